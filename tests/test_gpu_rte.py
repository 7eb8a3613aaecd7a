"""GPU relative_test_error (metrics.hpp:218-237) through the C-ABI
(htr_relative_error): against the oracle's restatement, against the generic
decode-then-compare chain, and on a full config-5 batch where the fused decode
kernel compares the reconstruction in HBM without writing it.

Bar: per-tensor relative errors within 1e-9 in
relative-error units of the oracle's.
"""
import numpy as np
import pytest

from oracle import htrise_oracle as ho
from oracle import ref_oracles as ro

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ht():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2412_16544_b200 import htrise

    htrise.set_default_context(htrise.Context(0))
    return htrise


@pytest.mark.parametrize("dims,ranks,tree", [
    ((64, 32, 6), (12, 5, 3), "1_23"),          # fused residual decode
    ((32, 32, 8, 4), (6, 4, 3, 2), "balanced"),  # fused, 4-way tree
    ((5, 6, 5, 4), (2, 3, 2, 2), "balanced"),     # extents outside the fused kernel
])
def test_rte_vs_oracle(ht, dims, ranks, tree):
    rng = np.random.default_rng(sum(dims) + 7 * sum(ranks))
    bases = [ro.random_orthonormal(n, r, rng) for n, r in zip(dims, ranks)]
    y0 = ro.tucker_family_batch(bases, 4, rng) + 1e-3 * rng.standard_normal(tuple(dims) + (4,))
    if tree == "1_23":
        gpu, _ = ht.bht_l2r(y0, ht.tree_1_23(), 1e-2)
        ref, _ = ho.bht_l2r(y0, ho.custom_tree_1_23(), 1e-2)
    else:
        gpu, _ = ht.bht_l2r(y0, ht.DimensionTree.balanced(len(dims)), 1e-2)
        ref, _ = ho.bht_l2r(y0, ho.DimensionTree.balanced(len(dims)), 1e-2)
    assert gpu.ranks() == ref.ranks()
    in_span = ro.tucker_family_batch(bases, 3, rng)
    tests = [
        in_span,                                   # order d + 1
        in_span[..., 0].copy(order="F"),           # order d: unit batch axis
        rng.standard_normal(tuple(dims) + (2,)),   # far from the span
        np.zeros(tuple(dims) + (2,)),              # adds 0, counts in the mean
    ]
    for t in tests:
        a, b = ht.relative_error(gpu, t), ho.relative_test_error(ref, [t])
        assert abs(a - b) <= 1e-9, (a, b)
    assert abs(ht.relative_test_error(gpu, tests) - ho.relative_test_error(ref, tests)) <= 1e-9
    # the same number as decode(encode(y)) compared on the host
    lat, _ = ht.encode(gpu, tests[2])
    back = ht.decode(gpu, lat)
    host = np.linalg.norm(tests[2] - back) / np.linalg.norm(tests[2])
    assert abs(ht.relative_error(gpu, tests[2]) - host) <= 1e-13
    assert ht.relative_error(gpu, tests[3]) == 0.0


def test_rte_errors(ht):
    rng = np.random.default_rng(3)
    y = rng.standard_normal((4, 5, 6, 2))
    gpu, _ = ht.bht_l2r(y, ht.DimensionTree.balanced(3), 0.3)
    with pytest.raises(ValueError):
        ht.relative_test_error(gpu, [])
    with pytest.raises(ValueError, match="encode"):
        ht.relative_error(gpu, rng.standard_normal((4, 5, 7, 2)))
    bad = y.copy()
    bad[1, 2, 3, 0] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        ht.relative_error(gpu, bad)


def test_rte_fused_matches_generic_and_runs(ht):
    """config 5's leaf shapes: the residual-mode fused kernel runs and equals
    the decode-to-scratch chain."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    rng = np.random.default_rng(237)
    bases = [ro.random_orthonormal(128, 20, rng) for _ in range(3)]
    # entries of the Tucker part are ~0.06: 1e-6 noise keeps the leaf ranks at 20
    y0 = ro.tucker_family_batch(bases, 3, rng) + 1e-6 * rng.standard_normal((128, 128, 128, 3))
    rep, _ = ht.bht_l2r(y0, ht.tree_1_23(), 1e-3)
    assert rep.ranks()[(1, 0)] == 20
    # samples the transfer node spans (its rank is set by 3 samples), plus noise
    t = y0[..., :2] + 1e-4 * rng.standard_normal((128, 128, 128, 2))
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        a = ht.relative_error(rep, t)
        rep.ctx.synchronize()
    names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    assert any("decode2_kernel" in n and "true" in n for n in names), names
    rep.ctx.set_option(ht.OPT_FUSED_ENCODE, 0)
    try:
        b = ht.relative_error(rep, t)
    finally:
        rep.ctx.set_option(ht.OPT_FUSED_ENCODE, 1)
    assert abs(a - b) <= 1e-12 * b
    assert 1e-4 < a < 1e-2


def test_rte_config5_full_batch(ht):
    """A full 4.3 GB config-5 batch: the in-HBM comparison equals
    decode-into-device-memory followed by a torch norm."""
    import torch
    from paper_2412_16544_b200.workloads import CONFIGS

    w = CONFIGS["c5"]
    shape = tuple(w.dims) + (w.batch,)
    rep, _ = ht.bht_l2r(ht.DeviceTensor(w.make_batch(0, "cuda"), shape), w.tree(), w.eps)
    y1 = w.make_batch(1, "cuda")
    a = ht.relative_error(rep, ht.DeviceTensor(y1, shape))
    lat, _ = ht.encode(rep, ht.DeviceTensor(y1, shape))
    import ctypes as C

    x = torch.empty_like(y1)
    dl = torch.from_numpy(np.ascontiguousarray(lat.transpose(2, 1, 0))).cuda()  # canonical r11 x r12 x N
    ls = (C.c_int64 * 3)(*lat.shape)
    dp = lambda u: C.cast(C.c_void_p(u.data_ptr()), C.POINTER(C.c_double))  # noqa: E731
    rep.ctx.check(ht.lib().htr_decode(rep.ctx.handle, rep._h, dp(dl), 1, ls, dp(x), 1))
    rep.ctx.synchronize()
    ref = (torch.linalg.norm(y1 - x) / torch.linalg.norm(y1)).item()
    del x
    assert abs(a - ref) <= 1e-12 * ref
    # config 5's relative noise is 1e-4 per sample, eps 1e-3: the error sits between
    assert 1e-5 < a < 1e-3
