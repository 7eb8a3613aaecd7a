"""GPU: the pipelined stream of updates (ht_rise_update_many, an extension
over the reference's per-batch ht_rise_update, ht_rise.hpp:99-186) must be
indistinguishable from calling ht_rise_update batch after batch: the same
skip decisions, reports, ranks and root slices bit for bit, through skips,
expansions (where the speculative encode of the next batch is discarded),
root-store growth, host inputs and trees outside the fused kernels."""
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


def _dev(ht, y):
    import torch

    t = torch.tensor(np.asarray(y).ravel(order="F"), dtype=torch.float64, device="cuda")
    return ht.DeviceTensor(t, tuple(y.shape))


def _family_stream(n, rng, grow_at=(), n_each=4, dims=(64, 64, 64), r=6, noise=1e-7):
    """Tucker-family batches; from each index in grow_at on, more
    components switch on (forcing an expansion at that batch)."""
    bases = [ro.random_orthonormal(d, 2 * r, rng) for d in dims]
    out = []
    k = r
    for i in range(n):
        if i in grow_at:
            k += 2
        b = [u[:, :k] for u in bases]
        y = ro.tucker_family_batch(b, n_each, rng)
        out.append(np.asfortranarray(y + noise * rng.standard_normal(y.shape)))
    return out


def _same_report(a, b):
    assert a.skipped == b.skipped
    assert a.proj_error == b.proj_error
    assert a.eps_des == b.eps_des
    assert a.new_ranks == b.new_ranks
    assert a.added_ranks == b.added_ranks
    assert a.used_fused_path == b.used_fused_path


def _check_stream(ht, rep0, batches, device, reserve=True):
    if reserve:
        rep0.reserve(sum(b.shape[-1] for b in batches) + rep0.accumulated + 8)
    args = [_dev(ht, b) if device else b for b in batches]
    seq, seq_reports = [], []
    r = rep0
    for a in args:
        r, u = ht.ht_rise_update(r, a)
        seq.append(r)
        seq_reports.append(u)
    many, reports = ht.ht_rise_update_many(rep0, args)
    assert len(many) == len(batches) == len(reports)
    for a, b in zip(reports, seq_reports):
        _same_report(a, b)
    for a, b in zip(many, seq):
        assert a.accumulated == b.accumulated
        assert a.ranks() == b.ranks()
    # the final value: identical bases and root slices
    fa, fb = many[-1], seq[-1]
    for l in range(1, fa.tree.depth + 1):
        for n in fa.tree.layer(l):
            assert np.array_equal(fa.basis_matrix(n.id), fb.basis_matrix(n.id)), n.id
    assert np.array_equal(fa.root(), fb.root())
    # every intermediate value still sees its own slices (value semantics)
    for a, b in zip(many, seq):
        m = a.accumulated
        assert np.array_equal(ht.reconstruct_slice(a, m), ht.reconstruct_slice(b, m))
    return many, reports


@pytest.mark.parametrize("device", [True, False])
def test_stream_matches_sequential_with_expansion(ht, device):
    rng = np.random.default_rng(2024)
    batches = _family_stream(9, rng, grow_at=(4,))
    rep0, _ = ht.bht_l2r(batches[0], ht.tree_1_23(), 1e-3)
    many, reports = _check_stream(ht, rep0, batches[1:], device)
    skipped = [u.skipped for u in reports]
    assert not skipped[3] and sum(skipped) >= 6, skipped  # batch 4 expands, the rest skip
    assert all(u.used_fused_path for u, s in zip(reports, skipped) if s)
    # against the oracle: the same decisions and ranks after every batch
    ref, _ = ho.bht_l2r(batches[0], ho.custom_tree_1_23(), 1e-3)
    for b, u, g in zip(batches[1:], reports, many):
        ref, ur = ho.ht_rise_update(ref, b)
        assert u.skipped == ur.skipped
        assert g.ranks() == ref.ranks()
    for m in range(1, ref.accumulated + 1):
        a, b = ht.reconstruct_slice(many[-1], m), ho.reconstruct_slice(ref, m)
        assert np.linalg.norm(a - b) <= 1e-9 * np.linalg.norm(b), m


def test_stream_root_store_growth(ht):
    # no reserve: the root store reallocates while speculative latents are in
    # flight (they land in a temporary and are appended on commit)
    rng = np.random.default_rng(77)
    batches = _family_stream(12, rng, n_each=3)
    rep0, _ = ht.bht_l2r(batches[0], ht.tree_1_23(), 1e-3)
    _, reports = _check_stream(ht, rep0, batches[1:], True, reserve=False)
    # (3 samples seed a transfer rank below the family's: the first updates expand)
    assert sum(u.skipped for u in reports) >= 6, [u.skipped for u in reports]


def test_stream_consecutive_expansions(ht):
    rng = np.random.default_rng(5)
    batches = _family_stream(7, rng, grow_at=(2, 3, 5), r=4)
    rep0, _ = ht.bht_l2r(batches[0], ht.tree_1_23(), 1e-3)
    _, reports = _check_stream(ht, rep0, batches[1:], True)
    assert sum(not u.skipped for u in reports) >= 2


def test_stream_generic_tree(ht):
    # a 4-way balanced tree of extent 10 is outside the fused kernels: the
    # stream enqueues the generic encode (deferred scalars) one batch ahead;
    # the results are still identical to the per-call loop
    rng = np.random.default_rng(31)
    bases = [ro.random_orthonormal(10, 3, rng) for _ in range(4)]
    batches = [np.asfortranarray(ro.tucker_family_batch(bases, 3, rng)) for _ in range(5)]
    rep0, _ = ht.bht_l2r(batches[0], ht.DimensionTree.balanced(4), 1e-6)
    _, reports = _check_stream(ht, rep0, batches[1:], True)
    assert all(u.skipped for u in reports)
    # a non-finite entry: the deferred encode's scan flags it, the per-call
    # path raises
    bad = batches[2].copy()
    bad[1, 2, 3, 1] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        ht.ht_rise_update_many(rep0, [_dev(ht, batches[1]), _dev(ht, bad)])


def test_stream_empty_and_errors(ht):
    rng = np.random.default_rng(3)
    batches = _family_stream(2, rng, n_each=2, dims=(64, 64, 8), r=2)
    rep0, _ = ht.bht_l2r(batches[0], ht.tree_1_23(), 1e-3)
    assert ht.ht_rise_update_many(rep0, []) == ([], [])
    bad = np.asfortranarray(np.ones((64, 64, 9, 2)))
    with pytest.raises(ValueError):
        ht.ht_rise_update_many(rep0, [batches[1], bad])
    nan = batches[1].copy()
    nan[3, 4, 5, 1] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        ht.ht_rise_update_many(rep0, [_dev(ht, batches[1]), _dev(ht, nan)])
    # the input value is untouched by the failed stream
    r, _ = ht.ht_rise_update(rep0, batches[1])
    assert r.accumulated == rep0.accumulated + 2


def test_stream_single_rank_nccl_matches_local(ht):
    """The stream API on the sharded runtime path: with a 1-rank NCCL
    communicator the skip norms and batch count go through ncclAllReduce and
    a D2H copy instead of the tail's mapped-memory write; results must equal
    the plain context's bit for bit (skips, an expansion, root slices)."""
    rng = np.random.default_rng(1212)
    plain = ht.Context(0)
    comm = ht.Context(0)
    comm.init_comm(ht.comm_unique_id(), 1, 0)
    batches = _family_stream(7, rng, grow_at=(3,))
    tree = ht.tree_1_23()
    outs = []
    for c in (plain, comm):
        r0, _ = ht.bht_l2r(batches[0], tree, 1e-3, ctx=c)
        r0.reserve(64)
        outs.append(ht.ht_rise_update_many(r0, [_dev(ht, b) for b in batches[1:]]))
    (va, ua), (vb, ub) = outs
    for a, b in zip(ua, ub):
        _same_report(a, b)
    assert any(not u.skipped for u in ua) and any(u.skipped for u in ua)
    assert np.array_equal(va[-1].root(), vb[-1].root())
    plain.close()
    comm.close()


def test_stream_ragged_batches_and_options(ht):
    """Batches of different sizes (the root slot of a speculative batch moves
    with the previous batch's size), an explicit epsilon and the adaptive
    budget: still identical to the per-call loop."""
    rng = np.random.default_rng(4242)
    bases = [ro.random_orthonormal(64, 8, rng) for _ in range(3)]
    sizes = [4, 1, 3, 6, 2, 5, 1]
    batches = []
    for k, n in enumerate(sizes):
        b = [u[:, : (4 if k < 4 else 6)] for u in bases]  # growth at batch 4
        y = ro.tucker_family_batch(b, n, rng)
        batches.append(np.asfortranarray(y + 1e-7 * rng.standard_normal(y.shape)))
    for eps, adaptive in ((None, False), (2e-3, False), (None, True)):
        rep0, _ = ht.bht_l2r(batches[0], ht.tree_1_23(), 1e-3)
        rep0.reserve(64)
        args = [_dev(ht, b) for b in batches[1:]]
        r, seq = rep0, []
        for a in args:
            r, u = ht.ht_rise_update(r, a, epsilon_rel=eps, adaptive_budget=adaptive)
            seq.append((r, u))
        many, reports = ht.ht_rise_update_many(rep0, args, epsilon_rel=eps, adaptive_budget=adaptive)
        for (rs, us), rm, um in zip(seq, many, reports):
            _same_report(us, um)
            assert rs.accumulated == rm.accumulated
        assert np.array_equal(many[-1].root(), seq[-1][0].root())
        assert any(u.skipped for u in reports) and not all(u.skipped for u in reports)


def test_stream_single_rank_nccl_generic_tree(ht):
    """The deferred generic encode on the sharded path: a 4-way tree outside
    the fused kernels, a 1-rank NCCL communicator (all-reduced scalars and
    batch count read back by copy): identical to the plain context."""
    rng = np.random.default_rng(4321)
    bases = [ro.random_orthonormal(10, 3, rng) for _ in range(4)]
    wide = [ro.random_orthonormal(10, 4, rng) for _ in range(4)]
    batches = [np.asfortranarray(ro.tucker_family_batch(bases, 3, rng)) for _ in range(4)]
    batches.append(np.asfortranarray(ro.tucker_family_batch(wide, 3, rng)))  # expands
    batches.append(np.asfortranarray(ro.tucker_family_batch(wide, 2, rng)))
    plain, comm = ht.Context(0), ht.Context(0)
    comm.init_comm(ht.comm_unique_id(), 1, 0)
    outs = []
    for c in (plain, comm):
        r0, _ = ht.bht_l2r(batches[0], ht.DimensionTree.balanced(4), 1e-6, ctx=c)
        outs.append(ht.ht_rise_update_many(r0, [_dev(ht, b) for b in batches[1:]]))
    (va, ua), (vb, ub) = outs
    for a, b in zip(ua, ub):
        _same_report(a, b)
    assert any(not u.skipped for u in ua) and any(u.skipped for u in ua)
    for m in range(1, va[-1].accumulated + 1):
        assert np.array_equal(ht.reconstruct_slice(va[-1], m), ht.reconstruct_slice(vb[-1], m))
    plain.close()
    comm.close()
