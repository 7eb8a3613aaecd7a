"""Skip-update throughput across sample shapes other than the five configs
(what a user of the reference with PDE / image / video tensors would meet):
which shapes take the fused kernels, which fall back to the generic engine,
and what each sustains. Tucker-family batches (fixed orthonormal bases,
random cores) + 1e-4 relative noise, eps 1e-3; BHT-l2r on batch 0, then a
stream of K skip updates over device-resident batches (CUDA events).

  python tools/shape_sweep.py > gpurun_out/shape_sweep.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_16544_b200 import htrise as ht  # noqa: E402

CASES = [
    # (name, dims, ranks, tree, samples per batch)
    ("128^3 r20 (c5 shape, reference point)", (128, 128, 128), 20, "1_23", 64),
    ("120x120x12 r8 (multispectral image patches)", (120, 120, 12), 8, "1_23", 1024),
    ("96^3 r12", (96, 96, 96), 12, "1_23", 128),
    ("100^3 r10", (100, 100, 100), 10, "1_23", 128),
    ("50^3 r8", (50, 50, 50), 8, "1_23", 512),
    ("128x64x32 r10", (128, 64, 32), 10, "1_23", 512),
    ("63^3 r8 (odd leading extent: generic engine)", (63, 63, 63), 8, "1_23", 256),
    ("256x256x16 r12 (2-D grids x channels; the 256 x 256 kernel)", (256, 256, 16), 12, "1_23", 128),
    ("512x512x4 r12 (extent > 256: generic engine)", (512, 512, 4), 12, "1_23", 128),
    ("64x64x64x5 r6 balanced (3-D fields x variables)", (64, 64, 64, 5), 6, "balanced", 64),
    ("120x120x12x4 r6 balanced", (120, 120, 12, 4), 4, "balanced", 128),
    ("64x64x3x16 r6 balanced (video clips)", (64, 64, 3, 16), 3, "balanced", 512),
    ("24^4 r5 balanced (padded 32 x 32 kernel)", (24, 24, 24, 24), 5, "balanced", 256),
]
K = 12


def family(dims, r, n, gen, bases):
    ranks = [min(r, d) for d in dims]
    core = torch.randn(*ranks, n, device="cuda", dtype=torch.float64, generator=gen)
    y = core
    for k, b in enumerate(bases):
        y = torch.tensordot(b, y, dims=([1], [k])).movedim(0, k)
    y = y + 1e-4 * y.norm() / y.numel() ** 0.5 * torch.randn(y.shape, device="cuda", dtype=torch.float64, generator=gen)
    # canonical layout: first index fastest
    return y.permute(*reversed(range(y.dim()))).contiguous()


ctx = ht.Context(0)
ht.set_default_context(ctx)
for name, dims, r, tree_kind, n in CASES:
    gen = torch.Generator(device="cuda").manual_seed(1234)
    bases = [torch.linalg.qr(torch.randn(d, min(r, d), device="cuda", dtype=torch.float64, generator=gen))[0] for d in dims]
    shape = tuple(dims) + (n,)
    tree = ht.tree_1_23() if tree_kind == "1_23" else ht.DimensionTree.balanced(len(dims))
    y0 = family(dims, r, n, gen, bases)
    rep, _ = ht.bht_l2r(ht.DeviceTensor(y0, shape), tree, 1e-3)
    pool = [ht.DeviceTensor(family(dims, r, n, gen, bases), shape) for _ in range(3)]
    rep.reserve(rep.accumulated + (2 * K + 4) * n)
    vals, reps = ht.ht_rise_update_many(rep, [pool[i % 3] for i in range(4)])
    rep = vals[-1]
    ctx.synchronize()
    st = torch.cuda.ExternalStream(ctx.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    vals, reps = ht.ht_rise_update_many(rep, [pool[i % 3] for i in range(K)])
    e1.record(st)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / K
    nbytes = 8 * n
    for d in dims:
        nbytes *= d
    print(json.dumps({"case": name, "dims": dims, "samples": n, "batch_MB": round(nbytes / 1e6, 1),
                      "skips": sum(int(u.skipped) for u in reps), "fused": sum(int(u.used_fused_path) for u in reps),
                      "exact_loss": sum(int(u.used_exact_loss) for u in reps),
                      "launches_per_batch": reps[-1].kernel_launches, "ms_per_batch": round(ms, 4),
                      "GBps": round(nbytes / ms / 1e6, 1), "ranks": {str(k): v for k, v in rep.ranks().items()}}),
          flush=True)
    del pool, vals, rep, y0
    torch.cuda.empty_cache()
