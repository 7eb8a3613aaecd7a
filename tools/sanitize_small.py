"""Small end-to-end runs of every fused path for compute-sanitizer
(memcheck / racecheck): 3-way fused3 + tail (per-sample, cluster-split and
sample-pair tails), the 8-way subtree kernels, the leading 32x32 slab pass,
the stream API, BHT-l2r with the packed and cluster Jacobi solvers and the
full-rank Cholesky test."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses

import numpy as np

from oracle import ref_oracles as ro
from paper_2412_16544_b200 import htrise as ht
from paper_2412_16544_b200.workloads import CONFIGS

ctx = ht.Context(0)
ht.set_default_context(ctx)
rng = np.random.default_rng(0)
# 3-way (1,(2,3)), 64^3: fused3 + tail (one sample per CTA / clusters / pairs)
bases = [ro.random_orthonormal(64, 5, rng) for _ in range(3)]
ys = [np.asfortranarray(ro.tucker_family_batch(bases, n, rng) + 1e-7 * rng.standard_normal((64, 64, 64, n)))
      for n in (4, 3, 2, 3)]
rep, _ = ht.bht_l2r(ys[0], ht.tree_1_23(), 1e-3)
for v in (0, 1, 2):
    ctx.set_option(ht.OPT_TAIL_KERNEL, v)
    r, u = ht.ht_rise_update(rep, ys[1])
    print("tail variant", v, "skipped", u.skipped, "fused", u.used_fused_path)
ctx.set_option(ht.OPT_TAIL_KERNEL, 0)
vals, reps = ht.ht_rise_update_many(rep, ys[1:])
print("stream", [x.skipped for x in reps])
# 8-way (config 4 shape, 1 sample)
w4 = dataclasses.replace(CONFIGS["c4"], batch=1)
shape4 = tuple(w4.dims) + (1,)
r4, _ = ht.bht_l2r(ht.DeviceTensor(w4.make_batch(0, "cuda"), shape4), w4.tree(), w4.eps)
r4b, u4 = ht.ht_rise_update(r4, ht.DeviceTensor(w4.make_batch(1, "cuda"), shape4))
print("8-way fused", u4.used_fused_path, u4.skipped)
# balanced(4) 32^3 x 8 (leading 32x32 slab pass), small batch
w3 = dataclasses.replace(CONFIGS["c3"], batch=2)
shape3 = tuple(w3.dims) + (2,)
r3, _ = ht.bht_l2r(ht.DeviceTensor(w3.make_batch(0, "cuda"), shape3), w3.tree(), w3.eps)
v3, rp3 = ht.ht_rise_update_many(r3, [ht.DeviceTensor(w3.make_batch(b, "cuda"), shape3) for b in (1, 2)])
print("4-way stream", [x.skipped for x in rp3])
# BHT-l2r on random full-rank data: a 200-row full-rank transfer (the
# Cholesky test replaces the cluster Jacobi), a 1600-row tall transfer
# (column-side Gram), leaves of 20/10/40 rows (packed Jacobi)
y = np.asfortranarray(rng.standard_normal((20, 10, 40, 40, 2)))
rb, rep_b = ht.bht_l2r(y, ht.DimensionTree.balanced(4), 1e-3)
print("bht ranks", rb.ranks())
# a 240-row transfer with fewer columns than rows (cluster Jacobi) and a
# 140-row leaf (A-in-smem Jacobi)
y2 = np.asfortranarray(rng.standard_normal((140, 4, 4, 8, 3)))
rc, _ = ht.bht_l2r(y2, ht.DimensionTree.balanced(4), 1e-3)
print("bht ranks", rc.ranks())
# round 2: the BASELINE configs c1-c3 at their stated sizes (c2/c3: first
# batches) -- tridiagonal eigensolver, DMMA mid-size Grams, the fused pair
# projection, the stream API with the explicit loss enqueued ahead -- and a
# machine-floor truncation (full eigenvector set, block inverse iteration)
for name, nb in (("c1", 1), ("c2", 4), ("c3", 3)):
    w = CONFIGS[name]
    r, _ = ht.bht_l2r(ht.DeviceTensor(w.make_batch(0, "cuda"), w.shape), w.tree(), w.eps)
    if nb > 1:
        vals, reps = ht.ht_rise_update_many(r, [ht.DeviceTensor(w.make_batch(b, "cuda"), w.shape) for b in range(1, nb)])
        print(name, "stream", [x.skipped for x in reps], vals[-1].ranks())
    else:
        print(name, "bht", r.ranks())
m = np.linalg.qr(rng.standard_normal((40, 10)))[0] @ rng.standard_normal((10, 90))
print("floor truncation rank", ht.truncated_svd(m, 1e-13 * np.linalg.norm(m), 0).rank)
