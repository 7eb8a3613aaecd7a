"""Host cost of one ht_rise_update call on a tiny fused-path batch (64^3 x 1,
tree (1,(2,3))): Python wall time per call vs the library's own
UpdateReport.seconds (C++ entry to exit) vs the device time of its kernels."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import ref_oracles as ro
from paper_2412_16544_b200 import htrise as ht

ctx = ht.Context(0)
ht.set_default_context(ctx)
rng = np.random.default_rng(1)
bases = [ro.random_orthonormal(64, 6, rng) for _ in range(3)]
y0 = ro.tucker_family_batch(bases, 4, rng)
rep, _ = ht.bht_l2r(y0, ht.tree_1_23(), 1e-3)
rep.reserve(100000)
y = torch.tensor(np.asfortranarray(ro.tucker_family_batch(bases, 1, rng)).ravel(order="F"), device="cuda")
dt = ht.DeviceTensor(y, (64, 64, 64, 1))
for _ in range(50):
    rep, u = ht.ht_rise_update(rep, dt)
torch.cuda.synchronize()
n = 2000
t0 = time.perf_counter()
secs = 0.0
for _ in range(n):
    rep, u = ht.ht_rise_update(rep, dt)
    secs += u.seconds
t1 = time.perf_counter()
print(f"per call: python wall {1e6 * (t1 - t0) / n:.1f} us, library (UpdateReport.seconds) {1e6 * secs / n:.1f} us, "
      f"skipped={u.skipped} fused={u.used_fused_path}")
vals, reps = ht.ht_rise_update_many(rep, [dt] * 10)
t0 = time.perf_counter()
for _ in range(n // 10):
    vals, reps = ht.ht_rise_update_many(vals[-1], [dt] * 10)
t1 = time.perf_counter()
print(f"stream API: {1e6 * (t1 - t0) / n:.1f} us per batch")
