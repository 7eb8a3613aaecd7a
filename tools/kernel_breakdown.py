"""Per-kernel device time of one HT-RISE skip update on config 5, measured
with CUPTI (torch.profiler) in a normal run: no replay, no serialisation.
Prints each kernel's mean duration per update and the update's span."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2412_16544_b200 import htrise as ht
from paper_2412_16544_b200.workloads import CONFIGS

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
iters = 10
w = CONFIGS[name]
ctx = ht.Context(0)
ht.set_default_context(ctx)
y0 = w.make_batch(0, "cuda")
rep, _ = ht.bht_l2r(ht.DeviceTensor(y0, w.shape), w.tree(), w.eps)
y1 = w.make_batch(1, "cuda")
torch.cuda.synchronize()
rep.reserve(64 * w.batch)
dt = ht.DeviceTensor(y1, w.shape)
for _ in range(3):
    rep, upd = ht.ht_rise_update(rep, dt)
ctx.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(iters):
        rep, upd = ht.ht_rise_update(rep, dt)
    ctx.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
tot = defaultdict(float)
cnt = defaultdict(int)
t0, t1 = float("inf"), 0.0
for e in evs:
    tot[e.name] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    cnt[e.name] += 1
    t0 = min(t0, e.time_range.start)
    t1 = max(t1, e.time_range.end)
busy = sum(tot.values())
print(f"{name}: skipped={upd.skipped} fused={upd.used_fused_path} span/update {(t1 - t0) / iters:.1f} us, "
      f"kernel busy/update {busy / iters:.1f} us")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"  {v / iters:9.1f} us/update  {cnt[k] / iters:5.1f} launches/update  {k[:90]}")
