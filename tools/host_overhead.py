"""Per-update host overhead on config 5: Python wall time per call vs the
library's own wall time (report.seconds, includes its syncs) vs device time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_16544_b200 import htrise as ht
from paper_2412_16544_b200.workloads import CONFIGS
w = CONFIGS["c5"]
ctx = ht.Context(0); ht.set_default_context(ctx)
y0 = w.make_batch(0, "cuda")
rep, _ = ht.bht_l2r(ht.DeviceTensor(y0, w.shape), w.tree(), w.eps)
y1 = w.make_batch(1, "cuda"); torch.cuda.synchronize()
rep.reserve(64 * 256)
dt = ht.DeviceTensor(y1, w.shape)
for i in range(3):
    rep, upd = ht.ht_rise_update(rep, dt)
stream = torch.cuda.ExternalStream(ctx.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ctx.set_option(ht.OPT_PROFILE_EVENTS, 1); ctx.reset_timing()
py, lib_s = [], []
e0.record(stream)
for i in range(20):
    t0 = time.perf_counter()
    rep, upd = ht.ht_rise_update(rep, dt)
    py.append(time.perf_counter() - t0); lib_s.append(upd.seconds)
e1.record(stream); e1.synchronize()
fm, fc, _, _ = ctx.kernel_timing()
print(f"python per call {1e3*sum(py)/20:.3f} ms, library wall {1e3*sum(lib_s)/20:.3f} ms, "
      f"event span per call {e0.elapsed_time(e1)/20:.3f} ms, fused kernel {fm/fc:.3f} ms")
