import os, sys
sys.path.insert(0, "/root/repo" if os.path.exists("/root/repo/bench.py") else os.getcwd())
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2412_16544_b200 import htrise as ht
from paper_2412_16544_b200.workloads import CONFIGS
w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
ctx = ht.Context(0); ht.set_default_context(ctx)
y0 = w.make_batch(0, "cuda")
ht.bht_l2r(ht.DeviceTensor(y0, w.shape), w.tree(), w.eps)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rep, _ = ht.bht_l2r(ht.DeviceTensor(y0, w.shape), w.tree(), w.eps)
    ctx.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start; prev = None
for e in ev:
    s, d = e.time_range.start - t0, e.time_range.end - e.time_range.start
    gap = "" if prev is None else f"gap {s - prev:7.1f}"
    print(f"{s:10.1f} + {d:8.1f}  {gap:12s} {e.name.replace('htr::(anonymous namespace)::','')[:60]}")
    prev = max(prev or 0, s + d)
