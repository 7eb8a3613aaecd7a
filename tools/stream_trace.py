"""Device timeline of a config-5 stream of skip updates (ht_rise_update_many):
kernels and copies with their start offsets and the idle gaps between them."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2412_16544_b200 import htrise as ht
from paper_2412_16544_b200.workloads import CONFIGS

w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
per_call = len(sys.argv) > 2 and sys.argv[2] == "call"
nb = int(sys.argv[3]) if len(sys.argv) > 3 else w.batch  # samples per batch (a rank's shard)
ctx = ht.Context(0)
ht.set_default_context(ctx)
shape = tuple(w.dims) + (nb,)
y0 = w.make_batch(0, "cuda", batch=nb)
rep, _ = ht.bht_l2r(ht.DeviceTensor(y0, shape), w.tree(), w.eps)
del y0
pool = [w.make_batch(1 + i, "cuda", batch=nb) for i in range(2)]
torch.cuda.synchronize()
rep.reserve(64 * nb)
bs = [ht.DeviceTensor(pool[i % 2], shape) for i in range(8)]
vals, _ = ht.ht_rise_update_many(rep, bs[:3])
rep = vals[-1]
ctx.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    if per_call:
        for b in bs:
            rep, _ = ht.ht_rise_update(rep, b)
    else:
        vals, _ = ht.ht_rise_update_many(rep, bs)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = None
for e in ev:
    s, d = e.time_range.start - t0, e.time_range.end - e.time_range.start
    gap = "" if prev_end is None else f"gap {s - prev_end:7.1f}"
    print(f"{s:10.1f} + {d:8.1f}  {gap:12s} {e.name[:70]}")
    prev_end = s + d
