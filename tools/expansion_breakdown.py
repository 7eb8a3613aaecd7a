"""Per-kernel device time of the non-skip (expansion) update of config 3
(batch 25, where six new components switch on), measured with CUPTI."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2412_16544_b200 import htrise as ht
from paper_2412_16544_b200.workloads import CONFIGS

w = CONFIGS["c3"]
ctx = ht.Context(0)
ht.set_default_context(ctx)
rep, _ = ht.bht_l2r(ht.DeviceTensor(w.make_batch(0, "cuda"), w.shape), w.tree(), w.eps)
for b in range(1, 24):
    rep, u = ht.ht_rise_update(rep, ht.DeviceTensor(w.make_batch(b, "cuda"), w.shape))
y = w.make_batch(24, "cuda")
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rep2, u = ht.ht_rise_update(rep, ht.DeviceTensor(y, w.shape))
    torch.cuda.synchronize()
print("skipped", u.skipped, "seconds", u.seconds, "added", u.added_ranks)
agg = defaultdict(lambda: [0.0, 0])
for e in prof.events():
    if e.device_type.name == "CUDA":
        a = agg[e.name[:90]]
        a[0] += e.time_range.end - e.time_range.start
        a[1] += 1
tot = sum(v[0] for v in agg.values())
print(f"kernel busy {tot:.1f} us")
for k, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:15]:
    print(f"{t:10.1f} us  x{n:<4d} {k}")
