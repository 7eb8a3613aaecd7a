"""Per-kernel device time of BHT-l2r (Alg. 1) on one config's first batch
(CUPTI through torch.profiler; kernels of this library only)."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2412_16544_b200 import htrise as ht
from paper_2412_16544_b200.workloads import CONFIGS

w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
ctx = ht.Context(0)
ht.set_default_context(ctx)
y0 = w.make_batch(0, "cuda")
ht.bht_l2r(ht.DeviceTensor(y0, w.shape), w.tree(), w.eps)  # warm (module loading)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rep, _ = ht.bht_l2r(ht.DeviceTensor(y0, w.shape), w.tree(), w.eps)
    ctx.synchronize()
tot, cnt = defaultdict(float), defaultdict(int)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and "htr::" in e.name:
        tot[e.name] += e.device_time_total
        cnt[e.name] += 1
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'c5'} bht_l2r: {sum(tot.values()) / 1e3:.1f} ms of kernels; ranks {rep.ranks()}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {v / 1e3:9.2f} ms  x{cnt[k]}  {k.replace('htr::(anonymous namespace)::', '')[:80]}")
