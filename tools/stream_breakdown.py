"""Per-kernel device time per batch of a skip stream (ht_rise_update_many on
device-resident batches), CUPTI through torch.profiler, no replay.

  python tools/stream_breakdown.py c2 [c3 ...]        # name+N: N updates first
                                                      # (c3+30: after its rank growth)
"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2412_16544_b200 import htrise as ht  # noqa: E402
from paper_2412_16544_b200.workloads import CONFIGS  # noqa: E402

K = 12
for arg in sys.argv[1:] or ["c2"]:
    name, _, adv = arg.partition("+")
    w = CONFIGS[name]
    ctx = ht.Context(0)
    ht.set_default_context(ctx)
    rep, _ = ht.bht_l2r(ht.DeviceTensor(w.make_batch(0, "cuda"), w.shape), w.tree(), w.eps)
    first = 1
    for b in range(1, 1 + int(adv or 0)):
        rep, _ = ht.ht_rise_update(rep, ht.DeviceTensor(w.make_batch(b, "cuda"), w.shape))
        first = b + 1
    P = 3
    pool = [ht.DeviceTensor(w.make_batch(b, "cuda"), w.shape) for b in range(first, first + P)]
    rep.reserve(rep.accumulated + 4 * K * w.batch)
    vals, _ = ht.ht_rise_update_many(rep, [pool[i % P] for i in range(4)])
    rep = vals[-1]
    ctx.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        vals, reps = ht.ht_rise_update_many(rep, [pool[i % P] for i in range(K)])
        ctx.synchronize()
    tot, cnt = defaultdict(float), defaultdict(int)
    first, last = None, None
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            if "htr::" in e.name or "Memcpy" in e.name or "Memset" in e.name:
                k = e.name.replace("htr::(anonymous namespace)::", "").replace("void ", "").split("(")[0]
                tot[k] += e.device_time_total
                cnt[k] += 1
    s = sum(tot.values()) / K
    print(f"{arg}: {s:.1f} us of kernels per batch; skips {sum(int(r.skipped) for r in reps)}/{K}; "
          f"exact {sum(int(r.used_exact_loss) for r in reps)}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:12]:
        print(f"   {v / K:8.1f} us  x{cnt[k] / K:.1f}  {k[:70]}")
    del pool, vals, rep
    torch.cuda.empty_cache()
