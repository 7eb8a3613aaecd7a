"""Per-rank step time of the config-5 skip update at the shard sizes of a
G-GPU run (256/G samples per rank) on one GPU: what each rank of
bench.py --gpus G computes, without the all-reduce. Stream API, K steps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2412_16544_b200 import htrise as ht
from paper_2412_16544_b200.workloads import CONFIGS

K = 10
w = CONFIGS["c5"]
ctx = ht.Context(0)
ht.set_default_context(ctx)
stream = torch.cuda.ExternalStream(ctx.stream())
for g in (1, 2, 4, 8):
    n = w.batch // g
    shape = tuple(w.dims) + (n,)
    y0 = w.make_batch(0, "cuda", batch=n)
    rep, _ = ht.bht_l2r(ht.DeviceTensor(y0, shape), w.tree(), w.eps)
    del y0
    pool = [w.make_batch(1 + i, "cuda", batch=n) for i in range(2)]
    rep.reserve((3 * K + 8) * n)
    bs = lambda k: [ht.DeviceTensor(pool[i % 2], shape) for i in range(k)]  # noqa: E731
    vals, _ = ht.ht_rise_update_many(rep, bs(3))
    rep = vals[-1]
    ctx.set_option(ht.OPT_PROFILE_EVENTS, 1)
    ctx.reset_timing()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    vals, reps = ht.ht_rise_update_many(rep, bs(K))
    e1.record(stream)
    e1.synchronize()
    fms, fcalls, _, _ = ctx.kernel_timing()
    ctx.set_option(ht.OPT_PROFILE_EVENTS, 0)
    ms = e0.elapsed_time(e1) / K
    print(f"G={g} samples/rank={n}: {ms:.4f} ms/step, fused3 {fms / max(fcalls, 1):.4f} ms, "
          f"per-rank {8 * n * 128**3 / ms / 1e6:.0f} GB/s, skipped {sum(u.skipped for u in reps)}/{K}", flush=True)
    del pool, vals, rep
    torch.cuda.empty_cache()
