"""Host-side cost of one ht_rise_update_many call on config 5: wall time of
the Python wrapper's argument preparation, the C call, and the result
construction, against the device time of the same K steps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2412_16544_b200 import htrise as ht
from paper_2412_16544_b200.workloads import CONFIGS

K = int(sys.argv[1]) if len(sys.argv) > 1 else 10
w = CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c5"]
ctx = ht.Context(0)
ht.set_default_context(ctx)
y0 = w.make_batch(0, "cuda")
rep, _ = ht.bht_l2r(ht.DeviceTensor(y0, w.shape), w.tree(), w.eps)
del y0
pool = [w.make_batch(1 + i, "cuda") for i in range(2)]
torch.cuda.synchronize()
rep.reserve(8 * K * w.batch)
stream = torch.cuda.ExternalStream(ctx.stream())
for trial in range(3):
    bs = [ht.DeviceTensor(pool[i % 2], w.shape) for i in range(K)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    vals, reps = ht.ht_rise_update_many(rep, bs)
    t1 = time.perf_counter()
    e1.record(stream)
    e1.synchronize()
    rep = vals[-1]
    print(f"K={K}: events {e0.elapsed_time(e1) / K:.4f} ms/step, wall {1e3 * (t1 - t0) / K:.4f} ms/step, "
          f"report seconds sum {sum(u.seconds for u in reps) * 1e3 / K:.4f}")
