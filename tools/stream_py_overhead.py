"""Python-side cost of ht_rise_update_many on config 5 (K batches): time
before the C call, inside it, and after it (result construction)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2412_16544_b200 import htrise as ht
from paper_2412_16544_b200.workloads import CONFIGS

K = 10
w = CONFIGS["c5"]
ctx = ht.Context(0)
ht.set_default_context(ctx)
rep, _ = ht.bht_l2r(ht.DeviceTensor(w.make_batch(0, "cuda"), w.shape), w.tree(), w.eps)
pool = [w.make_batch(1 + i, "cuda") for i in range(2)]
rep.reserve(10 * K * w.batch)
torch.cuda.synchronize()
real = ht._fn.ht_rise_update_many
marks = {}


def timed(*args):
    marks["c_in"] = time.perf_counter()
    r = real(*args)
    marks["c_out"] = time.perf_counter()
    return r


ht._fn.ht_rise_update_many = timed
for trial in range(4):
    bs = [ht.DeviceTensor(pool[i % 2], w.shape) for i in range(K)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    vals, reps = ht.ht_rise_update_many(rep, bs)
    t1 = time.perf_counter()
    rep = vals[-1]
    print(f"pre {1e6 * (marks['c_in'] - t0):.1f} us, C call {1e3 * (marks['c_out'] - marks['c_in']):.3f} ms, "
          f"post {1e6 * (t1 - marks['c_out']):.1f} us")
