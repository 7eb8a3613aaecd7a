"""Config-5 skip stream with a chosen tail kernel (HTR_OPT_TAIL_KERNEL: 0 the
default -- the unit-dealt TMA kernel when the transfer basis is the
identity --, 1 one CTA per sample): ms per batch by CUDA events.
  python tools/tail_probe.py <variant> [K]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_16544_b200 import htrise as ht  # noqa: E402
from paper_2412_16544_b200.workloads import CONFIGS  # noqa: E402

variant = int(sys.argv[1]) if len(sys.argv) > 1 else 0
K = int(sys.argv[2]) if len(sys.argv) > 2 else 12
w = CONFIGS["c5"]
ctx = ht.Context(0)
ht.set_default_context(ctx)
rep, _ = ht.bht_l2r(ht.DeviceTensor(w.make_batch(0, "cuda"), w.shape), w.tree(), w.eps)
ctx.set_option(ht.OPT_TAIL_KERNEL, variant)
pool = [ht.DeviceTensor(w.make_batch(b, "cuda"), w.shape) for b in range(1, 4)]
rep.reserve(rep.accumulated + (2 * K + 4) * w.batch)
vals, _ = ht.ht_rise_update_many(rep, [pool[i % 3] for i in range(3)])
rep = vals[-1]
ctx.synchronize()
st = torch.cuda.ExternalStream(ctx.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
vals, reps = ht.ht_rise_update_many(rep, [pool[i % 3] for i in range(K)])
e1.record(st)
e1.synchronize()
print(f"variant {variant}: {e0.elapsed_time(e1) / K:.4f} ms per batch, skips {sum(int(r.skipped) for r in reps)}/{K}")
