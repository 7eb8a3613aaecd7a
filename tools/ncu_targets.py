"""One pass over the round-2 kernels for an ncu capture (tools/ncu_lines.py
and tools/ncu_summary.py read the report): config 5's BHT-l2r (the fused
pair projection, the streaming and mode-0 Grams, the tridiagonal solver,
the blocked Cholesky certificate), config 1's BHT-l2r (mid-size Grams),
config 4's skip update (the 12-warp subtree pass + its finishing launch)
and a device normalisation."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_16544_b200 import htrise as ht  # noqa: E402
from paper_2412_16544_b200.workloads import CONFIGS  # noqa: E402

ctx = ht.Context(0)
ht.set_default_context(ctx)
for name in ("c5", "c1", "c4"):
    w = CONFIGS[name]
    rep, _ = ht.bht_l2r(ht.DeviceTensor(w.make_batch(0, "cuda"), w.shape), w.tree(), w.eps)
    if name == "c4":
        rep, _ = ht.ht_rise_update(rep, ht.DeviceTensor(w.make_batch(1, "cuda"), w.shape))
    torch.cuda.synchronize()
y = CONFIGS["c3"].make_batch(0, "cuda")
ht.normalize(ht.DeviceTensor(y, CONFIGS["c3"].shape), "zscore", 3)
torch.cuda.synchronize()
print("ok")
