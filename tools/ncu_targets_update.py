"""One pass over the skip-path update kernels of every config for an ncu
capture (tools/ncu_multi_summary.py reads the report): BHT-l2r on batch 0
(not captured: filter by kernel name), then two skip updates per config and
a device normalisation."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_16544_b200 import htrise as ht  # noqa: E402
from paper_2412_16544_b200.workloads import CONFIGS  # noqa: E402

ctx = ht.Context(0)
ht.set_default_context(ctx)
for name in (sys.argv[1:] or ["c2", "c3", "c4", "c5"]):
    w = CONFIGS[name]
    rep, _ = ht.bht_l2r(ht.DeviceTensor(w.make_batch(0, "cuda"), w.shape), w.tree(), w.eps)
    for b in (1, 2):
        rep, u = ht.ht_rise_update(rep, ht.DeviceTensor(w.make_batch(b, "cuda"), w.shape))
        assert u.skipped and u.used_fused_path, (name, b)
    torch.cuda.synchronize()
    del rep
    torch.cuda.empty_cache()
y = CONFIGS["c3"].make_batch(0, "cuda")
ht.normalize(ht.DeviceTensor(y, CONFIGS["c3"].shape), "zscore", 3)
torch.cuda.synchronize()
print("ok")
