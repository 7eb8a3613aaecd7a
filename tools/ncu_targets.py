"""BHT-l2r of the named configs' first batch for an ncu capture
(tools/ncu_multi_summary.py and tools/ncu_lines.py read the report): config
5 (the fused pair projection, the streaming and mode-0 Grams, the two-level-K
transfer Gram, the tridiagonal solver, the blocked Cholesky certificate) and
config 1 (mid-size Grams, clustered eigenvectors). The skip-update kernels
are captured with tools/ncu_targets_update.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_16544_b200 import htrise as ht  # noqa: E402
from paper_2412_16544_b200.workloads import CONFIGS  # noqa: E402

ctx = ht.Context(0)
ht.set_default_context(ctx)
for name in (sys.argv[1:] or ["c5", "c1"]):
    w = CONFIGS[name]
    rep, _ = ht.bht_l2r(ht.DeviceTensor(w.make_batch(0, "cuda"), w.shape), w.tree(), w.eps)
    torch.cuda.synchronize()
    del rep
    torch.cuda.empty_cache()
print("ok")
