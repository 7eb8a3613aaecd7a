"""Device time of the truncation eigensolvers per Gram size (CUPTI via
torch.profiler): the tridiagonal route's two kernels vs the Jacobi route.

  python tools/eig_probe.py [n ...]
"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2412_16544_b200 import htrise as ht  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [16, 32, 64, 128, 144, 160, 256, 400]
ctx = ht.Context(0)
ht.set_default_context(ctx)
rng = np.random.default_rng(1)
for n in sizes:
    r = min(20, n)
    m = np.linalg.qr(rng.standard_normal((n, r)))[0] @ rng.standard_normal((r, 3 * n + 8))
    m += 1e-6 * rng.standard_normal(m.shape)
    eps = 1e-3 * np.linalg.norm(m)
    for solver in (1, 0):
        ctx.set_option(ht.OPT_EIG_SOLVER, solver)
        ht.truncated_svd(m, eps)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(3):
                ht.truncated_svd(m, eps)
            ctx.synchronize()
        tot = defaultdict(float)
        for e in prof.events():
            if e.device_type == torch.autograd.DeviceType.CUDA and "htr::" in e.name:
                tot[e.name.replace("htr::(anonymous namespace)::", "").replace("void ", "").split("(")[0]] += e.device_time_total / 3
        top = sorted(tot.items(), key=lambda kv: -kv[1])[:4]
        print(f"n={n:4d} solver={'tridiag' if solver else 'jacobi '} total {sum(tot.values()):8.1f}us  "
              + "  ".join(f"{k[:28]} {v:8.1f}us" for k, v in top), flush=True)
ctx.set_option(ht.OPT_EIG_SOLVER, 1)
