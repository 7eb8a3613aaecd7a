"""Debug: truncations of residual-like matrices (exact null space) at a
machine-floor tolerance (the refine path with the full eigenvector set)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2412_16544_b200 import htrise as ht
from oracle import htrise_oracle as ho
rng = np.random.default_rng(3)
ctx = ht.Context(0); ht.set_default_context(ctx)
for n, r_old, cols in ((55, 35, 35), (55, 35, 300), (40, 20, 100), (64, 44, 200), (30, 10, 25)):
    U = np.linalg.qr(rng.standard_normal((n, r_old)))[0]
    C = rng.standard_normal((n, cols))
    R = C - U @ (U.T @ C)
    for eps_rel in (1e-12, 1e-9):
        eps = eps_rel * np.linalg.norm(C)
        b = ho.truncated_svd(R, eps, 0)
        for solver in (1, 0):
            ctx.set_option(ht.OPT_EIG_SOLVER, solver)
            a = ht.truncated_svd(R, eps, 0)
            leak = np.linalg.norm(U.T @ a.u) if a.rank else 0
            ang = np.linalg.norm(a.u - b.u @ (b.u.T @ a.u), 2) if a.rank == b.rank and a.rank else -1
            print(n, r_old, cols, eps_rel, "solver", solver, "rank", a.rank, b.rank, "leak %.2e angle %.2e" % (leak, ang), flush=True)
ctx.set_option(ht.OPT_EIG_SOLVER, 1)
