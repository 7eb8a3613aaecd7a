"""Debug: the expansion of test_fused_tail_tile_cases[ranks5-24-5-n015]."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2412_16544_b200 import htrise as ht
from oracle import htrise_oracle as ho, ref_oracles as ro
ranks, n2, nsamp, n01 = (7, 11, 5), 24, 5, (128, 64)
for solver in (1, 0):
    rng = np.random.default_rng(sum(ranks) * 1000 + n2)
    bases = [ro.random_orthonormal(n, r, rng) for n, r in zip((n01[0], n01[1], n2), ranks)]
    y0 = ro.tucker_family_batch(bases, nsamp, rng)
    ctx = ht.Context(0); ctx.set_option(ht.OPT_EIG_SOLVER, solver)
    rep, _ = ht.bht_l2r(y0, ht.tree_1_23(), 1e-9, ctx=ctx)
    ref, _ = ho.bht_l2r(y0, ho.custom_tree_1_23(), 1e-9)
    y1 = ro.tucker_family_batch(bases, 7, rng)
    _, pe = ht.encode(rep, y1); _, pr = ho.encode(ref, y1)
    print("solver", solver, "ranks", rep.ranks(), "pe", pe, pr, "ynorm", np.linalg.norm(y1), flush=True)
    r2, ur = ho.ht_rise_update(ref, y1)
    print("  oracle: skipped", ur.skipped, "added", ur.added_ranks, flush=True)
    try:
        g2, u = ht.ht_rise_update(rep, y1)
        print("  gpu: skipped", u.skipped, "added", u.added_ranks, g2.ranks(), flush=True)
    except Exception as e:
        print("  gpu error:", e, flush=True)
    for eps_solver in (1,):
        pass
