import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2412_16544_b200 import htrise as ht
from oracle import htrise_oracle as ho, ref_oracles as ro
ranks, n2, nsamp, n01 = (7, 11, 5), 24, 5, (128, 64)
rng = np.random.default_rng(sum(ranks) * 1000 + n2)
bases = [ro.random_orthonormal(n, r, rng) for n, r in zip((n01[0], n01[1], n2), ranks)]
y0 = ro.tucker_family_batch(bases, nsamp, rng)
for solver in (1, 0):
    for fused in (1, 0):
        ctx = ht.Context(0); ctx.set_option(ht.OPT_EIG_SOLVER, solver); ctx.set_option(ht.OPT_FUSED_ENCODE, fused)
        rep, _ = ht.bht_l2r(y0, ht.tree_1_23(), 1e-9, ctx=ctx)
        ref, _ = ho.bht_l2r(y0, ho.custom_tree_1_23(), 1e-9)
        print("solver", solver, "fused", fused, rep.ranks(), ref.ranks(), "defect", rep.orthonormality_defect())
        for l in (1, 2):
            for n in ref.tree.layer(l):
                a = rep.basis_matrix(n.id); b = ref.basis_matrix(n.id)
                if a.shape[1] == b.shape[1]:
                    print("  node", n.id, "angle", np.linalg.norm(a - b @ (b.T @ a), 2))
        rng2 = np.random.default_rng(5)
        y1 = ro.tucker_family_batch(bases, 7, rng2)
        la, pa = ht.encode(rep, y1); lb, pb = ho.encode(ref, y1)
        print("  encode pe", pa, pb, "ynorm", np.linalg.norm(y1))
        try:
            r2, u = ht.ht_rise_update(rep, y1); print("  update skipped", u.skipped, u.proj_error, u.eps_des)
        except Exception as e:
            print("  update error", e)
