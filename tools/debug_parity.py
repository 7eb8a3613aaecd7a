import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2412_16544_b200 import htrise as ht
from paper_2412_16544_b200.workloads import CONFIGS
from oracle import htrise_oracle as ho
ctx = ht.Context(0); ht.set_default_context(ctx)
def host(t, shape): return np.asfortranarray(t.cpu().numpy().reshape(tuple(reversed(shape))).transpose())

w = CONFIGS['c3']; shape = w.shape
y = host(w.make_batch(0, 'cuda'), shape)
M = ho.unfold(y, 0)
a = ht.truncated_svd(M, 1e-3*np.linalg.norm(y)/np.sqrt(6))
u, s, _ = np.linalg.svd(M, full_matrices=False)
R = u[:, :a.rank]
print("c3 mode0 rank", a.rank, "angle", np.linalg.norm(a.u - R @ (R.T @ a.u), 2), "sig", a.singular_values[:7], s[:7])
G = M @ M.T
lam, V = np.linalg.eigh(G); V = V[:, ::-1][:, :a.rank]
print("numpy eigh angle", np.linalg.norm(V - R @ (R.T @ V), 2))
# small matrix from the same data: first 5000 columns
M2 = np.ascontiguousarray(M[:, :5000])
a2 = ht.truncated_svd(M2, 0.0); u2, s2, _ = np.linalg.svd(M2, full_matrices=False)
R2 = u2[:, :6]
print("c3 first-5000 angle top6", np.linalg.norm(a2.u[:, :6] - R2 @ (R2.T @ a2.u[:, :6]), 2))

w = CONFIGS['c4']; shape = w.shape
yd = w.make_batch(0, 'cuda'); y0 = host(yd, shape)
rep, _ = ht.bht_l2r(ht.DeviceTensor(yd, shape), w.tree(), w.eps)
ref, _ = ho.bht_l2r(y0, ho.DimensionTree.balanced(8), w.eps)
y1d = w.make_batch(1, 'cuda'); y1 = host(y1d, shape)
print("c4 ranks", rep.ranks() == ref.ranks())
print("c4 |y|^2 gpu", ht.frobenius_norm(y1)**2, "np", np.sum(y1**2))
la, pa = ht.encode(rep, y1)
ctx.set_option(ht.OPT_EXACT_LOSS, 1); le, pe = ht.encode(rep, y1); ctx.set_option(ht.OPT_EXACT_LOSS, 0)
lb, pb = ho.encode(ref, y1)
print("c4 proj fast", pa, "exact", pe, "oracle", pb)
print("c4 |lat|^2 gpu", np.sum(la**2), "exact-path", np.sum(le**2), "oracle", np.sum(lb**2))
print("c4 decode diff", np.linalg.norm(ht.decode(rep, la) - ho.decode(ref, lb)) / np.linalg.norm(ho.decode(ref, lb)))
