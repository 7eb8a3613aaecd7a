import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2412_16544_b200 import htrise as ht
rng = np.random.default_rng(1)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
m = np.linalg.qr(rng.standard_normal((n, 20)))[0] @ rng.standard_normal((20, 3 * n + 8))
m += 1e-6 * rng.standard_normal(m.shape)
for _ in range(2):
    ht.truncated_svd(m, 1e-3 * np.linalg.norm(m))
