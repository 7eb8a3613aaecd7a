"""One small truncation (ncu target): n x 3n matrix, rank 5 + noise."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2412_16544_b200 import htrise as ht
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
rng = np.random.default_rng(2)
m = np.linalg.qr(rng.standard_normal((n, 5)))[0] @ rng.standard_normal((5, 3 * n))
m += 1e-6 * rng.standard_normal(m.shape)
for _ in range(2):
    ht.truncated_svd(m, 1e-2 * np.linalg.norm(m))
