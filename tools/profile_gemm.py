"""The skip tail's transfer projection shape through the public
mode_multiply API: [20, 400, 256] x_1 (400 x 400)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2412_16544_b200 import htrise as ht
ht.set_default_context(ht.Context(0))
rng = np.random.default_rng(0)
t = np.asfortranarray(rng.standard_normal((20, 400, 256)))
m = rng.standard_normal((400, 400))
for _ in range(3):
    out = ht.mode_multiply(t, 1, m)
ref = np.einsum("qj,ajs->aqs", m, t)
print("max err", np.max(np.abs(out - ref)) / np.max(np.abs(ref)))
