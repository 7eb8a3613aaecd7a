"""One config-5 skip update for ncu: BHT-l2r on batch 0, then `--updates`
ht_rise_update calls on a resident batch (the fused kernel dominates)."""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_16544_b200 import htrise as ht
from paper_2412_16544_b200.workloads import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--updates", type=int, default=2)
ap.add_argument("--config", default="c5")
a = ap.parse_args()
w = CONFIGS[a.config]
ctx = ht.Context(0); ht.set_default_context(ctx)
y0 = w.make_batch(0, "cuda")
rep, _ = ht.bht_l2r(ht.DeviceTensor(y0, w.shape), w.tree(), w.eps)
y1 = w.make_batch(1, "cuda")
torch.cuda.synchronize()
for i in range(a.updates):
    rep, upd = ht.ht_rise_update(rep, ht.DeviceTensor(y1, w.shape))
    print("update", i, "skipped", upd.skipped, "fused", upd.used_fused_path, "seconds", upd.seconds)
