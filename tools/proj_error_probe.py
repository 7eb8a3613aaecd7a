"""Per-batch projection error of the fused/telescoped path against the
explicit per-step loss (HTR_OPT_EXACT_LOSS) and the oracle, with the bases'
orthonormality defects: the accuracy floor of the telescoped skip test."""
import dataclasses
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import htrise_oracle as ho  # noqa: E402
from paper_2412_16544_b200 import htrise as ht  # noqa: E402
from paper_2412_16544_b200.workloads import CONFIGS  # noqa: E402


def host(t, shape):
    return np.asfortranarray(t.cpu().numpy().reshape(tuple(reversed(shape))).transpose())


def run(name, nb, batch=None):
    w = CONFIGS[name]
    if batch:
        w = dataclasses.replace(w, batch=batch)
    shape = tuple(w.dims) + (w.batch,)
    ctx = ht.Context(0)
    ex = ht.Context(0)
    ex.set_option(ht.OPT_EXACT_LOSS, 1)
    y0 = w.make_batch(0, "cuda")
    rep, _ = ht.bht_l2r(ht.DeviceTensor(y0, shape), w.tree(), w.eps, ctx=ctx)
    tree = ho.custom_tree_1_23() if w.tree_kind == "1_23" else ho.DimensionTree.balanced(len(w.dims))
    ref, _ = ho.bht_l2r(host(y0, shape), tree, w.eps)
    for b in range(1, nb):
        yb = w.make_batch(b, "cuda")
        ynorm = float(yb.norm())
        _, pe = ht.encode(rep, ht.DeviceTensor(yb, shape))
        # the same value's exact per-step loss on the exact context
        ctx.set_option(ht.OPT_EXACT_LOSS, 1)
        _, pe_x = ht.encode(rep, ht.DeviceTensor(yb, shape))
        ctx.set_option(ht.OPT_EXACT_LOSS, 0)
        _, pe_ref = ho.encode(ref, host(yb, shape))
        print(json.dumps({"config": name, "batch": b, "pe_over_y": pe / ynorm, "defect_max": rep.orthonormality_defect(),
                          "fast_minus_ref": (pe - pe_ref) / ynorm, "exact_minus_ref": (pe_x - pe_ref) / ynorm}),
              flush=True)
        rep, _ = ht.ht_rise_update(rep, ht.DeviceTensor(yb, shape))
        ref, _ = ho.ht_rise_update(ref, host(yb, shape))


if __name__ == "__main__":
    run("c2", 5)
    run("c3", 27)
    run("c5", 4, batch=6)
    run("c4", 3)
