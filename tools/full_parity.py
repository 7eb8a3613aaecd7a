"""Config parity at the BASELINE sizes: the library (device batches through
the C-ABI) against the CPU oracle fed the exact device bytes, batch by batch.

  python tools/full_parity.py c5 [--batches 40] [--compare all|some]

Per batch it records: skip decisions (GPU vs oracle), ranks at every node,
|proj_error - oracle| / ||y|| (north star: 1e-9), eps_des agreement, leaf
principal angles (north star: 1e-8) and, for the compared batches, the
largest relative error over every slice of the batch between the GPU's
decode of its latents and the oracle's decode of its own (north star: 1e-9).
One JSON line per batch, then a summary line, to stdout. The oracle is the
checker only; nothing here is timed against anything.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import htrise_oracle as ho  # noqa: E402
from paper_2412_16544_b200 import htrise as ht  # noqa: E402
from paper_2412_16544_b200.workloads import CONFIGS  # noqa: E402


def host(t, shape):
    return np.asfortranarray(t.cpu().numpy().reshape(tuple(reversed(shape))).transpose())


def sin_angle(u, v):
    if u.shape[1] == 0 and v.shape[1] == 0:
        return 0.0
    return float(np.linalg.norm(v - u @ (u.T @ v), 2))


def slice_errors(gpu_rep, ref, b, nb_samples, numel):
    """Largest per-slice relative difference of batch b's reconstructions."""
    root_g = gpu_rep.root()
    lat_g = np.asfortranarray(root_g[:, :, b * nb_samples:(b + 1) * nb_samples])
    lat_r = np.asfortranarray(ref.root()[:, :, b * nb_samples:(b + 1) * nb_samples])
    rec_g = ht.decode(gpu_rep, lat_g).reshape((numel, nb_samples), order="F")
    rec_r = ho.decode(ref, lat_r).reshape((numel, nb_samples), order="F")
    num = np.linalg.norm(rec_g - rec_r, axis=0)
    den = np.maximum(np.linalg.norm(rec_r, axis=0), 1e-300)
    return float(np.max(num / den))


def run(name, n_batches=None, batch=None, compare="some", out=sys.stdout):
    w = CONFIGS[name]
    if batch:
        w = dataclasses.replace(w, batch=batch)
    nb = w.n_batches if n_batches is None else n_batches
    shape = tuple(w.dims) + (w.batch,)
    numel = int(np.prod(w.dims))
    tree = ho.custom_tree_1_23() if w.tree_kind == "1_23" else ho.DimensionTree.balanced(len(w.dims))
    ctx = ht.Context(0)
    ht.set_default_context(ctx)
    summary = {"config": name, "batch": w.batch, "batches": nb, "ranks_identical": True, "skips_identical": True,
               "max_proj_error_diff": 0.0, "max_leaf_angle": 0.0, "max_slice_rel": 0.0, "compared_batches": [],
               "threads": torch.get_num_threads()}
    t_all = time.time()
    y = w.make_batch(0, "cuda")
    t0 = time.time()
    gpu, _ = ht.bht_l2r(ht.DeviceTensor(y, shape), w.tree(), w.eps)
    torch.cuda.synchronize()
    t_gpu = time.time() - t0
    yh = host(y, shape)
    del y
    t0 = time.time()
    ref, _ = ho.bht_l2r(yh, tree, w.eps)
    t_ref = time.time() - t0
    del yh
    check = set(range(nb)) if compare == "all" else {0, 1, nb // 2, nb - 1}
    for b in range(nb):
        rec = {"config": name, "batch": b}
        if b > 0:
            y = w.make_batch(b, "cuda")
            t0 = time.time()
            gpu, ug = ht.ht_rise_update(gpu, ht.DeviceTensor(y, shape))
            t_gpu = time.time() - t0
            ynorm = float(y.norm())
            yh = host(y, shape)
            del y
            t0 = time.time()
            ref, ur = ho.ht_rise_update(ref, yh)
            t_ref = time.time() - t0
            del yh
            rec.update({"skipped": bool(ug.skipped), "skipped_oracle": bool(ur.skipped),
                        "proj_error": ug.proj_error, "proj_error_oracle": ur.proj_error,
                        "proj_error_diff_rel_y": abs(ug.proj_error - ur.proj_error) / ynorm,
                        "eps_des_rel_diff": abs(ug.eps_des - ur.eps_des) / ur.eps_des,
                        "used_fused_path": bool(ug.used_fused_path), "used_exact_loss": bool(ug.used_exact_loss)})
            summary["skips_identical"] &= rec["skipped"] == rec["skipped_oracle"]
            summary["max_proj_error_diff"] = max(summary["max_proj_error_diff"], rec["proj_error_diff_rel_y"])
        rg, rr = gpu.ranks(), ref.ranks()
        rec["ranks"] = {f"{k[0]},{k[1]}": v for k, v in rg.items()}
        rec["ranks_identical"] = rg == rr
        summary["ranks_identical"] &= rec["ranks_identical"]
        ang = 0.0
        for l in range(1, ref.tree.depth + 1):
            for n in ref.tree.layer(l):
                if n.kind == ho.LEAF:
                    ang = max(ang, sin_angle(ref.basis_matrix(n.id), gpu.basis_matrix(n.id)))
        rec["max_leaf_angle"] = ang
        summary["max_leaf_angle"] = max(summary["max_leaf_angle"], ang)
        rec["seconds_gpu_call"] = t_gpu
        rec["seconds_oracle"] = t_ref
        if b in check:
            rec["max_slice_rel"] = slice_errors(gpu, ref, b, w.batch, numel)
            summary["max_slice_rel"] = max(summary["max_slice_rel"], rec["max_slice_rel"])
            summary["compared_batches"].append(b)
        print(json.dumps(rec), file=out, flush=True)
    if compare != "all":
        # every slice of every batch against the final representations
        for b in range(nb):
            if b in check:
                continue
            e = slice_errors(gpu, ref, b, w.batch, numel)
            summary["max_slice_rel"] = max(summary["max_slice_rel"], e)
            summary["compared_batches"].append(b)
    summary["seconds_total"] = time.time() - t_all
    summary["pass"] = bool(summary["ranks_identical"] and summary["skips_identical"] and
                           summary["max_proj_error_diff"] <= 1e-9 and summary["max_leaf_angle"] <= 1e-8 and
                           summary["max_slice_rel"] <= 1e-9)
    print(json.dumps({"summary": summary}), file=out, flush=True)
    return summary


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--batches", type=int, default=None)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--compare", default="some", choices=["some", "all"])
    a = ap.parse_args()
    s = run(a.config, a.batches, a.batch, a.compare)
    sys.exit(0 if s["pass"] else 1)
