"""One rank of a batch-sharded run of the library on a shared GPU (helper of
tests/test_gpu_multirank.py, not collected by pytest).

Every rank generates the full batch (same seeded bytes), keeps its own
sample range, and runs bht_l2r + ht_rise_update through the C-ABI with a
host-staged reducer (htr_context_set_reducer over a gloo group): the
runtime's nranks > 1 path — Gram and norm all-reduces, the global batch
count, the column scale of the rank rule, the sharded root — with no rank
ever waiting on another rank's kernels. The unsharded oracle's results
(computed once by the parent, pickled) are the checker.

argv: <spec.pkl> <out.json>; env RANK, WORLD_SIZE, MASTER_ADDR, MASTER_PORT.
"""
import hashlib
import json
import math
import os
import pickle
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import htrise_oracle as ho  # noqa: E402  (checker only)
from paper_2412_16544_b200 import htrise as ht  # noqa: E402
from paper_2412_16544_b200.workloads import CONFIGS  # noqa: E402


def shard_bounds(n: int, world: int, rank: int):
    """Samples [off, off + cnt) of an n-sample batch held by `rank` (the
    first n % world ranks take one more)."""
    base, extra = divmod(n, world)
    cnt = base + (1 if rank < extra else 0)
    off = rank * base + min(rank, extra)
    return off, cnt


def core_digest(rep) -> str:
    h = hashlib.sha256()
    for l in range(1, rep.tree.depth + 1):
        for n in rep.tree.layer(l):
            h.update(np.ascontiguousarray(rep.core(n.id)).tobytes())
    return h.hexdigest()


class TuckerWorkload:
    """A seeded Tucker-family stream on the (1,(2,3)) tree (test cases the
    BASELINE configs do not reach, e.g. a transfer node with more rows than
    its unfolding has columns)."""

    def __init__(self, spec):
        self.dims = tuple(spec["dims"])
        self.ranks = tuple(spec["ranks"])
        self.batch = spec["batch"]
        self.eps = spec["eps"]
        self.seed = spec["seed"]

    def tree(self):
        return ht.tree_1_23()

    def make_host(self, b):
        rng = np.random.default_rng(self.seed)
        bases = [np.linalg.qr(rng.standard_normal((n, r)))[0] for n, r in zip(self.dims, self.ranks)]
        rng_b = np.random.default_rng(self.seed * 1000 + b)
        cores = rng_b.standard_normal(tuple(self.ranks) + (self.batch,))
        y = np.einsum("abcs,ia,jb,kc->ijks", cores, *bases)
        return np.asfortranarray(y + 1e-9 * rng_b.standard_normal(y.shape))

    def make_batch(self, b, device="cuda"):
        y = self.make_host(b)
        return torch.from_numpy(np.ascontiguousarray(y.transpose(3, 2, 1, 0))).to(device).reshape(-1)


def workload_of(case):
    import dataclasses

    if case.get("custom"):
        return TuckerWorkload(case["custom"])
    w = CONFIGS[case["config"]]
    if case.get("batch"):
        w = dataclasses.replace(w, batch=case["batch"])
    return w


def run_case(case, rank, world, ctx):
    w = workload_of(case)
    ref = case["oracle"]  # per batch: ranks, skipped, proj_error, eps_des; final rep
    nb = case["n_batches"]
    numel = int(np.prod(w.dims))
    off, cnt = shard_bounds(w.batch, world, rank)
    shape = tuple(w.dims) + (cnt,)
    out = {"config": case["config"], "rank": rank, "shard": [off, cnt], "errors": []}

    def shard(b):
        y = w.make_batch(b, "cuda")
        return y[off * numel:(off + cnt) * numel].clone()

    y = shard(0)
    rep, _ = ht.bht_l2r(ht.DeviceTensor(y, shape), w.tree(), w.eps, ctx=ctx)
    if rep.ranks() != ref["ranks"][0]:
        out["errors"].append(f"bht_l2r ranks {rep.ranks()} vs oracle {ref['ranks'][0]}")
    worst_pe = 0.0
    for b in range(1, nb):
        y = shard(b)
        rep, upd = ht.ht_rise_update(rep, ht.DeviceTensor(y, shape))
        r = ref["updates"][b - 1]
        if bool(upd.skipped) != r["skipped"]:
            out["errors"].append(f"batch {b}: skipped {upd.skipped} vs oracle {r['skipped']}")
        if rep.ranks() != ref["ranks"][b]:
            out["errors"].append(f"batch {b}: ranks {rep.ranks()} vs oracle {ref['ranks'][b]}")
        ynorm = r["eps_des"] / w.eps
        if abs(upd.eps_des - r["eps_des"]) > 1e-12 * r["eps_des"]:
            out["errors"].append(f"batch {b}: eps_des {upd.eps_des} vs {r['eps_des']}")
        worst_pe = max(worst_pe, abs(upd.proj_error - r["proj_error"]) / ynorm)
    out["worst_proj_error_diff"] = worst_pe
    if rep.accumulated != nb * w.batch or rep.local_count != nb * cnt:
        out["errors"].append(f"counts {rep.accumulated}/{rep.local_count} vs {nb * w.batch}/{nb * cnt}")
    # this rank's slices against the unsharded oracle's
    final = ref["final"]
    worst = 0.0
    for b in range(nb):
        for j in range(cnt):
            a = ht.reconstruct_slice(rep, b * cnt + j + 1)
            e = ho.reconstruct_slice(final, b * w.batch + off + j + 1)
            worst = max(worst, float(np.linalg.norm(a - e) / max(np.linalg.norm(e), 1e-300)))
    out["worst_slice_rel"] = worst
    out["digest"] = core_digest(rep)
    digests = [None] * world
    dist.all_gather_object(digests, out["digest"])
    out["digests_identical"] = len(set(digests)) == 1
    return out


def main():
    spec_path, out_path = sys.argv[1], sys.argv[2]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    results = []
    try:
        with open(spec_path, "rb") as f:
            spec = pickle.load(f)
        ctx = ht.Context(0)
        ctx.set_reducer(ht.gloo_reducer(), world, rank)
        for case in spec:
            results.append(run_case(case, rank, world, ctx))
    except Exception:  # noqa: BLE001 - reported to the parent
        results.append({"rank": rank, "errors": [traceback.format_exc()]})
    with open(out_path, "w") as f:
        json.dump(results, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
