"""The sharded runtime (nranks > 1) executed: 2, 3 and 4 processes share one
B200, each one rank of a batch-sharded stream.

gpurun gives one GPU, and NCCL refuses two ranks on one device, so the ranks
reduce through the library's host-staged reducer (htr_context_set_reducer,
a gloo all-reduce on the host). Each rank drains its own stream before its
partial sums leave the device, so no kernel waits on another rank's kernel.
Everything above the reduction is the same runtime path as with NCCL: the
Gram and norm all-reduces of BHT-l2r, the skip test and the expansions, the
global batch count and the rank rule's global column count, the sharded root.

Bars (BASELINE.json north_star, checked per rank against the UNSHARDED
oracle run on the same bytes): identical ranks at every node after every
batch, identical skip decisions, proj_error within 1e-9 ||y|| and eps_des
within 1e-12 relative, every slice the rank holds within 1e-9 relative of
the oracle's reconstruction of the same global sample, and the non-root
cores bit-identical across ranks (the reduced Grams were identical).
"""
import dataclasses
import json
import os
import pickle
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import htrise_oracle as ho

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "multirank_worker.py")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _host(t, shape):
    return np.asfortranarray(t.cpu().numpy().reshape(tuple(reversed(shape))).transpose())


def _oracle_case(config, n_batches, batch=None, custom=None):
    from paper_2412_16544_b200.workloads import CONFIGS

    if custom:
        sys.path.insert(0, os.path.dirname(WORKER))
        from multirank_worker import TuckerWorkload

        w = TuckerWorkload(custom)
        tree = ho.custom_tree_1_23()
        host_batch = w.make_host
    else:
        w = CONFIGS[config]
        if batch:
            w = dataclasses.replace(w, batch=batch)
        tree = ho.custom_tree_1_23() if w.tree_kind == "1_23" else ho.DimensionTree.balanced(len(w.dims))
        shape = tuple(w.dims) + (w.batch,)
        host_batch = lambda b: _host(w.make_batch(b, "cuda"), shape)  # noqa: E731
    ref, _ = ho.bht_l2r(host_batch(0), tree, w.eps)
    ranks = [ref.ranks()]
    updates = []
    for b in range(1, n_batches):
        ref, r = ho.ht_rise_update(ref, host_batch(b))
        ranks.append(ref.ranks())
        updates.append({"skipped": bool(r.skipped), "proj_error": float(r.proj_error), "eps_des": float(r.eps_des)})
    return {"config": config, "batch": batch, "n_batches": n_batches, "custom": custom,
            "oracle": {"ranks": ranks, "updates": updates, "final": ref}}


def _run_world(world, cases, tmp_path):
    spec = tmp_path / f"spec{world}.pkl"
    with open(spec, "wb") as f:
        pickle.dump(cases, f)
    port = _free_port()
    procs, outs = [], []
    for r in range(world):
        out = tmp_path / f"out{world}_{r}.json"
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, WORKER, str(spec), str(out)], env=env, cwd=ROOT))
        outs.append(out)
    for p in procs:
        assert p.wait(timeout=1200) == 0
    results = []
    for out in outs:
        with open(out) as f:
            results.extend(json.load(f))
    return results


def _check(results, n_cases, world):
    assert len(results) == n_cases * world, results
    for r in results:
        assert not r["errors"], r
        assert r["digests_identical"], r
        assert r["worst_slice_rel"] <= 1e-9, r
        assert r["worst_proj_error_diff"] <= 1e-9, r


@pytest.fixture(scope="module")
def cuda():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"


def test_two_ranks_all_configs(cuda, tmp_path):
    """Every config's path sharded over 2 ranks: c1 (BHT-l2r, generic 4-way),
    c2 (fused 3-way leaf + tail kernels on 16-sample shards), c3 through its
    batch-25 expansion (residual Grams all-reduced), c4 (fused 8-way subtree
    kernels), c5's 128^3 rank-20 shapes (fused path, 3-sample shards)."""
    # + a 48 x 34 x 12 family: slabs that are no multiple of the fused kernel's
    # steps (the padded 64 x 64 kernel) through skip updates on 4-sample shards
    padded = {"dims": [48, 34, 12], "ranks": [5, 4, 3], "batch": 8, "eps": 1e-6, "seed": 11}
    cases = [_oracle_case("c1", 1), _oracle_case("c2", 4), _oracle_case("c3", 26),
             _oracle_case("c4", 2), _oracle_case("c5", 3, batch=6), _oracle_case("padded", 4, custom=padded)]
    _check(_run_world(2, cases, tmp_path), len(cases), 2)


def test_three_ranks_uneven_shards(cuda, tmp_path):
    """Uneven shards (c2: 11/11/10 samples, c3: 6/5/5) through skips and the
    expansion: the rank rule's global column count and the global batch
    count come from the all-reduce, not from world * local."""
    cases = [_oracle_case("c2", 3), _oracle_case("c3", 26)]
    _check(_run_world(3, cases, tmp_path), len(cases), 3)


def test_two_ranks_tall_transfer_gathered(cuda, tmp_path):
    """A transfer node whose unfolding has more rows (35 x 35 = 1225) than
    columns over all ranks (r0 x 6 samples): the column-side truncation
    needs every column, so the sharded runtime gathers the unfolding
    (all-reduce of a zero-initialised buffer) and every rank truncates the
    same bits -- BHT-l2r and an expanding update."""
    tall = {"dims": [24, 40, 40], "ranks": [5, 35, 35], "batch": 6, "eps": 1e-6, "seed": 7}
    cases = [_oracle_case("tall", 2, custom=tall)]
    _check(_run_world(2, cases, tmp_path), len(cases), 2)


def test_four_ranks(cuda, tmp_path):
    cases = [_oracle_case("c1", 1), _oracle_case("c2", 3)]
    _check(_run_world(4, cases, tmp_path), len(cases), 4)
