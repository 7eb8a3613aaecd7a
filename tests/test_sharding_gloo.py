"""Multi-rank (batch-axis sharded) decomposition, checked on the CPU with a
2-rank gloo process group.

The runtime shards every batch along its sample axis and all-reduces only
(a) the Grams Y_(k) Y_(k)^T that feed each truncation, (b) the norms of the
skip test and (c) the global batch count. This test restates
that decomposition in numpy — local Grams + all_reduce + identical
eigen-truncations on every rank + local projections — and checks it against
the unsharded CPU oracle: identical ranks, identical skip decisions and
identical reconstructions of each rank's own samples."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import htrise_oracle as ho
from oracle import ref_oracles as ro


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _allreduce(a: np.ndarray) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


def _truncate_gram(g, rows, cols, eps_abs, min_rank):
    lam, v = np.linalg.eigh(0.5 * (g + g.T))
    lam, v = lam[::-1], v[:, ::-1]
    k = min(rows, cols)
    if np.sum(np.maximum(lam, 0)) == 0.0:
        r = min(max(min_rank, 0), rows)
        return np.eye(rows, r), r
    rank, _ = ho.rank_rule(np.sqrt(np.maximum(lam[:k], 0.0)), eps_abs, min_rank)
    return v[:, :rank], rank


def _sharded_gram(c, mode, world_batch_cols):
    m = ho.unfold(c, mode)
    return _allreduce(m @ m.T), m.shape[0], world_batch_cols(m)


def sharded_bht_l2r(y_local, tree, eps_rel, n_global):
    """Runtime's bht_l2r with every global quantity all-reduced."""
    d, p = tree.dims(), tree.depth
    nloc = y_local.shape[-1]
    ysq = float(_allreduce(np.array([np.sum(y_local ** 2)]))[0])
    eps_abs = ho.effective_eps_rel(eps_rel) * math.sqrt(ysq)
    eps_nw = eps_abs / math.sqrt(2 * d - 2)
    cols = lambda m: m.shape[1] // nloc * n_global  # noqa: E731
    cores = [[None] * tree.layer_size(l) for l in range(p + 1)]
    c = y_local
    bases = []
    for n in tree.layer(p):
        g, rows, cc = _sharded_gram(c, n.leaf_dim, cols)
        bases.append(_truncate_gram(g, rows, cc, eps_nw, 1)[0])
    for i, n in enumerate(tree.layer(p)):
        cores[p][i] = bases[i]
        c = ho.mode_multiply(c, n.leaf_dim, bases[i].T)
    ranks = {n.id: cores[p][i].shape[1] for i, n in enumerate(tree.layer(p))}
    dims = list(y_local.shape[:d])
    for l in range(p - 1, 0, -1):
        ext = ho._layer_extents(tree, l, dims, ranks, nloc)
        c = ho.reshape(c, ext)
        lb = []
        for j in range(tree.layer_size(l)):
            g, rows, cc = _sharded_gram(c, j, cols)
            lb.append(_truncate_gram(g, rows, cc, eps_nw, 1)[0])
        for j, n in enumerate(tree.layer(l)):
            u = lb[j]
            cores[l][j] = u if n.kind == ho.LEAF else ho.reshape(
                u, [ranks[n.successors[0]], ranks[n.successors[1]], u.shape[1]])
            ranks[n.id] = u.shape[1]
        for j in range(tree.layer_size(l)):
            c = ho.mode_multiply(c, j, lb[j].T)
    rootn = tree.node((0, 0))
    cores[0][0] = ho.reshape(c, [ranks[rootn.successors[0]], ranks[rootn.successors[1]], nloc])
    return ho.HTRepresentation(tree, dims, cores, nloc, eps_rel)


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(2024)
        bases = [ro.random_orthonormal(6, 3, rng) for _ in range(4)]
        y = ro.tucker_family_batch(bases, 8, rng) + 1e-6 * rng.standard_normal((6, 6, 6, 6, 8))
        y2 = ro.tucker_family_batch(bases, 8, rng) + 1e-6 * rng.standard_normal((6, 6, 6, 6, 8))
        tree = ho.DimensionTree.balanced(4)
        n = y.shape[-1] // world
        sl = slice(rank * n, (rank + 1) * n)
        rep = sharded_bht_l2r(np.asfortranarray(y[..., sl]), tree, 1e-3, y.shape[-1])
        ref, _ = ho.bht_l2r(y, tree, 1e-3)
        ok_ranks = rep.ranks() == ref.ranks()
        # every rank reconstructs its own samples exactly like the unsharded run
        worst = 0.0
        for m in range(n):
            a = ho.reconstruct_slice(rep, m + 1)
            b = ho.reconstruct_slice(ref, rank * n + m + 1)
            worst = max(worst, float(np.linalg.norm(a - b) / np.linalg.norm(b)))
        # skip test of the next batch: two all-reduced norms
        lat, _ = ho.encode(rep, np.asfortranarray(y2[..., sl]))
        sums = _allreduce(np.array([np.sum(y2[..., sl] ** 2), np.sum(lat ** 2)]))
        proj = math.sqrt(max(0.0, sums[0] - sums[1]))
        _, upd = ho.ht_rise_update(ref, y2)
        skip_sharded = proj <= 1e-3 * math.sqrt(sums[0])
        out_q.put((rank, ok_ranks, worst, skip_sharded == upd.skipped, abs(proj - upd.proj_error) / upd.proj_error))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_decomposition_matches_unsharded():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_ranks, worst, same_skip, proj_rel in results:
        assert ok_ranks, rank
        assert worst <= 1e-9, (rank, worst)
        assert same_skip, rank
        assert proj_rel <= 1e-4, (rank, proj_rel)


def _reducer_worker(rank, world, port, out_q):
    """The library's host-reducer plumbing (htr_host_reduce_fn built by
    htrise.host_reduce_callback over a gloo group), called the way
    Context::allreduce calls it: a C double buffer summed in place."""
    import ctypes as C

    from paper_2412_16544_b200 import htrise as ht

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cb = ht.host_reduce_callback(ht.gloo_reducer())
        buf = (C.c_double * 5)(*[rank + 0.5 * i for i in range(5)])
        rc = cb(buf, 5, None)
        empty = cb(buf, 0, None)
        failing = ht.host_reduce_callback(lambda a: (_ for _ in ()).throw(RuntimeError("transport down")))
        rc_fail = failing(buf, 5, None)
        out_q.put((rank, rc, empty, rc_fail, list(buf)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_host_reducer_callback_sums_over_ranks(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_reducer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [sum(r + 0.5 * i for r in range(world)) for i in range(5)]
    for rank, rc, empty, rc_fail, vals in results:
        assert rc == 0 and empty == 0 and rc_fail == 1, rank
        assert vals == want, (rank, vals, want)
