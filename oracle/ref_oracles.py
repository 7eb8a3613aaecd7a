"""Restatement of the reference's loop-based test oracles
(/root/reference/proj/tests/oracles.hpp), independent of unfold/contract.
TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import itertools

import numpy as np

from . import htrise_oracle as ho


def random_tensor(shape, rng: np.random.Generator) -> np.ndarray:
    """oracles.hpp:189-194 (values differ: numpy normals, not libstdc++)."""
    return rng.standard_normal(int(np.prod(shape))).reshape(tuple(shape), order="F")


def random_orthonormal(rows, cols, rng) -> np.ndarray:
    """oracles.hpp:196-205: Householder Q of a Gaussian matrix."""
    g = rng.standard_normal((rows, cols))
    q, _ = np.linalg.qr(g, mode="reduced")
    return q


def naive_mode_multiply(t: np.ndarray, mode: int, m: np.ndarray) -> np.ndarray:
    """oracles.hpp:88-105, by explicit summation (einsum, no unfold)."""
    letters = "abcdefghijklmnop"
    src = letters[: t.ndim]
    dst = src[:mode] + "z" + src[mode + 1:]
    return np.einsum(f"z{src[mode]},{src}->{dst}", m, t)


def tucker_family_batch(bases, n, rng) -> np.ndarray:
    """oracles.hpp:209-236: random cores contracted with fixed bases."""
    dims = [b.shape[0] for b in bases]
    core_shape = [b.shape[1] for b in bases]
    out = np.zeros(dims + [n], order="F")
    for s in range(n):
        sl = random_tensor(core_shape, rng)
        for k, b in enumerate(bases):
            sl = naive_mode_multiply(sl, k, b)
        out[..., s] = sl
    return out


def dense_reconstruction(h: ho.HTRepresentation) -> np.ndarray:
    """oracles.hpp:110-146: bottom-up Kronecker frames."""
    def frame(nid):
        n = h.tree.node(nid)
        if n.kind == ho.LEAF:
            return h.core(nid), h.dims[n.leaf_dim]
        fl, sl = frame(n.successors[0])
        fr, sr = frame(n.successors[1])
        core = h.core(nid)
        # f(a + sl*b, k) = sum_ij core(i,j,k) fl(a,i) fr(b,j)
        f = np.einsum("ijk,ai,bj->abk", core, fl, fr).reshape(sl * sr, core.shape[2], order="F")
        return f, sl * sr
    full, _ = frame((0, 0))
    return full.reshape(list(h.dims) + [h.accumulated], order="F")


def span_matricization(y: np.ndarray, a: int, b: int) -> np.ndarray:
    """oracles.hpp:150-170: rows over dims [a..b] (first fastest), columns
    over the rest in canonical order."""
    d = y.ndim
    rows_axes = list(range(a, b + 1))
    rest = [k for k in range(d) if k < a or k > b]
    t = np.transpose(y, rows_axes + rest)
    rows = int(np.prod([y.shape[k] for k in rows_axes]))
    return t.reshape(rows, -1, order="F")


def tail_rank(m: np.ndarray, eps_abs: float) -> int:
    """oracles.hpp:174-185 with an independent dense SVD."""
    s = np.linalg.svd(m, compute_uv=False)
    tail = 0.0
    rank = len(s)
    for i in range(len(s) - 1, -1, -1):
        tail += s[i] * s[i]
        if np.sqrt(tail) > eps_abs:
            break
        rank = i
    return max(rank, 1)
