"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of the reference's BHT-l2r / HT-RISE algorithms
(/root/reference/proj/include/htrise/*.hpp), operation for operation, used
by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm as the *checker*. Nothing under paper_2412_16544_b200/ imports this file.

Why a restatement: the reference is header-only C++20 on Eigen3 (unpinned,
>=3.3, CMakeLists.txt:12) and Eigen is absent from this image and from the GPU
box, so the reference cannot be compiled here. The
arithmetic the reference delegates to Eigen is restated with numpy/LAPACK:

* Eigen::BDCSVD (divide and conquer bidiagonal SVD, truncated_svd.hpp:35,41)
  -> numpy.linalg.svd = LAPACK dgesdd (also divide and conquer).
* Eigen::HouseholderQR (truncated_svd.hpp:33) -> numpy.linalg.qr (dgeqrf).
* Eigen GEMM / norms -> numpy matmul / sum of squares.

Pinning (no stored golden arrays exist in the reference):
the known-answer tests and properties of test_truncated_svd.cpp,
test_dimension_tree.cpp, test_bht.cpp, test_ht_rise.cpp, test_metrics.cpp and
acceptance.cpp are ported in tests/test_oracle_*.py and must pass before the
oracle is trusted.

Layout: tensors are numpy arrays whose *canonical* linear order is the
reference's first-index-fastest order (tensor.hpp:36-41), i.e. numpy Fortran
order. ``flat(t)`` = ``t.ravel(order="F")``.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

ROOT, TRANSFER, LEAF = 0, 1, 2  # NodeKind order of dimension_tree.hpp:14


# ---------------------------------------------------------------------------
# tensor.hpp
# ---------------------------------------------------------------------------

def flat(t: np.ndarray) -> np.ndarray:
    return np.asarray(t).ravel(order="F")


def from_flat(data: np.ndarray, shape) -> np.ndarray:
    return np.asarray(data, dtype=np.float64).reshape(tuple(shape), order="F")


def _check_mode(t: np.ndarray, mode: int, who: str) -> None:
    if mode < 0 or mode >= t.ndim:
        raise ValueError(f"{who}: mode {mode} out of range for order {t.ndim}")


def unfold(t: np.ndarray, mode: int) -> np.ndarray:
    """tensor.hpp:150-172: rows = extent(mode), columns enumerate the remaining
    indices in canonical order with `mode` removed."""
    _check_mode(t, mode, "unfold")
    rows = t.shape[mode]
    return np.moveaxis(t, mode, 0).reshape(rows, -1, order="F")


def fold(m: np.ndarray, shape, mode: int) -> np.ndarray:
    """tensor.hpp:176-205: exact inverse of unfold."""
    shape = list(shape)
    if mode < 0 or mode >= len(shape):
        raise ValueError("fold: mode out of range")
    rows = shape[mode]
    total = int(np.prod(shape))
    if m.shape[0] != rows or m.size != total:
        raise ValueError("fold: matrix inconsistent with shape")
    rest = shape[:mode] + shape[mode + 1:]
    return np.moveaxis(m.reshape([rows] + rest, order="F"), 0, mode)


def reshape(t: np.ndarray, index_set) -> np.ndarray:
    """tensor.hpp:209-216: same canonical buffer under a new extent list."""
    if int(np.prod(index_set)) != t.size:
        raise ValueError("reshape: product mismatch")
    return np.asarray(t).reshape(tuple(index_set), order="F")


def frobenius_norm(t: np.ndarray) -> float:
    """tensor.hpp:269."""
    return float(np.linalg.norm(flat(t)))


def mode_multiply(t: np.ndarray, mode: int, m: np.ndarray) -> np.ndarray:
    """tensor.hpp:300-312: fold(M * unfold(t, mode))."""
    _check_mode(t, mode, "mode_multiply")
    if m.shape[1] != t.shape[mode]:
        raise ValueError("mode_multiply: factor/extent mismatch")
    prod = m @ unfold(t, mode)
    out_shape = list(t.shape)
    out_shape[mode] = m.shape[0]
    return fold(prod, out_shape, mode)


def contract3_split(t: np.ndarray, mode: int, core: np.ndarray) -> np.ndarray:
    """multi_contract with one 3-way factor contracting its last axis
    (tensor.hpp:353-374): mode `mode` (extent fs2) is replaced in place by
    the factor's two free axes (fs0, fs1)."""
    fs = core.shape
    m = core.reshape(fs[0] * fs[1], fs[2], order="F")
    if m.shape[1] != t.shape[mode]:
        raise ValueError("multi_contract: extent mismatch")
    prod = m @ unfold(t, mode)
    merged = list(t.shape)
    merged[mode] = fs[0] * fs[1]
    out_shape = list(t.shape)
    out_shape[mode] = fs[0]
    out_shape.insert(mode + 1, fs[1])
    return reshape(fold(prod, merged, mode), out_shape)


def concat(a: np.ndarray, b: np.ndarray, k: int) -> np.ndarray:
    """tensor.hpp:383-412."""
    _check_mode(a, k, "concat")
    if a.ndim != b.ndim:
        raise ValueError("concat: order mismatch")
    for m in range(a.ndim):
        if m != k and a.shape[m] != b.shape[m]:
            raise ValueError("concat: shapes differ off mode")
    return np.concatenate([a, b], axis=k)


def pad_zeros(t: np.ndarray, k: int, extra: int) -> np.ndarray:
    """tensor.hpp:415-422."""
    if extra == 0:
        return t
    if extra < 0:
        raise ValueError("pad_zeros: negative pad")
    zshape = list(t.shape)
    zshape[k] = extra
    return concat(t, np.zeros(zshape), k)


def slice_(t: np.ndarray, k: int, start: int, count: int) -> np.ndarray:
    """tensor.hpp:425-445."""
    _check_mode(t, k, "slice")
    if start < 0 or count < 1 or start + count > t.shape[k]:
        raise IndexError("slice: range out of bounds")
    idx = [slice(None)] * t.ndim
    idx[k] = slice(start, start + count)
    return t[tuple(idx)]


# ---------------------------------------------------------------------------
# truncated_svd.hpp
# ---------------------------------------------------------------------------

@dataclass
class TruncatedBasis:
    """truncated_svd.hpp:17-22."""
    u: np.ndarray
    rank: int
    discarded_norm: float
    singular_values: np.ndarray


def thin_svd(m: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """truncated_svd.hpp:29-45: tall inputs (rows > 2 cols) go through a
    Householder QR first, else a direct divide-and-conquer SVD."""
    rows, cols = m.shape
    if rows > 2 * cols:
        q, r = np.linalg.qr(m, mode="reduced")
        ur, s, _ = np.linalg.svd(r, full_matrices=False)
        return q @ ur, s
    u, s, _ = np.linalg.svd(m, full_matrices=False)
    return u, s


def rank_rule(sigma: np.ndarray, eps_abs: float, min_rank: int) -> Tuple[int, float]:
    """truncated_svd.hpp:74-99: tail[r] = sum_{i>=r} sigma_i^2 accumulated from
    the smallest; rank = smallest r with sqrt(tail[r]) <= eps_abs, floored at
    min_rank and capped at k = len(sigma)."""
    k = len(sigma)
    tail = [0.0] * (k + 1)
    for i in range(k - 1, -1, -1):
        tail[i] = tail[i + 1] + float(sigma[i]) * float(sigma[i])
    rank = k
    for r in range(k + 1):
        if math.sqrt(tail[r]) <= eps_abs:
            rank = r
            break
    rank = max(rank, min_rank)
    rank = min(rank, k)
    return rank, math.sqrt(tail[rank])


def truncated_svd(m: np.ndarray, eps_abs: float, min_rank: int = 1) -> TruncatedBasis:
    """truncated_svd.hpp:53-100."""
    m = np.asarray(m, dtype=np.float64)
    if m.size == 0:
        raise ValueError("truncated_svd: empty matrix")
    if not np.all(np.isfinite(m)):
        raise ValueError("truncated_svd: non-finite entries")
    if eps_abs < 0:
        raise ValueError("truncated_svd: negative tolerance")
    if np.linalg.norm(m) == 0.0:
        rank = min(max(min_rank, 0), m.shape[0])
        return TruncatedBasis(np.eye(m.shape[0], rank), rank, 0.0, np.zeros(rank))
    u, sigma = thin_svd(m)
    rank, disc = rank_rule(sigma, eps_abs, min_rank)
    return TruncatedBasis(u[:, :rank].copy(), rank, disc, sigma[:rank].copy())


def hosvd_layer(c: np.ndarray, modes, eps_nw: float, min_rank: int = 1) -> List[TruncatedBasis]:
    """truncated_svd.hpp:105-123: independent truncated SVD per listed mode of
    the same tensor."""
    seen = set()
    for m in modes:
        _check_mode(c, m, "hosvd_layer")
        if m in seen:
            raise ValueError("hosvd_layer: duplicate mode")
        seen.add(m)
    return [truncated_svd(unfold(c, m), eps_nw, min_rank) for m in modes]


# ---------------------------------------------------------------------------
# dimension_tree.hpp
# ---------------------------------------------------------------------------

@dataclass
class TreeNode:
    """dimension_tree.hpp:28-34. id = (layer, pos)."""
    id: Tuple[int, int]
    kind: int
    successors: List[Tuple[int, int]] = field(default_factory=list)
    parent: Tuple[int, int] = (0, 0)
    leaf_dim: int = -1


class DimensionTree:
    """dimension_tree.hpp:39-272."""

    def __init__(self):
        self.d = 0
        self.depth = 0
        self.layers: List[List[TreeNode]] = []

    @staticmethod
    def balanced(d: int) -> "DimensionTree":
        """dimension_tree.hpp:44-94: left-biased split ceil(len/2)."""
        if d < 2:
            raise ValueError(f"DimensionTree: need d >= 2, got {d}")
        spans = [[(0, d - 1)]]
        while True:
            nxt = []
            grew = False
            for a, b in spans[-1]:
                if a == b:
                    continue
                ln = b - a + 1
                left = (ln + 1) // 2
                nxt.append((a, a + left - 1))
                nxt.append((a + left, b))
                grew = True
            if not grew:
                break
            spans.append(nxt)
        t = DimensionTree()
        t.d = d
        t.depth = len(spans) - 1
        for l, layer in enumerate(spans):
            nodes = []
            nc = 0
            for i, (a, b) in enumerate(layer):
                if a == b:
                    nodes.append(TreeNode((l, i), LEAF, [], (0, 0), a))
                else:
                    kind = ROOT if l == 0 else TRANSFER
                    nodes.append(TreeNode((l, i), kind, [(l + 1, nc), (l + 1, nc + 1)]))
                    nc += 2
            t.layers.append(nodes)
        t._link_parents()
        t._validate()
        return t

    @staticmethod
    def from_layers(layers) -> "DimensionTree":
        """dimension_tree.hpp:99-113."""
        t = DimensionTree()
        t.layers = [[TreeNode(tuple(n.id), n.kind, [tuple(s) for s in n.successors],
                              tuple(n.parent), n.leaf_dim) for n in layer] for layer in layers]
        t.depth = len(t.layers) - 1
        t.d = sum(1 for layer in t.layers for n in layer if n.kind == LEAF)
        t._link_parents()
        t._validate()
        return t

    def dims(self) -> int:
        return self.d

    def node_count(self) -> int:
        return 2 * self.d - 1

    def layer_size(self, l: int) -> int:
        return len(self.layers[l])

    def layer(self, l: int) -> List[TreeNode]:
        return self.layers[l]

    def node(self, nid) -> TreeNode:
        l, p = nid
        if l < 0 or l >= len(self.layers) or p < 0 or p >= len(self.layers[l]):
            raise IndexError(f"DimensionTree: unknown node {nid}")
        return self.layers[l][p]

    def parent_slot(self, nid) -> int:
        """dimension_tree.hpp:133-140."""
        n = self.node(nid)
        if n.kind == ROOT:
            raise ValueError("parent_slot: root has no parent")
        p = self.node(n.parent)
        return 0 if tuple(p.successors[0]) == tuple(nid) else 1

    def _link_parents(self):
        for layer in self.layers:
            for n in layer:
                for s in n.successors:
                    self.layers[s[0]][s[1]].parent = n.id

    def _validate(self):
        """dimension_tree.hpp:170-250."""
        if not self.layers or len(self.layers[0]) != 1:
            raise ValueError("DimensionTree: need a single root")
        p_expected = math.ceil(math.log2(self.d)) if self.d > 0 else 0
        if self.depth != p_expected:
            raise ValueError("DimensionTree: depth mismatch")
        count = 0
        seen = [False] * self.d
        for layer in self.layers:
            for n in layer:
                count += 1
                internal = n.kind != LEAF
                if internal and len(n.successors) != 2:
                    raise ValueError("DimensionTree: internal node must have 2 successors")
                if not internal and n.successors:
                    raise ValueError("DimensionTree: leaf has successors")
                if internal:
                    s0, s1 = n.successors
                    if s0[1] + 1 != s1[1] or s0[0] != n.id[0] + 1 or s1[0] != n.id[0] + 1:
                        raise ValueError("DimensionTree: successors must be adjacent")
                if n.kind == LEAF:
                    if n.id[0] < self.depth - 1:
                        raise ValueError("DimensionTree: leaf above the last two layers")
                    if n.leaf_dim < 0 or n.leaf_dim >= self.d or seen[n.leaf_dim]:
                        raise ValueError("DimensionTree: bad leaf dimension")
                    seen[n.leaf_dim] = True
        if count != 2 * self.d - 1:
            raise ValueError("DimensionTree: node count")
        claimed: Dict[Tuple[int, int], int] = {}
        for layer in self.layers:
            for n in layer:
                for s in n.successors:
                    claimed[tuple(s)] = claimed.get(tuple(s), 0) + 1
        for layer in self.layers:
            for n in layer:
                expect = 0 if n.id[0] == 0 else 1
                if claimed.get(tuple(n.id), 0) != expect:
                    raise ValueError("DimensionTree: bad parent linkage")
        if self._dim_span(self.node((0, 0))) != (0, self.d - 1):
            raise ValueError("DimensionTree: dimensions must appear in order")

    def _dim_span(self, n: TreeNode):
        if n.kind == LEAF:
            return (n.leaf_dim, n.leaf_dim)
        left = self._dim_span(self.node(n.successors[0]))
        right = self._dim_span(self.node(n.successors[1]))
        if left[1] + 1 != right[0]:
            raise ValueError("DimensionTree: successors do not cover adjacent spans")
        return (left[0], right[1])


def custom_tree_1_23() -> DimensionTree:
    """The (1,(2,3)) tree of test_bht.cpp:246-252 (configs 2 and 5)."""
    layers = [
        [TreeNode((0, 0), ROOT, [(1, 0), (1, 1)])],
        [TreeNode((1, 0), LEAF, [], (0, 0), 0), TreeNode((1, 1), TRANSFER, [(2, 0), (2, 1)])],
        [TreeNode((2, 0), LEAF, [], (0, 0), 1), TreeNode((2, 1), LEAF, [], (0, 0), 2)],
    ]
    return DimensionTree.from_layers(layers)


class IndexSet:
    """dimension_tree.hpp:292-374."""

    def __init__(self):
        self.layer_sets: List[List[int]] = []
        self.node_sets: Dict[Tuple[int, int], List[int]] = {}

    @staticmethod
    def build(tree: DimensionTree, dims, ranks, batch) -> "IndexSet":
        s = IndexSet()
        s.layer_sets = [None] * (tree.depth + 1)
        for l in range(tree.depth + 1):
            s.update_layer(tree, l, dims, ranks, batch)
            for n in tree.layer(l):
                s.update_node(tree, n.id, dims, ranks, batch)
        return s

    @staticmethod
    def _rank(ranks, nid):
        if tuple(nid) not in ranks:
            raise IndexError(f"IndexSet: no rank for node {nid}")
        return ranks[tuple(nid)]

    def update_layer(self, tree, layer, dims, ranks, batch):
        ext = []
        for n in tree.layer(layer):
            if n.kind == LEAF:
                ext.append(dims[n.leaf_dim])
            else:
                ext.append(self._rank(ranks, n.successors[0]) * self._rank(ranks, n.successors[1]))
        ext.append(batch)
        self.layer_sets[layer] = ext

    def update_node(self, tree, nid, dims, ranks, batch):
        n = tree.node(nid)
        if n.kind == LEAF:
            ext = [dims[n.leaf_dim], self._rank(ranks, nid)]
        elif n.kind == TRANSFER:
            ext = [self._rank(ranks, n.successors[0]), self._rank(ranks, n.successors[1]),
                   self._rank(ranks, nid)]
        else:
            ext = [self._rank(ranks, n.successors[0]), self._rank(ranks, n.successors[1]), batch]
        self.node_sets[tuple(nid)] = ext

    def layer_set(self, l):
        return self.layer_sets[l]

    def node_set(self, nid):
        if tuple(nid) not in self.node_sets:
            raise IndexError(f"IndexSet: unknown node {nid}")
        return self.node_sets[tuple(nid)]


# ---------------------------------------------------------------------------
# bht.hpp
# ---------------------------------------------------------------------------

K_MACHINE_FLOOR_REL = 1e-14  # bht.hpp:20


def effective_eps_rel(eps_rel: float) -> float:
    """bht.hpp:22-27."""
    if eps_rel < 0 or eps_rel >= 1.0:
        raise ValueError("relative tolerance must lie in [0, 1)")
    return eps_rel if eps_rel > 0 else K_MACHINE_FLOOR_REL


class HTRepresentation:
    """bht.hpp:34-151. cores[layer][pos] are numpy arrays (Fortran layout)."""

    def __init__(self, tree, dims, cores, accumulated, epsilon_rel):
        self.tree = tree
        self.dims = list(dims)
        self.cores = cores
        self.accumulated = accumulated
        self.epsilon_rel = epsilon_rel

    def copy(self) -> "HTRepresentation":
        return HTRepresentation(self.tree, self.dims, [[c.copy() for c in layer] for layer in self.cores],
                                self.accumulated, self.epsilon_rel)

    def core(self, nid):
        return self.cores[nid[0]][nid[1]]

    def set_core(self, nid, value):
        self.cores[nid[0]][nid[1]] = value

    def root(self):
        return self.cores[0][0]

    def rank(self, nid) -> int:
        n = self.tree.node(nid)
        c = self.core(nid)
        if n.kind == LEAF:
            return c.shape[1]
        if n.kind == TRANSFER:
            return c.shape[2]
        raise ValueError("rank: root has no own rank")

    def ranks(self) -> Dict[Tuple[int, int], int]:
        return {n.id: self.rank(n.id) for l in range(1, self.tree.depth + 1) for n in self.tree.layer(l)}

    def max_rank(self) -> int:
        return max(self.ranks().values(), default=0)

    def basis_matrix(self, nid) -> np.ndarray:
        """bht.hpp:81-86: transfer cores flattened to (r_l*r_r) x r_own."""
        c = self.core(nid)
        if self.tree.node(nid).kind == LEAF:
            return c
        s = c.shape
        return c.reshape(s[0] * s[1], s[2], order="F")

    def stored_elements(self) -> int:
        return sum(c.size for layer in self.cores for c in layer)

    def index_sets(self, batch):
        return IndexSet.build(self.tree, self.dims, self.ranks(), batch)

    def orthonormality_defect(self) -> float:
        """bht.hpp:101-114."""
        worst = 0.0
        for l in range(1, self.tree.depth + 1):
            for n in self.tree.layer(l):
                u = self.basis_matrix(n.id)
                g = u.T @ u
                worst = max(worst, float(np.max(np.abs(g - np.eye(g.shape[0])))) if g.size else 0.0)
        return worst

    def validate(self, tol=1e-10):
        """bht.hpp:116-150."""
        if len(self.dims) != self.tree.dims():
            raise ValueError("HTRepresentation: dims/tree mismatch")
        for layer in self.cores:
            for c in layer:
                if not np.all(np.isfinite(c)):
                    raise RuntimeError("HTRepresentation: non-finite core entries")
        defect = self.orthonormality_defect()
        if not defect <= tol:
            raise RuntimeError(f"HTRepresentation: orthonormality defect {defect} exceeds {tol}")
        r = self.root()
        if r.ndim != 3 or r.shape[2] != self.accumulated:
            raise ValueError("HTRepresentation: root batch extent mismatch")
        sets = self.index_sets(self.accumulated)
        for l in range(self.tree.depth + 1):
            for n in self.tree.layer(l):
                if list(self.core(n.id).shape) != list(sets.node_set(n.id)):
                    raise ValueError("HTRepresentation: core shape inconsistent with its index set")


@dataclass
class NodeRecord:
    id: Tuple[int, int]
    rank: int
    discarded_norm: float


@dataclass
class BuildReport:
    """bht.hpp:170-174."""
    nodes: List[NodeRecord] = field(default_factory=list)
    layer_norms: List[float] = field(default_factory=list)
    eps_nw_initial: float = 0.0


def check_batch_input(y: np.ndarray, tree: DimensionTree, dims, who: str):
    """bht.hpp:187-213."""
    if y.ndim != tree.dims() + 1:
        raise ValueError(f"{who}: tensor order {y.ndim} does not match tree")
    if y.ndim < 3:
        raise ValueError(f"{who}: need d >= 2 plus a batch axis")
    if dims is not None:
        for k in range(tree.dims()):
            if y.shape[k] != dims[k]:
                raise ValueError(f"{who}: shape mismatch at mode {k}")
    if not np.all(np.isfinite(y)):
        raise ValueError(f"{who}: non-finite input")


def svds_below(tree: DimensionTree, l: int) -> int:
    """bht.hpp:216-220."""
    return sum(tree.layer_size(k) for k in range(1, l))


def adaptive_budget(eps_abs: float, achieved_err_sq: float, svd_remaining: int) -> float:
    """bht.hpp:227-245."""
    if svd_remaining < 1:
        raise ValueError("adaptive_budget: no SVDs remaining")
    budget_sq = eps_abs * eps_abs
    rem_sq = budget_sq - achieved_err_sq
    if rem_sq < 0:
        if achieved_err_sq > budget_sq * (1.0 + 1e-9) + 1e-300:
            raise RuntimeError("adaptive_budget: error budget exhausted")
        rem_sq = 0.0
    return math.sqrt(rem_sq) / math.sqrt(float(svd_remaining))


def _layer_extents(tree, l, dims, ranks, batch):
    """bht.hpp:312-321 / 385-395: reshape extents of layer l, batch last."""
    ext = []
    for n in tree.layer(l):
        if n.kind == LEAF:
            ext.append(dims[n.leaf_dim])
        else:
            ext.append(ranks[tuple(n.successors[0])] * ranks[tuple(n.successors[1])])
    ext.append(batch)
    return ext


def bht_l2r(y: np.ndarray, tree: DimensionTree, eps_rel: float, adaptive: bool = False):
    """bht.hpp:251-350 (Alg. 1)."""
    check_batch_input(y, tree, None, "bht_l2r")
    d = tree.dims()
    p = tree.depth
    batch = y.shape[d]
    norm_y = frobenius_norm(y)
    eps_abs = effective_eps_rel(eps_rel) * norm_y
    norm_y_sq = norm_y * norm_y

    report = BuildReport()
    report.eps_nw_initial = eps_abs / math.sqrt(2 * d - 2)
    report.layer_norms.append(norm_y)

    cores = [[None] * tree.layer_size(l) for l in range(p + 1)]
    eps_nw = report.eps_nw_initial
    c = y
    modes = [n.leaf_dim for n in tree.layer(p)]
    bases = hosvd_layer(c, modes, eps_nw)
    for i, b in enumerate(bases):
        n = tree.layer(p)[i]
        cores[p][i] = b.u
        report.nodes.append(NodeRecord(n.id, b.rank, b.discarded_norm))
    for i, b in enumerate(bases):
        c = mode_multiply(c, tree.layer(p)[i].leaf_dim, b.u.T)
    report.layer_norms.append(frobenius_norm(c))

    ranks = {n.id: cores[p][i].shape[1] for i, n in enumerate(tree.layer(p))}
    for l in range(p - 1, 0, -1):
        if adaptive:
            cn = report.layer_norms[-1]
            eps_nw = adaptive_budget(eps_abs, max(0.0, norm_y_sq - cn * cn), svds_below(tree, l + 1))
        c = reshape(c, _layer_extents(tree, l, _dims_of(y, d), ranks, batch))
        bases = hosvd_layer(c, list(range(tree.layer_size(l))), eps_nw)
        for j, b in enumerate(bases):
            n = tree.layer(l)[j]
            if n.kind == LEAF:
                cores[l][j] = b.u
            else:
                cores[l][j] = reshape(b.u, [ranks[n.successors[0]], ranks[n.successors[1]], b.rank])
            ranks[n.id] = b.rank
            report.nodes.append(NodeRecord(n.id, b.rank, b.discarded_norm))
        for j, b in enumerate(bases):
            c = mode_multiply(c, j, b.u.T)
        report.layer_norms.append(frobenius_norm(c))

    rootn = tree.node((0, 0))
    cores[0][0] = reshape(c, [ranks[rootn.successors[0]], ranks[rootn.successors[1]], batch])
    rep = HTRepresentation(tree, _dims_of(y, d), cores, batch, eps_rel)
    return rep, report


def _dims_of(y, d):
    return list(y.shape[:d])


def project_mode(c: np.ndarray, mode: int, basis: np.ndarray, loss: List[float]) -> np.ndarray:
    """bht.hpp:357-365: coefficient GEMM plus explicit residual energy."""
    m = unfold(c, mode)
    coeff = basis.T @ m
    loss[0] += float(np.sum((m - basis @ coeff) ** 2))
    out_shape = list(c.shape)
    out_shape[mode] = coeff.shape[0]
    return fold(coeff, out_shape, mode)


def encode(h: HTRepresentation, y: np.ndarray):
    """bht.hpp:373-401: (latent r11 x r12 x N, projection error)."""
    check_batch_input(y, h.tree, h.dims, "encode")
    p = h.tree.depth
    batch = y.shape[h.tree.dims()]
    loss = [0.0]
    c = y
    for n in h.tree.layer(p):
        c = project_mode(c, n.leaf_dim, h.basis_matrix(n.id), loss)
    ranks = h.ranks()
    for l in range(p - 1, 0, -1):
        c = reshape(c, _layer_extents(h.tree, l, h.dims, ranks, batch))
        for j in range(h.tree.layer_size(l)):
            c = project_mode(c, j, h.basis_matrix((l, j)), loss)
    return c, math.sqrt(loss[0])


def decode(h: HTRepresentation, latent: np.ndarray) -> np.ndarray:
    """bht.hpp:406-456: root-to-leaves reconstruction."""
    root = h.root()
    if latent.ndim != 3 or latent.shape[0] != root.shape[0] or latent.shape[1] != root.shape[1]:
        raise ValueError("decode: latent ranks do not match root")
    rootn = h.tree.node((0, 0))
    tags = [[tuple(rootn.successors[0]), True, -1], [tuple(rootn.successors[1]), True, -1]]
    c = latent
    for l in range(1, h.tree.depth + 1):
        pos = 0
        while pos < len(tags):
            tag = tags[pos]
            if not tag[1] or tag[0][0] != l:
                pos += 1
                continue
            n = h.tree.node(tag[0])
            if n.kind == LEAF:
                c = mode_multiply(c, pos, h.basis_matrix(n.id))
                tag[1] = False
                tag[2] = n.leaf_dim
            else:
                c = contract3_split(c, pos, h.core(n.id))
                tags[pos] = [tuple(n.successors[0]), True, -1]
                tags.insert(pos + 1, [tuple(n.successors[1]), True, -1])
                pos += 1
            pos += 1
    perm = [0] * (len(tags) + 1)
    for k, t in enumerate(tags):
        perm[t[2]] = k
    perm[-1] = len(tags)
    if any(perm[k] > perm[k + 1] for k in range(len(perm) - 1)):
        c = np.transpose(c, perm)
    return c


def pad_latent(latent: np.ndarray, r11: int, r12: int) -> np.ndarray:
    """bht.hpp:460-468."""
    if r11 < latent.shape[0] or r12 < latent.shape[1]:
        raise ValueError("pad_latent: ranks may only grow")
    s = pad_zeros(latent, 0, r11 - latent.shape[0])
    return pad_zeros(s, 1, r12 - s.shape[1])


def reconstruct_slice(h: HTRepresentation, m: int) -> np.ndarray:
    """bht.hpp:472-479 (m is 1-based)."""
    if m < 1 or m > h.accumulated:
        raise IndexError("reconstruct_slice: index outside 1..accumulated")
    one = slice_(h.root(), 2, m - 1, 1)
    return reshape(decode(h, one), h.dims)


# ---------------------------------------------------------------------------
# ht_rise.hpp
# ---------------------------------------------------------------------------

@dataclass
class UpdateReport:
    """ht_rise.hpp:20-27."""
    skipped: bool = False
    proj_error: float = 0.0
    eps_des: float = 0.0
    added_ranks: Dict[Tuple[int, int], int] = field(default_factory=dict)
    new_ranks: Dict[Tuple[int, int], int] = field(default_factory=dict)
    seconds: float = 0.0


def compute_residual(basis: np.ndarray, c_unfolded: np.ndarray) -> np.ndarray:
    """ht_rise.hpp:31-38: R = C - U (U^T C)."""
    if basis.shape[0] != c_unfolded.shape[0]:
        raise ValueError("compute_residual: row mismatch")
    return c_unfolded - basis @ (basis.T @ c_unfolded)


def expand_core(kind: int, core: np.ndarray, u_new: np.ndarray, orth_tol: float = 1e-8) -> np.ndarray:
    """ht_rise.hpp:53-79."""
    if u_new.shape[1] == 0:
        return core
    if kind == ROOT:
        raise ValueError("expand_core: root is not a basis core")
    s = core.shape
    alpha = s[0] if kind == LEAF else s[0] * s[1]
    r_old = s[1] if kind == LEAF else s[2]
    if u_new.shape[0] != alpha:
        raise ValueError("expand_core: row mismatch")
    u_old = core.reshape(alpha, r_old, order="F")
    defect = float(np.linalg.norm(u_old.T @ u_new))
    if defect > orth_tol * max(1.0, float(np.linalg.norm(u_new))):
        raise ValueError(f"expand_core: new directions not orthogonal to existing basis (defect {defect})")
    joined = np.concatenate([u_old, u_new], axis=1)
    if kind == LEAF:
        return joined
    return reshape(joined, [s[0], s[1], r_old + u_new.shape[1]])


def pad_with_zeros(core: np.ndarray, slot: int, r_extra: int) -> np.ndarray:
    """ht_rise.hpp:83-92."""
    if core.ndim != 3:
        raise ValueError("pad_with_zeros: core must be 3-way")
    if slot not in (0, 1):
        raise ValueError("pad_with_zeros: successor slot must be 0 or 1")
    return pad_zeros(core, slot, r_extra)


def ht_rise_update(h: HTRepresentation, y: np.ndarray, epsilon_rel: Optional[float] = None,
                   adaptive: bool = False):
    """ht_rise.hpp:99-186 (Alg. 2). Returns (new representation, report)."""
    t0 = time.perf_counter()
    check_batch_input(y, h.tree, h.dims, "ht_rise_update")
    tree = h.tree
    d = tree.dims()
    p = tree.depth
    batch = y.shape[d]
    eps_rel = effective_eps_rel(h.epsilon_rel if epsilon_rel is None else epsilon_rel)
    norm_y = frobenius_norm(y)

    report = UpdateReport()
    report.eps_des = eps_rel * norm_y
    for nid in h.ranks():
        report.added_ranks[nid] = 0

    def finish(rep):
        report.new_ranks = rep.ranks()
        report.seconds = time.perf_counter() - t0
        return rep, report

    latent, proj_error = encode(h, y)
    report.proj_error = proj_error
    if proj_error <= report.eps_des:
        report.skipped = True
        out = h.copy()
        out.set_core((0, 0), concat(out.root(), latent, 2))
        out.accumulated += batch
        return finish(out)

    out = h.copy()
    ranks = h.ranks()
    sets = IndexSet.build(tree, h.dims, ranks, batch)
    eps_nw = report.eps_des / math.sqrt(2 * d - 2)
    norm_y_sq = norm_y * norm_y
    c = y
    state = {"eps_nw": eps_nw}

    def expand_node(n: TreeNode, c_unf: np.ndarray):
        residual = compute_residual(out.basis_matrix(n.id), c_unf)
        tb = truncated_svd(residual, state["eps_nw"], 0)
        report.added_ranks[n.id] = tb.rank
        if tb.rank == 0:
            return
        out.set_core(n.id, expand_core(n.kind, out.core(n.id), tb.u))
        ranks[n.id] += tb.rank
        sets.update_node(tree, n.id, h.dims, ranks, batch)
        out.set_core(n.parent, pad_with_zeros(out.core(n.parent), tree.parent_slot(n.id), tb.rank))
        sets.update_node(tree, n.parent, h.dims, ranks, batch)

    for n in tree.layer(p):
        expand_node(n, unfold(c, n.leaf_dim))
    for n in tree.layer(p):
        c = mode_multiply(c, n.leaf_dim, out.basis_matrix(n.id).T)
    sets.update_layer(tree, p - 1, h.dims, ranks, batch)

    for l in range(p - 1, 0, -1):
        if adaptive:
            cn = frobenius_norm(c)
            state["eps_nw"] = adaptive_budget(report.eps_des, max(0.0, norm_y_sq - cn * cn),
                                              svds_below(tree, l + 1))
        c = reshape(c, sets.layer_set(l))
        for j in range(tree.layer_size(l)):
            expand_node(tree.layer(l)[j], unfold(c, j))
        for j in range(tree.layer_size(l)):
            c = mode_multiply(c, j, out.basis_matrix((l, j)).T)
        sets.update_layer(tree, l - 1, h.dims, ranks, batch)

    out.set_core((0, 0), concat(out.root(), c, 2))
    out.accumulated += batch
    return finish(out)


# ---------------------------------------------------------------------------
# metrics.hpp (CR / RR only)
# ---------------------------------------------------------------------------

def compression_ratio(h: HTRepresentation) -> float:
    """metrics.hpp:200-207."""
    if h.accumulated < 1:
        raise ValueError("compression_ratio: empty accumulation")
    return float(np.prod(h.dims)) * float(h.accumulated) / float(h.stored_elements())


def reduction_ratio(h: HTRepresentation) -> float:
    """metrics.hpp:210-214."""
    r = h.root()
    return float(np.prod(h.dims)) / float(r.shape[0] * r.shape[1])


def relative_test_error(h: HTRepresentation, test_set) -> float:
    """metrics.hpp:218-237: mean over the set of ||y - decode(encode(y))|| / ||y||;
    an order-d tensor gains a unit batch axis (224-226); zero tensors add 0
    but still count in the mean (230-231)."""
    test_set = list(test_set)
    if not test_set:
        raise ValueError("relative_test_error: empty test set")
    total = 0.0
    for t in test_set:
        y = t.reshape(t.shape + (1,), order="F") if t.ndim == h.tree.dims() else t
        back = decode(h, encode(h, y)[0])
        ny = float(np.linalg.norm(y))
        if ny == 0.0:
            continue
        total += float(np.linalg.norm(y - back)) / ny
    return total / len(test_set)
