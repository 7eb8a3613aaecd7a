"""BHTB batch and HTRS state containers (reference
/root/reference/proj/include/htrise/io.hpp: constants 23-25, UnitRecord 29-36,
RepresentationState 40-44, container layout 166-180, write_batch 208-217,
read_batch_file 224-239, write_state 249-299, read_state 301-387,
write/read_representation 390-396). Python twin of include/htrise/io.hpp:
the two write identical bytes (tests/test_io_containers.py).

Layout: magic (4 bytes), u16 format version, u32 header length, compact JSON
header, little-endian f64 payload. The header JSON follows the reference's
serialiser (nlohmann::json `dump()`): sorted keys, no whitespace, doubles in
shortest round-trip digits laid out in decimal when the decimal point sits
within (-4, 15] digits of the first digit and as d.ddde+XX otherwise
(nlohmann prints Grisu2 digits, which differ from the shortest ones in the
last place for ~0.1% of arbitrary doubles; both parse to the same value).

A device-resident representation is exported exactly (cores copied from
HBM) and `read_state` re-imports the cores bit for bit, so resuming a stream
from a state file reproduces the uninterrupted run exactly.
"""
from __future__ import annotations

import json as _json
import os
import struct
from dataclasses import dataclass, field
from decimal import Decimal
from typing import Any, Dict, List, Optional, Tuple

import numpy as np

FORMAT_VERSION = 1
BATCH_MAGIC = b"BHTB"
STATE_MAGIC = b"HTRS"
NORMALIZATION_METHODS = ("none", "maxabs", "unitvec", "zscore")
_KIND_NAMES = {0: "root", 1: "transfer", 2: "leaf"}  # NodeKind (dimension_tree.hpp:14)
_KIND_IDS = {v: k for k, v in _KIND_NAMES.items()}


# ---------------------------------------------------------------------------
# header JSON in the reference serialiser's layout
# ---------------------------------------------------------------------------

def _dump_float(x: float) -> str:
    if x != x or x in (float("inf"), float("-inf")):
        return "null"
    if x == 0.0:
        return "-0.0" if str(x).startswith("-") else "0.0"
    sign = "-" if x < 0 else ""
    dec = Decimal(repr(abs(x))).normalize()  # shortest round-trip digits
    _, digit_tuple, exp = dec.as_tuple()
    digits = "".join(str(d) for d in digit_tuple)
    k = len(digits)
    n = k + exp  # decimal point position relative to the first digit
    if k <= n <= 15:
        return sign + digits + "0" * (n - k) + ".0"
    if 0 < n <= 15:
        return sign + digits[:n] + "." + digits[n:]
    if -4 < n <= 0:
        return sign + "0." + "0" * (-n) + digits
    e = n - 1
    mant = digits[0] + ("." + digits[1:] if k > 1 else "")
    return f"{sign}{mant}e{'-' if e < 0 else '+'}{abs(e):02d}"


def _dump_string(s: str) -> str:
    out = ['"']
    for ch in s:
        o = ord(ch)
        if ch == '"':
            out.append('\\"')
        elif ch == "\\":
            out.append("\\\\")
        elif ch == "\b":
            out.append("\\b")
        elif ch == "\f":
            out.append("\\f")
        elif ch == "\n":
            out.append("\\n")
        elif ch == "\r":
            out.append("\\r")
        elif ch == "\t":
            out.append("\\t")
        elif o < 0x20:
            out.append(f"\\u{o:04x}")
        else:
            out.append(ch)
    out.append('"')
    return "".join(out)


def dump_json(v: Any) -> str:
    """Compact JSON with sorted keys, byte-compatible with the reference."""
    if v is None:
        return "null"
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    if isinstance(v, (float, np.floating)):
        return _dump_float(float(v))
    if isinstance(v, str):
        return _dump_string(v)
    if isinstance(v, dict):
        return "{" + ",".join(_dump_string(k) + ":" + dump_json(v[k]) for k in sorted(v)) + "}"
    if isinstance(v, (list, tuple)):
        return "[" + ",".join(dump_json(x) for x in v) + "]"
    raise TypeError(f"dump_json: unsupported {type(v).__name__}")


# ---------------------------------------------------------------------------
# containers
# ---------------------------------------------------------------------------

def _container(magic: bytes, header: dict, payload: List[np.ndarray]) -> bytes:
    h = dump_json(header).encode("utf-8")
    parts = [magic, struct.pack("<HI", FORMAT_VERSION, len(h)), h]
    for t in payload:
        parts.append(np.asarray(t, dtype="<f8").ravel(order="F").tobytes())
    return b"".join(parts)


def _publish(path: str, data: bytes) -> None:
    """Atomic publication: a sibling temporary, then rename."""
    tmp = path + ".tmp"
    try:
        with open(tmp, "wb") as f:
            f.write(data)
    except OSError as e:
        raise RuntimeError(f"{tmp}: cannot open for writing") from e
    os.replace(tmp, path)


class _Reader:
    def __init__(self, path: str, magic: bytes):
        self.path = path
        try:
            with open(path, "rb") as f:
                self.buf = f.read()
        except OSError as e:
            raise RuntimeError(f"{path}: cannot open") from e
        if len(self.buf) < 10:
            raise RuntimeError(f"{path}: truncated header")
        if self.buf[:4] != magic:
            raise RuntimeError(f"{path}: bad magic")
        version, hlen = struct.unpack_from("<HI", self.buf, 4)
        if version > FORMAT_VERSION:
            raise RuntimeError(f"{path}: unsupported format version {version}")
        self.pos = 10
        if len(self.buf) - self.pos < hlen:
            raise RuntimeError(f"{path}: truncated header")
        try:
            self.header = _json.loads(self.buf[self.pos:self.pos + hlen].decode("utf-8"))
        except (ValueError, UnicodeDecodeError) as e:
            raise RuntimeError(f"{path}: corrupt header: {e}") from e
        self.pos += hlen

    def payload(self, shape) -> np.ndarray:
        n = int(np.prod(shape, dtype=np.int64)) if len(shape) else 1
        if n < 0 or (len(self.buf) - self.pos) // 8 < n:
            raise RuntimeError(f"{self.path}: truncated payload")
        a = np.frombuffer(self.buf, dtype="<f8", count=n, offset=self.pos).astype(np.float64)
        self.pos += 8 * n
        return a.reshape(tuple(shape), order="F")

    def expect_end(self) -> None:
        if self.pos != len(self.buf):
            raise RuntimeError(f"{self.path}: trailing bytes after payload")


# ---------------------------------------------------------------------------
# normalisation ledger records (metrics.hpp:38-46)
# ---------------------------------------------------------------------------

@dataclass
class NormalizationParams:
    method: str = "none"
    field_axis: Optional[int] = None
    scale: List[float] = field(default_factory=list)
    offset: List[float] = field(default_factory=list)
    floored: List[bool] = field(default_factory=list)

    def to_json(self) -> dict:
        if self.method not in NORMALIZATION_METHODS:
            raise ValueError(f"unknown normalization method: {self.method}")
        j = {"method": self.method, "scale": [float(x) for x in self.scale],
             "offset": [float(x) for x in self.offset], "floored": [1 if b else 0 for b in self.floored]}
        if self.field_axis is not None:
            j["field_axis"] = int(self.field_axis)
        return j

    @staticmethod
    def from_json(j: dict) -> "NormalizationParams":
        m = j["method"]
        if m not in NORMALIZATION_METHODS:
            raise ValueError(f"unknown normalization method: {m}")
        return NormalizationParams(m, int(j["field_axis"]) if "field_axis" in j else None,
                                   [float(x) for x in j["scale"]], [float(x) for x in j["offset"]],
                                   [int(b) != 0 for b in j["floored"]])


@dataclass
class UnitRecord:
    first: int
    count: int
    source: str
    norm: NormalizationParams


@dataclass
class HostRepresentation:
    """A representation held as host arrays (what a state file stores)."""
    tree: Any
    dims: List[int]
    cores: Dict[Tuple[int, int], np.ndarray]
    accumulated: int
    epsilon_rel: float

    def core(self, nid) -> np.ndarray:
        return self.cores[(int(nid[0]), int(nid[1]))]


@dataclass
class RepresentationState:
    rep: Any
    units: List[UnitRecord] = field(default_factory=list)
    batches_processed: int = 0


# ---------------------------------------------------------------------------
# batches
# ---------------------------------------------------------------------------

def write_batch(t, path: str, normalization: Optional[NormalizationParams] = None) -> None:
    """Batch container (io.hpp:208-217): canonical (first-index-fastest) f64,
    batch axis last."""
    a = np.asarray(t, dtype=np.float64)
    header = {"dtype": "f64", "layout": "first-fastest", "shape": [int(x) for x in a.shape]}
    if normalization is not None:
        header["normalization"] = normalization.to_json()
    _publish(path, _container(BATCH_MAGIC, header, [a]))


def read_batch_file(path: str) -> Tuple[np.ndarray, Optional[NormalizationParams]]:
    r = _Reader(path, BATCH_MAGIC)
    h = r.header
    try:
        if h["dtype"] != "f64" or h["layout"] != "first-fastest":
            raise RuntimeError(f"{path}: unsupported dtype or layout")
        t = r.payload([int(x) for x in h["shape"]])
        r.expect_end()
        norm = NormalizationParams.from_json(h["normalization"]) if "normalization" in h else None
    except (KeyError, TypeError, ValueError) as e:
        raise RuntimeError(f"{path}: corrupt header: {e}") from e
    return t, norm


def read_batch(path: str) -> np.ndarray:
    return read_batch_file(path)[0]


# ---------------------------------------------------------------------------
# states
# ---------------------------------------------------------------------------

def _validate_host(rep: HostRepresentation, tol: float = 1e-10) -> None:
    """HTRepresentation::validate (bht.hpp:116-150) on host cores."""
    tree = rep.tree
    if len(rep.dims) != tree.dims():
        raise ValueError("HTRepresentation: dims/tree mismatch")
    for l in range(tree.depth + 1):
        for n in tree.layer(l):
            if not np.all(np.isfinite(rep.core(n.id))):
                raise RuntimeError("HTRepresentation: non-finite core entries")
    worst = 0.0
    for l in range(1, tree.depth + 1):
        for n in tree.layer(l):
            c = rep.core(n.id)
            u = c if n.kind == _KIND_IDS["leaf"] else c.reshape(c.shape[0] * c.shape[1], c.shape[2], order="F")
            with np.errstate(over="ignore", invalid="ignore"):
                g = u.T @ u
                d = float(np.max(np.abs(g - np.eye(g.shape[0])))) if g.size else 0.0
            worst = max(worst, d if d == d else float("inf"))
    if not worst <= tol:
        raise RuntimeError(f"HTRepresentation: orthonormality defect {worst} exceeds {tol}")
    root = rep.core((0, 0))
    if root.ndim != 3 or root.shape[2] != rep.accumulated:
        raise ValueError("HTRepresentation: root batch extent mismatch")


def write_state(state: RepresentationState, path: str) -> None:
    """io.hpp:249-299. `state.rep` is a device HTRepresentation or a
    HostRepresentation; invariants are checked before the file is written."""
    rep = state.rep
    if hasattr(rep, "validate"):
        rep.validate()
    else:
        _validate_host(rep)
    tree = rep.tree
    nodes, shapes, payload = [], [], []
    for l in range(tree.depth + 1):
        for n in tree.layer(l):
            kind = _KIND_NAMES[int(n.kind)]
            jn = {"layer": int(n.id[0]), "pos": int(n.id[1]), "kind": kind}
            if kind == "leaf":
                jn["leaf_dim"] = int(n.leaf_dim)
            else:
                jn["successors"] = [[int(s[0]), int(s[1])] for s in n.successors]
            if kind != "root":
                jn["parent"] = [int(n.parent[0]), int(n.parent[1])]
            nodes.append(jn)
            c = np.asarray(rep.core(n.id), dtype=np.float64)
            shapes.append([int(x) for x in c.shape])
            payload.append(c)
    header = {
        "dims": [int(x) for x in rep.dims],
        "epsilon_rel": float(rep.epsilon_rel),
        "accumulated": int(rep.accumulated),
        "batches_processed": int(state.batches_processed),
        "tree": {"d": int(tree.dims()), "nodes": nodes},
        "core_shapes": shapes,
        "units": [{"first": int(u.first), "count": int(u.count), "source": u.source, "norm": u.norm.to_json()}
                  for u in state.units],
    }
    _publish(path, _container(STATE_MAGIC, header, payload))


def read_state(path: str, device: bool = True, ctx=None) -> RepresentationState:
    """io.hpp:301-387. With `device` the representation is re-imported into
    HBM (bit-exact cores); otherwise a HostRepresentation is returned."""
    from . import htrise as ht

    r = _Reader(path, STATE_MAGIC)
    h = r.header
    try:
        jtree = h["tree"]
        layers: List[List[ht.TreeNode]] = []
        for jn in jtree["nodes"]:
            nid = (int(jn["layer"]), int(jn["pos"]))
            kind = jn["kind"]
            if kind not in _KIND_IDS:
                raise RuntimeError(f"{path}: unknown node kind {kind}")
            succ = [] if kind == "leaf" else [(int(s[0]), int(s[1])) for s in jn["successors"]]
            leaf_dim = int(jn["leaf_dim"]) if kind == "leaf" else -1
            if nid[0] < 0 or nid[1] < 0:
                raise RuntimeError(f"{path}: node records out of order")
            while len(layers) <= nid[0]:
                layers.append([])
            if len(layers[nid[0]]) != nid[1]:
                raise RuntimeError(f"{path}: node records out of order")
            layers[nid[0]].append(ht.TreeNode(nid, _KIND_IDS[kind], succ, (0, 0), leaf_dim))
        try:
            tree = ht.DimensionTree.from_layers(layers)
        except ValueError as e:
            raise RuntimeError(f"{path}: corrupt tree: {e}") from e
        if tree.dims() != int(jtree["d"]):
            raise RuntimeError(f"{path}: tree dimension mismatch")
        for jn in jtree["nodes"]:
            nid = (int(jn["layer"]), int(jn["pos"]))
            if nid[0] > 0 and tuple(tree.node(nid).parent) != (int(jn["parent"][0]), int(jn["parent"][1])):
                raise RuntimeError(f"{path}: corrupt parent link at node ({nid[0]},{nid[1]})")
        dims = [int(x) for x in h["dims"]]
        eps = float(h["epsilon_rel"])
        acc = int(h["accumulated"])
        batches = int(h["batches_processed"])
        shapes = h["core_shapes"]
        cores: Dict[Tuple[int, int], np.ndarray] = {}
        k = 0
        for l in range(tree.depth + 1):
            for n in tree.layer(l):
                cores[n.id] = r.payload([int(x) for x in shapes[k]])
                k += 1
        r.expect_end()
        units = [UnitRecord(int(u["first"]), int(u["count"]), str(u["source"]), NormalizationParams.from_json(u["norm"]))
                 for u in h["units"]]
    except (KeyError, TypeError, IndexError) as e:
        raise RuntimeError(f"{path}: corrupt header: {e}") from e
    host = HostRepresentation(tree, dims, cores, acc, eps)
    try:
        _validate_host(host)
    except (ValueError, RuntimeError) as e:
        raise RuntimeError(f"{path}: corrupt representation: {e}") from e
    rep = host
    if device:
        rep = ht.HTRepresentation.from_cores(tree, dims, cores, acc, eps, ctx)
    return RepresentationState(rep, units, batches)


def write_representation(rep, path: str) -> None:
    write_state(RepresentationState(rep, [], 0), path)


def read_representation(path: str, device: bool = True, ctx=None):
    return read_state(path, device, ctx).rep
