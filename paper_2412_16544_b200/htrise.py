"""Python mirror of the reference's htrise API, bound to libhtrise_cuda.so.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/htrise/*.hpp):

==========================  ==================================================
reference                   here (all compute runs in sm_100a kernels)
==========================  ==================================================
DimensionTree::balanced      DimensionTree.balanced        (dimension_tree.hpp:44)
DimensionTree::from_layers   DimensionTree.from_layers     (dimension_tree.hpp:99)
bht_l2r                      bht_l2r                       (bht.hpp:251)
encode / decode              encode / decode               (bht.hpp:373, 406)
pad_latent                   pad_latent                    (bht.hpp:460)
reconstruct_slice            reconstruct_slice             (bht.hpp:472)
ht_rise_update               ht_rise_update                (ht_rise.hpp:99)
compute_residual             compute_residual              (ht_rise.hpp:31)
truncated_svd                truncated_svd                 (truncated_svd.hpp:53)
mode_multiply                mode_multiply                 (tensor.hpp:300)
frobenius_norm               frobenius_norm                (tensor.hpp:269)
compression/reduction_ratio  compression_ratio / reduction_ratio (metrics.hpp:200-214)
==========================  ==================================================

Exceptions: std::invalid_argument -> ValueError, std::out_of_range ->
IndexError, std::runtime_error -> RuntimeError (status codes of the C-ABI).

Host tensors are numpy arrays in the reference's canonical order (first
index fastest = numpy Fortran order); device tensors are passed as
``DeviceTensor(torch_cuda_float64_tensor, canonical_shape)``. There is no CPU
fallback: if the CUDA library or a device is missing every call raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from collections.abc import Sequence as _SequenceABC
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

ROOT, TRANSFER, LEAF = 0, 1, 2  # NodeKind (dimension_tree.hpp:14)
MAX_NODES = 256
MAX_LAYERS = 16

OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_OUT_OF_RANGE = 2
ERR_RUNTIME = 3
ERR_CUDA = 4
ERR_NO_DEVICE = 5

OPT_EXACT_LOSS = 1
OPT_FUSED_ENCODE = 2
OPT_PROFILE_EVENTS = 3
OPT_TAIL_KERNEL = 4
OPT_EIG_SOLVER = 5

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhtrise_cuda.so")


class CudaError(RuntimeError):
    pass


class NoDeviceError(RuntimeError):
    pass


class _Node(C.Structure):
    _fields_ = [("layer", C.c_int32), ("pos", C.c_int32), ("kind", C.c_int32),
                ("leaf_dim", C.c_int32), ("succ0", C.c_int32), ("succ1", C.c_int32)]


class _BuildReport(C.Structure):
    _fields_ = [("eps_nw_initial", C.c_double), ("n_records", C.c_int32),
                ("rec_layer", C.c_int32 * MAX_NODES), ("rec_pos", C.c_int32 * MAX_NODES),
                ("rec_rank", C.c_int64 * MAX_NODES), ("rec_discarded", C.c_double * MAX_NODES),
                ("n_layer_norms", C.c_int32), ("layer_norms", C.c_double * MAX_LAYERS)]


class _UpdateReport(C.Structure):
    _fields_ = [("skipped", C.c_int32), ("proj_error", C.c_double), ("eps_des", C.c_double),
                ("seconds", C.c_double), ("n_nodes", C.c_int32),
                ("node_layer", C.c_int32 * MAX_NODES), ("node_pos", C.c_int32 * MAX_NODES),
                ("added_ranks", C.c_int64 * MAX_NODES), ("new_ranks", C.c_int64 * MAX_NODES),
                ("used_fused_path", C.c_int32), ("used_exact_loss", C.c_int32),
                ("kernel_launches", C.c_int64)]


_lib_handle = None

_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)

# htr_host_reduce_fn: int32 (*)(double* buf, int64 n, void* user)
_REDUCE_FN = C.CFUNCTYPE(C.c_int32, _D, C.c_int64, _P)

_SIGNATURES = {
    "htr_context_create": (C.c_int32, [C.c_int32, C.POINTER(_P)]),
    "htr_context_destroy": (C.c_int32, [_P]),
    "htr_last_error": (C.c_char_p, [_P]),
    "htr_context_stream": (C.c_int32, [_P, C.POINTER(_P)]),
    "htr_context_wait_stream": (C.c_int32, [_P, _P]),
    "htr_synchronize": (C.c_int32, [_P]),
    "htr_context_set_option": (C.c_int32, [_P, C.c_int32, C.c_double]),
    "htr_context_launch_count": (C.c_int64, [_P]),
    "htr_context_kernel_timing": (C.c_int32, [_P, _D, _I64, _D, _I64]),
    "htr_context_reset_timing": (C.c_int32, [_P]),
    "htr_comm_get_unique_id": (C.c_int32, [C.POINTER(C.c_uint8)]),
    "htr_context_init_comm": (C.c_int32, [_P, C.POINTER(C.c_uint8), C.c_int32, C.c_int32]),
    "htr_context_set_reducer": (C.c_int32, [_P, _REDUCE_FN, _P, C.c_int32, C.c_int32]),
    "htr_tree_balanced": (C.c_int32, [C.c_int64, C.POINTER(_Node), C.c_int64, _I64, C.c_char_p, C.c_int64]),
    "htr_tree_validate": (C.c_int32, [C.POINTER(_Node), C.c_int64, C.c_char_p, C.c_int64]),
    "htr_bht_l2r": (C.c_int32, [_P, _D, C.c_int32, _I64, C.c_int32, C.POINTER(_Node), C.c_int64, C.c_double,
                                C.c_int32, C.POINTER(_P), C.POINTER(_BuildReport)]),
    "htr_ht_rise_update": (C.c_int32, [_P, _P, _D, C.c_int32, _I64, C.c_int32, C.c_double, C.c_int32,
                                       C.POINTER(_P), C.POINTER(_UpdateReport)]),
    "htr_ht_rise_update_many": (C.c_int32, [_P, _P, C.c_int64, C.POINTER(_P), C.c_int32, _I64, C.c_int32,
                                            C.c_double, C.c_int32, C.POINTER(_P), C.POINTER(_UpdateReport)]),
    "htr_encode": (C.c_int32, [_P, _P, _D, C.c_int32, _I64, C.c_int32, _D, C.c_int32, _D]),
    "htr_decode": (C.c_int32, [_P, _P, _D, C.c_int32, _I64, _D, C.c_int32]),
    "htr_reconstruct_slice": (C.c_int32, [_P, _P, C.c_int64, _D, C.c_int32]),
    "htr_relative_error": (C.c_int32, [_P, _P, _D, C.c_int32, _I64, C.c_int32, _D]),
    "htr_rep_free": (C.c_int32, [_P]),
    "htr_rep_clone": (C.c_int32, [_P, _P, C.POINTER(_P)]),
    "htr_rep_info": (C.c_int32, [_P, C.POINTER(C.c_int32), _I64, _I64, _D, _I64]),
    "htr_rep_nodes": (C.c_int32, [_P, C.POINTER(_Node), C.c_int64]),
    "htr_rep_counts": (C.c_int32, [_P, _I64, _I64]),
    "htr_rep_core_shape": (C.c_int32, [_P, C.c_int32, C.c_int32, _I64, C.POINTER(C.c_int32)]),
    "htr_rep_core_get": (C.c_int32, [_P, _P, C.c_int32, C.c_int32, _D, C.c_int32]),
    "htr_rep_import": (C.c_int32, [_P, C.POINTER(_Node), C.c_int64, _I64, C.c_int32, C.POINTER(_D), _I64,
                                   C.c_int64, C.c_double, C.POINTER(_P)]),
    "htr_rep_reserve": (C.c_int32, [_P, _P, C.c_int64]),
    "htr_truncated_svd": (C.c_int32, [_P, _D, C.c_int32, C.c_int64, C.c_int64, C.c_double, C.c_int64, _D, _D,
                                      _I64, _D]),
    "htr_mode_multiply": (C.c_int32, [_P, _D, C.c_int32, _I64, C.c_int32, C.c_int32, _D, C.c_int64, _D,
                                      C.c_int32]),
    "htr_compute_residual": (C.c_int32, [_P, _D, C.c_int64, C.c_int64, _D, C.c_int64, _D]),
    "htr_frobenius_norm": (C.c_int32, [_P, _D, C.c_int32, C.c_int64, _D]),
    "htr_matmul": (C.c_int32, [_P, _D, C.c_int64, C.c_int64, _D, C.c_int64, _D]),
    "htr_contract": (C.c_int32, [_P, _D, _I64, C.c_int32, C.c_int32, _D, _I64, C.c_int32, C.c_int32, _D]),
    "htr_permute_axes": (C.c_int32, [_P, _D, _I64, C.c_int32, _I64, _D]),
    "htr_device_alloc": (C.c_int32, [_P, C.c_int64, C.POINTER(_D)]),
    "htr_device_free": (C.c_int32, [_P, _D]),
    "htr_copy": (C.c_int32, [_P, _D, C.c_int32, _D, C.c_int32, C.c_int64]),
    "htr_normalize": (C.c_int32, [_P, _D, C.c_int32, _I64, C.c_int32, C.c_int32, C.c_int32, _D, C.c_int32, _D, _D,
                                  C.POINTER(C.c_int32)]),
    "htr_denormalize": (C.c_int32, [_P, _D, C.c_int32, _I64, C.c_int32, C.c_int32, C.c_int32, _D, _D, _D,
                                    C.c_int32]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)


def library_path() -> str:
    return _LIB_PATH


class _Fns:
    """Bound foreign functions of the hot calls (attribute lookups cached)."""

    def __getattr__(self, name):
        f = getattr(lib(), "htr_" + name)
        setattr(self, name, f)
        return f


_fn = _Fns()


def lib():
    """Load libhtrise_cuda.so (fails loudly: there is no fallback path)."""
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"htrise-b200 CUDA library missing at {_LIB_PATH}; run __graft_entry__.build()")
        h = C.CDLL(_LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib_handle = h
    return _lib_handle


def _raise(code: int, msg: str):
    if code == ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if code == ERR_OUT_OF_RANGE:
        raise IndexError(msg)
    if code == ERR_CUDA:
        raise CudaError(msg)
    if code == ERR_NO_DEVICE:
        raise NoDeviceError(msg)
    raise RuntimeError(msg)


# ---------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------

class Context:
    """One device, one CUDA stream (htr_context)."""

    def __init__(self, device: int = 0):
        self._h = _P()
        code = lib().htr_context_create(device, C.byref(self._h))
        if code != OK:
            msg = lib().htr_last_error(self._h).decode()
            lib().htr_context_destroy(self._h)
            self._h = None
            _raise(code, msg)
        self.device = device
        self.world = 1
        self._update_report = _UpdateReport()

    def check(self, code: int):
        if code != OK:
            _raise(code, lib().htr_last_error(self._h).decode())

    @property
    def handle(self):
        return self._h

    def set_option(self, option: int, value: float):
        self.check(lib().htr_context_set_option(self._h, option, float(value)))

    def stream(self) -> int:
        s = _P()
        self.check(lib().htr_context_stream(self._h, C.byref(s)))
        return s.value or 0

    def synchronize(self):
        self.check(lib().htr_synchronize(self._h))

    def launch_count(self) -> int:
        return int(lib().htr_context_launch_count(self._h))

    def kernel_timing(self):
        fm, gm = C.c_double(), C.c_double()
        fc, gc = C.c_int64(), C.c_int64()
        self.check(lib().htr_context_kernel_timing(self._h, C.byref(fm), C.byref(fc), C.byref(gm), C.byref(gc)))
        return fm.value, fc.value, gm.value, gc.value

    def reset_timing(self):
        self.check(lib().htr_context_reset_timing(self._h))

    def init_comm(self, unique_id: bytes, nranks: int, rank: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        self.check(lib().htr_context_init_comm(self._h, buf, nranks, rank))
        self.world = nranks

    def set_reducer(self, reduce, nranks: int, rank: int):
        """Host-staged collective instead of NCCL (htr_context_set_reducer):
        ``reduce(array)`` must sum the float64 numpy array in place over all
        ranks (e.g. ``torch.distributed.all_reduce`` on a gloo group). The
        library hands it drained, pinned partial sums, so ranks never wait on
        one another's kernels."""

        self._reduce_cb = host_reduce_callback(reduce)  # kept alive with the context
        self.check(lib().htr_context_set_reducer(self._h, self._reduce_cb, None, int(nranks), int(rank)))
        self.world = nranks

    def close(self):
        if self._h:
            lib().htr_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def host_reduce_callback(reduce):
    """C callback (htr_host_reduce_fn) around ``reduce(array)``, which sums a
    float64 numpy view of the library's pinned buffer in place over all
    ranks. Exceptions become a non-zero status (the library then raises)."""

    def cb(buf, n, _user):
        try:
            if n > 0:
                reduce(np.ctypeslib.as_array(buf, shape=(int(n),)))
            return 0
        except Exception:  # noqa: BLE001 - reported as a runtime error by the library
            import traceback

            traceback.print_exc()
            return 1

    return _REDUCE_FN(cb)


def gloo_reducer(group=None):
    """``reduce`` for Context.set_reducer over a torch.distributed group
    (gloo on the host): an element-wise sum, the same bits on every rank."""
    import torch
    import torch.distributed as dist

    def reduce(a: np.ndarray):
        t = torch.from_numpy(a)  # shares the pinned buffer
        dist.all_reduce(t, group=group)

    return reduce


def comm_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    code = lib().htr_comm_get_unique_id(buf)
    if code != OK:
        _raise(code, "ncclGetUniqueId failed")
    return bytes(buf)


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def set_default_context(ctx: Context):
    global _default_ctx
    _default_ctx = ctx


# ---------------------------------------------------------------------------
# tensors
# ---------------------------------------------------------------------------

@dataclass
class DeviceTensor:
    """A contiguous float64 CUDA buffer (e.g. a torch tensor) read in the
    canonical first-index-fastest order with extents `shape`."""
    data: object
    shape: Tuple[int, ...]

    def ptr(self) -> int:
        d = self.data
        if hasattr(d, "data_ptr"):
            if d.dtype is not _torch_f64():
                raise ValueError("DeviceTensor: float64 storage required")
            if not d.is_contiguous():
                raise ValueError("DeviceTensor: contiguous storage required")
            if d.numel() != math.prod(self.shape):
                raise ValueError("DeviceTensor: element count does not match shape")
            return int(d.data_ptr())
        return int(d)


def _as_host(t) -> np.ndarray:
    a = np.asarray(t, dtype=np.float64)
    return np.asfortranarray(a)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _shape_arr(shape):
    return (C.c_int64 * len(shape))(*[int(s) for s in shape])


_torch_cache = {}


def _torch_f64():
    f = _torch_cache.get("f64")
    if f is None:
        import torch

        f = _torch_cache["f64"] = torch.float64
    return f


def _torch_stream(t) -> int:
    """Raw handle of torch's current stream on t's device."""
    raw = _torch_cache.get("raw")
    if raw is None:
        import torch

        raw = _torch_cache["raw"] = getattr(torch._C, "_cuda_getCurrentRawStream", None) or (
            lambda idx: torch.cuda.current_stream(idx).cuda_stream)
    return int(raw(t.get_device()))


def _tensor_arg(y, ctx: Optional["Context"] = None):
    """-> (pointer, on_device, shape, keepalive). Device inputs produced on
    torch's current stream are ordered before the library's stream."""
    if isinstance(y, DeviceTensor):
        if ctx is not None and hasattr(y.data, "data_ptr"):
            code = _fn.context_wait_stream(ctx._h, _torch_stream(y.data))
            if code:
                ctx.check(code)
        return C.cast(y.ptr(), _D), 1, tuple(map(int, y.shape)), y
    a = _as_host(y)
    if a.ndim == 0:
        a = a.reshape(1)
    return _ptr(a), 0, a.shape, a


# ---------------------------------------------------------------------------
# dimension tree (host metadata; validation runs in the C++ library)
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
    def __init__(self, nodes: Sequence[_Node]):
        self._nodes = list(nodes)
        depth = max(n.layer for n in self._nodes)
        self.layers: List[List[TreeNode]] = [[] for _ in range(depth + 1)]
        for n in sorted(self._nodes, key=lambda x: (x.layer, x.pos)):
            succ = [] if n.succ0 < 0 else [(n.layer + 1, n.succ0), (n.layer + 1, n.succ1)]
            self.layers[n.layer].append(TreeNode((n.layer, n.pos), n.kind, succ, (0, 0), n.leaf_dim))
        for layer in self.layers:
            for n in layer:
                for s in n.successors:
                    self.layers[s[0]][s[1]].parent = n.id
        self.depth = depth
        self.d = sum(1 for layer in self.layers for n in layer if n.kind == LEAF)

    @staticmethod
    def balanced(d: int) -> "DimensionTree":
        buf = (_Node * MAX_NODES)()
        n = C.c_int64()
        err = C.create_string_buffer(512)
        code = lib().htr_tree_balanced(int(d), buf, MAX_NODES, C.byref(n), err, 512)
        if code != OK:
            _raise(code, err.value.decode())
        return DimensionTree(buf[: n.value])

    @staticmethod
    def from_layers(layers) -> "DimensionTree":
        nodes = []
        for layer in layers:
            for t in layer:
                s0 = t.successors[0][1] if t.successors else -1
                s1 = t.successors[1][1] if t.successors else -1
                if t.successors and (t.successors[0][0] != t.id[0] + 1 or t.successors[1][0] != t.id[0] + 1):
                    raise ValueError(f"DimensionTree: successors of {t.id} must be adjacent, ordered, and one layer down")
                nodes.append(_Node(t.id[0], t.id[1], t.kind, t.leaf_dim, s0, s1))
        arr = (_Node * max(1, len(nodes)))(*nodes)
        err = C.create_string_buffer(512)
        code = lib().htr_tree_validate(arr, len(nodes), err, 512)
        if code != OK:
            _raise(code, err.value.decode())
        return DimensionTree(nodes)

    def c_nodes(self):
        arr = (_Node * len(self._nodes))(*self._nodes)
        return arr, len(self._nodes)

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
        n = self.node(nid)
        if n.kind == ROOT:
            raise ValueError("parent_slot: root has no parent")
        return 0 if tuple(self.node(n.parent).successors[0]) == tuple(nid) else 1

    def span(self, nid):
        n = self.node(nid)
        if n.kind == LEAF:
            return n.leaf_dim, n.leaf_dim
        return self.span(n.successors[0])[0], self.span(n.successors[1])[1]


def tree_1_23() -> DimensionTree:
    """The custom (1,(2,3)) tree of configs 2 and 5 (test_bht.cpp:246-252)."""
    layers = [
        [TreeNode((0, 0), ROOT, [(1, 0), (1, 1)])],
        [TreeNode((1, 0), LEAF, [], (0, 0), 0), TreeNode((1, 1), TRANSFER, [(2, 0), (2, 1)])],
        [TreeNode((2, 0), LEAF, [], (0, 0), 1), TreeNode((2, 1), LEAF, [], (0, 0), 2)],
    ]
    return DimensionTree.from_layers(layers)


# ---------------------------------------------------------------------------
# representation
# ---------------------------------------------------------------------------

@dataclass
class NodeRecord:
    id: Tuple[int, int]
    rank: int
    discarded_norm: float


@dataclass
class BuildReport:
    """bht.hpp:170-174."""
    nodes: List[NodeRecord]
    layer_norms: List[float]
    eps_nw_initial: float


@dataclass
class UpdateReport:
    """ht_rise.hpp:20-27 (+ device accounting)."""
    skipped: bool
    proj_error: float
    eps_des: float
    added_ranks: Dict[Tuple[int, int], int]
    new_ranks: Dict[Tuple[int, int], int]
    seconds: float
    used_fused_path: bool = False
    used_exact_loss: bool = False
    kernel_launches: int = 0


class HTRepresentation:
    """Device-resident batch-HT value (bht.hpp:34-151). Updates return new
    values; cores are fetched to host lazily for inspection."""

    def __init__(self, handle, ctx: Context, tree: Optional[DimensionTree] = None,
                 dims: Optional[List[int]] = None, accumulated: Optional[int] = None,
                 epsilon_rel: Optional[float] = None):
        self._h = handle
        self.ctx = ctx
        self._tree = tree
        self._dims = dims
        self._acc = accumulated
        self._eps = epsilon_rel
        self._cache: Dict[Tuple[int, int], np.ndarray] = {}

    def _info(self):
        d = C.c_int32()
        self.ctx.check(lib().htr_rep_info(self._h, C.byref(d), None, None, None, None))
        dims = (C.c_int64 * max(1, d.value))()
        acc = C.c_int64()
        eps = C.c_double()
        nn = C.c_int64()
        self.ctx.check(lib().htr_rep_info(self._h, C.byref(d), dims, C.byref(acc), C.byref(eps), C.byref(nn)))
        self._dims = [int(dims[i]) for i in range(d.value)]
        self._acc = int(acc.value)
        self._eps = float(eps.value)
        if self._tree is None:
            nodes = (_Node * nn.value)()
            self.ctx.check(lib().htr_rep_nodes(self._h, nodes, nn.value))
            self._tree = DimensionTree(nodes[:])

    @property
    def tree(self) -> DimensionTree:
        if self._tree is None:
            self._info()
        return self._tree

    @property
    def dims(self) -> List[int]:
        if self._dims is None:
            self._info()
        return self._dims

    @property
    def accumulated(self) -> int:
        """Tensors streamed so far, over all ranks."""
        if self._acc is None:
            self._info()
        return self._acc

    @property
    def local_count(self) -> int:
        """Slices held in this rank's root shard (== accumulated unsharded)."""
        loc = C.c_int64()
        self.ctx.check(lib().htr_rep_counts(self._h, C.byref(loc), None))
        return int(loc.value)

    @property
    def epsilon_rel(self) -> float:
        if self._eps is None:
            self._info()
        return self._eps

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            if self._h:
                lib().htr_rep_free(self._h)
                self._h = None
        except Exception:
            pass

    def core_shape(self, nid) -> Tuple[int, ...]:
        shape = (C.c_int64 * 3)()
        order = C.c_int32()
        self.ctx.check(lib().htr_rep_core_shape(self._h, int(nid[0]), int(nid[1]), shape, C.byref(order)))
        return tuple(int(shape[i]) for i in range(order.value))

    def core(self, nid) -> np.ndarray:
        nid = (int(nid[0]), int(nid[1]))
        if nid not in self._cache:
            shape = self.core_shape(nid)
            out = np.zeros(int(np.prod(shape)), dtype=np.float64)
            self.ctx.check(lib().htr_rep_core_get(self.ctx.handle, self._h, nid[0], nid[1], _ptr(out), 0))
            self._cache[nid] = out.reshape(shape, order="F")
        return self._cache[nid]

    def root(self) -> np.ndarray:
        return self.core((0, 0))

    def rank(self, nid) -> int:
        n = self.tree.node(nid)
        s = self.core_shape(nid)
        if n.kind == LEAF:
            return s[1]
        if n.kind == TRANSFER:
            return s[2]
        raise ValueError("rank: root has no own rank")

    def ranks(self) -> Dict[Tuple[int, int], int]:
        return {n.id: self.rank(n.id) for l in range(1, self.tree.depth + 1) for n in self.tree.layer(l)}

    def max_rank(self) -> int:
        return max(self.ranks().values(), default=0)

    def basis_matrix(self, nid) -> np.ndarray:
        c = self.core(nid)
        if self.tree.node(nid).kind == LEAF:
            return c
        return c.reshape(c.shape[0] * c.shape[1], c.shape[2], order="F")

    def stored_elements(self) -> int:
        return sum(int(np.prod(self.core_shape(n.id))) for layer in self.tree.layers for n in layer)

    def orthonormality_defect(self) -> float:
        worst = 0.0
        for l in range(1, self.tree.depth + 1):
            for n in self.tree.layer(l):
                u = self.basis_matrix(n.id)
                g = u.T @ u
                worst = max(worst, float(np.max(np.abs(g - np.eye(g.shape[0])))))
        return worst

    def validate(self, tol: float = 1e-10):
        """bht.hpp:116-150 (diagnostic; runs on fetched cores)."""
        for l in range(0, self.tree.depth + 1):
            for n in self.tree.layer(l):
                if not np.all(np.isfinite(self.core(n.id))):
                    raise RuntimeError("HTRepresentation: non-finite core entries")
        defect = self.orthonormality_defect()
        if not defect <= tol:
            raise RuntimeError(f"HTRepresentation: orthonormality defect {defect} exceeds {tol}")
        r = self.root()
        if r.ndim != 3 or r.shape[2] != self.local_count:
            raise ValueError("HTRepresentation: root batch extent mismatch")

    def reserve(self, samples: int):
        self.ctx.check(lib().htr_rep_reserve(self.ctx.handle, self._h, int(samples)))

    @staticmethod
    def from_cores(tree: DimensionTree, dims, cores, accumulated: int, epsilon_rel: float,
                   ctx: Optional[Context] = None) -> "HTRepresentation":
        """Device value from host cores (`cores[(layer, pos)]`, canonical
        layout, root included): uploads them bit for bit (htr_rep_import)."""
        ctx = ctx or default_context()
        nodes, nn = tree.c_nodes()
        arrays, shapes = [], []
        for i in range(nn):
            nid = (nodes[i].layer, nodes[i].pos)
            a = np.asfortranarray(np.asarray(cores[nid], dtype=np.float64))
            arrays.append(a)
            s = list(a.shape) + [1] * (3 - a.ndim)
            shapes.extend(int(x) for x in s[:3])
        ptrs = (_D * nn)(*[_ptr(a) for a in arrays])
        shp = (C.c_int64 * len(shapes))(*shapes)
        out = _P()
        ctx.check(lib().htr_rep_import(ctx.handle, nodes, nn, _shape_arr(dims), len(dims), ptrs, shp,
                                       int(accumulated), float(epsilon_rel), C.byref(out)))
        del arrays
        return HTRepresentation(out, ctx, tree, list(dims), int(accumulated), float(epsilon_rel))


# ---------------------------------------------------------------------------
# algorithms
# ---------------------------------------------------------------------------

def bht_l2r(y, tree: DimensionTree, eps_rel: float, adaptive_budget: bool = False,
            ctx: Optional[Context] = None):
    """Alg. 1 (bht.hpp:251-350). Returns (HTRepresentation, BuildReport)."""
    ctx = ctx or default_context()
    p, on_dev, shape, keep = _tensor_arg(y, ctx)
    nodes, nn = tree.c_nodes()
    out = _P()
    rep = _BuildReport()
    ctx.check(lib().htr_bht_l2r(ctx.handle, p, on_dev, _shape_arr(shape), len(shape), nodes, nn, float(eps_rel),
                                int(bool(adaptive_budget)), C.byref(out), C.byref(rep)))
    recs = [NodeRecord((rep.rec_layer[i], rep.rec_pos[i]), int(rep.rec_rank[i]), float(rep.rec_discarded[i]))
            for i in range(rep.n_records)]
    del keep
    return HTRepresentation(out, ctx), BuildReport(recs, [rep.layer_norms[i] for i in range(rep.n_layer_norms)],
                                                   rep.eps_nw_initial)


def ht_rise_update(h: HTRepresentation, y, epsilon_rel: Optional[float] = None, adaptive_budget: bool = False):
    """Alg. 2 (ht_rise.hpp:99-186). Returns (new HTRepresentation, UpdateReport)."""
    ctx = h.ctx
    p, on_dev, shape, keep = _tensor_arg(y, ctx)
    out = _P()
    rep = ctx._update_report  # reused: the C side overwrites every field it reports
    eps = -1.0 if epsilon_rel is None else float(epsilon_rel)
    code = _fn.ht_rise_update(ctx._h, h.handle, p, on_dev, _shape_arr(shape), len(shape), eps,
                              1 if adaptive_budget else 0, C.byref(out), C.byref(rep))
    if code:
        ctx.check(code)
    del keep
    n = rep.n_nodes
    ids = list(zip(rep.node_layer[:n], rep.node_pos[:n]))
    acc = None if (h._acc is None or ctx.world > 1) else h._acc + shape[-1]
    return HTRepresentation(out, ctx, h._tree, h._dims, acc, h._eps), UpdateReport(
        bool(rep.skipped), rep.proj_error, rep.eps_des, dict(zip(ids, rep.added_ranks[:n])),
        dict(zip(ids, rep.new_ranks[:n])), rep.seconds, bool(rep.used_fused_path), bool(rep.used_exact_loss),
        int(rep.kernel_launches))


def _update_report(rep) -> "UpdateReport":
    n = rep.n_nodes
    ids = list(zip(rep.node_layer[:n], rep.node_pos[:n]))
    return UpdateReport(
        bool(rep.skipped), rep.proj_error, rep.eps_des, dict(zip(ids, rep.added_ranks[:n])),
        dict(zip(ids, rep.new_ranks[:n])), rep.seconds, bool(rep.used_fused_path), bool(rep.used_exact_loss),
        int(rep.kernel_launches))


def ht_rise_update_many(h: HTRepresentation, batches, epsilon_rel: Optional[float] = None,
                        adaptive_budget: bool = False):
    """A stream of updates (extension; the reference's caller loops
    ht_rise_update over batches, tools/main.cpp:225-243). Identical to
    calling ht_rise_update on each batch in turn, each on the previous
    result; the library queues batch i+1's skip-path encode before batch i's
    skip decision is read back. Returns ([value after each batch], [report
    of each batch])."""
    ctx = h.ctx
    batches = list(batches)
    n = len(batches)
    if n == 0:
        return [], []
    dev = [isinstance(y, DeviceTensor) for y in batches]
    if any(dev) and not all(dev):
        raise ValueError("ht_rise_update_many: batches must be all on the device or all on the host")
    if dev[0]:
        # device batches: validate each distinct buffer once, and order the
        # library's stream after each distinct producing stream once
        ptr_of, streams = {}, set()
        for y in batches:
            key = id(y.data)
            if key not in ptr_of:
                ptr_of[key] = y.ptr()
                if hasattr(y.data, "data_ptr"):
                    streams.add(_torch_stream(y.data))
        for st in streams:
            code = _fn.context_wait_stream(ctx._h, st)
            if code:
                ctx.check(code)
        args = None
        ptr_list = [ptr_of[id(y.data)] for y in batches]
        shape_list = [tuple(y.shape) for y in batches]
        on_dev = 1
    else:
        args = [_tensor_arg(y) for y in batches]
        ptr_list = [C.cast(a[0], _P).value for a in args]
        shape_list = [a[2] for a in args]
        on_dev = 0
    order = len(shape_list[0])
    if any(len(sh) != order for sh in shape_list):
        raise ValueError("ht_rise_update_many: batches of different tensor order")
    ptrs = (_P * n)(*ptr_list)
    shapes = (C.c_int64 * (n * order))(*[int(e) for sh in shape_list for e in sh])
    outs = (_P * n)()
    reps = (_UpdateReport * n)()
    eps = -1.0 if epsilon_rel is None else float(epsilon_rel)
    code = _fn.ht_rise_update_many(ctx._h, h.handle, n, ptrs, on_dev, shapes, order, eps,
                                   1 if adaptive_budget else 0, outs, reps)
    if code:
        ctx.check(code)
    del args
    values = []
    acc = h._acc
    for i in range(n):
        if acc is not None:
            acc = None if ctx.world > 1 else acc + int(shapes[i * order + order - 1])
        values.append(HTRepresentation(_P(outs[i]), ctx, h._tree, h._dims, acc, h._eps))
    return values, _Reports(reps)


class _Reports(_SequenceABC):
    """The reports of ht_rise_update_many, decoded from the C structs on first
    access (the call returns as soon as the device work is done)."""

    def __init__(self, raw):
        self._raw = raw
        self._done: Dict[int, UpdateReport] = {}

    def __len__(self):
        return len(self._raw)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        r = self._done.get(i)
        if r is None:
            r = self._done[i] = _update_report(self._raw[i])
        return r

    def __eq__(self, other):
        return list(self) == list(other)


def _latent_shape(h: HTRepresentation, batch: int):
    r = h.core_shape((0, 0))
    return (r[0], r[1], batch)


def encode(h: HTRepresentation, y):
    """bht.hpp:373-401 -> (latent r11 x r12 x N, projection error)."""
    ctx = h.ctx
    p, on_dev, shape, keep = _tensor_arg(y, ctx)
    if len(shape) != h.tree.dims() + 1:
        raise ValueError(f"encode: tensor order {len(shape)} does not match tree over {h.tree.dims()} dims plus batch")
    lat = np.zeros(int(np.prod(_latent_shape(h, shape[-1]))), dtype=np.float64)
    err = C.c_double()
    ctx.check(lib().htr_encode(ctx.handle, h.handle, p, on_dev, _shape_arr(shape), len(shape), _ptr(lat), 0,
                               C.byref(err)))
    del keep
    return lat.reshape(_latent_shape(h, shape[-1]), order="F"), float(err.value)


def decode(h: HTRepresentation, latent, out: Optional[DeviceTensor] = None):
    """bht.hpp:406-456. With `out` (a DeviceTensor of prod(dims) x N
    elements) the reconstruction is written there in device memory and `out`
    is returned; otherwise a host array."""
    ctx = h.ctx
    p, on_dev, shape, keep = _tensor_arg(latent, ctx)
    if len(shape) != 3:
        raise ValueError(f"decode: latent ranks {list(shape)} do not match root")
    if out is not None:
        if not isinstance(out, DeviceTensor) or tuple(out.shape) != tuple(h.dims) + (shape[2],):
            raise ValueError("decode: out must be a DeviceTensor of shape dims + (N,)")
        ctx.check(lib().htr_decode(ctx.handle, h.handle, p, on_dev, _shape_arr(shape), C.cast(out.ptr(), _D), 1))
        del keep
        return out
    out = np.zeros(int(np.prod(h.dims)) * shape[2], dtype=np.float64)
    ctx.check(lib().htr_decode(ctx.handle, h.handle, p, on_dev, _shape_arr(shape), _ptr(out), 0))
    del keep
    return out.reshape(list(h.dims) + [shape[2]], order="F")


def pad_latent(latent, r11: int, r12: int) -> np.ndarray:
    """bht.hpp:460-468 (zero padding of a host latent)."""
    latent = _as_host(latent)
    if r11 < latent.shape[0] or r12 < latent.shape[1]:
        raise ValueError("pad_latent: ranks may only grow")
    out = np.zeros((r11, r12, latent.shape[2]), order="F")
    out[: latent.shape[0], : latent.shape[1], :] = latent
    return out


def reconstruct_slice(h: HTRepresentation, m: int) -> np.ndarray:
    """bht.hpp:472-479 (m is 1-based)."""
    out = np.zeros(int(np.prod(h.dims)), dtype=np.float64)
    h.ctx.check(lib().htr_reconstruct_slice(h.ctx.handle, h.handle, int(m), _ptr(out), 0))
    return out.reshape(h.dims, order="F")


@dataclass
class TruncatedBasis:
    """truncated_svd.hpp:17-22."""
    u: np.ndarray
    rank: int
    discarded_norm: float
    singular_values: np.ndarray


def truncated_svd(m, eps_abs: float, min_rank: int = 1, ctx: Optional[Context] = None) -> TruncatedBasis:
    """truncated_svd.hpp:53-100 on the GPU (Gram + one-CTA Jacobi)."""
    ctx = ctx or default_context()
    a = _as_host(m)
    if a.ndim != 2 or a.size == 0:
        raise ValueError("truncated_svd: empty matrix")
    rows, cols = a.shape
    k = min(rows, cols)
    u = np.zeros(rows * max(k, 1) + rows, dtype=np.float64)
    sig = np.zeros(max(k, 1) + 1, dtype=np.float64)
    rank = C.c_int64()
    disc = C.c_double()
    ctx.check(lib().htr_truncated_svd(ctx.handle, _ptr(a), 0, rows, cols, float(eps_abs), int(min_rank), _ptr(u),
                                      _ptr(sig), C.byref(rank), C.byref(disc)))
    r = int(rank.value)
    return TruncatedBasis(u[: rows * r].reshape(rows, r, order="F"), r, float(disc.value), sig[:r].copy())


def mode_multiply(t, mode: int, m, ctx: Optional[Context] = None) -> np.ndarray:
    """tensor.hpp:300-312."""
    ctx = ctx or default_context()
    a = _as_host(t)
    mm = _as_host(m)
    if mode < 0 or mode >= a.ndim:
        raise ValueError(f"mode_multiply: mode {mode} out of range for order {a.ndim}")
    if mm.shape[1] != a.shape[mode]:
        raise ValueError(f"mode_multiply: factor has {mm.shape[1]} cols, mode extent is {a.shape[mode]}")
    out_shape = list(a.shape)
    out_shape[mode] = mm.shape[0]
    out = np.zeros(int(np.prod(out_shape)), dtype=np.float64)
    ctx.check(lib().htr_mode_multiply(ctx.handle, _ptr(a), 0, _shape_arr(a.shape), a.ndim, mode, _ptr(mm),
                                      mm.shape[0], _ptr(out), 0))
    return out.reshape(out_shape, order="F")


def compute_residual(basis, c_unfolded, ctx: Optional[Context] = None) -> np.ndarray:
    """ht_rise.hpp:31-38: R = C - U (U^T C)."""
    ctx = ctx or default_context()
    u = _as_host(basis)
    cm = _as_host(c_unfolded)
    if u.shape[0] != cm.shape[0]:
        raise ValueError(f"compute_residual: basis has {u.shape[0]} rows, unfolding has {cm.shape[0]}")
    out = np.zeros(cm.size, dtype=np.float64)
    ctx.check(lib().htr_compute_residual(ctx.handle, _ptr(u), u.shape[0], u.shape[1], _ptr(cm), cm.shape[1],
                                         _ptr(out)))
    return out.reshape(cm.shape, order="F")


def frobenius_norm(t, ctx: Optional[Context] = None) -> float:
    """tensor.hpp:269."""
    ctx = ctx or default_context()
    p, on_dev, shape, keep = _tensor_arg(t, ctx)
    out = C.c_double()
    ctx.check(lib().htr_frobenius_norm(ctx.handle, p, on_dev, int(np.prod(shape)), C.byref(out)))
    del keep
    return float(out.value)


def relative_error(h: HTRepresentation, y) -> float:
    """||y - decode(encode(y))|| / ||y|| (0 for a zero tensor) of one test
    tensor (order d or d + 1, host or DeviceTensor), computed on the GPU."""
    ctx = h.ctx
    p, on_dev, shape, keep = _tensor_arg(y, ctx)
    out = C.c_double()
    ctx.check(lib().htr_relative_error(ctx.handle, h.handle, p, on_dev, _shape_arr(shape), len(shape), C.byref(out)))
    del keep
    return float(out.value)


_NORM_METHODS = {"none": 0, "maxabs": 1, "unitvec": 2, "zscore": 3}


@dataclass
class NormalizationParams:
    """metrics.hpp:38-46."""
    method: str
    field_axis: Optional[int]
    scale: List[float]
    offset: List[float]
    floored: List[bool]


def normalize(y, method: str = "none", field_axis: Optional[int] = None, ctx: Optional[Context] = None):
    """metrics.hpp:93-171 on the device (htr_normalize). Host arrays in,
    host array out; a DeviceTensor is scaled in place. Returns (scaled,
    NormalizationParams)."""
    ctx = ctx or default_context()
    if method not in _NORM_METHODS:
        raise ValueError("unknown normalization method: " + str(method))
    p, on_dev, shape, keep = _tensor_arg(y, ctx)
    fields = 1 if field_axis is None else int(shape[field_axis]) if 0 <= field_axis < len(shape) else 1
    sc = np.zeros(fields)
    off = np.zeros(fields)
    fl = (C.c_int32 * fields)()
    if on_dev:
        out_p, out = p, y
    else:
        out = np.zeros(int(np.prod(shape)), dtype=np.float64)
        out_p = _ptr(out)
    ctx.check(lib().htr_normalize(ctx.handle, p, on_dev, _shape_arr(shape), len(shape), _NORM_METHODS[method],
                                  -1 if field_axis is None else int(field_axis), out_p, on_dev, _ptr(sc), _ptr(off),
                                  fl))
    del keep
    params = NormalizationParams(method, field_axis, sc.tolist(), off.tolist(), [bool(x) for x in fl])
    if not on_dev:
        out = out.reshape(shape, order="F")
    return out, params


def denormalize(y, params: NormalizationParams, ctx: Optional[Context] = None):
    """metrics.hpp:174-197 on the device (htr_denormalize)."""
    ctx = ctx or default_context()
    p, on_dev, shape, keep = _tensor_arg(y, ctx)
    sc = np.asarray(params.scale, dtype=np.float64)
    off = np.asarray(params.offset, dtype=np.float64)
    out = np.zeros(int(np.prod(shape)), dtype=np.float64)
    ctx.check(lib().htr_denormalize(ctx.handle, p, on_dev, _shape_arr(shape), len(shape),
                                    _NORM_METHODS[params.method],
                                    -1 if params.field_axis is None else int(params.field_axis), _ptr(sc),
                                    _ptr(off), _ptr(out), 0))
    del keep
    return out.reshape(shape, order="F")


def relative_test_error(h: HTRepresentation, test_set) -> float:
    """metrics.hpp:218-237: mean per-tensor relative reconstruction error."""
    test_set = list(test_set)
    if not test_set:
        raise ValueError("relative_test_error: empty test set")
    return sum(relative_error(h, t) for t in test_set) / len(test_set)


def compression_ratio(h: HTRepresentation) -> float:
    """metrics.hpp:200-207."""
    if h.accumulated < 1:
        raise ValueError("compression_ratio: empty accumulation")
    return float(np.prod(h.dims)) * float(h.accumulated) / float(h.stored_elements())


def reduction_ratio(h: HTRepresentation) -> float:
    """metrics.hpp:210-214."""
    r = h.core_shape((0, 0))
    return float(np.prod(h.dims)) / float(r[0] * r[1])
