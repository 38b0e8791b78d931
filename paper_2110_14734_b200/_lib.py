"""ctypes binding of libw1g.so (include/w1g.h).

This is the thin host layer between the reference-shaped Python API and the
sm_100a kernels.  It loads the in-tree shared library, declares every entry
point, maps the library's error codes onto the exception types the reference
raises (ValueError, NetworkError, AssertionError, ...) and keeps one device
context per (host thread, device).  There is no CPU fallback: if the library
is missing or no B200 is visible, calls fail loudly.
"""

from __future__ import annotations

import ctypes
import math
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libw1g.so")

W1G_OK = 0
W1G_EINVAL = -1
W1G_ECUDA = -2
W1G_EOVERFLOW = -3
W1G_EDUPLICATE = -4
W1G_ECOUNT = -5
W1G_ENETWORK = -6
W1G_ENOMEM = -7
W1G_ESTATE = -8

NODES0 = 0
NODES = 1

_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_f64 = ctypes.c_double
_u64 = ctypes.c_uint64
_vp = ctypes.c_void_p
_I64P = ctypes.POINTER(ctypes.c_int64)
_I32P = ctypes.POINTER(ctypes.c_int32)
_F64P = ctypes.POINTER(ctypes.c_double)


class FrontEndInfo(ctypes.Structure):
    """w1g_front_end_info (include/w1g.h)."""

    _fields_ = [
        ("n_points0", _i64),
        ("n_points", _i64),
        ("n_tree_nodes", _i64),
        ("n_pairs", _i64),
        ("n_arcs", _i64),
        ("node_count", _i64),
        ("lower_bound", _f64),
        ("lower_bound_a", _f64),
        ("lower_bound_b", _f64),
        ("epsilon_condense", _f64),
        ("delta", _f64),
        ("short_circuit", _i32),
        ("tree_depth", _i32),
        ("n_levels_wspd", _i32),
        ("network_copied", _i32),
        ("stage_ms", ctypes.c_float * 8),
    ]


class BatchResult(ctypes.Structure):
    """w1g_batch_result (include/w1g.h)."""

    _fields_ = [
        ("pair", _i64),
        ("i", _i32),
        ("j", _i32),
        ("status", _i32),
        ("pad", _i32),
        ("info", FrontEndInfo),
        ("supplies", _vp),
        ("tails", _vp),
        ("heads", _vp),
        ("row_offsets", _vp),
        ("costs", _vp),
        ("block", _vp),
        ("message", ctypes.c_char * 256),
    ]


W1G_DONE = 1

STAGES = ("zero_condense", "rwmd", "delta_condense", "split_tree", "wspd", "emit_arcs", "assemble", "total")

# (name, restype, argtypes)
_PROTOS = [
    ("w1g_version", ctypes.c_int, []),
    ("w1g_host_alloc", ctypes.c_int, [ctypes.c_uint64, ctypes.POINTER(_vp)]),
    ("w1g_host_free", ctypes.c_int, [_vp]),
    ("w1g_launch_count", ctypes.c_uint64, []),
    ("w1g_profile_rwmd_tile", ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_float), _I64P]),
    ("w1g_profile_rwmd", ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_float), _I64P, _I64P]),
    ("w1g_debug_radix_sort", ctypes.c_int, [_vp, _vp, ctypes.c_int, _i64, _vp]),
    ("w1g_device_count", ctypes.c_int, [_I32P]),
    ("w1g_last_error", ctypes.c_char_p, []),
    ("w1g_ctx_create", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_vp)]),
    ("w1g_ctx_destroy", ctypes.c_int, [_vp]),
    ("w1g_ctx_stream", _vp, [_vp]),
    ("w1g_synchronize", ctypes.c_int, [_vp]),
    ("w1g_zero_condense", ctypes.c_int, [_vp, _F64P, _i64, _F64P, _i64, _I64P, _I32P]),
    ("w1g_zero_condense_device", ctypes.c_int, [_vp, _vp, _i64, _vp, _i64, _I64P, _I32P]),
    ("w1g_load_nodes", ctypes.c_int, [_vp, ctypes.c_int, _F64P, _I64P, _I64P, _i64, _i64, _i64]),
    ("w1g_nodes_size", ctypes.c_int, [_vp, ctypes.c_int, _I64P]),
    ("w1g_fetch_nodes", ctypes.c_int, [_vp, ctypes.c_int, _F64P, _I64P, _I64P]),
    ("w1g_rwmd", ctypes.c_int, [_vp, _F64P, _F64P, _F64P]),
    ("w1g_fetch_rwmd_best", ctypes.c_int, [_vp, ctypes.c_int, _F64P, _I64P]),
    ("w1g_set_rwmd_culling", ctypes.c_int, [_vp, ctypes.c_int]),
    ("w1g_member_counts", ctypes.c_int, [_vp, _I64P, _I64P]),
    ("w1g_rwmd_sharded", ctypes.c_int, [ctypes.POINTER(_vp), ctypes.c_int, _F64P, _F64P, _F64P]),
    ("w1g_rwmd_range", ctypes.c_int, [_vp, ctypes.c_int, _i64, _i64, _F64P, _I64P]),
    ("w1g_delta_condense", ctypes.c_int, [_vp, _f64, _f64, _f64, _u64, _I64P]),
    ("w1g_snap_points", ctypes.c_int, [_vp, _F64P, _i64, _f64, _F64P, _I64P]),
    ("w1g_split_tree", ctypes.c_int, [_vp, ctypes.c_int, _I64P, _I32P]),
    ("w1g_fetch_tree", ctypes.c_int, [_vp, _I64P, _I64P, _F64P, _I64P, _I64P]),
    ("w1g_load_tree", ctypes.c_int, [_vp, _F64P, _i64, _I64P, _I64P, _F64P, _I64P, _i64]),
    ("w1g_wspd", ctypes.c_int, [_vp, _f64, ctypes.c_int, _I64P]),
    ("w1g_fetch_pairs", ctypes.c_int, [_vp, _I64P, _I64P]),
    ("w1g_wspd_shard", ctypes.c_int, [_vp, _f64, ctypes.c_int, ctypes.c_int, _I64P]),
    ("w1g_emit_pair_arcs", ctypes.c_int, [_vp, ctypes.c_int, _I64P]),
    ("w1g_arcs_device", ctypes.c_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp), _I64P]),
    ("w1g_load_arcs_device", ctypes.c_int, [_vp, _vp, _vp, _vp, _i64]),
    ("w1g_pairs_device", ctypes.c_int, [_vp, ctypes.POINTER(_vp), _I64P]),
    ("w1g_load_pairs_device", ctypes.c_int, [_vp, _vp, _i64]),
    ("w1g_network_from_pairs", ctypes.c_int, [_vp, _I64P, _I64P]),
    ("w1g_fetch_pair_counts", ctypes.c_int, [_vp, _I64P, _I64P]),
    ("w1g_load_pairs", ctypes.c_int, [_vp, _I64P, _i64, _F64P, _i64]),
    ("w1g_emit_arcs", ctypes.c_int, [_vp, _I64P]),
    ("w1g_fetch_arcs", ctypes.c_int, [_vp, _I64P, _I64P, _F64P]),
    ("w1g_load_arcs", ctypes.c_int, [_vp, _I64P, _I64P, _F64P, _i64]),
    ("w1g_build_network", ctypes.c_int, [_vp, _I64P, _i64, _I64P]),
    ("w1g_assemble", ctypes.c_int, [_vp, _I64P, _I64P]),
    ("w1g_fetch_network", ctypes.c_int, [_vp, _I64P, _I64P, _I64P, _F64P, _I64P]),
    ("w1g_set_network_out", ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64]),
    ("w1g_front_end", ctypes.c_int,
     [_vp, _F64P, _i64, _F64P, _i64, _f64, ctypes.c_int, ctypes.c_int, _f64, _f64, _u64,
      ctypes.POINTER(FrontEndInfo)]),
    ("w1g_front_end_device", ctypes.c_int,
     [_vp, _vp, _i64, _vp, _i64, _f64, ctypes.c_int, ctypes.c_int, _f64, _f64, _u64,
      ctypes.POINTER(FrontEndInfo)]),
    ("w1g_front_end_batch", ctypes.c_int,
     [_vp, _vp, _i64, _f64, ctypes.c_int, ctypes.c_int, _f64, _f64, _u64, ctypes.c_int, ctypes.POINTER(FrontEndInfo),
      ctypes.POINTER(ctypes.c_float)]),
    ("w1g_batch_begin", ctypes.c_int,
     [_vp, _vp, _i64, _f64, ctypes.c_int, ctypes.c_int, _f64, _f64, _u64, ctypes.c_int, _i64]),
    ("w1g_batch_next", ctypes.c_int, [_vp, ctypes.POINTER(BatchResult)]),
    ("w1g_batch_release", ctypes.c_int, [_vp]),
    ("w1g_batch_end", ctypes.c_int, [_vp]),
    ("w1g_corpus_load", ctypes.c_int, [_vp, _F64P, _I64P, _i64]),
    ("w1g_corpus_set_host", ctypes.c_int, [_vp, _vp, _I64P, _i64]),
    ("w1g_wcd_corpus", ctypes.c_int, [_vp, _F64P, _i64, _I64P, _i64, _F64P]),
    ("w1g_rwmd_corpus", ctypes.c_int, [_vp, _F64P, _i64, _I64P, _i64, _F64P]),
    ("w1g_dense_network", ctypes.c_int, [_vp, _I64P, _I64P]),
]

EXPORTED = tuple(name for name, _, _ in _PROTOS)

_lib = None
_lib_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load libw1g.so and declare its prototypes (no device needed)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(path):
                raise ImportError(
                    f"{path} is missing: build it with `python -m paper_2110_14734_b200.build` "
                    "(there is no CPU fallback for the sparsify stages)"
                )
            L = ctypes.CDLL(path)
            for name, res, args in _PROTOS:
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


class NetworkError(ValueError):
    """Raised for unbalanced supplies, dangling arcs or invalid costs (network.py:18)."""


def _raise(code: int):
    raise_code(code, load().w1g_last_error().decode(errors="replace"))


def raise_code(code: int, msg: str):
    """The reference's exception type for a library error code."""
    if code in (W1G_EINVAL, W1G_EOVERFLOW, W1G_EDUPLICATE):
        raise ValueError(msg)
    if code == W1G_ENETWORK:
        raise NetworkError(msg)
    if code == W1G_ECOUNT:
        raise AssertionError(msg)
    if code == W1G_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"libw1g error {code}: {msg}")


def check(code: int):
    if code != W1G_OK:
        _raise(code)


def f64p(a: np.ndarray):
    return a.ctypes.data_as(_F64P)


def i64p(a: np.ndarray):
    return a.ctypes.data_as(_I64P)


def as_points(a) -> np.ndarray:
    p = np.ascontiguousarray(a, dtype=np.float64)
    if p.size == 0:
        return np.empty((0, 2), dtype=np.float64)
    return p.reshape(-1, 2)


def as_i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


class Context:
    """One device + one stream + device-resident stage state (w1g_ctx)."""

    def __init__(self, device: int = 0):
        self.lib = load()
        self.device = device
        h = _vp()
        check(self.lib.w1g_ctx_create(int(device), ctypes.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            self.lib.w1g_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(self.lib.w1g_ctx_stream(self.handle) or 0)

    def call(self, name: str, *args):
        check(getattr(self.lib, name)(self.handle, *args))


_tls = threading.local()


def context(device: int | None = None) -> Context:
    """The calling thread's context for `device` (default: $W1G_DEVICE or 0)."""
    if device is None:
        device = int(os.environ.get("W1G_DEVICE", "0"))
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    ctx = ctxs.get(device)
    if ctx is None:
        ctx = ctxs[device] = Context(device)
    return ctx


def device_count() -> int:
    n = ctypes.c_int32(0)
    check(load().w1g_device_count(ctypes.byref(n)))
    return int(n.value)


_pool_free: dict[int, list[int]] = {}
_pool_lock = threading.Lock()
_POOL_KEEP = 8  # free blocks kept per size class


def _size_class(n: int) -> int:
    c = 1 << 20
    while c < n:
        c <<= 1
    return c


def _pool_release(ptr: int, size: int):
    with _pool_lock:
        lst = _pool_free.setdefault(size, [])
        if len(lst) < _POOL_KEEP:
            lst.append(ptr)
            return
    load().w1g_host_free(ctypes.c_void_p(ptr))


class _PinnedHolder:
    """The numpy-visible owner of one pooled page-locked block: the arrays
    carved from it keep it alive (it is their .base), and when the last one is
    garbage-collected the block returns to the pool."""

    __slots__ = ("ptr", "size", "__array_interface__")

    def __init__(self, ptr: int, size: int):
        self.ptr = ptr
        self.size = size
        self.__array_interface__ = {"shape": (size,), "typestr": "|u1", "data": (ptr, False), "version": 3}

    def __del__(self):
        try:
            _pool_release(self.ptr, self.size)
        except Exception:
            pass


def pinned_arrays(specs):
    """numpy arrays [(shape, dtype), ...] carved from one pooled page-locked
    block, so device->host copies of results run at full link speed and the
    arrays are handed to the caller without a host-side copy."""
    offs, nbytes, total = [], [], 0
    for shape, dtype in specs:
        total = (total + 63) & ~63
        offs.append(total)
        nbytes.append(math.prod(shape) * np.dtype(dtype).itemsize)
        total += nbytes[-1]
    size = _size_class(max(total, 1))
    with _pool_lock:
        lst = _pool_free.get(size)
        ptr = lst.pop() if lst else None
    if ptr is None:
        p = _vp()
        check(load().w1g_host_alloc(size, ctypes.byref(p)))
        ptr = p.value
    base = np.asarray(_PinnedHolder(ptr, size))
    out = []
    for (shape, dtype), off, nb in zip(specs, offs, nbytes):
        out.append(base[off:off + nb].view(dtype).reshape(shape))
    return out


def addr(a: np.ndarray) -> int:
    """Raw data address of a contiguous array (a cheap ctypes void* argument)."""
    return a.__array_interface__["data"][0]




def launch_count() -> int:
    return int(load().w1g_launch_count())


class _BlockHolder:
    """Owner of one batch result block (w1g_batch_result.block): the numpy arrays
    viewing it keep it alive; when the last one dies the block goes back to the
    library's pool (w1g_batch_release)."""

    __slots__ = ("block", "__array_interface__")

    def __init__(self, block: int, nbytes: int):
        self.block = block
        self.__array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (block, False), "version": 3}

    def __del__(self):
        try:
            load().w1g_batch_release(ctypes.c_void_p(self.block))
        except Exception:
            pass


def result_arrays(r: "BatchResult"):
    """(supplies, tails, heads, costs, row_offsets) numpy views of a delivered
    network, zero-copy over its page-locked block."""
    n, m = int(r.info.node_count), int(r.info.n_arcs)
    lo = r.block
    hi = max(r.supplies + 8 * n, r.tails + 8 * m, r.heads + 8 * m, r.costs + 8 * m, r.row_offsets + 8 * (n + 1))
    base = np.asarray(_BlockHolder(lo, hi - lo))

    def view(addr_, count, dtype):
        off = addr_ - lo
        return base[off:off + count * 8].view(dtype)

    return (view(r.supplies, n, np.int64), view(r.tails, m, np.int64), view(r.heads, m, np.int64),
            view(r.costs, m, np.float64), view(r.row_offsets, n + 1, np.int64))
