"""ctypes binding of libgdgpu.so (C ABI declared in include/gd_api.h).

There is no CPU fallback: if the library or a CUDA device is missing, every
entry point raises DeviceError.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from .errors import (ConsistencyError, DeviceError, EdgeListParseError,
                     GraphSizeError)

LIB_PATH = Path(__file__).resolve().parent / "libgdgpu.so"

GD_OK, GD_EINVAL, GD_EPARSE, GD_ECAPACITY, GD_ECUDA, GD_ECONSISTENCY = 0, -1, -2, -3, -4, -5
GD_IDS_REMAP, GD_IDS_DECLARED, GD_IDS_MAX_ID, GD_IDS_SANITIZED = 0, 1, 2, 3
GD_INPUT_DEVICE, GD_OUTPUT_DEVICE = 1, 2
GD_PARSE_CR_NEWLINE, GD_PARSE_MM_SHIFT = 1, 2
NUM_SUMS, NUM_MICRO = 13, 10

_lib = None
_lock = threading.Lock()

_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_vp = ctypes.c_void_p

# (name, restype, argtypes) of every symbol include/gd_api.h declares
SIGNATURES = (
    ("gd_last_error", ctypes.c_char_p, []),
    ("gd_version", ctypes.c_int, []),
    ("gd_device_ok", ctypes.c_int, []),
    ("gd_graph_create", ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                       ctypes.c_int, ctypes.POINTER(_vp)]),
    ("gd_graph_create_batch", ctypes.c_int, [_vp, _i64p, _i64p, ctypes.c_int64, ctypes.c_int,
                                             ctypes.POINTER(_vp)]),
    ("gd_graph_create_batch_list", ctypes.c_int, [_vp, _i64p, _i64p, ctypes.c_int64,
                                                  ctypes.c_int, ctypes.POINTER(_vp)]),
    ("gd_graph_info", ctypes.c_int, [_vp, _i64p, _i64p, _i64p]),
    ("gd_graph_sizes", ctypes.c_int, [_vp, _i64p, _i64p]),
    ("gd_graph_export", ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("gd_graph_free", None, [_vp]),
    ("gd_census_global", ctypes.c_int, [_vp, _u64p, _i64p]),
    ("gd_census_per_edge", ctypes.c_int, [_vp, _vp, ctypes.c_int, _u64p, _i64p]),
    ("gd_sums_from_table", ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                          _u64p]),
    ("gd_census_global_edges", ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                              _u64p, _i64p]),
    ("gd_census_per_edge_edges", ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64,
                                                ctypes.c_int, _vp, _u64p, _i64p]),
    ("gd_graph_timings", ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_float), ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_char_p)]),
    ("gd_graph_stats", ctypes.c_int, [_vp, _i64p, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_char_p)]),
    ("gd_comm_unique_id", ctypes.c_int, [ctypes.c_char_p]),
    ("gd_comm_init", ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(_vp)]),
    ("gd_comm_free", None, [_vp]),
    ("gd_census_sharded", ctypes.c_int, [_vp, _vp, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int,
                                         _u64p, _i64p]),
    ("gd_shard_rows", ctypes.c_int, [ctypes.c_int64, ctypes.c_int, ctypes.c_int, _i64p, _i64p]),
    ("gd_close_counts", ctypes.c_int, [_u64p, _i64p, _i64p, ctypes.c_int64, _i64p,
                                       ctypes.POINTER(ctypes.c_int)]),
    ("gd_set_device", ctypes.c_int, [ctypes.c_int]),
    ("gd_device_alloc", _vp, [ctypes.c_int64]),
    ("gd_device_free", None, [_vp]),
    ("gd_host_alloc", _vp, [ctypes.c_int64]),
    ("gd_host_free", None, [_vp]),
    ("gd_flush_l2", ctypes.c_int, []),
    ("gd_trim_workspace", ctypes.c_int, []),
    ("gd_pool_stats", ctypes.c_int, [ctypes.POINTER(ctypes.c_uint64)]),
    ("gd_parse_edge_list", ctypes.c_int, [_vp, ctypes.c_int64,
                                          ctypes.POINTER(ctypes.c_char_p), ctypes.c_int,
                                          ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    ("gd_parsed_info", ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int64)]),
    ("gd_parsed_pairs", _vp, [_vp]),
    ("gd_parsed_free", None, [_vp]),
    ("gd_micro_roles", ctypes.c_int, [_vp, _vp, ctypes.c_int, _vp, _vp,
                                      ctypes.POINTER(ctypes.c_int64)]),
    ("gd_micro_csv", ctypes.c_int, [_vp, _vp, ctypes.c_int, _vp, ctypes.POINTER(ctypes.c_void_p),
                                    ctypes.POINTER(ctypes.c_int64)]),
    ("gd_text_size", ctypes.c_int64, [_vp]),
    ("gd_text_copy", ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, _vp]),
    ("gd_text_free", None, [_vp]),
    ("gd_edge_weights", ctypes.c_int, [_vp, _vp, ctypes.c_int, ctypes.c_int, _vp]),
    ("gd_rank_edges", ctypes.c_int, [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                     _vp, _vp, _vp, _vp]),
    ("gd_vertex_triangles", ctypes.c_int, [_vp, _vp, ctypes.c_int, _vp]),
    ("gd_selection_create", ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_void_p)]),
    ("gd_selection_apply", ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int64, _vp]),
    ("gd_selection_free", None, [_vp]),
)


def load_library(path: Path | None = None):
    """Load and type libgdgpu.so (no device call).  Raises DeviceError."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        # GD_LIBRARY: an alternative build of the same library (schedule
        # experiments, tools/build_variant.py); never a different backend
        p = Path(path) if path else Path(os.environ.get("GD_LIBRARY", LIB_PATH))
        if not p.exists():
            raise DeviceError(f"{p} is missing: build it with __graft_entry__.build() "
                              "(there is no CPU fallback)")
        try:
            lib = ctypes.CDLL(str(p))
        except OSError as exc:
            raise DeviceError(f"cannot load {p}: {exc}") from exc
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def lib():
    return _lib if _lib is not None else load_library()


def check(rc: int) -> None:
    if rc == GD_OK:
        return
    msg = (lib().gd_last_error() or b"").decode(errors="replace")
    if rc == GD_EINVAL:
        raise ValueError(msg)
    if rc == GD_EPARSE:
        raise EdgeListParseError(msg)
    if rc == GD_ECAPACITY:
        raise GraphSizeError(msg)
    if rc == GD_ECONSISTENCY:
        raise ConsistencyError(msg)
    raise DeviceError(f"libgdgpu error {rc}: {msg}")


_device_checked = False


def require_device() -> None:
    global _device_checked
    if not _device_checked:
        if not lib().gd_device_ok():
            raise DeviceError("no CUDA device is visible; the B200 path has no CPU fallback")
        _device_checked = True


def ptr(a: np.ndarray | None, t=ctypes.c_int64):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(t))


def vptr(a: np.ndarray | None):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def wide(sums: np.ndarray) -> list[int]:
    """(lo, hi) uint64 pairs -> Python ints."""
    s = sums.reshape(-1, 2)
    return [int(lo) + (int(hi) << 64) for lo, hi in s]


class _PinnedPool:
    """Library-owned cache of page-locked host blocks.  cudaHostAlloc of a
    per-edge table (1.26 GB at R-MAT-20) costs tens of milliseconds and its
    cudaFreeHost synchronises the device, so blocks released by the arrays
    that used them are kept (up to ``GD_PINNED_CACHE_MB``, default 16 GiB)
    and handed to the next request of the same or a slightly smaller size."""

    def __init__(self):
        self.lock = threading.Lock()
        self.free: list[tuple[int, int]] = []  # (nbytes, pointer)
        self.cached = 0
        self.cap = int(os.environ.get("GD_PINNED_CACHE_MB", 16384)) << 20

    def take(self, nbytes: int) -> tuple[int, int]:
        with self.lock:
            best = None
            for i, (size, p) in enumerate(self.free):
                if nbytes <= size <= 2 * nbytes and (best is None or size < self.free[best][0]):
                    best = i
            if best is not None:
                size, p = self.free.pop(best)
                self.cached -= size
                return p, size
        p = lib().gd_host_alloc(nbytes)
        if not p:  # pinned memory exhausted: drop the cache and retry once
            self.trim()
            p = lib().gd_host_alloc(nbytes)
        return (p or 0), nbytes

    def give(self, p: int, size: int) -> None:
        with self.lock:
            if self.cached + size <= self.cap:
                self.free.append((size, p))
                self.cached += size
                return
        lib().gd_host_free(p)

    def trim(self) -> None:
        with self.lock:
            blocks, self.free, self.cached = self.free, [], 0
        for _, p in blocks:
            lib().gd_host_free(p)


_pinned_pool = _PinnedPool()


class _PinnedBuffer:
    """Owns one page-locked block of the pool.  Exposed to numpy via
    __array_interface__, so every numpy view's base chain ends here and the
    block returns to the pool only when the last view is gone."""

    def __init__(self, p: int, nbytes: int):
        self.p = p
        self.size = nbytes
        self.__array_interface__ = {"data": (p, False), "shape": (nbytes,),
                                    "typestr": "|u1", "version": 3}

    def __del__(self):
        if self.p:
            try:
                _pinned_pool.give(self.p, self.size)
            except Exception:  # interpreter shutdown
                pass
            self.p = 0


def pinned_empty(shape, dtype=np.int64) -> np.ndarray:
    """np.empty in page-locked host memory from the library's pinned pool
    (D2H of per-edge tables at full PCIe rate, no per-call pinning)."""
    dtype = np.dtype(dtype)
    count = int(np.prod(shape)) if len(shape) else 1
    nbytes = max(count * dtype.itemsize, 1)
    p, size = _pinned_pool.take(nbytes)
    if not p:
        return np.empty(shape, dtype=dtype)  # pageable is still correct, only slower
    raw = np.asarray(_PinnedBuffer(p, size))
    return raw[:count * dtype.itemsize].view(dtype).reshape(shape)


def trim_pinned() -> None:
    """Release the cached page-locked host blocks."""
    _pinned_pool.trim()


def env_flag(name: str) -> bool:
    return os.environ.get(name, "") not in ("", "0", "false", "False")
