"""Device-resident graphs with the reference Graph's surface (graph.py:54-216).

``Graph`` keeps the sanitised CSR on the B200 (built there by
gd_graph_create: drop self-loops, canonicalise, dedupe, dense remap, degree
relabel) and materialises the reference's host arrays (``edges``,
``indptr``, ``indices``, ``edge_slot_ids``, ``degrees``, ``orig_ids``) only
when they are read.  Any object exposing ``n`` and ``edges`` (a reference
``graphlets.Graph`` in particular) is accepted by the census entry points.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from . import _native as N
from .errors import EdgeListParseError


@dataclass(frozen=True)
class ParseOptions:
    """Vertex-count conventions of Graph.from_edges (graph.py:36-51)."""

    comment_prefixes: tuple[str, ...] = ("#", "%")
    num_vertices: int | None = None
    use_max_id: bool = False


@dataclass(frozen=True)
class EdgeRef:
    index: int
    u: int
    v: int

    def __post_init__(self):
        if not self.u < self.v:
            raise ValueError(f"EdgeRef endpoints must satisfy u < v, got ({self.u}, {self.v})")


class _Handle:
    """Owns one gd_graph*."""

    __slots__ = ("p",)

    def __init__(self, p):
        self.p = p

    def __del__(self):
        if self.p:
            try:
                N.lib().gd_graph_free(self.p)
            except Exception:  # interpreter shutdown
                pass
            self.p = None


def _hostpack():
    """The CPython pointer-gathering helper, or None when it is not built."""
    try:
        from . import _hostpack as hp
        return hp
    except ImportError:
        return None


def _as_pairs(pairs) -> np.ndarray:
    if isinstance(pairs, np.ndarray) and pairs.dtype == np.int64 and pairs.ndim == 2 and \
            pairs.shape[1] == 2 and pairs.flags.c_contiguous:
        return pairs
    if isinstance(pairs, np.ndarray):
        arr = pairs
    else:
        arr = np.asarray(list(pairs), dtype=np.int64)
    arr = np.ascontiguousarray(arr, dtype=np.int64)
    if arr.size == 0:
        return np.zeros((0, 2), dtype=np.int64)
    if arr.ndim != 2 or arr.shape[1] != 2:
        arr = arr.reshape(-1, 2)
    return arr


def _create(pairs: np.ndarray, n: int, mode: int) -> _Handle:
    N.require_device()
    out = ctypes.c_void_p()
    N.check(N.lib().gd_graph_create(N.vptr(pairs), len(pairs), int(n), mode, 0,
                                    ctypes.byref(out)))
    return _Handle(out.value)


class Graph:
    """Immutable undirected simple graph living on the GPU.

    ``Graph(n, edges, orig_ids=None)`` has the reference constructor's
    contract (graph.py:68-81): edges must already be sanitised (no
    self-loops, no duplicates, endpoints in [0, n)); violations raise
    ValueError.  Use ``Graph.from_edges`` for raw pairs.
    """

    def __init__(self, n: int, edges, orig_ids=None, *, _handle: _Handle | None = None):
        if _handle is None:
            arr = _as_pairs(edges)
            _handle = _create(arr, int(n), N.GD_IDS_SANITIZED)
        self._h = _handle
        nn, mm, _ = (ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64())
        N.check(N.lib().gd_graph_info(self._h.p, ctypes.byref(nn), ctypes.byref(mm),
                                      ctypes.byref(_)))
        self.n = int(nn.value)
        self.m = int(mm.value)
        self._arrays: dict[str, np.ndarray] = {}
        self._micro_cache = None
        if orig_ids is not None:
            oi = np.asarray(orig_ids, dtype=np.int64).copy()
            if len(oi) != self.n:
                raise ValueError("orig_ids length must equal n")
            oi.setflags(write=False)
            self._arrays["orig_ids"] = oi

    # -- construction -------------------------------------------------------
    @staticmethod
    def from_edges(pairs: Iterable[Sequence[int]] | np.ndarray,
                   options: ParseOptions | None = None,
                   _declared_n: int | None = None) -> "Graph":
        """Sanitise raw pairs on the device with Graph.from_edges semantics
        (graph.py:118-157): drop self-loops, merge duplicate and reciprocal
        pairs, then the declared-n, max-id or dense-remap id convention."""
        options = options or ParseOptions()
        arr = _as_pairs(pairs)
        declared = options.num_vertices if options.num_vertices is not None else _declared_n
        if declared is not None:
            return Graph(0, None, _handle=_create(arr, int(declared), N.GD_IDS_DECLARED))
        if options.use_max_id:
            return Graph(0, None, _handle=_create(arr, 0, N.GD_IDS_MAX_ID))
        return Graph(0, None, _handle=_create(arr, 0, N.GD_IDS_REMAP))

    @staticmethod
    def from_file(path, options: ParseOptions | None = None) -> "Graph":
        """Edge-list file (graph.py:159-162), tokenised on the GPU."""
        from .edgelist import from_file
        return from_file(path, options)

    @staticmethod
    def from_text(text: str, options: ParseOptions | None = None) -> "Graph":
        """Edge-list text (graph.py:164-166), tokenised on the GPU."""
        from .edgelist import from_text
        return from_text(text, options)

    @staticmethod
    def from_reference(g) -> "Graph":
        """Device copy of any graph object with ``n``, ``edges`` (and
        optionally ``orig_ids``), e.g. a reference ``graphlets.Graph``."""
        if isinstance(g, Graph):
            return g
        return Graph(int(g.n), np.asarray(g.edges, dtype=np.int64),
                     orig_ids=getattr(g, "orig_ids", None))

    # -- host views ---------------------------------------------------------
    def _export(self, *names: str) -> None:
        want = [k for k in names if k not in self._arrays]
        if not want:
            return
        n, m = self.n, self.m
        shapes = {"edges": (m, 2), "orig_ids": (n,), "indptr": (n + 1,),
                  "indices": (2 * m,), "edge_slot_ids": (2 * m,), "degrees": (n,)}
        bufs = {k: np.empty(shapes[k], dtype=np.int64) for k in want}
        order = ("edges", "orig_ids", "indptr", "indices", "edge_slot_ids", "degrees")
        args = [N.vptr(bufs[k]) if k in bufs and bufs[k].size else None for k in order]
        N.check(N.lib().gd_graph_export(self._h.p, *args))
        for k, a in bufs.items():
            a.setflags(write=False)
            self._arrays[k] = a

    def _get(self, name):
        self._export(name)
        return self._arrays[name]

    edges = property(lambda self: self._get("edges"))
    orig_ids = property(lambda self: self._get("orig_ids"))
    indptr = property(lambda self: self._get("indptr"))
    indices = property(lambda self: self._get("indices"))
    edge_slot_ids = property(lambda self: self._get("edge_slot_ids"))
    degrees = property(lambda self: self._get("degrees"))

    # -- queries (graph.py:164-216) -----------------------------------------
    def neighbors(self, v: int) -> np.ndarray:
        return self.indices[self.indptr[v]:self.indptr[v + 1]]

    def degree(self, v: int) -> int:
        return int(self.degrees[v])

    def has_edge(self, u: int, v: int) -> bool:
        row = self.neighbors(u)
        pos = int(np.searchsorted(row, v))
        return pos < len(row) and row[pos] == v

    def edge_id(self, u: int, v: int) -> int | None:
        row = self.neighbors(u)
        pos = int(np.searchsorted(row, v))
        if pos < len(row) and row[pos] == v:
            return int(self.edge_slot_ids[self.indptr[u] + pos])
        return None

    def edge(self, index: int) -> EdgeRef:
        u, v = self.edges[index]
        return EdgeRef(int(index), int(u), int(v))

    def original_edges(self) -> np.ndarray:
        return self.orig_ids[self.edges]

    @property
    def handle(self):
        return self._h.p

    def __repr__(self):
        return f"Graph(n={self.n}, m={self.m}, device)"


class GraphBatch:
    """Many independent graphs packed as one device graph (disjoint union),
    counted in one launch sequence (config 4; replaces feature_matrix's
    per-graph loop, analytics.py:111-128)."""

    def __init__(self, pairs_list: Sequence[np.ndarray], n_list: Sequence[int]):
        N.require_device()
        if len(pairs_list) != len(n_list):
            raise ValueError("pairs_list and n_list differ in length")
        if not len(pairs_list):
            raise ValueError("empty batch")
        # the library gathers the per-graph arrays into its page-locked
        # staging with all host cores (no packing pass here); their pointers
        # and lengths are collected in one C pass (csrc/hostpack.c)
        arrs = pairs_list if isinstance(pairs_list, list) else list(pairs_list)
        offs = np.zeros(len(arrs) + 1, dtype=np.int64)
        ptrs = np.zeros(len(arrs), dtype=np.uint64)
        hp = _hostpack()
        if hp is None or hp.gather(arrs, ptrs, offs) >= 0:  # some array needs conversion
            arrs = [_as_pairs(p) for p in arrs]
            if hp is None or hp.gather(arrs, ptrs, offs) >= 0:
                np.cumsum([len(a) for a in arrs], out=offs[1:])
                ptrs = np.fromiter((a.__array_interface__["data"][0] for a in arrs),
                                   dtype=np.uint64, count=len(arrs))
        ns = np.ascontiguousarray(np.asarray(n_list, dtype=np.int64))
        out = ctypes.c_void_p()
        N.check(N.lib().gd_graph_create_batch_list(ctypes.c_void_p(ptrs.ctypes.data), N.ptr(offs),
                                                   N.ptr(ns), len(arrs), 0, ctypes.byref(out)))
        self._h = _Handle(out.value)
        self.num_graphs = len(arrs)
        self.n_per_graph = np.zeros(self.num_graphs, dtype=np.int64)
        self.m_per_graph = np.zeros(self.num_graphs, dtype=np.int64)
        N.check(N.lib().gd_graph_sizes(self._h.p, N.ptr(self.n_per_graph),
                                       N.ptr(self.m_per_graph)))

    @staticmethod
    def from_graphs(graphs: Sequence) -> "GraphBatch":
        """Batch of already-sanitised graphs (anything with n and edges)."""
        return GraphBatch([np.asarray(g.edges, dtype=np.int64) for g in graphs],
                          [int(g.n) for g in graphs])

    @property
    def handle(self):
        return self._h.p


def order_edges_by_degree(g) -> np.ndarray:
    """Edge job order of graph.py:314-325 (a hint only; results invariant)."""
    if g.m == 0:
        return np.zeros(0, dtype=np.int64)
    du = g.degrees[g.edges[:, 0]]
    dv = g.degrees[g.edges[:, 1]]
    return np.lexsort((-np.minimum(du, dv), -np.maximum(du, dv))).astype(np.int64)


__all__ = ["Graph", "GraphBatch", "ParseOptions", "EdgeRef", "order_edges_by_degree",
           "EdgeListParseError"]
