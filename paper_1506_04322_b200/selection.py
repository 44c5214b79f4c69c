"""Mutable induced-subgraph selections with localized incremental updates
(the reference's selection.py:1-229).

``SelectionState`` keeps the reference's API, validation and no-op rules.
The per-edge work runs on the GPU (gd_select.cu): a mutation marks the edges
incident to its region (the vertex and its base neighbours, or both endpoints
and theirs), and every such edge that is selected is recounted with the
reference's marks protocol over the selection-filtered adjacency, one CTA per
edge.  Instead of the reference's O(m_sel) re-summation of every stored tuple
after each operation (``_close``), the device maintains eleven exact 128-bit
moments of the selected edges' (t, su, sv, cl, cy) from which the 13 census
sums follow in O(1).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Iterable

import numpy as np

from . import _native as N
from .census import CensusSums, frequencies_from_sums, graphlet_census
from .errors import ConsistencyError
from .frequencies import GraphletFrequencies
from .graph import Graph

_ADD_VERTEX, _REMOVE_VERTEX, _READMIT_EDGE, _EXCLUDE_EDGE = 0, 1, 2, 3


@dataclass(frozen=True)
class SelectionOp:
    """One selection mutation (selection.py:22-35): add_vertex /
    remove_vertex use ``vertex``; add_edge / remove_edge use ``u``/``v``
    (dense base ids).  Edge adds re-admit a previously removed base edge."""

    action: str
    vertex: int | None = None
    u: int | None = None
    v: int | None = None

    VERTEX_ACTIONS = ("add_vertex", "remove_vertex")
    EDGE_ACTIONS = ("add_edge", "remove_edge")


def tuple_moments(tuples) -> list[int]:
    """The eleven moments of per-edge (t, su, sv, cl, cy) tuples (host
    restatement of what gd_select.cu maintains incrementally)."""
    m = [0] * 11
    for t, su, sv, cl, cy in (tuple(int(x) for x in r) for r in tuples):
        s = su + sv
        for k, v in enumerate((1, t, s, cl, cy, t * (t - 1) // 2, su * sv, t * s,
                               su * (su - 1) // 2 + sv * (sv - 1) // 2, t * t, s * s)):
            m[k] += v
    return m


def close_moments(moments, n_sel: int) -> GraphletFrequencies:
    """_close (selection.py:192-210) from the moments: every CensusSums
    field is a polynomial in them, with i3 = n_sel - 2 - t - s."""
    m_sel, s1, s2, s3, s4, s5, s6, s7, s8, s9, s10 = (int(x) for x in moments)
    k = n_sel - 2
    sum_i3 = m_sel * k - s1 - s2
    sum_i3_sq = m_sel * k * k - 2 * k * (s1 + s2) + (s9 + 2 * s7 + s10)
    sums = CensusSums(tri=s1, star=s2, indep3=sum_i3, clique4=s3, cycle4=s4, n_tt=s5,
                      n_susv=s6, n_ts=s7, n_ss_same=s8, n_ti=k * s1 - s9 - s7,
                      n_si=k * s2 - s7 - s10, n_ii=(sum_i3_sq - sum_i3) // 2,
                      outside=m_sel * (m_sel - 1) - 2 * s1 - s2)
    return frequencies_from_sums(sums, n_sel, m_sel)


def induced_subgraph(g, vertices: Iterable[int], excluded_edges: Iterable[int] = ()) -> Graph:
    """Subgraph induced by ``vertices`` (dense ids of ``g``), optionally
    masking some base edges out; ids re-densified, original ids carried
    through (graph.py:328-347)."""
    verts = np.asarray(sorted(set(int(v) for v in vertices)), dtype=np.int64)
    if len(verts) and (verts.min() < 0 or verts.max() >= g.n):
        raise ValueError("selection vertex out of range")
    excluded = set(int(e) for e in excluded_edges)
    member = np.zeros(g.n, dtype=bool)
    member[verts] = True
    edges = np.asarray(g.edges, dtype=np.int64).reshape(-1, 2)
    if len(edges):
        keep = member[edges[:, 0]] & member[edges[:, 1]]
        if excluded:
            keep &= ~np.isin(np.arange(len(edges)), np.fromiter(excluded, dtype=np.int64))
        sub = edges[keep]
    else:
        sub = np.zeros((0, 2), dtype=np.int64)
    dense = np.searchsorted(verts, sub)
    return Graph(len(verts), dense, orig_ids=np.asarray(g.orig_ids)[verts])


class SelectionState:
    """Single-writer selection over an immutable base graph
    (selection.py:38-229)."""

    def __init__(self, base, active: Iterable[int] = (), excluded_edges: Iterable[int] = ()):
        self.base = base
        self._g = Graph.from_reference(base)
        self.active: set[int] = set()
        self.excluded: set[int] = set(int(e) for e in excluded_edges)
        for e in self.excluded:
            if not 0 <= e < base.m:
                raise ValueError(f"excluded edge index {e} out of range")
        N.require_device()
        h = ctypes.c_void_p()
        N.check(N.lib().gd_selection_create(self._g.handle, ctypes.byref(h)))
        self._h = h
        self._mom = np.zeros(22, dtype=np.uint64)
        for e in sorted(self.excluded):
            self._device(_EXCLUDE_EDGE, e)
        self._freqs: GraphletFrequencies | None = None
        for v in active:
            self.apply_one(SelectionOp("add_vertex", vertex=int(v)))
        if self._freqs is None:
            self._freqs = self._close()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                N.lib().gd_selection_free(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    # -- queries -------------------------------------------------------------
    def frequencies(self) -> GraphletFrequencies:
        if self._freqs is None:
            self._freqs = self._close()
        return self._freqs

    def is_selected_edge(self, eid: int) -> bool:
        u, v = np.asarray(self.base.edges)[eid]
        return int(u) in self.active and int(v) in self.active and eid not in self.excluded

    def induced(self) -> Graph:
        return induced_subgraph(self.base, self.active, self.excluded)

    # -- mutation ------------------------------------------------------------
    def apply(self, ops: Iterable[SelectionOp]) -> GraphletFrequencies:
        for op in ops:
            self.apply_one(op)
        return self.frequencies()

    def apply_one(self, op: SelectionOp) -> GraphletFrequencies:
        base = self.base
        if op.action in SelectionOp.VERTEX_ACTIONS:
            x = op.vertex
            if x is None or not 0 <= x < base.n:
                raise ValueError(f"vertex {x} not in base graph")
            if op.action == "add_vertex":
                if x in self.active:
                    return self.frequencies()  # idempotent
                self.active.add(x)
                self._device(_ADD_VERTEX, x)
            else:
                if x not in self.active:
                    return self.frequencies()
                self.active.discard(x)
                self._device(_REMOVE_VERTEX, x)
        elif op.action in SelectionOp.EDGE_ACTIONS:
            if op.u is None or op.v is None:
                raise ValueError("edge op requires u and v")
            eid = self._g.edge_id(op.u, op.v)
            if eid is None:
                raise ValueError(f"({op.u}, {op.v}) is not a base-graph edge")
            if op.action == "add_edge":
                if op.u not in self.active or op.v not in self.active:
                    raise ValueError("add_edge endpoints must be in the active selection")
                if eid not in self.excluded:
                    return self.frequencies()
                self.excluded.discard(eid)
                self._device(_READMIT_EDGE, eid)
            else:
                if eid in self.excluded:
                    return self.frequencies()
                self.excluded.add(eid)
                self._device(_EXCLUDE_EDGE, eid)
        else:
            raise ValueError(f"unknown selection action {op.action!r}")
        self._freqs = self._close()
        return self._freqs

    # -- internals -----------------------------------------------------------
    def _device(self, action: int, a: int) -> None:
        N.check(N.lib().gd_selection_apply(self._h, action, int(a), N.vptr(self._mom)))

    def _moments(self) -> list[int]:
        out = []
        for k in range(11):
            v = int(self._mom[2 * k]) + (int(self._mom[2 * k + 1]) << 64)
            out.append(v - (1 << 128) if v >> 127 else v)
        return out

    def _close(self) -> GraphletFrequencies:
        return close_moments(self._moments(), len(self.active))

    def audit(self) -> GraphletFrequencies:
        """Full recount of the induced selection; ConsistencyError if the
        cached counts drifted (selection.py:212-222)."""
        fresh = graphlet_census(self.induced())
        cached = self.frequencies()
        if fresh != cached:
            raise ConsistencyError(
                "selection cache mismatch: cached counts differ from fresh census")
        return fresh


def selection_census(state: SelectionState, ops: Iterable[SelectionOp]) -> GraphletFrequencies:
    """Apply the operations; the counts of the induced active subgraph
    (selection.py:225-229)."""
    return state.apply(ops)
