"""Graph feature vectors and frequency distributions (analytics.py:44-131).

``feature_matrix`` keeps the reference signature, including its plugin seam
``census_fn``.  Without a ``census_fn`` every graph is counted in ONE batched
device pass (GraphBatch: disjoint union, per-graph 128-bit sums) instead of
the reference's serial per-graph loop; the float rows are then built on the
host exactly as the reference builds them (float(count), log1p, L1 scaling),
so they are bit-identical.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .census import (_STEP_NAMES, CensusSums, batch_counts, census_batch, counts_as_ints,
                     frequencies_from_sums, graphlet_census)
from .classes import classes_for
from .frequencies import GraphletFrequencies
from .graph import GraphBatch
from .parallel import ParallelConfig

GFD_SCOPES = ("connected", "all")


@dataclass(frozen=True)
class GfdVector:
    k: int
    scope: str
    class_ids: tuple[str, ...]
    values: tuple[float, ...]
    is_zero: bool = False


def gfd(freqs: GraphletFrequencies, k: int = 4, scope: str = "connected") -> GfdVector:
    """Normalised size-k frequencies (analytics.py:44-59)."""
    if k not in (3, 4):
        raise ValueError("gfd supports k in {3, 4}")
    if scope not in GFD_SCOPES:
        raise ValueError(f"scope must be one of {GFD_SCOPES}")
    ids = classes_for(k, connected_only=scope == "connected")
    raw = [freqs.counts[c] for c in ids]
    total = sum(raw)
    if total == 0:
        return GfdVector(k, scope, ids, tuple(0.0 for _ in ids), True)
    return GfdVector(k, scope, ids, tuple(v / total for v in raw))


@dataclass
class FeatureMatrix:
    class_ids: tuple[str, ...]
    labels: list[str]
    rows: np.ndarray
    seconds: list[float]
    skipped: list[tuple[str, str]] = field(default_factory=list)


def _row(freqs, class_ids, log_scale, normalize):
    row = [float(freqs.counts[c]) for c in class_ids]
    if log_scale:
        row = [math.log1p(v) for v in row]
    if normalize:
        total = sum(row)
        if total > 0:
            row = [v / total for v in row]
    return row


def feature_matrix(graphs, labels=None, config: ParallelConfig | None = None,
                   log_scale: bool = False, normalize: bool = False,
                   census_fn=None) -> FeatureMatrix:
    """One 17-dim count row per graph (analytics.py:91-131).  ``graphs`` is a
    sequence of graph-like objects (n, edges) or a GraphBatch."""
    class_ids = classes_for(2) + classes_for(3) + classes_for(4)
    kept, rows, seconds, skipped = [], [], [], []
    if census_fn is None:
        batch = graphs if isinstance(graphs, GraphBatch) else None
        if batch is None:
            graphs = list(graphs)
        count = batch.num_graphs if batch is not None else len(graphs)
        if labels is None:
            labels = [f"graph_{i}" for i in range(count)]
        labels = list(labels)
        count = min(count, len(labels))  # zip(labels, graphs), reference analytics.py:111
        if count == 0:
            return FeatureMatrix(class_ids, [], np.zeros((0, len(class_ids))), [], [])
        t0 = time.perf_counter()
        if batch is None:
            try:
                batch = GraphBatch.from_graphs(graphs[:count])
            except Exception:  # a malformed graph: per-graph route, as the reference
                return feature_matrix(graphs[:count], labels[:count], config, log_scale,
                                      normalize, census_fn=graphlet_census)
        counts, status, sums = batch_counts(batch, with_sums=True)
        per = (time.perf_counter() - t0) / count
        counts, status = counts[:count], status[:count]

        def skip(i):  # the reference's message: the closure re-run on the exact sums
            try:
                frequencies_from_sums(CensusSums.from_tuple(N.wide(sums[i])),
                                      int(batch.n_per_graph[i]), int(batch.m_per_graph[i]))
                msg = "ConsistencyError: " + _STEP_NAMES[int(status[i]) - 1] + " failed"
            except Exception as exc:
                msg = f"{type(exc).__name__}: {exc}"
            skipped.append((labels[i], msg))

        lo, hi = counts[..., 0], counts[..., 1]
        # float(count) exactly as the reference: int64 -> float64 is correctly
        # rounded; the rare counts beyond int64 go through Python ints
        small = (hi == 0) & (lo >= 0)
        fl = lo.astype(np.float64)
        if not log_scale and not normalize:
            # plain counts: whole-matrix conversion, per-row work only for
            # skipped graphs and counts beyond int64
            ok = status == 0
            keep = np.nonzero(ok)[0]
            matrix = fl[keep]
            wide = ~small[keep].all(axis=1)
            for r in np.nonzero(wide)[0]:
                matrix[r] = [float(v) for v in counts_as_ints(counts[keep[r]])]
            for i in np.nonzero(~ok)[0]:
                skip(i)
            kept = [labels[i] for i in keep]
            return FeatureMatrix(class_ids, kept, matrix.reshape(len(kept), len(class_ids)),
                                 [per] * len(kept), skipped)
        for i in range(count):
            if status[i]:
                skip(i)
                continue
            if small[i].all():
                row = fl[i].tolist()
            else:
                row = [float(v) for v in counts_as_ints(counts[i])]
            if log_scale:
                row = [math.log1p(v) for v in row]
            if normalize:
                total = sum(row)
                if total > 0:
                    row = [v / total for v in row]
            kept.append(labels[i])
            rows.append(row)
            seconds.append(per)
    else:
        graphs = list(graphs)
        if labels is None:
            labels = [f"graph_{i}" for i in range(len(graphs))]
        for label, g in zip(labels, graphs):
            t0 = time.perf_counter()
            try:
                freqs = census_fn(g, config) if config is not None else census_fn(g)
            except Exception as exc:  # per-graph failure: record, skip row
                skipped.append((label, f"{type(exc).__name__}: {exc}"))
                continue
            seconds.append(time.perf_counter() - t0)
            kept.append(label)
            rows.append(_row(freqs, class_ids, log_scale, normalize))
    matrix = np.asarray(rows, dtype=np.float64).reshape(len(rows), len(class_ids))
    return FeatureMatrix(class_ids, kept, matrix, seconds, skipped)


__all__ = ["GfdVector", "gfd", "FeatureMatrix", "feature_matrix", "graphlet_census"]


# ---------------------------------------------------------------------------
# edge analytics over the per-edge table (analytics.py:134-194)
# ---------------------------------------------------------------------------
RANK_PATTERNS = ("star4", "clique4", "triangle", "cycle4")
_PATTERN_CODE = {"triangle": 0, "clique4": 1, "cycle4": 2, "star4": 3}


@dataclass(frozen=True)
class RankedEdge:
    index: int
    u: int            # original ids
    v: int
    weight: int


class _TableArg:
    """The micro table for an analytics call: the caller's host table, or a
    fresh device table from the per-edge census (never copied to the host)."""

    def __init__(self, g, table, config):
        from . import _native as N
        from .census import micro_census_table
        from .graph import Graph
        self.N = N
        self.g = Graph.from_reference(g)
        self.dev = None
        if table is not None:
            self.host = np.ascontiguousarray(table, dtype=np.int64)
            if self.host.shape != (self.g.m, 10):
                raise ValueError(f"table must have shape ({self.g.m}, 10)")
            self.ptr, self.flags = N.vptr(self.host), 0
        elif self.g.m:
            self.dev = N.lib().gd_device_alloc(self.g.m * 80)
            if not self.dev:
                raise MemoryError("device table allocation failed")
            micro_census_table(self.g, config, device_out=self.dev)
            self.ptr, self.flags = self.dev, N.GD_INPUT_DEVICE
        else:
            self.ptr, self.flags = None, 0

    def close(self):
        if self.dev:
            self.N.lib().gd_device_free(self.dev)
            self.dev = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def _pattern(pattern: str) -> int:
    if pattern not in RANK_PATTERNS:
        raise ValueError(f"unknown pattern {pattern!r}; choose from {RANK_PATTERNS}")
    return _PATTERN_CODE[pattern]


def rank_edges(g, pattern: str, top_k: int | None = None, table: np.ndarray | None = None,
               config: ParallelConfig | None = None) -> list[RankedEdge]:
    """Edges by descending pattern participation, canonical index breaking
    ties (analytics.py:142-175); weights and the sort on the device."""
    from . import _native as N
    code = _pattern(pattern)
    with _TableArg(g, table, config) as t:
        m = t.g.m
        k = m if top_k is None else max(0, min(int(top_k), m))
        idx, u, v, w = (np.empty(k, dtype=np.int64) for _ in range(4))
        N.check(N.lib().gd_rank_edges(t.g.handle, t.ptr, t.flags, code, k, N.vptr(idx),
                                      N.vptr(u), N.vptr(v), N.vptr(w)))
    orig = np.asarray(g.orig_ids) if hasattr(g, "orig_ids") else np.asarray(t.g.orig_ids)
    ou, ov = orig[u], orig[v]
    return [RankedEdge(index=int(idx[i]), u=int(ou[i]), v=int(ov[i]), weight=int(w[i]))
            for i in range(k)]


def edge_weights(g, pattern: str, table: np.ndarray | None = None,
                 config: ParallelConfig | None = None) -> np.ndarray:
    """Per-edge weights in canonical edge order (analytics.py:178-186)."""
    from . import _native as N
    code = _pattern(pattern)
    with _TableArg(g, table, config) as t:
        out = np.zeros(t.g.m, dtype=np.int64)
        N.check(N.lib().gd_edge_weights(t.g.handle, t.ptr, t.flags, code, N.vptr(out)))
    return out


def vertex_triangle_counts(g, table: np.ndarray | None = None) -> np.ndarray:
    """Per-vertex triangle participation (analytics.py:189-194): half the sum
    of the triangle counts of the incident edges, on the device."""
    from . import _native as N
    with _TableArg(g, table, None) as t:
        out = np.zeros(t.g.n, dtype=np.int64)
        N.check(N.lib().gd_vertex_triangles(t.g.handle, t.ptr, t.flags, N.vptr(out)))
    return out
