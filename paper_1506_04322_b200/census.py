"""Drop-in counting entry points (graphlets/census.py:478-623 surface).

``graphlet_census`` / ``micro_table`` / ``frequencies_from_micro`` keep the
reference signatures and output layout; the per-edge kernels, the schedule
and the 128-bit reductions run on the B200 through libgdgpu.so.  Only the
O(1) closures (Eqs. 1-4, Lemmas 2-8, Eqs. 18-19; census.py:388-430) run on
the host, in Python ints, with the reference's exact-division checks.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, fields
from math import comb

import numpy as np

from . import _native as N
from .errors import ConsistencyError
from .frequencies import GraphletFrequencies
from .graph import Graph, GraphBatch
from .parallel import ParallelConfig

# Raw kernel output order (micro_table columns), census.py:95-97
RAW_MICRO_FIELDS = ("tri", "star_u", "star_v", "clique4", "cycle4",
                    "uu1", "vv1", "ts1", "ti1", "si1")


@dataclass
class CensusSums:
    """The 13 wide accumulators (census.py:359-385); FIELDS is the device ->
    host layout of gd_census_global."""

    tri: int = 0
    star: int = 0
    indep3: int = 0
    clique4: int = 0
    cycle4: int = 0
    n_tt: int = 0
    n_susv: int = 0
    n_ts: int = 0
    n_ss_same: int = 0
    n_ti: int = 0
    n_si: int = 0
    n_ii: int = 0
    outside: int = 0

    FIELDS = ("tri", "star", "indep3", "clique4", "cycle4", "n_tt", "n_susv",
              "n_ts", "n_ss_same", "n_ti", "n_si", "n_ii", "outside")

    def as_tuple(self):
        return tuple(getattr(self, f) for f in self.FIELDS)

    @staticmethod
    def from_tuple(values) -> "CensusSums":
        return CensusSums(**dict(zip(CensusSums.FIELDS, values)))


def _exact_div(value: int, divisor: int, what: str) -> int:
    q, r = divmod(value, divisor)
    if r:
        raise ConsistencyError(f"{what}: {value} not divisible by {divisor}")
    if q < 0:
        raise ConsistencyError(f"{what}: negative count {q}")
    return q


def _nonneg(value: int, what: str) -> int:
    if value < 0:
        raise ConsistencyError(f"{what}: negative count {value}")
    return value


def close_triads(tri_total: int, star_total: int, indep3_total: int, n: int) -> dict[str, int]:
    """Eqs. 1-4: each triangle is seen from 3 edges, each 2-star from 2."""
    f31 = _exact_div(tri_total, 3, "triangle closure")
    f32 = _exact_div(star_total, 2, "2-star closure")
    f33 = _nonneg(indep3_total, "3-node-1-edge closure")
    f34 = _nonneg(comb(n, 3) - f31 - f32 - f33, "3-node-independent closure")
    return {"g3_1": f31, "g3_2": f32, "g3_3": f33, "g3_4": f34}


def close_quads(sums: CensusSums, n: int, m: int) -> dict[str, int]:
    """Lemmas 2-8 and Eqs. 18-19 in dependency order (census.py:399-421)."""
    s = sums
    k41 = _exact_div(s.clique4, 6, "4-clique closure")
    k42 = _nonneg(s.n_tt - 6 * k41, "chordal-cycle closure")
    k44 = _exact_div(s.cycle4, 4, "4-cycle closure")
    k46 = _nonneg(s.n_susv - 4 * k44, "4-path closure")
    k43 = _exact_div(s.n_ts - 4 * k42, 2, "tailed-triangle closure")
    k45 = _exact_div(s.n_ss_same - k43, 3, "3-star closure")
    k47 = _exact_div(s.n_ti - k43, 3, "triangle-plus-isolated closure")
    k48 = _exact_div(s.n_si - 2 * k46, 2, "2-star-plus-isolated closure")
    k49 = _exact_div(s.outside - 6 * k41 - 4 * k42 - 2 * k43 - 4 * k44 - 2 * k46, 2,
                     "two-edge closure")
    k410 = _nonneg(s.n_ii - 2 * k49, "one-edge closure")
    k411 = _nonneg(comb(n, 4) - (k41 + k42 + k43 + k44 + k45 + k46 + k47 + k48 + k49 + k410),
                   "independent closure")
    return {"g4_1": k41, "g4_2": k42, "g4_3": k43, "g4_4": k44, "g4_5": k45,
            "g4_6": k46, "g4_7": k47, "g4_8": k48, "g4_9": k49, "g4_10": k410,
            "g4_11": k411}


def frequencies_from_sums(sums: CensusSums, n: int, m: int) -> GraphletFrequencies:
    counts = {"g2_1": m, "g2_2": comb(n, 2) - m}
    counts.update(close_triads(sums.tri, sums.star, sums.indep3, n))
    counts.update(close_quads(sums, n, m))
    freqs = GraphletFrequencies(counts=counts, n=n, m=m)
    freqs.validate()
    return freqs


def _check_config(config) -> None:
    if config is not None and not isinstance(config, ParallelConfig):
        # the reference ParallelConfig is accepted too (same fields)
        for f in ("workers", "batch_size", "ordering"):
            if not hasattr(config, f):
                raise TypeError("config must be a ParallelConfig")


def _device(g):
    """(handle owner, n, m) for our Graph or any graph-like object."""
    if isinstance(g, (Graph, GraphBatch)):
        return g
    return Graph.from_reference(g)


def graphlet_census(g, config: ParallelConfig | None = None) -> GraphletFrequencies:
    """All 17 global graphlet counts (census.py:478-491).  ``config`` is
    validated and ignored: results are schedule-invariant."""
    _check_config(config)
    n, m = int(g.n), int(g.m)
    if m == 0:  # closed form, no launch (all per-edge sums are empty)
        return frequencies_from_sums(CensusSums(), n, m)
    dg = _device(g)
    sums = np.zeros(2 * N.NUM_SUMS, dtype=np.uint64)
    seen = np.zeros(1, dtype=np.int64)
    N.check(N.lib().gd_census_global(dg.handle, N.ptr(sums, ctypes.c_uint64), N.ptr(seen)))
    if int(seen[0]) != m:
        raise ConsistencyError(f"processed {int(seen[0])} edges, expected {m}")
    return frequencies_from_sums(CensusSums.from_tuple(N.wide(sums)), n, m)


def micro_table(g, config: ParallelConfig | None = None, *, pinned: bool = True) -> np.ndarray:
    """Per-edge enumerated counts, (m, 10) int64 in canonical edge order with
    columns RAW_MICRO_FIELDS (census.py:503-518)."""
    table, _ = micro_census_table(g, config, pinned=pinned)
    return table


def micro_census_table(g, config: ParallelConfig | None = None, *, pinned: bool = True,
                       out: np.ndarray | None = None, device_out: int | None = None):
    """micro_table plus the global frequencies from the same device pass.

    ``out``: a C-contiguous int64 (m, 10) host array to fill (e.g. a reused
    pinned buffer); ``device_out``: a device pointer (int) of m*10 int64 to
    leave the table in HBM (then the returned table is None)."""
    _check_config(config)
    n, m = int(g.n), int(g.m)
    if m == 0:
        return np.zeros((0, len(RAW_MICRO_FIELDS)), dtype=np.int64), \
            frequencies_from_sums(CensusSums(), n, m)
    dg = _device(g)
    flags = 0
    if device_out is not None:
        table = None
        tptr = ctypes.c_void_p(int(device_out))
        flags = N.GD_OUTPUT_DEVICE
    else:
        if out is not None:
            if out.shape != (m, N.NUM_MICRO) or out.dtype != np.int64 or \
                    not out.flags["C_CONTIGUOUS"]:
                raise ValueError("out must be a C-contiguous int64 (m, 10) array")
            table = out
        else:
            table = N.pinned_empty((m, N.NUM_MICRO)) if pinned else \
                np.empty((m, N.NUM_MICRO), np.int64)
        tptr = N.vptr(table)
    sums = np.zeros(2 * N.NUM_SUMS, dtype=np.uint64)
    seen = np.zeros(1, dtype=np.int64)
    N.check(N.lib().gd_census_per_edge(dg.handle, tptr, flags,
                                       N.ptr(sums, ctypes.c_uint64), N.ptr(seen)))
    if int(seen[0]) != m:
        raise ConsistencyError(f"processed {int(seen[0])} edges, expected {m}")
    return table, frequencies_from_sums(CensusSums.from_tuple(N.wide(sums)), n, m)


def frequencies_from_micro(g, table: np.ndarray) -> GraphletFrequencies:
    """Dual route (census.py:521-544): global counts from a micro table,
    reduced on the device in 128-bit."""
    n, m = int(g.n), int(g.m)
    tab = np.ascontiguousarray(table, dtype=np.int64)
    if tab.shape != (m, len(RAW_MICRO_FIELDS)):
        raise ValueError(f"table shape {tab.shape} != ({m}, {len(RAW_MICRO_FIELDS)})")
    if m == 0:
        return frequencies_from_sums(CensusSums(), n, m)
    N.require_device()
    sums = np.zeros(2 * N.NUM_SUMS, dtype=np.uint64)
    N.check(N.lib().gd_sums_from_table(N.vptr(tab), m, n, 0, N.ptr(sums, ctypes.c_uint64)))
    return frequencies_from_sums(CensusSums.from_tuple(N.wide(sums)), n, m)


_STEP_NAMES = ("triangle closure", "2-star closure", "3-node-1-edge closure",
               "3-node-independent closure", "4-clique closure", "chordal-cycle closure",
               "4-cycle closure", "4-path closure", "tailed-triangle closure", "3-star closure",
               "triangle-plus-isolated closure", "2-star-plus-isolated closure",
               "two-edge closure", "one-edge closure", "independent closure")


def batch_counts(batch: GraphBatch, with_sums: bool = False):
    """One device census of every graph of the batch, closed in exact 128-bit
    integers by the library: (counts int64 [G][17][2] as (lo, hi) of signed
    128-bit values, status [G]: 0 ok, else 1 + failing closure step) and, with
    ``with_sums``, the raw 13 sums per graph (uint64 [G][26])."""
    G = batch.num_graphs
    sums = np.zeros(G * 2 * N.NUM_SUMS, dtype=np.uint64)
    seen = np.zeros(G, dtype=np.int64)
    N.check(N.lib().gd_census_global(batch.handle, N.ptr(sums, ctypes.c_uint64), N.ptr(seen)))
    if not np.array_equal(seen, batch.m_per_graph):
        bad = int(np.nonzero(seen != batch.m_per_graph)[0][0])
        raise ConsistencyError(f"graph {bad}: processed {int(seen[bad])} edges, "
                               f"expected {int(batch.m_per_graph[bad])}")
    counts = np.zeros((G, 17, 2), dtype=np.int64)
    status = np.zeros(G, dtype=np.int32)
    N.check(N.lib().gd_close_counts(N.ptr(sums, ctypes.c_uint64), N.ptr(batch.n_per_graph),
                                    N.ptr(batch.m_per_graph), G, N.ptr(counts),
                                    status.ctypes.data_as(ctypes.POINTER(ctypes.c_int))))
    if with_sums:
        return counts, status, sums.reshape(G, 2 * N.NUM_SUMS)
    return counts, status


def counts_as_ints(counts_lohi: np.ndarray) -> list[int]:
    lo = counts_lohi[..., 0].astype(np.uint64)
    hi = counts_lohi[..., 1]
    return [int(a) + (int(b) << 64) for a, b in zip(lo.tolist(), hi.tolist())]


def census_batch(batch: GraphBatch) -> list[GraphletFrequencies | Exception]:
    """Global counts of every graph of a batch from one device pass.  A graph
    whose closure fails yields its ConsistencyError in place of a result."""
    from .classes import CLASS_IDS
    counts, status, sums = batch_counts(batch, with_sums=True)
    out: list = []
    for i in range(batch.num_graphs):
        n, m = int(batch.n_per_graph[i]), int(batch.m_per_graph[i])
        if status[i]:
            # the reference's exception and message: the closure re-run on
            # the exact sums of this graph
            try:
                frequencies_from_sums(CensusSums.from_tuple(N.wide(sums[i])), n, m)
                out.append(ConsistencyError(_STEP_NAMES[int(status[i]) - 1] + " failed"))
            except Exception as exc:
                out.append(exc)
            continue
        f = GraphletFrequencies(counts=dict(zip(CLASS_IDS, counts_as_ints(counts[i]))), n=n, m=m)
        out.append(f)
    return out


def last_timings(g) -> dict[str, float]:
    """Device phase times (ms, CUDA events) of the last census on ``g``."""
    ms = (ctypes.c_float * 32)()
    names = ctypes.c_char_p()
    k = N.lib().gd_graph_timings(g.handle, ms, 32, ctypes.byref(names))
    labels = (names.value or b"").decode().split("\n")
    return {labels[i]: float(ms[i]) for i in range(k)}


def trim_workspace() -> None:
    """Release this thread's cached device workspace of the census kernels
    (kept between calls so censuses of fresh graphs do not re-allocate) and
    the cached page-locked host blocks of returned tables."""
    N.check(N.lib().gd_trim_workspace())
    N.trim_pinned()


def last_stats(g) -> dict[str, int]:
    vals = (ctypes.c_int64 * 32)()
    names = ctypes.c_char_p()
    k = N.lib().gd_graph_stats(g.handle, vals, 32, ctypes.byref(names))
    labels = (names.value or b"").decode().split("\n")
    return {labels[i]: int(vals[i]) for i in range(k)}
