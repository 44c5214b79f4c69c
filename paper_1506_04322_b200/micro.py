"""Per-edge role counts derived from the device micro table.

Host-side O(1)-per-edge algebra of the reference (census.py:32-92, 310-341,
574-623): Theorem 1, N_{.,.,0} = N_{.,.} - N_{.,.,1}.  The
enumerated inputs always come from the B200 per-edge census (micro_table);
nothing here counts graphlets on the CPU.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from math import comb

import numpy as np

from .errors import ConsistencyError
from .graph import EdgeRef


@dataclass(frozen=True)
class EdgeLocalCounts:
    """Neighbourhood class sizes of one edge plus its two enumerated quad
    counts; tri + star_u + star_v + 2 + indep3 == n (census.py:32-43)."""

    tri: int
    star_u: int
    star_v: int
    clique4: int
    cycle4: int
    indep3: int


@dataclass(frozen=True)
class UnrestrictedCounts:
    """Pair counts over the seven {w, r} classifications of an edge; the
    seven class fields sum to C(n-2, 2) (census.py:46-68)."""

    n_tt: int
    n_susv: int
    n_ts: int
    n_ss_same: int
    n_ti: int
    n_si: int
    n_ii: int
    n_ii_1: int

    def partition_total(self) -> int:
        return (self.n_tt + self.n_susv + self.n_ts + self.n_ss_same
                + self.n_ti + self.n_si + self.n_ii)


@dataclass(frozen=True)
class MicroCounts:
    """Exact per-edge counts of every 4-node pattern in every role the edge
    can play (census.py:71-92).  *_1: pair connected (enumerated on the
    device); *_0: by subtraction from the unrestricted pair counts."""

    edge: EdgeRef
    local: EdgeLocalCounts
    tt1: int
    tt0: int
    susv1: int
    susv0: int
    ts1: int
    ts0: int
    ss1: int
    ss0: int
    ti1: int
    ti0: int
    si1: int
    si0: int
    ii1: int
    ii0: int


def unrestricted_counts(local: EdgeLocalCounts, n: int, m: int,
                        micro: MicroCounts | None = None) -> UnrestrictedCounts:
    """Constant-time pair counts (census.py:310-341), with the reference's
    pair-partition check (C(n-2, 2))."""
    t, su, sv, i3 = local.tri, local.star_u, local.star_v, local.indep3
    raw_outside = m - (t + su) - (t + sv) - 1
    n_ii_1 = raw_outside
    if micro is not None:
        n_ii_1 = (raw_outside - (micro.tt1 + micro.ts1 + micro.ti1)
                  - (micro.ss1 + micro.susv1 + micro.si1))
    out = UnrestrictedCounts(n_tt=comb(t, 2), n_susv=su * sv, n_ts=t * (su + sv),
                             n_ss_same=comb(su, 2) + comb(sv, 2), n_ti=t * i3,
                             n_si=(su + sv) * i3, n_ii=comb(i3, 2), n_ii_1=n_ii_1)
    if out.partition_total() != comb(n - 2, 2):
        raise ConsistencyError(
            f"pair partition mismatch: {out.partition_total()} != C({n}-2,2)")
    return out


def derive_micro(e: EdgeRef, n: int, m: int, raw) -> MicroCounts:
    """The 14 role counts from one raw micro row (census.py:574-596)."""
    t, su, sv, cl, cy, uu1, vv1, ts1, ti1, si1 = (int(x) for x in raw)
    i3 = n - 2 - t - su - sv
    local = EdgeLocalCounts(tri=t, star_u=su, star_v=sv, clique4=cl, cycle4=cy, indep3=i3)
    ss1 = uu1 + vv1
    outside = m + 1 - (t + su + 1) - (t + sv + 1)
    ii1 = outside - (cl + ts1 + ti1) - (ss1 + cy + si1)
    mc = MicroCounts(
        edge=e, local=local,
        tt1=cl, tt0=comb(t, 2) - cl,
        susv1=cy, susv0=su * sv - cy,
        ts1=ts1, ts0=t * (su + sv) - ts1,
        ss1=ss1, ss0=comb(su, 2) + comb(sv, 2) - ss1,
        ti1=ti1, ti0=t * i3 - ti1,
        si1=si1, si0=(su + sv) * i3 - si1,
        ii1=ii1, ii0=comb(i3, 2) - ii1)
    for name in ("tt0", "susv0", "ts0", "ss0", "ti0", "ti1", "si0", "si1", "ii0", "ii1"):
        if getattr(mc, name) < 0:
            raise ConsistencyError(f"negative micro count {name} on edge {e}")
    return mc


_derive_micro = derive_micro


def micro_counts_from_table(g, table: np.ndarray, index: int) -> MicroCounts:
    u, v = (int(x) for x in np.asarray(g.edges)[index])
    return derive_micro(EdgeRef(int(index), u, v), int(g.n), int(g.m), table[index])


def micro_census(g, e: EdgeRef, marks=None) -> MicroCounts:
    """All role counts of one edge (census.py:551-571), read from the device
    per-edge table of ``g`` (computed once and cached on our Graph)."""
    from .census import micro_table
    table = getattr(g, "_micro_cache", None)
    if table is None:
        table = micro_table(g)
        try:
            g._micro_cache = table
        except AttributeError:
            pass
    return micro_counts_from_table(g, table, e.index)


MICRO_CSV_HEADER = [
    "src", "dst", "tri", "star_u", "star_v", "clique4", "cycle4",
    "chordal_chord", "cycle_mid_path", "chordal_cycle_edge", "tailed_tail",
    "star3", "tailed_detached", "tri_isolated", "path_end", "star_isolated",
    "pair_edge", "lone_edge", "indep3",
]


ROLE_COLUMNS = ("tt1", "tt0", "susv1", "susv0", "ts1", "ts0", "ss1", "ss0", "ti1", "ti0",
                "si1", "si0", "ii1", "ii0", "indep3")
_NEG_ORDER = ("tt0", "susv0", "ts0", "ss0", "ti0", "ti1", "si0", "si1", "ii0", "ii1")


def _device_args(g, table):
    """Our device graph for `g` (any object with n, edges, orig_ids) and the
    table as a C-contiguous int64 (m, 10) array."""
    from .graph import Graph
    dg = Graph.from_reference(g)
    tab = np.ascontiguousarray(table, dtype=np.int64)
    if tab.shape != (dg.m, 10):
        raise ValueError(f"table must have shape ({dg.m}, 10)")
    orig = np.ascontiguousarray(g.orig_ids if hasattr(g, "orig_ids") else dg.orig_ids,
                                dtype=np.int64)
    return dg, tab, orig


def _raise_negative(g, bad: int) -> None:
    idx, k = bad >> 4, bad & 15
    u, v = (int(x) for x in np.asarray(g.edges)[idx])
    raise ConsistencyError(f"negative micro count {_NEG_ORDER[k]} on edge {EdgeRef(idx, u, v)}")


def micro_roles(g, table: np.ndarray) -> np.ndarray:
    """_derive_micro over every edge on the device (census.py:574-596):
    int64 (m, 15) in ROLE_COLUMNS order.  ConsistencyError as the reference."""
    from . import _native as N
    dg, tab, orig = _device_args(g, table)
    out = np.empty((dg.m, len(ROLE_COLUMNS)), dtype=np.int64)
    bad = ctypes.c_int64(-1)
    rc = N.lib().gd_micro_roles(dg.handle, N.vptr(tab), 0, N.vptr(orig), N.vptr(out),
                                ctypes.byref(bad))
    if bad.value >= 0:
        _raise_negative(g, bad.value)
    N.check(rc)
    return out


class _Text:
    """A device CSV buffer (gd_micro_csv)."""

    def __init__(self, g, table):
        from . import _native as N
        self.N, self.L = N, N.lib()
        dg, tab, orig = _device_args(g, table)
        self.h = ctypes.c_void_p()
        bad = ctypes.c_int64(-1)
        rc = self.L.gd_micro_csv(dg.handle, N.vptr(tab), 0, N.vptr(orig), ctypes.byref(self.h),
                                 ctypes.byref(bad))
        if bad.value >= 0:
            _raise_negative(g, bad.value)
        N.check(rc)
        self.size = int(self.L.gd_text_size(self.h))

    def read(self, offset: int, length: int) -> bytearray:
        buf = bytearray(length)
        if length:
            view = (ctypes.c_char * length).from_buffer(buf)
            self.N.check(self.L.gd_text_copy(self.h, offset, length, view))
            del view
        return buf

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            self.L.gd_text_free(self.h)
            self.h = None


def micro_csv(g, table: np.ndarray) -> str:
    """Per-edge role CSV with original vertex ids (census.py:603-623),
    derived and formatted on the device."""
    t = _Text(g, table)
    return t.read(0, t.size).decode("ascii")


def write_micro_csv(g, table: np.ndarray, path, chunk: int = 256 << 20) -> int:
    """Stream micro_csv(g, table) into a file without building the string;
    returns the bytes written."""
    t = _Text(g, table)
    with open(path, "wb") as fh:
        for off in range(0, t.size, chunk):
            fh.write(t.read(off, min(chunk, t.size - off)))
    return t.size
