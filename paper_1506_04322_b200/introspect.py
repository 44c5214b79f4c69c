"""Single-edge introspection helpers with the reference's marks protocol
(census.py:104-187: 1 = Star_u, 2 = Tri_e, 3 = Star_v).

These are NOT the counting path (that is micro_table / graphlet_census on the
B200): they expose the neighbourhood classes of one edge for inspection and
tests, exactly as the reference's composed kernels do, over the host CSR view
of a graph.
"""

from __future__ import annotations

import numpy as np

from .graph import EdgeRef


def _nbrs(g, v: int) -> list[int]:
    ip = g.indptr
    return np.asarray(g.indices[ip[v]:ip[v + 1]]).tolist()


def edge_neighborhood_census(g, e: EdgeRef, marks: bytearray):
    """(Tri_e, Star_u, Star_v) of edge e; marks must be all zero on entry."""
    u, v = e.u, e.v
    au = _nbrs(g, u)
    for w in au:
        marks[w] = 1
    marks[v] = 0
    tri, star_v = [], []
    for w in _nbrs(g, v):
        if marks[w] == 1:
            marks[w] = 2
            tri.append(w)
        elif w != u:
            marks[w] = 3
            star_v.append(w)
    return tri, [w for w in au if marks[w] == 1], star_v


def clique_count(g, marks: bytearray, tri: list[int]) -> int:
    """Edges inside Tri_e (4-cliques through e); clears Tri marks."""
    count = 0
    for w in tri:
        count += sum(1 for r in _nbrs(g, w) if marks[r] == 2)
        marks[w] = 0
    return count


def cycle_count(g, marks: bytearray, star_u: list[int]) -> int:
    """Edges between Star_u and Star_v (4-cycles through e); clears Star_u."""
    count = 0
    for w in star_u:
        count += sum(1 for r in _nbrs(g, w) if marks[r] == 3)
        marks[w] = 0
    return count


def same_side_star_edges(g, marks: bytearray, star_u: list[int], star_v: list[int]):
    """(edges within Star_u, within Star_v, between Tri_e and the stars)."""
    uu = vv = ts = 0
    for w in star_u:
        for r in _nbrs(g, w):
            if marks[r] == 1 and w < r:
                uu += 1
            elif marks[r] == 2:
                ts += 1
    for w in star_v:
        for r in _nbrs(g, w):
            if marks[r] == 3 and w < r:
                vv += 1
            elif marks[r] == 2:
                ts += 1
    return uu, vv, ts


def clear_marks(g, marks: bytearray, e: EdgeRef) -> None:
    for w in _nbrs(g, e.u):
        marks[w] = 0
    for w in _nbrs(g, e.v):
        marks[w] = 0
