"""Seeded per-edge parity samples at full size: shared by the
fixture generator (tools/make_big_fixtures.py, build container) and the GPU
tests, so both draw exactly the same edges."""

from __future__ import annotations

import numpy as np

COUNT_CHUNK = 8192
SAMPLE_SEED = 1506


def degrees(edges: np.ndarray, n: int) -> np.ndarray:
    return np.bincount(edges.ravel(), minlength=n).astype(np.int64)


def micro_sample(edges: np.ndarray, n: int, uniform: int = 5000, top_w: int = 1000,
                 hubs: int = 100, per_hub: int = 100) -> np.ndarray:
    """Sorted canonical edge ids: ``uniform`` uniform edges, the ``top_w``
    edges with the largest w_e = d(lo) + S(lo) (the reference's _count_edge
    cost, census.py:259-303), and up to ``per_hub`` uniform edges incident to
    each of the ``hubs`` highest-degree vertices."""
    m = len(edges)
    rng = np.random.default_rng(SAMPLE_SEED)
    deg = degrees(edges, n)
    u, v = edges[:, 0], edges[:, 1]
    S = (np.bincount(u, weights=deg[v], minlength=n)
         + np.bincount(v, weights=deg[u], minlength=n)).astype(np.int64)
    lo = np.where(deg[u] <= deg[v], u, v)
    w = deg[lo] + S[lo]
    parts = [rng.choice(m, min(uniform, m), replace=False),
             np.argsort(-w, kind="stable")[:top_w]]
    ends = np.concatenate([u, v])
    eid = np.concatenate([np.arange(m), np.arange(m)])
    by_end = np.argsort(ends, kind="stable")
    ends, eid = ends[by_end], eid[by_end]
    for h in np.argsort(-deg, kind="stable")[:hubs]:
        inc = eid[np.searchsorted(ends, h):np.searchsorted(ends, h, side="right")]
        if len(inc) > per_hub:
            inc = rng.choice(inc, per_hub, replace=False)
        parts.append(inc)
    return np.unique(np.concatenate(parts)).astype(np.int64)


def count_sample(m: int, k: int) -> np.ndarray:
    """``k`` uniform edge ids (job order = ascending id)."""
    rng = np.random.default_rng(SAMPLE_SEED + 1)
    return np.sort(rng.choice(m, min(k, m), replace=False)).astype(np.int64)


def count_rows_from_table(tab: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """micro_table columns 0-4 (t, su, sv, cl, cy) of the sampled edges."""
    return np.ascontiguousarray(np.asarray(tab)[idx, :5])
