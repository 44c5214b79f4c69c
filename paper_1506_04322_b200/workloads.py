"""Seeded synthetic inputs for the five BASELINE.json configurations.

These stand in for the reference's benchmark graphs (the reference ships
generators only for config 1's G(n, m) shape: generate.py:19-37).  Every
generator returns RAW int64 (k, 2) pairs exactly as a user would hand them
to ``Graph.from_edges`` (graph.py:118-157): they may contain self-loops,
duplicates and reciprocal pairs, which the sanitising CSR build removes.
The vertex count ``n`` is returned alongside because isolated vertices
change the disconnected graphlet counts.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class RawGraph:
    name: str
    n: int
    pairs: np.ndarray          # int64 (k, 2) raw pairs, ids in [0, n)


def erdos_renyi_gnm(n: int, m: int, seed: int) -> RawGraph:
    """Config 1: uniform G(n, m) without loops or multi-edges.

    Oversample pairs, drop loops, canonicalise, dedupe and top up until m
    distinct edges exist; a seeded subset of exactly m is kept (the shape of
    the reference's ``random_graph_avg_degree``, generate.py:19-37)."""
    rng = np.random.default_rng(seed)
    keys = np.zeros(0, dtype=np.int64)
    while len(keys) < m:
        need = m - len(keys)
        d = rng.integers(0, n, size=(int(need * 1.3) + 16, 2), dtype=np.int64)
        d = d[d[:, 0] != d[:, 1]]
        lo = np.minimum(d[:, 0], d[:, 1])
        hi = np.maximum(d[:, 0], d[:, 1])
        keys = np.unique(np.concatenate([keys, lo * n + hi]))
    if len(keys) > m:
        keys = np.sort(rng.choice(keys, size=m, replace=False))
    return RawGraph(f"er_n{n}_m{m}", n, np.stack([keys // n, keys % n], axis=1))


def _chung_lu_weights(n: int, gamma: float, mean_deg: float, cap: float,
                      rng: np.random.Generator) -> np.ndarray:
    """Expected degrees w_i ~ Pareto tail P(w) ~ w^-gamma, rescaled to the
    requested mean and capped (cap/rescale iterated to a fixed point)."""
    u = rng.random(n)
    w = (1.0 - u) ** (-1.0 / (gamma - 1.0))
    for _ in range(50):
        w *= mean_deg / w.mean()
        over = w > cap
        if not over.any():
            break
        w[over] = cap
    return w


def _sample(cdf: np.ndarray, u: np.ndarray) -> np.ndarray:
    """np.searchsorted(cdf, u, side="right") computed on sorted queries (a
    linear merge instead of cache-missing binary searches); same result."""
    if len(u) < (1 << 20):
        return np.searchsorted(cdf, u, side="right")
    order = np.argsort(u, kind="stable")
    out = np.empty(len(u), dtype=np.int64)
    out[order] = np.searchsorted(cdf, u[order], side="right")
    return out


def chung_lu(n: int, gamma: float, mean_deg: float, cap: float, seed: int,
             draw_factor: float = 1.0) -> RawGraph:
    """Configs 2 and 5: Chung-Lu power-law graph.  Endpoints of
    ``draw_factor * n * mean_deg / 2`` raw pairs are sampled independently
    with probability proportional to the expected degrees; the CSR build
    symmetrises, dedupes and drops loops (realised m is reported)."""
    rng = np.random.default_rng(seed)
    w = _chung_lu_weights(n, gamma, mean_deg, cap, rng)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    k = int(round(draw_factor * n * mean_deg / 2))
    src = _sample(cdf, rng.random(k))
    dst = _sample(cdf, rng.random(k))
    np.minimum(src, n - 1, out=src)
    np.minimum(dst, n - 1, out=dst)
    return RawGraph(f"chung_lu_n{n}_g{gamma}_d{mean_deg}", n,
                    np.stack([src, dst], axis=1).astype(np.int64))


def rmat(scale: int, edge_factor: int, a: float, b: float, c: float,
         seed: int) -> RawGraph:
    """Config 3: R-MAT with per-bit quadrant draws and no noise."""
    rng = np.random.default_rng(seed)
    n = 1 << scale
    k = edge_factor * n
    src = np.zeros(k, dtype=np.int64)
    dst = np.zeros(k, dtype=np.int64)
    ab = a + b
    abc = a + b + c
    for bit in range(scale):
        r = rng.random(k)
        src |= (r >= ab).astype(np.int64) << bit
        dst |= (((r >= a) & (r < ab)) | (r >= abc)).astype(np.int64) << bit
    return RawGraph(f"rmat_s{scale}_ef{edge_factor}", n, np.stack([src, dst], axis=1))


def small_graph_batch(count: int, seed: int, n_lo: int = 20, n_hi: int = 500,
                      deg_lo: float = 3.0, deg_hi: float = 8.0) -> list[RawGraph]:
    """Config 4: ``count`` independent small graphs.  Per graph: n ~ U[20,500],
    mean degree ~ U[3,8] -> G(n, round(n*deg/2)) base, plus n//10 planted
    triangles and n//50 planted 4-cliques on random vertex subsets."""
    out = []
    for i, ss in enumerate(np.random.SeedSequence(seed).spawn(count)):
        rng = np.random.default_rng(ss)
        n = int(rng.integers(n_lo, n_hi + 1))
        deg = float(rng.uniform(deg_lo, deg_hi))
        m = int(round(n * deg / 2))
        base = rng.integers(0, n, size=(m, 2), dtype=np.int64)
        parts = [base]
        for size, reps in ((3, n // 10), (4, n // 50)):
            for _ in range(reps):
                vs = rng.choice(n, size=size, replace=False)
                iu = np.triu_indices(size, k=1)
                parts.append(np.stack([vs[iu[0]], vs[iu[1]]], axis=1))
        out.append(RawGraph(f"batch_{i}", n, np.concatenate(parts).astype(np.int64)))
    return out


CONFIGS = {
    "c1_er": lambda: erdos_renyi_gnm(2000, 10000, seed=1506),
    "c2_chung_lu": lambda: chung_lu(100_000, 2.1, 10.0, 5_000.0, seed=4322),
    "c3_rmat20": lambda: rmat(20, 16, 0.57, 0.19, 0.19, seed=20),
    "c5_chung_lu_4m": lambda: chung_lu(4_000_000, 1.9, 30.0, 100_000.0, seed=1904,
                                       draw_factor=1.45),
}


def config_graph(name: str) -> RawGraph:
    return CONFIGS[name]()


def config_batch(count: int = 4096, seed: int = 4096) -> list[RawGraph]:
    return small_graph_batch(count, seed)
