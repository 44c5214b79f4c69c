"""Synthetic config generators: shapes and determinism (CPU)."""

import numpy as np

from paper_1506_04322_b200 import workloads as W
from helpers import sha


def test_er_exact_m_no_loops():
    g = W.erdos_renyi_gnm(500, 2000, seed=3)
    assert g.pairs.shape == (2000, 2)
    assert np.all(g.pairs[:, 0] < g.pairs[:, 1])
    assert len(np.unique(g.pairs[:, 0] * 500 + g.pairs[:, 1])) == 2000


def test_deterministic():
    a = W.chung_lu(5000, 2.1, 10.0, 500.0, seed=1)
    b = W.chung_lu(5000, 2.1, 10.0, 500.0, seed=1)
    assert sha(a.pairs) == sha(b.pairs)
    r = W.rmat(10, 16, 0.57, 0.19, 0.19, seed=20)
    assert r.n == 1024 and len(r.pairs) == 16 * 1024
    assert r.pairs.min() >= 0 and r.pairs.max() < 1024


def test_batch_shapes():
    gs = W.small_graph_batch(8, seed=5)
    assert len(gs) == 8
    for g in gs:
        assert 20 <= g.n <= 500
        assert g.pairs.min() >= 0 and g.pairs.max() < g.n
