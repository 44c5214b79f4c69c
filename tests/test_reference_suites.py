"""Replay of the reference's own property suites against the drop-in
(SURVEY §4): the hypothesis graphs of pkg/tests/test_census.py:260-263, its
random-vs-oracle loop (:252-258), order invariance (:265-276), the complement
identity (:288-294), the named-graph expectations (:222-241), the beyond-64-bit
closure (:278-286) and the schedule-determinism matrix of
pkg/tests/test_parallel.py:31-45 (workers x batch sizes x orderings).  The
graphs are drawn here with the same shapes and ranges; the checker is the
pinned oracle (oracle/), never the product."""

from math import comb

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1506_04322_b200 as gd
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _gnp(n: int, p: float, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    iu = np.triu_indices(n, 1)
    mask = rng.random(len(iu[0])) < p
    return np.stack([iu[0][mask], iu[1][mask]], 1).astype(np.int64)


def _avg_degree(n: int, k: float, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    pairs = rng.integers(0, n, size=(int(n * k / 2 * 1.1), 2))
    return O.canonical_edges(pairs, n)[: int(n * k / 2)]


@st.composite
def small_graphs(draw, min_n=2, max_n=10):
    """Any simple graph on min_n..max_n vertices (every vertex pair drawn
    independently), as the reference's strategy does."""
    n = draw(st.integers(min_n, max_n))
    pairs = [(u, v) for u in range(n) for v in range(u + 1, n)]
    keep = draw(st.lists(st.booleans(), min_size=len(pairs), max_size=len(pairs)))
    edges = np.asarray([p for p, k in zip(pairs, keep) if k], dtype=np.int64).reshape(-1, 2)
    return n, edges


def _check(n, edges):
    g = gd.Graph(n, edges)
    f = gd.graphlet_census(g)
    assert f.counts == O.census(edges, n), (n, edges.tolist())
    f.validate()
    tab, f2 = gd.micro_census_table(g)
    assert f2 == f
    assert np.array_equal(np.asarray(tab), O.micro_rows(np.asarray(g.edges), n))


@settings(max_examples=50, deadline=None, derandomize=True)
@given(small_graphs(min_n=2, max_n=10))
def test_property_equals_oracle(case):
    _check(*case)


def test_random_equals_oracle():
    rng = np.random.default_rng(42)
    for _ in range(30):
        n = int(rng.integers(4, 31))
        p = float(rng.choice(np.arange(1, 10) / 10))
        _check(n, _gnp(n, p, int(rng.integers(1 << 30))))


def test_order_invariance():
    n, edges = 40, _gnp(40, 0.3, 9)
    base = gd.graphlet_census(gd.Graph(n, edges))
    base_tab = np.asarray(gd.micro_table(gd.Graph(n, edges)))
    rng = np.random.default_rng(5)
    for _ in range(3):
        perm = rng.permutation(len(edges))
        g = gd.Graph(n, edges[perm])
        assert gd.graphlet_census(g) == base
        # rows follow the graph's own edge order
        key = {tuple(e): i for i, e in enumerate(map(tuple, edges))}
        back = np.asarray([key[tuple(e)] for e in np.asarray(g.edges).tolist()])
        assert np.array_equal(np.asarray(gd.micro_table(g)), base_tab[back])
    assert gd.graphlet_census(gd.Graph(n, edges),
                              gd.ParallelConfig(workers=1, ordering="degree-desc")) == base


def test_determinism_matrix_workers_batches_orderings():
    """parallel.py:85-149 promises the same result for every worker count,
    batch size and ordering; the device schedule ignores them, so the whole
    matrix must give one answer (and the oracle's)."""
    n = 2000
    edges = _avg_degree(n, 10, 1)
    g = gd.Graph(n, edges)
    base = gd.graphlet_census(g, gd.ParallelConfig(workers=1))
    assert base.counts == O.census(np.asarray(g.edges), n)
    tab0 = np.asarray(gd.micro_table(g, gd.ParallelConfig(workers=1))).copy()
    for workers in (2, 4, 8):
        assert gd.graphlet_census(g, gd.ParallelConfig(workers=workers)) == base
    for batch in (1, 64, 256):
        cfg = gd.ParallelConfig(workers=4, batch_size=batch)
        assert gd.graphlet_census(g, cfg) == base
        assert np.array_equal(np.asarray(gd.micro_table(g, cfg)), tab0)
    n2, e2 = 120, _gnp(120, 0.1, 2)
    g2 = gd.Graph(n2, e2)
    a = gd.graphlet_census(g2, gd.ParallelConfig(workers=3, ordering="input"))
    b = gd.graphlet_census(g2, gd.ParallelConfig(workers=3, ordering="degree-desc"))
    assert a == b
    ta = np.asarray(gd.micro_table(g2, gd.ParallelConfig(workers=3, ordering="input")))
    tb = np.asarray(gd.micro_table(g2, gd.ParallelConfig(workers=3, ordering="degree-desc")))
    assert np.array_equal(ta, tb)  # rows stay in canonical edge order


def test_counts_are_exact_beyond_64_bits():
    n = 200_000
    g = gd.Graph(n, np.asarray([[0, 1], [1, 2], [5, 6]]))
    f = gd.graphlet_census(g)
    assert f.counts["g4_11"] > 2 ** 63
    assert sum(f.counts[c] for c in gd.CLASS_IDS if c.startswith("g4")) == comb(n, 4)
    f.validate()


def test_complement_identity_via_census():
    for seed in range(15):
        n = 13
        edges = _gnp(n, 0.35, seed)
        have = {tuple(e) for e in edges.tolist()}
        comp = np.asarray([(u, v) for u in range(n) for v in range(u + 1, n)
                           if (u, v) not in have], dtype=np.int64).reshape(-1, 2)
        fg = gd.graphlet_census(gd.Graph(n, edges))
        fc = gd.graphlet_census(gd.Graph(n, comp))
        for cid in gd.CLASS_IDS:
            assert fg.counts[cid] == fc.counts[gd.complement_class(cid)]


def test_named_graphs():
    def K(n):
        return n, np.stack(np.triu_indices(n, 1), 1).astype(np.int64)

    def cyc(n):
        return n, np.asarray([[i, (i + 1) % n] for i in range(n)], dtype=np.int64)

    def path(n):
        return n, np.asarray([[i, i + 1] for i in range(n - 1)], dtype=np.int64)

    def star(k):
        return k + 1, np.asarray([[0, i] for i in range(1, k + 1)], dtype=np.int64)

    cases = {
        "K4": (K(4), {"g4_1": 1, "g3_1": 4}),
        "C4": (cyc(4), {"g4_4": 1, "g3_2": 4}),
        "P4": (path(4), {"g4_6": 1, "g3_2": 2}),
        "S3": (star(3), {"g4_5": 1, "g3_2": 3}),
        "diamond": ((4, np.asarray([[0, 1], [0, 2], [0, 3], [1, 2], [1, 3]])), {"g4_2": 1, "g3_1": 2}),
        "paw": ((4, np.asarray([[0, 1], [0, 2], [1, 2], [2, 3]])), {"g4_3": 1, "g3_1": 1}),
        "2K2": ((4, np.asarray([[0, 1], [2, 3]])), {"g4_9": 1}),
        "K6": (K(6), {"g4_1": comb(6, 4), "g3_1": comb(6, 3)}),
        "C7": (cyc(7), {"g4_6": 7, "g4_4": 0}),
    }
    for name, ((n, edges), expected) in cases.items():
        f = gd.graphlet_census(gd.Graph(n, edges))
        for cid, val in expected.items():
            assert f.counts[cid] == val, (name, cid)
        assert f.counts == O.census(np.asarray(gd.Graph(n, edges).edges), n), name
