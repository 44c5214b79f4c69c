"""Device CSR build (Graph.from_edges / Graph(n, edges)) against the
reference's own construction (tests/golden/graph_build.json)."""

import numpy as np
import pytest

import paper_1506_04322_b200 as gd
from helpers import graph_build
from oracle import graph_oracle as GO

pytestmark = pytest.mark.gpu


def _check(g, c):
    assert g.n == c["n"] and g.m == c["m"], c["name"]
    for k in ("edges", "indptr", "indices", "edge_slot_ids", "degrees"):
        want = np.asarray(c[k], dtype=np.int64)
        assert np.array_equal(np.asarray(getattr(g, k)).reshape(-1), want.reshape(-1)), (c["name"], k)
    assert [int(x) for x in g.orig_ids] == [int(x) for x in c["orig_ids"]]


def test_from_edges_matches_reference_build():
    for c in graph_build()["cases"]:
        opts = gd.ParseOptions(**c["opts"])
        g = gd.Graph.from_edges(np.asarray(c["pairs"], dtype=np.int64).reshape(-1, 2), opts)
        _check(g, c)


def test_error_conventions():
    for e in graph_build()["errors"]:
        if "pairs" in e:
            with pytest.raises(gd.EdgeListParseError):
                gd.Graph.from_edges(np.asarray(e["pairs"]), gd.ParseOptions(**e["opts"]))
        else:
            with pytest.raises(ValueError):
                gd.Graph(e["n"], np.asarray(e["edges"]))


def test_random_builds_vs_numpy_restatement():
    rng = np.random.default_rng(9)
    for trial in range(6):
        k = int(rng.integers(1, 5000))
        hi = int(rng.integers(2, 3000))
        pairs = rng.integers(0, hi, size=(k, 2))
        for opts in ({}, {"num_vertices": hi}, {"use_max_id": True}):
            want = GO.from_edges_arrays(pairs, **opts)
            g = gd.Graph.from_edges(pairs, gd.ParseOptions(**opts))
            assert g.n == want["n"] and g.m == want["m"]
            for key in ("edges", "indptr", "indices", "edge_slot_ids", "degrees", "orig_ids"):
                assert np.array_equal(np.asarray(getattr(g, key)), want[key]), (trial, opts, key)


def test_large_remap_ids():
    rng = np.random.default_rng(4)
    ids = rng.integers(-(1 << 62), 1 << 62, size=20000)
    pairs = ids[rng.integers(0, len(ids), size=(100000, 2))]
    want = GO.from_edges_arrays(pairs)
    g = gd.Graph.from_edges(pairs)
    assert np.array_equal(np.asarray(g.orig_ids), want["orig_ids"])
    assert np.array_equal(np.asarray(g.edges), want["edges"])
