"""rank_edges / edge_weights / vertex_triangle_counts (analytics.py:142-194)
against the reference's outputs (tests/golden/analytics.json, made by
make_golden.py --analytics): a numpy restatement on CPU (pins the weight
definitions and tie-break), the device kernels (gd_rank.cu) on the GPU."""
import json
from types import SimpleNamespace

import numpy as np
import pytest

import paper_1506_04322_b200 as gd
from helpers import GOLDEN

CASES = json.loads((GOLDEN / "analytics.json").read_text())


def _np_weights(tab, p):
    if p == "triangle":
        return tab[:, 0]
    if p == "clique4":
        return tab[:, 3]
    if p == "cycle4":
        return tab[:, 4]
    su, sv = tab[:, 1], tab[:, 2]
    return su * (su - 1) // 2 + sv * (sv - 1) // 2 - tab[:, 5] - tab[:, 6]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_numpy_restatement_matches_reference(case):
    tab = np.asarray(case["micro"], dtype=np.int64)
    edges = np.asarray(case["edges"], dtype=np.int64).reshape(-1, 2)
    orig = np.asarray(case["orig_ids"])
    for p, want in case["patterns"].items():
        w = _np_weights(tab, p)
        assert w.tolist() == want["weights"]
        order = np.argsort(-w, kind="stable")
        ranked = [[int(i), int(orig[edges[i, 0]]), int(orig[edges[i, 1]]), int(w[i])] for i in order]
        assert ranked == want["ranked"]
    per = np.zeros(case["n"], dtype=np.int64)
    np.add.at(per, edges[:, 0], tab[:, 0])
    np.add.at(per, edges[:, 1], tab[:, 0])
    assert (per // 2).tolist() == case["vertex_triangles"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_device_analytics_match_reference(case):
    g = SimpleNamespace(n=case["n"], m=len(case["edges"]),
                        edges=np.asarray(case["edges"], dtype=np.int64).reshape(-1, 2),
                        orig_ids=np.asarray(case["orig_ids"]))
    tab = np.asarray(case["micro"], dtype=np.int64)
    dg = gd.Graph(case["n"], g.edges, orig_ids=g.orig_ids)
    for p, want in case["patterns"].items():
        assert gd.edge_weights(g, p, table=tab).tolist() == want["weights"]
        got = [[r.index, r.u, r.v, r.weight] for r in gd.rank_edges(g, p, table=tab)]
        assert got == want["ranked"]
        # no table: census on the device, table never copied to the host
        got = [[r.index, r.u, r.v, r.weight] for r in gd.rank_edges(dg, p, top_k=3)]
        assert got == want["top3"]
    assert gd.vertex_triangle_counts(g, tab).tolist() == case["vertex_triangles"]
    assert gd.vertex_triangle_counts(dg).tolist() == case["vertex_triangles"]
    with pytest.raises(ValueError):
        gd.rank_edges(dg, "pentagon")


@pytest.mark.gpu
def test_config2_rank_matches_numpy_on_the_same_table():
    from paper_1506_04322_b200 import workloads as W
    raw = W.config_graph("c2_chung_lu")
    g = gd.Graph.from_edges(raw.pairs, gd.ParseOptions(num_vertices=raw.n))
    tab = gd.micro_table(g)
    edges, orig = np.asarray(g.edges), np.asarray(g.orig_ids)
    for p in gd.RANK_PATTERNS:
        w = _np_weights(tab, p)
        assert np.array_equal(gd.edge_weights(g, p, table=tab), w)
        order = np.argsort(-w, kind="stable")[:1000]
        got = gd.rank_edges(g, p, top_k=1000)  # device census, device sort
        assert [r.index for r in got] == order.tolist()
        assert [r.weight for r in got] == w[order].tolist()
        assert [(r.u, r.v) for r in got] == [(int(orig[edges[i, 0]]), int(orig[edges[i, 1]]))
                                             for i in order]
    per = np.zeros(g.n, dtype=np.int64)
    np.add.at(per, edges[:, 0], tab[:, 0])
    np.add.at(per, edges[:, 1], tab[:, 0])
    assert np.array_equal(gd.vertex_triangle_counts(g), per // 2)
