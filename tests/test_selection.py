"""Incremental selections (selection.py) against the reference: the
closure-from-moments on CPU over golden per-edge tables, and the device op
streams (gd_select.cu) replayed against the reference's counts after every
operation (tests/golden/selection.json, make_golden.py --selection)."""
import json

import numpy as np
import pytest

import paper_1506_04322_b200 as gd
from helpers import GOLDEN, int_counts, small_graphs
from paper_1506_04322_b200.selection import close_moments, tuple_moments

STREAMS = json.loads((GOLDEN / "selection.json").read_text())


def test_close_from_moments_matches_reference_counts():
    """Whole-graph selection == full census: the moments of the reference
    micro rows (t, su, sv, cl, cy) closed with n give the golden counts."""
    for name, n, edges, counts, micro in small_graphs()[:80]:
        f = close_moments(tuple_moments(np.asarray(micro)[:, :5]), n)
        assert f.counts == counts, name


def _op(step):
    action, vertex, u, v = step["op"]
    return gd.SelectionOp(action, vertex=vertex, u=u, v=v)


@pytest.mark.gpu
@pytest.mark.parametrize("stream", STREAMS, ids=[s["name"] for s in STREAMS])
def test_device_op_stream_matches_reference(stream):
    base = gd.Graph(stream["n"], np.asarray(stream["edges"], dtype=np.int64).reshape(-1, 2))
    st = gd.SelectionState(base, active=stream["active"], excluded_edges=stream["excluded"])
    assert st.frequencies().counts == int_counts(stream["initial"])
    for i, step in enumerate(stream["steps"]):
        if "error" in step:
            with pytest.raises(Exception) as ei:
                st.apply_one(_op(step))
            assert type(ei.value).__name__ == step["error"], (i, step)
            continue
        f = st.apply_one(_op(step))
        assert (f.n, f.m) == (step["n"], step["m"]), (i, step["op"])
        assert f.counts == int_counts(step["counts"]), (i, step["op"])
    st.audit()


@pytest.mark.gpu
def test_selection_on_config2_hub_region():
    """Selections around hubs of config 2 (large regions) equal a fresh
    census of the induced subgraph."""
    from paper_1506_04322_b200 import workloads as W
    raw = W.config_graph("c2_chung_lu")
    g = gd.Graph.from_edges(raw.pairs, gd.ParseOptions(num_vertices=raw.n))
    deg = np.asarray(g.degrees)
    hubs = np.argsort(-deg)[:3]
    verts = set(int(h) for h in hubs)
    for h in hubs:
        verts.update(int(x) for x in g.neighbors(int(h))[:400])
    st = gd.SelectionState(g, active=sorted(verts))
    st.audit()
    st.apply_one(gd.SelectionOp("remove_vertex", vertex=int(hubs[0])))
    nb = g.neighbors(int(hubs[1]))
    st.apply_one(gd.SelectionOp("remove_edge", u=int(hubs[1]), v=int(nb[0])))
    assert st.audit() == st.frequencies()
