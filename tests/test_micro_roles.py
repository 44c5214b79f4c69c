"""Role-count derivation (_derive_micro) and micro_csv against the
reference's own MicroCounts / CSV output (CPU: inputs are golden tables)."""

import json
from types import SimpleNamespace

import numpy as np
import pytest

import paper_1506_04322_b200 as gd
from helpers import GOLDEN


def _load():
    return json.loads((GOLDEN / "micro_roles.json").read_text())


def test_derive_micro_matches_reference_roles():
    d = _load()
    for c in d["graphs"]:
        g = SimpleNamespace(n=c["n"], m=len(c["edges"]), edges=np.asarray(c["edges"]),
                            orig_ids=np.asarray(c["orig_ids"]))
        tab = np.asarray(c["micro"], dtype=np.int64)
        for i, want in enumerate(c["roles"]):
            mc = gd.micro_counts_from_table(g, tab, i)
            got = [getattr(mc, r) for r in d["roles"]] + [mc.local.indep3]
            assert got == want, (c["name"], i)
            gd.unrestricted_counts(mc.local, g.n, g.m, micro=mc)


def test_oracle_micro_csv_and_roles_match_reference():
    """The oracle restatement (checker of the device derive) is pinned to the
    reference's MicroCounts and CSV text."""
    from oracle import micro_oracle as MO
    d = _load()
    for c in d["graphs"]:
        tab = np.asarray(c["micro"], dtype=np.int64)
        assert MO.micro_csv(c["n"], c["edges"], c["orig_ids"], tab) == c["csv"], c["name"]
        roles = MO.roles_table(c["n"], len(c["edges"]), tab)
        assert roles.tolist() == [r for r in c["roles"]], c["name"]


@pytest.mark.gpu
def test_device_micro_csv_and_roles_match_reference():
    d = _load()
    for c in d["graphs"]:
        g = SimpleNamespace(n=c["n"], m=len(c["edges"]), edges=np.asarray(c["edges"]),
                            orig_ids=np.asarray(c["orig_ids"]))
        tab = np.asarray(c["micro"], dtype=np.int64)
        assert gd.micro_csv(g, tab) == c["csv"], c["name"]
        assert gd.micro_roles(g, tab).tolist() == c["roles"], c["name"]


@pytest.mark.gpu
def test_device_negative_role_raises_reference_message():
    g = gd.Graph(4, np.asarray([[0, 1], [1, 2]]))
    tab = np.zeros((2, 10), dtype=np.int64)
    tab[1] = [2, 0, 0, 5, 0, 0, 0, 0, 0, 0]  # cl > C(t, 2) on edge 1
    with pytest.raises(gd.ConsistencyError) as ei:
        gd.micro_csv(g, tab)
    assert str(ei.value) == "negative micro count tt0 on edge EdgeRef(index=1, u=1, v=2)"
    with pytest.raises(gd.ConsistencyError):
        gd.micro_roles(g, tab)


def test_negative_role_is_consistency_error():
    e = gd.EdgeRef(0, 0, 1)
    with pytest.raises(gd.ConsistencyError):
        gd.derive_micro(e, 4, 1, [2, 0, 0, 5, 0, 0, 0, 0, 0, 0])  # cl > C(t,2)


@pytest.mark.gpu
def test_micro_census_on_device_graph():
    d = _load()
    for c in d["graphs"]:
        g = gd.Graph(c["n"], np.asarray(c["edges"]), orig_ids=np.asarray(c["orig_ids"]))
        for i, want in enumerate(c["roles"]):
            mc = gd.micro_census(g, g.edge(i))
            assert [getattr(mc, r) for r in d["roles"]] + [mc.local.indep3] == want
        assert gd.micro_csv(g, gd.micro_table(g)) == c["csv"]


def test_introspection_helpers_match_golden_rows():
    """The marks-protocol helpers reproduce the reference micro rows."""
    from helpers import small_graphs
    from oracle import graph_oracle as GO
    for name, n, edges, counts, micro in small_graphs()[:40]:
        arr = GO.csr_arrays(n, edges)
        g = SimpleNamespace(n=n, m=len(edges), edges=arr["edges"], indptr=arr["indptr"],
                            indices=arr["indices"])
        marks = bytearray(n)
        for i, (u, v) in enumerate(arr["edges"].tolist()):
            e = gd.EdgeRef(i, u, v)
            tri, su, sv = gd.edge_neighborhood_census(g, e, marks)
            uu, vv, ts = gd.same_side_star_edges(g, marks, su, sv)
            cl = gd.clique_count(g, marks, tri)
            cy = gd.cycle_count(g, marks, su)
            gd.clear_marks(g, marks, e)
            assert not any(marks)
            assert [len(tri), len(su), len(sv), cl, cy, uu, vv, ts] == micro[i][:8].tolist(), name
