"""Device role derivation and CSV (gd_derive.cu) against the oracle
restatement (pinned to the reference's output in test_micro_roles.py) on
configs 1 and 2."""
import sys
import tempfile
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1506_04322_b200 as gd  # noqa: E402
from oracle import micro_oracle as MO  # noqa: E402
from paper_1506_04322_b200 import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu


def _graph(name):
    raw = W.config_graph(name)
    return gd.Graph.from_edges(raw.pairs, gd.ParseOptions(num_vertices=raw.n))


def test_config1_csv_and_roles_full():
    g = _graph("c1_er")
    tab = gd.micro_table(g)
    assert gd.micro_csv(g, tab) == MO.micro_csv(g.n, g.edges, g.orig_ids, tab)
    assert np.array_equal(gd.micro_roles(g, tab), MO.roles_table(g.n, g.m, tab))


def test_config2_csv_sampled_rows_and_file_stream():
    g = _graph("c2_chung_lu")
    tab = gd.micro_table(g)
    text = gd.micro_csv(g, tab)
    lines = text.split("\n")
    assert lines[0] == ",".join(MO.HEADER) and lines[-1] == "" and len(lines) == g.m + 2
    idx = np.random.default_rng(5).choice(g.m, 3000, replace=False)
    for k in idx:
        r = MO.derive_roles(g.n, g.m, tab[k], int(k))
        e = np.asarray(g.edges)[k]
        want = [int(g.orig_ids[e[0]]), int(g.orig_ids[e[1]]), r["tri"], r["star_u"], r["star_v"],
                r["tt1"], r["susv1"], r["tt0"], r["susv0"], r["ts1"], r["ss1"], r["ss0"],
                r["ti1"], r["ti0"], r["si1"], r["si0"], r["ii1"], r["ii0"], r["indep3"]]
        assert lines[k + 1] == ",".join(map(str, want))
    roles = gd.micro_roles(g, tab)
    assert np.array_equal(roles[idx], MO.roles_table(g.n, g.m, tab[idx]))
    with tempfile.NamedTemporaryFile(suffix=".csv") as fh:
        size = gd.write_micro_csv(g, tab, fh.name, chunk=1 << 20)
        assert Path(fh.name).read_text() == text and size == len(text)
