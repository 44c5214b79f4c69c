"""The independent CPU cross-check (oracle/crosscheck.c) is pinned to the
literal oracle (census_oracle.c, itself pinned to the reference by
test_oracle_golden.py) before its full-size fixtures are trusted by the GPU
tests.  CPU only."""

import json

import numpy as np
import pytest

from helpers import GOLDEN, configs, int_counts, sha
from oracle import oracle as O
from paper_1506_04322_b200 import workloads as W


def _cases():
    out = []
    for n, p, seed in ((40, 0.9, 1), (120, 0.5, 2), (300, 0.3, 3), (60, 1.0, 0), (8, 0.0, 4)):
        rng = np.random.default_rng(seed)
        iu = np.triu_indices(n, 1)
        mask = rng.random(len(iu[0])) < p
        out.append((f"gnp({n},{p})", n, np.stack([iu[0][mask], iu[1][mask]], 1).astype(np.int64)))
    raw = W.chung_lu(3000, 2.1, 8.0, 400.0, seed=11)
    out.append(("chung_lu3000", raw.n, O.canonical_edges(raw.pairs)))
    raw = W.rmat(11, 12, 0.57, 0.19, 0.19, seed=3)
    out.append(("rmat11", raw.n, O.canonical_edges(raw.pairs)))
    # isolated vertices, a star and a clique (degree ties in the orientation)
    star = np.array([[0, i] for i in range(1, 40)], dtype=np.int64)
    out.append(("star+isolated", 60, star))
    iu = np.triu_indices(12, 1)
    out.append(("K12", 12, np.stack(iu, 1).astype(np.int64)))
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c[0])
def test_crosscheck_equals_literal_oracle(case):
    name, n, edges = case
    rows, sums = O.crosscheck_table(edges, n, threads=2)
    assert np.array_equal(rows, O.micro_rows(edges, n, threads=2)), name
    want, seen = O.census_sums(edges, n, threads=2)
    assert sums == want and seen == len(edges)


def test_crosscheck_reference_configs():
    """C1 and C2: whole tables equal the reference's own micro_table (sha256
    recorded by make_golden.py from the Python reference)."""
    for name in ("c1_er", "c2_chung_lu"):
        c = configs()[name]
        raw = W.config_graph(name)
        edges = O.canonical_edges(raw.pairs)
        assert sha(edges) == c["edges_sha256"]
        rows, sums = O.crosscheck_table(edges, raw.n, threads=2)
        assert sha(rows) == c["micro_sha256"], name
        assert O.close(sums, raw.n, len(edges)) == int_counts(c["counts"])


@pytest.mark.parametrize("name", ["c1_er", "c2_chung_lu", "c3_rmat20", "c5_chung_lu_4m"])
def test_full_size_fixtures_are_pinned(name):
    """The committed full-size fixtures agree with every pin recorded when
    they were made (tools/make_crosscheck_fixtures.py refuses to write
    otherwise) and with each other."""
    p = GOLDEN / f"crosscheck_{name}.json"
    if not p.exists():
        pytest.skip(f"{p.name} not generated")
    d = json.loads(p.read_text())
    assert d["pinned_by"] and all(v for v in d["pinned_by"].values() if isinstance(v, bool))
    assert len(d["chunk_sha256"]) == -(-d["m"] // d["chunk_rows"])
    assert O.close([int(x) for x in d["sums"]], d["n"], d["m"]) == int_counts(d["counts"])
    full = GOLDEN / f"oracle_{name}.json"
    if full.exists():
        assert json.loads(full.read_text())["counts"] == d["counts"]
    if name in ("c3_rmat20", "c5_chung_lu_4m"):
        assert d["pinned_by"].get("oracle_micro_sample_rows") is True
        assert d["pinned_by"].get("oracle_count_sample_chunks") is True


def test_crosscheck_tiled_cycle_pass():
    """The tiled common-neighbour path (large centres at full size) gives the
    same tables: every centre tiled, tiles of 64 and 1000 vertices."""
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, %r)
from oracle import oracle as O
import test_crosscheck as T
for name, n, edges in T._cases():
    rows, sums = O.crosscheck_table(edges, n, threads=2)
    assert np.array_equal(rows, O.micro_rows(edges, n, threads=2)), name
print("ok")
''' % str(GOLDEN.parent.parent)
    for tile in ("64", "1000"):
        env = dict(__import__("os").environ, XC_TILE=tile, XC_TILE_S="0",
                   PYTHONPATH=str(GOLDEN.parent))
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
