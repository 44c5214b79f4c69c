"""Parity of the B200 path against the reference's golden vectors and the
oracle.  Bit-exact everywhere (integer counts)."""

import os
import subprocess
import sys
from types import SimpleNamespace

import numpy as np
import pytest

import paper_1506_04322_b200 as gd
from helpers import GOLDEN, configs, int_counts, sha, small_graphs
from sample_sets import count_rows_from_table, count_sample
from oracle import oracle as O
from paper_1506_04322_b200 import workloads as W

pytestmark = pytest.mark.gpu


def test_small_graphs_drop_in():
    for name, n, edges, counts, micro in small_graphs():
        g = gd.Graph(n, edges)
        f = gd.graphlet_census(g)
        assert f.counts == counts, name
        f.validate()
        tab = gd.micro_table(g)
        assert tab.dtype == np.int64 and tab.shape == (len(edges), 10)
        assert np.array_equal(np.asarray(tab), micro), name
        if len(edges):
            assert gd.frequencies_from_micro(g, tab) == f, name


def test_foreign_graph_objects_are_accepted():
    name, n, edges, counts, micro = small_graphs()[-1]
    foreign = SimpleNamespace(n=n, m=len(edges), edges=edges)
    assert gd.graphlet_census(foreign).counts == counts
    assert np.array_equal(np.asarray(gd.micro_table(foreign)), micro)
    # ParallelConfig is accepted and ignored for results
    cfg = gd.ParallelConfig(workers=3, batch_size=7, ordering="degree-desc")
    assert gd.graphlet_census(foreign, cfg).counts == counts


def test_edge_order_invariance():
    name, n, edges, counts, micro = small_graphs()[-1]
    perm = np.random.default_rng(5).permutation(len(edges))
    flipped = edges[perm][:, ::-1].copy()
    g = gd.Graph(n, flipped)
    assert gd.graphlet_census(g).counts == counts
    assert np.array_equal(np.asarray(gd.micro_table(g)), micro)


def test_degenerate_graphs():
    for n in (0, 1, 2, 3, 7):
        g = gd.Graph(n, np.zeros((0, 2), dtype=np.int64))
        f = gd.graphlet_census(g)
        f.validate()
        assert gd.micro_table(g).shape == (0, 10)
    g = gd.Graph(2, np.asarray([[0, 1]]))
    assert gd.graphlet_census(g).counts["g2_1"] == 1
    assert np.array_equal(np.asarray(gd.micro_table(g)), np.zeros((1, 10), dtype=np.int64))


FORCED = ["tri_gmem", "tri_small", "tri_blocks", "c4_coop", "c4_hub32", "c4_smem",
          "c4_flow", "tri_gmem,c4_coop", "tri_small,c4_hub32", "wide_slots", "c4_flow,wide_slots",
          "c4_tile64", "c4_coop,c4_tile64", "c4_coop,c4_tile64,wide_slots", "c4_coop,c4_cluster",
          "c4_coop,c4_flow", "pipeline", "c4_coop,c4_tile64,bits16", "c4_coop,c4_tile64,bits8",
          "c4_tile64,bits4", "c4_coop,c4_tile64,pieces1", "c4_coop,pieces1", "c4_coop,pieces8,bits16"]


def _dense_cases():
    out = []
    for n, p, seed in ((40, 0.9, 1), (120, 0.5, 2), (300, 0.3, 3), (60, 1.0, 0)):
        rng = np.random.default_rng(seed)
        iu = np.triu_indices(n, 1)
        mask = rng.random(len(iu[0])) < p
        out.append((f"gnp({n},{p})", n, np.stack([iu[0][mask], iu[1][mask]], 1)))
    raw = W.chung_lu(3000, 2.1, 8.0, 400.0, seed=11)
    out.append(("chung_lu3000", raw.n, O.canonical_edges(raw.pairs)))
    raw = W.rmat(11, 12, 0.57, 0.19, 0.19, seed=3)
    out.append(("rmat11", raw.n, O.canonical_edges(raw.pairs)))
    # leaves (degree 1: skipped by the pass-C tiles) beside degree-2 and hub vertices:
    # a star, and K_{2,50} with 100 leaves on either hub
    out.append(("star40", 41, np.asarray([[0, i] for i in range(1, 41)], dtype=np.int64)))
    k2 = [[h, 2 + i] for h in (0, 1) for i in range(50)]
    lv = [[h, 52 + 100 * h + i] for h in (0, 1) for i in range(100)]
    out.append(("k2_50+leaves", 252, O.canonical_edges(np.asarray(k2 + lv, dtype=np.int64), 252)))
    return out


@pytest.mark.parametrize("force", FORCED)
def test_forced_kernel_paths_match_oracle(force):
    """Every kernel variant (bins) checked against the oracle in a subprocess
    with GD_FORCE_PATH set (the schedule never changes results)."""
    code = r'''
import sys, numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r)
import paper_1506_04322_b200 as gd
from oracle import oracle as O
import test_gpu_parity as T
for name, n, edges in T._dense_cases():
    g = gd.Graph(n, edges)
    f = gd.graphlet_census(g)
    tab, f2 = gd.micro_census_table(g)
    want = O.census(edges, n)
    assert f.counts == want, (name, "global")
    assert f2 == f, (name, "per-edge sums")
    rows = O.micro_rows(edges, n)
    assert np.array_equal(np.asarray(tab), rows), (name, "micro")
print("ok")
''' % (str(GOLDEN.parent.parent), str(GOLDEN.parent))
    env = dict(os.environ, GD_FORCE_PATH=force)
    if force == "pipeline":  # the multi-pass pipeline where the small-graph kernel would run
        env = dict(os.environ, GD_SMALL="0")
    if "wide_slots" in force:  # 64-bit per-slot sums even where 32 bits suffice
        env["GD_WIDE_SLOTS"] = "1"
    if "pieces" in force:  # piece walk of the pass-C tiles from this average segment length
        env["GD_C4_PIECE_MIN"] = force.split("pieces")[1].split(",")[0]
        env["GD_FORCE_PATH"] = force.split(",pieces")[0]
        force = force.replace(",pieces" + env["GD_C4_PIECE_MIN"], "")
    if "bits" in force:  # narrowest counter width of the degree-aware pass-C tiles
        env["GD_C4_TILE_BITS"] = force.split("bits")[1]
        env["GD_FORCE_PATH"] = force.split(",bits")[0]
    if force == "tri_small,c4_hub32":
        env["GD_HIT_CAP"] = "5000"  # hit-buffer overflow: pass B re-probes some frames
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_default_paths_dense_cases():
    for name, n, edges in _dense_cases():
        g = gd.Graph(n, edges)
        tab, f = gd.micro_census_table(g)
        assert f.counts == O.census(edges, n), name
        assert np.array_equal(np.asarray(tab), O.micro_rows(edges, n)), name
        assert gd.graphlet_census(g) == f


def test_config1_exact():
    c = configs()["c1_er"]
    raw = W.config_graph("c1_er")
    g = gd.Graph.from_edges(raw.pairs, _declared_n=raw.n)
    assert sha(np.asarray(g.edges)) == c["edges_sha256"]
    f = gd.graphlet_census(g)
    assert f.counts == int_counts(c["counts"])
    tab = np.asarray(gd.micro_table(g))
    assert np.array_equal(tab, np.load(GOLDEN / "c1.npz")["micro"])
    assert sha(tab) == c["micro_sha256"]


def test_config2_against_reference():
    c = configs().get("c2_chung_lu")
    raw = W.config_graph("c2_chung_lu")
    g = gd.Graph.from_edges(raw.pairs, _declared_n=raw.n)
    tab, f = gd.micro_census_table(g)
    assert gd.graphlet_census(g) == f
    edges = np.asarray(g.edges)
    if c is None:
        assert f.counts == O.census(edges, raw.n)
    else:
        assert sha(edges) == c["edges_sha256"]
        assert f.counts == int_counts(c["counts"])
        assert sha(np.asarray(tab)) == c["micro_sha256"]
        idx = np.asarray(c["sample_idx"])
        assert np.array_equal(np.asarray(tab)[idx], np.asarray(c["sample_rows"]))
    idx = np.random.default_rng(1).choice(g.m, 3000, replace=False)
    assert np.array_equal(np.asarray(tab)[idx], O.micro_rows(edges, g.n, idx))


def test_config4_batch_feature_matrix():
    gold = np.load(GOLDEN / "c4_batch.npz")
    raws = W.config_batch()
    batch = gd.GraphBatch([r.pairs for r in raws], [r.n for r in raws])
    assert np.array_equal(batch.m_per_graph, gold["m"])
    fm = gd.feature_matrix(batch)
    assert fm.rows.shape == (4096, 17) and not fm.skipped
    assert np.array_equal(fm.rows, gold["counts"].astype(np.float64))
    # log/normalise rows equal the reference float math bit for bit
    fm2 = gd.feature_matrix(batch, log_scale=True, normalize=True)
    import math
    row = [math.log1p(float(v)) for v in gold["counts"][0]]
    tot = sum(row)
    assert fm2.rows[0].tolist() == [v / tot for v in row]
    # the plugin seam (census_fn) path gives the same rows
    some = [gd.Graph.from_edges(r.pairs, _declared_n=r.n) for r in raws[:16]]
    fm3 = gd.feature_matrix(some, census_fn=gd.graphlet_census)
    assert np.array_equal(fm3.rows, gold["counts"][:16].astype(np.float64))


def _chunk_sha(a, rows):
    a = np.ascontiguousarray(a)
    return [sha(a[i:i + rows]) for i in range(0, len(a), rows)]


def _big_parity(name, live_sample, require_xc=True):
    """Full-size parity of a config:
    * every row of the device per-edge table against the independent CPU
      cross-check (tests/golden/crosscheck_<cfg>.json, one sha256 per 65536
      rows; the cross-check is itself pinned to the literal oracle and the
      reference, tests/test_crosscheck.py);
    * the literal oracle's _micro_edge rows of the survey sample (uniform +
      top-1k by w_e + top-100-hub edges) and its _count_edge rows of 1M
      uniform edges (oracle_<cfg>_{micro,count}_sample, tools/make_big_fixtures.py);
    * a live oracle sample computed here, global counts against the full
      C-oracle census (C3) and the cross-check (C3, C5), and the two device
      routes / validate() identities."""
    import json
    raw = W.config_graph(name)
    g = gd.Graph.from_edges(raw.pairs, _declared_n=raw.n)
    f = gd.graphlet_census(g)
    tab, f2 = gd.micro_census_table(g)
    tab = np.asarray(tab)
    assert f2 == f  # two device routes (global closure vs per-edge sums)
    assert gd.frequencies_from_micro(g, tab) == f  # dual route over the table
    f.validate()
    edges = np.asarray(g.edges)
    xcp = GOLDEN / f"crosscheck_{name}.json"
    if xcp.exists():  # every row and the 17 counts against the independent cross-check
        xc = json.loads(xcp.read_text())
        assert xc["m"] == g.m and sha(edges) == xc["edges_sha256"]
        assert f.counts == int_counts(xc["counts"])
        got = _chunk_sha(tab, xc["chunk_rows"])
        bad = [i for i, (a, b) in enumerate(zip(got, xc["chunk_sha256"])) if a != b]
        assert len(got) == len(xc["chunk_sha256"]) and not bad, \
            f"{len(bad)} of {len(got)} table chunks differ, first rows {bad[:1] and bad[0] * xc['chunk_rows']}"
    else:
        assert require_xc is False, f"{xcp.name} missing"
    z = np.load(GOLDEN / f"oracle_{name}_micro_sample.npz")
    assert str(z["edges_sha256"]) == sha(edges)
    assert np.array_equal(tab[z["idx"]], z["rows"])
    cs = json.loads((GOLDEN / f"oracle_{name}_count_sample.json").read_text())
    idx = count_sample(g.m, cs["k"])
    assert sha(idx) == cs["idx_sha256"]
    assert _chunk_sha(count_rows_from_table(tab, idx), cs["chunk"]) == cs["chunk_sha256"]
    # a live literal-oracle sample on this box (independent of the fixtures)
    rng = np.random.default_rng(2024)
    idx = rng.choice(g.m, live_sample, replace=False)
    assert np.array_equal(tab[idx], O.micro_rows(edges, g.n, idx))
    full = GOLDEN / f"oracle_{name}.json"  # full census by the C oracle (tools/)
    if full.exists():
        d = json.loads(full.read_text())
        assert d["m"] == g.m and f.counts == int_counts(d["counts"])
    return g, f


def test_config3_rmat20_full_size():
    g, f = _big_parity("c3_rmat20", 400)
    assert g.m == 15702776
    assert f.counts["g3_1"] == 423856269 and f.counts["g4_1"] == 17041022655


@pytest.mark.slow
def test_config5_chung_lu_4m_full_size():
    # every row of the 64.6M-row table and the 17 counts against the committed
    # cross-check fixture (4.6 h of CPU, tools/make_crosscheck_fixtures.py),
    # plus the literal-oracle samples
    g, f = _big_parity("c5_chung_lu_4m", 100)
    assert g.n == 4_000_000 and g.m == 64623472
    assert f.counts["g4_4"] == 1254097230619 and f.counts["g3_1"] == 7146286343


@pytest.mark.parametrize("force", ["", "tri_gmem,c4_coop", "c4_hub32"])
def test_emulated_shards_match(force):
    """Frame sharding (multi-GPU partition) emulated on one GPU: every shard
    count gives the unsharded result bit for bit."""
    code = r'''
import sys, numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r)
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200.distributed import graphlet_census_sharded, micro_census_table_sharded
import test_gpu_parity as T
for name, n, edges in T._dense_cases():
    g = gd.Graph(n, edges)
    tab, f = gd.micro_census_table(g)
    for k in (2, 3, 5):
        assert graphlet_census_sharded(g, None, k) == f, (name, k)
        t2, f2 = micro_census_table_sharded(g, None, k)
        assert f2 == f and np.array_equal(np.asarray(t2), np.asarray(tab)), (name, k)
print("ok")
''' % (str(GOLDEN.parent.parent), str(GOLDEN.parent))
    env = dict(os.environ, GD_FORCE_PATH=force)
    if "wide_slots" in force:  # 64-bit per-slot sums even where 32 bits suffice
        env["GD_WIDE_SLOTS"] = "1"
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def _mixed_hub_graph():
    """K_{2,66000} (two frames whose counters may pass 16 bits: the u32 hub
    path) plus a dense block (u16 heavy frames): the schedule mixes both
    kinds of heavy frame, which a sharded census must deal out consistently."""
    hubs = np.array([[0, 2 + i] for i in range(66000)] + [[1, 2 + i] for i in range(66000)],
                    dtype=np.int64)
    rng = np.random.default_rng(9)
    base = 70000
    iu = np.triu_indices(400, 1)
    mask = rng.random(len(iu[0])) < 0.6
    block = np.stack([iu[0][mask], iu[1][mask]], 1).astype(np.int64) + base
    edges = np.concatenate([hubs, block])
    return base + 400, edges


@pytest.mark.parametrize("force", ["", "c4_coop", "c4_coop,c4_cluster", "c4_coop,c4_flow"])
def test_sharded_mixed_u16_u32_heavy_frames(force):
    """with u32 hub frames among the heavy frames, every shard
    count must still see every u16 frame (cluster, flow and tile paths)."""
    code = r'''
import sys, numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r)
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200.distributed import graphlet_census_sharded, micro_census_table_sharded
from oracle import oracle as O
import test_gpu_parity as T
n, edges = T._mixed_hub_graph()
g = gd.Graph(n, edges)
tab, f = gd.micro_census_table(g)
rows, sums = O.crosscheck_table(edges, n)
assert np.array_equal(np.asarray(tab), rows)
assert f.counts == O.close(sums, n, len(edges))
assert gd.last_stats(g)["c4_u32_hub_frames"] >= 1
for k in (2, 3):
    assert graphlet_census_sharded(g, None, k) == f, k
    t2, f2 = micro_census_table_sharded(g, None, k)
    assert f2 == f and np.array_equal(np.asarray(t2), np.asarray(tab)), k
print("ok")
''' % (str(GOLDEN.parent.parent), str(GOLDEN.parent))
    env = dict(os.environ, GD_FORCE_PATH=force)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_small_graph_kernel_and_pipeline_agree():
    """The one-launch small-graph kernel (reference marks protocol) and the
    multi-pass pipeline give identical tables on the golden graphs and the
    dense cases; the small path is the one taken by default for them."""
    code = r'''
import sys, numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r)
import paper_1506_04322_b200 as gd
from helpers import small_graphs
import test_gpu_parity as T
out = []
for name, n, edges, counts, micro in small_graphs():
    if not len(edges):
        continue
    g = gd.Graph(n, edges)
    tab, f = gd.micro_census_table(g)
    out.append((np.asarray(tab).copy(), f.counts, gd.last_stats(g).get("small_graph_path", 0)))
for name, n, edges in T._dense_cases():
    g = gd.Graph(n, edges)
    tab, f = gd.micro_census_table(g)
    out.append((np.asarray(tab).copy(), f.counts, gd.last_stats(g).get("small_graph_path", 0)))
np.save(sys.argv[1], np.array(out, dtype=object), allow_pickle=True)
print("ok")
''' % (str(GOLDEN.parent.parent), str(GOLDEN.parent))
    import tempfile
    res = {}
    with tempfile.TemporaryDirectory() as d:
        for small in ("1", "0"):
            path = os.path.join(d, f"r{small}.npy")
            r = subprocess.run([sys.executable, "-c", code, path], capture_output=True, text=True,
                               timeout=600, env=dict(os.environ, GD_SMALL=small))
            assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
            res[small] = np.load(path, allow_pickle=True)
    assert len(res["1"]) == len(res["0"])
    assert sum(int(x[2]) for x in res["1"]) >= len(res["1"]) - 8  # default: mostly the small path
    assert sum(int(x[2]) for x in res["0"]) == 0
    for a, b in zip(res["1"], res["0"]):
        assert np.array_equal(a[0], b[0]) and a[1] == b[1]
