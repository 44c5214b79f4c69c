"""Edge cases of the device census beyond the reference fixtures: pass-C
counters beyond 16 bits on the default schedule, concurrent censuses from
several host threads, and a seeded random sweep against the oracle (the
reference's hypothesis suite draws graphs with n <= 10,
test_census.py:260-263; this sweep goes wider and denser)."""

from concurrent.futures import ThreadPoolExecutor
from math import comb

import numpy as np
import pytest

import paper_1506_04322_b200 as gd
from oracle import oracle as O
from paper_1506_04322_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _k2n(N: int):
    """K_{2,N}: hubs 0 and 1, leaves 2..N+1."""
    leaves = np.arange(2, N + 2, dtype=np.int64)
    edges = np.concatenate([np.stack([np.zeros(N, np.int64), leaves], 1),
                            np.stack([np.ones(N, np.int64), leaves], 1)])
    return N + 2, edges


def test_hub_counters_beyond_16_bits_default_schedule():
    """The top hub's counter for the other hub reaches N = 70,000 > 65,535,
    so the default schedule must take the 32-bit hub path (no forcing)."""
    N = 70_000
    n, edges = _k2n(N)
    g = gd.Graph.from_edges(edges, gd.ParseOptions(num_vertices=n))
    tab, f = gd.micro_census_table(g)
    st = gd.last_stats(g)
    assert st["c4_u32_hub_frames"] >= 1
    assert st["narrow_slots"] == 0  # max degree 70,000: 64-bit per-slot sums
    f.validate()
    c = f.counts
    assert c["g4_4"] == comb(N, 2)          # 4-cycles: two leaves x the hub pair
    assert c["g4_5"] == 2 * comb(N, 3)      # 3-stars at either hub
    assert c["g3_1"] == c["g4_1"] == c["g4_2"] == c["g4_3"] == c["g4_6"] == 0
    tab = np.asarray(tab)
    # RAW_MICRO_FIELDS (census.py:95-97): t su sv cl cy uu vv ts ti si
    assert (tab[:, 0] == 0).all() and (tab[:, 3] == 0).all()
    assert (tab[:, 4] == N - 1).all()       # every hub-leaf edge: N - 1 cycles
    assert gd.graphlet_census(g) == f
    assert gd.frequencies_from_micro(g, tab) == f
    # the same graph at a size the oracle finishes: identical rows
    n2, e2 = _k2n(300)
    g2 = gd.Graph(n2, O.canonical_edges(e2, n2))
    assert np.array_equal(np.asarray(gd.micro_table(g2)), O.micro_rows(np.asarray(g2.edges), n2))


def _random_graphs(count: int, seed: int):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        n = int(rng.integers(2, 60))
        p = float(rng.choice([0.05, 0.2, 0.5, 0.9]))
        iu = np.triu_indices(n, 1)
        mask = rng.random(len(iu[0])) < p
        out.append((n, np.stack([iu[0][mask], iu[1][mask]], 1).astype(np.int64)))
    return out


def test_seeded_random_sweep_matches_oracle():
    for n, edges in _random_graphs(150, seed=2024):
        g = gd.Graph(n, edges)
        tab, f = gd.micro_census_table(g)
        assert f.counts == O.census(edges, n), (n, len(edges))
        assert np.array_equal(np.asarray(tab), O.micro_rows(edges, n)), (n, len(edges))


def test_concurrent_censuses_from_threads():
    """Calls are synchronous and thread-safe: several host threads counting
    the same graph and different graphs at once get the sequential results."""
    raws = [W.chung_lu(20_000, 2.1, 8.0, 800.0, seed=s) for s in (1, 2, 3)]
    graphs = [gd.Graph.from_edges(r.pairs, gd.ParseOptions(num_vertices=r.n)) for r in raws]
    want = [(gd.graphlet_census(g), np.asarray(gd.micro_table(g)).copy()) for g in graphs]
    jobs = [i % len(graphs) for i in range(12)]  # each graph from four threads

    def run(i):
        g = graphs[i]
        tab, f = gd.micro_census_table(g)
        return i, f, np.asarray(tab).copy(), gd.graphlet_census(g)

    with ThreadPoolExecutor(max_workers=6) as ex:
        for i, f, tab, fg in ex.map(run, jobs):
            assert f == want[i][0] and fg == want[i][0]
            assert np.array_equal(tab, want[i][1])


def test_nccl_sharded_path_single_rank():
    """The real-communicator path of the frame-sharded census (NCCL loaded
    with dlopen, communicator from a torch.distributed group, all-reduce of
    the 64-bit slot partials, all-gather of the totals) at world size 1 in a
    subprocess: identical table and counts to the single-GPU census."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    code = r'''
import sys, numpy as np
sys.path.insert(0, %r)
import torch.distributed as dist
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:29533", rank=0, world_size=1)
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import workloads as W
from paper_1506_04322_b200.distributed import CensusComm, micro_census_table_sharded, graphlet_census_sharded
raw = W.chung_lu(30_000, 2.1, 8.0, 1500.0, seed=9)
g = gd.Graph.from_edges(raw.pairs, gd.ParseOptions(num_vertices=raw.n))
tab0, f0 = gd.micro_census_table(g)
comm = CensusComm()
tab1, f1 = micro_census_table_sharded(g, comm)
f2 = graphlet_census_sharded(g, comm)
assert f1 == f0 and f2 == f0, (f0, f1, f2)
assert np.array_equal(np.asarray(tab1), np.asarray(tab0))
comm.close()
dist.destroy_process_group()
print("ok")
''' % str(root)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, MASTER_ADDR="127.0.0.1"))
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
