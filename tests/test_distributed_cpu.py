"""Multi-rank host logic on CPU (gloo, world_size 2): graph sharding and the
ordered gather of feature rows.  The per-graph census is the CPU oracle here
(the device path is covered by the -m gpu tests, incl. emulated shards)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1506_04322_b200.distributed import feature_matrix_distributed, shard_bounds


def test_shard_bounds_cover_everything():
    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 8):
        w = rng.integers(1, 1000, size=97)
        b = shard_bounds(w, world)
        assert b[0] == 0 and b[-1] == 97 and all(x <= y for x, y in zip(b, b[1:]))
        parts = [w[b[i]:b[i + 1]].sum() for i in range(world)]
        assert sum(parts) == w.sum()
        assert max(parts) <= w.sum() / world + w.max()
    assert shard_bounds([], 4) == [0, 0, 0, 0, 0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    from types import SimpleNamespace
    from helpers import small_graphs
    from oracle import oracle as O
    from paper_1506_04322_b200 import GraphletFrequencies
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cases = small_graphs()[:60]
    graphs = [SimpleNamespace(n=n, m=len(e), edges=e) for _, n, e, _, _ in cases]

    def oracle_census(g):
        return GraphletFrequencies(counts=O.census(g.edges, g.n), n=g.n, m=g.m)

    fm = feature_matrix_distributed(graphs, census_fn=oracle_census)
    want = np.asarray([[c[k] for k in fm.class_ids] for _, _, _, c, _ in cases], dtype=np.float64)
    out[rank] = bool(np.array_equal(fm.rows, want) and fm.labels == [f"graph_{i}" for i in range(60)])
    dist.destroy_process_group()


def test_feature_matrix_distributed_gloo_world2():
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        assert out[0] and out[1]


def test_shard_rows_match_the_library():
    """Python and C (gd_shard_rows) agree on the owned ranges; the ranges
    tile [0, m) in rank order."""
    import ctypes
    from paper_1506_04322_b200 import _native as N
    from paper_1506_04322_b200.distributed import shard_rows
    L = N.load_library()
    for m in (0, 1, 7, 10, 15702776, 64623472):
        for world in (1, 2, 3, 8):
            prev = 0
            for r in range(world):
                a, b = ctypes.c_int64(), ctypes.c_int64()
                assert L.gd_shard_rows(m, r, world, ctypes.byref(a), ctypes.byref(b)) == 0
                assert (a.value, b.value) == shard_rows(m, r, world)
                assert a.value == prev and b.value >= a.value
                prev = b.value
            assert prev == m


def _rows_worker(rank, world, port, out):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    from oracle import oracle as O
    from paper_1506_04322_b200 import workloads as W
    from paper_1506_04322_b200.distributed import gather_table, shard_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    raw = W.chung_lu(3000, 2.1, 8.0, 400.0, seed=11)
    edges = O.canonical_edges(raw.pairs)
    n, m = raw.n, len(edges)
    full, _ = O.crosscheck_table(edges, n, threads=1)
    e0, e1 = shard_rows(m, rank, world)
    block = full[e0:e1]  # what this rank's finalize writes
    table = gather_table(block, m)
    # the exact 128-bit totals: each rank's sums over its rows, gathered, added
    part = O.sums_from_rows(block, n, m)
    parts = [None] * world
    dist.all_gather_object(parts, part)
    total = [sum(p[k] for p in parts) for k in range(13)]
    out[rank] = bool(np.array_equal(table, full) and O.close(total, n, m) == O.census(edges, n))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_owned_rows_gather_and_exact_sums_gloo(world):
    """Host side of the multi-GPU census on CPU ranks: owned row blocks in
    rank order rebuild the whole table, and per-rank 128-bit sums over the
    owned rows add up to the global census."""
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_rows_worker, args=(world, port, out), nprocs=world, join=True)
        assert all(out[r] for r in range(world))
