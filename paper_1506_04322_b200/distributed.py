"""Multi-GPU census: one process per GPU, torch.distributed for bootstrap.

Single large graph: ``CensusComm`` wraps the library's NCCL communicator
(gd_comm_*); ``graphlet_census_sharded`` / ``micro_census_table_sharded``
deal the counting frames round-robin to the ranks.  Each rank owns the
contiguous canonical edge range ``shard_rows(m, rank, world)`` (SURVEY
8(e)): the per-edge triangle counters are all-reduced after pass A, the
per-edge partial sums of passes B and C are reduce-scattered onto their
owners, every rank finalizes only its rows, and the 128-bit totals are
all-gathered and added (the reference's fixed-order merge of worker
accumulators, parallel.py:138-143).  Every rank returns the global counts
and its own block of the per-edge table (``gather_table`` assembles the
whole table where it is wanted).  ``virtual_ranks=K`` without a
communicator emulates K shards on one GPU (the single-GPU check of the
partition: the packing, ownership and per-range finalize all run).

Many small graphs (config 4): ``feature_matrix_distributed`` shards the
graphs by rank (contiguous, balanced by edge count) with no data-path
collective, then all-gathers the rows.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .analytics import FeatureMatrix, feature_matrix
from .census import CensusSums, frequencies_from_sums
from .classes import classes_for
from .errors import ConsistencyError
from .graph import Graph


class CensusComm:
    """NCCL communicator of libgdgpu for the ranks of a torch.distributed
    group (the unique id is broadcast through the group)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        N.require_device()
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        uid = [None]
        if self.rank == 0:
            buf = ctypes.create_string_buffer(128)
            N.check(N.lib().gd_comm_unique_id(buf))
            uid[0] = bytes(buf.raw)
        dist.broadcast_object_list(uid, src=0, group=group)
        out = ctypes.c_void_p()
        N.check(N.lib().gd_comm_init(uid[0], self.rank, self.world, ctypes.byref(out)))
        self._p = out.value

    def close(self):
        if getattr(self, "_p", None):
            N.lib().gd_comm_free(self._p)
            self._p = None

    def __del__(self):
        self.close()


def _sharded(g, comm, virtual_ranks, per_edge, table_ptr, flags):
    dg = g if isinstance(g, Graph) else Graph.from_reference(g)
    sums = np.zeros(2 * N.NUM_SUMS, dtype=np.uint64)
    seen = np.zeros(1, dtype=np.int64)
    N.check(N.lib().gd_census_sharded(dg.handle, comm._p if comm else None,
                                      int(virtual_ranks), 1 if per_edge else 0, table_ptr,
                                      flags, N.ptr(sums, ctypes.c_uint64), N.ptr(seen)))
    if int(seen[0]) != dg.m:
        raise ConsistencyError(f"processed {int(seen[0])} edges, expected {dg.m}")
    return frequencies_from_sums(CensusSums.from_tuple(N.wide(sums)), dg.n, dg.m)


def graphlet_census_sharded(g, comm: CensusComm | None = None, virtual_ranks: int = 1):
    """graphlet_census with the frames split over the ranks of ``comm``."""
    if int(g.m) == 0:
        return frequencies_from_sums(CensusSums(), int(g.n), 0)
    return _sharded(g, comm, virtual_ranks, False, None, 0)


def shard_rows(m: int, rank: int, world: int) -> tuple[int, int]:
    """Owned canonical edge range [e0, e1) of ``rank``: blocks of
    ceil(m / world) edges (the library's gd_shard_rows)."""
    M = -(-int(m) // world) if world > 0 else int(m)
    e0 = min(int(m), rank * M)
    return e0, min(int(m), e0 + M)


def micro_census_table_sharded(g, comm: CensusComm | None = None, virtual_ranks: int = 1,
                               device_out: int | None = None):
    """micro_census_table with the frames split over the ranks of ``comm``.
    With a communicator the returned table holds this rank's rows
    ``shard_rows(m, comm.rank, comm.world)``; emulated (``virtual_ranks``)
    it is the whole table."""
    m = int(g.m)
    if m == 0:
        return np.zeros((0, N.NUM_MICRO), np.int64), frequencies_from_sums(CensusSums(), int(g.n), 0)
    if device_out is not None:
        return None, _sharded(g, comm, virtual_ranks, True, ctypes.c_void_p(int(device_out)),
                              N.GD_OUTPUT_DEVICE)
    e0, e1 = shard_rows(m, comm.rank, comm.world) if comm is not None else (0, m)
    table = N.pinned_empty((e1 - e0, N.NUM_MICRO))
    return table, _sharded(g, comm, virtual_ranks, True, N.vptr(table), 0)


def gather_table(block: np.ndarray, m: int, group=None) -> np.ndarray:
    """The whole (m, 10) table on every rank from the ranks' owned blocks
    (torch.distributed all-gather of the row blocks, in rank order)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    M = -(-int(m) // world)
    pad = np.zeros((M, N.NUM_MICRO), dtype=np.int64)
    pad[:len(block)] = block
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else \
        torch.device("cpu")
    mine = torch.from_numpy(pad).to(dev)
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    return torch.cat(parts).cpu().numpy()[:int(m)]


def shard_bounds(weights, world: int) -> list[int]:
    """Contiguous split of items with the given weights into ``world`` parts
    of near-equal total weight; returns world+1 boundaries."""
    w = np.asarray(weights, dtype=np.float64)
    if len(w) == 0:
        return [0] * (world + 1)
    c = np.concatenate([[0.0], np.cumsum(w)])
    targets = c[-1] * np.arange(world + 1) / world
    b = np.searchsorted(c, targets, side="left").tolist()
    b[0], b[-1] = 0, len(w)
    for i in range(1, world + 1):
        b[i] = max(b[i], b[i - 1])
    return b


def feature_matrix_distributed(graphs, labels=None, group=None, census_fn=None,
                               log_scale: bool = False, normalize: bool = False) -> FeatureMatrix:
    """feature_matrix over the ranks of ``group``: each rank counts a
    contiguous, edge-balanced slice of the graphs (one batched device pass,
    or ``census_fn`` per graph), then the rows are all-gathered in order."""
    import torch.distributed as dist
    graphs = list(graphs)
    if labels is None:
        labels = [f"graph_{i}" for i in range(len(graphs))]
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    b = shard_bounds([max(1, int(g.m)) for g in graphs], world)
    lo, hi = b[rank], b[rank + 1]
    if hi > lo:
        part = feature_matrix(graphs[lo:hi], labels[lo:hi], log_scale=log_scale,
                              normalize=normalize, census_fn=census_fn)
        payload = (part.labels, part.rows.tolist(), part.seconds, part.skipped)
    else:
        payload = ([], [], [], [])
    gathered = [None] * world
    dist.all_gather_object(gathered, payload, group=group)
    lab, rows, secs, skipped = [], [], [], []
    for p in gathered:
        lab += p[0]
        rows += p[1]
        secs += p[2]
        skipped += p[3]
    class_ids = classes_for(2) + classes_for(3) + classes_for(4)
    return FeatureMatrix(class_ids, lab,
                         np.asarray(rows, dtype=np.float64).reshape(len(rows), len(class_ids)),
                         secs, skipped)
