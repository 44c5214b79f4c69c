#!/usr/bin/env python
"""Benchmark of the B200 edge-centric graphlet census (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3_rmat20] [--mode per_edge|global]

One "step" is one census pass over the whole synthetic graph of the chosen
configuration (default: config 3, R-MAT scale 20, per-edge mode = the full
micro_table plus the 13 global sums).  `value` is edges/s with the graph
already resident in HBM (device CSR built before the timed region), timed
with the library's CUDA events; `e2e` is the public API from host memory:
H2D of the raw pairs + device sanitise/CSR build + census + D2H of the per-edge
table.  N>1 (torchrun): the same graph is counted once with its frames
sharded over the N GPUs (NCCL all-reduce of the per-slot partial counters
between passes), so total work is fixed (strong scaling).

`--impl reference` times the reference algorithm's CPU restatement
(oracle/census_oracle.c, all host threads) on bounded samples of the same
workload; it is the only other place this script executes oracle/.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "edges/sec for exact k=3,4 graphlet counts (1 B200); achieved HBM GB/s vs peak"
CONFIG_DESC = {
    "c1_er": "Erdos-Renyi G(n=2000, m=10000), seed 1506",
    "c2_chung_lu": "Chung-Lu n=100000, gamma 2.1, mean degree 10, cap 5000, seed 4322",
    "c3_rmat20": "R-MAT scale 20, edge factor 16, (a,b,c,d)=(0.57,0.19,0.19,0.05), seed 20",
    "c5_chung_lu_4m": "Chung-Lu n=4000000, gamma 1.9, mean degree 30, cap 100000, seed 1904",
}


DEBUG = bool(os.environ.get("GD_BENCH_DEBUG"))


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


class Dist:
    """torch.distributed plumbing (only imported for N > 1)."""

    def __init__(self, world: int, local_rank: int, backend: str):
        self.world = world
        self.torch = None
        if world > 1:
            import torch
            import torch.distributed as td
            self.torch = torch
            self.td = td
            if backend == "nccl":
                torch.cuda.set_device(local_rank)
                self.device = torch.device("cuda", local_rank)
            else:
                self.device = torch.device("cpu")
            td.init_process_group(backend=backend)

    def barrier(self):
        if self.torch is not None:
            self.td.barrier()
            if self.device.type == "cuda":
                self.torch.cuda.synchronize()

    def max(self, x: float) -> float:
        if self.torch is None:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.device)
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.torch is not None:
            self.td.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self) -> dict | None:
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
            out, _ = self.p.communicate()
        sms, maxes, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sms.append(float(f[1]))
                maxes.append(float(f[2]))
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sms:
            return None
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": max(maxes),
                "reasons": sorted(reasons), "samples": len(sms)}


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except (KeyError, ValueError):
            pass
    return 6650.0, "fallback"


PHASE_KERNELS = {  # census phase -> the kernels it launches (name prefixes)
    "c4_coop": ("k_c4_tiles", "k_c4_flow", "k_c4_cluster", "k_c4_hub", "k_c4_rounds"),
    "tri_frames": ("k_tri_frames",),
}


def ncu_traffic(config: str, mode: str, phase: str):
    """(DRAM bytes of the phase's kernels in one census, the largest of them by
    time with its share, DRAM bytes of one whole census) from the committed ncu
    launch-list summary (profiles/ncu_summary.json, made by tools/ncu_sum.py)."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None, None, None
    try:
        e = json.loads(p.read_text())[f"{config}/{mode}"]
        ks = [(k, v) for k, v in e["kernels"].items()
              if k.startswith(PHASE_KERNELS.get(phase, ()))]
        if not ks:
            return None, None, e["census_dram_bytes"]
        top = max(ks, key=lambda kv: kv[1]["ms"])
        total = sum(v["dram_bytes"] for _, v in ks)
        return total, {"name": top[0], "share": top[1]["share"],
                       "launches": sum(v["launches"] for _, v in ks)}, e["census_dram_bytes"]
    except (KeyError, ValueError):
        return None, None, None


def roofline_block(config, mode, phases, stats, n, m, deg, ms, peak, peak_kind) -> dict:
    """Roofline of the dominant kernel.

    achieved = algorithmic bytes of one launch / its live CUDA-event time.
    The algorithmic bytes are the item stream of the frame / wedge algorithm
    (what it must move through the memory system if nothing were cached):
      pass C heavy frames: 4 B (col[] entry of the wedge's end x) per heavy
        wedge per sweep, plus in per-edge mode a 4 B slot update per wedge
        (count + use sweeps: 12 B / wedge; global: 4 B / wedge);
      pass A triangle frames: 4 B per frame item (col[] entry probed).
    traffic = the ncu-measured DRAM bytes of that kernel (profiles/
    ncu_summary.json, same code); hbm_measured turns traffic into the HBM
    fraction actually used (always <= 1); compulsory = CSR read once + per-edge
    table written once; effective = SURVEY 8(d)'s B_alg over the census time
    (the per-edge formulation's bytes, which this algorithm never reads, so it
    may exceed 1 and is not a bound)."""
    per_edge = mode == "per_edge"
    wh = stats.get("c4_heavy_wedges", 0)
    items = stats.get("tri_items", 0)
    models = {
        "c4_coop": (4 * wh * (3 if per_edge else 1),
                    f"{wh} heavy wedges x {'(4 B col per sweep x 2 + 4 B slot update)' if per_edge else '4 B col'}"),
        "tri_frames": (4 * items, f"{items} frame items x 4 B col"),
    }
    dom = max(((k, v) for k, v in phases.items() if k in models), key=lambda kv: kv[1],
              default=("", 0.0))
    alg, model = models.get(dom[0], (0, ""))
    traffic, ncu_kernel, census_dram = ncu_traffic(config, mode, dom[0])
    t = max(dom[1], 1e-9) / 1e3
    achieved = alg / t / 1e9
    sum_d2 = int(np.dot(deg, deg))
    b_alg = m * (8 + 4 * 8 + 8 * (10 if per_edge else 0)) + 4 * sum_d2
    compulsory = 8 * (n + 1) + 8 * m * 2 + (80 * m if per_edge else 0)
    out = {"bound": "hbm", "kernel": (ncu_kernel or {}).get("name", dom[0]), "phase": dom[0],
           "phase_ms": dom[1], "share_of_census": dom[1] / max(ms, 1e-9),
           "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
           "algorithmic_bytes": alg, "model": model, "traffic": traffic,
           "phase_launches": (ncu_kernel or {}).get("launches"),
           "peak_source": peak_kind}
    if traffic:
        out["hbm_measured"] = {
            "kernel_gbs": traffic / t / 1e9, "kernel_frac": traffic / t / 1e9 / peak,
            "census_gbs": census_dram / (ms / 1e3) / 1e9 if census_dram else None,
            "census_frac": census_dram / (ms / 1e3) / 1e9 / peak if census_dram else None,
            "source": "ncu dram__bytes_read.sum + dram__bytes_write.sum (profiles/ncu_summary.json)"
                      " over this run's CUDA-event time"}
    out["compulsory"] = {"bytes": compulsory, "gbs": compulsory / (ms / 1e3) / 1e9,
                         "frac": compulsory / (ms / 1e3) / 1e9 / peak,
                         "model": "CSR offsets + neighbour lists read once" +
                                  (", int64 (m, 10) table written once" if per_edge else "")}
    out["effective_b_alg"] = {"bytes": b_alg, "gbs": b_alg / (ms / 1e3) / 1e9,
                              "frac_effective": b_alg / (ms / 1e3) / 1e9 / peak,
                              "model": "SURVEY 8(d): m(8+4o+8K) + 4 sum d^2 (both adjacency "
                                       "lists per edge; not read by this algorithm)"}
    return out


def load_graph(config: str):
    from paper_1506_04322_b200 import workloads as W
    return W.config_graph(config)


# ---------------------------------------------------------------------------
# CPU legs (oracle restatement of the reference algorithm)
# ---------------------------------------------------------------------------
def cpu_sample_run(og, mode: str, k: int, seed: int):
    """Time the reference algorithm on k uniformly sampled edge jobs."""
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(og.m, size=min(k, og.m), replace=False))
    t0 = time.perf_counter()
    if mode == "per_edge":
        og.micro_rows(idx)
    else:
        og.census_sums(order=idx, batch=1)
    return time.perf_counter() - t0, len(idx)


def cpu_calibrate(og, mode: str, budget_s: float):
    k = 64
    while True:
        t, kk = cpu_sample_run(og, mode, k, seed=1)
        if t > 0.5 or kk >= og.m:
            break
        k *= 4
    rate = kk / max(t, 1e-9)
    return int(max(16, min(og.m, rate * budget_s)))


def oracle_graph(raw):
    from oracle import oracle as O
    O.build()
    edges = O.canonical_edges(raw.pairs)
    return O.OracleGraph(edges, raw.n)


def cpu_baseline(raw, mode: str, budget_s: float) -> dict:
    og = oracle_graph(raw)
    k = cpu_calibrate(og, mode, budget_s)
    t, kk = cpu_sample_run(og, mode, k, seed=7)
    full = t * og.m / kk
    return {"value": og.m / full, "unit": "edges/s", "cores": os.cpu_count(), "kind": "port",
            "extrapolated": True,
            "sample": f"{kk} uniformly sampled edge jobs of the {og.m}-edge graph "
                      f"({'_micro_edge' if mode == 'per_edge' else '_count_edge'} C restatement, "
                      f"{os.cpu_count()} OpenMP threads) in {t:.2f} s; full census "
                      f"extrapolated = {full:.1f} s"}


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return 0
    raw = load_graph(args.config)
    og = oracle_graph(raw)
    k = cpu_calibrate(og, args.mode, args.cpu_budget)
    for i in range(args.warmup):
        cpu_sample_run(og, args.mode, max(16, k // 8), seed=100 + i)
    times = []
    for i in range(args.steps):
        t, kk = cpu_sample_run(og, args.mode, k, seed=1000 + i)
        times.append(t * og.m / kk)  # extrapolated full-census seconds
    full = statistics.mean(times)
    value = og.m / full
    line = {
        "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": full * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": args.config, "mode": args.mode, "graph": CONFIG_DESC[args.config],
                   "n": og.n, "m": og.m, "parallelism": "cpu threads"},
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": os.cpu_count(),
                         "kind": "port", "extrapolated": True,
                         "sample": f"each step: {k} uniformly sampled edge jobs, full census "
                                   f"time extrapolated x m/k"},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------
def run_ours(args, rank: int, world: int, local_rank: int):
    import paper_1506_04322_b200 as gd
    from paper_1506_04322_b200 import _native as N

    L = N.load_library()
    N.check(L.gd_set_device(local_rank))
    dist = Dist(world, local_rank, "nccl")
    raw = load_graph(args.config)
    pairs = N.pinned_empty(raw.pairs.shape, np.int64)
    pairs[...] = raw.pairs

    g = gd.Graph.from_edges(pairs, gd.ParseOptions(num_vertices=raw.n))
    n, m = g.n, g.m
    per_edge = args.mode == "per_edge"
    dtab = L.gd_device_alloc(max(1, m * 10 * 8)) if per_edge else None
    htab = N.pinned_empty((m, 10), np.int64) if per_edge else None
    comm = None
    if world > 1:
        from paper_1506_04322_b200.distributed import CensusComm
        comm = CensusComm()

    def census(graph, device_out=None, out=None):
        if comm is not None:
            from paper_1506_04322_b200.distributed import (graphlet_census_sharded,
                                                           micro_census_table_sharded)
            if per_edge:
                # this rank's rows (shard_rows) of the table
                t, f = micro_census_table_sharded(graph, comm, device_out=device_out)
                if out is not None:
                    from paper_1506_04322_b200.distributed import shard_rows
                    e0, e1 = shard_rows(graph.m, comm.rank, comm.world)
                    out[e0:e1] = t
                return f
            return graphlet_census_sharded(graph, comm)
        if per_edge:
            _, f = gd.micro_census_table(graph, device_out=device_out, out=out)
            return f
        return gd.graphlet_census(graph)

    def census_global(graph):
        if comm is not None:
            from paper_1506_04322_b200.distributed import graphlet_census_sharded
            return graphlet_census_sharded(graph, comm)
        return gd.graphlet_census(graph)

    def census_resident():
        return census(g, device_out=dtab)

    for _ in range(args.warmup):
        f_ref = census_resident()

    # --- device-resident timed region --------------------------------------
    clocks = ClockSampler(local_rank)
    clocks.start()
    dist.barrier()
    step_ms, phases, launches = [], {}, 0
    t_wall0 = time.perf_counter()
    for _ in range(args.steps):
        L.gd_flush_l2()
        f = census_resident()
        tm = gd.last_timings(g)
        step_ms.append(sum(tm.values()))
        for k, v in tm.items():
            phases[k] = phases.get(k, 0.0) + v / args.steps
        launches += gd.last_stats(g).get("launches", 0)
        if f != f_ref:
            raise SystemExit("census result changed between steps")
    dist.barrier()
    wall_ms = (time.perf_counter() - t_wall0) * 1e3 / args.steps
    clk = clocks.stop()
    ms = dist.max(statistics.mean(step_ms))
    stats = gd.last_stats(g)

    # secondary: the global-only census on the same resident graph
    glob = None
    if per_edge and args.global_too:
        gms = []
        for i in range(3):
            L.gd_flush_l2()
            fg = census_global(g)
            if i:
                gms.append(sum(gd.last_timings(g).values()))
        if fg != f_ref:
            raise SystemExit("global census differs from per-edge census")
        gm = dist.max(statistics.mean(gms))
        glob = {"ms_per_step": gm, "value": m / (gm / 1e3), "unit": "edges/s"}

    # the resident graph (and its census workspace) is released before the
    # end-to-end runs, which build their own device graph every step
    deg = np.asarray(g.degrees, dtype=np.int64)
    del g
    # --- end to end through the public API (host memory both ways) ----------
    # headline: the drop-in default call a user makes, from the pageable
    # numpy pairs the generator returned -> Graph.from_edges -> micro_table
    # (a fresh int64 table every step, returned as a numpy array; the library
    # recycles the page-locked blocks of tables the caller has dropped).
    # Beside it: the same calls from page-locked pairs into a reused output.
    dist.barrier()
    e2e_warm = max(1, args.warmup)

    def e2e_leg(src, out):
        times = []
        for i in range(args.steps + e2e_warm):
            t0 = time.perf_counter()
            g2 = gd.Graph.from_edges(src, gd.ParseOptions(num_vertices=raw.n))
            if comm is not None or not per_edge:
                f2 = census(g2, out=out if per_edge else None)
                tab2 = None
            elif out is None:
                tab2, f2 = gd.micro_census_table(g2)
            else:
                tab2, f2 = gd.micro_census_table(g2, out=out)
            dt = (time.perf_counter() - t0) * 1e3
            if DEBUG:
                print(f"e2e step {i}: {dt:.1f} ms (device {sum(gd.last_timings(g2).values()):.1f})",
                      file=sys.stderr, flush=True)
            del g2, tab2
            if i >= e2e_warm:
                times.append(dt)
            if f2 != f_ref:
                raise SystemExit("end-to-end census differs from the resident one")
        return times

    e2e_ms = e2e_leg(raw.pairs, None)
    e2e_pin_ms = e2e_leg(pairs, htab)
    dist.barrier()
    # median over steps (median of the runs); mean and max beside it
    e2e = dist.max(statistics.median(e2e_ms))
    e2e_mean = dist.max(statistics.mean(e2e_ms))
    e2e_pin = dist.max(statistics.median(e2e_pin_ms))

    # --- roofline -----------------------------------------------------------
    peak, peak_kind = measured_peak()
    roof = roofline_block(args.config, args.mode, phases, stats, n, m, deg, ms, peak, peak_kind)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(raw, args.mode, args.cpu_budget)

    batch = None
    if rank == 0 and args.batch:
        batch = bench_batch(gd, N, L, with_cpu=world == 1 and not args.no_cpu_baseline)

    big = None
    if rank == 0 and world == 1 and args.big and args.config == "c3_rmat20":
        big = bench_resident_config(gd, N, L, "c5_chung_lu_4m", peak)

    if rank == 0:
        line = {
            "metric": METRIC, "value": m / (ms / 1e3), "unit": "edges/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic",
            "config": {"workload": args.config, "mode": args.mode,
                       "graph": CONFIG_DESC[args.config], "n": n, "m": m,
                       "parallelism": f"frame-sharded x{world}, owned edge ranges (NCCL "
                                      "all-reduce + reduce-scatter)" if world > 1
                       else "single",
                       "l2": "flushed between steps (256 MiB device memset)",
                       "timing": "CUDA events on the library stream, whole census"},
            "roofline": roof,
            "phases_ms": {k: round(v, 3) for k, v in phases.items()},
            "work": {k: v for k, v in stats.items() if k != "launches"},
            "wall_ms_per_step": wall_ms,
            "e2e": {"value": m / (e2e / 1e3), "unit": "edges/s", "ms_per_step": e2e,
                    "ms_mean": e2e_mean, "ms_max": max(e2e_ms),
                    "ms_steps": [round(x, 2) for x in e2e_ms],
                    "call": "micro_table(Graph.from_edges(pairs)) from pageable numpy pairs, "
                            "fresh int64 table returned every step" if per_edge else
                            "graphlet_census(Graph.from_edges(pairs)) from pageable numpy pairs",
                    "h2d_bytes_per_step": int(raw.pairs.nbytes),
                    "d2h_bytes_per_step": int((m * 80 if per_edge else 0) + 13 * 16 + 8),
                    "pinned": {"value": m / (e2e_pin / 1e3), "ms_per_step": e2e_pin,
                               "ms_steps": [round(x, 2) for x in e2e_pin_ms],
                               "call": "page-locked pairs, output into a reused page-locked "
                                       "table (micro_census_table(out=...))"}},
            "gpu_launches": launches,
            "clocks": clk,
            "cpu_baseline": cpu,
            "global_mode": glob,
            "batch_c4": batch,
            "c5_chung_lu_4m": big,
            "counts": {"g3_1": str(f_ref.counts["g3_1"]), "g4_1": str(f_ref.counts["g4_1"]),
                       "g4_4": str(f_ref.counts["g4_4"])},
        }
        print(json.dumps(line), flush=True)
    if dtab:
        L.gd_device_free(dtab)
    if comm is not None:
        comm.close()
    dist.close()
    return 0


def bench_resident_config(gd, N, L, config: str, peak: float, steps: int = 3,
                          warmup: int = 3) -> dict:
    """A second BASELINE config measured resident (CSR on the device, L2
    flushed between steps, CUDA events over the whole census): per-edge and
    global census times, edges/s and SURVEY 8(d) roofline fraction.  Used for
    config 5 (the north star's 4M-vertex Chung-Lu run) beside config 3."""
    raw = load_graph(config)
    g = gd.Graph.from_edges(raw.pairs, gd.ParseOptions(num_vertices=raw.n))
    del raw
    n, m = g.n, g.m
    deg = np.asarray(g.degrees, dtype=np.int64)
    dtab = L.gd_device_alloc(m * 10 * 8)
    out = {"workload": config, "graph": CONFIG_DESC[config], "n": n, "m": m,
           "steps": steps, "warmup": warmup,
           "l2": "flushed between steps", "timing": "CUDA events, whole census"}
    try:
        for mode in ("per_edge", "global"):
            ms, ref = [], None
            for i in range(warmup + steps):
                L.gd_flush_l2()
                if mode == "per_edge":
                    _, f = gd.micro_census_table(g, device_out=dtab)
                else:
                    f = gd.graphlet_census(g)
                if ref is None:
                    ref = f
                elif f != ref:
                    raise SystemExit(f"{config} {mode}: census result changed between steps")
                if i >= warmup:
                    ms.append(sum(gd.last_timings(g).values()))
            t = statistics.mean(ms)
            ph = gd.last_timings(g)
            out[mode] = {"ms_per_step": t, "value": m / (t / 1e3), "unit": "edges/s",
                         "roofline": roofline_block(config, mode, ph, gd.last_stats(g), n, m,
                                                    deg, t, peak, "measured"),
                         "phases_ms": {k: round(v, 3) for k, v in ph.items()}}
        if out["per_edge"] and ref is not None:
            out["g4_4"] = str(ref.counts["g4_4"])
    finally:
        L.gd_device_free(dtab)
        del g
        gd.trim_workspace()
    return out


def bench_batch(gd, N, L, with_cpu: bool) -> dict:
    """Config 4: 4,096 small graphs -> 17-count feature rows (feature_matrix),
    end to end from host pairs (one batched device pass)."""
    from paper_1506_04322_b200 import workloads as W
    raws = W.config_batch()
    pairs = [r.pairs for r in raws]
    ns = [r.n for r in raws]
    times, dev = [], []
    for i in range(4):
        L.gd_flush_l2()
        t0 = time.perf_counter()
        b = gd.GraphBatch(pairs, ns)
        fm = gd.feature_matrix(b)
        dt = time.perf_counter() - t0
        if i:
            times.append(dt)
            dev.append(sum(gd.last_timings(b).values()))
    m = int(b.m_per_graph.sum())
    out = {"graphs": len(raws), "sum_m": m, "e2e_ms": statistics.median(times) * 1e3,
           "device_census_ms": statistics.median(dev),
           "e2e_edges_per_s": m / statistics.median(times),
           "graphs_per_s": len(raws) / statistics.median(times), "skipped": len(fm.skipped)}
    if with_cpu:
        from oracle import oracle as O
        idx = np.random.default_rng(3).choice(len(raws), 256, replace=False)
        t0 = time.perf_counter()
        for i in idx:
            O.census(O.canonical_edges(raws[i].pairs), raws[i].n, threads=1)
        t = (time.perf_counter() - t0) * len(raws) / len(idx)
        out["cpu_baseline"] = {"value": m / t, "unit": "edges/s", "cores": 1, "kind": "port",
                               "sample": "256 of the 4096 graphs, serial (the reference loops "
                                         "graphs serially in feature_matrix), extrapolated"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", default="c3_rmat20", choices=sorted(CONFIG_DESC))
    ap.add_argument("--mode", default="per_edge", choices=("per_edge", "global"))
    ap.add_argument("--cpu-budget", type=float, default=10.0,
                    help="seconds of CPU work per baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-global", dest="global_too", action="store_false")
    ap.add_argument("--no-batch", dest="batch", action="store_false",
                    help="skip the config-4 batch (feature_matrix) measurement")
    ap.add_argument("--no-big", dest="big", action="store_false",
                    help="skip the resident config-5 (Chung-Lu 4M) secondary measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
