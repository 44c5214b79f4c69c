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


def ncu_traffic(config: str, mode: str):
    """DRAM bytes (read + write) of one census, summed over its kernels, and
    the top kernel with its time share, from the committed ncu launch list
    summary (profiles/ncu_summary.json, made by tools/ncu_sum.py)."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None, None
    try:
        e = json.loads(p.read_text())[f"{config}/{mode}"]
        top = next(iter(e["kernels"].items()))
        return e["census_dram_bytes"], {"name": top[0], "share": top[1]["share"],
                                        "dram_bytes": top[1]["dram_bytes"]}
    except (KeyError, ValueError, StopIteration):
        return None, None


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
                         "kind": "port",
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
                t, f = micro_census_table_sharded(graph, comm, device_out=device_out)
                if out is not None:
                    out[...] = t
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
    dist.barrier()
    e2e_ms = []
    # the e2e leg gets the same W untimed warm-up steps as the resident leg
    # (measured with GD_BENCH_DEBUG=1: the first two fresh graphs after the
    # resident phase build in 300-450 ms, every later one in 12-17 ms)
    e2e_warm = max(1, args.warmup)
    for i in range(args.steps + e2e_warm):
        t0 = time.perf_counter()
        g2 = gd.Graph.from_edges(pairs, gd.ParseOptions(num_vertices=raw.n))
        tb = time.perf_counter()
        f2 = census(g2, out=htab if per_edge else None)
        tc = time.perf_counter()
        dev = sum(gd.last_timings(g2).values()) if DEBUG else 0.0
        del g2
        dt = (time.perf_counter() - t0) * 1e3
        if DEBUG:  # NVML (no CUDA context of its own) for the device memory in use
            import pynvml
            pynvml.nvmlInit()
            used = pynvml.nvmlDeviceGetMemoryInfo(pynvml.nvmlDeviceGetHandleByIndex(local_rank)).used
            ps = (ctypes.c_uint64 * 4)()
            L.gd_pool_stats(ps)
            print(f"e2e step {i}: build {1e3 * (tb - t0):.1f} census {1e3 * (tc - tb):.1f} "
                  f"(device {dev:.1f}) free {1e3 * (time.perf_counter() - tc):.1f} "
                  f"gpu used {used / 2**30:.2f} GiB pool reserved {ps[0] / 2**30:.2f} "
                  f"(high {ps[1] / 2**30:.2f}) used {ps[2] / 2**30:.2f} "
                  f"(high {ps[3] / 2**30:.2f}) GiB", file=sys.stderr, flush=True)
        if i >= e2e_warm:
            e2e_ms.append(dt)
        if f2 != f_ref:
            raise SystemExit("end-to-end census differs from the resident one")
    dist.barrier()
    # median over steps (median of the runs); the mean, which
    # host-side outliers of the box move (an occasional +100-300 ms step with
    # unchanged device time), is reported beside it
    e2e = dist.max(statistics.median(e2e_ms))
    e2e_mean = dist.max(statistics.mean(e2e_ms))

    # --- roofline: SURVEY 8(d) algorithmic bytes of one census ---------------
    sum_d2 = int(np.dot(deg, deg))
    o_bytes, k_out = 8, (10 if per_edge else 0)
    b_alg = m * (8 + 4 * o_bytes + 8 * k_out) + 4 * sum_d2
    peak, peak_kind = measured_peak()
    achieved = b_alg / (ms / 1e3) / 1e9
    traffic, ncu_kernel = ncu_traffic(args.config, args.mode)
    dom = max(phases.items(), key=lambda kv: kv[1]) if phases else ("", 0.0)

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
                       "parallelism": f"frame-sharded x{world} (NCCL all-reduce)" if world > 1
                       else "single",
                       "l2": "flushed between steps (256 MiB device memset)",
                       "timing": "CUDA events on the library stream, whole census"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": peak_kind,
                         "algorithmic_bytes": b_alg,
                         "kernel": "census pipeline (B_alg of SURVEY 8(d) / summed kernel time)",
                         "dominant_phase": dom[0],
                         "dominant_share": dom[1] / max(ms, 1e-9),
                         "ncu_kernel": ncu_kernel,
                         # the dominant phase's kernel: ncu DRAM bytes of one
                         # launch over its live CUDA-event time in this run
                         "dominant_dram_gbs": (ncu_kernel["dram_bytes"] / (dom[1] / 1e3) / 1e9
                                               if ncu_kernel and dom[1] > 0 else None)},
            "phases_ms": {k: round(v, 3) for k, v in phases.items()},
            "work": {k: v for k, v in stats.items() if k != "launches"},
            "wall_ms_per_step": wall_ms,
            "e2e": {"value": m / (e2e / 1e3), "unit": "edges/s", "ms_per_step": e2e,
                    "ms_mean": e2e_mean, "ms_steps": [round(x, 2) for x in e2e_ms],
                    "h2d_bytes_per_step": int(pairs.nbytes),
                    "d2h_bytes_per_step": int((m * 80 if per_edge else 0) + 13 * 16 + 8)},
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
    sum_d2 = int(np.dot(deg, deg))
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
            b_alg = m * (8 + 4 * 8 + 8 * (10 if mode == "per_edge" else 0)) + 4 * sum_d2
            out[mode] = {"ms_per_step": t, "value": m / (t / 1e3), "unit": "edges/s",
                         "roofline_frac": b_alg / (t / 1e3) / 1e9 / peak,
                         "algorithmic_bytes": b_alg,
                         "phases_ms": {k: round(v, 3) for k, v in gd.last_timings(g).items()}}
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
