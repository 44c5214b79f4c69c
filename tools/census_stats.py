"""Timings and schedule statistics of a few resident censuses of a config
(diagnostics): python tools/census_stats.py c5_chung_lu_4m per_edge [runs]"""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import _native as N, workloads as W

cfg, mode = sys.argv[1], sys.argv[2]
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 3
raw = W.config_graph(cfg)
L = N.load_library()
for r in range(runs):
    t0 = time.perf_counter()
    g = gd.Graph.from_edges(raw.pairs, gd.ParseOptions(num_vertices=raw.n))
    t1 = time.perf_counter()
    if mode == "per_edge":
        tab, f = gd.micro_census_table(g)
    else:
        f = gd.graphlet_census(g)
    t2 = time.perf_counter()
    ps = (__import__("ctypes").c_uint64 * 4)()
    L.gd_pool_stats(ps)
    print(json.dumps({"run": r, "build_ms": 1e3 * (t1 - t0), "census_call_ms": 1e3 * (t2 - t1),
                      "device_ms": gd.last_timings(g), "stats": gd.last_stats(g),
                      "pool_gib": [round(x / 2**30, 2) for x in ps]}), flush=True)
    del g
