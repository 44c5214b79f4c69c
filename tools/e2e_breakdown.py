"""Where the end-to-end time of a per-edge census goes (fresh graph each step,
as in bench.py's e2e leg): build from pinned host pairs, census into a device
table (first and second census of the graph), D2H of the table."""
import sys, time
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import _native as N, workloads as W
raw = W.config_graph(sys.argv[1] if len(sys.argv) > 1 else "c3_rmat20")
pairs = N.pinned_empty(raw.pairs.shape, np.int64); pairs[...] = raw.pairs
L = N.load_library()
g0 = gd.Graph.from_edges(pairs, gd.ParseOptions(num_vertices=raw.n))
m = g0.m
dtab = L.gd_device_alloc(m * 80)
htab = N.pinned_empty((m, 10), np.int64)
def sync():
    torch.cuda.synchronize()
for i in range(4):
    sync(); t0 = time.perf_counter()
    g = gd.Graph.from_edges(pairs, gd.ParseOptions(num_vertices=raw.n))
    sync(); t1 = time.perf_counter()
    gd.micro_census_table(g, device_out=dtab)
    sync(); t2 = time.perf_counter()
    t1d = {k: round(v, 1) for k, v in gd.last_timings(g).items()}
    ph1 = sum(t1d.values())
    gd.micro_census_table(g, device_out=dtab)
    sync(); t3 = time.perf_counter()
    ph2 = sum(gd.last_timings(g).values())
    _, f = gd.micro_census_table(g, out=htab)
    sync(); t4 = time.perf_counter()
    del g
    print(f"build {1e3*(t1-t0):.1f}  census#1 {1e3*(t2-t1):.1f} (phases {ph1:.1f})  "
          f"census#2 {1e3*(t3-t2):.1f} (phases {ph2:.1f})  census+d2h {1e3*(t4-t3):.1f}", t1d, flush=True)
