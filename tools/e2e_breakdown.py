import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import _native as N, workloads as W
raw = W.config_graph(sys.argv[1] if len(sys.argv) > 1 else "c3_rmat20")
pairs = N.pinned_empty(raw.pairs.shape, np.int64); pairs[...] = raw.pairs
g0 = gd.Graph.from_edges(pairs, gd.ParseOptions(num_vertices=raw.n))
htab = N.pinned_empty((g0.m, 10), np.int64)
for i in range(3):
    t0 = time.perf_counter()
    g = gd.Graph.from_edges(pairs, gd.ParseOptions(num_vertices=raw.n))
    t1 = time.perf_counter()
    _, f = gd.micro_census_table(g, out=htab)
    t2 = time.perf_counter()
    del g
    t3 = time.perf_counter()
    print(f"build {1e3*(t1-t0):.1f} census+d2h {1e3*(t2-t1):.1f} free {1e3*(t3-t2):.1f}", {k: round(v,1) for k,v in gd.last_timings(g0).items()} if i == 0 else "")
