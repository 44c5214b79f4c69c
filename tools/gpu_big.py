import sys, time, os
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1506_04322_b200 as gd
from oracle import oracle as O
from paper_1506_04322_b200 import workloads as W
print("cpus", os.cpu_count(), flush=True)
names = sys.argv[1:] or ["c3_rmat20"]
for name in names:
    t0 = time.time(); raw = W.config_graph(name); tg = time.time() - t0
    t0 = time.time(); g = gd.Graph.from_edges(raw.pairs, _declared_n=raw.n); tb = time.time() - t0
    print(name, g, f"gen {tg:.1f}s build {tb:.2f}s", flush=True)
    for rep in range(2):
        t0 = time.time(); f = gd.graphlet_census(g); t1 = time.time()
        print(" global", f"{t1-t0:.3f}s", gd.last_timings(g), gd.last_stats(g), flush=True)
    for rep in range(2):
        t0 = time.time(); table, f2 = gd.micro_census_table(g); t1 = time.time()
        print(" per-edge", f"{t1-t0:.3f}s", gd.last_timings(g), flush=True)
    print(" per-edge==global", f2 == f, flush=True)
    t0 = time.time(); f3 = gd.frequencies_from_micro(g, table); print(" dual route", f3 == f, f"{time.time()-t0:.2f}s")
    print(" counts", f.counts, flush=True)
    edges = np.asarray(g.edges)
    idx = np.random.default_rng(0).choice(g.m, 300, replace=False)
    t0 = time.time(); rows = O.micro_rows(edges, g.n, idx); 
    print(" sampled micro mismatches", int((np.asarray(table)[idx] != rows).any(1).sum()), f"oracle {time.time()-t0:.1f}s", flush=True)
