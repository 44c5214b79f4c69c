"""Latency breakdown of the small configs (C1 single graph, C4 batch):
build / census / closure host time and device phases."""
import ctypes, sys, time
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import _native as N, workloads as W

raw = W.config_graph("c1_er")
for it in range(6):
    t0 = time.perf_counter()
    g = gd.Graph.from_edges(raw.pairs, gd.ParseOptions(num_vertices=raw.n))
    t1 = time.perf_counter()
    tab, f = gd.micro_census_table(g)
    t2 = time.perf_counter()
    print(f"C1 build {1e3*(t1-t0):.3f} ms census+table {1e3*(t2-t1):.3f} ms",
          {k: round(v, 3) for k, v in gd.last_timings(g).items()}, gd.last_stats(g).get("launches"))
raws = W.config_batch()
pairs = [r.pairs for r in raws]; ns = [r.n for r in raws]
for it in range(4):
    t0 = time.perf_counter(); b = gd.GraphBatch(pairs, ns); t1 = time.perf_counter()
    counts, status = gd.census.batch_counts(b); t2 = time.perf_counter()
    fm = gd.feature_matrix(b); t3 = time.perf_counter()
    print(f"C4 build {1e3*(t1-t0):.2f} ms census+close {1e3*(t2-t1):.2f} ms feature_matrix(batch) {1e3*(t3-t2):.2f} ms",
          {k: round(v, 3) for k, v in gd.last_timings(b).items()}, gd.last_stats(b).get("launches"))
for it in range(3):
    t0 = time.perf_counter(); fm = gd.feature_matrix(gd.GraphBatch(pairs, ns)); t1 = time.perf_counter()
    print(f"C4 e2e {1e3*(t1-t0):.2f} ms")
