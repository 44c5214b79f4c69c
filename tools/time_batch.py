import sys, time
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import workloads as W
raws = W.config_batch()
pairs = [r.pairs for r in raws]; ns = [r.n for r in raws]
for it in range(3):
    t0 = time.perf_counter(); b = gd.GraphBatch(pairs, ns); t1 = time.perf_counter()
    res = gd.census_batch(b); t2 = time.perf_counter()
    print(f"build {1e3*(t1-t0):.1f} ms census {1e3*(t2-t1):.1f} ms  m={int(b.m_per_graph.sum())}", gd.last_timings(b), gd.last_stats(b))
t0 = time.perf_counter(); fm = gd.feature_matrix(b); t1 = time.perf_counter()
print("feature_matrix", 1e3*(t1-t0), "ms", fm.rows.shape)
