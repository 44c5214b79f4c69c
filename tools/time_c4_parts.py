"""C4 latency parts: batch build (gather + device build), census + closure,
feature rows."""
import sys, time
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import workloads as W

raws = W.config_batch()
pairs = [r.pairs for r in raws]; ns = [r.n for r in raws]
for it in range(5):
    t0 = time.perf_counter()
    b = gd.GraphBatch(pairs, ns)
    t1 = time.perf_counter()
    counts, status = gd.census.batch_counts(b)
    t2 = time.perf_counter()
    fm = gd.feature_matrix(b)
    t3 = time.perf_counter()
    print(f"batch build {1e3*(t1-t0):.2f} census+close {1e3*(t2-t1):.2f} "
          f"feature_matrix {1e3*(t3-t2):.2f}", gd.last_timings(b))
