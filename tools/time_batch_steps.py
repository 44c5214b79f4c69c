"""Where the config-4 feature_matrix e2e time goes (host packing, device
build, census + closures, row assembly)."""
import sys, time
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import workloads as W
from paper_1506_04322_b200.graph import _as_pairs, _staging_pairs
from paper_1506_04322_b200.census import batch_counts
raws = W.config_batch()
pairs = [r.pairs for r in raws]; ns = [r.n for r in raws]
for it in range(5):
    t0 = time.perf_counter()
    arrs = [_as_pairs(p) for p in pairs]
    t1 = time.perf_counter()
    flat = _staging_pairs(sum(len(a) for a in arrs)); np.concatenate(arrs, out=flat)
    t2 = time.perf_counter()
    b = gd.GraphBatch(pairs, ns)
    t3 = time.perf_counter()
    counts, status = batch_counts(b)
    t4 = time.perf_counter()
    fm = gd.feature_matrix(b)
    t5 = time.perf_counter()
    dev = gd.last_timings(b)
    print(f"as_pairs {1e3*(t1-t0):.2f} pack {1e3*(t2-t1):.2f} GraphBatch {1e3*(t3-t0):.2f} "
          f"batch_counts {1e3*(t4-t3):.2f} (device {sum(dev.values()):.2f}) feature_matrix {1e3*(t5-t4):.2f}", flush=True)
