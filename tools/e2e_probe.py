"""Step-by-step timing of the e2e path (fresh graph per step) with device
memory use, to find allocation / synchronisation spikes."""
import sys, time, gc
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import _native as N, workloads as W
raw = W.config_graph(sys.argv[1] if len(sys.argv) > 1 else "c3_rmat20")
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
pairs = N.pinned_empty(raw.pairs.shape, np.int64); pairs[...] = raw.pairs
L = N.load_library()
htab = None
for i in range(steps):
    t0 = time.perf_counter()
    g = gd.Graph.from_edges(pairs, gd.ParseOptions(num_vertices=raw.n))
    t1 = time.perf_counter()
    if htab is None:
        htab = N.pinned_empty((g.m, 10), np.int64)
    _, f = gd.micro_census_table(g, out=htab)
    t2 = time.perf_counter()
    ph = gd.last_timings(g)
    del g
    t3 = time.perf_counter()
    free, total = torch.cuda.mem_get_info()
    print(f"step {i}: build {1e3*(t1-t0):.1f} census+d2h {1e3*(t2-t1):.1f} (device phases {sum(ph.values()):.1f}) "
          f"free-graph {1e3*(t3-t2):.1f}  total {1e3*(t3-t0):.1f}  gpu used {(total-free)/2**30:.1f} GiB", flush=True)
