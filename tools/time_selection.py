"""Latency of incremental selection operations on a config graph (device
region refresh + O(1) closure), with a final audit against a fresh census."""
import json
import sys
import time
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2_chung_lu"
raw = W.config_graph(cfg)
g = gd.Graph.from_edges(raw.pairs, gd.ParseOptions(num_vertices=raw.n))
rng = np.random.default_rng(1)
seed_v = rng.choice(g.n, 2000, replace=False)
t0 = time.perf_counter()
st = gd.SelectionState(g, active=seed_v.tolist())
init_s = time.perf_counter() - t0
lat = []
edges = np.asarray(g.edges)
for i in range(300):
    k = int(rng.integers(0, 3))
    if k == 0:
        op = gd.SelectionOp("add_vertex", vertex=int(rng.integers(g.n)))
    elif k == 1:
        op = gd.SelectionOp("remove_vertex", vertex=int(rng.choice(list(st.active))))
    else:
        e = edges[int(rng.integers(g.m))]
        op = gd.SelectionOp("remove_edge", u=int(e[0]), v=int(e[1]))
    t0 = time.perf_counter()
    st.apply_one(op)
    lat.append((time.perf_counter() - t0) * 1e3)
t0 = time.perf_counter()
st.audit()
audit_s = time.perf_counter() - t0
print(json.dumps({"config": cfg, "n": g.n, "m": g.m, "initial_vertices": 2000,
                  "init_s": init_s, "ops": len(lat), "op_ms_median": float(np.median(lat)),
                  "op_ms_p90": float(np.percentile(lat, 90)), "op_ms_max": float(np.max(lat)),
                  "audit_s": audit_s}))
