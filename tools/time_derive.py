"""micro_csv / micro_roles throughput on a config's per-edge table: device
derive + format vs the CPython restatement (oracle/micro_oracle.py, the
reference's per-row algorithm) on a sample, extrapolated."""
import json
import sys
import tempfile
import time
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1506_04322_b200 as gd
from oracle import micro_oracle as MO
from paper_1506_04322_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3_rmat20"
raw = W.config_graph(cfg)
g = gd.Graph.from_edges(raw.pairs, gd.ParseOptions(num_vertices=raw.n))
tab = gd.micro_table(g)
orig = g.orig_ids
res = {"config": cfg, "m": g.m}
for name, fn in (("micro_roles", lambda: gd.micro_roles(g, tab)),
                 ("micro_csv_str", lambda: gd.micro_csv(g, tab))):
    ts = []
    for i in range(3):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    res[name + "_s"] = min(ts)
res["csv_bytes"] = len(out)
with tempfile.NamedTemporaryFile(suffix=".csv") as fh:
    t0 = time.perf_counter()
    gd.write_micro_csv(g, tab, fh.name)
    res["write_micro_csv_s"] = time.perf_counter() - t0
k = 100_000
idx = np.random.default_rng(1).choice(g.m, k, replace=False)
t0 = time.perf_counter()
MO.micro_csv(g.n, np.asarray(g.edges)[idx], orig, tab[idx], m=g.m)
res["cpython_rows_per_s"] = k / (time.perf_counter() - t0)
res["cpython_extrapolated_s"] = g.m / res["cpython_rows_per_s"]
print(json.dumps(res))
