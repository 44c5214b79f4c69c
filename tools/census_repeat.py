"""Phase times of N repeated resident censuses of one graph (variance check):
python tools/census_repeat.py c3_rmat20 global 20 [flush]"""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import _native as N, workloads as W

cfg, mode, runs = sys.argv[1], sys.argv[2], int(sys.argv[3])
flush = len(sys.argv) > 4
raw = W.config_graph(cfg)
g = gd.Graph.from_edges(raw.pairs, gd.ParseOptions(num_vertices=raw.n))
L = N.load_library()
d = L.gd_device_alloc(g.m * 80) if mode == "per_edge" else None
for i in range(runs):
    if flush:
        L.gd_flush_l2()
    if mode == "per_edge":
        gd.micro_census_table(g, device_out=d)
    else:
        gd.graphlet_census(g)
    t = gd.last_timings(g)
    print(i, round(sum(t.values()), 2), {k: round(v, 2) for k, v in t.items()}, flush=True)
