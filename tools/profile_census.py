"""One warm per-edge (or global) census of a config, for ncu captures."""
import sys
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import _native as N
from paper_1506_04322_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3_rmat20"
mode = sys.argv[2] if len(sys.argv) > 2 else "per_edge"
raw = W.config_graph(cfg)
g = gd.Graph.from_edges(raw.pairs, gd.ParseOptions(num_vertices=raw.n))
L = N.load_library()
dtab = L.gd_device_alloc(g.m * 80)
for _ in range(2):
    if mode == "per_edge":
        gd.micro_census_table(g, device_out=dtab)
    else:
        gd.graphlet_census(g)
print(gd.last_timings(g), gd.last_stats(g))
