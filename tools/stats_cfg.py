import sys, json
sys.path.insert(0, "/root/repo")
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import _native as N, workloads as W
raw = W.config_graph(sys.argv[1])
g = gd.Graph.from_edges(raw.pairs, gd.ParseOptions(num_vertices=raw.n))
L = N.load_library(); d = L.gd_device_alloc(g.m * 80)
for i in range(2):
    gd.micro_census_table(g, device_out=d)
print(json.dumps(gd.last_timings(g)), json.dumps(gd.last_stats(g)))
