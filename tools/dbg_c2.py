import sys
sys.path.insert(0, "/root/repo")
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import workloads as W
raw = W.config_graph("c2_chung_lu")
g = gd.Graph.from_edges(raw.pairs, gd.ParseOptions(num_vertices=raw.n))
print(gd.graphlet_census(g).counts["g4_4"])
