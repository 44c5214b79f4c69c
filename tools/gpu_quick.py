import sys, time, os
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1506_04322_b200 as gd
from oracle import oracle as O
from paper_1506_04322_b200 import workloads as W
import json
for name, raw in [("er300", W.erdos_renyi_gnm(300, 1500, seed=7)), ("c1", W.config_graph("c1_er")), ("c2", W.config_graph("c2_chung_lu"))]:
    g = gd.Graph.from_edges(raw.pairs, _declared_n=raw.n)
    t0=time.time(); f = gd.graphlet_census(g); t1=time.time()
    table, f2 = gd.micro_census_table(g); t2=time.time()
    print(name, g, "global", t1-t0, "micro", t2-t1, gd.last_timings(g), gd.last_stats(g), flush=True)
    edges = np.asarray(g.edges)
    if g.m <= 20000:
        want = O.census(edges, g.n)
        print(" global match", f.counts == want, " per-edge==global", f2 == f)
        rows = O.micro_rows(edges, g.n)
        bad = np.nonzero((np.asarray(table) != rows).any(1))[0]
        print(" micro mismatches", len(bad), bad[:5], table[bad[:3]] if len(bad) else "", rows[bad[:3]] if len(bad) else "")
    else:
        cfg = json.load(open("/root/repo/tests/golden/configs.json")).get(name.replace("c2","c2_chung_lu"))
        print(" per-edge==global", f2 == f)
        idx = np.random.default_rng(0).choice(g.m, 2000, replace=False)
        rows = O.micro_rows(edges, g.n, idx)
        print(" sampled micro mismatches", int((np.asarray(table)[idx] != rows).any(1).sum()))
