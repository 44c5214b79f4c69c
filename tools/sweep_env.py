"""Time one config under different env settings (each in a subprocess)."""
import json, os, subprocess, sys
cfg = sys.argv[1]
var = sys.argv[2]
vals = sys.argv[3].split(",")
mode = sys.argv[4] if len(sys.argv) > 4 else "per_edge"
code = r'''
import sys, json
sys.path.insert(0, %r)
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import _native as N, workloads as W
raw = W.config_graph(%r)
g = gd.Graph.from_edges(raw.pairs, gd.ParseOptions(num_vertices=raw.n))
L = N.load_library(); d = L.gd_device_alloc(g.m * 80)
res = []
for i in range(4):
    L.gd_flush_l2()
    try:
        if %r == "per_edge": gd.micro_census_table(g, device_out=d)
        else: gd.graphlet_census(g)
    except gd.GraphletError as exc:
        if i == 0: print("check failed (expected under GD_EXP):", exc)
    if i: res.append(gd.last_timings(g))
print(json.dumps(res[-1]), sum(sum(r.values()) for r in res) / len(res))
''' % (str(__import__('pathlib').Path(__file__).resolve().parent.parent), cfg, mode)
for v in vals:
    env = dict(os.environ, **{var: v})
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(var, v, r.stdout.strip()[-600:], r.stderr.strip()[-300:], flush=True)
