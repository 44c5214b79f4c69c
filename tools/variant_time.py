"""Time the census under several library builds (GD_LIBRARY variants from
tools/build_variant.py), each in a subprocess; prints per-phase timings and a
digest of the counts + per-edge table so variants can be checked against each
other.  Usage: python tools/variant_time.py CONFIG MODE lib1.so|default|ENV=VAL ..."""
import os, subprocess, sys
cfg, mode, libs = sys.argv[1], sys.argv[2], sys.argv[3:]
code = r'''
import sys, json, hashlib
sys.path.insert(0, %r)
import numpy as np, torch
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import _native as N, workloads as W
raw = W.config_graph(%r)
g = gd.Graph.from_edges(raw.pairs, gd.ParseOptions(num_vertices=raw.n))
L = N.load_library()
tot = []
for i in range(5):
    L.gd_flush_l2()
    try:
        if %r == "per_edge":
            t = torch.empty((g.m, 10), dtype=torch.int64, device="cuda")
            f = gd.micro_census_table(g, device_out=t.data_ptr())[1]
        else:
            f = gd.graphlet_census(g)
    except gd.GraphletError as exc:  # timing-only experiment builds fail the checks
        f = None
        if i == 0: print("check failed:", exc)
    tm = gd.last_timings(g)
    if i: tot.append(sum(tm.values()))
h = hashlib.sha256(repr(sorted(f.counts.items())).encode() if f else b"failed")
if %r == "per_edge" and f:
    h.update(t.cpu().numpy().tobytes())
print(json.dumps({k: round(v, 2) for k, v in tm.items()}), "total_ms %%.2f" %% (sum(tot) / len(tot)), "digest", h.hexdigest()[:16])
''' % (str(__import__('pathlib').Path(__file__).resolve().parent.parent), cfg, mode, mode)
for lib in libs:
    env = dict(os.environ)
    if "=" in lib:  # NAME=VALUE: the default library under an env setting
        k, v = lib.split("=", 1)
        env[k] = v
    elif lib != "default":
        env["GD_LIBRARY"] = lib
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), r.stdout.strip()[-500:], r.stderr.strip()[-400:], flush=True)
