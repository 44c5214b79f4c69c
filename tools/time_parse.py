"""Edge-list parsing throughput: device route (text -> device pairs -> device
graph) vs the reference's CPython loop (restated in edgelist._scan_lines, the
same algorithm as graph.py:239-285) on a sample of the same text."""
import io
import json
import sys
import time
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import edgelist as EL, workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3_rmat20"
raw = W.config_graph(cfg)
t0 = time.perf_counter()
s = raw.pairs.astype(str)
text = "\n".join(np.char.add(np.char.add(s[:, 0], " "), s[:, 1]).tolist()) + "\n"
gen_s = time.perf_counter() - t0
opts = gd.ParseOptions(num_vertices=raw.n)
ms = []
for i in range(4):
    t0 = time.perf_counter()
    g = gd.Graph.from_text(text, opts)
    ms.append((time.perf_counter() - t0) * 1e3)
assert EL.last_route == "device"
ref = gd.Graph.from_edges(raw.pairs, opts)
assert np.array_equal(np.asarray(g.edges), np.asarray(ref.edges))
# CPython loop on a 1M-line sample
lines = text.splitlines(keepends=True)
k = min(len(lines), 1_000_000)
t0 = time.perf_counter()
EL._scan_lines(io.StringIO("".join(lines[:k])), opts)
host_s = (time.perf_counter() - t0) * len(lines) / k
out = {"config": cfg, "lines": len(lines), "bytes": len(text),
       "device_ms_median": float(np.median(ms[1:])), "device_ms_all": ms,
       "device_GBps": len(text) / (np.median(ms[1:]) / 1e3) / 1e9,
       "cpython_loop_s_extrapolated": host_s, "cpython_sample_lines": k,
       "text_generation_s": gen_s}
print(json.dumps(out))

# breakdown of one device parse
import ctypes
from paper_1506_04322_b200 import _native as N
L = N.lib()
for i in range(3):
    t0 = time.perf_counter()
    data = text.encode("ascii")
    t1 = time.perf_counter()
    arr = (ctypes.c_char_p * 2)(b"#", b"%")
    h = ctypes.c_void_p()
    N.check(L.gd_parse_edge_list(data, len(data), arr, 2, 2, ctypes.byref(h)))
    t2 = time.perf_counter()
    info = (ctypes.c_int64 * 12)()
    N.check(L.gd_parsed_info(h, info))
    g = EL._graph_from_device_pairs(L.gd_parsed_pairs(h), info[0], raw.n, N.GD_IDS_DECLARED)
    t3 = time.perf_counter()
    L.gd_parsed_free(h)
    print(f"encode {1e3*(t1-t0):.1f} ms  parse {1e3*(t2-t1):.1f} ms  build {1e3*(t3-t2):.1f} ms")
