"""Full global census of a config by the C oracle (the restatement of the
reference's _count_edge/_census_batch), for a golden file the GPU tests can
check at full size.  Long-running: R-MAT-20 needs ~1.4e13 adjacency reads."""
import json, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import oracle as O
from paper_1506_04322_b200 import workloads as W

name = sys.argv[1]
raw = W.config_graph(name)
edges = O.canonical_edges(raw.pairs)
t0 = time.time()
og = O.OracleGraph(edges, raw.n)
sums, seen = og.census_sums(threads=0, batch=16)
counts = O.close(sums, raw.n, len(edges))
out = ROOT / "tests" / "golden" / f"oracle_{name}.json"
out.write_text(json.dumps({"config": name, "n": raw.n, "m": len(edges), "seen": seen,
                           "counts": {k: str(v) for k, v in counts.items()},
                           "seconds": time.time() - t0, "generator": "oracle/census_oracle.c"},
                          indent=1))
print("wrote", out, time.time() - t0)
