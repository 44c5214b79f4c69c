"""Per-edge parity fixtures for the full-size configs C3 / C5 (TEST
INFRASTRUCTURE: run in the build container, commits small files under
tests/golden/).

The literal C oracle (oracle/census_oracle.c, the restatement of the
reference's _micro_edge census.py:190-256 and _count_edge census.py:259-303,
pinned to the reference by tests/test_oracle_golden.py) is run on

* the SURVEY 8(c) per-edge sample: ``--uniform`` uniform edges, the top-1k
  edges by w_e = d(lo) + S(lo), and up to ``--per-hub`` uniformly chosen edges
  incident to each of the top-100 hubs -> full 10-column _micro_edge rows,
  stored verbatim (``oracle_<cfg>_micro_sample.npz``);
* ``--count`` uniformly chosen edges -> _count_edge rows (t, s_u, s_v, cl, cy)
  in canonical orientation, stored as one sha256 per chunk of 8192 jobs plus
  column sums (``oracle_<cfg>_count_sample.json``): 1M rows would be 40 MB.

The GPU tests regenerate the config, draw the same index set from the seed
(its sha256 is recorded) and compare the device table's columns.

usage: python tools/make_big_fixtures.py c3_rmat20 [--count 1000000] [--threads 6]
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import oracle as O  # noqa: E402
from paper_1506_04322_b200 import workloads as W  # noqa: E402
from sample_sets import COUNT_CHUNK, count_sample, micro_sample  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--count", type=int, default=1_000_000)
    ap.add_argument("--threads", type=int, default=6)
    ap.add_argument("--skip-micro", action="store_true")
    ap.add_argument("--skip-count", action="store_true")
    a = ap.parse_args()
    t0 = time.time()
    raw = W.config_graph(a.config)
    edges = O.canonical_edges(raw.pairs)
    n, m = raw.n, len(edges)
    print(f"{a.config}: n={n} m={m} generated in {time.time() - t0:.1f}s", flush=True)
    og = O.OracleGraph(edges, n)
    if not a.skip_micro:
        idx = micro_sample(edges, n)
        t1 = time.time()
        rows = og.micro_rows(idx, threads=a.threads)
        dt = time.time() - t1
        np.savez_compressed(GOLDEN / f"oracle_{a.config}_micro_sample.npz", idx=idx, rows=rows,
                            m=np.int64(m), edges_sha256=np.array(sha(edges)))
        print(f"micro sample: {len(idx)} edges in {dt:.1f}s", flush=True)
    if not a.skip_count:
        idx = count_sample(m, a.count)
        t1 = time.time()
        rows = og.count_rows(idx, threads=a.threads)
        dt = time.time() - t1
        chunks = [sha(rows[i:i + COUNT_CHUNK]) for i in range(0, len(idx), COUNT_CHUNK)]
        out = {"config": a.config, "n": n, "m": m, "edges_sha256": sha(edges),
               "k": len(idx), "idx_sha256": sha(idx), "chunk": COUNT_CHUNK,
               "columns": ["t", "su", "sv", "cl", "cy"],
               "col_sums": [str(int(rows[:, j].astype(object).sum())) for j in range(5)],
               "chunk_sha256": chunks, "seconds": dt, "threads": a.threads,
               "generator": "oracle/census_oracle.c oracle_count_rows_h (_count_edge)"}
        (GOLDEN / f"oracle_{a.config}_count_sample.json").write_text(json.dumps(out, indent=0))
        print(f"count sample: {len(idx)} edges in {dt:.1f}s", flush=True)


if __name__ == "__main__":
    main()
