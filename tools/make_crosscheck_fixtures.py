"""Full-size per-edge fixtures from the independent CPU cross-check
(oracle/crosscheck.c) -- TEST INFRASTRUCTURE, run in the build container.

For a config it computes the whole (m, 10) micro table and the 13 sums,
checks them against every literal-oracle / reference pin that exists for the
config (reference counts + table sha256 at C2, the full C-oracle census at C3,
the committed oracle samples oracle_<cfg>_{micro,count}_sample at C3 / C5) and
writes tests/golden/crosscheck_<cfg>.json: the 17 counts, the 13 sums and one
sha256 per 65536-row chunk of the table, so the GPU tests can compare every
row of the device table without shipping it.

usage: python tools/make_crosscheck_fixtures.py c3_rmat20 [--threads 8]
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
from sample_sets import COUNT_CHUNK, count_sample  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"
TABLE_CHUNK = 1 << 16


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--threads", type=int, default=0)
    a = ap.parse_args()
    raw = W.config_graph(a.config)
    edges = O.canonical_edges(raw.pairs)
    n, m = raw.n, len(edges)
    t0 = time.time()
    rows, sums = O.crosscheck_table(edges, n, threads=a.threads)
    dt = time.time() - t0
    counts = O.close(sums, n, m)
    print(f"{a.config}: m={m} cross-check table in {dt:.1f}s", flush=True)
    pins = {}
    # pins against the reference / the literal oracle
    cfg = json.loads((GOLDEN / "configs.json").read_text()).get(a.config, {})
    if "counts" in cfg:
        pins["reference_counts"] = {k: str(v) for k, v in counts.items()} == cfg["counts"]
    if "micro_sha256" in cfg:
        pins["reference_table_sha256"] = sha(rows) == cfg["micro_sha256"]
    full = GOLDEN / f"oracle_{a.config}.json"
    if full.exists():
        d = json.loads(full.read_text())
        pins["oracle_full_census_counts"] = {k: str(v) for k, v in counts.items()} == d["counts"]
    ms = GOLDEN / f"oracle_{a.config}_micro_sample.npz"
    if ms.exists():
        z = np.load(ms)
        pins["oracle_micro_sample_rows"] = bool(np.array_equal(rows[z["idx"]], z["rows"]))
        pins["oracle_micro_sample_size"] = int(len(z["idx"]))
    cs = GOLDEN / f"oracle_{a.config}_count_sample.json"
    if cs.exists():
        d = json.loads(cs.read_text())
        idx = count_sample(m, d["k"])
        assert sha(idx) == d["idx_sha256"]
        sub = np.ascontiguousarray(rows[idx, :5])
        got = [sha(sub[i:i + COUNT_CHUNK]) for i in range(0, len(idx), COUNT_CHUNK)]
        pins["oracle_count_sample_chunks"] = got == d["chunk_sha256"]
        pins["oracle_count_sample_size"] = int(d["k"])
    print("pins:", pins, flush=True)
    if not all(v for k, v in pins.items() if isinstance(v, bool)):
        raise SystemExit("cross-check disagrees with a pin: not writing the fixture")
    out = {"config": a.config, "n": n, "m": m, "edges_sha256": sha(edges),
           "chunk_rows": TABLE_CHUNK,
           "chunk_sha256": [sha(rows[i:i + TABLE_CHUNK]) for i in range(0, m, TABLE_CHUNK)],
           "table_sha256": sha(rows),
           "sums": [str(s) for s in sums],
           "counts": {k: str(v) for k, v in counts.items()},
           "pinned_by": pins, "seconds": dt,
           "generator": "oracle/crosscheck.c crosscheck_table (independent CPU computation)"}
    (GOLDEN / f"crosscheck_{a.config}.json").write_text(json.dumps(out, indent=0))
    print("wrote", GOLDEN / f"crosscheck_{a.config}.json", flush=True)


if __name__ == "__main__":
    main()
