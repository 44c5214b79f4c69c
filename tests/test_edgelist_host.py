"""Edge-list loading, host side (no GPU): the CPython-rules restatement of
the reference loop (edgelist._scan_lines) plus the numpy graph oracle
against the reference's own outputs on every golden parse case
(tests/golden/parse_cases.json, made by make_golden.py --parse)."""
import io
import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import graph_oracle as GO  # noqa: E402
from paper_1506_04322_b200 import ParseOptions  # noqa: E402
from paper_1506_04322_b200.edgelist import _scan_lines  # noqa: E402
from paper_1506_04322_b200.errors import EdgeListParseError  # noqa: E402

CASES = json.loads((ROOT / "tests" / "golden" / "parse_cases.json").read_text())


def _opts(d):
    d = dict(d)
    if "comment_prefixes" in d:
        d["comment_prefixes"] = tuple(d["comment_prefixes"])
    return ParseOptions(**d)


def _host_load(case):
    opts = _opts(case["opts"])
    if case["mode"] == "text":
        pairs, mm = _scan_lines(io.StringIO(case["text"]), opts)
    else:
        with tempfile.NamedTemporaryFile("wb", suffix=".txt", delete=False) as fh:
            fh.write(case["text"].encode("utf-8"))
        try:
            with open(fh.name, "r", encoding="utf-8") as f:
                pairs, mm = _scan_lines(f, opts)
        finally:
            os.unlink(fh.name)
    if mm is not None and opts.num_vertices is None and not opts.use_max_id:
        arr = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
        if len(arr) and (arr.min() < 1 or arr.max() > mm):
            raise EdgeListParseError(f"MatrixMarket ids outside [1, {mm}]")
        g = GO.from_edges_arrays(arr - 1, num_vertices=mm)
        g["orig_ids"] = np.arange(1, g["n"] + 1)
        return g
    return GO.from_edges_arrays(np.asarray(pairs, dtype=np.int64).reshape(-1, 2),
                                num_vertices=opts.num_vertices, use_max_id=opts.use_max_id)


@pytest.mark.parametrize("case", CASES, ids=[f"{c['name']}-{c['mode']}" for c in CASES])
def test_parse_case_matches_reference(case):
    if "error" in case:
        with pytest.raises(Exception) as ei:
            _host_load(case)
        exc = ei.value
        if case["error"] == "EdgeListParseError" and isinstance(exc, GO.OracleParseError):
            return  # range errors raised by the graph oracle (message differs)
        assert type(exc).__name__ == case["error"]
        assert str(exc) == case["message"]
        assert getattr(exc, "line", None) == case["line"]
        return
    g = _host_load(case)
    assert g["n"] == case["n"]
    assert np.asarray(g["edges"]).tolist() == case["edges"]
    assert [str(x) for x in g["orig_ids"]] == case["orig_ids"]
