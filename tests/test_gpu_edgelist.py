"""Edge-list parsing on the GPU (gd_parse_edge_list) against the reference's
own outputs (tests/golden/parse_cases.json): graph arrays, or error class,
message and line number.  ASCII inputs must take the device route."""
import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1506_04322_b200 as gd  # noqa: E402
from paper_1506_04322_b200 import edgelist as EL  # noqa: E402
from paper_1506_04322_b200 import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu
CASES = json.loads((ROOT / "tests" / "golden" / "parse_cases.json").read_text())


def _opts(d):
    d = dict(d)
    if "comment_prefixes" in d:
        d["comment_prefixes"] = tuple(d["comment_prefixes"])
    return gd.ParseOptions(**d)


def _load(case):
    opts = _opts(case["opts"])
    if case["mode"] == "text":
        return gd.Graph.from_text(case["text"], opts)
    with tempfile.NamedTemporaryFile("wb", suffix=".txt", delete=False) as fh:
        fh.write(case["text"].encode("utf-8"))
    try:
        return gd.Graph.from_file(fh.name, opts)
    finally:
        os.unlink(fh.name)


def _expected_route(case):
    t = case["text"]
    if not t.isascii() or "overflow" in case["name"]:
        return "host"
    if case["mode"] == "file" and "\r" in t.replace("\r\n", ""):
        return "host"  # a lone '\r' is a line break under universal newlines
    return "device"


@pytest.mark.parametrize("case", CASES, ids=[f"{c['name']}-{c['mode']}" for c in CASES])
def test_device_parse_matches_reference(case):
    EL.last_route = None
    if "error" in case:
        with pytest.raises(Exception) as ei:
            _load(case)
        exc = ei.value
        assert type(exc).__name__ == case["error"], exc
        assert str(exc) == case["message"]
        assert getattr(exc, "line", None) == case["line"]
    else:
        g = _load(case)
        assert g.n == case["n"]
        assert np.asarray(g.edges).tolist() == case["edges"]
        assert [str(x) for x in g.orig_ids] == case["orig_ids"]
    if EL.last_route is not None:
        assert EL.last_route == _expected_route(case)


def test_load_edge_list_io_objects():
    import io
    text = "# c\n0 1\n1 2\n"
    g = gd.load_edge_list(io.StringIO(text))
    assert g.n == 3 and g.m == 2 and EL.last_route == "device"
    g2 = gd.load_edge_list(["0 1\n", "1 2\n"])  # iterable of lines: CPython rules
    assert g2.n == 3 and g2.m == 2 and EL.last_route == "host"


def test_config2_text_round_trip():
    """A config-2-sized edge list (459k lines) parsed on the device equals the
    graph built from the same pairs; to_edge_list_text reproduces it."""
    raw = W.config_graph("c2_chung_lu")
    lines = "\n".join(f"{u}\t{v}" for u, v in raw.pairs.tolist()) + "\n"
    t0 = time.perf_counter()
    g = gd.Graph.from_text(lines, gd.ParseOptions(num_vertices=raw.n))
    dt = time.perf_counter() - t0
    assert EL.last_route == "device"
    ref = gd.Graph.from_edges(raw.pairs, gd.ParseOptions(num_vertices=raw.n))
    assert g.n == ref.n and np.array_equal(np.asarray(g.edges), np.asarray(ref.edges))
    g3 = gd.Graph.from_text(gd.to_edge_list_text(ref), gd.ParseOptions(num_vertices=raw.n))
    assert np.array_equal(np.asarray(g3.edges), np.asarray(ref.edges))
    print(f"parsed {len(lines) / 1e6:.1f} MB in {dt * 1e3:.1f} ms")
