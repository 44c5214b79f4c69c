"""INTEGRATION.md's reference-side binding (the `graphlets/_gpu.py` stub a
maintainer would add) run as written: the code block is extracted from
INTEGRATION.md into a stand-in `graphlets` package whose `census` / `errors`
modules provide the reference names the stub imports, then called through
the one-shot C entries gd_census_global_edges / gd_census_per_edge_edges on
duck-typed graphs, against the reference's golden outputs."""

import importlib
import os
import re
import sys
from types import SimpleNamespace

import numpy as np
import pytest

from helpers import GOLDEN, small_graphs

pytestmark = pytest.mark.gpu

ROOT = GOLDEN.parent.parent


def _stub_source() -> str:
    text = (ROOT / "INTEGRATION.md").read_text()
    m = re.search(r"```python\n(# graphlets/_gpu\.py.*?)```", text, re.S)
    assert m, "stub block missing from INTEGRATION.md"
    return m.group(1)


@pytest.fixture(scope="module")
def stub(tmp_path_factory):
    pkg = tmp_path_factory.mktemp("ref") / "graphlets"
    pkg.mkdir()
    (pkg / "__init__.py").write_text("")
    (pkg / "census.py").write_text(
        "from paper_1506_04322_b200.census import CensusSums, RAW_MICRO_FIELDS\n"
        "from paper_1506_04322_b200.census import frequencies_from_sums as _frequencies_from_sums\n")
    (pkg / "errors.py").write_text("from paper_1506_04322_b200.errors import ConsistencyError\n")
    (pkg / "_gpu.py").write_text(_stub_source())
    sys.path.insert(0, str(pkg.parent))
    os.environ["GD_LIBRARY"] = str(ROOT / "paper_1506_04322_b200" / "libgdgpu.so")
    try:
        yield importlib.import_module("graphlets._gpu")
    finally:
        sys.path.remove(str(pkg.parent))
        for k in [k for k in sys.modules if k == "graphlets" or k.startswith("graphlets.")]:
            del sys.modules[k]


def test_stub_global_and_per_edge_match_reference(stub):
    for name, n, edges, counts, micro in small_graphs():
        if not len(edges):
            continue
        g = SimpleNamespace(n=n, m=len(edges), edges=edges)  # a reference Graph's surface
        assert stub.graphlet_census(g).counts == counts, name
        assert np.array_equal(stub.micro_table(g), micro), name
