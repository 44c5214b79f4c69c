"""Host-side logic of the drop-in: closures, result type, config, classes,
C-ABI library surface.  CPU only (no device calls)."""

import re
from math import comb
from pathlib import Path

import numpy as np
import pytest

import paper_1506_04322_b200 as gd
from paper_1506_04322_b200 import _native as N
from paper_1506_04322_b200.census import CensusSums, frequencies_from_sums
from helpers import small_graphs
from oracle import oracle as O

ROOT = Path(__file__).resolve().parent.parent


def test_close_triads_hand_cases():
    # test_census.py:182-191 analogues
    assert gd.close_triads(3, 0, 0, 3) == {"g3_1": 1, "g3_2": 0, "g3_3": 0, "g3_4": 0}
    assert gd.close_triads(0, 4, 2, 4) == {"g3_1": 0, "g3_2": 2, "g3_3": 2, "g3_4": 0}
    with pytest.raises(gd.ConsistencyError):
        gd.close_triads(4, 0, 0, 5)
    with pytest.raises(gd.ConsistencyError):
        gd.close_triads(0, 3, 0, 5)


def test_close_quads_hand_cases():
    f = gd.close_quads(CensusSums(n_tt=1, n_ts=4, outside=4), n=4, m=5)
    assert f["g4_2"] == 1 and sum(f.values()) == 1
    f = gd.close_quads(CensusSums(cycle4=4, n_susv=4, outside=4), n=4, m=4)
    assert f["g4_4"] == 1 and f["g4_6"] == 0 and sum(f.values()) == 1
    with pytest.raises(gd.ConsistencyError):
        gd.close_quads(CensusSums(clique4=5), n=5, m=6)
    with pytest.raises(gd.ConsistencyError):
        gd.close_quads(CensusSums(cycle4=4, n_susv=2), n=5, m=4)


def test_closures_match_reference_on_golden_sums():
    for name, n, edges, counts, micro in small_graphs():
        sums = O.sums_from_rows(micro, n, len(edges))
        f = frequencies_from_sums(CensusSums.from_tuple(sums), n, len(edges))
        assert f.counts == counts, name


def test_beyond_64_bits_exact():
    n = 200_000
    f = frequencies_from_sums(CensusSums(), n, 0)
    assert f.counts["g4_11"] == comb(n, 4) > 2 ** 63
    f.validate()


def test_frequencies_validate_and_eq():
    f = frequencies_from_sums(CensusSums(), 5, 0)
    g = gd.GraphletFrequencies(counts=dict(f.counts), n=5, m=0)
    assert f == g
    bad = dict(f.counts)
    bad["g2_1"] = 1
    with pytest.raises(gd.ConsistencyError):
        gd.GraphletFrequencies(counts=bad, n=5, m=0).validate()
    with pytest.raises(ValueError):
        gd.GraphletFrequencies(counts={"g2_1": 0}, n=1, m=0)


def test_parallel_config_validation():
    gd.ParallelConfig(workers=4, batch_size=1, ordering="degree-desc")
    for kw in ({"workers": 0}, {"batch_size": 0}, {"batch_size": 4097}, {"ordering": "x"}):
        with pytest.raises(ValueError):
            gd.ParallelConfig(**kw)


def test_classes():
    assert len(gd.CLASS_IDS) == 17 and gd.CLASS_IDS[0] == "g2_1" and gd.CLASS_IDS[-1] == "g4_11"
    assert gd.classes_for(4, connected_only=True) == ("g4_1", "g4_2", "g4_3", "g4_4", "g4_5", "g4_6")
    for c in gd.CLASS_IDS:
        assert gd.complement_class(gd.complement_class(c)) == c


def test_gfd_host_math():
    name, n, edges, counts, _ = small_graphs()[-1]
    f = gd.GraphletFrequencies(counts=counts, n=n, m=len(edges))
    v = gd.gfd(f, 4, "all")
    assert abs(sum(v.values) - 1.0) < 1e-12


def _header_symbols():
    text = (ROOT / "include" / "gd_api.h").read_text()
    return sorted(set(re.findall(r"GD_API[^;]*?\b(gd_[a-z0-9_]+)\s*\(", text, re.S)))


def test_library_exports_every_declared_symbol():
    lib = N.load_library()
    declared = _header_symbols()
    assert len(declared) >= 15
    bound = {name for name, _, _ in N.SIGNATURES}
    assert set(declared) == bound
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.gd_version() == 1


def test_no_cpu_fallback_without_device():
    lib = N.load_library()
    if lib.gd_device_ok():
        pytest.skip("a device is present")
    with pytest.raises(gd.DeviceError):
        gd.Graph(3, np.asarray([[0, 1], [1, 2]]))


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(gd.DeviceError):
        N.load_library(tmp_path / "libgdgpu.so")


def test_product_does_not_import_oracle():
    pkg = ROOT / "paper_1506_04322_b200"
    for p in pkg.rglob("*.py"):
        txt = p.read_text()
        assert "import oracle" not in txt and "from oracle" not in txt, p


def test_library_closures_match_python_closures():
    """gd_close_counts (exact 128-bit closures for batches) == the Python-int
    closures, and flags the same failing identities."""
    import ctypes
    from paper_1506_04322_b200.census import counts_as_ints
    cases = small_graphs()
    G = len(cases)
    sums = np.zeros((G, 13, 2), dtype=np.uint64)
    ns = np.zeros(G, dtype=np.int64)
    ms = np.zeros(G, dtype=np.int64)
    for i, (name, n, edges, counts, micro) in enumerate(cases):
        for k, v in enumerate(O.sums_from_rows(micro, n, len(edges))):
            sums[i, k] = (v & ((1 << 64) - 1), v >> 64)
        ns[i], ms[i] = n, len(edges)
    bad = sums.copy()
    bad[0, 0, 0] += 1  # triangle total not divisible by 3
    L = N.load_library()
    for arr, expect_bad in ((sums, False), (bad, True)):
        out = np.zeros((G, 17, 2), dtype=np.int64)
        st = np.zeros(G, dtype=np.int32)
        N.check(L.gd_close_counts(N.ptr(np.ascontiguousarray(arr), ctypes.c_uint64), N.ptr(ns),
                                  N.ptr(ms), G, N.ptr(out),
                                  st.ctypes.data_as(ctypes.POINTER(ctypes.c_int))))
        for i, (name, n, edges, counts, micro) in enumerate(cases):
            if expect_bad and i == 0:
                assert st[0] == 1  # first identity: triangle closure
                continue
            assert st[i] == 0, name
            assert counts_as_ints(out[i]) == [counts[c] for c in gd.CLASS_IDS], name


def test_feature_matrix_skips_like_the_reference(monkeypatch):
    """Batched feature_matrix records a failing graph as the reference does
    (analytics.py:114-116: f"{type(exc).__name__}: {exc}" with the numbers)
    and zips labels with graphs (a shorter label list drops graphs)."""
    import numpy as np
    import paper_1506_04322_b200.analytics as A

    class FakeBatch:
        num_graphs = 3
        n_per_graph = np.array([5, 5, 5])
        m_per_graph = np.array([1, 1, 1])

    monkeypatch.setattr(A.GraphBatch, "from_graphs", staticmethod(lambda gs: FakeBatch()))
    sums = np.zeros((3, 26), np.uint64)
    sums[1, 0] = 4  # triangle sum 4: not divisible by 3
    counts = np.zeros((3, 17, 2), np.int64)
    status = np.array([0, 1, 0], dtype=np.int32)
    monkeypatch.setattr(A, "batch_counts", lambda b, with_sums=False: (counts, status, sums))
    fm = A.feature_matrix([object(), object(), object()], labels=["a", "b", "c"])
    assert fm.skipped == [("b", "ConsistencyError: triangle closure: 4 not divisible by 3")]
    assert fm.labels == ["a", "c"]
    fm = A.feature_matrix([object(), object(), object()], labels=["a", "b"])
    assert fm.labels == ["a"] and len(fm.skipped) == 1


def test_bench_roofline_block_is_a_bound():
    """bench.py's roofline block: the kernel and DRAM traffic belong to the
    phase that dominates the live timings (profiles/ncu_summary.json), the
    measured HBM fractions never exceed 1 and `frac` is achieved / peak."""
    import importlib.util
    import json
    root = Path(__file__).resolve().parent.parent
    spec = importlib.util.spec_from_file_location("bench_mod", root / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    summ = json.loads((root / "profiles" / "ncu_summary.json").read_text())
    deg = np.full(1000, 30, dtype=np.int64)
    for (cfg, mode), phases in {
        ("c3_rmat20", "per_edge"): {"schedule": 1.1, "tri_frames": 12.4, "trisum_frames": 5.3,
                                    "c4_coop": 19.6, "c4_smem": 2.0, "finalize": 1.4},
        ("c5_chung_lu_4m", "global"): {"schedule": 3.9, "tri_frames": 184.8, "c4_coop": 116.7,
                                       "c4_smem": 3.8, "finalize": 1.5},
    }.items():
        stats = {"c4_heavy_wedges": 5_570_596_165, "tri_items": 4_423_179_103}
        ms = sum(phases.values())
        r = bench.roofline_block(cfg, mode, phases, stats, 1000, 15000, deg, ms, 6457.1, "measured")
        dom = max(("c4_coop", "tri_frames"), key=lambda k: phases[k])
        assert r["phase"] == dom and r["bound"] == "hbm"
        assert r["kernel"].startswith(bench.PHASE_KERNELS[dom])
        assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
        names = [k for k in summ[f"{cfg}/{mode}"]["kernels"] if k.startswith(bench.PHASE_KERNELS[dom])]
        assert r["traffic"] == sum(summ[f"{cfg}/{mode}"]["kernels"][k]["dram_bytes"] for k in names)
        assert 0 < r["hbm_measured"]["kernel_frac"] <= 1.0
        assert 0 < r["hbm_measured"]["census_frac"] <= 1.0
