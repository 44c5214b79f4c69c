"""Generate the golden vectors of tests/golden/ by running the REFERENCE.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--c2]

Outputs (committed):
  small_graphs.json  reference graphlet_census + micro_table on the reference
                     test-suite graph families (canonical graphs, zoo, G(n,p)
                     corpus, degenerate n, beyond-64-bit case)
  c1.npz / configs.json   config 1 (ER 2000/10000): reference counts, the full
                     reference micro_table, and sha256 fingerprints of the
                     generated pairs and of the reference-sanitised edges
  c4_batch.npz       reference feature_matrix counts of all 4096 config-4
                     graphs (int64, 17 columns)
  c2 (with --c2)     config 2 global counts + micro_table sha256 and sampled
                     rows (the full reference per-edge run takes ~10 min on 8
                     cores)
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

import graphlets as R  # noqa: E402  (the reference)
from graphlets import generate as RG  # noqa: E402
from graphlets.analytics import feature_matrix  # noqa: E402

from paper_1506_04322_b200 import workloads as W  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def counts_json(f) -> dict:
    return {k: str(int(v)) for k, v in f.counts.items()}


def small_cases():
    cases = []
    canon = {
        "K3": RG.complete_graph(3), "K4": RG.complete_graph(4), "C4": RG.cycle_graph(4),
        "C5": RG.cycle_graph(5), "P4": RG.path_graph(4), "K1,3": RG.star_graph(3),
        "K1,5": RG.star_graph(5), "diamond": RG.diamond_graph(), "paw": RG.paw_graph(),
        "2K2": RG.two_disjoint_edges_graph(), "K5+pendant": RG.clique_plus_pendant(5),
    }
    cases += list(canon.items())
    for n in (0, 1, 2, 3):
        cases.append((f"empty{n}", RG.empty_graph(n)))
    # zoo (test_census.py:406-456 families)
    rng = np.random.default_rng(7)
    for seed in range(3):
        a, b = 6, 8
        r = np.random.default_rng(seed)
        e = [(i, a + j) for i in range(a) for j in range(b) if r.random() < 0.4]
        cases.append((f"bipartite{seed}", R.Graph(a + b, np.asarray(e, dtype=np.int64).reshape(-1, 2))))
    for seed in range(3):
        r = np.random.default_rng(seed)
        e = [(int(r.integers(0, v)), v) for v in range(1, 24)]
        cases.append((f"tree{seed}", R.Graph(24, np.asarray(e, dtype=np.int64))))
    grid = []
    for rr in range(4):
        for cc in range(5):
            v = rr * 5 + cc
            if cc + 1 < 5:
                grid.append((v, v + 1))
            if rr + 1 < 4:
                grid.append((v, v + 5))
    cases.append(("grid4x5", R.Graph(20, np.asarray(grid, dtype=np.int64))))
    cases.append(("tri+17isolated", R.Graph(20, np.asarray([[0, 1], [1, 2], [2, 0]]))))
    q3 = [(a, b) for a in range(8) for b in range(a + 1, 8) if bin(a ^ b).count("1") == 1]
    cases.append(("Q3", R.Graph(8, np.asarray(q3, dtype=np.int64))))
    for seed in range(3):
        cases.append((f"dense_complement{seed}",
                      R.complement(RG.gnp_random_graph(14, 0.2, seed=seed))))
    cases.append(("beyond64", R.Graph(200_000, np.asarray([[0, 1], [1, 2], [5, 6]]))))
    # G(n, p) corpus in the style of test_acceptance.py:43-56
    probs = np.arange(1, 10) / 10
    for i in range(120):
        n = int(rng.integers(4, 41))
        p = float(rng.choice(probs))
        cases.append((f"G({n},{p:.1f})#{i}", RG.gnp_random_graph(n, p, seed=int(rng.integers(1 << 31)))))
    # a few denser, larger ones with hubs
    for i in range(6):
        cases.append((f"BA(200,{i + 2})", RG.powerlaw_cluster_graph(200, i + 2, seed=i)))
    return cases


def make_small():
    out = []
    for name, g in small_cases():
        f = R.graphlet_census(g)
        if g.n <= 30:
            assert f == R.oracle_census(g), name
        tab = R.micro_table(g)
        out.append({"name": name, "n": g.n, "edges": g.edges.tolist(),
                    "counts": counts_json(f), "micro": tab.tolist()})
    (HERE / "small_graphs.json").write_text(json.dumps(out))
    print("small graphs:", len(out))


def ref_graph(raw: W.RawGraph):
    return R.Graph.from_edges(raw.pairs, R.ParseOptions(num_vertices=raw.n))


def make_configs(with_c2: bool):
    cfg_path = HERE / "configs.json"
    configs = json.loads(cfg_path.read_text()) if cfg_path.exists() else {}
    workers = os.cpu_count()
    names = ["c1_er"] + (["c2_chung_lu"] if with_c2 else [])
    for name in names:
        raw = W.config_graph(name)
        g = ref_graph(raw)
        g.adj_lists()
        g.edge_columns()
        t0 = time.time()
        f = R.graphlet_census(g, R.ParallelConfig(workers=workers))
        t_glob = time.time() - t0
        t0 = time.time()
        tab = R.micro_table(g, R.ParallelConfig(workers=workers))
        t_micro = time.time() - t0
        assert R.frequencies_from_micro(g, tab) == f
        rng = np.random.default_rng(99)
        sample = np.sort(rng.choice(g.m, size=min(g.m, 512), replace=False))
        configs[name] = {
            "n": g.n, "m": g.m,
            "pairs_sha256": sha(raw.pairs), "edges_sha256": sha(g.edges),
            "counts": counts_json(f), "micro_sha256": sha(tab),
            "sample_idx": sample.tolist(), "sample_rows": tab[sample].tolist(),
            "reference_seconds": {"graphlet_census": t_glob, "micro_table": t_micro,
                                  "workers": workers},
        }
        if name == "c1_er":
            np.savez_compressed(HERE / "c1.npz", micro=tab, edges=g.edges.astype(np.int32))
        print(name, g.n, g.m, f"global {t_glob:.1f}s micro {t_micro:.1f}s")
        cfg_path.write_text(json.dumps(configs, indent=1))


def make_batch():
    raws = W.config_batch()
    graphs = [ref_graph(r) for r in raws]
    t0 = time.time()
    fm = feature_matrix(graphs)
    dt = time.time() - t0
    counts = np.asarray([[int(R.graphlet_census(g).counts[c]) for c in R.CLASS_IDS]
                         for g in graphs[:32]], dtype=np.int64)
    rows = fm.rows
    assert np.array_equal(rows[:32], counts.astype(np.float64))
    exact = np.asarray([[int(x) for x in r] for r in rows], dtype=np.int64)
    assert np.array_equal(exact.astype(np.float64), rows)
    np.savez_compressed(HERE / "c4_batch.npz", counts=exact,
                        n=np.asarray([g.n for g in graphs], dtype=np.int64),
                        m=np.asarray([g.m for g in graphs], dtype=np.int64))
    meta_path = HERE / "configs.json"
    configs = json.loads(meta_path.read_text()) if meta_path.exists() else {}
    configs["c4_batch"] = {"graphs": len(graphs), "sum_m": int(sum(g.m for g in graphs)),
                           "sum_n": int(sum(g.n for g in graphs)),
                           "pairs_sha256": sha(np.concatenate([r.pairs for r in raws])),
                           "reference_seconds": {"feature_matrix_serial": dt}}
    meta_path.write_text(json.dumps(configs, indent=1))
    print("batch", len(graphs), f"{dt:.1f}s")


if __name__ == "__main__":
    if "--small" in sys.argv or len(sys.argv) == 1:
        make_small()
    if "--configs" in sys.argv or len(sys.argv) == 1 or "--c2" in sys.argv:
        make_configs("--c2" in sys.argv)
    if "--batch" in sys.argv or len(sys.argv) == 1:
        make_batch()


def make_graph_build():
    """Reference Graph.from_edges / Graph(n, edges) arrays on raw inputs with
    loops, duplicates, reciprocal pairs, sparse 64-bit and negative ids."""
    rng = np.random.default_rng(1234)
    cases = []
    cases.append(("spec_example", [[1, 2], [2, 1], [2, 2], [1, 3]], {}))
    big = rng.integers(-(1 << 62), 1 << 62, size=40)
    cases.append(("sparse64", big[rng.integers(0, 40, size=(300, 2))].tolist(), {}))
    cases.append(("negative_remap", [[-5, 3], [3, -5], [-5, -5], [7, 3], [-100, 7]], {}))
    cases.append(("declared_isolated", rng.integers(0, 30, size=(80, 2)).tolist(),
                  {"num_vertices": 50}))
    cases.append(("max_id", rng.integers(0, 30, size=(80, 2)).tolist(), {"use_max_id": True}))
    cases.append(("only_loops", [[3, 3], [4, 4]], {}))
    cases.append(("dups_heavy", rng.integers(0, 12, size=(500, 2)).tolist(), {}))
    out = []
    for name, pairs, opts in cases:
        g = R.Graph.from_edges(np.asarray(pairs, dtype=np.int64).reshape(-1, 2),
                               R.ParseOptions(**opts))
        out.append({"name": name, "pairs": [[int(a), int(b)] for a, b in pairs], "opts": opts,
                    "n": g.n, "m": g.m, "edges": g.edges.tolist(), "indptr": g.indptr.tolist(),
                    "indices": g.indices.tolist(), "edge_slot_ids": g.edge_slot_ids.tolist(),
                    "degrees": g.degrees.tolist(), "orig_ids": [str(x) for x in g.orig_ids]})
    errors = []
    for name, pairs, opts in (("declared_out_of_range", [[0, 5]], {"num_vertices": 5}),
                              ("declared_negative", [[-1, 2]], {"num_vertices": 5}),
                              ("max_id_negative", [[-1, 2]], {"use_max_id": True})):
        try:
            R.Graph.from_edges(np.asarray(pairs, dtype=np.int64), R.ParseOptions(**opts))
            errors.append({"name": name, "pairs": pairs, "opts": opts, "error": None})
        except Exception as exc:  # noqa: BLE001
            errors.append({"name": name, "pairs": pairs, "opts": opts,
                           "error": type(exc).__name__})
    for name, n, edges in (("init_loop", 4, [[1, 1]]), ("init_dup", 4, [[0, 1], [1, 0]]),
                           ("init_range", 4, [[0, 4]])):
        try:
            R.Graph(n, np.asarray(edges, dtype=np.int64))
            errors.append({"name": name, "n": n, "edges": edges, "error": None})
        except Exception as exc:  # noqa: BLE001
            errors.append({"name": name, "n": n, "edges": edges, "error": type(exc).__name__})
    (HERE / "graph_build.json").write_text(json.dumps({"cases": out, "errors": errors}))
    print("graph build cases:", len(out), "errors:", len(errors))


if __name__ == "__main__" and "--graphs" in sys.argv:
    make_graph_build()


def make_micro_roles():
    """Reference MicroCounts (all 14 roles) and micro_csv text for a few
    graphs, including original-id remapping."""
    from graphlets.census import micro_csv, micro_census, MicroCounts  # noqa: F401
    roles = ("tt1", "tt0", "susv1", "susv0", "ts1", "ts0", "ss1", "ss0", "ti1", "ti0",
             "si1", "si0", "ii1", "ii0")
    out = []
    graphs = [("paw", RG.paw_graph()), ("diamond", RG.diamond_graph()),
              ("gnp15", RG.gnp_random_graph(15, 0.5, seed=3)),
              ("remapped", R.Graph.from_edges(np.asarray([[100, 200], [200, 300], [300, 100],
                                                          [300, 4000], [7, 100]])))]
    for name, g in graphs:
        tab = R.micro_table(g)
        rows = []
        for e in g.edge_refs():
            mc = micro_census(g, e)
            rows.append([getattr(mc, r) for r in roles] + [mc.local.indep3])
        out.append({"name": name, "n": g.n, "edges": g.edges.tolist(),
                    "orig_ids": g.orig_ids.tolist(), "micro": tab.tolist(), "roles": rows,
                    "csv": micro_csv(g, tab)})
    (HERE / "micro_roles.json").write_text(json.dumps({"roles": roles, "graphs": out}))
    print("micro roles:", len(out))


if __name__ == "__main__" and "--roles" in sys.argv:
    make_micro_roles()


PARSE_CASES = [
    # (name, text, opts, modes)  modes: "text" (Graph.from_text), "file"
    # (Graph.from_file: UTF-8, universal newlines)
    ("simple", "0 1\n1 2\n2 0\n", {}, ("text", "file")),
    ("comments", "# header\n% mm comment\n0 1\n  # indented comment\n1 2\n", {}, ("text", "file")),
    ("commas_third_col", "0,1\n1,2,5.5\n2 3 w=7\n", {}, ("text", "file")),
    ("whitespace", "\t 3   4 \t\n\n   \n5\t6\n", {}, ("text", "file")),
    ("crlf", "0 1\r\n1 2\r\n2 0\r\n", {}, ("text", "file")),
    ("lone_cr", "0 1\r1 2\r2 3\r", {}, ("text", "file")),
    ("loops_dups_reciprocal", "1 1\n1 2\n2 1\n1 2\n3 1\n", {}, ("text", "file")),
    ("ids_64bit", "9223372036854775807 5\n-9223372036854775808 5\n", {}, ("text", "file")),
    ("negative_remap", "-5 3\n3 -5\n-100 7\n", {}, ("text", "file")),
    ("int_literals", "1_0 2\n+3 -4\n007 8\n0_0 9\n", {}, ("text", "file")),
    ("no_trailing_newline", "0 1\n1 2", {}, ("text", "file")),
    ("odd_whitespace", "0\x0b1\n2\x1c3\n4\x0c5\n", {}, ("text", "file")),
    ("commas_only_sep", ",,0,,1,,\n", {}, ("text", "file")),
    ("err_tokens", "0 1\n2\n3 4\n", {}, ("text", "file")),
    ("err_tokens_commas", "0 1\n,,,\n", {}, ("text", "file")),
    ("err_nonint", "0 1\n1 x\n", {}, ("text", "file")),
    ("err_float", "0 1.5\n", {}, ("text", "file")),
    ("err_underscore", "1_ 2\n", {}, ("text", "file")),
    ("err_double_underscore", "1__0 2\n", {}, ("text", "file")),
    ("err_first_of_two", "0 1\na b\nc\n", {}, ("text", "file")),
    ("err_nul", "0\x001\n", {}, ("text", "file")),
    ("err_empty", "", {}, ("text", "file")),
    ("err_comments_only", "# a\n% b\n\n", {}, ("text", "file")),
    ("mm_header", "%%MatrixMarket matrix coordinate pattern symmetric\n% c\n5 5 3\n1 2\n2 3\n3 1\n",
     {}, ("text", "file")),
    ("mm_no_header", "%%MatrixMarket matrix coordinate pattern\n1 2\n2 3\n", {}, ("text", "file")),
    ("mm_out_of_range", "%%MatrixMarket x\n3 3 2\n1 4\n", {}, ("text", "file")),
    ("mm_zero_id", "%%MatrixMarket x\n3 3 2\n0 2\n", {}, ("text", "file")),
    ("mm_bad_header", "%%MatrixMarket x\n3 x 2\n1 2\n", {}, ("text", "file")),
    ("mm_num_vertices", "%%MatrixMarket x\n4 4 2\n1 2\n2 3\n", {"num_vertices": 10}, ("text",)),
    ("mm_use_max_id", "%%MatrixMarket x\n4 4 2\n1 2\n2 3\n", {"use_max_id": True}, ("text",)),
    ("mm_after_data", "0 1\n%%MatrixMarket\n3 3 3\n", {}, ("text",)),
    ("mm_custom_prefix", "%%MatrixMarket x\n2 2 1\n1 2\n", {"comment_prefixes": ["#"]}, ("text",)),
    ("custom_prefix", "// c\n0 1\n", {"comment_prefixes": ["//"]}, ("text",)),
    ("custom_prefix_hash_data", "# c\n0 1\n", {"comment_prefixes": ["//"]}, ("text",)),
    ("empty_prefix", "0 1\n", {"comment_prefixes": [""]}, ("text",)),
    ("declared_n", "0 1\n2 3\n", {"num_vertices": 10}, ("text",)),
    ("declared_out_of_range", "0 1\n12 3\n", {"num_vertices": 10}, ("text",)),
    ("use_max_id", "0 5\n", {"use_max_id": True}, ("text",)),
    ("unicode_digit", "0 1\n١ 2\n", {}, ("text", "file")),
    ("unicode_space", "0\u00a01\n2\u20033\n", {}, ("text", "file")),
    ("overflow", "99999999999999999999 1\n", {}, ("text",)),
    ("overflow_then_error", "99999999999999999999 1\nx y\n", {}, ("text",)),
]


def _random_edge_text(seed: int, lines: int) -> str:
    rng = np.random.default_rng(seed)
    seps = [" ", "\t", ",", " , ", "  "]
    out = []
    for i in range(lines):
        r = rng.random()
        if r < 0.05:
            out.append("# comment %d" % i)
        elif r < 0.08:
            out.append("")
        else:
            u, v = rng.integers(0, 300, size=2)
            line = f"{u}{seps[rng.integers(0, len(seps))]}{v}"
            if rng.random() < 0.2:
                line += f" {rng.integers(0, 9)}"
            if rng.random() < 0.1:
                line = "  " + line + " \t"
            out.append(line)
    return "\n".join(out) + "\n"


PARSE_CASES.append(("random_2000", _random_edge_text(7, 2000), {}, ("text", "file")))
PARSE_CASES.append(("random_2000_crlf", _random_edge_text(8, 2000).replace("\n", "\r\n"), {},
                    ("text", "file")))


def make_parse():
    """Reference Graph.from_text / Graph.from_file on edge-list texts covering
    its parsing rules and error messages (graph.py:223-285)."""
    import tempfile
    out = []
    for name, text, opts, modes in PARSE_CASES:
        o = dict(opts)
        if "comment_prefixes" in o:
            o["comment_prefixes"] = tuple(o["comment_prefixes"])
        for mode in modes:
            try:
                if mode == "text":
                    g = R.Graph.from_text(text, R.ParseOptions(**o))
                else:
                    with tempfile.NamedTemporaryFile("wb", suffix=".txt", delete=False) as fh:
                        fh.write(text.encode("utf-8"))
                    try:
                        g = R.Graph.from_file(fh.name, R.ParseOptions(**o))
                    finally:
                        os.unlink(fh.name)
                res = {"n": g.n, "edges": g.edges.tolist(), "orig_ids": [str(x) for x in g.orig_ids]}
            except Exception as exc:  # noqa: BLE001
                res = {"error": type(exc).__name__, "message": str(exc),
                       "line": getattr(exc, "line", None)}
            out.append({"name": name, "mode": mode, "text": text, "opts": opts, **res})
    (HERE / "parse_cases.json").write_text(json.dumps(out, indent=0))
    print("parse cases:", len(out))


if __name__ == "__main__" and "--parse" in sys.argv:
    make_parse()


def make_analytics():
    """Reference rank_edges / edge_weights / vertex_triangle_counts
    (analytics.py:142-194) on graphs with ties, pendants and remapped ids."""
    from graphlets.analytics import RANK_PATTERNS, edge_weights, rank_edges, vertex_triangle_counts
    graphs = [("star5", RG.star_graph(5)), ("k5_pendant", None), ("cycle4", RG.cycle_graph(4)),
              ("gnp20", RG.gnp_random_graph(20, 0.3, seed=3)),
              ("gnp40", RG.gnp_random_graph(40, 0.25, seed=11)),
              ("remapped", R.Graph.from_edges(np.asarray([[100, 200], [200, 300], [300, 100],
                                                          [300, 4000], [7, 100], [7, 300]])))]
    out = []
    for name, g in graphs:
        if g is None:
            k5 = [[a, b] for a in range(5) for b in range(a + 1, 5)] + [[4, 5]]
            g = R.Graph(6, np.asarray(k5))
        tab = R.micro_table(g)
        rec = {"name": name, "n": g.n, "edges": g.edges.tolist(),
               "orig_ids": g.orig_ids.tolist(), "micro": tab.tolist(),
               "vertex_triangles": vertex_triangle_counts(g, tab).tolist(), "patterns": {}}
        for p in RANK_PATTERNS:
            rec["patterns"][p] = {
                "weights": edge_weights(g, p, table=tab).tolist(),
                "ranked": [[r.index, int(r.u), int(r.v), int(r.weight)] for r in rank_edges(g, p)],
                "top3": [[r.index, int(r.u), int(r.v), int(r.weight)]
                         for r in rank_edges(g, p, top_k=3)]}
        out.append(rec)
    (HERE / "analytics.json").write_text(json.dumps(out))
    print("analytics graphs:", len(out))


if __name__ == "__main__" and "--analytics" in sys.argv:
    make_analytics()


def make_selection():
    """Reference SelectionState op streams (selection.py) with the counts
    after every operation, and the errors of invalid operations."""
    from graphlets.selection import SelectionOp, SelectionState
    streams = []

    def run(name, base, ops, active=(), excluded=()):
        st = SelectionState(base, active=active, excluded_edges=excluded)
        rec = {"name": name, "n": base.n, "edges": base.edges.tolist(), "active": list(active),
               "excluded": list(excluded),
               "initial": {k: str(v) for k, v in st.frequencies().counts.items()}, "steps": []}
        for op in ops:
            step = {"op": [op.action, op.vertex, op.u, op.v]}
            try:
                f = st.apply_one(op)
                step["counts"] = {k: str(v) for k, v in f.counts.items()}
                step["n"], step["m"] = f.n, f.m
            except Exception as exc:  # noqa: BLE001
                step["error"] = type(exc).__name__
            rec["steps"].append(step)
        streams.append(rec)

    k4 = RG.complete_graph(4)
    run("k4_build", k4, [SelectionOp("add_vertex", vertex=v) for v in range(4)]
        + [SelectionOp("add_edge", u=0, v=1), SelectionOp("remove_edge", u=2, v=3),
           SelectionOp("add_edge", u=2, v=3), SelectionOp("remove_vertex", vertex=3),
           SelectionOp("remove_vertex", vertex=3), SelectionOp("add_vertex", vertex=99),
           SelectionOp("remove_edge", u=0, v=0), SelectionOp("teleport", vertex=1),
           SelectionOp("add_edge", u=0), SelectionOp("remove_edge", u=0, v=1),
           SelectionOp("remove_vertex", vertex=0), SelectionOp("add_edge", u=0, v=1)])
    run("k4_excluded_init", k4, [SelectionOp("add_edge", u=2, v=3)], active=[0, 1, 2, 3],
        excluded=[5])

    def random_stream(name, base, steps, seed):
        rng = np.random.default_rng(seed)
        active = set()
        ops = []
        for _ in range(steps):
            kind = int(rng.integers(0, 4))
            if kind == 0:
                op = SelectionOp("add_vertex", vertex=int(rng.integers(base.n)))
            elif kind == 1:
                op = SelectionOp("remove_vertex", vertex=int(rng.integers(base.n)))
            else:
                eid = int(rng.integers(base.m))
                u, v = (int(x) for x in base.edges[eid])
                if kind == 2:
                    op = SelectionOp("remove_edge", u=u, v=v)
                elif u in active and v in active:
                    op = SelectionOp("add_edge", u=u, v=v)
                else:
                    op = SelectionOp("add_vertex", vertex=u)
            if op.action == "add_vertex":
                active.add(op.vertex)
            elif op.action == "remove_vertex":
                active.discard(op.vertex)
            ops.append(op)
        run(name, base, ops)

    random_stream("random_300", RG.random_graph_avg_degree(300, 8, seed=8), 120, 23)
    cl = W.chung_lu(1500, 2.1, 10.0, 300.0, seed=31)
    random_stream("chung_lu_1500", ref_graph(cl), 150, 7)
    dense = RG.gnp_random_graph(60, 0.5, seed=5)
    random_stream("gnp60_dense", dense, 200, 9)
    (HERE / "selection.json").write_text(json.dumps(streams))
    print("selection streams:", len(streams), sum(len(s["steps"]) for s in streams))


if __name__ == "__main__" and "--selection" in sys.argv:
    make_selection()
