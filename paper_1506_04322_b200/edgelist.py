"""Edge-list loading: the reference's load_edge_list /
Graph.from_file / Graph.from_text (graph.py:159-166, 223-285) with the text
tokenised on the GPU.

ASCII input (the common case) goes through ``gd_parse_edge_list``: the bytes
are copied to the device once, every line is classified and its two ids are
parsed there, and the pairs are handed to the device graph build without
ever materialising a host pair array.  Input the ASCII rules cannot decide
exactly like CPython (non-ASCII bytes -- Unicode whitespace and digits --,
a lone carriage return under universal newlines, ids beyond int64) and
generic iterables of lines are parsed by ``_load_lines``, a line-for-line
restatement of the reference loop, so both routes raise the same
``EdgeListParseError`` (message and 1-based line number) on the same input.
"""

from __future__ import annotations

import ctypes
import io
from pathlib import Path
from typing import IO, Iterable

import numpy as np

from . import _native as N
from .errors import EdgeListParseError
from .graph import Graph, ParseOptions, _Handle

_ERR_TOKENS, _ERR_NONINT, _ERR_MM_HEADER, _ERR_NO_DATA = 1, 2, 3, 4
# which route parsed the last input: "device" or "host" (tests / bench)
last_route = None
_NO_DATA_MSG = "no data lines in input (empty or comments only)"


# ---------------------------------------------------------------------------
# device route
# ---------------------------------------------------------------------------
def _graph_from_device_pairs(ptr: int, k: int, n: int, mode: int, orig_ids=None) -> Graph:
    out = ctypes.c_void_p()
    N.check(N.lib().gd_graph_create(ctypes.c_void_p(ptr), k, int(n), mode, N.GD_INPUT_DEVICE,
                                    ctypes.byref(out)))
    return Graph(0, None, orig_ids=orig_ids, _handle=_Handle(out.value))


def _device_prefixes(options: ParseOptions):
    prefixes = options.comment_prefixes
    if isinstance(prefixes, str):
        prefixes = (prefixes,)
    enc = []
    for p in prefixes:
        if not isinstance(p, str) or not p.isascii() or len(p) >= 64:
            return None
        enc.append(p.encode("ascii"))
    if len(enc) > 16:
        return None
    return enc


def _parse_device(data, options: ParseOptions, cr_newline: bool, keep=None) -> Graph | None:
    """Parse `data` (bytes, or an (address, length) view of `keep`) on the
    GPU; None when the input needs CPython's rules."""
    enc = _device_prefixes(options)
    if enc is None:
        return None
    N.require_device()
    L = N.lib()
    arr = (ctypes.c_char_p * max(1, len(enc)))(*enc)
    mm_shift = options.num_vertices is None and not options.use_max_id
    flags = (N.GD_PARSE_CR_NEWLINE if cr_newline else 0) | (N.GD_PARSE_MM_SHIFT if mm_shift else 0)
    h = ctypes.c_void_p()
    ptr, size = data if isinstance(data, tuple) else (data, len(data))
    N.check(L.gd_parse_edge_list(ptr, size, arr, len(enc), flags, ctypes.byref(h)))
    global last_route
    try:
        info = (ctypes.c_int64 * 12)()
        N.check(L.gd_parsed_info(h, info))
        k, mm_rows, kind, line, off, ln, fallback, lo, hi = (int(info[i]) for i in range(9))
        if fallback:
            return None
        last_route = "device"
        if kind:
            raw = ctypes.string_at(ptr + off, ln) if isinstance(ptr, int) else ptr[off:off + ln]
            text = raw.decode("ascii").strip() if kind in (1, 2) else ""
            if kind == _ERR_TOKENS:
                raise EdgeListParseError(f"expected at least 2 integer tokens, got {text!r}", line)
            if kind == _ERR_NONINT:
                raise EdgeListParseError(f"non-integer vertex id in {text!r}", line)
            if kind == _ERR_MM_HEADER:
                raise EdgeListParseError("malformed MatrixMarket size header", line)
            raise EdgeListParseError(_NO_DATA_MSG)
        ptr = L.gd_parsed_pairs(h) or 0
        if mm_rows >= 0 and mm_shift:
            # graph.py:277-283: 1-based ids within [1, rows], reported as such
            if k and (lo < 1 or hi > mm_rows):
                raise EdgeListParseError(f"MatrixMarket ids outside [1, {mm_rows}]")
            g = _graph_from_device_pairs(ptr, k, mm_rows, N.GD_IDS_DECLARED)
            return Graph(0, None, orig_ids=np.arange(1, g.n + 1, dtype=np.int64), _handle=g._h)
        if options.num_vertices is not None:
            return _graph_from_device_pairs(ptr, k, options.num_vertices, N.GD_IDS_DECLARED)
        if options.use_max_id:
            return _graph_from_device_pairs(ptr, k, 0, N.GD_IDS_MAX_ID)
        return _graph_from_device_pairs(ptr, k, 0, N.GD_IDS_REMAP)
    finally:
        L.gd_parsed_free(h)


# ---------------------------------------------------------------------------
# CPython rules (restatement of graph.py:239-285, for the inputs above)
# ---------------------------------------------------------------------------
def _tokenize(line: str) -> list[str]:
    return line.replace(",", " ").split()


def _scan_lines(source: Iterable[str], options: ParseOptions):
    """The reference's line loop (graph.py:245-272): (pairs, MatrixMarket rows
    or None), raising EdgeListParseError like it."""
    pairs: list[tuple[int, int]] = []
    is_matrix_market = False
    mm_rows: int | None = None
    saw_data = False
    for lineno, raw in enumerate(source, start=1):
        line = raw.strip()
        if not line:
            continue
        if line.startswith("%%MatrixMarket"):
            is_matrix_market = True
            continue
        if line.startswith(options.comment_prefixes):
            continue
        tokens = _tokenize(line)
        if is_matrix_market and not saw_data:
            saw_data = True
            if len(tokens) == 3:
                try:
                    rows, cols = int(tokens[0]), int(tokens[1])
                except ValueError:
                    raise EdgeListParseError("malformed MatrixMarket size header", lineno)
                mm_rows = max(rows, cols)
                continue
        saw_data = True
        if len(tokens) < 2:
            raise EdgeListParseError(f"expected at least 2 integer tokens, got {line!r}", lineno)
        try:
            u, v = int(tokens[0]), int(tokens[1])
        except ValueError:
            raise EdgeListParseError(f"non-integer vertex id in {line!r}", lineno)
        pairs.append((u, v))
    if not saw_data:
        raise EdgeListParseError(_NO_DATA_MSG)
    return pairs, mm_rows


def _load_lines(source: Iterable[str], options: ParseOptions) -> Graph:
    global last_route
    last_route = "host"
    pairs, mm_rows = _scan_lines(source, options)
    if mm_rows is not None and options.num_vertices is None and not options.use_max_id:
        arr = np.asarray(pairs, dtype=np.int64) if pairs else np.zeros((0, 2), dtype=np.int64)
        if len(arr) and (arr.min() < 1 or arr.max() > mm_rows):
            raise EdgeListParseError(f"MatrixMarket ids outside [1, {mm_rows}]")
        g = Graph.from_edges(arr - 1, ParseOptions(), _declared_n=mm_rows)
        return Graph(0, None, orig_ids=np.arange(1, g.n + 1, dtype=np.int64), _handle=g._h)
    return Graph.from_edges(pairs, options)


# ---------------------------------------------------------------------------
# public entry points (graph.py:159-166, 223)
# ---------------------------------------------------------------------------
def load_edge_list(source: IO[str] | Iterable[str], options: ParseOptions | None = None) -> Graph:
    """Parse whitespace- or comma-separated integer pairs into a Graph
    (the reference's contract, graph.py:223-236)."""
    options = options or ParseOptions()
    if hasattr(source, "read"):
        text = source.read()
        if isinstance(text, bytes):
            text = text.decode("utf-8")
        if "\r" in text and not isinstance(source, io.StringIO):
            # a file opened with newline='' still breaks lines at lone '\r'
            return _load_lines(io.StringIO(text, newline=None), options)
        return from_text(text, options)
    return _load_lines(source, options)


def from_text(text: str, options: ParseOptions | None = None) -> Graph:
    """Graph.from_text (graph.py:164-166): lines split on '\\n' only."""
    options = options or ParseOptions()
    view = text.encode("ascii") if text.isascii() else None
    g = _parse_device(view, options, cr_newline=False) if view is not None else None
    return g if g is not None else _load_lines(io.StringIO(text), options)


def from_file(path: str | Path, options: ParseOptions | None = None) -> Graph:
    """Graph.from_file (graph.py:159-162): UTF-8 text, universal newlines."""
    options = options or ParseOptions()
    data = Path(path).read_bytes()
    g = _parse_device(data, options, cr_newline=True) if data.isascii() else None
    if g is not None:
        return g
    with open(path, "r", encoding="utf-8") as fh:
        return _load_lines(fh, options)


def to_edge_list_text(g) -> str:
    """Canonical text (graph.py:288-296): "u v" per edge in original ids,
    smaller id first, lines sorted."""
    out = np.asarray(g.orig_ids)[np.asarray(g.edges)]
    lo = np.minimum(out[:, 0], out[:, 1]) if len(out) else out.reshape(0)
    hi = np.maximum(out[:, 0], out[:, 1]) if len(out) else out.reshape(0)
    order = np.lexsort((hi, lo))
    lines = [f"{lo[i]} {hi[i]}" for i in order]
    return "\n".join(lines) + ("\n" if lines else "")
