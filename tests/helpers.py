"""Shared loaders for the golden fixtures (tests/golden, made by make_golden.py)."""

from __future__ import annotations

import hashlib
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@lru_cache(maxsize=None)
def small_graphs():
    out = []
    for c in json.loads((GOLDEN / "small_graphs.json").read_text()):
        edges = np.asarray(c["edges"], dtype=np.int64).reshape(-1, 2)
        micro = np.asarray(c["micro"], dtype=np.int64).reshape(-1, 10)
        counts = {k: int(v) for k, v in c["counts"].items()}
        out.append((c["name"], int(c["n"]), edges, counts, micro))
    return out


@lru_cache(maxsize=None)
def configs():
    return json.loads((GOLDEN / "configs.json").read_text())


@lru_cache(maxsize=None)
def graph_build():
    return json.loads((GOLDEN / "graph_build.json").read_text())


def int_counts(d):
    return {k: int(v) for k, v in d.items()}
