"""Work statistics of the triangle frames of a config, numpy only (no GPU):
frames, items (probes) and the row-bitmap bytes per out-degree bin.

python tools/frame_stats.py c5_chung_lu_4m
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import oracle as O  # noqa: E402
from paper_1506_04322_b200 import workloads as W  # noqa: E402

cfg = sys.argv[1]
raw = W.config_graph(cfg)
edges = O.canonical_edges(raw.pairs)
n, m = raw.n, len(edges)
deg = np.bincount(edges.ravel(), minlength=n)
order = np.lexsort((np.arange(n), deg))  # ascending (degree, id)
rank = np.empty(n, np.int64)
rank[order] = np.arange(n)
ru, rv = rank[edges[:, 0]], rank[edges[:, 1]]
lo, hi = np.minimum(ru, rv), np.maximum(ru, rv)
dplus = np.bincount(lo, minlength=n)       # out-degree in rank space
items = np.bincount(lo, weights=dplus[hi].astype(np.float64), minlength=n)
print(f"{cfg}: n={n} m={m} max deg {deg.max()} max d+ {dplus.max()} items {items.sum():.4g}")
bins = [2, 33, 65, 129, 257, 513, 1025, 2049, 4097, 8193, 16385, 1 << 30]
for a, b in zip(bins[:-1], bins[1:]):
    sel = (dplus >= a) & (dplus < b)
    D = dplus[sel].astype(np.float64)
    print(f"  D in [{a:6d},{b - 1:10d}]: frames {sel.sum():9d}  items {items[sel].sum():.4g}"
          f"  bitmap bytes sum {np.sum(D * np.ceil(D / 64) * 8):.4g}  max {np.max(D * np.ceil(D / 64) * 8, initial=0):.4g}")
# pass C: wedges of frame s = sum over lower neighbours w of #{x in N(w): x < s}
rows = np.concatenate([lo, hi])
cols = np.concatenate([hi, lo])
o2 = np.lexsort((cols, rows))
rows, cols = rows[o2], cols[o2]
rp = np.zeros(n + 1, np.int64)
np.cumsum(np.bincount(rows, minlength=n), out=rp[1:])
pos = np.arange(2 * m) - rp[rows]
up = cols > rows
Wd = np.bincount(cols[up], weights=pos[up].astype(np.float64), minlength=n)
dminus = np.bincount(hi, minlength=n)
print(f"  wedges {Wd.sum():.4g}")
wb = [1, 257, 1025, 4097, 12289, 24577, 1 << 20, 1 << 24, 1 << 62]
for a, b in zip(wb[:-1], wb[1:]):
    sel = (Wd >= a) & (Wd < b)
    print(f"  W in [{a:9d},{b - 1:20d}]: frames {sel.sum():9d}  wedges {Wd[sel].sum():.4g}"
          f"  lower slots {dminus[sel].sum():.4g}  mean d- {dminus[sel].mean() if sel.any() else 0:.1f}")
