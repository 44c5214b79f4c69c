"""TEST INFRASTRUCTURE ONLY: restatement of the reference's per-edge role
derivation and CSV writer, the checker for the device micro_roles /
micro_csv (gd_derive.cu).

  derive_roles  <- _derive_micro (census.py:574-596)
  micro_csv     <- micro_csv + serialize.write_csv (census.py:603-623,
                   serialize.py:39-44)

Pinned against the reference through tests/golden/micro_roles.json
(make_golden.py --roles).
"""

from __future__ import annotations

import csv
import io
from math import comb

import numpy as np

HEADER = [
    "src", "dst", "tri", "star_u", "star_v", "clique4", "cycle4",
    "chordal_chord", "cycle_mid_path", "chordal_cycle_edge", "tailed_tail",
    "star3", "tailed_detached", "tri_isolated", "path_end", "star_isolated",
    "pair_edge", "lone_edge", "indep3",
]
ROLES = ("tt1", "tt0", "susv1", "susv0", "ts1", "ts0", "ss1", "ss0", "ti1", "ti0",
         "si1", "si0", "ii1", "ii0", "indep3")
CHECK = ("tt0", "susv0", "ts0", "ss0", "ti0", "ti1", "si0", "si1", "ii0", "ii1")


class NegativeRole(Exception):
    def __init__(self, name, index):
        super().__init__(name, index)
        self.name, self.index = name, index


def derive_roles(n: int, m: int, raw, index: int = 0) -> dict:
    t, su, sv, cl, cy, uu1, vv1, ts1, ti1, si1 = (int(x) for x in raw)
    i3 = n - 2 - t - su - sv
    ss1 = uu1 + vv1
    outside = m + 1 - (t + su + 1) - (t + sv + 1)
    ii1 = outside - (cl + ts1 + ti1) - (ss1 + cy + si1)
    r = {"tri": t, "star_u": su, "star_v": sv, "indep3": i3,
         "tt1": cl, "tt0": comb(t, 2) - cl, "susv1": cy, "susv0": su * sv - cy,
         "ts1": ts1, "ts0": t * (su + sv) - ts1, "ss1": ss1,
         "ss0": comb(su, 2) + comb(sv, 2) - ss1, "ti1": ti1, "ti0": t * i3 - ti1,
         "si1": si1, "si0": (su + sv) * i3 - si1, "ii1": ii1, "ii0": comb(i3, 2) - ii1}
    for name in CHECK:
        if r[name] < 0:
            raise NegativeRole(name, index)
    return r


def roles_table(n: int, m: int, table) -> np.ndarray:
    tab = np.asarray(table)
    return np.asarray([[derive_roles(n, m, tab[i], i)[k] for k in ROLES] for i in range(len(tab))],
                      dtype=np.int64).reshape(-1, len(ROLES))


def micro_csv(n: int, edges, orig_ids, table, m: int | None = None) -> str:
    """`m` defaults to the number of rows (pass the graph's m for a subset)."""
    orig = np.asarray(orig_ids)[np.asarray(edges, dtype=np.int64)]
    tab = np.asarray(table)
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(HEADER)
    for i in range(len(tab)):
        r = derive_roles(n, len(tab) if m is None else m, tab[i], i)
        w.writerow([int(orig[i, 0]), int(orig[i, 1]), r["tri"], r["star_u"], r["star_v"],
                    r["tt1"], r["susv1"], r["tt0"], r["susv0"], r["ts1"], r["ss1"], r["ss0"],
                    r["ti1"], r["ti0"], r["si1"], r["si0"], r["ii1"], r["ii0"], r["indep3"]])
    return buf.getvalue()
