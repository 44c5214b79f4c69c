"""Summarise an ncu --metrics CSV launch list: per-kernel time share and DRAM
bytes of ONE census (the profiled script runs the census twice; the second
half of the launches is used)."""
import collections, csv, json, sys

def load(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[h], rows[h + 1:]
    ki, ii, mi, ui, vi = (hdr.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Unit", "Metric Value"))
    launches = collections.OrderedDict()
    for r in data:
        if len(r) <= vi:
            continue
        key = int(r[ii])
        d = launches.setdefault(key, {"kernel": r[ki]})
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        scale = {"ns": 1e-6, "usecond": 1e-3, "msecond": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                 "Gbyte": 1e9, "%": 1}.get(unit, 1)
        d[r[mi]] = v * scale
    return list(launches.values())

def summarise(path):
    ls = load(path)
    # the census is run twice: take the launches of the second census
    names = [l["kernel"] for l in ls]
    first_fin = [i for i, n in enumerate(names) if "finalize" in n]
    start = first_fin[0] + 1 if len(first_fin) >= 2 else 0
    # skip graph-build launches before the first census (second census starts after first finalize)
    ls = ls[start:]
    agg = collections.OrderedDict()
    for l in ls:
        short = l["kernel"].split("(")[0].replace("gd::<unnamed>::", "").replace("void ", "")
        a = agg.setdefault(short, {"ms": 0.0, "dram_bytes": 0.0, "launches": 0})
        a["ms"] += l.get("gpu__time_duration.sum", 0.0)
        a["dram_bytes"] += l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
        a["launches"] += 1
    tot_ms = sum(a["ms"] for a in agg.values())
    tot_b = sum(a["dram_bytes"] for a in agg.values())
    return {"census_kernel_ms": tot_ms, "census_dram_bytes": tot_b,
            "kernels": {k: {"ms": round(v["ms"], 3), "share": round(v["ms"] / tot_ms, 4),
                            "dram_bytes": v["dram_bytes"], "launches": v["launches"]}
                        for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["ms"])}}

if __name__ == "__main__":
    out = {}
    for spec in sys.argv[1:]:
        key, path = spec.split("=")
        out[key] = summarise(path)
    print(json.dumps(out, indent=1))
