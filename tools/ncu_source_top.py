"""Top CUDA source lines by warp-stall samples (with their instruction
share) of every kernel in an `ncu --import-source on` report, as JSON.
Usage: python tools/ncu_source_top.py report.ncu-rep [top] > out.json"""
import csv, io, json, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


per = defaultdict(dict)  # function -> (file:line) -> [stall, inst, source]
fn, path, hdr = None, None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] and len(r) >= len(hdr):
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        iI = hdr.index("Instructions Executed")
        key = f"{path}:{r[0]}"
        d = per[fn].setdefault(key, [0.0, 0.0, r[1].strip()[:90]])
        d[0] += num(r[iS])
        d[1] += num(r[iI])
res = {}
for fn, lines in per.items():
    ts = sum(v[0] for v in lines.values()) or 1.0
    ti = sum(v[1] for v in lines.values()) or 1.0
    name = fn.replace("gd::<unnamed>::", "").split("(")[0][:90]
    while name in res:
        name += "'"
    res[name] = [{"line": k, "source": v[2], "stall_share": round(v[0] / ts, 4),
                  "inst_share": round(v[1] / ti, 4)}
                 for k, v in sorted(lines.items(), key=lambda kv: -kv[1][0])[:top]]
print(json.dumps(res, indent=1))
