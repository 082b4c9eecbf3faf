"""Stall reasons and instruction counts per kernel phase (device function)
from an ncu source page (cuda,sass CSV of a -lineinfo build).

    ncu -i rep --page source --csv --print-source cuda,sass > x.csv
    python tools/ncu_phases.py x.csv [path/to/tilecast_b200.cu at the profiled revision]

Each SASS row is attributed to the CUDA source line above it; each line to
the device function whose definition encloses it in the .cu file.
"""
import csv
import re
import sys
from collections import defaultdict

src_csv = sys.argv[1]
cu = sys.argv[2] if len(sys.argv) > 2 else "paper_2605_19926_b200/csrc/tilecast_b200.cu"

# line -> enclosing device function (top-level definitions only)
func_at = {}
cur = "?"
pat = re.compile(r"^(?:__device__|__global__|__host__ __device__)[^(]*?(\w+)\s*\(")
for no, line in enumerate(open(cu), 1):
    m = pat.match(line)
    if m:
        cur = m.group(1)
    func_at[no] = cur

rows = list(csv.reader(open(src_csv)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
ie = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg = defaultdict(lambda: defaultdict(float))
cur_line = None
for r in rows[hi + 1:]:
    if len(r) <= ie:
        continue
    if r[0] not in ("", "-"):
        cur_line = int(r[0]) if r[0].isdigit() else None
        continue
    if cur_line is None:
        continue
    fn = func_at.get(cur_line, "?")
    a = agg[fn]
    try:
        a["inst"] += float(r[ie] or 0)
        for i in stall_cols:
            v = float(r[i] or 0)
            a[hdr[i]] += v
            a["samples"] += v
    except ValueError:
        pass

tot_i = sum(a["inst"] for a in agg.values())
tot_s = sum(a["samples"] for a in agg.values())
print(f"total warp-inst {tot_i:.0f}, stall samples {tot_s:.0f}")
for fn, a in sorted(agg.items(), key=lambda kv: -kv[1]["samples"]):
    if a["samples"] < 0.005 * tot_s and a["inst"] < 0.005 * tot_i:
        continue
    top = sorted(((k, v) for k, v in a.items() if k.startswith("stall_")), key=lambda kv: -kv[1])[:5]
    tops = ", ".join(f"{k[6:]} {100 * v / max(a['samples'], 1):.0f}%" for k, v in top if v)
    print(f"{fn:28s} inst {100 * a['inst'] / tot_i:5.1f}%  samples {100 * a['samples'] / tot_s:5.1f}%"
          f"  [{tops}]")
