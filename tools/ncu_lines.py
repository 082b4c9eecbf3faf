"""Aggregate an ncu source page (cuda,sass CSV) per CUDA source line.

    ncu -i rep --page source --csv --print-source cuda,sass > x.csv
    python tools/ncu_lines.py x.csv [top]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
ie_i = hdr.index("Instructions Executed")
s_i = hdr.index("Warp Stall Sampling (All Samples)")
agg = defaultdict(lambda: [0.0, 0.0, ""])
cur = None
for r in rows[hdr_i + 1:]:
    if len(r) <= ie_i:
        continue
    if r[0] not in ("", "-"):
        if not r[0].isdigit():
            continue
        cur = (int(r[0]), r[1])
    if r[2] in ("", "-") or cur is None:
        continue
    try:
        agg[cur[0]][0] += float(r[ie_i] or 0)
        agg[cur[0]][1] += float(r[s_i] or 0)
    except ValueError:
        continue
    agg[cur[0]][2] = cur[1]
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp-inst {ti:.0f}  stall samples {ts:.0f}")
for ln, (ie, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{100*ie/ti:5.1f}% inst {100*s/ts:5.1f}% samples  L{ln}: {src.strip()[:90]}")

if len(sys.argv) > 3:
    # range summary: "name:lo-hi,name:lo-hi"
    print("--- ranges")
    for part in sys.argv[3].split(","):
        name, rng_ = part.split(":")
        lo, hi = (int(x) for x in rng_.split("-"))
        ie = sum(v[0] for k, v in agg.items() if lo <= k <= hi)
        s = sum(v[1] for k, v in agg.items() if lo <= k <= hi)
        print(f"{name:12s} {100*ie/ti:5.1f}% inst {100*s/ts:5.1f}% samples")
