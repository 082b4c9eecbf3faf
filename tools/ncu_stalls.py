"""Per-source-range stall breakdown from an ncu cuda,sass source CSV.

    python tools/ncu_stalls.py x.csv "name:lo-hi,..."
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
ie_i = hdr.index("Instructions Executed")
per_line = defaultdict(lambda: defaultdict(float))
cur = None
for r in rows[hdr_i + 1:]:
    if len(r) <= max(cols):
        continue
    if r[0] not in ("", "-"):
        if not r[0].isdigit():
            continue
        cur = int(r[0])
    if r[2] in ("", "-") or cur is None:
        continue
    for c in cols + [ie_i]:
        try:
            per_line[cur][hdr[c]] += float(r[c] or 0)
        except ValueError:
            pass
ranges = [p.split(":") for p in sys.argv[2].split(",")]
tot = defaultdict(float)
for d in per_line.values():
    for k, v in d.items():
        tot[k] += v
allsamp = sum(v for k, v in tot.items() if k.startswith("stall_"))
names = [hdr[c] for c in cols]
print(f"{'range':14s} {'inst%':>6s} {'samp%':>6s}  top stalls")
for name, rg in ranges:
    lo, hi = (int(x) for x in rg.split("-"))
    acc = defaultdict(float)
    for ln, d in per_line.items():
        if lo <= ln <= hi:
            for k, v in d.items():
                acc[k] += v
    s = sum(acc[k] for k in names)
    top = sorted(((acc[k], k) for k in names), reverse=True)[:4]
    print(f"{name:14s} {100*acc['Instructions Executed']/tot['Instructions Executed']:6.1f} "
          f"{100*s/allsamp:6.1f}  " + ", ".join(f"{k[6:]}={100*v/max(s,1):.0f}%" for v, k in top))
