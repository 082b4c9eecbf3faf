"""Record DRAM traffic per step launch from an ncu capture of consecutive
launches (tools/ncu_c2.sh step 2) into profiles/ncu_traffic.json, keyed by
bench config and stamped with the kernel source hash, so bench.py reports
`roofline.traffic` only for the build that was measured.

    python tools/ncu_traffic.py gpurun_out/r02_dram8_c2.csv c2 <envs> <capture-name>
"""
import csv
import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
path, cfg, envs, name = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = {}
for r in rows[1:]:
    per.setdefault(r[ii], {"kernel": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
launches = [v for v in per.values() if "dram__bytes_write.sum" in v]
# steady state: skip the first launch (its predecessor's frames may not be in L2 yet)
steady = launches[1:] if len(launches) > 2 else launches
rd = sum(v["dram__bytes_read.sum"] for v in steady) / len(steady)
wr = sum(v["dram__bytes_write.sum"] for v in steady) / len(steady)
dur = sum(v["gpu__time_duration.sum"] for v in steady) / len(steady)
src = ROOT / "paper_2605_19926_b200" / "csrc" / "tilecast_b200.cu"
out = ROOT / "profiles" / "ncu_traffic.json"
db = json.loads(out.read_text()) if out.exists() else {}
db = {k: v for k, v in db.items() if isinstance(v, dict) and not k.startswith("_")}
db[cfg] = {"dram_bytes_per_launch": rd + wr, "dram_read_per_launch": rd,
           "dram_write_per_launch": wr, "ncu_duration_ns_mean": dur, "launches": len(steady),
           "kernel": steady[0]["kernel"][:60], "envs": envs,
           "source_sha16": hashlib.sha256(src.read_bytes()).hexdigest()[:16],
           "capture": f"{name}: ncu --cache-control none, {len(steady)} consecutive ring-rotated "
                      f"step launches after warm-up"}
out.write_text(json.dumps(db, indent=1) + "\n")
print(json.dumps(db[cfg], indent=1))
