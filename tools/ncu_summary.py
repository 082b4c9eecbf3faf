"""Summarise an ncu --set full report into profiles/<name>.json/.md.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep profiles/r01_c2_step [algo_bytes]
"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
algo = float(sys.argv[3]) if len(sys.argv) > 3 else None
# a report, or the `--page raw --csv` export of one (taken on the GPU box)
raw = open(rep).read() if rep.endswith(".csv") else \
    subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                   text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "ms": 1e6,
         "msecond": 1e6, "second": 1e9, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}


def f(k):
    """Value in base units (bytes, ns, Hz) using the report's unit row."""
    try:
        v = float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return None
    return v * SCALE.get(u.get(k, ""), 1)


keys = {
    "kernel": "Kernel Name",
    "duration_ns": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "ipc_active": "sm__inst_executed.avg.per_cycle_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_dyn": "launch__shared_mem_per_block_dynamic",
    "inst_executed": "smsp__inst_executed.sum",
    "thread_inst_per_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "branch_eff_pct": "smsp__sass_average_branch_targets_threads_uniform.pct",
    "smem_bank_conflicts_st": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "smem_bank_conflicts_ld": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smem_wavefronts_st": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "smem_wavefronts_ld": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "fp64_pipe_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm_clock_hz": "smsp__cycles_elapsed.avg.per_second",
    "icache_hit_pct": "sm__icc_request_hit_rate.pct",
    "local_ld_inst": "smsp__sass_inst_executed_op_local_ld.sum",
    "local_st_inst": "smsp__sass_inst_executed_op_local_st.sum",
}
res = {k: (d.get(v) if k == "kernel" else f(v)) for k, v in keys.items()}
stalls = {}
for k in hdr:
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        v = f(k)
        if v:
            stalls[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = v
tot = sum(stalls.values()) or 1.0
res["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in
                    sorted(stalls.items(), key=lambda kv: -kv[1])[:10]}
if res["dram_read_bytes"] is not None:
    res["traffic_bytes"] = res["dram_read_bytes"] + res["dram_write_bytes"]
if algo:
    res["algorithmic_bytes"] = algo
    if res["duration_ns"]:
        res["achieved_gbs_ncu_replay"] = algo / res["duration_ns"]
json.dump(res, open(out + ".json", "w"), indent=1)
with open(out + ".md", "w") as fh:
    fh.write(f"# ncu summary: {out.split('/')[-1]}\n\nreport: `{rep}`\n\n| metric | value |\n|---|---|\n")
    for k, v in res.items():
        if k != "stall_pct":
            fh.write(f"| {k} | {v} |\n")
    fh.write("\nTop warp stall reasons (% of samples): "
             + ", ".join(f"{k} {v}%" for k, v in res["stall_pct"].items()) + "\n")
print(json.dumps(res, indent=1))
