"""Key metrics of an ncu raw-page CSV (one row per kernel).
Usage: python tools/ncu_summary.py file.raw.csv"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__thread_inst_executed_per_inst_executed.ratio"]
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print(d.get("Kernel Name", "")[:100])
    for k in KEYS:
        if k in d:
            print(f"  {k:60s} {d[k]}")
    st = [(k, d[k]) for k in hdr if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")]
    st = sorted(((float(v or 0), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")) for k, v in st), reverse=True)
    print("  stalls/issue:", ", ".join(f"{n} {v:.2f}" for v, n in st[:8]))
