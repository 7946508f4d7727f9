"""Markdown table of bench.py lines (profiles/<session>/bench_*.json)."""
import glob
import json
import sys

rows = []
for f in sorted(glob.glob(sys.argv[1] + "/bench_*.json")):
    try:
        d = json.load(open(f))
    except Exception:
        continue
    r = d["roofline"]
    e = d.get("e2e") or {}
    rows.append((d["config"]["workload"], d["config"]["mode"], d["value"], d["ms_per_step"], r["kernel"].split(" (")[0],
                 r["kernel_ms"], r["frac"], e.get("value")))
print("| config | mode | GFLOP/s | ms / step | dominant kernel | its ms | roofline frac (HBM) | e2e GFLOP/s |")
print("|---|---|---|---|---|---|---|---|")
for w, m, v, ms, k, kms, fr, e in rows:
    print(f"| {w} | {m} | {v:.1f} | {ms:.3f} | {k} | {kms:.3f} | {fr:.3f} | {'' if e is None else f'{e:.1f}'} |")
