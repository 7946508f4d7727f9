"""Per-CUDA-line warp-instruction counts from an ncu source dump
(--page source --csv --print-source cuda,sass), SASS rows only, scaled by a
divisor (e.g. rows processed). Usage: python tools/ncu_sass_lines.py dump.csv divisor [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
agg = defaultdict(float)
stall = defaultdict(float)
fname, hdr, cur, tot, tots = "?", None, None, 0.0, 0.0
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        ws = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr) - 5:
        continue
    if r[0]:
        cur = (fname, r[0], r[1][:90])
        continue
    try:
        n = float(r[ie] or 0)
        s = float(r[ws] or 0)
    except ValueError:
        continue
    agg[cur] += n
    stall[cur] += s
    tot += n
    tots += s
print(f"total warp instr {tot:.4g} ({tot/div:.1f} per unit), stall samples {tots:.4g}")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{v/div:8.1f}/unit {100*v/tot:5.1f}% inst {100*stall[k]/max(tots,1):5.1f}% stall  {k[0]}:{k[1]} {k[2].strip()}")
