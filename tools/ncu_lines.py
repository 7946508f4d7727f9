"""Aggregate an `ncu --page source --csv --print-source cuda,sass` dump by
CUDA source line: instructions executed and warp-stall samples per line.
Usage: python tools/ncu_lines.py dump.csv [top_n]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
by_inst = len(sys.argv) > 3 and sys.argv[3] == "inst"
agg = defaultdict(lambda: [0, 0, ""])
fname = "?"
hdr = None
cur_line = None
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
        cur_line = (fname, r[0], r[1][:90])
    try:
        n = float(r[ie] or 0)
        s = float(r[ws] or 0)
    except ValueError:
        continue
    if cur_line:
        a = agg[cur_line[:2]]
        a[0] += n
        a[1] += s
        a[2] = cur_line[2]
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total instr {tot_i:.3g}  samples {tot_s:.3g}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0 if by_inst else 1])[:top]:
    print(f"{100*v[1]/tot_s:5.1f}% stall {100*v[0]/tot_i:5.1f}% inst  {k[0]}:{k[1]}  {v[2].strip()}")
