"""Shared-memory wavefronts (total / excessive = bank-conflict replays) and
stall samples per CUDA source line from an ncu source dump
(--page source --csv --print-source cuda,sass).
Usage: python tools/ncu_smem_lines.py dump.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = defaultdict(lambda: [0.0, 0.0, 0.0])
fname, hdr, cur = "?", None, None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iw = hdr.index("L1 Wavefronts Shared")
        ix = hdr.index("L1 Wavefronts Shared Excessive")
        iss = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr) - 5:
        continue
    if r[0]:
        cur = (fname, r[0], r[1][:80])
        continue
    f = lambda i: float(r[i] or 0) if r[i] not in ("-", "") else 0.0
    a = agg[cur]
    a[0] += f(iw)
    a[1] += f(ix)
    a[2] += f(iss)
tw = sum(v[0] for v in agg.values())
tx = sum(v[1] for v in agg.values())
ts = sum(v[2] for v in agg.values())
print(f"shared wavefronts {tw:.4g}, excessive {tx:.4g} ({100 * tx / max(tw, 1):.1f} %), stall samples {ts:.4g}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{v[0]:11.4g} wf {v[1]:11.4g} excess {100 * v[2] / max(ts, 1):5.1f}% stall  {k[0]}:{k[1]} {k[2]}")
