"""Print one line per bench JSON: value, ms/step, roofline and phase times.
Usage: python tools/bench_summary.py gpurun_out/<tag>/bench_*.json"""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:  # empty / failed run
        print(f, "FAILED", e)
        continue
    ph = d.get("phases_ms", {})
    r = d.get("roofline", {})
    print(f"{f.split('/')[-1]:42s} {d['value']:8.1f} {d['unit']} {d['ms_per_step']:8.3f} ms  roof {r.get('frac', 0):.3f} "
          f"({r.get('kernel', '')}, {r.get('kernel_ms', 0):.3f} ms)  "
          + " ".join(f"{k}={v:.3f}" for k, v in ph.items() if isinstance(v, float)))
