"""Experiment helper: time the numeric merge on one workload under the round
strategies (env BRM_STRATEGY) and print the device cycle counters
(env BRM_PROFILE=1). Usage: python tools/strategy_probe.py [workload] [mode]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(workload, mode):
    sys.path.insert(0, ROOT)
    import torch
    from bench import build_workload
    from paper_2206_06611_b200 import Context, TorchCsr
    A, B, _ = build_workload(workload, 1)
    ctx = Context()
    Ad, Bd = TorchCsr.from_csr(A), TorchCsr.from_csr(B)
    for _ in range(2):
        ctx.spgemm(Ad, Bd, mode)
    ctx.set_timing(True)
    ms = []
    for _ in range(3):
        ctx.spgemm(Ad, Bd, mode)
        s = ctx.stats()
        ms.append(s["ms_numeric"] + s["ms_symbolic"])
    torch.cuda.synchronize()
    s = ctx.stats()
    prof = s["prof"]
    rows = max(prof[6], 1)
    print(json.dumps({"strategy": os.environ.get("BRM_STRATEGY", "0"), "merge_ms": min(ms),
                      "bins": s["bin_rows"], "cycles_per_row": {"stage": prof[0] / rows, "seq": prof[1] / rows,
                      "chunked": prof[2] / rows, "store": prof[3] / rows},
                      "rounds_per_row": {"seq": prof[4] / rows, "chunked": prof[5] / rows}}))


if __name__ == "__main__":
    wl = sys.argv[1] if len(sys.argv) > 1 else "stencil27_64"
    mode = sys.argv[2] if len(sys.argv) > 2 else "upper"
    if os.environ.get("BRM_PROBE_CHILD"):
        child(wl, mode)
    else:
        for strat in ("0", "1", "2"):
            for prof in ("0", "1"):
                env = dict(os.environ, BRM_STRATEGY=strat, BRM_PROFILE=prof, BRM_PROBE_CHILD="1")
                out = subprocess.run([sys.executable, __file__, wl, mode], env=env, capture_output=True, text=True)
                print(f"strategy={strat} profile={prof}:", out.stdout.strip()[-600:], out.stderr.strip()[-300:])
