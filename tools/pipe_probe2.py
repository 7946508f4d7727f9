"""Host entry per call (ms) for a workload with the row-blocked pipeline forced on / off.
Usage: python tools/pipe_probe2.py cfg mode"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2206_06611_b200 import Context, TorchCsr
cfg, mode = sys.argv[1], sys.argv[2]
A, B, _ = bench.build_workload(cfg, 1)
ctx = Context(torch.device("cuda", 0))
Ah = TorchCsr.from_csr(A, pin=True)
Bh = Ah if B is A else TorchCsr.from_csr(B, pin=True)
for pipe in (1 << 62, 0):
    ctx.brm_set_host_pipeline(pipe)
    ctx.brmerge_spgemm_host(Ah, Bh, mode)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        ctx.brmerge_spgemm_host(Ah, Bh, mode)
        ts.append((time.perf_counter() - t0) * 1e3)
    print(cfg, mode, "pipelined" if pipe == 0 else "one-shot", " ".join(f"{t:.2f}" for t in ts), flush=True)
