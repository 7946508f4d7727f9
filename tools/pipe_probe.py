"""Time the host-buffer entry on a workload: full, and with BRM_PIPE_NOCOPY
set by the caller (blocks computed, no copies). Usage: python tools/pipe_probe.py cfg mode"""
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
ctx.brmerge_spgemm_host(Ah, Bh, mode)
for _ in range(3):
    t0 = time.perf_counter()
    ctx.brmerge_spgemm_host(Ah, Bh, mode)
    print(cfg, mode, "nocopy" if os.environ.get("BRM_PIPE_NOCOPY") else "full", f"{(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
