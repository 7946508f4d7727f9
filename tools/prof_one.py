"""One C = A*B of a named workload through the C ABI (for ncu captures)."""
import argparse
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs import workload
from paper_2206_06611_b200 import Context, TorchCsr

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="rmat20_ef16")
ap.add_argument("--mode", default="precise")
ap.add_argument("--reps", type=int, default=1)
args = ap.parse_args()
A, B = workload(args.config)
ctx = Context()
Ad, Bd = TorchCsr.from_csr(A), TorchCsr.from_csr(B)
for _ in range(args.reps):
    C = None
    C = ctx.spgemm(Ad, Bd, args.mode)
    torch.cuda.synchronize()
print("nnz", C.nnz)
