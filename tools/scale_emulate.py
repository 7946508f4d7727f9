"""Per-rank compute of the multi-GPU row partition, measured on ONE B200.

For N in --ns: the rows of A are split by balanced n_prod (brm_partition_rows,
§III.D), and each rank's row block runs through the C ABI alone on this GPU
(structure + fill, CUDA events, L2 flushed before each run). The N-GPU step
cannot be faster than its slowest block, so T_1 / (N * max_r T_r) bounds the
strong-scaling efficiency from above (NCCL's row_ptr all-gather and any
interference are not included). Ranks run one after another: no rank waits on
another. Prints one JSON line.
Usage: python tools/scale_emulate.py [--config rmat20_ef16] [--ns 1,2,4,8] [--reps 3]"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from inputs import generators as gen  # noqa: E402
from paper_2206_06611_b200 import Context, TorchCsr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="rmat20_ef16")
ap.add_argument("--mode", default="auto")
ap.add_argument("--ns", default="1,2,4,8")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--balance", default="nprod", choices=["nprod", "work", "cyclic"],
                help="work: weight n_prod * (1 + ceil(log2 nl)) per row, partitioned on the host by R7's rule; "
                     "cyclic: N * --chunks row ranges of equal n_prod (brm_partition_rows), range j to rank j mod N")
ap.add_argument("--chunks", type=int, default=8, help="cyclic: row ranges per rank")
args = ap.parse_args()

dev = torch.device("cuda", 0)
A, B, desc = bench.build_workload(args.config, 1)
ctx = Context(dev)
Bd = TorchCsr.from_csr(B)
Afull = TorchCsr.from_csr(A)
nprod = ctx.brm_row_nprod(Afull, Bd)
off = ctx.brm_exclusive_scan_i64(nprod)
nprod_h = nprod.cpu().numpy()
del Afull
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
mode = bench.resolve_mode(args.mode, int(nprod_h.sum()), torch.cuda.get_device_properties(dev).total_memory)


def rows_csr(ranges):
    """The rows of the given [r0, r1) ranges of A, concatenated, as a CSR."""
    lens = np.concatenate([np.diff(A.rpt[r0:r1 + 1]) for r0, r1 in ranges]) if ranges else np.zeros(0, np.int64)
    rpt = np.zeros(lens.size + 1, np.int64)
    np.cumsum(lens, out=rpt[1:])
    col = np.concatenate([A.col[int(A.rpt[r0]):int(A.rpt[r1])] for r0, r1 in ranges])
    val = np.concatenate([A.val[int(A.rpt[r0]):int(A.rpt[r1])] for r0, r1 in ranges])
    return gen.Csr(lens.size, A.cols, rpt, col, val)


def block_ms(r0, r1=None):
    Ab = rows_csr([(r0, r1)] if r1 is not None else r0)
    Ad = TorchCsr.from_csr(Ab)
    # a rank of the real run owns a whole GPU: give the cached blocks of the
    # previous (larger) C back first -- the heavy rows' level batches are sized
    # by the free memory
    torch.cuda.empty_cache()
    C = ctx.spgemm(Ad, Bd, mode)  # warm-up (its C blocks stay cached for the timed runs)
    del C
    ts = []
    for _ in range(args.reps):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        C = ctx.spgemm(Ad, Bd, mode)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        del C
    return float(np.mean(ts))


out = {"config": args.config, "mode": mode, "per_n": {}}
t1 = None
nl_h = np.diff(A.rpt)
work_h = nprod_h * (1 + np.ceil(np.log2(np.maximum(nl_h, 1))).astype(np.int64))
work_off = np.concatenate([[0], np.cumsum(work_h)])


def host_bounds(n):
    """R7: bounds[g] = first row r with prefix(r) * n >= g * total"""
    tot = work_off[-1]
    return np.array([0] + [int(np.searchsorted(work_off, (g * tot + n - 1) // n, side="left")) for g in range(1, n)]
                    + [A.rows])


out["balance"] = args.balance
for n in [int(x) for x in args.ns.split(",")]:
    if args.balance == "cyclic" and n > 1:
        cb = ctx.brm_partition_rows(off, n * args.chunks).cpu().numpy()
        parts = [[(int(cb[j]), int(cb[j + 1])) for j in range(r, n * args.chunks, n)] for r in range(n)]
        ms = [block_ms(p) for p in parts]
        share = [float(sum(nprod_h[a:b].sum() for a, b in p) / nprod_h.sum()) for p in parts]
        bounds = None
    else:
        bounds = ctx.brm_partition_rows(off, n).cpu().numpy() if args.balance != "work" else host_bounds(n)
        ms = [block_ms(int(bounds[r]), int(bounds[r + 1])) for r in range(n)]
        share = [float(nprod_h[bounds[r]:bounds[r + 1]].sum() / nprod_h.sum()) for r in range(n)]
    if n == 1:
        t1 = ms[0]
    eff = t1 / (n * max(ms)) if t1 else None
    out["per_n"][n] = {"block_ms": ms, "nprod_share": share, "max_ms": max(ms), "bound_efficiency": eff,
                       "rows": ([int(bounds[r + 1] - bounds[r]) for r in range(n)] if bounds is not None
                                else [sum(b - a for a, b in p) for p in parts])}
    print(f"N={n}: max {max(ms):.1f} ms, blocks {[round(x, 1) for x in ms]}, bound efficiency {eff}",
          file=sys.stderr, flush=True)
print(json.dumps(out))
