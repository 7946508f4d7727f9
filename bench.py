#!/usr/bin/env python
"""Benchmark of the BRMerge SpGEMM hot path on B200 (BASELINE.json metric:
SpGEMM GFLOPS = 2*nnz(C_hat)/s, fp64 C = A*A, + achieved HBM GB/s vs peak).

One step = one full C = A*B through the C ABI (n_prod + scan + binning,
symbolic merge, row_size scan, numeric merge; all kernels), inputs resident in
HBM. L2 is flushed (256 MiB write) between timed steps, outside the events.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME]
                  [--mode precise|upper] [--impl ours|reference]

Default workload: rmat20_ef16 (BASELINE configs[3], the largest single-GPU
C = A*A config), BRMerge-Precise (C_bar would need 251 GB).

N > 1 (torchrun, NCCL): rows are partitioned across ranks by balanced n_prod
(§III.D); B is NCCL-broadcast from rank 0 at setup; each timed step ends
with the NCCL all-gather of the C row blocks' row pointers into the global
row_ptr on every rank (--assemble full: the whole C). rmat20 / AMG are the
same problem at every N (strong scaling); stencil / uniform grow with N
(weak: 64 x 64 x 64N grid, N x rows). Time = max over ranks.
`--impl reference` times the CPU oracle (test infrastructure) on a bounded
row sample, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from inputs import generators as gen  # noqa: E402

def _baseline_metric() -> str:
    """BASELINE.json's metric string, verbatim (both arms report it)."""
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as f:
            return json.load(f)["metric"]
    except Exception:
        return "SpGEMM GFLOPS (2*nnz(C_hat)/s), fp64 C=A*A, + achieved HBM GB/s vs peak"


METRIC = _baseline_metric()

CONFIGS = {
    "uniform2k_k8": 0, "stencil27_64": 1, "uniform1m_k16": 2, "rmat20_ef16": 3, "amg_lap2048_agg2x2": 4,
}
DEFAULT_CONFIG = "rmat20_ef16"  # the largest single-GPU C = A*A config (BASELINE configs[3])
# stencil / uniform grow with the rank count (weak scaling); rmat20 and the AMG
# product are the same problem at every N (strong scaling)
SCALING = {"uniform2k_k8": "weak", "stencil27_64": "weak", "uniform1m_k16": "weak",
           "rmat20_ef16": "strong", "amg_lap2048_agg2x2": "strong"}


def build_workload(name: str, world: int):
    """(A, B, description) of the global workload for `world` ranks (weak scaling)."""
    if name == "stencil27_64":
        if world == 1:
            A = gen.stencil27(64, seed=1)
        else:  # 64 x 64 x (64*world) grid
            A = stencil27_box(64, 64, 64 * world, seed=1)
        return A, A, f"27-point stencil 64x64x{64 * world}, C=A*A"
    if name == "uniform2k_k8":
        A = gen.uniform_random(2000 * world, 2000 * world, 8, seed=1)
        return A, A, f"uniform {2000 * world}^2, 8/row, C=A*A"
    if name == "uniform1m_k16":
        A = gen.uniform_random((1 << 20) * world, (1 << 20) * world, 16, seed=1)
        return A, A, f"uniform 2^20*{world}, 16/row, C=A*A"
    if name == "rmat20_ef16":
        A = gen.rmat(20, 16, 0.57, 0.19, 0.19, 0.05, seed=1)
        return A, A, "R-MAT scale 20 ef 16 (.57,.19,.19,.05), C=A*A (same graph at every N)"
    if name == "amg_lap2048_agg2x2":
        A = gen.laplace2d_5pt(2048)
        P = gen.aggregation_prolongator(2048, seed=1)
        return A, P, "5-pt Laplacian 2048^2 x 2x2 aggregation, C=A*P (same at every N)"
    raise KeyError(name)


def stencil27_box(nx, ny, nz, seed):
    """27-point stencil on an nx*ny*nz box (row id (z*ny + y)*nx + x)."""
    rng = np.random.default_rng(seed)
    N = nx * ny * nz
    idx = np.arange(N, dtype=np.int64)
    x, y, z = idx % nx, (idx // nx) % ny, idx // (nx * ny)
    cols, diag = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                ok = ((x + dx >= 0) & (x + dx < nx) & (y + dy >= 0) & (y + dy < ny)
                      & (z + dz >= 0) & (z + dz < nz))
                cols.append(np.where(ok, idx + (dz * ny + dy) * nx + dx, -1))
                diag.append(dx == 0 and dy == 0 and dz == 0)
    cm = np.stack(cols, axis=1)
    valid = cm >= 0
    vm = np.where(np.array(diag)[None, :], 26.0, -1.0) + rng.uniform(-0.01, 0.01, size=cm.shape)
    rpt = np.zeros(N + 1, np.int64)
    np.cumsum(valid.sum(axis=1), out=rpt[1:])
    return gen.Csr(N, N, rpt, cm[valid].astype(np.int32), vm[valid])


# tier table mirrored from csrc/brm_internal.cuh (checked by tests/test_bench_host.py)
TIER_CAP = [0, 8, 32, 256, 768, 3072, 6656]
TIER_LCAP = [0, 8, 32, 64, 64, 256, 512]
NUM_BINS = 8
HV_LISTS = 512  # heavy rows of at most this many lists merge in one level (csrc/heavy.cuh kHvLists)


def tier_of(nprod: np.ndarray, nl: np.ndarray) -> np.ndarray:
    t = np.full(nprod.shape, NUM_BINS - 1, np.int64)
    for b in range(NUM_BINS - 2, 0, -1):
        t = np.where((nprod <= TIER_CAP[b]) & (nl <= TIER_LCAP[b]), b, t)
    return np.where(nprod == 0, 0, t)


def algorithmic_bytes(A, B, rows: np.ndarray, nnz_c_rows: int) -> int:
    """Compulsory HBM bytes for computing C's `rows`: A rows (rpt pair + 12 B
    per nonzero), every DISTINCT B row they touch (rpt pair + 12 B per
    nonzero), C rows written (12 B per nonzero + 8 B rpt). DESIGN.md §8(d)."""
    if rows.size == 0:
        return 0
    lens = A.rpt[rows + 1] - A.rpt[rows]
    a_bytes = int(rows.size) * 16 + int(lens.sum()) * 12
    idx = np.concatenate([np.arange(A.rpt[r], A.rpt[r + 1]) for r in rows]) if rows.size < 5000 else \
        np.repeat(A.rpt[rows], lens) + (np.arange(int(lens.sum())) - np.repeat(np.cumsum(lens) - lens, lens))
    touched = gen.sorted_unique(A.col[idx])
    b_bytes = int(touched.size) * 16 + int((B.rpt[touched + 1] - B.rpt[touched]).sum()) * 12
    c_bytes = int(nnz_c_rows) * 12 + int(rows.size) * 8
    return a_bytes + b_bytes + c_bytes


class ClockSampler:
    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        for line in (getattr(self, "out", "") or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def measured_traffic(config: str, mode: str, kernel: str):
    """DRAM bytes (read + write) per launch of the dominant kernel, from the
    `ncu --set full` capture recorded in profiles/traffic.json (None if this
    config/mode/kernel was not captured)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        e = t.get(f"{config}/{mode}/{kernel.split()[0]}")
        return None if e is None else float(e["dram_bytes"])
    except Exception:
        return None


def workload_config(name, desc, mode, A, nprod, nnz_c, world=1, assemble="rpt", partition=None):
    """`config` of a bench line (both arms: the same workload gives the same dict)."""
    return {"workload": name, "desc": desc, "mode": mode, "rows": A.rows,
            "nnz_a": A.nnz, "nprod": nprod, "nnz_c": nnz_c,
            "compression_ratio": nprod / max(nnz_c, 1),
            "l2": "flushed (256 MiB write) between timed steps, outside the events",
            "parallelism": f"dp{world} rows by balanced n_prod" + (f" ({partition})" if world > 1 and partition else ""),
            "assembly": ({"rpt": "global row_ptr all-gathered, C row-distributed",
                          "full": "whole C all-gathered",
                          "peer": "whole C on every rank, row blocks stored by the merge kernels over peer "
                                  "memory, row_ptr all-gathered"}[assemble] if world > 1 else "n/a (one GPU)")}


def resolve_mode(mode, nprod, total_mem):
    """auto: BRMerge-Upper when C_bar (12 B per intermediate product) fits in half the GPU memory."""
    if mode != "auto":
        return mode
    return "upper" if nprod * 12 < total_mem // 2 else "precise"


def run_reference(args):
    """--impl reference: the CPU oracle (Eq. (2) Gustavson, single thread) on
    the same workload, rank 0 only: the whole matrix when the K + W steps
    fit in about --ref-budget-s seconds (then `config` equals the GPU arm's),
    else an evenly strided row sample per step sized to that budget."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    A, B, desc = build_workload(args.config, 1)
    nprod = oracle.row_nprod(A, B)
    total = int(nprod.sum())
    # probe: the oracle's rate on a small sample
    prow, _ = _sample_rows(nprod, target_prod=args.cpu_sample_prod)
    t0 = time.perf_counter()
    oracle.spgemm_gustavson(A, B, rows=prow)
    rate = max(float(nprod[prow].sum()), 1.0) / max(time.perf_counter() - t0, 1e-6)
    per_step = args.ref_budget_s / (args.steps + args.warmup)
    whole = total / rate <= per_step
    if whole:
        rows = None
        sample = f"whole matrix ({A.rows} rows, n_prod {total})"
        sub_np = total
    else:
        rows, sample = _sample_rows(nprod, target_prod=rate * per_step)
        sub_np = int(nprod[rows].sum())
    times = []
    C = None
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        C = oracle.spgemm_gustavson(A, B, rows=rows) if rows is not None else oracle.spgemm_gustavson(A, B)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    sec = float(np.mean(times))
    v = 2.0 * sub_np / sec / 1e9
    try:
        import torch
        mem = torch.cuda.get_device_properties(0).total_memory if torch.cuda.is_available() else 0
    except Exception:
        mem = 0
    mode = resolve_mode(args.mode, total, mem or (178 << 30))
    if whole:
        nnz_c = int(C.nnz) if hasattr(C, "nnz") else int(C.rpt[-1])
        cfg = workload_config(args.config, desc, mode, A, total, nnz_c)
    else:
        cfg = {"workload": args.config, "desc": desc, "mode": mode, "rows": A.rows, "nnz_a": A.nnz,
               "nprod": total, "rows_sampled": int(rows.size)}
    line = {"impl": "reference", "metric": METRIC,
            "value": v, "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": SCALING[args.config], "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": cfg,
            "reference": "CPU oracle: Eq. (2) Gustavson with a sorted-map accumulator (oracle/oracle.cpp), "
                         "single thread; there is no reference implementation to install (the reference is a paper)",
            "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _sample_rows(nprod, target_prod):
    """Evenly strided row sample whose n_prod sum is about target_prod."""
    M = nprod.size
    total = int(nprod.sum())
    frac = min(1.0, target_prod / max(total, 1))
    n = max(1, int(M * frac))
    rows = gen.sorted_unique(np.linspace(0, M - 1, n).astype(np.int64))
    return rows, f"{rows.size} of {M} rows (evenly strided), n_prod {int(nprod[rows].sum())} of {total}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--mode", default="auto", choices=["auto", "precise", "upper"],
                    help="auto: BRMerge-Upper when its C_bar (12 B per intermediate product) fits in "
                         "half of the GPU memory, else BRMerge-Precise")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--assemble", default="rpt", choices=["rpt", "full", "peer"],
                    help="N > 1: all-gather the global row_ptr (C's col/val stay row-distributed), "
                         "or the whole C (row_ptr + col/val) on every rank, inside the timed step; "
                         "peer: the whole C on every rank too, but written by each rank's merge kernels "
                         "straight into its peers' arrays over NVLink P2P (brm_set_mirrors), only "
                         "row_ptr all-gathered")
    ap.add_argument("--partition", default=None, choices=["contiguous", "cyclic"],
                    help="N > 1: every rank gets the same n_prod either way (PAPER.md:281); contiguous: one "
                         "row block per rank; cyclic: N * --chunks row ranges of equal n_prod, range j to "
                         "rank j mod N (spreads the rows whose products cost more than average). Default: cyclic, "
                         "contiguous under --assemble peer")
    ap.add_argument("--chunks", type=int, default=8, help="--partition cyclic: row ranges per rank")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample-prod", type=float, default=2e6, help="probe sample (products)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target oracle time of the cpu_baseline")
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="--impl reference: oracle seconds for the whole K + W run")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist
    from paper_2206_06611_b200 import Context, TorchCsr
    from paper_2206_06611_b200 import dist as bdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    A, B, desc = build_workload(args.config, world)
    ctx = Context(dev)
    if world > 1:  # B broadcast with NCCL from rank 0 (setup)
        Bd = bdist.broadcast_csr(TorchCsr.from_csr(B) if rank == 0 else None, src=0, device=dev)
    else:
        Bd = TorchCsr.from_csr(B)
    Afull = TorchCsr.from_csr(A)
    # row partition by balanced n_prod (§III.D), computed by the library's kernels
    nprod_dev = ctx.brm_row_nprod(Afull, Bd)
    off = ctx.brm_exclusive_scan_i64(nprod_dev)
    if args.partition is None:
        args.partition = "contiguous" if args.assemble == "peer" else "cyclic"
    cyclic = world > 1 and args.partition == "cyclic"
    if cyclic and args.assemble == "peer":
        raise SystemExit("--assemble peer writes contiguous row blocks: use --partition contiguous")
    bounds = ctx.brm_partition_rows(off, world * args.chunks if cyclic else world).cpu().numpy()
    # this rank's rows: one block, or every world-th range of the world * chunks ranges
    ranges = bdist.cyclic_ranges(bounds, rank, world) if cyclic else [(int(bounds[rank]), int(bounds[rank + 1]))]
    my_rows = np.concatenate([np.arange(a, b) for a, b in ranges])
    r0, r1 = ranges[0][0], ranges[-1][1]  # (contiguous: the block itself)
    nprod_h = nprod_dev.cpu().numpy()
    del Afull
    lens = np.diff(A.rpt)[my_rows]
    brpt = np.zeros(my_rows.size + 1, np.int64)
    np.cumsum(lens, out=brpt[1:])
    Ablk = gen.Csr(my_rows.size, A.cols, brpt,
                   np.concatenate([A.col[int(A.rpt[a]):int(A.rpt[b])] for a, b in ranges]),
                   np.concatenate([A.val[int(A.rpt[a]):int(A.rpt[b])] for a, b in ranges]))
    Ad = TorchCsr.from_csr(Ablk)
    local_nprod = int(nprod_h[my_rows].sum())
    args.mode = resolve_mode(args.mode, local_nprod, torch.cuda.get_device_properties(dev).total_memory)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    peer = bdist.PeerAssembly(ctx) if world > 1 and args.assemble == "peer" else None
    order = bdist.cyclic_row_order(bounds, world, dev) if cyclic else None  # rank-major -> global rows (setup)

    def step():
        if peer is not None:  # the fill writes this rank's block into every rank's whole C
            Cg = peer.spgemm(Ad, Bd, args.mode, A.rows)
            o0, o1 = int(Cg.rpt[r0]), int(Cg.rpt[r1])
            return TorchCsr(Ablk.rows, Cg.cols, Cg.rpt[r0:r1 + 1] - o0, Cg.col[o0:o1], Cg.val[o0:o1])  # this rank's block
        C = ctx.spgemm(Ad, Bd, args.mode)
        if world > 1:  # C's row blocks assembled with all-gathers (NCCL)
            if args.assemble == "full":  # row_ptr + col/val of every block on every rank
                bdist.assemble_csr_cyclic(C, bounds, order=order) if cyclic else bdist.assemble_csr(C, A.rows)
            else:  # the global row_ptr on every rank; col/val stay row-distributed
                bdist.assemble_rpt_cyclic(C, bounds, order=order) if cyclic else bdist.assemble_rpt(C, A.rows)
        return C

    C = None
    for _ in range(args.warmup):
        C = None  # release the previous C first (rmat20's C alone is ~116 GB)
        C = step()
    torch.cuda.synchronize(dev)
    ctx.set_timing(True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    bin_ms = np.zeros(NUM_BINS)
    sym_ms = num_ms = pre_ms = scan_ms = cmp_ms = hv_plan_ms = hv_merge_ms = 0.0
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            C = None
            flush.zero_()
            ev[k][0].record(stream)
            C = step()
            ev[k][1].record(stream)
            s = ctx.stats()
            bin_ms += np.array(s["ms_bin_numeric"])
            sym_ms += s["ms_symbolic"]
            num_ms += s["ms_numeric"]
            pre_ms += s["ms_nprod_scan"]
            scan_ms += s["ms_rowsize_scan"]
            cmp_ms += s["ms_compact"]
            hv_plan_ms += s["ms_hv_plan"]
            hv_merge_ms += s["ms_hv_merge"]
            launches += s["launches"]
        torch.cuda.synchronize(dev)
    ctx.set_timing(False)
    if world > 1:
        dist.barrier()
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    stats = ctx.stats()
    nnz_local = C.nnz
    tot = torch.tensor([local_nprod, nnz_local], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(tot)
    nprod_all, nnz_all = int(tot[0]), int(tot[1])
    ms_step = total_ms / args.steps
    gflops = 2.0 * nprod_all / (ms_step * 1e-3) / 1e9

    # roofline of the dominant kernel: the single numeric-merge launch with the
    # largest event time -- a shared-memory tier (k_tier / k_tiny, one launch
    # per bin) or the windowed merge of the one-level heavy rows (k_hv_merge)
    peak, peak_kind = measured_peak_hbm()
    nl_loc = np.diff(Ablk.rpt)
    np_loc = nprod_h[my_rows]
    tiers = tier_of(np_loc, nl_loc)
    cand = {}
    for b in range(1, NUM_BINS - 1):
        cand[f"{'k_tiny' if b == 1 else 'k_tier'} (tier {b} numeric merge)"] = (
            bin_ms[b] / args.steps, np.nonzero(tiers == b)[0])
    if hv_merge_ms > 0:
        cand[f"k_hv_merge (heavy rows of <= {HV_LISTS} lists, windowed merge)"] = (
            hv_merge_ms / args.steps, np.nonzero((tiers == NUM_BINS - 1) & (nl_loc <= HV_LISTS))[0])
    dom_name = max(cand, key=lambda k: cand[k][0])
    dom_ms, dom_rows = cand[dom_name]
    crpt = C.rpt.cpu().numpy()
    nnz_dom = int((crpt[dom_rows + 1] - crpt[dom_rows]).sum())
    dom_bytes = algorithmic_bytes(Ablk, B, dom_rows, nnz_dom)
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9 if dom_ms > 0 else 0.0
    all_rows = np.arange(Ablk.rows)
    step_bytes = algorithmic_bytes(Ablk, B, all_rows, nnz_local)
    b_all = torch.tensor([step_bytes], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(b_all)
    step_gbs = int(b_all.item()) / (ms_step * 1e-3) / 1e9

    # end to end through the host-buffer C entry (pinned H2D, D2H inside)
    e2e = None
    host_ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    c_bytes = nnz_local * 12 + (Ablk.rows + 1) * 8
    if not args.no_e2e and c_bytes > 0.75 * host_ram:
        e2e = {"value": None, "unit": "GFLOP/s",
               "skipped": f"C is {c_bytes / 2**30:.0f} GiB, host RAM {host_ram / 2**30:.0f} GiB"}
    elif not args.no_e2e:
        del C  # the host entry computes C again on the device: release this one first
        C = None
        torch.cuda.empty_cache()
        Ah = TorchCsr.from_csr(Ablk, pin=True)
        Bh = Ah if (B is A and world == 1) else TorchCsr.from_csr(B, pin=True)
        ctx.brmerge_spgemm_host(Ah, Bh, args.mode)  # warm
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k_e2e = max(1, min(args.steps, 5 if c_bytes < (8 << 30) else 2))  # rmat20: ~116 GB over PCIe per step
        e0.record(stream)
        for _ in range(k_e2e):
            out = ctx.brmerge_spgemm_host(Ah, Bh, args.mode)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e_ms = e0.elapsed_time(e1) / k_e2e
        te = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e_ms = float(te.item())
        h2d = sum(x.numel() * x.element_size() for X in ((Ah,) if Bh is Ah else (Ah, Bh)) for x in (X.rpt, X.col, X.val))
        d2h = (Ablk.rows + 1) * 8 + out[3].size * 4 + out[4].size * 8
        e2e = {"value": 2.0 * nprod_all / (e_ms * 1e-3) / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": e_ms}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # the oracle baseline runs at N=1 only
        try:
            import oracle
            # a probe sample sizes the timed sample to ~args.cpu_seconds of oracle work
            rows, _ = _sample_rows(np_loc, args.cpu_sample_prod)
            t0 = time.perf_counter()
            oracle.spgemm_gustavson(Ablk, B, rows=rows)
            rate = int(np_loc[rows].sum()) / max(time.perf_counter() - t0, 1e-6)
            rows, sample = _sample_rows(np_loc, rate * args.cpu_seconds)
            t0 = time.perf_counter()
            oracle.spgemm_gustavson(Ablk, B, rows=rows)
            dt = time.perf_counter() - t0
            cpu = {"value": 2.0 * int(np_loc[rows].sum()) / dt / 1e9, "unit": "GFLOP/s", "cores": 1,
                   "kind": "oracle", "sample": sample + f"; {dt:.1f} s single-threaded"}
        except Exception as e:  # report, never fake
            cpu = {"value": None, "unit": "GFLOP/s", "cores": 1, "kind": "oracle", "sample": f"failed: {e}"}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC,
            "value": gflops, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": SCALING[args.config], "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.config, desc, args.mode, A, nprod_all, nnz_all, world, args.assemble,
                                      (f"{args.chunks} cyclic row ranges per rank" if cyclic else "one row block per rank")),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": measured_traffic(args.config, args.mode, dom_name),
                         "kernel": dom_name, "kernel_ms": dom_ms, "kernel_rows": int(dom_rows.size),
                         "algorithmic_bytes": dom_bytes, "peak_kind": peak_kind},
            "hbm_step": {"achieved_gbs": step_gbs, "frac": step_gbs / peak, "algorithmic_bytes": int(b_all.item())},
            "phases_ms": {"nprod_scan_bin": pre_ms / args.steps, "symbolic": sym_ms / args.steps,
                          "numeric": num_ms / args.steps, "rowsize_scan": scan_ms / args.steps,
                          "compact": cmp_ms / args.steps, "numeric_per_bin": (bin_ms / args.steps).tolist(),
                          "heavy_plan": hv_plan_ms / args.steps, "heavy_merge_one_level": hv_merge_ms / args.steps},
            "heavy_rows": {"one_level": stats["hv_rows_one"], f"levels_of_{HV_LISTS}_list_blocks": stats["hv_rows_multi"]},
            "bin_rows": stats["bin_rows"],
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
