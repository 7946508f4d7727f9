"""Multi-GPU plumbing of the BRMerge SpGEMM.

Output rows of Eq. (2) are independent, so the path shards by
rows: rank g computes the row block [bounds[g], bounds[g+1]) where the bounds
balance n_prod across ranks (§III.D; reading R7, computed on the
device by brm_partition_rows). B is broadcast from one rank, each rank runs
the whole path on its block through the C ABI, and C's row_ptr offsets (and
optionally the C row blocks themselves) are assembled with all-gathers -- or,
with PeerAssembly, the row blocks are written into every rank's copy of C by
the merge kernels themselves over peer memory (brm_set_mirrors), and only the
row pointers are all-gathered.

This module only moves and re-indexes tensors with torch.distributed (NCCL on
GPUs, gloo in the CPU tests); no step of the SpGEMM itself runs here.
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist

from .binding import TorchCsr


def broadcast_csr(X: Optional[TorchCsr], src: int = 0, device=None, group=None) -> TorchCsr:
    """Broadcast a CSR from rank `src` (X given there, None elsewhere).
    Shape (rows, cols, nnz) travels first as one int64 triple."""
    rank = dist.get_rank(group)
    dev = torch.device(device) if device is not None else (X.device if X is not None else torch.device("cpu"))
    hdr = torch.zeros(3, dtype=torch.int64, device=dev)
    if rank == src:
        hdr[0], hdr[1], hdr[2] = X.rows, X.cols, X.nnz
    dist.broadcast(hdr, src, group=group)
    rows, cols, nnz = (int(v) for v in hdr.tolist())
    if rank == src:
        out = X
    else:
        out = TorchCsr(rows, cols, torch.empty(rows + 1, dtype=torch.int64, device=dev),
                       torch.empty(nnz, dtype=torch.int32, device=dev),
                       torch.empty(nnz, dtype=torch.float64, device=dev))
    for t in (out.rpt, out.col, out.val):
        if t.numel():
            dist.broadcast(t, src, group=group)
    return out


def row_block(A: TorchCsr, r0: int, r1: int) -> TorchCsr:
    """Rows [r0, r1) of A as a CSR of its own (views of col/val, rpt rebased)."""
    if not (0 <= r0 <= r1 <= A.rows):
        raise ValueError(f"bad row block [{r0}, {r1}) of {A.rows} rows")
    a0, a1 = int(A.rpt[r0]), int(A.rpt[r1])
    return TorchCsr(r1 - r0, A.cols, (A.rpt[r0:r1 + 1] - a0).contiguous(), A.col[a0:a1], A.val[a0:a1])


def block_nnz(local_nnz: int, device, group=None) -> torch.Tensor:
    """All-gather every rank's nnz(C block): int64[world]. The global row_ptr
    of rank g's block starts at sum(counts[:g])."""
    world = dist.get_world_size(group)
    cnt = torch.tensor([local_nnz], dtype=torch.int64, device=device)
    allc = torch.empty(world, dtype=torch.int64, device=device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(allc, cnt, group=group)
    else:
        dist.all_gather(list(allc.split(1)), cnt, group=group)
    return allc


def _all_gather_varlen(x: torch.Tensor, counts: list[int], group=None) -> torch.Tensor:
    """Concatenate every rank's 1-D tensor (rank order); counts[g] = len on g."""
    world = len(counts)
    m = max(counts) if counts else 0
    buf = torch.zeros(m, dtype=x.dtype, device=x.device)
    buf[: x.numel()] = x
    parts = [torch.empty(m, dtype=x.dtype, device=x.device) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)])


def assemble_rpt(C_blk: TorchCsr, total_rows: int, group=None) -> torch.Tensor:
    """Global row_ptr of C on every rank (int64[total_rows + 1]) from the row
    blocks' row pointers: block g's entries shifted by the nnz of blocks < g.
    C's col/val stay row-distributed (each rank owns its rows)."""
    dev = C_blk.device
    world = dist.get_world_size(group)
    nnz = block_nnz(C_blk.nnz, dev, group).tolist()
    rows = block_nnz(C_blk.rows, dev, group).tolist()
    if sum(rows) != total_rows:
        raise ValueError(f"row blocks cover {sum(rows)} rows, expected {total_rows}")
    rp = _all_gather_varlen(C_blk.rpt[1:], rows, group)  # drop each block's leading 0
    shift = torch.repeat_interleave(
        torch.tensor([sum(nnz[:g]) for g in range(world)], dtype=torch.int64, device=dev),
        torch.tensor(rows, dtype=torch.int64, device=dev))
    return torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), rp + shift])


def assemble_csr(C_blk: TorchCsr, total_rows: int, group=None) -> TorchCsr:
    """Whole C on every rank from the row blocks (rank order = row order).
    rpt of block g is shifted by the nnz of blocks < g."""
    dev = C_blk.device
    world = dist.get_world_size(group)
    nnz = block_nnz(C_blk.nnz, dev, group).tolist()
    rows = block_nnz(C_blk.rows, dev, group).tolist()
    if sum(rows) != total_rows:
        raise ValueError(f"row blocks cover {sum(rows)} rows, expected {total_rows}")
    col = _all_gather_varlen(C_blk.col, nnz, group)
    val = _all_gather_varlen(C_blk.val, nnz, group)
    rp = _all_gather_varlen(C_blk.rpt[1:], rows, group)  # drop each block's leading 0
    shift = torch.repeat_interleave(
        torch.tensor([sum(nnz[:g]) for g in range(world)], dtype=torch.int64, device=dev),
        torch.tensor(rows, dtype=torch.int64, device=dev))
    rpt = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), rp + shift])
    return TorchCsr(total_rows, C_blk.cols, rpt, col, val)


# --- cyclic row ranges ------------------------------------------------------
# §III.D asks for p groups of rows with the same total n_prod;
# the groups need not be contiguous. Cutting the rows into world * k ranges of
# equal n_prod (brm_partition_rows with p = world * k) and dealing range j to
# rank j mod world keeps every rank's n_prod balanced AND spreads the rows
# whose products cost more than average (R-MAT's hub rows of many lists sit at
# the low row ids) over all ranks: rmat20_ef16's per-block emulation bound goes
# from 0.94 / 0.85 / 0.75 (contiguous blocks) to 0.98 / 0.97 / 0.93 at 2 / 4 /
# 8 ranks with k = 8.

def cyclic_ranges(chunk_bounds, rank: int, world: int) -> list[tuple[int, int]]:
    """Row ranges of `rank`: ranges j = rank, rank + world, ... of the
    world * k ranges whose bounds are chunk_bounds (world * k + 1 values)."""
    cb = [int(x) for x in chunk_bounds]
    if (len(cb) - 1) % world:
        raise ValueError("the number of ranges must be a multiple of the world size")
    return [(cb[j], cb[j + 1]) for j in range(rank, len(cb) - 1, world)]


def row_ranges_block(A: TorchCsr, ranges) -> TorchCsr:
    """The rows of the given [r0, r1) ranges of A, concatenated, as one CSR."""
    blocks = [row_block(A, r0, r1) for r0, r1 in ranges]
    if not blocks:
        raise ValueError("no row ranges")
    if len(blocks) == 1:
        return blocks[0]
    nnz0 = [0]
    for b in blocks:
        nnz0.append(nnz0[-1] + b.nnz)
    rpt = torch.cat([blocks[0].rpt[:1]] + [b.rpt[1:] + o for b, o in zip(blocks, nnz0)])
    return TorchCsr(sum(b.rows for b in blocks), A.cols, rpt, torch.cat([b.col for b in blocks]),
                    torch.cat([b.val for b in blocks]))


def cyclic_row_order(chunk_bounds, world: int, device="cpu") -> torch.Tensor:
    """Global row id of every row in rank-major order: rank 0's rows (its
    ranges concatenated), then rank 1's, ... (int64[total rows]). Depends only
    on the bounds: compute once per partition and pass to the assemblers."""
    cb = [int(x) for x in chunk_bounds]
    parts = [torch.arange(r0, r1, dtype=torch.int64, device=device)
             for g in range(world) for r0, r1 in cyclic_ranges(cb, g, world)]
    return torch.cat(parts) if parts else torch.zeros(0, dtype=torch.int64, device=device)


def _cyclic_row_sizes(C_blk: TorchCsr, chunk_bounds, group=None, order=None):
    """Row sizes of C in global row order from every rank's block (its ranges
    concatenated), plus the per-rank row-size lists."""
    dev = C_blk.device
    world = dist.get_world_size(group)
    cb = [int(x) for x in chunk_bounds]
    rows = block_nnz(C_blk.rows, dev, group).tolist()
    want = [sum(r1 - r0 for r0, r1 in cyclic_ranges(cb, g, world)) for g in range(world)]
    if rows != want:
        raise ValueError(f"the ranks hold {rows} rows, their ranges cover {want}")
    sizes_all = _all_gather_varlen(C_blk.rpt[1:] - C_blk.rpt[:-1], rows, group)
    if order is None:
        order = cyclic_row_order(cb, world, dev)
    glob = torch.empty(cb[-1], dtype=torch.int64, device=dev)
    glob[order] = sizes_all  # one scatter: rank-major order -> global row order
    return glob, list(sizes_all.split(rows))


def assemble_rpt_cyclic(C_blk: TorchCsr, chunk_bounds, group=None, order=None) -> torch.Tensor:
    """Global row_ptr of C on every rank when the ranks hold cyclic row ranges
    (cyclic_ranges of chunk_bounds); C's col/val stay with their ranks.
    order: cyclic_row_order(chunk_bounds, world, device), if already made."""
    glob, _ = _cyclic_row_sizes(C_blk, chunk_bounds, group, order)
    return torch.cat([torch.zeros(1, dtype=torch.int64, device=glob.device), torch.cumsum(glob, 0)])


def assemble_csr_cyclic(C_blk: TorchCsr, chunk_bounds, group=None, order=None) -> TorchCsr:
    """Whole C on every rank, rows in global order, from cyclic row ranges."""
    dev = C_blk.device
    world = dist.get_world_size(group)
    cb = [int(x) for x in chunk_bounds]
    glob, per_rank = _cyclic_row_sizes(C_blk, cb, group, order)
    rpt = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), torch.cumsum(glob, 0)])
    nnz = block_nnz(C_blk.nnz, dev, group).tolist()
    col_all = _all_gather_varlen(C_blk.col, nnz, group).split(nnz)
    val_all = _all_gather_varlen(C_blk.val, nnz, group).split(nnz)
    rb = rpt[torch.tensor(cb, dtype=torch.int64, device=dev)].tolist()  # row_ptr at the range bounds (one readback)
    col = torch.empty(rb[-1], dtype=C_blk.col.dtype, device=dev)
    val = torch.empty(rb[-1], dtype=C_blk.val.dtype, device=dev)
    for g in range(world):
        at = 0
        for j in range(g, len(cb) - 1, world):  # range j: rows [cb[j], cb[j+1]), entries [rb[j], rb[j+1])
            n = rb[j + 1] - rb[j]
            col[rb[j]:rb[j + 1]] = col_all[g][at:at + n]
            val[rb[j]:rb[j + 1]] = val_all[g][at:at + n]
            at += n
        if at != nnz[g]:
            raise ValueError(f"rank {g} holds {nnz[g]} entries, its ranges cover {at}")
    return TorchCsr(cb[-1], C_blk.cols, rpt, col, val)


def share_tensor(t: torch.Tensor, group=None) -> list[torch.Tensor]:
    """Every rank's `t` opened on every rank: out[g] is rank g's tensor (this
    rank's own `t` at its own index), mapped through CUDA IPC by torch's
    tensor-sharing machinery (the handle travels by all_gather_object). `t`
    must come from torch's caching allocator and stay alive on its owner while
    any peer uses the mapping."""
    from torch.multiprocessing.reductions import reduce_tensor
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    infos = [None] * world
    dist.all_gather_object(infos, reduce_tensor(t), group=group)
    return [t if g == rank else fn(*args) for g, (fn, args) in enumerate(infos)]


class PeerAssembly:
    """C = A*B over the ranks' row blocks with the write-out fused into the
    assembly: every rank holds a whole-C col/val array, opens its peers' arrays
    (share_tensor), and its fill stores each entry of its row block into its
    own array AND, through brm_set_mirrors, into every peer's at the block's
    global offset -- the numeric merge kernels' stores travel over NVLink P2P,
    so no all-gather of col/val follows the merge. Only the block sizes and the
    row pointers are all-gathered (assemble_rpt). At most 8 ranks (7 mirrors).

    The arrays are kept and re-shared only when C outgrows them (every rank
    sees the same total, so the ranks decide alike)."""

    def __init__(self, ctx, group=None):
        self.ctx, self.group = ctx, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        if self.world > 8:
            raise ValueError("PeerAssembly serves at most 8 ranks (7 mirrors)")
        self.cap = 0
        self.col = self.val = None
        self.peer_col = self.peer_val = None

    def _ensure(self, total: int):
        if total <= self.cap and self.col is not None:
            return
        dev = self.ctx.device
        self.peer_col = self.peer_val = None  # drop the old mappings first
        self.col = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
        self.val = torch.empty(max(total, 1), dtype=torch.float64, device=dev)
        self.cap = max(total, 1)
        self.peer_col = share_tensor(self.col, self.group)
        self.peer_val = share_tensor(self.val, self.group)
        for g, t in enumerate(self.peer_col):
            if g != self.rank and t.device != dev:
                self.ctx.brm_enable_peer_access(t.device.index)

    def spgemm(self, A_blk: TorchCsr, B: TorchCsr, mode, total_rows: int) -> TorchCsr:
        """This rank's row block A_blk (blocks in rank order cover A); returns
        the whole C on every rank (views of the kept arrays, valid until the
        next call)."""
        ctx, dev = self.ctx, self.ctx.device
        cdev = dev if dist.get_backend(self.group) == "nccl" else torch.device("cpu")  # where the collectives run
        c_rpt, nnz = ctx.brmerge_spgemm_structure(A_blk, B, mode)
        nnzs = block_nnz(nnz, cdev, self.group).tolist()
        total, off = sum(nnzs), sum(nnzs[: self.rank])
        self._ensure(total)
        # every rank has finished reading the previous C before anyone overwrites it
        torch.cuda.synchronize(dev)
        dist.barrier(self.group)
        others = [g for g in range(self.world) if g != self.rank]
        ctx.brm_set_mirrors([self.peer_col[g].data_ptr() + 4 * off for g in others],
                            [self.peer_val[g].data_ptr() + 8 * off for g in others])
        try:
            Cb = ctx.brmerge_spgemm_fill(A_blk.rows, B.cols, c_rpt, nnz,
                                         col=self.col[off:off + nnz], val=self.val[off:off + nnz])
        finally:
            ctx.brm_set_mirrors()
        # the peers' stores are complete once every rank's stream has drained
        torch.cuda.synchronize(dev)
        dist.barrier(self.group)
        # row_ptr offsets by all-gather (assemble_rpt reads only rpt, rows and nnz of the block)
        rpt = assemble_rpt(TorchCsr(Cb.rows, Cb.cols, Cb.rpt.to(cdev), Cb.col, Cb.val), total_rows, self.group)
        return TorchCsr(total_rows, B.cols, rpt.to(dev), self.col[:total], self.val[:total])
