"""World-size-2 gloo tests (CPU) of the multi-GPU plumbing in
paper_2206_06611_b200/dist.py: B broadcast, n_prod-balanced row blocks
(§III.D; contiguous, or cyclic ranges dealt round-robin), row_ptr
offsets and C row-block assembly. The per-rank
SpGEMM is stood in for by the oracle (no GPU here); the product path on GPUs
calls the C ABI instead (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q, partition="contiguous"):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from inputs import Csr, random_sparse, uniform_random
        from paper_2206_06611_b200 import TorchCsr
        from paper_2206_06611_b200 import dist as bd
        if case == "square":
            A = uniform_random(700, 700, 6, seed=3)
            B = A
        elif case == "skewed":
            A = random_sparse(300, 200, 0.02, seed=4)
            A.val[:] = 1.0
            B = random_sparse(200, 150, 0.1, seed=5)
        else:  # more ranks' worth of rows than rows: some blocks empty
            A = uniform_random(1, 5, 2, seed=6)
            B = uniform_random(5, 4, 2, seed=7)
        Bt = bd.broadcast_csr(TorchCsr.from_csr(B, device="cpu") if rank == 0 else None, src=0, device="cpu")
        assert torch.equal(Bt.rpt, torch.from_numpy(B.rpt)) and torch.equal(Bt.col, torch.from_numpy(B.col))
        assert torch.equal(Bt.val, torch.from_numpy(B.val))
        nprod = oracle.row_nprod(A, B)
        bounds = oracle.balance_by_nprod(nprod, world)
        At = TorchCsr.from_csr(A, device="cpu")
        if partition == "cyclic":  # 3 ranges of equal n_prod per rank, dealt round-robin
            bounds = oracle.balance_by_nprod(nprod, world * 3)
            ranges = bd.cyclic_ranges(bounds, rank, world)
            assert len(ranges) == 3 and ranges[0][0] == bounds[rank]
            blk = bd.row_ranges_block(At, ranges)
        else:
            blk = bd.row_block(At, bounds[rank], bounds[rank + 1])
        # per-rank compute (oracle stands in for the C ABI on the CPU)
        Ab = Csr(blk.rows, blk.cols, blk.rpt.numpy(), blk.col.numpy(), blk.val.numpy())
        Cb = oracle.spgemm_brmerge(Ab, B)[0]
        counts = bd.block_nnz(Cb.nnz, "cpu").tolist()
        ref = oracle.spgemm_brmerge(A, B)[0]
        if partition == "cyclic":
            Ct = TorchCsr.from_csr(Cb, device="cpu")
            C = bd.assemble_csr_cyclic(Ct, bounds)
            assert np.array_equal(bd.assemble_rpt_cyclic(Ct, bounds).numpy(), ref.rpt)
        else:
            C = bd.assemble_csr(TorchCsr.from_csr(Cb, device="cpu"), A.rows)
        ok = (np.array_equal(C.rpt.numpy(), ref.rpt) and np.array_equal(C.col.numpy(), ref.col)
              and np.array_equal(C.val.numpy(), ref.val) and sum(counts) == ref.nnz
              and counts[rank] == Cb.nnz)
        q.put((rank, ok, bounds))
    except Exception as e:  # surface in the parent
        q.put((rank, repr(e), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("partition", ["contiguous", "cyclic"])
@pytest.mark.parametrize("case", ["square", "skewed", "tiny"])
def test_two_rank_assembly(case, partition, oracle_mod):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q, partition)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, _ in res:
        assert ok is True, (rank, ok)
    b = [x[2] for x in res]
    assert b[0] == b[1]


def test_row_block_rebases():
    from inputs import uniform_random
    from paper_2206_06611_b200 import TorchCsr
    from paper_2206_06611_b200 import dist as bd
    A = TorchCsr.from_csr(uniform_random(50, 40, 3, seed=1), device="cpu")
    blk = bd.row_block(A, 10, 20)
    assert blk.rows == 10 and int(blk.rpt[0]) == 0 and int(blk.rpt[-1]) == 30
    assert torch.equal(blk.col, A.col[30:60])
    with pytest.raises(ValueError):
        bd.row_block(A, 20, 10)
