"""Two ranks on one GPU (gloo for the collectives), each running the C ABI on
its n_prod-balanced row block (§III.D): the partition comes from
the library's own kernels (brm_row_nprod -> brm_exclusive_scan_i64 ->
brm_partition_rows), B is broadcast from rank 0, each rank computes its block
of C on cuda:0, and dist.assemble_csr all-gathers the row blocks and row_ptr
offsets -- or ("peer") dist.PeerAssembly has each rank's fill store its block
into both ranks' whole-C arrays over peer memory (brm_set_mirrors, the other
rank's array opened through CUDA IPC) and all-gathers only the row pointers.
"cyclic" deals 4 ranges of equal n_prod per rank round-robin
(dist.cyclic_ranges) and reassembles C in global row order. The assembled C
must equal the oracle's bit for bit (columns, row pointers, Algorithm-1
values). This is the multi-GPU path of bench.py with
both ranks' kernels on one device (they never wait on each other's kernels)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, mode, q, assemble="allgather"):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from inputs import rmat, uniform_random
        from paper_2206_06611_b200 import Context, TorchCsr
        from paper_2206_06611_b200 import dist as bd
        if case == "rmat":  # heavy rows (windowed path) land on both ranks
            A = rmat(13, 16, 0.57, 0.19, 0.19, 0.05, seed=9)
        else:
            A = uniform_random(30001, 30001, 9, seed=10)
        B = A
        ctx = Context(torch.device("cuda", 0))
        Bd = TorchCsr.from_csr(B) if rank == 0 else None
        Bc = bd.broadcast_csr(Bd.to("cpu") if rank == 0 else None, src=0, device="cpu")  # gloo: host tensors
        Bd = Bc.to("cuda")
        Ad = TorchCsr.from_csr(A)
        nprod = ctx.brm_row_nprod(Ad, Bd)
        bounds = ctx.brm_partition_rows(ctx.brm_exclusive_scan_i64(nprod), world).cpu().tolist()
        assert bounds == oracle.balance_by_nprod(oracle.row_nprod(A, B), world)
        blk = bd.row_block(Ad, bounds[rank], bounds[rank + 1])
        ref, _ = oracle.spgemm_brmerge(A, B)
        if assemble == "peer":
            # write-out over peer memory: each rank's fill stores its block into
            # both ranks' whole-C arrays (the other rank's opened through CUDA IPC)
            pa = bd.PeerAssembly(ctx)
            small = uniform_random(4000, A.rows, 5, seed=3)  # a first, smaller product: the arrays regrow after it
            Sd = TorchCsr.from_csr(small)
            half = [0, 1500, 4000]
            Cs = pa.spgemm(bd.row_block(Sd, half[rank], half[rank + 1]), Bd, mode, small.rows).to("cpu")
            rs, _ = oracle.spgemm_brmerge(small, B)
            if not (np.array_equal(Cs.rpt.numpy(), rs.rpt) and np.array_equal(Cs.col.numpy(), rs.col)
                    and np.array_equal(Cs.val.numpy(), rs.val)):
                raise AssertionError("peer assembly of the first product differs from the oracle")
            for _ in range(2):  # the second call reuses the shared arrays
                C = pa.spgemm(blk, Bd, mode, A.rows).to("cpu")
        elif assemble == "cyclic":
            # 4 row ranges of equal n_prod per rank, dealt round-robin (the library's partition kernel)
            cb = ctx.brm_partition_rows(ctx.brm_exclusive_scan_i64(nprod), world * 4).cpu().tolist()
            assert cb == oracle.balance_by_nprod(oracle.row_nprod(A, B), world * 4)
            Cb = ctx.spgemm(bd.row_ranges_block(Ad, bd.cyclic_ranges(cb, rank, world)), Bd, mode)
            torch.cuda.synchronize()
            Cc = Cb.to("cpu")
            C = bd.assemble_csr_cyclic(Cc, cb)
            if not np.array_equal(bd.assemble_rpt_cyclic(Cc, cb).numpy(), ref.rpt):
                raise AssertionError("cyclic row_ptr assembly differs from the oracle")
        else:
            Cb = ctx.spgemm(blk, Bd, mode)
            torch.cuda.synchronize()
            C = bd.assemble_csr(Cb.to("cpu"), A.rows)
        ok = (np.array_equal(C.rpt.numpy(), ref.rpt) and np.array_equal(C.col.numpy(), ref.col)
              and np.array_equal(C.val.numpy(), ref.val))
        q.put((rank, ok, bounds))
        ctx.close()
    except Exception as e:  # surface in the parent
        import traceback
        q.put((rank, traceback.format_exc(), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,mode", [("uniform", "precise"), ("uniform", "upper"), ("rmat", "precise"),
                                       ("rmat", "upper")])
@pytest.mark.parametrize("assemble", ["allgather", "peer", "cyclic"])
def test_two_ranks_one_gpu(case, mode, assemble, oracle_mod):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, mode, q, assemble)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, _ in res:
        assert ok is True, (rank, ok)
    assert res[0][2] == res[1][2]
