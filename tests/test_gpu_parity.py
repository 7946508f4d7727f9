"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

Bar (BASELINE.json north_star): rpt and col bit-exact (structural zeros from
cancellation kept); fp64 values within |c - c_ref| <= 1e-12 * sum|a_ik b_kj|
per entry. Additionally the values must be bit-identical to Algorithm 1's
tree order (oracle.spgemm_brmerge), which the kernels follow exactly.
"""
import numpy as np
import pytest

from inputs import Csr, identity, random_sparse, uniform_random
from parity import compare

pytestmark = pytest.mark.gpu

MODES = ["upper", "precise"]


@pytest.fixture(scope="module")
def ctx():
    import torch
    from paper_2206_06611_b200 import Context
    assert torch.cuda.is_available()
    c = Context()
    yield c
    c.close()


def run(ctx, A: Csr, B: Csr, mode: str):
    from paper_2206_06611_b200 import TorchCsr
    C = ctx.spgemm(TorchCsr.from_csr(A), TorchCsr.from_csr(B), mode)
    return C.to_numpy()


def _lists_matrix(row_specs, list_len, ncols, seed, empty_rows_of_b=0):
    """A has one row per (num_lists) in row_specs, pointing at distinct rows of
    B; B rows have `list_len` entries (plus `empty_rows_of_b` empty rows)."""
    rng = np.random.default_rng(seed)
    kb = max(max(row_specs) if row_specs else 1, 1) + empty_rows_of_b
    Bfull = uniform_random(kb - empty_rows_of_b, ncols, list_len, seed=seed) if kb > empty_rows_of_b else None
    # interleave empty rows into B
    lens = np.full(kb, list_len, np.int64)
    empty = rng.choice(kb, size=empty_rows_of_b, replace=False) if empty_rows_of_b else np.zeros(0, np.int64)
    lens[empty] = 0
    rpt = np.zeros(kb + 1, np.int64)
    np.cumsum(lens, out=rpt[1:])
    B = Csr(kb, ncols, rpt, Bfull.col[:rpt[-1]].copy(), Bfull.val[:rpt[-1]].copy())
    arpt = [0]
    acol, aval = [], []
    for nl in row_specs:
        cols = np.sort(rng.choice(kb, size=nl, replace=False))
        acol.append(cols)
        aval.append(rng.uniform(-1, 1, size=nl))
        arpt.append(arpt[-1] + nl)
    A = Csr(len(row_specs), kb, np.array(arpt, np.int64),
            np.concatenate(acol).astype(np.int32) if acol else np.zeros(0, np.int32),
            np.concatenate(aval) if aval else np.zeros(0))
    return A, B


@pytest.mark.parametrize("mode", MODES)
def test_config0_full(ctx, oracle_mod, mode):
    """configs[0]: 2000x2000, 8 per row, seed 1, every row vs the oracle."""
    A = uniform_random(2000, 2000, 8, seed=1)
    compare(run(ctx, A, A, mode), A, A)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("seed", range(6))
def test_random_rectangular(ctx, oracle_mod, mode, seed):
    rng = np.random.default_rng(seed)
    m, k, n = (int(x) for x in rng.integers(1, 300, size=3))
    A = random_sparse(m, k, float(rng.uniform(0.005, 0.3)), seed=seed)
    B = random_sparse(k, n, float(rng.uniform(0.005, 0.3)), seed=seed + 99)
    compare(run(ctx, A, B, mode), A, B)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("list_len,specs", [
    (1, [1, 2, 3, 5, 8]),                        # tier 1 (register, 8 lanes)
    (2, [4, 5]),                                 # tier 1 edge P=8 / tier 2 P=10
    (1, [9, 17, 31, 32]),                        # tier 2 (register, warp), nl up to 32
    (4, [8, 9]),                                 # tier 2 edge P=32 / tier 3 P=36
    (16, [15, 16, 17]),                          # tier 3 edge (256)
    (4, [64, 65]),                               # tier 3 list cap 64 -> tier 5
    (27, [27, 28, 29]),                          # tier 4 (stencil-like, 768 edge)
    (33, [90, 93, 94]),                          # tier 5 (3072 edge)
    (64, [100, 104, 105]),                       # tier 6 (6656 edge) -> global
    (100, [90, 300]),                            # global tier
    (3, [40, 129, 257, 300, 513, 600, 1500]),    # many short lists (list caps 64 / 256 / 512)
])
def test_tier_boundaries(ctx, oracle_mod, mode, list_len, specs):
    A, B = _lists_matrix(specs, list_len, 5000, seed=list_len)
    compare(run(ctx, A, B, mode), A, B)


def _top_column_matrix(specs, list_len, ncols, seed, pool=64):
    """Like _lists_matrix, but every B row draws its columns from the `pool`
    highest columns of an ncols-wide B (ncols - 1 included in every row), so
    the merges see many duplicates right below the sentinel."""
    rng = np.random.default_rng(seed)
    kb = max(specs)
    top = ncols - pool + np.arange(pool)
    col = np.concatenate([np.sort(np.append(rng.choice(top[:-1], size=list_len - 1, replace=False), ncols - 1))
                          for _ in range(kb)]).astype(np.int32)
    B = Csr(kb, ncols, np.arange(kb + 1, dtype=np.int64) * list_len, col, rng.uniform(-1, 1, size=col.size))
    arpt, acol = [0], []
    for nl in specs:
        acol.append(np.sort(rng.choice(kb, size=nl, replace=False)))
        arpt.append(arpt[-1] + nl)
    acol = np.concatenate(acol).astype(np.int32)
    A = Csr(len(specs), kb, np.array(arpt, np.int64), acol, rng.uniform(-1, 1, size=acol.size))
    return A, B


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("tier,slot_bits,list_len,nl", [
    (3, 8, 12, 16),     # P = 192
    (4, 10, 16, 40),    # P = 640
    (5, 12, 24, 100),   # P = 2400
    (6, 13, 20, 300),   # P = 6000
])
@pytest.mark.parametrize("wide", [False, True])
def test_record_packing_boundary(ctx, oracle_mod, mode, tier, slot_bits, list_len, nl, wide):
    """Record tiers pack {col, slot} into 32 bits while B.cols <=
    2^(32 - slot_bits) - 1 (the sentinel's column) and fall back to 8-byte
    records one column above; both sides of the boundary, with column
    B.cols - 1 in every list."""
    ncols = (1 << (32 - slot_bits)) - 1 + int(wide)
    A, B = _top_column_matrix([nl, nl - 1, nl], list_len, ncols, seed=tier)
    compare(run(ctx, A, B, mode), A, B)


def _span_matrix(nl, list_len, span, base, seed, pool=96):
    """One A row of nl lists; B rows draw list_len sorted columns from a pool
    of `pool` columns in [base, base + span] holding both ends (first list:
    base, last list: base + span), so the row's column span is exactly span
    and its columns repeat across lists."""
    rng = np.random.default_rng(seed)
    pc = np.unique(np.concatenate([[base, base + span], rng.integers(base, base + span + 1, size=pool)]))
    rows = []
    for j in range(nl):
        c = rng.choice(pc, size=list_len, replace=False)
        if j == 0:
            c[0] = base
        if j == nl - 1:
            c[0] = base + span
        rows.append(np.unique(c))
    rpt = np.zeros(nl + 1, np.int64)
    np.cumsum([len(r) for r in rows], out=rpt[1:])
    col = np.concatenate(rows).astype(np.int32)
    B = Csr(nl, base + span + 1, rpt, col, rng.uniform(-1, 1, size=col.size))
    A = Csr(1, nl, np.array([0, nl], np.int64), np.arange(nl, dtype=np.int32), rng.uniform(-1, 1, size=nl))
    return A, B


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("nl,list_len", [(16, 16), (27, 27)])  # tier 3 (P 256) and tier 4 (P 729)
@pytest.mark.parametrize("span", [1, 32766, 32767, 32768, 40000])
@pytest.mark.parametrize("base", [0, 2_000_000_000])
def test_symbolic_direct_table_span(ctx, oracle_mod, mode, nl, list_len, span, base):
    """PRECISE symbolic of one-warp rows: a bitmap over the row's column span
    while span <= 32767 (the table's 32768 bits), hashing above; both sides
    of the boundary, near column 0 and near 2^31."""
    if span < list_len:
        list_len = span + 1
    A, B = _span_matrix(nl, list_len, span, base, seed=span + nl)
    compare(run(ctx, A, B, mode), A, B)


@pytest.mark.parametrize("mode", MODES)
def test_misaligned_b_arrays(ctx, oracle_mod, mode):
    """B's col/val arrays at addresses that are not 16-byte aligned (views one
    element into larger buffers): the gathers must give the same bits."""
    import torch
    from paper_2206_06611_b200 import TorchCsr
    A = uniform_random(3000, 3000, 13, seed=12)
    col = torch.empty(A.nnz + 1, dtype=torch.int32, device="cuda")[1:]
    val = torch.empty(A.nnz + 1, dtype=torch.float64, device="cuda")[1:]
    col.copy_(torch.from_numpy(A.col))
    val.copy_(torch.from_numpy(A.val))
    assert col.data_ptr() % 16 and val.data_ptr() % 16
    Bm = TorchCsr(A.rows, A.cols, torch.from_numpy(A.rpt).cuda(), col, val)
    C = ctx.spgemm(TorchCsr.from_csr(A), Bm, mode)
    compare(C.to_numpy(), A, A)


@pytest.mark.parametrize("mode", MODES)
def test_many_empty_lists(ctx, oracle_mod, mode):
    """Rows with many empty B rows among their lists: tree shape must keep them."""
    A, B = _lists_matrix([5, 50, 700, 1100, 2000], 4, 3000, seed=3, empty_rows_of_b=1500)
    compare(run(ctx, A, B, mode), A, B)


@pytest.mark.parametrize("mode", MODES)
def test_heavy_rows(ctx, oracle_mod, mode):
    """Rows far beyond the shared-memory tiers (n_prod up to ~200k): column
    slabs (20 and 200 lists) and the global tier (1000 and 2000 long lists)."""
    A, B = _lists_matrix([200, 1000, 2000, 20], 100, 20000, seed=11)
    compare(run(ctx, A, B, mode), A, B)


@pytest.mark.parametrize("mode", MODES)
def test_heavy_rows_global_route(oracle_mod, mode):
    """brm_set_heavy_route(BRM_HEAVY_GLOBAL): every heavy row on the
    global-memory tier gives the same bits."""
    from paper_2206_06611_b200 import Context
    c = Context()
    try:
        c.brm_set_heavy_route(c.HEAVY_GLOBAL)
        A, B = _lists_matrix([200, 1000, 2000, 20], 100, 20000, seed=11)
        compare(run(c, A, B, mode), A, B)
        A, B = _skewed_matrix([1, 2, 7, 64, 65, 300, 512, 513], 40000, seed=5)
        compare(run(c, A, B, mode), A, B)
    finally:
        c.close()


def _skewed_matrix(specs, ncols, seed, max_len=3000, identical=False):
    """A row per nl in specs over a B of rows with lengths spread over
    [0, max_len] (a tenth of them empty); identical=True gives every B row
    the same columns (every column repeats in every list)."""
    rng = np.random.default_rng(seed)
    kb = max(specs)
    lens = rng.integers(0, max_len + 1, size=kb)
    lens[rng.random(kb) < 0.1] = 0
    if identical:
        lens[:] = max_len
        base = np.sort(rng.choice(ncols, size=max_len, replace=False))
    cols = [base if identical else np.sort(rng.choice(ncols, size=n, replace=False)) for n in lens]
    rpt = np.zeros(kb + 1, np.int64)
    np.cumsum(lens, out=rpt[1:])
    bcol = np.concatenate(cols).astype(np.int32)
    B = Csr(kb, ncols, rpt, bcol, rng.uniform(-1, 1, size=bcol.size))
    arpt, acol = [0], []
    for nl in specs:
        acol.append(np.sort(rng.choice(kb, size=nl, replace=False)))
        arpt.append(arpt[-1] + nl)
    acol = np.concatenate(acol).astype(np.int32)
    A = Csr(len(specs), kb, np.array(arpt, np.int64), acol, rng.uniform(-1, 1, size=acol.size))
    return A, B


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("ncols", [40000, 1 << 21, 3_000_000])  # packed records up to 2^21 - 1 columns
def test_slab_rows(ctx, oracle_mod, mode, ncols):
    """Heavy rows in column slabs: one list, two, up to 64 (k_slab), then
    two levels of slabs (k_slab2) at 65, 256, 257, 512 and 513, over lists of
    skewed lengths with empty ones."""
    A, B = _skewed_matrix([1, 2, 7, 64, 65, 256, 257, 512, 513], ncols, seed=5)
    compare(run(ctx, A, B, mode), A, B)


@pytest.mark.parametrize("mode", MODES)
def test_slab_long_single_lists(ctx, oracle_mod, mode):
    """Heavy rows of one list (20,000 products: Alg. 1 only scales it), of
    two lists (20,000 + 5) and of three lists of which one is empty."""
    rng = np.random.default_rng(8)
    lens = np.array([20000, 5, 0, 9000])
    cols = [np.sort(rng.choice(50000, size=n, replace=False)) for n in lens]
    rpt = np.zeros(5, np.int64)
    np.cumsum(lens, out=rpt[1:])
    bcol = np.concatenate(cols).astype(np.int32)
    B = Csr(4, 50000, rpt, bcol, rng.uniform(-1, 1, size=bcol.size))
    acol = np.array([0, 0, 1, 0, 2, 3], np.int32)
    A = Csr(3, 4, np.array([0, 1, 3, 6], np.int64), acol, rng.uniform(-1, 1, size=6))
    compare(run(ctx, A, B, mode), A, B)


@pytest.mark.parametrize("mode", MODES)
def test_two_level_slab_rows(ctx, oracle_mod, mode):
    """Rows of > 64 lists: levels of column slabs over aligned 64-list blocks
    (k_slab2): two levels up to 4,096 lists, three beyond (short last blocks
    and groups at 700, 4,097, 16,383 and 16,385)."""
    A, B = _lists_matrix([700, 4096, 4097, 16383, 16384, 16385], 40, 200000, seed=17)
    compare(run(ctx, A, B, mode), A, B)


@pytest.mark.parametrize("mode", MODES)
def test_slab_rows_identical_lists(ctx, oracle_mod, mode):
    """Every list has the same 2,500 columns: each slab takes exactly q
    products from every list, and every column sums nl products."""
    A, B = _skewed_matrix([3, 40, 64, 200, 512], 10**6, seed=6, max_len=2500, identical=True)
    compare(run(ctx, A, B, mode), A, B)


@pytest.mark.parametrize("mode", MODES)
def test_edge_cases(ctx, oracle_mod, mode):
    # empty matrix
    E = Csr(0, 5, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0))
    B5 = uniform_random(5, 7, 2, seed=1)
    rpt, col, val = run(ctx, E, B5, mode)
    assert rpt.tolist() == [0] and col.size == 0
    # no nonzeros at all
    Z = Csr(4, 4, np.zeros(5, np.int64), np.zeros(0, np.int32), np.zeros(0))
    rpt, col, val = run(ctx, Z, Z, mode)
    assert rpt.tolist() == [0] * 5
    # A's lists all hit empty B rows (n_prod = 0 with num_list > 0)
    A = Csr(2, 3, np.array([0, 2, 3], np.int64), np.array([0, 2, 1], np.int32), np.ones(3))
    Bz = Csr(3, 4, np.array([0, 0, 2, 2], np.int64), np.array([1, 3], np.int32), np.array([2.0, 3.0]))
    compare(run(ctx, A, Bz, mode), A, Bz)
    # cancellation: C = [[0]] is stored
    A1 = Csr(1, 2, np.array([0, 2], np.int64), np.array([0, 1], np.int32), np.array([1.0, 1.0]))
    B1 = Csr(2, 1, np.array([0, 1, 2], np.int64), np.array([0, 0], np.int32), np.array([1.0, -1.0]))
    rpt, col, val = run(ctx, A1, B1, mode)
    assert rpt.tolist() == [0, 1] and col.tolist() == [0] and val.tolist() == [0.0]
    # identity both sides, exact
    X = uniform_random(3000, 3000, 5, seed=2)
    I = identity(3000)
    for L, R in ((X, I), (I, X)):
        rpt, col, val = run(ctx, L, R, mode)
        np.testing.assert_array_equal(rpt, X.rpt)
        np.testing.assert_array_equal(col, X.col)
        np.testing.assert_array_equal(val, X.val)


@pytest.mark.parametrize("mode", MODES)
def test_integer_values_exact(ctx, oracle_mod, mode):
    A = random_sparse(400, 300, 0.05, seed=5, integer_values=True)
    B = random_sparse(300, 500, 0.05, seed=6, integer_values=True)
    rpt, col, val = run(ctx, A, B, mode)
    np.testing.assert_array_equal(_dense(rpt, col, val, 400, 500), A.to_dense() @ B.to_dense())
    compare((rpt, col, val), A, B)


def _dense(rpt, col, val, m, n):
    d = np.zeros((m, n))
    r = np.repeat(np.arange(m), np.diff(rpt))
    d[r, col] = val
    return d


def test_repeatable_and_modes_agree(ctx):
    A = uniform_random(5000, 5000, 12, seed=4)
    r1 = run(ctx, A, A, "upper")
    r2 = run(ctx, A, A, "precise")
    r3 = run(ctx, A, A, "precise")
    for x, y in ((r1, r2), (r2, r3)):
        for a, b in zip(x, y):
            np.testing.assert_array_equal(a, b)


def test_onecall_and_host_forms(ctx, oracle_mod):
    import torch
    from paper_2206_06611_b200 import TorchCsr
    A = uniform_random(3000, 3000, 9, seed=7)
    c = ctx.brmerge_spgemm(TorchCsr.from_csr(A), TorchCsr.from_csr(A), "precise")
    torch.cuda.synchronize()
    n = c.nnz

    class _View:  # zero-copy view of a library-allocated device array
        def __init__(self, ptr, cnt, typestr):
            self.__cuda_array_interface__ = {"shape": (cnt,), "typestr": typestr,
                                             "data": (ptr, False), "version": 3}
    host = []
    for ptr, cnt, ts in ((c.rpt, c.rows + 1, "<i8"), (c.col, n, "<i4"), (c.val, n, "<f8")):
        host.append(torch.as_tensor(_View(ptr, cnt, ts), device="cuda").cpu().numpy().copy())
    ctx.brm_csr_free(c)
    compare(tuple(host), A, A)
    Ah = TorchCsr.from_csr(A, pin=True)
    rows, cols, rpt, col, val = ctx.brmerge_spgemm_host(Ah, Ah, "upper")
    assert (rows, cols) == (3000, 3000)
    compare((rpt.copy(), col.copy(), val.copy()), A, A)


def test_stage_nprod_scan_partition(ctx, oracle_mod):
    import torch
    from paper_2206_06611_b200 import TorchCsr
    A = random_sparse(3000, 2000, 0.01, seed=8)
    B = random_sparse(2000, 1000, 0.02, seed=9)
    nprod = ctx.brm_row_nprod(TorchCsr.from_csr(A), TorchCsr.from_csr(B)).cpu().numpy()
    np.testing.assert_array_equal(nprod, oracle_mod.row_nprod(A, B))
    # long rows (> 512 nonzeros: summed by a CTA each from 65,536 rows on,
    # by the warps below) between short and empty ones, in 32-row chunks with
    # several runs, and at the matrix end
    rng = np.random.default_rng(5)
    lens = np.zeros(70000, np.int64)
    lens[:700] = rng.integers(0, 40, size=700)
    lens[69000:] = rng.integers(0, 5, size=1000)
    lens[[3, 4, 31, 32, 60, 100, 101, 102, 699, 69998, 69999]] = [513, 2000, 900, 4000, 600, 513, 1, 3000, 1500,
                                                                  700, 800]
    lens[[5, 33]] = 0
    Bw = random_sparse(5000, 300, 0.02, seed=10)
    cols = [np.sort(rng.choice(5000, size=n, replace=False)).astype(np.int32) for n in lens]
    rpt = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    Al = Csr(lens.size, 5000, rpt, np.concatenate(cols), rng.uniform(-1, 1, size=int(rpt[-1])))
    for X in (Al, _row_slice(Al, 0, 700)):  # with and without the long-row pass
        got = ctx.brm_row_nprod(TorchCsr.from_csr(X), TorchCsr.from_csr(Bw)).cpu().numpy()
        np.testing.assert_array_equal(got, oracle_mod.row_nprod(X, Bw))
        compare(run(ctx, X, Bw, "precise"), X, Bw)
    rng = np.random.default_rng(0)
    for n in (0, 1, 2047, 2048, 2049, 100_000, 3_000_001):
        x = rng.integers(0, 1 << 40, size=n, dtype=np.int64)
        out = ctx.brm_exclusive_scan_i64(torch.from_numpy(x).cuda()).cpu().numpy()
        ref = np.zeros(n + 1, np.int64)
        np.cumsum(x, out=ref[1:])
        np.testing.assert_array_equal(out, ref)
    off = ctx.brm_exclusive_scan_i64(torch.from_numpy(nprod).cuda())
    for p in (1, 2, 3, 4, 8, 64):
        got = ctx.brm_partition_rows(off, p).cpu().tolist()
        assert got == oracle_mod.balance_by_nprod(nprod, p), p


def _row_slice(X, r0, r1):
    a0, a1 = int(X.rpt[r0]), int(X.rpt[r1])
    return Csr(r1 - r0, X.cols, (X.rpt[r0:r1 + 1] - a0).astype(np.int64), X.col[a0:a1].copy(), X.val[a0:a1].copy())


def test_errors_are_reported(ctx):
    from paper_2206_06611_b200 import BrmError, TorchCsr
    A = uniform_random(10, 8, 2, seed=1)
    B = uniform_random(9, 8, 2, seed=1)
    with pytest.raises(BrmError) as e:
        ctx.spgemm(TorchCsr.from_csr(A), TorchCsr.from_csr(B), "precise")
    assert e.value.code == 2  # BRM_ERR_DIM
    import torch
    from paper_2206_06611_b200 import Context
    fresh = Context()
    with pytest.raises(BrmError) as e:
        fresh.brmerge_spgemm_fill(10, 8, torch.zeros(11, dtype=torch.int64, device="cuda"), 0)
    assert e.value.code == 6  # BRM_ERR_STATE
    with pytest.raises(BrmError) as e:
        fresh.brm_set_host_pipeline(-1)
    assert e.value.code == 1  # BRM_ERR_INVALID
    fresh.close()


def test_stats_reported(ctx):
    from paper_2206_06611_b200 import TorchCsr
    A = uniform_random(20000, 20000, 8, seed=3)
    ctx.set_timing(True)
    ctx.spgemm(TorchCsr.from_csr(A), TorchCsr.from_csr(A), "precise")
    s = ctx.stats()
    ctx.set_timing(False)
    assert s["nprod_total"] == 20000 * 64 and s["nnz_c"] > 0
    assert sum(s["bin_rows"]) == 20000
    assert s["ms_numeric"] > 0


def _gather_rows(C, rows):
    """Rows of a device CSR (TorchCsr) as a numpy (rpt, col, val) triple."""
    import torch
    r = torch.as_tensor(np.asarray(rows, np.int64), device=C.rpt.device)
    s, e = C.rpt[r], C.rpt[r + 1]
    lens = (e - s)
    rpt = torch.zeros(r.numel() + 1, dtype=torch.int64, device=r.device)
    rpt[1:] = torch.cumsum(lens, 0)
    idx = torch.repeat_interleave(s - rpt[:-1], lens) + torch.arange(int(rpt[-1]), device=r.device)
    return rpt.cpu().numpy(), C.col[idx].cpu().numpy(), C.val[idx].cpu().numpy()


@pytest.mark.parametrize("mode", MODES)
def test_heavy_row_recursive_split(ctx, oracle_mod, mode):
    """A row of 20,000 one-element lists over 50 columns: its 32-list blocks
    go to the shared-memory tiers, and the 625 block results form a heavy row
    again (split a second time); plus a row of 3,000 two-element lists."""
    rng = np.random.default_rng(21)
    kb = 20000
    bcol = rng.integers(0, 50, size=kb).astype(np.int32)
    B = Csr(kb, 60, np.arange(kb + 1, dtype=np.int64), bcol, rng.uniform(-1, 1, size=kb))
    cols = [np.arange(kb, dtype=np.int32), np.sort(rng.choice(kb, size=3000, replace=False)).astype(np.int32)]
    A = Csr(2, kb, np.array([0, kb, kb + 3000], np.int64), np.concatenate(cols),
            rng.uniform(-1, 1, size=kb + 3000))
    compare(run(ctx, A, B, mode), A, B)


@pytest.mark.parametrize("mode", MODES)
def test_host_form_large(ctx, oracle_mod, mode):
    """The host-buffer entry on 70,001 rows: two calls in a row (pinned
    output grown, then reused), C = A*A (single upload) and C = A*B."""
    from paper_2206_06611_b200 import TorchCsr
    A = uniform_random(70001, 70001, 6, seed=31)
    B = random_sparse(70001, 300, 0.01, seed=32)
    Ah = TorchCsr.from_csr(A, pin=True)
    Bh = TorchCsr.from_csr(B, pin=True)
    for pipe in (0, 1 << 26):  # row-blocked pipeline forced, then the one-shot form (small product)
        ctx.brm_set_host_pipeline(pipe)
        for _ in range(2):
            rows, cols, rpt, col, val = ctx.brmerge_spgemm_host(Ah, Ah, mode)
            assert (rows, cols) == (70001, 70001)
            compare((rpt.copy(), col.copy(), val.copy()), A, A)
        rows, cols, rpt, col, val = ctx.brmerge_spgemm_host(Ah, Bh, mode)
        compare((rpt.copy(), col.copy(), val.copy()), A, B)


def test_alg1_pairing_order_hand_derived(ctx):
    """The hand-derived Algorithm-1 trees of test_oracle_pins
    straight against the CUDA path, no oracle in between."""
    from test_oracle_pins import _TREE_CASES, _one_column_row
    for vals, present, tree in _TREE_CASES:
        A, B = _one_column_row(vals, present)
        for mode in MODES:
            rpt, col, val = run(ctx, A, B, mode)
            assert rpt.tolist() == [0, 1] and col.tolist() == [0]
            assert val[0] == tree(vals), (vals, mode, val[0], tree(vals))


@pytest.mark.parametrize("mode", MODES)
def test_heavy_dense_refined_windows(ctx, oracle_mod, mode):
    """Heavy rows whose lists are dense over the same columns: every
    128-column histogram bin holds more products than a window (> 4096), so
    the windows are cut inside bins from per-column counts, in several
    refinement passes (> 64 such bins), with window starts inside refined
    bins; plus a row mixing dense and sparse lists and one of > 1024 lists."""
    rng = np.random.default_rng(41)
    ncols = 40000
    rows_b = []
    for k in range(100):  # 100 dense lists over columns [0, 10000) with a few gaps
        c = np.arange(10000)
        c = c[rng.random(c.size) > 0.02]
        rows_b.append(c)
    for k in range(1100):  # sparse lists over the whole range
        rows_b.append(np.sort(rng.choice(ncols, size=int(rng.integers(0, 60)), replace=False)))
    lens = np.array([r.size for r in rows_b])
    rpt = np.zeros(lens.size + 1, np.int64)
    np.cumsum(lens, out=rpt[1:])
    bcol = np.concatenate(rows_b).astype(np.int32)
    B = Csr(lens.size, ncols, rpt, bcol, rng.uniform(-1, 1, size=bcol.size))
    specs = [np.arange(100), np.concatenate([np.arange(0, 100, 3), np.arange(100, 600)]),
             np.arange(0, 1200)]
    acol = [np.sort(s).astype(np.int32) for s in specs]
    arpt = np.concatenate([[0], np.cumsum([a.size for a in acol])]).astype(np.int64)
    acol = np.concatenate(acol)
    A = Csr(len(specs), B.rows, arpt, acol, rng.uniform(-1, 1, size=acol.size))
    compare(run(ctx, A, B, mode), A, B)


@pytest.mark.parametrize("mode", MODES)
def test_host_form_heavy_rows(ctx, oracle_mod, mode):
    """The host-buffer entry on an R-MAT graph with heavy rows (windowed
    path, one level and 512-list blocks)."""
    from inputs import rmat
    from paper_2206_06611_b200 import TorchCsr
    A = rmat(14, 16, 0.57, 0.19, 0.19, 0.05, seed=12)
    Ah = TorchCsr.from_csr(A, pin=True)
    rows, cols, rpt, col, val = ctx.brmerge_spgemm_host(Ah, Ah, mode)
    assert (rows, cols) == (A.rows, A.cols)
    compare((rpt.copy(), col.copy(), val.copy()), A, A)


@pytest.mark.parametrize("mode", MODES)
def test_host_form_pipelined_heavy_rows(ctx, oracle_mod, mode):
    """The host-buffer entry's row-blocked pipeline (A of >= 65,536 rows: 8
    blocks of balanced n_prod, C copied back per block on a copy stream) on a
    matrix whose heavy rows (one level and 512-list blocks) sit in different
    blocks, plus empty rows; two calls (pinned output grown, then reused)."""
    from paper_2206_06611_b200 import TorchCsr
    rng = np.random.default_rng(77)
    M = 70001
    base = uniform_random(M, M, 3, seed=78)
    heavy = {5: 700, 20000: 300, 45000: 1100, 69999: 520}
    empty = {100, 30000}
    cols, rpt = [], [0]
    for i in range(M):
        if i in empty:
            c = np.zeros(0, np.int32)
        elif i in heavy:
            c = np.sort(rng.choice(M, size=heavy[i], replace=False)).astype(np.int32)
        else:
            c = base.col[base.rpt[i]:base.rpt[i + 1]]
        cols.append(c)
        rpt.append(rpt[-1] + c.size)
    col = np.concatenate(cols)
    A = Csr(M, M, np.array(rpt, np.int64), col, rng.uniform(-1, 1, size=col.size))
    Ah = TorchCsr.from_csr(A, pin=True)
    ctx.brm_set_host_pipeline(0)  # pipeline at any product count
    try:
        for _ in range(2):
            rows, ncols, hrpt, hcol, hval = ctx.brmerge_spgemm_host(Ah, Ah, mode)
            assert (rows, ncols) == (M, M)
            compare((hrpt.copy(), hcol.copy(), hval.copy()), A, A)
    finally:
        ctx.brm_set_host_pipeline(1 << 26)


@pytest.mark.parametrize("route", ["auto", "global"])
@pytest.mark.parametrize("mode", MODES)
def test_mirrors_receive_every_entry(oracle_mod, mode, route):
    """brm_set_mirrors: the fill stores each entry of C at the same index of
    every mirror (here: two more arrays on the same device, pre-filled with
    junk and offset by 5 entries) from every store site -- tiers 1-6, heavy
    rows of one level and of 512-list blocks (or the global tier), and the
    UPPER compaction. C itself still matches the oracle; clearing the mirrors
    stops the extra stores; bad arguments are rejected."""
    import torch
    from paper_2206_06611_b200 import BrmError, Context, TorchCsr
    c = Context()
    try:
        if route == "global":
            c.brm_set_heavy_route(c.HEAVY_GLOBAL)
        # rows of 1..600 lists over B rows of 12 entries: n_prod from 12 to 7200 covers every tier;
        # plus heavy rows (200 / 1000 lists of 100 entries)
        for A, B in (_lists_matrix([1, 2, 3, 8, 20, 21, 60, 64, 200, 250, 400, 512, 600, 0, 5], 12, 5000, seed=21),
                     _lists_matrix([200, 1000, 20], 100, 20000, seed=22)):
            At, Bt = TorchCsr.from_csr(A), TorchCsr.from_csr(B)
            c_rpt, nnz = c.brmerge_spgemm_structure(At, Bt, mode)
            off = 5
            mcol = [torch.full((nnz + off,), -7, dtype=torch.int32, device="cuda") for _ in range(2)]
            mval = [torch.full((nnz + off,), -7.0, dtype=torch.float64, device="cuda") for _ in range(2)]
            c.brm_set_mirrors([t.data_ptr() + 4 * off for t in mcol], [t.data_ptr() + 8 * off for t in mval])
            C = c.brmerge_spgemm_fill(A.rows, B.cols, c_rpt, nnz)
            c.brm_set_mirrors()
            torch.cuda.synchronize()
            compare(C.to_numpy(), A, B)
            for p in range(2):
                assert torch.equal(mcol[p][off:], C.col) and torch.equal(mval[p][off:], C.val), (mode, p)
                assert bool((mcol[p][:off] == -7).all()) and bool((mval[p][:off] == -7.0).all())
            # cleared: a second pair stays untouched
            c_rpt, nnz = c.brmerge_spgemm_structure(At, Bt, mode)
            mcol[0].fill_(-7)
            C2 = c.brmerge_spgemm_fill(A.rows, B.cols, c_rpt, nnz)
            torch.cuda.synchronize()
            assert bool((mcol[0] == -7).all()) and torch.equal(C2.val, C.val)
        t = torch.zeros(4, dtype=torch.int32, device="cuda")
        v = torch.zeros(4, dtype=torch.float64, device="cuda")
        with pytest.raises(BrmError) as e:
            c.brm_set_mirrors([t.data_ptr()] * 8, [v.data_ptr()] * 8)
        assert e.value.code == 1  # BRM_ERR_INVALID: more than 7 mirrors
        with pytest.raises(BrmError) as e:
            c.brm_set_mirrors([0], [v.data_ptr()])
        assert e.value.code == 1  # a null mirror pointer
        c.brm_enable_peer_access(0)  # the context's own device: a no-op
    finally:
        c.close()


def test_fill_into_caller_arrays(ctx, oracle_mod):
    """brmerge_spgemm_fill into caller-owned col/val (a slice of a larger
    array, as PeerAssembly passes); wrong sizes are rejected by the binding."""
    import torch
    from paper_2206_06611_b200 import TorchCsr
    A = uniform_random(3000, 3000, 7, seed=4)
    At = TorchCsr.from_csr(A)
    c_rpt, nnz = ctx.brmerge_spgemm_structure(At, At, "precise")
    col = torch.full((nnz + 9,), -1, dtype=torch.int32, device="cuda")
    val = torch.zeros(nnz + 9, dtype=torch.float64, device="cuda")
    C = ctx.brmerge_spgemm_fill(A.rows, A.cols, c_rpt, nnz, col=col[9:], val=val[9:])
    compare(C.to_numpy(), A, A)
    assert bool((col[:9] == -1).all())
    c_rpt, nnz = ctx.brmerge_spgemm_structure(At, At, "precise")
    with pytest.raises(ValueError):
        ctx.brmerge_spgemm_fill(A.rows, A.cols, c_rpt, nnz, col=col, val=val)


def _fuzz_matrix(seed):
    """A random product drawn from a family of shapes: power-law list counts
    per row of A (so one matrix spreads over many tiers), B rows of mixed
    lengths (empty, short, long) whose columns are clustered (many repeated
    columns per output row) or spread (few), values with exact zeros and
    cancelling pairs mixed in."""
    rng = np.random.default_rng(1000 + seed)
    kb = int(rng.integers(50, 1500))
    ncols = int(rng.choice([64, 700, 5000, 200000, 3_000_000]))
    max_len = int(rng.choice([1, 4, 30, 200, 1500]))
    lens = rng.integers(0, min(max_len, ncols) + 1, size=kb)
    lens[rng.random(kb) < 0.15] = 0
    clustered = rng.random() < 0.5
    cols = []
    for n in lens:
        if clustered:  # columns from a narrow band: heavy duplication across lists
            lo = int(rng.integers(0, max(ncols - 4 * max_len, 1)))
            hi = min(ncols, lo + max(4 * max_len, int(n)))
            cols.append(np.sort(rng.choice(np.arange(lo, hi), size=int(n), replace=False)))
        else:
            cols.append(np.sort(rng.choice(ncols, size=int(n), replace=False)))
    rpt = np.zeros(kb + 1, np.int64)
    np.cumsum(lens, out=rpt[1:])
    bcol = np.concatenate(cols).astype(np.int32) if rpt[-1] else np.zeros(0, np.int32)
    bval = rng.uniform(-1, 1, size=bcol.size)
    bval[rng.random(bcol.size) < 0.05] = 0.0  # stored zeros stay structural entries
    half = rng.random(bcol.size) < 0.2
    bval[half] = np.round(bval[half] * 4) / 4  # coarse values: exact cancellations happen
    B = Csr(kb, ncols, rpt, bcol, bval)
    m = int(rng.integers(1, 400))
    nls = np.minimum((rng.pareto(1.1, size=m) * 3).astype(np.int64), kb)
    nls[rng.random(m) < 0.1] = 0
    arpt = np.zeros(m + 1, np.int64)
    np.cumsum(nls, out=arpt[1:])
    acol = np.concatenate([np.sort(rng.choice(kb, size=int(n), replace=False)) for n in nls]).astype(np.int32) \
        if arpt[-1] else np.zeros(0, np.int32)
    aval = rng.uniform(-1, 1, size=acol.size)
    coarse = rng.random(acol.size) < 0.3
    aval[coarse] = np.round(aval[coarse] * 2) / 2
    return Csr(m, kb, arpt, acol, aval), B


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_shapes(ctx, oracle_mod, seed):
    """Random shapes across the tiers (see _fuzz_matrix), both modes: rpt and
    col bit-exact against Eq. (2), values within the tolerance and
    bit-identical to Algorithm 1."""
    A, B = _fuzz_matrix(seed)
    for mode in MODES:
        compare(run(ctx, A, B, mode), A, B)
