"""Every-row parity at BASELINE.json's full sizes (north_star: "CSR output
bit-exact in structure and within the stated fp64 tolerance of the oracle on
all five configs"), in the launch configuration bench.py times (PRECISE;
UPPER too where C_bar fits). See tests/fullsize.py for what is compared."""
import numpy as np
import pytest

import bench
import oracle
from fullsize import THREADS, compare_rows, row_sizes_parallel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch
    from paper_2206_06611_b200 import Context
    assert torch.cuda.is_available()
    c = Context()
    yield c
    c.close()


@pytest.mark.parametrize("name", ["uniform2k_k8", "stencil27_64", "uniform1m_k16", "amg_lap2048_agg2x2"])
def test_full_size_every_row(ctx, oracle_mod, name):
    """Every row of configs 0, 1, 2 and 4 in both modes: sizes and columns
    against Eq. (2), values within 1e-12*sum|ab| and bit-identical to Alg. 1."""
    import torch
    from inputs import workload
    from paper_2206_06611_b200 import TorchCsr
    A, B = workload(name)
    nprod = oracle.row_nprod(A, B)
    sizes = row_sizes_parallel(A, B)
    Ad, Bd = TorchCsr.from_csr(A), TorchCsr.from_csr(B)
    for mode in ("precise", "upper"):
        C = ctx.spgemm(Ad, Bd, mode)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(np.diff(C.rpt.cpu().numpy()), sizes)
        res = compare_rows(C, A, B, np.arange(A.rows), nprod)
        assert res["rows"] == A.rows and res["entries"] == C.nnz
        del C
        torch.cuda.empty_cache()


def test_full_size_rmat20(ctx, oracle_mod):
    """configs[3] (rmat20_ef16, PRECISE: C_bar would need 251 GB), every row:
    * C.rpt of all 1,048,576 rows against oracle.row_sizes (Eq. (2) pattern);
    * every row of tiers 1-6 (~800k rows) against Eq. (2) (columns, tolerance)
      and Algorithm 1 (bits);
    * every heavy row (245k rows, 97 % of the products) -- one-level windowed
      rows (<= 512 lists, bench.HV_LISTS) and rows of levels (> 512 lists) -- against
      Algorithm 1's oracle: columns exact, values bit-identical;
    * the Eq. (2) tolerance on heavy rows for the 16 heaviest one-level rows,
      16 two-level rows spread over their list counts, and 256 random heavy
      rows (the sorted-map oracle runs at ~2 M products/s on these rows)."""
    import torch
    from inputs import workload
    from paper_2206_06611_b200 import TorchCsr
    A, B = workload("rmat20_ef16")
    nprod = oracle.row_nprod(A, B)
    nl = np.diff(A.rpt)
    tiers = bench.tier_of(nprod, nl)
    sizes = row_sizes_parallel(A, B)
    C = ctx.spgemm(TorchCsr.from_csr(A), TorchCsr.from_csr(B), "precise")
    torch.cuda.synchronize()
    np.testing.assert_array_equal(np.diff(C.rpt.cpu().numpy()), sizes)
    light = np.nonzero((tiers >= 1) & (tiers <= 6))[0]
    heavy = np.nonzero(tiers == 7)[0]
    one = heavy[nl[heavy] <= bench.HV_LISTS]
    two = heavy[nl[heavy] > bench.HV_LISTS]
    assert one.size > 100_000 and two.size > 1000  # both heavy routes are exercised
    res = compare_rows(C, A, B, light, nprod)
    assert res["rows"] == light.size
    res = compare_rows(C, A, B, heavy, nprod, gust=False, tree=True)
    assert res["rows"] == heavy.size
    rng = np.random.default_rng(7)
    top_one = one[np.argsort(-nprod[one])[:16]]
    two_sorted = two[np.argsort(nl[two])]
    spread_two = two_sorted[np.linspace(0, two.size - 1, 16).astype(np.int64)]
    rand = rng.choice(heavy, 256, replace=False)
    sub = np.unique(np.concatenate([top_one, spread_two, rand]))
    res = compare_rows(C, A, B, sub, nprod, gust=True, tree=False)
    assert res["rows"] == sub.size and res["max_rel"] <= 1e-12
