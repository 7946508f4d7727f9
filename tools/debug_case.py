"""Debug aid (GPU): run one test matrix through the C ABI in both modes and
report, per wrong row, its n_prod / num_list / tier and the first wrong
values. Usage: python tools/debug_case.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from bench import tier_of  # noqa: E402
from paper_2206_06611_b200 import Context, TorchCsr  # noqa: E402
from test_gpu_parity import _lists_matrix  # noqa: E402


def check(ctx, A, B, label):
    ref, _ = oracle.spgemm_brmerge(A, B)
    nprod = oracle.row_nprod(A, B)
    nl = np.diff(A.rpt)
    for mode in ("upper", "precise"):
        C = ctx.spgemm(TorchCsr.from_csr(A), TorchCsr.from_csr(B), mode)
        rpt, col, val = C.to_numpy()
        bad = []
        for r in range(A.rows):
            s, e = ref.rpt[r], ref.rpt[r + 1]
            gs, ge = rpt[r], rpt[r + 1]
            if ge - gs != e - s or not np.array_equal(col[gs:ge], ref.col[s:e]) or not np.array_equal(val[gs:ge], ref.val[s:e]):
                bad.append(r)
        print(label, mode, "bad rows", len(bad), "of", A.rows)
        for r in bad[:6]:
            s, e = ref.rpt[r], ref.rpt[r + 1]
            gs = rpt[r]
            gv = val[gs:gs + (e - s)]
            w = np.nonzero(gv != ref.val[s:e])[0]
            print(f"  row {r} nprod {nprod[r]} nl {nl[r]} tier {tier_of(nprod[r:r+1], nl[r:r+1])[0]} nnz {e-s} "
                  f"wrong {w.size} first {w[:8].tolist()} gpu {gv[w[:3]].tolist()} ref {ref.val[s:e][w[:3]].tolist()}")


ctx = Context()
from inputs import random_sparse
for seed in range(6):
    rng = np.random.default_rng(seed)
    m, k, n = (int(x) for x in rng.integers(1, 300, size=3))
    Ar = random_sparse(m, k, float(rng.uniform(0.005, 0.3)), seed=seed)
    Br = random_sparse(k, n, float(rng.uniform(0.005, 0.3)), seed=seed + 99)
    check(ctx, Ar, Br, f"random{seed}")
check(ctx, *_lists_matrix([90, 93, 94], 33, 5000, seed=33), "t5/t6")
check(ctx, *_lists_matrix([90, 93], 33, 5000, seed=33), "t5 only")
check(ctx, *_lists_matrix([94, 100], 33, 5000, seed=33), "t6 only")
check(ctx, *_lists_matrix([100, 112, 113], 64, 20000, seed=64), "t6/t7")
check(ctx, *_lists_matrix([40, 129, 300, 513, 600, 1500], 3, 3000, seed=3), "short lists")
