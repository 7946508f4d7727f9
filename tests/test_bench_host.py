"""Host-side logic of bench.py (CPU): the tier table mirrors the kernels',
the algorithmic-byte count matches a brute-force count,
and the weak-scaling stencil box reduces to the configs[1] generator."""
import re
from pathlib import Path

import numpy as np

import bench
from inputs import random_sparse, stencil27, uniform_random

ROOT = Path(__file__).resolve().parents[1]


def test_tier_table_matches_kernels():
    src = (ROOT / "paper_2206_06611_b200" / "csrc" / "brm_internal.cuh").read_text()
    macros = {m: int(v) for m, v in re.findall(r"#define (BRM_T\d_ROUTE) (\d+)", src)}  # routing caps' defaults
    caps = {int(t): (int(macros.get(c, c)), int(l)) for t, c, l in
            re.findall(r"t\.cap\[(\d)\] = (\w+);\s+t\.lcap\[\d\] = (\d+);", src)}
    for t in range(1, bench.NUM_BINS - 1):
        assert caps[t] == (bench.TIER_CAP[t], bench.TIER_LCAP[t]), t
        m = re.search(rf"#define BRM_TIER{t} (\w+), (\d+), (\d+), (\w+)", src)
        assert int(m.group(2)) == bench.TIER_CAP[t] and int(m.group(3)) == bench.TIER_LCAP[t]
    assert f"#define BRM_NUM_BINS {bench.NUM_BINS}" in (ROOT / "include" / "brmerge.h").read_text()
    hv = (ROOT / "paper_2206_06611_b200" / "csrc" / "heavy.cuh").read_text()
    assert f"#define BRM_HV_LISTS {bench.HV_LISTS}" in hv  # one-level heavy rows (roofline rows)


def test_algorithmic_bytes_brute_force():
    A = random_sparse(40, 30, 0.1, seed=1)
    B = random_sparse(30, 25, 0.2, seed=2)
    rows = np.array([0, 3, 7, 8, 39])
    nnz_c = 17
    touched = set()
    a_bytes = 0
    for r in rows:
        a_bytes += 16 + 12 * int(A.rpt[r + 1] - A.rpt[r])
        touched.update(int(k) for k in A.col[A.rpt[r]:A.rpt[r + 1]])
    b_bytes = sum(16 + 12 * int(B.rpt[k + 1] - B.rpt[k]) for k in touched)
    c_bytes = 12 * nnz_c + 8 * rows.size
    assert bench.algorithmic_bytes(A, B, rows, nnz_c) == a_bytes + b_bytes + c_bytes
    big = np.arange(A.rows)
    assert bench.algorithmic_bytes(A, B, big, 0) > 0


def test_tier_of_matches_bounds():
    nprod = np.array([0, 1, 8, 9, 32, 33, 256, 257, 768, 769, 3072, 3073, 6656, 6657, 10, 40, 600, 300])
    nl = np.array([0, 1, 8, 1, 32, 1, 64, 1, 64, 1, 256, 1, 512, 1, 9, 65, 513, 257])
    assert bench.tier_of(nprod, nl).tolist() == [0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 2, 5, 7, 6]


def test_stencil_box_equals_cube():
    a = bench.stencil27_box(6, 6, 6, seed=1)
    b = stencil27(6, seed=1)
    np.testing.assert_array_equal(a.rpt, b.rpt)
    np.testing.assert_array_equal(a.col, b.col)
    np.testing.assert_array_equal(a.val, b.val)


def test_sample_rows_bounded():
    nprod = np.full(1000, 10, np.int64)
    rows, desc = bench._sample_rows(nprod, 2000)
    assert 150 <= rows.size <= 200 and "of 1000 rows" in desc
    A = uniform_random(10, 10, 2, seed=1)
    assert bench.build_workload("uniform2k_k8", 1)[0].rows == 2000
    assert A.rows == 10
