"""Seeded generators: valid CSR, deterministic, and the stated shapes."""
import numpy as np

from inputs import (aggregation_prolongator, laplace2d_5pt, rmat, stencil27, uniform_random,
                    random_sparse)


def test_uniform_random_exact_row_counts_and_determinism():
    A = uniform_random(2000, 2000, 8, seed=1)
    A.validate()
    assert np.all(np.diff(A.rpt) == 8)
    assert A.val.min() >= -1 and A.val.max() <= 1
    B = uniform_random(2000, 2000, 8, seed=1)
    np.testing.assert_array_equal(A.col, B.col)
    np.testing.assert_array_equal(A.val, B.val)


def test_stencil27_counts():
    n = 9
    A = stencil27(n, seed=1)
    A.validate()
    # per-dimension neighbour counts 2 (boundary) or 3 -> nnz = (3n-2)^3
    assert A.nnz == (3 * n - 2) ** 3
    diag = A.val[[np.searchsorted(A.col[A.rpt[i]:A.rpt[i + 1]], i) + A.rpt[i] for i in range(n ** 3)]]
    assert np.all(np.abs(diag - 26) <= 0.01)


def test_stencil27_full_size_nnz():
    A = stencil27(64, seed=1)
    assert A.rows == 262144 and A.nnz == 190 ** 3  # ~6.9M


def test_rmat_small():
    A = rmat(10, 16, 0.57, 0.19, 0.19, 0.05, seed=1)
    A.validate()
    assert A.rows == 1024 and 0 < A.nnz <= 16 * 1024
    assert A.val.min() >= 0 and A.val.max() <= 1
    deg = np.diff(A.rpt)
    assert deg.max() > 8 * deg.mean()  # skewed


def test_laplace_and_aggregation():
    L = laplace2d_5pt(16)
    L.validate()
    assert L.nnz == 5 * 256 - 4 * 16
    P = aggregation_prolongator(16, seed=1)
    P.validate()
    assert P.rows == 256 and P.cols == 64 and P.nnz == 256
    assert np.all(np.abs(P.val - 1) <= 0.1)


def test_random_sparse_valid():
    random_sparse(50, 60, 0.2, seed=3).validate()
