"""Helpers comparing the CUDA path's output with the oracle (tests only)."""
from __future__ import annotations

import numpy as np

import oracle
from inputs import Csr


def abs_csr(X: Csr) -> Csr:
    return Csr(X.rows, X.cols, X.rpt, X.col, np.abs(X.val))


def rows_of(rpt, col, val, rows):
    """Extract the given rows of a CSR (numpy) as a compact CSR triple."""
    rows = np.asarray(rows, dtype=np.int64)
    lens = rpt[rows + 1] - rpt[rows]
    out_rpt = np.zeros(rows.size + 1, np.int64)
    np.cumsum(lens, out=out_rpt[1:])
    idx = np.concatenate([np.arange(rpt[r], rpt[r + 1]) for r in rows]) if rows.size else np.zeros(0, np.int64)
    return out_rpt, col[idx], val[idx]


def compare(gpu, A: Csr, B: Csr, rows=None, tree_exact: bool = True, tol: float = 1e-12):
    """gpu = (rpt, col, val) numpy arrays of the GPU result (all rows, or
    only `rows` in that order when rows is given).

    Checks (north_star): rpt and col bit-exact against Eq. (2) (Gustavson,
    structural zeros kept); |c - c_ref| <= tol * sum|a_ik b_kj| per entry;
    and, when tree_exact, values bit-identical to Algorithm 1's tree order.
    Returns a dict of diagnostics."""
    rpt, col, val = gpu
    n = A.rows if rows is None else len(rows)
    if rows is not None and rpt.shape == (A.rows + 1,) and A.rows != len(rows):
        rpt, col, val = rows_of(rpt, col, val, rows)  # full result given: cut the rows
    assert rpt.shape == (n + 1,), rpt.shape
    assert rpt[0] == 0 and np.all(np.diff(rpt) >= 0)
    assert col.shape == val.shape == (int(rpt[-1]),)
    g_rpt, g_col, g_val = rpt, col, val
    ref = oracle.spgemm_gustavson(A, B, rows=rows)
    np.testing.assert_array_equal(g_rpt, ref.rpt, err_msg="row pointers differ")
    np.testing.assert_array_equal(g_col, ref.col, err_msg="column indices differ")
    bound = oracle.spgemm_gustavson(abs_csr(A), abs_csr(B), rows=rows).val
    err = np.abs(g_val - ref.val)
    bad = err > tol * bound
    assert not bad.any(), f"{bad.sum()} values outside {tol}*sum|ab|; max err {err.max()}"
    out = {"nnz": int(g_rpt[-1]), "max_rel": float((err / np.maximum(bound, 1e-300)).max()) if err.size else 0.0}
    if tree_exact:
        tree, _ = oracle.spgemm_brmerge(A, B, rows=rows)
        np.testing.assert_array_equal(g_val, tree.val, err_msg="values differ from Alg. 1 tree order")
    return out
