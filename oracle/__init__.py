"""CPU oracle for the BRMerge SpGEMM hot path (ctypes wrapper of oracle.cpp).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this package. The product
path (paper_2206_06611_b200/) never imports it and shares no code with it.

Functions and the PAPER.md passage each follows:
  row_nprod          §II.B.2, Alg. 1 line 1
  row_sizes          Eq. (2)'s pattern: distinct columns per row
  spgemm_gustavson   Eq. (2), sorted-map accumulator
  spgemm_brmerge     Algorithm 1, literal, tree order
  brmerge_trace      Alg. 1 accumulating phase, live totals per round
  merge_two          Fig. 2 caption
  balance_by_nprod   §III.D load balance
  compression_ratio  Eq. (5)
All pinned by tests/test_oracle_pins.py (no function is "parity unpinned").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "build" / "liboracle.so"
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> Path:
    """Compile oracle.cpp with g++ (no CUDA, -ffp-contract=off)."""
    src = _HERE / "oracle.cpp"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        _LIB_PATH.parent.mkdir(parents=True, exist_ok=True)
        tmp = _LIB_PATH.with_suffix(f".{os.getpid()}.tmp")
        subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-std=c++17", "-shared", "-fPIC", str(src), "-o", str(tmp)])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(str(build()))
        lib.oracle_row_nprod.restype = ctypes.c_int64
        lib.oracle_row_nprod.argtypes = [ctypes.c_int64, _i64p, _i32p, _i64p, _i64p]
        for name in ("oracle_gustavson", "oracle_brmerge"):
            f = getattr(lib, name)
            f.restype = ctypes.c_void_p
            f.argtypes = [ctypes.c_int64, _i64p, _i32p, _f64p, _i64p, _i32p, _f64p,
                          _i64p, ctypes.c_int64]
        lib.oracle_row_sizes.restype = None
        lib.oracle_row_sizes.argtypes = [ctypes.c_int64, _i64p, _i32p, _i64p, _i32p, ctypes.c_int64,
                                         _i64p, ctypes.c_int64, _i64p]
        lib.oracle_brmerge_trace.restype = ctypes.c_int64
        lib.oracle_brmerge_trace.argtypes = [_i64p, _i32p, _f64p, _i64p, _i32p, _f64p,
                                             ctypes.c_int64, _i64p, ctypes.c_int64]
        lib.oracle_merge_two.restype = ctypes.c_int64
        lib.oracle_merge_two.argtypes = [ctypes.c_int64, _i32p, _f64p, ctypes.c_int64,
                                         _i32p, _f64p, _i32p, _f64p]
        lib.oracle_result_nnz.restype = ctypes.c_int64
        lib.oracle_result_nnz.argtypes = [ctypes.c_void_p]
        lib.oracle_result_rows.restype = ctypes.c_int64
        lib.oracle_result_rows.argtypes = [ctypes.c_void_p]
        lib.oracle_result_copy.restype = None
        lib.oracle_result_copy.argtypes = [ctypes.c_void_p, _i64p, _i32p, _f64p, _i32p]
        lib.oracle_result_free.restype = None
        lib.oracle_result_free.argtypes = [ctypes.c_void_p]
        _lib = lib
    return _lib


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _check(A, B):
    from inputs import Csr  # generators only; no method arithmetic
    assert isinstance(A, Csr) and isinstance(B, Csr)
    if A.cols != B.rows:
        raise ValueError(f"dimension mismatch: A is {A.rows}x{A.cols}, B is {B.rows}x{B.cols}")


def row_nprod(A, B) -> np.ndarray:
    """n_prod per output row (§II.B.2): sum over k in A_i* of nnz(B_k*)."""
    _check(A, B)
    out = np.zeros(A.rows, dtype=np.int64)
    _load().oracle_row_nprod(A.rows, _p(A.rpt, ctypes.c_int64), _p(A.col, ctypes.c_int32),
                             _p(B.rpt, ctypes.c_int64), _p(out, ctypes.c_int64))
    return out


def row_sizes(A, B, rows=None) -> np.ndarray:
    """nnz of each output row (all rows, or `rows` in that order): the number
    of distinct columns over the row's intermediate products -- Eq. (2)'s
    pattern, structural zeros kept (R3). A set-membership count, no values."""
    _check(A, B)
    if rows is not None:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        rp, nr, n = _p(rows, ctypes.c_int64), rows.size, rows.size
    else:
        rp, nr, n = None, 0, A.rows
    out = np.zeros(n, np.int64)
    _load().oracle_row_sizes(A.rows, _p(A.rpt, ctypes.c_int64), _p(A.col, ctypes.c_int32),
                             _p(B.rpt, ctypes.c_int64), _p(B.col, ctypes.c_int32), B.cols,
                             rp, nr, _p(out, ctypes.c_int64))
    return out


def _run(fn, A, B, rows):
    from inputs import Csr
    _check(A, B)
    lib = _load()
    if rows is not None:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        rp, nr = _p(rows, ctypes.c_int64), rows.size
    else:
        rp, nr = None, 0
    h = fn(A.rows, _p(A.rpt, ctypes.c_int64), _p(A.col, ctypes.c_int32), _p(A.val, ctypes.c_double),
           _p(B.rpt, ctypes.c_int64), _p(B.col, ctypes.c_int32), _p(B.val, ctypes.c_double), rp, nr)
    try:
        n = lib.oracle_result_rows(h)
        nnz = lib.oracle_result_nnz(h)
        rpt = np.zeros(n + 1, np.int64)
        col = np.zeros(nnz, np.int32)
        val = np.zeros(nnz, np.float64)
        rounds = np.zeros(n, np.int32)
        lib.oracle_result_copy(h, _p(rpt, ctypes.c_int64), _p(col, ctypes.c_int32),
                               _p(val, ctypes.c_double), _p(rounds, ctypes.c_int32))
    finally:
        lib.oracle_result_free(h)
    return Csr(n, B.cols, rpt, col, val), rounds


def spgemm_gustavson(A, B, rows=None):
    """C = A*B by Eq. (2) with a sorted-map accumulator (rows subset optional:
    the result then has len(rows) rows, in the given order)."""
    return _run(_load().oracle_gustavson, A, B, rows)[0]


def spgemm_brmerge(A, B, rows=None):
    """C = A*B by Algorithm 1 literally; returns (C, rounds_per_row)."""
    return _run(_load().oracle_brmerge, A, B, rows)


def brmerge_trace(A, B, row: int) -> np.ndarray:
    """Live element totals: after the multiplying phase, then after each round."""
    _check(A, B)
    cap = 64
    out = np.zeros(cap, np.int64)
    n = _load().oracle_brmerge_trace(_p(A.rpt, ctypes.c_int64), _p(A.col, ctypes.c_int32),
                                     _p(A.val, ctypes.c_double), _p(B.rpt, ctypes.c_int64),
                                     _p(B.col, ctypes.c_int32), _p(B.val, ctypes.c_double),
                                     row, _p(out, ctypes.c_int64), cap)
    return out[:n].copy()


def merge_two(ac, av, bc, bv):
    """Fig. 2: merge two column-sorted lists, combining duplicate columns."""
    ac = np.ascontiguousarray(ac, np.int32); av = np.ascontiguousarray(av, np.float64)
    bc = np.ascontiguousarray(bc, np.int32); bv = np.ascontiguousarray(bv, np.float64)
    oc = np.zeros(ac.size + bc.size, np.int32)
    ov = np.zeros(ac.size + bc.size, np.float64)
    n = _load().oracle_merge_two(ac.size, _p(ac, ctypes.c_int32), _p(av, ctypes.c_double),
                                 bc.size, _p(bc, ctypes.c_int32), _p(bv, ctypes.c_double),
                                 _p(oc, ctypes.c_int32), _p(ov, ctypes.c_double))
    return oc[:n], ov[:n]


def balance_by_nprod(nprod, p: int) -> list[int]:
    """§III.D: rows split into p contiguous groups "to keep the
    same total n_prod in each group". Group g starts at the first row whose
    exclusive running n_prod sum reaches g*total/p (exact integer test
    prefix*p >= g*total); bounds[0] = 0, bounds[p] = M. Plain Python loop."""
    M = len(nprod)
    total = int(sum(int(x) for x in nprod))
    bounds = [0] * (p + 1)
    bounds[p] = M
    g = 1
    prefix = 0
    for i in range(M + 1):
        while g < p and prefix * p >= g * total:
            bounds[g] = i
            g += 1
        if i < M:
            prefix += int(nprod[i])
    while g < p:
        bounds[g] = M
        g += 1
    return bounds


def compression_ratio(nprod_total: int, nnz_c: int) -> float:
    """Eq. (5): total n_prod over total n_nz of C."""
    if nnz_c == 0:
        raise ZeroDivisionError("compression ratio undefined for nnz(C) = 0")
    return nprod_total / nnz_c
