"""Every-row parity at BASELINE.json's full sizes (tests only).

The oracle runs single-threaded per call (ctypes releases the GIL), over row
blocks on a thread pool; the GPU's rows are fetched from the device block by
block so host memory stays bounded.

Checks per row (north_star): row sizes and columns bit-exact against Eq. (2)
(oracle.spgemm_gustavson, or oracle.row_sizes for the sizes), values within
1e-12 * sum|a_ik b_kj| of the Gustavson sum, and values bit-identical to
Algorithm 1 (oracle.spgemm_brmerge). Where the Gustavson map oracle is too
slow (rmat20's heavy rows, ~2 M products/s), those rows are compared with
Algorithm 1's oracle (columns exact, values bit-identical) and the Gustavson
tolerance is checked on a stated subset.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

import oracle
from inputs import Csr
from parity import abs_csr

THREADS = max(1, min(32, os.cpu_count() or 1))


def gather_rows(C, rows: np.ndarray):
    """Rows (sorted or not) of a device CSR (TorchCsr) as numpy (rpt, col, val)."""
    import torch
    r = torch.as_tensor(np.asarray(rows, np.int64), device=C.rpt.device)
    s, e = C.rpt[r], C.rpt[r + 1]
    lens = e - s
    rpt = torch.zeros(r.numel() + 1, dtype=torch.int64, device=r.device)
    rpt[1:] = torch.cumsum(lens, 0)
    n = int(rpt[-1])
    idx = torch.repeat_interleave(s - rpt[:-1], lens, output_size=n) + torch.arange(n, device=r.device)
    return rpt.cpu().numpy(), C.col[idx].cpu().numpy(), C.val[idx].cpu().numpy()


def _split_by_weight(rows: np.ndarray, w: np.ndarray, parts: int):
    """Contiguous pieces of `rows` with about equal total weight."""
    if rows.size == 0:
        return []
    cw = np.cumsum(w.astype(np.float64))
    cuts = np.searchsorted(cw, np.linspace(0, cw[-1], parts + 1)[1:-1], side="right")
    return [p for p in np.split(rows, cuts) if p.size]


def _check_piece(A: Csr, B: Csr, rows, g_rpt, g_col, g_val, gust: bool, tree: bool, nonneg: bool, tol: float):
    """One block of rows: returns (n_rows, n_entries, max_rel) or raises."""
    if gust:
        ref = oracle.spgemm_gustavson(A, B, rows=rows)
        np.testing.assert_array_equal(g_rpt, ref.rpt, err_msg="row pointers differ from Eq. (2)")
        np.testing.assert_array_equal(g_col, ref.col, err_msg="columns differ from Eq. (2)")
        bound = ref.val if nonneg else oracle.spgemm_gustavson(abs_csr(A), abs_csr(B), rows=rows).val
        err = np.abs(g_val - ref.val)
        bad = err > tol * np.abs(bound)
        assert not bad.any(), f"{int(bad.sum())} values outside {tol}*sum|ab|"
        max_rel = float((err / np.maximum(np.abs(bound), 1e-300)).max()) if err.size else 0.0
    else:
        max_rel = float("nan")
    if tree:
        t, _ = oracle.spgemm_brmerge(A, B, rows=rows)
        np.testing.assert_array_equal(g_rpt, t.rpt, err_msg="row pointers differ from Alg. 1")
        np.testing.assert_array_equal(g_col, t.col, err_msg="columns differ from Alg. 1")
        np.testing.assert_array_equal(g_val, t.val, err_msg="values differ from Alg. 1 tree order")
    return len(rows), int(g_rpt[-1]), max_rel


def compare_rows(C, A: Csr, B: Csr, rows: np.ndarray, nprod: np.ndarray, *, gust=True, tree=True,
                 chunk_entries=40_000_000, tol=1e-12) -> dict:
    """Compare the GPU rows `rows` of device CSR C with the oracle, every row.
    Rows are taken in chunks of about `chunk_entries` output entries; each
    chunk is split over the thread pool by n_prod."""
    rows = np.asarray(rows, np.int64)
    if rows.size == 0:
        return {"rows": 0, "entries": 0}
    nonneg = bool((A.val >= 0).all() and (B.val >= 0).all())  # then sum|ab| = sum ab
    crpt = C.rpt.cpu().numpy()
    cs = np.concatenate([[0], np.cumsum(crpt[rows + 1] - crpt[rows])])
    starts = [0]
    while starts[-1] < rows.size:  # chunks of about chunk_entries output entries (at least one row)
        nxt = int(np.searchsorted(cs, cs[starts[-1]] + chunk_entries, side="right")) - 1
        starts.append(min(rows.size, max(nxt, starts[-1] + 1)))
    out_rows = out_entries = 0
    max_rel = 0.0
    with ThreadPoolExecutor(THREADS) as ex:
        for c0, c1 in zip(starts[:-1], starts[1:]):
            chunk = rows[c0:c1]
            g_rpt, g_col, g_val = gather_rows(C, chunk)
            pieces = _split_by_weight(np.arange(chunk.size), nprod[chunk] + 1, THREADS * 4)
            futs = []
            for p in pieces:
                a, b = int(p[0]), int(p[-1]) + 1
                e0, e1 = int(g_rpt[a]), int(g_rpt[b])
                futs.append(ex.submit(_check_piece, A, B, chunk[a:b], g_rpt[a:b + 1] - e0, g_col[e0:e1],
                                      g_val[e0:e1], gust, tree, nonneg, tol))
            for f in futs:
                n, e, m = f.result()
                out_rows += n
                out_entries += e
                if m == m:
                    max_rel = max(max_rel, m)
    return {"rows": out_rows, "entries": out_entries, "max_rel": max_rel}


def row_sizes_parallel(A: Csr, B: Csr) -> np.ndarray:
    """oracle.row_sizes of every row, over row blocks on the thread pool."""
    nprod = oracle.row_nprod(A, B)
    parts = _split_by_weight(np.arange(A.rows, dtype=np.int64), nprod + 1, THREADS * 4)
    with ThreadPoolExecutor(THREADS) as ex:
        res = list(ex.map(lambda p: oracle.row_sizes(A, B, rows=p), parts))
    return np.concatenate(res) if res else np.zeros(0, np.int64)
