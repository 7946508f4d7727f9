"""Seeded CSR generators for the five BASELINE.json workloads and for tests.

Every generator is deterministic in its arguments (numpy PCG64 seeded with
`seed`). Layout (the one the C-ABI consumes, include/brmerge.h):
  rpt : int64[rows+1], col : int32[nnz] strictly increasing per row,
  val : float64[nnz].
Recipes (also stated in DESIGN.md "Input recipe"):
  configs[0] uniform_random(2000, 2000, 8, seed=1)
  configs[1] stencil27(64)            -- 27-point stencil, 26 / -1 + U[-0.01,0.01]
  configs[2] uniform_random(2**20, 2**20, 16)
  configs[3] rmat(20, 16, .57, .19, .19, .05) duplicates removed, val U[0,1]
  configs[4] laplace2d_5pt(2048) x aggregation_prolongator(2048)
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Csr:
    rows: int
    cols: int
    rpt: np.ndarray  # int64[rows+1]
    col: np.ndarray  # int32[nnz]
    val: np.ndarray  # float64[nnz]

    @property
    def nnz(self) -> int:
        return int(self.rpt[-1])

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.rows, self.cols), dtype=np.float64)
        r = np.repeat(np.arange(self.rows), np.diff(self.rpt))
        d[r, self.col] = self.val
        return d

    def validate(self) -> None:
        assert self.rpt.dtype == np.int64 and self.col.dtype == np.int32
        assert self.val.dtype == np.float64
        assert self.rpt.shape == (self.rows + 1,) and self.rpt[0] == 0
        assert np.all(np.diff(self.rpt) >= 0)
        assert self.col.shape == (self.nnz,) and self.val.shape == (self.nnz,)
        if self.nnz:
            assert self.col.min() >= 0 and self.col.max() < self.cols
            d = np.diff(self.col.astype(np.int64))
            starts = np.zeros(self.nnz, dtype=bool)
            starts[self.rpt[:-1][np.diff(self.rpt) > 0]] = True
            assert np.all((d > 0) | starts[1:]), "columns not strictly increasing"


def sorted_unique(x: np.ndarray) -> np.ndarray:
    """np.unique(x) for a 1-D array (sort, then drop repeats): the same result,
    ~100x faster than numpy 2.3's np.unique on 16M int64 keys."""
    s = np.sort(x)
    if s.size == 0:
        return s
    return s[np.concatenate([[True], s[1:] != s[:-1]])]


def _from_sorted_keys(rows: int, cols: int, r: np.ndarray, c: np.ndarray,
                      v: np.ndarray) -> Csr:
    """Build CSR from (row, col) already sorted row-major and unique."""
    rpt = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=rows), out=rpt[1:])
    return Csr(rows, cols, rpt, c.astype(np.int32), v.astype(np.float64))


def _from_rows(rows: int, cols: int, colmat: np.ndarray, valmat: np.ndarray) -> Csr:
    """Equal-length rows given as 2-D arrays (each row sorted, distinct)."""
    k = colmat.shape[1] if colmat.ndim == 2 else 0
    rpt = np.arange(rows + 1, dtype=np.int64) * k
    return Csr(rows, cols, rpt, colmat.reshape(-1).astype(np.int32),
               valmat.reshape(-1).astype(np.float64))


def uniform_random(rows: int, cols: int, per_row: int, seed: int = 1,
                   lo: float = -1.0, hi: float = 1.0) -> Csr:
    """Each row has exactly `per_row` distinct uniformly random columns."""
    rng = np.random.default_rng(seed)
    c = np.sort(rng.integers(0, cols, size=(rows, per_row), dtype=np.int64), axis=1)
    while True:
        bad = np.nonzero(np.any(np.diff(c, axis=1) == 0, axis=1))[0]
        if bad.size == 0:
            break
        c[bad] = np.sort(rng.integers(0, cols, size=(bad.size, per_row),
                                      dtype=np.int64), axis=1)
    v = rng.uniform(lo, hi, size=(rows, per_row))
    return _from_rows(rows, cols, c, v)


def random_sparse(rows: int, cols: int, density: float, seed: int,
                  lo: float = -1.0, hi: float = 1.0, integer_values: bool = False) -> Csr:
    """Bernoulli(density) pattern; optional small-integer values (exact sums)."""
    rng = np.random.default_rng(seed)
    mask = rng.random((rows, cols)) < density
    r, c = np.nonzero(mask)
    if integer_values:
        v = rng.integers(-4, 5, size=r.size).astype(np.float64)
    else:
        v = rng.uniform(lo, hi, size=r.size)
    return _from_sorted_keys(rows, cols, r, c, v)


def stencil27(n: int, seed: int = 1, noise: float = 0.01) -> Csr:
    """3-D 27-point stencil on an n^3 grid, row id = (z*n + y)*n + x.

    Values: 26 on the diagonal, -1 off it, plus U[-noise, noise] on every entry.
    """
    rng = np.random.default_rng(seed)
    N = n * n * n
    idx = np.arange(N, dtype=np.int64)
    x, y, z = idx % n, (idx // n) % n, idx // (n * n)
    cols_list, diag_list = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                ok = ((x + dx >= 0) & (x + dx < n) & (y + dy >= 0) & (y + dy < n)
                      & (z + dz >= 0) & (z + dz < n))
                cols_list.append(np.where(ok, idx + (dz * n + dy) * n + dx, -1))
                diag_list.append(dx == 0 and dy == 0 and dz == 0)
    cm = np.stack(cols_list, axis=1)  # (N, 27), ascending where valid
    valid = cm >= 0
    base = np.where(np.array(diag_list)[None, :], 26.0, -1.0)
    vm = np.broadcast_to(base, cm.shape).copy()
    if noise:
        vm += rng.uniform(-noise, noise, size=cm.shape)
    rpt = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(valid.sum(axis=1), out=rpt[1:])
    return Csr(N, N, rpt, cm[valid].astype(np.int32), vm[valid])


def rmat(scale: int, edge_factor: int, a: float, b: float, c: float, d: float,
         seed: int = 1) -> Csr:
    """R-MAT graph (Chakrabarti et al. recursive quadrant choice), duplicates
    removed, values U[0,1]. Quadrant probabilities are applied with exact
    integer thresholds on a 0..9999 draw (params are multiples of 1e-4)."""
    assert abs(a + b + c + d - 1.0) < 1e-9
    rng = np.random.default_rng(seed)
    n = 1 << scale
    m = edge_factor * n
    ta, tb, tc = round(a * 10000), round((a + b) * 10000), round((a + b + c) * 10000)
    r = np.zeros(m, dtype=np.int64)
    cc = np.zeros(m, dtype=np.int64)
    for lvl in range(scale):
        u = rng.integers(0, 10000, size=m, dtype=np.int16)
        bit_c = ((u >= ta) & (u < tb)) | (u >= tc)
        bit_r = u >= tb
        r |= bit_r.astype(np.int64) << lvl
        cc |= bit_c.astype(np.int64) << lvl
    key = sorted_unique(r * n + cc)
    del r, cc
    rr, c2 = key // n, key % n
    v = rng.random(key.size)
    return _from_sorted_keys(n, n, rr, c2, v)


def laplace2d_5pt(n: int) -> Csr:
    """2-D 5-point Laplacian on an n x n grid: 4 on the diagonal, -1 to the
    (up to four) in-grid neighbours. Row id = y*n + x."""
    N = n * n
    idx = np.arange(N, dtype=np.int64)
    x, y = idx % n, idx // n
    offs = [(-n, y > 0), (-1, x > 0), (0, np.ones(N, bool)), (1, x < n - 1), (n, y < n - 1)]
    cm = np.stack([np.where(ok, idx + o, -1) for o, ok in offs], axis=1)
    vm = np.where(np.arange(5)[None, :] == 2, 4.0, -1.0) * np.ones((N, 1))
    valid = cm >= 0
    rpt = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(valid.sum(axis=1), out=rpt[1:])
    return Csr(N, N, rpt, cm[valid].astype(np.int32), vm[valid])


def aggregation_prolongator(n: int, seed: int = 1, perturb: float = 0.1) -> Csr:
    """n^2 x (n/2)^2 tentative prolongator of 2x2 block aggregation: fine node
    (x, y) -> aggregate (x//2, y//2), one nonzero 1 + U[-perturb, perturb]."""
    assert n % 2 == 0
    rng = np.random.default_rng(seed)
    N = n * n
    h = n // 2
    idx = np.arange(N, dtype=np.int64)
    x, y = idx % n, idx // n
    col = (y // 2) * h + (x // 2)
    v = 1.0 + rng.uniform(-perturb, perturb, size=N)
    return Csr(N, h * h, np.arange(N + 1, dtype=np.int64), col.astype(np.int32), v)


def identity(n: int) -> Csr:
    return Csr(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32),
               np.ones(n))


def permutation(n: int, seed: int) -> tuple[Csr, np.ndarray]:
    """Permutation matrix P with P[i, perm[i]] = 1 (so (P X)[i] = X[perm[i]])."""
    perm = np.random.default_rng(seed).permutation(n)
    return Csr(n, n, np.arange(n + 1, dtype=np.int64), perm.astype(np.int32),
               np.ones(n)), perm


# name -> (description, builder returning (A, B))
def _w0():
    A = uniform_random(2000, 2000, 8, seed=1)
    return A, A


def _w1():
    A = stencil27(64, seed=1)
    return A, A


def _w2():
    A = uniform_random(1 << 20, 1 << 20, 16, seed=1)
    return A, A


def _w3():
    A = rmat(20, 16, 0.57, 0.19, 0.19, 0.05, seed=1)
    return A, A


def _w4():
    return laplace2d_5pt(2048), aggregation_prolongator(2048, seed=1)


WORKLOADS = {
    "uniform2k_k8": ("configs[0]: C=A*A, 2000x2000, 8 nnz/row uniform, U[-1,1], seed 1", _w0),
    "stencil27_64": ("configs[1]: C=A*A, 27-point stencil on 64^3 (262,144 rows)", _w1),
    "uniform1m_k16": ("configs[2]: C=A*A, 2^20 x 2^20 uniform, 16 nnz/row, U[-1,1]", _w2),
    "rmat20_ef16": ("configs[3]: C=A*A, R-MAT scale 20, ef 16, (.57,.19,.19,.05), dedup, U[0,1]", _w3),
    "amg_lap2048_agg2x2": ("configs[4]: C=A*P, 5-pt Laplacian 2048^2 x 2x2 aggregation", _w4),
}


def workload(name: str) -> tuple[Csr, Csr]:
    return WORKLOADS[name][1]()
