"""Pins of the CPU oracle against things other than itself (③):
dense matmul, identity / permutation invariants, closed forms, exact-integer
agreement of two summation orders, the paper's Fig. 2 round count and the
paper's printed Table 2 compression ratios. CPU only."""
import math
import os

import numpy as np
import pytest

from inputs import (Csr, aggregation_prolongator, identity, laplace2d_5pt, permutation,
                    random_sparse, stencil27, uniform_random)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _pattern(X: Csr) -> np.ndarray:
    d = np.zeros((X.rows, X.cols), dtype=np.int64)
    r = np.repeat(np.arange(X.rows), np.diff(X.rpt))
    d[r, X.col] = 1
    return d


def _assert_same_csr(C: Csr, D: Csr, exact_values=True):
    assert C.rows == D.rows and C.cols == D.cols
    np.testing.assert_array_equal(C.rpt, D.rpt)
    np.testing.assert_array_equal(C.col, D.col)
    if exact_values:
        np.testing.assert_array_equal(C.val, D.val)


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("which", ["gustavson", "brmerge"])
def test_matches_dense_matmul(oracle_mod, seed, which):
    """Eq. (1)/(2): values equal the dense product within 1e-12*sum|a||b|, and
    the stored pattern equals the boolean product of the input patterns
    (structural zeros from cancellation are kept)."""
    rng = np.random.default_rng(100 + seed)
    m, k, n = rng.integers(1, 40, size=3)
    A = random_sparse(int(m), int(k), float(rng.uniform(0.02, 0.5)), seed=seed)
    B = random_sparse(int(k), int(n), float(rng.uniform(0.02, 0.5)), seed=seed + 1000)
    C = (oracle_mod.spgemm_gustavson(A, B) if which == "gustavson"
         else oracle_mod.spgemm_brmerge(A, B)[0])
    C.validate()
    np.testing.assert_array_equal(_pattern(C), (_pattern(A) @ _pattern(B)) > 0)
    dense = A.to_dense() @ B.to_dense()
    bound = np.abs(A.to_dense()) @ np.abs(B.to_dense())
    err = np.abs(C.to_dense() - dense)
    assert np.all(err <= 1e-12 * bound + 0.0)


@pytest.mark.parametrize("seed", range(8))
def test_integer_values_all_orders_exact(oracle_mod, seed):
    """Small-integer values make every partial sum exact in fp64, so Eq. (2)'s
    k-order sum, Algorithm 1's tree-order sum and dense matmul agree bit for
    bit -- including explicit zeros produced by cancellation."""
    A = random_sparse(30, 25, 0.3, seed=seed, integer_values=True)
    B = random_sparse(25, 35, 0.3, seed=seed + 50, integer_values=True)
    G = oracle_mod.spgemm_gustavson(A, B)
    T, _ = oracle_mod.spgemm_brmerge(A, B)
    _assert_same_csr(G, T)
    np.testing.assert_array_equal(G.to_dense(), A.to_dense() @ B.to_dense())


def test_cancellation_keeps_structural_zero(oracle_mod):
    # A = [[1, 1]], B = [[1], [-1]] -> C = [[0]] stored explicitly.
    A = Csr(1, 2, np.array([0, 2], np.int64), np.array([0, 1], np.int32), np.array([1.0, 1.0]))
    B = Csr(2, 1, np.array([0, 1, 2], np.int64), np.array([0, 0], np.int32), np.array([1.0, -1.0]))
    for C in (oracle_mod.spgemm_gustavson(A, B), oracle_mod.spgemm_brmerge(A, B)[0]):
        np.testing.assert_array_equal(C.rpt, [0, 1])
        np.testing.assert_array_equal(C.col, [0])
        assert C.val[0] == 0.0


@pytest.mark.parametrize("which", ["gustavson", "brmerge"])
def test_identity_invariant(oracle_mod, which):
    A = uniform_random(300, 300, 9, seed=5)
    I = identity(300)
    f = (oracle_mod.spgemm_gustavson if which == "gustavson"
         else (lambda x, y: oracle_mod.spgemm_brmerge(x, y)[0]))
    _assert_same_csr(f(A, I), A)
    _assert_same_csr(f(I, A), A)


@pytest.mark.parametrize("which", ["gustavson", "brmerge"])
def test_permutation_invariant(oracle_mod, which):
    """(P A)[i] = A[perm[i]] row-wise; (A P)[i, perm[k]] = A[i, k]. Exact."""
    A = uniform_random(257, 257, 7, seed=9)
    P, perm = permutation(257, seed=4)
    f = (oracle_mod.spgemm_gustavson if which == "gustavson"
         else (lambda x, y: oracle_mod.spgemm_brmerge(x, y)[0]))
    PA = f(P, A)
    for i in range(257):
        s, e = PA.rpt[i], PA.rpt[i + 1]
        r = perm[i]
        np.testing.assert_array_equal(PA.col[s:e], A.col[A.rpt[r]:A.rpt[r + 1]])
        np.testing.assert_array_equal(PA.val[s:e], A.val[A.rpt[r]:A.rpt[r + 1]])
    AP = f(A, P)
    for i in range(257):
        s, e = AP.rpt[i], AP.rpt[i + 1]
        src_c = perm[A.col[A.rpt[i]:A.rpt[i + 1]]]
        order = np.argsort(src_c)
        np.testing.assert_array_equal(AP.col[s:e], src_c[order])
        np.testing.assert_array_equal(AP.val[s:e], A.val[A.rpt[i]:A.rpt[i + 1]][order])


@pytest.mark.parametrize("seed", range(6))
def test_nprod_bounds_and_column_row_identity(oracle_mod, seed):
    """nnz(C_i) <= n_prod_i per row; and sum_i n_prod_i equals
    sum_k nnz(A_*k) * nnz(B_k*) (the outer-product count, Eq. (4))."""
    A = random_sparse(60, 50, 0.1, seed=seed)
    B = random_sparse(50, 70, 0.15, seed=seed + 7)
    nprod = oracle_mod.row_nprod(A, B)
    C = oracle_mod.spgemm_gustavson(A, B)
    assert np.all(np.diff(C.rpt) <= nprod)
    colcount = np.bincount(A.col, minlength=A.cols)
    assert nprod.sum() == int(np.sum(colcount * np.diff(B.rpt)))
    # brute force per row
    for i in range(A.rows):
        ks = A.col[A.rpt[i]:A.rpt[i + 1]]
        assert nprod[i] == sum(int(B.rpt[k + 1] - B.rpt[k]) for k in ks)


@pytest.mark.parametrize("n", [4, 5, 7])
def test_stencil27_closed_forms(oracle_mod, n):
    """27-point stencil on n^3: nnz(A^2) = (5n-6)^3, n_prod = (9n-10)^3, and
    with noise 0 each entry equals the common-neighbour count formula:
    |K| if i, j are not adjacent, |K| - 54 if adjacent (j != i),
    26^2 + |N(i)| - 1 on the diagonal, |K| = prod_d #{k_d : |k_d-i_d|<=1, |k_d-j_d|<=1}."""
    A = stencil27(n, noise=0.0)
    C = oracle_mod.spgemm_gustavson(A, A)
    T, _ = oracle_mod.spgemm_brmerge(A, A)
    _assert_same_csr(C, T)  # integer values -> both orders exact
    assert C.nnz == (5 * n - 6) ** 3
    assert int(oracle_mod.row_nprod(A, A).sum()) == (9 * n - 10) ** 3

    def coords(r):
        return (r % n, (r // n) % n, r // (n * n))

    for i in range(0, n ** 3, max(1, n ** 3 // 40)):
        ci = coords(i)
        nbrs = 1
        for d in range(3):
            nbrs *= sum(1 for t in (-1, 0, 1) if 0 <= ci[d] + t < n)
        for p in range(C.rpt[i], C.rpt[i + 1]):
            j = int(C.col[p])
            cj = coords(j)
            K = 1
            for d in range(3):
                K *= sum(1 for kd in range(n) if abs(kd - ci[d]) <= 1 and abs(kd - cj[d]) <= 1)
            if j == i:
                expect = 26 * 26 + nbrs - 1
            elif all(abs(ci[d] - cj[d]) <= 1 for d in range(3)):
                expect = K - 54
            else:
                expect = K
            assert C.val[p] == expect, (i, j)


@pytest.mark.parametrize("n", [4, 6, 10])
def test_laplace_times_aggregation_closed_form(oracle_mod, n):
    """5-pt Laplacian (n^2) x 2x2 aggregation: nnz(C) = 3n^2 - 4n; with
    perturbation 0, C[i, g] = sum of A_ik over neighbours k aggregated to g."""
    A = laplace2d_5pt(n)
    P = aggregation_prolongator(n, perturb=0.0)
    C = oracle_mod.spgemm_gustavson(A, P)
    assert C.nnz == 3 * n * n - 4 * n
    h = n // 2
    for i in range(n * n):
        x, y = i % n, i // n
        expect = {}
        for dx, dy, a in ((0, -1, -1.0), (-1, 0, -1.0), (0, 0, 4.0), (1, 0, -1.0), (0, 1, -1.0)):
            if 0 <= x + dx < n and 0 <= y + dy < n:
                g = ((y + dy) // 2) * h + (x + dx) // 2
                expect[g] = expect.get(g, 0.0) + a
        s, e = C.rpt[i], C.rpt[i + 1]
        assert list(C.col[s:e]) == sorted(expect)
        assert list(C.val[s:e]) == [expect[g] for g in sorted(expect)]


def test_fig2_six_lists_three_rounds(oracle_mod):
    """Fig. 2 caption: six lists need ceil(log 6) = 3 rounds."""
    # one row of A with 6 nonzeros hitting 6 non-empty rows of B
    A = Csr(1, 6, np.array([0, 6], np.int64), np.arange(6, dtype=np.int32), np.ones(6))
    B = uniform_random(6, 20, 3, seed=2)
    _, rounds = oracle_mod.spgemm_brmerge(A, B)
    assert rounds[0] == 3


@pytest.mark.parametrize("k", range(1, 34))
def test_round_count_and_monotone_shrink(oracle_mod, k):
    """Alg. 1 lines 21-35 halve num_list each round: ceil(log2 k) rounds; the
    live element total never grows ("the required memory size of
    the intermediate lists is reduced")."""
    A = Csr(1, k, np.array([0, k], np.int64), np.arange(k, dtype=np.int32), np.ones(k))
    B = uniform_random(k, 12, 4, seed=k)
    _, rounds = oracle_mod.spgemm_brmerge(A, B)
    assert rounds[0] == (math.ceil(math.log2(k)) if k > 1 else 0)
    tr = oracle_mod.brmerge_trace(A, B, 0)
    assert len(tr) == rounds[0] + 1
    assert tr[0] == 4 * k
    assert np.all(np.diff(tr) <= 0)


def test_merge_two_examples(oracle_mod):
    c, v = oracle_mod.merge_two([1], [1.0], [1], [2.0])
    assert list(c) == [1] and list(v) == [3.0]
    c, v = oracle_mod.merge_two([0, 2], [1.0, 1.0], [1], [5.0])
    assert list(c) == [0, 1, 2] and list(v) == [1.0, 5.0, 1.0]
    rng = np.random.default_rng(0)
    a = np.sort(rng.choice(400, 100, replace=False))
    b = np.sort(rng.choice(400, 100, replace=False))
    av, bv = rng.random(100), rng.random(100)
    c, v = oracle_mod.merge_two(a, av, b, bv)
    ref = {}
    for cc, vv in list(zip(a, av)) + list(zip(b, bv)):
        ref[int(cc)] = ref.get(int(cc), 0.0) + vv
    assert list(c) == sorted(ref)
    np.testing.assert_array_equal(v, [ref[x] for x in sorted(ref)])


def test_empty_rows_and_empty_matrix(oracle_mod):
    A = Csr(3, 3, np.zeros(4, np.int64), np.zeros(0, np.int32), np.zeros(0))
    for C in (oracle_mod.spgemm_gustavson(A, A), oracle_mod.spgemm_brmerge(A, A)[0]):
        np.testing.assert_array_equal(C.rpt, [0, 0, 0, 0])
    # nilpotent [[0,1],[0,0]]^2 = 0
    N = Csr(2, 2, np.array([0, 1, 1], np.int64), np.array([1], np.int32), np.array([1.0]))
    C = oracle_mod.spgemm_gustavson(N, N)
    np.testing.assert_array_equal(C.rpt, [0, 0, 0])


def test_row_subset_matches_full(oracle_mod):
    A = uniform_random(500, 500, 6, seed=3)
    full = oracle_mod.spgemm_gustavson(A, A)
    rows = np.array([7, 0, 499, 250, 7])
    sub = oracle_mod.spgemm_gustavson(A, A, rows=rows)
    for t, r in enumerate(rows):
        np.testing.assert_array_equal(sub.col[sub.rpt[t]:sub.rpt[t + 1]],
                                      full.col[full.rpt[r]:full.rpt[r + 1]])
        np.testing.assert_array_equal(sub.val[sub.rpt[t]:sub.rpt[t + 1]],
                                      full.val[full.rpt[r]:full.rpt[r + 1]])


def test_balance_by_nprod_examples(oracle_mod):
    assert oracle_mod.balance_by_nprod([1, 1, 1, 1], 2) == [0, 2, 4]
    assert oracle_mod.balance_by_nprod([10, 1, 1], 2) == [0, 1, 3]
    b = oracle_mod.balance_by_nprod([1, 1], 4)
    assert b[0] == 0 and b[-1] == 2 and all(x <= y for x, y in zip(b, b[1:]))
    # brute force: every group sum is within one row's n_prod of total/p
    rng = np.random.default_rng(1)
    w = rng.integers(0, 50, size=200)
    for p in (1, 2, 3, 8):
        b = oracle_mod.balance_by_nprod(w, p)
        assert b[0] == 0 and b[-1] == 200
        for g in range(p):
            s = int(w[b[g]:b[g + 1]].sum())
            assert abs(s - w.sum() / p) <= w.max() + 1e-9


def test_table2_compression_ratios(oracle_mod):
    """Eq. (5) against the ratios printed in Table 2 (tests/golden/table2.txt,
    PAPER.md:358-420)."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "table2.txt")) if not l.startswith("#")]
    assert len(rows) == 26
    for r in rows:
        nprod, nnz, cr = int(r[6]), int(r[7]), float(r[8])
        assert abs(oracle_mod.compression_ratio(nprod, nnz) - cr) <= 0.005 + 1e-12, r[1]


# ---------------------------------------------------------------------------
# Pin of Algorithm 1's pairing ORDER (lines 21-35): each
# round consumes the lists two at a time from the front of src_buffer --
# (0,1), (2,3), ... -- and copies an odd trailing list (lines 28-29); the
# next round pairs the results the same way. The value of a column is
# therefore the tree sum below, written out by hand per case. fp64 addition
# is not associative on these values (1e16 + 1 == 1e16), so a wrong pairing
# -- k-order summation, (0,2)(1,3), the odd list copied first, pairing from
# the back -- changes the bits. Every list is one B row with a single entry
# in column 0, scaled by A_ik = 1.0 (exact), so the products are the values.
# ---------------------------------------------------------------------------
def _one_column_row(vals, present=None):
    """One row of A with len(vals) nonzeros (all 1.0) over a B whose row k
    holds vals[k] in column 0 (or is empty when present[k] is False)."""
    k = len(vals)
    present = [True] * k if present is None else present
    lens = np.array([1 if p else 0 for p in present], np.int64)
    rpt = np.zeros(k + 1, np.int64)
    np.cumsum(lens, out=rpt[1:])
    bval = np.array([v for v, p in zip(vals, present) if p], np.float64)
    B = Csr(k, 1, rpt, np.zeros(bval.size, np.int32), bval)
    A = Csr(1, k, np.array([0, k], np.int64), np.arange(k, dtype=np.int32), np.ones(k))
    return A, B


_BIG = 1e16  # spacing of fp64 at 1e16 is 2: 1e16 + 1 rounds back to 1e16

# (values, present, the Algorithm-1 tree written out by hand)
_TREE_CASES = [
    # 3 lists: round 1 (0,1), 2 copied; round 2 (01, 2)
    ([_BIG, 1.0, -_BIG], None, lambda v: (v[0] + v[1]) + v[2]),
    ([1.0, -_BIG, _BIG], None, lambda v: (v[0] + v[1]) + v[2]),
    # 4 lists: (0,1), (2,3); then (01, 23)
    ([-_BIG, 1.0, _BIG, 1.0], None, lambda v: (v[0] + v[1]) + (v[2] + v[3])),
    ([1.0, 1.0, _BIG, -_BIG], None, lambda v: (v[0] + v[1]) + (v[2] + v[3])),
    # 5 lists: (0,1), (2,3), 4 copied; (01, 23), 4 copied; (0123, 4)
    ([1.0, _BIG, -_BIG, 1.0, 1.0], None, lambda v: ((v[0] + v[1]) + (v[2] + v[3])) + v[4]),
    ([_BIG, -_BIG, 1.0, 1.0, -_BIG], None, lambda v: ((v[0] + v[1]) + (v[2] + v[3])) + v[4]),
    # 6 lists (Fig. 2's shape): (0,1),(2,3),(4,5); (01,23), 45 copied; (0123, 45)
    ([1.0, _BIG, 1.0, -_BIG, 1.0, 1.0], None,
     lambda v: ((v[0] + v[1]) + (v[2] + v[3])) + (v[4] + v[5])),
    # 7 lists: (0,1),(2,3),(4,5), 6 copied; (01,23),(45,6); (0123, 456)
    ([_BIG, 1.0, 1.0, 1.0, -_BIG, 1.0, 1.0], None,
     lambda v: ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + v[6])),
    # an empty list keeps its place in the tree (Alg. 1 line 14 records its
    # offset): lists 1 and 4 lack the column, so pairs (0,1) and (4,5) pass
    # one value through; the tree is (v0 + (v2 + v3)) + v5
    ([1.0, 0.0, _BIG, 1.0, 0.0, -_BIG], [True, False, True, True, False, True],
     lambda v: (v[0] + (v[2] + v[3])) + v[5]),
    ([-_BIG, 0.0, 1.0, _BIG, 0.0, 1.0], [True, False, True, True, False, True],
     lambda v: (v[0] + (v[2] + v[3])) + v[5]),
]


def _alt_orders(n):
    """Plausible wrong orders (each must be refuted by some case)."""
    def seq(v, pres):
        s = None
        for x, p in zip(v, pres):
            if p:
                s = x if s is None else s + x
        return s

    def rounds(v, pres, pair):
        lists = [x if p else None for x, p in zip(v, pres)]
        while len(lists) > 1:
            lists = pair(lists)
        return lists[0]

    def add(a, b):
        return a if b is None else (b if a is None else a + b)

    def odd_first(ls):  # odd list copied FIRST, then (1,2), (3,4), ...
        if len(ls) % 2:
            return [ls[0]] + [add(ls[i], ls[i + 1]) for i in range(1, len(ls), 2)]
        return [add(ls[i], ls[i + 1]) for i in range(0, len(ls), 2)]

    def from_back(ls):  # pairs taken from the back: (n-2, n-1), ...
        r = [add(ls[i - 1], ls[i]) for i in range(len(ls) - 1, 0, -2)]
        if len(ls) % 2:
            r.append(ls[0])
        return r[::-1]

    def strided(ls):  # (0, h), (1, h+1), ... with h = ceil(n/2)
        h = (len(ls) + 1) // 2
        return [add(ls[i], ls[i + h]) if i + h < len(ls) else ls[i] for i in range(h)]

    return {"k-order": seq,
            "odd list copied first": lambda v, p: rounds(v, p, odd_first),
            "pairs from the back": lambda v, p: rounds(v, p, from_back),
            "strided pairs (i, i+n/2)": lambda v, p: rounds(v, p, strided)}


def test_alg1_pairing_order_pinned(oracle_mod):
    """Algorithm 1's tree order, bit for bit, on hand-derived non-associative
    cases; each plausible wrong order is refuted by at
    least one case, so the pin discriminates."""
    refuted = {name: False for name in _alt_orders(0)}
    for vals, present, tree in _TREE_CASES:
        pres = [True] * len(vals) if present is None else present
        expect = tree(vals)
        A, B = _one_column_row(vals, present)
        C, rounds = oracle_mod.spgemm_brmerge(A, B)
        assert C.nnz == 1 and C.col[0] == 0
        assert C.val[0] == expect and np.signbit(C.val[0]) == np.signbit(expect), (vals, C.val[0], expect)
        assert rounds[0] == math.ceil(math.log2(len(vals)))
        for name, alt in _alt_orders(len(vals)).items():
            if alt(vals, pres) != expect:
                refuted[name] = True
        # Gustavson (Eq. (2)) sums in k order: it must equal the k-order sum
        G = oracle_mod.spgemm_gustavson(A, B)
        assert G.val[0] == _alt_orders(0)["k-order"](vals, pres)
    assert all(refuted.values()), refuted


def test_alg1_pairing_order_multi_column(oracle_mod):
    """The same tree per column when columns differ across lists: 5 lists over
    2 columns; column 0 is in lists 0, 1, 3, 4 and column 1 in lists 1-4.
    Hand-derived: col 0 = ((v0 + v1) + v3) + v4 per Alg. 1 (list 2 lacks it:
    pair (2,3) passes v3 through), col 1 = (w1 + (w2 + w3)) + w4 (list 0
    lacks it: pair (0,1) passes w1 through). (fp64 addition commutes, so
    left + right vs right + left is not observable; grouping is.)"""
    v = [1.0, _BIG, None, -_BIG, 1.0]        # column 0 entries of lists 0..4
    w = [None, 1.0, 1.0, _BIG, -_BIG]        # column 1 entries
    rpt, col, val = [0], [], []
    for k in range(5):
        for c, x in ((0, v[k]), (1, w[k])):
            if x is not None:
                col.append(c)
                val.append(x)
        rpt.append(len(col))
    B = Csr(5, 2, np.array(rpt, np.int64), np.array(col, np.int32), np.array(val))
    A = Csr(1, 5, np.array([0, 5], np.int64), np.arange(5, dtype=np.int32), np.ones(5))
    C, _ = oracle_mod.spgemm_brmerge(A, B)
    e0 = ((v[0] + v[1]) + v[3]) + v[4]
    e1 = (w[1] + (w[2] + w[3])) + w[4]
    assert list(C.col) == [0, 1]
    assert C.val[0] == e0 and C.val[1] == e1
    # column 1's tree differs from its k-order sum, so the case discriminates
    assert e1 != ((w[1] + w[2]) + w[3]) + w[4]


@pytest.mark.parametrize("seed", range(6))
def test_row_sizes_definition(oracle_mod, seed):
    """oracle.row_sizes = the per-row count of the boolean product's nonzeros
    (dense pattern product, brute force), for all rows and for a row subset
    given out of order."""
    rng = np.random.default_rng(300 + seed)
    m, k, n = (int(x) for x in rng.integers(1, 60, size=3))
    A = random_sparse(m, k, float(rng.uniform(0.02, 0.4)), seed=seed)
    B = random_sparse(k, n, float(rng.uniform(0.02, 0.4)), seed=seed + 7)
    expect = ((_pattern(A) @ _pattern(B)) > 0).sum(axis=1)
    np.testing.assert_array_equal(oracle_mod.row_sizes(A, B), expect)
    rows = rng.permutation(m)[: max(1, m // 2)]
    np.testing.assert_array_equal(oracle_mod.row_sizes(A, B, rows=rows), expect[rows])


def test_row_sizes_closed_forms(oracle_mod):
    """27-point stencil squared: rows of C are the 5x5x5 neighbourhoods
    clipped to the grid, (5n-6)^3 nonzeros in total; identity: nnz(A_i*)."""
    n = 7
    S = stencil27(n, seed=1)
    rs = oracle_mod.row_sizes(S, S)
    assert rs.sum() == (5 * n - 6) ** 3
    X = uniform_random(300, 300, 7, seed=3)
    np.testing.assert_array_equal(oracle_mod.row_sizes(X, identity(300)), np.full(300, 7))
    np.testing.assert_array_equal(oracle_mod.row_sizes(identity(300), X), np.full(300, 7))
