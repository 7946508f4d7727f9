"""Debug aid: a line-by-line Python emulation of the chunk partition used by
csrc/engine.cuh rec_round (record tiers) and chunk_round (global tier):
sentinel-terminated lists, G chunks of odd VT positions, pair crossing,
dedupe at chunk starts; one row, G emulated threads. Used to check the partitioning logic on the CPU against
the oracle; not used by tests or the product path.
Usage: python tools/emulate_chunk.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
INF = 2**31 - 1


def merge_path(a, b, diag):
    lo, hi = max(0, diag - len(b)), min(diag, len(a))
    while lo < hi:
        mid = (lo + hi) // 2
        if a[mid] <= b[diag - 1 - mid]:
            lo = mid + 1
        else:
            hi = mid
    return lo


def chunk_round(G, sc, sv, off, nl, first, av):
    npairs = (nl + 1) // 2
    npos = off[nl] + (nl & 1)
    VT = (-(-npos // G)) | 1
    outs = []
    noff = {}
    for rank in range(G):
        g0 = min(rank * VT, npos)
        g1 = min(g0 + VT, npos)
        oc_l, ov_l, ent = [], [], []
        if g0 < g1:
            lo, hi = 0, npairs - 1
            while lo < hi:
                mid = (lo + hi + 1) // 2
                if off[2 * mid] <= g0:
                    lo = mid
                else:
                    hi = mid - 1
            p = lo
            as_, bs = off[2 * p], off[2 * p + 1]
            bend = off[2 * p + 2] if 2 * p + 2 <= nl else off[nl] + 1
            na, nb = bs - as_, bend - bs
            d = g0 - as_
            if d == 0:
                ent.append((p, 0))
            i = merge_path(sc[as_:bs], sc[bs:bend], d)
            j = d - i
            if i > 0 and j < nb and sc[as_ + i - 1] == sc[bs + j]:
                j += 1
            cur = None
            if i == na:
                if g0 + 1 < g1:
                    p += 1
                    ent.append((p, 0))
                    cur = [p, off[2 * p + 1], off[2 * p], off[2 * p + 1]]
            else:
                cur = [p, bs, as_ + i, bs + j]
            if cur is not None:
                p, bs, ia, ib = cur
                lim = g1 + bs
                for _ in range(VT):
                    if not ia + ib < lim:
                        break
                    ca, cb = sc[ia], sc[ib]
                    ta, tb = ca <= cb, cb <= ca
                    sa = av[2 * p] if first else 1.0
                    sb = (av[2 * p + 1] if 2 * p + 1 < nl else 0.0) if first else 1.0
                    x = sa * sv[ia] if ta else -0.0
                    y = sb * sv[ib] if tb else -0.0
                    oc_l.append(min(ca, cb))
                    ov_l.append(x + y)
                    ia += ta
                    ib += tb
                    if min(ca, cb) == INF and ia + ib < lim:
                        p += 1
                        ent.append((p, len(oc_l)))
                        bs = off[2 * p + 1]
                        ia, ib = off[2 * p], bs
                        lim = g1 + bs
        outs.append((oc_l, ov_l, ent))
    base = 0
    dc, dv = [], []
    for oc_l, ov_l, ent in outs:
        for q, c in ent:
            assert q not in noff, ("pair start recorded twice", q)
            noff[q] = base + c
        dc += oc_l
        dv += ov_l
        base += len(oc_l)
    noff[npairs] = base
    assert sorted(noff) == list(range(npairs + 1)), ("missing pair starts", sorted(noff))
    dc.append(INF)
    dv.append(0.0)
    return dc, dv, [noff[q] for q in range(npairs + 1)]


ROUND = chunk_round


def chunk_row(G, A, B, row):
    a0, a1 = A.rpt[row], A.rpt[row + 1]
    nl = a1 - a0
    sc, sv, off, av = [], [], [], []
    for l in range(nl):
        k = A.col[a0 + l]
        off.append(len(sc))
        sc += list(B.col[B.rpt[k]:B.rpt[k + 1]]) + [INF]
        sv += list(B.val[B.rpt[k]:B.rpt[k + 1]]) + [0.0]
        av.append(A.val[a0 + l])
    off.append(len(sc))
    sc.append(INF)
    sv.append(0.0)
    cur, first = nl, True
    while cur > 1:
        sc, sv, off = ROUND(G, sc, sv, off, cur, first, av)
        first = False
        cur = (cur + 1) // 2
    n = off[1] - 1 if nl > 1 else off[1] - 1
    vals = sv[:n] if nl > 1 else [av[0] * v for v in sv[:n]]
    return sc[:n], vals


if __name__ == "__main__":
    import oracle
    from inputs import stencil27, uniform_random
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    from test_gpu_parity import _lists_matrix
    cases = [(_lists_matrix([90, 93, 94], 33, 5000, seed=33), [32, 128, 256]),
             (_lists_matrix([5, 50, 700], 4, 3000, seed=3, empty_rows_of_b=1500), [32, 128, 256]),
             ((stencil27(6), stencil27(6)), [32, 8, 16])]
    for name, fn in (("chunk_round", chunk_round),):
      ROUND = fn
      for (A, B), Gs in cases:
        ref, _ = oracle.spgemm_brmerge(A, B)
        for G in Gs:
            for r in range(A.rows):
                c, v = chunk_row(G, A, B, r)
                s, e = ref.rpt[r], ref.rpt[r + 1]
                assert list(ref.col[s:e]) == c, (name, G, r, "cols")
                assert np.array_equal(ref.val[s:e], np.array(v)), (name, G, r, "vals")
            print(name, "ok", A.rows, "rows, G =", G)
