"""Analysis aid (not product, not tests): on a sample of rmat20_ef16's
one-level heavy rows (<= 512 lists, > 6656 products), cut each row into
windows of <= 4096 products by column (greedy, column granularity) and count,
per window, the element moves of Algorithm 1's rounds:
  all   -- every live element moves every round (the A-with-B merge of
           k_hv_merge: lists of a pair with an empty partner move too)
  both  -- only elements of pairs whose two lists are non-empty move
           (pass-through lists stay where they are).
Usage: python tools/sim_passthrough.py [nrows]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import workload  # noqa: E402


def rounds(lists):
    """lists: list of np arrays of columns (sorted, unique). Returns (all, both)."""
    tot_all = tot_both = 0
    cur = lists
    while len(cur) > 1:
        nxt = []
        for q in range(0, len(cur), 2):
            a = cur[q]
            b = cur[q + 1] if q + 1 < len(cur) else np.zeros(0, np.int64)
            tot_all += a.size + b.size
            if a.size and b.size:
                tot_both += a.size + b.size
                nxt.append(np.union1d(a, b))
            else:
                nxt.append(a if a.size else b)
        cur = nxt
    return tot_all, tot_both


def main():
    nrows = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    A, B = workload("rmat20_ef16")
    nl = np.diff(A.rpt)
    blen = np.diff(B.rpt)
    rng = np.random.default_rng(0)
    cs = np.concatenate([[0], np.cumsum(blen[A.col])])
    nprod = cs[A.rpt[1:]] - cs[A.rpt[:-1]]
    heavy = np.nonzero((nl <= 512) & (nprod > 6656))[0]
    print("one-level heavy rows", heavy.size, "products", int(nprod[heavy].sum()))
    w = nprod[heavy] / nprod[heavy].sum()
    pick = rng.choice(heavy, size=min(nrows, heavy.size), replace=False, p=w)
    S_all = S_both = S_p = 0
    nonempty = []
    for r in pick:
        ks = A.col[A.rpt[r]:A.rpt[r + 1]]
        lists = [B.col[B.rpt[k]:B.rpt[k + 1]].astype(np.int64) for k in ks]
        allc = np.sort(np.concatenate(lists))
        # greedy windows of <= 4096 products at column granularity
        uc, cnt = np.unique(allc, return_counts=True)
        cs = np.cumsum(cnt)
        cuts = [uc[0]]
        base = 0
        while True:
            j = np.searchsorted(cs, base + 4096, side="right")
            if j >= uc.size:
                break
            cuts.append(uc[j])
            base = cs[j - 1]
        cuts.append(uc[-1] + 1)
        for c0, c1 in zip(cuts[:-1], cuts[1:]):
            wl = [L[(L >= c0) & (L < c1)] for L in lists]
            a, b = rounds(wl)
            S_all += a
            S_both += b
            S_p += sum(x.size for x in wl)
            nonempty.append(sum(1 for x in wl if x.size) / len(wl))
    print(f"sample {len(pick)} rows, {S_p} products")
    print(f"element moves per product: all {S_all / S_p:.2f}  both-non-empty {S_both / S_p:.2f}")
    print(f"non-empty lists per window: mean fraction {np.mean(nonempty):.3f}")


if __name__ == "__main__":
    main()
