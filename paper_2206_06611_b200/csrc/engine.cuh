// engine.cuh -- the BRMerge accumulation of one output row by a thread group
// (Algorithm 1), in two GPU forms that compute exactly the
// rounds of Algorithm 1 (pairs (0,1),(2,3),... of the current lists merged,
// an odd trailing list copied, equal columns summed as left + right), so the
// values are bit-identical to the paper's sequential tree order (R1).
//
// reg_row  (tiers 1-2, P <= G <= 32): register-resident BRMerge. Lane e holds
//   product e of the row (multiplying phase, lines 10-15). Each round merges
//   list pairs in registers: a lane finds the rank of its column in the
//   partner list by a shuffle binary search (warp-shuffle merge path), left
//   lanes add the partner's equal-column value, right duplicates retire, and
//   every survivor moves to its merged position through a G-slot shared
//   ping-pong buffer.
//
// chunk_row (tiers 3-7): shared-memory (or global-workspace) ping-pong. The
//   multiplying phase copies the B rows of A_i* into `src` as compact sorted
//   lists, scaled by A_ik (one rounding per product, Alg. 1 line 12). Each
//   round is ONE pass: the round's merged positions (the concatenation of all
//   pairs) are split into G equal odd-length chunks; a thread locates its
//   chunk's pair and merge-path split, merges it sequentially with a
//   branch-free step (sum on equal columns) into `dst`, crossing into later
//   pairs when one ends; a group scan of the per-thread output counts gives
//   the compacted positions and the next round's list offsets, and each
//   thread copies its outputs back to `src` compacted.
#pragma once
#include "brm_internal.cuh"

namespace brm {

enum OutKind { OUT_SYMBOLIC = 0, OUT_CBAR = 1, OUT_C = 2 };

struct RowOut {
  const int64_t* base;  // OUT_CBAR: n_prod offsets; OUT_C: C.rpt
  int32_t* col;
  double* val;
  int64_t* row_size;    // OUT_SYMBOLIC / OUT_CBAR: nnz of each output row
};

// Shared scratch of one register-tier group (G slots each).
struct RegBufs {
  int* col;
  double* val;
  int* lid;
  int* owner;
};

template <int G, bool VALS>
__host__ __device__ constexpr int reg_group_bytes() {
  return align16(G * 4) * 3 + (VALS ? align16(G * 8) : 0);
}

// Working arrays of one chunk-tier group. Lists of a round are compact in
// col[0]/val[0] ("src"); col[1]/val[1] ("dst") receive the merged chunks.
// off[0] holds the current list offsets (nl + 1), off[1] the next round's.
struct ChunkBufs {
  int* col0;
  int* col1;
  double* val0;
  double* val1;
  int* off0;
  int* off1;
  int64_t* bst;  // B row start of each list
  double* av;    // A_ik of each list
  int* scan_tmp;
};

template <int G, int CAP, int LCAP, bool VALS>
__host__ __device__ constexpr int chunk_group_bytes() {
  return align16((CAP + 2) * 4) * 2 + (VALS ? align16((CAP + 2) * 8) * 2 : 0) + align16((LCAP + 2) * 4) * 2 +
         align16(LCAP * 8) + (VALS ? align16(LCAP * 8) : 0) + (G > 32 ? align16((G / 32 + 2) * 4) : 0);
}

// ===========================================================================
// Register tier
// ===========================================================================
template <int G>
__device__ __forceinline__ unsigned group_ballot(const Group<G>& g, bool p) {
  const unsigned b = __ballot_sync(g.mask, p);
  if constexpr (G >= 32)
    return b;
  else
    return (b >> g.base) & ((1u << G) - 1u);
}

template <int G, bool VALS, int OUT>
__device__ __forceinline__ void reg_row(const Group<G>& g, const CsrView& A, const CsrView& B, int64_t row,
                                        const RowOut& o, const RegBufs& rb) {
  constexpr int LOG = (G <= 8) ? 4 : 6;  // binary-search steps over <= G lanes
  const int lane = g.rank;
  const int64_t a0 = A.rpt[row];
  const int nl = static_cast<int>(A.rpt[row + 1] - a0);
  // multiplying phase (Alg. 1 lines 10-15): list l = B row A.col[a0 + l]
  int n = 0;
  int64_t st = 0;
  double av = 0.0;
  if (lane < nl) {
    const int k = __ldg(A.col + a0 + lane);
    st = __ldg(B.rpt + k);
    n = static_cast<int>(__ldg(B.rpt + k + 1) - st);
    if (VALS) av = __ldg(A.val + a0 + lane);
  }
  int T;
  const int off = group_excl_scan<G>(g, n, T, nullptr);
  const bool owns = lane < nl && n > 0;
  if (owns) rb.owner[off] = lane;
  const unsigned starts = __reduce_or_sync(g.mask, owns ? (1u << off) : 0u);
  g.sync();
  int s = 0, l = 0;
  if (lane < T) {
    s = 31 - __clz(starts & ((2u << lane) - 1u));  // start of the list holding product `lane`
    l = rb.owner[s];
  }
  const int64_t stl = __shfl_sync(g.mask, st, l, G);
  const double avl = VALS ? __shfl_sync(g.mask, av, l, G) : 0.0;
  int c = INT_MAX;
  double v = 0.0;
  if (lane < T) {
    c = __ldg(B.col + stl + (lane - s));
    if (VALS) v = __dmul_rn(avl, __ldg(B.val + stl + (lane - s)));
  }
  // accumulating phase (lines 21-35): ceil(log2 nl) rounds; at round r the
  // current list of a product is l >> r, pairs are (2m, 2m+1).
  const int R = nl <= 1 ? 0 : 32 - __clz(nl - 1);
  for (int r = 0; r < R; ++r) {
    const bool act = lane < T;
    const int m = act ? (l >> r) : -1;
    const int mprev = __shfl_up_sync(g.mask, m, 1, G);
    const bool start = act && (lane == 0 || mprev != m);
    const unsigned sm = group_ballot<G>(g, start);
    const unsigned le = (2u << lane) - 1u;  // lanes [0, lane]
    const int my_start = act ? 31 - __clz(sm & le) : 0;
    const unsigned above = sm & ~le;
    const int my_end = act ? (above ? __ffs(above) - 1 : T) : 0;
    const bool left = act && (m & 1) == 0;
    const int m_next = __shfl_sync(g.mask, m, my_end < G ? my_end : G - 1, G);
    const int m_prev = __shfl_sync(g.mask, m, my_start > 0 ? my_start - 1 : 0, G);
    int ps = my_start, pe = my_start;  // partner range [ps, pe)
    if (left) {
      ps = pe = my_end;
      if (my_end < T && m_next == (m ^ 1)) {
        const unsigned ab = sm & ~((2u << my_end) - 1u);
        pe = ab ? __ffs(ab) - 1 : T;
      }
    } else if (act && my_start > 0 && m_prev == (m ^ 1)) {
      ps = 31 - __clz(sm & ((1u << my_start) - 1u));
    }
    // rank of c in the partner list (lower bound) by shuffles
    int lo = ps, hi = pe;
#pragma unroll
    for (int it = 0; it < LOG; ++it) {
      const int mid = (lo + hi) >> 1;
      const int cm = __shfl_sync(g.mask, c, mid < G ? mid : G - 1, G);
      if (lo < hi) {
        if (cm < c)
          lo = mid + 1;
        else
          hi = mid;
      }
    }
    const int src = lo < G ? lo : G - 1;
    const int cq = __shfl_sync(g.mask, c, src, G);
    const bool found = act && lo < pe && cq == c;
    if (VALS) {
      const double pv = __shfl_sync(g.mask, v, src, G);
      if (left && found) v = __dadd_rn(v, pv);  // "vals with duplicate cols are combined"
    }
    const bool dead = found && !left;
    const unsigned dm = group_ballot<G>(g, dead);
    const unsigned mm = group_ballot<G>(g, found);
    const int matched_before = __popc(mm & ((1u << lane) - 1u) & ~((1u << my_start) - 1u));
    const int pair_start = left ? my_start : ps;
    const int newpos = pair_start - __popc(dm & ((1u << pair_start) - 1u)) + (lane - my_start) + (lo - ps) -
                       matched_before;
    const int newT = T - __popc(dm);
    if (act && !dead) {
      rb.col[newpos] = c;
      if (VALS) rb.val[newpos] = v;
      rb.lid[newpos] = l;
    }
    g.sync();
    c = INT_MAX;
    if (lane < newT) {
      c = rb.col[lane];
      if (VALS) v = rb.val[lane];
      l = rb.lid[lane];
    }
    g.sync();
    T = newT;
  }
  // Alg. 1 line 36: store the result row
  if (OUT != OUT_SYMBOLIC && lane < T) {
    const int64_t ob = o.base[row];
    o.col[ob + lane] = c;
    if (VALS) o.val[ob + lane] = v;
  }
  if (OUT != OUT_C && lane == 0) o.row_size[row] = T;
  g.sync();
}

// ===========================================================================
// Chunk tiers
// ===========================================================================

// One BRMerge round (Alg. 1 lines 22-34) over compact lists in sc/sv with
// offsets off[0..nl]; merged lists end up compact in sc/sv again with offsets
// noff[0..npairs]. Returns the new element total.
template <int G, bool VALS>
__device__ __forceinline__ int chunk_round(const Group<G>& g, int* __restrict__ sc, double* __restrict__ sv,
                                           int* __restrict__ dc, double* __restrict__ dv, const int* off,
                                           int* noff, int nl, int T, int* scan_tmp) {
  const int npairs = (nl + 1) >> 1;
  const int VT = ((T + G - 1) / G) | 1;  // odd: conflict-free strided smem access
  const int g0 = min(g.rank * VT, T), g1 = min(g0 + VT, T);
  int out = g0;
  int pf = 0, pl = -1;  // pairs whose start this thread records: [pf, pl]
  if (g0 < g1) {
    int lo = 0, hi = npairs - 1;  // last pair starting at or before g0 (it is non-empty)
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off[2 * mid] <= g0)
        lo = mid;
      else
        hi = mid - 1;
    }
    int p = lo;
    int as = off[2 * p];
    int bs = off[min(2 * p + 1, nl)];
    int be = off[min(2 * p + 2, nl)];
    const int d = g0 - as;
    if (d == 0) {  // this chunk starts pair p (and any empty pairs just before it)
      pf = p;
      while (pf > 0 && off[2 * (pf - 1)] == g0) --pf;
      for (int q = pf; q <= p; ++q) noff[q] = 0;
      pl = p;
    }
    const int i = merge_path(sc + as, bs - as, sc + bs, be - bs, d);
    int j = d - i;
    if (i > 0 && j < be - bs && sc[as + i - 1] == sc[bs + j]) ++j;  // b[j] was summed by the chunk on the left
    int ia = as + i, ib = bs + j;
    int lim = g1 + bs;  // merged position = ia + ib - bs
    int ca = ia < bs ? sc[ia] : INT_MAX;
    int cb = ib < be ? sc[ib] : INT_MAX;
    double va = 0.0, vb = 0.0;
    if (VALS) {
      va = sv[ia];
      vb = sv[ib];
    }
    while (ia + ib < lim) {
      if ((ca & cb) == INT_MAX) {  // both lists of pair p consumed: enter the next non-empty pair
        if (pl < 0) pf = p + 1;
        do {
          ++p;
          noff[p] = out - g0;
          as = off[2 * p];
          bs = off[min(2 * p + 1, nl)];
          be = off[min(2 * p + 2, nl)];
        } while (as == be);
        pl = p;
        ia = as;
        ib = bs;
        lim = g1 + bs;
        ca = ia < bs ? sc[ia] : INT_MAX;
        cb = ib < be ? sc[ib] : INT_MAX;
        if (VALS) {
          va = sv[ia];
          vb = sv[ib];
        }
      }
      const bool ta = ca <= cb, tb = cb <= ca;
      dc[out] = min(ca, cb);
      if (VALS) {
        const double x = ta ? va : -0.0;  // -0.0 is the exact additive identity
        const double y = tb ? vb : -0.0;
        dv[out] = __dadd_rn(x, y);
      }
      ++out;
      ia += ta;
      ib += tb;
      if (ta) {
        ca = ia < bs ? sc[ia] : INT_MAX;
        if (VALS) va = sv[ia];
      }
      if (tb) {
        cb = ib < be ? sc[ib] : INT_MAX;
        if (VALS) vb = sv[ib];
      }
    }
  }
  const int cnt = out - g0;
  int total;
  const int base = group_excl_scan<G>(g, cnt, total, scan_tmp);
  g.sync();  // every merge has finished reading sc
  for (int q = pf; q <= pl; ++q) noff[q] += base;
  for (int e = 0; e < cnt; ++e) {
    sc[base + e] = dc[g0 + e];
    if (VALS) sv[base + e] = dv[g0 + e];
  }
  if (g.rank == G - 1) {
    for (int q = npairs - 1; q >= 0 && off[2 * q] == T; --q) noff[q] = total;  // trailing empty pairs
    noff[npairs] = total;
  }
  g.sync();
  return total;
}

template <int G, bool VALS, int OUT>
__device__ __forceinline__ void chunk_row(const Group<G>& g, const CsrView& A, const CsrView& B, int64_t row,
                                          const RowOut& o, const ChunkBufs& cb) {
  const int rank = g.rank;
  const int64_t a0 = A.rpt[row];
  const int nl = static_cast<int>(A.rpt[row + 1] - a0);
  int* sc = cb.col0;
  double* sv = cb.val0;
  int* off = cb.off0;
  int* noff = cb.off1;
  // multiplying phase (Alg. 1 lines 10-15): list offsets by a group scan ...
  int T = 0;
  for (int lb = 0; lb < nl; lb += G) {
    const int l = lb + rank;
    int n = 0;
    if (l < nl) {
      const int k = __ldg(A.col + a0 + l);
      const int64_t st = __ldg(B.rpt + k);
      n = static_cast<int>(__ldg(B.rpt + k + 1) - st);
      cb.bst[l] = st;
      if (VALS) cb.av[l] = __ldg(A.val + a0 + l);
    }
    int tot;
    const int ex = group_excl_scan<G>(g, n, tot, cb.scan_tmp);
    if (l < nl) off[l] = T + ex;
    T += tot;
  }
  if (rank == 0) off[nl] = T;
  g.sync();
  // ... then the scaled B rows, S consecutive threads per list (S ~ mean list length)
  {
    const int avg = (T + nl - 1) / nl;
    int ls = 0;
    while ((1 << ls) < avg && (1 << ls) < G) ++ls;
    const int S = 1 << ls;
    const int per = G >> ls;
    const int sub = rank >> ls, e0 = rank & (S - 1);
    for (int lb = 0; lb < nl; lb += per) {
      const int l = lb + sub;
      if (l < nl) {
        const int o0 = off[l], n = off[l + 1] - o0;
        const int64_t st = cb.bst[l];
        const double a = VALS ? cb.av[l] : 0.0;
        for (int e = e0; e < n; e += 2 * S) {
          const int e1 = e + S;
          const bool h1 = e1 < n;
          const int c0 = __ldg(B.col + st + e);
          const int c1 = h1 ? __ldg(B.col + st + e1) : 0;
          double v0 = 0.0, v1 = 0.0;
          if (VALS) {
            v0 = __ldg(B.val + st + e);
            if (h1) v1 = __ldg(B.val + st + e1);
          }
          sc[o0 + e] = c0;
          if (VALS) sv[o0 + e] = __dmul_rn(a, v0);
          if (h1) {
            sc[o0 + e1] = c1;
            if (VALS) sv[o0 + e1] = __dmul_rn(a, v1);
          }
        }
      }
    }
  }
  g.sync();
  // accumulating phase (lines 21-35)
  int cur = nl;
  while (cur > 1) {
    T = chunk_round<G, VALS>(g, sc, sv, cb.col1, cb.val1, off, noff, cur, T, cb.scan_tmp);
    cur = (cur + 1) >> 1;
    int* t = off;
    off = noff;
    noff = t;
  }
  // line 36: the result row is list 0 of src, [0, T)
  if (OUT != OUT_SYMBOLIC) {
    const int64_t ob = o.base[row];
    for (int e = rank; e < T; e += G) {
      o.col[ob + e] = sc[e];
      if (VALS) o.val[ob + e] = sv[e];
    }
  }
  if (OUT != OUT_C && rank == 0) o.row_size[row] = T;
  g.sync();
}

}  // namespace brm
