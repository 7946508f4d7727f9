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
//   multiplying phase copies the B rows of A_i* into the ping buffer as
//   compact sorted lists (cp.async, coalesced); the scaling by A_ik is fused
//   into the first merge round (one rounding per product, Alg. 1 line 12).
//   Each round is ONE pass: the round's merged positions (the concatenation
//   of all pairs) are split into G equal odd-length chunks; a thread locates
//   its chunk's pair and merge-path split and merges it with a branch-free
//   predicated step (sum on equal columns), crossing into later pairs when
//   one ends, holding its outputs in registers; a group scan of the
//   per-thread output counts gives each thread its compacted position in the
//   pong buffer and the next round's list offsets; the buffers swap.
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
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// Predicated shared loads: one LDS under a predicate, never a branch.
__device__ __forceinline__ void lds_if(bool p, unsigned addr, int& v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.shared.b32 %0, [%1];\n\t}"
               : "+r"(v)
               : "r"(addr), "r"((unsigned)p));
}
__device__ __forceinline__ void lds_if(bool p, unsigned addr, double& v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.shared.f64 %0, [%1];\n\t}"
               : "+d"(v)
               : "r"(addr), "r"((unsigned)p));
}
__device__ __forceinline__ void cp_async_4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Merge state of one thread's chunk inside pair p = lists (2p, 2p+1):
// list a = [as, bs), list b = [bs, be) of src; heads ca/cb (INT_MAX once a
// list is consumed), head values va/vb; sa/sb = A_ik of the two lists (round
// 1 only: the scaling of Alg. 1 line 12 is fused into the first merge).
struct Cursor {
  int p, as, bs, be, ia, ib, lim, ca, cb;
  double va, vb, sa, sb;
};

template <bool VALS, bool FIRST>
__device__ __forceinline__ void cursor_load(Cursor& c, const int* sc, const double* sv, const double* av, int nl) {
  c.ca = c.ia < c.bs ? sc[c.ia] : INT_MAX;
  c.cb = c.ib < c.be ? sc[c.ib] : INT_MAX;
  if (VALS) {
    c.va = sv[c.ia];
    c.vb = sv[c.ib];
    if (FIRST) {
      c.sa = av[2 * c.p];
      c.sb = 2 * c.p + 1 < nl ? av[2 * c.p + 1] : 0.0;
    }
  }
}

// One BRMerge round (Alg. 1 lines 22-34) over compact lists in sc/sv with
// offsets off[0..nl]. The round's merged positions are split into G chunks of
// VT (odd) positions; the merged lists are written COMPACT with offsets
// noff[0..npairs]:
//   NV > 0: into dc/dv (the other ping-pong buffer), each thread holding its
//           <= NV outputs in registers until the group scan gives its base;
//   NV = 0: (global tier, unbounded VT) into dc/dv at the chunk's own
//           positions, then copied back compacted into sc/sv.
// Returns the new element total.
template <int G, int NV, bool VALS, bool FIRST, bool SMEM>
__device__ __forceinline__ int chunk_round(const Group<G>& g, int* __restrict__ sc, double* __restrict__ sv,
                                           int* __restrict__ dc, double* __restrict__ dv, const int* off,
                                           int* noff, int nl, int T, int* scan_tmp, const double* av) {
  const int npairs = (nl + 1) >> 1;
  const int VT = ((T + G - 1) / G) | 1;  // odd: conflict-free strided shared-memory access
  const int g0 = min(g.rank * VT, T), g1 = min(g0 + VT, T);
  int cnt = 0;
  int pf = 0, pl = -1;  // pairs whose output start this thread records: [pf, pl]
  Cursor c;
  c.ia = c.ib = c.lim = 0;
  c.ca = c.cb = INT_MAX;
  c.va = c.vb = c.sa = c.sb = 0.0;
  c.p = 0;
  c.as = c.bs = c.be = 0;
  if (g0 < g1) {
    int lo = 0, hi = npairs - 1;  // last pair starting at or before g0 (it is non-empty)
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off[2 * mid] <= g0)
        lo = mid;
      else
        hi = mid - 1;
    }
    c.p = lo;
    c.as = off[2 * c.p];
    c.bs = off[min(2 * c.p + 1, nl)];
    c.be = off[min(2 * c.p + 2, nl)];
    const int d = g0 - c.as;
    if (d == 0) {  // this chunk starts pair p (and any empty pairs just before it)
      pf = c.p;
      while (pf > 0 && off[2 * (pf - 1)] == g0) --pf;
      for (int q = pf; q <= c.p; ++q) noff[q] = 0;
      pl = c.p;
    }
    const int i = merge_path(sc + c.as, c.bs - c.as, sc + c.bs, c.be - c.bs, d);
    int j = d - i;
    if (i > 0 && j < c.be - c.bs && sc[c.as + i - 1] == sc[c.bs + j]) ++j;  // b[j] summed by the chunk on the left
    c.ia = c.as + i;
    c.ib = c.bs + j;
    c.lim = g1 + c.bs;  // merged position = ia + ib - bs
    cursor_load<VALS, FIRST>(c, sc, sv, av, nl);
  }
  const unsigned scb = SMEM ? smem_u32(sc) : 0u;
  const unsigned svb = (SMEM && VALS) ? smem_u32(sv) : 0u;
  constexpr int NR = NV > 0 ? NV : 1;
  int ocol[NR];
  double oval[NR];
  auto step = [&](int v) {
    const bool act = c.ia + c.ib < c.lim;
    if (act && (c.ca & c.cb) == INT_MAX) {  // pair p consumed: enter the next non-empty pair
      if (pl < 0) pf = c.p + 1;
      do {
        ++c.p;
        noff[c.p] = cnt;
        c.as = off[2 * c.p];
        c.bs = off[min(2 * c.p + 1, nl)];
        c.be = off[min(2 * c.p + 2, nl)];
      } while (c.as == c.be);
      pl = c.p;
      c.ia = c.as;
      c.ib = c.bs;
      c.lim = g1 + c.bs;
      cursor_load<VALS, FIRST>(c, sc, sv, av, nl);
    }
    const bool ta = act && c.ca <= c.cb;
    const bool tb = act && c.cb <= c.ca;
    const int oc = min(c.ca, c.cb);
    double ov = 0.0;
    if (VALS) {
      double x = FIRST ? __dmul_rn(c.sa, c.va) : c.va;  // the product, rounded once
      double y = FIRST ? __dmul_rn(c.sb, c.vb) : c.vb;
      x = ta ? x : -0.0;  // -0.0 is the exact additive identity
      y = tb ? y : -0.0;
      ov = __dadd_rn(x, y);  // "vals with duplicate cols are combined into one val"
    }
    if (NV > 0) {
      ocol[v] = oc;
      if (VALS) oval[v] = ov;
    } else if (act) {
      dc[g0 + cnt] = oc;
      if (VALS) dv[g0 + cnt] = ov;
    }
    cnt += act;
    c.ia += ta;
    c.ib += tb;
    if (SMEM) {
      lds_if(ta, scb + 4u * c.ia, c.ca);
      lds_if(tb, scb + 4u * c.ib, c.cb);
      if (VALS) {
        lds_if(ta, svb + 8u * c.ia, c.va);
        lds_if(tb, svb + 8u * c.ib, c.vb);
      }
    } else {
      if (ta) {
        c.ca = sc[c.ia];
        if (VALS) c.va = sv[c.ia];
      }
      if (tb) {
        c.cb = sc[c.ib];
        if (VALS) c.vb = sv[c.ib];
      }
    }
    c.ca = c.ia < c.bs ? c.ca : INT_MAX;
    c.cb = c.ib < c.be ? c.cb : INT_MAX;
  };
  if constexpr (NV > 0) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (v >= VT) break;  // group-uniform
      step(v);
    }
  } else {
    for (int v = 0; v < VT; ++v) step(0);
  }
  int total;
  const int base = group_excl_scan<G>(g, cnt, total, scan_tmp);
  for (int q = pf; q <= pl; ++q) noff[q] += base;
  if constexpr (NV > 0) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (v >= VT) break;
      if (v < cnt) {
        dc[base + v] = ocol[v];
        if (VALS) dv[base + v] = oval[v];
      }
    }
  } else {
    g.sync();  // every merge has finished reading sc
    for (int e = 0; e < cnt; ++e) {
      sc[base + e] = dc[g0 + e];
      if (VALS) sv[base + e] = dv[g0 + e];
    }
  }
  if (g.rank == G - 1) {
    for (int q = npairs - 1; q >= 0 && off[2 * q] == T; --q) noff[q] = total;  // trailing empty pairs
    noff[npairs] = total;
  }
  g.sync();
  return total;
}

// BRMerge of one output row by a group. NV > 0: buffers in shared memory,
// rounds ping-pong between (col0, val0) and (col1, val1); NV = 0: buffers in
// a global workspace, every round lands back in (col0, val0).
template <int G, int NV, bool VALS, int OUT>
__device__ __forceinline__ void chunk_row(const Group<G>& g, const CsrView& A, const CsrView& B, int64_t row,
                                          const RowOut& o, const ChunkBufs& cb) {
  constexpr bool SMEM = NV > 0;
  const int rank = g.rank;
  const int64_t a0 = A.rpt[row];
  const int nl = static_cast<int>(A.rpt[row + 1] - a0);
  int* sc = cb.col0;
  double* sv = cb.val0;
  int* dc = cb.col1;
  double* dv = cb.val1;
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
  // ... then the B rows themselves (unscaled; round 1 multiplies), S
  // consecutive threads per list (S ~ mean list length), coalesced.
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
        for (int e = e0; e < n; e += S) {
          if (SMEM) {
            cp_async_4(sc + o0 + e, B.col + st + e);
            if (VALS) cp_async_8(sv + o0 + e, B.val + st + e);
          } else {
            sc[o0 + e] = __ldg(B.col + st + e);
            if (VALS) sv[o0 + e] = __ldg(B.val + st + e);
          }
        }
      }
    }
    if (SMEM) cp_async_wait_all();
  }
  g.sync();
  // accumulating phase (lines 21-35)
  int cur = nl;
  bool first = true;
  while (cur > 1) {
    if (first)
      T = chunk_round<G, NV, VALS, true, SMEM>(g, sc, sv, dc, dv, off, noff, cur, T, cb.scan_tmp, cb.av);
    else
      T = chunk_round<G, NV, VALS, false, SMEM>(g, sc, sv, dc, dv, off, noff, cur, T, cb.scan_tmp, cb.av);
    first = false;
    cur = (cur + 1) >> 1;
    { int* t = off; off = noff; noff = t; }
    if (SMEM) {  // lines 33-34: swap the ping-pong buffers
      { int* t = sc; sc = dc; dc = t; }
      { double* t = sv; sv = dv; dv = t; }
    }
  }
  // line 36: the result row is list 0 of src, [0, T)
  if (OUT != OUT_SYMBOLIC) {
    const int64_t ob = o.base[row];
    const double s0 = (VALS && nl == 1) ? cb.av[0] : 1.0;  // a single list was never scaled
    for (int e = rank; e < T; e += G) {
      o.col[ob + e] = sc[e];
      if (VALS) o.val[ob + e] = nl == 1 ? __dmul_rn(s0, sv[e]) : sv[e];
    }
  }
  if (OUT != OUT_C && rank == 0) o.row_size[row] = T;
  g.sync();
}

}  // namespace brm
