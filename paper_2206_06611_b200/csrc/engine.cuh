// engine.cuh -- the BRMerge accumulation of one output row (Algorithm 1,
// PAPER.md:165-218) in four GPU forms. All compute exactly the rounds of
// Algorithm 1 -- pairs (0,1),(2,3),... of the current lists merged, an odd
// trailing list copied, equal columns combined as left + right -- so values
// are bit-identical to the paper's sequential tree order (R1).
//
// tiny_row  (tier 1, P <= 8): one thread per row runs Algorithm 1 literally,
//   its ping-pong buffers in thread-interleaved shared memory.
// reg_row   (tier 2, P <= 32): one warp; lane e holds product e; each round
//   merges list pairs in registers (shuffle rank search = warp-shuffle merge
//   path, ballot arithmetic for positions, a 32-slot shared exchange).
// rec_row   (tiers 3-6): a warp or CTA per row; rounds move records
//   {col, value slot} (32-bit packed or 8-byte) through one shared buffer,
//   values stay in place and duplicates accumulate into the left slot; each
//   round is one pass of G merge-path chunks of odd length VT; outputs wait
//   in registers until the group scan gives their compacted positions.
// chunk_row (tier 7 under BRM_HEAVY_GLOBAL): the chunk partition over
//   column/value ping-pong buffers in a global workspace, one 1024-thread CTA
//   per row. (The default heavy-row path is heavy.cuh.)
#pragma once
#include "brm_internal.cuh"

namespace brm {

enum OutKind { OUT_SYMBOLIC = 0, OUT_CBAR = 1, OUT_C = 2 };

constexpr int kHashEmpty = -1;  // empty slot of the shared hash tables (columns are >= 0)

// Mirrors (multi-GPU write-out over peer memory): under
// OUT_C every stored entry of C also goes, at the same index, into the
// peers' copies of C -- device pointers into peer memory (NVLink P2P), so the
// row blocks are assembled by the merge kernels' own stores instead of an
// all-gather after them.
constexpr int kMaxMirrors = 7;  // the peers of an 8-GPU node
struct Mirrors {
  int n;
  int32_t* col[kMaxMirrors];
  double* val[kMaxMirrors];
};
struct RowOut {
  const int64_t* base;  // OUT_CBAR: n_prod offsets; OUT_C: C.rpt
  int32_t* col;
  double* val;
  int64_t* row_size;    // OUT_SYMBOLIC / OUT_CBAR: nnz of each output row
  Mirrors mir;          // OUT_C only (n = 0: none)
};

// entry i of C into every mirror (static indices: the pointers stay kernel
// parameters); a uniform branch when there are none
template <bool VALS>
__device__ __forceinline__ void mirror_store(const Mirrors& m, int64_t i, int32_t c, double v) {
  if (m.n == 0) return;
#pragma unroll
  for (int p = 0; p < kMaxMirrors; ++p) {
    if (p < m.n) {
      m.col[p][i] = c;
      if (VALS) m.val[p][i] = v;
    }
  }
}

#ifndef BRM_OWNER_ROT
#define BRM_OWNER_ROT 4
#endif
// owner[e * ostr] = l for the products e0..e1-1 of list l, one thread per
// list. The fill starts at a different place in every list (rotation):
// lists of equal length would otherwise hit one shared-memory bank together
// (BRM_OWNER_ROT 0: no rotation, 1: by l mod n, 2: by l & 15 in two loops,
// 3: by l & 15 (0 for shorter lists) in one loop, 4: by l mod n only for
// lengths n that are multiples of 4; tuning switch). Measured (B200, same
// box): 0 -> 1 made uniform1m_k16's tier 3 14 % faster and stencil27_64's
// tier 4 2.8 % slower.
__device__ __forceinline__ void owner_fill(unsigned short* owner, int ostr, int e0, int e1, int l) {
  const unsigned short v = static_cast<unsigned short>(l);
#if BRM_OWNER_ROT == 0
  for (int e = e0; e < e1; ++e) owner[e * ostr] = v;
#elif BRM_OWNER_ROT == 1
  const int n = e1 - e0;
  int e = n > 0 ? e0 + l % n : e0;
  for (int i = 0; i < n; ++i) {
    owner[e * ostr] = v;
    if (++e == e1) e = e0;
  }
#elif BRM_OWNER_ROT == 3
  const int n = e1 - e0;
  int r = l & 15;
  if (r >= n) r = 0;
  int e = e0 + r;
  for (int i = 0; i < n; ++i) {
    owner[e * ostr] = v;
    if (++e == e1) e = e0;
  }
#elif BRM_OWNER_ROT == 4
  const int n = e1 - e0;
  if ((n & 3) == 0 && n > 0) {  // lengths that line lists up on one bank
    int e = e0 + l % n;
    for (int i = 0; i < n; ++i) {
      owner[e * ostr] = v;
      if (++e == e1) e = e0;
    }
  } else {
    for (int e = e0; e < e1; ++e) owner[e * ostr] = v;
  }
#else
  const int em = min(e1, e0 + (l & 15));
  for (int e = em; e < e1; ++e) owner[e * ostr] = v;
  for (int e = e0; e < em; ++e) owner[e * ostr] = v;
#endif
}

// Shared scratch of one register-tier (tier 2) group (G slots each).
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

// Working arrays of one global-tier row (global workspace slice). Lists of a
// round are compact in col0/val0 ("src"); col1/val1 ("dst") receive the
// merged chunks. off0 holds the current list offsets (nl + 1), off1 the
// next round's.
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

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// ===========================================================================
// Tiny tier (tier 1: P <= 8, nl <= 8): one THREAD per row runs Algorithm 1
// literally -- multiplying phase into its ping buffer, then rounds merging
// lists (0,1),(2,3),... into the pong buffer, odd trailing list copied,
// swap -- with both buffers in shared memory, thread-interleaved (slot s of
// thread t at s * NT + t: conflict-free when a warp touches equal slots).
// ===========================================================================
constexpr int kTinyP = 8;   // max n_prod of a tiny row
constexpr int kTinyL = 8;   // max num_list of a tiny row

template <int NT, bool VALS>
__host__ __device__ constexpr int tiny_block_bytes() {
  return NT * kTinyP * (4 + 4) + (VALS ? NT * kTinyP * 16 : 0);
}

template <int NT, bool VALS, int OUT>
__device__ __forceinline__ void tiny_row(const CsrView& A, const CsrView& B, int64_t row, int64_t a0, int nl,
                                         const RowOut& o, int* pc, int* qc, double* pv, double* qv) {
  // (a0 = A.rpt[row], nl = A.rpt[row + 1] - a0: loaded by the caller, one row ahead)
  // Alg. 1 lines 10-15: list l into the ping buffer at [off[l], off[l+1]);
  // the B row bounds of all lists are loaded before any list is gathered
#ifndef BRM_TINY_BATCH
#define BRM_TINY_BATCH 1  // tuning switch: 0 loads each list's bounds in the list loop
#endif
  int64_t bb[kTinyL], be[kTinyL];
  if (BRM_TINY_BATCH) {
#pragma unroll
    for (int l = 0; l < kTinyL; ++l) {
      bb[l] = be[l] = 0;
      if (l < nl) {
        const int k = __ldg(A.col + a0 + l);
        bb[l] = __ldg(B.rpt + k);
        be[l] = __ldg(B.rpt + k + 1);
      }
    }
#ifndef BRM_TINY_PREFETCH
#define BRM_TINY_PREFETCH 0  // tuning switch: 1 / 2 prefetch every list's first entry to L2 / L1 before the gather loop
#endif
    if constexpr (BRM_TINY_PREFETCH > 0) {
      // the gather loop below takes the lists one after another (a load
      // latency each); their first entries start towards the cache together
#pragma unroll
      for (int l = 0; l < kTinyL; ++l) {
        if (l < nl && bb[l] < be[l]) {
          if constexpr (BRM_TINY_PREFETCH == 1) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(B.col + bb[l]));
            if (VALS) asm volatile("prefetch.global.L2 [%0];" ::"l"(B.val + bb[l]));
          } else {
            asm volatile("prefetch.global.L1 [%0];" ::"l"(B.col + bb[l]));
            if (VALS) asm volatile("prefetch.global.L1 [%0];" ::"l"(B.val + bb[l]));
          }
        }
      }
    }
  }
  int off[kTinyL + 1];
  int P = 0;
#ifndef BRM_TINY_CPASYNC
#define BRM_TINY_CPASYNC 1  // the lists' entries staged by cp.async, all in flight at once (0: a load + store per entry, list after list)
#endif
  if constexpr (BRM_TINY_CPASYNC && BRM_TINY_BATCH) {
    // every entry of every list is copied by cp.async (4 + 8 bytes) straight
    // into its ping-buffer slot: no list waits for the one before it (the
    // plain loop below stalls on each list's load before issuing the next);
    // then the values are scaled in place, A_ik * B_kj rounded once (line 12)
#pragma unroll
    for (int l = 0; l < kTinyL; ++l) {
      off[l] = P;
      if (l < nl) {
        for (int64_t q = bb[l]; q < be[l]; ++q, ++P) {
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(pc + P * NT)), "l"(B.col + q) : "memory");
          if (VALS)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(pv + P * NT)), "l"(B.val + q) : "memory");
        }
      }
    }
    off[kTinyL] = P;
    double av[kTinyL];
#pragma unroll
    for (int l = 0; l < kTinyL; ++l) av[l] = (VALS && l < nl) ? __ldg(A.val + a0 + l) : 0.0;
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    if (VALS) {
#pragma unroll
      for (int l = 0; l < kTinyL; ++l)
        for (int e = off[l]; e < off[l + 1]; ++e) pv[e * NT] = __dmul_rn(av[l], pv[e * NT]);
    }
  } else {
#pragma unroll
  for (int l = 0; l < kTinyL; ++l) {
    off[l] = P;
    if (l < nl) {
      int64_t b0 = bb[l], b1 = be[l];
      if (!BRM_TINY_BATCH) {
        const int k = __ldg(A.col + a0 + l);
        b0 = __ldg(B.rpt + k);
        b1 = __ldg(B.rpt + k + 1);
      }
      const double a = VALS ? __ldg(A.val + a0 + l) : 0.0;
      for (int64_t q = b0; q < b1; ++q, ++P) {
        pc[P * NT] = __ldg(B.col + q);
        if (VALS) pv[P * NT] = __dmul_rn(a, __ldg(B.val + q));  // line 12: one rounding
      }
    }
  }
  off[kTinyL] = P;
  }
  // lines 21-35: rounds of pairwise merges between the two buffers
  int cur = nl;
  int n = P;
  while (cur > 1) {
    int noff[kTinyL + 1];
    int out = 0;
#pragma unroll
    for (int p = 0; p < kTinyL / 2; ++p) {
      noff[p] = out;
      if (2 * p < cur) {  // consume lists 2p and 2p+1 (empty if 2p+1 == cur: line 28 copy)
        int i = off[2 * p], j = off[2 * p + 1];
        const int ie = j, je = off[2 * p + 2];
        while (i < ie || j < je) {
          const int ci = i < ie ? pc[i * NT] : INT_MAX;
          const int cj = j < je ? pc[j * NT] : INT_MAX;
          const bool ti = ci <= cj, tj = cj <= ci;
          qc[out * NT] = ti ? ci : cj;
          if (VALS) {
            const double x = ti ? pv[i * NT] : -0.0;
            const double y = tj ? pv[j * NT] : -0.0;
            qv[out * NT] = __dadd_rn(x, y);  // "vals with duplicate cols are combined"
          }
          ++out;
          i += ti;
          j += tj;
        }
      }
    }
#pragma unroll
    for (int p = kTinyL / 2; p <= kTinyL; ++p) noff[p] = out;
#pragma unroll
    for (int p = 0; p < kTinyL / 2; ++p)
      if (2 * p + 1 >= cur + 1) noff[p] = out;  // lists past the last pair are empty
#pragma unroll
    for (int l = 0; l <= kTinyL; ++l) off[l] = noff[l];
    { int* t = pc; pc = qc; qc = t; }  // lines 33-34
    { double* t = pv; pv = qv; qv = t; }
    cur = (cur + 1) >> 1;
    n = out;
  }
  // line 36: store the result row
  if (OUT != OUT_SYMBOLIC) {
    const int64_t ob = o.base[row];  // (loading it with the row bounds measured slower: 0.1956 -> 0.2005 ms on AMG)
    for (int e = 0; e < n; ++e) {
      o.col[ob + e] = pc[e * NT];
      if (VALS) o.val[ob + e] = pv[e * NT];
      if (OUT == OUT_C) mirror_store<VALS>(o.mir, ob + e, pc[e * NT], VALS ? pv[e * NT] : 0.0);
    }
  }
  if (OUT != OUT_C) o.row_size[row] = n;
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
    if (OUT == OUT_C) mirror_store<VALS>(o.mir, ob + lane, c, v);
  }
  if (OUT != OUT_C && lane == 0) o.row_size[row] = T;
  g.sync();
}

// ===========================================================================
// Chunk tiers
// ===========================================================================
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

// Lists of a round are sentinel-terminated: list l = [off[l], off[l+1]-1)
// followed by one INT_MAX slot at off[l+1]-1. If nl is odd, the trailing
// list's empty partner is a lone sentinel at off[nl]. The round's position
// space is the src index space: pair p covers [off[2p], off[2p+2]) (the odd
// trailing pair [off[nl-1], off[nl]+1)). Merging a pair emits its merged
// list followed by ONE sentinel: the two input sentinels are equal columns
// and are consumed together, like any duplicate. Empty lists and pairs need
// no special case, and merge cursors need no bounds checks.
struct Cursor {
  int p, bs, ia, ib, lim, ca, cb;
  double va, vb, sa, sb;
};

template <bool VALS, bool FIRST>
__device__ __forceinline__ void enter_pair(Cursor& c, int p, const int* sc, const double* sv, const int* off,
                                           const double* av, int nl, int g1) {
  c.p = p;
  c.ia = off[2 * p];
  c.bs = off[2 * p + 1];  // 2p+1 == nl: the lone sentinel of an odd trailing list
  c.ib = c.bs;
  c.lim = g1 + c.bs;      // merged position = ia + ib - bs
  c.ca = sc[c.ia];
  c.cb = sc[c.ib];
  if (VALS) {
    c.va = sv[c.ia];
    c.vb = sv[c.ib];
    if (FIRST) {
      c.sa = av[2 * p];
      c.sb = 2 * p + 1 < nl ? av[2 * p + 1] : 0.0;
    }
  }
}

// One BRMerge round (Alg. 1 lines 22-34) of the global tier over the nl
// sentinel-terminated lists of sc/sv (offsets off[0..nl], global workspace).
// The round's positions are split into G chunks of VT (odd) positions; a
// thread merges its chunk into dc/dv at the chunk's own positions, then --
// once the group scan has given its compacted base -- copies it back into
// sc/sv; the next round's offsets go to noff[0..npairs]. Returns the new end
// offset (noff[npairs]).
template <int G, bool VALS, bool FIRST>
__device__ __forceinline__ int chunk_round(const Group<G>& g, int* sc, double* sv,
                                           int* dc, double* dv, const int* off,
                                           int* noff, int nl, int* scan_tmp, const double* av) {
  const int npairs = (nl + 1) >> 1;
  const int npos = off[nl] + (nl & 1);
  const int VT = ((npos + G - 1) / G) | 1;  // odd: conflict-free strided shared-memory access
  const int g0 = min(g.rank * VT, npos), g1 = min(g0 + VT, npos);
  int cnt = 0;
  int pf = 0, pl = -1;  // pairs whose output start this thread records: [pf, pl]
  Cursor c;
  c.p = 0;
  c.bs = c.ia = c.ib = c.lim = 0;
  c.ca = c.cb = INT_MAX;
  c.va = c.vb = c.sa = c.sb = 0.0;
  if (g0 < g1) {
    int lo = 0, hi = npairs - 1;  // last pair starting at or before g0
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off[2 * mid] <= g0)
        lo = mid;
      else
        hi = mid - 1;
    }
    const int p = lo;
    const int as = off[2 * p], bs = off[2 * p + 1];
    const int bend = 2 * p + 2 <= nl ? off[2 * p + 2] : off[nl] + 1;
    const int na = bs - as, nb = bend - bs;  // list lengths including the sentinels
    const int d = g0 - as;
    if (d == 0) {
      pf = pl = p;
      noff[p] = 0;
    }
    const int i = merge_path(sc + as, na, sc + bs, nb, d);
    int j = d - i;
    if (i > 0 && j < nb && sc[as + i - 1] == sc[bs + j]) ++j;  // b[j] was summed by the chunk on the left
    if (i == na) {  // pair p already finished (its two sentinels were consumed on the left)
      if (g0 + 1 < g1) {
        enter_pair<VALS, FIRST>(c, p + 1, sc, sv, off, av, nl, g1);
        pf = pl = p + 1;
        noff[p + 1] = 0;
      }
    } else {
      c.p = p;
      c.bs = bs;
      c.ia = as + i;
      c.ib = bs + j;
      c.lim = g1 + bs;
      c.ca = sc[c.ia];
      c.cb = sc[c.ib];
      if (VALS) {
        c.va = sv[c.ia];
        c.vb = sv[c.ib];
        if (FIRST) {
          c.sa = av[2 * p];
          c.sb = 2 * p + 1 < nl ? av[2 * p + 1] : 0.0;
        }
      }
    }
  }
  for (int v = 0; v < VT; ++v) {
    const bool act = c.ia + c.ib < c.lim;
    const bool ta = act && c.ca <= c.cb;
    const bool tb = act && c.cb <= c.ca;
    const int oc = min(c.ca, c.cb);
    if (act) {
      dc[g0 + cnt] = oc;
      if (VALS) {
        double x = FIRST ? __dmul_rn(c.sa, c.va) : c.va;  // the product, rounded once
        double y = FIRST ? __dmul_rn(c.sb, c.vb) : c.vb;
        x = ta ? x : -0.0;  // -0.0 is the exact additive identity
        y = tb ? y : -0.0;
        dv[g0 + cnt] = __dadd_rn(x, y);  // "vals with duplicate cols are combined into one val"
      }
    }
    cnt += act;
    c.ia += ta;
    c.ib += tb;
    if (ta) {
      c.ca = sc[c.ia];
      if (VALS) c.va = sv[c.ia];
    }
    if (tb) {
      c.cb = sc[c.ib];
      if (VALS) c.vb = sv[c.ib];
    }
    if (act && oc == INT_MAX && c.ia + c.ib < c.lim) {  // pair p done, chunk not: enter pair p+1
      if (pl < 0) pf = c.p + 1;
      pl = c.p + 1;
      noff[c.p + 1] = cnt;
      enter_pair<VALS, FIRST>(c, c.p + 1, sc, sv, off, av, nl, g1);
    }
  }
  int total;
  const int base = group_excl_scan<G>(g, cnt, total, scan_tmp);
  for (int q = pf; q <= pl; ++q) noff[q] += base;
  {
    g.sync();  // every merge has finished reading sc
    // copy back warp-cooperatively: the warp copies each of its 32 threads'
    // chunks in turn, coalesced (a thread-serial copy is latency-bound here)
    const int lane = threadIdx.x & 31;
    for (int j = 0; j < 32; ++j) {
      const int cj = __shfl_sync(0xffffffffu, cnt, j);
      const int gj = __shfl_sync(0xffffffffu, g0, j);
      const int bj = __shfl_sync(0xffffffffu, base, j);
      for (int e = lane; e < cj; e += 32) {
        sc[bj + e] = dc[gj + e];
        if (VALS) sv[bj + e] = dv[gj + e];
      }
    }
    if (g.rank == G - 1) {
      noff[npairs] = total;
      sc[total] = INT_MAX;
    }
  }
  g.sync();
  return total;
}

// ===========================================================================
// Record tiers (shared memory, tiers 3-6): the rounds move 8-byte records
// {col, slot} where `slot` names the value slot of the element's partial
// sum; values never move. A duplicate column adds the right element's
// partial sum into the left element's slot (left + right, Alg. 1's combine)
// and keeps the left slot, so after each round every record's slot holds
// the sum of its column over its subtree -- the Algorithm-1 tree order.
// ===========================================================================
__device__ __forceinline__ void lds_if(bool p, unsigned addr, int2& v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q ld.shared.v2.b32 {%0, %1}, [%2];\n\t}"
               : "+r"(v.x), "+r"(v.y)
               : "r"(addr), "r"((unsigned)p));
}

__device__ __forceinline__ void lds_if(bool p, unsigned addr, unsigned& v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.shared.b32 %0, [%1];\n\t}"
               : "+r"(v)
               : "r"(addr), "r"((unsigned)p));
}

// Record of a list element. Numeric rounds carry {col, value slot}: 8 bytes
// (RecWide) or, when the columns fit in 32 - SB bits, one 32-bit word
// col << SB | slot (RecPacked<SB>, half the shared-memory wavefronts per
// record move). Symbolic rounds carry the column only (RecCol). kSentCol is
// the sentinel's column, above every real column.
struct RecWide {
  using T = int2;
  static constexpr bool kVals = true;
  static constexpr int kBytes = 8;
  static constexpr int kSentCol = INT_MAX;
  __device__ static T make(int c, int s) { return make_int2(c, s); }
  __device__ static T sent() { return make_int2(INT_MAX, 0); }
  __device__ static int col(const T& r) { return r.x; }
  __device__ static int slot(const T& r) { return r.y; }
  __device__ static int col_at(const T* r, int i) { return reinterpret_cast<const int*>(r)[2 * i]; }  // 4-byte load
  __device__ static bool le(const T& a, const T& b) { return a.x <= b.x; }  // col(a) <= col(b)
  __device__ static bool le_at(const T* a, int i, const T* b, int j) { return col_at(a, i) <= col_at(b, j); }
  __device__ static bool is_sent(const T& r) { return r.x == INT_MAX; }
};
template <int SB>
struct RecPacked {
  using T = unsigned;
  static constexpr bool kVals = true;
  static constexpr int kBytes = 4;
  static constexpr int kSentCol = static_cast<int>(0xffffffffu >> SB);
  __device__ static T make(int c, int s) { return (static_cast<unsigned>(c) << SB) | static_cast<unsigned>(s); }
  __device__ static T sent() { return 0xffffffffu; }
  __device__ static int col(T r) { return static_cast<int>(r >> SB); }
  __device__ static int slot(T r) { return static_cast<int>(r & ((1u << SB) - 1u)); }
  __device__ static int col_at(const T* r, int i) { return col(r[i]); }
  // col(a) <= col(b) without unpacking: a <= b with b's slot bits set
  __device__ static bool le(T a, T b) { return a <= (b | ((1u << SB) - 1u)); }
  __device__ static bool le_at(const T* a, int i, const T* b, int j) { return le(a[i], b[j]); }
  __device__ static bool is_sent(T r) { return r == 0xffffffffu; }
};
struct RecCol {
  using T = int;
  static constexpr bool kVals = false;
  static constexpr int kBytes = 4;
  static constexpr int kSentCol = INT_MAX;
  __device__ static T make(int c, int) { return c; }
  __device__ static T sent() { return INT_MAX; }
  __device__ static int col(T r) { return r; }
  __device__ static int slot(T) { return 0; }
  __device__ static int col_at(const T* r, int i) { return r[i]; }
  __device__ static bool le(T a, T b) { return a <= b; }
  __device__ static bool le_at(const T* a, int i, const T* b, int j) { return a[i] <= b[j]; }
  __device__ static bool is_sent(T r) { return r == INT_MAX; }
};

// slot bits of a packed record for a tier of CAP products (slots 0..CAP-1)
__host__ __device__ constexpr int rec_slot_bits(int cap) {
  int b = 0;
  while ((1 << b) < cap) ++b;
  return b;
}
// packed records need every column of B below the sentinel's column
__host__ __device__ constexpr bool rec_pack_ok(int cap, int64_t b_cols) {
  return b_cols <= static_cast<int64_t>(0xffffffffu >> rec_slot_bits(cap));
}

struct RecBufs {
  void* rec;      // P + nl + 2 records (R::T): sentinel-terminated lists
  longlong2* lst; // per list {S index of product 0 (B index - product offset), A value bits}
  double* val;    // P value slots (products, then partial sums)
  unsigned short* owner;  // list of product e at owner[e * ostr] (multiplying phase);
  int ostr;               // laid over val (ostr 4: product e's slot) when there are values
  int* off0;
  int* off1;
  int64_t* bst;
  double* av;
  int* scan_tmp;
};

// CUR: the per-list cursor arrays bst / av (column slabs); the record tiers
// write the per-list table `lst` directly.
template <int G, int CAP, int LCAP, class R, bool CUR>
__host__ __device__ constexpr int rec_group_bytes() {
  constexpr bool VALS = R::kVals;
  return align16((CAP + LCAP + 2) * R::kBytes) + LCAP * 16 + (VALS ? align16(CAP * 8) : align16(CAP * 2)) +
         align16((LCAP + 2) * 4) * 2 + (CUR ? align16(LCAP * 8) + (VALS ? align16(LCAP * 8) : 0) : 0) +
         (G > 32 ? align16((G / 32 + 2) * 4) : 0);
}

// merge path over the columns of two record lists (R::col_at reads only the
// column of each probed record)
template <class R>
__device__ __forceinline__ int merge_path_rec(const typename R::T* a, int la, const typename R::T* b, int lb,
                                              int diag) {
  int lo = diag - lb > 0 ? diag - lb : 0;
  int hi = diag < la ? diag : la;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (R::le_at(a, mid, b, diag - 1 - mid))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// One round over the nl sentinel-terminated record lists of `rec` (offsets
// off[0..nl]); same partition as chunk_round (G chunks of VT odd positions,
// threads cross into the next pair when both sentinels merge). Outputs wait
// in registers and overwrite `rec` compacted once the group has read it.
// vote: the duplicate combine is skipped (one warp vote) when no lane of the
// warp has a duplicate -- cheaper for rounds with few repeated columns.
#ifndef BRM_PLAIN_DUP
#define BRM_PLAIN_DUP 0  // 1: plain combine in every record round (tuning switch)
#endif
#ifndef BRM_VOTE_MODE
#define BRM_VOTE_MODE 0
#endif
// 0: never vote; 1: vote chosen per round at run time; 2: per round, two
// non-inlined specialisations (tuning switch). Measured on B200: mode 1 made
// uniform1m_k16's tier 3 5 % faster and stencil27_64's tier 4 7 % slower (a
// predicate test on every step), mode 2 doubled the registers; mode 0 stays.
#if BRM_VOTE_MODE == 2
#define BRM_ROUND_INLINE __noinline__
#else
#define BRM_ROUND_INLINE __forceinline__
#endif
// PLAIN: the duplicate combine written as plain C++ (the compiler branches
// around it) instead of predicated loads: faster on rows with few
// duplicates, slower on rows with many (measured: uniform1m_k16's tier 3
// -9 %, stencil27_64's tier 4 +3.4 %); the record tiers take it for tier 3.
template <int G, int NV, class R, int VOTE, bool PLAIN = false>  // VOTE: -1 run time (vote), 0 never, 1 always
__device__ BRM_ROUND_INLINE int rec_round(const Group<G>& g, typename R::T* rec, double* val, const int* off,
                                          int* noff, int nl, int* scan_tmp, bool vote) {
  constexpr bool VALS = R::kVals;
  using T = typename R::T;
  constexpr unsigned RB = R::kBytes;
  const int npairs = (nl + 1) >> 1;
  const int npos = off[nl] + (nl & 1);
  const int VT = ((npos + G - 1) / G) | 1;
  const int g0 = min(g.rank * VT, npos), g1 = min(g0 + VT, npos);
  int pf = 0, pl = -1;
  int p = 0, bs = 0, ia = 0, ib = 0, lim = 0;
  T ra = R::sent(), rb = R::sent();
  if (g0 < g1) {
    int lo = 0, hi = npairs - 1;  // last pair starting at or before g0
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off[2 * mid] <= g0)
        lo = mid;
      else
        hi = mid - 1;
    }
    p = lo;
    const int as = off[2 * p];
    bs = off[2 * p + 1];
    const int bend = 2 * p + 2 <= nl ? off[2 * p + 2] : off[nl] + 1;
    const int na = bs - as, nb = bend - bs;
    const int d = g0 - as;
    if (d == 0) {
      pf = pl = p;
      noff[p] = 0;
    }
    const int i = merge_path_rec<R>(rec + as, na, rec + bs, nb, d);
    int j = d - i;
    if (i > 0 && j < nb && R::col_at(rec, as + i - 1) == R::col_at(rec, bs + j)) ++j;  // b[j] summed on the left
    if (i == na) {  // pair p finished on the left
      if (g0 + 1 < g1) {
        ++p;
        pf = pl = p;
        noff[p] = 0;
        ia = off[2 * p];
        bs = ib = off[2 * p + 1];
        lim = g1 + bs;
        ra = rec[ia];
        rb = rec[ib];
      }
    } else {
      ia = as + i;
      ib = bs + j;
      lim = g1 + bs;
      ra = rec[ia];
      rb = rec[ib];
    }
  }
  const unsigned recb = smem_u32(rec);
  const unsigned valb = VALS ? smem_u32(val) : 0u;
  T orec[NV];  // the chunk's outputs: the left record on ties (its slot keeps the sum)
  int cnt = 0;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    if (v >= VT) break;  // group-uniform
    const bool act = ia + ib < lim;
    const bool ta = act && R::le(ra, rb);
    const bool tb = act && R::le(rb, ra);
    const T out = ta ? ra : rb;
    orec[v] = out;
    if (VALS) {
      // equal columns: val[left] = val[left] + val[right]
      const bool dup = ta && tb && !R::is_sent(ra);
      const bool use_vote = VOTE < 0 ? vote : VOTE > 0;
      if (!use_vote || __any_sync(G < 32 ? g.mask : 0xffffffffu, dup)) {  // a uniform branch
        if constexpr (PLAIN || BRM_PLAIN_DUP) {
          if (dup) val[R::slot(ra)] = __dadd_rn(val[R::slot(ra)], val[R::slot(rb)]);
        } else {
          double x = 0.0, y = 0.0;
          lds_if(dup, valb + 8u * R::slot(ra), x);
          lds_if(dup, valb + 8u * R::slot(rb), y);
          if (dup) val[R::slot(ra)] = __dadd_rn(x, y);
        }
      }
    }
    cnt += act;
    ia += ta;
    ib += tb;
    lds_if(ta, recb + RB * ia, ra);
    lds_if(tb, recb + RB * ib, rb);
    if (act && R::is_sent(out) && ia + ib < lim) {  // pair p done, chunk not: enter pair p+1
      if (pl < 0) pf = p + 1;
      ++p;
      pl = p;
      noff[p] = cnt;
      ia = off[2 * p];
      bs = ib = off[2 * p + 1];
      lim = g1 + bs;
      ra = rec[ia];
      rb = rec[ib];
    }
  }
  int total;
  const int base = group_excl_scan<G>(g, cnt, total, scan_tmp);
  for (int q = pf; q <= pl; ++q) noff[q] += base;
  g.sync();  // every merge has finished reading rec: the outputs overwrite it in place
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    if (v >= VT) break;
    if (v < cnt) rec[base + v] = orec[v];
  }
  if (g.rank == G - 1) {
    noff[npairs] = total;
    rec[total] = R::sent();  // lone partner sentinel, used if npairs is odd
  }
  g.sync();
  return total;
}

// Multiplying phase (products of the lists, coalesced through a 16-bit
// product -> list owner table) and accumulating phase of one row's (or row
// slab's) nl lists. On entry: off[0..nl] = record offsets (list l at off[l],
// its P_l products then its sentinel), the sentinels written, rb.bst[l] = the
// B index of list l's first product, rb.av[l] = its A value. Returns the
// number T of merged records, left in rec[0..T).
// source loads: read-only path (B) or plain coherent loads (a workspace this
// kernel wrote earlier)
template <bool NC, class T>
__device__ __forceinline__ T src_ld(const T* p) {
  if constexpr (NC)
    return __ldg(p);
  else
    return *p;
}

// cbase: records carry col - cbase (the heavy-row windows pack columns
// relative to the window start, so 20 column bits serve any B.cols).
template <int G, int NV, class R, bool NC = true, bool BUILD = true, bool PLAIN = false>
__device__ __forceinline__ int rec_merge_lists(const Group<G>& g, const CsrView& B, int nl, int P, int* off,
                                               int* noff, const RecBufs& rb, int cbase = 0) {
  constexpr bool VALS = R::kVals;
  typename R::T* rec = static_cast<typename R::T*>(rb.rec);
  const int rank = g.rank;
  {
    // owner[e] = list of product e (16-bit table: nl <= 512 in these tiers),
    // filled by one thread per list; then the products are fetched coalesced
    unsigned short* owner = rb.owner;
    const int ostr = rb.ostr;
    for (int l = rank; l < nl; l += G) {
      const int e0 = off[l] - l, e1 = off[l + 1] - (l + 1);
      if (BUILD)  // {product 0's source index, A value}: one 16-byte load per product below
        rb.lst[l] = make_longlong2(rb.bst[l] - e0, VALS ? __double_as_longlong(rb.av[l]) : 0);
      owner_fill(owner, ostr, e0, e1, l);
    }
    g.sync();
#ifndef BRM_REC_CPASYNC
#define BRM_REC_CPASYNC 0  // 1: block-per-row tiers (G > 32) stage B by cp.async (A/B switch)
#endif
    if constexpr (BRM_REC_CPASYNC && G > 32 && VALS) {
      // every product's column (4 bytes) and value (8 bytes) copied by
      // cp.async straight into its record / value slot, all in flight at
      // once; then each list's entries become records {col, slot} and
      // products A_ik * B_kj (one rounding, line 12), a warp per list
      for (int e = rank; e < P; e += G) {
        const int l = owner[e * ostr];  // (read before the copy into val[e] lands on it)
        const int64_t src = rb.lst[l].x + e;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(rec + e + l)), "l"(B.col + src)
                     : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(rb.val + e)), "l"(B.val + src)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      g.sync();
      const int lane = rank & 31;
      for (int l = rank >> 5; l < nl; l += G / 32) {
        const int e0 = off[l] - l, e1 = off[l + 1] - (l + 1);
        const double a = __longlong_as_double(rb.lst[l].y);
        for (int e = e0 + lane; e < e1; e += 32) {
          const int c = *reinterpret_cast<const int*>(rec + e + l);  // the raw column (first 4 bytes)
          rec[e + l] = R::make(c - cbase, e);
          rb.val[e] = __dmul_rn(a, rb.val[e]);
        }
      }
    } else {
    // BRM_GATHER_BATCH products' loads in flight per thread (tuning switch)
#ifndef BRM_GATHER_BATCH
#define BRM_GATHER_BATCH 2
#endif
    for (int eb = rank; eb < P; eb += G * BRM_GATHER_BATCH) {
      constexpr int GB = BRM_GATHER_BATCH;
      int cg[GB], lg[GB];
      double vg[GB], ag[GB];
#pragma unroll
      for (int u = 0; u < GB; ++u) {
        const int e = eb + u * G;
        lg[u] = -1;
        cg[u] = 0;
        vg[u] = ag[u] = 0.0;
        if (e < P) {
          const int l = owner[e * ostr];  // (read before this thread overwrites val[e], which it may share)
          const longlong2 d = rb.lst[l];
          const int64_t src = d.x + e;
          lg[u] = l;
          cg[u] = src_ld<NC>(B.col + src);
          if (VALS) {
            vg[u] = src_ld<NC>(B.val + src);
            ag[u] = __longlong_as_double(d.y);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < GB; ++u) {
        const int e = eb + u * G;
        if (lg[u] >= 0) {
          rec[e + lg[u]] = R::make(cg[u] - cbase, e);
          if (VALS) rb.val[e] = __dmul_rn(ag[u], vg[u]);  // line 12: the product, rounded once
        }
      }
    }
    }
  }
  g.sync();
  // accumulating phase (lines 21-35)
  int cur = nl;
  int end = P + nl;
  // the combine of duplicates is voted away in rounds that follow a round
  // with few of them (fewer than 1 in 8 positions): adapts per row and round
  bool vote = false;
  while (cur > 1) {
    const int npos = off[cur] + (cur & 1);
#if BRM_VOTE_MODE == 0
    end = rec_round<G, NV, R, 0, PLAIN>(g, rec, rb.val, off, noff, cur, rb.scan_tmp, false);
#elif BRM_VOTE_MODE == 1
    end = rec_round<G, NV, R, -1>(g, rec, rb.val, off, noff, cur, rb.scan_tmp, vote);
#else
    if (vote)
      end = rec_round<G, NV, R, 1>(g, rec, rb.val, off, noff, cur, rb.scan_tmp, true);
    else
      end = rec_round<G, NV, R, 0>(g, rec, rb.val, off, noff, cur, rb.scan_tmp, false);
#endif
    const int dups = npos - end - ((cur + 1) >> 1);  // 2 positions -> 1 output: duplicates and sentinel pairs
    vote = 8 * dups < npos;
    cur = (cur + 1) >> 1;
    int* t = off;  // lines 33-34
    off = noff;
    noff = t;
  }
  return end - 1;  // list 0 = records [0, end - 1), then its sentinel
}

#ifndef BRM_REC_PREFETCH
#define BRM_REC_PREFETCH 0  // record tiers: L2 prefetch of up to 32 * this many entries of each list (0: none)
#endif
template <int G, int NV, class R, int OUT, bool PLAIN = false>
__device__ __forceinline__ void rec_row(const Group<G>& g, const CsrView& A, const CsrView& B, int64_t row,
                                        const RowOut& o, const RecBufs& rb) {
  constexpr bool VALS = R::kVals;
  typename R::T* rec = static_cast<typename R::T*>(rb.rec);
  const int rank = g.rank;
  const int64_t a0 = A.rpt[row];
  const int nl = static_cast<int>(A.rpt[row + 1] - a0);
  int* off = rb.off0;
  int* noff = rb.off1;
  // multiplying phase (Alg. 1 lines 10-15): list offsets (list l at record
  // off[l] = E_l + l, products E_l..), then the products themselves
  int P = 0;
  for (int lb = 0; lb < nl; lb += G) {
    const int l = lb + rank;
    int n = 0;
    int64_t st = 0;
    double av = 0.0;
    if (l < nl) {
      const int k = __ldg(A.col + a0 + l);
      st = __ldg(B.rpt + k);
      n = static_cast<int>(__ldg(B.rpt + k + 1) - st);
      if (VALS) av = __ldg(A.val + a0 + l);
      if constexpr (BRM_REC_PREFETCH > 0) {
        // the list's B entries start towards L2 now; the gather below reads
        // them after the scan, the owner fill and a group sync
        const int m = min(n, BRM_REC_PREFETCH * 32);
        for (int e = 0; e < m; e += 32) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(B.col + st + e));
          if (VALS) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(B.val + st + e));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(B.val + st + e + 16));
          }
        }
      }
    }
    int tot;
    const int ex = group_excl_scan<G>(g, n, tot, rb.scan_tmp);
    if (l < nl) {
      off[l] = P + ex + l;
      rec[P + ex + l + n] = R::sent();  // sentinel of list l
      rb.lst[l] = make_longlong2(st - (P + ex), VALS ? __double_as_longlong(av) : 0);
    }
    P += tot;
  }
  if (rank == 0) {
    off[nl] = P + nl;
    rec[P + nl] = R::sent();  // lone partner sentinel if nl is odd
  }
  g.sync();
  const int T = rec_merge_lists<G, NV, R, true, false, PLAIN>(g, B, nl, P, off, noff, rb);
  if (OUT != OUT_SYMBOLIC) {  // line 36
    const int64_t ob = o.base[row];
    for (int e = rank; e < T; e += G) {
      const typename R::T r = rec[e];
      o.col[ob + e] = R::col(r);
      double v = 0.0;
      if (VALS) o.val[ob + e] = v = rb.val[R::slot(r)];
      if (OUT == OUT_C) mirror_store<VALS>(o.mir, ob + e, R::col(r), v);
    }
  }
  if (OUT != OUT_C && rank == 0) o.row_size[row] = T;
  g.sync();
}

// BRMerge of one heavy output row by a CTA (global tier): the ping buffer
// (col0, val0) holds the sentinel-terminated lists, (col1, val1) receives a
// round's uncompacted chunks, and every round lands back in (col0, val0).
template <int G, bool VALS, int OUT>
__device__ __forceinline__ void chunk_row(const Group<G>& g, const CsrView& A, const CsrView& B, int64_t row,
                                          const RowOut& o, const ChunkBufs& cb) {
  const int rank = g.rank;
  const int64_t a0 = A.rpt[row];
  const int nl = static_cast<int>(A.rpt[row + 1] - a0);
  int* sc = cb.col0;
  double* sv = cb.val0;
  int* dc = cb.col1;
  double* dv = cb.val1;
  int* off = cb.off0;
  int* noff = cb.off1;
  // multiplying phase (Alg. 1 lines 10-15): list offsets by a group scan
  // (list l starts at product index E_l and at slot off[l] = E_l + l) ...
  int P = 0;
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
    if (l < nl) {
      off[l] = P + ex + l;
      sc[P + ex + l + n] = INT_MAX;  // sentinel of list l
    }
    P += tot;
  }
  if (rank == 0) {
    off[nl] = P + nl;
    sc[P + nl] = INT_MAX;  // lone partner sentinel if nl is odd
  }
  g.sync();
  // ... then the B rows themselves (unscaled; round 1 multiplies): a warp
  // per list, the list's products copied coalesced to its slots.
  {
    const int lane = threadIdx.x & 31, warp = rank >> 5;
    for (int l = warp; l < nl; l += G / 32) {
      const int o0 = off[l], n = off[l + 1] - 1 - o0;
      const int64_t st = cb.bst[l];
      for (int e = lane; e < n; e += 32) {
        sc[o0 + e] = __ldg(B.col + st + e);
        if (VALS) sv[o0 + e] = __ldg(B.val + st + e);
      }
    }
  }
  g.sync();
  // accumulating phase (lines 21-35)
  int cur = nl;
  int end = P + nl;
  bool first = true;
  while (cur > 1) {
    if (first)
      end = chunk_round<G, VALS, true>(g, sc, sv, dc, dv, off, noff, cur, cb.scan_tmp, cb.av);
    else
      end = chunk_round<G, VALS, false>(g, sc, sv, dc, dv, off, noff, cur, cb.scan_tmp, cb.av);
    first = false;
    cur = (cur + 1) >> 1;
    { int* t = off; off = noff; noff = t; }  // lines 33-34: the roles swap
  }
  const int T = end - 1;  // the result row: list 0 = [0, end - 1), then its sentinel
  // line 36: store the result row
  if (OUT != OUT_SYMBOLIC) {
    const int64_t ob = o.base[row];
    const double s0 = (VALS && nl == 1) ? cb.av[0] : 1.0;  // a single list was never scaled
    for (int e = rank; e < T; e += G) {
      o.col[ob + e] = sc[e];
      double v = 0.0;
      if (VALS) o.val[ob + e] = v = nl == 1 ? __dmul_rn(s0, sv[e]) : sv[e];
      if (OUT == OUT_C) mirror_store<VALS>(o.mir, ob + e, sc[e], v);
    }
  }
  if (OUT != OUT_C && rank == 0) o.row_size[row] = T;
  g.sync();
}

}  // namespace brm

namespace brm {

// ===========================================================================
// Hash symbolic phase (BRMerge-Precise step 3: "computes the
// row_size of the C matrix by the hashing method"), tiers 3-6: every product
// column of the row is inserted into a per-row shared-memory hash table
// (linear probing, atomicCAS); the row size is the number of first
// insertions. The table has H = the power of two >= P * HQ / 4 slots (per tier).
// ===========================================================================

// table of H = the power of two >= P * HQ / 4 slots (>= 64): HQ = 5 keeps the
// load factor <= 0.8 for the tiers whose rows repeat their columns; rows of
// mostly distinct columns take a sparser table (fewer, shorter probe chains)
template <int CAP, int HQ>
__host__ __device__ constexpr int hash_cap() {
  int h = 64;
  while (h < CAP * HQ / 4) h <<= 1;
  return h;
}

#ifndef BRM_HASH_CPASYNC
#define BRM_HASH_CPASYNC 0  // 1: hash symbolic with one load in flight per thread (tier 3) stages the row's columns by cp.async first (A/B switch)
#endif
// the hash loop with HB = 1 waits for a column load in every iteration (more
// loads in flight cost it registers: profiles/r02_variants); staged, all of
// the row's columns are in flight at once and the loop reads shared memory.
// Measured on B200 (profiles/r02m): uniform1m_k16's tier-3 symbolic 1.599 ->
// 1.670 ms (4 KB more shared memory per CTA: fewer resident rows), uniform2k_k8
// 0.0140 -> 0.0106 ms; off.
template <int G, int HB>
__host__ __device__ constexpr bool hash_staged() {
  return BRM_HASH_CPASYNC && HB == 1 && G <= 32;
}
struct HashBufs {
  int* stage;           // CAP columns (hash_staged only)
  int* table;           // HCAP slots
  unsigned short* owner;  // CAP: list of each product
  int* off;             // LCAP + 1 list offsets (product index)
  int64_t* bst;         // LCAP B row starts
  int* scan_tmp;
};

template <int G, int CAP, int LCAP, int HQ, bool STAGE = false>
__host__ __device__ constexpr int hash_group_bytes() {
  return align16(hash_cap<CAP, HQ>() * 4) + align16(CAP * 2) + align16((LCAP + 1) * 4) + align16(LCAP * 8) +
         (G > 32 ? align16((G / 32 + 2) * 4) : 0) + (STAGE ? align16(CAP * 4) : 0);
}

// DIRECT: insert by atomicCAS straight away; else read the slot first and
// CAS only an empty one (most products of rows that repeat their columns find
// their column already inserted)
template <int G, int CAP, int HB, int HQ, bool DIRECT>
__device__ __forceinline__ void hash_row(const Group<G>& g, const CsrView& A, const CsrView& B, int64_t row,
                                         const RowOut& o, const HashBufs& hb) {
  const int rank = g.rank;
  const int64_t a0 = A.rpt[row];
  const int nl = static_cast<int>(A.rpt[row + 1] - a0);
  constexpr bool BM = BRM_SYM_BITMAP && G <= 32;
  int P = 0;
  int cmin = INT_MAX, cmax = -1;  // BM: the row's column span (first / last column of every list)
  for (int lb = 0; lb < nl; lb += G) {
    const int l = lb + rank;
    int n = 0;
    if (l < nl) {
      const int k = __ldg(A.col + a0 + l);
      const int64_t st = __ldg(B.rpt + k);
      n = static_cast<int>(__ldg(B.rpt + k + 1) - st);
      hb.bst[l] = st;
      if (BM && n > 0) {
        cmin = min(cmin, __ldg(B.col + st));
        cmax = max(cmax, __ldg(B.col + st + n - 1));
      }
    }
    int tot;
    const int ex = group_excl_scan<G>(g, n, tot, hb.scan_tmp);
    if (l < nl) hb.off[l] = P + ex;
    P += tot;
  }
  if (rank == 0) hb.off[nl] = P;
  // Rows whose columns span at most the table's bits count with a
  // direct-mapped table instead: a bitmap over [cmin, cmax] (the hash is the
  // identity, no probing); a product is new iff it sets its bit first.
  bool use_bm = false;
  if constexpr (BM) {
    cmin = __reduce_min_sync(g.mask, cmin);
    cmax = __reduce_max_sync(g.mask, cmax);
    use_bm = cmax >= 0 && cmax - cmin < hash_cap<CAP, HQ>() * 32;
  }
  // a column's slot is the HIGH bits of its multiplicative hash (the low bits
  // of c * K follow c's low bits, which cluster for structured rows: the
  // stencil's symbolic pass ran 2.7x slower with them)
  int H = 64, hbits = 6;
  while (H < P * HQ / 4) {
    H <<= 1;
    ++hbits;
  }
  if (use_bm) {
    for (int e = rank; e < (((cmax - cmin) >> 7) + 1); e += G) reinterpret_cast<int4*>(hb.table)[e] = make_int4(0, 0, 0, 0);
  } else {
    for (int e = rank; e < (H >> 2); e += G)
      reinterpret_cast<int4*>(hb.table)[e] = make_int4(kHashEmpty, kHashEmpty, kHashEmpty, kHashEmpty);
  }
  g.sync();
  for (int l = rank; l < nl; l += G) owner_fill(hb.owner, 1, hb.off[l], hb.off[l + 1], l);
  g.sync();
  int cnt = 0;
  constexpr bool STAGE = hash_staged<G, HB>();
  if constexpr (STAGE) {
    // every column of the row copied to shared memory by cp.async; a thread
    // hashes the entries it copied (no other thread's copies are read)
    for (int e = rank; e < P; e += G) {
      const int l = hb.owner[e];
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(hb.stage + e)),
                   "l"(B.col + hb.bst[l] + (e - hb.off[l]))
                   : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  }
  // HB column loads in flight per thread before they are hashed
  for (int eb = rank; eb < P; eb += G * HB) {
    int cc[HB];
#pragma unroll
    for (int u = 0; u < HB; ++u) {
      const int e = eb + u * G;
      cc[u] = -1;
      if (e < P) {
        if constexpr (STAGE) {
          cc[u] = hb.stage[e];
        } else {
          const int l = hb.owner[e];
          cc[u] = __ldg(B.col + hb.bst[l] + (e - hb.off[l]));
        }
      }
    }
    if (use_bm) {
      const volatile unsigned* bv = reinterpret_cast<const volatile unsigned*>(hb.table);
#pragma unroll
      for (int u = 0; u < HB; ++u) {
        const int c = cc[u];
        if (c < 0) continue;
        const int rel = c - cmin;
        const unsigned bit = 1u << (rel & 31);
        if (!(bv[rel >> 5] & bit))  // a set bit is final: only a clear one is claimed
          cnt += !(atomicOr(reinterpret_cast<unsigned*>(hb.table) + (rel >> 5), bit) & bit);
      }
      continue;
    }
#pragma unroll
    for (int u = 0; u < HB; ++u) {
      const int c = cc[u];
      if (c < 0) continue;
      unsigned h = (static_cast<unsigned>(c) * 2654435761u) >> (32 - hbits);
      if constexpr (DIRECT) {
        while (true) {
          const int cur = atomicCAS(&hb.table[h], kHashEmpty, c);
          if (cur == kHashEmpty) {
            ++cnt;
            break;
          }
          if (cur == c) break;
          h = (h + 1) & (H - 1);
        }
      } else {
        // a plain load first (keys are never removed, so a non-empty slot read is final)
        const volatile int* tv = hb.table;
        while (true) {
          int cur = tv[h];
          if (cur == kHashEmpty) {
            cur = atomicCAS(&hb.table[h], kHashEmpty, c);
            if (cur == kHashEmpty) {
              ++cnt;
              break;
            }
          }
          if (cur == c) break;
          h = (h + 1) & (H - 1);
        }
      }
    }
  }
  int total;
  group_excl_scan<G>(g, cnt, total, hb.scan_tmp);
  if (rank == 0) o.row_size[row] = total;
  g.sync();
}

}  // namespace brm
