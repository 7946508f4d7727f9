// engine.cuh -- the BRMerge accumulation of one output row by a thread group
// (Algorithm 1), parallelised for a GPU:
//
//   multiplying phase (lines 10-15): the B rows selected by A_i* are copied
//     into the ping buffer as sorted intermediate lists. Shared-memory tiers
//     stage each list with ONE TMA bulk copy per array (cp.async.bulk on the
//     16-byte-aligned window around the B row, completion on an mbarrier);
//     where alignment or capacity forbids it, per-element cp.async is used.
//     The scaling by A_ik is fused into the first merge round (the product is
//     rounded once, exactly as in Alg. 1 line 12).
//   accumulating phase (lines 21-35): ceil(log2 num_list) rounds; round r
//     merges lists (0,1),(2,3),... of src into dst, an odd trailing list is
//     copied, then src/dst swap. A round is cut into chunks of VT merged
//     positions that never straddle a pair (chunk -> pair table, no search);
//     one thread merges one chunk: merge-path split inside the pair, then VT
//     branch-free merge steps into registers summing equal columns (Fig. 2).
//     A duplicate whose halves straddle a chunk boundary is taken by the left
//     chunk (look-ahead) and skipped by the right one. Each thread runs two
//     chunks interleaved (ILP). A group exclusive scan of the per-chunk output
//     counts gives every output its compacted dst position -- exactly Alg. 1's
//     sequential layout ("consume two lists and store to dst_buffer") -- and
//     the next round's list offsets.
//
// The same code runs with the buffers in shared memory (tiers 1-5) or in a
// global-memory workspace (tier 6); the SMEM template flag and the pointers
// decide.
#pragma once
#include "brm_internal.cuh"

namespace brm {

enum OutKind { OUT_SYMBOLIC = 0, OUT_CBAR = 1, OUT_C = 2 };

struct RowOut {
  const int64_t* base;  // OUT_CBAR: n_prod offsets; OUT_C: C.rpt
  int32_t* col;
  double* val;
  int64_t* row_size;    // OUT_SYMBOLIC / OUT_CBAR: nnz of each output row
  int strategy;          // round strategy: 0 cost model, 1 one thread per pair, 2 chunked
  unsigned long long* prof;  // optional cycle counters (kProf*), null = off
};

// Device cycle counters (env BRM_PROFILE=1): summed over groups, lane 0 of
// each group samples clock64() at phase boundaries.
enum ProfSlot { kProfStage = 0, kProfSeq = 1, kProfChunk = 2, kProfStore = 3, kProfSeqRounds = 4,
                kProfChunkRounds = 5, kProfRows = 6, kProfSlots = 8 };

// Working arrays of one row group. A list is (start, len) in a column buffer
// and is followed by one INT_MAX sentinel column, so merge cursors need no
// bounds checks. Lists of a round lie in increasing start order.
struct RowBufs {
  int* colA;
  int* colB;
  double* valA;
  double* valB;
  int* lstA;   // list starts, ping side (round 1: staged columns in colA)
  int* llnA;   // list lengths, ping side
  int* lstB;   // list starts, pong side
  int* llnB;   // list lengths, pong side
  int* vb;     // round 1: start of list l's values in valA
  int* cst;    // chunk table: first chunk of each pair
  int* cpair;  // chunk table: pair of each chunk
  unsigned long long* mbar;
  int* scan_tmp;
  int capc, capv;  // capacities of colA / valA (TMA windows need padding)
};


// ---------------------------------------------------------------------------
// async-copy primitives (sm_90+ PTX; SASS UBLKCP / LDGSTS / SYNCS)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async_4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void mbar_init(unsigned long long* m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* m, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* m) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(m))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(m)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_bulk_g2s(void* smem, const void* gmem, unsigned bytes, unsigned long long* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem)),
               "l"(gmem), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}

// ---------------------------------------------------------------------------
// Group reductions (sum and max of one int per thread).
// ---------------------------------------------------------------------------
template <int G>
__device__ __forceinline__ void group_sum_max(const Group<G>& g, int s, int m, int& sum, int& mx, int* tmp) {
  if constexpr (G <= 32) {
    sum = __reduce_add_sync(g.mask, s);
    mx = __reduce_max_sync(g.mask, m);
  } else {
    const int ws = __reduce_add_sync(0xffffffffu, s);
    const int wm = __reduce_max_sync(0xffffffffu, m);
    if (threadIdx.x == 0) {
      tmp[0] = 0;
      tmp[1] = 0;
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(&tmp[0], ws);
      atomicMax(&tmp[1], wm);
    }
    __syncthreads();
    sum = tmp[0];
    mx = tmp[1];
    __syncthreads();
  }
}

// Lengths of pair p (lists 2p, 2p+1; an odd trailing list has an empty
// partner). A list is [lst, lend) with its sentinel at lend.
__device__ __forceinline__ void pair_lens(const int* lst, const int* lend, int nl, int p, int& la, int& lb) {
  la = lend[2 * p] - lst[2 * p];
  lb = 2 * p + 1 < nl ? lend[2 * p + 1] - lst[2 * p + 1] : 0;
}

// ---------------------------------------------------------------------------
// Strategy S1: one thread merges one whole pair sequentially (Fig. 2's
// merge loop) -- no search, no scan; used when a round has many short pairs.
// ---------------------------------------------------------------------------
template <bool FIRST, bool VALS>
__device__ __forceinline__ int seq_merge(const int* sc, const double* sv, int pa, int pb, int qa, int qb, double sa,
                                         double sb, int* dc, double* dv, int out) {
  int ca = sc[pa], cb = sc[pb];
  const int o0 = out;
  while ((ca & cb) != INT_MAX) {  // both exhausted iff both heads are the sentinel
    const bool ta = ca <= cb;
    const bool tbb = cb <= ca;
    dc[out] = min(ca, cb);
    if (VALS) {
      double x = -0.0, y = -0.0;
      if (ta) x = FIRST ? __dmul_rn(sa, sv[qa]) : sv[pa];
      if (tbb) y = FIRST ? __dmul_rn(sb, sv[qb]) : sv[pb];
      dv[out] = __dadd_rn(x, y);  // "vals with duplicate cols are combined"
    }
    ++out;
    pa += ta;
    pb += tbb;
    if (FIRST) {
      qa += ta;
      qb += tbb;
    }
    if (ta) ca = sc[pa];
    if (tbb) cb = sc[pb];
  }
  dc[out] = INT_MAX;
  return out - o0;
}

template <int G, bool FIRST, bool VALS>
__device__ __forceinline__ int round_seq(const Group<G>& g, const RowBufs& rb, const int* sc, const double* sv,
                                         const int* lst, const int* lln, int nl, int* dc, double* dv, int* dst_st,
                                         int* dst_ln, const double* aval) {
  const int npairs = (nl + 1) >> 1;
  int run = 0;
  for (int qb0 = 0; qb0 < npairs; qb0 += G) {
    const int q = qb0 + g.rank;
    int la = 0, lb = 0;
    if (q < npairs) pair_lens(lst, lln, nl, q, la, lb);
    int tot;
    const int pre = group_excl_scan<G>(g, la + lb, tot, rb.scan_tmp);
    if (q < npairs) {
      const int ac = lst[2 * q];
      const int bc = 2 * q + 1 < nl ? lst[2 * q + 1] : ac + la;  // empty partner: a's sentinel
      int av = 0, bv = 0;
      double sa = 1.0, sb = 1.0;
      if (FIRST && VALS) {
        av = rb.vb[2 * q];
        bv = 2 * q + 1 < nl ? rb.vb[2 * q + 1] : av;
        sa = aval[2 * q];
        sb = 2 * q + 1 < nl ? aval[2 * q + 1] : 0.0;
      }
      const int pos = run + pre + q;  // upper-bound layout: pair q gets la + lb + 1 slots
      const int n = seq_merge<FIRST, VALS>(sc, sv, ac, bc, av, bv, sa, sb, dc, dv, pos);
      dst_st[q] = pos;
      dst_ln[q] = pos + n;
    }
    run += tot;
  }
  g.sync();
  return run;
}

// ---------------------------------------------------------------------------
// Strategy S2: chunks of VT merged positions (never straddling a pair), one
// merge-path split per chunk, two chunks per thread interleaved, outputs
// compacted over the whole round by a group scan.
// ---------------------------------------------------------------------------
template <int G, int VT>
__device__ __forceinline__ void build_chunks(const Group<G>& g, const int* lst, const int* lln, int nl, int npairs,
                                             int* cst, int* cpair, int* scan_tmp) {
  int run = 0;
  for (int pb = 0; pb < npairs; pb += G) {
    const int p = pb + g.rank;
    int c = 0;
    if (p < npairs) {
      int la, lb;
      pair_lens(lst, lln, nl, p, la, lb);
      c = (la + lb + VT - 1) / VT;
    }
    int tot;
    const int ex = group_excl_scan<G>(g, c, tot, scan_tmp);
    if (p < npairs) {
      cst[p] = run + ex;
      for (int q = 0; q < c; ++q) cpair[run + ex + q] = p;
    }
    run += tot;
  }
  if (g.rank == 0) cst[npairs] = run;
  g.sync();
}

// Merge state of one chunk: columns at sc[pa] / sc[pb] (physical cursors),
// values at sv[qa] / sv[qb]; merged position d of the next element, end dend.
struct Chunk {
  int pa, pb, qa, qb, d, dend, ca, cb, cnt, pair, pair_first;
  double sa, sb;
};

template <int VT, bool FIRST, bool VALS>
__device__ __forceinline__ void chunk_setup(Chunk& c, int t, int T, const int* sc, const int* lst, const int* lln,
                                            int nl, const RowBufs& rb, const double* aval) {
  c.cnt = 0;
  c.pair_first = -1;
  c.pair = 0;
  c.d = 0;
  c.dend = 0;  // inactive
  c.pa = c.pb = c.qa = c.qb = 0;
  c.ca = c.cb = INT_MAX;
  c.sa = c.sb = 1.0;
  if (t >= T) return;
  const int p = rb.cpair[t];
  const int k = t - rb.cst[p];
  int la, lb;
  pair_lens(lst, lln, nl, p, la, lb);
  const int ac = lst[2 * p];
  const int bc = 2 * p + 1 < nl ? lst[2 * p + 1] : ac + la;
  int av = ac, bv = bc;
  if (FIRST && VALS) {
    av = rb.vb[2 * p];
    bv = 2 * p + 1 < nl ? rb.vb[2 * p + 1] : av;
    c.sa = aval[2 * p];
    c.sb = 2 * p + 1 < nl ? aval[2 * p + 1] : 0.0;
  }
  c.pair = p;
  c.d = k * VT;
  c.dend = min(c.d + VT, la + lb);
  int i = merge_path(sc + ac, la, sc + bc, lb, c.d);
  int j = c.d - i;
  if (i > 0 && j < lb && sc[ac + i - 1] == sc[bc + j]) {
    ++j;  // b[j] duplicates a[i-1]: summed by the chunk to the left
    ++c.d;
  }
  c.pa = ac + i;
  c.pb = bc + j;
  c.qa = av + i;
  c.qb = bv + j;
  c.ca = sc[c.pa];
  c.cb = sc[c.pb];
  if (k == 0) c.pair_first = p;
}

// One branch-free merge step: emits min(ca, cb); on equal columns the two
// values are summed ("vals with duplicate cols are combined into one val").
// The value of a list not taken is -0.0, the exact additive identity, so the
// emitted value is bitwise x, y or x + y. Only consumed heads are reloaded.
template <bool FIRST, bool VALS>
__device__ __forceinline__ void chunk_step(Chunk& c, const int* sc, const double* sv, int& ocol, double& oval) {
  const bool act = c.d < c.dend;
  const bool ta = act && c.ca <= c.cb;
  const bool tbb = act && c.cb <= c.ca;
  ocol = min(c.ca, c.cb);
  if (VALS) {
    double x = -0.0, y = -0.0;
    if (ta) x = sv[FIRST ? c.qa : c.pa];
    if (tbb) y = sv[FIRST ? c.qb : c.pb];
    if (FIRST) {
      if (ta) x = __dmul_rn(c.sa, x);
      if (tbb) y = __dmul_rn(c.sb, y);
    }
    oval = __dadd_rn(x, y);
  }
  c.pa += ta;
  c.pb += tbb;
  if (FIRST) {
    c.qa += ta;
    c.qb += tbb;
  }
  c.d += (int)ta + (int)tbb;
  c.cnt += act;
  if (ta) c.ca = sc[c.pa];
  if (tbb) c.cb = sc[c.pb];
}

template <int G, int VT, bool FIRST, bool VALS>
__device__ __forceinline__ int round_chunked(const Group<G>& g, const RowBufs& rb, const int* sc, const double* sv,
                                             const int* lst, const int* lln, int nl, int T, int* dc, double* dv,
                                             int* dst_st, int* dst_ln, const double* aval) {
  const int npairs = (nl + 1) >> 1;
  build_chunks<G, VT>(g, lst, lln, nl, npairs, rb.cst, rb.cpair, rb.scan_tmp);
  int out_base = 0;
  for (int tb = 0; tb < T; tb += 2 * G) {
    Chunk c0, c1;
    const int t0 = tb + g.rank, t1 = tb + G + g.rank;
    chunk_setup<VT, FIRST, VALS>(c0, t0, T, sc, lst, lln, nl, rb, aval);
    chunk_setup<VT, FIRST, VALS>(c1, t1, T, sc, lst, lln, nl, rb, aval);
    int ocol0[VT], ocol1[VT];
    double oval0[VT], oval1[VT];
#pragma unroll
    for (int v = 0; v < VT; ++v) {
      chunk_step<FIRST, VALS>(c0, sc, sv, ocol0[v], oval0[v]);
      chunk_step<FIRST, VALS>(c1, sc, sv, ocol1[v], oval1[v]);
    }
    // packed scan: low 16 bits chunk t0, high 16 bits chunk t1
    int total;
    const int ex = group_excl_scan<G>(g, c0.cnt | (c1.cnt << 16), total, rb.scan_tmp);
    const int vbase0 = out_base + (ex & 0xffff);  // compacted (virtual) positions
    const int vbase1 = out_base + (total & 0xffff) + (ex >> 16);
    const int base0 = vbase0 + c0.pair;  // physical: one sentinel per earlier pair
    const int base1 = vbase1 + c1.pair;
#pragma unroll
    for (int v = 0; v < VT; ++v) {
      if (v < c0.cnt) {
        dc[base0 + v] = ocol0[v];
        if (VALS) dv[base0 + v] = oval0[v];
      }
      if (v < c1.cnt) {
        dc[base1 + v] = ocol1[v];
        if (VALS) dv[base1 + v] = oval1[v];
      }
    }
    // the last chunk of a pair writes the pair's sentinel and end
    if (t0 < T && t0 + 1 == rb.cst[c0.pair + 1]) {
      dc[base0 + c0.cnt] = INT_MAX;
      dst_ln[c0.pair] = base0 + c0.cnt;
    }
    if (t1 < T && t1 + 1 == rb.cst[c1.pair + 1]) {
      dc[base1 + c1.cnt] = INT_MAX;
      dst_ln[c1.pair] = base1 + c1.cnt;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int pf = h ? c1.pair_first : c0.pair_first;
      if (pf >= 0) {  // this pair's start; empty pairs just before it
        const int vb = h ? vbase1 : vbase0;
        int q = pf;
        const int k0 = rb.cst[q];
        dst_st[q] = vb + q;
        while (q > 0 && rb.cst[q - 1] == k0) {
          --q;
          dst_st[q] = dst_ln[q] = vb + q;
          dc[vb + q] = INT_MAX;  // sentinel of the empty pair q
        }
      }
    }
    out_base += (total & 0xffff) + (total >> 16);
  }
  if (g.rank == 0) {  // trailing empty pairs
    for (int q = npairs - 1; q >= 0 && rb.cst[q] == T; --q) {
      dst_st[q] = dst_ln[q] = out_base + q;
      dc[out_base + q] = INT_MAX;
    }
  }
  g.sync();
  return out_base;
}

// One BRMerge round (Alg. 1 lines 22-34): lists (0,1),(2,3),... of src merged
// into dst, an odd trailing list copied. Picks S1 or S2 by estimated cost.
template <int G, int VT, bool FIRST, bool VALS>
__device__ __forceinline__ int merge_round(const Group<G>& g, const RowBufs& rb, const int* sc, const double* sv,
                                           const int* lst, const int* lln, int nl, int* dc, double* dv,
                                           int* dst_st, int* dst_ln, const double* aval, int strategy,
                                           unsigned long long* acc) {
  const int npairs = (nl + 1) >> 1;
  int csum = 0, lmax = 0;
  {
    int cs = 0, lm = 0;
    for (int pb = 0; pb < npairs; pb += G) {
      const int p = pb + g.rank;
      if (p < npairs) {
        int la, lb;
        pair_lens(lst, lln, nl, p, la, lb);
        cs += (la + lb + VT - 1) / VT;
        lm = max(lm, la + lb);
      }
    }
    group_sum_max<G>(g, cs, lm, csum, lmax, rb.scan_tmp);
  }
  // latency model (cycles): a sequential step ~ kSeqStep, a chunk pass ~ kChunkIter
  const int seq_cost = lmax * (VALS ? 120 : 90) * ((npairs + G - 1) / G);
  const int chunk_cost = 1500 + ((csum + 2 * G - 1) / (2 * G)) * (VALS ? 3000 : 2400);
  const bool seq = strategy == 1 || (strategy == 0 && seq_cost <= chunk_cost);
  const long long t0 = acc ? clock64() : 0;
  int r;
  if (seq)
    r = round_seq<G, FIRST, VALS>(g, rb, sc, sv, lst, lln, nl, dc, dv, dst_st, dst_ln, aval);
  else
    r = round_chunked<G, VT, FIRST, VALS>(g, rb, sc, sv, lst, lln, nl, csum, dc, dv, dst_st, dst_ln, aval);
  if (acc) {
    acc[seq ? kProfSeq : kProfChunk] += clock64() - t0;
    acc[seq ? kProfSeqRounds : kProfChunkRounds] += 1;
  }
  return r;
}

// BRMerge of output row `row` (n_prod P) by group g.
// SMEM: buffers in shared memory (TMA / cp.async staging); phase: mbarrier
// parity of this group, toggled once per row.
template <int G, int VT, bool VALS, int OUT, bool SMEM>
__device__ __forceinline__ void process_row(const Group<G>& g, const CsrView& A, const CsrView& B, int64_t bnnz,
                                            int64_t row, int P, const RowOut& o, const RowBufs& rb,
                                            unsigned& phase, unsigned long long* acc) {
  const long long tp0 = acc ? clock64() : 0;
  const int64_t a0 = A.rpt[row];
  const int nl = static_cast<int>(A.rpt[row + 1] - a0);
  const double* aval = VALS ? A.val + a0 : nullptr;
  // TMA staging: every list's 16-byte window (+ room for its sentinel) must
  // fit the padded capacity and B's arrays must be 16-byte aligned
  const bool tma = SMEM && P + 7 * nl <= rb.capc && (!VALS || P + 2 * nl <= rb.capv) &&
                   ((reinterpret_cast<uintptr_t>(B.col) | (VALS ? reinterpret_cast<uintptr_t>(B.val) : 0)) & 15) == 0;
  if (tma) fence_proxy_async();  // order the previous row's generic accesses before async writes
  // multiplying phase (Alg. 1 lines 10-15): list l = B row k_l; each lane
  // computes its lists' lengths and staging positions and issues their copies
  int run = 0, runc = 0, runv = 0;
  for (int lbase = 0; lbase < nl; lbase += G) {
    const int l = lbase + g.rank;
    int len = 0, wc = 0, wv = 0;
    int64_t s = 0, wsc = 0, wsv = 0;
    if (l < nl) {
      const int k = A.col[a0 + l];
      s = B.rpt[k];
      len = static_cast<int>(B.rpt[k + 1] - s);
      wsc = wsv = s;
      if (tma) {
        wsc = s & ~3ll;
        wc = static_cast<int>(((s + len + 4) & ~3ll) - wsc);  // >= one slot after the list
        if (len > 0) {
          wsv = s & ~1ll;
          wv = static_cast<int>(((s + len + 1) & ~1ll) - wsv);
        }
      }
    }
    int tot;
    const int ex = group_excl_scan<G>(g, len, tot, rb.scan_tmp);
    int pex = 0, ptot = 0;
    if (tma) pex = group_excl_scan<G>(g, wc | (wv << 16), ptot, rb.scan_tmp);
    if (l < nl) {
      if (tma) {
        const int pc = runc + (pex & 0xffff), pv = runv + (pex >> 16);
        rb.lstA[l] = pc + static_cast<int>(s - wsc);
        rb.llnA[l] = pc + static_cast<int>(s - wsc) + len;
        if (VALS) rb.vb[l] = pv + static_cast<int>(s - wsv);
        if (len > 0) {
          // one bulk copy per array if the window stays inside B's arrays,
          // else element-wise cp.async into the same window positions
          const bool bulk_c = wsc + wc <= bnnz;
          const bool bulk_v = !VALS || wsv + wv <= bnnz;
          const unsigned bytes = (bulk_c ? wc * 4u : 0u) + (VALS && bulk_v ? wv * 8u : 0u);
          if (bytes) mbar_expect_tx(rb.mbar, bytes);
          if (bulk_c)
            tma_bulk_g2s(rb.colA + pc, B.col + wsc, wc * 4u, rb.mbar);
          else
            for (int e = 0; e < len; ++e) cp_async_4(rb.colA + pc + (s - wsc) + e, B.col + s + e);
          if (VALS) {
            if (bulk_v)
              tma_bulk_g2s(rb.valA + pv, B.val + wsv, wv * 8u, rb.mbar);
            else
              for (int e = 0; e < len; ++e) cp_async_8(rb.valA + pv + (s - wsv) + e, B.val + s + e);
          }
        }
      } else {
        rb.lstA[l] = run + ex + l;  // contiguous lists, one sentinel slot each
        rb.llnA[l] = run + ex + l + len;
        if (VALS) rb.vb[l] = run + ex + l;
      }
    }
    run += tot;
    if (tma) {
      runc += ptot & 0xffff;
      runv += ptot >> 16;
    }
  }
  g.sync();
  if (tma) {
    if (g.rank == 0) mbar_arrive(rb.mbar);
    cp_async_wait_all();
    mbar_wait(rb.mbar, phase);
    phase ^= 1u;
  } else {
    const bool per_list_group = P * 2 >= nl * G;
    for (int l = per_list_group ? 0 : g.rank; l < nl; l += per_list_group ? 1 : G) {
      const int dst = rb.lstA[l], n = rb.llnA[l] - rb.lstA[l];
      if (!n) continue;
      const int64_t s = B.rpt[A.col[a0 + l]];
      for (int e = per_list_group ? g.rank : 0; e < n; e += per_list_group ? G : 1) {
        if (SMEM) {
          cp_async_4(rb.colA + dst + e, B.col + s + e);
          if (VALS) cp_async_8(rb.valA + dst + e, B.val + s + e);
        } else {
          rb.colA[dst + e] = B.col[s + e];
          if (VALS) rb.valA[dst + e] = B.val[s + e];
        }
      }
    }
    if (SMEM) cp_async_wait_all();
  }
  g.sync();
  for (int l = g.rank; l < nl; l += G) rb.colA[rb.llnA[l]] = INT_MAX;  // sentinels
  g.sync();
  if (acc) acc[kProfStage] += clock64() - tp0;
  // accumulating phase (Alg. 1 lines 21-35)
  int* sc = rb.colA;
  double* sv = rb.valA;
  int* lst = rb.lstA;
  int* lln = rb.llnA;
  int* dc = rb.colB;
  double* dv = rb.valB;
  int* dst_st = rb.lstB;
  int* dst_ln = rb.llnB;
  int n_out = P;
  if (nl >= 2) {
    int cur = nl;
    n_out = merge_round<G, VT, true, VALS>(g, rb, sc, sv, lst, lln, cur, dc, dv, dst_st, dst_ln, aval, o.strategy,
                                           acc);
    cur = (cur + 1) >> 1;
    { int* t = sc; sc = dc; dc = t; }
    { double* t = sv; sv = dv; dv = t; }
    { int* t = lst; lst = dst_st; dst_st = t; }
    { int* t = lln; lln = dst_ln; dst_ln = t; }
    while (cur > 1) {
      n_out = merge_round<G, VT, false, VALS>(g, rb, sc, sv, lst, lln, cur, dc, dv, dst_st, dst_ln, nullptr,
                                              o.strategy, acc);
      cur = (cur + 1) >> 1;
      { int* t = sc; sc = dc; dc = t; }
      { double* t = sv; sv = dv; dv = t; }
      { int* t = lst; lst = dst_st; dst_st = t; }
      { int* t = lln; lln = dst_ln; dst_ln = t; }
    }
    n_out = lln[0] - lst[0];  // S1 rounds return the upper bound, the list length is exact
  }
  // Alg. 1 line 36: store the result row (list 0 of the last round)
  const long long ts0 = acc ? clock64() : 0;
  if (OUT != OUT_SYMBOLIC) {
    const int64_t dst = o.base[row];
    const int c0 = lst[0];
    if (nl == 1) {  // single list: the scaled B row is the result
      const double s0 = VALS ? aval[0] : 0.0;
      const int v0 = VALS ? rb.vb[0] : 0;
      for (int e = g.rank; e < n_out; e += G) {
        o.col[dst + e] = sc[c0 + e];
        if (VALS) o.val[dst + e] = __dmul_rn(s0, sv[v0 + e]);
      }
    } else {
      for (int e = g.rank; e < n_out; e += G) {
        o.col[dst + e] = sc[c0 + e];
        if (VALS) o.val[dst + e] = sv[c0 + e];
      }
    }
  }
  if (OUT != OUT_C && g.rank == 0) o.row_size[row] = n_out;
  g.sync();
  if (acc) {
    acc[kProfStore] += clock64() - ts0;
    acc[kProfRows] += 1;
  }
}

}  // namespace brm
