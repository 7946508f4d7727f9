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
};

// Working arrays of one row group.
struct RowBufs {
  int* colA;
  int* colB;
  double* valA;
  double* valB;
  int* cb;     // round 1: start of list l's columns in colA
  int* vb;     // round 1: start of list l's values in valA
  int* offA;   // list offsets (virtual, contiguous), ping
  int* offB;   // list offsets, pong
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
// Chunk table of a round: cst[p] = first chunk of pair p (cst[npairs] =
// total), cpair[t] = pair of chunk t.
// ---------------------------------------------------------------------------
template <int G, int VT>
__device__ __forceinline__ int build_chunks(const Group<G>& g, const int* so, int nl, int npairs, int* cst,
                                            int* cpair, int* scan_tmp) {
  int run = 0;
  for (int pb = 0; pb < npairs; pb += G) {
    const int p = pb + g.rank;
    int c = 0;
    if (p < npairs) {
      const int len = so[min(2 * p + 2, nl)] - so[2 * p];
      c = (len + VT - 1) / VT;
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
  return run;
}

// Buffer layout: every list is followed by one INT_MAX sentinel column, so a
// merge cursor needs no bounds check (an exhausted list reads INT_MAX). In the
// contiguous rounds list l starts at physical index off[l] + l (one sentinel
// slot per preceding list); round 1 uses the staged positions cb[l] / vb[l].

// Merge state of one chunk: columns at sc[pa] / sc[pb] (physical cursors),
// values at sv[qa] / sv[qb]; merged position d of the next element, end dend.
struct Chunk {
  int pa, pb, qa, qb, d, dend, ca, cb, cnt, pair, pair_first;
  double sa, sb;
};

template <int VT, bool FIRST, bool VALS>
__device__ __forceinline__ void chunk_setup(Chunk& c, int t, int T, const int* sc, const int* so, int nl,
                                            const int* cst, const int* cpair, const int* cb, const int* vb,
                                            const double* aval) {
  c.cnt = 0;
  c.pair_first = -1;
  c.pair = 0;
  c.d = 0;
  c.dend = 0;  // inactive
  c.pa = c.pb = c.qa = c.qb = 0;
  c.ca = c.cb = INT_MAX;
  c.sa = c.sb = 1.0;
  if (t >= T) return;
  const int p = cpair[t];
  const int k = t - cst[p];
  const int s0 = so[2 * p];
  const int s1 = so[min(2 * p + 1, nl)];
  const int s2 = so[min(2 * p + 2, nl)];
  const int la = s1 - s0, lb = s2 - s1;
  int ac, bc, av = 0, bv = 0;
  if (FIRST) {
    ac = cb[2 * p];
    if (VALS) av = vb[2 * p];
    if (2 * p + 1 < nl) {
      bc = cb[2 * p + 1];
      if (VALS) bv = vb[2 * p + 1];
    } else {
      bc = ac + la;  // empty partner: a's sentinel
      bv = av;
    }
  } else {
    ac = av = s0 + 2 * p;
    bc = bv = (2 * p + 1 < nl) ? s1 + 2 * p + 1 : ac + la;
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
  if (FIRST && VALS) {
    c.sa = aval[2 * p];
    c.sb = (2 * p + 1 < nl) ? aval[2 * p + 1] : 0.0;
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
// emitted value is bitwise x, y or x + y.
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
  c.ca = sc[c.pa];
  c.cb = sc[c.pb];
}

// One merge round over `nl` >= 2 lists of src (offsets `so`, nl + 1 entries).
// Writes ceil(nl/2) lists (each followed by its sentinel) to dst with offsets
// `dof`. Returns total outputs. Each thread merges two chunks (t and t + G)
// interleaved for ILP.
template <int G, int VT, bool FIRST, bool VALS>
__device__ __forceinline__ int merge_round(const Group<G>& g, const RowBufs& rb, const int* sc, const double* sv,
                                           const int* so, int nl, int* dc, double* dv, int* dof,
                                           const double* aval) {
  const int npairs = (nl + 1) >> 1;
  const int T = build_chunks<G, VT>(g, so, nl, npairs, rb.cst, rb.cpair, rb.scan_tmp);
  int out_base = 0;
  for (int tb = 0; tb < T; tb += 2 * G) {
    Chunk c0, c1;
    const int t0 = tb + g.rank, t1 = tb + G + g.rank;
    chunk_setup<VT, FIRST, VALS>(c0, t0, T, sc, so, nl, rb.cst, rb.cpair, rb.cb, rb.vb, aval);
    chunk_setup<VT, FIRST, VALS>(c1, t1, T, sc, so, nl, rb.cst, rb.cpair, rb.cb, rb.vb, aval);
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
    // the last chunk of a pair writes the pair's sentinel
    if (t0 < T && t0 + 1 == rb.cst[c0.pair + 1]) dc[base0 + c0.cnt] = INT_MAX;
    if (t1 < T && t1 + 1 == rb.cst[c1.pair + 1]) dc[base1 + c1.cnt] = INT_MAX;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int pf = h ? c1.pair_first : c0.pair_first;
      if (pf >= 0) {  // this pair's (and preceding empty pairs') dst offset
        const int vb = h ? vbase1 : vbase0;
        int q = pf;
        const int k0 = rb.cst[q];
        dof[q] = vb;
        while (q > 0 && rb.cst[q - 1] == k0) {
          dof[--q] = vb;
          dc[vb + q] = INT_MAX;  // sentinel of the empty pair q
        }
      }
    }
    out_base += (total & 0xffff) + (total >> 16);
  }
  if (g.rank == 0) {  // trailing empty pairs (sentinels too) and the end offset
    for (int q = npairs; q >= 0; --q) {
      if (q < npairs && rb.cst[q] != T) break;
      dof[q] = out_base;
      if (q < npairs) dc[out_base + q] = INT_MAX;
    }
  }
  g.sync();
  return out_base;
}

// BRMerge of output row `row` (n_prod P) by group g.
// SMEM: buffers in shared memory (TMA / cp.async staging); phase: mbarrier
// parity of this group, toggled once per row.
template <int G, int VT, bool VALS, int OUT, bool SMEM>
__device__ __forceinline__ void process_row(const Group<G>& g, const CsrView& A, const CsrView& B, int64_t bnnz,
                                            int64_t row, int P, const RowOut& o, const RowBufs& rb,
                                            unsigned& phase) {
  const int64_t a0 = A.rpt[row];
  const int nl = static_cast<int>(A.rpt[row + 1] - a0);
  const double* aval = VALS ? A.val + a0 : nullptr;
  // TMA staging: every list's 16-byte window (+ room for its sentinel) must
  // fit the padded capacity and B's arrays must be 16-byte aligned
  const bool tma = SMEM && P + 7 * nl <= rb.capc && (!VALS || P + 2 * nl <= rb.capv) &&
                   ((reinterpret_cast<uintptr_t>(B.col) | (VALS ? reinterpret_cast<uintptr_t>(B.val) : 0)) & 15) == 0;
  if (tma) fence_proxy_async();  // order the previous row's generic accesses before async writes
  // list offsets (exclusive scan of the selected B row lengths) and, for TMA,
  // the padded window layout; each lane stages its own lists
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
      rb.offA[l] = run + ex;
      if (tma) {
        const int pc = runc + (pex & 0xffff), pv = runv + (pex >> 16);
        rb.cb[l] = pc + static_cast<int>(s - wsc);
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
            for (int e = 0; e < len; ++e) cp_async_4(rb.colA + rb.cb[l] + e, B.col + s + e);
          if (VALS) {
            if (bulk_v)
              tma_bulk_g2s(rb.valA + pv, B.val + wsv, wv * 8u, rb.mbar);
            else
              for (int e = 0; e < len; ++e) cp_async_8(rb.valA + pv + (s - wsv) + e, B.val + s + e);
          }
        }
      } else {
        rb.cb[l] = run + ex + l;  // contiguous lists, one sentinel slot each
        if (VALS) rb.vb[l] = run + ex + l;
      }
    }
    run += tot;
    if (tma) {
      runc += ptot & 0xffff;
      runv += ptot >> 16;
    }
  }
  if (g.rank == 0) rb.offA[nl] = run;
  g.sync();
  if (tma) {
    if (g.rank == 0) mbar_arrive(rb.mbar);
    cp_async_wait_all();
    mbar_wait(rb.mbar, phase);
    phase ^= 1u;
  } else {
    // multiplying phase without TMA: copy list l to cb[l] .. cb[l] + len
    const bool per_list_group = P * 2 >= nl * G;
    for (int l = per_list_group ? 0 : g.rank; l < nl; l += per_list_group ? 1 : G) {
      const int dst = rb.cb[l], n = rb.offA[l + 1] - rb.offA[l];
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
  // sentinel after every gathered list
  for (int l = g.rank; l < nl; l += G) rb.colA[rb.cb[l] + rb.offA[l + 1] - rb.offA[l]] = INT_MAX;
  g.sync();
  int* sc = rb.colA;
  double* sv = rb.valA;
  int* so = rb.offA;
  int* dc = rb.colB;
  double* dv = rb.valB;
  int* dof = rb.offB;
  int n_out = P;
  if (nl >= 2) {
    int cur = nl;
    n_out = merge_round<G, VT, true, VALS>(g, rb, sc, sv, so, cur, dc, dv, dof, aval);
    cur = (cur + 1) >> 1;
    { int* t = sc; sc = dc; dc = t; }
    { double* t = sv; sv = dv; dv = t; }
    { int* t = so; so = dof; dof = t; }
    while (cur > 1) {
      n_out = merge_round<G, VT, false, VALS>(g, rb, sc, sv, so, cur, dc, dv, dof, nullptr);
      cur = (cur + 1) >> 1;
      { int* t = sc; sc = dc; dc = t; }
      { double* t = sv; sv = dv; dv = t; }
      { int* t = so; so = dof; dof = t; }
    }
  }
  // Alg. 1 line 36: store the result row
  if (OUT != OUT_SYMBOLIC) {
    const int64_t dst = o.base[row];
    if (nl == 1) {  // single list: the scaled B row is the result
      const double s0 = VALS ? aval[0] : 0.0;
      const int c0 = rb.cb[0], v0 = VALS ? rb.vb[0] : 0;
      for (int e = g.rank; e < n_out; e += G) {
        o.col[dst + e] = sc[c0 + e];
        if (VALS) o.val[dst + e] = __dmul_rn(s0, sv[v0 + e]);
      }
    } else {
      for (int e = g.rank; e < n_out; e += G) {
        o.col[dst + e] = sc[e];
        if (VALS) o.val[dst + e] = sv[e];
      }
    }
  }
  if (OUT != OUT_C && g.rank == 0) o.row_size[row] = n_out;
  g.sync();
}

}  // namespace brm
