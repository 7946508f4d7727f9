// engine.cuh -- the BRMerge accumulation of one output row by a thread group
// (Algorithm 1), parallelised for a GPU:
//
//   multiplying phase (lines 10-15): the B rows selected by A_i* are gathered,
//     coalesced, into the ping buffer as consecutive sorted lists; list
//     offsets come from a group scan of the B row lengths. The scaling by
//     A_ik is fused into the first merge round (same single rounding).
//   accumulating phase (lines 21-35): ceil(log2 num_list) rounds; round r
//     merges lists (0,1),(2,3),... of src into dst, an odd trailing list is
//     copied, then src/dst swap. A round is cut into chunks of VT merged
//     positions that never straddle a pair; one thread merges one chunk:
//     binary search of its pair over the chunk table, merge-path split inside
//     the pair, then VT branch-free merge steps into registers summing equal
//     columns (Fig. 2). A duplicate whose halves straddle a chunk boundary is
//     taken by the left chunk (look-ahead) and skipped by the right one. A
//     group exclusive scan of per-thread output counts gives each output its
//     compacted dst position -- exactly Alg. 1's sequential layout ("consume
//     two lists and store to dst_buffer") -- and the next round's offsets.
//
// The same code runs with the buffers in shared memory (tiers 1-5) or in a
// global-memory workspace (tier 6); the pointers decide.
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

// Chunk table of a round: cst[p] = first chunk of pair p, cst[npairs] = total.
template <int G, int VT>
__device__ __forceinline__ int build_chunks(const Group<G>& g, const int* so, int nl, int npairs, int* cst,
                                            int* scan_tmp) {
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
    if (p < npairs) cst[p] = run + ex;
    run += tot;
  }
  if (g.rank == 0) cst[npairs] = run;
  g.sync();
  return run;
}

// Merge state of one chunk: cursors i (list a) and j (list b) of pair p,
// merged position d of the next element, chunk end dend.
struct Chunk {
  int as, ae, la, lb, i, j, d, dend, ca, cb, cnt, pair_first;
  double sa, sb;
};

template <int VT, bool FIRST, bool VALS>
__device__ __forceinline__ void chunk_setup(Chunk& c, int t, int T, const int* sc, const int* so, int nl,
                                            int npairs, const int* cst, const double* scale) {
  c.cnt = 0;
  c.pair_first = -1;
  c.d = 0;
  c.dend = 0;  // inactive
  c.i = c.j = c.la = c.lb = c.as = c.ae = 0;
  c.ca = c.cb = INT_MAX;
  c.sa = c.sb = 1.0;
  if (t >= T) return;
  const int p = upper_search<1>(cst, npairs, t);
  const int k = t - cst[p];
  c.as = so[2 * p];
  c.ae = so[min(2 * p + 1, nl)];
  const int be = so[min(2 * p + 2, nl)];
  c.la = c.ae - c.as;
  c.lb = be - c.ae;
  c.d = k * VT;
  c.dend = min(c.d + VT, c.la + c.lb);
  c.i = merge_path(sc + c.as, c.la, sc + c.ae, c.lb, c.d);
  c.j = c.d - c.i;
  if (c.i > 0 && c.j < c.lb && sc[c.as + c.i - 1] == sc[c.ae + c.j]) {
    ++c.j;  // b[j] duplicates a[i-1]: summed by the chunk to the left
    ++c.d;
  }
  if (FIRST && VALS) {
    c.sa = scale[2 * p];
    c.sb = (2 * p + 1 < nl) ? scale[2 * p + 1] : 0.0;
  }
  c.ca = c.i < c.la ? sc[c.as + c.i] : INT_MAX;
  c.cb = c.j < c.lb ? sc[c.ae + c.j] : INT_MAX;
  if (k == 0) c.pair_first = p;
}

// One branch-free merge step: emits min(ca, cb); on equal columns the two
// values are summed ("vals with duplicate cols are combined into one val").
// The value of a list not taken is -0.0, the exact additive identity, so the
// emitted value is bitwise x, y or x + y.
template <bool FIRST, bool VALS>
__device__ __forceinline__ void chunk_step(Chunk& c, const int* sc, const double* sv, int& ocol,
                                           double& oval) {
  const bool act = c.d < c.dend;
  const bool ta = act && c.ca <= c.cb;
  const bool tbb = act && c.cb <= c.ca;
  ocol = min(c.ca, c.cb);
  if (VALS) {
    double x = -0.0, y = -0.0;
    if (ta) x = sv[c.as + c.i];
    if (tbb) y = sv[c.ae + c.j];
    if (FIRST) {
      if (ta) x = __dmul_rn(c.sa, x);
      if (tbb) y = __dmul_rn(c.sb, y);
    }
    oval = __dadd_rn(x, y);
  }
  c.i += ta;
  c.j += tbb;
  c.d += (int)ta + (int)tbb;
  c.cnt += act;
  const int na = c.as + min(c.i, c.la);  // in-bounds reload address (value masked below)
  const int nb = c.ae + min(c.j, c.lb - 1 < 0 ? 0 : c.lb - 1);
  const int xa = sc[na];
  const int xb = sc[nb];
  c.ca = c.i < c.la ? xa : INT_MAX;
  c.cb = c.j < c.lb ? xb : INT_MAX;
}

// One merge round over `nl` >= 2 lists of src (offsets `so`, nl + 1 entries).
// Writes ceil(nl/2) lists to dst with offsets `dof`. Returns total outputs.
// Each thread merges two chunks (t and t + G) interleaved for ILP.
template <int G, int VT, bool FIRST, bool VALS>
__device__ __forceinline__ int merge_round(const Group<G>& g, const int* sc, const double* sv,
                                           const int* so, int nl, int* dc, double* dv, int* dof,
                                           const double* scale, int* cst, int* scan_tmp) {
  const int npairs = (nl + 1) >> 1;
  const int T = build_chunks<G, VT>(g, so, nl, npairs, cst, scan_tmp);
  int out_base = 0;
  for (int tb = 0; tb < T; tb += 2 * G) {
    Chunk c0, c1;
    chunk_setup<VT, FIRST, VALS>(c0, tb + g.rank, T, sc, so, nl, npairs, cst, scale);
    chunk_setup<VT, FIRST, VALS>(c1, tb + G + g.rank, T, sc, so, nl, npairs, cst, scale);
    int ocol0[VT], ocol1[VT];
    double oval0[VT], oval1[VT];
#pragma unroll
    for (int v = 0; v < VT; ++v) {
      chunk_step<FIRST, VALS>(c0, sc, sv, ocol0[v], oval0[v]);
      chunk_step<FIRST, VALS>(c1, sc, sv, ocol1[v], oval1[v]);
    }
    // packed scan: low 16 bits chunk t, high 16 bits chunk t + G
    int total;
    const int ex = group_excl_scan<G>(g, c0.cnt | (c1.cnt << 16), total, scan_tmp);
    const int base0 = out_base + (ex & 0xffff);
    const int base1 = out_base + (total & 0xffff) + (ex >> 16);
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
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int pf = h ? c1.pair_first : c0.pair_first;
      if (pf >= 0) {  // this pair's (and preceding empty pairs') dst offset
        const int base = h ? base1 : base0;
        int q = pf;
        const int k0 = cst[q];
        dof[q] = base;
        while (q > 0 && cst[q - 1] == k0) dof[--q] = base;
      }
    }
    out_base += (total & 0xffff) + (total >> 16);
  }
  if (g.rank == 0) {  // trailing empty pairs and the end sentinel
    for (int q = npairs; q >= 0; --q) {
      if (q < npairs && cst[q] != T) break;
      dof[q] = out_base;
    }
  }
  g.sync();
  return out_base;
}

__device__ __forceinline__ void cp_async_4(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Multiplying phase (Alg. 1 lines 10-15, scaling deferred to round 1): copy
// list l = B row k_l to [offA[l], offA[l+1]). Shared-memory tiers use
// cp.async (LDGSTS) so every list of the row is in flight at once; long lists
// are copied by the whole group (coalesced), short ones one lane per list.
template <int G, bool VALS, bool SMEM>
__device__ __forceinline__ void gather_lists(const Group<G>& g, const CsrView& B, int nl, int P,
                                             const int* offA, const int64_t* bstart, int* colA,
                                             double* valA) {
  if (P * 2 >= nl * G || G == 1) {
    for (int l = 0; l < nl; ++l) {
      const int dst = offA[l], n = offA[l + 1] - dst;
      const int64_t s = bstart[l];
      for (int e = g.rank; e < n; e += G) {
        if (SMEM) {
          cp_async_4(colA + dst + e, B.col + s + e);
          if (VALS) cp_async_8(valA + dst + e, B.val + s + e);
        } else {
          colA[dst + e] = B.col[s + e];
          if (VALS) valA[dst + e] = B.val[s + e];
        }
      }
    }
  } else {
    for (int l = g.rank; l < nl; l += G) {
      const int dst = offA[l], n = offA[l + 1] - dst;
      const int64_t s = bstart[l];
      for (int e = 0; e < n; ++e) {
        if (SMEM) {
          cp_async_4(colA + dst + e, B.col + s + e);
          if (VALS) cp_async_8(valA + dst + e, B.val + s + e);
        } else {
          colA[dst + e] = B.col[s + e];
          if (VALS) valA[dst + e] = B.val[s + e];
        }
      }
    }
  }
  if (SMEM) cp_async_wait_all();
}

// BRMerge of output row `row` by group g. Buffers: colA/colB (>= n_prod),
// valA/valB (>= n_prod, VALS), offA (>= nl+1), offB (>= nl/2+2),
// cst (>= nl/2+2), bstart (>= nl), scale (>= nl, VALS), scan_tmp (G/32+1).
// SMEM: the buffers are in shared memory (cp.async gather).
template <int G, int VT, bool VALS, int OUT, bool SMEM>
__device__ __forceinline__ void process_row(const Group<G>& g, const CsrView& A, const CsrView& B,
                                            int64_t row, const RowOut& o, int* colA, int* colB,
                                            double* valA, double* valB, int* offA, int* offB, int* cst,
                                            int64_t* bstart, double* scale, int* scan_tmp) {
  const int64_t a0 = A.rpt[row];
  const int nl = static_cast<int>(A.rpt[row + 1] - a0);
  // list offsets: exclusive scan of the selected B row lengths
  int run = 0;
  for (int lbase = 0; lbase < nl; lbase += G) {
    const int l = lbase + g.rank;
    int len = 0;
    if (l < nl) {
      const int k = A.col[a0 + l];
      const int64_t s = B.rpt[k];
      len = static_cast<int>(B.rpt[k + 1] - s);
      bstart[l] = s;
      if (VALS) scale[l] = A.val[a0 + l];
    }
    int tot;
    const int ex = group_excl_scan<G>(g, len, tot, scan_tmp);
    if (l < nl) offA[l] = run + ex;
    run += tot;
  }
  const int P = run;
  if (g.rank == 0) offA[nl] = P;
  g.sync();
  // multiplying phase: gather the B rows into the ping buffer
  gather_lists<G, VALS, SMEM>(g, B, nl, P, offA, bstart, colA, valA);
  g.sync();
  int* sc = colA;
  double* sv = valA;
  int* so = offA;
  int* dc = colB;
  double* dv = valB;
  int* dof = offB;
  int n_out = P;
  if (nl >= 2) {
    int cur = nl;
    n_out = merge_round<G, VT, true, VALS>(g, sc, sv, so, cur, dc, dv, dof, scale, cst, scan_tmp);
    cur = (cur + 1) >> 1;
    { int* t = sc; sc = dc; dc = t; }
    { double* t = sv; sv = dv; dv = t; }
    { int* t = so; so = dof; dof = t; }
    while (cur > 1) {
      n_out = merge_round<G, VT, false, VALS>(g, sc, sv, so, cur, dc, dv, dof, nullptr, cst, scan_tmp);
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
      const double s0 = VALS ? scale[0] : 0.0;
      for (int e = g.rank; e < n_out; e += G) {
        o.col[dst + e] = sc[e];
        if (VALS) o.val[dst + e] = __dmul_rn(s0, sv[e]);
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
