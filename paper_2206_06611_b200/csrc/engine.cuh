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

// One merge round over `nl` >= 2 lists of src (offsets `so`, nl + 1 entries).
// Writes ceil(nl/2) lists to dst with offsets `dof`. Returns total outputs.
template <int G, int VT, bool FIRST, bool VALS>
__device__ __forceinline__ int merge_round(const Group<G>& g, const int* sc, const double* sv,
                                           const int* so, int nl, int* dc, double* dv, int* dof,
                                           const double* scale, int* cst, int* scan_tmp) {
  const int npairs = (nl + 1) >> 1;
  const int T = build_chunks<G, VT>(g, so, nl, npairs, cst, scan_tmp);
  int out_base = 0;
  for (int tb = 0; tb < T; tb += G) {
    const int t = tb + g.rank;
    int cnt = 0;
    int ocol[VT];
    double oval[VT];
    int first_of_pair = -1;
    if (t < T) {
      const int p = upper_search<1>(cst, npairs, t);
      const int k = t - cst[p];
      const int as = so[2 * p];
      const int ae = so[min(2 * p + 1, nl)];
      const int be = so[min(2 * p + 2, nl)];
      const int la = ae - as, lb = be - ae;
      int d = k * VT;
      const int dend = min(d + VT, la + lb);
      int i = merge_path(sc + as, la, sc + ae, lb, d);
      int j = d - i;
      if (i > 0 && j < lb && sc[as + i - 1] == sc[ae + j]) {
        ++j;  // b[j] duplicates a[i-1]: summed by the chunk to the left
        ++d;
      }
      double sa = 1.0, sb = 1.0;
      if (FIRST && VALS) {
        sa = scale[2 * p];
        sb = (2 * p + 1 < nl) ? scale[2 * p + 1] : 0.0;
      }
      int ca = i < la ? sc[as + i] : INT_MAX;
      int cb = j < lb ? sc[ae + j] : INT_MAX;
#pragma unroll
      for (int v = 0; v < VT; ++v) {
        if (d < dend) {
          const bool ta = ca <= cb;
          const bool tbb = cb <= ca;
          ocol[v] = ta ? ca : cb;
          if (VALS) {
            double x = 0.0, y = 0.0;
            if (ta) x = sv[as + i];
            if (tbb) y = sv[ae + j];
            if (FIRST) {
              x = __dmul_rn(sa, x);
              y = __dmul_rn(sb, y);
            }
            // "vals with duplicate cols are combined into one val"
            oval[v] = (ta && tbb) ? __dadd_rn(x, y) : (ta ? x : y);
          }
          i += ta;
          j += tbb;
          d += (int)ta + (int)tbb;
          if (ta) ca = i < la ? sc[as + i] : INT_MAX;
          if (tbb) cb = j < lb ? sc[ae + j] : INT_MAX;
          ++cnt;
        }
      }
      if (k == 0) first_of_pair = p;
    }
    int total;
    const int excl = group_excl_scan<G>(g, cnt, total, scan_tmp);
    const int base = out_base + excl;
#pragma unroll
    for (int v = 0; v < VT; ++v) {
      if (v < cnt) {
        dc[base + v] = ocol[v];
        if (VALS) dv[base + v] = oval[v];
      }
    }
    if (first_of_pair >= 0) {  // this pair's (and preceding empty pairs') dst offset
      int q = first_of_pair;
      const int c0 = cst[q];
      dof[q] = base;
      while (q > 0 && cst[q - 1] == c0) dof[--q] = base;
    }
    out_base += total;
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

// BRMerge of output row `row` by group g. Buffers: colA/colB (>= n_prod),
// valA/valB (>= n_prod, VALS), offA (>= nl+1), offB (>= nl/2+2),
// cst (>= nl/2+2), bstart (>= nl), scale (>= nl, VALS), scan_tmp (G/32+1).
template <int G, int VT, bool VALS, int OUT>
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
  // multiplying phase: gather the B rows, list by list (coalesced within a
  // list), U lists in flight per step for memory-level parallelism
  {
    constexpr int U = 4;
    for (int l0 = 0; l0 < nl; l0 += U) {
      int cv[U];
      double vv[U];
      int dst[U], n[U];
      int64_t src[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int l = l0 + u;
        n[u] = 0;
        if (l < nl) {
          dst[u] = offA[l];
          n[u] = offA[l + 1] - dst[u];
          src[u] = bstart[l];
        }
      }
      bool more = true;
      for (int e0 = 0; more; e0 += G) {
        more = false;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + g.rank;
          if (e < n[u]) {
            cv[u] = B.col[src[u] + e];
            if (VALS) vv[u] = B.val[src[u] + e];
          }
          more |= e0 + G < n[u];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + g.rank;
          if (e < n[u]) {
            colA[dst[u] + e] = cv[u];
            if (VALS) valA[dst[u] + e] = vv[u];
          }
        }
      }
    }
  }
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
