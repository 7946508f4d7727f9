// engine.cuh -- the BRMerge accumulation of one output row by a thread group
// (Algorithm 1), parallelised for a GPU:
//
//   multiplying phase (lines 10-15): the B rows selected by A_i* are gathered,
//     coalesced, into the ping buffer as consecutive sorted lists; list
//     offsets come from a group scan of the B row lengths. The scaling by
//     A_ik is fused into the first merge round (one rounding, same value).
//   accumulating phase (lines 21-35): ceil(log2 num_list) rounds; round r
//     merges lists (0,1),(2,3),... of src into dst, an odd trailing list is
//     copied, then src/dst swap. Every round is ONE segmented merge-path pass
//     over the whole concatenated merged space of all pairs: thread t owns
//     merged positions [t*VT, t*VT+VT) of each tile, finds its pair by binary
//     search over the pair starts and its split by a merge-path search, and
//     merges sequentially into registers, summing equal columns (Fig. 2). A
//     duplicate whose two halves straddle a thread boundary is taken by the
//     left thread (look-ahead) and skipped by the right one, so no cross-thread
//     fix-up is needed. A group exclusive scan of the per-thread output counts
//     gives every output its compacted dst position, which is exactly the
//     sequential layout of Alg. 1 ("consume two lists and store to
//     dst_buffer"), and the dst list offsets of the next round.
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

// One merge round over `nl` >= 2 lists of src (offsets `so`, nl + 1 entries).
// Writes ceil(nl/2) lists to dst with offsets `dof`. Returns total outputs.
template <int G, int VT, bool FIRST, bool VALS>
__device__ __forceinline__ int merge_round(const Group<G>& g, const int* sc, const double* sv,
                                           const int* so, int nl, int* dc, double* dv, int* dof,
                                           const double* scale, int* scan_tmp) {
  const int E = so[nl];
  const int npairs = (nl + 1) >> 1;
  int out_base = 0;
  for (int tile = 0; tile < E; tile += G * VT) {
    const int d0 = tile + g.rank * VT;
    const int dend = min(d0 + VT, E);
    int cnt = 0;
    int ocol[VT];
    double oval[VT];
    int pfirst = 0, plast = -1;  // pairs whose first output this thread emits
    if (d0 < E) {
      int p = upper_search<2>(so, npairs, d0);
      int as = so[2 * p];
      int ae = so[min(2 * p + 1, nl)];
      int be = so[min(2 * p + 2, nl)];
      int la = ae - as, lb = be - ae;
      const int dd = d0 - as;
      int i = merge_path(sc + as, la, sc + ae, lb, dd);
      int j = dd - i;
      int pos = d0;
      if (dd == 0) {
        // this thread starts pair p (and any empty pairs sharing its start)
        int q = p;
        while (q > 0 && so[2 * (q - 1)] == d0) --q;
        for (int r = q; r <= p; ++r) dof[r] = 0;
        pfirst = q;
        plast = p;
      } else if (i > 0 && j < lb && sc[as + i - 1] == sc[ae + j]) {
        // b[j] duplicates a[i-1], already summed by the thread to the left
        ++j;
        ++pos;
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
        if (pos < dend) {
          if (ca == INT_MAX && cb == INT_MAX) {
            // pair exhausted: the next non-empty pair starts exactly at pos
            const int q0 = p + 1;
            do {
              ++p;
              as = so[2 * p];
              ae = so[min(2 * p + 1, nl)];
              be = so[min(2 * p + 2, nl)];
            } while (as == be);
            for (int r = q0; r <= p; ++r) dof[r] = cnt;
            if (plast < 0) pfirst = q0;
            plast = p;
            la = ae - as;
            lb = be - ae;
            i = 0;
            j = 0;
            if (FIRST && VALS) {
              sa = scale[2 * p];
              sb = (2 * p + 1 < nl) ? scale[2 * p + 1] : 0.0;
            }
            ca = la > 0 ? sc[as] : INT_MAX;
            cb = lb > 0 ? sc[ae] : INT_MAX;
          }
          if (ca < cb) {
            ocol[v] = ca;
            if (VALS) oval[v] = FIRST ? __dmul_rn(sa, sv[as + i]) : sv[as + i];
            ++i;
            ++pos;
            ca = i < la ? sc[as + i] : INT_MAX;
          } else if (cb < ca) {
            ocol[v] = cb;
            if (VALS) oval[v] = FIRST ? __dmul_rn(sb, sv[ae + j]) : sv[ae + j];
            ++j;
            ++pos;
            cb = j < lb ? sc[ae + j] : INT_MAX;
          } else {  // equal columns: "vals with duplicate cols are combined"
            ocol[v] = ca;
            if (VALS) {
              const double x = FIRST ? __dmul_rn(sa, sv[as + i]) : sv[as + i];
              const double y = FIRST ? __dmul_rn(sb, sv[ae + j]) : sv[ae + j];
              oval[v] = __dadd_rn(x, y);
            }
            ++i;
            ++j;
            pos += 2;
            ca = i < la ? sc[as + i] : INT_MAX;
            cb = j < lb ? sc[ae + j] : INT_MAX;
          }
          ++cnt;
        }
      }
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
    for (int r = pfirst; r <= plast; ++r) dof[r] += base;
    out_base += total;
  }
  if (g.rank == 0) {
    // trailing empty pairs (start == E) and the end sentinel
    for (int q = npairs; q >= 0; --q) {
      if (q < npairs && so[2 * q] != E) break;
      dof[q] = out_base;
    }
  }
  g.sync();
  return out_base;
}

// BRMerge of output row `row` by group g. Buffers: colA/colB (>= n_prod),
// valA/valB (>= n_prod, VALS), offA (>= nl+1), offB (>= nl/2+2),
// bstart (>= nl), scale (>= nl, VALS), scan_tmp (G/32+1 ints, shared).
template <int G, int VT, bool VALS, int OUT>
__device__ __forceinline__ void process_row(const Group<G>& g, const CsrView& A, const CsrView& B,
                                            int64_t row, const RowOut& o, int* colA, int* colB,
                                            double* valA, double* valB, int* offA, int* offB,
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
  // multiplying phase: gather the B rows (coalesced within each list)
  for (int e = g.rank; e < P; e += G) {
    const int l = upper_search<1>(offA, nl, e);
    const int64_t src = bstart[l] + (e - offA[l]);
    colA[e] = B.col[src];
    if (VALS) valA[e] = B.val[src];
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
    n_out = merge_round<G, VT, true, VALS>(g, sc, sv, so, cur, dc, dv, dof, scale, scan_tmp);
    cur = (cur + 1) >> 1;
    { int* t = sc; sc = dc; dc = t; }
    { double* t = sv; sv = dv; dv = t; }
    { int* t = so; so = dof; dof = t; }
    while (cur > 1) {
      n_out = merge_round<G, VT, false, VALS>(g, sc, sv, so, cur, dc, dv, dof, nullptr, scan_tmp);
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
