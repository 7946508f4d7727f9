// heavy.cuh -- heavy rows (bin 7) by windowed BRMerge.
//
// A heavy output row is merged window by window: a window is a column range
// [c0, c1) holding at most kHvCap of the row's intermediate products.
// Restricting every list to [c0, c1) keeps the number of lists and therefore
// the pairing of every round of Algorithm 1 (an empty list keeps its place,
// PAPER.md:190), so each column receives exactly Algorithm 1's additions in
// Algorithm 1's order and the windows' results, in column
// order, concatenate to the row. A row of more than kHvLists lists is first
// cut into aligned blocks of kHvLists = 2^9 consecutive lists -- sub-trees
// of Algorithm 1's tree (pairs are (2m, 2m+1) at every level) -- whose
// results, scaled by 1.0 (exact), are the lists of the next level.
//
// Two kernels per level:
//   k_hv_plan   one CTA per virtual row: a column bitmap and a histogram of
//               its product columns in shared memory (one pass over the
//               products) give the windows (greedy, <= kHvCap products each)
//               and each window's output size (bits set in the window); the
//               total is the row size (BRMerge-Precise's symbolic step,
//               PAPER.md:298). count_only: the bitmap alone, any number of
//               lists (row sizes of rows that take several levels).
//   k_hv_merge  one CTA per task (a run of consecutive windows of one
//               virtual row): per window, each list's share by probes from
//               its cursor, the products gathered into shared memory, the
//               rounds of Algorithm 1 as one A-with-B merge per round (heavy.cu),
//               the result written at the window's output offset.
#pragma once
#include "engine.cuh"

namespace brm {

// (tuning overrides: BRM_NVCC_FLAGS="-DBRM_HV_CAP=3072 -DBRM_HV_MINB=3", tools/variants.sh)
#ifndef BRM_HV_CAP
#define BRM_HV_CAP 4096
#endif
#ifndef BRM_HV_LISTS
#define BRM_HV_LISTS 512
#endif
#ifndef BRM_HV_G
#define BRM_HV_G 256
#endif
#ifndef BRM_HV_MINB
#define BRM_HV_MINB 2
#endif
constexpr int kHvCap = BRM_HV_CAP;      // products per window
constexpr int kHvLists = BRM_HV_LISTS;  // lists per virtual row: an aligned 2^k-list sub-tree
constexpr int kHvG = BRM_HV_G;          // merge CTA
constexpr int kHvMinBlocks = BRM_HV_MINB;  // merge CTAs per SM (launch bounds)
constexpr int kHvPlanG = 512;      // plan CTA
constexpr int kHvRangeBits = 20;   // bitmap over 2^20 columns per pass ("range")
constexpr int kHvRange = 1 << kHvRangeBits;
constexpr int kHvBinBits = 7;      // histogram bins of 128 columns
constexpr int kHvBins = kHvRange >> kHvBinBits;
constexpr int kHvFine = 64;        // bins refined to single columns per refinement pass
// merge keys hold col - c0 in their low 20 bits (heavy.cu kColBits): a
// window spans at most 2^20 - 1 columns
constexpr int kHvSpan = (1 << 20) - 1;
static_assert(kHvCap <= 65535, "owner marks and the packed 16|16 round scan");
static_assert((kHvLists & (kHvLists - 1)) == 0, "a block of lists must be an aligned power-of-two sub-tree");
static_assert(kHvLists <= kHvCap, "a column holds at most one product per list: a single column fits a window");

struct HvRow {
  int64_t row;     // output row (row of A)
  int64_t first;   // src 0: index of list 0 among the A row's entries; src 1: list-table index of list 0
  int64_t nprod;   // products of this virtual row
  int64_t plan;    // offset of its plan: cuts / wout hold maxwin + 1 entries from here
  int64_t obase;   // out 1: workspace entry offset of its result
  int64_t task0;   // its first merge task
  int32_t nl;      // lists
  int32_t src;     // 0: B rows named by the A row; 1: workspace segments of the list table
  int32_t out;     // 0: output row of C / C_bar (RowOut base); 1: workspace at obase
  int32_t maxwin;  // plan capacity
  int32_t wch;     // windows per merge task
  int32_t pad;
};

struct HvArgs {
  CsrView A, B;
  int64_t ncols;          // B.cols
  const HvRow* rows;      // virtual rows
  int64_t nrows;
  const int64_t* lt;      // list table (src 1): list j = [lt[first + j], lt[first + j + 1]) of ws_col / ws_val
  const int32_t* ws_col;  // src 1 input
  const double* ws_val;
  int32_t* wo_col;        // out 1 output
  double* wo_val;
  int32_t* cuts;          // plan: window w = [cuts[plan + w], cuts[plan + w + 1])
  int32_t* wout;          // plan: output offset of window w (wout[plan + nwin] = total)
  int32_t* nwin;          // per virtual row
  int64_t* total;         // per virtual row: entries of its result
  int64_t* row_size;      // out 0 rows: row_size[row] = total (null: not written)
  unsigned int* err;      // bit 0: plan overflow; bit 1: window size mismatch
  const int32_t* tmap;    // merge: virtual row of each task (k_hv_taskmap)
  const int64_t* ntask_total;  // merge: number of tasks (device scalar)
};

// plan shared memory: bitmap, histogram, fine counts, bin slots, list table
constexpr int kHvGroups = kHvRange / 1024;  // popcount groups of 32 bitmap words
constexpr int hv_plan_smem() {
  return kHvRange / 8 + kHvBins * 4 + kHvFine * 128 * 4 + kHvBins + kHvLists * 8 + (kHvLists + 4) * 4 +
         align16((kHvLists + 4) * 4) + (kHvGroups + 4) * 4 + 256;
}
// merge shared memory
constexpr int hv_merge_smem() {
  return kHvLists * 16 /*lst*/ + kHvLists * 8 /*S*/ + kHvLists * 4 * 4 /*L, cur, head, cnt*/ +
         align16((kHvCap + 2) * 4) /*keys*/ + align16((kHvCap + 2) * 8) /*values*/ +
         kHvCap * 2 /*owner*/ +
         64 /*scan tmp*/;
}

// upper bound of the windows of a virtual row of P products whose columns
// lie in [0, ncols): two consecutive windows of one range hold more than
// kHvCap products; each range may end with a short window and a span cut.
inline int64_t hv_maxwin(int64_t P, int64_t ncols) {
  const int64_t ranges = (ncols + kHvRange - 1) / kHvRange;
  return 2 * ((P + kHvCap - 1) / kHvCap) + 3 * ranges + 1;
}

cudaError_t launch_hv_plan(const HvArgs& a, bool count_only, cudaStream_t st);
cudaError_t launch_hv_merge(int out_kind, const HvArgs& a, int64_t ntasks, const RowOut& o, cudaStream_t st);
// products of each virtual row (src 0 rows) -> a.total (as a staging array)
cudaError_t launch_hv_vrow_nprod(const HvArgs& a, int64_t* out, cudaStream_t st);
// merge tasks from the planned window counts: ntask[v] = ceil(nwin[v] / wch);
// then (after an exclusive scan toff of ntask) rows[v].task0 = toff[v] and
// tmap[toff[v] + j] = v for the row's tasks
cudaError_t launch_hv_ntask(const HvArgs& a, int64_t* ntask, cudaStream_t st);
cudaError_t launch_hv_taskmap(const HvArgs& a, HvRow* rows, const int64_t* toff, int32_t* tmap, cudaStream_t st);

}  // namespace brm
