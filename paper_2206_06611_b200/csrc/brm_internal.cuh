// brm_internal.cuh -- shared device-side definitions of libbrmerge (product
// path). Nothing here is shared with oracle/.
#pragma once
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#include "brmerge.h"

namespace brm {

struct CsrView {
  const int64_t* rpt;
  const int32_t* col;
  const double* val;
};

// ---------------------------------------------------------------------------
// Row tiers. A row with n_prod = P > 0 and num_list = nl
// (= nnz(A_i*)) goes to the first tier t whose (cap, lcap) admits it:
//   1  one thread per row (Alg. 1)      P <= 8,    nl <= 8
//   2  register BRMerge, one warp       P <= 32,   nl <= 32
//   3  record BRMerge, one warp         P <= 256,  nl <= 64   (smem records)
//   4  record BRMerge, one warp         P <= 768,  nl <= 64   (smem records)
//   5  record BRMerge, 256 threads      P <= 3072, nl <= 256  (smem records)
//   6  record BRMerge, 512 threads      P <= 6656, nl <= 512  (smem records)
//   7  heavy rows: windowed BRMerge (heavy.cuh; column windows of <= 4096
//      products, levels of 512-list blocks), or under BRM_HEAVY_GLOBAL the
//      chunked BRMerge on 1024 threads with ping-pong buffers in a global
//      workspace
// ---------------------------------------------------------------------------
constexpr int kBinEmpty = 0;
constexpr int kBinGlobal = 7;
static_assert(BRM_NUM_BINS == 8, "tier table below assumes 8 bins");

struct TierBounds {
  int cap[BRM_NUM_BINS];
  int lcap[BRM_NUM_BINS];
};

// (G threads per row group, CAP elements, LCAP lists, GPC groups per CTA)
// (G and GPC may be overridden at build time for tuning experiments, e.g.
// BRM_NVCC_FLAGS="-DBRM_T4_G=32 -DBRM_T4_GPC=2"; tools/variants.sh)
#ifndef BRM_T2_GPC
#define BRM_T2_GPC 8
#endif
#ifndef BRM_T3_G
#define BRM_T3_G 32
#endif
#ifndef BRM_T3_GPC
#define BRM_T3_GPC 8
#endif
#ifndef BRM_T4_G
#define BRM_T4_G 32
#endif
#ifndef BRM_T4_GPC
#define BRM_T4_GPC 2
#endif
// tiers 5-6 on 256 / 512 threads: 3.93 / 14.12 ms numeric on rmat20_ef16
// against 4.37 / 15.47 on 128 / 256 (profiles/r02c_scale/README.md)
#ifndef BRM_T5_G
#define BRM_T5_G 256
#endif
#ifndef BRM_T6_G
#define BRM_T6_G 512
#endif
// PLAIN (5th field): the record round's duplicate combine as plain code the
// compiler branches around (faster on rows with few duplicates) instead of
// predicated loads. Measured on B200: tier 3 on uniform1m_k16 -9 % with it;
// tier 4 on stencil27_64 +3.4 %, so only tier 3 takes it by default.
#ifndef BRM_T3_PLAIN
#define BRM_T3_PLAIN true
#endif
#ifndef BRM_T4_PLAIN
#define BRM_T4_PLAIN false
#endif
#define BRM_TIER1 8, 8, 8, 32, false
#define BRM_TIER2 32, 32, 32, BRM_T2_GPC, false
#define BRM_TIER3 BRM_T3_G, 256, 64, BRM_T3_GPC, BRM_T3_PLAIN
#define BRM_TIER4 BRM_T4_G, 768, 64, BRM_T4_GPC, BRM_T4_PLAIN
#define BRM_TIER5 BRM_T5_G, 3072, 256, 1, false
#define BRM_TIER6 BRM_T6_G, 6656, 512, 1, false
// PRECISE symbolic (hash counting) launch shapes of tiers 3-6, tuned apart
// from the merges: (G, CAP, LCAP, GPC)
#ifndef BRM_H3_GPC
#define BRM_H3_GPC 4
#endif
#ifndef BRM_H4_G
#define BRM_H4_G 32
#endif
#ifndef BRM_H4_GPC
#define BRM_H4_GPC 2
#endif
// 5th field: column loads in flight per thread before they are hashed.
// Measured on B200 (same box): tier 3 (uniform1m_k16) 2.45 ms with 1 vs
// 3.12 ms with 8 (registers); tier 4 (stencil27_64) 0.67 ms with 8 vs 0.78.
// 6th field: table slots per product x 4 (HQ: H = pow2 >= P * HQ / 4).
// 7th field: direct atomicCAS inserts (no read of the slot first).
// Measured on B200 (same box): stencil27_64's tier-4 symbolic 0.670 ms with
// HQ 6 -> 0.617 with HQ 5 (a smaller table to clear); uniform1m_k16's tier 3
// 2.43 ms with a read first vs 2.56 with direct CAS, and 2.43 / 1.82 / 2.42 ms
// with HQ 8 / 16 / 32 (uniform1m_k16 PRECISE 81.5 -> 90.0 GFLOP/s at 16);
// tier 4 on stencil27_64: 0.617 ms on 64 threads per row, 0.529 on one warp
// per row (2 rows per CTA; 4 per CTA 0.538), 8 loads in flight (4: 0.636,
// 2: 0.841), HQ 5 (4: 0.621, 8: 0.674) -- profiles/r02c_hash.
// PRECISE symbolic of one-warp rows: a direct-mapped table (a bitmap over
// the row's column span) when the span fits the table's bits, else hashing
#ifndef BRM_SYM_BITMAP
#define BRM_SYM_BITMAP 1
#endif
#ifndef BRM_H3_HB
#define BRM_H3_HB 1
#endif
#ifndef BRM_H3_HQ
#define BRM_H3_HQ 16
#endif
#ifndef BRM_H3_DIRECT
#define BRM_H3_DIRECT false
#endif
#define BRM_HASH3 32, 256, 64, BRM_H3_GPC, BRM_H3_HB, BRM_H3_HQ, BRM_H3_DIRECT
#ifndef BRM_H4_HB
#define BRM_H4_HB 8
#endif
#ifndef BRM_H4_HQ
#define BRM_H4_HQ 5
#endif
#define BRM_HASH4 BRM_H4_G, 768, 64, BRM_H4_GPC, BRM_H4_HB, BRM_H4_HQ, false
#ifndef BRM_H5_G
#define BRM_H5_G 128
#endif
#ifndef BRM_H6_G
#define BRM_H6_G 256
#endif
#define BRM_HASH5 BRM_H5_G, 3072, 256, 1, 8, 5, false
#define BRM_HASH6 BRM_H6_G, 6656, 512, 1, 8, 5, false
constexpr int kGlobalG = 1024;

// Routing caps of tiers 5-6 (<= their kernels' CAP; 0: the tier takes no
// rows, they go on to the next one / the windowed heavy path) -- tuning
// switches, BRM_NVCC_FLAGS="-DBRM_T6_ROUTE=0"
#ifndef BRM_T5_ROUTE
#define BRM_T5_ROUTE 3072
#endif
#ifndef BRM_T6_ROUTE
#define BRM_T6_ROUTE 6656
#endif
static_assert(BRM_T5_ROUTE <= 3072 && BRM_T6_ROUTE <= 6656, "routing caps within the kernels' capacity");
__host__ __device__ inline TierBounds tier_bounds() {
  TierBounds t{};
  t.cap[0] = 0;    t.lcap[0] = 0;
  t.cap[1] = 8;    t.lcap[1] = 8;
  t.cap[2] = 32;   t.lcap[2] = 32;
  t.cap[3] = 256;  t.lcap[3] = 64;
  t.cap[4] = 768;  t.lcap[4] = 64;
  t.cap[5] = BRM_T5_ROUTE; t.lcap[5] = 256;
  t.cap[6] = BRM_T6_ROUTE; t.lcap[6] = 512;
  t.cap[7] = INT_MAX; t.lcap[7] = INT_MAX;
  return t;
}

__host__ __device__ inline int tier_of(int64_t nprod, int64_t nl, const TierBounds& tb) {
  if (nprod == 0) return kBinEmpty;
#pragma unroll
  for (int t = 1; t < kBinGlobal; ++t)
    if (nprod <= tb.cap[t] && nl <= tb.lcap[t]) return t;
  return kBinGlobal;
}

__host__ __device__ constexpr int align16(int x) { return (x + 15) & ~15; }

// ---------------------------------------------------------------------------
// Thread groups: G <= 32 is a sub-warp (shuffles of width G), G > 32 is the
// whole CTA (blockDim.x == G).
// ---------------------------------------------------------------------------
template <int G>
struct Group {
  int rank;
  unsigned mask;
  int base;  // first lane of the group inside its warp (G <= 32)
  __device__ __forceinline__ void sync() const {
    if constexpr (G <= 32)
      __syncwarp(mask);
    else
      __syncthreads();
  }
};

template <int G>
__device__ __forceinline__ Group<G> make_group() {
  Group<G> g;
  g.rank = threadIdx.x % G;
  if constexpr (G >= 32) {
    g.mask = 0xffffffffu;
    g.base = 0;
  } else {
    g.base = (threadIdx.x & 31) & ~(G - 1);
    g.mask = ((1u << G) - 1u) << g.base;
  }
  return g;
}

// Exclusive scan of one int per thread over the group; `tmp` is shared memory
// of G/32+1 ints (unused for G <= 32). Ends with the group synchronised.
template <int G>
__device__ __forceinline__ int group_excl_scan(const Group<G>& g, int v, int& total, int* tmp) {
  if constexpr (G <= 32) {
    int x = v;
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
      const int y = __shfl_up_sync(g.mask, x, d, G);
      if (g.rank >= d) x += y;
    }
    total = __shfl_sync(g.mask, x, G - 1, G);
    return x - v;
  } else {
    constexpr int NW = G / 32;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) tmp[wid] = x;
    __syncthreads();
    if (wid == 0) {
      const int w = lane < NW ? tmp[lane] : 0;
      int wx = w;
#pragma unroll
      for (int d = 1; d < NW; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, wx, d);
        if (lane >= d) wx += y;
      }
      if (lane < NW) tmp[lane] = wx - w;
      if (lane == NW - 1) tmp[NW] = wx;
    }
    __syncthreads();
    const int res = tmp[wid] + x - v;
    total = tmp[NW];
    __syncthreads();
    return res;
  }
}

// Minimum / sum of one int per thread over the group; `tmp` as for
// group_excl_scan. Ends with the group synchronised.
template <int G, bool MIN>
__device__ __forceinline__ int group_reduce(const Group<G>& g, int v, int* tmp) {
  auto op = [](int a, int b) { return MIN ? min(a, b) : a + b; };
  if constexpr (G <= 32) {
#pragma unroll
    for (int d = G / 2; d >= 1; d >>= 1) v = op(v, __shfl_xor_sync(g.mask, v, d, G));
    return v;
  } else {
    constexpr int NW = G / 32;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, d));
    if (lane == 0) tmp[wid] = v;
    __syncthreads();
    int m = tmp[0];
#pragma unroll
    for (int w = 1; w < NW; ++w) m = op(m, tmp[w]);
    __syncthreads();
    return m;
  }
}

// Merge path: number of a-elements among the first `diag` merged elements,
// a-first on equal columns.
__device__ __forceinline__ int merge_path(const int* a, int la, const int* b, int lb, int diag) {
  int lo = diag - lb > 0 ? diag - lb : 0;
  int hi = diag < la ? diag : la;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] <= b[diag - 1 - mid])
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

}  // namespace brm
