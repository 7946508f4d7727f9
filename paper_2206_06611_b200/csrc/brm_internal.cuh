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
// Row tiers. A row with n_prod > 0 goes to the first tier t (1..5) with
// n_prod <= cap and num_list (= nnz(A_i*)) <= lcap, else to the global tier 6.
// Tier t's kernel runs `gpc` groups of `g` threads per CTA; each group owns one
// row at a time with both ping-pong buffers in shared memory.
// ---------------------------------------------------------------------------
constexpr int kBinEmpty = 0;
constexpr int kBinGlobal = 6;
static_assert(BRM_NUM_BINS == 7, "tier table below assumes 7 bins");

struct TierBounds {
  int cap[BRM_NUM_BINS];
  int lcap[BRM_NUM_BINS];
};

// (G threads per row group, VT merged positions per thread per chunk,
//  CAP elements, LCAP lists, GPC groups per CTA)
#define BRM_TIER1 8, 8, 64, 32, 16
#define BRM_TIER2 32, 8, 256, 128, 4
#define BRM_TIER3 32, 8, 768, 64, 1
#define BRM_TIER4 128, 8, 2560, 512, 1
#define BRM_TIER5 256, 8, 7168, 1024, 1
constexpr int kGlobalG = 512;
constexpr int kGlobalVT = 8;

__host__ __device__ inline TierBounds tier_bounds() {
  TierBounds t{};
  t.cap[0] = 0;    t.lcap[0] = 0;
  t.cap[1] = 64;   t.lcap[1] = 32;
  t.cap[2] = 256;  t.lcap[2] = 128;
  t.cap[3] = 768;  t.lcap[3] = 64;
  t.cap[4] = 2560; t.lcap[4] = 512;
  t.cap[5] = 7168; t.lcap[5] = 1024;
  t.cap[6] = INT_MAX; t.lcap[6] = INT_MAX;
  return t;
}

__host__ __device__ inline int tier_of(int64_t nprod, int64_t nl, const TierBounds& tb) {
  if (nprod == 0) return kBinEmpty;
#pragma unroll
  for (int t = 1; t < kBinGlobal; ++t)
    if (nprod <= tb.cap[t] && nl <= tb.lcap[t]) return t;
  return kBinGlobal;
}

// Shared-memory layout of one row group (bytes, 16-aligned pieces). colA /
// valA hold the gathered lists in 16-byte TMA windows, so they get padding
// (capc / capv elements); rows whose windows do not fit use cp.async.
struct GroupLayout {
  int valA, valB, colA, colB, lstA, llnA, lstB, llnB, vb, cst, cpair, mbar, scan, bytes, capc, capv;
};

__host__ __device__ constexpr int align16(int x) { return (x + 15) & ~15; }

template <int G, int VT, int CAP, int LCAP, bool VALS>
__host__ __device__ constexpr GroupLayout group_layout() {
  GroupLayout L{};
  L.capc = CAP + (LCAP > CAP / 4 ? LCAP : CAP / 4);
  L.capv = CAP + (LCAP > CAP / 8 ? LCAP : CAP / 8);
  int o = 0;
  L.valA = o;   o += VALS ? align16(L.capv * 8 + 16) : 0;
  L.valB = o;   o += VALS ? align16((CAP + LCAP / 2 + 2) * 8) : 0;
  L.colA = o;   o += align16(L.capc * 4 + 16);
  L.colB = o;   o += align16((CAP + LCAP / 2 + 2) * 4);
  L.lstA = o;   o += align16((LCAP + 1) * 4);
  L.llnA = o;   o += align16((LCAP + 1) * 4);
  L.lstB = o;   o += align16((LCAP / 2 + 2) * 4);
  L.llnB = o;   o += align16((LCAP / 2 + 2) * 4);
  L.vb = o;     o += VALS ? align16(LCAP * 4) : 0;
  L.cst = o;    o += align16((LCAP / 2 + 2) * 4);
  L.cpair = o;  o += align16((CAP / VT + LCAP / 2 + 2) * 4);
  L.mbar = o;   o += 16;
  L.scan = o;   o += G > 32 ? align16((G / 32 + 1) * 4) : 0;
  L.bytes = o;
  return L;
}

// ---------------------------------------------------------------------------
// Thread groups: G <= 32 is a sub-warp (shuffles of width G), G > 32 is the
// whole CTA (blockDim.x == G).
// ---------------------------------------------------------------------------
template <int G>
struct Group {
  int rank;
  unsigned mask;
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
  if constexpr (G >= 32)
    g.mask = 0xffffffffu;
  else
    g.mask = ((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1));
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

// Largest l in [0, n) with off[l * stride] <= e (n >= 1). With empty lists
// sharing a start, this is the non-empty list that contains position e.
template <int STRIDE>
__device__ __forceinline__ int upper_search(const int* off, int n, int e) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off[mid * STRIDE] <= e)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
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
