// kernels.cu -- every device kernel of libbrmerge (sm_100a).
//
//   k_nprod_scan     Step 1 of Fig. 4a/4b: n_prod per row
//                    (§II.B.2) fused with a single-pass decoupled look-back
//                    exclusive scan (CUB-free), the per-bin histogram and max.
//   k_bin_scatter    row binning by n_prod / list count into tiers.
//   k_tiny           tier 1: one thread per row runs Algorithm 1 literally.
//   k_tier<...>      tier 2: register BRMerge, one warp per row; tiers 3-6:
//                    record BRMerge (warp / warp / 128 / 256 threads per row).
//   k_hash_symbolic  BRMerge-Precise step 3 on tiers 3-6: per-row shared
//                    hash table counts the distinct columns.
//   (heavy.cu)       tier 7: k_hv_plan / k_hv_merge, windowed BRMerge.
//   k_global_tier    tier 7 under BRM_HEAVY_GLOBAL: ping-pong buffers in a
//                    global workspace, one 1024-thread CTA per row.
//   k_scan_i64       exclusive scan (row_size -> rpt; generic).
//   k_compact        Step 6 of Fig. 4a: C_bar -> C copy (BRMerge-Upper).
//   k_partition      §III.D row partition by balanced n_prod (multi-GPU).
//   k_row_nprod      n_prod per row (stage entry point).
#include <algorithm>
#include <cstdio>
#include <type_traits>

#include "engine.cuh"
#include "kernels.cuh"

namespace brm {

static int num_sms();

// ---------------------------------------------------------------------------
// Single-pass exclusive scan with decoupled look-back (Merrill & Garland
// style, hand-written). Tile status words pack a 2-bit flag over a 62-bit sum.
// ---------------------------------------------------------------------------
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPre = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Called by all threads of warp 0 of the tile's CTA; returns the exclusive
// prefix of this tile and publishes its inclusive prefix.
__device__ int64_t lookback(unsigned long long* status, int tile, int64_t aggregate) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_status(status, kFlagPre | (unsigned long long)aggregate);
    return 0;
  }
  if (lane == 0) st_status(status + tile, kFlagAgg | (unsigned long long)aggregate);
  int64_t excl = 0;
  int t = tile - 1;
  while (true) {
    const int idx = t - lane;
    unsigned long long w = kFlagPre;  // virtual prefix 0 before tile 0
    if (idx >= 0) {
      do {
        w = ld_status(status + idx);
      } while ((w >> 62) == 0);
    }
    const unsigned pmask = __ballot_sync(0xffffffffu, (w >> 62) == 2);
    int64_t v = (int64_t)(w & kValMask);
    if (pmask) {
      const int first = __ffs(pmask) - 1;  // closest tile with a full prefix
      if (lane > first) v = 0;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    excl += v;
    if (pmask) break;
    t -= 32;
  }
  if (lane == 0) st_status(status + tile, kFlagPre | (unsigned long long)(excl + aggregate));
  return excl;
}

constexpr int kScanThreads = 256;
constexpr int kScanIPT = 8;
constexpr int kScanTile = kScanThreads * kScanIPT;

// Block-wide exclusive scan of int64 thread sums; returns this thread's
// exclusive offset and the block total.
__device__ __forceinline__ int64_t block_scan_i64(int64_t x, int64_t& total, int64_t* wsum) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t inc = x;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += y;
  }
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    constexpr int NW = kScanThreads / 32;
    const int64_t w = lane < NW ? wsum[lane] : 0;
    int64_t wx = w;
#pragma unroll
    for (int d = 1; d < NW; d <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, wx, d);
      if (lane >= d) wx += y;
    }
    if (lane < NW) wsum[lane] = wx - w;
    if (lane == NW - 1) wsum[NW] = wx;
  }
  __syncthreads();
  total = wsum[kScanThreads / 32];
  return wsum[wid] + inc - x;
}

constexpr int kLongRow = 512;  // rows of more nonzeros: k_long_rows / k_long_nprod

// n_prod of the 32 rows [r0, r0 + 32) by one warp, nonzero-parallel: lanes
// stride over the rows' nonzeros (coalesced A.col reads, B.rpt gathers; four
// 32-nonzero batches in flight), find each nonzero's row by a shuffle search
// over the row starts, and sum runs of equal rows with a segmented shuffle
// scan; the last lane of a run adds it to out[row - r0]. *nl_out = lane's
// row length.
__device__ __forceinline__ void warp_rows_nprod(const CsrView& A, const int64_t* __restrict__ brpt, int64_t M,
                                                int64_t r0, int64_t* out, int* nl_out,
                                                const int64_t* __restrict__ long_np) {
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  const int64_t rs = A.rpt[min(r0 + lane, M)];  // start of row r0 + lane (clamped)
  const int64_t pend = A.rpt[min(r0 + 32, M)];
  const int64_t rnext = __shfl_down_sync(0xffffffffu, rs, 1);
  const int nl = lane < 31 ? (int)(rnext - rs) : (int)(pend - rs);
  *nl_out = nl;
  const bool valid = r0 + lane < M;
  // rows of more than kLongRow nonzeros were summed by k_long_nprod (if it ran)
  const bool lng = long_np != nullptr && valid && nl > kLongRow;
  const unsigned longm = __ballot_sync(0xffffffffu, lng);
  if (__reduce_max_sync(0xffffffffu, valid && !lng ? (unsigned)nl : 0u) <= 64u) {
    // short rows: one lane per row, independent gathers (no shuffles)
    int64_t acc = 0;
    if (lng) {
      acc = long_np[r0 + lane];
    } else if (valid) {
#ifndef BRM_NPS_U8
#define BRM_NPS_U8 0  // 1: eight of a row's gathers in flight instead of four (tuning switch)
#endif
#if BRM_NPS_U8
#pragma unroll 8
#else
#pragma unroll 4
#endif
      for (int64_t p = rs; p < rs + nl; ++p) {
        const int k = __ldg(A.col + p);
        acc += __ldg(brpt + k + 1) - __ldg(brpt + k);
      }
    }
    out[lane] = acc;
    __syncwarp();
    return;
  }
  out[lane] = lng ? long_np[r0 + lane] : 0;
  __syncwarp();
  // the other rows nonzero-parallel, one run of consecutive such rows at a time
  const int nvalid = (int)min((int64_t)32, M - r0);
  int ra = 0;
  while (ra < nvalid) {
    if ((longm >> ra) & 1u) {
      ++ra;
      continue;
    }
    const unsigned after = longm & ~((2u << ra) - 1u);  // long rows past ra
    const int rb = after ? __ffs(after) - 1 : nvalid;
    const int64_t pbeg = __shfl_sync(0xffffffffu, rs, ra);
    const int64_t rbs = __shfl_sync(0xffffffffu, rs, rb < nvalid ? rb : 0);
    const int64_t prun = rb < nvalid ? rbs : pend;  // the run's nonzeros: [pbeg, prun)
    ra = rb;
    for (int64_t pb = pbeg; pb < prun; pb += 32 * U) {
      int k[U];
      int64_t d[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t p = pb + 32 * u + lane;
        k[u] = p < prun ? __ldg(A.col + p) : -1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) d[u] = k[u] >= 0 ? __ldg(brpt + k[u] + 1) - __ldg(brpt + k[u]) : 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t p = pb + 32 * u + lane;
        if (pb + 32 * u >= prun) break;  // warp-uniform
        int lo = 0;  // row of nonzero p: last lane whose row start <= p
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const int64_t v = __shfl_sync(0xffffffffu, rs, lo + step);
          if (v <= p) lo += step;
        }
        int64_t x = d[u];  // segmented inclusive scan over lanes with equal rows
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
          const int ro = __shfl_up_sync(0xffffffffu, lo, o);
          if (lane >= o && ro == lo) x += y;
        }
        const int rn = __shfl_down_sync(0xffffffffu, lo, 1);
        if (p < prun && (lane == 31 || rn != lo || p + 1 >= prun)) out[lo] += x;
        __syncwarp();
      }
    }
  }
}

// Rows of more than kLongRow nonzeros (power-law rows): listed first, then
// summed by a CTA each, so no warp of k_nprod_scan carries a huge row alone
// (rmat20's 32-row chunk holding the first rows took the whole 10.8 ms).
__global__ void k_long_rows(CsrView A, int64_t M, int32_t* __restrict__ list, unsigned int* count) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < M && A.rpt[r + 1] - A.rpt[r] > kLongRow) list[atomicAdd(count, 1u)] = (int32_t)r;
}

__global__ void __launch_bounds__(256) k_long_nprod(CsrView A, const int64_t* __restrict__ brpt,
                                                    const int32_t* __restrict__ list, const unsigned int* count,
                                                    int64_t* __restrict__ long_np) {
  __shared__ int64_t red[8];
  const unsigned n = *count;
  for (unsigned i = blockIdx.x; i < n; i += gridDim.x) {
    const int64_t r = list[i];
    const int64_t p0 = A.rpt[r], p1 = A.rpt[r + 1];
    int64_t s = 0;
#pragma unroll 4
    for (int64_t p = p0 + threadIdx.x; p < p1; p += 256) {
      const int k = __ldg(A.col + p);
      s += __ldg(brpt + k + 1) - __ldg(brpt + k);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t t = 0;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += red[w];
      long_np[r] = t;
    }
    __syncthreads();
  }
}

// Step 1: n_prod per row + exclusive scan + bin histogram + max. A tile of
// 2048 rows per CTA: each warp computes 8 chunks of 32 rows (warp_rows_nprod)
// into shared memory, then the tile is scanned (8 consecutive rows per
// thread) with a decoupled look-back across tiles. Large tiles keep the
// look-back chain short (4.2M rows -> 2048 tiles).
constexpr int kNpTile = kScanTile;
#ifndef BRM_NPS_MINB
#define BRM_NPS_MINB 5  // launch-bounds CTAs per SM of k_nprod_scan: 48 registers, 5 CTAs (63 / 4 without a bound);
// the pass waits on dependent loads (long-scoreboard 10.7 per issue on AMG): AMG 0.1946 -> 0.1734 ms with 5,
// 0.1765 with 6 (spills); uniform1m_k16 0.1739 -> 0.1788 (profiles/r02k/nps)
#endif
__global__ void __launch_bounds__(kScanThreads, BRM_NPS_MINB) k_nprod_scan(CsrView A, const int64_t* __restrict__ brpt,
                                                             int64_t M, int64_t* __restrict__ nprod_off,
                                                             unsigned long long* status,
                                                             unsigned int* tile_counter,
                                                             DevSummary* summary,
                                                             const int64_t* __restrict__ long_np) {
  __shared__ int s_tile;
  __shared__ int64_t s_wsum[kScanThreads / 32 + 1];
  __shared__ int64_t s_prefix;
  __shared__ int64_t s_np[kNpTile];
  __shared__ unsigned long long s_bin_rows[BRM_NUM_BINS];
  __shared__ unsigned long long s_bin_nprod[BRM_NUM_BINS];
  __shared__ unsigned long long s_max, s_maxnl;
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(tile_counter, 1u);
  if (threadIdx.x < BRM_NUM_BINS) {
    s_bin_rows[threadIdx.x] = 0;
    s_bin_nprod[threadIdx.x] = 0;
  }
  if (threadIdx.x == 0) { s_max = 0; s_maxnl = 0; }
  __syncthreads();
  const int tile = s_tile;
  const TierBounds tb = tier_bounds();
  const int64_t t0 = (int64_t)tile * kNpTile;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kChunks = kNpTile / kScanThreads;  // chunks of 32 rows per warp
  for (int c = 0; c < kChunks; ++c) {
    const int loc = (wid * kChunks + c) * 32;
    const int64_t r0 = t0 + loc;
    if (r0 >= M) break;  // warp-uniform
    int nl;
    warp_rows_nprod(A, brpt, M, r0, s_np + loc, &nl, long_np);
    const bool valid = r0 + lane < M;
    const int64_t s = valid ? s_np[loc + lane] : 0;
    const int bin = valid ? tier_of(s, nl, tb) : -1;
    // warp-aggregated histogram: one shared atomic per distinct bin per warp
    unsigned todo = __ballot_sync(0xffffffffu, valid);
    while (todo) {
      const int leader = __ffs(todo) - 1;
      const int b = __shfl_sync(0xffffffffu, bin, leader);
      const unsigned m = __ballot_sync(0xffffffffu, bin == b);
      unsigned long long x = bin == b ? (unsigned long long)s : 0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == leader) {
        atomicAdd(&s_bin_rows[b], (unsigned long long)__popc(m));
        atomicAdd(&s_bin_nprod[b], x);
      }
      todo &= ~m;
    }
    const unsigned smax = __reduce_max_sync(0xffffffffu, (unsigned)min(s, (int64_t)0xffffffffll));
    const unsigned lmax = __reduce_max_sync(0xffffffffu, valid ? (unsigned)nl : 0u);
    if (lane == 0) {
      atomicMax(&s_max, (unsigned long long)smax);
      atomicMax(&s_maxnl, (unsigned long long)lmax);
    }
  }
  __syncthreads();
  const int64_t rb = t0 + (int64_t)threadIdx.x * kScanIPT;
  int64_t v[kScanIPT];
  int64_t tsum = 0;
#pragma unroll
  for (int t = 0; t < kScanIPT; ++t) {
    v[t] = rb + t < M ? s_np[threadIdx.x * kScanIPT + t] : 0;
    tsum += v[t];
  }
  int64_t total;
  const int64_t texcl = block_scan_i64(tsum, total, s_wsum);
  if (threadIdx.x < 32) {
    const int64_t pre = lookback(status, tile, total);
    if (threadIdx.x == 0) s_prefix = pre;
  }
  __syncthreads();
  int64_t run = s_prefix + texcl;
#pragma unroll
  for (int t = 0; t < kScanIPT; ++t) {
    const int64_t r = rb + t;
    if (r < M) nprod_off[r] = run;
    run += v[t];
    if (r == M - 1) {
      nprod_off[M] = run;
      summary->nprod_total = run;
    }
  }
  if (threadIdx.x < BRM_NUM_BINS) {
    if (s_bin_rows[threadIdx.x]) {
      atomicAdd(&summary->bin_rows[threadIdx.x], s_bin_rows[threadIdx.x]);
      atomicAdd(&summary->bin_nprod[threadIdx.x], s_bin_nprod[threadIdx.x]);
    }
  }
  if (threadIdx.x == 0) {
    atomicMax(&summary->nprod_max, s_max);
    atomicMax(&summary->nl_max, s_maxnl);
  }
}

// Generic exclusive scan: out[i] = sum_{r<i} in[r], out[n] = total.
__global__ void __launch_bounds__(kScanThreads) k_scan_i64(const int64_t* __restrict__ in, int64_t n,
                                                           int64_t* __restrict__ out,
                                                           unsigned long long* status,
                                                           unsigned int* tile_counter,
                                                           int64_t* total_out) {
  __shared__ int s_tile;
  __shared__ int64_t s_wsum[kScanThreads / 32 + 1];
  __shared__ int64_t s_prefix;
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(tile_counter, 1u);
  __syncthreads();
  const int tile = s_tile;
  const int64_t r0 = (int64_t)tile * kScanTile + (int64_t)threadIdx.x * kScanIPT;
  int64_t v[kScanIPT];
  int64_t tsum = 0;
#pragma unroll
  for (int t = 0; t < kScanIPT; ++t) {
    const int64_t r = r0 + t;
    v[t] = r < n ? in[r] : 0;
    tsum += v[t];
  }
  int64_t total;
  const int64_t texcl = block_scan_i64(tsum, total, s_wsum);
  if (threadIdx.x < 32) {
    const int64_t pre = lookback(status, tile, total);
    if (threadIdx.x == 0) s_prefix = pre;
  }
  __syncthreads();
  int64_t run = s_prefix + texcl;
#pragma unroll
  for (int t = 0; t < kScanIPT; ++t) {
    const int64_t r = r0 + t;
    if (r < n) out[r] = run;
    run += v[t];
    if (r == n - 1) {
      out[n] = run;
      if (total_out) *total_out = run;
    }
  }
}

// Row binning: rows of bin b are written to bins[bin_start[b] + ...]; rows with
// n_prod == 0 get row_size = 0 and are not stored. One global atomic per
// (CTA, bin).
constexpr int kBinThreads = 256;
constexpr int kBinRowsPerCta = 2048;
__global__ void __launch_bounds__(kBinThreads) k_bin_scatter(CsrView A, const int64_t* __restrict__ nprod_off,
                                                             int64_t M, const DevSummary* summary,
                                                             unsigned long long* bin_cursor,
                                                             int32_t* __restrict__ bins,
                                                             int64_t* __restrict__ row_size) {
  __shared__ unsigned int s_cnt[BRM_NUM_BINS];
  __shared__ unsigned long long s_base[BRM_NUM_BINS];
  __shared__ long long s_start[BRM_NUM_BINS];
  if (threadIdx.x < BRM_NUM_BINS) s_cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    long long acc = 0;
    for (int b = 0; b < BRM_NUM_BINS; ++b) {
      s_start[b] = acc;
      if (b != kBinEmpty) acc += (long long)summary->bin_rows[b];
    }
  }
  __syncthreads();
  const TierBounds tb = tier_bounds();
  constexpr int IPT = kBinRowsPerCta / kBinThreads;
  int bin[IPT];
  unsigned int rank[IPT];
  const int64_t base = (int64_t)blockIdx.x * kBinRowsPerCta;
#pragma unroll
  for (int t = 0; t < IPT; ++t) {
    const int64_t r = base + (int64_t)t * kBinThreads + threadIdx.x;
    bin[t] = -1;
    if (r < M) {
      const int64_t s = nprod_off[r + 1] - nprod_off[r];
      const int b = tier_of(s, A.rpt[r + 1] - A.rpt[r], tb);
      if (b == kBinEmpty) {
        row_size[r] = 0;
      } else {
        bin[t] = b;
        // warp-aggregated rank within the CTA
        const unsigned peers = __match_any_sync(__activemask(), b);
        const int leader = __ffs(peers) - 1;
        const int lane = threadIdx.x & 31;
        unsigned int off = 0;
        if (lane == leader) off = atomicAdd(&s_cnt[b], (unsigned)__popc(peers));
        off = __shfl_sync(peers, off, leader);
        rank[t] = off + __popc(peers & ((1u << lane) - 1u));
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < BRM_NUM_BINS && s_cnt[threadIdx.x])
    s_base[threadIdx.x] = atomicAdd(&bin_cursor[threadIdx.x], (unsigned long long)s_cnt[threadIdx.x]);
  __syncthreads();
#pragma unroll
  for (int t = 0; t < IPT; ++t) {
    const int64_t r = base + (int64_t)t * kBinThreads + threadIdx.x;
    if (bin[t] >= 0) bins[s_start[bin[t]] + s_base[bin[t]] + rank[t]] = (int32_t)r;
  }
}

// (n_prod, num_list) of the global-tier rows, for host-side batching.
__global__ void k_heavy_info(CsrView A, const int64_t* __restrict__ nprod_off,
                             const int32_t* __restrict__ rows, int64_t n, int64_t* __restrict__ info) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) {
    const int64_t r = rows[t];
    info[2 * t] = nprod_off[r + 1] - nprod_off[r];
    info[2 * t + 1] = A.rpt[r + 1] - A.rpt[r];
  }
}

// Tiers 2-6: GPC groups of G threads per CTA, one row per group at a time,
// the group's buffers in its slice of dynamic shared memory. CAP <= 32:
// register tier (reg_row), else record tier (rec_row) with records of type
// RecT<VALS, PACK, CAP> (PACK: 32-bit {col, slot} records).
template <bool VALS, bool PACK, int CAP>
using RecT = std::conditional_t<VALS, std::conditional_t<PACK, RecPacked<rec_slot_bits(CAP)>, RecWide>, RecCol>;

// carve one record group's buffers (rec_group_bytes) out of shared memory
template <int G, int CAP, int LCAP, class R, bool CUR>
__device__ __forceinline__ RecBufs rec_bufs(unsigned char* p) {
  auto take = [&](int n) {
    unsigned char* q = p;
    p += align16(n);
    return q;
  };
  RecBufs rb;
  rb.rec = take((CAP + LCAP + 2) * R::kBytes);
  rb.lst = reinterpret_cast<longlong2*>(take(LCAP * 16));
  if (R::kVals) {
    rb.val = reinterpret_cast<double*>(take(CAP * 8));
    rb.owner = reinterpret_cast<unsigned short*>(rb.val);  // laid over the value slots
    rb.ostr = 4;
  } else {
    rb.val = nullptr;
    rb.owner = reinterpret_cast<unsigned short*>(take(CAP * 2));
    rb.ostr = 1;
  }
  rb.off0 = reinterpret_cast<int*>(take((LCAP + 2) * 4));
  rb.off1 = reinterpret_cast<int*>(take((LCAP + 2) * 4));
  rb.bst = CUR ? reinterpret_cast<int64_t*>(take(LCAP * 8)) : nullptr;
  rb.av = CUR && R::kVals ? reinterpret_cast<double*>(take(LCAP * 8)) : nullptr;
  rb.scan_tmp = G > 32 ? reinterpret_cast<int*>(take((G / 32 + 2) * 4)) : nullptr;
  return rb;
}

template <int G, int CAP, int LCAP, int GPC, bool PLAIN, bool VALS, int OUT, bool PACK>
__global__ void __launch_bounds__(G * GPC) k_tier(CsrView A, CsrView B, const int32_t* __restrict__ rows,
                                                 int64_t nrows, RowOut o) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Group<G> g = make_group<G>();
  const int gid = threadIdx.x / G;
  if constexpr (CAP <= 32) {
    constexpr int bytes = reg_group_bytes<G, VALS>();
    unsigned char* base = smem + gid * bytes;
    RegBufs rb;
    rb.col = reinterpret_cast<int*>(base);
    rb.lid = reinterpret_cast<int*>(base + align16(G * 4));
    rb.owner = reinterpret_cast<int*>(base + 2 * align16(G * 4));
    rb.val = VALS ? reinterpret_cast<double*>(base + 3 * align16(G * 4)) : nullptr;
    for (int64_t r = (int64_t)blockIdx.x * GPC + gid; r < nrows; r += (int64_t)gridDim.x * GPC)
      reg_row<G, VALS, OUT>(g, A, B, rows[r], o, rb);
  } else {
    using R = RecT<VALS, PACK, CAP>;
    const RecBufs rb = rec_bufs<G, CAP, LCAP, R, false>(smem + gid * rec_group_bytes<G, CAP, LCAP, R, false>());
    for (int64_t r = (int64_t)blockIdx.x * GPC + gid; r < nrows; r += (int64_t)gridDim.x * GPC)
      rec_row<G, ((CAP + LCAP + 1 + G - 1) / G) | 1, R, OUT, PLAIN>(g, A, B, rows[r], o, rb);
  }
}

// PRECISE symbolic phase of tiers 3-6: hash_row per group (GPC groups of G).
template <int G, int CAP, int LCAP, int GPC, int HB, int HQ, bool DIRECT>
__global__ void __launch_bounds__(G * GPC) k_hash_symbolic(CsrView A, CsrView B, const int32_t* __restrict__ rows,
                                                          int64_t nrows, RowOut o) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Group<G> g = make_group<G>();
  const int gid = threadIdx.x / G;
  constexpr bool STAGE = hash_staged<G, HB>();
  unsigned char* p = smem + gid * hash_group_bytes<G, CAP, LCAP, HQ, STAGE>();
  auto take = [&](int n) {
    unsigned char* q = p;
    p += align16(n);
    return q;
  };
  HashBufs hb;
  hb.table = reinterpret_cast<int*>(take(hash_cap<CAP, HQ>() * 4));
  hb.owner = reinterpret_cast<unsigned short*>(take(CAP * 2));
  hb.off = reinterpret_cast<int*>(take((LCAP + 1) * 4));
  hb.bst = reinterpret_cast<int64_t*>(take(LCAP * 8));
  hb.scan_tmp = G > 32 ? reinterpret_cast<int*>(take((G / 32 + 2) * 4)) : nullptr;
  hb.stage = STAGE ? reinterpret_cast<int*>(take(CAP * 4)) : nullptr;
  for (int64_t r = (int64_t)blockIdx.x * GPC + gid; r < nrows; r += (int64_t)gridDim.x * GPC)
    hash_row<G, CAP, HB, HQ, DIRECT>(g, A, B, rows[r], o, hb);
}

// Tier 1: one thread per row (tiny_row), NT threads per CTA.
constexpr int kTinyNT = 128;
template <bool VALS, int OUT>
__global__ void __launch_bounds__(kTinyNT) k_tiny(CsrView A, CsrView B, const int32_t* __restrict__ rows,
                                                 int64_t nrows, RowOut o) {
  extern __shared__ __align__(16) unsigned char smem[];
  int* pc = reinterpret_cast<int*>(smem) + threadIdx.x;
  int* qc = pc + kTinyNT * kTinyP;
  double* pv = VALS ? reinterpret_cast<double*>(smem + kTinyNT * kTinyP * 8) + threadIdx.x : nullptr;
  double* qv = VALS ? pv + kTinyNT * kTinyP : nullptr;
  // (the row id two rows ahead and the row bounds one row ahead loaded while a
  // row merges -- two links off the row's chain of dependent loads -- measured
  // no faster at equal registers: 0.1978 vs 0.1956 ms on AMG, profiles/r02i/tiny_pipe)
  for (int64_t t = (int64_t)blockIdx.x * kTinyNT + threadIdx.x; t < nrows; t += (int64_t)gridDim.x * kTinyNT) {
    const int64_t row = rows[t];
    const int64_t a0 = A.rpt[row];
    tiny_row<kTinyNT, VALS, OUT>(A, B, row, a0, static_cast<int>(A.rpt[row + 1] - a0), o, pc, qc, pv, qv);
  }
}

// Global tier: one CTA per row, ping-pong buffers in a per-row slice of a
// global workspace at byte offset ws_off[2r] (host-batched; ws_off[2r+1] is
// the row's n_prod).
template <bool VALS, int OUT>
__global__ void __launch_bounds__(kGlobalG) k_global_tier(CsrView A, CsrView B, const int32_t* __restrict__ rows,
                                                         const int64_t* __restrict__ ws_off,
                                                         unsigned char* __restrict__ ws, RowOut o) {
  __shared__ int scan_tmp[kGlobalG / 32 + 2];
  const Group<kGlobalG> g = make_group<kGlobalG>();
  const int64_t row = rows[blockIdx.x];
  const int64_t P = ws_off[2 * blockIdx.x + 1];
  const int64_t nl = A.rpt[row + 1] - A.rpt[row];
  unsigned char* p = ws + ws_off[2 * blockIdx.x];
  auto take = [&](int64_t bytes) {
    unsigned char* q = p;
    p += (bytes + 15) & ~15ll;
    return q;
  };
  ChunkBufs cb;
  cb.col0 = reinterpret_cast<int*>(take((P + nl + 2) * 4));
  cb.col1 = reinterpret_cast<int*>(take((P + nl + 2) * 4));
  cb.val0 = VALS ? reinterpret_cast<double*>(take((P + nl + 2) * 8)) : nullptr;
  cb.val1 = VALS ? reinterpret_cast<double*>(take((P + nl + 2) * 8)) : nullptr;
  cb.off0 = reinterpret_cast<int*>(take((nl + 2) * 4));
  cb.off1 = reinterpret_cast<int*>(take((nl + 2) * 4));
  cb.bst = reinterpret_cast<int64_t*>(take(nl * 8));
  cb.av = VALS ? reinterpret_cast<double*>(take(nl * 8)) : nullptr;
  cb.scan_tmp = scan_tmp;
  chunk_row<kGlobalG, VALS, OUT>(g, A, B, row, o, cb);
}

// Step 6 of Fig. 4a: copy each row of C_bar (at its n_prod offset) to C.
// Work is cut by ELEMENTS of C, not rows, so a few very long rows (heavy
// rows, or a heavy-row decomposition's sub-products) spread over all warps:
// a warp takes chunks of kCompactChunk consecutive elements of C, finds the
// row of the chunk's first element by a binary search over C.rpt, then
// walks the chunk through windows of 32 consecutive rows; element e's row is
// found by a shuffle search over the window's row starts, its source is
// nprod_off[row] + (e - crpt[row]). Stores are coalesced.
constexpr int64_t kCompactChunk = 4096;
#ifndef BRM_COMPACT_U
#define BRM_COMPACT_U 4
#endif

__global__ void __launch_bounds__(256) k_compact(int64_t M, const int64_t* __restrict__ nprod_off,
                                                 const int64_t* __restrict__ crpt,
                                                 const int32_t* __restrict__ cbar_col,
                                                 const double* __restrict__ cbar_val,
                                                 int32_t* __restrict__ ccol, double* __restrict__ cval, Mirrors mir) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nnz = crpt[M];
  for (int64_t e0 = warp * kCompactChunk; e0 < nnz; e0 += nwarps * kCompactChunk) {
    const int64_t e1 = min(e0 + kCompactChunk, nnz);
    int64_t lo = 0, hi = M - 1;  // last row r with crpt[r] <= e0 (same on every lane)
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (crpt[mid] <= e0)
        lo = mid;
      else
        hi = mid - 1;
    }
    int64_t r0 = lo;
    int64_t eb0 = e0;
    while (eb0 < e1) {
      const int64_t r = min(r0 + lane, M);
      const int64_t cs = crpt[r];
      const int64_t delta = (r < M ? nprod_off[r] : 0) - cs;  // source - destination
      const int64_t wend = min(e1, crpt[min(r0 + 32, M)]);
      constexpr int U = BRM_COMPACT_U;  // 32-element batches in flight per warp
      for (int64_t eb = eb0; eb < wend; eb += 32 * U) {
        int32_t cv[U];
        double vv[U];
        int64_t dst[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t e = eb + 32 * u + lane;
          int l = 0;  // row of element e: last lane whose C start <= e
#pragma unroll
          for (int step = 16; step > 0; step >>= 1) {
            const int64_t v = __shfl_sync(0xffffffffu, cs, l + step);
            if (v <= e) l += step;
          }
          const int64_t d = __shfl_sync(0xffffffffu, delta, l);
          dst[u] = e < wend ? e : -1;
          cv[u] = 0;
          vv[u] = 0.0;
          if (e < wend) {
            cv[u] = cbar_col[e + d];
            vv[u] = cbar_val[e + d];
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (dst[u] >= 0) {
            ccol[dst[u]] = cv[u];
            cval[dst[u]] = vv[u];
          }
        if (mir.n) {  // (one test per batch)
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (dst[u] >= 0) mirror_store<true>(mir, dst[u], cv[u], vv[u]);
        }
      }
      eb0 = wend;
      r0 += 32;
    }
  }
}

// §III.D: bounds[g] = first row r with nprod_off[r] * p >= g * total.
__global__ void k_partition(const int64_t* __restrict__ nprod_off, int64_t M, int p,
                            int64_t* __restrict__ bounds) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g > p) return;
  if (g == 0) { bounds[0] = 0; return; }
  if (g == p) { bounds[p] = M; return; }
  const __int128 target = (__int128)g * nprod_off[M];
  int64_t lo = 0, hi = M;  // answer in [0, M]
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((__int128)nprod_off[mid] * p >= target)
      hi = mid;
    else
      lo = mid + 1;
  }
  bounds[g] = lo;
}

// n_prod per row only (stage entry point): 32 rows per warp as in k_nprod_scan.
__global__ void __launch_bounds__(256) k_row_nprod(CsrView A, const int64_t* __restrict__ brpt, int64_t M,
                                                   int64_t* __restrict__ nprod, const int64_t* __restrict__ long_np) {
  __shared__ int64_t s_np[256];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * 256 + wid * 32;
  if (r0 >= M) return;  // warp-uniform
  int nl;
  warp_rows_nprod(A, brpt, M, r0, s_np + wid * 32, &nl, long_np);
  if (r0 + lane < M) nprod[r0 + lane] = s_np[wid * 32 + lane];
}

// ---------------------------------------------------------------------------
// Host-side launchers.
// ---------------------------------------------------------------------------
// Launch setup is per DEVICE (the shared-memory attribute and the occupancy
// apply to the current device only): cached per device ordinal.
constexpr int kMaxDevices = 64;
static int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev < 0 || dev >= kMaxDevices ? 0 : dev;
}
static int num_sms() {
  static int n[kMaxDevices] = {};
  const int dev = current_device();
  if (!n[dev]) {
    cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev);
    if (n[dev] <= 0) n[dev] = 148;
  }
  return n[dev];
}

// One kernel instantiation's setup on the current device: raise its dynamic
// shared-memory limit to `smem` and return its resident CTAs per SM.
struct LaunchSetup {
  int per_sm[kMaxDevices] = {};
};
template <class K>
static cudaError_t kernel_setup(LaunchSetup& ls, K kern, int threads, int smem, int& per_sm) {
  const int dev = current_device();
  if (!ls.per_sm[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int n = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, smem);
    if (e != cudaSuccess) return e;
    ls.per_sm[dev] = n < 1 ? 1 : n;
  }
  per_sm = ls.per_sm[dev];
  return cudaSuccess;
}

int64_t scan_tiles(int64_t n) { return (n + kScanTile - 1) / kScanTile; }

int64_t nprod_tiles(int64_t M) { return (M + kNpTile - 1) / kNpTile; }

cudaError_t launch_long_rows(const CsrView& A, const int64_t* brpt, int64_t M, int32_t* list, unsigned int* count,
                             int64_t* long_np, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  k_long_rows<<<(unsigned)((M + 255) / 256), 256, 0, st>>>(A, M, list, count);
  k_long_nprod<<<(unsigned)(num_sms() * 2), 256, 0, st>>>(A, brpt, list, count, long_np);
  return cudaGetLastError();
}

cudaError_t launch_nprod_scan(const CsrView& A, const int64_t* brpt, int64_t M, int64_t* nprod_off,
                              unsigned long long* status, unsigned int* counter, DevSummary* summary,
                              const int64_t* long_np, cudaStream_t st) {
  const int64_t tiles = nprod_tiles(M);
  if (tiles > 0)
    k_nprod_scan<<<(unsigned)tiles, kScanThreads, 0, st>>>(A, brpt, M, nprod_off, status, counter, summary, long_np);
  return cudaGetLastError();
}

cudaError_t launch_scan_i64(const int64_t* in, int64_t n, int64_t* out, unsigned long long* status,
                            unsigned int* counter, int64_t* total_out, cudaStream_t st) {
  const int64_t tiles = scan_tiles(n);
  if (tiles > 0) k_scan_i64<<<(unsigned)tiles, kScanThreads, 0, st>>>(in, n, out, status, counter, total_out);
  return cudaGetLastError();
}

cudaError_t launch_bin_scatter(const CsrView& A, const int64_t* nprod_off, int64_t M, const DevSummary* summary,
                               unsigned long long* cursor, int32_t* bins, int64_t* row_size, cudaStream_t st) {
  const int64_t blocks = (M + kBinRowsPerCta - 1) / kBinRowsPerCta;
  if (blocks > 0) k_bin_scatter<<<(unsigned)blocks, kBinThreads, 0, st>>>(A, nprod_off, M, summary, cursor, bins, row_size);
  return cudaGetLastError();
}

cudaError_t launch_heavy_info(const CsrView& A, const int64_t* nprod_off, const int32_t* rows, int64_t n,
                              int64_t* info, cudaStream_t st) {
  if (n > 0) k_heavy_info<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(A, nprod_off, rows, n, info);
  return cudaGetLastError();
}

template <int G, int CAP, int LCAP, int GPC, bool PLAIN, bool VALS, int OUT, bool PACK>
static cudaError_t launch_tier_pk(const CsrView& A, const CsrView& B, const int32_t* rows, int64_t n, const RowOut& o,
                                  cudaStream_t st) {
  constexpr int per_group =
      CAP <= 32 ? reg_group_bytes<G, VALS>() : rec_group_bytes<G, CAP, LCAP, RecT<VALS, PACK, CAP>, false>();
  constexpr int smem = per_group * GPC;
  // registers hold <= NV chunk outputs; NV = 31 (G = 256, CAP 7168) miscompiled
  // (wrong values, no spills reported), so tiers keep NV <= 29
  static_assert(CAP <= 32 || (((CAP + LCAP + 1 + G - 1) / G) | 1) <= 29, "chunk tier NV must stay <= 29");
  static_assert(smem <= 232448, "tier shared memory exceeds 227 KB");
  static_assert(G <= 32 || GPC == 1, "a group of more than 32 threads is the whole CTA");
  auto kern = k_tier<G, CAP, LCAP, GPC, PLAIN, VALS, OUT, PACK>;
  static LaunchSetup ls;
  int per_sm = 0;
  if (cudaError_t e = kernel_setup(ls, kern, G * GPC, smem, per_sm); e != cudaSuccess) return e;
  const int64_t want = (n + GPC - 1) / GPC;
  const int64_t cap = (int64_t)per_sm * num_sms();
  const unsigned grid = (unsigned)(want < cap ? want : cap);
  kern<<<grid, G * GPC, smem, st>>>(A, B, rows, n, o);
  return cudaGetLastError();
}

// numeric record tiers take packed records when B's columns fit beside the slot
template <int G, int CAP, int LCAP, int GPC, bool PLAIN, bool VALS, int OUT>
static cudaError_t launch_tier_t(const CsrView& A, const CsrView& B, int64_t b_cols, const int32_t* rows, int64_t n,
                                 const RowOut& o, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if constexpr (VALS && CAP > 32) {
    if (rec_pack_ok(CAP, b_cols)) return launch_tier_pk<G, CAP, LCAP, GPC, PLAIN, VALS, OUT, true>(A, B, rows, n, o, st);
  }
  return launch_tier_pk<G, CAP, LCAP, GPC, PLAIN, VALS, OUT, false>(A, B, rows, n, o, st);
}

template <bool VALS, int OUT>
static cudaError_t launch_tiny(const CsrView& A, const CsrView& B, const int32_t* rows, int64_t n, const RowOut& o,
                              cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  constexpr int smem = tiny_block_bytes<kTinyNT, VALS>();
  auto kern = k_tiny<VALS, OUT>;
  static LaunchSetup ls;
  int per_sm = 0;
  if (cudaError_t e = kernel_setup(ls, kern, kTinyNT, smem, per_sm); e != cudaSuccess) return e;
  const int64_t want = (n + kTinyNT - 1) / kTinyNT;
  const int64_t cap = (int64_t)per_sm * num_sms();
  kern<<<(unsigned)(want < cap ? want : cap), kTinyNT, smem, st>>>(A, B, rows, n, o);
  return cudaGetLastError();
}

template <int G, int CAP, int LCAP, int GPC, int HB, int HQ, bool DIRECT>
static cudaError_t launch_hash_t(const CsrView& A, const CsrView& B, const int32_t* rows, int64_t n, const RowOut& o,
                                 cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  constexpr int smem = hash_group_bytes<G, CAP, LCAP, HQ, hash_staged<G, HB>()>() * GPC;
  static_assert(smem <= 232448, "hash tier shared memory exceeds 227 KB");
  static_assert(G <= 32 || GPC == 1, "a group of more than 32 threads is the whole CTA");
  auto kern = k_hash_symbolic<G, CAP, LCAP, GPC, HB, HQ, DIRECT>;
  static LaunchSetup ls;
  int per_sm = 0;
  if (cudaError_t e = kernel_setup(ls, kern, G * GPC, smem, per_sm); e != cudaSuccess) return e;
  const int64_t want = (n + GPC - 1) / GPC;
  const int64_t cap = (int64_t)per_sm * num_sms();
  kern<<<(unsigned)(want < cap ? want : cap), G * GPC, smem, st>>>(A, B, rows, n, o);
  return cudaGetLastError();
}

template <bool VALS, int OUT>
static cudaError_t launch_tier_dispatch(int bin, const CsrView& A, const CsrView& B, int64_t b_cols, const int32_t* rows,
                                        int64_t n, const RowOut& o, cudaStream_t st) {
#ifndef BRM_SYM_MERGE_T56
#define BRM_SYM_MERGE_T56 1  // tiers 5-6 count by the column-only record merge (0: hashing; A/B switch)
#endif
  if constexpr (OUT == OUT_SYMBOLIC) {  // PRECISE step 3: hash counting on tiers 3-6
    switch (bin) {
      case 3: return launch_hash_t<BRM_HASH3>(A, B, rows, n, o, st);
      case 4: return launch_hash_t<BRM_HASH4>(A, B, rows, n, o, st);
      case 5:
        if (!BRM_SYM_MERGE_T56) return launch_hash_t<BRM_HASH5>(A, B, rows, n, o, st);
        break;
      case 6:
        if (!BRM_SYM_MERGE_T56) return launch_hash_t<BRM_HASH6>(A, B, rows, n, o, st);
        break;
      default: break;
    }
  }
  switch (bin) {
    case 1: return launch_tiny<VALS, OUT>(A, B, rows, n, o, st);
    case 2: return launch_tier_t<BRM_TIER2, VALS, OUT>(A, B, b_cols, rows, n, o, st);
    case 3: return launch_tier_t<BRM_TIER3, VALS, OUT>(A, B, b_cols, rows, n, o, st);
    case 4: return launch_tier_t<BRM_TIER4, VALS, OUT>(A, B, b_cols, rows, n, o, st);
    case 5: return launch_tier_t<BRM_TIER5, VALS, OUT>(A, B, b_cols, rows, n, o, st);
    case 6: return launch_tier_t<BRM_TIER6, VALS, OUT>(A, B, b_cols, rows, n, o, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_tier(int bin, int out_kind, const CsrView& A, const CsrView& B, int64_t b_cols, const int32_t* rows,
                        int64_t n, const RowOut& o, cudaStream_t st) {
  switch (out_kind) {
    case OUT_SYMBOLIC: return launch_tier_dispatch<false, OUT_SYMBOLIC>(bin, A, B, b_cols, rows, n, o, st);
    case OUT_CBAR: return launch_tier_dispatch<true, OUT_CBAR>(bin, A, B, b_cols, rows, n, o, st);
    case OUT_C: return launch_tier_dispatch<true, OUT_C>(bin, A, B, b_cols, rows, n, o, st);
    default: return cudaErrorInvalidValue;
  }
}

int64_t global_row_bytes(int64_t nprod, int64_t nl, bool vals) {
  auto a = [](int64_t b) { return (b + 15) & ~15ll; };
  int64_t s = a((nprod + nl + 2) * 4) * 2 + a((nl + 2) * 4) * 2 + a(nl * 8);
  if (vals) s += a((nprod + nl + 2) * 8) * 2 + a(nl * 8);
  return s;
}

cudaError_t launch_global_tier(int out_kind, const CsrView& A, const CsrView& B, const int32_t* rows, int64_t n,
                               const int64_t* ws_off, unsigned char* ws, const RowOut& o, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  switch (out_kind) {
    case OUT_SYMBOLIC: k_global_tier<false, OUT_SYMBOLIC><<<(unsigned)n, kGlobalG, 0, st>>>(A, B, rows, ws_off, ws, o); break;
    case OUT_CBAR: k_global_tier<true, OUT_CBAR><<<(unsigned)n, kGlobalG, 0, st>>>(A, B, rows, ws_off, ws, o); break;
    case OUT_C: k_global_tier<true, OUT_C><<<(unsigned)n, kGlobalG, 0, st>>>(A, B, rows, ws_off, ws, o); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_compact(int64_t M, int64_t nnz, const int64_t* nprod_off, const int64_t* crpt, const int32_t* cbar_col,
                           const double* cbar_val, int32_t* ccol, double* cval, const Mirrors& mir, cudaStream_t st) {
  if (M <= 0 || nnz <= 0) return cudaSuccess;
  int64_t blocks = (nnz + 8 * kCompactChunk - 1) / (8 * kCompactChunk);  // one chunk per warp
  const int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  k_compact<<<(unsigned)blocks, 256, 0, st>>>(M, nprod_off, crpt, cbar_col, cbar_val, ccol, cval, mir);
  return cudaGetLastError();
}

cudaError_t launch_partition(const int64_t* nprod_off, int64_t M, int p, int64_t* bounds, cudaStream_t st) {
  k_partition<<<(p + 1 + 127) / 128, 128, 0, st>>>(nprod_off, M, p, bounds);
  return cudaGetLastError();
}

cudaError_t launch_row_nprod(const CsrView& A, const int64_t* brpt, int64_t M, int64_t* nprod, const int64_t* long_np,
                             cudaStream_t st) {
  if (M > 0) k_row_nprod<<<(unsigned)((M + 255) / 256), 256, 0, st>>>(A, brpt, M, nprod, long_np);
  return cudaGetLastError();
}

// Device -> pinned host copy by the SMs (stores through the host mapping of
// the pinned buffer) instead of a copy engine: a bulk copy on a copy engine
// queues the library's small readbacks (row-size summaries, heavy-row info)
// behind it. W-byte words, coalesced, grid-stride.
template <class W>
__global__ void __launch_bounds__(256) k_copy_to_host(W* __restrict__ dst, const W* __restrict__ src, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  constexpr int U = 4;  // loads in flight per thread
  for (; i + (U - 1) * stride < n; i += U * stride) {
    W v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(dst + i + u * stride, v[u]);
  }
  for (; i < n; i += stride) __stcs(dst + i, __ldcs(src + i));
}

cudaError_t launch_copy_to_host(void* dst, const void* src, int64_t bytes, int ctas, cudaStream_t st) {
  if (bytes <= 0) return cudaSuccess;
  const uintptr_t a = reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | (uintptr_t)bytes;
  if ((a & 15) == 0)
    k_copy_to_host<int4><<<ctas, 256, 0, st>>>(static_cast<int4*>(dst), static_cast<const int4*>(src), bytes / 16);
  else if ((a & 7) == 0)
    k_copy_to_host<long long><<<ctas, 256, 0, st>>>(static_cast<long long*>(dst), static_cast<const long long*>(src),
                                                   bytes / 8);
  else if ((a & 3) == 0)
    k_copy_to_host<int><<<ctas, 256, 0, st>>>(static_cast<int*>(dst), static_cast<const int*>(src), bytes / 4);
  else
    k_copy_to_host<char><<<ctas, 256, 0, st>>>(static_cast<char*>(dst), static_cast<const char*>(src), bytes);
  return cudaGetLastError();
}

}  // namespace brm
