// heavy.cu -- kernels of the windowed heavy-row path (heavy.cuh).
#include <climits>

#include "heavy.cuh"
#include "kernels.cuh"

namespace brm {

namespace {

// first index i in [0, n) with p[i] >= key (n if none); p is read-only here
__device__ __forceinline__ int lower_bound_g(const int32_t* p, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(p + mid) < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// Largest i in [lo, hi] with pred(i), pred monotone (true ... true false ...)
// and pred(lo) true; evaluated by one warp, 32 probes per step.
template <class Pred>
__device__ __forceinline__ int warp_last_true(int lo, int hi, Pred pred) {
  const int lane = threadIdx.x & 31;
  while (lo < hi) {
    const int step = (hi - lo + 31) / 32;
    const int i = lo + (lane + 1) * step;
    const bool p = i <= hi && pred(i);
    const int k = __popc(__ballot_sync(0xffffffffu, p));  // probes 1..k hold
    const int nlo = lo + k * step;
    hi = min(hi, nlo + step - 1);
    lo = nlo;
  }
  return lo;
}

// List j of virtual row r: its start in the column source and its length.
struct ListRef {
  int64_t start;
  int len;
};
__device__ __forceinline__ ListRef hv_list(const HvArgs& a, const HvRow& r, int64_t a0, int64_t j) {
  if (r.src == 0) {
    const int k = __ldg(a.A.col + a0 + r.first + j);
    const int64_t s = __ldg(a.B.rpt + k);
    return {s, static_cast<int>(__ldg(a.B.rpt + k + 1) - s)};
  }
  const int64_t s = __ldg(a.lt + r.first + j);
  return {s, static_cast<int>(__ldg(a.lt + r.first + j + 1) - s)};
}

// block-wide exclusive scan of n <= kHvLists ints in place (512 threads, two
// entries each); returns the total. Ends synchronised.
__device__ int plan_scan(int* x, int n, int* wtmp) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int i0 = 2 * t, i1 = 2 * t + 1;
  const int v0 = i0 < n ? x[i0] : 0, v1 = i1 < n ? x[i1] : 0;
  int s = v0 + v1, inc = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += y;
  }
  if (lane == 31) wtmp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    constexpr int NW = kHvPlanG / 32;
    const int w = lane < NW ? wtmp[lane] : 0;
    int wx = w;
#pragma unroll
    for (int d = 1; d < NW; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wx, d);
      if (lane >= d) wx += y;
    }
    if (lane < NW) wtmp[lane] = wx - w;
    if (lane == NW - 1) wtmp[NW] = wx;
  }
  __syncthreads();
  const int ex = wtmp[wid] + inc - s;
  if (i0 < n) x[i0] = ex;
  if (i1 < n) x[i1] = ex + v0;
  const int total = wtmp[kHvPlanG / 32];
  if (t == 0) x[n] = total;
  __syncthreads();
  return total;
}

// The products [0, pc) of a chunk of lists (list j at lstart[j], products
// loff[j] .. loff[j+1]) visited by the CTA in items of <= 1024 consecutive
// products of ONE list (item offsets ioff, built here): a warp takes items
// round-robin, its lanes read consecutive columns (coalesced, four loads in
// flight per lane); no per-product list search. fn(col, list) on every lane
// (col < 0: none).
template <class Fn>
__device__ __forceinline__ void plan_for_products(const int32_t* scol, const int64_t* lstart, const int* loff, int nc,
                                                  int pc, int* ioff, int* wtmp, Fn fn) {
#ifndef BRM_PLAN_U
#define BRM_PLAN_U 16  // column loads in flight per lane in the plan's product pass (4 / 8 / 16: rmat20 one-level plan 47.6 / 45.7 / 45.5 ms)
#endif
  constexpr int NW = kHvPlanG / 32, U = BRM_PLAN_U, ITEM = 1024;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int j = threadIdx.x; j < nc; j += kHvPlanG) ioff[j] = (loff[j + 1] - loff[j] + ITEM - 1) / ITEM;
  __syncthreads();
  const int nitems = plan_scan(ioff, nc, wtmp);
  for (int it = wid; it < nitems; it += NW) {
    int lo = 0, hi = nc - 1;  // the list of item it: last j with ioff[j] <= it
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (ioff[mid] <= it)
        lo = mid;
      else
        hi = mid - 1;
    }
    const int l = lo;
    const int b0 = (it - ioff[l]) * ITEM;
    const int n = min(ITEM, loff[l + 1] - loff[l] - b0);
    const int32_t* base = scol + lstart[l] + b0;
    for (int i0 = 0; i0 < n; i0 += 32 * U) {
      int c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + 32 * u + lane;
        c[u] = i < n ? __ldg(base + i) : -1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) fn(c[u], l);
    }
  }
}

#ifndef BRM_PLAN_AGG
#define BRM_PLAN_AGG 0  // plan product pass: 0 an atomic per product (kept); 1 bitmap words OR-ed per warp run; 2 also bin counts per run
// (measured on B200, rmat20 PRECISE one-level plan: 45.5 / 91.1 / 101.0 ms for 0 / 1 / 2 -- the shuffles cost more than the serialised atomics)
#endif
// The plan's product pass hands a warp 32 consecutive entries of ONE sorted
// list (plan_for_products; lanes past the list's end invalid, at the tail),
// so lanes on one bitmap word / histogram bin form contiguous runs. A run's
// bits are OR-ed by a segmented shuffle reduction and its first lane sets
// them with one atomicOr; likewise one atomicAdd of the run's length per bin
// (same-word atomics from several lanes serialise: rmat20's bitmap atomicOr
// cost 8.5 shared wavefronts per warp instruction). Called by all 32 lanes.
template <bool HIST>
__device__ __forceinline__ void plan_mark_sorted(unsigned* bm, unsigned* hist, int rel, bool valid) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const unsigned upto = (2u << lane) - 1u;  // lanes <= this one (all of them for lane 31)
  {
    const int w = valid ? rel >> 5 : -1;
    const int wp = __shfl_up_sync(FULL, w, 1);
    const bool head = lane == 0 || w != wp;
    const unsigned above = __ballot_sync(FULL, head) & ~upto;
    const int next = above ? __ffs(above) - 1 : 32;  // end of this lane's run
    unsigned x = valid ? 1u << (rel & 31) : 0u;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned y = __shfl_down_sync(FULL, x, d);
      if (lane + d < next) x |= y;
    }
    if (head && valid) atomicOr(&bm[w], x);
  }
  if constexpr (HIST) {
    if constexpr (BRM_PLAN_AGG >= 2) {
      const int b = valid ? rel >> kHvBinBits : -1;
      const int bp = __shfl_up_sync(FULL, b, 1);
      const bool head = lane == 0 || b != bp;
      const unsigned above = __ballot_sync(FULL, head) & ~upto;
      const int next = above ? __ffs(above) - 1 : 32;
      if (head && valid) atomicAdd(&hist[b], static_cast<unsigned>(next - lane));
    } else if (valid) {
      atomicAdd(&hist[rel >> kHvBinBits], 1u);
    }
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// Plan of one virtual row per CTA (see heavy.cuh). Columns are processed in
// ranges of 2^20 (one range when B.cols <= 2^20); per range:
//   1. bitmap of the product columns (atomicOr) and histogram of products per
//      128-column bin (atomicAdd), one pass over the products;
//   2. inclusive prefix of the histogram;
//   3. windows, greedily: from x0, the largest cut x with
//      count(x) <= count(x0) + kHvCap, at a bin boundary, or inside a bin of
//      more than kHvCap products whose per-column counts were refined by an
//      extra pass (64 such bins at a time); warp 0, 32 probes per step;
//   4. each window's output size = bits set in [x0, x) (warp 0).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kHvPlanG, 1) k_hv_plan(HvArgs a, int count_only) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned* bm = reinterpret_cast<unsigned*>(smem);
  unsigned* hist = bm + kHvRange / 32;
  unsigned* fine = hist + kHvBins;
  unsigned char* slot = reinterpret_cast<unsigned char*>(fine + kHvFine * 128);
  int64_t* lstart = reinterpret_cast<int64_t*>(slot + kHvBins);
  int* ioff = reinterpret_cast<int*>(lstart + kHvLists);  // items of each list (plan_for_products)
  int* loff = ioff + kHvLists + 4;
  unsigned* gp = reinterpret_cast<unsigned*>(loff + kHvLists + 4);  // gp[g] = bits set in groups < g
  __shared__ int s_wtmp[kHvPlanG / 32 + 1];
  __shared__ unsigned long long s_cnt;
  __shared__ int s_cmin, s_cmax;
  __shared__ int s_x0, s_nw, s_need, s_done, s_running;
  __shared__ int s_nwr;  // windows of the ranges done
  __shared__ int s_refined_lo, s_refined_hi;  // bins [lo, hi] may hold refined slots

  const HvRow r = a.rows[blockIdx.x];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int64_t a0 = r.src == 0 ? a.A.rpt[r.row] : 0;
  const int32_t* scol = r.src == 0 ? a.B.col : a.ws_col;
  const int nl = r.nl;
  // column span of the virtual row: first / last column of every list
  if (t == 0) {
    s_cmin = INT_MAX;
    s_cmax = -1;
    s_cnt = 0;
    s_nw = 0;
    s_nwr = 0;
    s_running = 0;
  }
  __syncthreads();
  {
    int cmin = INT_MAX, cmax = -1;
    for (int j = t; j < nl; j += kHvPlanG) {
      const ListRef L = hv_list(a, r, a0, j);
      if (L.len > 0) {
        cmin = min(cmin, __ldg(scol + L.start));
        cmax = max(cmax, __ldg(scol + L.start + L.len - 1));
      }
    }
    cmin = __reduce_min_sync(0xffffffffu, cmin);
    cmax = __reduce_max_sync(0xffffffffu, cmax);
    if (lane == 0) {
      atomicMin(&s_cmin, cmin);
      atomicMax(&s_cmax, cmax);
    }
  }
  __syncthreads();
  const int cmin = s_cmin, cmax = s_cmax;
  if (cmax < 0) {  // no products at all (a block of empty lists)
    if (t == 0) {
      if (!count_only) {
        a.nwin[blockIdx.x] = 0;
        a.wout[r.plan] = 0;
        a.cuts[r.plan] = 0;
      }
      a.total[blockIdx.x] = 0;
      if (r.out == 0 && a.row_size) a.row_size[r.row] = 0;
    }
    return;
  }
  const bool multi = (cmin >> kHvRangeBits) != (cmax >> kHvRangeBits);
  const int nchunks = (nl + kHvLists - 1) / kHvLists;  // plan rows: nl <= kHvLists, one chunk
  for (int rg = cmin >> kHvRangeBits; rg <= (cmax >> kHvRangeBits); ++rg) {
    const int64_t rs0 = static_cast<int64_t>(rg) << kHvRangeBits;
    const int rlen = static_cast<int>(min(static_cast<int64_t>(kHvRange), a.ncols - rs0));
    const int lo_c = static_cast<int>(max(static_cast<int64_t>(cmin), rs0) - rs0);             // relative
    const int hi_c = static_cast<int>(min(static_cast<int64_t>(cmax) + 1, rs0 + rlen) - rs0);  // relative, exclusive
    // the whole range's bitmap (windows reach bin boundaries outside [lo_c, hi_c))
    for (int w = t; w < (((rlen + 31) >> 5) + 3) >> 2; w += kHvPlanG) reinterpret_cast<uint4*>(bm)[w] = make_uint4(0, 0, 0, 0);
    if (!count_only) {
      for (int b = t; b < kHvBins / 4; b += kHvPlanG) reinterpret_cast<uint4*>(hist)[b] = make_uint4(0, 0, 0, 0);
      for (int b = t; b < kHvBins / 16; b += kHvPlanG)
        reinterpret_cast<uint4*>(slot)[b] = make_uint4(~0u, ~0u, ~0u, ~0u);
    }
    __syncthreads();
    int prange = 0;
    for (int ch = 0; ch < nchunks; ++ch) {
      const int j0 = ch * kHvLists, nc = min(kHvLists, nl - j0);
      for (int j = t; j < nc; j += kHvPlanG) {
        const ListRef L = hv_list(a, r, a0, j0 + j);
        int lo = 0, hi = L.len;
        if (multi) {
          lo = lower_bound_g(scol + L.start, L.len, static_cast<int>(rs0));
          hi = rs0 + kHvRange >= a.ncols ? L.len
                                         : lower_bound_g(scol + L.start, L.len, static_cast<int>(rs0 + kHvRange));
        }
        lstart[j] = L.start + lo;
        loff[j] = hi - lo;
      }
      __syncthreads();
      const int pc = plan_scan(loff, nc, s_wtmp);
      // one pass over the chunk's products
      const int irs0 = static_cast<int>(rs0);
      if (count_only) {
        plan_for_products(scol, lstart, loff, nc, pc, ioff, s_wtmp, [&](int c, int) {
          if constexpr (BRM_PLAN_AGG >= 1) {
            plan_mark_sorted<false>(bm, hist, c - irs0, c >= 0);
          } else if (c >= 0) {
            const int rel = c - irs0;
            atomicOr(&bm[rel >> 5], 1u << (rel & 31));
          }
        });
      } else {
        plan_for_products(scol, lstart, loff, nc, pc, ioff, s_wtmp, [&](int c, int) {
          if constexpr (BRM_PLAN_AGG >= 1) {
            plan_mark_sorted<true>(bm, hist, c - irs0, c >= 0);
          } else if (c >= 0) {
            const int rel = c - irs0;
            atomicOr(&bm[rel >> 5], 1u << (rel & 31));
            atomicAdd(&hist[rel >> kHvBinBits], 1u);
          }
        });
      }
      __syncthreads();
      prange += pc;
    }
    if (count_only) {
      unsigned long long c = 0;
      for (int w = (lo_c >> 5) + t; w <= ((hi_c - 1) >> 5); w += kHvPlanG) c += __popc(bm[w]);
      c = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(c));
      if (lane == 0 && c) atomicAdd(&s_cnt, c);
      __syncthreads();
      continue;
    }
    if (prange == 0) continue;
    // inclusive prefix of the histogram: warp w owns bins [w * 512, w * 512 +
    // 512); its lanes read consecutive bins (a thread reading 16 consecutive
    // bins would put lanes t and t + 2 on one bank)
    {
      constexpr int SPAN = kHvBins / (kHvPlanG / 32), ITER = SPAN / 32;
      unsigned v[ITER];
      unsigned carry = 0;
#pragma unroll
      for (int i = 0; i < ITER; ++i) {
        unsigned x = hist[wid * SPAN + i * 32 + lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, x, d);
          if (lane >= d) x += y;
        }
        v[i] = x + carry;
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) s_wtmp[wid] = static_cast<int>(carry);
      __syncthreads();
      unsigned pre = 0;
      for (int w = 0; w < wid; ++w) pre += static_cast<unsigned>(s_wtmp[w]);
#pragma unroll
      for (int i = 0; i < ITER; ++i) hist[wid * SPAN + i * 32 + lane] = v[i] + pre;  // hist is now the inclusive prefix H
      __syncthreads();
    }
    const unsigned* H = hist;
    auto bin_count = [&](int b) { return H[b] - (b > 0 ? H[b - 1] : 0u); };
    // greedy windows, with refinement passes as the walk meets bins of more
    // than kHvCap products
    if (t == 0) {
      s_x0 = lo_c & ~((1 << kHvBinBits) - 1);  // a bin boundary: count 0
      if (rg != (cmin >> kHvRangeBits)) s_x0 = 0;
      s_need = -1;
      s_done = 0;
      s_refined_lo = 1;
      s_refined_hi = 0;
    }
    __syncthreads();
    const int nb = (rlen + (1 << kHvBinBits) - 1) >> kHvBinBits;
    const int nwords = (rlen + 31) >> 5, ngroups = (nwords + 31) >> 5;
    bool gp_done = false;
    while (true) {
      if (s_need >= 0) {
        // refine the next kHvFine overflow bins from s_need on (whole CTA)
        const int from = s_need;
        if (wid == 0) {
          for (int b = s_refined_lo + lane; b <= s_refined_hi; b += 32) slot[b] = 0xff;
          __syncwarp();
          int nsl = 0, last = from;
          for (int b0 = from; b0 < nb && nsl < kHvFine; b0 += 32) {
            const int b = b0 + lane;
            const bool ov = b < nb && bin_count(b) > static_cast<unsigned>(kHvCap);
            const unsigned m = __ballot_sync(0xffffffffu, ov);
            const int rank = nsl + __popc(m & ((1u << lane) - 1u));
            if (ov && rank < kHvFine) {
              slot[b] = static_cast<unsigned char>(rank);
              last = b;
            }
            nsl += __popc(m);
            last = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(last));
          }
          if (lane == 0) {
            s_refined_lo = from;
            s_refined_hi = last;
          }
        }
        for (int i = t; i < kHvFine * 128; i += kHvPlanG) fine[i] = 0u;
        __syncthreads();
        const int irs0 = static_cast<int>(rs0);
        plan_for_products(scol, lstart, loff, nl, loff[nl], ioff, s_wtmp, [&](int c, int) {  // plan rows: one chunk of lists
          if (c >= 0) {
            const int rel = c - irs0;
            const int sl = slot[rel >> kHvBinBits];
            if (sl != 0xff) atomicAdd(&fine[sl * 128 + (rel & 127)], 1u);
          }
        });
        __syncthreads();
        // inclusive prefix per refined bin (a warp per bin)
        for (int sl = wid; sl < kHvFine; sl += kHvPlanG / 32) {
          unsigned* f = fine + sl * 128;
          unsigned carry = 0;
          for (int i0 = 0; i0 < 128; i0 += 32) {
            unsigned x = f[i0 + lane];
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
              const unsigned y = __shfl_up_sync(0xffffffffu, x, d);
              if (lane >= d) x += y;
            }
            f[i0 + lane] = x + carry;
            carry += __shfl_sync(0xffffffffu, x, 31);
          }
        }
        if (t == 0) s_need = -1;
        __syncthreads();
      }
      if (wid == 0) {
        int x0 = s_x0;
        int nw = s_nw;
        int need = -1;
        // count(x): products of this range with relative column < x (x a bin
        // boundary, or inside a refined bin)
        auto count_at = [&](int x) -> unsigned {
          const int b = x >> kHvBinBits, w = x & 127;
          const unsigned base = b > 0 ? H[b - 1] : 0u;
          if (w == 0) return base;
          return base + fine[slot[b] * 128 + w - 1];
        };
        const unsigned ptot = H[nb - 1];
        while (x0 < rlen && count_at(x0) < ptot) {
          const unsigned T = count_at(x0) + kHvCap;
          const int b0 = x0 >> kHvBinBits;
          int cut;
          if (H[b0] <= T) {  // the next bin boundary fits: the last one that does
            const int B = warp_last_true(b0 + 1, nb, [&](int i) { return H[i - 1] <= T; });
            cut = B << kHvBinBits;
            if (B < nb && bin_count(B) > static_cast<unsigned>(kHvCap)) {  // continue inside bin B
              if (slot[B] == 0xff) {
                need = B;
                break;
              }
              const int w = warp_last_true(0, 127, [&](int i) { return i == 0 || count_at(cut + i) <= T; });
              cut += w;
            }
          } else {  // bin b0 alone holds too much: cut inside it (refined)
            if (slot[b0] == 0xff) {
              need = b0;
              break;
            }
            const int w0 = x0 & 127;
            const int w = warp_last_true(w0, 127, [&](int i) { return i == w0 || count_at((b0 << kHvBinBits) + i) <= T; });
            cut = (b0 << kHvBinBits) + w;  // > x0: one column holds <= nl <= kHvCap products
          }
          if (cut - x0 > kHvSpan) cut = (x0 + kHvSpan) & ~((1 << kHvBinBits) - 1);
          cut = min(cut, rlen);
          if (nw >= r.maxwin) {
            if (lane == 0) atomicOr(a.err, 1u);
            need = -2;
            break;
          }
          if (lane == 0) a.cuts[r.plan + nw] = static_cast<int>(rs0 + x0);
          ++nw;
          x0 = cut;
        }
        if (lane == 0) {
          s_x0 = x0;
          s_nw = nw;
          // a window start inside a refined bin keeps that bin refined: the
          // next group of refined bins starts at x0's bin
          if (need >= 0) s_need = (x0 & 127) ? min(need, x0 >> kHvBinBits) : need; else s_done = 1;
          if (need == -2) s_done = 2;
          if (need == -1 && ptot > 0) s_cnt = static_cast<unsigned long long>(rs0 + x0);  // end of the last window
        }
      } else if (!gp_done) {
        // while warp 0 cuts the windows, the other warps count the bits of
        // every group of 32 bitmap words (16-byte loads: 8 lanes per group)
        // and warp 1 turns the counts into the exclusive prefix gp
        gp_done = true;
        constexpr int NWK = kHvPlanG / 32 - 1;
        const int sub = lane >> 3, part = lane & 7;
        for (int g0 = 4 * (wid - 1); g0 < ngroups; g0 += 4 * NWK) {
          const int g = g0 + sub;
          const int w = 32 * g + 4 * part;
          unsigned c = 0;
          if (g < ngroups && w < nwords) {
            const uint4 x = *reinterpret_cast<const uint4*>(bm + w);  // (words past nwords are cleared)
            c = __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
          }
          c += __shfl_xor_sync(0xffffffffu, c, 4);
          c += __shfl_xor_sync(0xffffffffu, c, 2);
          c += __shfl_xor_sync(0xffffffffu, c, 1);
          if (part == 0 && g < ngroups) gp[g + 1] = c;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kHvPlanG - 32) : "memory");  // warps 1.. only
        if (wid == 1) {
          unsigned carry = 0;
          if (lane == 0) gp[0] = 0;
          for (int g0 = 1; g0 <= ngroups; g0 += 32) {
            unsigned x = g0 + lane <= ngroups ? gp[g0 + lane] : 0u;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
              const unsigned y = __shfl_up_sync(0xffffffffu, x, d);
              if (lane >= d) x += y;
            }
            if (g0 + lane <= ngroups) gp[g0 + lane] = x + carry;
            carry += __shfl_sync(0xffffffffu, x, 31);
          }
        }
      }
      __syncthreads();
      if (s_done) break;
    }
    if (s_done == 2) break;
    // output size of each window of this range = bits set in it: the group
    // prefix gp (made above, beside the window cutting), then two partial
    // prefixes per window (a warp per window)
    {
      auto bits_below = [&](int x) -> unsigned {  // bits set in [0, x), by one warp
        unsigned c = 0;
        const int w = x >> 5, g = w >> 5;
        const int wi = 32 * g + lane;
        if (wi < w) c = __popc(bm[wi]);
        else if (wi == w && (x & 31)) c = __popc(bm[wi] & ((1u << (x & 31)) - 1u));
        return gp[g] + __reduce_add_sync(0xffffffffu, c);
      };
      const int nw1 = s_nw, nw0 = s_nwr;
      for (int w = nw0 + wid; w < nw1; w += kHvPlanG / 32) {
        const int x0 = a.cuts[r.plan + w] - static_cast<int>(rs0);
        const int x1 = w + 1 < nw1 ? a.cuts[r.plan + w + 1] - static_cast<int>(rs0) : rlen;
        const unsigned c = bits_below(x1) - bits_below(x0);
        if (lane == 0) a.wout[r.plan + w] = static_cast<int>(c);  // a count for now
      }
      __syncthreads();
      if (wid == 0) {  // counts -> output offsets (exclusive, continuing over ranges)
        int carry = s_running;
        for (int w0 = nw0; w0 < nw1; w0 += 32) {
          const int w = w0 + lane;
          const int c = w < nw1 ? a.wout[r.plan + w] : 0;
          int x = c;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
          }
          if (w < nw1) a.wout[r.plan + w] = carry + x - c;
          carry += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) {
          s_running = carry;
          s_nwr = nw1;
        }
      }
      __syncthreads();
    }
  }
  __syncthreads();
  if (t == 0) {
    if (count_only) {
      a.total[blockIdx.x] = static_cast<int64_t>(s_cnt);
      if (r.out == 0 && a.row_size) a.row_size[r.row] = static_cast<int64_t>(s_cnt);
    } else {
      const int nw = s_nw;
      a.cuts[r.plan + nw] = static_cast<int>(s_cnt);
      a.wout[r.plan + nw] = s_running;
      a.nwin[blockIdx.x] = nw;
      a.total[blockIdx.x] = s_running;
      if (r.out == 0 && a.row_size) a.row_size[r.row] = s_running;
    }
  }
}

// ---------------------------------------------------------------------------
// Merge: one CTA per task = windows [w0, w1) of one virtual row.
//
// The window's rounds of Algorithm 1 run on 32-bit keys
//   key = (pair index q) << 20 | (col - c0)
// with the values moving alongside: list m of the current round belongs to
// pair q = m >> 1 (lines 22-29: lists (2q, 2q+1) are consumed together; an
// odd trailing list has an empty partner). The even lists are stored
// concatenated as sequence A, the odd lists as sequence B; both are sorted by
// (q, col), so a whole round is ONE merge of A with B: equal keys are the
// duplicate columns of pair q and combine as left + right (A holds the left
// list). An output of pair q is an element of list q of the next round: it
// goes to A' if q is even, to B' if odd, with key q >> 1.
// ---------------------------------------------------------------------------
namespace {

// 32-bit keys (q << kColBits | col - c0), values moving with them
constexpr int kColBits = 20;
constexpr unsigned kColMask = (1u << kColBits) - 1u;
constexpr unsigned kKey32Sent = 0xffffffffu;
static_assert(kHvLists / 2 <= (1 << (32 - kColBits)) - 2, "pair indices fit the key's high bits");

__device__ __forceinline__ int key32_merge_path(const unsigned* A, int na, const unsigned* B, int nb, int diag) {
  int lo = diag - nb > 0 ? diag - nb : 0;
  int hi = diag < na ? diag : na;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (A[mid] <= B[diag - 1 - mid])
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// inclusive max-scan of u16 owner marks over [0, n) by the CTA (n <= kHvCap)
__device__ __forceinline__ void owner_max_scan(unsigned short* m, int n, int* wtmp) {
  constexpr int PER = (kHvCap + kHvG - 1) / kHvG;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int b0 = t * PER;
  unsigned short v[PER];
  unsigned run = 0;
  if constexpr (PER % 8 == 0) {  // 16-byte loads: a thread's 2*PER bytes (u16 loads at a 2*PER-byte stride conflict)
#pragma unroll
    for (int i = 0; i < PER; i += 8) {
      const uint4 x = *reinterpret_cast<const uint4*>(m + b0 + i);
      const unsigned w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        v[i + 2 * h] = static_cast<unsigned short>(w4[h] & 0xffffu);
        v[i + 2 * h + 1] = static_cast<unsigned short>(w4[h] >> 16);
      }
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) run = max(run, static_cast<unsigned>(v[i]));
  } else {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      v[i] = b0 + i < n ? m[b0 + i] : 0;
      run = max(run, static_cast<unsigned>(v[i]));
    }
  }
  unsigned inc = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc = max(inc, y);
  }
  if (lane == 31) wtmp[wid] = static_cast<int>(inc);
  __syncthreads();
  unsigned pre = 0;
  for (int w = 0; w < wid; ++w) pre = max(pre, static_cast<unsigned>(wtmp[w]));
  unsigned ex = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) ex = 0;
  run = max(pre, ex);
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    run = max(run, static_cast<unsigned>(v[i]));
    v[i] = static_cast<unsigned short>(run);
  }
  if constexpr (PER % 8 == 0) {  // (positions >= n get values too: the marks are cleared per window)
#pragma unroll
    for (int i = 0; i < PER; i += 8) {
      uint4 x;
      x.x = v[i] | (static_cast<unsigned>(v[i + 1]) << 16);
      x.y = v[i + 2] | (static_cast<unsigned>(v[i + 3]) << 16);
      x.z = v[i + 4] | (static_cast<unsigned>(v[i + 5]) << 16);
      x.w = v[i + 6] | (static_cast<unsigned>(v[i + 7]) << 16);
      *reinterpret_cast<uint4*>(m + b0 + i) = x;
    }
  } else {
#pragma unroll
    for (int i = 0; i < PER; ++i)
      if (b0 + i < n) m[b0 + i] = v[i];
  }
  __syncthreads();
}

}  // namespace

template <int OUT>
__global__ void __launch_bounds__(kHvG, kHvMinBlocks) k_hv_merge(HvArgs a, RowOut o) {
  constexpr int NVC = ((kHvCap + kHvG - 1) / kHvG) | 1;
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* p = smem;
  auto take = [&](int n) {
    unsigned char* q = p;
    p += align16(n);
    return q;
  };
  longlong2* lst = reinterpret_cast<longlong2*>(take(kHvLists * 16));  // {src of layout position 0, A value}
  int64_t* S = reinterpret_cast<int64_t*>(take(kHvLists * 8));
  int* L = reinterpret_cast<int*>(take(kHvLists * 4));
  int* cur = reinterpret_cast<int*>(take(kHvLists * 4));
  int* head = reinterpret_cast<int*>(take(kHvLists * 4));
  int* cnt = reinterpret_cast<int*>(take(kHvLists * 4));
  unsigned* rk = reinterpret_cast<unsigned*>(take((kHvCap + 2) * 4));  // keys (q, col - c0)
  double* rv = reinterpret_cast<double*>(take((kHvCap + 2) * 8));     // their values (move with them)
  unsigned short* own = reinterpret_cast<unsigned short*>(take(kHvCap * 2));
  int* wtmp = reinterpret_cast<int*>(take(64));
  __shared__ int s_na;
  const int rank = threadIdx.x;
  const int64_t t = blockIdx.x;
  // the grid covers the plan's upper bound of tasks; the task map holds the
  // virtual row of each of the planned windows' tasks
  if (t >= *a.ntask_total) return;
  const int v = a.tmap[t];
  const HvRow r = a.rows[v];
  const int nwin = a.nwin[v];
  const int w0 = static_cast<int>(t - r.task0) * r.wch;
  if (w0 >= nwin) return;
  const int w1 = min(nwin, w0 + r.wch);
  const int nl = r.nl;
  const int ne = (nl + 1) >> 1;  // even lists: layout ranks [0, ne), odd lists: [ne, nl)
  const int64_t a0 = r.src == 0 ? a.A.rpt[r.row] : 0;
  const int32_t* scol = r.src == 0 ? a.B.col : a.ws_col;
  const double* sval = r.src == 0 ? a.B.val : a.ws_val;
  const int cfirst = a.cuts[r.plan + w0];
  for (int l = rank; l < nl; l += kHvG) {
    const ListRef Lr = hv_list(a, r, a0, l);
    const int c0 = w0 == 0 ? 0 : lower_bound_g(scol + Lr.start, Lr.len, cfirst);
    S[l] = Lr.start;
    L[l] = Lr.len;
    lst[l].y = __double_as_longlong(r.src == 0 ? __ldg(a.A.val + a0 + r.first + l) : 1.0);
    cur[l] = c0;
    head[l] = c0 < Lr.len ? __ldg(scol + Lr.start + c0) : INT_MAX;
  }
  __syncthreads();
  int32_t* ocol;
  double* oval;
  int64_t obase;
  if (r.out == 0) {
    ocol = o.col;
    oval = o.val;
    obase = o.base[r.row];
  } else {
    ocol = a.wo_col;
    oval = a.wo_val;
    obase = r.obase;
  }
  for (int w = w0; w < w1; ++w) {
    const int c0 = a.cuts[r.plan + w], c1 = a.cuts[r.plan + w + 1];
    // (1) each list's share of [c0, c1): 8 probes past the cursor (one
    // latency), then a binary search only if the list goes on inside; the
    // first column >= c1 becomes the list's new head
    {
      // a thread's lists l = rank + j * kHvG: the probes of all of them are
      // issued before any is resolved (one memory latency for the batch)
      constexpr int LPT = (kHvLists + kHvG - 1) / kHvG;
      int pr[LPT][8];
#pragma unroll
      for (int j = 0; j < LPT; ++j) {
        const int l = rank + j * kHvG;
        const bool live = l < nl && head[l] < c1;
        const int cu = live ? cur[l] : 0;
        const int rem = live ? L[l] - cu : 0;
        const int32_t* q = scol + (live ? S[l] + cu : 0);
#pragma unroll
        for (int k = 0; k < 8; ++k) pr[j][k] = k + 1 < rem ? __ldg(q + k + 1) : INT_MAX;
      }
#pragma unroll
      for (int j = 0; j < LPT; ++j) {
        const int l = rank + j * kHvG;
        if (l >= nl) break;
        int n = 0;
        if (head[l] < c1) {
          const int cu = cur[l];
          const int rem = L[l] - cu;  // >= 1
          n = 1;
          int nh = INT_MAX;
          bool more = true;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (more) {
              if (pr[j][k] < c1) {
                ++n;
              } else {
                nh = pr[j][k];
                more = false;
              }
            }
          }
          if (more && n < rem) {  // all 8 probes inside the window: 16-ary search on
            const int32_t* q = scol + S[l] + cu;
            int lo = n, hi = min(rem, kHvCap + 1);  // first index >= c1 lies in [lo, hi]
            while (hi - lo > 16) {
              const int st = (hi - lo + 15) / 16;
              int k = 0;
              int pv[16];
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                const int ix = lo + (u + 1) * st - 1;
                pv[u] = ix < hi ? __ldg(q + ix) : INT_MAX;
              }
#pragma unroll
              for (int u = 0; u < 16; ++u) k += pv[u] < c1;
              const int nlo = lo + k * st;
              hi = min(hi, nlo + st - 1);
              lo = nlo;
            }
            n = lo + lower_bound_g(q + lo, hi - lo, c1);
            nh = n < rem ? __ldg(q + n) : INT_MAX;
          }
          head[l] = nh;
        }
        cnt[l] = n;
      }
    }
    __syncthreads();
    // (2) layout: even lists (A) then odd lists (B), in list order; owner
    // marks at each non-empty list's first position
    for (int i = rank; i < kHvCap / 8; i += kHvG) reinterpret_cast<uint4*>(own)[i] = make_uint4(0, 0, 0, 0);
    int P = 0;
    for (int vb = 0; vb < nl; vb += kHvG) {
      const int vr = vb + rank;
      const int m = vr < ne ? 2 * vr : 2 * (vr - ne) + 1;
      const int n = vr < nl ? cnt[m] : 0;
      int tot;
      const int ex = group_excl_scan<kHvG>(Group<kHvG>{rank, 0xffffffffu, 0}, n, tot, wtmp);
      if (vr < nl) {
        const int pos = P + ex;
        lst[m].x = S[m] + cur[m] - pos;
        if (n) own[pos] = static_cast<unsigned short>(vr);
        if (vr == ne - 1) s_na = pos + n;  // nA: the even lists' products
      }
      P += tot;
    }
    __syncthreads();
    const int nA0 = s_na;
    owner_max_scan(own, P, wtmp);
    // (3) gather: product at layout position e, record key (m >> 1, col - c0, slot e)
    // A occupies rk/rv[0, nA), a sentinel at nA, B at [nA + 1, P + 1), a sentinel at P + 1
#ifndef BRM_HV_CPASYNC
#define BRM_HV_CPASYNC 0  // 1: the gather by cp.async straight into the key/value arrays (A/B switch)
#endif
#if BRM_HV_CPASYNC
    {
      // every product's column and value copied by cp.async (4 + 8 bytes) to
      // its layout position, all in flight at once; then keys and products
      // formed in place
      for (int e = rank; e < P; e += kHvG) {
        const int vr = own[e];
        const int m = vr < ne ? 2 * vr : 2 * (vr - ne) + 1;
        const int64_t src = lst[m].x + e;
        const int pos = e + (e >= nA0 ? 1 : 0);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(rk + pos)), "l"(scol + src) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(rv + pos)), "l"(sval + src) : "memory");
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      for (int e = rank; e < P; e += kHvG) {  // (each thread converts the entries it copied)
        const int vr = own[e];
        const int m = vr < ne ? 2 * vr : 2 * (vr - ne) + 1;
        const int pos = e + (e >= nA0 ? 1 : 0);
        rv[pos] = __dmul_rn(__longlong_as_double(lst[m].y), rv[pos]);  // line 12: the product, rounded once
        rk[pos] = (static_cast<unsigned>(m >> 1) << kColBits) | (rk[pos] - static_cast<unsigned>(c0));
      }
    }
#else
    {
      // a batch of a thread's loads is issued before its products are formed
      constexpr int PPT = ((kHvCap + kHvG - 1) / kHvG + 1) / 2;
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
      int cg[PPT], mq[PPT];
      double bv[PPT], av[PPT];
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        const int e = rank + (k + half * PPT) * kHvG;
        cg[k] = 0;
        bv[k] = 0.0;
        av[k] = 0.0;
        mq[k] = 0;
        if (e < P) {
          const int vr = own[e];
          const int m = vr < ne ? 2 * vr : 2 * (vr - ne) + 1;
          const longlong2 d = lst[m];
          const int64_t src = d.x + e;
          cg[k] = __ldg(scol + src);
          bv[k] = __ldg(sval + src);
          av[k] = __longlong_as_double(d.y);
          mq[k] = m >> 1;
        }
      }
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        const int e = rank + (k + half * PPT) * kHvG;
        if (e < P) {
          const int pos = e + (e >= nA0 ? 1 : 0);
          const unsigned key = (static_cast<unsigned>(mq[k]) << kColBits) | static_cast<unsigned>(cg[k] - c0);
          rv[pos] = __dmul_rn(av[k], bv[k]);  // line 12: the product, rounded once
          rk[pos] = key;
        }
      }
      }
    }
#endif
    if (rank == 0) {
      rk[nA0] = kKey32Sent;
      rk[P + 1] = kKey32Sent;
    }
    __syncthreads();
    // (4) accumulating phase: ceil(log2 nl) rounds (lines 21-35)
    int nA = nA0, nB = P - nA0, lists = nl;
    while (lists > 1) {
      const unsigned* A = rk;
      const unsigned* B = rk + nA + 1;
      const int n = nA + nB;
      const int VT = min(((n + kHvG - 1) / kHvG) | 1, NVC);  // odd: strided accesses spread over the banks
      const int g0 = min(rank * VT, n), g1 = min(g0 + VT, n);
      int cntv = 0, cntE = 0;
      const int i = key32_merge_path(A, nA, B, nB, g0);
      int j = g0 - i;
      if (i > 0 && j < nB && A[i - 1] == B[j]) ++j;  // B[j] was combined on the left
      int ia = i;
      int ib = nA + 1 + j;  // ib indexes rk directly
      const int lim = g0 < g1 ? g1 + nA + 1 : 0;  // ia + ib < lim <=> positions consumed < g1
      unsigned ra = A[ia], rb = rk[ib];
      unsigned ok[NVC];
      double ov[NVC];
      double va = rv[ia], vb = rv[ib];
      const unsigned kb = smem_u32(rk), vbase = smem_u32(rv);
#pragma unroll
      for (int k = 0; k < NVC; ++k) {
        if (k >= VT) break;
        const bool act = ia + ib < lim;
        const bool ta = act && ra <= rb;
        const bool tb = act && rb <= ra;
        ok[k] = ta ? ra : rb;
        // equal keys: a duplicate column of pair q, left + right (Fig. 2)
        ov[k] = ta ? (tb ? __dadd_rn(va, vb) : va) : vb;
        cntv += act;
        cntE += act && !((ok[k] >> kColBits) & 1u);  // outputs of even pairs (-> A')
        ia += ta;
        ib += tb;
        lds_if(ta, kb + 4u * ia, ra);
        lds_if(ta, vbase + 8u * ia, va);
        lds_if(tb, kb + 4u * ib, rb);
        lds_if(tb, vbase + 8u * ib, vb);
      }
      // outputs of even pairs go to A', odd pairs to B' (one packed 16 | 16 scan)
      int tot;
      const int packed = group_excl_scan<kHvG>(Group<kHvG>{rank, 0xffffffffu, 0}, cntE | ((cntv - cntE) << 16), tot, wtmp);
      const int nA2 = tot & 0xffff, nB2 = tot >> 16;
      // every thread has read its inputs (group_excl_scan ends synchronised)
      int e_ = packed & 0xffff, o_ = nA2 + 1 + (packed >> 16);
#pragma unroll
      for (int k = 0; k < NVC; ++k) {
        if (k >= cntv) break;
        const unsigned key = ok[k];
        const unsigned q = key >> kColBits;
        const unsigned odd = q & 1u;
        const int dst = odd ? o_ : e_;
        o_ += odd;
        e_ += 1 - odd;
        const unsigned nkey = ((q >> 1) << kColBits) | (key & kColMask);
        rk[dst] = nkey;
        rv[dst] = ov[k];
      }
      if (rank == 0) {
        rk[nA2] = kKey32Sent;
        rk[nA2 + 1 + nB2] = kKey32Sent;
      }
      __syncthreads();
      nA = nA2;
      nB = nB2;
      lists = (lists + 1) >> 1;
    }
    // (5) line 36: the window's part of the row (list 0 = A)
    const int T = nA;
    const int ob = a.wout[r.plan + w];
    if (rank == 0 && T != a.wout[r.plan + w + 1] - ob) atomicOr(a.err, 2u);
    for (int e = rank; e < T; e += kHvG) {
      const int c = static_cast<int>(rk[e] & kColMask) + c0;
      const double v = rv[e];
      ocol[obase + ob + e] = c;
      oval[obase + ob + e] = v;
      if (OUT == OUT_C && r.out == 0) mirror_store<true>(o.mir, obase + ob + e, c, v);
    }
    for (int l = rank; l < nl; l += kHvG) cur[l] += cnt[l];
    __syncthreads();
  }
}

__global__ void k_hv_ntask(HvArgs a, int64_t* ntask) {
  const int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= a.nrows) return;
  const int wch = a.rows[v].wch;
  ntask[v] = (a.nwin[v] + wch - 1) / wch;
}

__global__ void k_hv_taskmap(HvArgs a, HvRow* rows, const int64_t* toff, int32_t* tmap) {
  const int64_t v = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= a.nrows) return;
  const int64_t t0 = toff[v], n = toff[v + 1] - t0;
  if (lane == 0) rows[v].task0 = t0;
  for (int64_t j = lane; j < n; j += 32) tmap[t0 + j] = static_cast<int32_t>(v);
}

// products of each (src 0) virtual row: one warp per row
__global__ void k_hv_vrow_nprod(HvArgs a, int64_t* out) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= a.nrows) return;
  const HvRow r = a.rows[w];
  const int64_t a0 = r.src == 0 ? a.A.rpt[r.row] : 0;
  int64_t s = 0;
  for (int j = lane; j < r.nl; j += 32) s += hv_list(a, r, a0, j).len;
#pragma unroll
  for (int d = 16; d; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
  if (lane == 0) out[w] = s;
}

cudaError_t launch_hv_plan(const HvArgs& a, bool count_only, cudaStream_t st) {
  if (a.nrows <= 0) return cudaSuccess;
  constexpr int smem = hv_plan_smem();
  static_assert(smem <= 232448, "plan shared memory exceeds 227 KB");
  static bool set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_hv_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    set[dev] = true;
  }
  k_hv_plan<<<static_cast<unsigned>(a.nrows), kHvPlanG, smem, st>>>(a, count_only ? 1 : 0);
  return cudaGetLastError();
}

template <int OUT>
static cudaError_t launch_hv_merge_t(const HvArgs& a, int64_t ntasks, const RowOut& o, cudaStream_t st) {
  constexpr int smem = hv_merge_smem();
  static_assert(smem <= 232448, "merge shared memory exceeds 227 KB");
  static bool set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_hv_merge<OUT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    set[dev] = true;
  }
  k_hv_merge<OUT><<<static_cast<unsigned>(ntasks), kHvG, smem, st>>>(a, o);
  return cudaGetLastError();
}

cudaError_t launch_hv_merge(int out_kind, const HvArgs& a, int64_t ntasks, const RowOut& o, cudaStream_t st) {
  if (ntasks <= 0) return cudaSuccess;
  switch (out_kind) {
    case OUT_CBAR: return launch_hv_merge_t<OUT_CBAR>(a, ntasks, o, st);
    case OUT_C: return launch_hv_merge_t<OUT_C>(a, ntasks, o, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_hv_ntask(const HvArgs& a, int64_t* ntask, cudaStream_t st) {
  if (a.nrows <= 0) return cudaSuccess;
  k_hv_ntask<<<static_cast<unsigned>((a.nrows + 255) / 256), 256, 0, st>>>(a, ntask);
  return cudaGetLastError();
}

cudaError_t launch_hv_taskmap(const HvArgs& a, HvRow* rows, const int64_t* toff, int32_t* tmap, cudaStream_t st) {
  if (a.nrows <= 0) return cudaSuccess;
  k_hv_taskmap<<<static_cast<unsigned>((a.nrows * 32 + 255) / 256), 256, 0, st>>>(a, rows, toff, tmap);
  return cudaGetLastError();
}

cudaError_t launch_hv_vrow_nprod(const HvArgs& a, int64_t* out, cudaStream_t st) {
  if (a.nrows <= 0) return cudaSuccess;
  const int64_t threads = a.nrows * 32;
  k_hv_vrow_nprod<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(a, out);
  return cudaGetLastError();
}

}  // namespace brm
