// api.cu -- the C ABI of include/brmerge.h: context, workspace, and the
// orchestration of Fig. 4a (BRMerge-Upper) and Fig. 4b (BRMerge-Precise),
// PAPER.md:284-300, on one device stream.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "brmerge.h"
#include "heavy.cuh"
#include "kernels.cuh"

using namespace brm;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
};

struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
};

}  // namespace

struct brm_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  bool timing = false;
  int heavy_route = BRM_HEAVY_AUTO;
  // workspace (grow-only)
  DevBuf nprod_off, row_size, bins, status, small, cbar_col, cbar_val, gws, gws_off, heavy_info, long_list, long_np;
  DevBuf stA_rpt, stA_col, stA_val, stB_rpt, stB_col, stB_val, stC_rpt, stC_col, stC_val;
  HostBuf h_small, h_heavy, h_gws_off, h_C;
  // plan (structure -> fill)
  bool planned = false;
  brm_mode_t mode = BRM_PRECISE;
  CsrView A{}, B{};
  int64_t M = 0, K = 0, N = 0, nnz_c = 0, bnnz = 0;
  int64_t bin_start[BRM_NUM_BINS] = {};
  int64_t bin_rows[BRM_NUM_BINS] = {};
  DevSummary sum{};
  bool heavy_loaded = false;
  std::vector<int64_t> heavy;  // (n_prod, nl) per global-tier row
  std::vector<int32_t> heavy_rows;  // the global-tier rows (bin order)
  cudaEvent_t ev_heavy = nullptr;   // their readback landed
  brm_stats_t stats{};
  cudaEvent_t ev[32] = {};
  cudaEvent_t handoff = nullptr;  // orders a stream switch after the old stream's work
  unsigned ev_mask = 0;  // events recorded since the last structure call
  int64_t launches = 0;  // kernels launched since the last structure call
  DevBuf glob_rows;
  HostBuf h_rows;
  // windowed heavy rows (heavy.cuh): rows of <= kHvLists lists ("single",
  // planned in structure, merged in fill under PRECISE) and the levels of
  // rows of more lists ("multi", planned and merged within one call)
  struct HvSet {
    std::vector<HvRow> rows;
    int64_t ntasks = 0;  // upper bound (from the plan capacities): the merge grid
    DevBuf d_rows, cuts, wout, nwin, total, ntask, toff, tmap;
  } hv_single, hv_multi;
  bool hv_single_planned = false;
  DevBuf hv_lt[2], hv_ws_col[2], hv_ws_val[2], hv_tmp;
  HostBuf h_hv;
  // host-buffer form for large A: row blocks, C copied back per block on a
  // copy stream (brmerge_spgemm_host, "pipelined")
  static constexpr int kPipeBlocks = 16;
  cudaStream_t copy_st = nullptr;
  cudaEvent_t ev_blk[kPipeBlocks] = {};
  DevBuf blk_rpt[kPipeBlocks], blk_col[kPipeBlocks], blk_val[kPipeBlocks], hb_nprod, hb_off, hb_bounds;
  HostBuf h_prpt, h_pcol, h_pval, h_bounds, h_rb;
  // readbacks by a copy kernel instead of a copy engine (set while the
  // pipelined host entry keeps a copy engine busy with C)
  bool kernel_readback = false;
  int64_t pipe_min_products = int64_t(1) << 26;  // brm_set_host_pipeline
  Mirrors mirrors{};  // brm_set_mirrors: peers' copies of C written by brmerge_spgemm_fill
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

brm_status_t fail(brm_context_t* c, brm_status_t s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}

brm_status_t cuda_fail(brm_context_t* c, cudaError_t e, const char* what) {
  const bool oom = e == cudaErrorMemoryAllocation;
  cudaGetLastError();
  return fail(c, oom ? BRM_ERR_OOM : BRM_ERR_CUDA,
              std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}

#define CK(call, what)                               \
  do {                                               \
    cudaError_t e_ = (call);                         \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, what); \
  } while (0)

cudaError_t ensure(brm_context_t* ctx, DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return cudaSuccess;
  if (b.p) {
    cudaError_t e = cudaFreeAsync(b.p, ctx->stream);
    if (e != cudaSuccess) return e;
    b.p = nullptr;
    b.cap = 0;
  }
  const size_t want = (bytes + 255) & ~size_t(255);
  cudaError_t e = cudaMallocAsync(&b.p, want, ctx->stream);
  if (e == cudaErrorMemoryAllocation) {
    // blocks freed on the stream stay reserved in the pool until it is
    // trimmed: return them to the device and retry once
    (void)cudaGetLastError();
    cudaMemPool_t pool;
    if (cudaStreamSynchronize(ctx->stream) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, ctx->device) == cudaSuccess &&
        cudaMemPoolTrimTo(pool, 0) == cudaSuccess)
      e = cudaMallocAsync(&b.p, want, ctx->stream);
  }
  if (e != cudaSuccess) {
    b.p = nullptr;
    return e;
  }
  b.cap = want;
  return cudaSuccess;
}

cudaError_t ensure_host(HostBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return cudaSuccess;
  const size_t want = std::max(bytes, b.cap * 3 / 2);
  if (b.p) cudaFreeHost(b.p);
  b.p = nullptr;
  b.cap = 0;
  cudaError_t e = cudaMallocHost(&b.p, want);
  if (e != cudaSuccess) {
    b.p = nullptr;
    return e;
  }
  b.cap = want;
  return cudaSuccess;
}

// Small device -> host readbacks of the library's own host logic (summaries,
// heavy-row info) into PINNED memory: a copy engine normally, a copy kernel
// (SM stores through the pinned buffer's host mapping) while the pipelined
// host entry's bulk copies occupy the copy engine -- queued behind them, a
// readback would stall the compute stream until the bulk copy ended.
cudaError_t readback(brm_context_t* ctx, void* pinned_dst, const void* src, size_t bytes) {
  if (ctx->kernel_readback) return launch_copy_to_host(pinned_dst, src, (int64_t)bytes, 4, ctx->stream);
  return cudaMemcpyAsync(pinned_dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream);
}

void free_dev(brm_context_t* ctx, DevBuf& b) {
  if (b.p) cudaFreeAsync(b.p, ctx->stream);
  b.p = nullptr;
  b.cap = 0;
}

brm_status_t check_csr(brm_context_t* ctx, const brm_csr_t* X, const char* name) {
  if (!X) return fail(ctx, BRM_ERR_INVALID, std::string(name) + " is null");
  if (X->rows < 0 || X->cols < 0 || X->nnz < 0)
    return fail(ctx, BRM_ERR_INVALID, std::string(name) + " has a negative size");
  if (!X->rpt) return fail(ctx, BRM_ERR_INVALID, std::string(name) + ".rpt is null");
  if (X->nnz > 0 && (!X->col || !X->val))
    return fail(ctx, BRM_ERR_INVALID, std::string(name) + ".col/.val is null");
  return BRM_OK;
}

// Small device block: summary + scan counters + bin cursor + nnz total.
struct SmallDev {
  DevSummary summary;
  unsigned long long cursor[BRM_NUM_BINS];
  unsigned int counter[4];
  int64_t nnz_total;
  unsigned int hv_err;  // heavy-row windows: inconsistency flags (heavy.cuh HvArgs::err)
  unsigned int pad;
};

SmallDev* small_dev(brm_context_t* ctx) { return static_cast<SmallDev*>(ctx->small.p); }

// n_prod of A's rows of more than kLongRow nonzeros, ahead of the per-warp
// n_prod passes (needs ctx->small; uses its counter[2]); *long_np = their
// values for those passes. Below 65,536 rows the warps take long rows
// themselves (*long_np = null): no skew worth the pass's fixed cost.
brm_status_t long_rows(brm_context_t* ctx, const CsrView& A, const int64_t* brpt, int64_t M,
                       const int64_t** long_np) {
  *long_np = nullptr;
  if (M < 65536) return BRM_OK;
  CK(ensure(ctx, ctx->long_np, (size_t)M * 8), "alloc long rows");
  CK(ensure(ctx, ctx->long_list, (size_t)M * 4), "alloc long rows");
  CK(ensure(ctx, ctx->long_np, (size_t)M * 8), "alloc long rows");
  CK(cudaMemsetAsync(&small_dev(ctx)->counter[2], 0, 4, ctx->stream), "memset long-row counter");
  CK(launch_long_rows(A, brpt, M, static_cast<int32_t*>(ctx->long_list.p), &small_dev(ctx)->counter[2],
                      static_cast<int64_t*>(ctx->long_np.p), ctx->stream), "k_long_rows");
  ctx->launches += 2;
  *long_np = static_cast<const int64_t*>(ctx->long_np.p);
  return BRM_OK;
}

// Timing events (no synchronisation when recorded; resolved in brm_get_stats):
// 0/1 n_prod+scan+bin, 2/3 structure merge, 3/4 row_size scan, 5/6 fill,
// 10+2b / 11+2b numeric merge of bin b.
constexpr int kEvBin = 10;
constexpr int kEvHv = 26;  // 26/27 heavy plan (single-level rows), 28/29 heavy merge
void ev_record(brm_context_t* ctx, int i) {
  if (!ctx->timing) return;
  cudaEventRecord(ctx->ev[i], ctx->stream);
  ctx->ev_mask |= 1u << i;
}

float ev_ms(const brm_context_t* ctx, int a, int b) {
  float ms = 0.f;
  if (ctx->timing && (ctx->ev_mask >> a & 1u) && (ctx->ev_mask >> b & 1u))
    cudaEventElapsedTime(&ms, ctx->ev[a], ctx->ev[b]);
  return ms;
}

// Exclusive scan with fresh look-back state.
brm_status_t run_scan(brm_context_t* ctx, const int64_t* in, int64_t n, int64_t* out, int64_t* total_out) {
  const int64_t tiles = scan_tiles(n);
  CK(ensure(ctx, ctx->status, (size_t)(tiles + 1) * 8), "alloc scan status");
  CK(cudaMemsetAsync(ctx->status.p, 0, (size_t)(tiles + 1) * 8, ctx->stream), "memset scan status");
  SmallDev* sd = small_dev(ctx);
  CK(cudaMemsetAsync(&sd->counter[1], 0, 4, ctx->stream), "memset scan counter");
  if (n == 0) {
    CK(cudaMemsetAsync(out, 0, 8, ctx->stream), "memset scan out");
    if (total_out) CK(cudaMemsetAsync(total_out, 0, 8, ctx->stream), "memset scan total");
    return BRM_OK;
  }
  CK(launch_scan_i64(in, n, out, static_cast<unsigned long long*>(ctx->status.p), &sd->counter[1],
                     total_out, ctx->stream),
     "k_scan_i64");
  ++ctx->launches;
  return BRM_OK;
}

// ---------------------------------------------------------------------------
// Windowed heavy rows (heavy.cuh).
// ---------------------------------------------------------------------------
using HvSet = brm_context::HvSet;
constexpr int kHvWch = 16;  // windows per merge task

HvArgs hv_args(brm_context_t* ctx, HvSet& set) {
  HvArgs a{};
  a.A = ctx->A;
  a.B = ctx->B;
  a.ncols = ctx->N;
  a.rows = static_cast<const HvRow*>(set.d_rows.p);
  a.nrows = static_cast<int64_t>(set.rows.size());
  a.cuts = static_cast<int32_t*>(set.cuts.p);
  a.wout = static_cast<int32_t*>(set.wout.p);
  a.nwin = static_cast<int32_t*>(set.nwin.p);
  a.total = static_cast<int64_t*>(set.total.p);
  a.err = &small_dev(ctx)->hv_err;
  return a;
}

// Sort the virtual rows by n_prod (heaviest first: a launch lasts as long as
// its heaviest rows), give each its plan slice and merge tasks, upload.
brm_status_t hv_upload(brm_context_t* ctx, HvSet& set, bool sort) {
  if (sort) {
    // heaviest first, by octave of n_prod (a counting sort, stable inside an
    // octave): the plan runs one CTA per virtual row, so a heavy row started
    // last would trail the launch; a full comparison sort of the 64-byte rows
    // cost ~50 ms of host time on rmat20's 239K rows
    constexpr int NB = 64;
    size_t cnt[NB + 1] = {};
    auto oct = [](int64_t p) { return p > 0 ? 63 - __builtin_clzll(static_cast<unsigned long long>(p)) : 0; };
    for (const HvRow& r : set.rows) ++cnt[NB - 1 - oct(r.nprod) + 1];
    for (int b = 0; b < NB; ++b) cnt[b + 1] += cnt[b];
    std::vector<HvRow> sorted(set.rows.size());
    for (const HvRow& r : set.rows) sorted[cnt[NB - 1 - oct(r.nprod)]++] = r;
    set.rows.swap(sorted);
  }
  int64_t plan = 0, task = 0;
  for (HvRow& r : set.rows) {
    r.maxwin = static_cast<int32_t>(hv_maxwin(r.nprod, ctx->N));
    r.plan = plan;
    plan += r.maxwin + 1;
    r.wch = kHvWch;
    r.task0 = task;
    task += (r.maxwin + kHvWch - 1) / kHvWch;
  }
  set.ntasks = task;
  const size_t n = set.rows.size();
  CK(ensure(ctx, set.d_rows, n * sizeof(HvRow)), "alloc heavy rows");
  CK(ensure(ctx, set.cuts, (size_t)plan * 4), "alloc heavy plan");
  CK(ensure(ctx, set.wout, (size_t)plan * 4), "alloc heavy plan");
  CK(ensure(ctx, set.nwin, n * 4), "alloc heavy plan");
  CK(ensure(ctx, set.total, n * 8), "alloc heavy plan");
  // pageable source: the copy is complete when the call returns
  if (n) CK(cudaMemcpyAsync(set.d_rows.p, set.rows.data(), n * sizeof(HvRow), cudaMemcpyHostToDevice, ctx->stream),
            "copy heavy rows");
  return BRM_OK;
}

brm_status_t hv_check_err(brm_context_t* ctx) {
  CK(ensure_host(ctx->h_rb, 16), "alloc pinned readback");
  CK(readback(ctx, ctx->h_rb.p, &small_dev(ctx)->hv_err, 4), "copy heavy flags");
  CK(cudaStreamSynchronize(ctx->stream), "sync heavy flags");
  const unsigned int e = *static_cast<const unsigned int*>(ctx->h_rb.p);
  if (e) return fail(ctx, BRM_ERR_CUDA, "heavy rows: internal inconsistency (flags " + std::to_string(e) + ")");
  return BRM_OK;
}

// Rows of <= kHvLists lists: plan (bitmap + histogram windows; row sizes).
brm_status_t hv_plan_single(brm_context_t* ctx, const std::vector<int32_t>& rows, const std::vector<int64_t>& info,
                            int64_t* row_size) {
  HvSet& set = ctx->hv_single;
  set.rows.clear();
  for (size_t i = 0; i < rows.size(); ++i) {
    HvRow r{};
    r.row = rows[i];
    r.nprod = info[2 * i];
    r.nl = static_cast<int32_t>(info[2 * i + 1]);
    set.rows.push_back(r);
  }
  brm_status_t s = hv_upload(ctx, set, true);
  if (s != BRM_OK) return s;
  HvArgs a = hv_args(ctx, set);
  a.row_size = row_size;
  ev_record(ctx, kEvHv);
  CK(launch_hv_plan(a, false, ctx->stream), "k_hv_plan");
  ev_record(ctx, kEvHv + 1);
  ++ctx->launches;
  ctx->hv_single_planned = true;
  return BRM_OK;
}

// The merge tasks of a planned set: ceil(windows / kHvWch) per virtual row,
// their offsets (scan) and the task -> virtual row map, on the device.
brm_status_t hv_tasks(brm_context_t* ctx, HvSet& set, HvArgs& a) {
  const size_t n = set.rows.size();
  CK(ensure(ctx, set.ntask, n * 8), "alloc heavy tasks");
  CK(ensure(ctx, set.toff, (n + 1) * 8), "alloc heavy tasks");
  CK(ensure(ctx, set.tmap, (size_t)set.ntasks * 4), "alloc heavy task map");
  CK(launch_hv_ntask(a, static_cast<int64_t*>(set.ntask.p), ctx->stream), "k_hv_ntask");
  brm_status_t s = run_scan(ctx, static_cast<const int64_t*>(set.ntask.p), (int64_t)n,
                            static_cast<int64_t*>(set.toff.p), nullptr);
  if (s != BRM_OK) return s;
  CK(launch_hv_taskmap(a, static_cast<HvRow*>(set.d_rows.p), static_cast<const int64_t*>(set.toff.p),
                       static_cast<int32_t*>(set.tmap.p), ctx->stream), "k_hv_taskmap");
  ctx->launches += 3;
  a.tmap = static_cast<const int32_t*>(set.tmap.p);
  a.ntask_total = static_cast<const int64_t*>(set.toff.p) + n;
  return BRM_OK;
}

brm_status_t hv_merge_single(brm_context_t* ctx, int out, const RowOut& o) {
  HvSet& set = ctx->hv_single;
  if (set.rows.empty()) return BRM_OK;
  if (!ctx->hv_single_planned) return fail(ctx, BRM_ERR_STATE, "heavy rows merged without a plan");
  HvArgs a = hv_args(ctx, set);
  brm_status_t s = hv_tasks(ctx, set, a);
  if (s != BRM_OK) return s;
  ev_record(ctx, kEvHv + 2);
  CK(launch_hv_merge(out, a, set.ntasks, o, ctx->stream), "k_hv_merge");
  ev_record(ctx, kEvHv + 3);
  ++ctx->launches;
  return BRM_OK;
}

// Row sizes of rows of more than kHvLists lists (PRECISE symbolic): a bitmap
// over all their lists.
brm_status_t hv_count_multi(brm_context_t* ctx, const std::vector<int32_t>& rows, const std::vector<int64_t>& info,
                            int64_t* row_size) {
  if (rows.empty()) return BRM_OK;
  HvSet& set = ctx->hv_multi;
  set.rows.clear();
  for (size_t i = 0; i < rows.size(); ++i) {
    HvRow r{};
    r.row = rows[i];
    r.nprod = info[2 * i];
    r.nl = static_cast<int32_t>(info[2 * i + 1]);
    set.rows.push_back(r);
  }
  brm_status_t s = hv_upload(ctx, set, true);
  if (s != BRM_OK) return s;
  HvArgs a = hv_args(ctx, set);
  a.row_size = row_size;
  CK(launch_hv_plan(a, true, ctx->stream), "k_hv_plan (count)");
  ++ctx->launches;
  return BRM_OK;
}

// Rows of more than kHvLists lists, all levels: aligned blocks of kHvLists
// lists (sub-trees of Algorithm 1's tree) merged into a workspace, whose
// results are the next level's lists (scale 1.0), until a row has at most
// kHvLists lists; that last level writes the output row. Rows are batched so
// a level's workspace stays within a memory budget.
brm_status_t hv_run_multi(brm_context_t* ctx, int out, const RowOut& o, const std::vector<int32_t>& rows,
                          const std::vector<int64_t>& info) {
  if (rows.empty()) return BRM_OK;
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  int64_t maxP = 0;
  for (size_t i = 0; i < rows.size(); ++i) maxP = std::max(maxP, info[2 * i]);
#ifndef BRM_HV_BUDGET_DIV
#define BRM_HV_BUDGET_DIV 4  // a batch's level-1 workspace takes at most 1/4 of the free memory (tuning switch)
#endif
  const int64_t budget =
      std::max<int64_t>(std::min<int64_t>((int64_t)(free_b / BRM_HV_BUDGET_DIV), 48ll << 30), maxP * 12);
  HvSet& set = ctx->hv_multi;
  size_t b0 = 0;
  while (b0 < rows.size()) {
    size_t b1 = b0;
    int64_t bytes = 0;
    while (b1 < rows.size() && (b1 == b0 || bytes + info[2 * b1] * 12 <= budget)) bytes += info[2 * b1++] * 12;
    struct Cur {
      int64_t row, first, nlist, P;
      int src;
    };
    std::vector<Cur> cur;
    for (size_t i = b0; i < b1; ++i) cur.push_back({rows[i], 0, info[2 * i + 1], info[2 * i], 0});
    int lvl = 0;
    while (!cur.empty()) {
      set.rows.clear();
      std::vector<int64_t> owner;  // the Cur entry of each virtual row
      bool blocks = false;
      for (size_t i = 0; i < cur.size(); ++i) {
        const Cur& c = cur[i];
        if (c.nlist <= kHvLists) {
          HvRow r{};
          r.row = c.row;
          r.first = c.first;
          r.nprod = c.P;
          r.nl = static_cast<int32_t>(c.nlist);
          r.src = c.src;
          r.out = 0;
          set.rows.push_back(r);
          owner.push_back(static_cast<int64_t>(i));
        } else {
          blocks = true;
          for (int64_t l0 = 0; l0 < c.nlist; l0 += kHvLists) {
            HvRow r{};
            r.row = c.row;
            r.first = c.first + l0;
            r.nprod = -1;
            r.nl = static_cast<int32_t>(std::min<int64_t>(kHvLists, c.nlist - l0));
            r.src = c.src;
            r.out = 1;
            set.rows.push_back(r);
            owner.push_back(static_cast<int64_t>(i));
          }
        }
      }
      const size_t nv = set.rows.size();
      const int in = (lvl + 1) & 1, outb = lvl & 1;  // workspace / list-table ping-pong
      if (blocks) {  // products of each block
        for (HvRow& r : set.rows) r.nprod = 0;
        brm_status_t s = hv_upload(ctx, set, false);
        if (s != BRM_OK) return s;
        HvArgs a = hv_args(ctx, set);
        a.lt = static_cast<const int64_t*>(ctx->hv_lt[in].p);
        a.ws_col = static_cast<const int32_t*>(ctx->hv_ws_col[in].p);
        CK(ensure(ctx, ctx->hv_tmp, nv * 8), "alloc heavy block sizes");
        CK(launch_hv_vrow_nprod(a, static_cast<int64_t*>(ctx->hv_tmp.p), ctx->stream), "k_hv_vrow_nprod");
        ++ctx->launches;
        CK(ensure_host(ctx->h_rb, nv * 8), "alloc pinned readback");
        CK(readback(ctx, ctx->h_rb.p, ctx->hv_tmp.p, nv * 8), "copy block sizes");
        CK(cudaStreamSynchronize(ctx->stream), "sync block sizes");
        const int64_t* np = static_cast<const int64_t*>(ctx->h_rb.p);
        for (size_t v = 0; v < nv; ++v) set.rows[v].nprod = np[v];
      }
      // sort heaviest first, keeping each virtual row's Cur entry
      std::vector<size_t> ord(nv);
      for (size_t v = 0; v < nv; ++v) ord[v] = v;
      std::stable_sort(ord.begin(), ord.end(), [&](size_t x, size_t y) { return set.rows[x].nprod > set.rows[y].nprod; });
      {
        std::vector<HvRow> sr(nv);
        std::vector<int64_t> so(nv);
        for (size_t v = 0; v < nv; ++v) {
          sr[v] = set.rows[ord[v]];
          so[v] = owner[ord[v]];
        }
        set.rows.swap(sr);
        owner.swap(so);
      }
      brm_status_t s = hv_upload(ctx, set, false);
      if (s != BRM_OK) return s;
      HvArgs a = hv_args(ctx, set);
      a.lt = static_cast<const int64_t*>(ctx->hv_lt[in].p);
      a.ws_col = static_cast<const int32_t*>(ctx->hv_ws_col[in].p);
      a.ws_val = static_cast<const double*>(ctx->hv_ws_val[in].p);
      a.row_size = out == OUT_C ? nullptr : o.row_size;
      CK(launch_hv_plan(a, false, ctx->stream), "k_hv_plan");
      ++ctx->launches;
      std::vector<Cur> next;
      if (blocks) {
        // block results: contiguous per row, in block order
        CK(ensure_host(ctx->h_rb, nv * 8), "alloc pinned readback");
        CK(readback(ctx, ctx->h_rb.p, set.total.p, nv * 8), "copy block totals");
        CK(cudaStreamSynchronize(ctx->stream), "sync block totals");
        const std::vector<int64_t> tot(static_cast<const int64_t*>(ctx->h_rb.p),
                                       static_cast<const int64_t*>(ctx->h_rb.p) + nv);
        std::vector<std::vector<size_t>> of(cur.size());  // block virtual rows of each Cur, in block order
        for (size_t v = 0; v < nv; ++v)
          if (set.rows[v].out == 1) of[owner[v]].push_back(v);
        std::vector<int64_t> lt;
        int64_t pos = 0;
        for (size_t i = 0; i < cur.size(); ++i) {
          if (of[i].empty()) continue;
          std::sort(of[i].begin(), of[i].end(), [&](size_t x, size_t y) { return set.rows[x].first < set.rows[y].first; });
          Cur nc{cur[i].row, static_cast<int64_t>(lt.size()), static_cast<int64_t>(of[i].size()), 0, 1};
          for (size_t v : of[i]) {
            set.rows[v].obase = pos;
            lt.push_back(pos);
            pos += tot[v];
            nc.P += tot[v];
          }
          lt.push_back(pos);
          next.push_back(nc);
        }
        CK(ensure(ctx, ctx->hv_ws_col[outb], (size_t)pos * 4), "alloc heavy workspace");
        CK(ensure(ctx, ctx->hv_ws_val[outb], (size_t)pos * 8), "alloc heavy workspace");
        CK(ensure(ctx, ctx->hv_lt[outb], lt.size() * 8), "alloc heavy list table");
        CK(cudaMemcpyAsync(ctx->hv_lt[outb].p, lt.data(), lt.size() * 8, cudaMemcpyHostToDevice, ctx->stream),
           "copy heavy list table");
        CK(cudaMemcpyAsync(set.d_rows.p, set.rows.data(), nv * sizeof(HvRow), cudaMemcpyHostToDevice, ctx->stream),
           "copy heavy rows");
        a.wo_col = static_cast<int32_t*>(ctx->hv_ws_col[outb].p);
        a.wo_val = static_cast<double*>(ctx->hv_ws_val[outb].p);
      }
      if ((s = hv_tasks(ctx, set, a)) != BRM_OK) return s;
      CK(launch_hv_merge(out == OUT_C ? OUT_C : OUT_CBAR, a, set.ntasks, o, ctx->stream), "k_hv_merge");
      ++ctx->launches;
      // the next level reads this level's workspace (ordered on the stream)
      cur.swap(next);
      ++lvl;
    }
    b0 = b1;
  }
  return BRM_OK;
}

// Launch the merge of every non-empty bin with output kind `out`.
brm_status_t run_merge(brm_context_t* ctx, int out, const RowOut& o, bool per_bin) {
  const int32_t* bins = static_cast<const int32_t*>(ctx->bins.p);
  const int64_t nh = ctx->bin_rows[kBinGlobal];
  const int32_t* hrows = bins + ctx->bin_start[kBinGlobal];
  // the heavy rows' (n_prod, nl) and ids are read back first (once per
  // structure call), so the host prepares their plans while the tier
  // kernels launched below run
  const bool load = nh && !ctx->heavy_loaded;
  if (load) {
    CK(ensure(ctx, ctx->heavy_info, (size_t)nh * 16), "alloc heavy info");
    CK(launch_heavy_info(ctx->A, static_cast<const int64_t*>(ctx->nprod_off.p), hrows, nh,
                         static_cast<int64_t*>(ctx->heavy_info.p), ctx->stream),
       "k_heavy_info");
    ++ctx->launches;
    CK(ensure_host(ctx->h_heavy, (size_t)nh * 16), "alloc pinned heavy info");
    CK(ensure_host(ctx->h_rows, (size_t)nh * 4), "alloc pinned heavy rows");
    CK(readback(ctx, ctx->h_heavy.p, ctx->heavy_info.p, (size_t)nh * 16), "copy heavy info");
    CK(readback(ctx, ctx->h_rows.p, hrows, (size_t)nh * 4), "copy heavy rows");
    if (!ctx->ev_heavy) CK(cudaEventCreateWithFlags(&ctx->ev_heavy, cudaEventDisableTiming), "create event");
    CK(cudaEventRecord(ctx->ev_heavy, ctx->stream), "record heavy readback");
  }
  for (int b = 1; b < kBinGlobal; ++b) {
    if (!ctx->bin_rows[b]) continue;
    if (per_bin) ev_record(ctx, kEvBin + 2 * b);
    CK(launch_tier(b, out, ctx->A, ctx->B, ctx->N, bins + ctx->bin_start[b], ctx->bin_rows[b], o, ctx->stream),
       "k_tier");
    ++ctx->launches;
    if (per_bin) ev_record(ctx, kEvBin + 2 * b + 1);
  }
  if (!nh) return BRM_OK;
  if (per_bin) ev_record(ctx, kEvBin + 2 * kBinGlobal);
  if (load) {
    CK(cudaEventSynchronize(ctx->ev_heavy), "sync heavy readback");
    const int64_t* hi = static_cast<const int64_t*>(ctx->h_heavy.p);
    ctx->heavy.assign(hi, hi + 2 * nh);
    const int32_t* hr0 = static_cast<const int32_t*>(ctx->h_rows.p);
    ctx->heavy_rows.assign(hr0, hr0 + nh);
    ctx->heavy_loaded = true;
  }
  const int32_t* hr = ctx->heavy_rows.data();
  if (ctx->heavy_route == BRM_HEAVY_AUTO) {
    // windowed BRMerge (heavy.cuh): rows of <= kHvLists lists in one level,
    // the rest in levels of aligned kHvLists-list blocks
    std::vector<int32_t> r1, rm;
    std::vector<int64_t> i1, im;
    for (int64_t t = 0; t < nh; ++t) {
      const int64_t P = ctx->heavy[2 * t], nl = ctx->heavy[2 * t + 1];
      (nl <= kHvLists ? r1 : rm).push_back(hr[t]);
      (nl <= kHvLists ? i1 : im).push_back(P);
      (nl <= kHvLists ? i1 : im).push_back(nl);
    }
    ctx->stats.hv_rows_one = static_cast<int64_t>(r1.size());
    ctx->stats.hv_rows_multi = static_cast<int64_t>(rm.size());
    brm_status_t st = BRM_OK;
    if (out == OUT_SYMBOLIC) {  // PRECISE step 3: row sizes (+ the windows of the one-level rows, kept for fill)
      if ((st = hv_plan_single(ctx, r1, i1, o.row_size)) != BRM_OK) return st;
      if ((st = hv_count_multi(ctx, rm, im, o.row_size)) != BRM_OK) return st;
    } else {
      if (out == OUT_CBAR && (st = hv_plan_single(ctx, r1, i1, o.row_size)) != BRM_OK) return st;
      if ((st = hv_merge_single(ctx, out, o)) != BRM_OK) return st;
      if ((st = hv_run_multi(ctx, out, o, rm, im)) != BRM_OK) return st;
      if ((st = hv_check_err(ctx)) != BRM_OK) return st;
    }
    if (per_bin) ev_record(ctx, kEvBin + 2 * kBinGlobal + 1);
    return BRM_OK;
  }
  // BRM_HEAVY_GLOBAL: every heavy row on the global-memory tier, heaviest
  // first (a launch lasts as long as its heaviest rows)
  std::vector<int64_t> order(nh);
  for (int64_t t = 0; t < nh; ++t) order[t] = t;
  std::sort(order.begin(), order.end(),
            [&](int64_t x, int64_t y) { return ctx->heavy[2 * x] > ctx->heavy[2 * y]; });
  std::vector<int32_t> g_rows;
  std::vector<int64_t> g_info;
  for (const int64_t t : order) {
    g_rows.push_back(hr[t]);
    g_info.push_back(ctx->heavy[2 * t]);
    g_info.push_back(ctx->heavy[2 * t + 1]);
  }
  const int64_t ng = (int64_t)g_rows.size();
  CK(ensure(ctx, ctx->glob_rows, (size_t)ng * 4), "alloc heavy rows");
  CK(cudaMemcpyAsync(ctx->glob_rows.p, g_rows.data(), (size_t)ng * 4, cudaMemcpyHostToDevice, ctx->stream),
     "copy heavy rows");  // pageable source: copied when the call returns
  if (ng > 0) {
    const int32_t* grows = static_cast<const int32_t*>(ctx->glob_rows.p);
    const bool vals = out != OUT_SYMBOLIC;
    // batch the rows so their workspace slices fit the budget
    auto row_bytes = [&](int64_t t) { return global_row_bytes(g_info[2 * t], g_info[2 * t + 1], vals); };
    int64_t max_row = 0;
    for (int64_t t = 0; t < ng; ++t) max_row = std::max(max_row, row_bytes(t));
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    // a workspace already held is reused as is; a new one takes at most half
    // the free memory
    int64_t budget = std::min<int64_t>(std::max<int64_t>((int64_t)(free_b / 2), (int64_t)ctx->gws.cap), 64ll << 30);
    budget = std::max(budget, max_row);
    CK(ensure_host(ctx->h_gws_off, (size_t)ng * 16), "alloc pinned ws offsets");
    CK(ensure(ctx, ctx->gws_off, (size_t)ng * 16), "alloc ws offsets");
    int64_t* hoff = static_cast<int64_t*>(ctx->h_gws_off.p);
    std::vector<int64_t> cuts{0};
    int64_t acc = 0, need = 0;
    for (int64_t t = 0; t < ng; ++t) {
      const int64_t bytes = row_bytes(t);
      if (t > 0 && acc + bytes > budget) {
        cuts.push_back(t);
        acc = 0;
      }
      hoff[2 * t] = acc;
      hoff[2 * t + 1] = g_info[2 * t];
      acc += bytes;
      need = std::max(need, acc);
    }
    cuts.push_back(ng);
    CK(ensure(ctx, ctx->gws, (size_t)need), "alloc global-tier workspace");
    CK(cudaMemcpyAsync(ctx->gws_off.p, hoff, (size_t)ng * 16, cudaMemcpyHostToDevice, ctx->stream),
       "copy ws offsets");
    for (size_t c = 0; c + 1 < cuts.size(); ++c) {
      const int64_t b0 = cuts[c], n = cuts[c + 1] - b0;
      if (n <= 0) continue;
      const int64_t* woff = static_cast<const int64_t*>(ctx->gws_off.p) + 2 * b0;
      unsigned char* ws = static_cast<unsigned char*>(ctx->gws.p);
      CK(launch_global_tier(out, ctx->A, ctx->B, grows + b0, n, woff, ws, o, ctx->stream), "k_global_tier");
      ++ctx->launches;
    }
  }
  if (per_bin) ev_record(ctx, kEvBin + 2 * kBinGlobal + 1);
  return BRM_OK;
}

brm_status_t structure_impl(brm_context_t* ctx, const brm_csr_t* A, const brm_csr_t* B, brm_mode_t mode,
                            int64_t* c_rpt, int64_t* c_nnz) {
  brm_status_t s;
  if ((s = check_csr(ctx, A, "A")) != BRM_OK) return s;
  if ((s = check_csr(ctx, B, "B")) != BRM_OK) return s;
  if (mode != BRM_UPPER && mode != BRM_PRECISE) return fail(ctx, BRM_ERR_INVALID, "mode must be BRM_UPPER or BRM_PRECISE");
  if (A->cols != B->rows) return fail(ctx, BRM_ERR_DIM, "A.cols != B.rows");
  if (B->cols >= INT32_MAX) return fail(ctx, BRM_ERR_INVALID, "B.cols must be < 2^31 - 1");
  if (!c_rpt || !c_nnz) return fail(ctx, BRM_ERR_INVALID, "c_rpt / c_nnz is null");
  ctx->planned = false;
  ctx->heavy_loaded = false;
  ctx->hv_single_planned = false;
  ctx->hv_single.rows.clear();
  ctx->mode = mode;
  ctx->A = CsrView{A->rpt, A->col, A->val};
  ctx->B = CsrView{B->rpt, B->col, B->val};
  ctx->M = A->rows;
  ctx->K = A->cols;
  ctx->N = B->cols;
  ctx->bnnz = B->nnz;
  const int64_t M = ctx->M;
  memset(&ctx->stats, 0, sizeof(ctx->stats));
  ctx->ev_mask = 0;
  ctx->launches = 0;
  ctx->stats.rows = M;
  ctx->stats.mode = mode;
  ctx->stats.timing_enabled = ctx->timing ? 1 : 0;

  CK(ensure(ctx, ctx->small, sizeof(SmallDev)), "alloc small");
  CK(ensure_host(ctx->h_small, sizeof(SmallDev)), "alloc pinned small");
  CK(ensure(ctx, ctx->nprod_off, (size_t)(M + 1) * 8), "alloc nprod_off");
  CK(ensure(ctx, ctx->row_size, (size_t)(M + 1) * 8), "alloc row_size");
  CK(ensure(ctx, ctx->bins, (size_t)M * 4), "alloc bins");
  const int64_t tiles = nprod_tiles(M);  // >= scan_tiles(M): the status array serves both scans
  CK(ensure(ctx, ctx->status, (size_t)(tiles + 1) * 8), "alloc scan status");
  SmallDev* sd = small_dev(ctx);
  ev_record(ctx, 0);
  CK(cudaMemsetAsync(sd, 0, sizeof(SmallDev), ctx->stream), "memset small");
  CK(cudaMemsetAsync(ctx->status.p, 0, (size_t)(tiles + 1) * 8, ctx->stream), "memset status");
  int64_t* nprod_off = static_cast<int64_t*>(ctx->nprod_off.p);
  int64_t* row_size = static_cast<int64_t*>(ctx->row_size.p);
  if (M == 0) {
    CK(cudaMemsetAsync(nprod_off, 0, 8, ctx->stream), "memset");
  }
  // Step 1: n_prod per row + prefix sum (+ bin histogram)
  const int64_t* lnp = nullptr;
  if ((s = long_rows(ctx, ctx->A, B->rpt, M, &lnp)) != BRM_OK) return s;
  CK(launch_nprod_scan(ctx->A, B->rpt, M, nprod_off, static_cast<unsigned long long*>(ctx->status.p),
                       &sd->counter[0], &sd->summary, lnp, ctx->stream),
     "k_nprod_scan");
  // row binning
  CK(launch_bin_scatter(ctx->A, nprod_off, M, &sd->summary, sd->cursor, static_cast<int32_t*>(ctx->bins.p),
                        row_size, ctx->stream),
     "k_bin_scatter");
  if (M > 0) ctx->launches += 2;
  ev_record(ctx, 1);
  CK(readback(ctx, ctx->h_small.p, sd, sizeof(SmallDev)), "copy summary");
  CK(cudaStreamSynchronize(ctx->stream), "sync summary");
  ctx->sum = static_cast<SmallDev*>(ctx->h_small.p)->summary;
  ctx->stats.nprod_total = ctx->sum.nprod_total;
  ctx->stats.nprod_max = (int64_t)ctx->sum.nprod_max;
  if (ctx->sum.nprod_max >= (1ull << 31))
    return fail(ctx, BRM_ERR_OVERFLOW, "a row has n_prod >= 2^31");
  int64_t acc = 0;
  for (int b = 0; b < BRM_NUM_BINS; ++b) {
    ctx->bin_rows[b] = (int64_t)ctx->sum.bin_rows[b];
    ctx->stats.bin_rows[b] = ctx->bin_rows[b];
    ctx->stats.bin_nprod[b] = (int64_t)ctx->sum.bin_nprod[b];
    ctx->bin_start[b] = acc;
    if (b != kBinEmpty) acc += ctx->bin_rows[b];
  }
  // UPPER: Steps 3-4 (C_bar by n_prod offsets, numeric merge);
  // PRECISE: Step 3 (symbolic merge)
  RowOut o{};
  int out;
  if (mode == BRM_UPPER) {
    const int64_t np = ctx->sum.nprod_total;
    CK(ensure(ctx, ctx->cbar_col, (size_t)np * 4), "alloc C_bar col");
    CK(ensure(ctx, ctx->cbar_val, (size_t)np * 8), "alloc C_bar val");
    o.base = nprod_off;
    o.col = static_cast<int32_t*>(ctx->cbar_col.p);
    o.val = static_cast<double*>(ctx->cbar_val.p);
    o.row_size = row_size;
    out = OUT_CBAR;
  } else {
    o.row_size = row_size;
    out = OUT_SYMBOLIC;
  }
  ev_record(ctx, 2);
  if ((s = run_merge(ctx, out, o, mode == BRM_UPPER)) != BRM_OK) return s;
  ev_record(ctx, 3);
  // Step 5 (UPPER) / Step 4 (PRECISE): prefix sum of row sizes -> rpt, nnz(C)
  if ((s = run_scan(ctx, row_size, M, c_rpt, &sd->nnz_total)) != BRM_OK) return s;
  ev_record(ctx, 4);
  CK(readback(ctx, ctx->h_small.p, sd, sizeof(SmallDev)), "copy nnz");
  CK(cudaStreamSynchronize(ctx->stream), "sync nnz");
  ctx->nnz_c = static_cast<SmallDev*>(ctx->h_small.p)->nnz_total;
  *c_nnz = ctx->nnz_c;
  ctx->stats.nnz_c = ctx->nnz_c;
  ctx->planned = true;
  return BRM_OK;
}

// mir: the peers' copies of C (brmerge_spgemm_fill only; the other forms
// pass none)
brm_status_t fill_impl(brm_context_t* ctx, brm_csr_t* C, const Mirrors& mir = Mirrors{}) {
  if (!ctx->planned) return fail(ctx, BRM_ERR_STATE, "fill without a preceding structure call");
  if (!C || !C->rpt || (ctx->nnz_c > 0 && (!C->col || !C->val)))
    return fail(ctx, BRM_ERR_INVALID, "C arrays are null");
  C->rows = ctx->M;
  C->cols = ctx->N;
  C->nnz = ctx->nnz_c;
  ev_record(ctx, 5);
  if (ctx->mode == BRM_UPPER) {
    // Step 6 of Fig. 4a: copy C_bar -> C
    CK(launch_compact(ctx->M, ctx->nnz_c, static_cast<const int64_t*>(ctx->nprod_off.p), C->rpt,
                      static_cast<const int32_t*>(ctx->cbar_col.p), static_cast<const double*>(ctx->cbar_val.p),
                      C->col, C->val, mir, ctx->stream),
       "k_compact");
    ++ctx->launches;
    ev_record(ctx, 6);
  } else {
    // Step 5 of Fig. 4b: numeric merge straight into C
    RowOut o{};
    o.base = C->rpt;
    o.col = C->col;
    o.val = C->val;
    o.mir = mir;
    brm_status_t s = run_merge(ctx, OUT_C, o, true);
    if (s != BRM_OK) return s;
    ev_record(ctx, 6);
  }
  return BRM_OK;
}

// Host-buffer form for large A (>= 65,536 rows, >= 2^26 intermediate
// products by default: brm_set_host_pipeline), pipelined: the rows are cut into 8 or 16 blocks of balanced n_prod (the §III.D rule, by the library's
// own n_prod / scan / partition kernels), and each block runs structure +
// fill on the context stream into its own device C slice; an event then
// lets a separate copy stream bring the block's rpt / col / val back to
// pinned host memory while the next block computes. The compute stream never
// waits for a copy (every block has its own slice), so the device-to-host
// copies of C -- the e2e step's bound on large outputs -- overlap all but the
// first block's SpGEMM. A row block is a view of the uploaded A (its rpt
// values stay absolute offsets into A's col/val); block-local C.rpt values
// are rebased on the host after the copies.
constexpr int64_t kPipeMinRows = 65536;

brm_status_t host_pipelined(brm_context_t* ctx, const brm_csr_t* Ah, const brm_csr_t* Bh, const brm_csr_t* Ad,
                            const brm_csr_t* Bd, brm_mode_t mode, brm_csr_t* Ch, bool* declined) {
  constexpr int KMAX = brm_context::kPipeBlocks;
  static const bool diag_nocopy = getenv("BRM_PIPE_NOCOPY") != nullptr;  // diagnostics: skip the copies
  static const bool diag_trace = getenv("BRM_PIPE_TRACE") != nullptr;    // diagnostics: block timeline
  cudaEvent_t tr0 = nullptr, trc[KMAX] = {}, trd[KMAX] = {};
  if (diag_trace) {
    cudaEventCreate(&tr0);
    for (int k = 0; k < KMAX; ++k) {
      cudaEventCreate(&trc[k]);
      cudaEventCreate(&trd[k]);
    }
    cudaEventRecord(tr0, ctx->stream);
  }
  const int64_t M = Ah->rows;
  brm_status_t s;
  if (Ad->cols != Bd->rows) return fail(ctx, BRM_ERR_DIM, "A.cols != B.rows");
  // (1) row blocks of balanced n_prod
  CK(ensure(ctx, ctx->hb_nprod, (size_t)M * 8), "alloc n_prod");
  CK(ensure(ctx, ctx->hb_off, (size_t)(M + 1) * 8), "alloc n_prod offsets");
  CK(ensure(ctx, ctx->hb_bounds, (size_t)(KMAX + 1) * 8), "alloc block bounds");
  CK(ensure(ctx, ctx->small, sizeof(SmallDev)), "alloc small");
  const int64_t* lnp = nullptr;
  if ((s = long_rows(ctx, CsrView{Ad->rpt, Ad->col, Ad->val}, Bd->rpt, M, &lnp)) != BRM_OK) return s;
  CK(launch_row_nprod(CsrView{Ad->rpt, Ad->col, Ad->val}, Bd->rpt, M, static_cast<int64_t*>(ctx->hb_nprod.p),
                      lnp, ctx->stream), "k_row_nprod");
  if ((s = run_scan(ctx, static_cast<const int64_t*>(ctx->hb_nprod.p), M, static_cast<int64_t*>(ctx->hb_off.p),
                    nullptr)) != BRM_OK)
    return s;
  // blocks: 16 for large outputs (the first block's SpGEMM is the part no
  // copy overlaps), else 8
  CK(ensure_host(ctx->h_bounds, (size_t)(KMAX + 1) * 8), "alloc pinned bounds");
  int64_t* bounds = static_cast<int64_t*>(ctx->h_bounds.p);
  CK(cudaMemcpyAsync(bounds, static_cast<const int64_t*>(ctx->hb_off.p) + M, 8, cudaMemcpyDeviceToHost, ctx->stream),
     "D2H n_prod total");
  CK(cudaStreamSynchronize(ctx->stream), "sync n_prod total");
  // small outputs: the blocks' fixed costs (host syncs, launches) outweigh
  // the copy they hide -- the one-shot form runs instead
  *declined = bounds[0] < ctx->pipe_min_products;
  if (*declined) return BRM_OK;
  const int K = bounds[0] >= (4ll << 30) ? KMAX : KMAX / 2;
  CK(launch_partition(static_cast<const int64_t*>(ctx->hb_off.p), M, K, static_cast<int64_t*>(ctx->hb_bounds.p),
                      ctx->stream), "k_partition");
  CK(cudaMemcpyAsync(bounds, ctx->hb_bounds.p, (size_t)(K + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream),
     "D2H block bounds");
  CK(cudaStreamSynchronize(ctx->stream), "sync block bounds");
  // the blocks hold C: release the one-shot form's C buffers
  free_dev(ctx, ctx->stC_col);
  free_dev(ctx, ctx->stC_val);
  if (!ctx->copy_st) CK(cudaStreamCreateWithFlags(&ctx->copy_st, cudaStreamNonBlocking), "create copy stream");
  for (auto& e : ctx->ev_blk)
    if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "create block event");
  CK(ensure_host(ctx->h_prpt, (size_t)(M + 1) * 8), "alloc pinned C.rpt");
  int64_t* hrpt = static_cast<int64_t*>(ctx->h_prpt.p);
  // (2) the blocks: compute on the context stream, copies on the copy stream
  int64_t boff[KMAX + 1] = {};
  bool fits = true;
  // bulk copies on a copy engine (a copy kernel on the SMs measured ~29 GB/s
  // against the engine's ~48); the blocks' own small readbacks go through a
  // copy kernel meanwhile (readback()), so they do not queue behind the bulk
  auto d2h = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->copy_st);
  };
  struct ReadbackMode {
    brm_context_t* c;
    ~ReadbackMode() { c->kernel_readback = false; }
  } rb_mode{ctx};
  ctx->kernel_readback = true;
  auto copy_block = [&](int k) -> cudaError_t {
    const int64_t r0 = bounds[k], r1 = bounds[k + 1], nb = boff[k + 1] - boff[k];
    cudaError_t e = cudaSuccess;
    if (r1 > r0) e = d2h(hrpt + r0, ctx->blk_rpt[k].p, (size_t)(r1 - r0) * 8);
    if (e == cudaSuccess && nb)
      e = d2h(static_cast<double*>(ctx->h_pval.p) + boff[k], ctx->blk_val[k].p, (size_t)nb * 8);
    if (e == cudaSuccess && nb)
      e = d2h(static_cast<int32_t*>(ctx->h_pcol.p) + boff[k], ctx->blk_col[k].p, (size_t)nb * 4);
    return e;
  };
  for (int k = 0; k < K; ++k) {
    const int64_t r0 = bounds[k], r1 = bounds[k + 1];
    int64_t nb = 0;
    if (r1 > r0) {
      const brm_csr_t Ab{r1 - r0, Ad->cols, Ah->rpt[r1] - Ah->rpt[r0], Ad->rpt + r0, Ad->col, Ad->val};
      CK(ensure(ctx, ctx->blk_rpt[k], (size_t)(r1 - r0 + 1) * 8), "alloc block C.rpt");
      if ((s = structure_impl(ctx, &Ab, Bd, mode, static_cast<int64_t*>(ctx->blk_rpt[k].p), &nb)) != BRM_OK)
        return s;
      CK(ensure(ctx, ctx->blk_col[k], (size_t)nb * 4), "alloc block C.col");
      CK(ensure(ctx, ctx->blk_val[k], (size_t)nb * 8), "alloc block C.val");
      brm_csr_t Cb{0, 0, 0, static_cast<int64_t*>(ctx->blk_rpt[k].p), static_cast<int32_t*>(ctx->blk_col[k].p),
                   static_cast<double*>(ctx->blk_val[k].p)};
      if ((s = fill_impl(ctx, &Cb)) != BRM_OK) return s;
    }
    boff[k + 1] = boff[k] + nb;
    CK(cudaEventRecord(ctx->ev_blk[k], ctx->stream), "record block event");
    fits = fits && ctx->h_pcol.cap >= (size_t)boff[k + 1] * 4 && ctx->h_pval.cap >= (size_t)boff[k + 1] * 8;
    if (fits && !diag_nocopy) {
      CK(cudaStreamWaitEvent(ctx->copy_st, ctx->ev_blk[k], 0), "copy waits for block");
      CK(copy_block(k), "D2H block");
    }
    if (diag_trace) {
      cudaEventRecord(trc[k], ctx->stream);
      cudaEventRecord(trd[k], ctx->copy_st);
    }
  }
  const int64_t nnz = boff[K];
  if (diag_nocopy) {
    CK(ensure_host(ctx->h_pcol, (size_t)nnz * 4), "alloc pinned C.col");
    CK(ensure_host(ctx->h_pval, (size_t)nnz * 8), "alloc pinned C.val");
    fits = true;
  }
  if (!fits) {  // first call at this size: grow the pinned output, then copy every block
    CK(cudaStreamSynchronize(ctx->copy_st), "sync copies");
    CK(ensure_host(ctx->h_pcol, (size_t)nnz * 4), "alloc pinned C.col");
    CK(ensure_host(ctx->h_pval, (size_t)nnz * 8), "alloc pinned C.val");
    CK(cudaStreamWaitEvent(ctx->copy_st, ctx->ev_blk[K - 1], 0), "copy waits for the blocks");
    for (int k = 0; k < K; ++k) CK(copy_block(k), "D2H block");
  }
  CK(cudaStreamSynchronize(ctx->copy_st), "sync copies");
  CK(cudaStreamSynchronize(ctx->stream), "sync blocks");
  if (diag_trace) {
    for (int k = 0; k < K; ++k) {
      float tc = 0, td = 0;
      cudaEventElapsedTime(&tc, tr0, trc[k]);
      cudaEventElapsedTime(&td, tr0, trd[k]);
      fprintf(stderr, "block %d: rows %lld nnz %lld compute done %.1f ms, copy done %.1f ms\n", k,
              (long long)(bounds[k + 1] - bounds[k]), (long long)(boff[k + 1] - boff[k]), tc, td);
    }
    for (int k = 0; k < KMAX; ++k) {
      cudaEventDestroy(trc[k]);
      cudaEventDestroy(trd[k]);
    }
    cudaEventDestroy(tr0);
  }
  for (int k = 0; k < K; ++k)
    for (int64_t r = bounds[k]; r < bounds[k + 1]; ++r) hrpt[r] += boff[k];
  hrpt[M] = nnz;
  Ch->rows = M;
  Ch->cols = Bh->cols;
  Ch->nnz = nnz;
  Ch->rpt = hrpt;
  Ch->val = static_cast<double*>(ctx->h_pval.p);
  Ch->col = static_cast<int32_t*>(ctx->h_pcol.p);
  return BRM_OK;
}

}  // namespace

extern "C" {

const char* brm_status_string(brm_status_t s) {
  switch (s) {
    case BRM_OK: return "BRM_OK";
    case BRM_ERR_INVALID: return "BRM_ERR_INVALID";
    case BRM_ERR_DIM: return "BRM_ERR_DIM";
    case BRM_ERR_CUDA: return "BRM_ERR_CUDA";
    case BRM_ERR_OOM: return "BRM_ERR_OOM";
    case BRM_ERR_OVERFLOW: return "BRM_ERR_OVERFLOW";
    case BRM_ERR_STATE: return "BRM_ERR_STATE";
  }
  return "BRM_ERR_UNKNOWN";
}

brm_status_t brm_create(brm_context_t** out, int device, void* stream) {
  if (!out) return BRM_ERR_INVALID;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
    cudaGetLastError();
    return BRM_ERR_CUDA;
  }
  brm_context_t* ctx = new brm_context_t;
  ctx->device = device;
  ctx->stream = static_cast<cudaStream_t>(stream);
  DeviceGuard g(device);
  for (auto& e : ctx->ev) cudaEventCreate(&e);
  cudaEventCreateWithFlags(&ctx->handoff, cudaEventDisableTiming);
  *out = ctx;
  return BRM_OK;
}

brm_status_t brm_destroy(brm_context_t* ctx) {
  if (!ctx) return BRM_ERR_INVALID;
  {
    DeviceGuard g(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (DevBuf* b : {&ctx->nprod_off, &ctx->row_size, &ctx->bins, &ctx->status, &ctx->small, &ctx->cbar_col,
                      &ctx->long_list, &ctx->long_np,
                      &ctx->cbar_val, &ctx->gws, &ctx->gws_off, &ctx->heavy_info, &ctx->stA_rpt, &ctx->stA_col,
                      &ctx->stA_val, &ctx->stB_rpt, &ctx->stB_col, &ctx->stB_val, &ctx->stC_rpt, &ctx->stC_col,
                      &ctx->stC_val, &ctx->glob_rows, &ctx->hv_single.d_rows,
                      &ctx->hv_single.cuts, &ctx->hv_single.wout, &ctx->hv_single.nwin, &ctx->hv_single.total,
                      &ctx->hv_single.ntask, &ctx->hv_single.toff, &ctx->hv_single.tmap, &ctx->hv_multi.ntask,
                      &ctx->hv_multi.toff, &ctx->hv_multi.tmap,
                      &ctx->hv_multi.d_rows, &ctx->hv_multi.cuts, &ctx->hv_multi.wout, &ctx->hv_multi.nwin,
                      &ctx->hv_multi.total, &ctx->hv_lt[0], &ctx->hv_lt[1], &ctx->hv_ws_col[0], &ctx->hv_ws_col[1],
                      &ctx->hv_ws_val[0], &ctx->hv_ws_val[1], &ctx->hv_tmp, &ctx->hb_nprod, &ctx->hb_off,
                      &ctx->hb_bounds})
      free_dev(ctx, *b);
    for (int k = 0; k < brm_context::kPipeBlocks; ++k)
      for (DevBuf* b : {&ctx->blk_rpt[k], &ctx->blk_col[k], &ctx->blk_val[k]}) free_dev(ctx, *b);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->copy_st) {
      cudaStreamSynchronize(ctx->copy_st);
      cudaStreamDestroy(ctx->copy_st);
    }
    for (HostBuf* b : {&ctx->h_small, &ctx->h_heavy, &ctx->h_gws_off, &ctx->h_C, &ctx->h_rows, &ctx->h_prpt,
                       &ctx->h_pcol, &ctx->h_pval, &ctx->h_bounds, &ctx->h_rb})
      if (b->p) cudaFreeHost(b->p);
    for (auto& e : ctx->ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : ctx->ev_blk)
      if (e) cudaEventDestroy(e);
    if (ctx->handoff) cudaEventDestroy(ctx->handoff);
    if (ctx->ev_heavy) cudaEventDestroy(ctx->ev_heavy);
  }
  delete ctx;
  return BRM_OK;
}

brm_status_t brm_set_stream(brm_context_t* ctx, void* stream) {
  if (!ctx) return BRM_ERR_INVALID;
  cudaStream_t ns = static_cast<cudaStream_t>(stream);
  if (ns == ctx->stream) return BRM_OK;
  // the workspace (n_prod offsets, bins, C_bar, heavy-row plans) may still be
  // read by kernels enqueued on the old stream: the new stream waits for them
  DeviceGuard g(ctx->device);
  CK(cudaEventRecord(ctx->handoff, ctx->stream), "record stream hand-off");
  CK(cudaStreamWaitEvent(ns, ctx->handoff, 0), "wait for stream hand-off");
  ctx->stream = ns;
  return BRM_OK;
}

brm_status_t brm_set_timing(brm_context_t* ctx, int enable) {
  if (!ctx) return BRM_ERR_INVALID;
  ctx->timing = enable != 0;
  return BRM_OK;
}

brm_status_t brm_set_host_pipeline(brm_context_t* ctx, int64_t min_products) {
  if (!ctx) return BRM_ERR_INVALID;
  if (min_products < 0) return fail(ctx, BRM_ERR_INVALID, "min_products < 0");
  ctx->pipe_min_products = min_products;
  return BRM_OK;
}

brm_status_t brm_set_mirrors(brm_context_t* ctx, int n, int32_t* const* col, double* const* val) {
  if (!ctx) return BRM_ERR_INVALID;
  if (n < 0 || n > kMaxMirrors) return fail(ctx, BRM_ERR_INVALID, "mirror count outside [0, 7]");
  if (n > 0 && (!col || !val)) return fail(ctx, BRM_ERR_INVALID, "mirror arrays are null");
  Mirrors m{};
  for (int p = 0; p < n; ++p) {
    if (!col[p] || !val[p]) return fail(ctx, BRM_ERR_INVALID, "a mirror pointer is null");
    m.col[p] = col[p];
    m.val[p] = val[p];
  }
  m.n = n;
  ctx->mirrors = m;
  return BRM_OK;
}

brm_status_t brm_enable_peer_access(brm_context_t* ctx, int peer_device) {
  if (!ctx) return BRM_ERR_INVALID;
  if (peer_device == ctx->device) return BRM_OK;
  DeviceGuard g(ctx->device);
  int can = 0;
  CK(cudaDeviceCanAccessPeer(&can, ctx->device, peer_device), "cudaDeviceCanAccessPeer");
  if (!can) return fail(ctx, BRM_ERR_INVALID, "the peer device is not reachable over P2P");
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return BRM_OK;
  }
  CK(e, "cudaDeviceEnablePeerAccess");
  return BRM_OK;
}

brm_status_t brm_set_heavy_route(brm_context_t* ctx, int route) {
  if (!ctx || (route != BRM_HEAVY_AUTO && route != BRM_HEAVY_GLOBAL)) return BRM_ERR_INVALID;
  ctx->heavy_route = route;
  return BRM_OK;
}

const char* brm_last_error(const brm_context_t* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

brm_status_t brm_get_stats(const brm_context_t* ctx, brm_stats_t* out) {
  if (!ctx || !out) return BRM_ERR_INVALID;
  *out = ctx->stats;
  out->launches = ctx->launches;
  if (ctx->timing && ctx->ev_mask) {
    DeviceGuard g(ctx->device);
    for (int i = 31; i >= 0; --i)  // wait for everything recorded
      if (ctx->ev_mask >> i & 1u) cudaEventSynchronize(ctx->ev[i]);
    out->ms_nprod_scan = ev_ms(ctx, 0, 1);
    if (ctx->mode == BRM_UPPER) {
      out->ms_numeric = ev_ms(ctx, 2, 3);
      out->ms_compact = ev_ms(ctx, 5, 6);
    } else {
      out->ms_symbolic = ev_ms(ctx, 2, 3);
      out->ms_numeric = ev_ms(ctx, 5, 6);
    }
    out->ms_rowsize_scan = ev_ms(ctx, 3, 4);
    for (int b = 0; b < BRM_NUM_BINS; ++b) out->ms_bin_numeric[b] = ev_ms(ctx, kEvBin + 2 * b, kEvBin + 2 * b + 1);
    out->ms_hv_plan = ev_ms(ctx, kEvHv, kEvHv + 1);
    out->ms_hv_merge = ev_ms(ctx, kEvHv + 2, kEvHv + 3);
  }
  return BRM_OK;
}

brm_status_t brmerge_spgemm_structure(brm_context_t* ctx, const brm_csr_t* A, const brm_csr_t* B,
                                      brm_mode_t mode, int64_t* c_rpt, int64_t* c_nnz) {
  if (!ctx) return BRM_ERR_INVALID;
  DeviceGuard g(ctx->device);
  return structure_impl(ctx, A, B, mode, c_rpt, c_nnz);
}

brm_status_t brmerge_spgemm_fill(brm_context_t* ctx, brm_csr_t* C) {
  if (!ctx) return BRM_ERR_INVALID;
  DeviceGuard g(ctx->device);
  return fill_impl(ctx, C, ctx->mirrors);
}

brm_status_t brmerge_spgemm(brm_context_t* ctx, const brm_csr_t* A, const brm_csr_t* B, brm_mode_t mode,
                            brm_csr_t* C) {
  if (!ctx) return BRM_ERR_INVALID;
  if (!C) return fail(ctx, BRM_ERR_INVALID, "C is null");
  brm_status_t s0;
  if ((s0 = check_csr(ctx, A, "A")) != BRM_OK) return s0;  // before sizing C.rpt by A->rows
  if ((s0 = check_csr(ctx, B, "B")) != BRM_OK) return s0;
  DeviceGuard g(ctx->device);
  memset(C, 0, sizeof(*C));
  int64_t* rpt = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&rpt), (size_t)(A->rows + 1) * 8, ctx->stream), "alloc C.rpt");
  int64_t nnz = 0;
  brm_status_t s = structure_impl(ctx, A, B, mode, rpt, &nnz);
  if (s != BRM_OK) {
    cudaFreeAsync(rpt, ctx->stream);
    return s;
  }
  C->rpt = rpt;
  cudaError_t e1 = cudaMallocAsync(reinterpret_cast<void**>(&C->col), (size_t)std::max<int64_t>(nnz, 1) * 4, ctx->stream);
  cudaError_t e2 = e1 == cudaSuccess
                       ? cudaMallocAsync(reinterpret_cast<void**>(&C->val), (size_t)std::max<int64_t>(nnz, 1) * 8, ctx->stream)
                       : e1;
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    brm_csr_free(ctx, C);
    return cuda_fail(ctx, e1 != cudaSuccess ? e1 : e2, "alloc C.col/val");
  }
  s = fill_impl(ctx, C);
  if (s != BRM_OK) brm_csr_free(ctx, C);
  return s;
}

brm_status_t brm_csr_free(brm_context_t* ctx, brm_csr_t* C) {
  if (!ctx || !C) return BRM_ERR_INVALID;
  DeviceGuard g(ctx->device);
  if (C->rpt) cudaFreeAsync(C->rpt, ctx->stream);
  if (C->col) cudaFreeAsync(C->col, ctx->stream);
  if (C->val) cudaFreeAsync(C->val, ctx->stream);
  C->rpt = nullptr;
  C->col = nullptr;
  C->val = nullptr;
  return BRM_OK;
}

brm_status_t brmerge_spgemm_host(brm_context_t* ctx, const brm_csr_t* Ah, const brm_csr_t* Bh, brm_mode_t mode,
                                 brm_csr_t* Ch) {
  if (!ctx) return BRM_ERR_INVALID;
  brm_status_t s;
  if ((s = check_csr(ctx, Ah, "A")) != BRM_OK) return s;
  if ((s = check_csr(ctx, Bh, "B")) != BRM_OK) return s;
  if (!Ch) return fail(ctx, BRM_ERR_INVALID, "C is null");
  DeviceGuard g(ctx->device);
  auto up = [&](DevBuf& d, const void* h, size_t bytes) -> cudaError_t {
    cudaError_t e = ensure(ctx, d, bytes);
    if (e != cudaSuccess) return e;
    if (bytes) e = cudaMemcpyAsync(d.p, h, bytes, cudaMemcpyHostToDevice, ctx->stream);
    return e;
  };
  CK(up(ctx->stA_rpt, Ah->rpt, (size_t)(Ah->rows + 1) * 8), "H2D A.rpt");
  CK(up(ctx->stA_col, Ah->col, (size_t)Ah->nnz * 4), "H2D A.col");
  CK(up(ctx->stA_val, Ah->val, (size_t)Ah->nnz * 8), "H2D A.val");
  // C = A * A (the same host arrays): one upload serves both operands
  const bool same = Ah->rpt == Bh->rpt && Ah->col == Bh->col && Ah->val == Bh->val && Ah->rows == Bh->rows &&
                    Ah->nnz == Bh->nnz;
  if (!same) {
    CK(up(ctx->stB_rpt, Bh->rpt, (size_t)(Bh->rows + 1) * 8), "H2D B.rpt");
    CK(up(ctx->stB_col, Bh->col, (size_t)Bh->nnz * 4), "H2D B.col");
    CK(up(ctx->stB_val, Bh->val, (size_t)Bh->nnz * 8), "H2D B.val");
  }
  brm_csr_t Ad{Ah->rows, Ah->cols, Ah->nnz, static_cast<int64_t*>(ctx->stA_rpt.p),
               static_cast<int32_t*>(ctx->stA_col.p), static_cast<double*>(ctx->stA_val.p)};
  const DevBuf& br = same ? ctx->stA_rpt : ctx->stB_rpt;
  const DevBuf& bc = same ? ctx->stA_col : ctx->stB_col;
  const DevBuf& bv = same ? ctx->stA_val : ctx->stB_val;
  brm_csr_t Bd{Bh->rows, Bh->cols, Bh->nnz, static_cast<int64_t*>(br.p), static_cast<int32_t*>(bc.p),
               static_cast<double*>(bv.p)};
  if (Ah->rows >= kPipeMinRows) {
    bool declined = false;
    s = host_pipelined(ctx, Ah, Bh, &Ad, &Bd, mode, Ch, &declined);
    if (s != BRM_OK || !declined) return s;
  }
  CK(ensure(ctx, ctx->stC_rpt, (size_t)(Ah->rows + 1) * 8), "alloc C.rpt");
  int64_t nnz = 0;
  if ((s = structure_impl(ctx, &Ad, &Bd, mode, static_cast<int64_t*>(ctx->stC_rpt.p), &nnz)) != BRM_OK) return s;
  CK(ensure(ctx, ctx->stC_col, (size_t)nnz * 4), "alloc C.col");
  CK(ensure(ctx, ctx->stC_val, (size_t)nnz * 8), "alloc C.val");
  brm_csr_t Cd{0, 0, 0, static_cast<int64_t*>(ctx->stC_rpt.p), static_cast<int32_t*>(ctx->stC_col.p),
               static_cast<double*>(ctx->stC_val.p)};
  if ((s = fill_impl(ctx, &Cd)) != BRM_OK) return s;
  const size_t brpt = (size_t)(Ah->rows + 1) * 8, bcol = (size_t)nnz * 4, bval = (size_t)nnz * 8;
  CK(ensure_host(ctx->h_C, brpt + bcol + bval + 32), "alloc pinned C");
  unsigned char* h = static_cast<unsigned char*>(ctx->h_C.p);
  CK(cudaMemcpyAsync(h, Cd.rpt, brpt, cudaMemcpyDeviceToHost, ctx->stream), "D2H C.rpt");
  unsigned char* hv = h + ((brpt + 15) & ~size_t(15));
  if (bval) CK(cudaMemcpyAsync(hv, Cd.val, bval, cudaMemcpyDeviceToHost, ctx->stream), "D2H C.val");
  unsigned char* hc = hv + ((bval + 15) & ~size_t(15));
  if (bcol) CK(cudaMemcpyAsync(hc, Cd.col, bcol, cudaMemcpyDeviceToHost, ctx->stream), "D2H C.col");
  CK(cudaStreamSynchronize(ctx->stream), "sync D2H");
  Ch->rows = Ah->rows;
  Ch->cols = Bh->cols;
  Ch->nnz = nnz;
  Ch->rpt = reinterpret_cast<int64_t*>(h);
  Ch->val = reinterpret_cast<double*>(hv);
  Ch->col = reinterpret_cast<int32_t*>(hc);
  return BRM_OK;
}

brm_status_t brm_row_nprod(brm_context_t* ctx, const brm_csr_t* A, const brm_csr_t* B, int64_t* nprod) {
  if (!ctx) return BRM_ERR_INVALID;
  brm_status_t s;
  if ((s = check_csr(ctx, A, "A")) != BRM_OK) return s;
  if ((s = check_csr(ctx, B, "B")) != BRM_OK) return s;
  if (A->cols != B->rows) return fail(ctx, BRM_ERR_DIM, "A.cols != B.rows");
  if (!nprod && A->rows) return fail(ctx, BRM_ERR_INVALID, "nprod is null");
  DeviceGuard g(ctx->device);
  CK(ensure(ctx, ctx->small, sizeof(SmallDev)), "alloc small");
  const int64_t* lnp = nullptr;
  if ((s = long_rows(ctx, CsrView{A->rpt, A->col, A->val}, B->rpt, A->rows, &lnp)) != BRM_OK) return s;
  CK(launch_row_nprod(CsrView{A->rpt, A->col, A->val}, B->rpt, A->rows, nprod, lnp, ctx->stream), "k_row_nprod");
  return BRM_OK;
}

brm_status_t brm_exclusive_scan_i64(brm_context_t* ctx, const int64_t* in, int64_t* out, int64_t n) {
  if (!ctx) return BRM_ERR_INVALID;
  if (n < 0 || !out || (n > 0 && !in)) return fail(ctx, BRM_ERR_INVALID, "bad scan arguments");
  DeviceGuard g(ctx->device);
  CK(ensure(ctx, ctx->small, sizeof(SmallDev)), "alloc small");
  return run_scan(ctx, in, n, out, nullptr);
}

brm_status_t brm_partition_rows(brm_context_t* ctx, const int64_t* nprod_off, int64_t rows, int p,
                                int64_t* bounds) {
  if (!ctx) return BRM_ERR_INVALID;
  if (p < 1 || rows < 0 || !nprod_off || !bounds) return fail(ctx, BRM_ERR_INVALID, "bad partition arguments");
  DeviceGuard g(ctx->device);
  CK(launch_partition(nprod_off, rows, p, bounds, ctx->stream), "k_partition");
  return BRM_OK;
}

}  // extern "C"
