/*
 * brmerge.h -- C ABI of the B200-native BRMerge SpGEMM library
 * (libbrmerge.so, built from paper_2206_06611_b200/csrc/).
 *
 * Computes C = A * B for CSR matrices in fp64 with the row-wise (Gustavson)
 * dataflow, Eq. (2) of arxiv 2206.06611 ("C_{i*} = sum_k A_ik * B_k*"),
 * accumulating every output row with the BRMerge method of Algorithm 1
 * (PAPER.md:165-218): the scaled rows A_ik * B_k* are laid out as sorted
 * intermediate lists in one contiguous ping buffer, then merged two by two in
 * a binary tree between two ping-pong buffers, duplicate columns summed
 * (Fig. 2). Pairing is (0,1),(2,3),... each round with an odd
 * trailing list copied (Alg. 1 lines 21-35), so every output value is the
 * Algorithm-1 tree sum of its products, bit for bit.
 *
 * Two allocation variants (§III.D):
 *   BRM_UPPER   -- BRMerge-Upper: rows are computed into a temporary C_bar
 *                  sized by n_prod per row (the upper bound),
 *                  then compacted into the final CSR (Step 6).
 *   BRM_PRECISE -- BRMerge-Precise: a symbolic merge (columns only) counts
 *                  nnz per row first, the prefix sum gives rpt, and the
 *                  numeric merge writes rows straight into C.
 *
 * ---------------------------------------------------------------------------
 * Layout (every matrix, host or device):
 *   rpt : int64_t[rows + 1], rpt[0] = 0, non-decreasing, rpt[rows] = nnz
 *   col : int32_t[nnz], strictly increasing inside each row, in [0, cols)
 *   val : double[nnz]
 * Preconditions (not re-checked on the device): A.cols == B.rows; B's rows
 * sorted strictly increasing (Alg. 1 relies on it: "each generated list is
 * naturally sorted since each row of B is sorted"); A's
 * column indices in [0, B.rows). B.cols < 2^31 - 1. No single output row may
 * have n_prod >= 2^31 (BRM_ERR_OVERFLOW).
 * Output: C has rows = A.rows, cols = B.cols, rows sorted strictly
 * increasing; entries that cancel to 0.0 are KEPT (structural nonzeros).
 *
 * Pointers are device pointers unless the function name ends in _host.
 * All device work is enqueued on the context's stream; functions that must
 * return a size to the host (structure, one-call forms) synchronise that
 * stream. Functions return BRM_OK or an error code; on error the context's
 * brm_last_error() string says what failed and the output is undefined.
 * The library never falls back to the CPU.
 * ---------------------------------------------------------------------------
 */
#ifndef BRMERGE_H_
#define BRMERGE_H_

#include <stdint.h>

#if defined(__GNUC__)
#define BRM_API __attribute__((visibility("default")))
#else
#define BRM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BRM_UPPER = 0,   /* BRMerge-Upper (upper-bound allocation)   */
  BRM_PRECISE = 1  /* BRMerge-Precise (symbolic merge first) */
} brm_mode_t;

typedef enum {
  BRM_OK = 0,
  BRM_ERR_INVALID = 1,  /* null pointer, bad mode, cols too large, bad size   */
  BRM_ERR_DIM = 2,      /* A.cols != B.rows                                   */
  BRM_ERR_CUDA = 3,     /* a CUDA runtime error (see brm_last_error)          */
  BRM_ERR_OOM = 4,      /* device or pinned allocation failed                 */
  BRM_ERR_OVERFLOW = 5, /* a row has n_prod >= 2^31 (per-row index space)     */
  BRM_ERR_STATE = 6     /* fill called without a matching structure call      */
} brm_status_t;

typedef struct {
  int64_t rows, cols, nnz;
  int64_t* rpt; /* rows + 1 */
  int32_t* col; /* nnz      */
  double* val;  /* nnz      */
} brm_csr_t;

/* Number of row bins (tiers) the binning pass sorts rows into; see DESIGN.md
 * "Kernels": 0 = empty rows (n_prod == 0), 1 = one thread per row (Alg. 1
 * literally, P <= 8), 2 = one warp per row in registers (P <= 32), 3-6 =
 * shared-memory record tiers (warp, warp, 256 and 512 threads per row),
 * 7 = heavy rows (windowed BRMerge in column windows, in levels of
 * 512-list blocks beyond 512 lists; or the global-memory tier, see
 * brm_set_heavy_route).                                                     */
#define BRM_NUM_BINS 8

typedef struct {
  int64_t rows;                     /* A.rows                                  */
  int64_t nprod_total;              /* sum_i n_prod_i (= nnz(C_hat))           */
  int64_t nprod_max;                /* max_i n_prod_i ("max_row_nprod_C")     */
  int64_t nnz_c;                    /* nnz(C)                                  */
  int64_t bin_rows[BRM_NUM_BINS];   /* rows per bin                            */
  int64_t bin_nprod[BRM_NUM_BINS];  /* n_prod per bin                          */
  int32_t mode;                     /* brm_mode_t of the last call             */
  int32_t timing_enabled;           /* 1 if the fields below are filled        */
  float ms_nprod_scan;              /* n_prod + scan + bin kernels             */
  float ms_symbolic;                /* PRECISE: symbolic merge (all tiers)     */
  float ms_numeric;                 /* numeric merge (all tiers)               */
  float ms_rowsize_scan;            /* row_size scan -> rpt                    */
  float ms_compact;                 /* UPPER: C_bar -> C compaction            */
  float ms_bin_numeric[BRM_NUM_BINS]; /* numeric merge per tier              */
  int64_t launches;                 /* kernels launched by the last structure+fill */
  float ms_hv_plan;                 /* heavy rows of <= 512 lists: window plan (k_hv_plan)  */
  float ms_hv_merge;                /* heavy rows of <= 512 lists: windowed merge (k_hv_merge)  */
  int64_t hv_rows_one;              /* heavy rows merged in one level (<= 512 lists)           */
  int64_t hv_rows_multi;            /* heavy rows merged in levels of 512-list blocks          */
} brm_stats_t;

typedef struct brm_context brm_context_t;

/* Create a context bound to CUDA device `device` and stream `stream`
 * (a cudaStream_t; NULL = the legacy default stream). The context owns a
 * grow-only device workspace (n_prod offsets, bins, row sizes, C_bar,
 * global-tier ping-pong buffers) reused across calls; it is not thread-safe.
 * Errors: BRM_ERR_INVALID (ctx null), BRM_ERR_CUDA (bad device).          */
BRM_API brm_status_t brm_create(brm_context_t** ctx, int device, void* stream);
BRM_API brm_status_t brm_destroy(brm_context_t* ctx);
BRM_API brm_status_t brm_set_stream(brm_context_t* ctx, void* stream);
/* Record per-phase CUDA-event times into brm_stats_t (adds syncs; off by default). */
BRM_API brm_status_t brm_set_timing(brm_context_t* ctx, int enable);
/* Route of the heavy rows (bin 7): BRM_HEAVY_AUTO (0,
 * default): each row is merged in column windows of <= 4096 products in
 * shared memory (k_hv_plan picks the windows, k_hv_merge merges them); a
 * row of more than 512 lists first merges aligned 512-list blocks into a
 * workspace (sub-trees of Algorithm 1's tree) whose results are the next
 * level's lists. BRM_HEAVY_GLOBAL (1): every heavy row runs on the
 * global-memory tier instead (one 1024-thread CTA per row, ping-pong
 * buffers in global memory; testing and comparison). Results are identical,
 * bit for bit. Errors: BRM_ERR_INVALID.                                     */
#define BRM_HEAVY_AUTO 0
#define BRM_HEAVY_GLOBAL 1
BRM_API brm_status_t brm_set_heavy_route(brm_context_t* ctx, int route);
/* Host-buffer form (brmerge_spgemm_host) for A of >= 65,536 rows: row blocks
 * of balanced n_prod whose C is copied back on a copy stream while the next
 * block computes, used when A*B has at least `min_products` intermediate
 * products (default 2^26; 0: always). Smaller products run the one-shot
 * form. Results are identical. Errors: BRM_ERR_INVALID (negative).        */
BRM_API brm_status_t brm_set_host_pipeline(brm_context_t* ctx, int64_t min_products);
/* Multi-GPU write-out over peer memory (the row partition
 * of PAPER.md:281 gives every rank a block of C's rows, Eq. (2) rows being
 * independent). After brm_set_mirrors(ctx, n, col, val), every
 * brmerge_spgemm_fill on this context stores each entry of C -- the column
 * and the value it writes at index i of C->col / C->val -- also at index i of
 * col[p] / val[p] for p < n, so a rank's row block lands in its peers' copies
 * of C by the merge kernels' (UPPER: the compaction kernel's) own stores and
 * no all-gather of col/val follows. col[p] / val[p] are DEVICE pointers that
 * this device can write: peer memory opened through CUDA IPC or enabled with
 * brm_enable_peer_access, normally a peer's whole-C array advanced by this
 * rank's first entry. They are host arrays of n pointers, copied by the
 * call; the memory they name stays owned by the caller and must outlive the
 * fill and the work it enqueues. n = 0 clears. The other forms (one-call,
 * host-buffer) never mirror. The stores are plain global stores: a peer may
 * read them after this stream's work has completed and the ranks have
 * synchronised. Errors: BRM_ERR_INVALID (n outside [0, 7], null pointers). */
#define BRM_MAX_MIRRORS 7
BRM_API brm_status_t brm_set_mirrors(brm_context_t* ctx, int n, int32_t* const* col, double* const* val);
/* Let the context's device write `peer_device`'s memory (cudaDeviceEnablePeerAccess;
 * already enabled is not an error; the context's own device is a no-op).
 * Errors: BRM_ERR_INVALID (no P2P path), BRM_ERR_CUDA.                      */
BRM_API brm_status_t brm_enable_peer_access(brm_context_t* ctx, int peer_device);
/* Last error message of this context (static storage owned by ctx). */
BRM_API const char* brm_last_error(const brm_context_t* ctx);
BRM_API const char* brm_status_string(brm_status_t s);
/* Statistics of the last structure/fill pair (host copy). With timing on,
 * waits for the recorded events (no other synchronisation is added). */
BRM_API brm_status_t brm_get_stats(const brm_context_t* ctx, brm_stats_t* out);

/* --- one-call form (north_star: brmerge_spgemm(A, B, mode, &C)) ----------
 * A, B: device CSR. On success C->rows/cols/nnz are set and C->rpt/col/val
 * are NEW device arrays allocated with cudaMallocAsync on the context
 * stream; the caller owns them and releases them with brm_csr_free().
 * Synchronises the context stream twice (n_prod/bin summary, nnz(C)).     */
BRM_API brm_status_t brmerge_spgemm(brm_context_t* ctx, const brm_csr_t* A, const brm_csr_t* B,
                            brm_mode_t mode, brm_csr_t* C);
BRM_API brm_status_t brm_csr_free(brm_context_t* ctx, brm_csr_t* C);

/* --- two-phase form (caller-owned output) --------------------------------
 * structure: runs Steps 1-5 of Fig. 4a (UPPER: n_prod, scan, bins, numeric
 * merge into C_bar, row_size scan) or Steps 1-4 of Fig. 4b (PRECISE: n_prod,
 * scan, bins, symbolic merge, row_size scan). Writes C's rpt (rows + 1
 * int64, caller-allocated device array) and *c_nnz (host). The context keeps
 * A, B (by pointer: they must stay alive and unchanged) and the plan.
 * fill: C->rpt must be the array structure filled; C->col/val caller-allocated
 * device arrays of *c_nnz entries. UPPER: Step 6 compaction C_bar -> C.
 * PRECISE: Step 5 numeric merge straight into C. Does not synchronise.
 * Errors: BRM_ERR_STATE if fill is not preceded by structure.             */
BRM_API brm_status_t brmerge_spgemm_structure(brm_context_t* ctx, const brm_csr_t* A,
                                      const brm_csr_t* B, brm_mode_t mode,
                                      int64_t* c_rpt, int64_t* c_nnz);
BRM_API brm_status_t brmerge_spgemm_fill(brm_context_t* ctx, brm_csr_t* C);

/* --- host-buffer form (end-to-end) ---------------------------------------
 * A_h, B_h: HOST CSR (pinned memory recommended). Copies A and B to the
 * device (once if A_h and B_h name the same host arrays, as for C = A*A),
 * runs brmerge_spgemm, copies C back. C_h's arrays point into a
 * pinned host buffer owned by the context, valid until the next _host call
 * or brm_destroy (caller must not free them).                            */
BRM_API brm_status_t brmerge_spgemm_host(brm_context_t* ctx, const brm_csr_t* A_h,
                                 const brm_csr_t* B_h, brm_mode_t mode, brm_csr_t* C_h);

/* --- stage entry points (each is one step of the hot path) ---------------
 * n_prod per output row (§II.B.2; Alg. 1 line 1):
 *   nprod[i] = sum_{k in A_i*} (B.rpt[k+1] - B.rpt[k]),  nprod: int64[A.rows]. */
BRM_API brm_status_t brm_row_nprod(brm_context_t* ctx, const brm_csr_t* A, const brm_csr_t* B,
                           int64_t* nprod);
/* Exclusive prefix sum (hand-written single-pass decoupled look-back scan):
 *   out[0] = 0, out[i+1] = out[i] + in[i] for i < n;  out: int64[n + 1].
 * in and out may alias only if in == out + 1 is false (no overlap).      */
BRM_API brm_status_t brm_exclusive_scan_i64(brm_context_t* ctx, const int64_t* in, int64_t* out,
                                    int64_t n);
/* Row partition for p ranks by balanced n_prod (§III.D):
 * nprod_off = exclusive scan of n_prod (rows + 1 entries, device);
 * bounds[g] = first row r with nprod_off[r] * p >= g * nprod_off[rows],
 * bounds[0] = 0, bounds[p] = rows. bounds: int64[p + 1] device.           */
BRM_API brm_status_t brm_partition_rows(brm_context_t* ctx, const int64_t* nprod_off, int64_t rows,
                                int p, int64_t* bounds);

#ifdef __cplusplus
}
#endif
#endif /* BRMERGE_H_ */
