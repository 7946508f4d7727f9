// kernels.cuh -- host-side launchers of kernels.cu (internal to libbrmerge).
#pragma once
#include <cuda_runtime.h>

#include "brm_internal.cuh"
#include "engine.cuh"

namespace brm {

// Device-side summary written by the n_prod/scan pass (read back once).
struct DevSummary {
  long long nprod_total;
  unsigned long long nprod_max;
  unsigned long long nl_max;
  unsigned long long bin_rows[BRM_NUM_BINS];
  unsigned long long bin_nprod[BRM_NUM_BINS];
  long long nnz_c;
};

int64_t scan_tiles(int64_t n);
int64_t nprod_tiles(int64_t M);
// rows of A with more than kLongRow nonzeros: listed (list, *count) and their
// n_prod summed into long_np[row] by a CTA each; run before the two below
cudaError_t launch_long_rows(const CsrView& A, const int64_t* brpt, int64_t M, int32_t* list, unsigned int* count,
                             int64_t* long_np, cudaStream_t st);
cudaError_t launch_nprod_scan(const CsrView& A, const int64_t* brpt, int64_t M, int64_t* nprod_off,
                              unsigned long long* status, unsigned int* counter, DevSummary* summary,
                              const int64_t* long_np, cudaStream_t st);
cudaError_t launch_scan_i64(const int64_t* in, int64_t n, int64_t* out, unsigned long long* status,
                            unsigned int* counter, int64_t* total_out, cudaStream_t st);
cudaError_t launch_bin_scatter(const CsrView& A, const int64_t* nprod_off, int64_t M, const DevSummary* summary,
                               unsigned long long* cursor, int32_t* bins, int64_t* row_size, cudaStream_t st);
cudaError_t launch_heavy_info(const CsrView& A, const int64_t* nprod_off, const int32_t* rows, int64_t n,
                              int64_t* info, cudaStream_t st);
// b_cols = B's column count (numeric record tiers pack {col, slot} into 32
// bits when the columns fit)
cudaError_t launch_tier(int bin, int out_kind, const CsrView& A, const CsrView& B, int64_t b_cols, const int32_t* rows,
                        int64_t n, const RowOut& o, cudaStream_t st);
int64_t global_row_bytes(int64_t nprod, int64_t nl, bool vals);
cudaError_t launch_global_tier(int out_kind, const CsrView& A, const CsrView& B, const int32_t* rows, int64_t n,
                               const int64_t* ws_off, unsigned char* ws, const RowOut& o, cudaStream_t st);
cudaError_t launch_compact(int64_t M, int64_t nnz, const int64_t* nprod_off, const int64_t* crpt, const int32_t* cbar_col,
                           const double* cbar_val, int32_t* ccol, double* cval, const Mirrors& mir, cudaStream_t st);
cudaError_t launch_partition(const int64_t* nprod_off, int64_t M, int p, int64_t* bounds, cudaStream_t st);
cudaError_t launch_row_nprod(const CsrView& A, const int64_t* brpt, int64_t M, int64_t* nprod, const int64_t* long_np,
                             cudaStream_t st);
// device -> pinned (host-mapped) memory copy by `ctas` CTAs of the SMs
cudaError_t launch_copy_to_host(void* dst, const void* src, int64_t bytes, int ctas, cudaStream_t st);

}  // namespace brm
