// ks_sell.cu -- sliced-ELL copy of the CSR pattern used by the block-PCG SpMM.
//
// Why: a multi-RHS CSR row kernel issues, per nonzero, one broadcast load of col and one of val next to
// the gather of the orbital row; on sm_100a those broadcast loads cost as many L1 wavefronts and LSU
// issue slots as the gathers themselves (profiles/r01_ncu_summary.md). In SELL-8 with 4-slot groups one
// 16-byte col load and one 32-byte value load serve 4 nonzeros of a row, and the 8 rows of a slice read
// one contiguous 128-byte col line (256-byte value lines) per slot group.
//
// Layout (C = KS_SELL_C = 8 rows per slice, slot groups of 4):
//   slice s = rows 8s .. 8s+7; K_s = 4 ceil(max row length in the slice / 4) slots (>= 4);
//   sell_ptr[s] = sum_{s' < s} 8 K_s' (entries);  entry (row i, slot k) at
//   sell_ptr[i / 8] + (k / 4) * 32 + (i % 8) * 4 + (k % 4).
//   Slot k < len(i) holds CSR entry row_ptr[i] + k (same order, so row sums are accumulated in CSR
//   order); padding slots hold col = i (own row, a valid gather) and value 0.
#include <cub/cub.cuh>

#include "ks_internal.cuh"

namespace {

__global__ void k_sell_count(const int32_t *__restrict__ row_ptr, int64_t n, int64_t n_slices,
                             int32_t *__restrict__ cnt) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n_slices) return;
  int m = 0;
  for (int64_t i = s * KS_SELL_C; i < min((s + 1) * KS_SELL_C, n); i++) m = max(m, row_ptr[i + 1] - row_ptr[i]);
  const int K = max(4, (m + 3) & ~3);
  cnt[s] = KS_SELL_C * K;
}

__global__ void k_sell_fill_col(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col, int64_t n,
                                const int32_t *__restrict__ sell_ptr, int32_t *__restrict__ scol) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t s = i / KS_SELL_C;
  const int32_t b = sell_ptr[s], K = (sell_ptr[s + 1] - b) / KS_SELL_C;
  const int32_t k0 = row_ptr[i], len = row_ptr[i + 1] - k0;
  const int64_t base = b + (i % KS_SELL_C) * 4;
  for (int k = 0; k < K; k++) scol[base + (k >> 2) * (4 * KS_SELL_C) + (k & 3)] = k < len ? col[k0 + k] : (int32_t)i;
}

__global__ void k_sell_fill_val(const int32_t *__restrict__ row_ptr, const double *__restrict__ val, int64_t n,
                                const int32_t *__restrict__ sell_ptr, double *__restrict__ sval) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t s = i / KS_SELL_C;
  const int32_t b = sell_ptr[s], K = (sell_ptr[s + 1] - b) / KS_SELL_C;
  const int32_t k0 = row_ptr[i], len = row_ptr[i + 1] - k0;
  const int64_t base = b + (i % KS_SELL_C) * 4;
  for (int k = 0; k < K; k++) sval[base + (k >> 2) * (4 * KS_SELL_C) + (k & 3)] = k < len ? val[k0 + k] : 0.0;
}

__global__ void k_sell_fill_csr(const int32_t *__restrict__ row_ptr, int64_t n, const int32_t *__restrict__ sell_ptr,
                                int32_t *__restrict__ scsr) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t s = i / KS_SELL_C;
  const int32_t b = sell_ptr[s], K = (sell_ptr[s + 1] - b) / KS_SELL_C;
  const int32_t k0 = row_ptr[i], len = row_ptr[i + 1] - k0;
  const int64_t base = b + (i % KS_SELL_C) * 4;
  for (int k = 0; k < K; k++) scsr[base + (k >> 2) * (4 * KS_SELL_C) + (k & 3)] = k < len ? k0 + k : -1;
}

__global__ void k_inv_diag(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                           const double *__restrict__ val, int64_t n, double *__restrict__ dinv) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int32_t k = row_ptr[i]; k < row_ptr[i + 1]; k++)
    if (col[k] == i) dinv[i] = 1.0 / val[k];
}

}  // namespace

// cnt [n_slices + 1] and cub (cub_bytes) are setup temporaries; total = the plan's entry count (checked)
ks_status ks_sell_build(ks_ctx *ctx, int32_t *cnt, void *cub, size_t cub_bytes, int64_t planned_total) {
  cudaStream_t s = ctx->stream;
  const int64_t n = ctx->n_free;
  const int64_t ns = (n + KS_SELL_C - 1) / KS_SELL_C;
  ctx->n_slices = ns;
  KS_CUDA(ctx, cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (ns + 1), s));
  k_sell_count<<<ks_blocks(ns, 256), 256, 0, s>>>(ctx->row_ptr, n, ns, cnt);
  KS_LAUNCHED(ctx);
  size_t tmp_bytes = cub_bytes;
  KS_CUDA(ctx, cub::DeviceScan::ExclusiveSum(cub, tmp_bytes, cnt, ctx->sell_ptr, (int)(ns + 1), s));
  ctx->launches++;
  int32_t total = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&total, ctx->sell_ptr + ns, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  if (total != planned_total)
    return ks_fail(ctx, KS_E_CUDA, "sliced-ELL entries %d differ from the plan's %lld", total, (long long)planned_total);
  ctx->sell_total = total;
  k_sell_fill_col<<<ks_blocks(n, 256), 256, 0, s>>>(ctx->row_ptr, ctx->col, n, ctx->sell_ptr, ctx->sell_col);
  KS_LAUNCHED(ctx);
  k_sell_fill_val<<<ks_blocks(n, 256), 256, 0, s>>>(ctx->row_ptr, ctx->M, n, ctx->sell_ptr, ctx->sell_M);
  KS_LAUNCHED(ctx);
  k_sell_fill_val<<<ks_blocks(n, 256), 256, 0, s>>>(ctx->row_ptr, ctx->K, n, ctx->sell_ptr, ctx->sell_K);
  KS_LAUNCHED(ctx);
  k_inv_diag<<<ks_blocks(n, 256), 256, 0, s>>>(ctx->row_ptr, ctx->col, ctx->K, n, ctx->dinvK);
  KS_LAUNCHED(ctx);
  k_sell_fill_csr<<<ks_blocks(n, 256), 256, 0, s>>>(ctx->row_ptr, n, ctx->sell_ptr, ctx->sell_csr);
  KS_LAUNCHED(ctx);
  return KS_OK;
}
