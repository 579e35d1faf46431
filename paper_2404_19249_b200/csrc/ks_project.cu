// ks_project.cu -- projection of H and M onto the augmented subspace W = [P | U~]:
//   F_A = [[A_H, b_H], [b_H^T, beta]],  F_B = [[B_H, c_H], [c_H^T, gamma]]                (st1)-(st2)
//   A_H = P^T H P (st5), b_H = P^T H U~ (st6), beta = U~^T H U~ (st7);
//   B_H = P^T M P (cached per mesh pair), c_H = P^T M U~, gamma = U~^T M U~ (717-731).
// Kernels (all deterministic: fixed partitions, fixed summation orders, no float atomics):
//   K8  Y_H = H U~ and Y_M = M U~ in one pass over the shared column stream
//   K8b beta, gamma: tall-skinny Gram products U~^T Y (register-tiled, per-block partials + fixed reduce)
//   K9  b_H, c_H = P^T Y: coarse-major P^T lists, one block per coarse node
//   K10 A_H = P^T (H P): G = H P per fine row on the precomputed pattern of H P, then one block per
//       coarse row accumulating P^T G into per-warp dense rows in shared memory, combined in fixed order.
#include <cub/cub.cuh>

#include "ks_internal.cuh"
#include "ks_rowops.cuh"

namespace {

constexpr int GROW_MAX = 512;  // max entries of a row of H P before dedup (row_len * 4)

__global__ void k_check_P(const int32_t *__restrict__ ptr, const int32_t *__restrict__ col, int64_t n_free,
                          int64_t n_H, int64_t p_nnz, unsigned long long *bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_free) return;
  int32_t a = ptr[i], b = ptr[i + 1];
  bool ok = a >= 0 && b >= a && b - a <= 4 && b <= p_nnz;
  for (int32_t k = a; ok && k < b; k++) ok = col[k] >= 0 && col[k] < n_H;
  if (!ok) atomicMin(bad, (unsigned long long)i);
}

// expand P entries: key = coarse col, value = entry index (stable sort -> ascending fine row)
__global__ void k_P_rows(const int32_t *__restrict__ ptr, int64_t n_free, int32_t *__restrict__ row_of) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_free) return;
  for (int32_t k = ptr[i]; k < ptr[i + 1]; k++) row_of[k] = (int32_t)i;
}

__global__ void k_iota(int32_t *__restrict__ v, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int32_t)i;
}

__global__ void k_PT_fill(const int32_t *__restrict__ order, const int32_t *__restrict__ row_of,
                          const double *__restrict__ Pval, int64_t p_nnz, int32_t *__restrict__ PT_row,
                          double *__restrict__ PT_val) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= p_nnz) return;
  int32_t k = order[j];
  PT_row[j] = row_of[k];
  PT_val[j] = Pval[k];
}

__global__ void k_lower_bound_ptr(const int32_t *__restrict__ keys, int64_t nk, int64_t nrows,
                                  int32_t *__restrict__ ptr) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r > nrows) return;
  int64_t lo = 0, hi = nk;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < (int32_t)r) lo = mid + 1; else hi = mid;
  }
  ptr[r] = (int32_t)lo;
}

// pattern of G = H P: row i = sorted unique coarse columns of the P rows of the columns of row i.
// pass 0 counts, pass 1 fills.
__global__ void k_G_pattern(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                            const int32_t *__restrict__ Pptr, const int32_t *__restrict__ Pcol, int64_t n_free,
                            const int32_t *__restrict__ G_ptr, int32_t *__restrict__ G_cnt,
                            int32_t *__restrict__ G_col, unsigned long long *bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_free) return;
  int32_t buf[GROW_MAX];
  int m = 0;
  for (int32_t k = row_ptr[i]; k < row_ptr[i + 1]; k++) {
    int32_t j = col[k];
    for (int32_t t = Pptr[j]; t < Pptr[j + 1]; t++) {
      if (m >= GROW_MAX) { atomicMin(bad, (unsigned long long)i); return; }
      buf[m++] = Pcol[t];
    }
  }
  // insertion sort + unique
  for (int x = 1; x < m; x++) {
    int32_t v = buf[x];
    int y = x - 1;
    while (y >= 0 && buf[y] > v) { buf[y + 1] = buf[y]; y--; }
    buf[y + 1] = v;
  }
  int u = 0;
  for (int x = 0; x < m; x++)
    if (u == 0 || buf[x] != buf[u - 1]) buf[u++] = buf[x];
  if (G_cnt) G_cnt[i] = u;
  if (G_col) {
    int32_t g0 = G_ptr[i];
    for (int x = 0; x < u; x++) G_col[g0 + x] = buf[x];
  }
}

// G values: half-warp per fine row; lane s owns G slots s, s+16, ...; each slot sums the matching
// (k, t) products in ascending (k, t) order.
__global__ void __launch_bounds__(256) k_G_values(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                                  const double *__restrict__ val, const int32_t *__restrict__ Pptr,
                                                  const int32_t *__restrict__ Pcol, const double *__restrict__ Pval,
                                                  const int32_t *__restrict__ G_ptr, const int32_t *__restrict__ G_col,
                                                  int64_t n_free, double *__restrict__ G_val) {
  int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 4;
  int s = threadIdx.x & 15;
  if (i >= n_free) return;
  const int32_t g0 = G_ptr[i], g1 = G_ptr[i + 1];
  const int32_t k0 = row_ptr[i], k1 = row_ptr[i + 1];
  for (int32_t g = g0 + s; g < g1; g += 16) {
    const int32_t d = G_col[g];
    double acc = 0.0;
    for (int32_t k = k0; k < k1; k++) {
      const int32_t j = __ldg(col + k);
      const double h = __ldg(val + k);
      for (int32_t t = __ldg(Pptr + j); t < __ldg(Pptr + j + 1); t++)
        if (__ldg(Pcol + t) == d) acc = fma(h, __ldg(Pval + t), acc);
    }
    G_val[g] = acc;
  }
}

// out[c][d] (row stride ld) = sum_{j in P^T row c} P^T_val[j] * G[PT_row[j]][d]; RS warps each keep a
// dense row of n_H partial sums in shared memory, combined in warp order.
__global__ void k_PtG(const int32_t *__restrict__ PT_ptr, const int32_t *__restrict__ PT_row,
                      const double *__restrict__ PT_val, const int32_t *__restrict__ G_ptr,
                      const int32_t *__restrict__ G_col, const double *__restrict__ G_val, int64_t n_H,
                      double *__restrict__ out, int64_t ld) {
  extern __shared__ double acc[];  // [RS][n_H]
  const int RS = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = blockIdx.x;
  for (int64_t x = threadIdx.x; x < RS * n_H; x += blockDim.x) acc[x] = 0.0;
  __syncthreads();
  double *mine = acc + warp * n_H;
  for (int32_t j = PT_ptr[c] + warp; j < PT_ptr[c + 1]; j += RS) {
    const int32_t i = __ldg(PT_row + j);
    const double wgt = __ldg(PT_val + j);
    const int32_t g1 = __ldg(G_ptr + i + 1);
    for (int32_t g = __ldg(G_ptr + i) + lane; g < g1; g += 32) {
      const int32_t d = __ldg(G_col + g);
      mine[d] = fma(wgt, __ldg(G_val + g), mine[d]);
    }
    __syncwarp();
  }
  __syncthreads();
  for (int64_t d = threadIdx.x; d < n_H; d += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < RS; w++) s += acc[w * n_H + d];
    out[c * ld + d] = s;
  }
}

// Y_H = H U~, Y_M = M U~ (fast layout, N == NP)
template <int NP>
__global__ void __launch_bounds__(256) k_HM_times(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                                  const double *__restrict__ H, const double *__restrict__ M,
                                                  const double *__restrict__ X, double *__restrict__ YH,
                                                  double *__restrict__ YM, int64_t n) {
  constexpr int VEC = Lay<NP>::VEC, LPR = Lay<NP>::LPR;
  const int64_t gl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t row = gl / LPR;
  const int sub = (int)(gl % LPR);
  if (row >= n) return;
  Vec<VEC> yh, ym;
  row_spmv2<NP>(col, H, M, __ldg(row_ptr + row), __ldg(row_ptr + row + 1), X, sub, yh, ym);
  yh.store(YH + row * NP + sub * VEC);
  ym.store(YM + row * NP + sub * VEC);
}

__global__ void k_HM_times_generic(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                   const double *__restrict__ H, const double *__restrict__ M,
                                   const double *__restrict__ X, double *__restrict__ YH, double *__restrict__ YM,
                                   int64_t n, int N) {
  const int64_t gl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gl >= n * N) return;
  const int64_t row = gl / N;
  const int c = (int)(gl % N);
  double sh = 0.0, sm = 0.0;
  for (int32_t k = row_ptr[row]; k < row_ptr[row + 1]; k++) {
    const double x = X[(int64_t)col[k] * N + c];
    sh = fma(H[k], x, sh);
    sm = fma(M[k], x, sm);
  }
  YH[gl] = sh;
  YM[gl] = sm;
}

// Gram partials: part[blk][m][a][b] = sum over the block's rows of U[i][a] * Y_m[i][b], m in {H, M}.
// Outputs are tiled 4x4 per thread; threads beyond the tiles form row groups (rows r = g mod ngroups).
constexpr int GR_ROWS = 32;
__global__ void __launch_bounds__(256) k_gram(const double *__restrict__ U, const double *__restrict__ YH,
                                              const double *__restrict__ YM, int64_t n, int N, int64_t rows_per_blk,
                                              double *__restrict__ part) {
  extern __shared__ double sm[];
  const int NT = (N + 3) / 4, NQ = NT * 4;
  double *sU = sm, *sH = sm + GR_ROWS * NQ, *sM = sm + 2 * GR_ROWS * NQ;
  double *sRed = sm + 3 * GR_ROWS * NQ;  // [ngroups][2 N N] reduction scratch reuses after loop
  const int ntiles = 2 * NT * NT;
  const int ngroups = max(1, (int)blockDim.x / ntiles);
  const int64_t r0 = blockIdx.x * rows_per_blk;
  const int64_t r1 = min(n, r0 + rows_per_blk);
  double acc[2][16];  // up to 2 tiles per thread when ntiles > blockDim
  for (int z = 0; z < 2; z++)
    for (int k = 0; k < 16; k++) acc[z][k] = 0.0;
  const int my_group = threadIdx.x / ntiles;
  for (int64_t rb = r0; rb < r1; rb += GR_ROWS) {
    const int nr = (int)min((int64_t)GR_ROWS, r1 - rb);
    __syncthreads();
    for (int x = threadIdx.x; x < GR_ROWS * NQ; x += blockDim.x) {
      const int rr = x / NQ, cc = x % NQ;
      const bool in = rr < nr && cc < N;
      const int64_t g = (rb + rr) * N + cc;
      sU[x] = in ? U[g] : 0.0;
      sH[x] = in ? YH[g] : 0.0;
      sM[x] = in ? YM[g] : 0.0;
    }
    __syncthreads();
    for (int z = 0; z < 2; z++) {
      const int tile = (ntiles > (int)blockDim.x) ? threadIdx.x + z * blockDim.x : (z == 0 ? threadIdx.x % ntiles : -1);
      if (tile < 0 || tile >= ntiles) continue;
      if (ntiles <= (int)blockDim.x && my_group >= ngroups) continue;
      const int m = tile / (NT * NT), ta = (tile % (NT * NT)) / NT, tb = tile % NT;
      const double *sY = m ? sM : sH;
      const int rstart = (ntiles <= (int)blockDim.x) ? my_group : 0;
      const int rstep = (ntiles <= (int)blockDim.x) ? ngroups : 1;
      for (int rr = rstart; rr < nr; rr += rstep) {
        double ua[4], yb[4];
#pragma unroll
        for (int k = 0; k < 4; k++) { ua[k] = sU[rr * NQ + ta * 4 + k]; yb[k] = sY[rr * NQ + tb * 4 + k]; }
#pragma unroll
        for (int x = 0; x < 4; x++)
#pragma unroll
          for (int y = 0; y < 4; y++) acc[z][x * 4 + y] = fma(ua[x], yb[y], acc[z][x * 4 + y]);
      }
    }
  }
  __syncthreads();
  // combine row groups in fixed order via shared memory, write 2 N N partial
  const int NN2 = 2 * N * N;
  for (int x = threadIdx.x; x < ngroups * NN2; x += blockDim.x) sRed[x] = 0.0;
  __syncthreads();
  for (int z = 0; z < 2; z++) {
    const int tile = (ntiles > (int)blockDim.x) ? threadIdx.x + z * blockDim.x : (z == 0 ? threadIdx.x % ntiles : -1);
    if (tile < 0 || tile >= ntiles) continue;
    const int grp = (ntiles > (int)blockDim.x) ? 0 : my_group;
    if (grp >= ngroups) continue;
    const int m = tile / (NT * NT), ta = (tile % (NT * NT)) / NT, tb = tile % NT;
    for (int x = 0; x < 4; x++)
      for (int y = 0; y < 4; y++) {
        const int a = ta * 4 + x, b = tb * 4 + y;
        if (a < N && b < N) sRed[grp * NN2 + m * N * N + a * N + b] = acc[z][x * 4 + y];
      }
  }
  __syncthreads();
  for (int x = threadIdx.x; x < NN2; x += blockDim.x) {
    double s = 0.0;
    for (int g = 0; g < ngroups; g++) s += sRed[g * NN2 + x];
    part[(int64_t)blockIdx.x * NN2 + x] = s;
  }
}

// beta / gamma = sum of block partials in block order -> bottom-right blocks of F_A / F_B
__global__ void k_gram_final(const double *__restrict__ part, int nblk, int N, int64_t n_H, int64_t D,
                             double *__restrict__ FA, double *__restrict__ FB) {
  const int NN2 = 2 * N * N;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < NN2; x += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblk; b++) s += part[(int64_t)b * NN2 + x];
    const int m = x / (N * N), a = (x % (N * N)) / N, bb = x % N;
    (m ? FB : FA)[(n_H + a) * D + n_H + bb] = s;
  }
}

// b_H = P^T Y_H, c_H = P^T Y_M: block per coarse node c; thread (rs, a) sums entries j = rs mod RS.
__global__ void k_PtY(const int32_t *__restrict__ PT_ptr, const int32_t *__restrict__ PT_row,
                      const double *__restrict__ PT_val, const double *__restrict__ YH, const double *__restrict__ YM,
                      int N, int64_t n_H, int64_t D, double *__restrict__ FA, double *__restrict__ FB) {
  extern __shared__ double red[];  // [RS][2N]
  const int RS = blockDim.x / N;
  const int rs = threadIdx.x / N, a = threadIdx.x % N;
  const int64_t c = blockIdx.x;
  double sh = 0.0, sm = 0.0;
  if (rs < RS) {
    for (int32_t j = PT_ptr[c] + rs; j < PT_ptr[c + 1]; j += RS) {
      const int64_t i = __ldg(PT_row + j);
      const double w = __ldg(PT_val + j);
      sh = fma(w, YH[i * N + a], sh);
      sm = fma(w, YM[i * N + a], sm);
    }
    red[rs * 2 * N + a] = sh;
    red[rs * 2 * N + N + a] = sm;
  }
  __syncthreads();
  if (threadIdx.x < N) {
    double th = 0.0, tm = 0.0;
    for (int r = 0; r < RS; r++) { th += red[r * 2 * N + a]; tm += red[r * 2 * N + N + a]; }
    FA[c * D + n_H + a] = th;
    FA[(n_H + a) * D + c] = th;
    FB[c * D + n_H + a] = tm;
    FB[(n_H + a) * D + c] = tm;
  }
}

__global__ void k_copy_block(const double *__restrict__ src, int64_t n_H, double *__restrict__ dst, int64_t D) {
  int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= n_H * n_H) return;
  dst[(x / n_H) * D + x % n_H] = src[x];
}

int pow2_at_least(int N) {
  int np = 1;
  while (np < N) np <<= 1;
  return np;
}

ks_status ptg_launch(ks_ctx *ctx, const double *Gv, double *out, int64_t ld) {
  int RS = 4;
  size_t sm = (size_t)RS * ctx->n_H * sizeof(double);
  while (sm > 200 * 1024 && RS > 1) { RS >>= 1; sm = (size_t)RS * ctx->n_H * sizeof(double); }
  if (sm > 200 * 1024) return ks_fail(ctx, KS_E_ARG, "n_H = %lld too large for the dense-row triple product", (long long)ctx->n_H);
  KS_CUDA(ctx, cudaFuncSetAttribute(k_PtG, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_PtG<<<(unsigned)ctx->n_H, 32 * RS, sm, ctx->stream>>>(ctx->PT_ptr, ctx->PT_row, ctx->PT_val, ctx->G_ptr,
                                                          ctx->G_col, Gv, ctx->n_H, out, ld);
  KS_LAUNCHED(ctx);
  return KS_OK;
}

ks_status g_values_launch(ks_ctx *ctx, const double *val) {
  k_G_values<<<ks_blocks(16 * ctx->n_free, 256), 256, 0, ctx->stream>>>(
      ctx->row_ptr, ctx->col, val, ctx->P_ptr, ctx->P_col, ctx->P_val, ctx->G_ptr, ctx->G_col, ctx->n_free,
      ctx->G_val);
  KS_LAUNCHED(ctx);
  return KS_OK;
}

}  // namespace

ks_status ks_set_coarse_impl(ks_ctx *ctx, int64_t n_H, const int32_t *Pptr, const int32_t *Pcol, const double *Pval) {
  cudaStream_t s = ctx->stream;
  const int64_t nf = ctx->n_free;
  // read p_nnz from the row pointer
  int32_t h_pn = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&h_pn, Pptr + nf, 4, cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  const int64_t pn = h_pn;
  if (pn < 0) return ks_fail(ctx, KS_E_ARG, "P row_ptr[n_free] = %lld < 0", (long long)pn);
  // drop a previous coarse space
  for (void **b : {(void **)&ctx->P_ptr, (void **)&ctx->P_col, (void **)&ctx->P_val, (void **)&ctx->PT_ptr,
                   (void **)&ctx->PT_row, (void **)&ctx->PT_val, (void **)&ctx->G_ptr, (void **)&ctx->G_col,
                   (void **)&ctx->G_val, (void **)&ctx->B_H})
    if (*b) { cudaFree(*b); *b = nullptr; }
  ctx->n_H = n_H;
  ctx->p_nnz = pn;
  KS_TRY(ks_alloc_t(ctx, &ctx->P_ptr, nf + 1, "P_ptr"));
  KS_TRY(ks_alloc_t(ctx, &ctx->P_col, pn, "P_col"));
  KS_TRY(ks_alloc_t(ctx, &ctx->P_val, pn, "P_val"));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->P_ptr, Pptr, 4 * (nf + 1), cudaMemcpyDeviceToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->P_col, Pcol, 4 * pn, cudaMemcpyDeviceToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->P_val, Pval, 8 * pn, cudaMemcpyDeviceToDevice, s));

  unsigned long long *bad = nullptr;
  KS_CUDA(ctx, cudaMalloc((void **)&bad, 8));
  struct Guard { void *p; ~Guard() { cudaFree(p); } } gbad{bad};
  KS_CUDA(ctx, cudaMemsetAsync(bad, 0xff, 8, s));
  k_check_P<<<ks_blocks(nf, 256), 256, 0, s>>>(ctx->P_ptr, ctx->P_col, nf, n_H, pn, bad);
  KS_LAUNCHED(ctx);
  unsigned long long h_bad = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&h_bad, bad, 8, cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  if (h_bad != ~0ull)
    return ks_fail(ctx, KS_E_ARG, "P row %llu invalid (more than 4 entries, or column outside [0, n_H))", h_bad);

  // ---- P^T (coarse-major) by a stable sort of the entries on their coarse column ----
  int32_t *row_of, *keys_sorted, *idx, *idx_sorted;
  KS_CUDA(ctx, cudaMalloc((void **)&row_of, 4 * (pn + 1)));
  Guard g1{row_of};
  KS_CUDA(ctx, cudaMalloc((void **)&keys_sorted, 4 * (pn + 1)));
  Guard g2{keys_sorted};
  KS_CUDA(ctx, cudaMalloc((void **)&idx, 4 * (pn + 1)));
  Guard g3{idx};
  KS_CUDA(ctx, cudaMalloc((void **)&idx_sorted, 4 * (pn + 1)));
  Guard g4{idx_sorted};
  k_P_rows<<<ks_blocks(nf, 256), 256, 0, s>>>(ctx->P_ptr, nf, row_of);
  KS_LAUNCHED(ctx);
  k_iota<<<ks_blocks(pn, 256), 256, 0, s>>>(idx, pn);
  KS_LAUNCHED(ctx);
  size_t tb = 0;
  int end_bit = 1;
  while ((1ll << end_bit) <= n_H) end_bit++;
  KS_CUDA(ctx, cub::DeviceRadixSort::SortPairs(nullptr, tb, ctx->P_col, keys_sorted, idx, idx_sorted, (int)pn, 0,
                                               end_bit, s));
  void *tmp;
  KS_CUDA(ctx, cudaMalloc(&tmp, tb ? tb : 1));
  Guard g5{tmp};
  KS_CUDA(ctx, cub::DeviceRadixSort::SortPairs(tmp, tb, ctx->P_col, keys_sorted, idx, idx_sorted, (int)pn, 0,
                                               end_bit, s));
  ctx->launches++;
  KS_TRY(ks_alloc_t(ctx, &ctx->PT_ptr, n_H + 1, "PT_ptr"));
  KS_TRY(ks_alloc_t(ctx, &ctx->PT_row, pn, "PT_row"));
  KS_TRY(ks_alloc_t(ctx, &ctx->PT_val, pn, "PT_val"));
  k_lower_bound_ptr<<<ks_blocks(n_H + 1, 256), 256, 0, s>>>(keys_sorted, pn, n_H, ctx->PT_ptr);
  KS_LAUNCHED(ctx);
  k_PT_fill<<<ks_blocks(pn, 256), 256, 0, s>>>(idx_sorted, row_of, ctx->P_val, pn, ctx->PT_row, ctx->PT_val);
  KS_LAUNCHED(ctx);

  // ---- pattern of G = H P ----
  int32_t *cnt;
  KS_CUDA(ctx, cudaMalloc((void **)&cnt, 4 * (nf + 1)));
  Guard g6{cnt};
  KS_CUDA(ctx, cudaMemsetAsync(bad, 0xff, 8, s));
  k_G_pattern<<<ks_blocks(nf, 128), 128, 0, s>>>(ctx->row_ptr, ctx->col, ctx->P_ptr, ctx->P_col, nf, nullptr, cnt,
                                                 nullptr, bad);
  KS_LAUNCHED(ctx);
  KS_TRY(ks_alloc_t(ctx, &ctx->G_ptr, nf + 1, "G_ptr"));
  KS_CUDA(ctx, cudaMemsetAsync(cnt + nf, 0, 4, s));
  size_t tb2 = 0;
  KS_CUDA(ctx, cub::DeviceScan::ExclusiveSum(nullptr, tb2, cnt, ctx->G_ptr, (int)(nf + 1), s));
  void *tmp2;
  KS_CUDA(ctx, cudaMalloc(&tmp2, tb2 ? tb2 : 1));
  Guard g7{tmp2};
  KS_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp2, tb2, cnt, ctx->G_ptr, (int)(nf + 1), s));
  ctx->launches++;
  int32_t h_g = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&h_g, ctx->G_ptr + nf, 4, cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaMemcpyAsync(&h_bad, bad, 8, cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  if (h_bad != ~0ull) return ks_fail(ctx, KS_E_ARG, "row %llu of H P has more than %d entries", h_bad, GROW_MAX);
  ctx->g_nnz = h_g;
  KS_TRY(ks_alloc_t(ctx, &ctx->G_col, h_g, "G_col"));
  KS_TRY(ks_alloc_t(ctx, &ctx->G_val, h_g, "G_val"));
  k_G_pattern<<<ks_blocks(nf, 128), 128, 0, s>>>(ctx->row_ptr, ctx->col, ctx->P_ptr, ctx->P_col, nf, ctx->G_ptr,
                                                 nullptr, ctx->G_col, bad);
  KS_LAUNCHED(ctx);

  // ---- cached B_H = P^T M P ----
  KS_TRY(ks_alloc_t(ctx, &ctx->B_H, n_H * n_H, "B_H"));
  KS_TRY(g_values_launch(ctx, ctx->M));
  KS_TRY(ptg_launch(ctx, ctx->G_val, ctx->B_H, n_H));
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  return KS_OK;
}

ks_status ks_project_impl(ks_ctx *ctx, int N, const double *Ut, double *FA, double *FB) {
  cudaStream_t s = ctx->stream;
  const int64_t n = ctx->n_free, nH = ctx->n_H, D = nH + N;
  if (ctx->y_cap < n * N) {
    if (ctx->Y_H) { cudaFree(ctx->Y_H); ctx->Y_H = nullptr; }
    if (ctx->Y_M) { cudaFree(ctx->Y_M); ctx->Y_M = nullptr; }
    KS_TRY(ks_alloc_t(ctx, &ctx->Y_H, n * N, "Y_H"));
    KS_TRY(ks_alloc_t(ctx, &ctx->Y_M, n * N, "Y_M"));
    ctx->y_cap = n * N;
  }
  // K8: Y_H = H U~, Y_M = M U~
  const bool fast = pow2_at_least(N) == N && ((uintptr_t)Ut & 15) == 0;
  if (fast) {
    switch (N) {
#define KS_HM(NPV)                                                                                              \
  case NPV:                                                                                                     \
    k_HM_times<NPV><<<ks_blocks(n * Lay<NPV>::LPR, 256), 256, 0, s>>>(ctx->row_ptr, ctx->col, ctx->H, ctx->M, Ut, \
                                                                      ctx->Y_H, ctx->Y_M, n);                    \
    break;
      KS_HM(1) KS_HM(2) KS_HM(4) KS_HM(8) KS_HM(16) KS_HM(32) KS_HM(64)
#undef KS_HM
    }
  } else {
    k_HM_times_generic<<<ks_blocks(n * N, 256), 256, 0, s>>>(ctx->row_ptr, ctx->col, ctx->H, ctx->M, Ut, ctx->Y_H,
                                                             ctx->Y_M, n, N);
  }
  KS_LAUNCHED(ctx);

  // K8b: beta, gamma
  const int nblk = 2 * ctx->sm_count;
  const int64_t rows_per_blk = ((n + nblk - 1) / nblk + GR_ROWS - 1) / GR_ROWS * GR_ROWS;
  const int nb = (int)((n + rows_per_blk - 1) / rows_per_blk);
  const int64_t need = (int64_t)nb * 2 * N * N;
  if (ctx->gram_cap < need) {
    if (ctx->gram_part) { cudaFree(ctx->gram_part); ctx->gram_part = nullptr; }
    KS_TRY(ks_alloc_t(ctx, &ctx->gram_part, need, "gram partials"));
    ctx->gram_cap = need;
  }
  {
    const int NQ = (N + 3) / 4 * 4, NT = NQ / 4;
    const int ntiles = 2 * NT * NT;
    const int ngroups = ntiles >= 256 ? 1 : 256 / ntiles;
    const size_t sm = sizeof(double) * (3 * GR_ROWS * NQ + (size_t)ngroups * 2 * N * N);
    if (ntiles > 512) return ks_fail(ctx, KS_E_ARG, "N=%d too large for the Gram kernel", N);
    KS_CUDA(ctx, cudaFuncSetAttribute(k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_gram<<<nb, 256, sm, s>>>(Ut, ctx->Y_H, ctx->Y_M, n, N, rows_per_blk, ctx->gram_part);
    KS_LAUNCHED(ctx);
    k_gram_final<<<ks_blocks(2 * N * N, 128), 128, 0, s>>>(ctx->gram_part, nb, N, nH, D, FA, FB);
    KS_LAUNCHED(ctx);
  }

  // K9: b_H, c_H
  {
    const int T = N * (256 / N >= 1 ? 256 / N : 1);
    k_PtY<<<(unsigned)nH, T, sizeof(double) * 2 * T, s>>>(ctx->PT_ptr, ctx->PT_row, ctx->PT_val, ctx->Y_H, ctx->Y_M,
                                                          N, nH, D, FA, FB);
    KS_LAUNCHED(ctx);
  }

  // K10: A_H = P^T (H P) into F_A, cached B_H into F_B
  KS_TRY(g_values_launch(ctx, ctx->H));
  KS_TRY(ptg_launch(ctx, ctx->G_val, FA, D));
  k_copy_block<<<ks_blocks(nH * nH, 256), 256, 0, s>>>(ctx->B_H, nH, FB, D);
  KS_LAUNCHED(ctx);
  return KS_OK;
}
