// ks_outer.cu -- NEXT-1: close the linear Algorithm-3 loop.
//   ks_pencil_eig       lowest k eigenpairs of F_A y = lambda F_B y, the "small-scale algebraic eigenvalue
//                       problem" on W (Nonlinear_Eig_Hh); dense, D = n_H + N
//                       <= ~1400, by the cuSOLVER generalized symmetric eigensolver (a plain library call,
//                       like cuBLAS for a plain GEMM): Cholesky of F_B, tridiagonal reduction, and only the
//                       lowest k eigenpairs (index range, dsygvdx).
//   ks_lift             U_new = P y_H + U~ y_t (the new orbitals in S_H + span{psi~}), own kernel.
//   ks_augmented_solve  outer iterations with a fixed potential: block solve -> projection -> pencil
//                       eig -> lift, until max |lambda_new - lambda| <= tol_eig * max |lambda|.
#include <cusolverDn.h>

#include <algorithm>

#include "ks_internal.cuh"
#include "ks_sell.cuh"

namespace {

// eigenvectors: cuSOLVER leaves them column-major in A (column j = eigenvector j); out [D][k] row-major
__global__ void k_take_evecs(const double *__restrict__ A, int64_t D, int k, double *__restrict__ out) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= D * k) return;
  const int64_t i = x / k, j = x % k;
  out[x] = A[j * D + i];
}

// U_new[i][j] = sum_t P_it Y[col_t][j] + sum_m U~[i][m] Y[n_H + m][j]; one thread per (row, output column)
// U_new = P y_H + U~ y_t (the lift of the Ritz vectors). One warp per 8 rows: the dense
// part U~[8 rows][N] x y_t[N][k] on the FP64 tensor cores (mma.m8n8k4.f64, k-steps of 4 orbitals; A[m = row]
// [k = orbital] from global, B = y_t staged in shared memory per block), then the <= 4 coarse parents of
// each row added from y_H in the epilogue (fragment C[m = lane/4][n = 2(lane%4) + v]). Ragged N and k are
// masked by select.
constexpr int LIFT_WARPS = 8;
// row stride of the staged y_t: S = 4 (mod 16) doubles, so the B-fragment loads of a half-warp (rows tig,
// columns grp: addresses tig*S + grp) hit 16 distinct 8-byte bank pairs (K8 = 32 would be 4-way conflicted)
__host__ __device__ inline int lift_stride(int k) {
  const int K8 = (k + 7) & ~7;
  return K8 + ((4 - K8) % 16 + 16) % 16;
}
__global__ void __launch_bounds__(LIFT_WARPS * 32) k_lift(const int32_t *__restrict__ Pptr,
                                                          const int32_t *__restrict__ Pcol,
                                                          const double *__restrict__ Pval,
                                                          const double *__restrict__ Ut, int N, int ldu,
                                                          const double *__restrict__ Y, int k, int64_t n_H, int64_t n,
                                                          double *__restrict__ Unew, int ldo) {
  extern __shared__ double yt[];   // [N4][S] zero-padded y_t
  const int N4 = (N + 3) & ~3, K8 = (k + 7) & ~7, S = lift_stride(k);
  for (int x = threadIdx.x; x < N4 * S; x += blockDim.x) {
    const int m = x / S, j = x % S;
    yt[x] = (m < N && j < k) ? __ldg(Y + (n_H + m) * k + j) : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, grp = lane >> 2, tig = lane & 3;
  const int64_t ntile = (n + 7) / 8;     // 8-row warp tiles, strided over the (persistent) grid
  for (int64_t tile = (int64_t)blockIdx.x * LIFT_WARPS + (threadIdx.x >> 5); tile < ntile;
       tile += (int64_t)gridDim.x * LIFT_WARPS) {
  const int64_t i = tile * 8 + grp;      // this lane's row (A fragments and outputs)
  const bool rv = i < n;
  // the row's coarse parents (<= 4), loaded ahead of the MMA loop so their latency overlaps it
  int32_t pc[4] = {0, 0, 0, 0};
  double pw[4] = {0.0, 0.0, 0.0, 0.0};
  int np = 0;
  if (rv) {
    const int32_t p0 = __ldg(Pptr + i);
    np = min(__ldg(Pptr + i + 1) - p0, 4);
#pragma unroll
    for (int q = 0; q < 4; q++)
      if (q < np) {
        pc[q] = __ldg(Pcol + p0 + q);
        pw[q] = __ldg(Pval + p0 + q);
      }
  }
  for (int t0 = 0; t0 < K8; t0 += 32) {  // up to 4 column tiles of 8 per pass
    double c[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    for (int k0 = 0; k0 < N4; k0 += 16) {  // 4 k-steps per batch: independent A loads in flight
      double a[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int m = k0 + 4 * u + tig;
        a[u] = (rv && m < N) ? __ldg(Ut + i * ldu + m) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int m = k0 + 4 * u + tig;
        if (k0 + 4 * u >= N4) break;
#pragma unroll
        for (int t = 0; t < 4; t++) {
          if (t0 + 8 * t >= K8) break;
          const double b = yt[m * S + t0 + 8 * t + grp];
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a[u]), "d"(b));
        }
      }
    }
    if (rv) {
#pragma unroll
      for (int q = 0; q < 4; q++) {
        if (q >= np) break;
        const double *yh = Y + (int64_t)pc[q] * k;
#pragma unroll
        for (int t = 0; t < 4; t++) {
          const int j = t0 + 8 * t + 2 * tig;
          if (j < k) c[t][0] = fma(pw[q], __ldg(yh + j), c[t][0]);
          if (j + 1 < k) c[t][1] = fma(pw[q], __ldg(yh + j + 1), c[t][1]);
        }
      }
#pragma unroll
      for (int t = 0; t < 4; t++) {
        const int j = t0 + 8 * t + 2 * tig;
        if (j < k) Unew[i * ldo + j] = c[t][0];
        if (j + 1 < k) Unew[i * ldo + j + 1] = c[t][1];
      }
    }
  }
  }
}

}  // namespace

static ks_status ensure_solver_handle(ks_ctx *ctx) {
  if (!ctx->cusolver) {
    cusolverDnHandle_t h = nullptr;
    if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS) return ks_fail(ctx, KS_E_CUDA, "cusolverDnCreate failed");
    ctx->cusolver = h;
  }
  if (cusolverDnSetStream((cusolverDnHandle_t)ctx->cusolver, ctx->stream) != CUSOLVER_STATUS_SUCCESS)
    return ks_fail(ctx, KS_E_CUDA, "cusolverDnSetStream failed");
  return KS_OK;
}

void ks_free_outer(ks_ctx *ctx) {
  if (ctx->cusolver) cusolverDnDestroy((cusolverDnHandle_t)ctx->cusolver);
  ctx->cusolver = nullptr;
}

__global__ void k_mirror_lower(double *A, int64_t n) {   // column-major lower -> full symmetric
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= n * n) return;
  const int64_t i = x % n, j = x / n;   // A(i, j) = A[i + j n]
  if (i < j) A[i + j * n] = A[j + i * n];
}

// A <- A^-1 for a symmetric positive definite [n][n] (Cholesky: potrf + potri, then mirrored); *spd = false
// (A left unusable) when the factorisation finds a non-positive pivot.
ks_status ks_spd_inverse(ks_ctx *ctx, double *A, int64_t n, bool *spd) {
  KS_TRY(ensure_solver_handle(ctx));
  cusolverDnHandle_t h = (cusolverDnHandle_t)ctx->cusolver;
  int lw1 = 0, lw2 = 0;
  if (cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, (int)n, A, (int)n, &lw1) != CUSOLVER_STATUS_SUCCESS ||
      cusolverDnDpotri_bufferSize(h, CUBLAS_FILL_MODE_LOWER, (int)n, A, (int)n, &lw2) != CUSOLVER_STATUS_SUCCESS)
    return ks_fail(ctx, KS_E_CUDA, "potrf/potri bufferSize failed");
  const int lw = lw1 > lw2 ? lw1 : lw2;
  double *work = nullptr;
  int *info = nullptr;
  KS_CUDA(ctx, cudaMallocAsync((void **)&work, sizeof(double) * (size_t)(lw > 0 ? lw : 1), ctx->stream));
  KS_CUDA(ctx, cudaMallocAsync((void **)&info, sizeof(int), ctx->stream));
  int hinfo = 0;
  bool ok = cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, (int)n, A, (int)n, work, lw, info) == CUSOLVER_STATUS_SUCCESS;
  if (ok) {
    KS_CUDA(ctx, cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    ok = hinfo == 0;
  }
  if (ok) {
    ok = cusolverDnDpotri(h, CUBLAS_FILL_MODE_LOWER, (int)n, A, (int)n, work, lw, info) == CUSOLVER_STATUS_SUCCESS;
    if (ok) {
      KS_CUDA(ctx, cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
      ok = hinfo == 0;
    }
  }
  KS_CUDA(ctx, cudaFreeAsync(work, ctx->stream));
  KS_CUDA(ctx, cudaFreeAsync(info, ctx->stream));
  if (ok) {
    k_mirror_lower<<<ks_blocks(n * n, 256), 256, 0, ctx->stream>>>(A, n);
    KS_LAUNCHED(ctx);
  }
  *spd = ok;
  return KS_OK;
}

ks_status ks_pencil_eig_impl(ks_ctx *ctx, int64_t D, int k, const double *FA, const double *FB, double *evals,
                             double *evecs) {
  KS_TRY(ensure_solver_handle(ctx));
  cusolverDnHandle_t h = (cusolverDnHandle_t)ctx->cusolver;
  if (ctx->eig_cap < D) {
    ks_free_t(ctx, ctx->eig_A);
    ks_free_t(ctx, ctx->eig_B);
    ks_free_t(ctx, ctx->eig_w);
    KS_TRY(ks_alloc_t(ctx, &ctx->eig_A, D * D, "pencil A"));
    KS_TRY(ks_alloc_t(ctx, &ctx->eig_B, D * D, "pencil B"));
    KS_TRY(ks_alloc_t(ctx, &ctx->eig_w, D, "pencil eigenvalues"));
    ctx->eig_cap = D;
  }
  // symmetric matrices: row-major == column-major
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->eig_A, FA, sizeof(double) * D * D, cudaMemcpyDeviceToDevice, ctx->stream));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->eig_B, FB, sizeof(double) * D * D, cudaMemcpyDeviceToDevice, ctx->stream));
  // only the lowest k eigenpairs are needed: the index-range solver (bisection + inverse iteration on the
  // tridiagonal form, k back-transformed vectors) instead of all D (KS_PENCIL_ALL=1 selects dsygvd)
  const char *all = getenv("KS_PENCIL_ALL");
  const bool subset = !(all && all[0] == '1') && k < D;
  int lwork = 0, meig = 0;
  if (subset) {
    if (cusolverDnDsygvdx_bufferSize(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I,
                                     CUBLAS_FILL_MODE_LOWER, (int)D, ctx->eig_A, (int)D, ctx->eig_B, (int)D, 0.0, 0.0,
                                     1, k, &meig, ctx->eig_w, &lwork) != CUSOLVER_STATUS_SUCCESS)
      return ks_fail(ctx, KS_E_CUDA, "cusolverDnDsygvdx_bufferSize failed (D = %lld)", (long long)D);
  } else if (cusolverDnDsygvd_bufferSize(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                         (int)D, ctx->eig_A, (int)D, ctx->eig_B, (int)D, ctx->eig_w, &lwork) !=
             CUSOLVER_STATUS_SUCCESS)
    return ks_fail(ctx, KS_E_CUDA, "cusolverDnDsygvd_bufferSize failed (D = %lld)", (long long)D);
  if (ctx->eig_work_cap < lwork) {
    ks_free_t(ctx, ctx->eig_work);
    KS_TRY(ks_alloc_t(ctx, &ctx->eig_work, lwork, "pencil workspace"));
    ctx->eig_work_cap = lwork;
  }
  if (!ctx->eig_info) KS_TRY(ks_alloc_t(ctx, &ctx->eig_info, 1, "pencil info"));
  cusolverStatus_t cst;
  if (subset)
    cst = cusolverDnDsygvdx(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I,
                            CUBLAS_FILL_MODE_LOWER, (int)D, ctx->eig_A, (int)D, ctx->eig_B, (int)D, 0.0, 0.0, 1, k,
                            &meig, ctx->eig_w, ctx->eig_work, lwork, ctx->eig_info);
  else
    cst = cusolverDnDsygvd(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)D, ctx->eig_A,
                           (int)D, ctx->eig_B, (int)D, ctx->eig_w, ctx->eig_work, lwork, ctx->eig_info);
  if (cst != CUSOLVER_STATUS_SUCCESS)
    return ks_fail(ctx, KS_E_CUDA, "cusolver generalized eigensolver failed (D = %lld, status %d)", (long long)D,
                   (int)cst);
  ctx->launches++;
  int info = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&info, ctx->eig_info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (info > D)
    return ks_fail(ctx, KS_E_RANK, "F_B is not positive definite (leading minor %d): W = [P | U~] is rank deficient",
                   info - (int)D);
  if (info != 0) return ks_fail(ctx, KS_E_NONFINITE, "pencil eigensolver did not converge (info %d)", info);
  KS_CUDA(ctx, cudaMemcpyAsync(evals, ctx->eig_w, sizeof(double) * k, cudaMemcpyDeviceToDevice, ctx->stream));
  k_take_evecs<<<ks_blocks(D * k, 256), 256, 0, ctx->stream>>>(ctx->eig_A, D, k, evecs);
  KS_LAUNCHED(ctx);
  return KS_OK;
}

ks_status ks_lift_impl(ks_ctx *ctx, int N, const double *Ut, int k, const double *Y, double *Unew) {
  const int64_t n = ctx->n_free;
  const size_t sm = sizeof(double) * (size_t)((N + 3) & ~3) * lift_stride(k);
  if (sm > 200 * 1024) return ks_fail(ctx, KS_E_ARG, "lift: N = %d, k = %d too large for the staged y_t", N, k);
  if (sm > 48 * 1024) KS_CUDA(ctx, cudaFuncSetAttribute(k_lift, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_lift<<<(unsigned)std::min<int64_t>(ks_blocks(n, 8 * LIFT_WARPS), 8 * (int64_t)ctx->sm_count), LIFT_WARPS * 32, sm,
           ctx->stream>>>(ctx->P_ptr, ctx->P_col, ctx->P_val, Ut, N, N,
                                                                              Y, k, ctx->n_H, n, Unew, k);
  KS_LAUNCHED(ctx);
  return KS_OK;
}

ks_status ks_augmented_solve_impl(ks_ctx *ctx, int N, double *lambda, double *U, double tol_eig, int max_outer,
                                  double tol_bvp, int32_t max_iter_bvp, int32_t *h_outer, double *h_history) {
  const int64_t n = ctx->n_free, D = ctx->n_H + N;
  if (ctx->outer_cap < n * N || ctx->outer_D < D) {
    ks_free_t(ctx, ctx->outer_Ut);
    ks_free_t(ctx, ctx->outer_FA);
    ks_free_t(ctx, ctx->outer_FB);
    ks_free_t(ctx, ctx->outer_Y);
    ks_free_t(ctx, ctx->outer_lam);
    KS_TRY(ks_alloc_t(ctx, &ctx->outer_Ut, n * N, "outer U~"));
    KS_TRY(ks_alloc_t(ctx, &ctx->outer_FA, D * D, "outer F_A"));
    KS_TRY(ks_alloc_t(ctx, &ctx->outer_FB, D * D, "outer F_B"));
    KS_TRY(ks_alloc_t(ctx, &ctx->outer_Y, D * N, "outer Y"));
    KS_TRY(ks_alloc_t(ctx, &ctx->outer_lam, N, "outer lambda"));
    ctx->outer_cap = n * N;
    ctx->outer_D = D;
  }
  std::vector<double> prev(N), cur(N);
  KS_CUDA(ctx, cudaMemcpyAsync(prev.data(), lambda, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx->stream));
  KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  int it = 0;
  ks_status result = KS_E_NOT_CONVERGED;
  while (it < max_outer) {
    KS_TRY(ks_solve_impl(ctx, N, lambda, U, ctx->outer_Ut, tol_bvp, max_iter_bvp, nullptr, nullptr));
    KS_TRY(ks_project_impl(ctx, N, ctx->outer_Ut, ctx->outer_FA, ctx->outer_FB));
    KS_TRY(ks_pencil_eig_impl(ctx, D, N, ctx->outer_FA, ctx->outer_FB, ctx->outer_lam, ctx->outer_Y));
    KS_TRY(ks_lift_impl(ctx, N, ctx->outer_Ut, N, ctx->outer_Y, U));
    KS_CUDA(ctx, cudaMemcpyAsync(lambda, ctx->outer_lam, sizeof(double) * N, cudaMemcpyDeviceToDevice, ctx->stream));
    KS_CUDA(ctx, cudaMemcpyAsync(cur.data(), ctx->outer_lam, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx->stream));
    KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    double dmax = 0.0, lmax = 0.0;
    for (int j = 0; j < N; j++) {
      dmax = fmax(dmax, fabs(cur[j] - prev[j]));
      lmax = fmax(lmax, fabs(cur[j]));
      if (h_history) h_history[(int64_t)it * N + j] = cur[j];
    }
    it++;
    prev = cur;
    if (!(dmax == dmax)) { result = KS_E_NONFINITE; break; }
    if (dmax <= tol_eig * lmax) { result = KS_OK; break; }
  }
  if (h_outer) *h_outer = it;
  if (result != KS_OK)
    return ks_fail(ctx, result, "ks_augmented_solve: %d outer iterations without reaching tol %g", it, tol_eig);
  return KS_OK;
}
