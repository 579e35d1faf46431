// ks_outer.cu -- NEXT-1: close the linear Algorithm-3 loop.
//   ks_pencil_eig       lowest k eigenpairs of F_A y = lambda F_B y, the "small-scale algebraic eigenvalue
//                       problem" on W (Nonlinear_Eig_Hh), D = n_H + N <= ~1400.
//                       Default: reduction to standard form (with the coarse block's Cholesky factor cached per
//                       coarse space, coarse_chol_reduction) and a Chebyshev-filtered subspace iteration on
//                       k + 8 vectors (pencil_eig_filtered: k_sym_gemm, k_gram_pair, k_rotate_resid, the m x m
//                       eigenproblems on the host). Fallback, and KS_PENCIL_DENSE=1: the dense cuSOLVER
//                       generalized symmetric eigensolver (lowest k by index range, dsygvdx).
//   ks_lift             U_new = P y_H + U~ y_t (the new orbitals in S_H + span{psi~}), own kernel (FP64 MMA).
//   ks_augmented_solve  outer iterations with a fixed potential: block solve -> projection -> pencil
//                       eig -> lift, until max |lambda_new - lambda| <= tol_eig * max |lambda|.
#include <cusolverDn.h>

#include <algorithm>

#include <cublas_v2.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <vector>

#include "ks_internal.cuh"
#include "ks_layout.cuh"
#include "ks_sell.cuh"

namespace {

// eigenvectors: cuSOLVER leaves them column-major in A (column j = eigenvector j); out [D][k] row-major
__global__ void k_take_evecs(const double *__restrict__ A, int64_t D, int k, double *__restrict__ out) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= D * k) return;
  const int64_t i = x / k, j = x % k;
  out[x] = A[j * D + i];
}

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
  if (ctx->cublas) cublasDestroy((cublasHandle_t)ctx->cublas);
  ctx->cublas = nullptr;
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
  if (lw > ctx->ext_lwork) return ks_fail(ctx, KS_E_WORKSPACE, "Cholesky workspace %d exceeds the ext plan", lw);
  double *work = ctx->eig_work;
  int *info = ctx->eig_info;
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
  if (ok) {
    k_mirror_lower<<<ks_blocks(n * n, 256), 256, 0, ctx->stream>>>(A, n);
    KS_LAUNCHED(ctx);
  }
  *spd = ok;
  return KS_OK;
}

// cuSOLVER workspace (doubles) of the pencil routes for dimension D (k = 1..D) and of the Cholesky inverse of
// the n_H x n_H coarse stiffness (two-level Hartree solve)
ks_status ks_cusolver_lwork(ks_ctx *ctx, int64_t D, int64_t nH, int64_t *lwork) {
  KS_TRY(ensure_solver_handle(ctx));
  cusolverDnHandle_t h = (cusolverDnHandle_t)ctx->cusolver;
  int lw = 1, x = 0, meig = 0;
  double *p = nullptr, *w = nullptr;
  auto mx = [&](cusolverStatus_t st) {
    if (st != CUSOLVER_STATUS_SUCCESS) return false;
    lw = lw > x ? lw : x;
    return true;
  };
  const int d = (int)D;
  bool ok = mx(cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, d, p, d, &x)) &&
            mx(cusolverDnDsygvd_bufferSize(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, d,
                                           p, d, p, d, w, &x));
  for (int k : {1, d}) {
    ok = ok && mx(cusolverDnDsygvdx_bufferSize(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I,
                                               CUBLAS_FILL_MODE_LOWER, d, p, d, p, d, 0.0, 0.0, 1, k, &meig, w, &x));
  }
  if (nH > 0) {
    const int c = (int)nH;
    ok = ok && mx(cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, c, p, c, &x)) &&
         mx(cusolverDnDpotri_bufferSize(h, CUBLAS_FILL_MODE_LOWER, c, p, c, &x));
  }
  if (!ok) return ks_fail(ctx, KS_E_CUDA, "cuSOLVER bufferSize query failed (D = %lld)", (long long)D);
  *lwork = lw;
  return KS_OK;
}

// ------------------------------------------------------------------------------------------------------
// Filtered eigensolver for the lowest k eigenpairs of the pencil. After the reduction to
// standard form, B = L L^T (potrf) and C = L^-1 A L^-T (two trsm), it runs a Chebyshev-filtered subspace
// iteration on a block of m = k + g vectors.
//   start   X = L^T Y0, Y0 = [unit vectors on the last k coordinates | g seeded random columns]: the Ritz
//           vectors of W = [P | U~] lie mostly on the U~ block.
//   repeat  SVQB-orthonormalise X; Rayleigh-Ritz (X^T C X, m x m, host Jacobi); stop when every wanted
//           residual ||C x_j - lambda_j x_j|| <= tol * (Gershgorin bound of C); otherwise a degree-DEG
//           Chebyshev filter damping [lambda_m, bound] (3-term recurrence, one GEMM per degree).
//   end     y_j = L^-T x_j, F_B-orthonormal by construction.
// The small dense problems (m <= k + 8 <= 72) are solved on the host: Householder tridiagonalisation + implicit
// QL (cyclic Jacobi as its fallback and A/B, KS_EF_HOSTEIG=jacobi). It falls back to the dense cuSOLVER path if
// it does not converge.
namespace {

constexpr int EF_GUARD = 8, EF_GUARD_MAX = KS_EXT_EF_GUARD, EF_DEG = 20, EF_DEG_GROW = 0, EF_DEG_MAX = 20, EF_MAXIT = 40;

// cyclic Jacobi for a symmetric n x n (column-major, overwritten): ascending eigenvalues w, eigenvectors V
void host_jacobi_eig(std::vector<double> &A, int n, std::vector<double> &w, std::vector<double> &V) {
  V.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; i++) V[(size_t)i * n + i] = 1.0;
  for (int sweep = 0; sweep < 60; sweep++) {
    int rotated = 0;
    for (int p = 0; p < n - 1; p++)
      for (int q = p + 1; q < n; q++) {
        const double apq = A[(size_t)q * n + p];
        const double app = A[(size_t)p * n + p], aqq = A[(size_t)q * n + q];
        // negligible against both diagonal entries (at working precision): no rotation
        if (std::fabs(apq) <= 1e-18 * std::sqrt(std::fabs(app * aqq)) || apq == 0.0) continue;
        rotated++;
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), sn = t * c;
        for (int r = 0; r < n; r++) {   // columns p, q
          const double arp = A[(size_t)p * n + r], arq = A[(size_t)q * n + r];
          A[(size_t)p * n + r] = c * arp - sn * arq;
          A[(size_t)q * n + r] = sn * arp + c * arq;
        }
        for (int r = 0; r < n; r++) {   // rows p, q
          const double apr = A[(size_t)r * n + p], aqr = A[(size_t)r * n + q];
          A[(size_t)r * n + p] = c * apr - sn * aqr;
          A[(size_t)r * n + q] = sn * apr + c * aqr;
        }
        for (int r = 0; r < n; r++) {
          const double vp = V[(size_t)p * n + r], vq = V[(size_t)q * n + r];
          V[(size_t)p * n + r] = c * vp - sn * vq;
          V[(size_t)q * n + r] = sn * vp + c * vq;
        }
      }
    if (rotated == 0) break;
  }
  std::vector<int> idx(n);
  for (int i = 0; i < n; i++) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return A[(size_t)a * n + a] < A[(size_t)b * n + b]; });
  std::vector<double> V2((size_t)n * n);
  w.resize(n);
  for (int j = 0; j < n; j++) {
    w[j] = A[(size_t)idx[j] * n + idx[j]];
    for (int r = 0; r < n; r++) V2[(size_t)j * n + r] = V[(size_t)idx[j] * n + r];
  }
  V.swap(V2);
}

// symmetric n x n (column-major, overwritten): ascending eigenvalues w, eigenvectors V (column j = V[j*n..]).
// Householder reduction to tridiagonal form, then the implicit QL iteration with Wilkinson shifts on (d, e),
// the rotations accumulated into the Householder basis. false if a QL sweep count runs out.
bool host_tridiag_ql_eig(std::vector<double> &A, int n, std::vector<double> &w, std::vector<double> &V) {
  std::vector<double> d(n), e(n, 0.0), v(n), p(n), beta(n, 0.0);
  // A <- H_k ... A ... H_k, the Householder vectors kept below the subdiagonal (v_0 implicit in beta/first entry)
  std::vector<double> Hv((size_t)n * n, 0.0);
  for (int k = 0; k + 2 < n; k++) {
    double *col = &A[(size_t)k * n];
    double nrm2 = 0.0;
    for (int i = k + 1; i < n; i++) nrm2 += col[i] * col[i];
    const double nrm = std::sqrt(nrm2);
    d[k] = col[k];
    if (nrm == 0.0) { e[k] = 0.0; continue; }
    const double alpha = col[k + 1] > 0.0 ? -nrm : nrm;
    for (int i = k + 1; i < n; i++) v[i] = col[i];
    v[k + 1] -= alpha;
    double vv = 0.0;
    for (int i = k + 1; i < n; i++) vv += v[i] * v[i];
    const double b = 2.0 / vv;
    // p = b A22 v, w = p - (b/2)(v.p) v, A22 -= v w^T + w v^T
    for (int i = k + 1; i < n; i++) p[i] = 0.0;
    for (int j = k + 1; j < n; j++) {
      const double *aj = &A[(size_t)j * n];
      const double vj = v[j];
      for (int i = k + 1; i < n; i++) p[i] += aj[i] * vj;
    }
    double vp = 0.0;
    for (int i = k + 1; i < n; i++) { p[i] *= b; vp += v[i] * p[i]; }
    const double K = 0.5 * b * vp;
    for (int i = k + 1; i < n; i++) p[i] -= K * v[i];
    for (int j = k + 1; j < n; j++) {
      double *aj = &A[(size_t)j * n];
      const double vj = v[j], pj = p[j];
      for (int i = k + 1; i < n; i++) aj[i] -= v[i] * pj + p[i] * vj;
    }
    e[k] = alpha;
    beta[k] = b;
    for (int i = k + 1; i < n; i++) Hv[(size_t)k * n + i] = v[i];
  }
  if (n >= 2) {
    d[n - 2] = A[(size_t)(n - 2) * n + (n - 2)];
    e[n - 2] = A[(size_t)(n - 2) * n + (n - 1)];
  }
  d[n - 1] = A[(size_t)(n - 1) * n + (n - 1)];
  // Z = H_0 H_1 ... H_{n-3}, stored by rows of Z^T: Zt[j*n + r] = Z[r][j] (column j contiguous)
  std::vector<double> Z((size_t)n * n, 0.0);
  for (int i = 0; i < n; i++) Z[(size_t)i * n + i] = 1.0;
  for (int k = n - 3; k >= 0; k--) {
    if (beta[k] == 0.0) continue;
    const double *hv = &Hv[(size_t)k * n];
    for (int j = k + 1; j < n; j++) {   // column j of Z: z -= beta v (v.z)
      double *zj = &Z[(size_t)j * n];
      double s = 0.0;
      for (int i = k + 1; i < n; i++) s += hv[i] * zj[i];
      s *= beta[k];
      for (int i = k + 1; i < n; i++) zj[i] -= s * hv[i];
    }
  }
  // implicit QL on (d, e): e[i] couples i and i+1
  for (int l = 0; l < n; l++) {
    for (int iter = 0;; iter++) {
      int m = l;
      for (; m + 1 < n; m++) {
        const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
        if (std::fabs(e[m]) <= 2.3e-16 * dd) break;
      }
      if (m == l) break;
      if (iter == 80) return false;
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = std::sqrt(g * g + 1.0);
      g = d[m] - d[l] + e[l] / (g + (g >= 0.0 ? r : -r));
      double s = 1.0, c = 1.0, pp = 0.0;
      int i = m - 1;
      for (; i >= l; i--) {
        double f = s * e[i];
        const double bb = c * e[i];
        r = std::sqrt(f * f + g * g);
        e[i + 1] = r;
        if (r == 0.0) { d[i + 1] -= pp; e[m] = 0.0; break; }
        s = f / r;
        c = g / r;
        g = d[i + 1] - pp;
        r = (d[i] - g) * s + 2.0 * c * bb;
        pp = s * r;
        d[i + 1] = g + pp;
        g = c * r - bb;
        double *zi = &Z[(size_t)i * n], *zi1 = &Z[(size_t)(i + 1) * n];
        for (int k = 0; k < n; k++) {
          f = zi1[k];
          zi1[k] = s * zi[k] + c * f;
          zi[k] = c * zi[k] - s * f;
        }
      }
      if (r == 0.0 && i >= l) continue;
      d[l] -= pp;
      e[l] = g;
      e[m] = 0.0;
    }
  }
  std::vector<int> idx(n);
  for (int i = 0; i < n; i++) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return d[a] < d[b]; });
  w.resize(n);
  V.resize((size_t)n * n);
  for (int j = 0; j < n; j++) {
    w[j] = d[idx[j]];
    for (int r2 = 0; r2 < n; r2++) V[(size_t)j * n + r2] = Z[(size_t)idx[j] * n + r2];
  }
  return true;
}

// Gershgorin bound max_j sum_i |C_ij| (symmetric, column-major): one warp per column, the maximum through
// an integer atomicMax on the bits of the non-negative column sums (order-independent). *out must be 0.
__global__ void k_row_abs_max(const double *__restrict__ C, int64_t D, unsigned long long *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (j >= D) return;
  double s = 0.0;
  for (int64_t i = lane; i < D; i += 32) s += fabs(C[j * D + i]);
  s = warp_sum(s);
  if (lane == 0) atomicMax(out, (unsigned long long)__double_as_longlong(s));
}

// Yn = alpha (CY - c Y) + beta Xp  (element-wise on D x m blocks)
__global__ void k_cheb(const double *__restrict__ CY, const double *__restrict__ Y, const double *__restrict__ Xp,
                       int64_t len, double alpha, double c, double beta, double *__restrict__ Yn) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= len) return;
  Yn[x] = alpha * (CY[x] - c * Y[x]) + (Xp ? beta * Xp[x] : 0.0);
}

// A <- A - c I with the diagonal saved (save[i] = A_ii), and its exact restoration: the Chebyshev steps take
// alpha (A - c I) Y + beta Y_prev as one GEMM (beta accumulates into Y_prev's buffer)
__global__ void k_shift_diag(double *__restrict__ A, int64_t D, double c, double *__restrict__ save) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= D) return;
  const double a = A[i * D + i];
  save[i] = a;
  A[i * D + i] = a - c;
}
__global__ void k_restore_diag(double *__restrict__ A, int64_t D, const double *__restrict__ save) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < D) A[i * D + i] = save[i];
}

// Out = alpha (A - c I) Y + beta Out for a symmetric A [D][D] and column-major D x m blocks (ld D), m small: the
// product of the filtered iteration in one launch (instead of a cuBLAS GEMM and its split-K reduction, DESIGN.md
// §8.2), on the FP64 tensor cores with the operands staged through shared memory. One CTA per RT output rows and all
// m columns. Chunks of SG2_KC values of k of the CTA's RT rows of A (= its columns: A is symmetric) and
// of all m columns of Y are copied by cp.async (8 bytes each, no alignment needed: D may be odd) into a ring of
// SG2_STAGES stages with a row pitch = 4 (mod 16) doubles (conflict-free fragment loads), so the bytes in flight do
// not occupy registers. A unit is an 8 x 8 output tile; KSPLIT warps share a unit, each taking a contiguous part of
// every chunk in k-steps of 4 (mma.m8n8k4.f64: A[m = lane/4][k = lane%4], B[k = lane%4][n = lane/4],
// C[m = lane/4][n = 2 (lane%4) + v]) with four accumulator pairs in rotation; the KSPLIT partial tiles are added in
// ascending order: deterministic.
constexpr int SG_WARPS = 12;
constexpr int SG2_KC = 128, SG2_STAGES = 3, SG2_PITCH = SG2_KC + 4;
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void sg_mma884(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int RT>
__global__ void __launch_bounds__(SG_WARPS * 32, 1) k_sym_gemm(const double *__restrict__ A, const double *__restrict__ Y,
                                                                  double *__restrict__ Out, int D, int m, int KSPLIT,
                                                                  double alpha, double c, double beta) {
  extern __shared__ __align__(16) double sg2[];   // [STAGES][RT + m][PITCH], then red [SG_WARPS][8][8]
  const int rows = RT + m;
  double *red = sg2 + (size_t)SG2_STAGES * rows * SG2_PITCH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, grp = lane >> 2, tig = lane & 3;
  const int i0 = blockIdx.x * RT;
  const int nct = (m + 7) / 8;
  const int nchunks = (D + SG2_KC - 1) / SG2_KC;
  auto fill = [&](int chunk) {
    double *st = sg2 + (size_t)(chunk % SG2_STAGES) * rows * SG2_PITCH;
    const int kbase = chunk * SG2_KC;
    for (int row = warp; row < rows; row += SG_WARPS) {   // a warp per staged row, lanes on consecutive k
      const double *src = (row < RT ? A + (int64_t)min(i0 + row, D - 1) * D : Y + (int64_t)(row - RT) * D) + kbase;
      double *dst = st + row * SG2_PITCH;
#pragma unroll
      for (int u = 0; u < SG2_KC / 32; u++) {
        const int kk = u * 32 + lane;
        if (kbase + kk < D) cp_async8(dst + kk, src + kk);
        else dst[kk] = 0.0;
      }
    }
  };
  for (int sgi = 0; sgi < SG2_STAGES - 1; sgi++) {
    if (sgi < nchunks) fill(sgi);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  const int unit = warp / KSPLIT, kq = warp - unit * KSPLIT;
  const int rt = unit / nct, ct = unit - rt * nct;
  const bool active = unit < (RT / 8) * nct;
  const int arow = rt * 8 + grp, brow = RT + min(ct * 8 + grp, m - 1);
  const int klen = SG2_KC / KSPLIT, k0 = kq * klen;
  double c0[4] = {0.0, 0.0, 0.0, 0.0}, c1[4] = {0.0, 0.0, 0.0, 0.0};
  for (int ch = 0; ch < nchunks; ch++) {
    asm volatile("cp.async.wait_group %0;" ::"n"(SG2_STAGES - 2) : "memory");
    __syncthreads();   // chunk ch has landed for every thread; every warp is done with chunk ch - 1
    if (ch + SG2_STAGES - 1 < nchunks) fill(ch + SG2_STAGES - 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (active) {
      const double *st = sg2 + (size_t)(ch % SG2_STAGES) * rows * SG2_PITCH;
      const double *pa = st + arow * SG2_PITCH + k0 + tig, *pb = st + brow * SG2_PITCH + k0 + tig;
      for (int kk = 0; kk < klen; kk += 16) {
        double av[4], bv[4];
#pragma unroll
        for (int u = 0; u < 4; u++) { av[u] = pa[kk + 4 * u]; bv[u] = pb[kk + 4 * u]; }
#pragma unroll
        for (int u = 0; u < 4; u++) sg_mma884(c0[u], c1[u], av[u], bv[u]);
      }
    }
  }
  if (active) {
    red[(warp * 8 + grp) * 8 + 2 * tig] = (c0[0] + c0[1]) + (c0[2] + c0[3]);
    red[(warp * 8 + grp) * 8 + 2 * tig + 1] = (c1[0] + c1[1]) + (c1[2] + c1[3]);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < RT * m; t += blockDim.x) {
    const int j = t / RT, r = t - j * RT, i = i0 + r;
    if (i >= D) continue;
    const int u = (r >> 3) * nct + (j >> 3);
    double sacc = 0.0;
    for (int q = 0; q < KSPLIT; q++) sacc += red[((u * KSPLIT + q) * 8 + (r & 7)) * 8 + (j & 7)];
    const int64_t o = (int64_t)j * D + i;
    double v = alpha * (sacc - c * Y[o]);
    if (beta != 0.0) v = fma(beta, Out[o], v);
    Out[o] = v;
  }
}

// The two Gram matrices of the Rayleigh-Ritz step in one launch: G = X^T X and H = X^T (C X), m x m column-major,
// for column-major D x m blocks. One warp per pair a <= b (lanes on consecutive k, four k per lane in flight),
// butterfly sums, the entry mirrored (H is symmetric up to rounding; the host symmetrises the reduced matrix).
__global__ void __launch_bounds__(SG_WARPS * 32) k_gram_pair(const double *__restrict__ X, const double *__restrict__ CXb,
                                                             int D, int m, double *__restrict__ G, double *__restrict__ H) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * SG_WARPS + (threadIdx.x >> 5);
  if (gw >= m * m) return;
  const int a = gw % m, b = gw / m;
  if (a > b) return;
  const double *xa = X + (int64_t)a * D, *xb = X + (int64_t)b * D, *cb = CXb + (int64_t)b * D;
  double g = 0.0, h = 0.0;
  int k = lane;
  for (; k + 96 < D; k += 128) {
    double va[4], vb[4], vc[4];
#pragma unroll
    for (int u = 0; u < 4; u++) { va[u] = xa[k + 32 * u]; vb[u] = xb[k + 32 * u]; vc[u] = cb[k + 32 * u]; }
#pragma unroll
    for (int u = 0; u < 4; u++) { g = fma(va[u], vb[u], g); h = fma(va[u], vc[u], h); }
  }
  for (; k < D; k += 32) { const double va = xa[k]; g = fma(va, xb[k], g); h = fma(va, cb[k], h); }
  g = warp_sum(g);
  h = warp_sum(h);
  if (lane == 0) {
    G[b * m + a] = g; G[a * m + b] = g;
    H[b * m + a] = h; H[a * m + b] = h;
  }
}

// The Rayleigh-Ritz rotation and the residuals in one launch: Xn = X T, CXn = (C X) T for the m x m matrix T
// (column-major), and per block of RR_ROWS rows the partial sums of (CXn_ij - lam_j Xn_ij)^2 for the k wanted
// columns (part [row blocks][k], summed on the host in ascending block order). A CTA takes RR_ROWS rows and 8
// output columns: its rows of X and C X staged in shared memory (a thread per row), T's 8 columns l-major.
constexpr int RR_ROWS = 128, RR_JB = 8;
__global__ void __launch_bounds__(RR_ROWS) k_rotate_resid(const double *__restrict__ X, const double *__restrict__ CXb,
                                                          const double *__restrict__ T, const double *__restrict__ lam,
                                                          int D, int m, int k, double *__restrict__ Xn,
                                                          double *__restrict__ CXn, double *__restrict__ part) {
  extern __shared__ __align__(16) double rr_s[];   // xs [m][RR_ROWS], cs [m][RR_ROWS], ts [m][RR_JB], wsum [4][RR_JB]
  double *xs = rr_s, *cs = xs + (size_t)m * RR_ROWS, *ts = cs + (size_t)m * RR_ROWS, *wsum = ts + (size_t)m * RR_JB;
  const int tid = threadIdx.x, i = blockIdx.x * RR_ROWS + tid, jb = blockIdx.y * RR_JB;
  const bool row_ok = i < D;
  for (int l = 0; l < m; l++) {
    xs[l * RR_ROWS + tid] = row_ok ? X[(int64_t)l * D + i] : 0.0;
    cs[l * RR_ROWS + tid] = row_ok ? CXb[(int64_t)l * D + i] : 0.0;
  }
  for (int x = tid; x < m * RR_JB; x += RR_ROWS) {
    const int l = x / RR_JB, q = x - l * RR_JB;
    ts[x] = jb + q < m ? T[(int64_t)(jb + q) * m + l] : 0.0;
  }
  __syncthreads();
  double ax[RR_JB], ac[RR_JB];
#pragma unroll
  for (int q = 0; q < RR_JB; q++) ax[q] = ac[q] = 0.0;
  for (int l = 0; l < m; l++) {
    const double xv = xs[l * RR_ROWS + tid], cv = cs[l * RR_ROWS + tid];
#pragma unroll
    for (int q = 0; q < RR_JB; q++) {
      const double w = ts[l * RR_JB + q];
      ax[q] = fma(xv, w, ax[q]);
      ac[q] = fma(cv, w, ac[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < RR_JB; q++) {
    const int j = jb + q;
    if (j < m && row_ok) {
      Xn[(int64_t)j * D + i] = ax[q];
      CXn[(int64_t)j * D + i] = ac[q];
    }
    double r = 0.0;
    if (j < k && row_ok) {
      r = ac[q] - lam[j] * ax[q];
      r *= r;
    }
    r = warp_sum(r);
    if ((tid & 31) == 0) wsum[(tid >> 5) * RR_JB + q] = r;
  }
  __syncthreads();
  if (tid < RR_JB && jb + tid < k) {
    double sacc = 0.0;
    for (int w = 0; w < RR_ROWS / 32; w++) sacc += wsum[w * RR_JB + tid];
    part[(int64_t)blockIdx.x * k + jb + tid] = sacc;
  }
}

// number of entries of the leading n x n block of F (column-major, ld D) that differ from B (n x n)
__global__ void k_block_mismatch(const double *__restrict__ F, int64_t D, const double *__restrict__ B, int64_t n,
                                 int *__restrict__ count) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool bad = false;
  if (x < n * n) bad = F[(x / n) * D + x % n] != B[x];
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicAdd(count, 1);
}

// explicit L = [[L_H, 0], [K, L_S]] and L^-1 = [[L_H^-1, 0], [BL, L_S^-1]] (D x D, column-major, upper zero)
// from the cached coarse factor and the Schur-complement pieces (K = Kt^T, Kt [nH][Nc] column-major)
__global__ void k_build_L(const double *__restrict__ LH, const double *__restrict__ LHinv, const double *__restrict__ Kt,
                          const double *__restrict__ LS, const double *__restrict__ LSinv, int64_t nH, int64_t Nc,
                          double *__restrict__ L, double *__restrict__ Linv) {
  const int64_t D = nH + Nc;
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= D * D) return;
  const int64_t i = x % D, j = x / D;   // row, column
  double l = 0.0, li = 0.0;
  if (i >= j) {
    if (j < nH && i < nH) {
      l = LH[j * nH + i];
      li = LHinv[j * nH + i];
    } else if (j < nH) {         // bottom-left: K (L^-1's block is written by a GEMM afterwards)
      l = Kt[(i - nH) * nH + j];
    } else {
      l = LS[(j - nH) * Nc + (i - nH)];
      li = LSinv[(j - nH) * Nc + (i - nH)];
    }
  }
  L[x] = l;
  Linv[x] = li;
}

__global__ void k_lower_only(double *__restrict__ A, int64_t n) {   // zero the strict upper triangle
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= n * n) return;
  if (x % n < x / n) A[x] = 0.0;
}

__global__ void k_identity(double *__restrict__ A, int64_t n) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x < n * n) A[x] = (x % n == x / n) ? 1.0 : 0.0;
}

// T[j * D + i] = Y[i * k + j] for the first k columns of a column-major D x m block (Y row-major D x k)
__global__ void k_put_cols(const double *__restrict__ Y, int64_t D, int k, double *__restrict__ T) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= D * k) return;
  const int64_t i = x / k, j = x % k;
  T[j * D + i] = Y[x];
}

// squared residual norms of the first k columns: sum_i (CX_ij - lam_j X_ij)^2 (one warp per column)
__global__ void k_resid(const double *__restrict__ CX, const double *__restrict__ X, const double *__restrict__ lam,
                        int64_t D, int k, double *__restrict__ out) {
  const int j = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < D; i += blockDim.x) {
    const double r = CX[j * D + i] - lam[j] * X[j * D + i];
    s += r * r;
  }
  s = warp_sum(s);
  if (threadIdx.x == 0) out[j] = s;
}

// guard vectors of the filtered iteration: EF_GUARD, or KS_EF_GUARD (A/B) up to the extension region's capacity
int ef_guard() {
  int g = EF_GUARD;
  if (const char *e = getenv("KS_EF_GUARD")) g = std::min(EF_GUARD_MAX, std::max(1, atoi(e)));
  return g;
}

}  // namespace

extern "C" ks_status ks_host_sym_eig(int32_t n, const double *h_A, double *h_w, double *h_V, int32_t method) {
  if (n < 1 || !h_A || !h_w || !h_V || method < 0 || method > 1) return KS_E_ARG;
  std::vector<double> A(h_A, h_A + (size_t)n * n), w, V;
  if (method == 0) {
    if (!host_tridiag_ql_eig(A, n, w, V)) return KS_E_NOT_CONVERGED;
  } else {
    host_jacobi_eig(A, n, w, V);
  }
  std::copy(w.begin(), w.end(), h_w);
  std::copy(V.begin(), V.end(), h_V);
  return KS_OK;
}

static ks_status ensure_blas(ks_ctx *ctx) {
  if (!ctx->cublas) {
    cublasHandle_t b = nullptr;
    if (cublasCreate(&b) != CUBLAS_STATUS_SUCCESS) return ks_fail(ctx, KS_E_CUDA, "cublasCreate failed");
    ctx->cublas = b;
  }
  if (cublasSetStream((cublasHandle_t)ctx->cublas, ctx->stream) != CUBLAS_STATUS_SUCCESS)
    return ks_fail(ctx, KS_E_CUDA, "cublasSetStream failed");
  // the GEMM workspace comes from the caller's extension region (cuBLAS allocates none of its own)
  if (cublasSetWorkspace((cublasHandle_t)ctx->cublas, ctx->blas_ws, KS_EXT_BLAS_WS) != CUBLAS_STATUS_SUCCESS)
    return ks_fail(ctx, KS_E_CUDA, "cublasSetWorkspace failed");
  return KS_OK;
}

// plan of k_sym_gemm: warps per 8 x 8 output tile and dynamic shared memory; false when the sizes do not fit, i.e.
// more than one wave of 8-row CTAs (D > 8 SMs: with 16-row CTAs every CTA still stages all of Y, and at C5's
// D = 1363 that was slower than cuBLAS) or more column tiles than warps: cuBLAS serves those
struct SymGemmPlan {
  int KSPLIT = 1;
  size_t smem = 0;
};
constexpr int SG_RT = 8;
static bool sym_gemm_plan(const ks_ctx *ctx, int64_t D, int m, SymGemmPlan *pl) {
  const int nct = (m + 7) / 8;
  if (D < 64 || m < 1 || (D + SG_RT - 1) / SG_RT > ctx->sm_count || nct > SG_WARPS) return false;
  int KSPLIT = 1;
  while (KSPLIT < 4 && nct * KSPLIT * 2 <= SG_WARPS) KSPLIT *= 2;
  const size_t smem = sizeof(double) * ((size_t)SG2_STAGES * (SG_RT + m) * SG2_PITCH + (size_t)SG_WARPS * 64);
  if (smem > 220 * 1024) return false;
  pl->KSPLIT = KSPLIT;
  pl->smem = smem;
  return true;
}
static bool sym_gemm_fits(const ks_ctx *ctx, int64_t D, int m) {
  SymGemmPlan pl;
  return sym_gemm_plan(ctx, D, m, &pl);
}
static bool sym_gemm(ks_ctx *ctx, const double *A, const double *Y, double *Out, int64_t D, int m, double alpha,
                     double c, double beta) {
  SymGemmPlan pl;
  if (!sym_gemm_plan(ctx, D, m, &pl)) return false;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute((const void *)k_sym_gemm<SG_RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  const int grid = (int)((D + SG_RT - 1) / SG_RT);
  k_sym_gemm<SG_RT><<<grid, SG_WARPS * 32, pl.smem, ctx->stream>>>(A, Y, Out, (int)D, m, pl.KSPLIT, alpha, c, beta);
  return true;
}

#define KS_BLAS(ctx, call)                                                                         \
  do {                                                                                             \
    if ((call) != CUBLAS_STATUS_SUCCESS) return ks_fail(ctx, KS_E_CUDA, "cuBLAS call failed: " #call); \
  } while (0)

// the filtered path on ctx->eig_A (A, overwritten by C) and ctx->eig_B (B, overwritten by L), after potrf.
// *done = false: not converged (the caller runs the dense path on fresh copies)
static ks_status pencil_eig_filtered(ks_ctx *ctx, int64_t D, int k, double *evals, double *evecs, bool *done,
                                     const double *Ywarm, const double *Linv) {
  *done = false;
  KS_TRY(ensure_blas(ctx));
  cublasHandle_t hb = (cublasHandle_t)ctx->cublas;
  cudaStream_t st = ctx->stream;
  const int m = k + ef_guard();
  const double one = 1.0, zero = 0.0;
  double *A = ctx->eig_A, *L = ctx->eig_B;
  // C = L^-1 A L^-T (in A): two GEMMs with the explicit inverse when it is given (the coarse block's factor is
  // cached, ks_pencil_eig_impl), else two triangular solves
  if (Linv) {
    KS_BLAS(ctx, cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, (int)D, (int)D, (int)D, &one, Linv, (int)D, A, (int)D, &zero,
                             ctx->ef_TD, (int)D));
    KS_BLAS(ctx, cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_T, (int)D, (int)D, (int)D, &one, ctx->ef_TD, (int)D, Linv,
                             (int)D, &zero, A, (int)D));
  } else {
    KS_BLAS(ctx, cublasDtrsm(hb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, (int)D,
                             (int)D, &one, L, (int)D, A, (int)D));
    KS_BLAS(ctx, cublasDtrsm(hb, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, (int)D,
                             (int)D, &one, L, (int)D, A, (int)D));
  }
  // ef_buf [4][D][m], ef_small [2 m m + m + 1] (two m x m Grams, then V and lambda): the extension workspace
  // holds them for m <= max_N + EF_GUARD and D <= ext_D (ks_pencil_eig_impl routes larger k to the dense path)
  double *X = ctx->ef_buf, *CX = X + D * m, *T1 = CX + D * m, *T2 = T1 + D * m, *sm = ctx->ef_small;
  // start block: Y0 in T1, X = L^T Y0
  {
    std::vector<double> y0((size_t)D * m, 0.0);
    uint64_t sd = 0x9E3779B97F4A7C15ull;
    for (int j = 0; j < m; j++) {
      if (j < k) {
        y0[(size_t)j * D + (D - k + j)] = 1.0;
      } else {
        for (int64_t i = 0; i < D; i++) {
          sd = sd * 6364136223846793005ull + 1442695040888963407ull;
          y0[(size_t)j * D + i] = (double)(sd >> 11) * 0x1.0p-53 - 0.5;
        }
      }
    }
    KS_CUDA(ctx, cudaMemcpyAsync(T1, y0.data(), sizeof(double) * D * m, cudaMemcpyHostToDevice, st));
    if (Ywarm) {   // the caller's start vectors replace the unit vectors
      k_put_cols<<<ks_blocks(D * k, 256), 256, 0, st>>>(Ywarm, D, k, T1);
      KS_LAUNCHED(ctx);
    }
    KS_CUDA(ctx, cudaStreamSynchronize(st));
    KS_BLAS(ctx, cublasDtrmm(hb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, (int)D, m,
                             &one, L, (int)D, T1, (int)D, X, (int)D));
  }
  double bound = 0.0;
  KS_CUDA(ctx, cudaMemsetAsync(sm, 0, sizeof(double), st));
  k_row_abs_max<<<ks_blocks(32 * D, 256), 256, 0, st>>>(A, D, reinterpret_cast<unsigned long long *>(sm));
  KS_LAUNCHED(ctx);
  const double tol = 1e-12;
  int maxit = EF_MAXIT;   // KS_PENCIL_EF_MAXIT: test hook to exercise the dense fallback
  if (const char *e = getenv("KS_PENCIL_EF_MAXIT")) maxit = atoi(e);
  // KS_PENCIL_DEVICE=1: the whole iteration as one cooperative kernel (ks_efdev.cu, measured slower)
  const char *devrr = getenv("KS_PENCIL_DEVICE");
  // KS_EF_FUSED=0: the Chebyshev step as a GEMM plus an element-wise kernel (the round-1 form; A/B only)
  const char *fe = getenv("KS_EF_FUSED");
  const bool fused_cheb = !(fe && fe[0] == '0');
  // KS_EF_GEMM=cublas: the D x D by D x m products through cuBLAS instead of k_sym_gemm (A/B)
  const char *ge = getenv("KS_EF_GEMM");
  const bool own_gemm = !(ge && ge[0] == 'c') && sym_gemm_fits(ctx, D, m);
  // KS_EF_RR=cublas: the Gram matrices, the rotation and the residuals of the Rayleigh-Ritz step by cuBLAS GEMMs and
  // k_resid (5 launches) instead of k_gram_pair and k_rotate_resid (A/B)
  const char *re = getenv("KS_EF_RR");
  const int64_t rr_blocks = (D + RR_ROWS - 1) / RR_ROWS;
  const size_t rr_smem = sizeof(double) * ((size_t)2 * m * RR_ROWS + (size_t)m * RR_JB + (RR_ROWS / 32) * RR_JB);
  const bool own_rr = !(re && re[0] == 'c') && rr_blocks * k <= (int64_t)m * m && rr_smem <= 200 * 1024;
  if (own_rr && rr_smem > 48 * 1024)
    KS_CUDA(ctx, cudaFuncSetAttribute((const void *)k_rotate_resid, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)rr_smem));
  std::vector<double> rpart;
  if (devrr && devrr[0] == '1' && ctx->ef_dev) {
    int stv = 0, rounds = 0;
    bool ran = false;
    double *lam_dev = nullptr;
    KS_TRY(ks_ef_device(ctx, D, k, m, A, X, CX, sm, ctx->ef_dev, maxit, EF_DEG, tol, &stv, &rounds, &ran, &lam_dev));
    if (ran) {
      ctx->ef_rounds = rounds;
      if (stv != 1) return KS_OK;   // not converged or a collapsed block: the dense path
      // the orthonormal block is in CX: y = L^-T x, eigenvalues, eigenvectors [D][k] row-major
      if (Linv) {
        KS_BLAS(ctx, cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, (int)D, k, (int)D, &one, Linv, (int)D, CX, (int)D, &zero,
                                 T2, (int)D));
      } else {
        KS_CUDA(ctx, cudaMemcpyAsync(T2, CX, sizeof(double) * D * k, cudaMemcpyDeviceToDevice, st));
        KS_BLAS(ctx, cublasDtrsm(hb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, (int)D,
                                 k, &one, L, (int)D, T2, (int)D));
      }
      KS_CUDA(ctx, cudaMemcpyAsync(evals, lam_dev, sizeof(double) * k, cudaMemcpyDeviceToDevice, st));
      k_take_evecs<<<ks_blocks(D * k, 256), 256, 0, st>>>(T2, D, k, evecs);
      KS_LAUNCHED(ctx);
      *done = true;
      return KS_OK;
    }
  }
  KS_CUDA(ctx, cudaMemcpyAsync(&bound, sm, sizeof(double), cudaMemcpyDeviceToHost, st));
  KS_CUDA(ctx, cudaStreamSynchronize(st));
  std::vector<double> G((size_t)m * m), w, V, Tm, lam(m), res(k);
  // host: Cholesky of the column-scaled Gram G = D R^T R D (upper R, column-major); false on a collapsed pivot
  auto host_chol = [&](const std::vector<double> &Gm, std::vector<double> &dsc, std::vector<double> &Rinv) -> bool {
    dsc.resize(m);
    for (int j = 0; j < m; j++) dsc[j] = std::sqrt(Gm[(size_t)j * m + j]);
    if (!(dsc[0] > 0.0)) return false;
    std::vector<double> R((size_t)m * m, 0.0);
    for (int j = 0; j < m; j++)
      for (int i = 0; i <= j; i++) {
        double v = Gm[(size_t)j * m + i] / (dsc[i] * dsc[j]);
        for (int l = 0; l < i; l++) v -= R[(size_t)i * m + l] * R[(size_t)j * m + l];
        if (i == j) {
          if (!(v > 1e-12)) return false;
          R[(size_t)j * m + j] = std::sqrt(v);
        } else {
          R[(size_t)j * m + i] = v / R[(size_t)i * m + i];
        }
      }
    Rinv.assign((size_t)m * m, 0.0);   // R^-1 (upper), by columns
    for (int j = 0; j < m; j++) {
      Rinv[(size_t)j * m + j] = 1.0 / R[(size_t)j * m + j];
      for (int i = j - 1; i >= 0; i--) {
        double v = 0.0;
        for (int l = i + 1; l <= j; l++) v += R[(size_t)l * m + i] * Rinv[(size_t)j * m + l];
        Rinv[(size_t)j * m + i] = -v / R[(size_t)i * m + i];
      }
    }
    return true;
  };
  std::vector<double> G2((size_t)m * m), dsc, Rinv, Hs((size_t)m * m), Hq;
  double host_us = 0.0;   // host share of the Rayleigh-Ritz steps (KS_EF_VERBOSE)
  const char *he = getenv("KS_EF_HOSTEIG");
  const bool jacobi_rr = he && he[0] == 'j';
  // filter degree of round it: min(deg_max, deg0 + grow * it) (KS_EF_DEG / KS_EF_DEG_GROW / KS_EF_DEG_MAX; A/B)
  int deg0 = EF_DEG, deg_grow = EF_DEG_GROW, deg_max = EF_DEG_MAX;
  if (const char *e = getenv("KS_EF_DEG")) deg0 = std::max(2, atoi(e));
  if (const char *e = getenv("KS_EF_DEG_GROW")) deg_grow = std::max(0, atoi(e));
  if (const char *e = getenv("KS_EF_DEG_MAX")) deg_max = std::max(2, atoi(e));
  for (int it = 0; it < maxit; it++) {
    ctx->ef_rounds = it + 1;
    // Rayleigh-Ritz on span(X) with the orthonormalisation folded in: T2 = C X, G = X^T X and H = X^T C X in
    // one round trip; on the host the small pencil (H, G) is reduced by the Cholesky factor of the scaled G
    // and diagonalised by Jacobi: V = D^-1 R^-1 W, X <- X V (orthonormal), CX <- (C X) V
    if (own_gemm) {
      sym_gemm(ctx, A, X, T2, D, m, 1.0, 0.0, 0.0);
      KS_LAUNCHED(ctx);
    } else {
      KS_BLAS(ctx, cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, (int)D, m, (int)D, &one, A, (int)D, X, (int)D, &zero, T2,
                               (int)D));
    }
    if (own_rr) {
      k_gram_pair<<<(m * m + SG_WARPS - 1) / SG_WARPS, SG_WARPS * 32, 0, st>>>(X, T2, (int)D, m, sm, sm + (int64_t)m * m);
      KS_LAUNCHED(ctx);
    } else {
      KS_BLAS(ctx, cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, m, m, (int)D, &one, X, (int)D, X, (int)D, &zero, sm, m));
      KS_BLAS(ctx, cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, m, m, (int)D, &one, X, (int)D, T2, (int)D, &zero,
                               sm + (int64_t)m * m, m));
    }
    KS_CUDA(ctx, cudaMemcpyAsync(G.data(), sm, sizeof(double) * m * m, cudaMemcpyDeviceToHost, st));
    KS_CUDA(ctx, cudaMemcpyAsync(G2.data(), sm + (int64_t)m * m, sizeof(double) * m * m, cudaMemcpyDeviceToHost, st));
    KS_CUDA(ctx, cudaStreamSynchronize(st));
    const auto h0 = std::chrono::steady_clock::now();
    if (!host_chol(G, dsc, Rinv)) {   // the block lost rank: dense path
      if (getenv("KS_EF_VERBOSE")) fprintf(stderr, "ks_pencil_eig: round %d: Gram pivot collapsed\n", it + 1);
      return KS_OK;
    }
    // Hs = R^-T (D^-1 H D^-1) R^-1
    for (int j = 0; j < m; j++)
      for (int i = 0; i < m; i++) G2[(size_t)j * m + i] /= dsc[i] * dsc[j];
    {
      std::vector<double> HR((size_t)m * m, 0.0);   // (D^-1 H D^-1) R^-1
      for (int j = 0; j < m; j++)
        for (int l = 0; l <= j; l++) {
          const double r = Rinv[(size_t)j * m + l];
          for (int i = 0; i < m; i++) HR[(size_t)j * m + i] += G2[(size_t)l * m + i] * r;
        }
      for (int j = 0; j < m; j++)
        for (int i = 0; i < m; i++) {
          double v = 0.0;
          for (int l = 0; l <= i; l++) v += Rinv[(size_t)i * m + l] * HR[(size_t)j * m + l];
          Hs[(size_t)j * m + i] = v;
        }
      for (int j = 0; j < m; j++)
        for (int i = 0; i < j; i++) Hs[(size_t)j * m + i] = Hs[(size_t)i * m + j] = 0.5 * (Hs[(size_t)j * m + i] + Hs[(size_t)i * m + j]);
    }
    // the small symmetric eigenproblem: Householder + implicit QL (KS_EF_HOSTEIG=jacobi: cyclic Jacobi, which is
    // also the fallback should a QL iteration count run out)
    if (jacobi_rr) {
      host_jacobi_eig(Hs, m, w, V);
    } else {
      Hq = Hs;
      if (!host_tridiag_ql_eig(Hq, m, w, V)) host_jacobi_eig(Hs, m, w, V);
    }
    lam = w;
    Tm.assign((size_t)m * m, 0.0);   // D^-1 R^-1 W
    for (int j = 0; j < m; j++)
      for (int i = 0; i < m; i++) {
        double v = 0.0;
        for (int l = i; l < m; l++) v += Rinv[(size_t)l * m + i] * V[(size_t)j * m + l];
        Tm[(size_t)j * m + i] = v / dsc[i];
      }
    host_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count();
    KS_CUDA(ctx, cudaMemcpyAsync(sm, Tm.data(), sizeof(double) * m * m, cudaMemcpyHostToDevice, st));
    KS_CUDA(ctx, cudaMemcpyAsync(sm + (int64_t)m * m, lam.data(), sizeof(double) * m, cudaMemcpyHostToDevice, st));
    double rmax = 0.0;
    if (own_rr) {   // rotation and wanted residuals in one launch; the row-block partials summed here in order
      double *part = sm + (int64_t)m * m + m;
      k_rotate_resid<<<dim3((unsigned)rr_blocks, (unsigned)((m + RR_JB - 1) / RR_JB)), RR_ROWS, rr_smem, st>>>(
          X, T2, sm, sm + (int64_t)m * m, (int)D, m, k, T1, CX, part);
      KS_LAUNCHED(ctx);
      std::swap(X, T1);
      rpart.resize((size_t)rr_blocks * k);
      KS_CUDA(ctx, cudaMemcpyAsync(rpart.data(), part, sizeof(double) * rr_blocks * k, cudaMemcpyDeviceToHost, st));
      KS_CUDA(ctx, cudaStreamSynchronize(st));
      for (int j = 0; j < k; j++) {
        double sacc = 0.0;
        for (int64_t rb = 0; rb < rr_blocks; rb++) sacc += rpart[(size_t)rb * k + j];
        rmax = std::fmax(rmax, std::sqrt(sacc));
      }
    } else {
      KS_BLAS(ctx, cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, (int)D, m, m, &one, X, (int)D, sm, m, &zero, T1, (int)D));
      KS_BLAS(ctx, cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, (int)D, m, m, &one, T2, (int)D, sm, m, &zero, CX, (int)D));
      std::swap(X, T1);
      // wanted residuals
      k_resid<<<k, 32, 0, st>>>(CX, X, sm + (int64_t)m * m, D, k, T2);
      KS_LAUNCHED(ctx);
      KS_CUDA(ctx, cudaMemcpyAsync(res.data(), T2, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
      KS_CUDA(ctx, cudaStreamSynchronize(st));
      for (int j = 0; j < k; j++) rmax = std::fmax(rmax, std::sqrt(res[j]));
    }
    if (getenv("KS_EF_VERBOSE"))
      fprintf(stderr, "ks_pencil_eig: round %d rmax %.3e (tol %.3e), host Rayleigh-Ritz so far %.0f us\n", it + 1, rmax,
              tol * bound, host_us);
    if (!std::isfinite(rmax)) return KS_OK;
    if (rmax <= tol * bound) {
      // one more Cholesky-QR pass (X V is orthonormal only up to cond(X)^2 eps), then y = L^-T x, evals
      KS_BLAS(ctx, cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, m, m, (int)D, &one, X, (int)D, X, (int)D, &zero, sm, m));
      KS_CUDA(ctx, cudaMemcpyAsync(G.data(), sm, sizeof(double) * m * m, cudaMemcpyDeviceToHost, st));
      KS_CUDA(ctx, cudaStreamSynchronize(st));
      if (!host_chol(G, dsc, Rinv)) return KS_OK;
      for (int j = 0; j < m; j++)
        for (int i = 0; i < m; i++) Tm[(size_t)j * m + i] = Rinv[(size_t)j * m + i] / dsc[i];
      KS_CUDA(ctx, cudaMemcpyAsync(sm, Tm.data(), sizeof(double) * m * m, cudaMemcpyHostToDevice, st));
      KS_CUDA(ctx, cudaMemcpyAsync(sm + (int64_t)m * m, lam.data(), sizeof(double) * m, cudaMemcpyHostToDevice, st));
      KS_BLAS(ctx, cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, (int)D, m, m, &one, X, (int)D, sm, m, &zero, T1, (int)D));
      if (Linv) {   // y = L^-T x
        KS_BLAS(ctx, cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, (int)D, k, (int)D, &one, Linv, (int)D, T1, (int)D, &zero,
                                 T2, (int)D));
        std::swap(T1, T2);
      } else {
        KS_BLAS(ctx, cublasDtrsm(hb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, (int)D,
                                 k, &one, L, (int)D, T1, (int)D));
      }
      KS_CUDA(ctx, cudaMemcpyAsync(evals, sm + (int64_t)m * m, sizeof(double) * k, cudaMemcpyDeviceToDevice, st));
      k_take_evecs<<<ks_blocks(D * k, 256), 256, 0, st>>>(T1, D, k, evecs);
      KS_LAUNCHED(ctx);
      *done = true;
      return KS_OK;
    }
    // Chebyshev filter damping [lam_m, bound]
    const double a = lam[m - 1], b = bound, e = 0.5 * (b - a), c = 0.5 * (b + a);
    if (!(e > 0.0)) return KS_OK;
    double sigma = e / (lam[0] - c);
    const double s1 = 2.0 / sigma;
    const int64_t len = D * m;
    const int deg = std::max(2, std::min(std::max(deg_max, deg0), deg0 + deg_grow * it));
    double *Xp = X, *Y = T1, *Yn = T2;
    k_cheb<<<ks_blocks(len, 256), 256, 0, st>>>(CX, X, nullptr, len, sigma / e, c, 0.0, Y);
    KS_LAUNCHED(ctx);
    if (fused_cheb && own_gemm) {
      // Y_{d} = (2 s2 / e) (C - c I) Y_{d-1} - sigma s2 Y_{d-2}: one k_sym_gemm launch per degree, accumulated into
      // Y_{d-2}'s buffer
      for (int d = 2; d <= deg; d++) {
        const double s2 = 1.0 / (s1 - sigma), al = 2.0 * s2 / e, be = -sigma * s2;
        if (!sym_gemm(ctx, A, Y, Xp, D, m, al, c, be)) return ks_fail(ctx, KS_E_STATE, "ks_pencil_eig: k_sym_gemm sizes");
        KS_LAUNCHED(ctx);
        std::swap(Xp, Y);
        sigma = s2;
      }
    } else if (fused_cheb) {
      // the same with one cuBLAS GEMM per degree; C's diagonal is shifted for the filter and restored bitwise after
      // it (T2 holds the saved diagonal)
      k_shift_diag<<<ks_blocks(D, 256), 256, 0, st>>>(A, D, c, T2);
      KS_LAUNCHED(ctx);
      for (int d = 2; d <= deg; d++) {
        const double s2 = 1.0 / (s1 - sigma), al = 2.0 * s2 / e, be = -sigma * s2;
        KS_BLAS(ctx, cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, (int)D, m, (int)D, &al, A, (int)D, Y, (int)D, &be, Xp,
                                 (int)D));
        std::swap(Xp, Y);
        sigma = s2;
      }
      k_restore_diag<<<ks_blocks(D, 256), 256, 0, st>>>(A, D, T2);
      KS_LAUNCHED(ctx);
    } else {
      for (int d = 2; d <= deg; d++) {
        const double s2 = 1.0 / (s1 - sigma);
        KS_BLAS(ctx, cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, (int)D, m, (int)D, &one, A, (int)D, Y, (int)D, &zero, CX,
                                 (int)D));
        k_cheb<<<ks_blocks(len, 256), 256, 0, st>>>(CX, Y, Xp, len, 2.0 * s2 / e, c, -sigma * s2, Yn);
        KS_LAUNCHED(ctx);
        double *t = Xp;
        Xp = Y;
        Y = Yn;
        Yn = t;
        sigma = s2;
      }
    }
    if (Y != X) KS_CUDA(ctx, cudaMemcpyAsync(X, Y, sizeof(double) * len, cudaMemcpyDeviceToDevice, st));
  }
  return KS_OK;
}

// The pencil of ks_project_augmented has F_B = [[B_H, c], [c^T, gamma]] with B_H = P^T M P fixed per coarse space.
// Its Cholesky factor is L = [[L_H, 0], [K, L_S]] with L_H = chol(B_H) (cached once per coarse space, with
// L_H^-1), K = c^T L_H^-T and L_S = chol(gamma - K K^T) (N x N), so L and L^-1 are formed in O(n_H^2 N) and
// the reduction C = L^-1 F_A L^-T takes two GEMMs instead of a D x D factorisation and two triangular solves
// (DESIGN.md §8.2). Returns false (caller: the general path) when the leading block of F_B is not bitwise the
// cached B_H, N > max_N, or a factor is not positive definite. eig_B <- L, ctx->ef_Linv <- L^-1.
static ks_status coarse_chol_reduction(ks_ctx *ctx, int64_t D, const double *FB, bool *ok) {
  *ok = false;
  const int64_t nH = ctx->n_H, Nc = D - nH;
  if (nH < 1 || Nc < 1 || Nc > ctx->max_N || !ctx->ef_LH || !ctx->B_H) return KS_OK;
  KS_TRY(ensure_blas(ctx));
  cublasHandle_t hb = (cublasHandle_t)ctx->cublas;
  cusolverDnHandle_t h = (cusolverDnHandle_t)ctx->cusolver;
  cudaStream_t st = ctx->stream;
  const double one = 1.0, mone = -1.0, zero = 0.0;
  int lw = 0;
  if (ctx->ef_LH_state == 0) {   // once per coarse space: L_H = chol(B_H), L_H^-1
    ctx->ef_LH_state = -1;
    KS_CUDA(ctx, cudaMemcpyAsync(ctx->ef_LH, ctx->B_H, sizeof(double) * nH * nH, cudaMemcpyDeviceToDevice, st));
    if (cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, (int)nH, ctx->ef_LH, (int)nH, &lw) !=
            CUSOLVER_STATUS_SUCCESS || lw > ctx->ext_lwork)
      return KS_OK;
    if (cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, (int)nH, ctx->ef_LH, (int)nH, ctx->eig_work, lw, ctx->eig_info) !=
        CUSOLVER_STATUS_SUCCESS)
      return KS_OK;
    ctx->launches++;
    int info = 0;
    KS_CUDA(ctx, cudaMemcpyAsync(&info, ctx->eig_info, sizeof(int), cudaMemcpyDeviceToHost, st));
    KS_CUDA(ctx, cudaStreamSynchronize(st));
    if (info != 0) return KS_OK;
    k_lower_only<<<ks_blocks(nH * nH, 256), 256, 0, st>>>(ctx->ef_LH, nH);
    KS_LAUNCHED(ctx);
    k_identity<<<ks_blocks(nH * nH, 256), 256, 0, st>>>(ctx->ef_LHinv, nH);
    KS_LAUNCHED(ctx);
    KS_BLAS(ctx, cublasDtrsm(hb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, (int)nH,
                             (int)nH, &one, ctx->ef_LH, (int)nH, ctx->ef_LHinv, (int)nH));
    ctx->ef_LH_state = 1;
  }
  if (ctx->ef_LH_state != 1) return KS_OK;
  double *Kt = ctx->ef_aux, *S = Kt + nH * Nc, *LSinv = S + Nc * Nc, *T = LSinv + Nc * Nc;   // T [Nc][nH]
  int *mism = reinterpret_cast<int *>(T + Nc * nH);
  KS_CUDA(ctx, cudaMemsetAsync(mism, 0, sizeof(int), st));
  k_block_mismatch<<<ks_blocks(nH * nH, 256), 256, 0, st>>>(FB, D, ctx->B_H, nH, mism);
  KS_LAUNCHED(ctx);
  // Kt = L_H^-1 c (nH x Nc), S = gamma - Kt^T Kt
  KS_BLAS(ctx, cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, (int)nH, (int)Nc, (int)nH, &one, ctx->ef_LHinv, (int)nH,
                           FB + nH * D, (int)D, &zero, Kt, (int)nH));
  KS_CUDA(ctx, cudaMemcpy2DAsync(S, sizeof(double) * Nc, FB + nH * D + nH, sizeof(double) * D, sizeof(double) * Nc, Nc,
                                 cudaMemcpyDeviceToDevice, st));
  KS_BLAS(ctx, cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, (int)Nc, (int)Nc, (int)nH, &mone, Kt, (int)nH, Kt, (int)nH,
                           &one, S, (int)Nc));
  if (cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, (int)Nc, S, (int)Nc, &lw) != CUSOLVER_STATUS_SUCCESS ||
      lw > ctx->ext_lwork)
    return KS_OK;
  if (cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, (int)Nc, S, (int)Nc, ctx->eig_work, lw, ctx->eig_info) !=
      CUSOLVER_STATUS_SUCCESS)
    return KS_OK;
  ctx->launches++;
  int hv[2] = {0, 0};
  KS_CUDA(ctx, cudaMemcpyAsync(&hv[0], mism, sizeof(int), cudaMemcpyDeviceToHost, st));
  KS_CUDA(ctx, cudaMemcpyAsync(&hv[1], ctx->eig_info, sizeof(int), cudaMemcpyDeviceToHost, st));
  KS_CUDA(ctx, cudaStreamSynchronize(st));
  if (hv[0] != 0 || hv[1] != 0) return KS_OK;   // not the cached coarse block, or the Schur complement not SPD
  k_lower_only<<<ks_blocks(Nc * Nc, 256), 256, 0, st>>>(S, Nc);
  KS_LAUNCHED(ctx);
  k_identity<<<ks_blocks(Nc * Nc, 256), 256, 0, st>>>(LSinv, Nc);
  KS_LAUNCHED(ctx);
  KS_BLAS(ctx, cublasDtrsm(hb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, (int)Nc,
                           (int)Nc, &one, S, (int)Nc, LSinv, (int)Nc));
  k_build_L<<<ks_blocks(D * D, 256), 256, 0, st>>>(ctx->ef_LH, ctx->ef_LHinv, Kt, S, LSinv, nH, Nc, ctx->eig_B,
                                                     ctx->ef_Linv);
  KS_LAUNCHED(ctx);
  // bottom-left block of L^-1: -L_S^-1 K L_H^-1 = -L_S^-1 (Kt^T L_H^-1)
  KS_BLAS(ctx, cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, (int)Nc, (int)nH, (int)nH, &one, Kt, (int)nH, ctx->ef_LHinv,
                           (int)nH, &zero, T, (int)Nc));
  KS_BLAS(ctx, cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, (int)Nc, (int)nH, (int)Nc, &mone, LSinv, (int)Nc, T, (int)Nc,
                           &zero, ctx->ef_Linv + nH, (int)D));
  *ok = true;
  return KS_OK;
}

ks_status ks_pencil_eig_impl(ks_ctx *ctx, int64_t D, int k, const double *FA, const double *FB, double *evals,
                             double *evecs, const double *Ywarm, bool same_B) {
  KS_TRY(ensure_solver_handle(ctx));
  cusolverDnHandle_t h = (cusolverDnHandle_t)ctx->cusolver;
  if (!(ctx->ext_features & (KS_EXT_EIG | KS_EXT_SCF)))
    return ks_fail(ctx, KS_E_STATE, "ks_pencil_eig: attach an extension workspace planned with KS_EXT_EIG");
  if (D > ctx->ext_D)
    return ks_fail(ctx, KS_E_WORKSPACE, "ks_pencil_eig: D = %lld exceeds the ext plan's %lld", (long long)D,
                   (long long)ctx->ext_D);
  // symmetric matrices: row-major == column-major
  const char *dense = getenv("KS_PENCIL_DENSE");
  const bool filtered = !(dense && dense[0] == '1') && k <= ctx->max_N && k + ef_guard() <= D / 2;
  const bool have_L = filtered && same_B && ctx->ef_L_D == D;
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->eig_A, FA, sizeof(double) * D * D, cudaMemcpyDeviceToDevice, ctx->stream));
  if (!have_L)
    KS_CUDA(ctx, cudaMemcpyAsync(ctx->eig_B, FB, sizeof(double) * D * D, cudaMemcpyDeviceToDevice, ctx->stream));
  ctx->ef_L_D = 0;   // eig_B holds F_B (or L below)
  // the filtered subspace iteration for the lowest k when the block is small against D (KS_PENCIL_DENSE=1:
  // always the dense cuSOLVER path below; it is also the fallback)
  bool fast = false;
  if (filtered && !have_L) KS_TRY(coarse_chol_reduction(ctx, D, FB, &fast));
  if (filtered) {
    if (!have_L && !fast) {
    int lw = 0;
    if (cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, (int)D, ctx->eig_B, (int)D, &lw) !=
        CUSOLVER_STATUS_SUCCESS)
      return ks_fail(ctx, KS_E_CUDA, "cusolverDnDpotrf_bufferSize failed");
    if (lw > ctx->ext_lwork) return ks_fail(ctx, KS_E_WORKSPACE, "potrf workspace %d exceeds the ext plan", lw);
    if (cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, (int)D, ctx->eig_B, (int)D, ctx->eig_work, lw, ctx->eig_info) !=
        CUSOLVER_STATUS_SUCCESS)
      return ks_fail(ctx, KS_E_CUDA, "cusolverDnDpotrf failed");
    ctx->launches++;
    int pinfo = 0;
    KS_CUDA(ctx, cudaMemcpyAsync(&pinfo, ctx->eig_info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (pinfo > 0)
      return ks_fail(ctx, KS_E_RANK, "F_B is not positive definite (leading minor %d): W = [P | U~] is rank deficient",
                     pinfo);
    }
    ctx->ef_L_D = D;   // eig_B = L
    bool done = false;
    KS_TRY(pencil_eig_filtered(ctx, D, k, evals, evecs, &done, Ywarm, fast ? ctx->ef_Linv : nullptr));
    if (done) return KS_OK;
    ctx->ef_L_D = 0;
    // not converged: the dense path on fresh copies
    KS_CUDA(ctx, cudaMemcpyAsync(ctx->eig_A, FA, sizeof(double) * D * D, cudaMemcpyDeviceToDevice, ctx->stream));
    KS_CUDA(ctx, cudaMemcpyAsync(ctx->eig_B, FB, sizeof(double) * D * D, cudaMemcpyDeviceToDevice, ctx->stream));
  }
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
  if (lwork > ctx->ext_lwork)
    return ks_fail(ctx, KS_E_WORKSPACE, "eigensolver workspace %d exceeds the ext plan", lwork);
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
  const int64_t D = ctx->n_H + N;
  if (!(ctx->ext_features & (KS_EXT_EIG | KS_EXT_SCF)) || N > ctx->max_N)
    return ks_fail(ctx, KS_E_STATE, "ks_augmented_solve: attach an extension workspace planned with KS_EXT_EIG");
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
