// ks_scf.cu -- NEXT-2: the nonlinear terms of the Kohn-Sham operator on the fine mesh.
//   ks_density   nodal density rho = f sum_i psi_i^2 (occupation f, reading R6)
//   ks_vxc       LDA exchange + Perdew-Zunger correlation potential (Eqs. expot, copot)
// Pointwise over all nodes, fp64 (libdevice cbrt / log / sqrt).
#include <cmath>
#include <cstdlib>
#include <vector>

#include "ks_internal.cuh"
#include "ks_layout.cuh"

namespace {

// 4 lanes per node: lane q sums u_ij^2 over j = q, q + 4, ... (each warp load covers 8 full 32-byte row
// segments), then a fixed 2-step butterfly; Dirichlet nodes get 0.
__global__ void k_density(const int32_t *__restrict__ free_of_node, const double *__restrict__ U, int N, double f,
                          int64_t n_nodes, double *__restrict__ rho) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t v = g >> 2;
  const int q = (int)(g & 3);
  const bool valid = v < n_nodes;   // no early return: the butterfly needs all 4 lanes
  const int32_t i = valid ? __ldg(free_of_node + v) : -1;
  double s = 0.0;
  if (i >= 0)
    for (int j = q; j < N; j += 4) {
      const double u = __ldg(U + (int64_t)i * N + j);
      s = fma(u, u, s);
    }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  if (valid && q == 0) rho[v] = f * s;
}

__global__ void k_vxc(const double *__restrict__ rho, int64_t n, double *__restrict__ vxc, double *__restrict__ eps) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  const double A = 0.0311, B = -0.048, C = 0.0020, D = -0.0116, G = -0.1423, B1 = 1.0529, B2 = 0.3334;
  const double r = rho[v];
  double vv = 0.0, ee = 0.0;
  if (r > 0.0) {
    const double vx = -cbrt(3.0 * r / CUDART_PI);
    const double rs = cbrt(3.0 / (4.0 * CUDART_PI * r));
    double vc, ec;
    if (rs < 1.0) {
      const double l = log(rs);
      ec = A * l + B + C * rs * l + D * rs;
      vc = A * l + (B - A / 3.0) + (2.0 / 3.0) * C * rs * l + (1.0 / 3.0) * (2.0 * D - C) * rs;
    } else {
      const double sq = sqrt(rs), den = 1.0 + B1 * sq + B2 * rs;
      ec = G / den;
      vc = ec * (1.0 + (7.0 / 6.0) * B1 * sq + (4.0 / 3.0) * B2 * rs) / den;
    }
    vv = vx + vc;
    ee = 0.75 * vx + ec;
  }
  vxc[v] = vv;
  if (eps) eps[v] = ee;
}

}  // namespace

ks_status ks_density_impl(ks_ctx *ctx, int N, const double *U, double f, double *rho) {
  k_density<<<ks_blocks(4 * ctx->n_nodes, 256), 256, 0, ctx->stream>>>(ctx->free_of_node, U, N, f, ctx->n_nodes, rho);
  KS_LAUNCHED(ctx);
  return KS_OK;
}

ks_status ks_vxc_impl(ks_ctx *ctx, const double *rho, double *vxc, double *eps) {
  k_vxc<<<ks_blocks(ctx->n_nodes, 256), 256, 0, ctx->stream>>>(rho, ctx->n_nodes, vxc, eps);
  KS_LAUNCHED(ctx);
  return KS_OK;
}

// ---------------------------------------------------------------------------------------------
// Hartree potential: -Lap V = 4 pi rho, V = w_D (multipole expansion, Eq. bd, with the
// 1/2 of the quadrupole Taylor term: DESIGN.md reading R5) on the boundary; P1 Galerkin with the Dirichlet
// lift, free values by the batched PCG (N = 1) on the stiffness matrix.
// ---------------------------------------------------------------------------------------------
namespace {

constexpr int HB = 256;   // threads per block of the moment / element kernels

// tet geometry: |T| and grad lambda_a (a = 0..3) from the node coordinates
__device__ __forceinline__ void tet_grads(const double *__restrict__ xyz, int4 v, double &vol, double g[4][3]) {
  const double x0 = xyz[3 * v.x], y0 = xyz[3 * v.x + 1], z0 = xyz[3 * v.x + 2];
  const double J00 = xyz[3 * v.y] - x0, J10 = xyz[3 * v.y + 1] - y0, J20 = xyz[3 * v.y + 2] - z0;
  const double J01 = xyz[3 * v.z] - x0, J11 = xyz[3 * v.z + 1] - y0, J21 = xyz[3 * v.z + 2] - z0;
  const double J02 = xyz[3 * v.w] - x0, J12 = xyz[3 * v.w + 1] - y0, J22 = xyz[3 * v.w + 2] - z0;
  const double det = J00 * (J11 * J22 - J12 * J21) - J01 * (J10 * J22 - J12 * J20) + J02 * (J10 * J21 - J11 * J20);
  vol = det / 6.0;
  // rows of J^-1 are grad lambda_1..3
  g[1][0] = (J11 * J22 - J12 * J21) / det; g[1][1] = (J02 * J21 - J01 * J22) / det; g[1][2] = (J01 * J12 - J02 * J11) / det;
  g[2][0] = (J12 * J20 - J10 * J22) / det; g[2][1] = (J00 * J22 - J02 * J20) / det; g[2][2] = (J02 * J10 - J00 * J12) / det;
  g[3][0] = (J10 * J21 - J11 * J20) / det; g[3][1] = (J01 * J20 - J00 * J21) / det; g[3][2] = (J00 * J11 - J01 * J10) / det;
  for (int d = 0; d < 3; d++) g[0][d] = -(g[1][d] + g[2][d] + g[3][d]);
}

// block partials of NV moment values, fixed order (per-thread values, then a shared-memory tree)
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double *sm, double *out) {
  for (int k = 0; k < NV; k++) sm[k * HB + threadIdx.x] = v[k];
  __syncthreads();
  for (int s = HB / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int k = 0; k < NV; k++) sm[k * HB + threadIdx.x] += sm[k * HB + threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x < NV) out[(int64_t)blockIdx.x * NV + threadIdx.x] = sm[threadIdx.x * HB];
}

// pass 1: Q = int rho, m1 = int rho x (exact for P1 rho: int lambda_a lambda_b = |T| (1 + delta_ab) / 20)
__global__ void __launch_bounds__(HB) k_moments1(const int32_t *__restrict__ tets, const double *__restrict__ vol,
                                                 const double *__restrict__ xyz, const double *__restrict__ rho,
                                                 int64_t nt, double *__restrict__ part) {
  __shared__ double sm[4 * HB];
  double v[4] = {0, 0, 0, 0};
  for (int64_t t = blockIdx.x * (int64_t)HB + threadIdx.x; t < nt; t += (int64_t)gridDim.x * HB) {
    const int4 tv = __ldg(reinterpret_cast<const int4 *>(tets) + t);
    const int32_t id[4] = {tv.x, tv.y, tv.z, tv.w};
    const double V = __ldg(vol + t);
    double r[4], sr = 0.0;
    for (int a = 0; a < 4; a++) { r[a] = __ldg(rho + id[a]); sr += r[a]; }
    v[0] += V * sr / 4.0;
    for (int b = 0; b < 4; b++) {
      const double wb = V * (sr + r[b]) / 20.0;   // sum_a rho_a (1 + delta_ab) |T| / 20
      for (int i = 0; i < 3; i++) v[1 + i] += wb * __ldg(xyz + 3 * id[b] + i);
    }
  }
  block_sum<4>(v, sm, part);
}

// pass 2 about the centre c: p = int rho (x - c), q_ij = int rho (x - c)_i (x - c)_j
// (int lambda_a lambda_b lambda_c = alpha! |T| / 120)
__global__ void __launch_bounds__(HB) k_moments2(const int32_t *__restrict__ tets, const double *__restrict__ vol,
                                                 const double *__restrict__ xyz, const double *__restrict__ rho,
                                                 const double *__restrict__ mom, int64_t nt,
                                                 double *__restrict__ part) {
  __shared__ double sm[9 * HB];
  double v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};   // p0..2, q00 q11 q22 q01 q02 q12
  const double c0 = mom[1], c1 = mom[2], c2 = mom[3];
  for (int64_t t = blockIdx.x * (int64_t)HB + threadIdx.x; t < nt; t += (int64_t)gridDim.x * HB) {
    const int4 tv = __ldg(reinterpret_cast<const int4 *>(tets) + t);
    const int32_t id[4] = {tv.x, tv.y, tv.z, tv.w};
    const double V = __ldg(vol + t);
    double r[4], y[4][3];
    for (int a = 0; a < 4; a++) {
      r[a] = __ldg(rho + id[a]);
      y[a][0] = __ldg(xyz + 3 * id[a]) - c0;
      y[a][1] = __ldg(xyz + 3 * id[a] + 1) - c1;
      y[a][2] = __ldg(xyz + 3 * id[a] + 2) - c2;
    }
    for (int a = 0; a < 4; a++)
      for (int b = 0; b < 4; b++) {
        const double w2 = r[a] * V * (a == b ? 2.0 : 1.0) / 20.0;
        for (int i = 0; i < 3; i++) v[i] += w2 * y[b][i];
        for (int cc = 0; cc < 4; cc++) {
          const double al = (a == b && b == cc) ? 6.0 : ((a == b || b == cc || a == cc) ? 2.0 : 1.0);
          const double w3 = r[a] * V * al / 120.0;
          v[3] += w3 * y[b][0] * y[cc][0];
          v[4] += w3 * y[b][1] * y[cc][1];
          v[5] += w3 * y[b][2] * y[cc][2];
          v[6] += w3 * y[b][0] * y[cc][1];
          v[7] += w3 * y[b][0] * y[cc][2];
          v[8] += w3 * y[b][1] * y[cc][2];
        }
      }
  }
  block_sum<9>(v, sm, part);
}

// fixed-order sum of block partials (warp k sums value k: lane-strided, then a butterfly); pass 1 also forms
// the centre of charge. Launch with 32 * nv threads.
__global__ void k_moments_final(const double *__restrict__ part, int nblk, int nv, int pass, double *__restrict__ mom) {
  __shared__ double s[9];
  const int lane = threadIdx.x & 31, k = threadIdx.x >> 5;
  if (k < nv) {
    double v = 0.0;
    for (int b = lane; b < nblk; b += 32) v += part[(int64_t)b * nv + k];
    v = warp_sum(v);
    if (lane == 0) s[k] = v;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (pass == 1) {
    mom[0] = s[0];
    for (int i = 0; i < 3; i++) mom[1 + i] = s[0] != 0.0 ? s[1 + i] / s[0] : 0.0;
  } else {
    for (int kk = 0; kk < 9; kk++) mom[4 + kk] = s[kk];
  }
}

// multipole boundary values w_D at the Dirichlet nodes (0 elsewhere)
__global__ void k_hartree_boundary(const int32_t *__restrict__ free_of_node, const double *__restrict__ xyz,
                                   const double *__restrict__ mom, int64_t nn, double *__restrict__ w) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= nn) return;
  if (__ldg(free_of_node + v) >= 0) { w[v] = 0.0; return; }
  const double Q = mom[0];
  const double d[3] = {xyz[3 * v] - mom[1], xyz[3 * v + 1] - mom[2], xyz[3 * v + 2] - mom[3]};
  const double q[3][3] = {{mom[7], mom[10], mom[11]}, {mom[10], mom[8], mom[12]}, {mom[11], mom[12], mom[9]}};
  const double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2], r = sqrt(r2);
  double s = Q / r;
  for (int i = 0; i < 3; i++) s += mom[4 + i] * d[i] / (r2 * r);
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) s += 0.5 * q[i][j] * (3.0 * d[i] * d[j] - (i == j ? r2 : 0.0)) / (r2 * r2 * r);
  w[v] = s;
}

// element contributions to the load vector: c[4t + a] = sum_b (4 pi M_T(a,b) rho_b - [b Dirichlet] K_T(a,b) w_b)
__global__ void __launch_bounds__(HB) k_hartree_elem(const int32_t *__restrict__ tets, const double *__restrict__ xyz,
                                                     const int32_t *__restrict__ free_of_node,
                                                     const double *__restrict__ rho, const double *__restrict__ w,
                                                     int64_t nt, double *__restrict__ c) {
  const int64_t t = blockIdx.x * (int64_t)HB + threadIdx.x;
  if (t >= nt) return;
  const int4 tv = __ldg(reinterpret_cast<const int4 *>(tets) + t);
  const int32_t id[4] = {tv.x, tv.y, tv.z, tv.w};
  double V, g[4][3];
  tet_grads(xyz, tv, V, g);
  bool dir[4];
  double r[4], wb[4];
  for (int b = 0; b < 4; b++) {
    dir[b] = __ldg(free_of_node + id[b]) < 0;
    r[b] = __ldg(rho + id[b]);
    wb[b] = dir[b] ? __ldg(w + id[b]) : 0.0;
  }
  for (int a = 0; a < 4; a++) {
    double s = 0.0;
    for (int b = 0; b < 4; b++) {
      s += 4.0 * CUDART_PI * V * (a == b ? 2.0 : 1.0) / 20.0 * r[b];
      if (dir[b]) s -= V * (g[a][0] * g[b][0] + g[a][1] * g[b][1] + g[a][2] * g[b][2]) * wb[b];
    }
    c[4 * t + a] = s;
  }
}

// per free node: sum of its element contributions in ascending element order (the inverse map of the
// diagonal entry lists exactly the (t, a) with v_a = node)
__global__ void k_hartree_rhs(const int32_t *__restrict__ diag_pos, const int32_t *__restrict__ inv_ptr,
                              const int32_t *__restrict__ inv_idx, const double *__restrict__ c, int64_t n,
                              double *__restrict__ b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t e = __ldg(diag_pos + i);
  double s = 0.0;
  for (int32_t q = __ldg(inv_ptr + e); q < __ldg(inv_ptr + e + 1); q++) {
    const int32_t m = __ldg(inv_idx + q);   // 16 t + 4 a + a
    s += __ldg(c + 4 * (int64_t)(m >> 4) + ((m >> 2) & 3));
  }
  b[i] = s;
}

__global__ void k_gather_free(const int32_t *__restrict__ node_of_free, const double *__restrict__ vn, int64_t n,
                              double *__restrict__ x) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[i] = vn[__ldg(node_of_free + i)];
}

__global__ void k_hartree_out(const int32_t *__restrict__ free_of_node, const double *__restrict__ x,
                              const double *__restrict__ w, int64_t nn, double *__restrict__ vh) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= nn) return;
  const int32_t i = __ldg(free_of_node + v);
  vh[v] = i >= 0 ? x[i] : w[v];
}

}  // namespace

ks_status ks_hartree_impl(ks_ctx *ctx, const double *rho, double tol, int max_iter, double *vh, int warm,
                          double *h_mom, int32_t *h_iters) {
  cudaStream_t s = ctx->stream;
  const int64_t nn = ctx->n_nodes, nt = ctx->n_tets, n = ctx->n_free;
  if (!(ctx->ext_features & KS_EXT_SCF))
    return ks_fail(ctx, KS_E_STATE, "ks_hartree: attach an extension workspace planned with KS_EXT_SCF");
  const int nblk = 8 * ctx->sm_count;   // latency-bound gathers over the tets: 8 blocks per SM
  k_moments1<<<nblk, HB, 0, s>>>(ctx->tets, ctx->vol, ctx->xyz, rho, nt, ctx->har_part);
  KS_LAUNCHED(ctx);
  k_moments_final<<<1, 32 * 4, 0, s>>>(ctx->har_part, nblk, 4, 1, ctx->har_mom);
  KS_LAUNCHED(ctx);
  k_moments2<<<nblk, HB, 0, s>>>(ctx->tets, ctx->vol, ctx->xyz, rho, ctx->har_mom, nt, ctx->har_part);
  KS_LAUNCHED(ctx);
  k_moments_final<<<1, 32 * 9, 0, s>>>(ctx->har_part, nblk, 9, 2, ctx->har_mom);
  KS_LAUNCHED(ctx);
  k_hartree_boundary<<<ks_blocks(nn, 256), 256, 0, s>>>(ctx->free_of_node, ctx->xyz, ctx->har_mom, nn, ctx->har_w);
  KS_LAUNCHED(ctx);
  k_hartree_elem<<<ks_blocks(nt, HB), HB, 0, s>>>(ctx->tets, ctx->xyz, ctx->free_of_node, rho, ctx->har_w, nt,
                                                 ctx->har_c);
  KS_LAUNCHED(ctx);
  k_hartree_rhs<<<ks_blocks(n, 256), 256, 0, s>>>(ctx->diag_pos, ctx->inv_ptr, ctx->inv_idx, ctx->har_c, n,
                                                  ctx->har_b);
  KS_LAUNCHED(ctx);
  if (warm) {
    k_gather_free<<<ks_blocks(n, 256), 256, 0, s>>>(ctx->node_of_free, vh, n, ctx->har_x0);
    KS_LAUNCHED(ctx);
  } else {
    KS_CUDA(ctx, cudaMemsetAsync(ctx->har_x0, 0, sizeof(double) * n, s));
  }
  // two-level preconditioner on the coarse space of ks_set_coarse when one is set (ks_pcg2l.cu, DESIGN.md
  // §8.4); KS_HARTREE_2L=0 or no coarse space: the Jacobi-PCG of ks_pcg.cu
  const char *e2l = getenv("KS_HARTREE_2L");
  ks_status st2 = KS_E_STATE;
  if (!(e2l && e2l[0] == '0')) {
    st2 = ks_pcg2l_run(ctx, ctx->har_b, ctx->har_x0, ctx->har_x, tol, max_iter, ctx->har_iters);
    if (st2 != KS_OK && st2 != KS_E_STATE) return st2;
  }
  if (st2 != KS_OK)
    KS_TRY(ks_pcg_run(ctx, ctx->sell_K, ctx->dinvK, 0.0, 1, nullptr, ctx->har_b, ctx->har_x0, ctx->har_x, tol,
                      max_iter, ctx->har_iters, nullptr));
  k_hartree_out<<<ks_blocks(nn, 256), 256, 0, s>>>(ctx->free_of_node, ctx->har_x, ctx->har_w, nn, vh);
  KS_LAUNCHED(ctx);
  if (h_mom || h_iters) {
    double mom[13];
    int32_t it = 0;
    KS_CUDA(ctx, cudaMemcpyAsync(mom, ctx->har_mom, sizeof(double) * 13, cudaMemcpyDeviceToHost, s));
    KS_CUDA(ctx, cudaMemcpyAsync(&it, ctx->har_iters, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    KS_CUDA(ctx, cudaStreamSynchronize(s));
    if (h_mom) {   // Q, centre, dipole, diagonal quadrupole (the oracle's layout)
      for (int k = 0; k < 10; k++) h_mom[k] = mom[k];
    }
    if (h_iters) *h_iters = it;
  }
  return KS_OK;
}

// ---------------------------------------------------------------------------------------------
// Algorithm 3 for the Kohn-Sham equation with Anderson mixing
// ---------------------------------------------------------------------------------------------
namespace {

constexpr int SB = 256;
constexpr int AMAX = 8;   // largest Anderson depth

__global__ void k_veff(const double *__restrict__ vext, const double *__restrict__ vh, const double *__restrict__ vxc,
                       int64_t n, double *__restrict__ veff) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v < n) veff[v] = vext[v] + vh[v] + vxc[v];
}

// partials of x_f^T (M x_f) for the free part of a nodal vector x = a - b (b may be null): one SELL row per
// thread, fixed-order block tree
__global__ void __launch_bounds__(SB) k_mnorm2(const int32_t *__restrict__ sell_ptr, const int32_t *__restrict__ sell_col,
                                               const double *__restrict__ M, const int32_t *__restrict__ node_of_free,
                                               const double *__restrict__ a, const double *__restrict__ b, int64_t n,
                                               double *__restrict__ part) {
  __shared__ double sm[SB];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)SB + threadIdx.x; i < n; i += (int64_t)gridDim.x * SB) {
    const int64_t s = i / KS_SELL_C;
    const int32_t bs = __ldg(sell_ptr + s), e = __ldg(sell_ptr + s + 1);
    const int K = (e - bs) / KS_SELL_C;
    const int64_t base = bs + (i % KS_SELL_C) * 4;
    const int64_t vi = __ldg(node_of_free + i);
    const double xi = __ldg(a + vi) - (b ? __ldg(b + vi) : 0.0);
    double mx = 0.0;
    for (int k = 0; k < K; k++) {
      const int64_t o = base + (k >> 2) * (4 * KS_SELL_C) + (k & 3);
      const int64_t vj = __ldg(node_of_free + __ldg(sell_col + o));
      const double xj = __ldg(a + vj) - (b ? __ldg(b + vj) : 0.0);
      mx = fma(__ldg(M + o), xj, mx);
    }
    acc = fma(xi, mx, acc);
  }
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int st = SB / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) sm[threadIdx.x] += sm[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}

// Anderson Gram: with F_j = out_j - in_j (slots in age order, m = newest), D_j = F_m - F_j (j < m):
// G[j][k] = (D_j, D_k), r[j] = (D_j, F_m); partials [nblk][m*m + m]
__global__ void __launch_bounds__(SB) k_anderson_gram(const double *__restrict__ hin, const double *__restrict__ hout,
                                                      const int *__restrict__ slot, int m, int64_t n,
                                                      double *__restrict__ part) {
  __shared__ double sm[(AMAX * AMAX + AMAX) * 32];
  const int nv = m * m + m;
  double acc[AMAX * AMAX + AMAX];
  for (int k = 0; k < nv; k++) acc[k] = 0.0;
  const int64_t sm_ = slot[m];
  for (int64_t v = blockIdx.x * (int64_t)SB + threadIdx.x; v < n; v += (int64_t)gridDim.x * SB) {
    const double Fm = hout[sm_ * n + v] - hin[sm_ * n + v];
    double D[AMAX];
    for (int j = 0; j < m; j++) D[j] = Fm - (hout[(int64_t)slot[j] * n + v] - hin[(int64_t)slot[j] * n + v]);
    for (int j = 0; j < m; j++) {
      for (int k = 0; k < m; k++) acc[j * m + k] += D[j] * D[k];
      acc[m * m + j] += D[j] * Fm;
    }
  }
  // fixed-order: warp butterflies, then warps in order
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = 0; k < nv; k++) {
    double s = acc[k];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) sm[k * 32 + warp] = s;
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double s = 0.0;
    for (int w = 0; w < SB / 32; w++) s += sm[threadIdx.x * 32 + w];
    part[(int64_t)blockIdx.x * nv + threadIdx.x] = s;
  }
}

__global__ void k_sum_partials(const double *__restrict__ part, int nblk, int nv, double *__restrict__ out) {
  const int k = threadIdx.x;
  if (k >= nv) return;
  double s = 0.0;
  for (int b = 0; b < nblk; b++) s += part[(int64_t)b * nv + k];
  out[k] = s;
}

// rho = beta (out_m + sum a_j (out_j - out_m)) + (1 - beta)(in_m + sum a_j (in_j - in_m))
__global__ void k_anderson_combine(const double *__restrict__ hin, const double *__restrict__ hout,
                                   const int *__restrict__ slot, const double *__restrict__ alpha, int m,
                                   double beta, int64_t n, double *__restrict__ rho) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int64_t sm_ = slot[m];
  const double im = hin[sm_ * n + v], om = hout[sm_ * n + v];
  double ti = im, to = om;
  for (int j = 0; j < m; j++) {
    ti += alpha[j] * (hin[(int64_t)slot[j] * n + v] - im);
    to += alpha[j] * (hout[(int64_t)slot[j] * n + v] - om);
  }
  rho[v] = beta * to + (1.0 - beta) * ti;
}

}  // namespace

static ks_status scf_alloc(ks_ctx *ctx, int N, int depth) {
  if (!(ctx->ext_features & KS_EXT_SCF) || ctx->ext_nH != ctx->n_H)
    return ks_fail(ctx, KS_E_STATE, "ks_scf_solve: attach an extension workspace planned with KS_EXT_SCF for this "
                   "coarse space");
  if (N > ctx->max_N || depth > KS_EXT_DEPTH_MAX || ctx->n_H + N > ctx->ext_D)
    return ks_fail(ctx, KS_E_WORKSPACE, "ks_scf_solve: N = %d / depth = %d exceed the extension plan", N, depth);
  return KS_OK;
}

// ||a - b||_M over the free nodes (b may be null), synchronises
static ks_status mnorm(ks_ctx *ctx, const double *a, const double *b, double *out) {
  const int nblk = 4 * ctx->sm_count;
  k_mnorm2<<<nblk, SB, 0, ctx->stream>>>(ctx->sell_ptr, ctx->sell_col, ctx->sell_M, ctx->node_of_free, a, b,
                                          ctx->n_free, ctx->scf_part);
  KS_LAUNCHED(ctx);
  k_sum_partials<<<1, 32, 0, ctx->stream>>>(ctx->scf_part, nblk, 1, ctx->scf_red);
  KS_LAUNCHED(ctx);
  double v = 0.0;
  KS_CUDA(ctx, cudaMemcpyAsync(&v, ctx->scf_red, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  *out = std::sqrt(v > 0.0 ? v : 0.0);
  return KS_OK;
}

static ks_status make_veff(ks_ctx *ctx, const double *vext, const double *rho, double hartree_tol, bool warm) {
  KS_TRY(ks_hartree_impl(ctx, rho, hartree_tol, 100000, ctx->scf_vh, warm ? 1 : 0, nullptr, nullptr));
  KS_TRY(ks_vxc_impl(ctx, rho, ctx->scf_vxc, nullptr));
  k_veff<<<ks_blocks(ctx->n_nodes, 256), 256, 0, ctx->stream>>>(vext, ctx->scf_vh, ctx->scf_vxc, ctx->n_nodes,
                                                                ctx->scf_veff);
  KS_LAUNCHED(ctx);
  return KS_OK;
}

// Anderson step over the history slots (age order in `order`, newest last): rho_next into ctx->scf_in
static ks_status anderson(ks_ctx *ctx, const std::vector<int> &order, double beta) {
  const int m = (int)order.size() - 1;
  const int64_t nn = ctx->n_nodes;
  std::vector<int> slot(order);
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->scf_slot, slot.data(), sizeof(int) * slot.size(), cudaMemcpyHostToDevice, ctx->stream));
  std::vector<double> alpha(AMAX, 0.0);
  if (m > 0) {
    const int nv = m * m + m, nblk = 4 * ctx->sm_count;
    k_anderson_gram<<<nblk, SB, 0, ctx->stream>>>(ctx->scf_hin, ctx->scf_hout, ctx->scf_slot, m, nn, ctx->scf_part);
    KS_LAUNCHED(ctx);
    k_sum_partials<<<1, 128, 0, ctx->stream>>>(ctx->scf_part, nblk, nv, ctx->scf_red);
    KS_LAUNCHED(ctx);
    std::vector<double> g(nv);
    KS_CUDA(ctx, cudaMemcpyAsync(g.data(), ctx->scf_red, sizeof(double) * nv, cudaMemcpyDeviceToHost, ctx->stream));
    KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    // (mix6): G alpha = r by Gaussian elimination with partial pivoting (m <= AMAX - 1)
    std::vector<double> A(m * m), r(m);
    for (int j = 0; j < m; j++) {
      r[j] = g[m * m + j];
      for (int k = 0; k < m; k++) A[j * m + k] = g[j * m + k];
    }
    for (int c = 0; c < m; c++) {
      int piv = c;
      for (int q = c + 1; q < m; q++)
        if (std::fabs(A[q * m + c]) > std::fabs(A[piv * m + c])) piv = q;
      if (!(std::fabs(A[piv * m + c]) > 0.0)) return ks_fail(ctx, KS_E_NONFINITE, "Anderson mixing: singular system");
      if (piv != c) {
        for (int k = 0; k < m; k++) std::swap(A[c * m + k], A[piv * m + k]);
        std::swap(r[c], r[piv]);
      }
      for (int q = c + 1; q < m; q++) {
        const double l = A[q * m + c] / A[c * m + c];
        for (int k = c; k < m; k++) A[q * m + k] -= l * A[c * m + k];
        r[q] -= l * r[c];
      }
    }
    for (int c = m - 1; c >= 0; c--) {
      double s = r[c];
      for (int k = c + 1; k < m; k++) s -= A[c * m + k] * alpha[k];
      alpha[c] = s / A[c * m + c];
    }
  }
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->scf_alpha, alpha.data(), sizeof(double) * AMAX, cudaMemcpyHostToDevice, ctx->stream));
  k_anderson_combine<<<ks_blocks(nn, 256), 256, 0, ctx->stream>>>(ctx->scf_hin, ctx->scf_hout, ctx->scf_slot,
                                                                   ctx->scf_alpha, m, beta, nn, ctx->scf_in);
  KS_LAUNCHED(ctx);
  KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));   // the host vectors above must outlive the copies
  return KS_OK;
}

ks_status ks_scf_solve_impl(ks_ctx *ctx, int N, const double *vext, double f, double mu, double *lambda, double *U,
                            double tol, int max_outer, int inner, double inner_tol, double beta, int depth,
                            double bvp_tol, double hartree_tol, int32_t *h_outer, int32_t *h_inner, double *h_dres,
                            double *h_lams) {
  KS_TRY(scf_alloc(ctx, N, depth));
  const int64_t nn = ctx->n_nodes, D = ctx->n_H + N;
  cudaStream_t s = ctx->stream;
  KS_TRY(ks_density_impl(ctx, N, U, f, ctx->scf_rho));
  bool warm = false;
  int it = 0;
  ks_status result = KS_E_NOT_CONVERGED;
  while (it < max_outer) {
    KS_TRY(make_veff(ctx, vext, ctx->scf_rho, hartree_tol, warm));
    warm = true;
    KS_TRY(ks_assemble_impl(ctx, ctx->scf_veff, mu));
    KS_TRY(ks_solve_impl(ctx, N, lambda, U, ctx->scf_Ut, bvp_tol, 100000, nullptr, nullptr));
    KS_CUDA(ctx, cudaMemcpyAsync(ctx->scf_in, ctx->scf_rho, sizeof(double) * nn, cudaMemcpyDeviceToDevice, s));
    std::vector<int> order;   // Anderson history slots, oldest first
    int next_slot = 0, k = 0;
    for (k = 0; k < inner; k++) {
      KS_TRY(ks_project_impl(ctx, N, ctx->scf_Ut, ctx->scf_FA, ctx->scf_FB));
      // within the inner loop U~ (hence F_B) is fixed: reuse its Cholesky factor and start the filtered
      // eigensolver from the previous inner step's eigenvectors
      KS_TRY(ks_pencil_eig_impl(ctx, D, N, ctx->scf_FA, ctx->scf_FB, lambda, ctx->scf_Y, k > 0 ? ctx->scf_Y : nullptr,
                                k > 0));
      KS_TRY(ks_lift_impl(ctx, N, ctx->scf_Ut, N, ctx->scf_Y, U));
      KS_TRY(ks_density_impl(ctx, N, U, f, ctx->scf_out));
      double dn = 0.0, on = 0.0;
      KS_TRY(mnorm(ctx, ctx->scf_out, ctx->scf_in, &dn));
      KS_TRY(mnorm(ctx, ctx->scf_out, nullptr, &on));
      if (dn <= inner_tol * on || k == inner - 1) break;
      // push (rho_in, rho_out) into the history ring, then mix
      const int sl = next_slot;
      next_slot = (next_slot + 1) % depth;
      if ((int)order.size() == depth) order.erase(order.begin());
      order.push_back(sl);
      KS_CUDA(ctx, cudaMemcpyAsync(ctx->scf_hin + (int64_t)sl * nn, ctx->scf_in, sizeof(double) * nn,
                                   cudaMemcpyDeviceToDevice, s));
      KS_CUDA(ctx, cudaMemcpyAsync(ctx->scf_hout + (int64_t)sl * nn, ctx->scf_out, sizeof(double) * nn,
                                   cudaMemcpyDeviceToDevice, s));
      KS_TRY(anderson(ctx, order, beta));
      KS_TRY(make_veff(ctx, vext, ctx->scf_in, hartree_tol, true));
      KS_TRY(ks_assemble_impl(ctx, ctx->scf_veff, mu));
    }
    double ch = 0.0, on = 0.0;
    KS_TRY(mnorm(ctx, ctx->scf_out, ctx->scf_rho, &ch));
    KS_TRY(mnorm(ctx, ctx->scf_out, nullptr, &on));
    const double change = on > 0.0 ? ch / on : ch;
    if (h_dres) h_dres[it] = change;
    if (h_inner) h_inner[it] = k + 1;
    if (h_lams) {
      KS_CUDA(ctx, cudaMemcpyAsync(h_lams + (int64_t)it * N, lambda, sizeof(double) * N, cudaMemcpyDeviceToHost, s));
      KS_CUDA(ctx, cudaStreamSynchronize(s));
    }
    KS_CUDA(ctx, cudaMemcpyAsync(ctx->scf_rho, ctx->scf_out, sizeof(double) * nn, cudaMemcpyDeviceToDevice, s));
    it++;
    if (!(change == change)) { result = KS_E_NONFINITE; break; }
    if (change <= tol) { result = KS_OK; break; }
  }
  if (h_outer) *h_outer = it;
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  if (result != KS_OK) return ks_fail(ctx, result, "ks_scf_solve: %d outer iterations without reaching tol %g", it, tol);
  return KS_OK;
}
