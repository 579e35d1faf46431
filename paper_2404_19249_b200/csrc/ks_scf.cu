// ks_scf.cu -- NEXT-2: the nonlinear terms of the Kohn-Sham operator on the fine mesh.
//   ks_density   nodal density rho = f sum_i psi_i^2 (occupation f, reading R6)
//   ks_vxc       LDA exchange + Perdew-Zunger correlation potential (Eqs. expot, copot)
// Pointwise over all nodes, fp64 (libdevice cbrt / log / sqrt).
#include "ks_internal.cuh"

namespace {

__global__ void k_density(const int32_t *__restrict__ free_of_node, const double *__restrict__ U, int N, double f,
                          int64_t n_nodes, double *__restrict__ rho) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n_nodes) return;
  const int32_t i = __ldg(free_of_node + v);
  double s = 0.0;
  if (i >= 0)
    for (int j = 0; j < N; j++) {
      const double u = __ldg(U + (int64_t)i * N + j);
      s += u * u;
    }
  rho[v] = f * s;
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
  k_density<<<ks_blocks(ctx->n_nodes, 256), 256, 0, ctx->stream>>>(ctx->free_of_node, U, N, f, ctx->n_nodes, rho);
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

// fixed-order sum of block partials; pass 1 also forms the centre of charge
__global__ void k_moments_final(const double *__restrict__ part, int nblk, int nv, int pass, double *__restrict__ mom) {
  if (threadIdx.x != 0) return;
  double s[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int b = 0; b < nblk; b++)
    for (int k = 0; k < nv; k++) s[k] += part[(int64_t)b * nv + k];
  if (pass == 1) {
    mom[0] = s[0];
    for (int i = 0; i < 3; i++) mom[1 + i] = s[0] != 0.0 ? s[1 + i] / s[0] : 0.0;
  } else {
    for (int k = 0; k < 9; k++) mom[4 + k] = s[k];
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
  if (!ctx->har_w) {
    KS_TRY(ks_alloc_t(ctx, &ctx->har_w, nn, "hartree w"));
    KS_TRY(ks_alloc_t(ctx, &ctx->har_c, 4 * nt, "hartree element loads"));
    KS_TRY(ks_alloc_t(ctx, &ctx->har_b, n, "hartree rhs"));
    KS_TRY(ks_alloc_t(ctx, &ctx->har_x0, n, "hartree x0"));
    KS_TRY(ks_alloc_t(ctx, &ctx->har_x, n, "hartree x"));
    KS_TRY(ks_alloc_t(ctx, &ctx->har_mom, 16, "hartree moments"));
    KS_TRY(ks_alloc_t(ctx, &ctx->har_part, 9 * 2 * (int64_t)ctx->sm_count, "hartree partials"));
    KS_TRY(ks_alloc_t(ctx, &ctx->har_iters, 1, "hartree iterations"));
  }
  const int nblk = 2 * ctx->sm_count;
  k_moments1<<<nblk, HB, 0, s>>>(ctx->tets, ctx->vol, ctx->xyz, rho, nt, ctx->har_part);
  KS_LAUNCHED(ctx);
  k_moments_final<<<1, 32, 0, s>>>(ctx->har_part, nblk, 4, 1, ctx->har_mom);
  KS_LAUNCHED(ctx);
  k_moments2<<<nblk, HB, 0, s>>>(ctx->tets, ctx->vol, ctx->xyz, rho, ctx->har_mom, nt, ctx->har_part);
  KS_LAUNCHED(ctx);
  k_moments_final<<<1, 32, 0, s>>>(ctx->har_part, nblk, 9, 2, ctx->har_mom);
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
  KS_TRY(ks_pcg_run(ctx, ctx->sell_K, ctx->dinvK, 0.0, 1, nullptr, ctx->har_b, ctx->har_x0, ctx->har_x, tol, max_iter,
                    ctx->har_iters, nullptr));
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
