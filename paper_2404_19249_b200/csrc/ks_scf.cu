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
