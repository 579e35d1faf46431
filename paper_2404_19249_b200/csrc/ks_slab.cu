// ks_slab.cu -- the row-slab partition of one block solve over several GPUs (
// the paper's work model of the BVPs split over processes).
//
// Rank r owns a contiguous range of rows [row0, row1) of the free numbering (balanced by nonzeros). The phases
// of the fused two-phase Jacobi-PCG (ks_pcg.cu k_block_pcg_fused) run as separate launches over that range,
// so that a multi-process driver (paper_2404_19249_b200/slab.py) can exchange the halo rows of z with the
// neighbouring ranks before each S phase and all-gather the per-column dot products after each phase:
//   init  b = (lambda+mu) M u, r = b - A u, z = r / d, p = z                 dots: b.b, r.z, r.r
//   S     w = A z (rows of z up to the halo), q = w + beta q, p' = z + beta p, x += alpha_x p   dots: p'.q
//   U     z -= alpha q / d                                                  dots: r.z = d z^2, r.r = (d z)^2
//   X     x += alpha_x p (the deferred update after the last iteration)
// The partition itself (slab bounds, halo ranges, exchange schedule) is host logic of the driver.
// Vectors are [n][NP] row-major in the global numbering (NP = a power of two >= N, pad columns zero); a rank
// reads and writes only its own rows (and reads the halo rows of z and u). The per-block partial sums are
// reduced in a fixed order into dots[k][NP] (deterministic); the coefficients alpha, beta come from the driver,
// which sums the ranks' dots in rank order, so every rank holds the same coefficients.
#include "ks_internal.cuh"
#include "ks_layout.cuh"
#include "ks_sell.cuh"

namespace {

constexpr int SB_THREADS = 256;
constexpr int SB_WARPS = SB_THREADS / 32;

struct SlabCoef {
  double a[KS_MAX_N], b[KS_MAX_N];
};

// per-block column sums acc[d][v] (column (VEC lane + v) % NP) -> part[blockIdx][d][NP], fixed order
template <int NP, int ND>
__device__ __forceinline__ void slab_block_cols(double (&acc)[ND][SL<NP, SB_THREADS>::VEC], double *red,
                                                double *part) {
  constexpr int VEC = SL<NP, SB_THREADS>::VEC, LPR = SL<NP, SB_THREADS>::LPR;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 0; d < ND; d++)
#pragma unroll
    for (int v = 0; v < VEC; v++) {
      double s = acc[d][v];
#pragma unroll
      for (int o = LPR; o < 32; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane < LPR) red[(warp * ND + d) * NP + lane * VEC + v] = s;
    }
  __syncthreads();
  for (int i = threadIdx.x; i < ND * NP; i += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < SB_WARPS; w++) s += red[w * ND * NP + i];
    part[(int64_t)blockIdx.x * ND * NP + i] = s;
  }
}

template <int NP>
__global__ void __launch_bounds__(SB_THREADS) k_slab_init(const int32_t *__restrict__ sell_ptr,
                                                          const int32_t *__restrict__ sell_col,
                                                          const double *__restrict__ A, const double *__restrict__ M,
                                                          const double *__restrict__ dinv,
                                                          const double *__restrict__ lambda, double mu,
                                                          const double *__restrict__ U, double *__restrict__ Z,
                                                          double *__restrict__ P, int64_t row0, int64_t row1,
                                                          double *__restrict__ part) {
  constexpr int VEC = SL<NP, SB_THREADS>::VEC, LPR = SL<NP, SB_THREADS>::LPR, RPW = SL<NP, SB_THREADS>::RPW,
                TILE = SL<NP, SB_THREADS>::TILE;
  __shared__ double red[SB_WARPS * 3 * NP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, slot = lane / LPR, sub = lane % LPR;
  double acc[3][VEC], sh[VEC];
#pragma unroll
  for (int v = 0; v < VEC; v++) {
    acc[0][v] = acc[1][v] = acc[2][v] = 0.0;
    sh[v] = __ldg(lambda + sub * VEC + v) + mu;
  }
  const int64_t ntiles = (row1 - row0 + TILE - 1) / TILE;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t row = row0 + t * TILE + warp * RPW + slot;
    if (row < row1) {
      DV<VEC> au, mu_;
      sell_row<NP, 2>(sell_ptr, sell_col, A, M, row, U, sub, au, mu_);
      const int64_t off = row * NP + sub * VEC;
      const double di = __ldg(dinv + row);
      DV<VEC> z;
#pragma unroll
      for (int v = 0; v < VEC; v++) {
        const double b = sh[v] * mu_.v[v];
        const double r = b - au.v[v];
        z.v[v] = r * di;
        acc[0][v] += b * b;
        acc[1][v] += r * z.v[v];
        acc[2][v] += r * r;
      }
      z.st(Z + off);
      z.st(P + off);
    }
  }
  slab_block_cols<NP, 3>(acc, red, part);
}

template <int NP>
__global__ void __launch_bounds__(SB_THREADS) k_slab_s(const int32_t *__restrict__ sell_ptr,
                                                       const int32_t *__restrict__ sell_col,
                                                       const double *__restrict__ A, const double *__restrict__ Z,
                                                       double *__restrict__ Q, double *__restrict__ P,
                                                       const double *Xin, double *X,   // may alias (x in place)
                                                       int64_t row0, int64_t row1, int first, SlabCoef c,
                                                       double *__restrict__ part) {
  constexpr int VEC = SL<NP, SB_THREADS>::VEC, LPR = SL<NP, SB_THREADS>::LPR, RPW = SL<NP, SB_THREADS>::RPW,
                TILE = SL<NP, SB_THREADS>::TILE;
  __shared__ double red[SB_WARPS * NP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, slot = lane / LPR, sub = lane % LPR;
  double acc[1][VEC], be[VEC], xa[VEC];
#pragma unroll
  for (int v = 0; v < VEC; v++) {
    acc[0][v] = 0.0;
    xa[v] = c.a[sub * VEC + v];
    be[v] = c.b[sub * VEC + v];
  }
  const int64_t ntiles = (row1 - row0 + TILE - 1) / TILE;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t row = row0 + t * TILE + warp * RPW + slot;
    if (row < row1) {
      DV<VEC> w, unused;
      sell_row<NP, 1>(sell_ptr, sell_col, A, nullptr, row, Z, sub, w, unused);
      const int64_t off = row * NP + sub * VEC;
      if (first) {   // p = z (init), q = A p
        const DV<VEC> pv = DV<VEC>::ld(P + off);
#pragma unroll
        for (int v = 0; v < VEC; v++) acc[0][v] += pv.v[v] * w.v[v];
        w.st(Q + off);
      } else {
        DV<VEC> qv = DV<VEC>::ld(Q + off), pv = DV<VEC>::ld(P + off), xv = DV<VEC>::ld(Xin + off);
        const DV<VEC> zv = DV<VEC>::ld(Z + off);
#pragma unroll
        for (int v = 0; v < VEC; v++) {
          xv.v[v] += xa[v] * pv.v[v];
          pv.v[v] = zv.v[v] + be[v] * pv.v[v];
          qv.v[v] = w.v[v] + be[v] * qv.v[v];
          acc[0][v] += pv.v[v] * qv.v[v];
        }
        qv.st(Q + off);
        pv.st(P + off);
        xv.st(X + off);
      }
    }
  }
  slab_block_cols<NP, 1>(acc, red, part);
}

template <int NP>
__global__ void __launch_bounds__(SB_THREADS) k_slab_u(double *__restrict__ Z, const double *__restrict__ Q,
                                                       const double *__restrict__ dinv, const double *__restrict__ dg,
                                                       int64_t row0, int64_t row1, SlabCoef c,
                                                       double *__restrict__ part) {
  constexpr int VEC = SL<NP, SB_THREADS>::VEC, LPR = SL<NP, SB_THREADS>::LPR, RPW = SL<NP, SB_THREADS>::RPW,
                TILE = SL<NP, SB_THREADS>::TILE;
  __shared__ double red[SB_WARPS * 2 * NP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, slot = lane / LPR, sub = lane % LPR;
  double acc[2][VEC], al[VEC];
#pragma unroll
  for (int v = 0; v < VEC; v++) {
    acc[0][v] = acc[1][v] = 0.0;
    al[v] = c.a[sub * VEC + v];
  }
  const int64_t ntiles = (row1 - row0 + TILE - 1) / TILE;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t row = row0 + t * TILE + warp * RPW + slot;
    if (row < row1) {
      const int64_t off = row * NP + sub * VEC;
      DV<VEC> z = DV<VEC>::ld(Z + off);
      const DV<VEC> q = DV<VEC>::ld(Q + off);
      const double di = __ldg(dinv + row), dd = __ldg(dg + row);
#pragma unroll
      for (int v = 0; v < VEC; v++) {
        z.v[v] -= al[v] * (q.v[v] * di);
        const double r = dd * z.v[v];
        acc[0][v] += r * z.v[v];
        acc[1][v] += r * r;
      }
      z.st(Z + off);
    }
  }
  slab_block_cols<NP, 2>(acc, red, part);
}

template <int NP>
__global__ void __launch_bounds__(SB_THREADS) k_slab_x(const double *__restrict__ P, const double *Xin, double *X,
                                                       int64_t row0, int64_t row1,
                                                       SlabCoef c) {
  const int64_t e = row0 * NP + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= row1 * NP) return;
  X[e] = Xin[e] + c.a[e % NP] * P[e];
}

// dots[j] = sum over blocks b (ascending) of part[b][j]
__global__ void k_slab_dots(const double *__restrict__ part, int nblk, int nv, double *__restrict__ dots) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nv) return;
  double s = 0.0;
  for (int b = 0; b < nblk; b++) s += part[(int64_t)b * nv + j];
  dots[j] = s;
}

int slab_grid(const ks_ctx *ctx, int64_t rows, int tile) {
  const int64_t nt = (rows + tile - 1) / tile;
  const int64_t g = 4 * (int64_t)ctx->sm_count;
  return (int)(nt < 1 ? 1 : (nt < g ? nt : g));
}

SlabCoef make_coef(int NP, const double *ha, const double *hb) {
  SlabCoef c;
  for (int j = 0; j < KS_MAX_N; j++) {
    c.a[j] = (ha && j < NP) ? ha[j] : 0.0;
    c.b[j] = (hb && j < NP) ? hb[j] : 0.0;
  }
  return c;
}

template <int NP>
ks_status slab_phase(ks_ctx *ctx, int phase, int64_t row0, int64_t row1, int first, const SlabCoef &c,
                     const double *lambda, const double *U, double *Z, double *Q, double *P, const double *Xin,
                     double *X, double *dots) {
  constexpr int TILE = SL<NP, SB_THREADS>::TILE;
  cudaStream_t s = ctx->stream;
  const int G = slab_grid(ctx, row1 - row0, TILE);
  const int nk = phase == 0 ? 3 : phase == 1 ? 1 : 2;
  KsScratch scratch(ctx, KS_R_WORK);
  double *part = nullptr;
  if (phase <= 2) KS_TRY(ks_alloc_t(ctx, &part, (int64_t)G * nk * NP, "slab partials"));
  switch (phase) {
    case 0:
      k_slab_init<NP><<<G, SB_THREADS, 0, s>>>(ctx->sell_ptr, ctx->sell_col, ctx->sell_A, ctx->sell_M, ctx->dinv,
                                               lambda, ctx->mu, U, Z, P, row0, row1, part);
      break;
    case 1:
      k_slab_s<NP><<<G, SB_THREADS, 0, s>>>(ctx->sell_ptr, ctx->sell_col, ctx->sell_A, Z, Q, P, Xin, X, row0, row1,
                                            first, c, part);
      break;
    case 2:
      k_slab_u<NP><<<G, SB_THREADS, 0, s>>>(Z, Q, ctx->dinv, ctx->diag, row0, row1, c, part);
      break;
    default:
      k_slab_x<NP><<<ks_blocks((row1 - row0) * NP, 256), 256, 0, s>>>(P, Xin, X, row0, row1, c);
      break;
  }
  KS_LAUNCHED(ctx);
  if (phase <= 2) {
    k_slab_dots<<<ks_blocks(nk * NP, 128), 128, 0, s>>>(part, G, nk * NP, dots);
    KS_LAUNCHED(ctx);
  }
  return KS_OK;
}

}  // namespace

ks_status ks_slab_phase_impl(ks_ctx *ctx, int phase, int NP, int64_t row0, int64_t row1, int first,
                             const double *h_alpha, const double *h_beta, const double *lambda, const double *U,
                             double *Z, double *Q, double *P, const double *Xin, double *X, double *dots) {
  const SlabCoef c = make_coef(NP, h_alpha, h_beta);
  switch (NP) {
    case 1: return slab_phase<1>(ctx, phase, row0, row1, first, c, lambda, U, Z, Q, P, Xin, X, dots);
    case 2: return slab_phase<2>(ctx, phase, row0, row1, first, c, lambda, U, Z, Q, P, Xin, X, dots);
    case 4: return slab_phase<4>(ctx, phase, row0, row1, first, c, lambda, U, Z, Q, P, Xin, X, dots);
    case 8: return slab_phase<8>(ctx, phase, row0, row1, first, c, lambda, U, Z, Q, P, Xin, X, dots);
    case 16: return slab_phase<16>(ctx, phase, row0, row1, first, c, lambda, U, Z, Q, P, Xin, X, dots);
    case 32: return slab_phase<32>(ctx, phase, row0, row1, first, c, lambda, U, Z, Q, P, Xin, X, dots);
    case 64: return slab_phase<64>(ctx, phase, row0, row1, first, c, lambda, U, Z, Q, P, Xin, X, dots);
  }
  return ks_fail(ctx, KS_E_ARG, "slab: NP = %d must be a power of two <= 64", NP);
}
