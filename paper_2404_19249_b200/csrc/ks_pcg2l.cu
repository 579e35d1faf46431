// ks_pcg2l.cu -- two-level preconditioned CG for the Hartree Poisson solve K x = b (NEXT-2 / NEXT-4,
// DESIGN.md §9): the Jacobi smoother of ks_pcg.cu plus a coarse correction on the method's own coarse space
// (the nonnested interpolation P of ks_set_coarse),
//     z = D^-1 r + P K_H^-1 P^T r,      K_H = P^T K P  (dense, inverted once per coarse space by Cholesky).
// Same stopping rule as ks_pcg.cu (||r|| <= tol ||b||), x0 given. One persistent cooperative launch; per
// iteration five grid-barrier-separated phases:
//   S   q = K p, p.q                                                                       | barrier
//   U   r' = r - alpha q (second buffer), r'.D^-1 r', r'.r'; item restriction partials
//       sum_{i in item} P_ic (r_i - alpha q_i) from the unchanged r (so both run in one phase)  | barrier
//   C1  r_H[c] = sum over the items of coarse node c (CT lists, fixed order)                    | barrier
//   C2  y = K_H^-1 r_H (warp per coarse row), r_H.y                                             | barrier
//   P   x += alpha p, z = D^-1 r' + P y, p = z + beta p,   rho' = r'.D^-1 r' + r_H.y (= r'.z)  | barrier
// All reductions are fixed-order (lane-strided + butterfly, warps in order, blocks in order), so the solve
// is bitwise reproducible. Data written by other blocks inside the launch is read with ld.global.cg (L2).
#include <algorithm>

#include "ks_grid.cuh"
#include "ks_internal.cuh"
#include "ks_layout.cuh"
#include "ks_sell.cuh"

namespace {

constexpr int T2 = 512, W2 = T2 / 32;
constexpr int NSLOT = KS_EXT_NSLOT2L;   // block partial slots: 0 S, 1-2 U, 3 C2, 4-6 init

struct P2Args {
  const int32_t *sell_ptr, *sell_col;
  const double *K, *dinv, *B, *X0;
  double *X, *r, *r2, *p, *q;
  const int32_t *Pc4, *perm, *item_ptr, *CT_ptr, *CT_val;
  const double *Pv4, *Pv4p, *KHinv;
  double *rpart, *rH, *y, *part;
  unsigned *bar, *flags;
  int32_t *iters_out;
  int64_t n, n_items, nH;
  double tol;
  int max_iter;
};

// block sum of ND per-thread values, fixed order; result in out[0..ND) for every thread
template <int ND>
__device__ __forceinline__ void block_sum(const double (&v)[ND], double *red, double *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 0; d < ND; d++) {
    const double s = warp_sum(v[d]);
    if (lane == 0) red[warp * ND + d] = s;
  }
  __syncthreads();
  if (threadIdx.x < ND) {
    double t = 0.0;
    for (int w = 0; w < W2; w++) t += red[w * ND + threadIdx.x];
    out[threadIdx.x] = t;
  }
  __syncthreads();
}

// sum over the blocks of partial slots [s0, s0 + ns): warp j takes slot s0 + j (lane-strided, butterfly)
__device__ __forceinline__ void grid_sum(const double *part, int s0, int ns, double *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < ns; j += W2) {
    double s = 0.0;
    for (int g = lane; g < (int)gridDim.x; g += 32) s += __ldcg(part + g * NSLOT + s0 + j);
    s = warp_sum(s);
    if (lane == 0) out[j] = s;
  }
  __syncthreads();
}

#ifndef KS_P2_UNR
#define KS_P2_UNR 2
#endif
constexpr int P2_UNR = KS_P2_UNR;   // slot groups loaded ahead of their gathers
// (K x)_row on the sliced-ELL copy (N = 1: one thread per row). The row's first 4 slot groups (16 slots:
// the whole row on these meshes) are loaded before their gathers, so the gathers overlap.
__device__ __forceinline__ double spmv_row(const P2Args &a, int64_t row, const double *x) {
  const int64_t sl = row / KS_SELL_C;
  const int32_t b = __ldg(a.sell_ptr + sl), e = __ldg(a.sell_ptr + sl + 1);
  const int groups = (e - b) / (4 * KS_SELL_C);
  const int64_t base = b + (row % KS_SELL_C) * 4;
  double s = 0.0;
  for (int g0 = 0; g0 < groups; g0 += P2_UNR) {
    int4 c[P2_UNR];
    double w[P2_UNR][4];
#pragma unroll
    for (int u = 0; u < P2_UNR; u++) {
      if (g0 + u < groups) {
        const int64_t o = base + (int64_t)(g0 + u) * (4 * KS_SELL_C);
        c[u] = __ldg(reinterpret_cast<const int4 *>(a.sell_col + o));
        ldnc_v4(a.K + o, w[u][0], w[u][1], w[u][2], w[u][3]);
      } else {
        c[u] = make_int4(0, 0, 0, 0);
        w[u][0] = w[u][1] = w[u][2] = w[u][3] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < P2_UNR; u++) {
      if (g0 + u >= groups) break;
      s = fma(w[u][0], __ldcg(x + c[u].x), s);
      s = fma(w[u][1], __ldcg(x + c[u].y), s);
      s = fma(w[u][2], __ldcg(x + c[u].z), s);
      s = fma(w[u][3], __ldcg(x + c[u].w), s);
    }
  }
  return s;
}

// item restriction partials rpart[4 it + k] = sum_{pos in item} Pv4p[4 pos + k] (r - alpha q)[perm[pos]],
// one warp per item (positions lane-strided, then a butterfly)
__device__ __forceinline__ void restrict_items(const P2Args &a, const double *r, const double *q, double alpha) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * T2 + threadIdx.x) >> 5, nw = (int64_t)gridDim.x * W2;
  for (int64_t it = gw; it < a.n_items; it += nw) {
    const int32_t p0 = __ldg(a.item_ptr + it), p1 = __ldg(a.item_ptr + it + 1);
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int32_t pos = p0 + lane; pos < p1; pos += 32) {
      const int32_t i = __ldg(a.perm + pos);
      const double v = q ? __ldcg(r + i) - alpha * __ldcg(q + i) : __ldcg(r + i);
      double w0, w1, w2, w3;
      ldnc_v4(a.Pv4p + 4 * (int64_t)pos, w0, w1, w2, w3);
      s[0] = fma(w0, v, s[0]);
      s[1] = fma(w1, v, s[1]);
      s[2] = fma(w2, v, s[2]);
      s[3] = fma(w3, v, s[3]);
    }
#pragma unroll
    for (int k = 0; k < 4; k++) s[k] = warp_sum(s[k]);
    if (lane == 0) *reinterpret_cast<double4 *>(a.rpart + 4 * it) = make_double4(s[0], s[1], s[2], s[3]);
  }
}

// r_H[c] = sum over the (item, slot) entries of coarse node c, in list order (one warp per coarse node)
__device__ __forceinline__ void coarse_rhs(const P2Args &a) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * T2 + threadIdx.x) >> 5, nw = (int64_t)gridDim.x * W2;
  for (int64_t c = gw; c < a.nH; c += nw) {
    const int32_t e0 = __ldg(a.CT_ptr + c), e1 = __ldg(a.CT_ptr + c + 1);
    double s = 0.0;
    for (int32_t e = e0 + lane; e < e1; e += 32) s += __ldcg(a.rpart + __ldg(a.CT_val + e));
    s = warp_sum(s);
    if (lane == 0) a.rH[c] = s;
  }
}

// y = K_H^-1 r_H (one warp per coarse row); returns this thread's share of r_H . y
__device__ __forceinline__ double coarse_solve(const P2Args &a) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * T2 + threadIdx.x) >> 5, nw = (int64_t)gridDim.x * W2;
  double dot = 0.0;
  for (int64_t c = gw; c < a.nH; c += nw) {
    const double *row = a.KHinv + c * a.nH;
    double s = 0.0;
    for (int64_t d = lane; d < a.nH; d += 32) s = fma(__ldg(row + d), __ldcg(a.rH + d), s);
    s = warp_sum(s);
    if (lane == 0) {
      a.y[c] = s;
      dot = fma(__ldcg(a.rH + c), s, dot);
    }
  }
  return dot;
}

// (P y)_row: the row's <= 4 coarse parents from the 4-wide tables (absent parents: column 0, weight 0)
__device__ __forceinline__ double prolong_row(const P2Args &a, int64_t row) {
  const int4 c = __ldg(reinterpret_cast<const int4 *>(a.Pc4) + row);
  double w0, w1, w2, w3;
  ldnc_v4(a.Pv4 + 4 * row, w0, w1, w2, w3);
  double s = w0 * __ldcg(a.y + c.x);
  s = fma(w1, __ldcg(a.y + c.y), s);
  s = fma(w2, __ldcg(a.y + c.z), s);
  return fma(w3, __ldcg(a.y + c.w), s);
}

__global__ void k_pc4(const int32_t *__restrict__ P_ptr, const int32_t *__restrict__ P_col, int64_t n,
                      int32_t *__restrict__ Pc4) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t p0 = P_ptr[i], np = P_ptr[i + 1] - p0;
  for (int k = 0; k < 4; k++) Pc4[4 * i + k] = k < np ? P_col[p0 + k] : 0;
}

#ifndef KS_P2_MINB
#define KS_P2_MINB 2
#endif
__global__ void __launch_bounds__(T2, KS_P2_MINB) k_pcg2l(P2Args a) {
  __shared__ double red[W2 * 4];
  __shared__ double tot[8];
  __shared__ double s_rho, s_bn, s_alpha, s_beta;
  __shared__ int s_done, s_iters;
  unsigned target = 0;
  const int64_t n = a.n, gtid = (int64_t)blockIdx.x * T2 + threadIdx.x, gstride = (int64_t)gridDim.x * T2;
  double *part = a.part + blockIdx.x * NSLOT;

  // ---- init: r = b - K x0, x = x0; b.b, r.D^-1 r, r.r ----
  {
    double v[3] = {0.0, 0.0, 0.0};
    for (int64_t row = gtid; row < n; row += gstride) {
      const double b = __ldg(a.B + row), x0 = __ldg(a.X0 + row);
      const double r = b - spmv_row(a, row, a.X0);
      a.r[row] = r;
      a.X[row] = x0;
      v[0] = fma(b, b, v[0]);
      v[1] = fma(r * __ldg(a.dinv + row), r, v[1]);
      v[2] = fma(r, r, v[2]);
    }
    block_sum<3>(v, red, tot);
    if (threadIdx.x < 3) part[4 + threadIdx.x] = tot[threadIdx.x];
  }
  grid_barrier(a.bar, target);
  restrict_items(a, a.r, nullptr, 0.0);
  grid_barrier(a.bar, target);
  coarse_rhs(a);
  grid_barrier(a.bar, target);
  {
    const double d[1] = {coarse_solve(a)};
    block_sum<1>(d, red, tot);
    if (threadIdx.x == 0) part[3] = tot[0];
  }
  grid_barrier(a.bar, target);
  grid_sum(a.part, 3, 4, tot);   // r_H.y, b.b, r.D^-1 r, r.r
  if (threadIdx.x == 0) {
    const double bn = sqrt(tot[1]), rr = tot[3];
    s_bn = bn;
    s_rho = tot[2] + tot[0];
    s_iters = 0;
    const bool finite = isfinite(bn) && isfinite(rr) && isfinite(s_rho);
    if (!finite && blockIdx.x == 0) atomicOr(a.flags, KSF_NONFINITE);
    s_done = !finite || sqrt(rr) <= a.tol * bn;
  }
  __syncthreads();
  if (!s_done)
    for (int64_t row = gtid; row < n; row += gstride)
      a.p[row] = __ldg(a.dinv + row) * __ldcg(a.r + row) + prolong_row(a, row);
  grid_barrier(a.bar, target);

  double *r = a.r, *r2 = a.r2;
  for (int it = 0; !s_done; it++) {
    if (it >= a.max_iter) {
      if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(a.flags, KSF_NOT_CONVERGED);
      break;
    }
    // ---- S: q = K p, p.q ----
    {
      double v[1] = {0.0};
      for (int64_t row = gtid; row < n; row += gstride) {
        const double qv = spmv_row(a, row, a.p);
        a.q[row] = qv;
        v[0] = fma(__ldcg(a.p + row), qv, v[0]);
      }
      block_sum<1>(v, red, tot);
      if (threadIdx.x == 0) part[0] = tot[0];
    }
    grid_barrier(a.bar, target);
    grid_sum(a.part, 0, 1, tot);
    if (threadIdx.x == 0) {
      const double pq = tot[0];
      if (!(pq > 0.0)) {
        if (blockIdx.x == 0) atomicOr(a.flags, isfinite(pq) ? KSF_NOT_SPD : KSF_NONFINITE);
        s_done = 1;
      }
      s_alpha = s_rho / pq;
    }
    __syncthreads();
    if (s_done) break;
    const double al = s_alpha;
    // ---- U: r' = r - alpha q, dots; item restriction of r - alpha q ----
    {
      double v[2] = {0.0, 0.0};
      for (int64_t row = gtid; row < n; row += gstride) {
        const double rn = __ldcg(r + row) - al * __ldcg(a.q + row);
        r2[row] = rn;
        v[0] = fma(rn * __ldg(a.dinv + row), rn, v[0]);
        v[1] = fma(rn, rn, v[1]);
      }
      restrict_items(a, r, a.q, al);
      block_sum<2>(v, red, tot);
      if (threadIdx.x < 2) part[1 + threadIdx.x] = tot[threadIdx.x];
    }
    grid_barrier(a.bar, target);
    coarse_rhs(a);
    grid_barrier(a.bar, target);
    {
      const double d[1] = {coarse_solve(a)};
      block_sum<1>(d, red, tot);
      if (threadIdx.x == 0) part[3] = tot[0];
    }
    grid_barrier(a.bar, target);
    grid_sum(a.part, 1, 3, tot);   // r'.D^-1 r', r'.r', r_H.y
    if (threadIdx.x == 0) {
      const double rho = tot[0] + tot[2], rr = tot[1];
      s_iters = it + 1;
      if (!isfinite(rho) || !isfinite(rr)) {
        if (blockIdx.x == 0) atomicOr(a.flags, KSF_NONFINITE);
        s_done = 1;
      } else {
        s_done = sqrt(rr) <= a.tol * s_bn;
      }
      s_beta = rho / s_rho;
      s_rho = rho;
    }
    __syncthreads();
    // ---- P: x += alpha p; p = D^-1 r' + P y + beta p ----
    {
      const double be = s_beta;
      const bool upd = !s_done;
      for (int64_t row = gtid; row < n; row += gstride) {
        const double pv = __ldcg(a.p + row);
        a.X[row] = __ldcg(a.X + row) + al * pv;
        if (upd) a.p[row] = __ldg(a.dinv + row) * __ldcg(r2 + row) + prolong_row(a, row) + be * pv;
      }
    }
    double *t = r;
    r = r2;
    r2 = t;
    grid_barrier(a.bar, target);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.iters_out = s_iters;
}

}  // namespace

void ks_free_pcg2l(ks_ctx *ctx) { ctx->har2l_state = 0; }

// K_H^-1 and the work vectors for the current coarse space (once per ks_set_coarse)
static ks_status pcg2l_setup(ks_ctx *ctx) {
  if (ctx->har2l_state != 0) return KS_OK;
  // the tables live in the extension workspace (ks_layout_ext), planned for the current coarse space
  if (ctx->ext_nH != ctx->n_H || !ctx->har2l_KHinv) {
    ctx->har2l_state = -1;
    return KS_OK;
  }
  const int64_t n = ctx->n_free, nH = ctx->n_H;
  k_pc4<<<ks_blocks(n, 256), 256, 0, ctx->stream>>>(ctx->P_ptr, ctx->P_col, n, ctx->har2l_Pc4);
  KS_LAUNCHED(ctx);
  KS_TRY(ks_coarse_galerkin(ctx, ctx->sell_K, ctx->har2l_KHinv));
  bool spd = false;
  KS_TRY(ks_spd_inverse(ctx, ctx->har2l_KHinv, nH, &spd));
  ctx->har2l_state = spd ? 1 : -1;
  return KS_OK;
}

// returns KS_E_STATE when no usable coarse space is set (the caller falls back to Jacobi-PCG)
ks_status ks_pcg2l_run(ks_ctx *ctx, const double *b, const double *x0, double *x, double tol, int max_iter,
                       int32_t *d_iters) {
  if (ctx->n_H <= 0 || !ctx->Pv4 || !ctx->CT_ptr) return KS_E_STATE;
  KS_TRY(pcg2l_setup(ctx));
  if (ctx->har2l_state != 1) return KS_E_STATE;
  int per_sm = 0;
  KS_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg2l, T2, 0));
  if (per_sm < 1) return ks_fail(ctx, KS_E_CUDA, "k_pcg2l cannot be resident");
  const int G = std::min(per_sm, 4) * ctx->sm_count;
  P2Args a;
  a.sell_ptr = ctx->sell_ptr;
  a.sell_col = ctx->sell_col;
  a.K = ctx->sell_K;
  a.dinv = ctx->dinvK;
  a.B = b;
  a.X0 = x0;
  a.X = x;
  a.r = ctx->har2l_r;
  a.r2 = ctx->har2l_r2;
  a.p = ctx->har2l_p;
  a.q = ctx->har2l_q;
  a.Pc4 = ctx->har2l_Pc4;
  a.perm = ctx->perm;
  a.item_ptr = ctx->item_ptr;
  a.CT_ptr = ctx->CT_ptr;
  a.CT_val = ctx->CT_val;
  a.Pv4 = ctx->Pv4;
  a.Pv4p = ctx->Pv4p;
  a.KHinv = ctx->har2l_KHinv;
  a.rpart = ctx->har2l_rpart;
  a.rH = ctx->har2l_rH;
  a.y = ctx->har2l_y;
  a.part = ctx->har2l_part;
  a.bar = ctx->barrier;
  a.flags = ctx->d_flags;
  a.iters_out = d_iters;
  a.n = ctx->n_free;
  a.n_items = ctx->n_items;
  a.nH = ctx->n_H;
  a.tol = tol;
  a.max_iter = max_iter;
  KS_CUDA(ctx, cudaMemsetAsync(ctx->barrier, 0, sizeof(unsigned), ctx->stream));
  void *args[] = {&a};
  KS_CUDA(ctx, cudaLaunchCooperativeKernel((const void *)k_pcg2l, dim3(G), dim3(T2), args, 0, ctx->stream));
  ctx->launches++;
  return KS_OK;
}
