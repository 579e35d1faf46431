// ks_assemble.cu -- (st4) reassembly of the V_eff-weighted mass on the fixed pattern,
// H = 1/2 K + M_V and the shifted operator A = H + mu M. Deterministic, no atomics.
//
// The element integral of the P1 interpolant of V against lambda_a lambda_b is
//     MV_T(a,b) = |T| (1+delta_ab) (V_a + V_b + S_T) / 120,      S_T = V_0 + V_1 + V_2 + V_3.
// Summed over the tets of an entry it splits into a part proportional to the mass entry and a part that
// only needs one scalar per tet, w_T = |T| S_T ("assembly"):
//     off-diagonal (i != j):  (M_V)_ij = (V_i + V_j) M_ij / 6 + sum_{T ∋ i,j} w_T / 120
//     diagonal:               (M_V)_ii =  V_i M_ii / 3      + sum_{T ∋ i}   w_T / 60
// since |T| (V_a + V_b)/120 = (V_a + V_b) M_T(a,b)/6 and 2|T| 2V_a/120 = V_a M_T(a,a)/3.
// Kernel 1 computes w_T per tet and V at free nodes; kernel 2 gathers w_T through the inverse scatter map
// (the element-to-nnz map grouped by target entry, ascending element) -- a fixed summation order.
#include "ks_internal.cuh"

namespace {

__global__ void k_tet_weights(const int32_t *__restrict__ tets, const double *__restrict__ vol,
                              const double *__restrict__ V, int64_t n_tets, const int32_t *__restrict__ node_of_free,
                              int64_t n_free, double *__restrict__ w, double *__restrict__ v_free,
                              unsigned *__restrict__ flags) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool bad = false;
  if (i < n_tets) {
    int4 t = __ldg(reinterpret_cast<const int4 *>(tets) + i);
    double s = __ldg(V + t.x) + __ldg(V + t.y) + __ldg(V + t.z) + __ldg(V + t.w);
    bad = !isfinite(s);
    w[i] = __ldg(vol + i) * s;
  }
  if (i < n_free) {
    double v = __ldg(V + __ldg(node_of_free + i));
    bad |= !isfinite(v);
    v_free[i] = v;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, KSF_NONFINITE);
}

// Half-warp per row: lane j of the half handles entries row_ptr[i] + j, + 16, ... The contributions of an
// entry (its slice of the inverse map, ascending element) are loaded ASM_UNR at a time before their w_T
// gathers, and summed in that order. VIEWS = false (the hot path) writes the operators the solver and the
// projection read: the sliced-ELL copies of A and H, diag(A) and 1 / diag(A). VIEWS = true writes the CSR
// value arrays M_V, H, A behind ks_values / ks_spmm (materialised on demand, same arithmetic).
constexpr int ASM_UNR = 8;
template <bool VIEWS>
__global__ void __launch_bounds__(256) k_assemble_rows(
    const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col, const int32_t *__restrict__ inv_ptr,
    const int32_t *__restrict__ inv_idx, const double *__restrict__ w, const double *__restrict__ v_free,
    const double *__restrict__ K, const double *__restrict__ M, double mu, int64_t n_free, double *__restrict__ MV,
    double *__restrict__ H, double *__restrict__ A, double *__restrict__ diag, double *__restrict__ dinv,
    const int32_t *__restrict__ sell_ptr, double *__restrict__ sell_A, double *__restrict__ sell_H) {
  int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 4;
  int j = threadIdx.x & 15;
  if (row >= n_free) return;
  const double vi = __ldg(v_free + row);
  const int32_t kr = __ldg(row_ptr + row), k1 = __ldg(row_ptr + row + 1);
  const int64_t sbase = VIEWS ? 0 : __ldg(sell_ptr + row / KS_SELL_C) + (row % KS_SELL_C) * 4;
  for (int32_t e = kr + j; e < k1; e += 16) {
    const int32_t c = __ldg(col + e);
    const double m = __ldg(M + e), kk = __ldg(K + e), vc = __ldg(v_free + c);
    const int32_t q0 = __ldg(inv_ptr + e), q1 = __ldg(inv_ptr + e + 1);
    double s = 0.0;
    for (int32_t qb = q0; qb < q1; qb += ASM_UNR) {
      int32_t t[ASM_UNR];
#pragma unroll
      for (int u = 0; u < ASM_UNR; u++) t[u] = qb + u < q1 ? (__ldg(inv_idx + qb + u) >> 4) : -1;
      double wt[ASM_UNR];
#pragma unroll
      for (int u = 0; u < ASM_UNR; u++) wt[u] = t[u] >= 0 ? __ldg(w + t[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < ASM_UNR; u++)
        if (t[u] >= 0) s += wt[u];
    }
    double mv;
    if (c == row) mv = vi * m / 3.0 + s / 60.0;
    else mv = (vi + vc) * m / 6.0 + s / 120.0;
    const double h = 0.5 * kk + mv;
    const double a = h + mu * m;
    if (VIEWS) {
      MV[e] = mv;
      H[e] = h;
      A[e] = a;
    } else {
      const int k = e - kr;   // slot of the entry in the sliced-ELL copy (ks_sell.cu)
      const int64_t sp = sbase + (k >> 2) * (4 * KS_SELL_C) + (k & 3);
      sell_A[sp] = a;
      sell_H[sp] = h;
      if (c == row) {
        diag[row] = a;
        dinv[row] = 1.0 / a;
      }
    }
  }
}

// Hot-path assembly in sliced-ELL order: one warp per 8-row slice, one slot group (8 rows x 4
// slots = 32 entries) per step, lane = (row % 8) * 4 + slot % 4. The entry's K and M come from their sliced-ELL
// copies and the SELL values of A and H are written in place: every read of the fixed data and every write is
// one coalesced 256-byte segment per warp. Each lane walks its entry's slice of the inverse map (through the
// entry's CSR index) in ascending element order, as k_assemble_rows does: the same arithmetic and order per
// entry. The ~24-long diagonal lists of a slice fall in one slot group, so per slice the walk costs about one
// long group plus the short ones (the half-warp per row kernel waits for its diagonal lane on every row).
template <int UNR>
__global__ void __launch_bounds__(256) k_assemble_sell(const int32_t *__restrict__ sell_ptr,
                                                       const int32_t *__restrict__ sell_col,
                                                       const int32_t *__restrict__ sell_csr,
                                                       const double *__restrict__ sK, const double *__restrict__ sM,
                                                       const int32_t *__restrict__ inv_ptr,
                                                       const int32_t *__restrict__ inv_idx, const double *__restrict__ w,
                                                       const double *__restrict__ v_free, double mu, int64_t n_free,
                                                       int64_t n_slices, double *__restrict__ sell_A,
                                                       double *__restrict__ sell_H, double *__restrict__ diag,
                                                       double *__restrict__ dinv) {
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= n_slices) return;
  const int32_t b = __ldg(sell_ptr + s), ng = (__ldg(sell_ptr + s + 1) - b) / (4 * KS_SELL_C);
  const int64_t row = s * KS_SELL_C + (lane >> 2);
  const double vi = row < n_free ? __ldg(v_free + row) : 0.0;
  for (int g = 0; g < ng; g++) {
    const int64_t sp = b + (int64_t)g * (4 * KS_SELL_C) + lane;
    const int32_t e = __ldg(sell_csr + sp);
    if (e < 0) continue;   // padding slot (stays 0)
    const int32_t c = __ldg(sell_col + sp);
    const double m = __ldg(sM + sp), kk = __ldg(sK + sp), vc = __ldg(v_free + c);
    const int32_t q0 = __ldg(inv_ptr + e), q1 = __ldg(inv_ptr + e + 1);
    double sum = 0.0;
    for (int32_t qb = q0; qb < q1; qb += UNR) {
      int32_t t[UNR];
#pragma unroll
      for (int u = 0; u < UNR; u++) t[u] = qb + u < q1 ? (__ldg(inv_idx + qb + u) >> 4) : -1;
      double wt[UNR];
#pragma unroll
      for (int u = 0; u < UNR; u++) wt[u] = t[u] >= 0 ? __ldg(w + t[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < UNR; u++)
        if (t[u] >= 0) sum += wt[u];
    }
    double mv;
    if (c == row) mv = vi * m / 3.0 + sum / 60.0;
    else mv = (vi + vc) * m / 6.0 + sum / 120.0;
    const double h = 0.5 * kk + mv;
    const double a = h + mu * m;
    sell_A[sp] = a;
    sell_H[sp] = h;
    if (c == row) {
      diag[row] = a;
      dinv[row] = 1.0 / a;
    }
  }
}

}  // namespace

ks_status ks_assemble_impl(ks_ctx *ctx, const double *d_veff, double mu) {
  cudaStream_t s = ctx->stream;
  const int64_t n = ctx->n_tets > ctx->n_free ? ctx->n_tets : ctx->n_free;
  k_tet_weights<<<ks_blocks(n, 256), 256, 0, s>>>(ctx->tets, ctx->vol, d_veff, ctx->n_tets, ctx->node_of_free,
                                                  ctx->n_free, ctx->w_tet, ctx->v_free, ctx->d_flags);
  KS_LAUNCHED(ctx);
#ifndef KS_ASM_SELL
#define KS_ASM_SELL 1
#endif
  if (KS_ASM_SELL) {
    k_assemble_sell<ASM_UNR><<<ks_blocks(32 * ctx->n_slices, 256), 256, 0, s>>>(
        ctx->sell_ptr, ctx->sell_col, ctx->sell_csr, ctx->sell_K, ctx->sell_M, ctx->inv_ptr, ctx->inv_idx, ctx->w_tet,
        ctx->v_free, mu, ctx->n_free, ctx->n_slices, ctx->sell_A, ctx->sell_H, ctx->diag, ctx->dinv);
  } else {
    k_assemble_rows<false><<<ks_blocks(16 * ctx->n_free, 256), 256, 0, s>>>(
        ctx->row_ptr, ctx->col, ctx->inv_ptr, ctx->inv_idx, ctx->w_tet, ctx->v_free, ctx->K, ctx->M, mu,
        ctx->n_free, nullptr, nullptr, nullptr, ctx->diag, ctx->dinv, ctx->sell_ptr, ctx->sell_A, ctx->sell_H);
  }
  KS_LAUNCHED(ctx);
  ctx->views_fresh = false;
  ctx->mu = mu;
  ctx->assembled = true;
  return KS_OK;
}

// CSR value views (M_V, H, A) of the last assembly, recomputed from the kept per-tet weights and nodal V
ks_status ks_materialize_views(ks_ctx *ctx) {
  if (!ctx->assembled || ctx->views_fresh) return KS_OK;
  k_assemble_rows<true><<<ks_blocks(16 * ctx->n_free, 256), 256, 0, ctx->stream>>>(
      ctx->row_ptr, ctx->col, ctx->inv_ptr, ctx->inv_idx, ctx->w_tet, ctx->v_free, ctx->K, ctx->M, ctx->mu,
      ctx->n_free, ctx->MV, ctx->H, ctx->A, nullptr, nullptr, nullptr, nullptr, nullptr);
  KS_LAUNCHED(ctx);
  ctx->views_fresh = true;
  return KS_OK;
}
