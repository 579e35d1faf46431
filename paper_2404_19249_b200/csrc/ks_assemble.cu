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
#include <cstdlib>
#include <cstring>

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

// Sum of w_T over an entry's slice [q0, q1) of the inverse map, ascending element. Off-diagonal entries
// (4-6 tets) sum in that order; the diagonal (the row's whole star, ~24 tets) in four interleaved partial sums
// p_r over the positions k = q - q0 with k % 4 = r, combined as (p0 + p1) + (p2 + p3): the order the star-mask
// kernel's four lanes per row produce, so every assembly kernel writes bitwise the same values.
template <int UNR>
__device__ __forceinline__ double walk_sum(const int32_t *__restrict__ inv_idx, const double *__restrict__ w,
                                           int32_t q0, int32_t q1, bool diag) {
  static_assert(UNR % 4 == 0, "batches must keep k % 4 static");
  double ps[4] = {0.0, 0.0, 0.0, 0.0};
  for (int32_t qb = q0; qb < q1; qb += UNR) {
    int32_t t[UNR];
#pragma unroll
    for (int u = 0; u < UNR; u++) t[u] = qb + u < q1 ? (__ldg(inv_idx + qb + u) >> 4) : -1;
    double wt[UNR];
#pragma unroll
    for (int u = 0; u < UNR; u++) wt[u] = t[u] >= 0 ? __ldg(w + t[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < UNR; u++)
      if (t[u] >= 0) {
        if (diag) ps[u & 3] += wt[u];
        else ps[0] += wt[u];
      }
  }
  return diag ? (ps[0] + ps[1]) + (ps[2] + ps[3]) : ps[0];
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
    const double s = walk_sum<ASM_UNR>(inv_idx, w, q0, q1, c == row);
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
    const double sum = walk_sum<UNR>(inv_idx, w, q0, q1, c == row);
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

// Star-mask variant (default when every free node's star has <= STAR_MAX tets). Every tet contributing to an
// entry of row i contains node i, so it lies in the row's star: the tets containing node i, which is exactly the
// inverse-map slice of the row's diagonal entry (ascending tet). A setup-time bit mask per sliced-ELL slot marks
// which star tets contribute to the slot's entry (bit k = the k-th tet of the star; 0 = padding slot). A warp
// first gathers the w_T of its slice's 8 stars (~24 tets each) into shared memory, 4 lanes per row; each lane
// then sums the set bits of its slot's mask in ascending order (the diagonal: the whole star, summed while it is
// staged, in walk_sum's order). That is the entry's inverse-map slice in walk_sum's order, so the values are
// bitwise those of k_assemble_sell, without the per-entry inverse-map walk (no
// sell_csr, inv_ptr or inv_idx reads per entry: one coalesced 8-byte mask per slot instead).
// Stars of <= 32 tets (every Kuhn mesh: 24) use 32-bit masks, halving the mask stream.
constexpr int STAR_MAX = 64, ASM_WARPS = 8;
#ifdef KS_ASM_MINB
#define KS_ASM_BOUNDS __launch_bounds__(ASM_WARPS * 32, KS_ASM_MINB)
#else
#define KS_ASM_BOUNDS __launch_bounds__(ASM_WARPS * 32)
#endif
#ifndef KS_ASM_NGC
#define KS_ASM_NGC 2   // slot groups whose loads are issued together (before the star staging for the first chunk)
#endif
template <class MT>
__global__ void KS_ASM_BOUNDS k_assemble_mask(
    const int32_t *__restrict__ sell_ptr, const int32_t *__restrict__ sell_col, const MT *__restrict__ slot_mask,
    const double *__restrict__ sK, const double *__restrict__ sM, const int2 *__restrict__ star,
    const int32_t *__restrict__ inv_idx, const double *__restrict__ w, const double *__restrict__ v_free, double mu,
    int64_t n_free, int64_t n_slices, double *__restrict__ sell_A, double *__restrict__ sell_H,
    double *__restrict__ diag, double *__restrict__ dinv) {
  constexpr int NGC = KS_ASM_NGC;
  constexpr int KPL = (sizeof(MT) == 8 ? STAR_MAX : 32) / 4;   // star entries per lane (4 lanes per row)
  __shared__ double ws[ASM_WARPS][KS_SELL_C][STAR_MAX + 1];   // +1: the 8 rows on different banks
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t s = (int64_t)blockIdx.x * ASM_WARPS + warp;
  if (s >= n_slices) return;   // whole warps
  double (*st)[STAR_MAX + 1] = ws[warp];
  const int rl = lane >> 2;
  const int64_t row = s * KS_SELL_C + rl;
  const int32_t b = __ldg(sell_ptr + s), ng = (__ldg(sell_ptr + s + 1) - b) / (4 * KS_SELL_C);
  // the entry loads of the first NGC slot groups go out first: they do not depend on the star
  MT mk[NGC];
  int32_t cg[NGC];
  double mg[NGC], kg[NGC];
  auto load_groups = [&](int g0) {
#pragma unroll
    for (int q = 0; q < NGC; q++) {
      mk[q] = 0;
      if (g0 + q < ng) {
        const int64_t sp = b + (int64_t)(g0 + q) * (4 * KS_SELL_C) + lane;
        mk[q] = __ldg(slot_mask + sp);
        cg[q] = __ldg(sell_col + sp);
        mg[q] = __ldg(sM + sp);
        kg[q] = __ldg(sK + sp);
      }
    }
  };
  load_groups(0);
  // 4 lanes per row stage its star: every inverse-map index first, then every w_T gather
  double dsum = 0.0;   // the diagonal's sum: the whole star, in walk_sum's four-partial order
  if (row < n_free) {
    const int2 sd = __ldg(star + row);
    int32_t ix[KPL];
#pragma unroll
    for (int j = 0; j < KPL; j++) {
      const int k = (lane & 3) + 4 * j;
      ix[j] = k < sd.y ? __ldg(inv_idx + sd.x + k) : -1;
    }
    double x[KPL];
#pragma unroll
    for (int j = 0; j < KPL; j++) x[j] = ix[j] >= 0 ? __ldg(w + (ix[j] >> 4)) : 0.0;
#pragma unroll
    for (int j = 0; j < KPL; j++) {
      const int k = (lane & 3) + 4 * j;
      if (k < sd.y) {
        st[rl][k] = x[j];
        dsum += x[j];
      }
    }
  }
  dsum += __shfl_xor_sync(0xffffffffu, dsum, 1);   // p0 + p1 (= p1 + p0), p2 + p3
  dsum += __shfl_xor_sync(0xffffffffu, dsum, 2);   // (p0 + p1) + (p2 + p3) on all four lanes
  __syncwarp();
  const double vi = row < n_free ? __ldg(v_free + row) : 0.0;
  for (int g0 = 0; g0 < ng; g0 += NGC) {
    if (g0 > 0) load_groups(g0);
    double vc[NGC];
#pragma unroll
    for (int q = 0; q < NGC; q++) vc[q] = mk[q] ? __ldg(v_free + cg[q]) : 0.0;
#pragma unroll
    for (int q = 0; q < NGC; q++) {
      MT m_ = mk[q];
      if (!m_) continue;   // padding slot (stays 0) or past the slice
      const int64_t sp = b + (int64_t)(g0 + q) * (4 * KS_SELL_C) + lane;
      const int32_t c = cg[q];
      const double m = mg[q], kk = kg[q];
      double sum = dsum;
      if (c != row) {
        sum = 0.0;
        do {
          sum += st[rl][sizeof(MT) == 8 ? __ffsll((long long)m_) - 1 : __ffs((int)m_) - 1];
          m_ &= m_ - 1;
        } while (m_);
      }
      double mv;
      if (c == row) mv = vi * m / 3.0 + sum / 60.0;
      else mv = (vi + vc[q]) * m / 6.0 + sum / 120.0;
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
}

// setup, thread per free row: star[i] = (first, length) of the row's diagonal inverse-map slice; *max_star =
// the largest star
__global__ void k_star(const int32_t *__restrict__ diag_pos, const int32_t *__restrict__ inv_ptr, int64_t n_free,
                       int2 *__restrict__ star, int *__restrict__ max_star) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_free) return;
  const int32_t ed = diag_pos[i];
  const int32_t d0 = inv_ptr[ed], nd = inv_ptr[ed + 1] - d0;
  star[i] = make_int2(d0, nd);
  atomicMax(max_star, nd);
}

// setup, thread per free row (stars <= STAR_MAX): the bit mask of every sliced-ELL slot of the row (slot layout
// of k_sell_fill_csr); bit k set = the k-th tet of the row's star contributes to the slot's entry
template <class MT>
__global__ void k_slot_masks(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ sell_ptr,
                             const int2 *__restrict__ star, const int32_t *__restrict__ inv_ptr,
                             const int32_t *__restrict__ inv_idx, int64_t n_free, MT *__restrict__ slot_mask) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_free) return;
  const int64_t sl = i / KS_SELL_C;
  const int32_t b = sell_ptr[sl], K = (sell_ptr[sl + 1] - b) / KS_SELL_C;
  const int64_t base = b + (i % KS_SELL_C) * 4;
  const int32_t k0 = row_ptr[i], len = row_ptr[i + 1] - k0;
  const int2 sd = star[i];
  for (int k = 0; k < K; k++) {
    MT mk = 0;
    if (k < len)
      for (int32_t q = inv_ptr[k0 + k]; q < inv_ptr[k0 + k + 1]; q++) {
        const int32_t t = inv_idx[q] >> 4;
        int lo = 0, hi = sd.y;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if ((inv_idx[sd.x + mid] >> 4) < t) lo = mid + 1; else hi = mid;
        }
        mk |= (MT)1 << lo;
      }
    slot_mask[base + (k >> 2) * (4 * KS_SELL_C) + (k & 3)] = mk;
  }
}

}  // namespace

ks_status ks_star_setup(ks_ctx *ctx, int *d) {
  KS_CUDA(ctx, cudaMemsetAsync(d, 0, sizeof(int), ctx->stream));
  k_star<<<ks_blocks(ctx->n_free, 256), 256, 0, ctx->stream>>>(ctx->diag_pos, ctx->inv_ptr, ctx->n_free, ctx->star, d);
  KS_LAUNCHED(ctx);
  int h = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->max_star = h;
  // KS_ASM_MASK (read here, at ks_create; A/B and tests): "0" = no masks (the k_assemble_sell walk), "64" =
  // 64-bit masks even for stars <= 32; unset: the narrowest mask the mesh allows
  const char *e = getenv("KS_ASM_MASK");
  ctx->mask_bits = h <= 32 ? 32 : h <= STAR_MAX ? 64 : 0;
  if (e && !strcmp(e, "0")) ctx->mask_bits = 0;
  if (e && !strcmp(e, "64") && ctx->mask_bits) ctx->mask_bits = 64;
  if (ctx->mask_bits == 32) {
    k_slot_masks<<<ks_blocks(ctx->n_free, 256), 256, 0, ctx->stream>>>(
        ctx->row_ptr, ctx->sell_ptr, ctx->star, ctx->inv_ptr, ctx->inv_idx, ctx->n_free,
        reinterpret_cast<uint32_t *>(ctx->slot_mask));
    KS_LAUNCHED(ctx);
  } else if (ctx->mask_bits == 64) {
    k_slot_masks<<<ks_blocks(ctx->n_free, 256), 256, 0, ctx->stream>>>(ctx->row_ptr, ctx->sell_ptr, ctx->star,
                                                                       ctx->inv_ptr, ctx->inv_idx, ctx->n_free,
                                                                       ctx->slot_mask);
    KS_LAUNCHED(ctx);
  }
  return KS_OK;
}

ks_status ks_assemble_impl(ks_ctx *ctx, const double *d_veff, double mu) {
  cudaStream_t s = ctx->stream;
  const int64_t n = ctx->n_tets > ctx->n_free ? ctx->n_tets : ctx->n_free;
  k_tet_weights<<<ks_blocks(n, 256), 256, 0, s>>>(ctx->tets, ctx->vol, d_veff, ctx->n_tets, ctx->node_of_free,
                                                  ctx->n_free, ctx->w_tet, ctx->v_free, ctx->d_flags);
  KS_LAUNCHED(ctx);
#ifndef KS_ASM_SELL
#define KS_ASM_SELL 1
#endif
#ifndef KS_ASM_STAR
#define KS_ASM_STAR 1
#endif
  const unsigned mask_blocks = (unsigned)((ctx->n_slices + ASM_WARPS - 1) / ASM_WARPS);
  if (KS_ASM_STAR && ctx->mask_bits == 32) {
    k_assemble_mask<<<mask_blocks, ASM_WARPS * 32, 0, s>>>(
        ctx->sell_ptr, ctx->sell_col, reinterpret_cast<const uint32_t *>(ctx->slot_mask), ctx->sell_K, ctx->sell_M,
        ctx->star, ctx->inv_idx, ctx->w_tet, ctx->v_free, mu, ctx->n_free, ctx->n_slices, ctx->sell_A, ctx->sell_H,
        ctx->diag, ctx->dinv);
  } else if (KS_ASM_STAR && ctx->mask_bits == 64) {
    k_assemble_mask<<<mask_blocks, ASM_WARPS * 32, 0, s>>>(
        ctx->sell_ptr, ctx->sell_col, ctx->slot_mask, ctx->sell_K, ctx->sell_M, ctx->star, ctx->inv_idx, ctx->w_tet,
        ctx->v_free, mu, ctx->n_free, ctx->n_slices, ctx->sell_A, ctx->sell_H, ctx->diag, ctx->dinv);
  } else if (KS_ASM_SELL) {
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
  ctx->ah_fresh = 0;   // H changed: the projection's A_H partials are stale
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
