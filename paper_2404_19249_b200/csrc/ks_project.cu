// ks_project.cu -- projection of H and M onto the augmented subspace W = [P | U~]:
//   F_A = [[A_H, b_H], [b_H^T, beta]],  F_B = [[B_H, c_H], [c_H^T, gamma]]                (st1)-(st2)
//   A_H = P^T H P (st5), b_H = P^T H U~ (st6), beta = U~^T H U~ (st7);
//   B_H = P^T M P (cached per mesh pair), c_H = P^T M U~, gamma = U~^T M U~ (717-731).
//
// Design (DESIGN.md §4.4 "projection"). Fine rows are grouped by their coarse parent set S (the <= 4
// coarse nodes with P_ic != 0) and cut into "items" of <= ITEM_ROWS rows. Every contribution of a row
// lands in coarse rows c in S, so one warp can accumulate an item privately:
//   K8a k_proj_y      Y_H = H U~ and Y_M = M U~ on the sliced-ELL copies (one pass, shared col stream)
//   K8b k_proj_ai     item partials sum_i P_ic (H P)_{i,d}, d in the item's coarse window D, on an item-ordered
//                     sliced-ELL copy of the pattern (columns, window slots) built by ks_set_coarse; k_proj_a (the
//                     same sums with per-entry loads) serves Op = M (cached B_H) and Op = K (Hartree coarse operator)
//   K8c k_proj_bg     item partials sum_i P_ic Y_H[i] / Y_M[i] (b_H, c_H) and, per warp, the Gram
//                     partials beta, gamma = U~^T Y (symmetric: upper 4x4 tiles), rows in item order
//   K9  k_proj_final  one block per coarse node c: fixed-order sums over the items containing c;
//       k_gram_fin    fixed-order sums of the Gram partials.
// Everything is deterministic (fixed partitions and orders, no float atomics).
#include <cub/cub.cuh>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "ks_internal.cuh"
#include "ks_layout.cuh"
#include "ks_rowops.cuh"
#include "ks_sell.cuh"

namespace {

constexpr int ITEM_ROWS = 128;   // rows per item (chunk of a parent-set group)
constexpr int DMAX = 255;        // max coarse window of an item (u8 slots; 255 = "no slot")

// ---------------------------------------------------------------------------------------------
// setup kernels
// ---------------------------------------------------------------------------------------------
// validate P rows (<= 4 entries, columns in range), sort each row by column, build the parent-set key
__global__ void k_P_rows_keys(int32_t *__restrict__ ptr, int32_t *__restrict__ col, double *__restrict__ val,
                              int64_t n_free, int64_t n_H, int64_t p_nnz, uint64_t *__restrict__ key,
                              int32_t *__restrict__ rows, unsigned long long *bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_free) return;
  int32_t a = ptr[i], b = ptr[i + 1];
  bool ok = a >= 0 && b >= a && b - a <= 4 && b <= p_nnz;
  int32_t c[4];
  double v[4];
  int m = ok ? b - a : 0;
  for (int q = 0; q < m; q++) {
    c[q] = col[a + q];
    v[q] = val[a + q];
    ok &= c[q] >= 0 && c[q] < n_H;
  }
  for (int x = 1; x < m; x++)
    for (int y = x; y > 0 && c[y - 1] > c[y]; y--) {
      int32_t tc = c[y]; c[y] = c[y - 1]; c[y - 1] = tc;
      double tv = v[y]; v[y] = v[y - 1]; v[y - 1] = tv;
    }
  for (int x = 1; x < m; x++) ok &= c[x] != c[x - 1];
  if (!ok) {
    atomicMin(bad, (unsigned long long)i);
    return;
  }
  uint64_t B = (uint64_t)n_H + 1, k = 0;
  for (int q = 0; q < 4; q++) k = k * B + (uint64_t)(q < m ? c[q] : n_H);
  for (int q = 0; q < m; q++) { col[a + q] = c[q]; val[a + q] = v[q]; }
  key[i] = k;
  rows[i] = (int32_t)i;
}

__global__ void k_group_flags(const uint64_t *__restrict__ ks, int64_t n, int32_t *__restrict__ flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) flag[i] = (i == 0 || ks[i] != ks[i - 1]) ? 1 : 0;
}

__global__ void k_group_first(const int32_t *__restrict__ flag, const int32_t *__restrict__ gincl, int64_t n,
                              int32_t *__restrict__ gfirst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && flag[i]) gfirst[gincl[i] - 1] = (int32_t)i;
}

__global__ void k_item_flags(const int32_t *__restrict__ gincl, const int32_t *__restrict__ gfirst, int64_t n,
                             int32_t *__restrict__ iflag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) iflag[i] = ((i - gfirst[gincl[i] - 1]) % ITEM_ROWS) == 0 ? 1 : 0;
}

__global__ void k_item_ptr(const int32_t *__restrict__ iflag, const int32_t *__restrict__ iincl, int64_t n,
                           int32_t *__restrict__ item_ptr, int32_t *__restrict__ item_of_pos) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  item_of_pos[i] = iincl[i] - 1;
  if (iflag[i]) item_ptr[iincl[i] - 1] = (int32_t)i;
}

__global__ void k_item_S(const int32_t *__restrict__ item_ptr, const int32_t *__restrict__ perm,
                         const int32_t *__restrict__ Pptr, const int32_t *__restrict__ Pcol, int64_t n_items,
                         int32_t *__restrict__ item_S, int32_t *__restrict__ ct_key, int32_t *__restrict__ ct_val,
                         int32_t n_H) {
  int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (it >= n_items) return;
  int32_t i = perm[item_ptr[it]];
  int32_t a = Pptr[i], m = Pptr[i + 1] - a;
  for (int q = 0; q < 4; q++) {
    int32_t c = q < m ? Pcol[a + q] : -1;
    item_S[4 * it + q] = c;
    ct_key[4 * it + q] = c >= 0 ? c : n_H;
    ct_val[4 * it + q] = (int32_t)(4 * it + q);
  }
}

// Per item: the sorted set D of coarse columns of P rows of all neighbours of the item's rows.
// Bitmap over coarse ids in shared memory (order-independent -> deterministic). pass 0: counts.
__global__ void k_item_D(const int32_t *__restrict__ item_ptr, const int32_t *__restrict__ perm,
                         const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                         const int32_t *__restrict__ Pptr, const int32_t *__restrict__ Pcol, int32_t n_H,
                         int32_t *__restrict__ D_cnt, const int32_t *__restrict__ D_ptr, int32_t *__restrict__ D) {
  extern __shared__ unsigned bits[];
  __shared__ int32_t wsum[33];
  const int64_t it = blockIdx.x;
  const int nw = (n_H + 31) / 32;
  for (int w = threadIdx.x; w < nw; w += blockDim.x) bits[w] = 0u;
  __syncthreads();
  const int32_t p0 = item_ptr[it], p1 = item_ptr[it + 1];
  for (int32_t pos = p0 + threadIdx.x / 32; pos < p1; pos += blockDim.x / 32) {
    const int32_t i = perm[pos];
    for (int32_t k = row_ptr[i] + (threadIdx.x & 31); k < row_ptr[i + 1]; k += 32) {
      const int32_t j = col[k];
      for (int32_t t = Pptr[j]; t < Pptr[j + 1]; t++) {
        const int32_t d = Pcol[t];
        atomicOr(&bits[d >> 5], 1u << (d & 31));
      }
    }
  }
  __syncthreads();
  // contiguous chunk of words per thread -> popcounts -> block exclusive scan (fixed)
  const int per = (nw + blockDim.x - 1) / blockDim.x;
  const int w0 = threadIdx.x * per, w1 = min(nw, w0 + per);
  int cnt = 0;
  for (int w = w0; w < w1; w++) cnt += __popc(bits[w]);
  if (D_cnt) {
    // block reduce
    int v = cnt;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      int s = 0;
      for (int w = 0; w < (int)blockDim.x / 32; w++) s += wsum[w];
      D_cnt[it] = s;
    }
    return;
  }
  // exclusive scan of cnt over threads
  int v = cnt;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    int u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  if (lane == 31) wsum[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < (int)blockDim.x / 32; w++) { int t = wsum[w]; wsum[w] = s; s += t; }
  }
  __syncthreads();
  int off = D_ptr[it] + wsum[warp] + v - cnt;
  for (int w = w0; w < w1; w++) {
    unsigned b = bits[w];
    while (b) {
      int l = __ffs(b) - 1;
      D[off++] = w * 32 + l;
      b &= b - 1;
    }
  }
}

// slot of each (entry k, parent t of col[k]) inside the D list of the row's item
__global__ void k_slotmap(const int32_t *__restrict__ perm, const int32_t *__restrict__ item_of_pos,
                          const int32_t *__restrict__ D_ptr, const int32_t *__restrict__ D,
                          const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                          const int32_t *__restrict__ Pptr, const int32_t *__restrict__ Pcol, int64_t n_free,
                          uint8_t *__restrict__ slotmap) {
  int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (pos >= n_free) return;
  const int32_t i = perm[pos], it = item_of_pos[pos];
  const int32_t d0 = D_ptr[it], dn = D_ptr[it + 1] - d0;
  for (int32_t k = row_ptr[i]; k < row_ptr[i + 1]; k++) {
    const int32_t j = col[k];
    const int32_t a = Pptr[j], m = Pptr[j + 1] - a;
    for (int t = 0; t < 4; t++) {
      uint8_t s = 255;
      if (t < m) {
        const int32_t c = Pcol[a + t];
        int lo = 0, hi = dn;
        while (lo < hi) {
          int mid = (lo + hi) >> 1;
          if (D[d0 + mid] < c) lo = mid + 1; else hi = mid;
        }
        s = (uint8_t)lo;
      }
      slotmap[4 * (int64_t)k + t] = s;
    }
  }
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

// ---- item-ordered sliced-ELL copy of the pattern (k_proj_ai): items padded to whole 8-row slices ----
__global__ void k_item_nslices(const int32_t *__restrict__ item_ptr, int64_t ni, int32_t *__restrict__ cnt) {
  const int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (it < ni) cnt[it] = (item_ptr[it + 1] - item_ptr[it] + KS_SELL_C - 1) / KS_SELL_C;
}
// slots of every item slice: 8 rows x its longest row rounded up to a 4-slot group
__global__ void k_islice_width(const int32_t *__restrict__ item_ptr, const int32_t *__restrict__ islice0,
                               const int32_t *__restrict__ perm, const int32_t *__restrict__ row_ptr, int64_t ni,
                               int32_t *__restrict__ isw) {
  const int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (it >= ni) return;
  const int32_t p0 = item_ptr[it], nr = item_ptr[it + 1] - p0;
  for (int32_t r0 = 0; r0 < nr; r0 += KS_SELL_C) {
    int32_t w = 0;
    for (int32_t r = r0; r < nr && r < r0 + KS_SELL_C; r++) {
      const int32_t i = perm[p0 + r];
      w = max(w, row_ptr[i + 1] - row_ptr[i]);
    }
    isw[islice0[it] + r0 / KS_SELL_C] = (w + 3) / 4 * 4 * KS_SELL_C;
  }
}
// thread per item position: the row's item-layout columns (padding: own row) and window-slot words
// (word (g, t): byte u = slot of parent t of column 4g+u, 255 absent or padding), and its natural sliced-ELL base
// and slot groups (H is read there)
__global__ void k_isell_fill(const int32_t *__restrict__ perm, const int32_t *__restrict__ item_of_pos,
                             const int32_t *__restrict__ item_ptr, const int32_t *__restrict__ islice0,
                             const int32_t *__restrict__ isell_ptr, const int32_t *__restrict__ row_ptr,
                             const int32_t *__restrict__ col, const int32_t *__restrict__ sell_ptr,
                             const uint8_t *__restrict__ slotmap, int64_t n_free, int2 *__restrict__ inat,
                             int32_t *__restrict__ icol, uint32_t *__restrict__ islot) {
  const int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (pos >= n_free) return;
  const int32_t i = perm[pos], it = item_of_pos[pos];
  const int64_t ip = (int64_t)KS_SELL_C * islice0[it] + (pos - item_ptr[it]);
  const int32_t sb = isell_ptr[ip / KS_SELL_C], groups = (isell_ptr[ip / KS_SELL_C + 1] - sb) / (4 * KS_SELL_C);
  const int32_t base = sb + (int32_t)(ip % KS_SELL_C) * 4;
  const int32_t k0 = row_ptr[i], len = row_ptr[i + 1] - k0;
  const int32_t nb = sell_ptr[i / KS_SELL_C] + (i % KS_SELL_C) * 4;
  inat[pos] = make_int2(nb, (len + 3) / 4);
  for (int g = 0; g < groups; g++)
    for (int q = 0; q < 4; q++) {
      const int k = 4 * g + q;
      const int64_t o = base + (int64_t)g * (4 * KS_SELL_C) + q;
      icol[o] = k < len ? col[k0 + k] : i;
      uint32_t w = 0;
      for (int u = 3; u >= 0; u--) {
        const int ku = 4 * g + u;
        w = (w << 8) | (ku < len ? (uint32_t)slotmap[4 * (int64_t)(k0 + ku) + q] : 255u);
      }
      islot[o] = w;
    }
}

// ---------------------------------------------------------------------------------------------
// projection kernels (v2)
// ---------------------------------------------------------------------------------------------
// K8a  k_proj_y   Y_H = H U~, Y_M = M U~ on the sliced-ELL copies (rows in natural order, coalesced)
// K8b  k_proj_a   per item: sum_i P_ic (Op P)_{i,d} for c in S, d in the item window D  (A_H / B_H)
// K8c  k_proj_bg  per item: b/c partials sum_i P_ic Y[i]; per warp: Gram partials U~^T Y (upper tiles)
// K9   k_proj_final / k_gram_fin: fixed-order sums of the partials into F_A, F_B.

template <int NP>
#ifndef KS_PY_MINB
#define KS_PY_MINB 4   // <= 64 registers: 4 blocks/SM (A/B: 436 vs 468 us at C4, same box)
#endif
__global__ void __launch_bounds__(256, KS_PY_MINB) k_proj_y(const int32_t *__restrict__ sell_ptr, const int32_t *__restrict__ sell_col,
                                                const double *__restrict__ H, const double *__restrict__ M,
                                                const double *__restrict__ U, const int32_t *__restrict__ pos_of_row,
                                                double *__restrict__ Up, double *__restrict__ YHp,
                                                double *__restrict__ YMp, int64_t n, bool write_up) {
  // rows in natural order (coalesced operator stream); outputs scattered, one full row each, into item
  // order (position pos_of_row[row] of the coarse-parent grouping) for the item pass k_proj_bg; the
  // item-ordered copy of U~ only for the FFMA pass (write_up; the tensor-core pass copies U~ rows itself)
  constexpr int VEC = SL<NP>::VEC, LPR = SL<NP>::LPR;
  const int64_t gl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t row = gl / LPR;
  const int sub = (int)(gl % LPR);
  if (row >= n) return;
  DV<VEC> yh, ym;
  sell_row<NP, 2>(sell_ptr, sell_col, H, M, row, U, sub, yh, ym);
  const int64_t o = (int64_t)__ldg(pos_of_row + row) * NP + sub * VEC;
  if (write_up) DV<VEC>::ld(U + row * NP + sub * VEC).st(Up + o);
  yh.st(YHp + o);
  ym.st(YMp + o);
}

// Item partials of P^T Op P (A_H with Op = H, B_H with Op = M), G[c][d] = sum_{i in item} P_ic (Op P)_{i,d}
// for the item's parents c and window slots d. No float atomics; the partition and all orders are fixed.
#ifndef KS_PA_UNR
#define KS_PA_UNR 16   // A/B: 389 -> 367 us at C4, 1.23 -> 1.15 ms at C5 (vs 8)
#endif
constexpr int PA_UNR = KS_PA_UNR;   // nonzeros of a row in flight per thread

// Row part: the row's contributions are added in place in its shared row of the item window. The 4 parents of one nonzero have distinct slots (distinct coarse nodes), so their 4
// read-modify-writes are issued together (one shared-memory latency per nonzero); absent parents write
// the pad column wcap. Nonzeros in CSR order, parents ascending: fixed order.
__device__ __forceinline__ void proj_a_row_smem(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                                const int32_t *__restrict__ sell_ptr, const double *__restrict__ sval,
                                                const uint8_t *__restrict__ slotmap, const double *__restrict__ Pv4,
                                                int32_t i, double *Wl, int wcap) {
  const int32_t k0 = __ldg(row_ptr + i), k1 = __ldg(row_ptr + i + 1);
  const int64_t sb = __ldg(sell_ptr + i / KS_SELL_C) + (i % KS_SELL_C) * 4;
  for (int32_t kb = k0; kb < k1; kb += PA_UNR) {
    int32_t j[PA_UNR];
    double h[PA_UNR];
    uchar4 sl[PA_UNR];
#pragma unroll
    for (int u = 0; u < PA_UNR; u++) {
      const bool in = kb + u < k1;
      const int32_t k = in ? kb + u : k0, kl = k - k0;
      j[u] = __ldg(col + k);
      h[u] = in ? __ldg(sval + sb + (kl >> 2) * (4 * KS_SELL_C) + (kl & 3)) : 0.0;
      sl[u] = in ? __ldg(reinterpret_cast<const uchar4 *>(slotmap) + k) : make_uchar4(255, 255, 255, 255);
    }
    double q[PA_UNR][4];
#pragma unroll
    for (int u = 0; u < PA_UNR; u++) ldnc_v4(Pv4 + 4 * (int64_t)j[u], q[u][0], q[u][1], q[u][2], q[u][3]);
#pragma unroll
    for (int u = 0; u < PA_UNR; u++) {
      const int s0 = sl[u].x == 255 ? wcap : sl[u].x, s1 = sl[u].y == 255 ? wcap : sl[u].y;
      const int s2 = sl[u].z == 255 ? wcap : sl[u].z, s3 = sl[u].w == 255 ? wcap : sl[u].w;
      const double w0 = Wl[s0], w1 = Wl[s1], w2 = Wl[s2], w3 = Wl[s3];
      Wl[s0] = fma(h[u], q[u][0], w0);
      Wl[s1] = fma(h[u], q[u][1], w1);
      Wl[s2] = fma(h[u], q[u][2], w2);
      Wl[s3] = fma(h[u], q[u][3], w3);
    }
  }
}

// One block of ITEM_ROWS threads per item (all of its rows at once):
//   1. thread = row r of the item: its row W[r][0..dn) of the item window (proj_a_row_smem), and P_r;
//   2. G = P_item^T W on the FP64 tensor cores (mma.m8n8k4.f64), one warp per 8-column tile of the window.
#ifndef KS_PA_MINB
#define KS_PA_MINB 1
#endif
__global__ void __launch_bounds__(ITEM_ROWS, KS_PA_MINB) k_proj_a(const int32_t *__restrict__ row_ptr,
                                                     const int32_t *__restrict__ col,
                                                     const int32_t *__restrict__ sell_ptr,
                                                     const double *__restrict__ sval,
                                                     const uint8_t *__restrict__ slotmap,
                                                     const double *__restrict__ Pv4,
                                                     const int32_t *__restrict__ perm,
                                                     const int32_t *__restrict__ item_ptr,
                                                     const int32_t *__restrict__ D_ptr, int64_t n_items, int wcap,
                                                     double *__restrict__ AH_part) {
  extern __shared__ double smem[];
  const int ws = wcap + 1;                       // odd row stride; column wcap is the pad (absent parents)
  double *W = smem;                              // [ITEM_ROWS][ws]
  double *Ps = smem + ITEM_ROWS * ws;            // [ITEM_ROWS][4]
  const int tid = threadIdx.x;
  for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int32_t p0 = __ldg(item_ptr + it), p1 = __ldg(item_ptr + it + 1);
    const int32_t d0 = __ldg(D_ptr + it), dn = __ldg(D_ptr + it + 1) - d0;
    const int nr = p1 - p0;
    double *Wl = W + tid * ws;
    for (int d = 0; d < dn; d++) Wl[d] = 0.0;
    if (tid < nr) {
      const int32_t i = __ldg(perm + p0 + tid);
      double pi0, pi1, pi2, pi3;
      ldnc_v4(Pv4 + 4 * (int64_t)i, pi0, pi1, pi2, pi3);
      Ps[tid * 4 + 0] = pi0; Ps[tid * 4 + 1] = pi1; Ps[tid * 4 + 2] = pi2; Ps[tid * 4 + 3] = pi3;
      proj_a_row_smem(row_ptr, col, sell_ptr, sval, slotmap, Pv4, i, Wl, wcap);
    }
    __syncthreads();
    // G = P_item^T W on the FP64 tensor cores: warp w takes the 8-column tiles w, w + 4, ... of the window;
    // k-steps of 4 rows; A[m = c][k = r] = P_rc (rows 4..7 zero), B[k = r][n = d] = W[r][d]. Rows past nr
    // and columns past dn are zeroed by select (stale shared memory).
    const int lane = tid & 31, warp = tid >> 5, grp = lane >> 2, tig = lane & 3;
    double *out = AH_part + 4 * (int64_t)d0;
    for (int t = warp; 8 * t < dn; t += ITEM_ROWS / 32) {
      const int d = 8 * t + grp;
      double c0 = 0.0, c1 = 0.0;
      for (int r0 = 0; r0 < nr; r0 += 4) {
        const int r = r0 + tig;
        const double av = (grp < 4 && r < nr) ? Ps[r * 4 + grp] : 0.0;
        const double bv = (r < nr && d < dn) ? W[r * ws + d] : 0.0;
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c0), "+d"(c1) : "d"(av), "d"(bv));
      }
      if (grp < 4) {
        const int dd = 8 * t + 2 * tig;
        if (dd < dn) out[grp * dn + dd] = c0;
        if (dd + 1 < dn) out[grp * dn + dd + 1] = c1;
      }
    }
    __syncthreads();
  }
}

// k_proj_a on the item-ordered sliced-ELL copy (default; KS_PROJ_AI=0: k_proj_a): thread = row of the item as in k_proj_a, but each
// 4-slot group of the row is one coalesced 16-byte column load, one 16-byte window-slot load (the 4 parents' words)
// and one 32-byte H sector (natural layout), instead of per-entry loads scattered over the rows of the item. Same
// entries in the same order into the same window rows and the same k-step chain: bitwise k_proj_a's partials.
#ifndef KS_PAI_G
#define KS_PAI_G 4
#endif
#ifndef KS_PAI_MINB
#define KS_PAI_MINB 1
#endif
constexpr int PAI_G = KS_PAI_G;   // slot groups (16 entries) in flight per thread
__global__ void __launch_bounds__(ITEM_ROWS, KS_PAI_MINB) k_proj_ai(
    const int32_t *__restrict__ item_ptr, const int32_t *__restrict__ islice0, const int32_t *__restrict__ isell_ptr,
    const int32_t *__restrict__ isell_col, const int2 *__restrict__ inat, const double *__restrict__ sval,
    const uint32_t *__restrict__ islot, const double *__restrict__ Pv4, const double *__restrict__ Pv4p,
    const int32_t *__restrict__ D_ptr, int64_t n_items, int wcap, double *__restrict__ AH_part) {
  extern __shared__ double smem[];
  const int ws = wcap + 1;
  double *W = smem;                              // [ITEM_ROWS][ws]
  double *Ps = smem + ITEM_ROWS * ws;            // [ITEM_ROWS][4]
  const int tid = threadIdx.x;
  for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int32_t p0 = __ldg(item_ptr + it), nr = __ldg(item_ptr + it + 1) - p0, s0 = __ldg(islice0 + it);
    const int32_t d0 = __ldg(D_ptr + it), dn = __ldg(D_ptr + it + 1) - d0;
    double *Wl = W + tid * ws;
    for (int d = 0; d < dn; d++) Wl[d] = 0.0;
    if (tid < nr) {
      double pi0, pi1, pi2, pi3;
      ldnc_v4(Pv4p + 4 * (int64_t)(p0 + tid), pi0, pi1, pi2, pi3);
      Ps[tid * 4 + 0] = pi0; Ps[tid * 4 + 1] = pi1; Ps[tid * 4 + 2] = pi2; Ps[tid * 4 + 3] = pi3;
      const int2 nat = __ldg(inat + p0 + tid);
      const int64_t ib = __ldg(isell_ptr + s0 + tid / KS_SELL_C) + (tid % KS_SELL_C) * 4;
      for (int g0 = 0; g0 < nat.y; g0 += PAI_G) {
        int4 c[PAI_G];
        uint4 sw[PAI_G];
        double h[PAI_G][4];
#pragma unroll
        for (int q = 0; q < PAI_G; q++) {
          const int g = g0 + q < nat.y ? g0 + q : g0;   // past the row: a repeat, masked below
          const int64_t o = ib + (int64_t)g * (4 * KS_SELL_C);
          c[q] = __ldg(reinterpret_cast<const int4 *>(isell_col + o));
          sw[q] = __ldg(reinterpret_cast<const uint4 *>(islot + o));
          ldnc_v4(sval + nat.x + (int64_t)g * (4 * KS_SELL_C), h[q][0], h[q][1], h[q][2], h[q][3]);
        }
        double pv[PAI_G][4][4];
#pragma unroll
        for (int q = 0; q < PAI_G; q++) {
          ldnc_v4(Pv4 + 4 * (int64_t)c[q].x, pv[q][0][0], pv[q][0][1], pv[q][0][2], pv[q][0][3]);
          ldnc_v4(Pv4 + 4 * (int64_t)c[q].y, pv[q][1][0], pv[q][1][1], pv[q][1][2], pv[q][1][3]);
          ldnc_v4(Pv4 + 4 * (int64_t)c[q].z, pv[q][2][0], pv[q][2][1], pv[q][2][2], pv[q][2][3]);
          ldnc_v4(Pv4 + 4 * (int64_t)c[q].w, pv[q][3][0], pv[q][3][1], pv[q][3][2], pv[q][3][3]);
        }
#pragma unroll
        for (int q = 0; q < PAI_G; q++) {
          if (g0 + q >= nat.y) break;
          const uint32_t w4[4] = {sw[q].x, sw[q].y, sw[q].z, sw[q].w};
#pragma unroll
          for (int u = 0; u < 4; u++) {   // entry 4g+u; parent t's slot is byte u of word t
            int sl[4];
#pragma unroll
            for (int t = 0; t < 4; t++) {
              const int v = (int)((w4[t] >> (8 * u)) & 255u);
              sl[t] = v == 255 ? wcap : v;
            }
            const double w0 = Wl[sl[0]], w1 = Wl[sl[1]], w2 = Wl[sl[2]], w3 = Wl[sl[3]];
            Wl[sl[0]] = fma(h[q][u], pv[q][u][0], w0);
            Wl[sl[1]] = fma(h[q][u], pv[q][u][1], w1);
            Wl[sl[2]] = fma(h[q][u], pv[q][u][2], w2);
            Wl[sl[3]] = fma(h[q][u], pv[q][u][3], w3);
          }
        }
      }
    }
    __syncthreads();
    const int lane = tid & 31, warp = tid >> 5, grp = lane >> 2, tig = lane & 3;
    double *out = AH_part + 4 * (int64_t)d0;
    for (int t = warp; 8 * t < dn; t += ITEM_ROWS / 32) {
      const int d = 8 * t + grp;
      double c0 = 0.0, c1 = 0.0;
      for (int r0 = 0; r0 < nr; r0 += 4) {
        const int r = r0 + tig;
        const double av = (grp < 4 && r < nr) ? Ps[r * 4 + grp] : 0.0;
        const double bv = (r < nr && d < dn) ? W[r * ws + d] : 0.0;
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c0), "+d"(c1) : "d"(av), "d"(bv));
      }
      if (grp < 4) {
        const int dd = 8 * t + 2 * tig;
        if (dd < dn) out[grp * dn + dd] = c0;
        if (dd + 1 < dn) out[grp * dn + dd + 1] = c1;
      }
    }
    __syncthreads();
  }
}

// Item pass (item order: Up, YHp, YMp, Pv4p are stored by position, so every item's rows are contiguous):
// b/c partials per item and Gram partials per warp. Each warp owns a contiguous range of items and streams
// its rows through a 2-stage shared-memory ring with bulk (TMA) copies, lane 0 producing, all lanes
// consuming. Gram: 4x4 register tiles (op, ta, tb), ta <= tb (the blocks are symmetric), lane l owns tiles
// l, l + 32, ...; b/c: lane l owns (op, c) = l / 4 and the orbitals b of quarter l % 4.
constexpr int PBG_WARPS = 8;     // warps per block of k_proj_bg
constexpr int PBG_STAGES = 2;
template <int NP>
struct PbgLayout {
  static constexpr int CH = NP <= 16 ? 16 : NP == 32 ? 8 : 4;           // rows per stage
  static constexpr int STAGE = CH * (3 * NP + 4);                        // doubles per stage
  static constexpr size_t WARP_BYTES = sizeof(double) * PBG_STAGES * STAGE;
};

template <int NP, bool GRAM>
__global__ void __launch_bounds__(PBG_WARPS * 32) k_proj_bg(const double *__restrict__ Up, const double *__restrict__ YHp,
                                                            const double *__restrict__ YMp,
                                                            const double *__restrict__ Pv4p,
                                                            const int32_t *__restrict__ item_ptr, int64_t n_items,
                                                            double *__restrict__ bH_part, double *__restrict__ cH_part,
                                                            double *__restrict__ gram_part) {
  constexpr int T4 = NP >= 4 ? NP / 4 : 1;                 // 4-wide tiles per dimension
  constexpr int NT2 = T4 * (T4 + 1) / 2;                   // upper tiles per operator
  constexpr int MAXT = (2 * NT2 + 31) / 32;                // tiles per lane
  constexpr int BQ = NP >= 4 ? NP / 4 : NP;                // b/c orbitals per lane (NP >= 4: a quarter)
  constexpr int CH = PbgLayout<NP>::CH, STAGE = PbgLayout<NP>::STAGE;
  extern __shared__ __align__(16) double dsm[];
  __shared__ __align__(8) uint64_t bars[PBG_WARPS][PBG_STAGES];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *ring = dsm + (size_t)warp * PBG_STAGES * STAGE;
  const int64_t gw = (int64_t)blockIdx.x * PBG_WARPS + warp, nw = (int64_t)gridDim.x * PBG_WARPS;
  // contiguous item range of this warp, and its rows
  const int64_t ia = n_items * gw / nw, ib = n_items * (gw + 1) / nw;
  const int32_t ra = __ldg(item_ptr + ia), rb = __ldg(item_ptr + ib);
  const int nchunks = (rb - ra + CH - 1) / CH;

  int t_op[MAXT], t_a[MAXT], t_b[MAXT];
#pragma unroll
  for (int q = 0; q < MAXT; q++) {
    int id = lane + 32 * q, op = -1, ta = 0, tb = 0;
    if (id < 2 * NT2) {
      op = id / NT2;
      int r = id % NT2;
      while (r >= T4 - ta) { r -= T4 - ta; ta++; }
      tb = ta + r;
    }
    t_op[q] = op; t_a[q] = ta; t_b[q] = tb;
  }
  double g[MAXT][16];
#pragma unroll
  for (int q = 0; q < MAXT; q++)
#pragma unroll
    for (int e = 0; e < 16; e++) g[q][e] = 0.0;
  const int bc_op = lane >> 4, bc_c = (lane >> 2) & 3, bc_b0 = NP >= 4 ? (lane & 3) * BQ : 0;
  const bool bc_on = NP >= 4 || (lane & 3) == 0;

  auto issue = [&](int c) {   // lane 0: chunk c of this warp's rows into stage c % PBG_STAGES
    const int st = c % PBG_STAGES;
    const int32_t r0 = ra + c * CH, cnt = min(CH, rb - r0);
    double *S = ring + st * STAGE;
    const unsigned bv = (unsigned)cnt * NP * 8u, bp = (unsigned)cnt * 32u;
    mbar_expect_tx(&bars[warp][st], 3 * bv + bp);
    bulk_g2s(S, Up + (int64_t)r0 * NP, bv, &bars[warp][st]);
    bulk_g2s(S + CH * NP, YHp + (int64_t)r0 * NP, bv, &bars[warp][st]);
    bulk_g2s(S + 2 * CH * NP, YMp + (int64_t)r0 * NP, bv, &bars[warp][st]);
    bulk_g2s(S + 3 * CH * NP, Pv4p + 4 * (int64_t)r0, bp, &bars[warp][st]);
  };
  if (lane == 0) {
    for (int st = 0; st < PBG_STAGES; st++) mbar_init(&bars[warp][st], 1);
    mbar_fence_init();
    for (int c = 0; c < PBG_STAGES && c < nchunks; c++) issue(c);
  }
  __syncwarp();

  int64_t it = ia;
  int32_t iend = __ldg(item_ptr + ia + 1);
  double bc[BQ];
#pragma unroll
  for (int v = 0; v < BQ; v++) bc[v] = 0.0;
  auto flush = [&]() {
    if (bc_on) {
      double *dst = (bc_op ? cH_part : bH_part) + (4 * it + bc_c) * NP + bc_b0;
#pragma unroll
      for (int v = 0; v < BQ; v++) dst[v] = bc[v];
    }
#pragma unroll
    for (int v = 0; v < BQ; v++) bc[v] = 0.0;
  };

  for (int c = 0; c < nchunks; c++) {
    const int st = c % PBG_STAGES;
    mbar_wait(&bars[warp][st], (unsigned)(c / PBG_STAGES) & 1u);
    const double *S = ring + st * STAGE;
    const int32_t r0 = ra + c * CH, cnt = min(CH, rb - r0);
    for (int rr = 0; rr < cnt; rr++) {
      while (r0 + rr >= iend) {     // item boundary (warp-uniform)
        flush();
        it++;
        iend = __ldg(item_ptr + it + 1);
      }
      const double *Ur = S + rr * NP, *Hr = S + CH * NP + rr * NP, *Mr = S + 2 * CH * NP + rr * NP;
      const double *Pr = S + 3 * CH * NP + rr * 4;
      if (GRAM) {
#pragma unroll
        for (int q = 0; q < MAXT; q++) {
          if (t_op[q] < 0) continue;
          const double *ua = Ur + 4 * t_a[q], *yb = (t_op[q] ? Mr : Hr) + 4 * t_b[q];
          double u4[4], y4[4];
          if (NP >= 4) {
            const double2 u01 = reinterpret_cast<const double2 *>(ua)[0], u23 = reinterpret_cast<const double2 *>(ua)[1];
            const double2 y01 = reinterpret_cast<const double2 *>(yb)[0], y23 = reinterpret_cast<const double2 *>(yb)[1];
            u4[0] = u01.x; u4[1] = u01.y; u4[2] = u23.x; u4[3] = u23.y;
            y4[0] = y01.x; y4[1] = y01.y; y4[2] = y23.x; y4[3] = y23.y;
          } else {
#pragma unroll
            for (int e = 0; e < 4; e++) { u4[e] = e < NP ? ua[e] : 0.0; y4[e] = e < NP ? yb[e] : 0.0; }
          }
#pragma unroll
          for (int x = 0; x < 4; x++)
#pragma unroll
            for (int y = 0; y < 4; y++) g[q][x * 4 + y] = fma(u4[x], y4[y], g[q][x * 4 + y]);
        }
      }
      if (bc_on) {
        const double pc = Pr[bc_c];
        const double *yv = (bc_op ? Mr : Hr) + bc_b0;
#pragma unroll
        for (int v = 0; v < BQ; v++) bc[v] = fma(pc, yv[v], bc[v]);
      }
    }
    __syncwarp();
    if (lane == 0 && c + PBG_STAGES < nchunks) issue(c + PBG_STAGES);
  }
  if (ib > ia) flush();   // the last item of the range
  if (GRAM) {
    // per-warp partial [2][NP][NP], both triangles (the lower one mirrored from the upper tiles)
    double *out = gram_part + gw * 2 * NP * NP;
#pragma unroll
    for (int q = 0; q < MAXT; q++) {
      if (t_op[q] < 0) continue;
      double *o = out + t_op[q] * NP * NP;
      for (int x = 0; x < 4; x++)
        for (int y = 0; y < 4; y++) {
          const int a = 4 * t_a[q] + x, b = 4 * t_b[q] + y;
          if (a < NP && b < NP) {
            o[a * NP + b] = g[q][x * 4 + y];
            if (t_a[q] != t_b[q]) o[b * NP + a] = g[q][x * 4 + y];
          }
        }
    }
  }
}

// The same item pass on the FP64 tensor cores (NP = 8, 16, 32): both products are dense
// contractions over the warp's rows, taken 4 rows (one k-step) at a time with mma.m8n8k4.f64:
//   Gram   G_op[8ta.., 8tb..] += U~[rows, 8ta..]^T Y_op[rows, 8tb..]      (upper tiles ta <= tb)
//   b / c  bc_op[c, 8tb..]    += P_item[rows, c]^T  Y_op[rows, 8tb..]      (A rows 0..3 = the 4 parent
//                                                                          slots, rows 4..7 zero)
// Fragments (PTX m8n8k4 .f64): A[m = lane/4][k = lane%4], B[k = lane%4][n = lane/4], C[m = lane/4][n =
// 2(lane%4) + v]. The Y fragments serve both products, so every staged double is read from shared memory
// once per lane group instead of once per register tile. A k-step that crosses an item boundary is split
// into masked segments (P = 0 outside the segment); rows past the chunk are zeroed by select (never by a
// multiply: stale shared memory may hold NaN patterns).
// U~ rows: NP <= 16 gathered from the natural-order block through perm with TMA tile::gather4 (4 rows per
// copy; no item-ordered copy of U~ is written by the Y pass: C4 net -45 us); NP = 32 from the item-ordered
// copy (per-row bulk copies cost the item pass +0.3 ms at C5, gather4 +0.22 ms: no net gain over the 0.24 ms
// the Y pass saves).
#ifndef KS_PBG_GATHER_MAXNP
#define KS_PBG_GATHER_MAXNP 16
#endif
#ifndef KS_PBG_G4
#define KS_PBG_G4 1   // the per-row U~ copies as TMA tile::gather4 (4 rows per copy, tensor map of U~): C4 item pass 165 -> 156 us
#endif
template <int NP>
__host__ __device__ constexpr bool pbg_gather_u() { return NP <= KS_PBG_GATHER_MAXNP; }

// TMA gather of 4 rows (row indices r0..r3, columns [0, box width)) of a 2-D tensor into shared memory
__device__ __forceinline__ void tma_gather4(void *dst, const CUtensorMap *map, int32_t r0, int32_t r1, int32_t r2,
                                            int32_t r3, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

template <int NP>
__global__ void __launch_bounds__(PBG_WARPS * 32, NP == 32 ? 1 : 2) k_proj_bg_mma(const double *__restrict__ U,
                                                                const int32_t *__restrict__ perm,
                                                                const double *__restrict__ YHp,
                                                                const double *__restrict__ YMp,
                                                                const double *__restrict__ Pv4p,
                                                                const int32_t *__restrict__ item_ptr, int64_t n_items,
                                                                double *__restrict__ bH_part,
                                                                double *__restrict__ cH_part,
                                                                double *__restrict__ gram_part,
                                                                const __grid_constant__ CUtensorMap tmapU) {
  static_assert(NP == 8 || NP == 16 || NP == 32, "mma item pass: NP in {8, 16, 32}");
  constexpr int TT = NP / 8;                       // 8-wide tiles per dimension
  constexpr int NU = TT * (TT + 1) / 2;            // upper tiles per operator
  constexpr int CH = PbgLayout<NP>::CH, STAGE = PbgLayout<NP>::STAGE;
  static_assert(CH % 4 == 0, "chunks of whole k-steps");
  extern __shared__ __align__(16) double dsm[];
  __shared__ __align__(8) uint64_t bars[PBG_WARPS][PBG_STAGES];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, grp = lane >> 2, tig = lane & 3;
  double *ring = dsm + (size_t)warp * PBG_STAGES * STAGE;
  const int64_t gw = (int64_t)blockIdx.x * PBG_WARPS + warp, nw = (int64_t)gridDim.x * PBG_WARPS;
  const int64_t ia = n_items * gw / nw, ib = n_items * (gw + 1) / nw;
  const int32_t ra = __ldg(item_ptr + ia), rb = __ldg(item_ptr + ib);
  const int nchunks = (rb - ra + CH - 1) / CH;

  double g[2][NU][2], bc[2][TT][2];
#pragma unroll
  for (int op = 0; op < 2; op++) {
#pragma unroll
    for (int t = 0; t < NU; t++) g[op][t][0] = g[op][t][1] = 0.0;
#pragma unroll
    for (int t = 0; t < TT; t++) bc[op][t][0] = bc[op][t][1] = 0.0;
  }

  // all lanes: lane 0 registers the stage's bytes and copies the contiguous item-ordered Y_H, Y_M and P
  // rows; the U~ rows come either per row (lane l < cnt: natural-order row perm[r0 + l], pbg_gather_u) or
  // as one contiguous copy of the item-ordered block (U = that copy)
  auto issue = [&](int c) {
    const int st = c % PBG_STAGES;
    const int32_t r0 = ra + c * CH, cnt = min(CH, rb - r0);
    double *S = ring + st * STAGE;
    const unsigned bv = (unsigned)cnt * NP * 8u, bp = (unsigned)cnt * 32u;
    const unsigned bu = (pbg_gather_u<NP>() && KS_PBG_G4) ? (unsigned)((cnt + 3) / 4) * 4u * NP * 8u : bv;
    if (lane == 0) {
      mbar_expect_tx(&bars[warp][st], bu + 2 * bv + bp);
      if constexpr (!pbg_gather_u<NP>()) bulk_g2s(S, U + (int64_t)r0 * NP, bv, &bars[warp][st]);
      bulk_g2s(S + CH * NP, YHp + (int64_t)r0 * NP, bv, &bars[warp][st]);
      bulk_g2s(S + 2 * CH * NP, YMp + (int64_t)r0 * NP, bv, &bars[warp][st]);
      bulk_g2s(S + 3 * CH * NP, Pv4p + 4 * (int64_t)r0, bp, &bars[warp][st]);
    }
    if constexpr (pbg_gather_u<NP>()) {
      __syncwarp();
#if KS_PBG_G4
      if (lane < (cnt + 3) / 4) {   // rows past cnt repeat the last valid row (masked in the fragments)
        int32_t rr[4];
#pragma unroll
        for (int q = 0; q < 4; q++) rr[q] = __ldg(perm + r0 + min(4 * lane + q, cnt - 1));
        tma_gather4(S + 4 * lane * NP, &tmapU, rr[0], rr[1], rr[2], rr[3], &bars[warp][st]);
      }
#else
      if (lane < cnt) bulk_g2s(S + lane * NP, U + (int64_t)__ldg(perm + r0 + lane) * NP, NP * 8u, &bars[warp][st]);
#endif
    }
  };
  if (lane == 0) {
    for (int st = 0; st < PBG_STAGES; st++) mbar_init(&bars[warp][st], 1);
    mbar_fence_init();
  }
  __syncwarp();
  for (int c = 0; c < PBG_STAGES && c < nchunks; c++) issue(c);

  int64_t it = ia;
  int32_t iend = __ldg(item_ptr + ia + 1);
  auto flush = [&]() {
    if (grp < 4) {
#pragma unroll
      for (int op = 0; op < 2; op++) {
        double *dst = (op ? cH_part : bH_part) + (4 * it + grp) * NP + 2 * tig;
#pragma unroll
        for (int t = 0; t < TT; t++) *reinterpret_cast<double2 *>(dst + 8 * t) = make_double2(bc[op][t][0], bc[op][t][1]);
      }
    }
#pragma unroll
    for (int op = 0; op < 2; op++)
#pragma unroll
      for (int t = 0; t < TT; t++) bc[op][t][0] = bc[op][t][1] = 0.0;
  };

  for (int c = 0; c < nchunks; c++) {
    const int st = c % PBG_STAGES;
    mbar_wait(&bars[warp][st], (unsigned)(c / PBG_STAGES) & 1u);
    const double *S = ring + st * STAGE;
    const int32_t r0 = ra + c * CH, cnt = min(CH, rb - r0);
    for (int kk = 0; kk < cnt; kk += 4) {
      const bool rv = kk + tig < cnt;
      const int so = (kk + tig) * NP + grp;
      double fu[TT], fh[TT], fm[TT];
#pragma unroll
      for (int t = 0; t < TT; t++) {
        fu[t] = rv ? S[so + 8 * t] : 0.0;
        fh[t] = rv ? S[CH * NP + so + 8 * t] : 0.0;
        fm[t] = rv ? S[2 * CH * NP + so + 8 * t] : 0.0;
      }
      int u = 0;
#pragma unroll
      for (int ta = 0; ta < TT; ta++)
#pragma unroll
        for (int tb = ta; tb < TT; tb++, u++) {
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(g[0][u][0]), "+d"(g[0][u][1]) : "d"(fu[ta]), "d"(fh[tb]));
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(g[1][u][0]), "+d"(g[1][u][1]) : "d"(fu[ta]), "d"(fm[tb]));
        }
      const double pv = (rv && grp < 4) ? S[3 * CH * NP + (kk + tig) * 4 + grp] : 0.0;
      const int32_t kb = r0 + kk, ke = min(kb + 4, r0 + cnt), r = kb + tig;
      int32_t lo = kb;
      while (true) {                       // segments of the k-step by item (warp-uniform)
        while (lo >= iend) {
          flush();
          it++;
          iend = __ldg(item_ptr + it + 1);
        }
        const int32_t hi = min(ke, iend);
        const double pa = (r >= lo && r < hi) ? pv : 0.0;
#pragma unroll
        for (int t = 0; t < TT; t++) {
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(bc[0][t][0]), "+d"(bc[0][t][1]) : "d"(pa), "d"(fh[t]));
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(bc[1][t][0]), "+d"(bc[1][t][1]) : "d"(pa), "d"(fm[t]));
        }
        lo = hi;
        if (lo >= ke) break;
      }
    }
    __syncwarp();
    if (c + PBG_STAGES < nchunks) issue(c + PBG_STAGES);
  }
  if (ib > ia) flush();
  // per-warp partial [2][NP][NP], both triangles
  double *out = gram_part + gw * 2 * NP * NP;
#pragma unroll
  for (int op = 0; op < 2; op++) {
    int u = 0;
#pragma unroll
    for (int ta = 0; ta < TT; ta++)
#pragma unroll
      for (int tb = ta; tb < TT; tb++, u++)
#pragma unroll
        for (int v = 0; v < 2; v++) {
          const int a = 8 * ta + grp, b = 8 * tb + 2 * tig + v;
          out[op * NP * NP + a * NP + b] = g[op][u][v];
          if (ta != tb) out[op * NP * NP + b * NP + a] = g[op][u][v];
        }
  }
}

// beta / gamma blocks: one warp per entry sums the per-warp Gram partials (lane-strided, then a fixed
// butterfly: deterministic)
__global__ void k_gram_fin(const double *__restrict__ part, int nparts, int N, int NP, int64_t n_H, int64_t D,
                           double *__restrict__ FA, double *__restrict__ FB) {
  const int lane = threadIdx.x & 31;
  const int64_t x = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (x >= 2 * N * N) return;
  const int m = (int)(x / (N * N)), a = (int)((x % (N * N)) / N), b = (int)(x % N);
  const double *src = part + m * NP * NP + a * NP + b;
  double s = 0.0;
  for (int w = lane; w < nparts; w += 32) s += __ldcg(src + (int64_t)w * 2 * NP * NP);
  s = warp_sum(s);
  if (lane == 0) (m ? FB : FA)[(n_H + a) * D + n_H + b] = s;
}

// one block per coarse node c: A row from the item partials (dense rows per warp, combined in warp
// order), and, with WITH_B, b_H / c_H entries (per-warp register sums over the warp's items, combined in
// warp order). Items are visited 4 at a time per warp so their metadata loads overlap. Fixed order.
constexpr int PF_BATCH = 4;
template <bool WITH_B>
__global__ void k_proj_final(const int32_t *__restrict__ CT_ptr, const int32_t *__restrict__ CT_val,
                             const int32_t *__restrict__ D_ptr, const int32_t *__restrict__ D,
                             const double *__restrict__ AH_part, const double *__restrict__ bH_part,
                             const double *__restrict__ cH_part, int64_t n_H, int N, int NP, double *__restrict__ FA,
                             double *__restrict__ FB, int64_t ldA, int64_t D2) {
  extern __shared__ double acc[];  // [W][n_H], then (WITH_B) [W][2N]
  const int W = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = blockIdx.x;
  for (int64_t x = threadIdx.x; x < W * n_H; x += blockDim.x) acc[x] = 0.0;
  __syncthreads();
  const int32_t e0 = __ldg(CT_ptr + c), e1 = __ldg(CT_ptr + c + 1);
  double *mine = acc + warp * n_H;
  constexpr int BQ = 4;                  // b/c columns per lane: 2N <= 128
  double bacc[BQ] = {0.0, 0.0, 0.0, 0.0};
  for (int32_t eb = e0 + warp; eb < e1; eb += PF_BATCH * W) {
    int32_t v[PF_BATCH], d0[PF_BATCH], dn[PF_BATCH];
#pragma unroll
    for (int k = 0; k < PF_BATCH; k++) {
      const int32_t e = eb + k * W;
      v[k] = e < e1 ? __ldg(CT_val + e) : -1;
    }
#pragma unroll
    for (int k = 0; k < PF_BATCH; k++) {
      d0[k] = 0;
      dn[k] = 0;
      if (v[k] >= 0) {
        d0[k] = __ldg(D_ptr + (v[k] >> 2));
        dn[k] = __ldg(D_ptr + (v[k] >> 2) + 1) - d0[k];
      }
    }
#pragma unroll
    for (int k = 0; k < PF_BATCH; k++) {
      if (v[k] < 0) continue;
      const double *src = AH_part + 4 * (int64_t)d0[k] + (v[k] & 3) * dn[k];
      for (int s = lane; s < dn[k]; s += 32) mine[__ldg(D + d0[k] + s)] += __ldcg(src + s);
      __syncwarp();
      if (WITH_B) {
#pragma unroll
        for (int q = 0; q < BQ; q++) {
          const int a = lane + 32 * q;
          if (a < 2 * N) bacc[q] += __ldcg((a < N ? bH_part : cH_part) + (int64_t)v[k] * NP + (a < N ? a : a - N));
        }
      }
    }
  }
  if (WITH_B) {
    double *bs = acc + W * n_H;
#pragma unroll
    for (int q = 0; q < BQ; q++)
      if (lane + 32 * q < 2 * N) bs[warp * 2 * N + lane + 32 * q] = bacc[q];
  }
  __syncthreads();
  for (int64_t d = threadIdx.x; d < n_H; d += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < W; w++) s += acc[w * n_H + d];
    FA[c * ldA + d] = s;
  }
  if (WITH_B) {
    const double *bs = acc + W * n_H;
    for (int a = threadIdx.x; a < 2 * N; a += blockDim.x) {
      const int col = a % N;
      double s = 0.0;
      for (int w = 0; w < W; w++) s += bs[w * 2 * N + a];
      double *F = a < N ? FA : FB;
      F[c * D2 + n_H + col] = s;
      F[(n_H + col) * D2 + c] = s;
    }
  }
}

// Gram partials: part[blk][m][a][b] = sum over the block's rows of U[i][a] * Y_m[i][b], m in {H, M}.
// Inputs with row stride ld. Outputs tiled 4x4 per thread; spare threads form row groups.
constexpr int GR_ROWS = 32;
__global__ void __launch_bounds__(256) k_gram(const double *__restrict__ U, const double *__restrict__ YH,
                                              const double *__restrict__ YM, int64_t n, int N, int ld,
                                              int64_t rows_per_blk, double *__restrict__ part) {
  extern __shared__ double sm[];
  const int NT = (N + 3) / 4, NQ = NT * 4;
  double *sU = sm, *sH = sm + GR_ROWS * NQ, *sM = sm + 2 * GR_ROWS * NQ;
  double *sRed = sm + 3 * GR_ROWS * NQ;
  const int ntiles = 2 * NT * NT;
  const bool many = ntiles > (int)blockDim.x;
  const int ngroups = many ? 1 : (int)blockDim.x / ntiles;
  const int my_group = many ? 0 : (int)threadIdx.x / ntiles;
  const int64_t r0 = blockIdx.x * rows_per_blk;
  const int64_t r1 = min(n, r0 + rows_per_blk);
  double acc[2][16];
#pragma unroll
  for (int z = 0; z < 2; z++)
#pragma unroll
    for (int k = 0; k < 16; k++) acc[z][k] = 0.0;
  for (int64_t rb = r0; rb < r1; rb += GR_ROWS) {
    const int nr = (int)min((int64_t)GR_ROWS, r1 - rb);
    __syncthreads();
    for (int x = threadIdx.x; x < GR_ROWS * NQ; x += blockDim.x) {
      const int rr = x / NQ, cc = x % NQ;
      const bool in = rr < nr && cc < N;
      const int64_t g = (rb + rr) * ld + cc;
      sU[x] = in ? U[g] : 0.0;
      sH[x] = in ? YH[g] : 0.0;
      sM[x] = in ? YM[g] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int z = 0; z < 2; z++) {
      const int tile = many ? (int)threadIdx.x + z * (int)blockDim.x : (z == 0 ? (int)threadIdx.x % ntiles : -1);
      if (tile < 0 || tile >= ntiles || my_group >= ngroups) continue;
      const int m = tile / (NT * NT), ta = (tile % (NT * NT)) / NT, tb = tile % NT;
      const double *sY = m ? sM : sH;
      for (int rr = my_group; rr < nr; rr += ngroups) {
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
  const int NN2 = 2 * N * N;
  for (int x = threadIdx.x; x < ngroups * NN2; x += blockDim.x) sRed[x] = 0.0;
  __syncthreads();
#pragma unroll
  for (int z = 0; z < 2; z++) {
    const int tile = many ? (int)threadIdx.x + z * (int)blockDim.x : (z == 0 ? (int)threadIdx.x % ntiles : -1);
    if (tile < 0 || tile >= ntiles || my_group >= ngroups) continue;
    const int m = tile / (NT * NT), ta = (tile % (NT * NT)) / NT, tb = tile % NT;
    for (int x = 0; x < 4; x++)
      for (int y = 0; y < 4; y++) {
        const int aa = ta * 4 + x, bb = tb * 4 + y;
        if (aa < N && bb < N) sRed[my_group * NN2 + m * N * N + aa * N + bb] = acc[z][x * 4 + y];
      }
  }
  __syncthreads();
  for (int x = threadIdx.x; x < NN2; x += blockDim.x) {
    double s = 0.0;
    for (int g = 0; g < ngroups; g++) s += sRed[g * NN2 + x];
    part[(int64_t)blockIdx.x * NN2 + x] = s;
  }
}

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

__global__ void k_copy_block(const double *__restrict__ src, int64_t n_H, double *__restrict__ dst, int64_t D) {
  int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= n_H * n_H) return;
  dst[(x / n_H) * D + x % n_H] = src[x];
}

__global__ void k_pad_proj(const double *__restrict__ src, int N, double *__restrict__ dst, int NP, int64_t n) {
  const int64_t gl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gl >= n * NP) return;
  const int64_t row = gl / NP;
  const int c = (int)(gl % NP);
  dst[gl] = c < N ? src[row * N + c] : 0.0;
}

int pow2_at_least(int N) {
  int np = 1;
  while (np < N) np <<= 1;
  return np;
}

// P rows as a dense 4-wide table (columns ascending, zero padded): the gather of a neighbour's P row
// is one 32-byte load instead of the row_ptr -> values chain
__global__ void k_pv4(const int32_t *__restrict__ Pptr, const double *__restrict__ Pval, int64_t n,
                      double *__restrict__ Pv4) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t a = Pptr[i], m = Pptr[i + 1] - a;
  for (int t = 0; t < 4; t++) Pv4[4 * i + t] = t < m ? Pval[a + t] : 0.0;
}

// item order: pos_of_row = inverse of perm, Pv4p[pos] = Pv4[perm[pos]]
__global__ void k_item_order(const int32_t *__restrict__ perm, const double *__restrict__ Pv4, int64_t n,
                             int32_t *__restrict__ pos_of_row, double *__restrict__ Pv4p) {
  const int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (pos >= n) return;
  const int32_t i = perm[pos];
  pos_of_row[i] = (int32_t)pos;
  for (int t = 0; t < 4; t++) Pv4p[4 * pos + t] = Pv4[4 * (int64_t)i + t];
}

ks_status launch_proj_ai(ks_ctx *ctx, const double *op_sell_vals) {   // Op in the natural sliced-ELL layout
  const int wcap = ctx->d_max;
  const size_t sm = sizeof(double) * (size_t)ITEM_ROWS * (wcap + 1 + 4);
  if (sm > 200 * 1024) return ks_fail(ctx, KS_E_ARG, "coarse window %d too large", ctx->d_max);
  KS_CUDA(ctx, cudaFuncSetAttribute(k_proj_ai, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per_sm = 0;
  KS_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_proj_ai, ITEM_ROWS, sm));
  int64_t grid = (int64_t)(per_sm > 0 ? per_sm : 1) * ctx->sm_count * 4;
  if (grid > ctx->n_items) grid = ctx->n_items;
  k_proj_ai<<<(unsigned)(grid > 0 ? grid : 1), ITEM_ROWS, sm, ctx->stream>>>(
      ctx->item_ptr, ctx->islice0, ctx->isell_ptr, ctx->isell_col, ctx->inat, op_sell_vals, ctx->islot, ctx->Pv4,
      ctx->Pv4p, ctx->item_D_ptr, ctx->n_items, wcap, ctx->AH_part);
  KS_LAUNCHED(ctx);
  return KS_OK;
}

ks_status launch_proj_a(ks_ctx *ctx, const double *op_sell_vals) {   // Op in the sliced-ELL layout
  const int wcap = ctx->d_max;
  const size_t sm = sizeof(double) * (size_t)ITEM_ROWS * (wcap + 1 + 4);
  if (sm > 200 * 1024) return ks_fail(ctx, KS_E_ARG, "coarse window %d too large", ctx->d_max);
  KS_CUDA(ctx, cudaFuncSetAttribute(k_proj_a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per_sm = 0;
  KS_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_proj_a, ITEM_ROWS, sm));
  int64_t grid = (int64_t)(per_sm > 0 ? per_sm : 1) * ctx->sm_count * 4;
  if (grid > ctx->n_items) grid = ctx->n_items;
  k_proj_a<<<(unsigned)(grid > 0 ? grid : 1), ITEM_ROWS, sm, ctx->stream>>>(
      ctx->row_ptr, ctx->col, ctx->sell_ptr, op_sell_vals, ctx->slotmap, ctx->Pv4, ctx->perm, ctx->item_ptr,
      ctx->item_D_ptr, ctx->n_items, wcap, ctx->AH_part);
  KS_LAUNCHED(ctx);
  return KS_OK;
}

// KS_PROJ_AI=0 selects k_proj_a (per-row entry loads) for the A_H pass (A/B knob; read per call, so
// tests can compare both in one process); default: k_proj_ai on the item-ordered copy
bool proj_ai_enabled() {
  const char *e = getenv("KS_PROJ_AI");
  return !(e && e[0] == '0');
}

// KS_PROJ_MMA=0 selects the FFMA item pass (A/B knob); default: tensor cores
bool proj_mma_enabled() {
  static const bool on = [] {
    const char *e = getenv("KS_PROJ_MMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

// tensor map of a row-major [n][np] f64 block for TMA row gathers: box = one full row (gather4 takes 4)
ks_status make_row_map(ks_ctx *ctx, const double *base, int64_t n, int np, CUtensorMap *map) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return ks_fail(ctx, KS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {(cuuint64_t)np, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)np * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)np, 1u}, estr[2] = {1u, 1u};
  if (encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return ks_fail(ctx, KS_E_CUDA, "cuTensorMapEncodeTiled failed (n = %lld, np = %d)", (long long)n, np);
  return KS_OK;
}

template <int NP>
ks_status launch_proj_yb(ks_ctx *ctx, int N, const double *u, double *FA, double *FB, int64_t D) {
  cudaStream_t s = ctx->stream;
  const int64_t n = ctx->n_free;
  constexpr bool MMA_NP = NP == 8 || NP == 16 || NP == 32;
  const bool mma = MMA_NP && proj_mma_enabled();
  const bool gather_u = mma && pbg_gather_u<NP>();
  k_proj_y<NP><<<ks_blocks(n * SL<NP>::LPR, 256), 256, 0, s>>>(ctx->sell_ptr, ctx->sell_col, ctx->sell_H,
                                                               ctx->sell_M, u, ctx->pos_of_row, ctx->proj_up,
                                                               ctx->Y_H, ctx->Y_M, n, !gather_u);
  KS_LAUNCHED(ctx);
  constexpr bool GRAM = NP <= 32;
  const int grid = 2 * ctx->sm_count;
  const int nparts = grid * PBG_WARPS;
  if (GRAM && (int64_t)nparts * 2 * NP * NP > ctx->gram_cap)
    return ks_fail(ctx, KS_E_WORKSPACE, "gram partials exceed the coarse plan");
  const size_t bsm = PBG_WARPS * PbgLayout<NP>::WARP_BYTES;
  if constexpr (NP == 8 || NP == 16 || NP == 32) {
    if (mma) {
      KS_CUDA(ctx, cudaFuncSetAttribute(k_proj_bg_mma<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
      CUtensorMap tmapU;
      memset(&tmapU, 0, sizeof(tmapU));
      if (gather_u && KS_PBG_G4) KS_TRY(make_row_map(ctx, u, n, NP, &tmapU));
      k_proj_bg_mma<NP><<<grid, PBG_WARPS * 32, bsm, s>>>(gather_u ? u : ctx->proj_up, ctx->perm, ctx->Y_H, ctx->Y_M,
                                                          ctx->Pv4p, ctx->item_ptr,
                                                          ctx->n_items, ctx->bH_part, ctx->cH_part, ctx->gram_part,
                                                          tmapU);
    } else {
      KS_CUDA(ctx, cudaFuncSetAttribute(k_proj_bg<NP, GRAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
      k_proj_bg<NP, GRAM><<<grid, PBG_WARPS * 32, bsm, s>>>(ctx->proj_up, ctx->Y_H, ctx->Y_M, ctx->Pv4p,
                                                             ctx->item_ptr, ctx->n_items, ctx->bH_part, ctx->cH_part,
                                                             ctx->gram_part);
    }
  } else {
    KS_CUDA(ctx, cudaFuncSetAttribute(k_proj_bg<NP, GRAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
    k_proj_bg<NP, GRAM><<<grid, PBG_WARPS * 32, bsm, s>>>(ctx->proj_up, ctx->Y_H, ctx->Y_M, ctx->Pv4p, ctx->item_ptr,
                                                           ctx->n_items, ctx->bH_part, ctx->cH_part, ctx->gram_part);
  }
  KS_LAUNCHED(ctx);
  if (GRAM) {
    k_gram_fin<<<ks_blocks(2 * N * N * 32, 128), 128, 0, s>>>(ctx->gram_part, nparts, N, NP, ctx->n_H, D, FA, FB);
    KS_LAUNCHED(ctx);
  } else {
    // NP = 64: register tiles of the fused pass would not fit; row-block Gram kernel (natural order)
    const int nblk = 2 * ctx->sm_count;
    const int64_t rows_per_blk = ((n + nblk - 1) / nblk + GR_ROWS - 1) / GR_ROWS * GR_ROWS;
    const int nb = (int)((n + rows_per_blk - 1) / rows_per_blk);
    if ((int64_t)nb * 2 * N * N > ctx->gram_cap)
      return ks_fail(ctx, KS_E_WORKSPACE, "gram partials exceed the coarse plan");
    const int NQ = (N + 3) / 4 * 4, NT = NQ / 4;
    const int ntiles = 2 * NT * NT;
    if (ntiles > 512) return ks_fail(ctx, KS_E_ARG, "N = %d too large for the Gram kernel", N);
    const int ngroups = ntiles > 256 ? 1 : 256 / ntiles;
    const size_t sm = sizeof(double) * (3 * GR_ROWS * NQ + (size_t)ngroups * 2 * N * N);
    KS_CUDA(ctx, cudaFuncSetAttribute(k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_gram<<<nb, 256, sm, s>>>(ctx->proj_up, ctx->Y_H, ctx->Y_M, n, N, NP, rows_per_blk, ctx->gram_part);
    KS_LAUNCHED(ctx);
    k_gram_final<<<ks_blocks(2 * N * N, 128), 128, 0, s>>>(ctx->gram_part, nb, N, ctx->n_H, D, FA, FB);
    KS_LAUNCHED(ctx);
  }
  return KS_OK;
}

template <bool WITH_B>
ks_status launch_final(ks_ctx *ctx, int N, int NP, double *FA, double *FB, int64_t ldA, int64_t D2) {
  int W = 8;
  size_t sm = sizeof(double) * W * (ctx->n_H + 2 * N);
  while (sm > 200 * 1024 && W > 1) { W >>= 1; sm = sizeof(double) * W * (ctx->n_H + 2 * N); }
  if (sm > 200 * 1024) return ks_fail(ctx, KS_E_ARG, "n_H = %lld too large for the dense-row reduction", (long long)ctx->n_H);
  KS_CUDA(ctx, cudaFuncSetAttribute(k_proj_final<WITH_B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_proj_final<WITH_B><<<(unsigned)ctx->n_H, 32 * W, sm, ctx->stream>>>(ctx->CT_ptr, ctx->CT_val, ctx->item_D_ptr,
                                                                        ctx->item_D, ctx->AH_part, ctx->bH_part,
                                                                        ctx->cH_part, ctx->n_H, N, NP, FA, FB, ldA, D2);
  KS_LAUNCHED(ctx);
  return KS_OK;
}

// gram partial slots of launch_proj_yb for any block width up to np_max (NP <= 32: one N x N pair per warp of
// the item pass; NP = 64: one per row block of k_gram)
int64_t proj_gram_cap(int sm_count, int np_max) {
  int64_t cap = 0;
  for (int np = 2; np <= np_max; np <<= 1) {
    const int64_t c = np <= 32 ? (int64_t)2 * sm_count * PBG_WARPS * 2 * np * np : (int64_t)2 * sm_count * 2 * np * np;
    cap = c > cap ? c : cap;
  }
  return cap;
}

}  // namespace

// dense P^T Op P [n_H][n_H] for an operator in the sliced-ELL layout (the A-part of the item pass)
ks_status ks_coarse_galerkin(ks_ctx *ctx, const double *op_sell_vals, double *out) {
  if (ctx->n_H <= 0) return ks_fail(ctx, KS_E_STATE, "no coarse space");
  ctx->ah_fresh = 0;   // AH_part is reused for this operator
  KS_TRY(launch_proj_a(ctx, op_sell_vals));
  return launch_final<false>(ctx, 0, 16, out, nullptr, ctx->n_H, 0);
}

void ks_free_coarse(ks_ctx *ctx) {
  ks_free_pcg2l(ctx);
  ctx->P_ptr = ctx->P_col = nullptr;
  ctx->P_val = ctx->Pv4 = ctx->Pv4p = nullptr;
  ctx->pos_of_row = nullptr;
  ctx->perm = ctx->item_ptr = ctx->item_S = ctx->item_D_ptr = ctx->item_D = ctx->CT_ptr = ctx->CT_val = nullptr;
  ctx->slotmap = nullptr;
  ctx->B_H = ctx->AH_part = nullptr;
  ctx->Y_H = ctx->Y_M = ctx->proj_u = ctx->proj_up = ctx->bH_part = ctx->cH_part = ctx->gram_part = nullptr;
  ctx->gram_cap = 0;
  ctx->n_H = 0;
  ctx->islice0 = ctx->isell_ptr = ctx->isell_col = nullptr;
  ctx->inat = nullptr;
  ctx->islot = nullptr;
  ctx->n_islices = ctx->isell_total = 0;
  ctx->ah_fresh = 0;
}

static int proj_np(int max_N) {
  const int np = ks_pow2_at_least(max_N);
  return np < 2 ? 2 : np;
}

// The coarse space of (st5)-(st7): P copied, fine rows grouped by parent set into items, coarse windows,
// slot map, coarse node -> item lists, cached B_H = P^T M P. The grouping runs in call scratch of the
// workspace; plan_only stops once the item count and window total are known and returns the coarse region
// size (ks_coarse_plan); otherwise the coarse layout is carved from the caller's coarse region.
ks_status ks_set_coarse_impl(ks_ctx *ctx, int64_t n_H, const int32_t *Pptr, const int32_t *Pcol, const double *Pval,
                             bool plan_only, size_t *coarse_bytes) {
  cudaStream_t s = ctx->stream;
  const int64_t nf = ctx->n_free;
  if (n_H >= 55000) return ks_fail(ctx, KS_E_ARG, "n_H = %lld >= 55000 not supported (parent-set key)", (long long)n_H);
  int32_t h_pn = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&h_pn, Pptr + nf, 4, cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  const int64_t pn = h_pn;
  if (pn < 0 || pn > 4 * nf) return ks_fail(ctx, KS_E_ARG, "P row_ptr[n_free] = %lld out of range", (long long)pn);
  size_t cub_cap = 0;
  if (ks_coarse_cub_bytes(nf, &cub_cap) != KS_OK) return ks_fail(ctx, KS_E_CUDA, "CUB temporary-size query failed");

  KsScratch scratch(ctx, KS_R_WORK);
  KsCoarseTemps t;
  KsCarver cv(ctx);
  ks_layout_coarse_temps_rows(cv, t, nf, pn, cub_cap);
  KS_TRY(cv.st);
  uint8_t *cub_tmp = t.cub;
  KS_CUDA(ctx, cudaMemcpyAsync(t.P_ptr, Pptr, 4 * (nf + 1), cudaMemcpyDeviceToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(t.P_col, Pcol, 4 * pn, cudaMemcpyDeviceToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(t.P_val, Pval, 8 * pn, cudaMemcpyDeviceToDevice, s));
  KS_CUDA(ctx, cudaMemsetAsync(t.bad, 0xff, 8, s));
  k_P_rows_keys<<<ks_blocks(nf, 256), 256, 0, s>>>(t.P_ptr, t.P_col, t.P_val, nf, n_H, pn, t.key, t.rows, t.bad);
  KS_LAUNCHED(ctx);
  unsigned long long h_bad = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&h_bad, t.bad, 8, cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  if (h_bad != ~0ull)
    return ks_fail(ctx, KS_E_ARG, "P row %llu invalid (more than 4 entries, repeated column, or column outside [0, n_H))", h_bad);
  k_pv4<<<ks_blocks(nf, 256), 256, 0, s>>>(t.P_ptr, t.P_val, nf, t.Pv4);
  KS_LAUNCHED(ctx);

  // ---- group rows by parent set (stable: ascending row inside a group), cut into items ----
  int end_bit = 1;
  {
    double bits = 4.0 * log2((double)n_H + 1.0);
    end_bit = (int)ceil(bits) + 1;
    if (end_bit > 64) end_bit = 64;
  }
  size_t tb = cub_cap;
  KS_CUDA(ctx, cub::DeviceRadixSort::SortPairs(cub_tmp, tb, t.key, t.key_sorted, t.rows, t.perm, (int)nf, 0, end_bit, s));
  ctx->launches++;
  k_item_order<<<ks_blocks(nf, 256), 256, 0, s>>>(t.perm, t.Pv4, nf, t.pos_of_row, t.Pv4p);
  KS_LAUNCHED(ctx);
  k_group_flags<<<ks_blocks(nf, 256), 256, 0, s>>>(t.key_sorted, nf, t.flag);
  KS_LAUNCHED(ctx);
  tb = cub_cap;
  KS_CUDA(ctx, cub::DeviceScan::InclusiveSum(cub_tmp, tb, t.flag, t.gincl, (int)nf, s));
  ctx->launches++;
  k_group_first<<<ks_blocks(nf, 256), 256, 0, s>>>(t.flag, t.gincl, nf, t.gfirst);
  KS_LAUNCHED(ctx);
  k_item_flags<<<ks_blocks(nf, 256), 256, 0, s>>>(t.gincl, t.gfirst, nf, t.iflag);
  KS_LAUNCHED(ctx);
  tb = cub_cap;
  KS_CUDA(ctx, cub::DeviceScan::InclusiveSum(cub_tmp, tb, t.iflag, t.iincl, (int)nf, s));
  ctx->launches++;
  int32_t h_items = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&h_items, t.iincl + nf - 1, 4, cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  const int64_t ni = h_items;
  ks_layout_coarse_temps_items(cv, t, ni, nf);
  KS_TRY(cv.st);
  int32_t h_nf = (int32_t)nf;
  KS_CUDA(ctx, cudaMemcpyAsync(t.item_ptr + ni, &h_nf, 4, cudaMemcpyHostToDevice, s));
  k_item_ptr<<<ks_blocks(nf, 256), 256, 0, s>>>(t.iflag, t.iincl, nf, t.item_ptr, t.item_of_pos);
  KS_LAUNCHED(ctx);
  k_item_S<<<ks_blocks(ni, 256), 256, 0, s>>>(t.item_ptr, t.perm, t.P_ptr, t.P_col, ni, t.item_S, t.ct_key, t.ct_val,
                                              (int32_t)n_H);
  KS_LAUNCHED(ctx);

  // ---- coarse windows D per item: sizes ----
  const size_t bsm = sizeof(unsigned) * (size_t)((n_H + 31) / 32);
  KS_CUDA(ctx, cudaFuncSetAttribute(k_item_D, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
  k_item_D<<<(unsigned)ni, 256, bsm, s>>>(t.item_ptr, t.perm, ctx->row_ptr, ctx->col, t.P_ptr, t.P_col, (int32_t)n_H,
                                          t.dcnt, nullptr, nullptr);
  KS_LAUNCHED(ctx);
  KS_CUDA(ctx, cudaMemsetAsync(t.dcnt + ni, 0, 4, s));
  tb = cub_cap;
  KS_CUDA(ctx, cub::DeviceScan::ExclusiveSum(cub_tmp, tb, t.dcnt, t.item_D_ptr, (int)(ni + 1), s));
  ctx->launches++;
  tb = cub_cap;
  KS_CUDA(ctx, cub::DeviceReduce::Max(cub_tmp, tb, t.dcnt, t.dmax, (int)ni, s));
  ctx->launches++;
  int32_t h_dtot = 0, h_dmax = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&h_dtot, t.item_D_ptr + ni, 4, cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaMemcpyAsync(&h_dmax, t.dmax, 4, cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  if (h_dmax > DMAX - 1)
    return ks_fail(ctx, KS_E_ARG, "an item touches %d coarse nodes (> %d): coarse mesh too fine for the fine mesh",
                   h_dmax, DMAX - 1);
  // ---- item slices of the item-ordered sliced-ELL copy (k_proj_ai): counts, widths, slot offsets ----
  KS_CUDA(ctx, cudaMemsetAsync(t.isw + ni, 0, 4, s));
  k_item_nslices<<<ks_blocks(ni, 256), 256, 0, s>>>(t.item_ptr, ni, t.isw);
  KS_LAUNCHED(ctx);
  tb = cub_cap;
  KS_CUDA(ctx, cub::DeviceScan::ExclusiveSum(cub_tmp, tb, t.isw, t.islice0, (int)(ni + 1), s));
  ctx->launches++;
  int32_t h_nis = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&h_nis, t.islice0 + ni, 4, cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  k_islice_width<<<ks_blocks(ni, 128), 128, 0, s>>>(t.item_ptr, t.islice0, t.perm, ctx->row_ptr, ni, t.isw);
  KS_LAUNCHED(ctx);
  KS_CUDA(ctx, cudaMemsetAsync(t.isw + h_nis, 0, 4, s));
  tb = cub_cap;
  KS_CUDA(ctx, cub::DeviceScan::ExclusiveSum(cub_tmp, tb, t.isw, t.isell_ptr, (int)(h_nis + 1), s));
  ctx->launches++;
  int32_t h_istot = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&h_istot, t.isell_ptr + h_nis, 4, cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  if (h_istot < 0) return ks_fail(ctx, KS_E_ARG, "item-ordered sliced-ELL copy exceeds 2^31 slots");

  KsCoarseSizes cs;
  cs.nis = h_nis;
  cs.istot = h_istot;
  cs.nf = nf;
  cs.nnz = ctx->nnz;
  cs.pn = pn;
  cs.ni = ni;
  cs.dtot = h_dtot;
  cs.nH = n_H;
  cs.np = proj_np(ctx->max_N);
  cs.gram = proj_gram_cap(ctx->sm_count, cs.np);
  if (plan_only) {
    KsSizer sz;
    ks_layout_coarse(sz, ctx, cs);
    *coarse_bytes = sz.bytes;
    return KS_OK;
  }

  // ---- the coarse region: carve the layout, move the grouping arrays in, build the rest ----
  ks_free_coarse(ctx);
  ctx->reg[KS_R_COARSE].off = 0;
  {
    KsRegion rg(ctx, KS_R_COARSE);
    KsCarver cc(ctx);
    ks_layout_coarse(cc, ctx, cs);
    KS_TRY(cc.st);
  }
  ctx->p_nnz = pn;
  ctx->n_items = ni;
  ctx->d_total = h_dtot;
  ctx->d_max = h_dmax > 0 ? h_dmax : 1;
  ctx->gram_cap = cs.gram;
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->P_ptr, t.P_ptr, 4 * (nf + 1), cudaMemcpyDeviceToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->P_col, t.P_col, 4 * pn, cudaMemcpyDeviceToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->P_val, t.P_val, 8 * pn, cudaMemcpyDeviceToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->perm, t.perm, 4 * nf, cudaMemcpyDeviceToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->Pv4, t.Pv4, 32 * nf, cudaMemcpyDeviceToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->pos_of_row, t.pos_of_row, 4 * nf, cudaMemcpyDeviceToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->Pv4p, t.Pv4p, 32 * nf, cudaMemcpyDeviceToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->item_ptr, t.item_ptr, 4 * (ni + 1), cudaMemcpyDeviceToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->item_S, t.item_S, 16 * ni, cudaMemcpyDeviceToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->item_D_ptr, t.item_D_ptr, 4 * (ni + 1), cudaMemcpyDeviceToDevice, s));
  k_item_D<<<(unsigned)ni, 256, bsm, s>>>(ctx->item_ptr, ctx->perm, ctx->row_ptr, ctx->col, ctx->P_ptr, ctx->P_col,
                                          (int32_t)n_H, nullptr, ctx->item_D_ptr, ctx->item_D);
  KS_LAUNCHED(ctx);
  k_slotmap<<<ks_blocks(nf, 128), 128, 0, s>>>(ctx->perm, t.item_of_pos, ctx->item_D_ptr, ctx->item_D, ctx->row_ptr,
                                               ctx->col, ctx->P_ptr, ctx->P_col, nf, ctx->slotmap);
  KS_LAUNCHED(ctx);

  // ---- the item-ordered sliced-ELL copy of the pattern (columns, window slots) for k_proj_ai ----
  ctx->n_islices = h_nis;
  ctx->isell_total = h_istot;
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->islice0, t.islice0, 4 * (ni + 1), cudaMemcpyDeviceToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->isell_ptr, t.isell_ptr, 4 * ((int64_t)h_nis + 1), cudaMemcpyDeviceToDevice, s));
  KS_CUDA(ctx, cudaMemsetAsync(ctx->isell_col, 0, 4 * (size_t)h_istot, s));   // pad rows gather row 0
  KS_CUDA(ctx, cudaMemsetAsync(ctx->islot, 0xff, 4 * (size_t)h_istot, s));
  k_isell_fill<<<ks_blocks(nf, 128), 128, 0, s>>>(ctx->perm, t.item_of_pos, ctx->item_ptr, ctx->islice0,
                                                  ctx->isell_ptr, ctx->row_ptr, ctx->col, ctx->sell_ptr, ctx->slotmap, nf, ctx->inat, ctx->isell_col,
                                                  ctx->islot);
  KS_LAUNCHED(ctx);

  // ---- coarse node -> items list (stable sort on the coarse id; pads sort last) ----
  int ct_bits = 1;
  while ((1ll << ct_bits) <= n_H) ct_bits++;
  tb = cub_cap;
  KS_CUDA(ctx, cub::DeviceRadixSort::SortPairs(cub_tmp, tb, t.ct_key, t.ct_key_sorted, t.ct_val, ctx->CT_val,
                                               (int)(4 * ni), 0, ct_bits, s));
  ctx->launches++;
  k_lower_bound_ptr<<<ks_blocks(n_H + 1, 256), 256, 0, s>>>(t.ct_key_sorted, 4 * ni, n_H, ctx->CT_ptr);
  KS_LAUNCHED(ctx);

  // ---- cached B_H = P^T M P (A-part of the item pass with M) ----
  ctx->n_H = n_H;
  ctx->ah_fresh = 0;
  KS_TRY(launch_proj_a(ctx, ctx->sell_M));
  KS_TRY(launch_final<false>(ctx, 0, 16, ctx->B_H, nullptr, n_H, 0));
  KS_CUDA(ctx, cudaStreamSynchronize(s));   // the call scratch is released at return
  return KS_OK;
}

ks_status ks_project_impl(ks_ctx *ctx, int N, const double *Ut, double *FA, double *FB) {
  cudaStream_t s = ctx->stream;
  const int64_t n = ctx->n_free, nH = ctx->n_H, D = nH + N;
  // NP >= 2: item-ordered rows are then multiples of 16 bytes (bulk-copy granularity)
  const int np = pow2_at_least(N) < 2 ? 2 : pow2_at_least(N);
  if (N > ctx->max_N) return ks_fail(ctx, KS_E_ARG, "N = %d exceeds max_N = %d", N, ctx->max_N);
  const double *u = Ut;
  if (np != N || ((uintptr_t)Ut & 31)) {
    k_pad_proj<<<ks_blocks(n * np, 256), 256, 0, s>>>(Ut, N, ctx->proj_u, np, n);
    KS_LAUNCHED(ctx);
    u = ctx->proj_u;
  }
  // K8a + K8c (+ Gram partials) for the orbital blocks
  switch (np) {
    case 2: KS_TRY(launch_proj_yb<2>(ctx, N, u, FA, FB, D)); break;
    case 4: KS_TRY(launch_proj_yb<4>(ctx, N, u, FA, FB, D)); break;
    case 8: KS_TRY(launch_proj_yb<8>(ctx, N, u, FA, FB, D)); break;
    case 16: KS_TRY(launch_proj_yb<16>(ctx, N, u, FA, FB, D)); break;
    case 32: KS_TRY(launch_proj_yb<32>(ctx, N, u, FA, FB, D)); break;
    case 64: KS_TRY(launch_proj_yb<64>(ctx, N, u, FA, FB, D)); break;
    default: return ks_fail(ctx, KS_E_ARG, "N = %d unsupported", N);
  }
  // K8b: A_H item partials (unshifted H, reading Q1)
  // (A_H depends on H only: repeated projections of one assembly, e.g. the outer iterations of
  // ks_augmented_solve at a fixed potential, reuse the item partials)
  const int ah_mode = proj_ai_enabled() && ctx->isell_col ? 1 : 2;
  if (ctx->ah_fresh != ah_mode) {
    if (ah_mode == 1) KS_TRY(launch_proj_ai(ctx, ctx->sell_H));
    else KS_TRY(launch_proj_a(ctx, ctx->sell_H));
    ctx->ah_fresh = ah_mode;
  }
  // K9: A_H, b_H, c_H
  KS_TRY(launch_final<true>(ctx, N, np, FA, FB, D, D));
  k_copy_block<<<ks_blocks(nH * nH, 256), 256, 0, s>>>(ctx->B_H, nH, FB, D);
  KS_LAUNCHED(ctx);
  return KS_OK;
}
