// ks_pcg.cu -- the N shifted boundary value problems of Algorithm 3 (Aux_Linear_Problem,
// PAPER.md:634-639):   A u~_i = (lambda_i + mu) M u_i,  A = H + mu M,  i = 1..N,
// solved as ONE batched Jacobi-preconditioned CG over the [n][NP] orbital block by a persistent
// cooperative kernel (one launch per solve, no host round trip). Per iteration, with per-column
// alpha_i, beta_i and masks (DESIGN.md §4.3 "block PCG"):
//   S  q = A p                      (multi-RHS CSR SpMM, fused p.q partials)          | grid barrier
//   U  r -= alpha q, z = r / d      (fused r.z and r.r partials)                       | grid barrier
//   P  x += alpha p, p = z + beta p (x update deferred to here so p is read once)      | grid barrier
// Memory-level parallelism (the kernel is HBM-latency bound without it, profiles/r01_ncu_summary.md):
//   * S stages each warp's rows of a tile (their slices of row_ptr / col / A values) into shared memory
//     with bulk (TMA) copies, cp.async.bulk + one mbarrier per (warp, stage), STAGES tiles ahead; each
//     warp runs its own pipeline (no block-wide sync per tile) and the next iteration's first tiles are
//     prefetched while the U and P phases stream. The gathers of p then only wait on shared memory, and
//     every lane issues 8 independent 16-byte gathers at a time (rows padded with the own row and a zero
//     weight, so the loads are unconditional).
//   * U and P stream UNR chunks per thread with all loads issued before any use.
//   * The Jacobi preconditioner is applied as a product with 1/diag(A) (precomputed by the assembly).
// Reductions are deterministic: each block owns a fixed, interleaved set of row tiles, reduces in a fixed
// order and writes one partial per column; after the barrier every block sums the partials in the same
// fixed order, so all blocks hold bitwise-identical alpha/beta and the result is reproducible run to run.
// Tiles are interleaved across blocks (tile t -> block t mod G) so that the gathered rows of p form a
// sweeping front that stays L2-resident. The U/P chunk of 2*PCG_THREADS doubles is the
// same row range as the S tile, so U and P touch only rows the block itself produced in S.
#include <cooperative_groups.h>

#include "ks_internal.cuh"
#include "ks_rowops.cuh"

namespace {

#ifndef KS_PCG_THREADS
#define KS_PCG_THREADS 512
#endif
#ifndef KS_PCG_MINB
#define KS_PCG_MINB 2
#endif
constexpr int PCG_THREADS = KS_PCG_THREADS;   // 512 threads x 2 blocks/SM: 64 registers, no spills
constexpr int PCG_WARPS = PCG_THREADS / 32;
constexpr int CHUNK = 2 * PCG_THREADS;   // doubles per streaming chunk (one double2 per thread)
constexpr int STAGES = 3;                // bulk-copy pipeline depth of the S phase
#ifndef KS_PCG_GATHER
#define KS_PCG_GATHER 8
#endif
#ifndef KS_PCG_UNR_U
#define KS_PCG_UNR_U 1
#endif
#ifndef KS_PCG_UNR_P
#define KS_PCG_UNR_P 1
#endif
constexpr int GATHER = KS_PCG_GATHER;    // independent gathers per lane in flight
constexpr int UNR_U = KS_PCG_UNR_U, UNR_P = KS_PCG_UNR_P;  // streaming chunks per thread per step (U, P)

struct PcgArgs {
  const int32_t *row_ptr, *col;
  const double *A, *M, *dinv;
  const double *lambda;
  double mu, tol;
  const double *U;      // [n][NP] input (possibly padded copy)
  double *X;            // [n][NP] solution
  double *r, *p, *q;    // [n][NP] workspace
  double *partials;     // [G][4*NP]
  unsigned *bar;
  unsigned *flags;
  int32_t *iters_out;   // [N] or null
  double *relres_out;   // [N] or null
  int32_t *block_iters_out;
  int64_t n;
  int N, ntiles, max_iter;
  int stage_nnz;        // capacity (elements) of one stage's col / value buffers (STAGED path)
  unsigned long long *trace;  // optional phase-end timestamps (%globaltimer, block 0), KS_PCG_TRACE=1
  int *trace_count;
  int trace_cap;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier for a cooperative launch (all blocks co-resident). Monotonic counter, reset to 0
// before the launch; `target` advances by gridDim.x per barrier in every block. The gpu-scope fences
// make the other blocks' writes visible (and invalidate this SM's L1 lines read before the barrier).
__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned &target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (ld_acquire(bar) < target) __nanosleep(20);
    __threadfence();
  }
  __syncthreads();
}

// out[j] = sum_{g < G} part[g*stride + j] for j < nv, fixed order, one warp per value.
__device__ __forceinline__ void reduce_partials(const double *part, int stride, int nv, double *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < nv; j += PCG_WARPS) {
    double s = 0.0;
    for (int g = lane; g < (int)gridDim.x; g += 32) s += __ldcg(part + (int64_t)g * stride + j);
    s = warp_sum(s);
    if (lane == 0) out[j] = s;
  }
  __syncthreads();
}

// ---- bulk (TMA) copies global -> shared, completion on an mbarrier ----
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Shared-memory layout of one warp's S-phase stage: row_ptr slice, col slice, value slice (16-byte aligned).
template <int NP>
struct Stage {
  static constexpr int TR = Lay<NP>::RPW;               // rows of a warp tile
  static constexpr int RP_CAP = (TR + 8 + 3) & ~3;     // row_ptr entries (aligned superset of TR + 1), x4
  __host__ __device__ static size_t bytes(int cap) {    // cap: col / value elements (multiple of 4)
    return sizeof(int32_t) * (RP_CAP + cap) + sizeof(double) * cap;
  }
};

// Issue the bulk copies of the warp tile starting at row r0 (rows [r0, min(r0 + TR, n)), empty if r0 >= n)
// into one stage's buffers (one thread).
__device__ __forceinline__ void issue_tile(const PcgArgs &a, int TR, int64_t r0, int32_t *srp, int32_t *scol,
                                           double *sval, uint64_t *bar) {
  r0 = min(r0, a.n);
  const int64_t r1 = min(r0 + TR, a.n);
  const int32_t kb = __ldg(a.row_ptr + r0), ke = __ldg(a.row_ptr + r1);
  const int64_t ra = r0 & ~3LL, re = (r1 + 1 + 3) & ~3LL;
  const int32_t ca = kb & ~3, ce = (ke + 3) & ~3;
  const int32_t va = kb & ~1, ve = (ke + 1) & ~1;
  const unsigned b_rp = (unsigned)(re - ra) * 4u, b_col = (unsigned)(ce - ca) * 4u, b_val = (unsigned)(ve - va) * 8u;
  mbar_expect_tx(bar, b_rp + b_col + b_val);
  bulk_g2s(srp, a.row_ptr + ra, b_rp, bar);
  if (b_col) bulk_g2s(scol, a.col + ca, b_col, bar);
  if (b_val) bulk_g2s(sval, a.A + va, b_val, bar);
}

// y = sum_k val[k] X[col[k]] for one row, col/val from shared memory (already offset to the row's first
// entry), GATHER unconditional gathers in flight (pad entries gather the own row with weight 0).
template <int NP>
__device__ __forceinline__ Vec<Lay<NP>::VEC> row_spmv_smem(const int32_t *scol, const double *sval, int len,
                                                           int64_t row, const double *X, int sub) {
  constexpr int VEC = Lay<NP>::VEC;
  Vec<VEC> acc;
  acc.zero();
  for (int k = 0; k < len; k += GATHER) {
    Vec<VEC> x[GATHER];
    double w[GATHER];
#pragma unroll
    for (int j = 0; j < GATHER; j++) {
      const bool in = k + j < len;
      const int64_t c = in ? (int64_t)scol[k + j] : row;
      w[j] = in ? sval[k + j] : 0.0;
      x[j] = Vec<VEC>::load(X + c * NP + sub * VEC);
    }
#pragma unroll
    for (int j = 0; j < GATHER; j++)
#pragma unroll
      for (int v = 0; v < VEC; v++) acc.v[v] = fma(w[j], x[j].v[v], acc.v[v]);
  }
  return acc;
}

template <int NP, bool STAGED>
__global__ void __launch_bounds__(PCG_THREADS, KS_PCG_MINB) k_block_pcg(PcgArgs a) {
  constexpr int VEC = Lay<NP>::VEC, LPR = Lay<NP>::LPR, RPW = Lay<NP>::RPW;
  constexpr int TILE = PCG_WARPS * RPW;              // rows per tile
  constexpr int STRIDE = 4 * NP;                     // partial slots per block
  static_assert(TILE * NP == CHUNK || NP == 1, "S tile and U/P chunk must cover the same rows");

  __shared__ double red[PCG_WARPS * 3 * NP];
  __shared__ double tot[3 * NP];
  __shared__ double s_alpha[NP], s_beta[NP], s_rho[NP], s_bnorm[NP], s_rr[NP];
  __shared__ int s_active[NP], s_conv[NP], s_iters[NP];
  __shared__ int s_any;
  __shared__ __align__(8) uint64_t s_bar[PCG_WARPS][STAGES];
  extern __shared__ __align__(16) unsigned char dyn[];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = lane / LPR, sub = lane % LPR;
  const int G = gridDim.x;
  const int64_t n = a.n;
  const int64_t nel = n * NP;
  const int nchunks = (int)((nel + CHUNK - 1) / CHUNK);
  unsigned target = 0;
  double *part_init = a.partials;                      // region 0: 3 dots (init) / 2 dots (U)
  double *part_s = a.partials + (int64_t)G * STRIDE;   // region 1: 1 dot (S)

  // ---- S-phase stage buffers and the per-warp tile pipelines ----
  const int cap = a.stage_nnz;
  const size_t stage_bytes = Stage<NP>::bytes(cap);
  unsigned char *wdyn = dyn + (size_t)warp * STAGES * stage_bytes;
  auto st_rp = [&](int s) { return reinterpret_cast<int32_t *>(wdyn + s * stage_bytes); };
  auto st_col = [&](int s) { return reinterpret_cast<int32_t *>(wdyn + s * stage_bytes) + Stage<NP>::RP_CAP; };
  auto st_val = [&](int s) {
    return reinterpret_cast<double *>(wdyn + s * stage_bytes + sizeof(int32_t) * (Stage<NP>::RP_CAP + cap));
  };
  auto wtile_row = [&](int ti) { return (int64_t)(blockIdx.x + ti * G) * TILE + warp * RPW; };
  const int my_tiles = a.ntiles > blockIdx.x ? (a.ntiles - blockIdx.x + G - 1) / G : 0;
  unsigned seq = 0;  // tiles consumed so far (all phases); stage = seq % STAGES, parity = (seq / STAGES) & 1
  if (STAGED) {
    if (lane == 0) {
      for (int s = 0; s < STAGES; s++) mbar_init(&s_bar[warp][s], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      // the S phases consume this block's tiles periodically: consumption number q is tile index
      // q mod my_tiles; stage q mod STAGES always holds consumption q (prefetched STAGES ahead)
      if (my_tiles > 0)
        for (int q = 0; q < STAGES; q++)
          issue_tile(a, RPW, wtile_row(q % my_tiles), st_rp(q), st_col(q), st_val(q), &s_bar[warp][q]);
    }
    __syncwarp();
  }
  unsigned long long *trace = (a.trace && blockIdx.x == 0 && threadIdx.x == 0) ? a.trace : nullptr;
  int ntr = 0;
  auto stamp = [&]() {
    if (trace && ntr < a.trace_cap) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[ntr++] = t;
    }
  };
  stamp();

  // ---------------- init: b = (lambda+mu) M u, r = b - A u, x = u, z = r/d, p = z ----------------
  {
    double acc[3][VEC];
#pragma unroll
    for (int d = 0; d < 3; d++)
#pragma unroll
      for (int v = 0; v < VEC; v++) acc[d][v] = 0.0;
    double sh[VEC];
#pragma unroll
    for (int v = 0; v < VEC; v++) {
      int c = sub * VEC + v;
      sh[v] = (c < a.N ? __ldg(a.lambda + c) : 0.0) + a.mu;
    }
    for (int tile = blockIdx.x; tile < a.ntiles; tile += G) {
      int64_t row = (int64_t)tile * TILE + warp * RPW + slot;
      if (row < n) {
        Vec<VEC> au, mu_;
        row_spmv2<NP>(a.col, a.A, a.M, __ldg(a.row_ptr + row), __ldg(a.row_ptr + row + 1), a.U, sub, au, mu_);
        const int64_t off = row * NP + sub * VEC;
        Vec<VEC> u = Vec<VEC>::load(a.U + off);
        const double dinv = __ldg(a.dinv + row);
        Vec<VEC> r, z;
#pragma unroll
        for (int v = 0; v < VEC; v++) {
          double b = sh[v] * mu_.v[v];
          r.v[v] = b - au.v[v];
          z.v[v] = r.v[v] * dinv;
          acc[0][v] += b * b;
          acc[1][v] += r.v[v] * z.v[v];
          acc[2][v] += r.v[v] * r.v[v];
        }
        r.store(a.r + off);
        z.store(a.p + off);
        u.store(a.X + off);
      }
    }
    block_reduce_cols<NP, 3>(acc, red, tot);
    for (int i = threadIdx.x; i < 3 * NP; i += blockDim.x) part_init[(int64_t)blockIdx.x * STRIDE + i] = tot[i];
    grid_barrier(a.bar, target);
    stamp();
    reduce_partials(part_init, STRIDE, 3 * NP, tot);
    if (threadIdx.x < NP) {
      const int c = threadIdx.x;
      double bn = sqrt(tot[c]), rz = tot[NP + c], rr = tot[2 * NP + c];
      s_bnorm[c] = bn;
      s_rho[c] = rz;
      s_rr[c] = rr;
      s_iters[c] = 0;
      s_conv[c] = 0;
      bool real = c < a.N;
      bool finite = isfinite(bn) && isfinite(rr) && isfinite(rz);
      if (real && !finite && blockIdx.x == 0) atomicOr(a.flags, KSF_NONFINITE);
      s_active[c] = real && finite && !(sqrt(rr) <= a.tol * bn);
    }
    __syncthreads();
  }

  // ---------------- iterations ----------------
  int it = 0;
  // streaming layout: element e = chunk * CHUNK + 2 * threadIdx.x; columns c0, c0 + 1 (NP >= 2)
  const int c0 = (2 * threadIdx.x) % NP;
  const int c1 = NP == 1 ? 0 : c0 + 1;
  for (;;) {
    if (threadIdx.x == 0) {
      int any = 0;
      for (int c = 0; c < NP; c++) any |= s_active[c];
      s_any = any;
    }
    __syncthreads();
    if (!s_any) break;
    if (it >= a.max_iter) {
      if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(a.flags, KSF_NOT_CONVERGED);
      break;
    }

    // ---- S: q = A p, p.q ----
    {
      double acc[1][VEC];
#pragma unroll
      for (int v = 0; v < VEC; v++) acc[0][v] = 0.0;
      for (int i = 0; i < my_tiles; i++) {
        const int tile = blockIdx.x + i * G;
        const int64_t r0 = (int64_t)tile * TILE;
        const int64_t row = r0 + warp * RPW + slot;
        Vec<VEC> q;
        if (STAGED) {
          const int s = seq % STAGES;
          mbar_wait(&s_bar[warp][s], (seq / STAGES) & 1u);
          const int32_t *srp = st_rp(s);
          const int64_t w0 = r0 + warp * RPW;   // first row of the warp tile
          const int64_t ra = w0 & ~3LL;
          const int32_t kb = srp[w0 - ra];       // first nnz of the warp tile; slices start at kb & ~3 / kb & ~1
          if (row < n) {
            const int32_t k0 = srp[row - ra], k1 = srp[row - ra + 1];
            q = row_spmv_smem<NP>(st_col(s) + (k0 - (kb & ~3)), st_val(s) + (k0 - (kb & ~1)), k1 - k0, row, a.p,
                                  sub);
          }
        } else if (row < n) {
          q = row_spmv<NP>(a.col, a.A, __ldg(a.row_ptr + row), __ldg(a.row_ptr + row + 1), a.p, sub);
        }
        if (row < n) {
          const int64_t off = row * NP + sub * VEC;
          Vec<VEC> pv = Vec<VEC>::load(a.p + off);
#pragma unroll
          for (int v = 0; v < VEC; v++) acc[0][v] += pv.v[v] * q.v[v];
          q.store(a.q + off);
        }
        if (STAGED) {
          __syncwarp();  // the warp is done with this stage's buffers
          if (lane == 0) {
            // refill the stage with consumption seq + STAGES (wrapping into the next iteration's S phase:
            // the matrix never changes, so the prefetch overlaps the U and P phases)
            const int s = seq % STAGES;
            const int nxt = (int)((seq + STAGES) % (unsigned)my_tiles);
            issue_tile(a, RPW, wtile_row(nxt), st_rp(s), st_col(s), st_val(s), &s_bar[warp][s]);
          }
          seq++;
        }
      }
      block_reduce_cols<NP, 1>(acc, red, tot);
      for (int i = threadIdx.x; i < NP; i += blockDim.x) part_s[(int64_t)blockIdx.x * STRIDE + i] = tot[i];
      grid_barrier(a.bar, target);
      stamp();
      reduce_partials(part_s, STRIDE, NP, tot);
      if (threadIdx.x < NP) {
        const int c = threadIdx.x;
        double al = 0.0;
        if (s_active[c]) {
          double pq = tot[c];
          if (!(pq > 0.0)) {
            if (blockIdx.x == 0) atomicOr(a.flags, isfinite(pq) ? KSF_NOT_SPD : KSF_NONFINITE);
            s_active[c] = 0;
          } else {
            al = s_rho[c] / pq;
          }
        }
        s_alpha[c] = al;
      }
      __syncthreads();
    }

    // ---- U: r -= alpha q; r.z, r.r (z = r / d) ----
    {
      const double al0 = s_alpha[c0], al1 = s_alpha[c1];
      double acc[2][VEC];
#pragma unroll
      for (int d = 0; d < 2; d++)
#pragma unroll
        for (int v = 0; v < VEC; v++) acc[d][v] = 0.0;
      for (int ch = blockIdx.x; ch < nchunks; ch += UNR_U * G) {
        double2 r[UNR_U], q[UNR_U];
        double d0[UNR_U], d1[UNR_U];
#pragma unroll
        for (int u = 0; u < UNR_U; u++) {
          const int64_t e = (int64_t)(ch + u * G) * CHUNK + 2 * threadIdx.x;
          if (ch + u * G < nchunks && e < nel) {
            r[u] = *reinterpret_cast<const double2 *>(a.r + e);
            q[u] = *reinterpret_cast<const double2 *>(a.q + e);
            if (NP == 1) { d0[u] = __ldg(a.dinv + e); d1[u] = __ldg(a.dinv + e + 1); }
            else { d0[u] = d1[u] = __ldg(a.dinv + e / NP); }
          }
        }
#pragma unroll
        for (int u = 0; u < UNR_U; u++) {
          const int64_t e = (int64_t)(ch + u * G) * CHUNK + 2 * threadIdx.x;
          if (ch + u * G < nchunks && e < nel) {
            r[u].x -= al0 * q[u].x;
            r[u].y -= al1 * q[u].y;
            acc[0][0] += r[u].x * (r[u].x * d0[u]);
            acc[0][VEC - 1] += r[u].y * (r[u].y * d1[u]);
            acc[1][0] += r[u].x * r[u].x;
            acc[1][VEC - 1] += r[u].y * r[u].y;
            *reinterpret_cast<double2 *>(a.r + e) = r[u];
          }
        }
      }
      block_reduce_cols<NP, 2>(acc, red, tot);
      for (int i = threadIdx.x; i < 2 * NP; i += blockDim.x) part_init[(int64_t)blockIdx.x * STRIDE + i] = tot[i];
      grid_barrier(a.bar, target);
      stamp();
      reduce_partials(part_init, STRIDE, 2 * NP, tot);
      if (threadIdx.x < NP) {
        const int c = threadIdx.x;
        double be = 0.0;
        int conv = 0;
        if (s_active[c]) {
          double rz = tot[c], rr = tot[NP + c];
          s_iters[c] += 1;
          if (!isfinite(rz) || !isfinite(rr)) {
            if (blockIdx.x == 0) atomicOr(a.flags, KSF_NONFINITE);
            conv = 1;
          } else {
            be = rz / s_rho[c];
            s_rho[c] = rz;
            s_rr[c] = rr;
            conv = sqrt(rr) <= a.tol * s_bnorm[c];
          }
          if (conv) be = 0.0;
        }
        s_beta[c] = be;
        s_conv[c] = conv;
      }
      __syncthreads();
    }

    // ---- P: x += alpha p; p = r/d + beta p ----
    {
      const double al0 = s_alpha[c0], al1 = s_alpha[c1];
      const double be0 = s_beta[c0], be1 = s_beta[c1];
      for (int ch = blockIdx.x; ch < nchunks; ch += UNR_P * G) {
        double2 r[UNR_P], p[UNR_P], x[UNR_P];
        double d0[UNR_P], d1[UNR_P];
#pragma unroll
        for (int u = 0; u < UNR_P; u++) {
          const int64_t e = (int64_t)(ch + u * G) * CHUNK + 2 * threadIdx.x;
          if (ch + u * G < nchunks && e < nel) {
            r[u] = *reinterpret_cast<const double2 *>(a.r + e);
            p[u] = *reinterpret_cast<const double2 *>(a.p + e);
            x[u] = *reinterpret_cast<const double2 *>(a.X + e);
            if (NP == 1) { d0[u] = __ldg(a.dinv + e); d1[u] = __ldg(a.dinv + e + 1); }
            else { d0[u] = d1[u] = __ldg(a.dinv + e / NP); }
          }
        }
#pragma unroll
        for (int u = 0; u < UNR_P; u++) {
          const int64_t e = (int64_t)(ch + u * G) * CHUNK + 2 * threadIdx.x;
          if (ch + u * G < nchunks && e < nel) {
            x[u].x += al0 * p[u].x;
            x[u].y += al1 * p[u].y;
            p[u].x = r[u].x * d0[u] + be0 * p[u].x;
            p[u].y = r[u].y * d1[u] + be1 * p[u].y;
            *reinterpret_cast<double2 *>(a.X + e) = x[u];
            *reinterpret_cast<double2 *>(a.p + e) = p[u];
          }
        }
      }
      if (threadIdx.x < NP && s_conv[threadIdx.x]) s_active[threadIdx.x] = 0;
      it++;
      grid_barrier(a.bar, target);
      stamp();
    }
  }

  if (blockIdx.x == 0) {
    for (int c = threadIdx.x; c < a.N; c += blockDim.x) {
      if (a.iters_out) a.iters_out[c] = s_iters[c];
      if (a.relres_out) a.relres_out[c] = s_bnorm[c] > 0.0 ? sqrt(s_rr[c]) / s_bnorm[c] : sqrt(s_rr[c]);
    }
    if (threadIdx.x == 0) {
      *a.block_iters_out = it;
      if (a.trace_count) *a.trace_count = ntr;
    }
  }
  if (STAGED) {
    // drain the prefetches issued for an S phase that did not run, so no bulk copy outlives the block
    const int pending = my_tiles > 0 ? STAGES : 0;
    for (int i = 0; i < pending; i++) {
      const unsigned q = seq + i;
      mbar_wait(&s_bar[warp][q % STAGES], (q / STAGES) & 1u);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// standalone multi-RHS SpMM (parity / benchmarking) and helpers
// ---------------------------------------------------------------------------------------------
template <int NP>
__global__ void __launch_bounds__(256) k_spmm(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                              const double *__restrict__ val, const double *__restrict__ X,
                                              double *__restrict__ Y, int64_t n) {
  constexpr int VEC = Lay<NP>::VEC, LPR = Lay<NP>::LPR;
  const int64_t gl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t row = gl / LPR;
  const int sub = (int)(gl % LPR);
  if (row >= n) return;
  Vec<VEC> y = row_spmv<NP>(col, val, __ldg(row_ptr + row), __ldg(row_ptr + row + 1), X, sub);
  y.store(Y + row * NP + sub * VEC);
}

__global__ void k_spmm_generic(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                               const double *__restrict__ val, const double *__restrict__ X, double *__restrict__ Y,
                               int64_t n, int N) {
  const int64_t gl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gl >= n * N) return;
  const int64_t row = gl / N;
  const int c = (int)(gl % N);
  double s = 0.0;
  for (int32_t k = row_ptr[row]; k < row_ptr[row + 1]; k++) s = fma(val[k], X[(int64_t)col[k] * N + c], s);
  Y[gl] = s;
}

// [n][N] <-> [n][NP] with zero padding
__global__ void k_pad(const double *__restrict__ src, int N, double *__restrict__ dst, int NP, int64_t n) {
  const int64_t gl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gl >= n * NP) return;
  const int64_t row = gl / NP;
  const int c = (int)(gl % NP);
  dst[gl] = c < N ? src[row * N + c] : 0.0;
}

__global__ void k_unpad(const double *__restrict__ src, int NP, double *__restrict__ dst, int N, int64_t n) {
  const int64_t gl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gl >= n * N) return;
  dst[gl] = src[(gl / N) * NP + gl % N];
}

// true residual partials: per block sums of b^2 and (b - A ut)^2 per column (generic layout)
__global__ void k_true_residual(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                const double *__restrict__ A, const double *__restrict__ M,
                                const double *__restrict__ lambda, double mu, const double *__restrict__ U,
                                const double *__restrict__ Ut, int64_t n, int N, double *__restrict__ part) {
  // one thread per (row, column); block handles a contiguous range; partial per block per column
  extern __shared__ double sh[];  // [2][blockDim]
  const int64_t gl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double bb = 0.0, rr = 0.0;
  int c = -1;
  if (gl < n * N) {
    const int64_t row = gl / N;
    c = (int)(gl % N);
    double mu_ = 0.0, au = 0.0;
    for (int32_t k = row_ptr[row]; k < row_ptr[row + 1]; k++) {
      mu_ = fma(M[k], U[(int64_t)col[k] * N + c], mu_);
      au = fma(A[k], Ut[(int64_t)col[k] * N + c], au);
    }
    double b = (lambda[c] + mu) * mu_;
    bb = b * b;
    rr = (b - au) * (b - au);
  }
  sh[threadIdx.x] = bb;
  sh[blockDim.x + threadIdx.x] = rr;
  __syncthreads();
  // column-wise sums in fixed order by thread 0..N-1
  for (int cc = threadIdx.x; cc < N; cc += blockDim.x) {
    double sb = 0.0, sr = 0.0;
    const int64_t first = blockIdx.x * (int64_t)blockDim.x;
    for (int t = 0; t < (int)blockDim.x; t++) {
      const int64_t g = first + t;
      if (g < n * N && (int)(g % N) == cc) { sb += sh[t]; sr += sh[blockDim.x + t]; }
    }
    part[(int64_t)blockIdx.x * 2 * N + cc] = sb;
    part[(int64_t)blockIdx.x * 2 * N + N + cc] = sr;
  }
}

__global__ void k_true_residual_final(const double *__restrict__ part, int nblk, int N, double *__restrict__ out) {
  for (int c = threadIdx.x; c < N; c += blockDim.x) {
    double sb = 0.0, sr = 0.0;
    for (int b = 0; b < nblk; b++) { sb += part[(int64_t)b * 2 * N + c]; sr += part[(int64_t)b * 2 * N + N + c]; }
    out[c] = sb > 0.0 ? sqrt(sr) / sqrt(sb) : sqrt(sr);
  }
}

int pad_np(int N) {
  int np = 1;
  while (np < N) np <<= 1;
  return np;
}

// largest nnz count of a TR-row tile (sizes the S-phase stage buffers)
__global__ void k_tile_max_nnz(const int32_t *__restrict__ row_ptr, int64_t n, int TR, int ntiles,
                               int *__restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  int v = 0;
  if (t < ntiles) {
    const int64_t r0 = (int64_t)t * TR, r1 = min(r0 + TR, n);
    v = row_ptr[r1] - row_ptr[r0];
  }
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0 && v > 0) atomicMax(out, v);
}

static ks_status tile_max_nnz(ks_ctx *ctx, int TR, int ntiles, int *out) {
  for (auto &e : ctx->tile_nnz_cache)
    if (e.first == TR) { *out = e.second; return KS_OK; }
  int *d = nullptr;
  KS_TRY(ks_alloc_t(ctx, &d, 1, "tile nnz"));
  k_tile_max_nnz<<<ks_blocks(ntiles, 256), 256, 0, ctx->stream>>>(ctx->row_ptr, ctx->n_free, TR, ntiles, d);
  KS_LAUNCHED(ctx);
  int h = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  cudaFree(d);
  ctx->bytes -= sizeof(int);
  ctx->tile_nnz_cache.push_back({TR, h});
  *out = h;
  return KS_OK;
}

template <int NP, bool STAGED>
ks_status launch_pcg_t(ks_ctx *ctx, PcgArgs &a, size_t dyn) {
  auto kern = k_block_pcg<NP, STAGED>;
  KS_CUDA(ctx, cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  int per_sm = 0;
  KS_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PCG_THREADS, dyn));
  if (per_sm < 1) return ks_fail(ctx, KS_E_CUDA, "k_block_pcg<%d,%d> cannot be resident", NP, (int)STAGED);
  int G = per_sm * ctx->sm_count;
  if (G > a.ntiles) G = a.ntiles;
  if ((int64_t)G * 4 * NP * 2 > ctx->partial_cap) {
    if (ctx->partials) { cudaFree(ctx->partials); ctx->partials = nullptr; }
    ctx->partial_cap = (int64_t)G * 4 * NP * 2;
    KS_TRY(ks_alloc_t(ctx, &ctx->partials, ctx->partial_cap, "pcg partials"));
  }
  a.partials = ctx->partials;
  KS_CUDA(ctx, cudaMemsetAsync(ctx->barrier, 0, sizeof(unsigned), ctx->stream));
  void *args[] = {&a};
  KS_CUDA(ctx, cudaLaunchCooperativeKernel((const void *)kern, dim3(G), dim3(PCG_THREADS), args, dyn, ctx->stream));
  ctx->launches++;
  return KS_OK;
}

// STAGED (bulk-copied matrix tiles) when STAGES stage buffers fit next to a second block on the SM;
// KS_PCG_STAGED=0 in the environment forces the direct path (A/B measurements).
constexpr size_t STAGE_SMEM_MAX = 96 * 1024;

template <int NP>
ks_status launch_pcg(ks_ctx *ctx, PcgArgs &a) {
  constexpr int TILE = PCG_WARPS * Lay<NP>::RPW;
  a.ntiles = (int)((a.n + TILE - 1) / TILE);
  int mx = 0;
  KS_TRY(tile_max_nnz(ctx, Lay<NP>::RPW, (int)((a.n + Lay<NP>::RPW - 1) / Lay<NP>::RPW), &mx));
  const int cap = ((mx + 8) + 3) & ~3;   // + alignment slack of both slices
  a.stage_nnz = cap;
  const size_t dyn = (size_t)PCG_WARPS * STAGES * Stage<NP>::bytes(cap);
  const char *env = getenv("KS_PCG_STAGED");
  const bool want = !(env && env[0] == '0');
  if (want && dyn <= STAGE_SMEM_MAX) return launch_pcg_t<NP, true>(ctx, a, dyn);
  a.stage_nnz = 0;
  return launch_pcg_t<NP, false>(ctx, a, 0);
}

template <int NP>
void launch_spmm(ks_ctx *ctx, const double *val, const double *X, double *Y) {
  const int64_t threads = ctx->n_free * Lay<NP>::LPR;
  k_spmm<NP><<<ks_blocks(threads, 256), 256, 0, ctx->stream>>>(ctx->row_ptr, ctx->col, val, X, Y, ctx->n_free);
}

}  // namespace

static bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

ks_status ks_spmm_impl(ks_ctx *ctx, const double *val, int N, const double *X, double *Y) {
  const int np = pad_np(N);
  if (np == N && aligned16(X) && aligned16(Y)) {
    switch (N) {
      case 1: launch_spmm<1>(ctx, val, X, Y); break;
      case 2: launch_spmm<2>(ctx, val, X, Y); break;
      case 4: launch_spmm<4>(ctx, val, X, Y); break;
      case 8: launch_spmm<8>(ctx, val, X, Y); break;
      case 16: launch_spmm<16>(ctx, val, X, Y); break;
      case 32: launch_spmm<32>(ctx, val, X, Y); break;
      case 64: launch_spmm<64>(ctx, val, X, Y); break;
    }
  } else {
    k_spmm_generic<<<ks_blocks(ctx->n_free * N, 256), 256, 0, ctx->stream>>>(ctx->row_ptr, ctx->col, val, X, Y,
                                                                             ctx->n_free, N);
  }
  KS_LAUNCHED(ctx);
  return KS_OK;
}

static ks_status ensure_solver_ws(ks_ctx *ctx, int np) {
  if (ctx->ws_np >= np && ctx->ws_rows == ctx->n_free) return KS_OK;
  for (double **b : {&ctx->r, &ctx->p, &ctx->q, &ctx->xpad, &ctx->upad})
    if (*b) { cudaFree(*b); *b = nullptr; }
  const int64_t cnt = ctx->n_free * (int64_t)np + 2;  // +2: NP=1 streaming reads pairs
  KS_TRY(ks_alloc_t(ctx, &ctx->r, cnt, "pcg r"));
  KS_TRY(ks_alloc_t(ctx, &ctx->p, cnt, "pcg p"));
  KS_TRY(ks_alloc_t(ctx, &ctx->q, cnt, "pcg q"));
  KS_TRY(ks_alloc_t(ctx, &ctx->xpad, cnt, "pcg x pad"));
  KS_TRY(ks_alloc_t(ctx, &ctx->upad, cnt, "pcg u pad"));
  ctx->ws_np = np;
  ctx->ws_rows = ctx->n_free;
  return KS_OK;
}

ks_status ks_solve_impl(ks_ctx *ctx, int N, const double *lambda, const double *U, double *Ut, double tol,
                        int max_iter, int32_t *iters, double *relres) {
  const int np = pad_np(N);
  KS_TRY(ensure_solver_ws(ctx, np));
  const int64_t n = ctx->n_free;
  // NP = 1 streams element pairs: pad to an even element count via the internal buffers
  const bool direct = (np == N) && aligned16(U) && aligned16(Ut) && !(np == 1 && (n & 1));
  const double *u = U;
  double *x = Ut;
  if (!direct) {
    KS_CUDA(ctx, cudaMemsetAsync(ctx->upad, 0, sizeof(double) * (n * np + 2), ctx->stream));
    KS_CUDA(ctx, cudaMemsetAsync(ctx->xpad, 0, sizeof(double) * (n * np + 2), ctx->stream));
    k_pad<<<ks_blocks(n * np, 256), 256, 0, ctx->stream>>>(U, N, ctx->upad, np, n);
    KS_LAUNCHED(ctx);
    u = ctx->upad;
    x = ctx->xpad;
  }
  if (np == 1) {
    // keep the odd tail element finite for the pairwise streaming phases
    KS_CUDA(ctx, cudaMemsetAsync(ctx->r + n, 0, sizeof(double) * 2, ctx->stream));
    KS_CUDA(ctx, cudaMemsetAsync(ctx->q + n, 0, sizeof(double) * 2, ctx->stream));
    KS_CUDA(ctx, cudaMemsetAsync(ctx->p + n, 0, sizeof(double) * 2, ctx->stream));
  }
  PcgArgs a;
  a.row_ptr = ctx->row_ptr;
  a.col = ctx->col;
  a.A = ctx->A;
  a.M = ctx->M;
  a.dinv = ctx->dinv;
  a.lambda = lambda;
  a.mu = ctx->mu;
  a.tol = tol;
  a.U = u;
  a.X = x;
  a.r = ctx->r;
  a.p = ctx->p;
  a.q = ctx->q;
  a.bar = ctx->barrier;
  a.flags = ctx->d_flags;
  a.iters_out = iters;
  a.relres_out = relres;
  a.block_iters_out = ctx->d_block_iters;
  a.trace = nullptr;
  a.trace_count = nullptr;
  a.trace_cap = 0;
  const char *tr = getenv("KS_PCG_TRACE");
  if (tr && tr[0] == '1') {
    if (!ctx->trace) {
      KS_TRY(ks_alloc_t(ctx, &ctx->trace, KS_TRACE_CAP, "pcg trace"));
      KS_TRY(ks_alloc_t(ctx, &ctx->trace_count, 1, "pcg trace count"));
    }
    a.trace = ctx->trace;
    a.trace_count = ctx->trace_count;
    a.trace_cap = KS_TRACE_CAP;
  }
  a.n = n;
  a.N = N;
  a.max_iter = max_iter;
  switch (np) {
    case 1: KS_TRY(launch_pcg<1>(ctx, a)); break;
    case 2: KS_TRY(launch_pcg<2>(ctx, a)); break;
    case 4: KS_TRY(launch_pcg<4>(ctx, a)); break;
    case 8: KS_TRY(launch_pcg<8>(ctx, a)); break;
    case 16: KS_TRY(launch_pcg<16>(ctx, a)); break;
    case 32: KS_TRY(launch_pcg<32>(ctx, a)); break;
    case 64: KS_TRY(launch_pcg<64>(ctx, a)); break;
    default: return ks_fail(ctx, KS_E_ARG, "N=%d unsupported", N);
  }
  if (!direct) {
    k_unpad<<<ks_blocks(n * N, 256), 256, 0, ctx->stream>>>(ctx->xpad, np, Ut, N, n);
    KS_LAUNCHED(ctx);
  }
  return KS_OK;
}

ks_status ks_true_residual_impl(ks_ctx *ctx, int N, const double *lambda, const double *U, const double *Ut,
                                double *relres) {
  const int64_t total = ctx->n_free * N;
  const int T = 256;
  const int nblk = ks_blocks(total, T);
  double *part = nullptr;
  KS_CUDA(ctx, cudaMallocAsync((void **)&part, sizeof(double) * 2 * N * (size_t)nblk, ctx->stream));
  k_true_residual<<<nblk, T, 2 * T * sizeof(double), ctx->stream>>>(ctx->row_ptr, ctx->col, ctx->A, ctx->M, lambda,
                                                                     ctx->mu, U, Ut, ctx->n_free, N, part);
  KS_LAUNCHED(ctx);
  k_true_residual_final<<<1, 64, 0, ctx->stream>>>(part, nblk, N, relres);
  KS_LAUNCHED(ctx);
  KS_CUDA(ctx, cudaFreeAsync(part, ctx->stream));
  return KS_OK;
}
