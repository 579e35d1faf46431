// ks_pcg.cu -- the N shifted boundary value problems of Algorithm 3 (Aux_Linear_Problem,
// PAPER.md:634-639):   A u~_i = (lambda_i + mu) M u_i,  A = H + mu M,  i = 1..N,
// solved as ONE batched Jacobi-preconditioned CG over the [n][NP] orbital block by a persistent
// cooperative kernel (one launch per solve, no host round trip). Per iteration, with per-column
// alpha_i, beta_i and masks (DESIGN.md §4.3 "block PCG"):
//   S  q = A p                      (multi-RHS SpMM on the sliced-ELL copy, fused p.q partials)  | barrier
//   U  r -= alpha q, z = r / d      (fused r.z and r.r partials)                                  | barrier
//   P  x += alpha p, p = z + beta p (x update deferred to here so p is read once)                 | barrier
// Throughput design (profiles/r01_ncu_summary.md):
//   * S reads the operator in SELL-8 (ks_sell.cu): per 4 nonzeros of a row one 16-byte col load and one
//     32-byte value load, shared by the lanes of the row; the orbital rows are gathered with 32-byte
//     loads (LDG.256), 4 lanes per 128-byte row at N = 16. The CSR form spent as many L1 wavefronts on
//     broadcast col/val loads as on the gathers.
//   * U and P stream 32-byte vectors (one row segment of 4 orbitals per thread).
//   * The Jacobi preconditioner is a product with 1/diag(A) (precomputed by the assembly).
// Reductions are deterministic: each block owns a fixed, interleaved set of row tiles, reduces in a fixed
// order and writes one partial per column; after the barrier every block sums the partials in the same
// fixed order, so all blocks hold bitwise-identical alpha/beta and the result is reproducible run to run.
// Tiles are interleaved across blocks (tile t -> block t mod G) so that the gathered rows of p form a
// sweeping front that stays L2-resident. The U/P chunk (VEC doubles per thread) is the
// same row range as the S tile, so U and P touch only rows the block itself produced in S.
#include "ks_internal.cuh"
#include "ks_rowops.cuh"
#include "ks_sell.cuh"
#include "ks_grid.cuh"

namespace {

#ifndef KS_PCG_THREADS
#define KS_PCG_THREADS 512
#endif
#ifndef KS_PCG_MINB
#define KS_PCG_MINB 1
#endif
constexpr int PCG_THREADS = KS_PCG_THREADS;   // 512 threads x 1 block/SM: 128 registers, no spills
constexpr int PCG_WARPS = PCG_THREADS / 32;

// Block-level column sums: acc[d][v] per lane (column (VEC*lane+v) % NP) -> out[d*NP + c], fixed order
// (butterfly over the lanes of a column within the warp, then warps 0..W-1 in order).
template <int NP, int ND, int VEC = SL<NP, PCG_THREADS>::VEC, int LPR = SL<NP, PCG_THREADS>::LPR>
__device__ __forceinline__ void block_cols(double (&acc)[ND][VEC], double *red, double *out) {
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
    for (int w = 0; w < PCG_WARPS; w++) s += red[w * ND * NP + i];
    out[i] = s;
  }
  __syncthreads();
}

struct PcgArgs {
  const int32_t *sell_ptr, *sell_col;
  const double *A, *M, *dinv;   // A, M: sliced-ELL values
  const double *lambda;
  double mu, tol;
  const double *U;      // [n][NP] input (possibly padded copy): u_i, and x0 (warm start)
  const double *B;      // [n][NP] given right-hand side (Poisson mode), or null: b = (lambda + mu) M u
  double *X;            // [n][NP] solution
  double *r, *p, *q;    // [n][NP] workspace
  double *partials;     // [G][4*NP]
  unsigned *bar;
  unsigned *flags;
  int32_t *iters_out;   // [N] or null
  double *relres_out;   // [N] or null
  int32_t *block_iters_out;
  unsigned long long *trace;  // optional phase-end timestamps (%globaltimer, block 0), KS_PCG_TRACE=1
  int *trace_count;
  int trace_cap;
  int64_t n;
  int N, ntiles, max_iter;
  // staged S phase (ks_stage.cu)
  const int32_t *meta;        // [n_groups] KS_META_BYTES records
  const uint16_t *slcol;      // [sell_total] local column of every slot
  const uint16_t *dlc;        // [n] local index of the row itself
  int64_t ngroups;
  int stage_cap;              // staged rows per stage buffer
};

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

// ---- staged S phase: the p rows a group of GRP rows references are copied (bulk, TMA) into shared memory
constexpr int PSTAGES = 3;
constexpr int META_SLOT = 128;   // bytes reserved for the group record in a stage (KS_META_BYTES <= 128)

template <int NP>
struct SP {   // staged layout: 2 orbitals per lane (NP >= 4)
  static constexpr int VEC = 2, LPR = NP >= 4 ? NP / 2 : 2, RPW = 32 / LPR, GRP = PCG_WARPS * RPW;
  static_assert(GRP * NP == 1024, "group size of ks_stage_build");
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// thread 0: copy the staged rows of consumption k (group g) into stage st, plus the record of group k + PSTAGES
// (the producer reads records only from shared memory after the prologue). rec: the record of group g.
template <int NP>
__device__ __forceinline__ void issue_group(const PcgArgs &a, const int32_t *rec, int64_t g, int64_t g_next,
                                            unsigned char *stage, uint64_t *bar, int *staged_flag) {
  const int nruns = rec[0];
  *staged_flag = nruns > 0;
  unsigned bytes = nruns > 0 ? (unsigned)rec[1] * NP * 8u : 0u;
  if (g_next >= 0) bytes += KS_META_BYTES;
  if (bytes == 0) {
    mbar_arrive(bar);
    return;
  }
  mbar_expect_tx(bar, bytes);
  double *buf = reinterpret_cast<double *>(stage + META_SLOT);
  int off = 0;
  for (int r = 0; r < nruns; r++) {
    const int start = rec[4 + 2 * r], len = rec[5 + 2 * r];
    bulk_g2s(buf + (int64_t)off * NP, a.p + (int64_t)start * NP, (unsigned)len * NP * 8u, bar);
    off += len;
  }
  if (g_next >= 0) bulk_g2s(stage, a.meta + g_next * (KS_META_BYTES / 4), KS_META_BYTES, bar);
}

// q = A p for this CTA's groups, p.q partials in acc (staged layout); returns the consumptions done
template <int NP>
__device__ __forceinline__ void s_phase_staged(const PcgArgs &a, unsigned char *dyn, uint64_t *pbar, int *s_staged,
                                               unsigned &pseq, double (&acc)[1][2]) {
  constexpr int LPR = SP<NP>::LPR, RPW = SP<NP>::RPW, GRP = SP<NP>::GRP;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = lane / LPR, sub = lane % LPR;
  const int G = gridDim.x;
  const int64_t n = a.n;
  const size_t stage_bytes = META_SLOT + (size_t)a.stage_cap * NP * 8;
  const int64_t my = a.ngroups > blockIdx.x ? (a.ngroups - blockIdx.x + G - 1) / G : 0;
  auto stage_of = [&](unsigned q) { return dyn + (size_t)(q % PSTAGES) * stage_bytes; };
  if (threadIdx.x == 0) {
    // p was written by other CTAs before the grid barrier: order the bulk (async-proxy) reads after it
    asm volatile("fence.proxy.async.global;" ::: "memory");
    for (int k = 0; k < PSTAGES && k < my; k++) {
      const int64_t g = blockIdx.x + (int64_t)k * G;
      const int64_t gn = k + PSTAGES < my ? g + (int64_t)PSTAGES * G : -1;
      const int32_t *rec = a.meta + g * (KS_META_BYTES / 4);
      int32_t r[KS_META_BYTES / 4];
      for (int x = 0; x < KS_META_BYTES / 4; x++) r[x] = __ldg(rec + x);
      issue_group<NP>(a, r, g, gn, stage_of(pseq + k), &pbar[(pseq + k) % PSTAGES], &s_staged[(pseq + k) % PSTAGES]);
    }
  }
  for (int64_t k = 0; k < my; k++) {
    const unsigned q = pseq + (unsigned)k;
    const int st = q % PSTAGES;
    mbar_wait(&pbar[st], (q / PSTAGES) & 1u);
    unsigned char *stage = stage_of(q);
    const double *buf = reinterpret_cast<const double *>(stage + META_SLOT);
    const int64_t g = blockIdx.x + k * G;
    const int64_t row = g * GRP + warp * RPW + slot;
    const bool staged = s_staged[st];
    if (row < n) {
      const int64_t sl = row / KS_SELL_C;
      const int32_t b = __ldg(a.sell_ptr + sl), e = __ldg(a.sell_ptr + sl + 1);
      const int groups = (e - b) / (4 * KS_SELL_C);
      const int64_t base = b + (row % KS_SELL_C) * 4;
      double q0 = 0.0, q1 = 0.0, p0, p1;
      if (staged) {
        for (int gg = 0; gg < groups; gg++) {
          const int64_t o = base + (int64_t)gg * (4 * KS_SELL_C);
          const ushort4 lc = __ldg(reinterpret_cast<const ushort4 *>(a.slcol + o));
          double w0, w1, w2, w3;
          ldnc_v4(a.A + o, w0, w1, w2, w3);
          const double2 x0 = *reinterpret_cast<const double2 *>(buf + (int64_t)lc.x * NP + 2 * sub);
          const double2 x1 = *reinterpret_cast<const double2 *>(buf + (int64_t)lc.y * NP + 2 * sub);
          const double2 x2 = *reinterpret_cast<const double2 *>(buf + (int64_t)lc.z * NP + 2 * sub);
          const double2 x3 = *reinterpret_cast<const double2 *>(buf + (int64_t)lc.w * NP + 2 * sub);
          q0 = fma(w0, x0.x, q0); q1 = fma(w0, x0.y, q1);
          q0 = fma(w1, x1.x, q0); q1 = fma(w1, x1.y, q1);
          q0 = fma(w2, x2.x, q0); q1 = fma(w2, x2.y, q1);
          q0 = fma(w3, x3.x, q0); q1 = fma(w3, x3.y, q1);
        }
        const double2 pv = *reinterpret_cast<const double2 *>(buf + (int64_t)__ldg(a.dlc + row) * NP + 2 * sub);
        p0 = pv.x; p1 = pv.y;
      } else {   // group too irregular to stage: gathers from global memory
        for (int gg = 0; gg < groups; gg++) {
          const int64_t o = base + (int64_t)gg * (4 * KS_SELL_C);
          const int4 c = __ldg(reinterpret_cast<const int4 *>(a.sell_col + o));
          double w0, w1, w2, w3;
          ldnc_v4(a.A + o, w0, w1, w2, w3);
          const double2 x0 = *reinterpret_cast<const double2 *>(a.p + (int64_t)c.x * NP + 2 * sub);
          const double2 x1 = *reinterpret_cast<const double2 *>(a.p + (int64_t)c.y * NP + 2 * sub);
          const double2 x2 = *reinterpret_cast<const double2 *>(a.p + (int64_t)c.z * NP + 2 * sub);
          const double2 x3 = *reinterpret_cast<const double2 *>(a.p + (int64_t)c.w * NP + 2 * sub);
          q0 = fma(w0, x0.x, q0); q1 = fma(w0, x0.y, q1);
          q0 = fma(w1, x1.x, q0); q1 = fma(w1, x1.y, q1);
          q0 = fma(w2, x2.x, q0); q1 = fma(w2, x2.y, q1);
          q0 = fma(w3, x3.x, q0); q1 = fma(w3, x3.y, q1);
        }
        const double2 pv = *reinterpret_cast<const double2 *>(a.p + row * NP + 2 * sub);
        p0 = pv.x; p1 = pv.y;
      }
      acc[0][0] += p0 * q0;
      acc[0][1] += p1 * q1;
      *reinterpret_cast<double2 *>(a.q + row * NP + 2 * sub) = make_double2(q0, q1);
    }
    __syncthreads();   // every warp is done with stage st
    if (threadIdx.x == 0 && k + PSTAGES < my) {
      int32_t r[KS_META_BYTES / 4];
      const int32_t *rec = reinterpret_cast<const int32_t *>(stage);   // arrived with consumption k
      for (int x = 0; x < KS_META_BYTES / 4; x++) r[x] = rec[x];
      const int64_t g2 = g + (int64_t)PSTAGES * G;
      const int64_t gn = k + 2 * PSTAGES < my ? g2 + (int64_t)PSTAGES * G : -1;
      issue_group<NP>(a, r, g2, gn, stage, &pbar[st], &s_staged[st]);
    }
  }
  pseq += (unsigned)my;
}

template <int NP, bool STAGEP>
__global__ void __launch_bounds__(PCG_THREADS, KS_PCG_MINB) k_block_pcg(PcgArgs a) {
  constexpr int VEC = SL<NP, PCG_THREADS>::VEC, LPR = SL<NP, PCG_THREADS>::LPR, RPW = SL<NP, PCG_THREADS>::RPW, TILE = SL<NP, PCG_THREADS>::TILE;
  constexpr int CHUNK = SL<NP, PCG_THREADS>::CHUNK;
  constexpr int STRIDE = 4 * NP;                     // partial slots per block

  __shared__ double red[PCG_WARPS * 3 * NP];
  __shared__ double tot[3 * NP];
  __shared__ double s_alpha[NP], s_beta[NP], s_rho[NP], s_bnorm[NP], s_rr[NP];
  __shared__ int s_active[NP], s_conv[NP], s_iters[NP];
  __shared__ int s_any;
  __shared__ __align__(8) uint64_t s_pbar[PSTAGES];
  __shared__ int s_staged[PSTAGES];
  extern __shared__ __align__(128) unsigned char dyn[];
  unsigned pseq = 0;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = lane / LPR, sub = lane % LPR;
  const int G = gridDim.x;
  const int64_t n = a.n;
  unsigned target = 0;
  double *part_init = a.partials;                      // region 0: 3 dots (init) / 2 dots (U)
  double *part_s = a.partials + (int64_t)G * STRIDE;   // region 1: 1 dot (S)
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
  if constexpr (STAGEP) {
    if (threadIdx.x == 0) {
      for (int st = 0; st < PSTAGES; st++) mbar_init(&s_pbar[st], 1);
      mbar_fence_init();
    }
    __syncthreads();
  }

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
      sh[v] = (c < a.N && a.lambda ? __ldg(a.lambda + c) : 0.0) + a.mu;
    }
    for (int tile = blockIdx.x; tile < a.ntiles; tile += G) {
      int64_t row = (int64_t)tile * TILE + warp * RPW + slot;
      if (row < n) {
        DV<VEC> au, mu_;
        const int64_t off = row * NP + sub * VEC;
        if (a.B) {   // Poisson mode: the right-hand side is given (grid-uniform branch)
          sell_row<NP, 1>(a.sell_ptr, a.sell_col, a.A, nullptr, row, a.U, sub, au, mu_);
          mu_ = DV<VEC>::ld(a.B + off);
#pragma unroll
          for (int v = 0; v < VEC; v++) sh[v] = 1.0;
        } else {
          sell_row<NP, 2>(a.sell_ptr, a.sell_col, a.A, a.M, row, a.U, sub, au, mu_);
        }
        const double dinv = __ldg(a.dinv + row);
        DV<VEC> r, z;
#pragma unroll
        for (int v = 0; v < VEC; v++) {
          double b = sh[v] * mu_.v[v];
          r.v[v] = b - au.v[v];
          z.v[v] = r.v[v] * dinv;
          acc[0][v] += b * b;
          acc[1][v] += r.v[v] * z.v[v];
          acc[2][v] += r.v[v] * r.v[v];
        }
        r.st(a.r + off);
        z.st(a.p + off);   // x0 = u is not copied: the first P phase reads it from U (saves a vector write)
      }
    }
    block_cols<NP, 3>(acc, red, tot);
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
  const int64_t nel = n * NP;
  const int nchunks = (int)((nel + CHUNK - 1) / CHUNK);
  const int cb = (VEC * threadIdx.x) % NP;           // first column of this thread's stream vector
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
    if constexpr (STAGEP) {
      double acc[1][2] = {{0.0, 0.0}};
      s_phase_staged<NP>(a, dyn, s_pbar, s_staged, pseq, acc);
      block_cols<NP, 1, 2, NP / 2>(acc, red, tot);
    } else {
      double acc[1][VEC];
#pragma unroll
      for (int v = 0; v < VEC; v++) acc[0][v] = 0.0;
      for (int tile = blockIdx.x; tile < a.ntiles; tile += G) {
        const int64_t row = (int64_t)tile * TILE + warp * RPW + slot;
        if (row < n) {
          DV<VEC> q, unused;
          sell_row<NP, 1>(a.sell_ptr, a.sell_col, a.A, nullptr, row, a.p, sub, q, unused);
          const int64_t off = row * NP + sub * VEC;
          const DV<VEC> pv = DV<VEC>::ld(a.p + off);
#pragma unroll
          for (int v = 0; v < VEC; v++) acc[0][v] += pv.v[v] * q.v[v];
          q.st(a.q + off);
        }
      }
      block_cols<NP, 1>(acc, red, tot);
    }
    {
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
      double al[VEC];
#pragma unroll
      for (int v = 0; v < VEC; v++) al[v] = s_alpha[cb + v];
      double acc[2][VEC];
#pragma unroll
      for (int d = 0; d < 2; d++)
#pragma unroll
        for (int v = 0; v < VEC; v++) acc[d][v] = 0.0;
      for (int ch = blockIdx.x; ch < nchunks; ch += G) {
        const int64_t e = (int64_t)ch * CHUNK + VEC * threadIdx.x;
        if (e < nel) {
          DV<VEC> r = DV<VEC>::ld(a.r + e);
          const DV<VEC> q = DV<VEC>::ld(a.q + e);
          const double di = __ldg(a.dinv + e / NP);
#pragma unroll
          for (int v = 0; v < VEC; v++) {
            r.v[v] -= al[v] * q.v[v];
            acc[0][v] += r.v[v] * (r.v[v] * di);
            acc[1][v] += r.v[v] * r.v[v];
          }
          r.st(a.r + e);
        }
      }
      block_cols<NP, 2>(acc, red, tot);
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
      double al[VEC], be[VEC];
#pragma unroll
      for (int v = 0; v < VEC; v++) {
        al[v] = s_alpha[cb + v];
        be[v] = s_beta[cb + v];
      }
      for (int ch = blockIdx.x; ch < nchunks; ch += G) {
        const int64_t e = (int64_t)ch * CHUNK + VEC * threadIdx.x;
        if (e < nel) {
          const DV<VEC> r = DV<VEC>::ld(a.r + e);
          DV<VEC> p = DV<VEC>::ld(a.p + e);
          DV<VEC> x = DV<VEC>::ld((it == 0 ? a.U : a.X) + e);   // x0 = u
          const double di = __ldg(a.dinv + e / NP);
#pragma unroll
          for (int v = 0; v < VEC; v++) {
            x.v[v] += al[v] * p.v[v];
            p.v[v] = r.v[v] * di + be[v] * p.v[v];
          }
          x.st(a.X + e);
          p.st(a.p + e);
        }
      }
      if (threadIdx.x < NP && s_conv[threadIdx.x]) s_active[threadIdx.x] = 0;
      it++;
      grid_barrier(a.bar, target);
      stamp();
    }
  }

  if (it == 0) {   // no P phase ran (converged at the initial check, or stopped before it): x = x0 = u
    for (int ch = blockIdx.x; ch < nchunks; ch += G) {
      const int64_t e = (int64_t)ch * CHUNK + VEC * threadIdx.x;
      if (e < nel) DV<VEC>::ld(a.U + e).st(a.X + e);
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
}

// ---------------------------------------------------------------------------------------------
// standalone multi-RHS SpMM on the sliced-ELL copy (A, M): parity helper and benchmark of phase S
// ---------------------------------------------------------------------------------------------
template <int NP>
__global__ void __launch_bounds__(256) k_spmm_sell(const int32_t *__restrict__ sell_ptr,
                                                   const int32_t *__restrict__ sell_col,
                                                   const double *__restrict__ val, const double *__restrict__ X,
                                                   double *__restrict__ Y, int64_t n) {
  constexpr int VEC = SL<NP, PCG_THREADS>::VEC, LPR = SL<NP, PCG_THREADS>::LPR;
  const int64_t gl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t row = gl / LPR;
  const int sub = (int)(gl % LPR);
  if (row >= n) return;
  DV<VEC> y, unused;
  sell_row<NP, 1>(sell_ptr, sell_col, val, nullptr, row, X, sub, y, unused);
  y.st(Y + row * NP + sub * VEC);
}

// CSR multi-RHS SpMM for the operators without a sliced-ELL copy (K, M_V, H)
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

template <int NP, bool STAGEP>
ks_status launch_pcg_t(ks_ctx *ctx, PcgArgs &a, size_t dyn) {
  auto kern = k_block_pcg<NP, STAGEP>;
  if (dyn > 0) KS_CUDA(ctx, cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  int per_sm = 0;
  KS_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PCG_THREADS, dyn));
  if (per_sm < 1) return ks_fail(ctx, KS_E_CUDA, "k_block_pcg<%d,%d> cannot be resident", NP, (int)STAGEP);
  int G = per_sm * ctx->sm_count;
  if (G > a.ntiles) G = a.ntiles;
  if ((int64_t)G * 4 * NP * 2 > ctx->partial_cap) {
    ks_free_t(ctx, ctx->partials);
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

// Staged S phase (opt-in, KS_PCG_STAGE=1): for NP >= 4 when the group tables fit three stages of shared
// memory. Measured slower on the lexicographically numbered meshes (C4: S 471 us vs 296 us gathering,
// r01ad): a 64-row group references ~7 runs of ~66 rows, so each p row is copied into ~7 stage buffers and
// the L2 -> shared traffic (7.2x the vector per S phase) saturates L2, while L1 gathers hit ~50 %. It needs
// 3-D-local row groups to pay off.
constexpr size_t PSTAGE_SMEM_MAX = 200 * 1024;

template <int NP>
ks_status launch_pcg(ks_ctx *ctx, PcgArgs &a) {
  a.ntiles = (int)((a.n + SL<NP, PCG_THREADS>::TILE - 1) / SL<NP, PCG_THREADS>::TILE);
  a.meta = nullptr;
  a.slcol = nullptr;
  a.dlc = nullptr;
  a.ngroups = 0;
  a.stage_cap = 0;
  const char *env = getenv("KS_PCG_STAGE");
  const bool want = NP >= 4 && env && env[0] == '1';
  if constexpr (NP >= 4 && PCG_THREADS == 512) {   // the staged layout assumes 512 threads (SP<NP>)
    if (want) {
      const int max_rows = (int)((PSTAGE_SMEM_MAX / PSTAGES - META_SLOT) / (NP * 8));
      KS_TRY(ks_stage_build(ctx, NP, max_rows));
      if (ctx->stage_staged > 0) {
        a.meta = ctx->stage_meta;
        a.slcol = ctx->stage_slcol;
        a.dlc = ctx->stage_dlc;
        a.ngroups = ctx->stage_groups;
        a.stage_cap = ctx->stage_cap;
        const size_t dyn = (size_t)PSTAGES * (META_SLOT + (size_t)ctx->stage_cap * NP * 8);
        return launch_pcg_t<NP, true>(ctx, a, dyn);
      }
    }
  }
  return launch_pcg_t<NP, false>(ctx, a, 0);
}

template <int NP>
void launch_spmm(ks_ctx *ctx, const double *sell_val, const double *csr_val, const double *X, double *Y) {
  if (sell_val) {
    const int64_t threads = ctx->n_free * SL<NP, PCG_THREADS>::LPR;
    k_spmm_sell<NP><<<ks_blocks(threads, 256), 256, 0, ctx->stream>>>(ctx->sell_ptr, ctx->sell_col, sell_val, X, Y,
                                                                      ctx->n_free);
  } else {
    const int64_t threads = ctx->n_free * Lay<NP>::LPR;
    k_spmm<NP><<<ks_blocks(threads, 256), 256, 0, ctx->stream>>>(ctx->row_ptr, ctx->col, csr_val, X, Y,
                                                                 ctx->n_free);
  }
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

}  // namespace

static bool aligned32(const void *p) { return ((uintptr_t)p & 31u) == 0; }

ks_status ks_spmm_impl(ks_ctx *ctx, ks_op op, const double *val, int N, const double *X, double *Y) {
  const int np = pad_np(N);
  const double *sv = op == KS_OP_A ? ctx->sell_A : op == KS_OP_M ? ctx->sell_M : nullptr;
  if (np == N && aligned32(X) && aligned32(Y)) {
    switch (N) {
      case 1: launch_spmm<1>(ctx, sv, val, X, Y); break;
      case 2: launch_spmm<2>(ctx, sv, val, X, Y); break;
      case 4: launch_spmm<4>(ctx, sv, val, X, Y); break;
      case 8: launch_spmm<8>(ctx, sv, val, X, Y); break;
      case 16: launch_spmm<16>(ctx, sv, val, X, Y); break;
      case 32: launch_spmm<32>(ctx, sv, val, X, Y); break;
      case 64: launch_spmm<64>(ctx, sv, val, X, Y); break;
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
  for (double **b : {&ctx->r, &ctx->p, &ctx->q, &ctx->xpad, &ctx->upad, &ctx->bpad})
    ks_free_t(ctx, *b);
  const int64_t cnt = ctx->n_free * (int64_t)np;
  KS_TRY(ks_alloc_t(ctx, &ctx->r, cnt, "pcg r"));
  KS_TRY(ks_alloc_t(ctx, &ctx->p, cnt, "pcg p"));
  KS_TRY(ks_alloc_t(ctx, &ctx->q, cnt, "pcg q"));
  KS_TRY(ks_alloc_t(ctx, &ctx->xpad, cnt, "pcg x pad"));
  KS_TRY(ks_alloc_t(ctx, &ctx->upad, cnt, "pcg u pad"));
  KS_TRY(ks_alloc_t(ctx, &ctx->bpad, cnt, "pcg b pad"));
  ctx->ws_np = np;
  ctx->ws_rows = ctx->n_free;
  return KS_OK;
}

ks_status ks_solve_impl(ks_ctx *ctx, int N, const double *lambda, const double *U, double *Ut, double tol,
                        int max_iter, int32_t *iters, double *relres) {
  return ks_pcg_run(ctx, ctx->sell_A, ctx->dinv, ctx->mu, N, lambda, nullptr, U, Ut, tol, max_iter, iters, relres);
}

// General batched Jacobi-PCG on a sliced-ELL operator: A x = b with b = (lambda + mu) M u (B == null, the BVPs)
// or b = B (given, [n][N]; the Poisson solve of the Hartree potential), x0 = U.
ks_status ks_pcg_run(ks_ctx *ctx, const double *sell_vals, const double *dinv, double mu, int N,
                     const double *lambda, const double *B, const double *U, double *Ut, double tol, int max_iter,
                     int32_t *iters, double *relres) {
  const int np = pad_np(N);
  KS_TRY(ensure_solver_ws(ctx, np));
  const int64_t n = ctx->n_free;
  const bool direct = (np == N) && aligned32(U) && aligned32(Ut) && (!B || aligned32(B));
  const double *u = U, *bb = B;
  double *x = Ut;
  if (!direct) {
    k_pad<<<ks_blocks(n * np, 256), 256, 0, ctx->stream>>>(U, N, ctx->upad, np, n);
    KS_LAUNCHED(ctx);
    u = ctx->upad;
    x = ctx->xpad;
    if (B) {   // the given right-hand side is padded into the (not yet used) q buffer
      k_pad<<<ks_blocks(n * np, 256), 256, 0, ctx->stream>>>(B, N, ctx->bpad, np, n);
      KS_LAUNCHED(ctx);
      bb = ctx->bpad;
    }
  }
  PcgArgs a;
  a.sell_ptr = ctx->sell_ptr;
  a.sell_col = ctx->sell_col;
  a.A = sell_vals;
  a.M = ctx->sell_M;
  a.dinv = dinv;
  a.lambda = lambda;
  a.mu = mu;
  a.tol = tol;
  a.U = u;
  a.B = bb;
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
  KS_TRY(ks_materialize_views(ctx));
  k_true_residual<<<nblk, T, 2 * T * sizeof(double), ctx->stream>>>(ctx->row_ptr, ctx->col, ctx->A, ctx->M, lambda,
                                                                     ctx->mu, U, Ut, ctx->n_free, N, part);
  KS_LAUNCHED(ctx);
  k_true_residual_final<<<1, 64, 0, ctx->stream>>>(part, nblk, N, relres);
  KS_LAUNCHED(ctx);
  KS_CUDA(ctx, cudaFreeAsync(part, ctx->stream));
  return KS_OK;
}
