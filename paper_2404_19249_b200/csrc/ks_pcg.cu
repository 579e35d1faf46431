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
#include "ks_layout.cuh"
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
  const double *dg;             // diag(A) [n] (fused kernel: r = d z)
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
  // staged S phase of the fused kernel: the largest sliced-ELL entry count of one tile and the stage size
  int emax;
  unsigned stage_bytes;
  int stage_init;   // the init phase's A, M values and columns fit a stage (20 bytes per slot): staged too
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

template <int NP>
__global__ void __launch_bounds__(PCG_THREADS, KS_PCG_MINB) k_block_pcg(PcgArgs a) {
  constexpr int VEC = SL<NP, PCG_THREADS>::VEC, LPR = SL<NP, PCG_THREADS>::LPR, RPW = SL<NP, PCG_THREADS>::RPW, TILE = SL<NP, PCG_THREADS>::TILE;
  constexpr int CHUNK = SL<NP, PCG_THREADS>::CHUNK;
  constexpr int STRIDE = 4 * NP;                     // partial slots per block

  __shared__ double red[PCG_WARPS * 3 * NP];
  __shared__ double tot[3 * NP];
  __shared__ double s_alpha[NP], s_beta[NP], s_rho[NP], s_bnorm[NP], s_rr[NP];
  __shared__ int s_active[NP], s_conv[NP], s_iters[NP];
  __shared__ int s_any;

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
    {
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


// L2 prefetch of the streamed operands of a warp's rows one tile ahead (cp.async.bulk.prefetch: no register,
// no L1 wavefront; the later loads hit L2): the sliced-ELL values and columns of its slice and, in the fused S
// phase, its row segments of q, p and x. Sizes are multiples of 16 bytes for NP >= 4 (KS_PCG_PREFETCH=0: off).
#ifndef KS_PCG_PREFETCH
#define KS_PCG_PREFETCH 1
#endif
#ifndef KS_PCG_STG_MBAR
#define KS_PCG_STG_MBAR 1   // staged S phase: per-stage empty mbarriers instead of a block barrier per tile
#endif
#ifndef KS_PCG_CONTIG
#define KS_PCG_CONTIG 0   // fused kernel: contiguous tile chunks per block instead of interleaved tiles
#endif
#ifndef KS_PCG_PFDIST
#define KS_PCG_PFDIST 1   // tiles ahead
#endif
__device__ __forceinline__ void l2_prefetch(const void *ptr, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr), "r"(bytes) : "memory");
}
template <int NP, int RPW>
__device__ __forceinline__ void prefetch_rows(const PcgArgs &a, int64_t row0, const double *xin, bool streams) {
  if (row0 >= a.n) return;
  const int64_t rows = min((int64_t)RPW, a.n - row0);
  const int32_t e0 = __ldg(a.sell_ptr + row0 / KS_SELL_C), e1 = __ldg(a.sell_ptr + (row0 + rows - 1) / KS_SELL_C + 1);
  l2_prefetch(a.A + e0, (unsigned)(e1 - e0) * 8u);
  l2_prefetch(a.sell_col + e0, (unsigned)(e1 - e0) * 4u);
  if (streams) {
    const unsigned vb = (unsigned)(rows * NP * 8);
    l2_prefetch(a.q + row0 * NP, vb);
    l2_prefetch(a.p + row0 * NP, vb);
    l2_prefetch(xin + row0 * NP, vb);
  }
}

// One row of w = A z with the row's sliced-ELL values and columns in shared memory (a staged tile, below):
// the same slot groups and accumulation order as sell_row; the gathers of z stay global loads. OWN: also return
// the row's own gathered vector (its diagonal slot; padding slots gather the own row as well).
template <int NP, bool OWN = false>
__device__ __forceinline__ void sell_row_s(const double *vs, const int32_t *cs, int base, int groups,
                                           const double *X, int sub, DV<SL<NP>::VEC> &ya,
                                           int64_t row = 0, DV<SL<NP>::VEC> *own = nullptr) {
  constexpr int VEC = SL<NP>::VEC;
  auto take = [&](int32_t col, const DV<VEC> &x) {
    if (OWN && col == row) *own = x;
  };
#pragma unroll
  for (int v = 0; v < VEC; v++) ya.v[v] = 0.0;
  const double *xs = X + sub * VEC;
  int g = 0;
  for (; g + 2 <= groups; g += 2) {
    const int o = base + g * (4 * KS_SELL_C), o2 = o + 4 * KS_SELL_C;
    const int4 c = *reinterpret_cast<const int4 *>(cs + o);
    const int4 d = *reinterpret_cast<const int4 *>(cs + o2);
    double av[8];
    {
      const double2 t0 = *reinterpret_cast<const double2 *>(vs + o), t1 = *reinterpret_cast<const double2 *>(vs + o + 2);
      const double2 t2 = *reinterpret_cast<const double2 *>(vs + o2), t3 = *reinterpret_cast<const double2 *>(vs + o2 + 2);
      av[0] = t0.x; av[1] = t0.y; av[2] = t1.x; av[3] = t1.y; av[4] = t2.x; av[5] = t2.y; av[6] = t3.x; av[7] = t3.y;
    }
    DV<VEC> x[8];
    x[0] = DV<VEC>::ld(xs + (int64_t)c.x * NP);
    x[1] = DV<VEC>::ld(xs + (int64_t)c.y * NP);
    x[2] = DV<VEC>::ld(xs + (int64_t)c.z * NP);
    x[3] = DV<VEC>::ld(xs + (int64_t)c.w * NP);
    x[4] = DV<VEC>::ld(xs + (int64_t)d.x * NP);
    x[5] = DV<VEC>::ld(xs + (int64_t)d.y * NP);
    x[6] = DV<VEC>::ld(xs + (int64_t)d.z * NP);
    x[7] = DV<VEC>::ld(xs + (int64_t)d.w * NP);
#pragma unroll
    for (int j = 0; j < 8; j++)
#pragma unroll
      for (int v = 0; v < VEC; v++) ya.v[v] = fma(av[j], x[j].v[v], ya.v[v]);
    if (OWN) {
      take(c.x, x[0]); take(c.y, x[1]); take(c.z, x[2]); take(c.w, x[3]);
      take(d.x, x[4]); take(d.y, x[5]); take(d.z, x[6]); take(d.w, x[7]);
    }
  }
  for (; g < groups; g++) {
    const int o = base + g * (4 * KS_SELL_C);
    const int4 c = *reinterpret_cast<const int4 *>(cs + o);
    const double2 t0 = *reinterpret_cast<const double2 *>(vs + o), t1 = *reinterpret_cast<const double2 *>(vs + o + 2);
    const DV<VEC> x0 = DV<VEC>::ld(xs + (int64_t)c.x * NP), x1 = DV<VEC>::ld(xs + (int64_t)c.y * NP);
    const DV<VEC> x2 = DV<VEC>::ld(xs + (int64_t)c.z * NP), x3 = DV<VEC>::ld(xs + (int64_t)c.w * NP);
    if (OWN) {
      take(c.x, x0); take(c.y, x1); take(c.z, x2); take(c.w, x3);
    }
#pragma unroll
    for (int v = 0; v < VEC; v++) {
      ya.v[v] = fma(t0.x, x0.v[v], ya.v[v]);
      ya.v[v] = fma(t0.y, x1.v[v], ya.v[v]);
      ya.v[v] = fma(t1.x, x2.v[v], ya.v[v]);
      ya.v[v] = fma(t1.y, x3.v[v], ya.v[v]);
    }
  }
}

// One row of ya = A x, yb = M x from a staged tile (A values, M values and columns in shared memory): the slot
// groups and the accumulation order of sell_row<NP, 2>; the gathers of x stay global loads.
template <int NP>
__device__ __forceinline__ void sell_row_s2(const double *vs, const double *ms, const int32_t *cs, int base, int groups,
                                            const double *X, int sub, DV<SL<NP>::VEC> &ya, DV<SL<NP>::VEC> &yb) {
  constexpr int VEC = SL<NP>::VEC;
#pragma unroll
  for (int v = 0; v < VEC; v++) ya.v[v] = yb.v[v] = 0.0;
  const double *xs = X + sub * VEC;
  int g = 0;
  for (; g + 2 <= groups; g += 2) {
    const int o = base + g * (4 * KS_SELL_C), o2 = o + 4 * KS_SELL_C;
    const int4 c = *reinterpret_cast<const int4 *>(cs + o);
    const int4 d = *reinterpret_cast<const int4 *>(cs + o2);
    double av[8], bv[8];
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int oo = h ? o2 : o;
      const double2 t0 = *reinterpret_cast<const double2 *>(vs + oo), t1 = *reinterpret_cast<const double2 *>(vs + oo + 2);
      const double2 u0 = *reinterpret_cast<const double2 *>(ms + oo), u1 = *reinterpret_cast<const double2 *>(ms + oo + 2);
      av[4 * h] = t0.x; av[4 * h + 1] = t0.y; av[4 * h + 2] = t1.x; av[4 * h + 3] = t1.y;
      bv[4 * h] = u0.x; bv[4 * h + 1] = u0.y; bv[4 * h + 2] = u1.x; bv[4 * h + 3] = u1.y;
    }
    DV<VEC> x[8];
    x[0] = DV<VEC>::ld(xs + (int64_t)c.x * NP);
    x[1] = DV<VEC>::ld(xs + (int64_t)c.y * NP);
    x[2] = DV<VEC>::ld(xs + (int64_t)c.z * NP);
    x[3] = DV<VEC>::ld(xs + (int64_t)c.w * NP);
    x[4] = DV<VEC>::ld(xs + (int64_t)d.x * NP);
    x[5] = DV<VEC>::ld(xs + (int64_t)d.y * NP);
    x[6] = DV<VEC>::ld(xs + (int64_t)d.z * NP);
    x[7] = DV<VEC>::ld(xs + (int64_t)d.w * NP);
#pragma unroll
    for (int j = 0; j < 8; j++)
#pragma unroll
      for (int v = 0; v < VEC; v++) {
        ya.v[v] = fma(av[j], x[j].v[v], ya.v[v]);
        yb.v[v] = fma(bv[j], x[j].v[v], yb.v[v]);
      }
  }
  for (; g < groups; g++) {
    const int o = base + g * (4 * KS_SELL_C);
    const int4 c = *reinterpret_cast<const int4 *>(cs + o);
    const double2 t0 = *reinterpret_cast<const double2 *>(vs + o), t1 = *reinterpret_cast<const double2 *>(vs + o + 2);
    const double2 u0 = *reinterpret_cast<const double2 *>(ms + o), u1 = *reinterpret_cast<const double2 *>(ms + o + 2);
    const DV<VEC> x0 = DV<VEC>::ld(xs + (int64_t)c.x * NP), x1 = DV<VEC>::ld(xs + (int64_t)c.y * NP);
    const DV<VEC> x2 = DV<VEC>::ld(xs + (int64_t)c.z * NP), x3 = DV<VEC>::ld(xs + (int64_t)c.w * NP);
#pragma unroll
    for (int v = 0; v < VEC; v++) {
      ya.v[v] = fma(t0.x, x0.v[v], ya.v[v]);
      ya.v[v] = fma(t0.y, x1.v[v], ya.v[v]);
      ya.v[v] = fma(t1.x, x2.v[v], ya.v[v]);
      ya.v[v] = fma(t1.y, x3.v[v], ya.v[v]);
      yb.v[v] = fma(u0.x, x0.v[v], yb.v[v]);
      yb.v[v] = fma(u0.y, x1.v[v], yb.v[v]);
      yb.v[v] = fma(u1.x, x2.v[v], yb.v[v]);
      yb.v[v] = fma(u1.y, x3.v[v], yb.v[v]);
    }
  }
}

// the init phase's operators (A and M values, columns) of a warp's rows, one tile ahead
template <int RPW>
__device__ __forceinline__ void prefetch_init(const PcgArgs &a, int64_t row0) {
  if (row0 >= a.n) return;
  const int64_t rows = min((int64_t)RPW, a.n - row0);
  const int32_t e0 = __ldg(a.sell_ptr + row0 / KS_SELL_C), e1 = __ldg(a.sell_ptr + (row0 + rows - 1) / KS_SELL_C + 1);
  l2_prefetch(a.A + e0, (unsigned)(e1 - e0) * 8u);
  l2_prefetch(a.M + e0, (unsigned)(e1 - e0) * 8u);
  l2_prefetch(a.sell_col + e0, (unsigned)(e1 - e0) * 4u);
}

// ---------------------------------------------------------------------------------------------
// Fused two-phase iteration (the default for the BVPs, KS_PCG_FUSED=0 selects the three-phase kernel above).
// z = D^-1 r is stored instead of r, and q = A p is carried by the recurrence
//     q_{k+1} = A z_{k+1} + beta_k q_k        (p_{k+1} = z_{k+1} + beta_k p_k, exact-arithmetic identical)
// so that neither the p update nor the x update needs its own pass: both run inside the SpMM pass, on the rows
// the pass produces, while the gathers of z keep the load/store unit busy:
//   S  w = A z (gathered), q = w + beta q, p' = z + beta p, x += alpha_prev p, partials p'.q     | barrier
//   U  z -= alpha D^-1 q, partials d z^2 (= r.z) and d^2 z^2 (= r.r)                            | barrier
// The same 10 vector touches per iteration as the three-phase form, one grid barrier fewer. The deferred
// x_{k+1} = x_k + alpha_k p_k of the last iteration runs in a final streaming pass. Per-column freezing,
// NOT_SPD / NONFINITE / NOT_CONVERGED semantics and the fixed reduction order are those of k_block_pcg.
// STG: the S phases after the first stream each tile's sliced-ELL values and columns and its rows of q, p, x and
// z into shared memory with bulk copies (cp.async.bulk, SASS UBLKCP), two stages, one producer thread: the
// only global loads left on a row's dependency chain are the gathers of z.
template <int NP, bool STG>
__global__ void __launch_bounds__(PCG_THREADS, KS_PCG_MINB) k_block_pcg_fused(PcgArgs a) {
  constexpr int VEC = SL<NP, PCG_THREADS>::VEC, LPR = SL<NP, PCG_THREADS>::LPR, RPW = SL<NP, PCG_THREADS>::RPW,
                TILE = SL<NP, PCG_THREADS>::TILE, CHUNK = SL<NP, PCG_THREADS>::CHUNK;
  constexpr int STRIDE = 4 * NP;
  constexpr unsigned VB = TILE * NP * 8;   // bytes of one vector's tile rows
  extern __shared__ __align__(128) unsigned char dyn[];
  __shared__ __align__(8) uint64_t s_full[2], s_empty[2];
  unsigned pseq = 0;                        // stage uses so far (stage pseq & 1, parity (pseq >> 1) & 1)
  // the k-th row tile (= U/P chunk) of this block: interleaved over the blocks (t = b + k G, one sweeping
  // front of gathers, KS_PCG_CONTIG=0) or contiguous chunks (t = b per + k: consecutive tiles of a block are
  // grid neighbours, their gathers reuse L1)
  const int tper = (a.ntiles + (int)gridDim.x - 1) / (int)gridDim.x;
  const int64_t my_tiles = KS_PCG_CONTIG ? max(0, min(tper, a.ntiles - (int)blockIdx.x * tper))
                                         : (a.ntiles > (int)blockIdx.x ? (a.ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0);
  auto tile_k = [&](int64_t kk) -> int64_t {
    return KS_PCG_CONTIG ? (int64_t)blockIdx.x * tper + kk : (int64_t)blockIdx.x + kk * gridDim.x;
  };

  __shared__ double red[PCG_WARPS * 3 * NP];
  __shared__ double tot[3 * NP];
  __shared__ double s_alpha[NP], s_xalpha[NP], s_beta[NP], s_rho[NP], s_bnorm[NP], s_rr[NP];
  __shared__ int s_active[NP], s_iters[NP];
  __shared__ int s_any;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = lane / LPR, sub = lane % LPR;
  const int G = gridDim.x;
  const int64_t n = a.n;
  unsigned target = 0;
  double *part_a = a.partials;                        // region 0: init (3 dots) / U (2 dots)
  double *part_s = a.partials + (int64_t)G * STRIDE;  // region 1: S (1 dot)
  double *Z = a.r;                                    // the r buffer holds z = D^-1 r
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
  if constexpr (STG) {
    if (threadIdx.x == 0) {
      mbar_init(&s_full[0], 1);
      mbar_init(&s_full[1], 1);
      mbar_init(&s_empty[0], PCG_WARPS);   // one arrival per warp when it is done with a stage
      mbar_init(&s_empty[1], PCG_WARPS);
      mbar_fence_init();
    }
    __syncthreads();
  }

  // ---------------- init: b = (lambda+mu) M u, r = b - A u, z = r / d, p = z (x = u stays implicit) ------------
  {
    double acc[3][VEC];
#pragma unroll
    for (int d = 0; d < 3; d++)
#pragma unroll
      for (int v = 0; v < VEC; v++) acc[d][v] = 0.0;
    double sh[VEC];
#pragma unroll
    for (int v = 0; v < VEC; v++) {
      const int c = sub * VEC + v;
      sh[v] = (c < a.N ? __ldg(a.lambda + c) : 0.0) + a.mu;
    }
    constexpr bool PFI = KS_PCG_PREFETCH && NP >= 4;
    const bool sti = STG && a.stage_init;   // staged init: each tile's A, M values and columns by bulk copies
    const unsigned EB = (unsigned)a.emax;
    auto issue_init = [&](int64_t k) {   // one thread: the bulk copies of tile k into stage (pseq + k) & 1
      const int64_t r0 = tile_k(k) * TILE;
      const int64_t rows = min((int64_t)TILE, n - r0);
      const int32_t e0 = __ldg(a.sell_ptr + r0 / KS_SELL_C);
      const int32_t e1 = __ldg(a.sell_ptr + (r0 + rows + KS_SELL_C - 1) / KS_SELL_C);
      const unsigned q = pseq + (unsigned)k, eb = (unsigned)(e1 - e0);
      unsigned char *st = dyn + (size_t)(q & 1u) * a.stage_bytes;
      uint64_t *bar = &s_full[q & 1u];
      mbar_expect_tx(bar, eb * 20u);
      bulk_g2s(st, a.A + e0, eb * 8u, bar);
      bulk_g2s(st + 8u * EB, a.sell_col + e0, eb * 4u, bar);
      bulk_g2s(st + 12u * EB, a.M + e0, eb * 8u, bar);
    };
    if (sti && threadIdx.x == 0)
      for (int64_t k = 0; k < 2 && k < my_tiles; k++) issue_init(k);
    if (!sti && PFI && lane == 0 && my_tiles > 0) prefetch_init<RPW>(a, tile_k(0) * TILE + warp * RPW);
    for (int64_t kk = 0; kk < my_tiles; kk++) {
      const int64_t row = tile_k(kk) * TILE + warp * RPW + slot;
      if (!sti && PFI && lane == 0 && kk + 1 < my_tiles) prefetch_init<RPW>(a, tile_k(kk + 1) * TILE + warp * RPW);
      const unsigned q = pseq + (unsigned)kk;
      if (sti) mbar_wait(&s_full[q & 1u], (q >> 1) & 1u);
      if (row < n) {
        DV<VEC> au, mu_;
        if (sti) {
          const unsigned char *st = dyn + (size_t)(q & 1u) * a.stage_bytes;
          const int64_t t = tile_k(kk);
          const int32_t e0 = __ldg(a.sell_ptr + t * (TILE / KS_SELL_C));
          const int32_t b = __ldg(a.sell_ptr + row / KS_SELL_C), e = __ldg(a.sell_ptr + row / KS_SELL_C + 1);
          sell_row_s2<NP>(reinterpret_cast<const double *>(st), reinterpret_cast<const double *>(st + 12u * EB),
                          reinterpret_cast<const int32_t *>(st + 8u * EB), (b - e0) + (int)(row % KS_SELL_C) * 4,
                          (e - b) / (4 * KS_SELL_C), a.U, sub, au, mu_);
        } else {
          sell_row<NP, 2>(a.sell_ptr, a.sell_col, a.A, a.M, row, a.U, sub, au, mu_);
        }
        const int64_t off = row * NP + sub * VEC;
        const double dinv = __ldg(a.dinv + row);
        DV<VEC> z;
#pragma unroll
        for (int v = 0; v < VEC; v++) {
          const double b = sh[v] * mu_.v[v];
          const double r = b - au.v[v];
          z.v[v] = r * dinv;
          acc[0][v] += b * b;
          acc[1][v] += r * z.v[v];
          acc[2][v] += r * r;
        }
        z.st(Z + off);
        z.st(a.p + off);
      }
      if (sti) {   // this warp is done with the stage; the producer refills it once all warps are
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[q & 1u]);
        if (threadIdx.x == 0 && kk + 2 < my_tiles) {
          mbar_wait(&s_empty[q & 1u], (q >> 1) & 1u);
          issue_init(kk + 2);
        }
      }
    }
    if (sti) pseq += (unsigned)my_tiles;
    block_cols<NP, 3>(acc, red, tot);
    for (int i = threadIdx.x; i < 3 * NP; i += blockDim.x) part_a[(int64_t)blockIdx.x * STRIDE + i] = tot[i];
    grid_barrier(a.bar, target);
    stamp();
    reduce_partials(part_a, STRIDE, 3 * NP, tot);
    if (threadIdx.x < NP) {
      const int c = threadIdx.x;
      const double bn = sqrt(tot[c]), rz = tot[NP + c], rr = tot[2 * NP + c];
      s_bnorm[c] = bn;
      s_rho[c] = rz;
      s_rr[c] = rr;
      s_iters[c] = 0;
      s_alpha[c] = 0.0;
      s_xalpha[c] = 0.0;
      s_beta[c] = 0.0;
      const bool real = c < a.N;
      const bool finite = isfinite(bn) && isfinite(rr) && isfinite(rz);
      if (real && !finite && blockIdx.x == 0) atomicOr(a.flags, KSF_NONFINITE);
      s_active[c] = real && finite && !(sqrt(rr) <= a.tol * bn);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int any = 0;
      for (int c = 0; c < NP; c++) any |= s_active[c];
      s_any = any;
    }
    __syncthreads();
  }

  int it = 0;
  bool xwritten = false;   // x = u until the first deferred x update
  const int64_t nel = n * NP;
  const int nchunks = (int)((nel + CHUNK - 1) / CHUNK);
  const int cb = (VEC * threadIdx.x) % NP;
  if (s_any) {
    for (bool first = true;; first = false) {
      // ---- S: w = A z; q = w + beta q; p' = z + beta p; x += alpha_prev p; p'.q ----
      {
        double be[VEC], xa[VEC], acc[1][VEC];
#pragma unroll
        for (int v = 0; v < VEC; v++) {
          be[v] = s_beta[sub * VEC + v];
          xa[v] = s_xalpha[sub * VEC + v];
          acc[0][v] = 0.0;
        }
        const double *xin = xwritten ? a.X : a.U;
        if (STG) {
          // ---- staged: tile k of this block in stage (pseq + k) & 1 (first S phase: the operator slices only) ----
          const int64_t my = my_tiles;
          const unsigned EB = (unsigned)a.emax;
          auto issue = [&](int64_t k) {   // one thread: the bulk copies of tile k
            const int64_t r0 = tile_k(k) * TILE;
            const int64_t rows = min((int64_t)TILE, n - r0);
            const int32_t e0 = __ldg(a.sell_ptr + r0 / KS_SELL_C);
            const int32_t e1 = __ldg(a.sell_ptr + (r0 + rows + KS_SELL_C - 1) / KS_SELL_C);
            const unsigned q = pseq + (unsigned)k, eb = (unsigned)(e1 - e0), vb = (unsigned)(rows * NP * 8);
            unsigned char *st = dyn + (size_t)(q & 1u) * a.stage_bytes;
            uint64_t *bar = &s_full[q & 1u];
            mbar_expect_tx(bar, eb * 12u + (first ? 0u : 4u * vb));
            bulk_g2s(st, a.A + e0, eb * 8u, bar);
            bulk_g2s(st + 8u * EB, a.sell_col + e0, eb * 4u, bar);
            if (!first) {
              unsigned char *vbase = st + 12u * EB;
              bulk_g2s(vbase, a.q + r0 * NP, vb, bar);
              bulk_g2s(vbase + VB, a.p + r0 * NP, vb, bar);
              bulk_g2s(vbase + 2 * VB, xin + r0 * NP, vb, bar);
              bulk_g2s(vbase + 3 * VB, Z + r0 * NP, vb, bar);
            }
          };
          if (threadIdx.x == 0) {
            // q, p, x, z were written by the generic proxy before the grid barrier: order the bulk reads after
            asm volatile("fence.proxy.async.global;" ::: "memory");
            for (int64_t k = 0; k < 2 && k < my; k++) issue(k);
          }
          for (int64_t k = 0; k < my; k++) {
            const unsigned q = pseq + (unsigned)k;
            mbar_wait(&s_full[q & 1u], (q >> 1) & 1u);
            const unsigned char *st = dyn + (size_t)(q & 1u) * a.stage_bytes;
            const double *vs = reinterpret_cast<const double *>(st);
            const int32_t *cs = reinterpret_cast<const int32_t *>(st + 8u * EB);
            const double *qs = reinterpret_cast<const double *>(st + 12u * EB);
            const int64_t t = tile_k(k);
            const int lr = warp * RPW + slot;
            const int64_t row = t * TILE + lr;
            if (row < n) {
              const int32_t e0 = __ldg(a.sell_ptr + t * (TILE / KS_SELL_C));
              const int32_t b = __ldg(a.sell_ptr + row / KS_SELL_C), e = __ldg(a.sell_ptr + row / KS_SELL_C + 1);
              DV<VEC> w;
              const int64_t off0 = row * NP + sub * VEC;
              if (first) {   // p = z (init: bitwise), q = A p; p's row is the own gathered row of z
                DV<VEC> pv0;
                sell_row_s<NP, true>(vs, cs, (b - e0) + (int)(row % KS_SELL_C) * 4, (e - b) / (4 * KS_SELL_C), Z, sub,
                                     w, row, &pv0);
#pragma unroll
                for (int v = 0; v < VEC; v++) acc[0][v] += pv0.v[v] * w.v[v];
                w.st(a.q + off0);
              } else {
              sell_row_s<NP>(vs, cs, (b - e0) + (int)(row % KS_SELL_C) * 4, (e - b) / (4 * KS_SELL_C), Z, sub, w);
              const int so = lr * NP + sub * VEC;
              double qv[VEC], pv[VEC], xv[VEC], zv[VEC];
#pragma unroll
              for (int v = 0; v < VEC; v += 2) {
                const double2 q2 = *reinterpret_cast<const double2 *>(qs + so + v);
                const double2 p2 = *reinterpret_cast<const double2 *>(qs + VB / 8 + so + v);
                const double2 x2 = *reinterpret_cast<const double2 *>(qs + 2 * (VB / 8) + so + v);
                const double2 z2 = *reinterpret_cast<const double2 *>(qs + 3 * (VB / 8) + so + v);
                qv[v] = q2.x; qv[v + 1] = q2.y; pv[v] = p2.x; pv[v + 1] = p2.y;
                xv[v] = x2.x; xv[v + 1] = x2.y; zv[v] = z2.x; zv[v + 1] = z2.y;
              }
              DV<VEC> qo, po, xo;
#pragma unroll
              for (int v = 0; v < VEC; v++) {
                xo.v[v] = xv[v] + xa[v] * pv[v];
                po.v[v] = zv[v] + be[v] * pv[v];
                qo.v[v] = w.v[v] + be[v] * qv[v];
                acc[0][v] += po.v[v] * qo.v[v];
              }
              const int64_t off = row * NP + sub * VEC;
              qo.st(a.q + off);
              po.st(a.p + off);
              xo.st(a.X + off);
              }
            }
#if KS_PCG_STG_MBAR
            // this warp is done with the stage; the producer refills it once all warps are (no block barrier)
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[q & 1u]);
            if (threadIdx.x == 0 && k + 2 < my) {
              mbar_wait(&s_empty[q & 1u], (q >> 1) & 1u);
              issue(k + 2);
            }
#else
            __syncthreads();   // every warp is done with this stage
            if (threadIdx.x == 0 && k + 2 < my) issue(k + 2);
#endif
          }
          pseq += (unsigned)my;
        } else {
        constexpr bool PF = KS_PCG_PREFETCH && NP >= 4;
        if (PF && lane == 0)
          for (int d = 0; d < KS_PCG_PFDIST; d++)
            if (d < my_tiles) prefetch_rows<NP, RPW>(a, tile_k(d) * TILE + warp * RPW, xin, !first);
        for (int64_t kk = 0; kk < my_tiles; kk++) {
          const int64_t row = tile_k(kk) * TILE + warp * RPW + slot;
          if (PF && lane == 0 && kk + KS_PCG_PFDIST < my_tiles)
            prefetch_rows<NP, RPW>(a, tile_k(kk + KS_PCG_PFDIST) * TILE + warp * RPW, xin, !first);
          if (row < n) {
            DV<VEC> w, unused;
            sell_row<NP, 1>(a.sell_ptr, a.sell_col, a.A, nullptr, row, Z, sub, w, unused);
            const int64_t off = row * NP + sub * VEC;
            if (first) {   // p = z (init), q = A p
              const DV<VEC> pv = DV<VEC>::ld(a.p + off);
#pragma unroll
              for (int v = 0; v < VEC; v++) acc[0][v] += pv.v[v] * w.v[v];
              w.st(a.q + off);
            } else {
              DV<VEC> qv = DV<VEC>::ld(a.q + off), pv = DV<VEC>::ld(a.p + off);
              const DV<VEC> zv = DV<VEC>::ld(Z + off);
              DV<VEC> xv = DV<VEC>::ld(xin + off);
#pragma unroll
              for (int v = 0; v < VEC; v++) {
                xv.v[v] += xa[v] * pv.v[v];
                pv.v[v] = zv.v[v] + be[v] * pv.v[v];
                qv.v[v] = w.v[v] + be[v] * qv.v[v];
                acc[0][v] += pv.v[v] * qv.v[v];
              }
              qv.st(a.q + off);
              pv.st(a.p + off);
              xv.st(a.X + off);
            }
          }
        }
        }   // unstaged
        if (!first) xwritten = true;
        block_cols<NP, 1>(acc, red, tot);
        for (int i = threadIdx.x; i < NP; i += blockDim.x) part_s[(int64_t)blockIdx.x * STRIDE + i] = tot[i];
        grid_barrier(a.bar, target);
        stamp();
        reduce_partials(part_s, STRIDE, NP, tot);
        if (threadIdx.x < NP) {
          const int c = threadIdx.x;
          double al = 0.0;
          if (s_active[c]) {
            const double pq = tot[c];
            if (!(pq > 0.0)) {
              if (blockIdx.x == 0) atomicOr(a.flags, isfinite(pq) ? KSF_NOT_SPD : KSF_NONFINITE);
              s_active[c] = 0;
            } else {
              al = s_rho[c] / pq;
            }
          }
          s_alpha[c] = al;
          s_xalpha[c] = al;   // applied to x with this p in the next S pass (or the final pass)
        }
        __syncthreads();
      }

      // ---- U: z -= alpha D^-1 q; r.z = d z^2, r.r = (d z)^2 ----
      {
        double al[VEC], acc[2][VEC];
#pragma unroll
        for (int v = 0; v < VEC; v++) {
          al[v] = s_alpha[cb + v];
          acc[0][v] = acc[1][v] = 0.0;
        }
        for (int64_t kk = 0; kk < my_tiles; kk++) {
          const int64_t ch = tile_k(kk);
          const int64_t e = (int64_t)ch * CHUNK + VEC * threadIdx.x;
          if (e < nel) {
            DV<VEC> z = DV<VEC>::ld(Z + e);
            const DV<VEC> q = DV<VEC>::ld(a.q + e);
            const double di = __ldg(a.dinv + e / NP), dd = __ldg(a.dg + e / NP);
#pragma unroll
            for (int v = 0; v < VEC; v++) {
              z.v[v] -= al[v] * (q.v[v] * di);
              const double r = dd * z.v[v];
              acc[0][v] += r * z.v[v];
              acc[1][v] += r * r;
            }
            z.st(Z + e);
          }
        }
        block_cols<NP, 2>(acc, red, tot);
        for (int i = threadIdx.x; i < 2 * NP; i += blockDim.x) part_a[(int64_t)blockIdx.x * STRIDE + i] = tot[i];
        grid_barrier(a.bar, target);
        stamp();
        reduce_partials(part_a, STRIDE, 2 * NP, tot);
        if (threadIdx.x < NP) {
          const int c = threadIdx.x;
          double be = 0.0;
          if (s_active[c]) {
            const double rz = tot[c], rr = tot[NP + c];
            s_iters[c] += 1;
            bool conv;
            if (!isfinite(rz) || !isfinite(rr)) {
              if (blockIdx.x == 0) atomicOr(a.flags, KSF_NONFINITE);
              conv = true;
            } else {
              be = rz / s_rho[c];
              s_rho[c] = rz;
              s_rr[c] = rr;
              conv = sqrt(rr) <= a.tol * s_bnorm[c];
            }
            if (conv) {
              be = 0.0;
              s_active[c] = 0;
            }
          }
          s_beta[c] = be;
        }
        __syncthreads();
        it++;
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
      }
    }
  }

  // ---- final: the deferred x_{k+1} = x_k + alpha_k p_k (x = u when no iteration ran) ----
  {
    double xa[VEC];
#pragma unroll
    for (int v = 0; v < VEC; v++) xa[v] = s_xalpha[cb + v];
    const double *xin = xwritten ? a.X : a.U;
    for (int64_t kk = 0; kk < my_tiles; kk++) {
          const int64_t ch = tile_k(kk);
      const int64_t e = (int64_t)ch * CHUNK + VEC * threadIdx.x;
      if (e < nel) {
        DV<VEC> x = DV<VEC>::ld(xin + e);
        if (it > 0) {
          const DV<VEC> pv = DV<VEC>::ld(a.p + e);
#pragma unroll
          for (int v = 0; v < VEC; v++) x.v[v] += xa[v] * pv.v[v];
        }
        x.st(a.X + e);
      }
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

// largest sliced-ELL entry count of a tile of `slices` consecutive slices
__global__ void k_tile_emax(const int32_t *__restrict__ sell_ptr, int64_t n_slices, int slices, int *emax) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t s0 = t * slices;
  if (s0 >= n_slices) return;
  const int64_t s1 = s0 + slices < n_slices ? s0 + slices : n_slices;
  atomicMax(emax, sell_ptr[s1] - sell_ptr[s0]);
}

#ifndef KS_PCG_STAGED
#define KS_PCG_STAGED 1   // the staged S phase of the fused kernel when its two stages fit in shared memory
#endif
#ifndef KS_PCG_STAGED_MAXNP
#define KS_PCG_STAGED_MAXNP 32   // up to which block width (NP = 64: two stages do not fit)
#endif
constexpr size_t PCG_STAGE_SMEM_MAX = 200 * 1024;

template <int NP, bool FUSED, bool STG>
ks_status launch_pcg_t(ks_ctx *ctx, PcgArgs &a, size_t dyn) {
  auto kern = FUSED ? k_block_pcg_fused<NP, STG> : k_block_pcg<NP>;
  if (dyn > 0) KS_CUDA(ctx, cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  int per_sm = 0;
  KS_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PCG_THREADS, dyn));
  if (per_sm < 1) return ks_fail(ctx, KS_E_CUDA, "k_block_pcg<%d> cannot be resident", NP);
  if (per_sm > KS_PCG_GMAX_PER_SM) per_sm = KS_PCG_GMAX_PER_SM;   // the partials are planned for this many
  int G = per_sm * ctx->sm_count;
  if (G > a.ntiles) G = a.ntiles;
  a.partials = ctx->partials;
  KS_CUDA(ctx, cudaMemsetAsync(ctx->barrier, 0, sizeof(unsigned), ctx->stream));
  void *args[] = {&a};
  KS_CUDA(ctx, cudaLaunchCooperativeKernel((const void *)kern, dim3(G), dim3(PCG_THREADS), args, dyn, ctx->stream));
  ctx->launches++;
  return KS_OK;
}

template <int NP>
ks_status launch_pcg(ks_ctx *ctx, PcgArgs &a) {
  constexpr int TILE = SL<NP, PCG_THREADS>::TILE;
  a.ntiles = (int)((a.n + TILE - 1) / TILE);
  a.emax = 0;
  a.stage_bytes = 0;
  a.stage_init = 0;
  // the fused two-phase kernel serves the BVPs (right-hand side (lambda + mu) M u); the Poisson mode of the
  // Hartree solve (given B, up to ~10^3 iterations to 1e-12) keeps the three-phase recurrences
  const char *fz = getenv("KS_PCG_FUSED");
  if (a.B || (fz && fz[0] == '0')) return launch_pcg_t<NP, false, false>(ctx, a, 0);
  if constexpr (NP >= 4 && NP <= KS_PCG_STAGED_MAXNP && KS_PCG_STAGED) {
    const char *sg = getenv("KS_PCG_STAGED");
    if (!(sg && sg[0] == '0')) {
      int &em = ctx->tile_emax[__builtin_ctz(NP)];
      if (em == 0) {   // once per context and block width
        KsScratch scratch(ctx, KS_R_WORK);
        int *d = nullptr;
        KS_TRY(ks_alloc_t(ctx, &d, 1, "tile emax"));
        const int slices = TILE / KS_SELL_C;
        const int64_t nt = (ctx->n_slices + slices - 1) / slices;
        k_tile_emax<<<ks_blocks(nt, 256), 256, 0, ctx->stream>>>(ctx->sell_ptr, ctx->n_slices, slices, d);
        KS_LAUNCHED(ctx);
        KS_CUDA(ctx, cudaMemcpyAsync(&em, d, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        if (em <= 0) em = -1;
      }
      const size_t stage = (size_t)em * 12 + 4 * (size_t)TILE * NP * 8;
      if (em > 0 && 2 * stage <= PCG_STAGE_SMEM_MAX) {
        a.emax = em;
        a.stage_bytes = (unsigned)stage;
        a.stage_init = (size_t)em * 20 <= stage;   // the init phase's A, M values and columns fit a stage
        return launch_pcg_t<NP, true, true>(ctx, a, 2 * stage);
      }
    }
  }
  return launch_pcg_t<NP, true, false>(ctx, a, 0);
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

// true residual partials: per block sums of b^2 and (b - A ut)^2 per column (generic layout). A block of
// R * N threads covers a contiguous row range; thread t owns column t % N and every R-th row; the per-column
// sums are combined in a fixed order (deterministic, no atomics).
__global__ void k_true_residual(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                const double *__restrict__ A, const double *__restrict__ M,
                                const double *__restrict__ lambda, double mu, const double *__restrict__ U,
                                const double *__restrict__ Ut, int64_t n, int N, double *__restrict__ part) {
  __shared__ double sb[256], sr[256];
  const int R = blockDim.x / N;
  const int c = threadIdx.x % N, rs = threadIdx.x / N;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  double bb = 0.0, rr = 0.0;
  if (rs < R)
    for (int64_t row = r0 + rs; row < r1; row += R) {
      double mu_ = 0.0, au = 0.0;
      for (int32_t k = row_ptr[row]; k < row_ptr[row + 1]; k++) {
        mu_ = fma(M[k], U[(int64_t)col[k] * N + c], mu_);
        au = fma(A[k], Ut[(int64_t)col[k] * N + c], au);
      }
      const double b = (lambda[c] + mu) * mu_;
      bb += b * b;
      rr += (b - au) * (b - au);
    }
  sb[threadIdx.x] = bb;
  sr[threadIdx.x] = rr;
  __syncthreads();
  if (threadIdx.x < N) {
    double tb = 0.0, tr = 0.0;
    for (int q = 0; q < R; q++) {
      tb += sb[q * N + threadIdx.x];
      tr += sr[q * N + threadIdx.x];
    }
    part[(int64_t)blockIdx.x * 2 * N + threadIdx.x] = tb;
    part[(int64_t)blockIdx.x * 2 * N + N + threadIdx.x] = tr;
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
  if (N > ctx->max_N)
    return ks_fail(ctx, KS_E_ARG, "N = %d exceeds the max_N = %d the workspace was planned for", N, ctx->max_N);
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
  a.dg = ctx->diag;
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
  if (N > ctx->max_N) return ks_fail(ctx, KS_E_ARG, "N = %d exceeds max_N = %d", N, ctx->max_N);
  const int T = (256 / N) * N;
  const int nblk = 4 * ctx->sm_count;
  KsScratch scratch(ctx, KS_R_WORK);
  double *part = nullptr;
  KS_TRY(ks_alloc_t(ctx, &part, (int64_t)2 * N * nblk, "true residual partials"));
  KS_TRY(ks_materialize_views(ctx));
  k_true_residual<<<nblk, T, 0, ctx->stream>>>(ctx->row_ptr, ctx->col, ctx->A, ctx->M, lambda, ctx->mu, U, Ut,
                                                ctx->n_free, N, part);
  KS_LAUNCHED(ctx);
  k_true_residual_final<<<1, 64, 0, ctx->stream>>>(part, nblk, N, relres);
  KS_LAUNCHED(ctx);
  return KS_OK;
}
