// ks_efdev.cu -- the Chebyshev-filtered subspace iteration of ks_pencil_eig (NEXT-1) as ONE
// persistent cooperative kernel: every Rayleigh-Ritz step, convergence test and filter step runs on the device,
// with no host round trip and no library launch inside the loop (the small eigenvalue problem
// on W = [P | U~]; PAPER.md:1016-1019 solves it "in serial" on a CPU core).
//
// Input: C = L^-1 F_A L^-T (D x D symmetric), the start block X (D x m), the Gershgorin bound of C. Internally the
// D x m blocks are row-major with a row pitch mp = 4 (mod 8) >= m and ldp = D rounded up to 32 rows (zero padding),
// and C is tiled by 32-column chunks ([chunk][row][36]), so that a chunk of the GEMM is two contiguous bulk copies.
// Each CTA owns rt (8 or 16) rows of every block. A round:
//   1. T = C X for the CTA's rows on the FP64 tensor cores (mma.m8n8k4.f64). 64 k-rows of X and the CTA's C rows
//      per chunk stream through a shared-memory ring, filled by a producer warp with bulk copies (cp.async.bulk,
//      mbarrier completion) and drained by 8 consumer warps (two k-steps of 4 rows each per chunk); the warps'
//      partials are added in warp order;
//   2. Gram partials G = X^T X, H = X^T T over the CTA's rows; a two-level fixed-order sum over the CTAs;
//   3. Rayleigh-Ritz with the orthonormalisation folded in, computed redundantly (bitwise identically) by every
//      CTA from the summed G, H: column scaling d, Cholesky G~ = R^T R, R^-1, H~ = R^-T (d^-1 H d^-1) R^-1,
//      parallel cyclic Jacobi (round-robin pairs, the host routine's rotation and skip rule), ascending sort,
//      T = d^-1 R^-1 V; then X <- X T and C X <- T T (own rows);
//   4. wanted residuals ||C x_j - lambda_j x_j|| (fixed-order sums over the CTAs): stop at <= tol * bound;
//   5. otherwise the degree-deg Chebyshev filter damping [lambda_m, bound]: deg - 1 GEMM steps, each followed by
//      the three-term recurrence on the CTA's own rows (fused epilogue), one grid barrier per step.
// At convergence one more Cholesky-QR pass makes the block orthonormal; the kernel writes it, lambda and a status.
// All sums have fixed partitions and orders: the result is bitwise reproducible run to run.
#include "ks_grid.cuh"
#include "ks_internal.cuh"
#include "ks_sell.cuh"

namespace {

constexpr int EFD_CW = 8;                          // consumer warps of the GEMM; warp EFD_CW produces the ring
constexpr int EFD_NW = EFD_CW + 1, EFD_THREADS = 32 * EFD_NW;
constexpr int EFD_MMAX = 72;                       // m = k + 8 <= max_N + 8
constexpr int EFD_MT = 2, EFD_NT = EFD_MMAX / 8;   // m-tiles (rt <= 16) and n-tiles
constexpr int EFD_KC = 8 * EFD_CW;                 // k-rows per chunk: two k-steps per consumer warp
constexpr int EFD_KS = EFD_KC + 4;                 // C tile row stride (doubles): = 4 (mod 16), conflict-free
constexpr int EFD_NSMAX = 12;                      // ring stages (at most; as many as fit)

struct EfdArgs {
  const double *Ct;       // [ldp / KC][D][KS] C by 64-column chunks (columns past D zero)
  const double *x0;       // [m][D] start block (column-major, pitch D)
  double *blk[3];         // [ldp][mp] internal blocks (row-major), padding rows zero
  double *part;           // [grid][2 m m] per-CTA partials
  double *gsum;           // [2 m m] their sums
  const double *bound;    // device scalar: Gershgorin bound of C
  double *x_out;          // [m][D] the final orthonormal block (pitch D)
  double *lam_out;        // [m] Ritz values, ascending
  int *status;            // [2]: 1 converged, 0 not within maxit, -1 breakdown (dense fallback); rounds
  unsigned *bar;          // grid barrier counter (0 at launch)
  unsigned long long *trace;   // KS_EF_TRACE=1: (tag, %globaltimer) pairs of CTA 0, else null
  int *trace_count;
  int64_t D, ldp;
  int m, mp, k, rt, maxit, deg, ns;
  double tol;
};

__device__ __forceinline__ void mma884(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned long long efd_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct EfdRing {
  double *buf;         // [ns][KC mp + rt KS]
  uint64_t *full, *empty;
  unsigned g = 0;      // chunks consumed so far (uniform over the CTA)
};

// producer lane: chunk c (k-rows [KC c, KC c + KC)) of Y and of the CTA's C rows into stage g % ns (two bulk
// copies), after the stage's previous consumption
__device__ void efd_issue(const EfdArgs &a, EfdRing &R, const double *Y, int64_t r0, int c, unsigned g) {
  const int ns = a.ns, st = g % ns, rt = a.rt, mp = a.mp;
  if (g >= (unsigned)ns) mbar_wait(&R.empty[st], ((g / ns) - 1) & 1u);
  const int nrows = a.D - r0 < rt ? (int)(a.D - r0) : rt;
  double *S = R.buf + (size_t)st * (EFD_KC * mp + rt * EFD_KS);
  const unsigned by = (unsigned)(EFD_KC * mp) * 8u, bc = (unsigned)(nrows * EFD_KS) * 8u;
  mbar_expect_tx(&R.full[st], by + bc);
  bulk_g2s(S, Y + (int64_t)c * EFD_KC * mp, by, &R.full[st]);
  bulk_g2s(S + EFD_KC * mp, a.Ct + ((int64_t)c * a.D + r0) * EFD_KS, bc, &R.full[st]);
}

// out[r][j] (shared, [rt][m]) = sum_k C[r0 + r][k] Y[k][j] for the CTA's rows (Y: an internal block written by every
// CTA before the last grid barrier). Rows past D are zero.
__device__ void efd_gemm(const EfdArgs &a, EfdRing &R, const double *Y, int64_t r0, double *red, double *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, grp = lane >> 2, tig = lane & 3;
  const int m = a.m, mp = a.mp, rt = a.rt, MT = rt / 8, NT = (m + 7) / 8, ns = a.ns;
  const int nch = (int)(a.ldp / EFD_KC);
  if (warp == EFD_CW) {   // producer
    if (lane == 0) {
      asm volatile("fence.proxy.async.global;" ::: "memory");   // generic writes before the barrier -> bulk copies
      for (int c = 0; c < nch; c++) efd_issue(a, R, Y, r0, c, R.g + c);
    }
  } else {
    double acc[EFD_MT][EFD_NT][2];
#pragma unroll
    for (int mt = 0; mt < EFD_MT; mt++)
#pragma unroll
      for (int nt = 0; nt < EFD_NT; nt++) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    for (int c = 0; c < nch; c++) {
      const unsigned g = R.g + c;
      const int st = g % ns;
      mbar_wait(&R.full[st], (g / ns) & 1u);
      const double *S = R.buf + (size_t)st * (EFD_KC * mp + rt * EFD_KS), *SC = S + EFD_KC * mp;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int kl = 8 * warp + 4 * h + tig;   // k-row within the chunk (rows past D are zero in Y and C)
        double bf[EFD_NT];
#pragma unroll
        for (int nt = 0; nt < EFD_NT; nt++) {
          const int j = 8 * nt + grp;
          bf[nt] = (nt < NT && j < m) ? S[kl * mp + j] : 0.0;
        }
#pragma unroll
        for (int mt = 0; mt < EFD_MT; mt++) {
          if (mt >= MT) break;
          // C rows past D were not copied (stale shared memory): zero by select
          const double af = r0 + 8 * mt + grp < a.D ? SC[(8 * mt + grp) * EFD_KS + kl] : 0.0;
#pragma unroll
          for (int nt = 0; nt < EFD_NT; nt++)
            if (nt < NT) mma884(acc[mt][nt][0], acc[mt][nt][1], af, bf[nt]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&R.empty[st]);
    }
    const int rtm = rt * m;
#pragma unroll
    for (int mt = 0; mt < EFD_MT; mt++)
#pragma unroll
      for (int nt = 0; nt < EFD_NT; nt++)
#pragma unroll
        for (int v = 0; v < 2; v++) {
          const int i = 8 * mt + grp, j = 8 * nt + 2 * tig + v;
          if (mt < MT && nt < NT && j < m) red[warp * rtm + i * m + j] = acc[mt][nt][v];
        }
  }
  R.g += nch;
  __syncthreads();
  // fixed-order reduction over the consumer warps
  for (int r = warp; r < rt; r += EFD_NW)
    for (int j = lane; j < m; j += 32) {
      double s = 0.0;
      for (int w = 0; w < EFD_CW; w++) s += red[(w * rt + r) * m + j];
      out[r * m + j] = r0 + r < a.D ? s : 0.0;
    }
  __syncthreads();
}

// this CTA's partials [2][m][m] (column-major: G[b*m + a] = sum_r X[r][a] X[r][b], H likewise with T) -> part
__device__ void efd_gram_partial(const EfdArgs &a, const double *xo, const double *t, bool with_h) {
  const int m = a.m, rt = a.rt, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *dst = a.part + (int64_t)blockIdx.x * 2 * m * m;
  for (int cb = warp; cb < (with_h ? 2 : 1) * m; cb += EFD_NW) {   // column cb of [G | H]
    const int op = cb >= m, ib = op ? cb - m : cb;
    const double *y = op ? t : xo;
    for (int ia = lane; ia < m; ia += 32) {
      double s = 0.0;
      for (int r = 0; r < rt; r++) s = fma(xo[r * m + ia], y[r * m + ib], s);
      dst[(op * m + ib) * m + ia] = s;
    }
  }
}

// two-level sum of the per-CTA partials: CTA b sums entries [b E / G, (b+1) E / G) over all CTAs in CTA order
__device__ void efd_sum_partials(const EfdArgs &a, int nent) {
  const int64_t G = gridDim.x;
  const int e0 = (int)(nent * (int64_t)blockIdx.x / G), e1 = (int)(nent * (int64_t)(blockIdx.x + 1) / G);
  const int stride = 2 * a.m * a.m;
  for (int e = e0 + threadIdx.x; e < e1; e += EFD_THREADS) {
    double s = 0.0;
    for (int64_t b = 0; b < G; b++) s += __ldcg(a.part + b * stride + e);
    a.gsum[e] = s;
  }
}

// The small dense matrices are m x m column-major with an odd leading dimension ld. Cholesky of the column-scaled
// Gram G (pitch m) into B1 (upper factor R, G~ = R^T R) and R^-1 in B2; dsc[j] = sqrt(G_jj). One warp factors (lane
// = column: no block barriers), every warp then inverts columns of R. Returns false (uniform over the CTA) on a
// collapsed pivot (<= 1e-12), as the host routine.
__device__ bool efd_chol(int m, int ld, const double *G, double *B1, double *B2, double *dsc, int *flag) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int j = warp; j < m; j += EFD_NW) {
    const double dj = sqrt(G[j * m + j]);
    for (int i = lane; i < m; i += 32) {
      B1[j * ld + i] = G[j * m + i] / (sqrt(G[i * m + i]) * dj);
      B2[j * ld + i] = 0.0;
    }
    if (lane == 0) dsc[j] = dj;
  }
  __syncthreads();
  if (!(dsc[0] > 0.0)) return false;
  if (warp == 0) {
    int ok = 1;
    for (int p = 0; p < m; p++) {
      const double piv = B1[p * ld + p];
      if (!(piv > 1e-12)) { ok = 0; break; }   // warp-uniform
      const double rpp = sqrt(piv);
      __syncwarp();
      for (int j = p + lane; j < m; j += 32) B1[j * ld + p] = j == p ? rpp : B1[j * ld + p] / rpp;
      __syncwarp();
      for (int j = p + 1 + lane; j < m; j += 32) {   // lane owns column j of the trailing upper triangle
        const double rj = B1[j * ld + p];
        for (int i = p + 1; i <= j; i++) B1[j * ld + i] -= B1[i * ld + p] * rj;
      }
      __syncwarp();
    }
    if (lane == 0) *flag = ok;
  }
  __syncthreads();
  if (!*flag) return false;
  // R^-1 (upper) by back substitution, one warp per column: the lanes split each dot product (fixed butterfly)
  for (int j = warp; j < m; j += EFD_NW) {
    if (lane == 0) B2[j * ld + j] = 1.0 / B1[j * ld + j];
    __syncwarp();
    for (int i = j - 1; i >= 0; i--) {
      double v = 0.0;
      for (int l = i + 1 + lane; l <= j; l += 32) v = fma(B1[l * ld + i], B2[j * ld + l], v);
      v = warp_sum(v);
      if (lane == 0) B2[j * ld + i] = -v / B1[i * ld + i];
      __syncwarp();
    }
  }
  __syncthreads();
  return true;
}

// parallel cyclic Jacobi on A (m x m symmetric, pitch ld), V <- eigenvectors. A round rotates n/2 disjoint pairs
// (round-robin ordering, table pr[r][i] = (p, q)); each rotation zeroes a_pq (t = sgn(d) 2 a_pq / (|d| +
// sqrt(d^2 + 4 a_pq^2)), d = a_qq - a_pp: tan of the Jacobi angle; c = rsqrt(1 + t^2), s = t c; skipped when
// a_pq^2 <= 1e-36 |a_pp a_qq|, the host routine's rule). Disjoint rotations commute, so every 2 x 2 block of A is
// updated as J_a^T B J_b in one pass (columns first, as the host routine) and V <- V J. Sweeps until one without a
// rotation (at most 60).
__device__ int efd_jacobi(int m, int ld, double *A, double *V, double *rc, const unsigned char *pr, int *cnt) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = m + (m & 1), half = n / 2;
  for (int j = warp; j < m; j += EFD_NW)
    for (int i = lane; i < m; i += 32) V[j * ld + i] = i == j ? 1.0 : 0.0;
  __syncthreads();
  for (int sweep = 0; sweep < 60; sweep++) {
    if (tid == 0) *cnt = 0;
    __syncthreads();
    for (int r = 0; r < n - 1; r++) {
      const unsigned char *prr = pr + 2 * half * r;
      if (tid < half) {
        const int p = prr[2 * tid], q = prr[2 * tid + 1];
        double c = 1.0, s = 0.0;
        if (q < m) {
          const double apq = A[q * ld + p], app = A[p * ld + p], aqq = A[q * ld + q];
          if (!(apq * apq <= 1e-36 * fabs(app * aqq) || apq == 0.0)) {
            const double d = aqq - app;
            const double t = (d >= 0.0 ? 2.0 : -2.0) * apq / (fabs(d) + sqrt(d * d + 4.0 * apq * apq));
            c = rsqrt(1.0 + t * t);
            s = t * c;
            atomicAdd(cnt, 1);
          }
        }
        rc[2 * tid] = c;
        rc[2 * tid + 1] = s;
      }
      __syncthreads();
      for (int ia = warp; ia < half; ia += EFD_NW)   // 2 x 2 blocks (pair ia rows, pair ib columns)
        for (int ib = lane; ib < half; ib += 32) {
          const double ca = rc[2 * ia], sa = rc[2 * ia + 1], cb = rc[2 * ib], sb = rc[2 * ib + 1];
          if (sa == 0.0 && sb == 0.0) continue;
          const int pa = prr[2 * ia], qa = prr[2 * ia + 1], pb = prr[2 * ib], qb = prr[2 * ib + 1];
          const bool va = qa < m, vb = qb < m;
          const double b00 = A[pb * ld + pa], b01 = vb ? A[qb * ld + pa] : 0.0;
          const double b10 = va ? A[pb * ld + qa] : 0.0, b11 = (va && vb) ? A[qb * ld + qa] : 0.0;
          const double c00 = cb * b00 - sb * b01, c01 = sb * b00 + cb * b01;   // columns (J_b)
          const double c10 = cb * b10 - sb * b11, c11 = sb * b10 + cb * b11;
          A[pb * ld + pa] = ca * c00 - sa * c10;                                // rows (J_a^T)
          if (vb) A[qb * ld + pa] = ca * c01 - sa * c11;
          if (va) A[pb * ld + qa] = sa * c00 + ca * c10;
          if (va && vb) A[qb * ld + qa] = sa * c01 + ca * c11;
        }
      for (int ib = warp; ib < half; ib += EFD_NW) {   // V <- V J (columns pb, qb)
        const double cb = rc[2 * ib], sb = rc[2 * ib + 1];
        if (sb == 0.0) continue;
        const int pb = prr[2 * ib], qb = prr[2 * ib + 1];
        for (int i = lane; i < m; i += 32) {
          const double vp = V[pb * ld + i], vq = V[qb * ld + i];
          V[pb * ld + i] = cb * vp - sb * vq;
          V[qb * ld + i] = sb * vp + cb * vq;
        }
      }
      __syncthreads();
    }
    const int rotated = *cnt;
    __syncthreads();
    if (rotated == 0) return sweep + 1;
  }
  return 60;
}

__global__ void __launch_bounds__(EFD_THREADS, 1) k_ef_iterate(EfdArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bars[2 * EFD_NSMAX];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, m = a.m, rt = a.rt, k = a.k, ld = m | 1;
  const int64_t D = a.D, r0 = (int64_t)blockIdx.x * rt;
  const int mm = m * m, rtm = rt * m, n = m + (m & 1), half = n / 2;
  // shared layout: [union: GEMM ring ns x (KC mp + rt KS) | Rayleigh-Ritz buffers] (the ring is idle between GEMMs)
  //                [GEMM warp partials CW x rt x m] [xo][tt][cx] rt x m each [dsc lam rc] [ints] [pair table]
  const int mld = m * ld;
  const size_t ring = (size_t)a.ns * (EFD_KC * a.mp + rt * EFD_KS), rrb = 4 * (size_t)mld + 2 * (size_t)mm;
  EfdRing R;
  R.buf = sm;
  R.full = bars;
  R.empty = bars + EFD_NSMAX;
  double *B1 = sm, *B2 = sm + mld, *B3 = sm + 2 * mld, *B4 = sm + 3 * mld;   // RR buffers (pitch ld)
  double *GH = sm + 4 * mld;                                               // summed G, H (pitch m)
  double *red = sm + (ring > rrb ? ring : rrb);                            // [CW][rt][m]
  double *xo = red + EFD_CW * rtm, *tt = xo + rtm, *cx = tt + rtm;
  double *dsc = cx + rtm, *lam = dsc + EFD_MMAX, *rc = lam + EFD_MMAX;   // rc [2 * 36]
  int *ip = reinterpret_cast<int *>(rc + EFD_MMAX);                       // perm [72], flags [8]
  int *perm = ip, *flag = perm + EFD_MMAX;
  unsigned char *pr = reinterpret_cast<unsigned char *>(flag + 8);        // [n - 1][half][2]
  if (tid == 0) {
    for (int s = 0; s < a.ns; s++) {
      mbar_init(&R.full[s], 1);
      mbar_init(&R.empty[s], EFD_CW);
    }
    mbar_fence_init();
  }
  for (int x = tid; x < (n - 1) * half; x += EFD_THREADS) {   // round-robin pairs: round r, pair i
    const int r = x / half, i = x % half;
    const int a0 = i == 0 ? 0 : 1 + (i - 1 + r) % (n - 1), a1 = 1 + (n - 2 - i + r) % (n - 1);
    pr[2 * x] = (unsigned char)min(a0, a1);
    pr[2 * x + 1] = (unsigned char)max(a0, a1);
  }
  unsigned bt = 0;
  int xi = 0, status = 0, rounds = 0, nt = 0;
  // KS_EF_TRACE: (tag, %globaltimer) pairs at phase ends of CTA 0; tags 0 round start, 1 GEMM, 2 Gram sums,
  // 3 Cholesky, 4 reduced matrix, 5 Jacobi, 6 block update, 7 residual barrier, 8 filter
  auto stamp = [&](int tag) {
    if (a.trace && blockIdx.x == 0 && tid == 0 && nt + 1 < KS_TRACE_CAP) {
      a.trace[nt] = (unsigned long long)tag;
      a.trace[nt + 1] = efd_now();
    }
    nt += 2;
  };
  auto own_rows = [&](const double *Y, double *dst) {   // dst[r][j] = Y[r0 + r][j] (0 past D)
    for (int r = warp; r < rt; r += EFD_NW)
      for (int j = lane; j < m; j += 32) dst[r * m + j] = r0 + r < D ? __ldcg(Y + (r0 + r) * a.mp + j) : 0.0;
  };
  auto store_rows = [&](const double *src, double *Y) {
    for (int r = warp; r < rt; r += EFD_NW)
      if (r0 + r < D)
        for (int j = lane; j < m; j += 32) Y[(r0 + r) * a.mp + j] = src[r * m + j];
  };
  // [rt][m] = [rt][m] x T (m x m, pitch ld, in shared)
  auto times_T = [&](const double *src, const double *T, double *dst) {
    for (int r = warp; r < rt; r += EFD_NW)
      for (int j = lane; j < m; j += 32) {
        double s = 0.0;
        for (int l = 0; l < m; l++) s = fma(src[r * m + l], T[j * ld + l], s);
        dst[r * m + j] = s;
      }
  };
  // the start block's own rows into the internal block 0 (its padding rows were zeroed before the launch)
  for (int r = warp; r < rt; r += EFD_NW)
    if (r0 + r < D)
      for (int j = lane; j < m; j += 32) a.blk[0][(r0 + r) * a.mp + j] = a.x0[(int64_t)j * D + r0 + r];
  grid_barrier(a.bar, bt);
  const double bound = *a.bound, tol_abs = a.tol * bound;
  for (int it = 0; it < a.maxit; it++) {
    rounds = it + 1;
    // 1. T = C X (own rows), own X rows
    if (it > 0) grid_barrier(a.bar, bt);
    stamp(0);
    efd_gemm(a, R, a.blk[xi], r0, red, tt);
    own_rows(a.blk[xi], xo);
    __syncthreads();
    stamp(1);
    // 2. Gram partials, two-level sums
    efd_gram_partial(a, xo, tt, true);
    grid_barrier(a.bar, bt);
    efd_sum_partials(a, 2 * mm);
    grid_barrier(a.bar, bt);
    stamp(2);
    // 3. Rayleigh-Ritz (every CTA, identically)
    for (int x = tid; x < 2 * mm; x += EFD_THREADS) GH[x] = __ldcg(a.gsum + x);
    __syncthreads();
    if (!efd_chol(m, ld, GH, B1, B2, dsc, flag)) { status = -1; break; }
    stamp(3);
    // H~ = d^-1 H d^-1 (B4); B3 <- H~ R^-1; B1 <- R^-T B3 (symmetrised)
    for (int j = warp; j < m; j += EFD_NW)
      for (int i = lane; i < m; i += 32) B4[j * ld + i] = GH[mm + j * m + i] / (dsc[i] * dsc[j]);
    __syncthreads();
    for (int j = warp; j < m; j += EFD_NW)
      for (int i = lane; i < m; i += 32) {
        double s = 0.0;
        for (int l = 0; l <= j; l++) s = fma(B4[l * ld + i], B2[j * ld + l], s);
        B3[j * ld + i] = s;
      }
    __syncthreads();
    for (int j = warp; j < m; j += EFD_NW)
      for (int i = lane; i < m; i += 32) {
        double s = 0.0;
        for (int l = 0; l <= i; l++) s = fma(B2[i * ld + l], B3[j * ld + l], s);
        B4[j * ld + i] = s;
      }
    __syncthreads();
    for (int j = warp; j < m; j += EFD_NW)
      for (int i = lane; i < m; i += 32) B1[j * ld + i] = i == j ? B4[j * ld + i] : 0.5 * (B4[j * ld + i] + B4[i * ld + j]);
    __syncthreads();
    stamp(4);
    const int sweeps = efd_jacobi(m, ld, B1, B3, rc, pr, flag + 1);   // eigenvalues on diag(B1), vectors in B3
    stamp(5 + 100 * sweeps);   // (the trace records the sweep count with the Jacobi stamp)
    // ascending order (ties by index)
    for (int j = tid; j < m; j += EFD_THREADS) {
      const double dj = B1[j * ld + j];
      int rank = 0;
      for (int l = 0; l < m; l++) {
        const double dl = B1[l * ld + l];
        rank += (dl < dj || (dl == dj && l < j)) ? 1 : 0;
      }
      perm[rank] = j;
    }
    __syncthreads();
    for (int j = tid; j < m; j += EFD_THREADS) lam[j] = B1[perm[j] * ld + perm[j]];
    // T = d^-1 R^-1 V (B4)
    for (int j = warp; j < m; j += EFD_NW)
      for (int i = lane; i < m; i += 32) {
        const double *v = B3 + perm[j] * ld;
        double s = 0.0;
        for (int l = i; l < m; l++) s = fma(B2[l * ld + i], v[l], s);
        B4[j * ld + i] = s / dsc[i];
      }
    __syncthreads();
    // X <- X T (written back: nobody reads the block until the next barrier), C X <- T_gemm T
    times_T(xo, B4, cx);          // cx temporarily holds the new X rows
    __syncthreads();
    for (int x = tid; x < rtm; x += EFD_THREADS) xo[x] = cx[x];
    __syncthreads();
    times_T(tt, B4, cx);
    __syncthreads();
    store_rows(xo, a.blk[xi]);
    stamp(6);
    // 4. residual partials of the wanted columns, and the first filter step (own rows, speculative)
    for (int j = tid; j < k; j += EFD_THREADS) {
      double s = 0.0;
      for (int r = 0; r < rt; r++) {
        const double d = cx[r * m + j] - lam[j] * xo[r * m + j];
        s = fma(d, d, s);
      }
      a.part[(int64_t)blockIdx.x * 2 * mm + j] = s;
    }
    const double fa = lam[m - 1], fe = 0.5 * (bound - fa), fc = 0.5 * (bound + fa);
    double sigma = fe / (lam[0] - fc);
    const int yi = (xi + 1) % 3, zi = (xi + 2) % 3;
    for (int x = tid; x < rtm; x += EFD_THREADS) tt[x] = sigma / fe * (cx[x] - fc * xo[x]);
    __syncthreads();
    store_rows(tt, a.blk[yi]);
    grid_barrier(a.bar, bt);
    stamp(7);
    // residual sums (every CTA, CTA order) -> the same decision everywhere
    double rmax = 0.0;
    for (int j = 0; j < k; j++) {
      double s = 0.0;
      for (int64_t b = 0; b < (int64_t)gridDim.x; b++) s += __ldcg(a.part + b * 2 * mm + j);
      rmax = fmax(rmax, sqrt(s));
    }
    if (!isfinite(rmax)) { status = -1; break; }
    if (rmax <= tol_abs) { status = 1; break; }
    if (!(fe > 0.0)) { status = -1; break; }
    // 5. Chebyshev filter: Xp = X, Y = Y1; Yn = 2 s2 / e (C Y - c Y) - sigma s2 Xp
    const double s1 = 2.0 / sigma;
    int pi = xi, ci = yi, ni = zi;
    for (int d = 2; d <= a.deg; d++) {
      const double s2 = 1.0 / (s1 - sigma);
      if (d > 2) grid_barrier(a.bar, bt);
      efd_gemm(a, R, a.blk[ci], r0, red, tt);
      own_rows(a.blk[ci], xo);
      own_rows(a.blk[pi], cx);
      __syncthreads();
      for (int x = tid; x < rtm; x += EFD_THREADS) tt[x] = 2.0 * s2 / fe * (tt[x] - fc * xo[x]) - sigma * s2 * cx[x];
      __syncthreads();
      store_rows(tt, a.blk[ni]);
      const int t0 = pi;
      pi = ci;
      ci = ni;
      ni = t0;
      sigma = s2;
    }
    xi = ci;   // the next round's first barrier completes the filtered block
    stamp(8);
  }
  if (status == 1) {
    // one more Cholesky-QR pass: X <- X d^-1 R^-1 (the barrier: every CTA is done reading the residual partials)
    grid_barrier(a.bar, bt);
    efd_gram_partial(a, xo, tt, false);
    grid_barrier(a.bar, bt);
    efd_sum_partials(a, mm);
    grid_barrier(a.bar, bt);
    for (int x = tid; x < mm; x += EFD_THREADS) GH[x] = __ldcg(a.gsum + x);
    __syncthreads();
    if (!efd_chol(m, ld, GH, B1, B2, dsc, flag)) {
      status = -1;
    } else {
      for (int j = warp; j < m; j += EFD_NW)
        for (int i = lane; i < m; i += 32) B4[j * ld + i] = B2[j * ld + i] / dsc[i];
      __syncthreads();
      times_T(xo, B4, cx);
      __syncthreads();
      for (int r = warp; r < rt; r += EFD_NW)   // the result column-major, pitch D
        if (r0 + r < D)
          for (int j = lane; j < m; j += 32) a.x_out[(int64_t)j * D + r0 + r] = cx[r * m + j];
      if (blockIdx.x == 0)
        for (int j = tid; j < m; j += EFD_THREADS) a.lam_out[j] = lam[j];
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    a.status[0] = status;
    a.status[1] = rounds;
    if (a.trace) *a.trace_count = nt < KS_TRACE_CAP ? nt : KS_TRACE_CAP;
  }
}

// C by 64-column chunks: Ct[(c D + row) KS + kk] = C[row][64 c + kk] (0 past D; kk in [64, KS) never read)
__global__ void k_efd_tile_c(const double *__restrict__ C, int64_t D, int64_t nch, double *__restrict__ Ct) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= nch * D * EFD_KC) return;
  const int64_t kk = x % EFD_KC, row = (x / EFD_KC) % D, c = x / (EFD_KC * D), col = c * EFD_KC + kk;
  Ct[(c * D + row) * EFD_KS + kk] = col < D ? C[row * D + col] : 0.0;
}

}  // namespace

static int64_t efd_ldp(int64_t D) { return (D + EFD_KC - 1) / EFD_KC * EFD_KC; }
static int efd_mp(int m) { return (m + 3) / 8 * 8 + 4 >= m ? (m + 3) / 8 * 8 + 4 : (m + 3) / 8 * 8 + 12; }

// shared memory of k_ef_iterate for (m, rt, ns stages)
static size_t efd_smem(int m, int rt, int ns) {
  const size_t ld = (size_t)(m | 1), rtm = (size_t)rt * m;
  const size_t uni = std::max((size_t)ns * (EFD_KC * efd_mp(m) + rt * EFD_KS), 4 * (size_t)m * ld + 2 * (size_t)m * m);
  return sizeof(double) * (uni + (size_t)EFD_CW * rtm + 3 * rtm + 3 * EFD_MMAX) + sizeof(int) * (EFD_MMAX + 8) +
         2 * EFD_MMAX * EFD_MMAX;
}

// doubles of device scratch for dimension D: per-CTA partials, their sums, status words, the Ritz values, the tiled
// copy of C and the three internal blocks
int64_t ks_ef_device_scratch(int sm_count, int m, int64_t D) {
  const int64_t ldp = efd_ldp(D);
  return (int64_t)sm_count * 2 * m * m + 2 * m * m + 8 + m + 4 + (ldp / EFD_KC) * D * EFD_KS + 3 * ldp * efd_mp(m);
}

// Runs the whole filtered iteration on the device. C [D][D] (pitch D) is copied to a padded pitch first; x0 [m][D]:
// the start block; x_out [m][D]: the final block; scratch: ks_ef_device_scratch(sm_count, m, D) doubles (*lam_dev:
// the Ritz values in it); bound_dev: the Gershgorin bound. *status: 1 converged, 0 not within maxit, -1 breakdown;
// *ran = false when the kernel does not fit (the host-driven loop runs instead).
ks_status ks_ef_device(ks_ctx *ctx, int64_t D, int k, int m, const double *C, const double *x0, double *x_out,
                       const double *bound_dev, double *scratch, int maxit, int deg, double tol, int *status,
                       int *rounds, bool *ran, double **lam_dev) {
  *ran = false;
  if (m > EFD_MMAX || m < 2 || D < 2 * m) return KS_OK;
  int rt = (D + 7) / 8 <= ctx->sm_count ? 8 : 16;
  if (const char *e = getenv("KS_EF_RT")) rt = atoi(e) == 16 ? 16 : rt;   // A/B: rows per CTA
  if ((D + rt - 1) / rt > ctx->sm_count) return KS_OK;
  const int grid = (int)((D + rt - 1) / rt);
  int max_smem = 0;
  KS_CUDA(ctx, cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  // as many ring stages as fit (at most EFD_NSMAX, at least 2), leaving room for the static mbarriers
  int ns = EFD_NSMAX;
  while (ns > 2 && efd_smem(m, rt, ns) + 1024 > (size_t)max_smem) ns--;
  const size_t smem = efd_smem(m, rt, ns);
  if (smem + 1024 > (size_t)max_smem) return KS_OK;
  KS_CUDA(ctx, cudaFuncSetAttribute(k_ef_iterate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  KS_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ef_iterate, EFD_THREADS, smem));
  if (per_sm < 1) return KS_OK;
  const int64_t ldp = efd_ldp(D);
  const int mp = efd_mp(m);
  EfdArgs a;
  a.part = scratch;
  a.gsum = scratch + (int64_t)ctx->sm_count * 2 * m * m;
  int *st = reinterpret_cast<int *>(a.gsum + 2 * m * m);
  a.lam_out = a.gsum + 2 * m * m + 8;
  double *Ct = scratch + ((int64_t)ctx->sm_count * 2 * m * m + 2 * m * m + 8 + m + 3) / 4 * 4;   // 32-byte aligned
  const int64_t nch = ldp / EFD_KC;
  a.blk[0] = Ct + nch * D * EFD_KS;
  a.blk[1] = a.blk[0] + ldp * mp;
  a.blk[2] = a.blk[1] + ldp * mp;
  // the tiled C; the internal blocks zeroed (padding rows and columns)
  k_efd_tile_c<<<ks_blocks(nch * D * EFD_KC, 256), 256, 0, ctx->stream>>>(C, D, nch, Ct);
  KS_LAUNCHED(ctx);
  KS_CUDA(ctx, cudaMemsetAsync(a.blk[0], 0, sizeof(double) * 3 * ldp * mp, ctx->stream));
  a.Ct = Ct;
  a.x0 = x0;
  *lam_dev = a.lam_out;
  a.bound = bound_dev;
  a.x_out = x_out;
  a.status = st;
  a.bar = ctx->barrier;
  const char *tr = getenv("KS_EF_TRACE");
  a.trace = tr && tr[0] == '1' ? ctx->trace : nullptr;
  a.trace_count = ctx->trace_count;
  a.D = D;
  a.ldp = ldp;
  a.m = m;
  a.mp = mp;
  a.ns = ns;
  a.k = k;
  a.rt = rt;
  a.maxit = maxit;
  a.deg = deg;
  a.tol = tol;
  KS_CUDA(ctx, cudaMemsetAsync(ctx->barrier, 0, sizeof(unsigned), ctx->stream));
  void *args[] = {&a};
  KS_CUDA(ctx, cudaLaunchCooperativeKernel((const void *)k_ef_iterate, dim3(grid), dim3(EFD_THREADS), args, smem,
                                           ctx->stream));
  KS_LAUNCHED(ctx);
  int hs[2] = {0, 0};
  KS_CUDA(ctx, cudaMemcpyAsync(hs, st, sizeof(hs), cudaMemcpyDeviceToHost, ctx->stream));
  KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  *status = hs[0];
  *rounds = hs[1];
  *ran = true;
  return KS_OK;
}
