// Microbenchmark ("route the gathers through the TMA unit"): the sliced-ELL SpMM
// Y = A X of the block PCG's S phase and the projection's Y pass, X, Y [n][16] fp64 row-major, A the
// 15-point Kuhn stencil of an nx^3 node grid in natural order (the C4 pattern's interior: own node + 14
// neighbours), SELL-8 with 4-slot groups, padding slots gather the own row with weight 0 (ks_sell.cu layout).
// Two ways, same FMA order per output (up to the order of the 4 products of a slot group: tma takes them
// in a rotated order so the shared-memory reads are bank-conflict free; values in [-0.5, 0.5), |error| ~ 1e-15):
//   ldg : ks_sell.cuh's sell_row: 4 lanes per row, 32-byte gathers (LDG.256), 8 in flight per lane;
//   tma : a producer warp per CTA issues, per 8-row slice, one cp.async.bulk.tensor tile::gather4 per (row,
//         slot group) -- the 4 gathered rows of X land in shared memory -- plus one bulk copy of the slice's
//         values; W consumer warps (one slice each per ring slot) read the rows with shared loads.
// NV = 2 reads a second value stream on the same columns (the Y pass's H and M).
// Prints us per SpMM, gathered rows/s and the HBM-side algorithmic bytes rate; checks tma == ldg bitwise.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o gather_bench gather_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cmath>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

constexpr int NP = 16, C = 8;

__device__ __forceinline__ void ldnc_v4(const double *p, double &a, double &b, double &c, double &d) {
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ void ld_v4(const double *p, double *r) {
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_v4(double *p, const double *v) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]) : "memory");
}

template <int NV>
__global__ void __launch_bounds__(256) k_ldg(const int32_t *__restrict__ sp, const int32_t *__restrict__ sc,
                                             const double *__restrict__ va, const double *__restrict__ vb,
                                             const double *X, double *Ya, double *Yb, long n) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const long row = t >> 2;
  const int sub = t & 3;
  if (row >= n) return;
  double ya[4] = {0, 0, 0, 0}, yb[4] = {0, 0, 0, 0};
  const long s = row / C;
  const int b = __ldg(sp + s), e = __ldg(sp + s + 1);
  const int groups = (e - b) / (4 * C);
  const long base = b + (row % C) * 4;
  const double *xs = X + sub * 4;
  int g = 0;
  for (; g + 2 <= groups; g += 2) {
    const long o = base + (long)g * (4 * C), o2 = o + 4 * C;
    const int4 c = __ldg(reinterpret_cast<const int4 *>(sc + o));
    const int4 d = __ldg(reinterpret_cast<const int4 *>(sc + o2));
    double a[8], bb[8], x[8][4];
    ldnc_v4(va + o, a[0], a[1], a[2], a[3]);
    ldnc_v4(va + o2, a[4], a[5], a[6], a[7]);
    if (NV == 2) { ldnc_v4(vb + o, bb[0], bb[1], bb[2], bb[3]); ldnc_v4(vb + o2, bb[4], bb[5], bb[6], bb[7]); }
    ld_v4(xs + (long)c.x * NP, x[0]); ld_v4(xs + (long)c.y * NP, x[1]);
    ld_v4(xs + (long)c.z * NP, x[2]); ld_v4(xs + (long)c.w * NP, x[3]);
    ld_v4(xs + (long)d.x * NP, x[4]); ld_v4(xs + (long)d.y * NP, x[5]);
    ld_v4(xs + (long)d.z * NP, x[6]); ld_v4(xs + (long)d.w * NP, x[7]);
#pragma unroll
    for (int j = 0; j < 8; j++)
#pragma unroll
      for (int v = 0; v < 4; v++) {
        ya[v] = fma(a[j], x[j][v], ya[v]);
        if (NV == 2) yb[v] = fma(bb[j], x[j][v], yb[v]);
      }
  }
  for (; g < groups; g++) {
    const long o = base + (long)g * (4 * C);
    const int4 c = __ldg(reinterpret_cast<const int4 *>(sc + o));
    double a[4], bb[4] = {0, 0, 0, 0}, x[4][4];
    ldnc_v4(va + o, a[0], a[1], a[2], a[3]);
    if (NV == 2) ldnc_v4(vb + o, bb[0], bb[1], bb[2], bb[3]);
    ld_v4(xs + (long)c.x * NP, x[0]); ld_v4(xs + (long)c.y * NP, x[1]);
    ld_v4(xs + (long)c.z * NP, x[2]); ld_v4(xs + (long)c.w * NP, x[3]);
#pragma unroll
    for (int j = 0; j < 4; j++)
#pragma unroll
      for (int v = 0; v < 4; v++) {
        ya[v] = fma(a[j], x[j][v], ya[v]);
        if (NV == 2) yb[v] = fma(bb[j], x[j][v], yb[v]);
      }
  }
  st_v4(Ya + row * NP + sub * 4, ya);
  if (NV == 2) st_v4(Yb + row * NP + sub * 4, yb);
}

// ---- TMA ----
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile("{\n .reg .pred P1;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra W_%=;\n}\n" ::"r"(su32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void gather4(void *dst, const CUtensorMap *map, int r0, int r1, int r2, int r3, uint64_t *bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
               ::"r"(su32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(bar)) : "memory");
}

constexpr int GMAX = 4;                             // slot groups per slice (the stencil's 15 -> 16 slots)
constexpr int SLOT_X = GMAX * C * 4 * NP;           // doubles of gathered rows per ring slot (16 KB)
constexpr int SLOT_V = GMAX * C * 4;                // doubles of one value stream per ring slot (1 KB)

template <int W, int ST, int NV>
__global__ void __launch_bounds__((W + 1) * 32, 1) k_tma(const int32_t *__restrict__ sp, const int32_t *__restrict__ sc,
                                                         const double *__restrict__ va, const double *__restrict__ vb,
                                                         double *Ya, double *Yb, long n_slices,
                                                         const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *xr = reinterpret_cast<double *>(smem);                         // [W][ST][SLOT_X]
  double *vr = xr + (size_t)W * ST * SLOT_X;                             // [W][ST][NV][SLOT_V]
  uint64_t *full = reinterpret_cast<uint64_t *>(vr + (size_t)W * ST * NV * SLOT_V);
  uint64_t *empty = full + W * ST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < W * ST; i++) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long stride = (long)gridDim.x * W;
  if (warp == W) {   // producer
    long k = 0;
    for (long s0 = (long)blockIdx.x * W; s0 < n_slices; s0 += stride, k++) {
      const int slot = (int)(k % ST);
      const unsigned ph = (unsigned)((k / ST) & 1);
      for (int w = 0; w < W; w++) {
        const long s = s0 + w;
        if (s >= n_slices) break;
        uint64_t *fb = full + w * ST + slot;
        mbar_wait(empty + w * ST + slot, ph ^ 1);
        const int b = __ldg(sp + s), e = __ldg(sp + s + 1);
        const int groups = (e - b) / (4 * C);
        if (lane == 0) mbar_expect_tx(fb, (unsigned)(groups * C * 4 * NP * 8 + NV * groups * 4 * C * 8));
        __syncwarp();
        double *xd = xr + ((size_t)w * ST + slot) * SLOT_X;
        if (lane < groups * C) {   // lane = g*8 + r: the slice's column blocks are contiguous
          const int4 c = __ldg(reinterpret_cast<const int4 *>(sc + b) + lane);
          gather4(xd + lane * 4 * NP, &tmap, c.x, c.y, c.z, c.w, fb);
        }
        if (lane == 0) bulk_g2s(vr + (((size_t)w * ST + slot) * NV) * SLOT_V, va + b, groups * 4 * C * 8, fb);
        if (NV == 2 && lane == 1) bulk_g2s(vr + (((size_t)w * ST + slot) * NV + 1) * SLOT_V, vb + b, groups * 4 * C * 8, fb);
      }
    }
    return;
  }
  const int r = lane >> 2, sub = lane & 3;
  long k = 0;
  for (long s = (long)blockIdx.x * W + warp; s < n_slices; s += stride, k++) {
    const int slot = (int)(k % ST);
    const unsigned ph = (unsigned)((k / ST) & 1);
    const int b = __ldg(sp + s), e = __ldg(sp + s + 1);
    const int groups = (e - b) / (4 * C);
    mbar_wait(full + warp * ST + slot, ph);
    const double *xs = xr + ((size_t)warp * ST + slot) * SLOT_X;
    const double *vs = vr + (((size_t)warp * ST + slot) * NV) * SLOT_V;
    double ya[4] = {0, 0, 0, 0}, yb[4] = {0, 0, 0, 0};
    for (int g = 0; g < groups; g++) {
      const double4 a = *reinterpret_cast<const double4 *>(vs + g * 32 + r * 4);
      double4 bb = make_double4(0, 0, 0, 0);
      if (NV == 2) bb = *reinterpret_cast<const double4 *>(vs + SLOT_V + g * 32 + r * 4);
      const double *xg = xs + ((g * C + r) * 4) * NP;
#pragma unroll
      for (int jj = 0; jj < 4; jj++) {
        // rows of the 128B-swizzled gather: 16-byte chunk c of a row at smem line L sits at c ^ (L % 8); row
        // j = (jj + r/2) % 4 makes the 8 rows of a warp hit 8 distinct lines mod 8 (conflict-free)
        const int j = (jj + (r >> 1)) & 3;
        const double *ln = xg + j * NP;
        const int L = (int)((su32(ln) >> 7) & 7);
        const double2 x0 = *reinterpret_cast<const double2 *>(ln + 2 * ((2 * sub) ^ L));
        const double2 x1 = *reinterpret_cast<const double2 *>(ln + 2 * ((2 * sub + 1) ^ L));
        const double x[4] = {x0.x, x0.y, x1.x, x1.y};
        const double aj = j == 0 ? a.x : j == 1 ? a.y : j == 2 ? a.z : a.w;
        const double bj = j == 0 ? bb.x : j == 1 ? bb.y : j == 2 ? bb.z : bb.w;
#pragma unroll
        for (int v = 0; v < 4; v++) {
          ya[v] = fma(aj, x[v], ya[v]);
          if (NV == 2) yb[v] = fma(bj, x[v], yb[v]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + warp * ST + slot);
    const long row = s * C + r;
    st_v4(Ya + row * NP + sub * 4, ya);
    if (NV == 2) st_v4(Yb + row * NP + sub * 4, yb);
  }
}


// self-issuing variant: every warp is its own producer (ST ring slots per warp, slice k + ST issued into the
// slot of slice k once the warp has consumed it): W warps issue gathers instead of one producer warp
template <int W, int ST, int NV>
__global__ void __launch_bounds__(W * 32, 1) k_tma_self(const int32_t *__restrict__ sp, const int32_t *__restrict__ sc,
                                                       const double *__restrict__ va, const double *__restrict__ vb,
                                                       double *Ya, double *Yb, long n_slices,
                                                       const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *xr = reinterpret_cast<double *>(smem);
  double *vr = xr + (size_t)W * ST * SLOT_X;
  uint64_t *full = reinterpret_cast<uint64_t *>(vr + (size_t)W * ST * NV * SLOT_V);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < W * ST; i++) mbar_init(full + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long stride = (long)gridDim.x * W;
  const long s_first = (long)blockIdx.x * W + warp;
  auto issue = [&](long k) {
    const long s = s_first + k * stride;
    if (s >= n_slices) return;
    const int slot = (int)(k % ST);
    uint64_t *fb = full + warp * ST + slot;
    const int b = __ldg(sp + s), e = __ldg(sp + s + 1);
    const int groups = (e - b) / (4 * C);
    if (lane == 0) mbar_expect_tx(fb, (unsigned)(groups * C * 4 * NP * 8 + NV * groups * 4 * C * 8));
    __syncwarp();
    double *xd = xr + ((size_t)warp * ST + slot) * SLOT_X;
    if (lane < groups * C) {
      const int4 c = __ldg(reinterpret_cast<const int4 *>(sc + b) + lane);
      gather4(xd + lane * 4 * NP, &tmap, c.x, c.y, c.z, c.w, fb);
    }
    if (lane == 0) bulk_g2s(vr + (((size_t)warp * ST + slot) * NV) * SLOT_V, va + b, groups * 4 * C * 8, fb);
    if (NV == 2 && lane == 1) bulk_g2s(vr + (((size_t)warp * ST + slot) * NV + 1) * SLOT_V, vb + b, groups * 4 * C * 8, fb);
  };
  for (int k = 0; k < ST; k++) issue(k);
  const int r = lane >> 2, sub = lane & 3;
  long k = 0;
  for (long s = s_first; s < n_slices; s += stride, k++) {
    const int slot = (int)(k % ST);
    const unsigned ph = (unsigned)((k / ST) & 1);
    const int b = __ldg(sp + s), e = __ldg(sp + s + 1);
    const int groups = (e - b) / (4 * C);
    mbar_wait(full + warp * ST + slot, ph);
    const double *xs = xr + ((size_t)warp * ST + slot) * SLOT_X;
    const double *vs = vr + (((size_t)warp * ST + slot) * NV) * SLOT_V;
    double ya[4] = {0, 0, 0, 0}, yb[4] = {0, 0, 0, 0};
    for (int g = 0; g < groups; g++) {
      const double4 a = *reinterpret_cast<const double4 *>(vs + g * 32 + r * 4);
      double4 bb = make_double4(0, 0, 0, 0);
      if (NV == 2) bb = *reinterpret_cast<const double4 *>(vs + SLOT_V + g * 32 + r * 4);
      const double *xg = xs + ((g * C + r) * 4) * NP;
#pragma unroll
      for (int jj = 0; jj < 4; jj++) {
        const int j = (jj + (r >> 1)) & 3;
        const double *ln = xg + j * NP;
        const int L = (int)((su32(ln) >> 7) & 7);
        const double2 x0 = *reinterpret_cast<const double2 *>(ln + 2 * ((2 * sub) ^ L));
        const double2 x1 = *reinterpret_cast<const double2 *>(ln + 2 * ((2 * sub + 1) ^ L));
        const double x[4] = {x0.x, x0.y, x1.x, x1.y};
        const double aj = j == 0 ? a.x : j == 1 ? a.y : j == 2 ? a.z : a.w;
        const double bj = j == 0 ? bb.x : j == 1 ? bb.y : j == 2 ? bb.z : bb.w;
#pragma unroll
        for (int v = 0; v < 4; v++) {
          ya[v] = fma(aj, x[v], ya[v]);
          if (NV == 2) yb[v] = fma(bj, x[v], yb[v]);
        }
      }
    }
    __syncwarp();
    issue(k + ST);
    const long row = s * C + r;
    st_v4(Ya + row * NP + sub * 4, ya);
    if (NV == 2) st_v4(Yb + row * NP + sub * 4, yb);
  }
}

typedef CUresult (*encode_fn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static double timeit(cudaEvent_t a, cudaEvent_t b, int reps) { float ms; cudaEventElapsedTime(&ms, a, b); return 1e3 * ms / reps; }

template <int W, int ST, int NV, bool SELF = false>
void run_tma(const char *name, int grid, const int32_t *sp, const int32_t *sc, const double *va, const double *vb,
             double *Ya, double *Yb, long ns, const CUtensorMap &map, int reps, double *ref_a, double *ref_b, long n,
             double alg_bytes, long nnz_slots) {
  const size_t sm = (size_t)W * ST * SLOT_X * 8 + (size_t)W * ST * NV * SLOT_V * 8 + 2 * W * ST * 8;
  auto kfn = SELF ? k_tma_self<W, ST, NV> : k_tma<W, ST, NV>;
  const int threads = SELF ? W * 32 : (W + 1) * 32;
  CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  CK(cudaMemset(Ya, 0, n * NP * 8));
  kfn<<<grid, threads, sm>>>(sp, sc, va, vb, Ya, Yb, ns, map);
  CK(cudaDeviceSynchronize());
  std::vector<double> h(n * NP), hr(n * NP);
  CK(cudaMemcpy(h.data(), Ya, n * NP * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hr.data(), ref_a, n * NP * 8, cudaMemcpyDeviceToHost));
  double err = 0;
  for (long i = 0; i < n * NP; i++) err = std::max(err, std::fabs(h[i] - hr[i]));
  if (NV == 2) {
    CK(cudaMemcpy(h.data(), Yb, n * NP * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hr.data(), ref_b, n * NP * 8, cudaMemcpyDeviceToHost));
    for (long i = 0; i < n * NP; i++) err = std::max(err, std::fabs(h[i] - hr[i]));
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; i++) kfn<<<grid, threads, sm>>>(sp, sc, va, vb, Ya, Yb, ns, map);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  const double us = timeit(e0, e1, reps);
  printf("{\"kernel\": \"%s\", \"NV\": %d, \"W\": %d, \"stages\": %d, \"grid\": %d, \"smem\": %zu, \"us\": %.1f, \"Grows_s\": %.1f, \"alg_GBs\": %.0f, \"maxabs_vs_ldg\": %.3g}\n",
         name, NV, W, ST, grid, sm, us, nnz_slots / us * 1e-3, alg_bytes / us * 1e-3, err);
}

int main(int argc, char **argv) {
  const int nx = argc > 1 ? atoi(argv[1]) : 128;
  const int reps = 20;
  const long n = (long)nx * nx * nx;
  // 15-point Kuhn stencil, natural order (x fastest); columns ascending, padded to whole groups with the own row
  const int off[15][3] = {{0, 0, 0},  {1, 0, 0},  {-1, 0, 0}, {0, 1, 0},  {0, -1, 0}, {0, 0, 1},  {0, 0, -1}, {1, 1, 0},
                          {-1, -1, 0}, {1, 0, 1}, {-1, 0, -1}, {0, 1, 1}, {0, -1, -1}, {1, 1, 1}, {-1, -1, -1}};
  const long ns = (n + C - 1) / C;
  std::vector<int32_t> sp(ns + 1);
  std::vector<std::vector<int32_t>> cols(n);
  for (long i = 0; i < n; i++) {
    const int x = i % nx, y = (i / nx) % nx, z = i / ((long)nx * nx);
    for (auto &o : off) {
      const int a = x + o[0], b = y + o[1], c = z + o[2];
      if (a < 0 || b < 0 || c < 0 || a >= nx || b >= nx || c >= nx) continue;
      cols[i].push_back((int32_t)(a + (long)nx * (b + (long)nx * c)));
    }
    std::sort(cols[i].begin(), cols[i].end());
  }
  long tot = 0;
  for (long s = 0; s < ns; s++) {
    sp[s] = (int32_t)tot;
    size_t w = 0;
    for (int r = 0; r < C; r++) if (s * C + r < n) w = std::max(w, (cols[s * C + r].size() + 3) / 4);
    tot += (long)w * 4 * C;
  }
  sp[ns] = (int32_t)tot;
  std::vector<int32_t> sc(tot);
  std::vector<double> va(tot), vb(tot);
  long nnz = 0;
  uint64_t st = 12345;
  auto rnd = [&]() { st = st * 6364136223846793005ULL + 1442695040888963407ULL; return (double)(st >> 11) / 9007199254740992.0 - 0.5; };
  for (long s = 0; s < ns; s++) {
    const int w = (sp[s + 1] - sp[s]) / (4 * C);
    if (w > GMAX) { printf("slice width %d > GMAX\n", w); return 1; }
    for (int g = 0; g < w; g++)
      for (int r = 0; r < C; r++)
        for (int q = 0; q < 4; q++) {
          const long row = s * C + r, o = sp[s] + (long)g * 4 * C + r * 4 + q;
          const size_t j = (size_t)g * 4 + q;
          if (row < n && j < cols[row].size()) { sc[o] = cols[row][j]; va[o] = rnd(); vb[o] = rnd(); nnz++; }
          else { sc[o] = (int32_t)std::min(row, n - 1); va[o] = 0; vb[o] = 0; }
        }
  }
  std::vector<double> X(n * NP);
  for (auto &v : X) v = rnd();
  int32_t *d_sp, *d_sc;
  double *d_va, *d_vb, *d_X, *d_Ya, *d_Yb, *d_Ra, *d_Rb;
  CK(cudaMalloc(&d_sp, (ns + 1) * 4)); CK(cudaMalloc(&d_sc, tot * 4));
  CK(cudaMalloc(&d_va, tot * 8)); CK(cudaMalloc(&d_vb, tot * 8));
  CK(cudaMalloc(&d_X, n * NP * 8)); CK(cudaMalloc(&d_Ya, n * NP * 8)); CK(cudaMalloc(&d_Yb, n * NP * 8));
  CK(cudaMalloc(&d_Ra, n * NP * 8)); CK(cudaMalloc(&d_Rb, n * NP * 8));
  CK(cudaMemcpy(d_sp, sp.data(), (ns + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_sc, sc.data(), tot * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_va, va.data(), tot * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_vb, vb.data(), tot * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_X, X.data(), n * NP * 8, cudaMemcpyHostToDevice));

  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)NP, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)NP * 8};
  const cuuint32_t box[2] = {(cuuint32_t)NP, 1u}, es[2] = {1u, 1u};
  if (((encode_fn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d_X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n"); return 1;
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  printf("{\"n\": %ld, \"nnz\": %ld, \"sell_slots\": %ld, \"sms\": %d}\n", n, nnz, tot, sms);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int NV = 1; NV <= 2; NV++) {
    // algorithmic HBM bytes: values (8 NV) + col (4) per slot, X read once, Y written (NV rows)
    const double alg = (double)tot * (8 * NV + 4) + 8.0 * NP * n * (1 + NV);
    const int grid = (int)((n * 4 + 255) / 256);
    auto lk = [&]() { if (NV == 1) k_ldg<1><<<grid, 256>>>(d_sp, d_sc, d_va, d_vb, d_X, d_Ra, d_Rb, n);
                      else k_ldg<2><<<grid, 256>>>(d_sp, d_sc, d_va, d_vb, d_X, d_Ra, d_Rb, n); };
    lk(); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int i = 0; i < reps; i++) lk();
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    const double us = timeit(e0, e1, reps);
    printf("{\"kernel\": \"ldg\", \"NV\": %d, \"us\": %.1f, \"Grows_s\": %.1f, \"alg_GBs\": %.0f}\n", NV, us, tot / us * 1e-3, alg / us * 1e-3);
    if (NV == 1) {
      run_tma<4, 3, 1>("tma", sms, d_sp, d_sc, d_va, d_vb, d_Ya, d_Yb, ns, map, reps, d_Ra, d_Rb, n, alg, tot);
      run_tma<6, 2, 1>("tma", sms, d_sp, d_sc, d_va, d_vb, d_Ya, d_Yb, ns, map, reps, d_Ra, d_Rb, n, alg, tot);
      run_tma<8, 1, 1>("tma", sms, d_sp, d_sc, d_va, d_vb, d_Ya, d_Yb, ns, map, reps, d_Ra, d_Rb, n, alg, tot);
      run_tma<3, 4, 1>("tma", sms, d_sp, d_sc, d_va, d_vb, d_Ya, d_Yb, ns, map, reps, d_Ra, d_Rb, n, alg, tot);
      run_tma<6, 2, 1, true>("tma_self", sms, d_sp, d_sc, d_va, d_vb, d_Ya, d_Yb, ns, map, reps, d_Ra, d_Rb, n, alg, tot);
      run_tma<12, 1, 1, true>("tma_self", sms, d_sp, d_sc, d_va, d_vb, d_Ya, d_Yb, ns, map, reps, d_Ra, d_Rb, n, alg, tot);
      run_tma<3, 2, 1, true>("tma_self", 2 * sms, d_sp, d_sc, d_va, d_vb, d_Ya, d_Yb, ns, map, reps, d_Ra, d_Rb, n, alg, tot);
      run_tma<2, 3, 1>("tma", 2 * sms, d_sp, d_sc, d_va, d_vb, d_Ya, d_Yb, ns, map, reps, d_Ra, d_Rb, n, alg, tot);
    } else {
      run_tma<4, 3, 2>("tma", sms, d_sp, d_sc, d_va, d_vb, d_Ya, d_Yb, ns, map, reps, d_Ra, d_Rb, n, alg, tot);
      run_tma<6, 2, 2>("tma", sms, d_sp, d_sc, d_va, d_vb, d_Ya, d_Yb, ns, map, reps, d_Ra, d_Rb, n, alg, tot);
      run_tma<2, 3, 2>("tma", 2 * sms, d_sp, d_sc, d_va, d_vb, d_Ya, d_Yb, ns, map, reps, d_Ra, d_Rb, n, alg, tot);
    }
  }
  return 0;
}
