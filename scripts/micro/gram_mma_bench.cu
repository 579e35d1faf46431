// Microbenchmark ("FP64 tensor-core MMA is justified only if a microbenchmark on the box
// shows it beating FP64 FFMA for the Gram epilogue"): G = U^T Y for U, Y [n][N] fp64 row-major, N = 16 / 32,
// per-warp partial Grams (no final reduction), two ways with the same row partition:
//   ffma: each lane owns 4x4 register tiles of G, rows read from L1/L2 (like k_proj_bg's Gram part);
//   dmma: mma.sync.aligned.m8n8k4.row.col.f64 (A = U^T tile 8x4, B = Y tile 4x8, 4 rows per k-step).
// Prints ms and achieved GFLOP/s (2 N^2 n flops) and checks both against each other.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <int N>
__global__ void __launch_bounds__(256) k_ffma(const double *__restrict__ U, const double *__restrict__ Y, long n,
                                              double *__restrict__ part) {
  constexpr int T4 = N / 4, NT = T4 * T4, MAXT = (NT + 31) / 32;
  const int lane = threadIdx.x & 31;
  const long gw = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5, nw = ((long)gridDim.x * blockDim.x) >> 5;
  double g[MAXT][16];
  for (int q = 0; q < MAXT; q++) for (int e = 0; e < 16; e++) g[q][e] = 0.0;
  const long r0 = n * gw / nw, r1 = n * (gw + 1) / nw;
  for (long i = r0; i < r1; i++) {
#pragma unroll
    for (int q = 0; q < MAXT; q++) {
      const int t = lane + 32 * q;
      if (t >= NT) continue;
      const int ta = t / T4, tb = t % T4;
      double u[4], y[4];
      for (int e = 0; e < 4; e++) { u[e] = __ldg(U + i * N + 4 * ta + e); y[e] = __ldg(Y + i * N + 4 * tb + e); }
#pragma unroll
      for (int x = 0; x < 4; x++)
#pragma unroll
        for (int z = 0; z < 4; z++) g[q][x * 4 + z] = fma(u[x], y[z], g[q][x * 4 + z]);
    }
  }
  for (int q = 0; q < MAXT; q++) {
    const int t = lane + 32 * q;
    if (t >= NT) continue;
    const int ta = t / T4, tb = t % T4;
    for (int x = 0; x < 4; x++) for (int z = 0; z < 4; z++) part[gw * N * N + (4 * ta + x) * N + 4 * tb + z] = g[q][x * 4 + z];
  }
}

template <int N>
__global__ void __launch_bounds__(256) k_dmma(const double *__restrict__ U, const double *__restrict__ Y, long n,
                                              double *__restrict__ part) {
  constexpr int TT = N / 8;                        // 8x8 tiles per dimension
  const int lane = threadIdx.x & 31, grp = lane >> 2, tig = lane & 3;
  const long gw = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5, nw = ((long)gridDim.x * blockDim.x) >> 5;
  double c[TT][TT][2];
  for (int a = 0; a < TT; a++) for (int b = 0; b < TT; b++) c[a][b][0] = c[a][b][1] = 0.0;
  long r0 = n * gw / nw, r1 = n * (gw + 1) / nw;
  r0 = (r0 + 3) & ~3L; r1 = (r1 + 3) & ~3L; if (r1 > n) r1 = n;   // k-steps of 4 rows (n multiple of 4 here)
  for (long i = r0; i + 4 <= r1; i += 4) {
    double af[TT], bf[TT];
#pragma unroll
    for (int a = 0; a < TT; a++) af[a] = __ldg(U + (i + tig) * N + 8 * a + grp);   // A[m=grp][k=tig] = U[i+k][8a+m]
#pragma unroll
    for (int b = 0; b < TT; b++) bf[b] = __ldg(Y + (i + tig) * N + 8 * b + grp);   // B[k=tig][n=grp] = Y[i+k][8b+n]
#pragma unroll
    for (int a = 0; a < TT; a++)
#pragma unroll
      for (int b = 0; b < TT; b++)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[a][b][0]), "+d"(c[a][b][1]) : "d"(af[a]), "d"(bf[b]));
  }
  for (int a = 0; a < TT; a++)
    for (int b = 0; b < TT; b++)
      for (int v = 0; v < 2; v++) part[gw * N * N + (8 * a + grp) * N + 8 * b + 2 * tig + v] = c[a][b][v];
}

template <int N>
void run(long n) {
  std::vector<double> hU(n * N), hY(n * N);
  unsigned long long s = 12345;
  for (auto &x : hU) { s = s * 6364136223846793005ULL + 1442695040888963407ULL; x = (double)(s >> 11) * 0x1.0p-53 - 0.5; }
  for (auto &x : hY) { s = s * 6364136223846793005ULL + 1442695040888963407ULL; x = (double)(s >> 11) * 0x1.0p-53 - 0.5; }
  double *U, *Y, *p1, *p2;
  const int blocks = 148 * 8, threads = 256;
  const long nwarps = (long)blocks * threads / 32;
  CK(cudaMalloc(&U, sizeof(double) * n * N)); CK(cudaMalloc(&Y, sizeof(double) * n * N));
  CK(cudaMalloc(&p1, sizeof(double) * nwarps * N * N)); CK(cudaMalloc(&p2, sizeof(double) * nwarps * N * N));
  CK(cudaMemcpy(U, hU.data(), sizeof(double) * n * N, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(Y, hY.data(), sizeof(double) * n * N, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best[2] = {1e30f, 1e30f};
  for (int rep = 0; rep < 6; rep++) {
    for (int v = 0; v < 2; v++) {
      cudaEventRecord(e0);
      if (v == 0) k_ffma<N><<<blocks, threads>>>(U, Y, n, p1); else k_dmma<N><<<blocks, threads>>>(U, Y, n, p2);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep > 0 && ms < best[v]) best[v] = ms;
    }
  }
  CK(cudaGetLastError());
  std::vector<double> g1(nwarps * N * N), g2(nwarps * N * N), s1(N * N, 0.0), s2(N * N, 0.0);
  CK(cudaMemcpy(g1.data(), p1, sizeof(double) * g1.size(), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(g2.data(), p2, sizeof(double) * g2.size(), cudaMemcpyDeviceToHost));
  for (long w = 0; w < nwarps; w++) for (int k = 0; k < N * N; k++) { s1[k] += g1[w * N * N + k]; s2[k] += g2[w * N * N + k]; }
  double md = 0, mx = 0; for (int k = 0; k < N * N; k++) { md = fmax(md, fabs(s1[k] - s2[k])); mx = fmax(mx, fabs(s1[k])); }
  const double fl = 2.0 * N * N * (double)n;
  const double gb = 2.0 * n * N * 8.0;
  printf("{\"N\": %d, \"n\": %ld, \"ffma_ms\": %.4f, \"dmma_ms\": %.4f, \"ffma_TFLOPs\": %.2f, \"dmma_TFLOPs\": %.2f, "
         "\"ffma_GBs\": %.0f, \"dmma_GBs\": %.0f, \"max_rel_diff\": %.2e}\n", N, n, best[0], best[1],
         fl / best[0] / 1e9, fl / best[1] / 1e9, gb / best[0] / 1e6, gb / best[1] / 1e6, md / mx);
  cudaFree(U); cudaFree(Y); cudaFree(p1); cudaFree(p2);
}

int main() {
  run<16>(2048384L);   // C4 rows (rounded to 4)
  run<32>(6967872L);   // C5 rows
  return 0;
}
