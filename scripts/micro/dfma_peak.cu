// Peak rate of the vector FP64 pipe (DFMA) and of the FP64 tensor cores (DMMA m8n8k4) on this GPU:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dfma_peak scripts/micro/dfma_peak.cu && ./dfma_peak
// Every thread runs ILP independent dependent-FMA chains from registers (no memory traffic); one JSON line per
// (kind, warps per SM, ILP): FMA per clock per SM and TFLOP/s. DESIGN.md §4 uses the result for the ALU bound of the
// gather kernels (k_proj_y) and of k_sym_gemm.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void k_dfma(double *out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int u = 0; u < ILP; u++) x[u] = threadIdx.x * 1e-3 + u;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < ILP; u++) x[u] = fma(x[u], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < ILP; u++) s += x[u];
  if (s == 123.456) out[0] = s;
}

template <int ILP>
__global__ void k_dmma(double *out, int iters, double a, double b) {
  double c0[ILP], c1[ILP];
#pragma unroll
  for (int u = 0; u < ILP; u++) { c0[u] = threadIdx.x; c1[u] = u; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < ILP; u++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c0[u]), "+d"(c1[u]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < ILP; u++) s += c0[u] + c1[u];
  if (s == 123.456) out[0] = s;
}

template <class F>
static void run(const char *kind, int ilp, int warps, F launch, double fma_per_thread_iter) {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch(p.multiProcessorCount, warps * 32, iters);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  launch(p.multiProcessorCount, warps * 32, iters);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double fma = fma_per_thread_iter * ilp * (double)iters * warps * 32 * p.multiProcessorCount;
  printf("{\"kind\": \"%s\", \"ilp\": %d, \"warps_per_sm\": %d, \"ms\": %.4f, \"TFLOPs\": %.2f, "
         "\"fma_per_clk_per_sm_at_max_clock\": %.1f}\n",
         kind, ilp, warps, ms, 2.0 * fma / (ms * 1e-3) / 1e12, fma / (ms * 1e-3) / (khz * 1e3) / p.multiProcessorCount);
}

int main() {
  double *out;
  cudaMalloc(&out, 8);
  for (int warps : {4, 8, 16, 32}) {
    run("dfma", 8, warps, [&](int g, int b, int it) { k_dfma<8><<<g, b>>>(out, it, 1.0000001, 1e-9); }, 1.0);
    run("dmma_m8n8k4", 4, warps, [&](int g, int b, int it) { k_dmma<4><<<g, b>>>(out, it, 1.0000001, 1e-9); },
        256.0 / 32.0);
  }
  return 0;
}
