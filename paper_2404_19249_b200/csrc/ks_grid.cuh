// ks_grid.cuh -- grid-wide barrier for the persistent cooperative kernels (ks_pcg.cu, ks_pcg2l.cu).
#pragma once
#include <cstdint>

namespace {

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

}  // namespace
