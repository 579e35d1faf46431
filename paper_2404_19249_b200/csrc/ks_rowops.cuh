// ks_rowops.cuh -- the multi-RHS CSR row kernel of the standalone SpMM (ks_spmm) for the operators without
// a sliced-ELL copy (K, M_V, H views). The hot path uses the sliced-ELL row kernel of ks_sell.cuh.
//
// Layout of a block of vectors: X[n][NP] row-major, NP a power of two <= 64. A "row group" of LPR lanes
// owns one row; lane `sub` of the group owns the VEC = 2 consecutive columns sub*VEC .. sub*VEC+1
// (NP = 1: one lane per row, VEC = 1). For NP >= 16 one group reads whole 128-byte lines of the gathered
// row with 16-byte loads, so every L1 wavefront of the gather carries useful bytes. A warp holds
// RPW = 32 / LPR row groups. The column owned by lane l is (VEC * l) % NP in every layout used here,
// which lets all reductions share one lane -> column map.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

template <int NP>
struct Lay {
  static_assert(NP == 1 || NP == 2 || NP == 4 || NP == 8 || NP == 16 || NP == 32 || NP == 64, "NP");
  static constexpr int VEC = NP >= 2 ? 2 : 1;
  static constexpr int LPR = NP / VEC;     // lanes per row
  static constexpr int RPW = 32 / LPR;     // rows per warp
};

template <int VEC>
struct Vec;
template <>
struct Vec<1> {
  double v[1];
  __device__ __forceinline__ static Vec load(const double *p) { Vec r; r.v[0] = *p; return r; }
  __device__ __forceinline__ static Vec ldcg(const double *p) { Vec r; r.v[0] = __ldcg(p); return r; }
  __device__ __forceinline__ static Vec ldg(const double *p) { Vec r; r.v[0] = __ldg(p); return r; }
  __device__ __forceinline__ void store(double *p) const { *p = v[0]; }
  __device__ __forceinline__ void zero() { v[0] = 0.0; }
};
template <>
struct Vec<2> {
  double v[2];
  __device__ __forceinline__ static Vec load(const double *p) {
    double2 t = *reinterpret_cast<const double2 *>(p);
    Vec r; r.v[0] = t.x; r.v[1] = t.y; return r;
  }
  __device__ __forceinline__ static Vec ldcg(const double *p) {
    double2 t = __ldcg(reinterpret_cast<const double2 *>(p));
    Vec r; r.v[0] = t.x; r.v[1] = t.y; return r;
  }
  __device__ __forceinline__ static Vec ldg(const double *p) {
    double2 t = __ldg(reinterpret_cast<const double2 *>(p));
    Vec r; r.v[0] = t.x; r.v[1] = t.y; return r;
  }
  __device__ __forceinline__ void store(double *p) const {
    *reinterpret_cast<double2 *>(p) = make_double2(v[0], v[1]);
  }
  __device__ __forceinline__ void zero() { v[0] = v[1] = 0.0; }
};

// y = sum_k val[k] * X[col[k]][sub*VEC ..] over the CSR row [k0, k1). X may be written elsewhere in the
// same kernel (PCG), so it is read with plain (L1-cached, coherent after the grid barrier) loads.
// The matrix stream (col, val) is read-only for the kernel's lifetime and goes through the
// non-coherent path. Unrolled by 4 so that 4 independent gathers are in flight per lane.
template <int NP>
__device__ __forceinline__ Vec<Lay<NP>::VEC> row_spmv(const int32_t *__restrict__ col,
                                                      const double *__restrict__ val, int32_t k0, int32_t k1,
                                                      const double *X, int sub) {
  constexpr int VEC = Lay<NP>::VEC;
  Vec<VEC> acc;
  acc.zero();
  int32_t k = k0;
  for (; k + 4 <= k1; k += 4) {
    int32_t c0 = __ldg(col + k), c1 = __ldg(col + k + 1), c2 = __ldg(col + k + 2), c3 = __ldg(col + k + 3);
    double a0 = __ldg(val + k), a1 = __ldg(val + k + 1), a2 = __ldg(val + k + 2), a3 = __ldg(val + k + 3);
    Vec<VEC> x0 = Vec<VEC>::load(X + (int64_t)c0 * NP + sub * VEC);
    Vec<VEC> x1 = Vec<VEC>::load(X + (int64_t)c1 * NP + sub * VEC);
    Vec<VEC> x2 = Vec<VEC>::load(X + (int64_t)c2 * NP + sub * VEC);
    Vec<VEC> x3 = Vec<VEC>::load(X + (int64_t)c3 * NP + sub * VEC);
#pragma unroll
    for (int v = 0; v < VEC; v++) {
      acc.v[v] = fma(a0, x0.v[v], acc.v[v]);
      acc.v[v] = fma(a1, x1.v[v], acc.v[v]);
      acc.v[v] = fma(a2, x2.v[v], acc.v[v]);
      acc.v[v] = fma(a3, x3.v[v], acc.v[v]);
    }
  }
  for (; k < k1; k++) {
    int32_t c0 = __ldg(col + k);
    double a0 = __ldg(val + k);
    Vec<VEC> x0 = Vec<VEC>::load(X + (int64_t)c0 * NP + sub * VEC);
#pragma unroll
    for (int v = 0; v < VEC; v++) acc.v[v] = fma(a0, x0.v[v], acc.v[v]);
  }
  return acc;
}
