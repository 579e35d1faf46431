// ks_sell.cuh -- the sliced-ELL row kernel (ks_sell.cu layout) and the 32-byte vector types shared by the
// block PCG (ks_pcg.cu) and the projection (ks_project.cu). Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ks_internal.cuh"

// Solver layout of an [n][NP] block: a row group of LPR lanes owns one row, lane `sub` owns the VEC
// consecutive orbitals sub*VEC .. sub*VEC+VEC-1 (32-byte vectors for NP >= 4). Lane l therefore owns
// columns (VEC*l) % NP + v, in the S phase (row groups) and in the U/P streams (element VEC*thread).
template <int NP, int THREADS = 512>
struct SL {
  static_assert(NP == 1 || NP == 2 || NP == 4 || NP == 8 || NP == 16 || NP == 32 || NP == 64, "NP");
  static constexpr int VEC = NP >= 4 ? 4 : NP;
  static constexpr int LPR = NP / VEC;
  static constexpr int RPW = 32 / LPR;
  static constexpr int TILE = (THREADS / 32) * RPW;   // rows per tile of a THREADS-thread block
  static constexpr int CHUNK = THREADS * VEC;         // doubles per U/P chunk (= TILE * NP)
  static_assert(TILE * NP == CHUNK, "S tile and U/P chunk must cover the same rows");
};

template <int V>
struct DV;  // V consecutive doubles
template <>
struct DV<1> {
  double v[1];
  __device__ __forceinline__ static DV ld(const double *p) { DV r; r.v[0] = *p; return r; }
  __device__ __forceinline__ void st(double *p) const { *p = v[0]; }
};
template <>
struct DV<2> {
  double v[2];
  __device__ __forceinline__ static DV ld(const double *p) {
    double2 t = *reinterpret_cast<const double2 *>(p);
    DV r; r.v[0] = t.x; r.v[1] = t.y; return r;
  }
  __device__ __forceinline__ void st(double *p) const { *reinterpret_cast<double2 *>(p) = make_double2(v[0], v[1]); }
};
template <>
struct DV<4> {
  double v[4];
  __device__ __forceinline__ static DV ld(const double *p) {   // LDG.256 (32-byte aligned)
    DV r;
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3]) : "l"(p) : "memory");
    return r;
  }
  __device__ __forceinline__ void st(double *p) const {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
                 : "memory");
  }
};

__device__ __forceinline__ void ldnc_v4(const double *p, double &a, double &b, double &c, double &d) {
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

// One row of Y = Op X on the sliced-ELL copy (ks_sell.cu): slot groups of 4, CSR order within the row,
// padding slots gather the own row with weight 0. NV = 1 (ya = A x) or 2 (ya = A x, yb = B x on the
// same col stream). The operator arrays are read-only for the kernel's lifetime (non-coherent path);
// X may have been written by other blocks before a grid barrier and is read with coherent loads.
#ifndef KS_PCG_SUNR
#define KS_PCG_SUNR 2
#endif
constexpr int SUNR = KS_PCG_SUNR;             // slot groups (4 gathers each) in flight per lane

template <int NP, int NV>
__device__ __forceinline__ void sell_row(const int32_t *__restrict__ sell_ptr, const int32_t *__restrict__ scol,
                                         const double *__restrict__ va, const double *__restrict__ vb, int64_t row,
                                         const double *X, int sub, DV<SL<NP>::VEC> &ya, DV<SL<NP>::VEC> &yb) {
  constexpr int VEC = SL<NP>::VEC;
#pragma unroll
  for (int v = 0; v < VEC; v++) ya.v[v] = yb.v[v] = 0.0;
  const int64_t s = row / KS_SELL_C;
  const int32_t b = __ldg(sell_ptr + s), e = __ldg(sell_ptr + s + 1);
  const int groups = (e - b) / (4 * KS_SELL_C);
  const int64_t base = b + (row % KS_SELL_C) * 4;
  const double *xs = X + sub * VEC;
  int g = 0;
  if (SUNR == 2) {
    for (; g + 2 <= groups; g += 2) {   // two slot groups: 8 gathers in flight per lane
      const int64_t o = base + (int64_t)g * (4 * KS_SELL_C), o2 = o + 4 * KS_SELL_C;
      const int4 c = __ldg(reinterpret_cast<const int4 *>(scol + o));
      const int4 d = __ldg(reinterpret_cast<const int4 *>(scol + o2));
      double a[8], bb[8];
      ldnc_v4(va + o, a[0], a[1], a[2], a[3]);
      ldnc_v4(va + o2, a[4], a[5], a[6], a[7]);
      if (NV == 2) {
        ldnc_v4(vb + o, bb[0], bb[1], bb[2], bb[3]);
        ldnc_v4(vb + o2, bb[4], bb[5], bb[6], bb[7]);
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
          ya.v[v] = fma(a[j], x[j].v[v], ya.v[v]);
          if (NV == 2) yb.v[v] = fma(bb[j], x[j].v[v], yb.v[v]);
        }
    }
  }
  for (; g < groups; g++) {
    const int64_t o = base + (int64_t)g * (4 * KS_SELL_C);
    const int4 c = __ldg(reinterpret_cast<const int4 *>(scol + o));
    double a0, a1, a2, a3, b0 = 0, b1 = 0, b2 = 0, b3 = 0;
    ldnc_v4(va + o, a0, a1, a2, a3);
    if (NV == 2) ldnc_v4(vb + o, b0, b1, b2, b3);
    // padding slots gather the own row (cached) with weight 0: unconditional loads measured faster
    // than predicated ones (r01w: +2 % solve, +17 % Y pass)
    const DV<VEC> x0 = DV<VEC>::ld(xs + (int64_t)c.x * NP), x1 = DV<VEC>::ld(xs + (int64_t)c.y * NP);
    const DV<VEC> x2 = DV<VEC>::ld(xs + (int64_t)c.z * NP), x3 = DV<VEC>::ld(xs + (int64_t)c.w * NP);
#pragma unroll
    for (int v = 0; v < VEC; v++) {
      ya.v[v] = fma(a0, x0.v[v], ya.v[v]);
      ya.v[v] = fma(a1, x1.v[v], ya.v[v]);
      ya.v[v] = fma(a2, x2.v[v], ya.v[v]);
      ya.v[v] = fma(a3, x3.v[v], ya.v[v]);
      if (NV == 2) {
        yb.v[v] = fma(b0, x0.v[v], yb.v[v]);
        yb.v[v] = fma(b1, x1.v[v], yb.v[v]);
        yb.v[v] = fma(b2, x2.v[v], yb.v[v]);
        yb.v[v] = fma(b3, x3.v[v], yb.v[v]);
      }
    }
  }
}


// ---- bulk (TMA) copies global -> shared with mbarrier completion (cp.async.bulk, SASS UBLKCP) ----
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// bytes: multiple of 16, src and dst 16-byte aligned
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
