// ks_interp.cu -- NEXT-3: the nonnested interpolation operator P = I_H^h of Algorithm 1
// on the GPU: every fine free node is located in an independent (nonnested, possibly
// unstructured) coarse tet mesh and its row of P holds the barycentric coordinates of that coarse tet.
//
// Algorithm 1 in B200 form:
//   * the paper's quadtree over the coarse vertices -> a uniform bucket grid (cell ~ coarse vertex spacing),
//     built on the host with the coarse face adjacency and one incident tet per vertex (coarse meshes are
//     small: n_H + N is the size of the dense pencil);
//   * per fine node (one thread): nearest coarse vertex from the buckets (rings of cells until one holds a
//     vertex, plus one ring), then the paper's barycentric walk from one of its tets: while a coordinate is
//     negative, step to the neighbour across the face opposite the most negative one (the lowest local
//     index on ties, where the paper picks at random); a walk that leaves the mesh or exceeds its step
//     budget falls back to a scan of all coarse tets (the containing tet with the largest minimal
//     coordinate), so the result is always the containing tet.
// Row i keeps the coarse FREE vertices (Dirichlet vertices carry zero data) with |lambda| > KS_INTERP_DROP
// (reading R4), sorted by coarse free index. Deterministic.
#include <algorithm>
#include <array>
#include <cmath>
#include <cub/cub.cuh>

#include "ks_internal.cuh"
#include "ks_layout.cuh"

#define KS_INTERP_DROP 1e-13
#define KS_INTERP_ACCEPT (-1e-12)

namespace {

struct Locate {
  const double *xyz;        // fine coordinates
  const int32_t *node_of_free;
  const double *xc;         // coarse coordinates [3 n_c]
  const int32_t *tc;        // coarse tets [4 m_c]
  const double *Jinv;       // [9 m_c]
  const int32_t *nbr;       // [4 m_c] tet across the face opposite local vertex a, -1 on the boundary
  const int32_t *vtet;      // [n_c] one tet incident to the vertex
  const int32_t *cell_ptr;  // [ncell + 1]
  const int32_t *cell_v;    // [n_c] vertices by cell
  const int32_t *cfree;     // [n_c] coarse free index or -1
  double bmin[3], inv_h;
  int g[3];
  int64_t n_free, m_c;
  int max_walk;
  int32_t *cnt;             // [n_free] entries of the row
  int32_t *col4;            // [4 n_free]
  double *val4;             // [4 n_free]
  unsigned *flags;          // bit 1: walk fell back to the scan; bit 2: point outside the coarse mesh
};

__device__ __forceinline__ void bary(const Locate &a, int64_t t, const double q[3], double l[4]) {
  const int32_t v0 = __ldg(a.tc + 4 * t);
  const double d0 = q[0] - __ldg(a.xc + 3 * v0), d1 = q[1] - __ldg(a.xc + 3 * v0 + 1), d2 = q[2] - __ldg(a.xc + 3 * v0 + 2);
  const double *J = a.Jinv + 9 * t;
  l[1] = __ldg(J + 0) * d0 + __ldg(J + 1) * d1 + __ldg(J + 2) * d2;
  l[2] = __ldg(J + 3) * d0 + __ldg(J + 4) * d1 + __ldg(J + 5) * d2;
  l[3] = __ldg(J + 6) * d0 + __ldg(J + 7) * d1 + __ldg(J + 8) * d2;
  l[0] = 1.0 - l[1] - l[2] - l[3];
}

__global__ void k_locate(Locate a) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= a.n_free) return;
  const int64_t node = __ldg(a.node_of_free + i);
  const double q[3] = {__ldg(a.xyz + 3 * node), __ldg(a.xyz + 3 * node + 1), __ldg(a.xyz + 3 * node + 2)};
  int c[3];
  for (int d = 0; d < 3; d++) c[d] = min(a.g[d] - 1, max(0, (int)floor((q[d] - a.bmin[d]) * a.inv_h)));
  // nearest coarse vertex: rings of cells until one holds a vertex, then one more ring
  int32_t best_v = -1;
  double best_d = 1e300;
  int found_ring = -1;
  const int gmax = max(a.g[0], max(a.g[1], a.g[2]));
  for (int r = 0; r <= gmax; r++) {
    for (int z = c[2] - r; z <= c[2] + r; z++)
      for (int y = c[1] - r; y <= c[1] + r; y++)
        for (int x = c[0] - r; x <= c[0] + r; x++) {
          if (x < 0 || y < 0 || z < 0 || x >= a.g[0] || y >= a.g[1] || z >= a.g[2]) continue;
          if (max(abs(x - c[0]), max(abs(y - c[1]), abs(z - c[2]))) != r) continue;   // the ring only
          const int64_t cell = x + (int64_t)a.g[0] * (y + (int64_t)a.g[1] * z);
          for (int32_t k = __ldg(a.cell_ptr + cell); k < __ldg(a.cell_ptr + cell + 1); k++) {
            const int32_t v = __ldg(a.cell_v + k);
            const double e0 = q[0] - __ldg(a.xc + 3 * v), e1 = q[1] - __ldg(a.xc + 3 * v + 1),
                         e2 = q[2] - __ldg(a.xc + 3 * v + 2);
            const double dd = e0 * e0 + e1 * e1 + e2 * e2;
            if (dd < best_d || (dd == best_d && v < best_v)) { best_d = dd; best_v = v; }
          }
        }
    if (best_v >= 0 && found_ring < 0) found_ring = r;
    if (found_ring >= 0 && r >= found_ring + 1) break;
  }
  // barycentric walk (Algorithm 1)
  int64_t t = best_v >= 0 ? __ldg(a.vtet + best_v) : 0;
  double l[4];
  bool ok = false;
  for (int step = 0; step < a.max_walk; step++) {
    bary(a, t, q, l);
    int k = 0;
    for (int m = 1; m < 4; m++)
      if (l[m] < l[k]) k = m;
    if (l[k] >= KS_INTERP_ACCEPT) { ok = true; break; }
    const int32_t nt = __ldg(a.nbr + 4 * t + k);
    if (nt < 0) break;
    t = nt;
  }
  if (!ok) {  // fallback: the containing tet by a scan (largest minimal coordinate, first on ties)
    atomicOr(a.flags, 1u);
    double best_min = -1e300;
    int64_t bt = 0;
    for (int64_t s = 0; s < a.m_c; s++) {
      double ls[4];
      bary(a, s, q, ls);
      const double mn = fmin(fmin(ls[0], ls[1]), fmin(ls[2], ls[3]));
      if (mn > best_min) { best_min = mn; bt = s; }
    }
    if (best_min < -1e-10) atomicOr(a.flags, 2u);
    t = bt;
    bary(a, t, q, l);
  }
  // free coarse vertices with |lambda| > drop, sorted by coarse free index
  int32_t cc[4];
  double vv[4];
  int m = 0;
  for (int k = 0; k < 4; k++) {
    const int32_t cf = __ldg(a.cfree + __ldg(a.tc + 4 * t + k));
    if (cf < 0 || !(fabs(l[k]) > KS_INTERP_DROP)) continue;
    int pos = m;
    while (pos > 0 && cc[pos - 1] > cf) { cc[pos] = cc[pos - 1]; vv[pos] = vv[pos - 1]; pos--; }
    cc[pos] = cf;
    vv[pos] = l[k];
    m++;
  }
  a.cnt[i] = m;
  for (int k = 0; k < 4; k++) {
    a.col4[4 * i + k] = k < m ? cc[k] : -1;
    a.val4[4 * i + k] = k < m ? vv[k] : 0.0;
  }
}

__global__ void k_compact_rows(const int32_t *__restrict__ rowptr, const int32_t *__restrict__ col4,
                               const double *__restrict__ val4, int64_t n, int32_t *__restrict__ col,
                               double *__restrict__ val) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t b = rowptr[i], m = rowptr[i + 1] - b;
  for (int k = 0; k < m; k++) {
    col[b + k] = col4[4 * i + k];
    val[b + k] = val4[4 * i + k];
  }
}

struct InterpBufs {
  double *xc = nullptr, *J = nullptr, *val4 = nullptr;
  int32_t *tc = nullptr, *nbr = nullptr, *vtet = nullptr, *cptr = nullptr, *cv = nullptr, *cfree = nullptr;
  int32_t *cnt = nullptr, *col4 = nullptr;
  unsigned *flags = nullptr;
  uint8_t *cub = nullptr;
};

// the call's device buffers (caller-provided scratch, ks_interpolation_plan sizes it with the same list)
template <class A>
void interp_layout(A &a, InterpBufs &b, int64_t n_c, int64_t m_c, int64_t ncell, int64_t nf, size_t cub) {
  a.add(&b.xc, 3 * n_c, "coarse xyz");
  a.add(&b.J, 9 * m_c, "coarse inverse Jacobians");
  a.add(&b.tc, 4 * m_c, "coarse tets");
  a.add(&b.nbr, 4 * m_c, "coarse face neighbours");
  a.add(&b.vtet, n_c, "vertex tet");
  a.add(&b.cptr, ncell + 1, "bucket ptr");
  a.add(&b.cv, n_c, "bucket vertices");
  a.add(&b.cfree, n_c, "coarse free numbering");
  a.add(&b.cnt, nf + 1, "row counts");
  a.add(&b.col4, 4 * nf, "4-wide columns");
  a.add(&b.val4, 4 * nf, "4-wide values");
  a.add(&b.flags, 1, "flags");
  a.add(&b.cub, (int64_t)cub, "scan temporary");
}

// bucket grid over the coarse vertices: cell ~ the mean vertex spacing, <= 1024 cells per axis
void interp_grid(const double *xc, int64_t n_c, double bmin[3], double bmax[3], double *h, int g[3]) {
  for (int d = 0; d < 3; d++) { bmin[d] = 1e300; bmax[d] = -1e300; }
  for (int64_t v = 0; v < n_c; v++)
    for (int d = 0; d < 3; d++) {
      bmin[d] = std::min(bmin[d], xc[3 * v + d]);
      bmax[d] = std::max(bmax[d], xc[3 * v + d]);
    }
  double vol = 1.0;
  for (int d = 0; d < 3; d++) vol *= std::max(bmax[d] - bmin[d], 1e-300);
  *h = std::cbrt(vol / (double)std::max<int64_t>(n_c, 1));
  for (int d = 0; d < 3; d++) g[d] = std::max(1, std::min(1024, (int)std::ceil((bmax[d] - bmin[d]) / *h)));
}

}  // namespace

static ks_status interp_cub_bytes(int64_t nf, size_t *bytes) {
  int32_t *p = nullptr;
  *bytes = 0;
  return cub::DeviceScan::ExclusiveSum(nullptr, *bytes, p, p, (int)(nf + 1)) == cudaSuccess ? KS_OK : KS_E_CUDA;
}

ks_status ks_interpolation_plan_impl(ks_ctx *ctx, int64_t n_c, const double *xc, int64_t m_c, size_t *bytes) {
  double bmin[3], bmax[3], h;
  int g[3];
  interp_grid(xc, n_c, bmin, bmax, &h, g);
  size_t cub = 0;
  if (interp_cub_bytes(ctx->n_free, &cub) != KS_OK) return ks_fail(ctx, KS_E_CUDA, "CUB temporary-size query failed");
  KsSizer sz;
  InterpBufs b;
  interp_layout(sz, b, n_c, m_c, (int64_t)g[0] * g[1] * g[2], ctx->n_free, cub);
  *bytes = sz.bytes;
  return KS_OK;
}

ks_status ks_interpolation_impl(ks_ctx *ctx, int64_t n_c, const double *xc, int64_t m_c, const int32_t *tc,
                                const uint8_t *dc, void *d_work, size_t work_bytes, int32_t *d_rowptr, int32_t *d_col,
                                double *d_val, int64_t *h_nH, int64_t *h_pnnz) {
  cudaStream_t s = ctx->stream;
  // ---- host: coarse structures (free numbering, inverse Jacobians, face adjacency, vertex -> tet, buckets)
  std::vector<int32_t> cfree(n_c);
  int64_t nH = 0;
  for (int64_t v = 0; v < n_c; v++) cfree[v] = dc[v] ? -1 : (int32_t)nH++;
  std::vector<double> Jinv(9 * m_c);
  for (int64_t t = 0; t < m_c; t++) {
    double J[3][3];
    for (int k = 0; k < 4; k++) {
      const int32_t v = tc[4 * t + k];
      if (v < 0 || v >= n_c) return ks_fail(ctx, KS_E_MESH, "coarse tet %lld: node %d out of range", (long long)t, v);
    }
    const double *x0 = xc + 3 * (int64_t)tc[4 * t];
    for (int k = 0; k < 3; k++)
      for (int r = 0; r < 3; r++) J[r][k] = xc[3 * (int64_t)tc[4 * t + 1 + k] + r] - x0[r];
    const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                       J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    if (!(std::fabs(det) > 0.0)) return ks_fail(ctx, KS_E_MESH, "coarse tet %lld is degenerate", (long long)t);
    double *Ji = &Jinv[9 * t];
    Ji[0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
    Ji[1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
    Ji[2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
    Ji[3] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
    Ji[4] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
    Ji[5] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
    Ji[6] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
    Ji[7] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
    Ji[8] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
  }
  // faces: key = sorted vertex triple of the face opposite local vertex a
  std::vector<std::pair<std::array<int32_t, 3>, int64_t>> faces(4 * m_c);
  for (int64_t t = 0; t < m_c; t++)
    for (int a = 0; a < 4; a++) {
      std::array<int32_t, 3> f;
      int k = 0;
      for (int b = 0; b < 4; b++)
        if (b != a) f[k++] = tc[4 * t + b];
      std::sort(f.begin(), f.end());
      faces[4 * t + a] = {f, 4 * t + a};
    }
  std::sort(faces.begin(), faces.end());
  std::vector<int32_t> nbr(4 * m_c, -1);
  for (size_t k = 0; k + 1 < faces.size(); k++)
    if (faces[k].first == faces[k + 1].first) {
      nbr[faces[k].second] = (int32_t)(faces[k + 1].second / 4);
      nbr[faces[k + 1].second] = (int32_t)(faces[k].second / 4);
    }
  std::vector<int32_t> vtet(n_c, -1);
  for (int64_t t = m_c - 1; t >= 0; t--)
    for (int a = 0; a < 4; a++) vtet[tc[4 * t + a]] = (int32_t)t;   // smallest incident tet id
  double bmin[3], bmax[3], h;
  int g[3];
  interp_grid(xc, n_c, bmin, bmax, &h, g);
  const int64_t ncell = (int64_t)g[0] * g[1] * g[2];
  std::vector<int32_t> cell_of(n_c), cell_ptr(ncell + 1, 0), cell_v(n_c);
  for (int64_t v = 0; v < n_c; v++) {
    int c[3];
    for (int d = 0; d < 3; d++) c[d] = std::min(g[d] - 1, std::max(0, (int)std::floor((xc[3 * v + d] - bmin[d]) / h)));
    cell_of[v] = c[0] + g[0] * (c[1] + g[1] * c[2]);
    cell_ptr[cell_of[v] + 1]++;
  }
  for (int64_t k = 0; k < ncell; k++) cell_ptr[k + 1] += cell_ptr[k];
  {
    std::vector<int32_t> fill(cell_ptr.begin(), cell_ptr.end() - 1);
    for (int64_t v = 0; v < n_c; v++) cell_v[fill[cell_of[v]]++] = (int32_t)v;   // ascending ids per cell
  }
  // ---- device: the call's buffers carved from the caller's scratch
  const int64_t nf = ctx->n_free;
  size_t cub_bytes = 0;
  if (interp_cub_bytes(nf, &cub_bytes) != KS_OK) return ks_fail(ctx, KS_E_CUDA, "CUB temporary-size query failed");
  if (((uintptr_t)d_work & (KS_ALIGN - 1)) != 0) return ks_fail(ctx, KS_E_ARG, "ks_interpolation: d_work not aligned");
  struct CallRegion {
    ks_ctx *c;
    ~CallRegion() { c->reg[KS_R_CALL] = ks_region(); }
  } unbind{ctx};
  ctx->reg[KS_R_CALL].base = (uint8_t *)d_work;
  ctx->reg[KS_R_CALL].cap = work_bytes;
  ctx->reg[KS_R_CALL].off = 0;
  InterpBufs bf;
  {
    KsRegion rg(ctx, KS_R_CALL);
    KsCarver cv(ctx);
    interp_layout(cv, bf, n_c, m_c, ncell, nf, cub_bytes);
    KS_TRY(cv.st);
  }
  double *d_xc = bf.xc, *d_J = bf.J, *d_val4 = bf.val4;
  int32_t *d_tc = bf.tc, *d_nbr = bf.nbr, *d_vtet = bf.vtet, *d_cptr = bf.cptr, *d_cv = bf.cv, *d_cfree = bf.cfree;
  int32_t *d_cnt = bf.cnt, *d_col4 = bf.col4;
  unsigned *d_flags = bf.flags;
  KS_CUDA(ctx, cudaMemcpyAsync(d_xc, xc, sizeof(double) * 3 * n_c, cudaMemcpyHostToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(d_J, Jinv.data(), sizeof(double) * 9 * m_c, cudaMemcpyHostToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(d_tc, tc, sizeof(int32_t) * 4 * m_c, cudaMemcpyHostToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(d_nbr, nbr.data(), sizeof(int32_t) * 4 * m_c, cudaMemcpyHostToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(d_vtet, vtet.data(), sizeof(int32_t) * n_c, cudaMemcpyHostToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(d_cptr, cell_ptr.data(), sizeof(int32_t) * (ncell + 1), cudaMemcpyHostToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(d_cv, cell_v.data(), sizeof(int32_t) * n_c, cudaMemcpyHostToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(d_cfree, cfree.data(), sizeof(int32_t) * n_c, cudaMemcpyHostToDevice, s));
  KS_CUDA(ctx, cudaMemsetAsync(d_flags, 0, sizeof(unsigned), s));
  KS_CUDA(ctx, cudaMemsetAsync(d_cnt + nf, 0, sizeof(int32_t), s));
  Locate a;
  a.xyz = ctx->xyz;
  a.node_of_free = ctx->node_of_free;
  a.xc = d_xc;
  a.tc = d_tc;
  a.Jinv = d_J;
  a.nbr = d_nbr;
  a.vtet = d_vtet;
  a.cell_ptr = d_cptr;
  a.cell_v = d_cv;
  a.cfree = d_cfree;
  for (int d = 0; d < 3; d++) { a.bmin[d] = bmin[d]; a.g[d] = g[d]; }
  a.inv_h = 1.0 / h;
  a.n_free = nf;
  a.m_c = m_c;
  a.max_walk = (int)std::min<int64_t>(m_c + 8, 100000);
  a.cnt = d_cnt;
  a.col4 = d_col4;
  a.val4 = d_val4;
  a.flags = d_flags;
  k_locate<<<ks_blocks(nf, 128), 128, 0, s>>>(a);
  KS_LAUNCHED(ctx);
  size_t tmp_bytes = cub_bytes;
  KS_CUDA(ctx, cub::DeviceScan::ExclusiveSum(bf.cub, tmp_bytes, d_cnt, d_rowptr, (int)(nf + 1), s));
  ctx->launches++;
  k_compact_rows<<<ks_blocks(nf, 256), 256, 0, s>>>(d_rowptr, d_col4, d_val4, nf, d_col, d_val);
  KS_LAUNCHED(ctx);
  int32_t pnnz = 0;
  unsigned flags = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&pnnz, d_rowptr + nf, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaMemcpyAsync(&flags, d_flags, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  if (flags & 2u) return ks_fail(ctx, KS_E_MESH, "a fine node lies outside the coarse mesh");
  ctx->interp_fallbacks = (flags & 1u) ? 1 : 0;
  *h_nH = nH;
  *h_pnnz = pnnz;
  return KS_OK;
}
