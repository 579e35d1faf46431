// ks_setup.cu -- once-per-mesh setup on the device:
//   free numbering (Dirichlet elimination), CSR pattern of the P1 operators
//   (radix sort + unique of the 16 (row, col) pairs of every tet), element-to-nnz scatter map emap and
//   its inverse (emap indices grouped by target nnz), tet geometry, stiffness K and mass M of (st3)
//    gathered through the inverse map in a fixed order (no float atomics).
// CUB (shipped with the CUDA toolkit) provides the sort / scan / unique primitives of this setup step.
#include <cub/cub.cuh>

#include "ks_internal.cuh"
#include "ks_layout.cuh"

namespace {

__global__ void k_check_tets(const int32_t *__restrict__ tets, int64_t n_tets, int64_t n_nodes,
                             unsigned long long *bad) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_tets) return;
  for (int a = 0; a < 4; a++) {
    int32_t v = tets[4 * t + a];
    if (v < 0 || v >= n_nodes) atomicMin(bad, (unsigned long long)t);
  }
}

__global__ void k_notdir(const uint8_t *__restrict__ dir, int64_t n, int32_t *__restrict__ flag) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v < n) flag[v] = dir[v] ? 0 : 1;
}

__global__ void k_free_numbering(const uint8_t *__restrict__ dir, const int32_t *__restrict__ scan, int64_t n,
                                 int32_t *__restrict__ free_of_node, int32_t *__restrict__ node_of_free) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  if (dir[v]) {
    free_of_node[v] = -1;
  } else {
    free_of_node[v] = scan[v];
    node_of_free[scan[v]] = (int32_t)v;
  }
}

// |T| and grad lambda_a: J = [x1-x0, x2-x0, x3-x0]; rows of J^{-1} are
// grad lambda_1..3, grad lambda_0 = -(sum). Inverted / degenerate tets latch the smallest bad id.
__global__ void k_geometry(const double *__restrict__ xyz, const int32_t *__restrict__ tets, int64_t n_tets,
                           double *__restrict__ vol, double *__restrict__ grad, unsigned long long *bad) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_tets) return;
  int4 v = reinterpret_cast<const int4 *>(tets)[t];
  double x0 = xyz[3 * v.x], y0 = xyz[3 * v.x + 1], z0 = xyz[3 * v.x + 2];
  double J00 = xyz[3 * v.y] - x0, J10 = xyz[3 * v.y + 1] - y0, J20 = xyz[3 * v.y + 2] - z0;
  double J01 = xyz[3 * v.z] - x0, J11 = xyz[3 * v.z + 1] - y0, J21 = xyz[3 * v.z + 2] - z0;
  double J02 = xyz[3 * v.w] - x0, J12 = xyz[3 * v.w + 1] - y0, J22 = xyz[3 * v.w + 2] - z0;
  double c00 = J11 * J22 - J12 * J21, c01 = J12 * J20 - J10 * J22, c02 = J10 * J21 - J11 * J20;
  double det = J00 * c00 + J01 * c01 + J02 * c02;
  if (!(det > 0.0)) {
    atomicMin(bad, (unsigned long long)t);
    det = 1.0;
  }
  double id = 1.0 / det;
  double g[12];
  // row 0 of J^{-1}
  g[3] = c00 * id; g[4] = (J02 * J21 - J01 * J22) * id; g[5] = (J01 * J12 - J02 * J11) * id;
  // row 1
  g[6] = c01 * id; g[7] = (J00 * J22 - J02 * J20) * id; g[8] = (J02 * J10 - J00 * J12) * id;
  // row 2
  g[9] = c02 * id; g[10] = (J01 * J20 - J00 * J21) * id; g[11] = (J00 * J11 - J01 * J10) * id;
  g[0] = -(g[3] + g[6] + g[9]);
  g[1] = -(g[4] + g[7] + g[10]);
  g[2] = -(g[5] + g[8] + g[11]);
  vol[t] = det / 6.0;
#pragma unroll
  for (int k = 0; k < 12; k++) grad[12 * t + k] = g[k];
}

// 16 (row, col) keys per tet; pairs touching a Dirichlet node get the sentinel n_free << 32.
__global__ void k_pair_keys(const int32_t *__restrict__ tets, const int32_t *__restrict__ fon, int64_t n_tets,
                            uint64_t sentinel, uint64_t *__restrict__ keys) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= 16 * n_tets) return;
  int64_t t = i >> 4;
  int a = (int)((i >> 2) & 3), b = (int)(i & 3);
  int32_t fa = fon[tets[4 * t + a]], fb = fon[tets[4 * t + b]];
  keys[i] = (fa >= 0 && fb >= 0) ? (((uint64_t)(uint32_t)fa << 32) | (uint32_t)fb) : sentinel;
}

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t *a, int64_t n, uint64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int64_t lower_bound_i32(const int32_t *a, int64_t n, int32_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_row_ptr(const uint64_t *__restrict__ uniq, int64_t n_uniq, int64_t n_free,
                          int32_t *__restrict__ row_ptr) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r > n_free) return;
  row_ptr[r] = (int32_t)lower_bound_u64(uniq, n_uniq, (uint64_t)r << 32);
}

__global__ void k_cols(const uint64_t *__restrict__ uniq, int64_t nnz, int32_t *__restrict__ col) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < nnz) col[e] = (int32_t)(uniq[e] & 0xffffffffull);
}

__device__ __forceinline__ int32_t find_col(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                            int32_t r, int32_t c) {
  int32_t lo = row_ptr[r], hi = row_ptr[r + 1];
  int32_t p = lo + (int32_t)lower_bound_i32(col + lo, hi - lo, c);
  return (p < hi && col[p] == c) ? p : -1;
}

__global__ void k_diag_pos(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col, int64_t n_free,
                           int32_t *__restrict__ diag_pos) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n_free) diag_pos[i] = find_col(row_ptr, col, (int32_t)i, (int32_t)i);
}

// emap[16t+4a+b] = CSR position of (free(v_a), free(v_b)) or -1; inverse-map keys (nnz for -1).
__global__ void k_emap(const int32_t *__restrict__ tets, const int32_t *__restrict__ fon,
                       const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col, int64_t n_tets,
                       int64_t nnz, int32_t *__restrict__ emap, uint32_t *__restrict__ inv_key,
                       int32_t *__restrict__ inv_val) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= 16 * n_tets) return;
  int64_t t = i >> 4;
  int a = (int)((i >> 2) & 3), b = (int)(i & 3);
  int32_t fa = fon[tets[4 * t + a]], fb = fon[tets[4 * t + b]];
  int32_t e = (fa >= 0 && fb >= 0) ? find_col(row_ptr, col, fa, fb) : -1;
  emap[i] = e;
  inv_key[i] = e >= 0 ? (uint32_t)e : (uint32_t)nnz;
  inv_val[i] = (int32_t)i;
}

__global__ void k_inv_ptr(const uint32_t *__restrict__ keys, int64_t n_keys, int64_t nnz,
                          int32_t *__restrict__ inv_ptr) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e > nnz) return;
  int64_t lo = 0, hi = n_keys;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < (uint32_t)e) lo = mid + 1; else hi = mid;
  }
  inv_ptr[e] = (int32_t)lo;
}

// K_e = sum_T |T| grad l_a . grad l_b ; M_e = sum_T |T| (1+delta_ab)/20   (st3), gathered through the
// inverse map in ascending (t, a, b) order: deterministic, no atomics.
__global__ void k_stiffness_mass(const int32_t *__restrict__ inv_ptr, const int32_t *__restrict__ inv_idx,
                                 const double *__restrict__ vol, const double *__restrict__ grad, int64_t nnz,
                                 double *__restrict__ K, double *__restrict__ M) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  double k = 0.0, m = 0.0;
  for (int32_t j = inv_ptr[e]; j < inv_ptr[e + 1]; j++) {
    int32_t idx = inv_idx[j];
    int64_t t = idx >> 4;
    int a = (idx >> 2) & 3, b = idx & 3;
    const double *g = grad + 12 * t;
    double v = vol[t];
    k += v * (g[3 * a] * g[3 * b] + g[3 * a + 1] * g[3 * b + 1] + g[3 * a + 2] * g[3 * b + 2]);
    m += v * (a == b ? 2.0 : 1.0) / 20.0;
  }
  K[e] = k;
  M[e] = m;
}

int bitlen(uint64_t x) {
  int b = 0;
  while (x) { b++; x >>= 1; }
  return b;
}

}  // namespace


ks_status ks_setup_mesh(ks_ctx *ctx, const double *h_xyz, const int32_t *h_tets, const uint8_t *h_dir) {
  cudaStream_t s = ctx->stream;
  const int64_t nn = ctx->n_nodes, nt = ctx->n_tets;
  const int T = 256;
  // sizes of the setup products counted on the host (the plan's count), then every buffer carved up front:
  // the persistent layout from the caller's persistent region, the temporaries from the setup region
  KsMeshSizes z;
  KS_TRY(ks_count_mesh(nn, h_tets, nt, h_dir, &z, &ctx->err));
  size_t cub_cap = 0;
  if (ks_setup_cub_bytes(z, &cub_cap) != KS_OK) return ks_fail(ctx, KS_E_CUDA, "CUB temporary-size query failed");
  {
    KsRegion rg(ctx, KS_R_PERSIST);
    KsCarver cv(ctx);
    ks_layout_persist(cv, ctx, z);
    KS_TRY(cv.st);
  }
  KsSetupTemps tp;
  {
    KsRegion rg(ctx, KS_R_SETUP);
    KsCarver cv(ctx);
    ks_layout_setup(cv, tp, z, cub_cap);
    KS_TRY(cv.st);
  }
  double *xyz = ctx->xyz;
  uint8_t *dir = tp.dir;
  int32_t *flag = tp.flag, *scan = tp.scan;
  unsigned long long *bad = tp.bad;
  void *cub_tmp = tp.cub;
  KS_CUDA(ctx, cudaMemcpyAsync(xyz, h_xyz, sizeof(double) * 3 * nn, cudaMemcpyHostToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(dir, h_dir, nn, cudaMemcpyHostToDevice, s));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->tets, h_tets, sizeof(int32_t) * 4 * nt, cudaMemcpyHostToDevice, s));
  KS_CUDA(ctx, cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));

  k_check_tets<<<ks_blocks(nt, T), T, 0, s>>>(ctx->tets, nt, nn, bad);
  KS_LAUNCHED(ctx);
  unsigned long long h_bad = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&h_bad, bad, sizeof h_bad, cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  if (h_bad != ~0ull) return ks_fail(ctx, KS_E_MESH, "tet %llu has a node index outside [0, %lld)", h_bad, (long long)nn);

  // --- free numbering (exclusive scan of non-Dirichlet flags) ---
  k_notdir<<<ks_blocks(nn, T), T, 0, s>>>(dir, nn, flag);
  KS_LAUNCHED(ctx);
  size_t tmp_bytes = cub_cap;
  KS_CUDA(ctx, cub::DeviceScan::ExclusiveSum(cub_tmp, tmp_bytes, flag, scan, (int)nn, s));
  ctx->launches++;
  int32_t last_scan = 0, last_flag = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&last_scan, scan + nn - 1, 4, cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaMemcpyAsync(&last_flag, flag + nn - 1, 4, cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  const int64_t nf = (int64_t)last_scan + last_flag;
  ctx->n_free = nf;
  if (nf != z.nf) return ks_fail(ctx, KS_E_CUDA, "free count %lld differs from the plan's %lld", (long long)nf, (long long)z.nf);
  k_free_numbering<<<ks_blocks(nn, T), T, 0, s>>>(dir, scan, nn, ctx->free_of_node, ctx->node_of_free);
  KS_LAUNCHED(ctx);

  // --- geometry ---
  double *grad = tp.grad;
  k_geometry<<<ks_blocks(nt, T), T, 0, s>>>(xyz, ctx->tets, nt, ctx->vol, grad, bad);
  KS_LAUNCHED(ctx);
  KS_CUDA(ctx, cudaMemcpyAsync(&h_bad, bad, sizeof h_bad, cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  if (h_bad != ~0ull) return ks_fail(ctx, KS_E_MESH, "tet %llu is inverted or degenerate (det <= 0)", h_bad);

  // --- pattern: sort + unique of (free row, free col) keys ---
  const int64_t nk = 16 * nt;
  uint64_t *keys = tp.keys, *keys_sorted = tp.keys_sorted, *uniq;
  int *n_sel = tp.n_sel;
  const uint64_t sentinel = (uint64_t)nf << 32;
  k_pair_keys<<<ks_blocks(nk, T), T, 0, s>>>(ctx->tets, ctx->free_of_node, nt, sentinel, keys);
  KS_LAUNCHED(ctx);
  const int end_bit = 32 + bitlen((uint64_t)nf);
  tmp_bytes = cub_cap;
  KS_CUDA(ctx, cub::DeviceRadixSort::SortKeys(cub_tmp, tmp_bytes, keys, keys_sorted, (int)nk, 0, end_bit, s));
  ctx->launches++;
  tmp_bytes = cub_cap;
  uniq = keys;  // reuse
  KS_CUDA(ctx, cub::DeviceSelect::Unique(cub_tmp, tmp_bytes, keys_sorted, uniq, n_sel, (int)nk, s));
  ctx->launches++;
  int h_nsel = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&h_nsel, n_sel, sizeof(int), cudaMemcpyDeviceToHost, s));
  uint64_t last_key = 0;
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  KS_CUDA(ctx, cudaMemcpyAsync(&last_key, uniq + h_nsel - 1, 8, cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  const int64_t nnz = (last_key == sentinel) ? h_nsel - 1 : h_nsel;
  ctx->nnz = nnz;
  if (nnz != z.nnz) return ks_fail(ctx, KS_E_CUDA, "nnz %lld differs from the plan's %lld", (long long)nnz, (long long)z.nnz);
  k_row_ptr<<<ks_blocks(nf + 1, T), T, 0, s>>>(uniq, nnz, nf, ctx->row_ptr);
  KS_LAUNCHED(ctx);
  k_cols<<<ks_blocks(nnz, T), T, 0, s>>>(uniq, nnz, ctx->col);
  KS_LAUNCHED(ctx);
  k_diag_pos<<<ks_blocks(nf, T), T, 0, s>>>(ctx->row_ptr, ctx->col, nf, ctx->diag_pos);
  KS_LAUNCHED(ctx);

  // --- scatter map and its inverse (stable sort of emap targets keeps ascending index order) ---
  uint32_t *ik = reinterpret_cast<uint32_t *>(keys_sorted);          // reuse 8-byte buffers as 2 x 4-byte
  uint32_t *ik_sorted = ik + nk;
  int32_t *iv = reinterpret_cast<int32_t *>(keys);
  int32_t *iv_sorted = iv + nk;
  k_emap<<<ks_blocks(nk, T), T, 0, s>>>(ctx->tets, ctx->free_of_node, ctx->row_ptr, ctx->col, nt, nnz, ctx->emap,
                                        ik, iv);
  KS_LAUNCHED(ctx);
  const int end_bit2 = bitlen((uint64_t)nnz);
  tmp_bytes = cub_cap;
  KS_CUDA(ctx, cub::DeviceRadixSort::SortPairs(cub_tmp, tmp_bytes, ik, ik_sorted, iv, iv_sorted, (int)nk, 0,
                                               end_bit2, s));
  ctx->launches++;
  k_inv_ptr<<<ks_blocks(nnz + 1, T), T, 0, s>>>(ik_sorted, nk, nnz, ctx->inv_ptr);
  KS_LAUNCHED(ctx);
  int32_t h_nc = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&h_nc, ctx->inv_ptr + nnz, 4, cudaMemcpyDeviceToHost, s));
  KS_CUDA(ctx, cudaStreamSynchronize(s));
  ctx->n_contrib = h_nc;
  if (h_nc != z.nc) return ks_fail(ctx, KS_E_CUDA, "contributions %d differ from the plan's %lld", h_nc, (long long)z.nc);
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->inv_idx, iv_sorted, sizeof(int32_t) * h_nc, cudaMemcpyDeviceToDevice, s));

  // --- K and M ---
  k_stiffness_mass<<<ks_blocks(nnz, T), T, 0, s>>>(ctx->inv_ptr, ctx->inv_idx, ctx->vol, grad, nnz, ctx->K, ctx->M);
  KS_LAUNCHED(ctx);
  KS_TRY(ks_sell_build(ctx, tp.sell_cnt, cub_tmp, cub_cap, z.sell_total));
  KS_TRY(ks_star_setup(ctx, tp.n_sel));
  KS_CUDA(ctx, cudaStreamSynchronize(s));  // the setup temporaries are not referenced after this point
  return KS_OK;
}
