// ks_plan.cu -- memory plans of libks (include/ks.h, "Memory"): the caller allocates every device byte the
// library uses; the library carves it with a bump allocator (ks_alloc, ks_api.cu) and never calls
// cudaMalloc / cudaFree.
//
// The sizes of the setup products (n_free, nnz, contributions, sliced-ELL entries) are counted on the host
// from the mesh (the same definitions the device setup computes); every region is
// then the sum of its allocations, listed once in a layout function that serves both the size query (KsSizer)
// and the allocation (KsCarver), so plan and use cannot drift apart.
#include <cub/cub.cuh>

#include <algorithm>
#include <thread>
#include <vector>

#include "ks_internal.cuh"
#include "ks_layout.cuh"

// ---------------------------------------------------------------------------------------------
// host count of the pattern sizes (threads over row ranges, one "last seen" stamp array per thread)
// ---------------------------------------------------------------------------------------------
ks_status ks_count_mesh(int64_t nn, const int32_t *tets, int64_t nt, const uint8_t *dir, KsMeshSizes *z,
                        std::string *err) {
  std::vector<int32_t> fidx(nn);
  int64_t nf = 0;
  for (int64_t v = 0; v < nn; v++) fidx[v] = dir[v] ? -1 : (int32_t)nf++;
  if (nf < 1) {
    *err = "KS_E_MESH: mesh has no free (non-Dirichlet) node";
    return KS_E_MESH;
  }
  // incidence of free nodes: tets containing each free node
  std::vector<int64_t> start(nf + 1, 0);
  int64_t nc = 0;
  for (int64_t t = 0; t < nt; t++) {
    int f = 0;
    for (int a = 0; a < 4; a++) {
      const int32_t v = tets[4 * t + a];
      if (v < 0 || v >= nn) {
        *err = "KS_E_MESH: tet " + std::to_string(t) + " has a node index outside [0, " + std::to_string(nn) + ")";
        return KS_E_MESH;
      }
      if (fidx[v] >= 0) {
        start[fidx[v] + 1]++;
        f++;
      }
    }
    nc += (int64_t)f * f;
  }
  for (int64_t i = 0; i < nf; i++) start[i + 1] += start[i];
  std::vector<int32_t> inc(start[nf]);
  {
    std::vector<int64_t> pos(start.begin(), start.end() - 1);
    for (int64_t t = 0; t < nt; t++)
      for (int a = 0; a < 4; a++) {
        const int32_t f = fidx[tets[4 * t + a]];
        if (f >= 0) inc[pos[f]++] = (int32_t)t;
      }
  }
  std::vector<int32_t> len(nf);
  const int nth = (int)std::max<unsigned>(1, std::min<unsigned>(16, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (int w = 0; w < nth; w++)
    th.emplace_back([&, w]() {
      std::vector<int32_t> stamp(nf, -1);
      for (int64_t i = w; i < nf; i += nth) {
        int32_t c = 0;
        for (int64_t k = start[i]; k < start[i + 1]; k++) {
          const int32_t *tv = tets + 4 * (int64_t)inc[k];
          for (int a = 0; a < 4; a++) {
            const int32_t f = fidx[tv[a]];
            if (f >= 0 && stamp[f] != (int32_t)i) {
              stamp[f] = (int32_t)i;
              c++;
            }
          }
        }
        len[i] = c;
      }
    });
  for (auto &x : th) x.join();
  int64_t nnz = 0;
  for (int64_t i = 0; i < nf; i++) nnz += len[i];
  const int64_t ns = (nf + KS_SELL_C - 1) / KS_SELL_C;
  int64_t sell = 0;
  for (int64_t s = 0; s < ns; s++) {
    int m = 0;
    for (int64_t i = s * KS_SELL_C; i < std::min<int64_t>((s + 1) * KS_SELL_C, nf); i++) m = std::max(m, len[i]);
    sell += (int64_t)KS_SELL_C * std::max(4, (m + 3) & ~3);
  }
  if (nnz > 0x7fffffffLL || sell > 0x7fffffffLL || nc > 0x7fffffffLL) {
    *err = "KS_E_ARG: pattern exceeds int32 indexing";
    return KS_E_ARG;
  }
  z->nn = nn;
  z->nt = nt;
  z->nf = nf;
  z->nnz = nnz;
  z->nc = nc;
  z->ns = ns;
  z->sell_total = sell;
  return KS_OK;
}

static int bitlen64(uint64_t x) {
  int b = 0;
  while (x) { b++; x >>= 1; }
  return b;
}

// CUB temporary storage of the setup's scans / sorts (the same calls as ks_setup.cu, ks_sell.cu)
ks_status ks_setup_cub_bytes(const KsMeshSizes &z, size_t *bytes) {
  const int64_t nk = 16 * z.nt;
  size_t m = 0, b = 0;
  int32_t *i32 = nullptr;
  uint64_t *u64 = nullptr;
  uint32_t *u32 = nullptr;
  int *ip = nullptr;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, b, i32, i32, (int)z.nn);
  m = std::max(m, b);
  if (e == cudaSuccess) e = cub::DeviceRadixSort::SortKeys(nullptr, b, u64, u64, (int)nk, 0, 32 + bitlen64(z.nf));
  m = std::max(m, b);
  if (e == cudaSuccess) e = cub::DeviceSelect::Unique(nullptr, b, u64, u64, ip, (int)nk);
  m = std::max(m, b);
  if (e == cudaSuccess) e = cub::DeviceRadixSort::SortPairs(nullptr, b, u32, u32, i32, i32, (int)nk, 0, bitlen64(z.nnz));
  m = std::max(m, b);
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(nullptr, b, i32, i32, (int)(z.ns + 1));
  m = std::max(m, b);
  *bytes = m;
  return e == cudaSuccess ? KS_OK : KS_E_CUDA;
}

// CUB temporary storage of ks_set_coarse's sorts / scans for n_free rows (n_items <= n_free)
ks_status ks_coarse_cub_bytes(int64_t nf, size_t *bytes) {
  size_t m = 0, b = 0;
  uint64_t *u64 = nullptr;
  int32_t *i32 = nullptr;
  int *ip = nullptr;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, b, u64, u64, i32, i32, (int)nf, 0, 64);
  m = std::max(m, b);
  if (e == cudaSuccess) e = cub::DeviceScan::InclusiveSum(nullptr, b, i32, i32, (int)nf);
  m = std::max(m, b);
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(nullptr, b, i32, i32, (int)(nf + 1));
  m = std::max(m, b);
  // item slices of the item-ordered sliced-ELL copy: at most n_items + n_free / 8 <= 9 n_free / 8 (+ 1)
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(nullptr, b, i32, i32, (int)(nf + (nf + 7) / 8 + 1));
  m = std::max(m, b);
  if (e == cudaSuccess) e = cub::DeviceReduce::Max(nullptr, b, i32, ip, (int)nf);
  m = std::max(m, b);
  if (e == cudaSuccess) e = cub::DeviceRadixSort::SortPairs(nullptr, b, i32, i32, i32, i32, (int)(4 * nf), 0, 32);
  m = std::max(m, b);
  *bytes = m;
  return e == cudaSuccess ? KS_OK : KS_E_CUDA;
}

int ks_pow2_at_least(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

ks_status ks_plan_sizes(const KsMeshSizes &z, int max_N, int sm_count, size_t *persist, size_t *work,
                        size_t *setup) {
  ks_ctx tmp;   // host struct only: the layouts take the addresses of its pointer fields
  KsSizer a;
  ks_layout_persist(a, &tmp, z);
  *persist = a.bytes;
  size_t cub_setup = 0, cub_coarse = 0;
  KS_TRY(ks_setup_cub_bytes(z, &cub_setup));
  KS_TRY(ks_coarse_cub_bytes(z.nf, &cub_coarse));
  KsSizer b;
  KsSetupTemps st;
  ks_layout_setup(b, st, z, cub_setup);
  *setup = b.bytes;
  KsSizer c;
  ks_layout_work(c, &tmp, z.nf, max_N, sm_count);
  c.bytes += ks_scratch_bound(z, max_N, sm_count, cub_coarse);
  *work = c.bytes;
  return KS_OK;
}
