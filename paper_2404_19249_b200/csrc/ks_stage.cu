// ks_stage.cu -- per-group tables for the S phase of the block PCG with the orbital block staged in shared
// memory (DESIGN.md §4.3 "staged S phase").
//
// The rows of the block PCG are cut into groups of GRP consecutive rows (GRP = 1024 / NP: one CTA step of the
// staged layout, 2 orbitals per lane). A group references a set of columns (its rows' CSR columns); sorted and
// cut into runs of consecutive indices it is what the CTA copies into shared memory with bulk (TMA) copies
// before the group's SpMM: each run is rows [start, start + len) of p, contiguous in memory. For the Kuhn
// meshes of the configs a 64-row group needs 7 runs of ~66 rows (the stencil's offset groups).
// Tables (device):
//   meta   [n_groups] records of KS_META_BYTES: {n_runs, rows, -, -, (start, len) x KS_STAGE_RMAX}; n_runs = 0
//          marks a group that does not fit (more runs or rows than the caps) and is gathered from global memory;
//   slcol  [sell_total] u16: for every sliced-ELL slot, the position of its column in the group's staged rows
//          (padding slots: the own row);
//   dlc    [n_free] u16: the position of the row itself (for p_i in p.q).
#include <algorithm>
#include <vector>

#include "ks_internal.cuh"

ks_status ks_stage_build(ks_ctx *ctx, int NP, int max_rows) {
  if (ctx->stage_np == NP) return KS_OK;
  const int64_t n = ctx->n_free, nnz = ctx->nnz;
  const int GRP = 1024 / NP;
  const int64_t ng = (n + GRP - 1) / GRP;
  std::vector<int32_t> rp(n + 1), col(nnz), sptr(ctx->n_slices + 1);
  KS_CUDA(ctx, cudaMemcpyAsync(rp.data(), ctx->row_ptr, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, ctx->stream));
  KS_CUDA(ctx, cudaMemcpyAsync(col.data(), ctx->col, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, ctx->stream));
  KS_CUDA(ctx, cudaMemcpyAsync(sptr.data(), ctx->sell_ptr, sizeof(int32_t) * (ctx->n_slices + 1), cudaMemcpyDeviceToHost,
                               ctx->stream));
  KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  std::vector<int32_t> meta(ng * (KS_META_BYTES / 4), 0);
  std::vector<uint16_t> slcol(ctx->sell_total, 0), dlc(n, 0);
  std::vector<int32_t> u;
  int cap = 0;
  int64_t staged = 0;
  for (int64_t g = 0; g < ng; g++) {
    const int64_t r0 = g * GRP, r1 = std::min(n, r0 + GRP);
    u.assign(col.begin() + rp[r0], col.begin() + rp[r1]);
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    int nruns = 0;
    for (size_t k = 0; k < u.size(); k++)
      if (k == 0 || u[k] != u[k - 1] + 1) nruns++;
    int32_t *m = &meta[g * (KS_META_BYTES / 4)];
    if (nruns > KS_STAGE_RMAX || (int)u.size() > max_rows || u.size() >= 65535) continue;   // gathered path
    m[0] = nruns;
    m[1] = (int32_t)u.size();
    int r = -1;
    for (size_t k = 0; k < u.size(); k++) {
      if (k == 0 || u[k] != u[k - 1] + 1) {
        r++;
        m[4 + 2 * r] = u[k];
        m[4 + 2 * r + 1] = 0;
      }
      m[4 + 2 * r + 1]++;
    }
    cap = std::max(cap, (int)u.size());
    staged++;
    for (int64_t i = r0; i < r1; i++) {
      const int64_t s = i / KS_SELL_C;
      const int32_t b = sptr[s], K = (sptr[s + 1] - b) / KS_SELL_C;
      const int32_t len = rp[i + 1] - rp[i];
      const int64_t base = b + (i % KS_SELL_C) * 4;
      const uint16_t own = (uint16_t)(std::lower_bound(u.begin(), u.end(), (int32_t)i) - u.begin());
      dlc[i] = own;
      for (int k = 0; k < K; k++) {
        uint16_t l = own;
        if (k < len) l = (uint16_t)(std::lower_bound(u.begin(), u.end(), col[rp[i] + k]) - u.begin());
        slcol[base + (k >> 2) * (4 * KS_SELL_C) + (k & 3)] = l;
      }
    }
  }
  ks_free_t(ctx, ctx->stage_meta);
  ks_free_t(ctx, ctx->stage_slcol);
  ks_free_t(ctx, ctx->stage_dlc);
  KS_TRY(ks_alloc_t(ctx, &ctx->stage_meta, (int64_t)meta.size(), "stage meta"));
  KS_TRY(ks_alloc_t(ctx, &ctx->stage_slcol, (int64_t)slcol.size(), "stage local cols"));
  KS_TRY(ks_alloc_t(ctx, &ctx->stage_dlc, n, "stage diagonal local"));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->stage_meta, meta.data(), sizeof(int32_t) * meta.size(), cudaMemcpyHostToDevice,
                               ctx->stream));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->stage_slcol, slcol.data(), sizeof(uint16_t) * slcol.size(), cudaMemcpyHostToDevice,
                               ctx->stream));
  KS_CUDA(ctx, cudaMemcpyAsync(ctx->stage_dlc, dlc.data(), sizeof(uint16_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->stage_np = NP;
  ctx->stage_cap = cap;
  ctx->stage_groups = ng;
  ctx->stage_staged = staged;
  return KS_OK;
}
