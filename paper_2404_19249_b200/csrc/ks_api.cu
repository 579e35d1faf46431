// ks_api.cu -- C-ABI entry points of libks (include/ks.h): argument validation, context lifetime,
// status latching, dispatch to the kernels in ks_setup.cu / ks_assemble.cu / ks_pcg.cu / ks_project.cu.
#include <stdarg.h>

#include <mutex>

#include "ks_internal.cuh"

static std::mutex g_err_mu;
static std::string g_create_err;

const char *ks_status_name(ks_status s) {
  switch (s) {
    case KS_OK: return "KS_OK";
    case KS_E_ARG: return "KS_E_ARG";
    case KS_E_MESH: return "KS_E_MESH";
    case KS_E_NONFINITE: return "KS_E_NONFINITE";
    case KS_E_NOT_SPD: return "KS_E_NOT_SPD";
    case KS_E_NOT_CONVERGED: return "KS_E_NOT_CONVERGED";
    case KS_E_CUDA: return "KS_E_CUDA";
    case KS_E_NOMEM: return "KS_E_NOMEM";
    case KS_E_STATE: return "KS_E_STATE";
    case KS_E_RANK: return "KS_E_RANK";
  }
  return "KS_E_?";
}

ks_status ks_fail(ks_ctx *ctx, ks_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  std::string msg = std::string(ks_status_name(s)) + ": " + buf;
  if (ctx) ctx->err = msg;
  return s;
}

ks_status ks_cuda_check(ks_ctx *ctx, cudaError_t e, const char *what) {
  if (e == cudaSuccess) return KS_OK;
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return ks_fail(ctx, KS_E_NOMEM, "%s: %s", what, cudaGetErrorString(e));
  }
  return ks_fail(ctx, KS_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

ks_status ks_alloc(ks_ctx *ctx, void **ptr, size_t bytes, const char *what) {
  *ptr = nullptr;
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *ptr = nullptr;
    return ks_fail(ctx, KS_E_NOMEM, "cudaMalloc(%zu bytes) for %s: %s", bytes, what, cudaGetErrorString(e));
  }
  ctx->bytes += bytes;
  ctx->allocs.push_back({*ptr, bytes});
  // zero-filled: padding tails past the logical ends (read by the bulk tile copies) stay defined
  e = cudaMemsetAsync(*ptr, 0, bytes, ctx->stream);
  if (e != cudaSuccess) return ks_cuda_check(ctx, e, "cudaMemsetAsync (new allocation)");
  return KS_OK;
}

void ks_free(ks_ctx *ctx, void *ptr) {
  if (!ptr) return;
  for (size_t k = 0; k < ctx->allocs.size(); k++)
    if (ctx->allocs[k].first == ptr) {
      ctx->bytes -= ctx->allocs[k].second;
      ctx->allocs.erase(ctx->allocs.begin() + k);
      break;
    }
  cudaFree(ptr);
}

static void free_all(ks_ctx *ctx) {
  ks_free_stream(ctx);
  ks_free_outer(ctx);
  for (auto &a : ctx->allocs) cudaFree(a.first);
  ctx->allocs.clear();
  ctx->bytes = 0;
}

extern "C" {

int ks_abi_version(void) { return KS_ABI_VERSION; }

#define KS_STR2(x) #x
#define KS_STR(x) KS_STR2(x)
const char *ks_build_info(void) {
  return "libks sm_100a fp64 (nvcc " KS_STR(__CUDACC_VER_MAJOR__) "." KS_STR(__CUDACC_VER_MINOR__) ") " __DATE__;
}

ks_status ks_create(int64_t n_nodes, const double *h_xyz, int64_t n_tets, const int32_t *h_tets,
                    const uint8_t *h_dirichlet, void *stream, ks_ctx **out) {
  if (!out) return KS_E_ARG;
  *out = nullptr;
  auto set_err = [](const std::string &m) {
    std::lock_guard<std::mutex> g(g_err_mu);
    g_create_err = m;
  };
  if (n_nodes < 4 || n_tets < 1 || !h_xyz || !h_tets || !h_dirichlet) {
    set_err("KS_E_ARG: ks_create needs n_nodes >= 4, n_tets >= 1 and non-null host arrays");
    return KS_E_ARG;
  }
  if (n_nodes > 0x7fffffffLL || 16 * n_tets > 0x7fffffffLL) {
    set_err("KS_E_ARG: mesh too large for int32 indexing (n_nodes < 2^31, 16 n_tets < 2^31)");
    return KS_E_ARG;
  }
  ks_ctx *ctx = new ks_ctx();
  ctx->stream = (cudaStream_t)stream;
  ctx->n_nodes = n_nodes;
  ctx->n_tets = n_tets;
  ks_status st = KS_OK;
  do {
    if ((st = ks_cuda_check(ctx, cudaGetDevice(&ctx->device), "cudaGetDevice")) != KS_OK) break;
    if ((st = ks_cuda_check(ctx, cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, ctx->device),
                            "cudaDeviceGetAttribute")) != KS_OK)
      break;
    int coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device);
    if (!coop) { st = ks_fail(ctx, KS_E_CUDA, "device does not support cooperative launch"); break; }
    if ((st = ks_alloc_t(ctx, &ctx->d_flags, 1, "flags")) != KS_OK) break;
    if ((st = ks_alloc_t(ctx, &ctx->d_block_iters, 1, "block iters")) != KS_OK) break;
    if ((st = ks_alloc_t(ctx, &ctx->barrier, 1, "barrier")) != KS_OK) break;
    if ((st = ks_cuda_check(ctx, cudaMemsetAsync(ctx->d_flags, 0, 4, ctx->stream), "memset")) != KS_OK) break;
    if ((st = ks_cuda_check(ctx, cudaMemsetAsync(ctx->d_block_iters, 0, 4, ctx->stream), "memset")) != KS_OK) break;
    st = ks_setup_mesh(ctx, h_xyz, h_tets, h_dirichlet);
  } while (0);
  if (st != KS_OK) {
    set_err(ctx->err);
    free_all(ctx);
    delete ctx;
    return st;
  }
  *out = ctx;
  return KS_OK;
}

void ks_destroy(ks_ctx *ctx) {
  if (!ctx) return;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  else cudaDeviceSynchronize();
  free_all(ctx);
  delete ctx;
}

ks_status ks_set_stream(ks_ctx *ctx, void *stream) {
  if (!ctx) return KS_E_ARG;
  ctx->stream = (cudaStream_t)stream;
  return KS_OK;
}

ks_status ks_pattern(const ks_ctx *ctx, int64_t *n_free, int64_t *nnz, const int32_t **d_row_ptr,
                     const int32_t **d_col, const int32_t **d_emap, const int32_t **d_free_of_node,
                     const int32_t **d_inv_ptr, const int32_t **d_inv_idx) {
  if (!ctx) return KS_E_ARG;
  if (n_free) *n_free = ctx->n_free;
  if (nnz) *nnz = ctx->nnz;
  if (d_row_ptr) *d_row_ptr = ctx->row_ptr;
  if (d_col) *d_col = ctx->col;
  if (d_emap) *d_emap = ctx->emap;
  if (d_free_of_node) *d_free_of_node = ctx->free_of_node;
  if (d_inv_ptr) *d_inv_ptr = ctx->inv_ptr;
  if (d_inv_idx) *d_inv_idx = ctx->inv_idx;
  return KS_OK;
}

ks_status ks_values(const ks_ctx *ctx, const double **d_K, const double **d_M, const double **d_MV,
                    const double **d_H, const double **d_A, const double **d_diag) {
  if (!ctx) return KS_E_ARG;
  if (d_K) *d_K = ctx->K;
  if (d_M) *d_M = ctx->M;
  if ((d_MV || d_H || d_A || d_diag) && !ctx->assembled)
    return ks_fail(const_cast<ks_ctx *>(ctx), KS_E_STATE, "ks_values: call ks_assemble_veff first");
  if (d_MV || d_H || d_A) {
    ks_status st = ks_materialize_views(const_cast<ks_ctx *>(ctx));
    if (st != KS_OK) return st;
  }
  if (d_MV) *d_MV = ctx->MV;
  if (d_H) *d_H = ctx->H;
  if (d_A) *d_A = ctx->A;
  if (d_diag) *d_diag = ctx->diag;
  return KS_OK;
}

ks_status ks_assemble_veff(ks_ctx *ctx, const double *d_veff, double mu) {
  if (!ctx) return KS_E_ARG;
  if (!d_veff) return ks_fail(ctx, KS_E_ARG, "ks_assemble_veff: d_veff is NULL");
  if (!(mu >= 0.0) || !isfinite(mu)) return ks_fail(ctx, KS_E_ARG, "ks_assemble_veff: mu = %g must be finite and >= 0", mu);
  return ks_assemble_impl(ctx, d_veff, mu);
}

static const double *op_values(const ks_ctx *ctx, ks_op op) {
  switch (op) {
    case KS_OP_K: return ctx->K;
    case KS_OP_M: return ctx->M;
    case KS_OP_MV: return ctx->assembled ? ctx->MV : nullptr;
    case KS_OP_H: return ctx->assembled ? ctx->H : nullptr;
    case KS_OP_A: return ctx->assembled ? ctx->A : nullptr;
  }
  return nullptr;
}

ks_status ks_spmm(ks_ctx *ctx, ks_op op, int32_t N, const double *d_X, double *d_Y) {
  if (!ctx) return KS_E_ARG;
  if (N < 1 || N > KS_MAX_N) return ks_fail(ctx, KS_E_ARG, "ks_spmm: N = %d outside [1, %d]", N, KS_MAX_N);
  if (!d_X || !d_Y || d_X == d_Y) return ks_fail(ctx, KS_E_ARG, "ks_spmm: X, Y must be distinct non-null");
  if (((uintptr_t)d_X & 7) || ((uintptr_t)d_Y & 7)) return ks_fail(ctx, KS_E_ARG, "ks_spmm: X, Y must be 8-byte aligned");
  const double *v = op_values(ctx, op);
  if (!v) return ks_fail(ctx, KS_E_STATE, "ks_spmm: operator %d not assembled", (int)op);
  if (op == KS_OP_MV || op == KS_OP_H) KS_TRY(ks_materialize_views(ctx));
  return ks_spmm_impl(ctx, op, v, N, d_X, d_Y);
}

ks_status ks_block_solve(ks_ctx *ctx, int32_t N, const double *d_lambda, const double *d_U, double *d_Ut,
                         double tol, int32_t max_iter, int32_t *d_iters, double *d_relres) {
  if (!ctx) return KS_E_ARG;
  if (N < 1 || N > KS_MAX_N) return ks_fail(ctx, KS_E_ARG, "ks_block_solve: N = %d outside [1, %d]", N, KS_MAX_N);
  if (!d_lambda || !d_U || !d_Ut) return ks_fail(ctx, KS_E_ARG, "ks_block_solve: null lambda/U/Ut");
  if (d_U == d_Ut) return ks_fail(ctx, KS_E_ARG, "ks_block_solve: U and Ut must not alias");
  if (((uintptr_t)d_U & 7) || ((uintptr_t)d_Ut & 7)) return ks_fail(ctx, KS_E_ARG, "ks_block_solve: U/Ut must be 8-byte aligned");
  if (!(tol > 0.0) || !isfinite(tol)) return ks_fail(ctx, KS_E_ARG, "ks_block_solve: tol = %g must be > 0", tol);
  if (max_iter < 1) return ks_fail(ctx, KS_E_ARG, "ks_block_solve: max_iter = %d must be >= 1", max_iter);
  if (!ctx->assembled) return ks_fail(ctx, KS_E_STATE, "ks_block_solve: call ks_assemble_veff first");
  return ks_solve_impl(ctx, N, d_lambda, d_U, d_Ut, tol, max_iter, d_iters, d_relres);
}

ks_status ks_last_iterations(ks_ctx *ctx, int32_t *h_block_iters) {
  if (!ctx || !h_block_iters) return KS_E_ARG;
  KS_CUDA(ctx, cudaMemcpyAsync(h_block_iters, ctx->d_block_iters, 4, cudaMemcpyDeviceToHost, ctx->stream));
  KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return KS_OK;
}

ks_status ks_pencil_eig(ks_ctx *ctx, int64_t D, int32_t k, const double *d_FA, const double *d_FB, double *d_evals,
                        double *d_evecs) {
  if (!ctx) return KS_E_ARG;
  if (D < 1 || k < 1 || k > D || D > 65536) return ks_fail(ctx, KS_E_ARG, "ks_pencil_eig: need 1 <= k <= D <= 65536");
  if (!d_FA || !d_FB || !d_evals || !d_evecs) return ks_fail(ctx, KS_E_ARG, "ks_pencil_eig: null pointer");
  return ks_pencil_eig_impl(ctx, D, k, d_FA, d_FB, d_evals, d_evecs);
}

ks_status ks_lift(ks_ctx *ctx, int32_t N, const double *d_Ut, int32_t k, const double *d_Y, double *d_Unew) {
  if (!ctx) return KS_E_ARG;
  if (N < 1 || N > KS_MAX_N || k < 1 || !d_Ut || !d_Y || !d_Unew || d_Ut == d_Unew)
    return ks_fail(ctx, KS_E_ARG, "ks_lift: bad arguments");
  if (ctx->n_H < 1) return ks_fail(ctx, KS_E_STATE, "ks_lift: call ks_set_coarse first");
  return ks_lift_impl(ctx, N, d_Ut, k, d_Y, d_Unew);
}

ks_status ks_augmented_solve(ks_ctx *ctx, int32_t N, double *d_lambda, double *d_U, double tol_eig, int32_t max_outer,
                             double tol_bvp, int32_t max_iter_bvp, int32_t *h_outer, double *h_history) {
  if (!ctx) return KS_E_ARG;
  if (N < 1 || N > KS_MAX_N || !d_lambda || !d_U || !(tol_eig >= 0.0) || max_outer < 1 || !(tol_bvp > 0.0) ||
      max_iter_bvp < 1)
    return ks_fail(ctx, KS_E_ARG, "ks_augmented_solve: bad arguments");
  if (!ctx->assembled) return ks_fail(ctx, KS_E_STATE, "ks_augmented_solve: call ks_assemble_veff first");
  if (ctx->n_H < 1) return ks_fail(ctx, KS_E_STATE, "ks_augmented_solve: call ks_set_coarse first");
  return ks_augmented_solve_impl(ctx, N, d_lambda, d_U, tol_eig, max_outer, tol_bvp, max_iter_bvp, h_outer, h_history);
}

ks_status ks_interpolation(ks_ctx *ctx, int64_t n_c, const double *h_xyz_c, int64_t m_c, const int32_t *h_tets_c,
                           const uint8_t *h_dirichlet_c, int32_t *d_P_row_ptr, int32_t *d_P_col, double *d_P_val,
                           int64_t *h_n_H, int64_t *h_p_nnz) {
  if (!ctx) return KS_E_ARG;
  if (n_c < 4 || m_c < 1 || n_c > 0x7fffffffLL || m_c > 0x7fffffffLL || !h_xyz_c || !h_tets_c || !h_dirichlet_c ||
      !d_P_row_ptr || !d_P_col || !d_P_val || !h_n_H || !h_p_nnz)
    return ks_fail(ctx, KS_E_ARG, "ks_interpolation: bad arguments");
  return ks_interpolation_impl(ctx, n_c, h_xyz_c, m_c, h_tets_c, h_dirichlet_c, d_P_row_ptr, d_P_col, d_P_val,
                               h_n_H, h_p_nnz);
}

ks_status ks_density(ks_ctx *ctx, int32_t N, const double *d_U, double f, double *d_rho) {
  if (!ctx) return KS_E_ARG;
  if (N < 1 || N > KS_MAX_N || !d_U || !d_rho || !(f >= 0.0)) return ks_fail(ctx, KS_E_ARG, "ks_density: bad arguments");
  return ks_density_impl(ctx, N, d_U, f, d_rho);
}

ks_status ks_vxc(ks_ctx *ctx, const double *d_rho, double *d_vxc, double *d_eps) {
  if (!ctx) return KS_E_ARG;
  if (!d_rho || !d_vxc) return ks_fail(ctx, KS_E_ARG, "ks_vxc: null pointer");
  return ks_vxc_impl(ctx, d_rho, d_vxc, d_eps);
}

ks_status ks_hartree(ks_ctx *ctx, const double *d_rho, double tol, int32_t max_iter, double *d_vh, int32_t warm,
                     double *h_mom, int32_t *h_iters) {
  if (!ctx) return KS_E_ARG;
  if (!d_rho || !d_vh || !(tol > 0.0) || max_iter < 1) return ks_fail(ctx, KS_E_ARG, "ks_hartree: bad arguments");
  return ks_hartree_impl(ctx, d_rho, tol, max_iter, d_vh, warm, h_mom, h_iters);
}

ks_status ks_scf_solve(ks_ctx *ctx, int32_t N, const double *d_vext, double f, double mu, double *d_lambda,
                       double *d_U, double tol, int32_t max_outer, int32_t inner, double inner_tol, double beta,
                       int32_t depth, double bvp_tol, double hartree_tol, int32_t *h_outer, int32_t *h_inner,
                       double *h_dres, double *h_lams) {
  if (!ctx) return KS_E_ARG;
  if (N < 1 || N > KS_MAX_N || !d_vext || !d_lambda || !d_U || !(f >= 0.0) || !(mu >= 0.0) || !(tol > 0.0) ||
      max_outer < 1 || inner < 1 || !(inner_tol > 0.0) || !(beta > 0.0 && beta <= 1.0) || depth < 1 || depth > 7 ||
      !(bvp_tol > 0.0) || !(hartree_tol > 0.0))
    return ks_fail(ctx, KS_E_ARG, "ks_scf_solve: bad arguments");
  if (ctx->n_H < 1) return ks_fail(ctx, KS_E_STATE, "ks_scf_solve: call ks_set_coarse first");
  return ks_scf_solve_impl(ctx, N, d_vext, f, mu, d_lambda, d_U, tol, max_outer, inner, inner_tol, beta, depth,
                           bvp_tol, hartree_tol, h_outer, h_inner, h_dres, h_lams);
}

ks_status ks_step_submit(ks_ctx *ctx, int32_t N, const double *h_V, double mu, const double *h_lambda,
                         const double *h_U, double tol, int32_t max_iter, double *h_FA, double *h_FB) {
  if (!ctx) return KS_E_ARG;
  if (N < 1 || N > KS_MAX_N || !h_V || !h_lambda || !h_U || !h_FA || !h_FB || !(tol > 0.0) || max_iter < 1 ||
      !(mu >= 0.0))
    return ks_fail(ctx, KS_E_ARG, "ks_step_submit: bad arguments");
  if (ctx->n_H < 1) return ks_fail(ctx, KS_E_STATE, "ks_step_submit: call ks_set_coarse first");
  return ks_step_submit_impl(ctx, N, h_V, mu, h_lambda, h_U, tol, max_iter, h_FA, h_FB);
}

ks_status ks_step_wait(ks_ctx *ctx) {
  if (!ctx) return KS_E_ARG;
  return ks_step_wait_impl(ctx);
}

ks_status ks_solve_trace(ks_ctx *ctx, int32_t cap, uint64_t *h_ns, int32_t *h_count) {
  if (!ctx || !h_count || (cap > 0 && !h_ns)) return KS_E_ARG;
  *h_count = 0;
  if (!ctx->trace) return KS_OK;
  int n = 0;
  KS_CUDA(ctx, cudaMemcpyAsync(&n, ctx->trace_count, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (n > cap) n = cap;
  if (n > 0) {
    KS_CUDA(ctx, cudaMemcpyAsync(h_ns, ctx->trace, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, ctx->stream));
    KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  }
  *h_count = n;
  return KS_OK;
}

ks_status ks_true_residual(ks_ctx *ctx, int32_t N, const double *d_lambda, const double *d_U, const double *d_Ut,
                           double *d_relres) {
  if (!ctx) return KS_E_ARG;
  if (N < 1 || N > KS_MAX_N || !d_lambda || !d_U || !d_Ut || !d_relres)
    return ks_fail(ctx, KS_E_ARG, "ks_true_residual: bad arguments");
  if (!ctx->assembled) return ks_fail(ctx, KS_E_STATE, "ks_true_residual: call ks_assemble_veff first");
  return ks_true_residual_impl(ctx, N, d_lambda, d_U, d_Ut, d_relres);
}

ks_status ks_set_coarse(ks_ctx *ctx, int64_t n_H, const int32_t *d_P_row_ptr, const int32_t *d_P_col,
                        const double *d_P_val) {
  if (!ctx) return KS_E_ARG;
  if (n_H < 1 || n_H > 0x7fffffffLL) return ks_fail(ctx, KS_E_ARG, "ks_set_coarse: n_H = %lld", (long long)n_H);
  if (!d_P_row_ptr || !d_P_col || !d_P_val) return ks_fail(ctx, KS_E_ARG, "ks_set_coarse: null P arrays");
  ks_status st = ks_set_coarse_impl(ctx, n_H, d_P_row_ptr, d_P_col, d_P_val);
  if (st != KS_OK) ctx->n_H = 0;
  return st;
}

ks_status ks_project_augmented(ks_ctx *ctx, int32_t N, const double *d_Ut, double *d_FA, double *d_FB) {
  if (!ctx) return KS_E_ARG;
  if (N < 1 || N > KS_MAX_N) return ks_fail(ctx, KS_E_ARG, "ks_project_augmented: N = %d outside [1, %d]", N, KS_MAX_N);
  if (!d_Ut || !d_FA || !d_FB || d_FA == d_FB) return ks_fail(ctx, KS_E_ARG, "ks_project_augmented: bad pointers");
  if (!ctx->assembled) return ks_fail(ctx, KS_E_STATE, "ks_project_augmented: call ks_assemble_veff first");
  if (ctx->n_H < 1) return ks_fail(ctx, KS_E_STATE, "ks_project_augmented: call ks_set_coarse first");
  return ks_project_impl(ctx, N, d_Ut, d_FA, d_FB);
}

ks_status ks_memory_bytes(const ks_ctx *ctx, size_t *bytes) {
  if (!ctx || !bytes) return KS_E_ARG;
  *bytes = ctx->bytes;
  return KS_OK;
}

ks_status ks_launch_count(const ks_ctx *ctx, int64_t *count) {
  if (!ctx || !count) return KS_E_ARG;
  *count = ctx->launches;
  return KS_OK;
}

ks_status ks_sync(ks_ctx *ctx) {
  if (!ctx) return KS_E_ARG;
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return ks_cuda_check(ctx, e, "cudaStreamSynchronize");
  unsigned f = 0;
  KS_CUDA(ctx, cudaMemcpy(&f, ctx->d_flags, 4, cudaMemcpyDeviceToHost));
  KS_CUDA(ctx, cudaMemset(ctx->d_flags, 0, 4));
  if (f & KSF_NONFINITE) return ks_fail(ctx, KS_E_NONFINITE, "non-finite value met (V_eff or a solver reduction)");
  if (f & KSF_NOT_SPD) return ks_fail(ctx, KS_E_NOT_SPD, "p.Ap <= 0 in some column: A = H + mu M not SPD (mu too small)");
  if (f & KSF_NOT_CONVERGED) return ks_fail(ctx, KS_E_NOT_CONVERGED, "max_iter reached with columns above tolerance");
  return KS_OK;
}

const char *ks_last_error(const ks_ctx *ctx) {
  if (ctx) return ctx->err.c_str();
  std::lock_guard<std::mutex> g(g_err_mu);
  return g_create_err.c_str();
}

}  // extern "C"
