// ks_api.cu -- C-ABI entry points of libks (include/ks.h): argument validation, context lifetime,
// status latching, dispatch to the kernels in ks_setup.cu / ks_assemble.cu / ks_pcg.cu / ks_project.cu.
#include <stdarg.h>

#include <mutex>

#include <nvtx3/nvToolsExt.h>

#include "ks_internal.cuh"
#include "ks_layout.cuh"

// NVTX range per ABI call (SURVEY.md §5 tracing): nsys / ncu timelines show each call by name. NVTX3 is
// header-only; without a tool attached a push/pop costs a few nanoseconds.
struct KsNvtx {
  explicit KsNvtx(const char *name) { nvtxRangePushA(name); }
  ~KsNvtx() { nvtxRangePop(); }
};
#define KS_RANGE() KsNvtx ks_nvtx_range_(__func__)

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
    case KS_E_WORKSPACE: return "KS_E_WORKSPACE";
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

static const char *region_name(int r) {
  static const char *names[KS_R_N] = {"persistent", "workspace", "setup", "coarse", "ext", "call"};
  return (r >= 0 && r < KS_R_N) ? names[r] : "?";
}

ks_status ks_alloc(ks_ctx *ctx, void **ptr, size_t bytes, const char *what) {
  *ptr = nullptr;
  ks_region &g = ctx->reg[ctx->region];
  const size_t need = ks_round(bytes > 0 ? bytes : 1);
  if (!g.base || g.off + need > g.cap)
    return ks_fail(ctx, KS_E_WORKSPACE, "%s region: %s needs %zu bytes at offset %zu of %zu (plan it with the "
                   "matching ks_*_plan call)", region_name(ctx->region), what, need, g.off, g.cap);
  *ptr = g.base + g.off;
  g.off += need;
  if (g.off > g.peak) g.peak = g.off;
  // zero-filled: padding tails past the logical ends (read by the vector and bulk copies) stay defined
  cudaError_t e = cudaMemsetAsync(*ptr, 0, bytes > 0 ? bytes : 1, ctx->stream);
  if (e != cudaSuccess) return ks_cuda_check(ctx, e, "cudaMemsetAsync (new allocation)");
  return KS_OK;
}

static ks_status bind_region(ks_ctx *ctx, int r, void *base, size_t bytes, const char *what) {
  if (((uintptr_t)base & (KS_ALIGN - 1)) != 0)
    return ks_fail(ctx, KS_E_ARG, "%s: device pointer must be %d-byte aligned", what, KS_ALIGN);
  ctx->reg[r].base = (uint8_t *)base;
  ctx->reg[r].cap = base ? bytes : 0;
  ctx->reg[r].off = 0;
  ctx->reg[r].peak = 0;
  return KS_OK;
}

static void free_all(ks_ctx *ctx) {
  ks_free_stream(ctx);
  ks_free_outer(ctx);
}

extern "C" {

int ks_abi_version(void) { return KS_ABI_VERSION; }

#define KS_STR2(x) #x
#define KS_STR(x) KS_STR2(x)
const char *ks_build_info(void) {
  return "libks sm_100a fp64 (nvcc " KS_STR(__CUDACC_VER_MAJOR__) "." KS_STR(__CUDACC_VER_MINOR__) ") " __DATE__;
}

static void set_create_err(const std::string &m) {
  std::lock_guard<std::mutex> g(g_err_mu);
  g_create_err = m;
}

static ks_status check_mesh_args(int64_t n_nodes, const double *h_xyz, int64_t n_tets, const int32_t *h_tets,
                                 const uint8_t *h_dirichlet, int32_t max_N) {
  if (n_nodes < 4 || n_tets < 1 || !h_xyz || !h_tets || !h_dirichlet) {
    set_create_err("KS_E_ARG: needs n_nodes >= 4, n_tets >= 1 and non-null host arrays");
    return KS_E_ARG;
  }
  if (n_nodes > 0x7fffffffLL || 16 * n_tets > 0x7fffffffLL) {
    set_create_err("KS_E_ARG: mesh too large for int32 indexing (n_nodes < 2^31, 16 n_tets < 2^31)");
    return KS_E_ARG;
  }
  if (max_N < 1 || max_N > KS_MAX_N) {
    set_create_err("KS_E_ARG: max_N must be in [1, 64]");
    return KS_E_ARG;
  }
  return KS_OK;
}

static int device_sm_count() {
  int dev = 0, sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return sm;
}

ks_status ks_plan(int64_t n_nodes, const double *h_xyz, int64_t n_tets, const int32_t *h_tets,
                  const uint8_t *h_dirichlet, int32_t max_N, size_t *persistent_bytes, size_t *workspace_bytes,
                  size_t *setup_bytes) {
  KS_RANGE();
  KS_TRY(check_mesh_args(n_nodes, h_xyz, n_tets, h_tets, h_dirichlet, max_N));
  if (!persistent_bytes || !workspace_bytes || !setup_bytes) {
    set_create_err("KS_E_ARG: ks_plan needs non-null size outputs");
    return KS_E_ARG;
  }
  KsMeshSizes z;
  std::string err;
  ks_status st = ks_count_mesh(n_nodes, h_tets, n_tets, h_dirichlet, &z, &err);
  if (st != KS_OK) {
    set_create_err(err);
    return st;
  }
  const int sm = device_sm_count();
  if (sm < 1) {
    set_create_err("KS_E_CUDA: no CUDA device");
    return KS_E_CUDA;
  }
  st = ks_plan_sizes(z, max_N, sm, persistent_bytes, workspace_bytes, setup_bytes);
  if (st != KS_OK) set_create_err("KS_E_CUDA: CUB temporary-size query failed");
  return st;
}

ks_status ks_create(int64_t n_nodes, const double *h_xyz, int64_t n_tets, const int32_t *h_tets,
                    const uint8_t *h_dirichlet, int32_t max_N, void *d_persistent, size_t persistent_bytes,
                    void *d_workspace, size_t workspace_bytes, void *d_setup, size_t setup_bytes, void *stream,
                    ks_ctx **out) {
  KS_RANGE();
  if (!out) return KS_E_ARG;
  *out = nullptr;
  KS_TRY(check_mesh_args(n_nodes, h_xyz, n_tets, h_tets, h_dirichlet, max_N));
  if (!d_persistent || !d_workspace) {
    set_create_err("KS_E_ARG: ks_create needs the persistent and workspace regions (sizes from ks_plan)");
    return KS_E_ARG;
  }
  ks_ctx *ctx = new ks_ctx();
  ctx->stream = (cudaStream_t)stream;
  ctx->n_nodes = n_nodes;
  ctx->n_tets = n_tets;
  ctx->max_N = max_N;
  ks_status st = KS_OK;
  do {
    if ((st = ks_cuda_check(ctx, cudaGetDevice(&ctx->device), "cudaGetDevice")) != KS_OK) break;
    if ((st = ks_cuda_check(ctx, cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, ctx->device),
                            "cudaDeviceGetAttribute")) != KS_OK)
      break;
    int coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device);
    if (!coop) { st = ks_fail(ctx, KS_E_CUDA, "device does not support cooperative launch"); break; }
    if ((st = bind_region(ctx, KS_R_PERSIST, d_persistent, persistent_bytes, "d_persistent")) != KS_OK) break;
    if ((st = bind_region(ctx, KS_R_WORK, d_workspace, workspace_bytes, "d_workspace")) != KS_OK) break;
    // setup temporaries: the caller's setup region, or the workspace (free until the solver carves it)
    if ((st = d_setup ? bind_region(ctx, KS_R_SETUP, d_setup, setup_bytes, "d_setup")
                      : bind_region(ctx, KS_R_SETUP, d_workspace, workspace_bytes, "d_workspace")) != KS_OK)
      break;
    st = ks_setup_mesh(ctx, h_xyz, h_tets, h_dirichlet);
    ctx->reg[KS_R_SETUP] = ks_region();   // the setup region is not referenced after ks_create returns
    if (st != KS_OK) break;
    KsRegion rg(ctx, KS_R_WORK);
    KsCarver cv(ctx);
    ks_layout_work(cv, ctx, ctx->n_free, max_N, ctx->sm_count);
    if ((st = cv.st) != KS_OK) break;
    st = ks_cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize (ks_create)");
  } while (0);
  if (st != KS_OK) {
    set_create_err(ctx->err);
    free_all(ctx);
    delete ctx;
    return st;
  }
  *out = ctx;
  return KS_OK;
}

void ks_destroy(ks_ctx *ctx) {
  KS_RANGE();
  if (!ctx) return;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  else cudaDeviceSynchronize();
  free_all(ctx);
  delete ctx;
}

ks_status ks_set_stream(ks_ctx *ctx, void *stream) {
  KS_RANGE();
  if (!ctx) return KS_E_ARG;
  cudaStream_t ns = (cudaStream_t)stream;
  if (ns == ctx->stream) return KS_OK;
  // Work still queued on the old stream shares the context's workspaces (grid-barrier counter, solver
  // vectors, status flags): the new stream waits for it before anything enqueued after this call runs.
  cudaEvent_t ev;
  KS_CUDA(ctx, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  cudaError_t e = cudaEventRecord(ev, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(ns, ev, 0);
  cudaEventDestroy(ev);
  KS_CUDA(ctx, e);
  ctx->stream = ns;
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
  KS_RANGE();
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
  KS_RANGE();
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
  KS_RANGE();
  if (!ctx) return KS_E_ARG;
  if (N < 1 || N > KS_MAX_N) return ks_fail(ctx, KS_E_ARG, "ks_spmm: N = %d outside [1, %d]", N, KS_MAX_N);
  if (!d_X || !d_Y || d_X == d_Y) return ks_fail(ctx, KS_E_ARG, "ks_spmm: X, Y must be distinct non-null");
  if (((uintptr_t)d_X & 7) || ((uintptr_t)d_Y & 7)) return ks_fail(ctx, KS_E_ARG, "ks_spmm: X, Y must be 8-byte aligned");
  const double *v = op_values(ctx, op);
  if (!v) return ks_fail(ctx, KS_E_STATE, "ks_spmm: operator %d not assembled", (int)op);
  // the CSR views M_V, H, A are recomputed after an assembly on first use (the generic CSR kernel reads A
  // for ragged N or unaligned blocks, so A is refreshed as well)
  if (op == KS_OP_MV || op == KS_OP_H || op == KS_OP_A) KS_TRY(ks_materialize_views(ctx));
  return ks_spmm_impl(ctx, op, v, N, d_X, d_Y);
}

ks_status ks_block_solve(ks_ctx *ctx, int32_t N, const double *d_lambda, const double *d_U, double *d_Ut,
                         double tol, int32_t max_iter, int32_t *d_iters, double *d_relres) {
  KS_RANGE();
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
  KS_RANGE();
  if (!ctx || !h_block_iters) return KS_E_ARG;
  KS_CUDA(ctx, cudaMemcpyAsync(h_block_iters, ctx->d_block_iters, 4, cudaMemcpyDeviceToHost, ctx->stream));
  KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return KS_OK;
}

ks_status ks_pencil_eig(ks_ctx *ctx, int64_t D, int32_t k, const double *d_FA, const double *d_FB, double *d_evals,
                        double *d_evecs) {
  KS_RANGE();
  if (!ctx) return KS_E_ARG;
  if (D < 1 || k < 1 || k > D || D > 65536) return ks_fail(ctx, KS_E_ARG, "ks_pencil_eig: need 1 <= k <= D <= 65536");
  if (!d_FA || !d_FB || !d_evals || !d_evecs) return ks_fail(ctx, KS_E_ARG, "ks_pencil_eig: null pointer");
  return ks_pencil_eig_impl(ctx, D, k, d_FA, d_FB, d_evals, d_evecs);
}

ks_status ks_lift(ks_ctx *ctx, int32_t N, const double *d_Ut, int32_t k, const double *d_Y, double *d_Unew) {
  KS_RANGE();
  if (!ctx) return KS_E_ARG;
  if (N < 1 || N > KS_MAX_N || k < 1 || !d_Ut || !d_Y || !d_Unew || d_Ut == d_Unew)
    return ks_fail(ctx, KS_E_ARG, "ks_lift: bad arguments");
  if (ctx->n_H < 1) return ks_fail(ctx, KS_E_STATE, "ks_lift: call ks_set_coarse first");
  return ks_lift_impl(ctx, N, d_Ut, k, d_Y, d_Unew);
}

ks_status ks_augmented_solve(ks_ctx *ctx, int32_t N, double *d_lambda, double *d_U, double tol_eig, int32_t max_outer,
                             double tol_bvp, int32_t max_iter_bvp, int32_t *h_outer, double *h_history) {
  KS_RANGE();
  if (!ctx) return KS_E_ARG;
  if (N < 1 || N > KS_MAX_N || !d_lambda || !d_U || !(tol_eig >= 0.0) || max_outer < 1 || !(tol_bvp > 0.0) ||
      max_iter_bvp < 1)
    return ks_fail(ctx, KS_E_ARG, "ks_augmented_solve: bad arguments");
  if (!ctx->assembled) return ks_fail(ctx, KS_E_STATE, "ks_augmented_solve: call ks_assemble_veff first");
  if (ctx->n_H < 1) return ks_fail(ctx, KS_E_STATE, "ks_augmented_solve: call ks_set_coarse first");
  return ks_augmented_solve_impl(ctx, N, d_lambda, d_U, tol_eig, max_outer, tol_bvp, max_iter_bvp, h_outer, h_history);
}

ks_status ks_interpolation_plan(ks_ctx *ctx, int64_t n_c, const double *h_xyz_c, int64_t m_c,
                                size_t *work_bytes) {
  KS_RANGE();
  if (!ctx) return KS_E_ARG;
  if (n_c < 4 || m_c < 1 || n_c > 0x7fffffffLL || m_c > 0x7fffffffLL || !h_xyz_c || !work_bytes)
    return ks_fail(ctx, KS_E_ARG, "ks_interpolation_plan: bad arguments");
  return ks_interpolation_plan_impl(ctx, n_c, h_xyz_c, m_c, work_bytes);
}

ks_status ks_interpolation(ks_ctx *ctx, int64_t n_c, const double *h_xyz_c, int64_t m_c, const int32_t *h_tets_c,
                           const uint8_t *h_dirichlet_c, void *d_work, size_t work_bytes, int32_t *d_P_row_ptr,
                           int32_t *d_P_col, double *d_P_val, int64_t *h_n_H, int64_t *h_p_nnz) {
  KS_RANGE();
  if (!ctx) return KS_E_ARG;
  if (n_c < 4 || m_c < 1 || n_c > 0x7fffffffLL || m_c > 0x7fffffffLL || !h_xyz_c || !h_tets_c || !h_dirichlet_c ||
      !d_work || !d_P_row_ptr || !d_P_col || !d_P_val || !h_n_H || !h_p_nnz)
    return ks_fail(ctx, KS_E_ARG, "ks_interpolation: bad arguments");
  return ks_interpolation_impl(ctx, n_c, h_xyz_c, m_c, h_tets_c, h_dirichlet_c, d_work, work_bytes, d_P_row_ptr,
                               d_P_col, d_P_val, h_n_H, h_p_nnz);
}

ks_status ks_density(ks_ctx *ctx, int32_t N, const double *d_U, double f, double *d_rho) {
  KS_RANGE();
  if (!ctx) return KS_E_ARG;
  if (N < 1 || N > KS_MAX_N || !d_U || !d_rho || !(f >= 0.0)) return ks_fail(ctx, KS_E_ARG, "ks_density: bad arguments");
  return ks_density_impl(ctx, N, d_U, f, d_rho);
}

ks_status ks_vxc(ks_ctx *ctx, const double *d_rho, double *d_vxc, double *d_eps) {
  KS_RANGE();
  if (!ctx) return KS_E_ARG;
  if (!d_rho || !d_vxc) return ks_fail(ctx, KS_E_ARG, "ks_vxc: null pointer");
  return ks_vxc_impl(ctx, d_rho, d_vxc, d_eps);
}

ks_status ks_hartree(ks_ctx *ctx, const double *d_rho, double tol, int32_t max_iter, double *d_vh, int32_t warm,
                     double *h_mom, int32_t *h_iters) {
  KS_RANGE();
  if (!ctx) return KS_E_ARG;
  if (!d_rho || !d_vh || !(tol > 0.0) || max_iter < 1) return ks_fail(ctx, KS_E_ARG, "ks_hartree: bad arguments");
  return ks_hartree_impl(ctx, d_rho, tol, max_iter, d_vh, warm, h_mom, h_iters);
}

ks_status ks_scf_solve(ks_ctx *ctx, int32_t N, const double *d_vext, double f, double mu, double *d_lambda,
                       double *d_U, double tol, int32_t max_outer, int32_t inner, double inner_tol, double beta,
                       int32_t depth, double bvp_tol, double hartree_tol, int32_t *h_outer, int32_t *h_inner,
                       double *h_dres, double *h_lams) {
  KS_RANGE();
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
  KS_RANGE();
  if (!ctx) return KS_E_ARG;
  if (N < 1 || N > KS_MAX_N || !h_V || !h_lambda || !h_U || !h_FA || !h_FB || !(tol > 0.0) || max_iter < 1 ||
      !(mu >= 0.0))
    return ks_fail(ctx, KS_E_ARG, "ks_step_submit: bad arguments");
  if (ctx->n_H < 1) return ks_fail(ctx, KS_E_STATE, "ks_step_submit: call ks_set_coarse first");
  return ks_step_submit_impl(ctx, N, h_V, mu, h_lambda, h_U, tol, max_iter, h_FA, h_FB);
}

ks_status ks_step_wait(ks_ctx *ctx) {
  KS_RANGE();
  if (!ctx) return KS_E_ARG;
  return ks_step_wait_impl(ctx);
}

ks_status ks_solve_trace(ks_ctx *ctx, int32_t cap, uint64_t *h_ns, int32_t *h_count) {
  KS_RANGE();
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
  KS_RANGE();
  if (!ctx) return KS_E_ARG;
  if (N < 1 || N > KS_MAX_N || !d_lambda || !d_U || !d_Ut || !d_relres)
    return ks_fail(ctx, KS_E_ARG, "ks_true_residual: bad arguments");
  if (!ctx->assembled) return ks_fail(ctx, KS_E_STATE, "ks_true_residual: call ks_assemble_veff first");
  return ks_true_residual_impl(ctx, N, d_lambda, d_U, d_Ut, d_relres);
}

static ks_status check_coarse_args(ks_ctx *ctx, int64_t n_H, const int32_t *d_P_row_ptr, const int32_t *d_P_col,
                                   const double *d_P_val) {
  if (n_H < 1 || n_H > 0x7fffffffLL) return ks_fail(ctx, KS_E_ARG, "coarse space: n_H = %lld", (long long)n_H);
  if (!d_P_row_ptr || !d_P_col || !d_P_val) return ks_fail(ctx, KS_E_ARG, "coarse space: null P arrays");
  return KS_OK;
}

ks_status ks_coarse_plan(ks_ctx *ctx, int64_t n_H, const int32_t *d_P_row_ptr, const int32_t *d_P_col,
                         const double *d_P_val, size_t *coarse_bytes) {
  KS_RANGE();
  if (!ctx || !coarse_bytes) return KS_E_ARG;
  KS_TRY(check_coarse_args(ctx, n_H, d_P_row_ptr, d_P_col, d_P_val));
  return ks_set_coarse_impl(ctx, n_H, d_P_row_ptr, d_P_col, d_P_val, true, coarse_bytes);
}

ks_status ks_set_coarse(ks_ctx *ctx, int64_t n_H, const int32_t *d_P_row_ptr, const int32_t *d_P_col,
                        const double *d_P_val, void *d_coarse, size_t coarse_bytes) {
  KS_RANGE();
  if (!ctx) return KS_E_ARG;
  KS_TRY(check_coarse_args(ctx, n_H, d_P_row_ptr, d_P_col, d_P_val));
  if (!d_coarse) return ks_fail(ctx, KS_E_ARG, "ks_set_coarse: null coarse region (size from ks_coarse_plan)");
  // a new coarse space invalidates the old one and the extension workspace planned for it
  KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  ks_free_coarse(ctx);
  ctx->ext_features = 0;
  ctx->reg[KS_R_EXT] = ks_region();
  KS_TRY(bind_region(ctx, KS_R_COARSE, d_coarse, coarse_bytes, "d_coarse"));
  ks_status st = ks_set_coarse_impl(ctx, n_H, d_P_row_ptr, d_P_col, d_P_val, false, nullptr);
  if (st != KS_OK) {
    ks_free_coarse(ctx);
    ctx->reg[KS_R_COARSE] = ks_region();
  }
  return st;
}

static ks_status ext_sizes(ks_ctx *ctx, uint32_t features, int64_t max_D, KsExtSizes *e) {
  if (features & KS_EXT_SCF) features |= KS_EXT_EIG;
  e->features = features;
  e->nn = ctx->n_nodes;
  e->nt = ctx->n_tets;
  e->nf = ctx->n_free;
  e->nH = ctx->n_H;
  e->ni = ctx->n_items;
  e->N = ctx->max_N;
  e->sm_count = ctx->sm_count;
  e->D = ctx->n_H + ctx->max_N;
  if (max_D > e->D) e->D = max_D;
  e->lwork = 1;
  if (features & KS_EXT_EIG) KS_TRY(ks_cusolver_lwork(ctx, e->D, ctx->n_H, &e->lwork));
  return KS_OK;
}

ks_status ks_ext_plan(ks_ctx *ctx, uint32_t features, int64_t max_D, size_t *ext_bytes) {
  KS_RANGE();
  if (!ctx || !ext_bytes) return KS_E_ARG;
  if (features == 0 || (features & ~(uint32_t)(KS_EXT_EIG | KS_EXT_SCF | KS_EXT_STEP)))
    return ks_fail(ctx, KS_E_ARG, "ks_ext_plan: features must be a nonempty KS_EXT_* mask");
  if (max_D < 0 || max_D > 65536) return ks_fail(ctx, KS_E_ARG, "ks_ext_plan: max_D = %lld", (long long)max_D);
  KsExtSizes e;
  KS_TRY(ext_sizes(ctx, features, max_D, &e));
  KsSizer sz;
  ks_ctx tmp;
  ks_layout_ext(sz, &tmp, e);
  *ext_bytes = sz.bytes;
  return KS_OK;
}

ks_status ks_attach_ext(ks_ctx *ctx, uint32_t features, int64_t max_D, void *d_ext, size_t ext_bytes) {
  KS_RANGE();
  if (!ctx) return KS_E_ARG;
  if (features == 0 || (features & ~(uint32_t)(KS_EXT_EIG | KS_EXT_SCF | KS_EXT_STEP)) || !d_ext || max_D < 0 ||
      max_D > 65536)
    return ks_fail(ctx, KS_E_ARG, "ks_attach_ext: bad arguments");
  KsExtSizes e;
  KS_TRY(ext_sizes(ctx, features, max_D, &e));
  KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->ext_features = 0;
  ctx->har2l_state = 0;
  ctx->ef_LH_state = 0;
  ctx->ef_L_D = 0;
  ctx->ef_LH = ctx->ef_LHinv = ctx->ef_Linv = ctx->ef_TD = ctx->ef_aux = nullptr;
  KS_TRY(bind_region(ctx, KS_R_EXT, d_ext, ext_bytes, "d_ext"));
  {
    KsRegion rg(ctx, KS_R_EXT);
    KsCarver cv(ctx);
    ks_layout_ext(cv, ctx, e);
    if (cv.st != KS_OK) {
      ctx->reg[KS_R_EXT] = ks_region();
      return cv.st;
    }
  }
  ctx->ext_features = e.features;
  ctx->ext_nH = ctx->n_H;
  ctx->ext_D = e.D;
  ctx->ext_lwork = e.lwork;
  return KS_OK;
}

ks_status ks_project_augmented(ks_ctx *ctx, int32_t N, const double *d_Ut, double *d_FA, double *d_FB) {
  KS_RANGE();
  if (!ctx) return KS_E_ARG;
  if (N < 1 || N > KS_MAX_N) return ks_fail(ctx, KS_E_ARG, "ks_project_augmented: N = %d outside [1, %d]", N, KS_MAX_N);
  if (!d_Ut || !d_FA || !d_FB || d_FA == d_FB) return ks_fail(ctx, KS_E_ARG, "ks_project_augmented: bad pointers");
  if (!ctx->assembled) return ks_fail(ctx, KS_E_STATE, "ks_project_augmented: call ks_assemble_veff first");
  if (ctx->n_H < 1) return ks_fail(ctx, KS_E_STATE, "ks_project_augmented: call ks_set_coarse first");
  return ks_project_impl(ctx, N, d_Ut, d_FA, d_FB);
}

static ks_status check_slab(ks_ctx *ctx, int32_t NP, int64_t row0, int64_t row1, const void *const *ptrs, int np) {
  if (!ctx) return KS_E_ARG;
  if (NP < 1 || NP > KS_MAX_N || (NP & (NP - 1)))
    return ks_fail(ctx, KS_E_ARG, "slab: NP = %d must be a power of two in [1, 64]", NP);
  if (row0 < 0 || row1 <= row0 || row1 > ctx->n_free)
    return ks_fail(ctx, KS_E_ARG, "slab: rows [%lld, %lld) outside [0, %lld)", (long long)row0, (long long)row1,
                   (long long)ctx->n_free);
  for (int i = 0; i < np; i++) {
    if (!ptrs[i]) return ks_fail(ctx, KS_E_ARG, "slab: null pointer argument %d", i);
    if (NP >= 4 && ((uintptr_t)ptrs[i] & 31)) return ks_fail(ctx, KS_E_ARG, "slab: blocks must be 32-byte aligned");
  }
  if (!ctx->assembled) return ks_fail(ctx, KS_E_STATE, "slab: call ks_assemble_veff first");
  return KS_OK;
}

ks_status ks_slab_init(ks_ctx *ctx, int32_t NP, int64_t row0, int64_t row1, const double *d_lambda, const double *d_U,
                       double *d_Z, double *d_P, double *d_dots) {
  KS_RANGE();
  const void *p[] = {d_U, d_Z, d_P};
  KS_TRY(check_slab(ctx, NP, row0, row1, p, 3));
  if (!d_lambda || !d_dots) return ks_fail(ctx, KS_E_ARG, "ks_slab_init: null lambda / dots");
  return ks_slab_phase_impl(ctx, 0, NP, row0, row1, 0, nullptr, nullptr, d_lambda, d_U, d_Z, nullptr, d_P, nullptr,
                            nullptr, d_dots);
}

ks_status ks_slab_spmm(ks_ctx *ctx, int32_t NP, int64_t row0, int64_t row1, int32_t first, const double *h_alpha_x,
                       const double *h_beta, const double *d_Z, double *d_Q, double *d_P, const double *d_Xin,
                       double *d_X, double *d_dots) {
  KS_RANGE();
  const void *p[] = {d_Z, d_Q, d_P, d_Xin, d_X};
  KS_TRY(check_slab(ctx, NP, row0, row1, p, 5));
  if (!h_alpha_x || !h_beta || !d_dots) return ks_fail(ctx, KS_E_ARG, "ks_slab_spmm: null coefficients / dots");
  return ks_slab_phase_impl(ctx, 1, NP, row0, row1, first, h_alpha_x, h_beta, nullptr, nullptr,
                            const_cast<double *>(d_Z), d_Q, d_P, d_Xin, d_X, d_dots);
}

ks_status ks_slab_update(ks_ctx *ctx, int32_t NP, int64_t row0, int64_t row1, const double *h_alpha, double *d_Z,
                         const double *d_Q, double *d_dots) {
  KS_RANGE();
  const void *p[] = {d_Z, d_Q};
  KS_TRY(check_slab(ctx, NP, row0, row1, p, 2));
  if (!h_alpha || !d_dots) return ks_fail(ctx, KS_E_ARG, "ks_slab_update: null coefficients / dots");
  return ks_slab_phase_impl(ctx, 2, NP, row0, row1, 0, h_alpha, nullptr, nullptr, nullptr, d_Z,
                            const_cast<double *>(d_Q), nullptr, nullptr, nullptr, d_dots);
}

ks_status ks_slab_finish(ks_ctx *ctx, int32_t NP, int64_t row0, int64_t row1, const double *h_alpha_x,
                         const double *d_P, const double *d_Xin, double *d_X) {
  KS_RANGE();
  const void *p[] = {d_P, d_Xin, d_X};
  KS_TRY(check_slab(ctx, NP, row0, row1, p, 3));
  if (!h_alpha_x) return ks_fail(ctx, KS_E_ARG, "ks_slab_finish: null coefficients");
  return ks_slab_phase_impl(ctx, 3, NP, row0, row1, 0, h_alpha_x, nullptr, nullptr, nullptr, nullptr, nullptr,
                            const_cast<double *>(d_P), d_Xin, d_X, nullptr);
}

ks_status ks_memory_bytes(const ks_ctx *ctx, size_t *bytes) {
  if (!ctx || !bytes) return KS_E_ARG;
  size_t b = 0;
  for (int r = 0; r < KS_R_N; r++) b += ctx->reg[r].cap;
  *bytes = b;
  return KS_OK;
}

ks_status ks_memory_usage(const ks_ctx *ctx, int32_t region, size_t *capacity, size_t *used, size_t *peak) {
  if (!ctx || region < 0 || region >= KS_R_N) return KS_E_ARG;
  if (capacity) *capacity = ctx->reg[region].cap;
  if (used) *used = ctx->reg[region].off;
  if (peak) *peak = ctx->reg[region].peak;
  return KS_OK;
}

ks_status ks_launch_count(const ks_ctx *ctx, int64_t *count) {
  if (!ctx || !count) return KS_E_ARG;
  *count = ctx->launches;
  return KS_OK;
}

ks_status ks_sync(ks_ctx *ctx) {
  KS_RANGE();
  if (!ctx) return KS_E_ARG;
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return ks_cuda_check(ctx, e, "cudaStreamSynchronize");
  unsigned f = 0;
  // read and clear on the context's stream, so the clear is ordered before work enqueued afterwards
  KS_CUDA(ctx, cudaMemcpyAsync(&f, ctx->d_flags, 4, cudaMemcpyDeviceToHost, ctx->stream));
  KS_CUDA(ctx, cudaMemsetAsync(ctx->d_flags, 0, 4, ctx->stream));
  KS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
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
