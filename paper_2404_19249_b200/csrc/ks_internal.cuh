// ks_internal.cuh -- context struct and device helpers of libks (sm_100a, fp64).
// Not part of the ABI; see include/ks.h.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>
#include <stdio.h>
#include <string>
#include <vector>

#include "../../include/ks.h"

// device status bits latched by kernels (reported by ks_sync)
enum : unsigned {
  KSF_NONFINITE = 1u,
  KSF_NOT_SPD = 2u,
  KSF_NOT_CONVERGED = 4u,
  KSF_MESH = 8u,
};

// Device memory is owned by the caller (include/ks.h, "Memory"): the library carves every buffer out of
// caller-provided regions with a bump allocator (ks_alloc); it never calls cudaMalloc / cudaFree.
enum : int {
  KS_R_PERSIST = 0,   // ks_create: mesh, pattern, maps, values, sliced-ELL copies (ctx lifetime)
  KS_R_WORK = 1,      // ks_create: solver workspace for N <= max_N + call scratch (ctx lifetime)
  KS_R_SETUP = 2,     // ks_create only: setup temporaries (may be the workspace)
  KS_R_COARSE = 3,    // ks_set_coarse: P, item tables, B_H, projection workspace (until the next set_coarse)
  KS_R_EXT = 4,       // ks_attach_ext: NEXT-1/2 and host-step workspaces
  KS_R_CALL = 5,      // one call's caller-provided scratch (ks_interpolation)
  KS_R_N = 6
};
struct ks_region {
  uint8_t *base = nullptr;
  size_t cap = 0, off = 0, peak = 0;
};
#define KS_ALIGN 256
static inline size_t ks_round(size_t b) { return (b + KS_ALIGN - 1) / KS_ALIGN * KS_ALIGN; }

struct ks_ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  int64_t n_nodes = 0, n_tets = 0, n_free = 0, nnz = 0, n_contrib = 0;
  int64_t launches = 0;
  int max_N = 0;                    // largest N the workspace was planned for (ks_plan / ks_create)
  ks_region reg[KS_R_N];
  int region = KS_R_PERSIST;        // region ks_alloc carves from
  unsigned ext_features = 0;        // KS_EXT_* of the attached extension workspace (0: none attached)
  int64_t ext_nH = -1;              // n_H it was planned for (a new coarse space detaches it)
  int64_t ext_D = 0;                // largest pencil dimension it holds
  int64_t ext_lwork = 0;            // cuSOLVER workspace (doubles) it holds
  uint8_t *blas_ws = nullptr;       // cuBLAS workspace (KS_EXT_BLAS_WS bytes)

  // mesh / pattern (library-owned device memory)
  int32_t *tets = nullptr;          // [4 n_tets]
  double *xyz = nullptr;            // [3 n_nodes] node coordinates
  int32_t *free_of_node = nullptr;  // [n_nodes]
  int32_t *node_of_free = nullptr;  // [n_free]
  int32_t *row_ptr = nullptr;       // [n_free+1]
  int32_t *col = nullptr;           // [nnz]
  int32_t *diag_pos = nullptr;      // [n_free] position of (i,i)
  int32_t *emap = nullptr;          // [16 n_tets]
  int32_t *inv_ptr = nullptr;       // [nnz+1]
  int32_t *inv_idx = nullptr;       // [n_contrib] emap indices 16t+4a+b sorted by target nnz, then index
  double *vol = nullptr;            // [n_tets]
  double *K = nullptr, *M = nullptr, *MV = nullptr, *H = nullptr, *A = nullptr;  // [nnz]
  double *diag = nullptr;           // [n_free] diag(A)
  double *dinv = nullptr;           // [n_free + 2] 1 / diag(A) (Jacobi preconditioner), zero padded
  double *w_tet = nullptr;          // [n_tets] |T| S_T (assembly scratch)
  // sliced-ELL copy of the pattern for the block-PCG SpMM (ks_sell.cu): A (per assembly) and M (fixed)
  int64_t n_slices = 0, sell_total = 0;
  int32_t *sell_ptr = nullptr;      // [n_slices+1] first entry of each 8-row slice
  int32_t *sell_col = nullptr;      // [sell_total]
  double *sell_A = nullptr, *sell_M = nullptr, *sell_H = nullptr;  // [sell_total]
  double *sell_K = nullptr;         // [sell_total] stiffness (Poisson operator of the Hartree solve)
  int32_t *sell_csr = nullptr;      // [sell_total] CSR index of each slot (-1: padding), for the assembly
  uint64_t *slot_mask = nullptr;    // [sell_total] star tets contributing to each slot's entry (ks_assemble.cu)
  int2 *star = nullptr;             // [n_free] (first, length) of each row's star in inv_idx
  int max_star = 1 << 30;           // largest star (tets containing a free node); set at ks_create
  int mask_bits = 0;                // width of slot_mask's entries (32 / 64), 0 = masks not built
  double *dinvK = nullptr;          // [n_free + 2] 1 / diag(K)
  double *v_free = nullptr;         // [n_free] V at free nodes (assembly scratch)
  double mu = 0.0;
  bool assembled = false;
  bool views_fresh = false;         // CSR views MV, H, A match the last assembly (ks_materialize_views)

  // device status
  unsigned *d_flags = nullptr;      // latched KSF_* bits
  int32_t *d_block_iters = nullptr; // [1] block iterations of the last solve
  unsigned long long *trace = nullptr;  // [KS_TRACE_CAP] phase-end timestamps of the last traced solve
  int *trace_count = nullptr;

  // solver workspace (KS_R_WORK, carved at ks_create for N <= max_N)
  int tile_emax[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // largest sliced-ELL entries of a PCG tile, per log2(NP)
  double *r = nullptr, *p = nullptr, *q = nullptr, *xpad = nullptr, *upad = nullptr, *bpad = nullptr;
  double *partials = nullptr;       // [grid][4 * 64]
  unsigned *barrier = nullptr;      // grid barrier counter

  // coarse space (ks_set_coarse) and projection workspace
  int64_t n_H = 0, p_nnz = 0;
  int32_t *P_ptr = nullptr, *P_col = nullptr;   // own copy, columns ascending within a row
  double *P_val = nullptr;
  double *Pv4 = nullptr;         // [4 n_free] P rows as a zero-padded 4-wide table
  double *Pv4p = nullptr;        // [4 n_free] the same in item order (position of the parent grouping)
  int32_t *pos_of_row = nullptr; // [n_free] inverse of perm
  int64_t n_items = 0, d_total = 0;
  int d_max = 0;
  int32_t *perm = nullptr;       // [n_free] fine rows grouped by parent set ("items" of <= ITEM_ROWS rows)
  int32_t *item_ptr = nullptr;   // [n_items+1] ranges of perm
  int32_t *item_S = nullptr;     // [4 n_items] parent coarse ids of the item (-1 padded)
  int32_t *item_D_ptr = nullptr; // [n_items+1]
  int32_t *item_D = nullptr;     // [d_total] sorted coarse ids touched by P rows of the item's neighbours
  uint8_t *slotmap = nullptr;    // [4 nnz] slot of (entry k, parent t of col[k]) in its row's item D list
  int32_t *CT_ptr = nullptr;     // [n_H+1] coarse node -> (item, local parent) list
  int32_t *CT_val = nullptr;     // [4 n_items] entries 4 item + q
  double *B_H = nullptr;         // [n_H n_H] cached P^T M P
  double *AH_part = nullptr;     // [4 d_total] per-item partials of P^T Op P
  int ah_fresh = 0;              // AH_part holds the A_H partials of the current H (1: k_proj_ai, 2: k_proj_a); reset by
                                 // an assembly, a coarse space and every other use of AH_part
  double *bH_part = nullptr, *cH_part = nullptr;  // [4 n_items NP]
  double *Y_H = nullptr, *Y_M = nullptr, *proj_u = nullptr;  // [n_free][NP] (Y_H, Y_M in item order)
  double *proj_up = nullptr;     // [n_free][NP] U~ in item order
  double *gram_part = nullptr;   // [blocks][2 N N]
  int64_t gram_cap = 0;
  // item-ordered sliced-ELL copy of the pattern for the A_H pass (ks_project.cu k_proj_ai): every item starts on
  // an 8-row slice; row position r of item it is slice islice0[it] + r / 8, lane row r % 8
  int64_t n_islices = 0, isell_total = 0;
  int32_t *islice0 = nullptr;    // [n_items+1] first item slice of each item
  int32_t *isell_ptr = nullptr;  // [n_islices+1] first slot of each item slice
  int2 *inat = nullptr;          // [n_free] per item position: (natural sliced-ELL slot of the row's slot 0, its
                                 // slot groups); H is read in the natural layout the assembly writes
  int32_t *isell_col = nullptr;  // [isell_total] natural column (padding: own row, pad rows: 0)
  uint32_t *islot = nullptr;     // [isell_total] word (row, group g, parent t): bytes u = window slot of parent t
                                 // of the column of slot 4g+u (255: absent)

  // NEXT-2 Hartree workspace (ks_scf.cu)
  double *har_w = nullptr, *har_c = nullptr, *har_b = nullptr, *har_x0 = nullptr, *har_x = nullptr;
  double *har_mom = nullptr, *har_part = nullptr;
  int32_t *har_iters = nullptr;
  // two-level preconditioner of the Hartree solve (ks_pcg2l.cu): K_H^-1 = (P^T K P)^-1 on the coarse space
  int har2l_state = 0;              // 0: not built for the current coarse space, 1: built, -1: unusable
  double *har2l_KHinv = nullptr;    // [n_H n_H]
  double *har2l_rpart = nullptr;    // [4 n_items] item restriction partials
  double *har2l_rH = nullptr, *har2l_y = nullptr;                       // [n_H]
  double *har2l_r = nullptr, *har2l_r2 = nullptr, *har2l_p = nullptr, *har2l_q = nullptr;  // [n_free]
  double *har2l_part = nullptr;     // [grid][8] block partials
  int32_t *har2l_Pc4 = nullptr;     // [4 n_free] P columns as a 4-wide table (pairs with Pv4)
  // NEXT-2 SCF driver workspace
  double *scf_rho = nullptr, *scf_in = nullptr, *scf_out = nullptr, *scf_vh = nullptr, *scf_vxc = nullptr;
  double *scf_veff = nullptr, *scf_Ut = nullptr, *scf_FA = nullptr, *scf_FB = nullptr, *scf_Y = nullptr;
  double *scf_hin = nullptr, *scf_hout = nullptr, *scf_part = nullptr, *scf_red = nullptr, *scf_alpha = nullptr;
  int *scf_slot = nullptr;
  // pipelined host-buffer steps (ks_stream.cu)
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr}, ev_d2h[2] = {nullptr, nullptr};
  double *st_V[2] = {nullptr, nullptr}, *st_lam[2] = {nullptr, nullptr}, *st_U[2] = {nullptr, nullptr};
  double *st_Ut[2] = {nullptr, nullptr}, *st_FA[2] = {nullptr, nullptr}, *st_FB[2] = {nullptr, nullptr};
  int64_t step_count = 0;
  int interp_fallbacks = 0;         // last ks_interpolation needed the scan fallback of the walk
  // NEXT-1 (ks_outer.cu): cuSOLVER handle, pencil and outer-loop workspaces
  void *cusolver = nullptr;
  void *cublas = nullptr;           // cuBLAS handle of the filtered pencil eigensolver (ks_outer.cu)
  double *ef_buf = nullptr;         // [4][D][m] work blocks of the filtered eigensolver
  double *ef_small = nullptr;       // [m][m] device staging of the small Rayleigh-Ritz / SVQB matrices
  double *ef_dev = nullptr;         // scratch of the device-resident filtered iteration (ks_efdev.cu)
  int ef_rounds = 0;                // Rayleigh-Ritz rounds of the last filtered solve
  int64_t ef_L_D = 0;                // D of the Cholesky factor held in eig_B (0: none)
  // cached Cholesky factor of the coarse block B_H (ks_outer.cu coarse_chol_reduction), per coarse space
  int ef_LH_state = 0;              // 0: not built, 1: built, -1: unusable
  double *ef_LH = nullptr, *ef_LHinv = nullptr;   // [n_H][n_H]
  double *ef_Linv = nullptr, *ef_TD = nullptr;    // [D][D] L^-1, GEMM temporary
  double *ef_aux = nullptr;                       // Kt, S, L_S^-1, T and a counter
  double *eig_A = nullptr, *eig_B = nullptr, *eig_w = nullptr, *eig_work = nullptr;
  int *eig_info = nullptr;
  double *outer_Ut = nullptr, *outer_FA = nullptr, *outer_FB = nullptr, *outer_Y = nullptr, *outer_lam = nullptr;

  std::string err;
};

#define KS_MAX_N 64
// elements of padding behind row_ptr, col and the value arrays: the bulk (TMA) tile copies round their
// ranges out to 16-byte boundaries and may read up to this far past the logical end.
#define KS_PAD 8
#define KS_TRACE_CAP 8192
#define KS_SELL_C 8   // rows per slice of the sliced-ELL operator copy

const char *ks_status_name(ks_status s);
ks_status ks_fail(ks_ctx *ctx, ks_status s, const char *fmt, ...);
ks_status ks_cuda_check(ks_ctx *ctx, cudaError_t e, const char *what);
// carves `bytes` (KS_ALIGN-aligned, zero-filled on the stream) from region ctx->region; KS_E_WORKSPACE when
// the caller's region is smaller than its plan said
ks_status ks_alloc(ks_ctx *ctx, void **ptr, size_t bytes, const char *what);

// the allocation region for a scope
struct KsRegion {
  ks_ctx *c;
  int prev;
  KsRegion(ks_ctx *c_, int r) : c(c_), prev(c_->region) { c->region = r; }
  ~KsRegion() { c->region = prev; }
};
// temporaries of one call: allocations from region r inside the scope are released at its end
struct KsScratch {
  ks_ctx *c;
  int r, prev;
  size_t mark;
  KsScratch(ks_ctx *c_, int r_) : c(c_), r(r_), prev(c_->region), mark(c_->reg[r_].off) { c->region = r_; }
  ~KsScratch() {
    c->reg[r].off = mark;
    c->region = prev;
  }
};

// byte counter with the allocator's rounding: plans add exactly what the allocation sites carve
struct KsSizer {
  size_t bytes = 0;
  template <typename T>
  void add(T **, int64_t count, const char * = nullptr) {
    bytes += ks_round(sizeof(T) * (size_t)(count > 0 ? count : 1));
  }
};

#define KS_TRY(expr)                      \
  do {                                    \
    ks_status _s = (expr);                \
    if (_s != KS_OK) return _s;           \
  } while (0)
#define KS_CUDA(ctx, expr) KS_TRY(ks_cuda_check((ctx), (expr), #expr))

template <typename T>
static inline ks_status ks_alloc_t(ks_ctx *ctx, T **ptr, int64_t count, const char *what) {
  return ks_alloc(ctx, (void **)ptr, sizeof(T) * (size_t)(count > 0 ? count : 1), what);
}

static inline int ks_blocks(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 0x7fffffff) b = 0x7fffffff;
  return (int)b;
}

// launch bookkeeping + error check
#define KS_LAUNCHED(ctx) \
  do { (ctx)->launches++; KS_CUDA((ctx), cudaGetLastError()); } while (0)

// ---------------------------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// internal entry points implemented in the .cu files
ks_status ks_setup_mesh(ks_ctx *ctx, const double *h_xyz, const int32_t *h_tets, const uint8_t *h_dir);
ks_status ks_sell_build(ks_ctx *ctx, int32_t *cnt, void *cub, size_t cub_bytes, int64_t planned_total);
ks_status ks_coarse_galerkin(ks_ctx *ctx, const double *op_sell_vals, double *out);   // P^T Op P, dense [n_H][n_H]
ks_status ks_spd_inverse(ks_ctx *ctx, double *A, int64_t n, bool *spd);              // A <- A^-1 (Cholesky)
ks_status ks_cusolver_lwork(ks_ctx *ctx, int64_t D, int64_t nH, int64_t *lwork);
ks_status ks_pcg2l_run(ks_ctx *ctx, const double *b, const double *x0, double *x, double tol, int max_iter,
                       int32_t *d_iters);
void ks_free_pcg2l(ks_ctx *ctx);
ks_status ks_assemble_impl(ks_ctx *ctx, const double *d_veff, double mu);
ks_status ks_materialize_views(ks_ctx *ctx);
int64_t ks_ef_device_scratch(int sm_count, int m, int64_t D);
ks_status ks_ef_device(ks_ctx *ctx, int64_t D, int k, int m, const double *C, const double *x0, double *x_out,
                       const double *bound_dev, double *scratch, int maxit, int deg, double tol, int *status,
                       int *rounds, bool *ran, double **lam_dev);

ks_status ks_star_setup(ks_ctx *ctx, int *d_tmp);  // d_tmp: one int of setup scratch
ks_status ks_spmm_impl(ks_ctx *ctx, ks_op op, const double *val, int N, const double *X, double *Y);
ks_status ks_solve_impl(ks_ctx *ctx, int N, const double *lambda, const double *U, double *Ut, double tol,
                        int max_iter, int32_t *iters, double *relres);
ks_status ks_pcg_run(ks_ctx *ctx, const double *sell_vals, const double *dinv, double mu, int N,
                     const double *lambda, const double *B, const double *U, double *Ut, double tol, int max_iter,
                     int32_t *iters, double *relres);
ks_status ks_true_residual_impl(ks_ctx *ctx, int N, const double *lambda, const double *U,
                                const double *Ut, double *relres);
ks_status ks_set_coarse_impl(ks_ctx *ctx, int64_t n_H, const int32_t *Pptr, const int32_t *Pcol,
                             const double *Pval, bool plan_only, size_t *coarse_bytes);
ks_status ks_project_impl(ks_ctx *ctx, int N, const double *Ut, double *FA, double *FB);
void ks_free_coarse(ks_ctx *ctx);
void ks_free_outer(ks_ctx *ctx);
void ks_free_stream(ks_ctx *ctx);
ks_status ks_step_submit_impl(ks_ctx *ctx, int N, const double *h_V, double mu, const double *h_lambda,
                              const double *h_U, double tol, int max_iter, double *h_FA, double *h_FB);
ks_status ks_step_wait_impl(ks_ctx *ctx);
ks_status ks_density_impl(ks_ctx *ctx, int N, const double *U, double f, double *rho);
ks_status ks_vxc_impl(ks_ctx *ctx, const double *rho, double *vxc, double *eps);
ks_status ks_scf_solve_impl(ks_ctx *ctx, int N, const double *vext, double f, double mu, double *lambda, double *U,
                            double tol, int max_outer, int inner, double inner_tol, double beta, int depth,
                            double bvp_tol, double hartree_tol, int32_t *h_outer, int32_t *h_inner, double *h_dres,
                            double *h_lams);
ks_status ks_hartree_impl(ks_ctx *ctx, const double *rho, double tol, int max_iter, double *vh, int warm,
                          double *h_mom, int32_t *h_iters);
ks_status ks_interpolation_impl(ks_ctx *ctx, int64_t n_c, const double *h_xyz_c, int64_t m_c, const int32_t *h_tets_c,
                                const uint8_t *h_dir_c, void *d_work, size_t work_bytes, int32_t *d_rowptr,
                                int32_t *d_col, double *d_val, int64_t *h_nH, int64_t *h_pnnz);
ks_status ks_interpolation_plan_impl(ks_ctx *ctx, int64_t n_c, const double *h_xyz_c, int64_t m_c, size_t *bytes);
ks_status ks_pencil_eig_impl(ks_ctx *ctx, int64_t D, int k, const double *FA, const double *FB, double *evals,
                             double *evecs, const double *Ywarm = nullptr, bool same_B = false);
// Ywarm [D][k] (device, may alias evecs): start block of the filtered path (e.g. the previous inner step's
// eigenvectors); same_B: F_B equals the previous call's (its Cholesky factor is reused)
ks_status ks_slab_phase_impl(ks_ctx *ctx, int phase, int NP, int64_t row0, int64_t row1, int first,
                             const double *h_alpha, const double *h_beta, const double *lambda, const double *U,
                             double *Z, double *Q, double *P, const double *Xin, double *X, double *dots);
ks_status ks_lift_impl(ks_ctx *ctx, int N, const double *Ut, int k, const double *Y, double *Unew);
ks_status ks_augmented_solve_impl(ks_ctx *ctx, int N, double *lambda, double *U, double tol_eig, int max_outer,
                                  double tol_bvp, int32_t max_iter_bvp, int32_t *h_outer, double *h_history);
