/*
 * ks.h -- C ABI of libks, the B200 (sm_100a) hot path of the nonnested augmented subspace method for
 * the Kohn-Sham equation (arXiv 2404.19249). Citations "PAPER.md:L" are lines of the paper's source.
 *
 * The library computes, on one GPU in fp64:
 *   ks_create             setup once per fine mesh: free numbering (Dirichlet elimination), the CSR
 *                         pattern of the P1 operators, the element-to-nnz scatter map and its inverse,
 *                         tet geometry, stiffness K and mass M (st3).
 *   ks_assemble_veff      V_eff-weighted mass M_V (st4) reassembled on the fixed
 *                         pattern, H = 1/2 K + M_V, shifted operator A = H + mu M (H~)
 *                         and its diagonal. Deterministic, no floating-point atomics.
 *   ks_block_solve        the N linear boundary value problems of Algorithm 3
 *                         (Aux_Linear_Problem): A u~_i = (lambda_i + mu) M u_i,
 *                         batched Jacobi-PCG over all N orbitals.
 *   ks_set_coarse         the interpolation operator P = I_H^h, cached mass blocks.
 *   ks_project_augmented  F_A, F_B of (st1)-(st2): A_H = P^T H P (st5), b_H = P^T H U~ (st6),
 *                         beta = U~^T H U~ (st7), B_H = P^T M P, c_H = P^T M U~, gamma = U~^T M U~
 *                         (PAPER.md:682-759).
 *
 * Conventions
 *   - Pointers named d_* are DEVICE pointers on the context's device; h_* are HOST pointers. The caller
 *     owns every pointer it passes; the library never frees them and never keeps host pointers past the
 *     call. Device inputs/outputs must stay valid until the stream work that uses them completes.
 *   - Memory: the caller owns ALL device memory. libks never allocates or frees device memory (no cudaMalloc,
 *     cudaMallocAsync or cudaFree anywhere in the library); it carves every buffer it uses out of regions
 *     the caller allocates from the sizes the plan calls return:
 *       ks_plan(mesh, max_N)          -> persistent, workspace, setup bytes      -> ks_create
 *       ks_coarse_plan(ctx, n_H, P)   -> coarse bytes                            -> ks_set_coarse
 *       ks_ext_plan(ctx, features, .) -> extension bytes (NEXT rows, host steps) -> ks_attach_ext
 *       ks_interpolation_plan(...)    -> scratch bytes of one ks_interpolation call
 *     Regions are device memory on the context's device, 256-byte aligned (torch's allocator gives 512),
 *     borrowed by the context: they must stay valid until ks_destroy (persistent, workspace), the next
 *     ks_set_coarse (coarse, extension) or the end of the call (setup, interpolation scratch), and until the
 *     stream work that uses them has completed. A region smaller than its plan returns KS_E_WORKSPACE.
 *     The cuSOLVER / cuBLAS handles of NEXT-1 are the libraries' own host objects; cuBLAS is given its GEMM
 *     workspace from the extension region (cublasSetWorkspace).
 *   - Every compute call is asynchronous on the context's stream (a cudaStream_t passed as void*).
 *     Device-detected conditions (non-finite values, NOT_SPD columns, non-convergence) are latched in a
 *     device flag word and returned by the next ks_sync. Argument errors are returned immediately and
 *     launch nothing.
 *   - Free numbering: free index = rank of a non-Dirichlet node among non-Dirichlet nodes, ascending node
 *     id. Blocks of orbitals are row-major [n_free][N] (orbital index fastest), 8-byte aligned; 16-byte
 *     alignment enables the vectorised path.
 *   - CSR: row_ptr int32 [n_free+1], col int32 [nnz] sorted ascending within a row, diagonal present.
 *   - emap int32 [16*n_tets]: emap[16 t + 4 a + b] = CSR position of (free(v_a), free(v_b)), -1 if
 *     either vertex is a Dirichlet node.
 *   - No exceptions cross the ABI. ks_last_error returns a NUL-terminated message for the last failure.
 */
#ifndef KS_H_
#define KS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KS_ABI_VERSION 2

typedef struct ks_ctx ks_ctx;

typedef enum {
  KS_OK = 0,
  KS_E_ARG = 1,            /* invalid argument (null pointer, size, alignment, range) */
  KS_E_MESH = 2,           /* inverted / degenerate tet or node index out of range (tet id in message) */
  KS_E_NONFINITE = 3,      /* NaN/Inf met in V_eff or in a solver reduction */
  KS_E_NOT_SPD = 4,        /* p.Ap <= 0 in some column: A = H + mu M not positive definite (mu too
                              small, Theorem 1) */
  KS_E_NOT_CONVERGED = 5,  /* max_iter reached with some column above tolerance; last iterate written */
  KS_E_CUDA = 6,           /* CUDA runtime error (message has the CUDA error string) */
  KS_E_NOMEM = 7,          /* device allocation failed */
  KS_E_STATE = 8,          /* call order: e.g. solve before assemble, project before set_coarse */
  KS_E_RANK = 9,           /* F_B not positive definite: W = [P | U~] rank deficient (ks_pencil_eig) */
  KS_E_WORKSPACE = 10      /* a caller-provided region is smaller than its plan (see "Memory") */
} ks_status;

/* Features of the extension workspace (ks_ext_plan / ks_attach_ext). */
enum {
  KS_EXT_EIG = 1u,   /* ks_pencil_eig, ks_augmented_solve (NEXT-1) */
  KS_EXT_SCF = 2u,   /* ks_hartree, ks_scf_solve (NEXT-2; implies KS_EXT_EIG) */
  KS_EXT_STEP = 4u   /* ks_step_submit / ks_step_wait (the hot-path step from host buffers) */
};

/* Operator selector for ks_spmm / ks_values. */
typedef enum { KS_OP_K = 0, KS_OP_M = 1, KS_OP_MV = 2, KS_OP_H = 3, KS_OP_A = 4 } ks_op;

/* ABI version (KS_ABI_VERSION) and a static build string. */
int ks_abi_version(void);
const char *ks_build_info(void);

/*
 * Memory plan of one fine mesh: the three region sizes ks_create needs (see "Memory").
 *   h_xyz, h_tets, h_dirichlet: as ks_create (host, read during the call); max_N: largest block of orbitals
 *   (1 <= max_N <= 64) any later call will use.
 *   *persistent_bytes: mesh, CSR pattern, scatter map and inverse, K, M, M_V, H, A values, sliced-ELL copies
 *                      (the context's lifetime);
 *   *workspace_bytes:  the block solver's vectors for N <= max_N plus call scratch (the context's lifetime);
 *   *setup_bytes:      temporaries of ks_create only (sort keys, geometry); may be freed after it returns.
 * The sizes come from a host count of the pattern (the definitions of SURVEY.md §8(c) items 1-3). Needs a CUDA
 * device (CUB temporary sizes). Errors: KS_E_ARG, KS_E_MESH (node index out of range, no free node), KS_E_CUDA;
 * the message is ks_last_error(NULL).
 */
ks_status ks_plan(int64_t n_nodes, const double *h_xyz, int64_t n_tets, const int32_t *h_tets,
                  const uint8_t *h_dirichlet, int32_t max_N, size_t *persistent_bytes, size_t *workspace_bytes,
                  size_t *setup_bytes);

/*
 * Setup of one fine mesh (section 2 of the paper; st3 PAPER.md:733-738).
 *   h_xyz       [n_nodes][3] f64 node coordinates (host)
 *   h_tets      [n_tets][4]  i32 node ids, positively oriented (host)
 *   h_dirichlet [n_nodes]    u8, nonzero = Dirichlet node (psi = 0 on dOmega)
 *   max_N       as passed to ks_plan
 *   d_persistent, d_workspace: caller-owned device regions of at least the planned sizes (context lifetime)
 *   d_setup     caller-owned region of setup_bytes, used only during this call; NULL = the workspace serves
 *               (then workspace_bytes >= setup_bytes is required)
 *   stream      cudaStream_t (NULL = legacy default stream) on the current device
 * On success *out is a new context; the call synchronises the stream (setup is not async).
 * Errors: KS_E_ARG, KS_E_MESH (first bad tet id in ks_last_error(NULL)), KS_E_WORKSPACE, KS_E_CUDA.
 * On error *out is NULL.
 */
ks_status ks_create(int64_t n_nodes, const double *h_xyz, int64_t n_tets, const int32_t *h_tets,
                    const uint8_t *h_dirichlet, int32_t max_N, void *d_persistent, size_t persistent_bytes,
                    void *d_workspace, size_t workspace_bytes, void *d_setup, size_t setup_bytes, void *stream,
                    ks_ctx **out);

/* Synchronises the stream and frees the host struct (the caller frees its regions afterwards). Safe on NULL. */
void ks_destroy(ks_ctx *ctx);

/* Re-targets the context to another stream (same device). Ordering: the new stream waits (event) for all
 * work already enqueued on the old stream, because both share the context's workspaces; work enqueued on
 * the new stream after this call therefore runs after it. */
ks_status ks_set_stream(ks_ctx *ctx, void *stream);

/* Sizes and read-only device views of the setup products (owned by the library). Any out-pointer may
 * be NULL. d_inv_ptr [nnz+1] / d_inv_idx [contributions] is the inverse scatter map: for nnz e the
 * entries d_inv_idx[d_inv_ptr[e] .. d_inv_ptr[e+1]) are the emap indices 16 t + 4 a + b that target e,
 * ascending. */
ks_status ks_pattern(const ks_ctx *ctx, int64_t *n_free, int64_t *nnz, const int32_t **d_row_ptr,
                     const int32_t **d_col, const int32_t **d_emap, const int32_t **d_free_of_node,
                     const int32_t **d_inv_ptr, const int32_t **d_inv_idx);

/* Device views of the value arrays [nnz] (CSR order of ks_pattern) and the diagonal of A [n_free]. MV, H, A,
 * diag are defined after the first ks_assemble_veff (KS_E_STATE before). The hot path keeps A and H in a
 * sliced-ELL layout; the CSR arrays MV, H, A are recomputed from the last assembly's state on the
 * context's stream when first requested after an assembly (one extra kernel; also by ks_spmm with
 * KS_OP_MV / KS_OP_H and by ks_true_residual). Synchronise the stream before reading them. */
ks_status ks_values(const ks_ctx *ctx, const double **d_K, const double **d_M, const double **d_MV,
                    const double **d_H, const double **d_A, const double **d_diag);

/*
 * (st4) reassembly, and the shifted operator of PAPER.md:553-561:
 *   (M_V)_ij = sum_T |T| (1+delta_ab) (V_a + V_b + S_T) / 120,  S_T = sum of V over the 4 vertices
 * (exact integral of the P1 interpolant of the nodal V), then H = 1/2 K + M_V, A = H + mu M, diag(A).
 *   d_veff [n_nodes] f64, ALL nodes (boundary values enter S_T).   mu >= 0 (shift).
 * Asynchronous. Deterministic (fixed summation order), no float atomics. Non-finite V latches
 * KS_E_NONFINITE (reported by ks_sync).
 */
ks_status ks_assemble_veff(ks_ctx *ctx, const double *d_veff, double mu);

/* Y = Op X for X, Y [n_free][N] f64 row-major (X != Y). Asynchronous. Parity / benchmarking helper. */
ks_status ks_spmm(ks_ctx *ctx, ks_op op, int32_t N, const double *d_X, double *d_Y);

/*
 * Algorithm 3 step 1 (Aux_Linear_Problem): for i = 0..N-1 independently solve
 *     A u~_i = (lambda_i + mu) M u_i,      A = H + mu M (from the last ks_assemble_veff)
 * by Jacobi-preconditioned CG from x0 = u_i, batched over the N columns in one persistent kernel:
 * per-column alpha/beta, a column stops when ||r||_2 <= tol ||b||_2 (recursive residual) and is frozen.
 *   d_lambda [N] f64, d_U [n_free][N] f64 (input), d_Ut [n_free][N] f64 (output, may not alias d_U)
 *   tol > 0, max_iter >= 1, 1 <= N <= max_N (ks_plan)
 *   d_iters [N] i32 (output, may be NULL): iterations applied to each column
 *   d_relres [N] f64 (output, may be NULL): recursive ||r||/||b|| at exit
 * Asynchronous; the status (NOT_SPD, NONFINITE, NOT_CONVERGED) is latched for ks_sync. The last iterate
 * is always written. Deterministic: fixed partition and reduction order, bitwise reproducible.
 */
ks_status ks_block_solve(ks_ctx *ctx, int32_t N, const double *d_lambda, const double *d_U, double *d_Ut,
                         double tol, int32_t max_iter, int32_t *d_iters, double *d_relres);

/* Number of block iterations (max over columns) of the last ks_block_solve; synchronises the stream. */
ks_status ks_last_iterations(ks_ctx *ctx, int32_t *h_block_iters);

/* Phase timestamps of the last ks_block_solve, for profiling. Recorded only when the environment variable
 * KS_PCG_TRACE=1 was set at that call: block 0 stamps %globaltimer (ns) at kernel start and after every
 * grid barrier, i.e. [start, init, then per iteration: S (q = Ap), U (r update), P (x, p update)].
 *   cap       capacity of h_ns;   h_ns [cap] u64 (host, output);   *h_count (host, output) = entries written
 *             (0 when tracing was off). Synchronises the stream. */
ks_status ks_solve_trace(ks_ctx *ctx, int32_t cap, uint64_t *h_ns, int32_t *h_count);

/* True relative residual ||(lambda_i+mu) M u_i - A u~_i|| / ||(lambda_i+mu) M u_i|| per column into
 * d_relres [N] (parity helper, one extra SpMM pass). Asynchronous. */
ks_status ks_true_residual(ks_ctx *ctx, int32_t N, const double *d_lambda, const double *d_U,
                           const double *d_Ut, double *d_relres);

/*
 * The interpolation operator P = I_H^h from the coarse space (Alg. 1, 747-753 st5):
 *   n_H coarse free nodes; d_P_row_ptr [n_free+1] i32, d_P_col [p_nnz] i32 (< n_H), d_P_val [p_nnz] f64.
 * ks_coarse_plan groups the fine rows by parent set (in the workspace's call scratch) and returns the size of
 * the coarse region; ks_set_coarse builds, in the caller's d_coarse region: the copy of P, the item tables,
 * the pattern of H P (window slots, also as an item-ordered sliced-ELL copy for the A_H pass), cached
 * B_H = P^T M P and the projection workspace for N <= max_N. Both synchronise the
 * stream. Requires n_H >= 1, at most 4 entries per row. A new coarse space detaches the extension workspace.
 */
ks_status ks_coarse_plan(ks_ctx *ctx, int64_t n_H, const int32_t *d_P_row_ptr, const int32_t *d_P_col,
                         const double *d_P_val, size_t *coarse_bytes);
ks_status ks_set_coarse(ks_ctx *ctx, int64_t n_H, const int32_t *d_P_row_ptr, const int32_t *d_P_col,
                        const double *d_P_val, void *d_coarse, size_t coarse_bytes);

/*
 * Extension workspace of the NEXT rows and the host-buffer steps: features = KS_EXT_* mask; max_D = largest
 * pencil dimension ks_pencil_eig will see (0: n_H + max_N, the projected pencil). Plan after ks_set_coarse
 * (the sizes depend on n_H); ks_attach_ext binds the caller's region (valid until the next ks_set_coarse or
 * ks_destroy). Calls that need a feature that is not attached return KS_E_STATE.
 */
ks_status ks_ext_plan(ks_ctx *ctx, uint32_t features, int64_t max_D, size_t *ext_bytes);
ks_status ks_attach_ext(ks_ctx *ctx, uint32_t features, int64_t max_D, void *d_ext, size_t ext_bytes);

/*
 * Projection onto W = [P | U~] (st1-st7), unshifted H (reading Q1):
 *   F_A = [[A_H, b_H], [b_H^T, beta]],  F_B = [[B_H, c_H], [c_H^T, gamma]]
 *   d_Ut [n_free][N] f64; d_FA, d_FB [(n_H+N)][(n_H+N)] f64 row-major, coarse block first.
 * Asynchronous, deterministic.
 */
ks_status ks_project_augmented(ks_ctx *ctx, int32_t N, const double *d_Ut, double *d_FA, double *d_FB);

/*
 * NEXT-1: the small eigenvalue problem of Algorithm 3 and the linear outer loop.
 *
 * ks_pencil_eig: lowest k eigenpairs of F_A y = lambda F_B y (Nonlinear_Eig_Hh on W; "a
 * small-scale algebraic eigenvalue problem solved in serial"), on the context's stream.
 * It reduces to standard form by Cholesky, then runs a Chebyshev-filtered subspace iteration on k + 8 vectors
 * when k + 8 <= D / 2 (its D x D by D x m products, Gram matrices and rotations are the library's
 * own kernels, the m x m eigenproblems run on the host, see ks_host_sym_eig; KS_PENCIL_DEVICE=1 runs the iteration
 * as one cooperative kernel with the Rayleigh-Ritz steps on the device). The fallback is the dense cuSOLVER
 * generalized symmetric eigensolver, which is always used when the environment variable KS_PENCIL_DENSE=1 is set.
 *   D = n_H + N >= 1, 1 <= k <= D; d_FA, d_FB [D][D] f64 symmetric (e.g. from ks_project_augmented), not
 *   modified; d_evals [k] f64 ascending; d_evecs [D][k] f64 row-major, column j = eigenvector j, normalised
 *   y^T F_B y = 1 (sign arbitrary). Synchronises the stream (reads the solver status).
 *   Errors: KS_E_ARG, KS_E_RANK (F_B not SPD), KS_E_NONFINITE (no convergence), KS_E_CUDA.
 */
ks_status ks_pencil_eig(ks_ctx *ctx, int64_t D, int32_t k, const double *d_FA, const double *d_FB,
                        double *d_evals, double *d_evecs);

/* The host routine behind the Rayleigh-Ritz steps of ks_pencil_eig's filtered iteration: all
 * eigenpairs of a small dense symmetric matrix. Host only: no context, no device work, callable without a GPU.
 *   n >= 1; h_A [n][n] f64 symmetric (host, not modified); h_w [n] f64 (host, output) ascending eigenvalues;
 *   h_V [n][n] f64 (host, output): h_V[j*n + i] = component i of eigenvector j, orthonormal.
 *   method 0: Householder tridiagonalisation + implicit QL (the default of the filtered iteration);
 *   method 1: cyclic Jacobi (its fallback, KS_EF_HOSTEIG=jacobi).
 *   Errors: KS_E_ARG (null pointer, n < 1, unknown method), KS_E_NOT_CONVERGED (QL iteration count ran out). */
ks_status ks_host_sym_eig(int32_t n, const double *h_A, double *h_w, double *h_V, int32_t method);

/*
 * ks_lift: the new orbitals in W (Algorithm 3: psi in S_H + span{psi~}):
 *   U_new[i][j] = sum_c P_ic Y[c][j] + sum_m U~[i][m] Y[n_H + m][j]
 *   d_Ut [n_free][N], d_Y [(n_H + N)][k], d_Unew [n_free][k] (may not alias d_Ut). Requires ks_set_coarse.
 *   Asynchronous.
 */
ks_status ks_lift(ks_ctx *ctx, int32_t N, const double *d_Ut, int32_t k, const double *d_Y, double *d_Unew);

/*
 * ks_augmented_solve: outer iterations of Algorithm 3 with the operators of the last ks_assemble_veff
 * (a fixed potential): ks_block_solve (tol_bvp, max_iter_bvp) -> ks_project_augmented
 * -> ks_pencil_eig (lowest N) -> ks_lift, repeated until max_j |lambda_j new - old| <= tol_eig max_j
 * |lambda_j| or max_outer iterations.
 *   d_lambda [N] (in: initial guesses, out: Ritz values), d_U [n_free][N] (in/out: orbitals), both updated
 *   in place; h_outer (host, may be NULL): iterations done; h_history (host, may be NULL) [max_outer][N]:
 *   the Ritz values of every iteration. Synchronises once per outer iteration.
 *   Errors: as the four calls; KS_E_NOT_CONVERGED if max_outer is reached (last iterate kept).
 */
ks_status ks_augmented_solve(ks_ctx *ctx, int32_t N, double *d_lambda, double *d_U, double tol_eig,
                             int32_t max_outer, double tol_bvp, int32_t max_iter_bvp, int32_t *h_outer,
                             double *h_history);

/*
 * NEXT-4 / SURVEY.md §8(e): the row-slab partition of ONE block solve over several processes (one GPU each;
 * the paper splits the BVPs over processes). The phases of the fused two-phase
 * Jacobi-PCG of ks_block_solve run as separate launches over one rank's contiguous rows [row0, row1); the
 * driver (paper_2404_19249_b200/slab.py) owns the partition (slab bounds balanced by nonzeros, halo ranges),
 * exchanges the halo rows of z between neighbouring ranks before every ks_slab_spmm and all-gathers the
 * per-column dots after every phase, summing them in rank order so all ranks derive the same alpha, beta.
 *   NP: padded block width (power of two, 1..64); every block d_* is [n_free][NP] f64 in the global row
 *   numbering (32-byte aligned for NP >= 4); a call reads the rows of d_U / d_Z referenced by its rows (own
 *   rows + halo) and writes only its own rows. d_lambda [NP] (pad entries 0). h_* coefficient arrays [NP]
 *   (host). d_dots: per-column sums over the rank's rows, [3][NP] (init: b.b, r.z, r.r), [NP] (spmm: p.q),
 *   [2][NP] (update: r.z, r.r), deterministic.
 *   ks_slab_init    b = (lambda+mu) M u, r = b - A u, z = r / d, p = z                (Aux_Linear_Problem)
 *   ks_slab_spmm    w = A z; q = w + beta q, p = z + beta p, x = xin + alpha_x p (first != 0: q = A z only)
 *   ks_slab_update  z -= alpha q / d
 *   ks_slab_finish  x = xin + alpha_x p
 * Asynchronous on the context's stream. Errors: KS_E_ARG (range, alignment), KS_E_STATE (not assembled).
 */
ks_status ks_slab_init(ks_ctx *ctx, int32_t NP, int64_t row0, int64_t row1, const double *d_lambda, const double *d_U,
                       double *d_Z, double *d_P, double *d_dots);
ks_status ks_slab_spmm(ks_ctx *ctx, int32_t NP, int64_t row0, int64_t row1, int32_t first, const double *h_alpha_x,
                       const double *h_beta, const double *d_Z, double *d_Q, double *d_P, const double *d_Xin,
                       double *d_X, double *d_dots);
ks_status ks_slab_update(ks_ctx *ctx, int32_t NP, int64_t row0, int64_t row1, const double *h_alpha, double *d_Z,
                         const double *d_Q, double *d_dots);
ks_status ks_slab_finish(ks_ctx *ctx, int32_t NP, int64_t row0, int64_t row1, const double *h_alpha_x,
                         const double *d_P, const double *d_Xin, double *d_X);

/*
 * NEXT-3: the nonnested interpolation operator P = I_H^h of Algorithm 1
 * from an independent coarse tet mesh (nonnested, possibly unstructured, covering the
 * fine mesh's domain): row i holds the barycentric coordinates of fine free node i in the coarse tet that
 * contains it, restricted to coarse FREE vertices (Dirichlet vertices carry zero data) with |lambda| > 1e-13,
 * sorted by coarse free index (coarse free index = rank of a non-Dirichlet coarse node, ascending id).
 *   h_xyz_c [n_c][3] f64, h_tets_c [m_c][4] i32, h_dirichlet_c [n_c] u8 (host, read during the call);
 *   d_work: caller-owned device scratch of at least ks_interpolation_plan's bytes (used during the call only);
 *   d_P_row_ptr [n_free+1] i32, d_P_col [4 n_free] i32, d_P_val [4 n_free] f64 (device, caller-owned outputs,
 *   ready for ks_set_coarse); *h_n_H = coarse free nodes, *h_p_nnz = entries written.
 * Synchronises the stream. Errors: KS_E_ARG, KS_E_MESH (degenerate coarse tet, node id out of range, or a fine
 * node outside the coarse mesh), KS_E_WORKSPACE, KS_E_CUDA.
 */
ks_status ks_interpolation_plan(ks_ctx *ctx, int64_t n_c, const double *h_xyz_c, int64_t m_c, size_t *work_bytes);
ks_status ks_interpolation(ks_ctx *ctx, int64_t n_c, const double *h_xyz_c, int64_t m_c, const int32_t *h_tets_c,
                           const uint8_t *h_dirichlet_c, void *d_work, size_t work_bytes, int32_t *d_P_row_ptr,
                           int32_t *d_P_col, double *d_P_val, int64_t *h_n_H, int64_t *h_p_nnz);

/*
 * NEXT-2: the nonlinear terms of the Kohn-Sham operator, on all nodes.
 * ks_density: rho(x_v) = f sum_j psi_j(x_v)^2 (f = occupation per orbital, 2 for the
 *   paper's closed shells, reading R6); d_U [n_free][N]; d_rho [n_nodes] (0 on Dirichlet nodes).
 * ks_vxc: LDA exchange -(3 rho / pi)^(1/3) + Perdew-Zunger correlation (Eqs. expot, copot,
 *   PAPER.md:330-362) -> d_vxc [n_nodes]; d_eps [n_nodes] (may be NULL) = eps_x + eps_c, the
 *   exchange-correlation energy per electron; rho <= 0 gives 0.
 * Asynchronous.
 */
ks_status ks_density(ks_ctx *ctx, int32_t N, const double *d_U, double f, double *d_rho);
ks_status ks_vxc(ks_ctx *ctx, const double *d_rho, double *d_vxc, double *d_eps);

/*
 * ks_hartree: the Hartree potential: -Lap V = 4 pi rho, V = w_D on the boundary with the
 * multipole expansion of Eq. bd about the centre of charge (monopole, dipole, quadrupole with the 1/2 of the
 * Taylor term, reading R5; moments exact for the P1 density); P1 Galerkin with the Dirichlet lift,
 * the free values by a preconditioned CG on the stiffness matrix to ||r|| <= tol ||b||. When a coarse
 * space is set (ks_set_coarse), the preconditioner is two-level: Jacobi + P (P^T K P)^-1 P^T, with the
 * coarse operator built and Cholesky-inverted on the first call after ks_set_coarse. That is NEXT-4
 * (DESIGN.md §8.4); it falls back to Jacobi if P^T K P is not SPD. Without a coarse space, or with the
 * environment variable KS_HARTREE_2L=0, it is the batched Jacobi-PCG (N = 1).
 *   d_rho [n_nodes]; d_vh [n_nodes] (out: free values and w_D; in when warm != 0: the warm start);
 *   h_mom [10] (host, may be NULL): Q, centre (3), dipole (3), diagonal of the second moment (3);
 *   h_iters (host, may be NULL): PCG iterations. Synchronises the stream when h_mom or h_iters is given.
 *   Latches KS_E_NOT_CONVERGED (ks_sync) when max_iter is reached.
 */
ks_status ks_hartree(ks_ctx *ctx, const double *d_rho, double tol, int32_t max_iter, double *d_vh, int32_t warm,
                     double *h_mom, int32_t *h_iters);

/*
 * ks_scf_solve: Algorithm 3 for the Kohn-Sham equation on the context's mesh and coarse
 * space (ks_set_coarse), with Anderson mixing:
 *   outer: V_eff = V_ext + V_Har[rho] + V_xc[rho] -> ks_assemble_veff(V_eff, mu) -> the N BVPs from
 *          (lambda, Psi) -> Psi~;
 *   inner (the small Kohn-Sham equation on S_H + span{Psi~}, self-consistent with Psi~ fixed, at most `inner`
 *          steps; reading R8): projection -> pencil eig -> lift -> rho_out = f sum psi^2; stop when
 *          ||rho_out - rho_in||_M <= inner_tol ||rho_out||_M, else Anderson-mix (depth <= 7, beta) and
 *          reassemble with the mixed density;
 *   stop when the outer density change ||rho^(l) - rho^(l-1)||_M <= tol ||rho^(l)||_M.
 *   d_vext [n_nodes] (the external potential, e.g. smoothed Coulomb); f occupation per orbital; mu shift;
 *   d_lambda [N], d_U [n_free][N] (in: initial, out: converged); host outputs (may be NULL): h_outer,
 *   h_inner [max_outer] inner steps, h_dres [max_outer] outer density changes, h_lams [max_outer][N].
 *   Synchronises. Errors: as the calls it makes; KS_E_NOT_CONVERGED after max_outer (last iterate kept).
 */
ks_status ks_scf_solve(ks_ctx *ctx, int32_t N, const double *d_vext, double f, double mu, double *d_lambda,
                       double *d_U, double tol, int32_t max_outer, int32_t inner, double inner_tol, double beta,
                       int32_t depth, double bvp_tol, double hartree_tol, int32_t *h_outer, int32_t *h_inner,
                       double *h_dres, double *h_lams);

/*
 * The hot-path step from HOST buffers, pipelined. ks_step_submit enqueues one step: copy V_eff [n_nodes],
 * lambda [N], U [n_free][N] from host memory (pinned for asynchronous copies), ks_assemble_veff(V_eff, mu),
 * ks_block_solve(tol, max_iter), ks_project_augmented, and copy F_A, F_B [(n_H+N)^2] to host memory. It
 * returns without waiting. Consecutive steps alternate between two device slots; input copies run on an
 * internal host-to-device stream and result copies on an internal device-to-host stream, ordered against the
 * context's stream by events, so the input copy of one step overlaps the compute of the previous one.
 * The caller must not modify a step's host inputs, or read its outputs, before ks_step_wait returns.
 * ks_step_wait waits for every submitted step. Device-detected conditions are reported by ks_sync.
 */
ks_status ks_step_submit(ks_ctx *ctx, int32_t N, const double *h_V, double mu, const double *h_lambda,
                         const double *h_U, double tol, int32_t max_iter, double *h_FA, double *h_FB);
ks_status ks_step_wait(ks_ctx *ctx);

/* Bytes of caller memory the context currently references (sum of the bound regions' sizes). */
ks_status ks_memory_bytes(const ks_ctx *ctx, size_t *bytes);
/* Capacity, bytes in use and peak use of one region: 0 persistent, 1 workspace, 3 coarse, 4 extension
 * (2 setup and 5 call scratch are unbound after their call). Any out-pointer may be NULL. */
ks_status ks_memory_usage(const ks_ctx *ctx, int32_t region, size_t *capacity, size_t *used, size_t *peak);

/* Number of kernel launches issued by this context since creation (for the bench's gpu_launches). */
ks_status ks_launch_count(const ks_ctx *ctx, int64_t *count);

/* Synchronises the stream, clears and returns the latched device status (worst condition seen since
 * the previous ks_sync): KS_OK, KS_E_NONFINITE, KS_E_NOT_SPD, KS_E_NOT_CONVERGED, or KS_E_CUDA. */
ks_status ks_sync(ks_ctx *ctx);

/* Message of the last failure on ctx (or of the last failed ks_create when ctx is NULL). */
const char *ks_last_error(const ks_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* KS_H_ */
