/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY. A plain, slow, single-threaded CPU implementation of the
 * hot path of the nonnested augmented subspace method (arXiv 2404.19249). It exists to check the
 * CUDA library (paper_2404_19249_b200/csrc) element by element. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it. It shares no code, header,
 * table or helper with the CUDA path.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (no fast-math; no OpenMP).
 *
 * Every function follows a passage of /root/reference/PAPER.md ("PAPER.md:L"), with the readings
 * of SURVEY.md §8c / DESIGN.md §2 where the paper is silent:
 *   or_create          P1 space S_h in H^1_0 on a tet mesh, Dirichlet elimination (
 *                      readings Q3, pattern item 2), element-to-nnz map,
 *                      stiffness and mass of (st3).
 *   or_assemble_veff   V_eff-weighted mass (st4), H = 1/2 K + M_V, shifted
 *                      operator A = H + mu M of H~.
 *   or_spmm            Y = Op X for a block of vectors (definition).
 *   or_block_pcg       N independent BVPs (Aux_Linear_Problem) by textbook
 *                      Jacobi-preconditioned CG, one column at a time (reading Q6, Q7).
 *   or_project         F_A, F_B of (st1)-(st2) with A_H = P^T H P (st5), b_H = P^T H U~ (st6),
 *                      beta = U~^T H U~ (st7), and the mass counterparts B_H, c_H, gamma
 *                      (readings Q1, Q4).
 * Pinning: every function is pinned in tests/test_oracle_*.py against closed forms, invariants and
 * brute-force dense solves (no function here is "parity unpinned").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>

enum { OR_OK = 0, OR_E_ARG = 1, OR_E_MESH = 2, OR_E_NONFINITE = 3, OR_E_NOT_SPD = 4,
       OR_E_NOT_CONVERGED = 5, OR_E_NOMEM = 6 };

typedef struct {
  int64_t n_nodes, n_tets, n_free, nnz;
  int32_t *free_of_node;   /* [n_nodes], -1 on Dirichlet nodes */
  int32_t *node_of_free;   /* [n_free] */
  int64_t *row_ptr;        /* [n_free+1] */
  int32_t *col;            /* [nnz], sorted within each row */
  int32_t *emap;           /* [16*n_tets]: emap[16t+4a+b] = CSR position of (free(v_a), free(v_b)) or -1 */
  int32_t *tets;           /* copy [4*n_tets] */
  double *vol;             /* [n_tets] |T| */
  double *grad;            /* [12*n_tets] grad lambda_a, a=0..3 */
  double *K, *M, *MV, *H, *A, *diag; /* [nnz], [nnz], ..., diag [n_free] */
  double mu;               /* shift used by the last or_assemble_veff */
  char err[256];
} or_mesh;

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

void or_destroy(or_mesh *h) {
  if (!h) return;
  free(h->free_of_node); free(h->node_of_free); free(h->row_ptr); free(h->col); free(h->emap);
  free(h->tets); free(h->vol); free(h->grad); free(h->K); free(h->M); free(h->MV); free(h->H);
  free(h->A); free(h->diag);
  free(h);
}

const char *or_last_error(const or_mesh *h) { return h ? h->err : "null handle"; }

/* position of column c in row r (binary search over the sorted row), -1 if absent */
static int64_t find_in_row(const or_mesh *h, int64_t r, int32_t c) {
  int64_t lo = h->row_ptr[r], hi = h->row_ptr[r + 1] - 1;
  while (lo <= hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (h->col[mid] == c) return mid;
    if (h->col[mid] < c) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

/*
 * Geometry of one tet (PAPER.md:256-261, P1 on a shape-regular tet mesh):
 * J = [x1-x0, x2-x0, x3-x0] (columns); |T| = det(J)/6 must be > 0.
 * grad lambda_a (a=1..3) are the rows of J^{-1}; grad lambda_0 = -(sum of the others).
 */
static int tet_geometry(const double *xyz, const int32_t *v, double *vol, double g[4][3]) {
  double J[3][3];
  for (int c = 0; c < 3; c++)
    for (int r = 0; r < 3; r++) J[r][c] = xyz[3 * v[c + 1] + r] - xyz[3 * v[0] + r];
  double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1])
             - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0])
             + J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
  if (!(det > 0.0)) return 0;
  /* inverse = adj(J)/det; row a of J^{-1} is grad lambda_{a+1} */
  double inv[3][3];
  inv[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
  inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
  inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
  inv[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
  inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
  inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
  inv[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
  inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
  inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
  for (int a = 0; a < 3; a++)
    for (int d = 0; d < 3; d++) g[a + 1][d] = inv[a][d];
  for (int d = 0; d < 3; d++) g[0][d] = -(g[1][d] + g[2][d] + g[3][d]);
  *vol = det / 6.0;
  return 1;
}

/*
 * Build the P1 discretization on the fine mesh:
 *  1. free[v] = rank of v among non-Dirichlet nodes (Dirichlet elimination, PAPER.md:1120 psi=0 on dOmega).
 *  2. CSR pattern over free nodes: row i lists the sorted unique free(w) with w sharing a tet with i
 *     (diagonal included); nothing beyond the FEM stencil.
 *  3. emap[16t+4a+b] = CSR position of (free(v_a), free(v_b)) or -1 (element-to-nnz scatter map).
 *  4. |T| and grad lambda_a per tet.
 *  5. K_ij = sum_T |T| grad l_a . grad l_b,  M_ij = sum_T |T|(1+delta_ab)/20  (st3),
 *     accumulated val[emap] += elem(a,b) for t ascending, then a, then b.
 * Returns NULL only on allocation failure; *status reports mesh errors (inverted tet id in err).
 */
or_mesh *or_create(int64_t n_nodes, const double *xyz, int64_t n_tets, const int32_t *tets,
                   const uint8_t *dirichlet, int *status) {
  or_mesh *h = (or_mesh *)calloc(1, sizeof(or_mesh));
  if (!h) { *status = OR_E_NOMEM; return NULL; }
  *status = OR_OK;
  h->n_nodes = n_nodes; h->n_tets = n_tets;

  /* 1. free numbering */
  h->free_of_node = (int32_t *)malloc(sizeof(int32_t) * (n_nodes > 0 ? n_nodes : 1));
  int64_t nf = 0;
  for (int64_t v = 0; v < n_nodes; v++) h->free_of_node[v] = dirichlet[v] ? -1 : (int32_t)(nf++);
  h->n_free = nf;
  h->node_of_free = (int32_t *)malloc(sizeof(int32_t) * (nf > 0 ? nf : 1));
  for (int64_t v = 0; v < n_nodes; v++) if (!dirichlet[v]) h->node_of_free[h->free_of_node[v]] = (int32_t)v;

  for (int64_t t = 0; t < 4 * n_tets; t++)
    if (tets[t] < 0 || tets[t] >= n_nodes) {
      snprintf(h->err, sizeof h->err, "tet %lld has node index %d out of range", (long long)(t / 4), tets[t]);
      *status = OR_E_MESH; return h;
    }
  h->tets = (int32_t *)malloc(sizeof(int32_t) * 4 * (n_tets > 0 ? n_tets : 1));
  memcpy(h->tets, tets, sizeof(int32_t) * 4 * n_tets);

  /* 2. pattern: node -> incident tets, then per free row collect, sort, unique */
  int64_t *inc_ptr = (int64_t *)calloc(n_nodes + 1, sizeof(int64_t));
  for (int64_t t = 0; t < n_tets; t++)
    for (int a = 0; a < 4; a++) inc_ptr[tets[4 * t + a] + 1]++;
  for (int64_t v = 0; v < n_nodes; v++) inc_ptr[v + 1] += inc_ptr[v];
  int32_t *inc = (int32_t *)malloc(sizeof(int32_t) * (4 * n_tets > 0 ? 4 * n_tets : 1));
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (n_nodes > 0 ? n_nodes : 1));
  for (int64_t v = 0; v < n_nodes; v++) fill[v] = inc_ptr[v];
  for (int64_t t = 0; t < n_tets; t++)
    for (int a = 0; a < 4; a++) inc[fill[tets[4 * t + a]]++] = (int32_t)t;
  free(fill);

  h->row_ptr = (int64_t *)malloc(sizeof(int64_t) * (nf + 1));
  h->row_ptr[0] = 0;
  int32_t *buf = NULL; int64_t bufcap = 0;
  /* first pass: counts */
  for (int pass = 0; pass < 2; pass++) {
    for (int64_t i = 0; i < nf; i++) {
      int64_t v = h->node_of_free[i];
      int64_t deg = inc_ptr[v + 1] - inc_ptr[v];
      if (4 * deg > bufcap) { bufcap = 4 * deg; buf = (int32_t *)realloc(buf, sizeof(int32_t) * bufcap); }
      int64_t m = 0;
      for (int64_t e = inc_ptr[v]; e < inc_ptr[v + 1]; e++) {
        int64_t t = inc[e];
        for (int a = 0; a < 4; a++) {
          int32_t f = h->free_of_node[tets[4 * t + a]];
          if (f >= 0) buf[m++] = f;
        }
      }
      qsort(buf, (size_t)m, sizeof(int32_t), cmp_i32);
      int64_t u = 0;
      for (int64_t k = 0; k < m; k++) if (u == 0 || buf[k] != buf[u - 1]) buf[u++] = buf[k];
      if (pass == 0) h->row_ptr[i + 1] = h->row_ptr[i] + u;
      else memcpy(h->col + h->row_ptr[i], buf, sizeof(int32_t) * u);
    }
    if (pass == 0) {
      h->nnz = h->row_ptr[nf];
      h->col = (int32_t *)malloc(sizeof(int32_t) * (h->nnz > 0 ? h->nnz : 1));
    }
  }
  free(buf); free(inc); free(inc_ptr);

  /* 3. element-to-nnz scatter map */
  h->emap = (int32_t *)malloc(sizeof(int32_t) * 16 * (n_tets > 0 ? n_tets : 1));
  for (int64_t t = 0; t < n_tets; t++)
    for (int a = 0; a < 4; a++)
      for (int b = 0; b < 4; b++) {
        int32_t fa = h->free_of_node[tets[4 * t + a]], fb = h->free_of_node[tets[4 * t + b]];
        h->emap[16 * t + 4 * a + b] = (fa >= 0 && fb >= 0) ? (int32_t)find_in_row(h, fa, fb) : -1;
      }

  /* 4. geometry */
  h->vol = (double *)malloc(sizeof(double) * (n_tets > 0 ? n_tets : 1));
  h->grad = (double *)malloc(sizeof(double) * 12 * (n_tets > 0 ? n_tets : 1));
  for (int64_t t = 0; t < n_tets; t++) {
    double g[4][3];
    if (!tet_geometry(xyz, tets + 4 * t, &h->vol[t], g)) {
      snprintf(h->err, sizeof h->err, "tet %lld is inverted or degenerate", (long long)t);
      *status = OR_E_MESH; return h;
    }
    for (int a = 0; a < 4; a++) for (int d = 0; d < 3; d++) h->grad[12 * t + 3 * a + d] = g[a][d];
  }

  /* 5. K and M values */
  size_t nb = sizeof(double) * (h->nnz > 0 ? h->nnz : 1);
  h->K = (double *)calloc(1, nb); h->M = (double *)calloc(1, nb);
  h->MV = (double *)calloc(1, nb); h->H = (double *)calloc(1, nb); h->A = (double *)calloc(1, nb);
  h->diag = (double *)calloc(nf > 0 ? nf : 1, sizeof(double));
  for (int64_t t = 0; t < n_tets; t++) {
    const double *g = h->grad + 12 * t;
    for (int a = 0; a < 4; a++)
      for (int b = 0; b < 4; b++) {
        int32_t e = h->emap[16 * t + 4 * a + b];
        if (e < 0) continue;
        double dot = g[3 * a] * g[3 * b] + g[3 * a + 1] * g[3 * b + 1] + g[3 * a + 2] * g[3 * b + 2];
        h->K[e] += h->vol[t] * dot;
        h->M[e] += h->vol[t] * (a == b ? 2.0 : 1.0) / 20.0;
      }
  }
  return h;
}

void or_sizes(const or_mesh *h, int64_t *n_free, int64_t *nnz) { *n_free = h->n_free; *nnz = h->nnz; }

/* copy-out accessors (row_ptr as int64) */
void or_get_pattern(const or_mesh *h, int64_t *row_ptr, int32_t *col, int32_t *emap, int32_t *free_of_node) {
  if (row_ptr) memcpy(row_ptr, h->row_ptr, sizeof(int64_t) * (h->n_free + 1));
  if (col) memcpy(col, h->col, sizeof(int32_t) * h->nnz);
  if (emap) memcpy(emap, h->emap, sizeof(int32_t) * 16 * h->n_tets);
  if (free_of_node) memcpy(free_of_node, h->free_of_node, sizeof(int32_t) * h->n_nodes);
}

void or_get_values(const or_mesh *h, double *K, double *M, double *MV, double *H, double *A, double *diag,
                   double *vol) {
  size_t nb = sizeof(double) * h->nnz;
  if (K) memcpy(K, h->K, nb);
  if (M) memcpy(M, h->M, nb);
  if (MV) memcpy(MV, h->MV, nb);
  if (H) memcpy(H, h->H, nb);
  if (A) memcpy(A, h->A, nb);
  if (diag) memcpy(diag, h->diag, sizeof(double) * h->n_free);
  if (vol) memcpy(vol, h->vol, sizeof(double) * h->n_tets);
}

/*
 * (st4) nonlinear part: (M_V)_ij = ((V_Har+V_xc) phi_i, phi_j), here for a nodal P1
 * potential V (all nodes, boundary included). The exact element integral of the P1 interpolant
 * V = sum_k V_k lambda_k against lambda_a lambda_b, from int_T lambda^alpha = 3! alpha! |T| / (3+|alpha|)!:
 *     MV_T(a,b) = |T| (1 + delta_ab) (V_a + V_b + S_T) / 120,   S_T = sum_{k in T} V_k   (reading Q2).
 * Accumulated through emap for t ascending, then a, then b. Then H = 1/2 K + M_V and the shifted
 * operator A = H + mu M (H~ of PAPER.md:553-561), diag = diag(A) (Jacobi preconditioner).
 * Returns OR_E_NONFINITE if any V is not finite (values are still computed).
 */
int or_assemble_veff(or_mesh *h, const double *V, double mu) {
  int st = OR_OK;
  for (int64_t v = 0; v < h->n_nodes; v++) if (!isfinite(V[v])) { st = OR_E_NONFINITE; break; }
  memset(h->MV, 0, sizeof(double) * h->nnz);
  h->mu = mu;
  for (int64_t t = 0; t < h->n_tets; t++) {
    const int32_t *v = h->tets + 4 * t;
    double S = V[v[0]] + V[v[1]] + V[v[2]] + V[v[3]];
    for (int a = 0; a < 4; a++)
      for (int b = 0; b < 4; b++) {
        int32_t e = h->emap[16 * t + 4 * a + b];
        if (e < 0) continue;
        h->MV[e] += h->vol[t] * (a == b ? 2.0 : 1.0) * (V[v[a]] + V[v[b]] + S) / 120.0;
      }
  }
  for (int64_t e = 0; e < h->nnz; e++) {
    h->H[e] = 0.5 * h->K[e] + h->MV[e];
    h->A[e] = h->H[e] + mu * h->M[e];
  }
  for (int64_t i = 0; i < h->n_free; i++) h->diag[i] = h->A[find_in_row(h, i, (int32_t)i)];
  return st;
}

static const double *pick(const or_mesh *h, int which) {
  switch (which) { case 0: return h->K; case 1: return h->M; case 2: return h->MV;
                   case 3: return h->H; case 4: return h->A; default: return NULL; }
}

/* Y = Op X, X and Y are [n_free][N] row-major. which: 0 K, 1 M, 2 MV, 3 H, 4 A. */
int or_spmm(const or_mesh *h, int which, int N, const double *X, double *Y) {
  const double *val = pick(h, which);
  if (!val || N < 1) return OR_E_ARG;
  for (int64_t i = 0; i < h->n_free; i++)
    for (int c = 0; c < N; c++) {
      double s = 0.0;
      for (int64_t k = h->row_ptr[i]; k < h->row_ptr[i + 1]; k++) s += val[k] * X[(int64_t)h->col[k] * N + c];
      Y[i * N + c] = s;
    }
  return OR_OK;
}

static double dot_n(const double *a, const double *b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; i++) s += a[i] * b[i];
  return s;
}

static void matvec(const or_mesh *h, const double *val, const double *x, double *y) {
  for (int64_t i = 0; i < h->n_free; i++) {
    double s = 0.0;
    for (int64_t k = h->row_ptr[i]; k < h->row_ptr[i + 1]; k++) s += val[k] * x[h->col[k]];
    y[i] = s;
  }
}

/*
 * Algorithm 3, first step (Eq. Aux_Linear_Problem): for i = 1..N independently,
 *     (H~ psi^_i, v) = (lambda_i + mu)(psi_i, v)  for all v in S_h,
 * i.e. A u~_i = b_i with A = H + mu M and b_i = (lambda_i + mu) M u_i. Solved by textbook
 * Jacobi-preconditioned CG (readings Q6, Q7): x0 = u_i, r0 = b - A x0, z = D^{-1} r, p = z;
 * loop: stop when ||r||_2 <= tol ||b||_2; q = A p; if p.q <= 0 -> NOT_SPD; alpha = r.z / p.q;
 * x += alpha p; r -= alpha q; z = D^{-1} r; beta = r.z_new / r.z_old; p = z + beta p.
 * iters[i] = completed updates; relres_rec[i] = ||r||/||b|| (recursive), relres_true[i] =
 * ||b - A x||/||b||. Returns the worst status over the columns.
 */
int or_block_pcg(const or_mesh *h, int N, const double *lambda, const double *U, double *Ut,
                 double tol, int max_iter, int32_t *iters, double *relres_rec, double *relres_true) {
  int64_t n = h->n_free;
  double mu = h->mu;
  int worst = OR_OK;
  double *u = (double *)malloc(sizeof(double) * n), *x = (double *)malloc(sizeof(double) * n);
  double *b = (double *)malloc(sizeof(double) * n), *r = (double *)malloc(sizeof(double) * n);
  double *z = (double *)malloc(sizeof(double) * n), *p = (double *)malloc(sizeof(double) * n);
  double *q = (double *)malloc(sizeof(double) * n);
  for (int c = 0; c < N; c++) {
    int st = OR_OK;
    for (int64_t i = 0; i < n; i++) u[i] = U[i * N + c];
    matvec(h, h->M, u, b);
    for (int64_t i = 0; i < n; i++) b[i] *= (lambda[c] + mu);
    matvec(h, h->A, u, q);
    for (int64_t i = 0; i < n; i++) { x[i] = u[i]; r[i] = b[i] - q[i]; z[i] = r[i] / h->diag[i]; p[i] = z[i]; }
    double bnorm = sqrt(dot_n(b, b, n));
    double rz = dot_n(r, z, n);
    int it = 0;
    for (;;) {
      double rnorm = sqrt(dot_n(r, r, n));
      if (!isfinite(rnorm) || !isfinite(bnorm)) { st = OR_E_NONFINITE; break; }
      if (rnorm <= tol * bnorm) break;
      if (it >= max_iter) { st = OR_E_NOT_CONVERGED; break; }
      matvec(h, h->A, p, q);
      double pq = dot_n(p, q, n);
      if (!(pq > 0.0)) { st = OR_E_NOT_SPD; break; }
      double alpha = rz / pq;
      for (int64_t i = 0; i < n; i++) { x[i] += alpha * p[i]; r[i] -= alpha * q[i]; z[i] = r[i] / h->diag[i]; }
      double rz_new = dot_n(r, z, n);
      double beta = rz_new / rz;
      rz = rz_new;
      for (int64_t i = 0; i < n; i++) p[i] = z[i] + beta * p[i];
      it++;
    }
    iters[c] = it;
    relres_rec[c] = bnorm > 0.0 ? sqrt(dot_n(r, r, n)) / bnorm : sqrt(dot_n(r, r, n));
    matvec(h, h->A, x, q);
    for (int64_t i = 0; i < n; i++) q[i] = b[i] - q[i];
    relres_true[c] = bnorm > 0.0 ? sqrt(dot_n(q, q, n)) / bnorm : sqrt(dot_n(q, q, n));
    for (int64_t i = 0; i < n; i++) Ut[i * N + c] = x[i];
    if (st > worst) worst = st;
  }
  free(u); free(x); free(b); free(r); free(z); free(p); free(q);
  return worst;
}

/*
 * Projection onto the augmented subspace W = [P | U~]:
 *   F_A = [[A_H, b_H], [b_H^T, beta]],  F_B = [[B_H, c_H], [c_H^T, gamma]]     (st1-st2)
 *   A_H = P^T H P (st5), b_H = P^T H U~ (st6), beta = U~^T H U~ (st7),
 *   B_H = P^T M P, c_H = P^T M U~, gamma = U~^T M U~        (reading Q4)
 * with the unshifted H = 1/2 K + M_V (reading Q1). P: n_free x n_H CSR. F_* row-major
 * [(n_H+N)][(n_H+N)], coarse block first. Plain loops over the definitions.
 */
int or_project(const or_mesh *h, int64_t n_H, const int32_t *Pptr, const int32_t *Pcol, const double *Pval,
               int N, const double *Ut, double *FA, double *FB) {
  int64_t n = h->n_free, D = n_H + N;
  double *HU = (double *)calloc(n * N > 0 ? n * N : 1, sizeof(double));
  double *MU = (double *)calloc(n * N > 0 ? n * N : 1, sizeof(double));
  or_spmm(h, 3, N, Ut, HU);
  or_spmm(h, 1, N, Ut, MU);
  memset(FA, 0, sizeof(double) * D * D);
  memset(FB, 0, sizeof(double) * D * D);
  /* A_H[c][d] = sum_i sum_j P_ic H_ij P_jd ; B_H with M */
  for (int64_t i = 0; i < n; i++)
    for (int64_t k = h->row_ptr[i]; k < h->row_ptr[i + 1]; k++) {
      int64_t j = h->col[k];
      for (int32_t s = Pptr[i]; s < Pptr[i + 1]; s++)
        for (int32_t t = Pptr[j]; t < Pptr[j + 1]; t++) {
          int64_t c = Pcol[s], d = Pcol[t];
          FA[c * D + d] += Pval[s] * h->H[k] * Pval[t];
          FB[c * D + d] += Pval[s] * h->M[k] * Pval[t];
        }
    }
  /* b_H[c][a] = sum_i P_ic (H U~)_ia ; c_H with M */
  for (int64_t i = 0; i < n; i++)
    for (int32_t s = Pptr[i]; s < Pptr[i + 1]; s++)
      for (int a = 0; a < N; a++) {
        FA[(int64_t)Pcol[s] * D + n_H + a] += Pval[s] * HU[i * N + a];
        FB[(int64_t)Pcol[s] * D + n_H + a] += Pval[s] * MU[i * N + a];
      }
  for (int64_t c = 0; c < n_H; c++)
    for (int a = 0; a < N; a++) {
      FA[(n_H + a) * D + c] = FA[c * D + n_H + a];
      FB[(n_H + a) * D + c] = FB[c * D + n_H + a];
    }
  /* beta[a][b] = sum_i U~_ia (H U~)_ib ; gamma with M */
  for (int a = 0; a < N; a++)
    for (int b = 0; b < N; b++) {
      double sa = 0.0, sb = 0.0;
      for (int64_t i = 0; i < n; i++) { sa += Ut[i * N + a] * HU[i * N + b]; sb += Ut[i * N + a] * MU[i * N + b]; }
      FA[(n_H + a) * D + n_H + b] = sa;
      FB[(n_H + a) * D + n_H + b] = sb;
    }
  free(HU); free(MU);
  return OR_OK;
}

/*
 * NEXT-1: the small eigenvalue problem of Algorithm 3 and the lift of its eigenvectors.
 *
 * or_pencil_eig: the generalized symmetric eigenproblem of (Nonlinear_Eig_Hh) restricted to W,
 * F_A y = lambda F_B y, "a small-scale algebraic eigenvalue problem solved in
 * serial". Textbook reduction: Cholesky F_B = L L^T (F_B must be SPD), C = L^-1 F_A L^-T,
 * cyclic Jacobi rotations on C until every off-diagonal |c_pq| <= 1e-15 sqrt(|c_pp c_qq|) (or 100 sweeps),
 * eigenvalues sorted ascending, eigenvectors y = L^-T z (then F_B-orthonormal). The lowest k are returned:
 * evals [k], evecs [D][k] row-major (column j = eigenvector j).
 * Returns OR_OK, OR_E_NOT_SPD when the Cholesky factorisation of F_B breaks down, OR_E_NOMEM.
 */
int or_pencil_eig(int64_t D, const double *FA, const double *FB, int k, double *evals, double *evecs) {
  if (D < 1 || k < 1 || k > D) return OR_E_ARG;
  double *L = (double *)calloc(D * D, sizeof(double));
  double *C = (double *)calloc(D * D, sizeof(double));
  double *Z = (double *)calloc(D * D, sizeof(double));
  double *T = (double *)calloc(D * D, sizeof(double));
  int64_t *ord = (int64_t *)calloc(D, sizeof(int64_t));
  if (!L || !C || !Z || !T || !ord) { free(L); free(C); free(Z); free(T); free(ord); return OR_E_NOMEM; }
  /* Cholesky (lower), F_B symmetric: use the lower triangle */
  for (int64_t j = 0; j < D; j++) {
    double s = FB[j * D + j];
    for (int64_t m = 0; m < j; m++) s -= L[j * D + m] * L[j * D + m];
    if (!(s > 0.0)) { free(L); free(C); free(Z); free(T); free(ord); return OR_E_NOT_SPD; }
    L[j * D + j] = sqrt(s);
    for (int64_t i = j + 1; i < D; i++) {
      double t = FB[i * D + j];
      for (int64_t m = 0; m < j; m++) t -= L[i * D + m] * L[j * D + m];
      L[i * D + j] = t / L[j * D + j];
    }
  }
  /* T = L^-1 F_A (forward substitution, column by column of F_A) */
  for (int64_t c = 0; c < D; c++)
    for (int64_t i = 0; i < D; i++) {
      double t = FA[i * D + c];
      for (int64_t m = 0; m < i; m++) t -= L[i * D + m] * T[m * D + c];
      T[i * D + c] = t / L[i * D + i];
    }
  /* C = T L^-T, i.e. C^T = L^-1 T^T: row r of C solves L x = (row r of T)^T */
  for (int64_t r = 0; r < D; r++)
    for (int64_t i = 0; i < D; i++) {
      double t = T[r * D + i];
      for (int64_t m = 0; m < i; m++) t -= L[i * D + m] * C[r * D + m];
      C[r * D + i] = t / L[i * D + i];
    }
  /* symmetrise (rounding) and run cyclic Jacobi: C = Z diag Z^T */
  for (int64_t i = 0; i < D; i++)
    for (int64_t j = i + 1; j < D; j++) {
      double a = 0.5 * (C[i * D + j] + C[j * D + i]);
      C[i * D + j] = C[j * D + i] = a;
    }
  for (int64_t i = 0; i < D; i++) Z[i * D + i] = 1.0;
  for (int sweep = 0; sweep < 100; sweep++) {
    int rotated = 0;
    for (int64_t p = 0; p < D - 1; p++)
      for (int64_t q = p + 1; q < D; q++) {
        double apq = C[p * D + q], app = C[p * D + p], aqq = C[q * D + q];
        if (fabs(apq) <= 1e-15 * sqrt(fabs(app * aqq)) || apq == 0.0) continue;
        rotated = 1;
        /* rotation angle: tan(2 theta) = 2 apq / (aqq - app), smaller root (Golub & Van Loan 8.5.2) */
        double tau = (aqq - app) / (2.0 * apq);
        double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
        for (int64_t r = 0; r < D; r++) {   /* columns p, q */
          double crp = C[r * D + p], crq = C[r * D + q];
          C[r * D + p] = c * crp - s * crq;
          C[r * D + q] = s * crp + c * crq;
        }
        for (int64_t r = 0; r < D; r++) {   /* rows p, q */
          double cpr = C[p * D + r], cqr = C[q * D + r];
          C[p * D + r] = c * cpr - s * cqr;
          C[q * D + r] = s * cpr + c * cqr;
        }
        C[p * D + q] = C[q * D + p] = 0.0;
        for (int64_t r = 0; r < D; r++) {
          double zrp = Z[r * D + p], zrq = Z[r * D + q];
          Z[r * D + p] = c * zrp - s * zrq;
          Z[r * D + q] = s * zrp + c * zrq;
        }
      }
    if (!rotated) break;
  }
  /* ascending order (insertion sort of indices, ties by index) */
  for (int64_t i = 0; i < D; i++) ord[i] = i;
  for (int64_t i = 1; i < D; i++) {
    int64_t x = ord[i], j = i;
    while (j > 0 && C[ord[j - 1] * D + ord[j - 1]] > C[x * D + x]) { ord[j] = ord[j - 1]; j--; }
    ord[j] = x;
  }
  /* y = L^-T z for the lowest k (back substitution with L^T) */
  for (int j = 0; j < k; j++) {
    int64_t e = ord[j];
    evals[j] = C[e * D + e];
    for (int64_t i = D - 1; i >= 0; i--) {
      double t = Z[i * D + e];
      for (int64_t m = i + 1; m < D; m++) t -= L[m * D + i] * evecs[m * k + j];
      evecs[i * k + j] = t / L[i * D + i];
    }
  }
  free(L); free(C); free(Z); free(T); free(ord);
  return OR_OK;
}

/*
 * or_lift: the new orbitals in W = [P_H | U~] (Algorithm 3: psi in S_H + span{psi~}):
 *   U_new[i][j] = sum_c P_ic Y[c][j] + sum_m U~[i][m] Y[n_H + m][j],   Y [(n_H + N)][k] row-major.
 * U_new [n_free][k].
 */
int or_lift(const or_mesh *h, int64_t n_H, const int32_t *Pptr, const int32_t *Pcol, const double *Pval, int N,
            const double *Ut, int k, const double *Y, double *Unew) {
  int64_t n = h->n_free;
  for (int64_t i = 0; i < n; i++)
    for (int j = 0; j < k; j++) {
      double s = 0.0;
      for (int32_t t = Pptr[i]; t < Pptr[i + 1]; t++) s += Pval[t] * Y[(int64_t)Pcol[t] * k + j];
      for (int m = 0; m < N; m++) s += Ut[i * N + m] * Y[(n_H + m) * k + j];
      Unew[i * k + j] = s;
    }
  return OR_OK;
}

/*
 * NEXT-3: the nonnested interpolation operator P = I_H^h of Algorithm 1
 * (PAPER.md:499-548): for every vertex q of the fine mesh, the P1 interpolant of a coarse function at q,
 * g(q) = sum_j lambda_j f(q_j), lambda = the barycentric coordinates of q in the coarse tet K that
 * contains it. Plain definition (no quadtree, no walk): K = the coarse tet maximising min_j lambda_j(q; K)
 * (the containing tet; on shared faces/edges every containing tet gives the same nonzero weights), first
 * index on ties. Row i of P (fine FREE node i = free_nodes[i]) keeps the coarse FREE vertices (coarse
 * Dirichlet vertices carry zero data) with |lambda| > drop (reading R4), sorted by
 * coarse free index. O(n_free x n_coarse_tets): tiny meshes only.
 *   xyz_f [*][3] fine coordinates, free_nodes [n_free] fine node ids of the rows; xyz_c [n_c][3],
 *   tets_c [m_c][4], dir_c [n_c] (nonzero = Dirichlet); out: rowptr [n_free+1], col [4 n_free],
 *   val [4 n_free]; *n_H = number of coarse free nodes. Returns OR_E_MESH if a tet is degenerate or a
 *   point lies outside the coarse mesh (min lambda < -1e-10).
 */
int or_interpolation(const double *xyz_f, int64_t n_free, const int64_t *free_nodes, int64_t n_c,
                     const double *xyz_c, int64_t m_c, const int32_t *tets_c, const uint8_t *dir_c, double drop,
                     int32_t *rowptr, int32_t *col, double *val, int64_t *n_H) {
  int32_t *cfree = (int32_t *)malloc(sizeof(int32_t) * (n_c > 0 ? n_c : 1));
  double *Jinv = (double *)malloc(sizeof(double) * 9 * (m_c > 0 ? m_c : 1));
  if (!cfree || !Jinv) { free(cfree); free(Jinv); return OR_E_NOMEM; }
  int64_t nh = 0;
  for (int64_t v = 0; v < n_c; v++) cfree[v] = dir_c[v] ? -1 : (int32_t)nh++;
  *n_H = nh;
  /* inverse of the edge matrix J = [x1-x0, x2-x0, x3-x0] (columns) per coarse tet: lambda_{1..3} = J^-1 (q - x0) */
  for (int64_t t = 0; t < m_c; t++) {
    const double *x0 = xyz_c + 3 * (int64_t)tets_c[4 * t];
    double J[3][3];
    for (int a = 0; a < 3; a++)
      for (int r = 0; r < 3; r++) J[r][a] = xyz_c[3 * (int64_t)tets_c[4 * t + 1 + a] + r] - x0[r];
    double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                 J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    if (!(fabs(det) > 0.0)) { free(cfree); free(Jinv); return OR_E_MESH; }
    double *Ji = Jinv + 9 * t;
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
  int64_t nnz = 0;
  rowptr[0] = 0;
  for (int64_t i = 0; i < n_free; i++) {
    const double *q = xyz_f + 3 * free_nodes[i];
    int64_t best = -1;
    double best_min = -1e300, bl[4] = {0, 0, 0, 0};
    for (int64_t t = 0; t < m_c; t++) {
      const double *x0 = xyz_c + 3 * (int64_t)tets_c[4 * t];
      const double d0 = q[0] - x0[0], d1 = q[1] - x0[1], d2 = q[2] - x0[2];
      const double *Ji = Jinv + 9 * t;
      double l1 = Ji[0] * d0 + Ji[1] * d1 + Ji[2] * d2;
      double l2 = Ji[3] * d0 + Ji[4] * d1 + Ji[5] * d2;
      double l3 = Ji[6] * d0 + Ji[7] * d1 + Ji[8] * d2;
      double l0 = 1.0 - l1 - l2 - l3;
      double m = fmin(fmin(l0, l1), fmin(l2, l3));
      if (m > best_min) { best_min = m; best = t; bl[0] = l0; bl[1] = l1; bl[2] = l2; bl[3] = l3; }
    }
    if (best < 0 || best_min < -1e-10) { free(cfree); free(Jinv); return OR_E_MESH; }
    /* keep free coarse vertices with |lambda| > drop, sorted by coarse free index */
    int32_t cc[4];
    double vv[4];
    int m = 0;
    for (int a = 0; a < 4; a++) {
      int32_t cf = cfree[tets_c[4 * best + a]];
      if (cf < 0 || !(fabs(bl[a]) > drop)) continue;
      int pos = m;
      while (pos > 0 && cc[pos - 1] > cf) { cc[pos] = cc[pos - 1]; vv[pos] = vv[pos - 1]; pos--; }
      cc[pos] = cf;
      vv[pos] = bl[a];
      m++;
    }
    for (int a = 0; a < m; a++) { col[nnz] = cc[a]; val[nnz] = vv[a]; nnz++; }
    rowptr[i + 1] = (int32_t)nnz;
  }
  free(cfree); free(Jinv);
  return OR_OK;
}

/*
 * NEXT-2: the nonlinear terms of the Kohn-Sham operator.
 *
 * or_density: nodal density rho(x_v) = f sum_i psi_i(x_v)^2 (rho_Psi = sum |psi_i|^2;
 * occupation f per orbital: DESIGN.md reading R6 -- the paper's examples put 2 electrons in each orbital,
 * He N = 1, HLi N = 2, CH4 N = 5, C6H6 N = 21), on ALL nodes (psi = 0 on Dirichlet nodes).
 *   U [n_free][N], rho [n_nodes].
 */
int or_density(const or_mesh *h, int N, const double *U, double f, double *rho) {
  for (int64_t v = 0; v < h->n_nodes; v++) {
    int32_t i = h->free_of_node[v];
    double s = 0.0;
    if (i >= 0)
      for (int j = 0; j < N; j++) s += U[(int64_t)i * N + j] * U[(int64_t)i * N + j];
    rho[v] = f * s;
  }
  return OR_OK;
}

/*
 * or_vxc: LDA exchange V_x = -(3 rho / pi)^(1/3) (Eq. expot) plus Perdew-Zunger correlation
 * (Eq. copot) with r_s = (3 / (4 pi rho))^(1/3), A = 0.0311, B = -0.048, C = 0.0020,
 * D = -0.0116, gamma = -0.1423, beta1 = 1.0529, beta2 = 0.3334:
 *   r_s < 1:  V_c = A ln r_s + (B - A/3) + (2/3) C r_s ln r_s + (1/3)(2D - C) r_s
 *   r_s >= 1: V_c = eps_c (1 + 7/6 beta1 sqrt(r_s) + 4/3 beta2 r_s) / (1 + beta1 sqrt(r_s) + beta2 r_s),
 *             eps_c = gamma / (1 + beta1 sqrt(r_s) + beta2 r_s).
 * rho <= 0 gives V_xc = 0 (no electrons). Also returns eps_xc = eps_x + eps_c per node when eps != NULL
 * (eps_x = -(3/4)(3 rho / pi)^(1/3), the energy per electron of E_x^LDA).
 */
int or_vxc(int64_t n, const double *rho, double *vxc, double *eps) {
  const double A = 0.0311, B = -0.048, C = 0.0020, D = -0.0116, G = -0.1423, B1 = 1.0529, B2 = 0.3334;
  const double PI = 3.14159265358979323846;
  for (int64_t v = 0; v < n; v++) {
    double r = rho[v];
    if (!(r > 0.0)) { vxc[v] = 0.0; if (eps) eps[v] = 0.0; continue; }
    double vx = -cbrt(3.0 * r / PI);
    double rs = cbrt(3.0 / (4.0 * PI * r));
    double vc, ec;
    if (rs < 1.0) {
      double l = log(rs);
      ec = A * l + B + C * rs * l + D * rs;
      vc = A * l + (B - A / 3.0) + (2.0 / 3.0) * C * rs * l + (1.0 / 3.0) * (2.0 * D - C) * rs;
    } else {
      double sq = sqrt(rs), den = 1.0 + B1 * sq + B2 * rs;
      ec = G / den;
      vc = ec * (1.0 + (7.0 / 6.0) * B1 * sq + (4.0 / 3.0) * B2 * rs) / den;
    }
    vxc[v] = vx + vc;
    if (eps) eps[v] = 0.75 * vx + ec;
  }
  return OR_OK;
}

/*
 * or_hartree: the Hartree potential: -Lap V = 4 pi rho in Omega, V = w_D on dOmega, with
 * w_D the multipole expansion (Eq. bd) about the centre of charge x'' = int x rho / int rho:
 *   w_D(x) = Q/|d| + sum_i p_i d_i/|d|^3 + 1/2 sum_ij q_ij (3 d_i d_j - delta_ij |d|^2)/|d|^5,  d = x - x'',
 *   Q = int rho, p_i = int rho (x'-x'')_i, q_ij = int rho (x'-x'')_i (x'-x'')_j.
 * (reading R5: the factor 1/2 of the second-order Taylor term of 1/|x - x'|, missing in the printed
 * Eq. bd.) Moments are exact integrals of the P1 density: int_T lambda^alpha = 3! alpha! |T| / (3+|alpha|)!.
 * P1 Galerkin with the Dirichlet lift: for free i, sum_j K_ij V_j = 4 pi sum_{all b} M_ib rho_b
 *   - sum_{Dirichlet b} K_ib w_D(x_b), accumulated element by element (t ascending); the free values by Jacobi-PCG
 * on K from zero to ||r|| <= tol ||b||. vh [n_nodes] = the free values and w_D on Dirichlet nodes.
 * mom [10] (may be NULL) = Q, x''_0..2, p_0..2, q_00, q_11, q_22 (diagonal). Returns OR_E_NOT_CONVERGED if
 * max_iter is reached (vh still written), *iters = iterations.
 */
int or_hartree(const or_mesh *h, const double *xyz, const double *rho, double tol, int max_iter, double *vh,
               double *mom, int *iters) {
  const double PI = 3.14159265358979323846;
  int64_t nt = h->n_tets, n = h->n_free, nn = h->n_nodes;
  /* moments */
  double Q = 0.0, m1[3] = {0, 0, 0};
  for (int64_t t = 0; t < nt; t++) {
    const int32_t *v = h->tets + 4 * t;
    double V = h->vol[t], sr = 0.0;
    for (int a = 0; a < 4; a++) sr += rho[v[a]];
    Q += V * sr / 4.0;
    for (int a = 0; a < 4; a++)
      for (int b = 0; b < 4; b++)
        for (int i = 0; i < 3; i++) m1[i] += rho[v[a]] * xyz[3 * (int64_t)v[b] + i] * V * (a == b ? 2.0 : 1.0) / 20.0;
  }
  double c[3] = {0, 0, 0}, p[3] = {0, 0, 0}, q[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  if (Q != 0.0)
    for (int i = 0; i < 3; i++) c[i] = m1[i] / Q;
  for (int64_t t = 0; t < nt; t++) {
    const int32_t *v = h->tets + 4 * t;
    double V = h->vol[t];
    double y[4][3];
    for (int a = 0; a < 4; a++)
      for (int i = 0; i < 3; i++) y[a][i] = xyz[3 * (int64_t)v[a] + i] - c[i];
    for (int a = 0; a < 4; a++)
      for (int b = 0; b < 4; b++) {
        double w2 = V * (a == b ? 2.0 : 1.0) / 20.0;
        for (int i = 0; i < 3; i++) p[i] += rho[v[a]] * y[b][i] * w2;
        for (int cc = 0; cc < 4; cc++) {
          /* int lambda_a lambda_b lambda_c = alpha! |T| / 120 */
          double al = (a == b && b == cc) ? 6.0 : ((a == b || b == cc || a == cc) ? 2.0 : 1.0);
          double w3 = V * al / 120.0;
          for (int i = 0; i < 3; i++)
            for (int j = 0; j < 3; j++) q[i][j] += rho[v[a]] * y[b][i] * y[cc][j] * w3;
        }
      }
  }
  if (mom) {
    mom[0] = Q;
    for (int i = 0; i < 3; i++) { mom[1 + i] = c[i]; mom[4 + i] = p[i]; mom[7 + i] = q[i][i]; }
  }
  /* boundary values */
  double *w = (double *)calloc(nn, sizeof(double));
  double *bvec = (double *)calloc(n > 0 ? n : 1, sizeof(double));
  if (!w || !bvec) { free(w); free(bvec); return OR_E_NOMEM; }
  for (int64_t vtx = 0; vtx < nn; vtx++) {
    if (h->free_of_node[vtx] >= 0) continue;
    double d[3], r2 = 0.0;
    for (int i = 0; i < 3; i++) { d[i] = xyz[3 * vtx + i] - c[i]; r2 += d[i] * d[i]; }
    double r = sqrt(r2);
    double s = Q / r;
    for (int i = 0; i < 3; i++) s += p[i] * d[i] / (r2 * r);
    for (int i = 0; i < 3; i++)
      for (int j = 0; j < 3; j++) s += 0.5 * q[i][j] * (3.0 * d[i] * d[j] - (i == j ? r2 : 0.0)) / (r2 * r2 * r);
    w[vtx] = s;
  }
  /* load vector with the Dirichlet lift, element by element */
  for (int64_t t = 0; t < nt; t++) {
    const int32_t *v = h->tets + 4 * t;
    const double *g = h->grad + 12 * t;
    double V = h->vol[t];
    for (int a = 0; a < 4; a++) {
      int32_t ia = h->free_of_node[v[a]];
      if (ia < 0) continue;
      double s = 0.0;
      for (int b = 0; b < 4; b++) {
        s += 4.0 * PI * V * (a == b ? 2.0 : 1.0) / 20.0 * rho[v[b]];
        if (h->free_of_node[v[b]] < 0) {
          double kab = V * (g[3 * a] * g[3 * b] + g[3 * a + 1] * g[3 * b + 1] + g[3 * a + 2] * g[3 * b + 2]);
          s -= kab * w[v[b]];
        }
      }
      bvec[ia] += s;
    }
  }
  /* Jacobi-PCG on K from x0 = 0 */
  double *x = (double *)calloc(n > 0 ? n : 1, sizeof(double));
  double *r = (double *)malloc(sizeof(double) * (n > 0 ? n : 1));
  double *z = (double *)malloc(sizeof(double) * (n > 0 ? n : 1));
  double *pp = (double *)malloc(sizeof(double) * (n > 0 ? n : 1));
  double *qq = (double *)malloc(sizeof(double) * (n > 0 ? n : 1));
  double *dK = (double *)malloc(sizeof(double) * (n > 0 ? n : 1));
  for (int64_t i = 0; i < n; i++)
    for (int64_t k = h->row_ptr[i]; k < h->row_ptr[i + 1]; k++)
      if (h->col[k] == i) dK[i] = h->K[k];
  double bn = 0.0;
  for (int64_t i = 0; i < n; i++) { r[i] = bvec[i]; z[i] = r[i] / dK[i]; pp[i] = z[i]; bn += bvec[i] * bvec[i]; }
  bn = sqrt(bn);
  double rz = 0.0;
  for (int64_t i = 0; i < n; i++) rz += r[i] * z[i];
  int it = 0, st = OR_OK;
  for (;;) {
    double rr = 0.0;
    for (int64_t i = 0; i < n; i++) rr += r[i] * r[i];
    if (sqrt(rr) <= tol * bn) break;
    if (it >= max_iter) { st = OR_E_NOT_CONVERGED; break; }
    matvec(h, h->K, pp, qq);
    double pq = 0.0;
    for (int64_t i = 0; i < n; i++) pq += pp[i] * qq[i];
    double al = rz / pq;
    for (int64_t i = 0; i < n; i++) { x[i] += al * pp[i]; r[i] -= al * qq[i]; z[i] = r[i] / dK[i]; }
    double rz2 = 0.0;
    for (int64_t i = 0; i < n; i++) rz2 += r[i] * z[i];
    double be = rz2 / rz;
    rz = rz2;
    for (int64_t i = 0; i < n; i++) pp[i] = z[i] + be * pp[i];
    it++;
  }
  for (int64_t vtx = 0; vtx < nn; vtx++) {
    int32_t i = h->free_of_node[vtx];
    vh[vtx] = i >= 0 ? x[i] : w[vtx];
  }
  if (iters) *iters = it;
  free(w); free(bvec); free(x); free(r); free(z); free(pp); free(qq); free(dK);
  return st;
}
