/* A plain C99 consumer of libks (no Python, no torch): builds a small Kuhn mesh of the cube [-1, 1]^3 with
 * n^3 cells (6 tets per cell, Dirichlet boundary), uploads V = |x|^2 / 2 and N = 2 orbitals, and runs
 * ks_plan -> ks_create -> ks_assemble_veff -> ks_block_solve -> ks_sync through the ABI of include/ks.h. All
 * device memory is the consumer's own (CUDA runtime C API): the library's regions are allocated from the
 * sizes ks_plan returns (include/ks.h, "Memory"); the setup region is freed right after ks_create. Prints "ok <n_free> <iterations> <relres0> <relres1>" and returns 0,
 * or prints the ks_last_error message and returns 1. Used by tests/test_abi.py (compile + link, CPU) and
 * tests/test_gpu_c_abi.py (run, GPU). */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "ks.h"

#define CHECK(call)                                                                                      \
  do {                                                                                                   \
    ks_status s_ = (call);                                                                               \
    if (s_ != KS_OK) {                                                                                   \
      printf("fail %s: status %d: %s\n", #call, (int)s_, ks_last_error(ctx));                           \
      return 1;                                                                                          \
    }                                                                                                    \
  } while (0)

int main(void) {
  const int n = 4, n1 = n + 1, N = 2;
  const int64_t nn = (int64_t)n1 * n1 * n1, nt = 6LL * n * n * n;
  double *xyz = malloc(sizeof(double) * 3 * nn);
  int32_t *tets = malloc(sizeof(int32_t) * 4 * nt);
  uint8_t *dir = malloc(nn);
  double *V = malloc(sizeof(double) * nn);
  for (int k = 0; k < n1; k++)
    for (int j = 0; j < n1; j++)
      for (int i = 0; i < n1; i++) {
        const int64_t v = i + n1 * (j + (int64_t)n1 * k);
        const double x = -1.0 + 2.0 * i / n, y = -1.0 + 2.0 * j / n, z = -1.0 + 2.0 * k / n;
        xyz[3 * v] = x;
        xyz[3 * v + 1] = y;
        xyz[3 * v + 2] = z;
        dir[v] = (i == 0 || j == 0 || k == 0 || i == n || j == n || k == n);
        V[v] = 0.5 * (x * x + y * y + z * z);
      }
  /* Kuhn split: the 6 paths from corner 0 to corner 7 of each cell (positive orientation) */
  static const int perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  int64_t t = 0;
  for (int k = 0; k < n; k++)
    for (int j = 0; j < n; j++)
      for (int i = 0; i < n; i++)
        for (int p = 0; p < 6; p++) {
          int c[3] = {i, j, k};
          int32_t id[4];
          id[0] = (int32_t)(c[0] + n1 * (c[1] + n1 * c[2]));
          for (int s = 0; s < 3; s++) {
            c[perm[p][s]]++;
            id[s + 1] = (int32_t)(c[0] + n1 * (c[1] + n1 * c[2]));
          }
          /* orientation: det of (x1 - x0, x2 - x0, x3 - x0) must be positive; swap the last two if not */
          double e[3][3];
          for (int a = 0; a < 3; a++)
            for (int d = 0; d < 3; d++) e[a][d] = xyz[3 * id[a + 1] + d] - xyz[3 * id[0] + d];
          const double det = e[0][0] * (e[1][1] * e[2][2] - e[1][2] * e[2][1]) -
                             e[0][1] * (e[1][0] * e[2][2] - e[1][2] * e[2][0]) +
                             e[0][2] * (e[1][0] * e[2][1] - e[1][1] * e[2][0]);
          if (det < 0) {
            int32_t tmp = id[2];
            id[2] = id[3];
            id[3] = tmp;
          }
          for (int a = 0; a < 4; a++) tets[4 * t + a] = id[a];
          t++;
        }
  ks_ctx *ctx = NULL;
  size_t b_persist = 0, b_work = 0, b_setup = 0;
  CHECK(ks_plan(nn, xyz, nt, tets, dir, N, &b_persist, &b_work, &b_setup));
  void *d_persist = NULL, *d_work = NULL, *d_setup = NULL;
  if (cudaMalloc(&d_persist, b_persist) || cudaMalloc(&d_work, b_work) || cudaMalloc(&d_setup, b_setup)) {
    printf("fail cudaMalloc (regions)\n");
    return 1;
  }
  CHECK(ks_create(nn, xyz, nt, tets, dir, N, d_persist, b_persist, d_work, b_work, d_setup, b_setup, NULL, &ctx));
  cudaFree(d_setup);   /* used only during ks_create */
  int64_t n_free = 0, nnz = 0;
  CHECK(ks_pattern(ctx, &n_free, &nnz, NULL, NULL, NULL, NULL, NULL, NULL));
  double *dV, *dlam, *dU, *dUt, *drel;
  int32_t *dit;
  if (cudaMalloc((void **)&dV, sizeof(double) * nn) || cudaMalloc((void **)&dlam, sizeof(double) * N) ||
      cudaMalloc((void **)&dU, sizeof(double) * n_free * N) || cudaMalloc((void **)&dUt, sizeof(double) * n_free * N) ||
      cudaMalloc((void **)&drel, sizeof(double) * N) || cudaMalloc((void **)&dit, sizeof(int32_t) * N)) {
    printf("fail cudaMalloc\n");
    return 1;
  }
  double *U = malloc(sizeof(double) * n_free * N), lam[2] = {1.5, 2.5}, rel[2];
  for (int64_t r = 0; r < n_free; r++)
    for (int c = 0; c < N; c++) U[r * N + c] = 1.0 + 0.1 * c + 0.01 * (double)(r % 7);
  cudaMemcpy(dV, V, sizeof(double) * nn, cudaMemcpyHostToDevice);
  cudaMemcpy(dlam, lam, sizeof(double) * N, cudaMemcpyHostToDevice);
  cudaMemcpy(dU, U, sizeof(double) * n_free * N, cudaMemcpyHostToDevice);
  CHECK(ks_assemble_veff(ctx, dV, 10.0));
  CHECK(ks_block_solve(ctx, N, dlam, dU, dUt, 1e-10, 1000, dit, drel));
  CHECK(ks_sync(ctx));
  int32_t iters = 0;
  CHECK(ks_last_iterations(ctx, &iters));
  cudaMemcpy(rel, drel, sizeof(double) * N, cudaMemcpyDeviceToHost);
  printf("ok %lld %d %.3e %.3e\n", (long long)n_free, iters, rel[0], rel[1]);
  ks_destroy(ctx);
  cudaFree(d_persist);
  cudaFree(d_work);
  cudaFree(dV);
  cudaFree(dlam);
  cudaFree(dU);
  cudaFree(dUt);
  cudaFree(drel);
  cudaFree(dit);
  free(xyz);
  free(tets);
  free(dir);
  free(V);
  free(U);
  return (rel[0] <= 1e-10 && rel[1] <= 1e-10 && iters > 0) ? 0 : 1;
}
