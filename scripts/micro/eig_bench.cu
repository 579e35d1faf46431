// Microbenchmark (NEXT-1): cuSOLVER routes for the lowest k eigenpairs of a dense SPD pencil
// (A, B), D = 745 / 1363, k = 16 / 32: sygvd (all), sygvdx (subset), and the reduction to standard form
// (potrf + 2 trsm) followed by syevd / syevdx / Xsyevd / Xsyevdx. Prints ms per route (events, median of 5).
#include <cublas_v2.h>
#include <cusolverDn.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#define CK(x) do { auto e = (x); if ((int)e != 0) { printf("err %d at %d\n", (int)e, __LINE__); exit(1); } } while (0)

int main() {
  cusolverDnHandle_t h; CK(cusolverDnCreate(&h));
  cublasHandle_t cb; CK(cublasCreate(&cb));
  cusolverDnParams_t prm; CK(cusolverDnCreateParams(&prm));
  for (int D : {745, 1363}) {
    const int k = D == 745 ? 16 : 32;
    std::vector<double> A(D * D), B(D * D);
    unsigned long long s = 7;
    auto rnd = [&]() { s = s * 6364136223846793005ULL + 1442695040888963407ULL; return (double)(s >> 11) * 0x1.0p-53 - 0.5; };
    for (int i = 0; i < D; i++) for (int j = 0; j <= i; j++) { double a = rnd(), b = 0.1 * rnd(); A[i * D + j] = A[j * D + i] = a; B[i * D + j] = B[j * D + i] = b; }
    for (int i = 0; i < D; i++) { A[i * D + i] += 4.0 * i / D; B[i * D + i] += D * 0.2; }
    double *dA, *dB, *dA0, *dB0, *w, *work; int *info;
    CK(cudaMalloc(&dA, 8ull * D * D)); CK(cudaMalloc(&dB, 8ull * D * D)); CK(cudaMalloc(&dA0, 8ull * D * D)); CK(cudaMalloc(&dB0, 8ull * D * D));
    CK(cudaMalloc(&w, 8ull * D)); CK(cudaMalloc(&info, 4));
    CK(cudaMemcpy(dA0, A.data(), 8ull * D * D, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dB0, B.data(), 8ull * D * D, cudaMemcpyHostToDevice));
    size_t wsz = 64ull << 20; CK(cudaMalloc(&work, wsz)); void *hwork = malloc(64 << 20);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](const char *name, auto fn) {
      std::vector<float> t;
      for (int r = 0; r < 6; r++) {
        CK(cudaMemcpy(dA, dA0, 8ull * D * D, cudaMemcpyDeviceToDevice)); CK(cudaMemcpy(dB, dB0, 8ull * D * D, cudaMemcpyDeviceToDevice));
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0); fn(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (r) t.push_back(ms);
      }
      std::sort(t.begin(), t.end());
      std::vector<double> wh(k); CK(cudaMemcpy(wh.data(), w, 8 * k, cudaMemcpyDeviceToHost));
      printf("{\"D\": %d, \"k\": %d, \"route\": \"%s\", \"ms\": %.3f, \"w0\": %.12f, \"wk\": %.12f}\n", D, k, name, t[t.size() / 2], wh[0], wh[k - 1]);
    };
    const int lw = (int)(wsz / 8);
    int meig = 0;
    timeit("sygvd", [&] { CK(cusolverDnDsygvd(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, D, dA, D, dB, D, w, work, lw, info)); });
    timeit("sygvdx", [&] { CK(cusolverDnDsygvdx(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, D, dA, D, dB, D, 0, 0, 1, k, &meig, w, work, lw, info)); });
    const double one = 1.0;
    auto reduce = [&] {   // B = L L^T, A <- L^-1 A L^-T
      CK(cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, D, dB, D, work, lw, info));
      CK(cublasDtrsm(cb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, D, D, &one, dB, D, dA, D));
      CK(cublasDtrsm(cb, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, D, D, &one, dB, D, dA, D));
    };
    cudaStream_t st; cusolverDnGetStream(h, &st); cublasSetStream(cb, st);
    timeit("reduce_only", [&] { reduce(); });
    timeit("reduce+syevd", [&] { reduce(); CK(cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, D, dA, D, w, work, lw, info)); });
    timeit("reduce+syevdx", [&] { reduce(); CK(cusolverDnDsyevdx(h, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, D, dA, D, 0, 0, 1, k, &meig, w, work, lw, info)); });
    size_t dws = 0, hws = 0;
    CK(cusolverDnXsyevd_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, D, CUDA_R_64F, dA, D, CUDA_R_64F, w, CUDA_R_64F, &dws, &hws));
    timeit("reduce+Xsyevd", [&] { reduce(); CK(cusolverDnXsyevd(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, D, CUDA_R_64F, dA, D, CUDA_R_64F, w, CUDA_R_64F, work, wsz, hwork, 64 << 20, info)); });
    int64_t me = 0;
    CK(cusolverDnXsyevdx_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, D, CUDA_R_64F, dA, D, nullptr, nullptr, 1, k, &me, CUDA_R_64F, w, CUDA_R_64F, &dws, &hws));
    timeit("reduce+Xsyevdx", [&] { reduce(); CK(cusolverDnXsyevdx(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, D, CUDA_R_64F, dA, D, nullptr, nullptr, 1, k, &me, CUDA_R_64F, w, CUDA_R_64F, work, wsz, hwork, 64 << 20, info)); });
    cudaFree(dA); cudaFree(dB); cudaFree(dA0); cudaFree(dB0); cudaFree(w); cudaFree(work); cudaFree(info); free(hwork);
  }
  return 0;
}
