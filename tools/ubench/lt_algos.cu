// Time every cublasLt heuristic algorithm for the batch-1 projection shapes
// (x[M,K] @ W[K,N], bf16 in, bf16 or fp32 out), weights cycled over 16 copies
// so they stream from HBM.  nvcc -O2 -arch=sm_100a lt_algos.cu -lcublasLt -o lt_algos
#include <cublasLt.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <vector>
#define CK(x) do { auto e = (x); if ((int)e) { printf("err %d at %s:%d\n", (int)e, __FILE__, __LINE__); return; } } while (0)

static void run(int M, int N, int K, bool f32out) {
  cublasLtHandle_t h; cublasLtCreate(&h);
  const int L = 16;
  std::vector<void*> W(L);
  for (auto &w : W) cudaMalloc(&w, (size_t)K * N * 2), cudaMemset(w, 0, (size_t)K * N * 2);
  void *x, *out, *ws; size_t wsz = 64 << 20;
  cudaMalloc(&x, (size_t)M * K * 2); cudaMemset(x, 0, (size_t)M * K * 2);
  cudaMalloc(&out, (size_t)M * N * 4); cudaMalloc(&ws, wsz);
  cublasLtMatmulDesc_t d; CK(cublasLtMatmulDescCreate(&d, CUBLAS_COMPUTE_32F, CUDA_R_32F));
  cublasOperation_t nt = CUBLAS_OP_N;
  cublasLtMatmulDescSetAttribute(d, CUBLASLT_MATMUL_DESC_TRANSA, &nt, sizeof(nt));
  cublasLtMatmulDescSetAttribute(d, CUBLASLT_MATMUL_DESC_TRANSB, &nt, sizeof(nt));
  cublasLtMatrixLayout_t A, B, C;  // column-major: C[N,M] = W^T-view A[N,K] * x-view B[K,M]
  CK(cublasLtMatrixLayoutCreate(&A, CUDA_R_16BF, N, K, N));
  CK(cublasLtMatrixLayoutCreate(&B, CUDA_R_16BF, K, M, K));
  CK(cublasLtMatrixLayoutCreate(&C, f32out ? CUDA_R_32F : CUDA_R_16BF, N, M, N));
  cublasLtMatmulPreference_t pref; cublasLtMatmulPreferenceCreate(&pref);
  cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsz, sizeof(wsz));
  cublasLtMatmulHeuristicResult_t res[32]; int nres = 0;
  CK(cublasLtMatmulAlgoGetHeuristic(h, d, A, B, C, C, pref, 32, res, &nres));
  float alpha = 1.f, beta = 0.f;
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("M %d N %d K %d %s: %d algos\n", M, N, K, f32out ? "f32" : "bf16", nres);
  for (int i = 0; i < nres; ++i) {
    if (res[i].state) continue;
    bool bad = false;
    for (int r = 0; r < 2 && !bad; ++r)
      for (int l = 0; l < L; ++l)
        if (cublasLtMatmul(h, d, &alpha, W[l], A, x, B, &beta, out, C, out, C, &res[i].algo, ws, wsz, s)) bad = true;
    if (bad) { printf("  algo %d failed\n", i); continue; }
    cudaEventRecord(e0, s);
    for (int r = 0; r < 5; ++r)
      for (int l = 0; l < L; ++l)
        cublasLtMatmul(h, d, &alpha, W[l], A, x, B, &beta, out, C, out, C, &res[i].algo, ws, wsz, s);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double us = ms * 1000 / (5 * L);
    printf("  algo %2d: %7.2f us  %5.2f TB/s  ws %zu\n", i, us, (double)K * N * 2 / us / 1e6, res[i].workspaceSize);
  }
}
int main() {
  int shapes[4][2] = {{4096, 6144}, {4096, 4096}, {4096, 28672}, {14336, 4096}};
  for (auto &sh : shapes) run(44, sh[1], sh[0], false);
  run(44, 4096, 4096, true); run(44, 4096, 14336, true);
  return 0;
}
