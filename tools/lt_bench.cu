// cuBLASLt algorithm sweep for the recompute GEMM shapes (row-major
// C[M,N] (+)= A[M,K] . W[K,N], bf16 operands, fp32 accumulate): times every
// heuristic candidate so the default choice can be compared with the best.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/lt_bench.cu -lcublasLt -o tools/_lt_bench
#include <cublasLt.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    auto e = (x);                                                          \
    if ((int)e != 0) {                                                     \
      printf("error %d at %s:%d\n", (int)e, __FILE__, __LINE__);          \
      return 1;                                                            \
    }                                                                      \
  } while (0)

__global__ void fill_rand(__nv_bfloat16* p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    p[i] = __float2bfloat16(((x & 0xffff) / 32768.f - 1.f));
  }
}

struct Shape {
  const char* name;
  int M, N, K;
  bool f32_out;  // fp32 C with beta = 1 (residual epilogue), else bf16 C
};

int main() {
  const Shape shapes[] = {{"qkv", 4916, 6144, 4096, false},
                          {"o+res", 4916, 4096, 4096, true},
                          {"gate_up", 4916, 28672, 4096, false},
                          {"down+res", 4916, 4096, 14336, true}};
  cublasLtHandle_t lt;
  CK(cublasLtCreate(&lt));
  size_t ws_bytes = 64 << 20;
  void* ws;
  CK(cudaMalloc(&ws, ws_bytes));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  for (const Shape& s : shapes) {
    void *A, *W, *C;
    CK(cudaMalloc(&A, (size_t)s.M * s.K * 2));
    CK(cudaMalloc(&W, (size_t)s.K * s.N * 2));
    CK(cudaMalloc(&C, (size_t)s.M * s.N * 4));
    fill_rand<<<1184, 256>>>((__nv_bfloat16*)A, (size_t)s.M * s.K, 1);
    fill_rand<<<1184, 256>>>((__nv_bfloat16*)W, (size_t)s.K * s.N, 2);
    CK(cudaMemset(C, 0, (size_t)s.M * s.N * 4));
    cublasLtMatmulDesc_t op;
    CK(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
    // column-major view: C^T[N,M] = W^T[N,K] . A^T[K,M]
    cublasLtMatrixLayout_t la, lb, lc;
    CK(cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, s.N, s.K, s.N));
    CK(cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, s.K, s.M, s.K));
    CK(cublasLtMatrixLayoutCreate(&lc, s.f32_out ? CUDA_R_32F : CUDA_R_16BF, s.N, s.M, s.N));
    cublasLtMatmulPreference_t pref;
    CK(cublasLtMatmulPreferenceCreate(&pref));
    CK(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws_bytes,
                                            sizeof(ws_bytes)));
    std::vector<cublasLtMatmulHeuristicResult_t> res(32);
    int n = 0;
    CK(cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, lc, lc, pref, 32, res.data(), &n));
    const float alpha = 1.f, beta = s.f32_out ? 1.f : 0.f;
    const double flop = 2.0 * s.M * s.N * (double)s.K;
    double best = 1e30, first = 0;
    int best_i = -1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < n; ++i) {
      if (res[i].state != CUBLAS_STATUS_SUCCESS) continue;
      bool ok = true;
      for (int w = 0; w < 3 && ok; ++w)
        ok = cublasLtMatmul(lt, op, &alpha, W, la, A, lb, &beta, C, lc, C, lc, &res[i].algo, ws, ws_bytes, st) ==
             CUBLAS_STATUS_SUCCESS;
      if (!ok) continue;
      const int it = 30;
      cudaEventRecord(e0, st);
      for (int r = 0; r < it; ++r)
        cublasLtMatmul(lt, op, &alpha, W, la, A, lb, &beta, C, lc, C, lc, &res[i].algo, ws, ws_bytes, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = 1e3 * ms / it;
      if (i == 0) first = us;
      if (us < best) best = us, best_i = i;
      printf("%-9s algo %2d: %8.1f us  %6.0f TF/s  ws %zu\n", s.name, i, us, flop / us / 1e6,
             res[i].workspaceSize);
    }
    printf("%-9s heuristic #0 %.1f us, best #%d %.1f us (%.1f %%)\n\n", s.name, first, best_i, best,
           100.0 * (first - best) / first);
    cudaFree(A);
    cudaFree(W);
    cudaFree(C);
  }
  return 0;
}
