// MUFU exp2 throughput: ex2.approx.f32 vs ex2.approx.f16x2 vs ex2.approx.ftz.bf16x2
// (elements per clock per SM).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 mufu_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

template <int KIND>
__global__ void k(float* out, int iters) {
  float a[8];
  uint32_t h[8];
  for (int i = 0; i < 8; ++i) { a[i] = -0.001f * (threadIdx.x + i); h[i] = 0xBC00BC00u + i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (KIND == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[i]));
      if (KIND == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h[i]));
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(h[i]);
  if (s == 12345.f) out[0] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096, blocks = sms * 4, threads = 512;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[3] = {"ex2.f32", "ex2.f16x2", "ex2.bf16x2"};
  for (int kind = 0; kind < 3; ++kind) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (kind == 0) k<0><<<blocks, threads>>>(out, iters);
      if (kind == 1) k<1><<<blocks, threads>>>(out, iters);
      if (kind == 2) k<2><<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * iters * 8;  // instructions (lane ops)
      double elems = ops * (kind == 0 ? 1 : 2);
      if (rep) printf("%-10s %.3f ms  %.1f lane-instr/clk/SM  %.1f exps/clk/SM (at %d MHz nominal)\n", names[kind], ms,
                      ops / (ms * 1e-3) / sms / (clk * 1e3), elems / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
