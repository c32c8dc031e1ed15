// tcgen05 MMA issue-stream throughput by shape / operand source (clocks per
// MMA, one CTA per SM, one warp issuing back to back, operands' contents
// irrelevant).  Patterns: SS N=128, SS N=64, TS N=128 (A in TMEM), and the
// per-block instruction mixes of the v10 / v11 recompute-attention schedules.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//      -I paper_2603_05353_b200/csrc -I include tools/micro/mma_shape_bench.cu -o /tmp/mma_shape_bench -lcuda
#include <cstdio>

#include "tc_common.cuh"

using namespace ifkv;

constexpr int kPanel = 128 * 128;

template <int PAT>
__global__ void __launch_bounds__(128, 1) bench(long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* qa = base;               // 32 KB
  uint8_t* kb = base + 2 * kPanel;  // 32 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tbase);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp == 0) {
    constexpr uint32_t id128 = tc::idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t id64 = tc::idesc_bf16(128, 64, 0, 0);
    constexpr uint32_t idpv = tc::idesc_bf16(128, 128, 0, 1);
    const uint64_t da = tc::smem_desc_sw128(tc::smem_u32(qa), 16, 1024);
    const uint64_t db = tc::smem_desc_sw128(tc::smem_u32(kb), 16, 1024);
    const uint64_t db_hi = tc::smem_desc_sw128(tc::smem_u32(kb + 64 * 128), 16, 1024);
    const uint64_t dv = tc::smem_desc_sw128(tc::smem_u32(kb), kPanel, 1024);
    auto ss = [&](uint32_t d, uint64_t b, uint32_t id) {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const uint64_t step = (uint64_t)((t >> 2) * (kPanel >> 4) + (t & 3) * 2);
        tc::mma_bf16_ss_ws(tmem + d, da + step, b + step, id, t > 0);
      }
    };
    auto ts = [&](uint32_t d, uint32_t a, int n) {
      for (int t = 0; t < n; ++t) tc::mma_bf16_ts_ws(tmem + d, tmem + a + 8 * t, dv + (uint64_t)(t * 128), idpv, 1);
    };
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (PAT == 0) ss(0, db, id128);                 // 8 SS N=128
      if (PAT == 1) ss(0, db, id64);                  // 8 SS N=64
      if (PAT == 2) ts(256, 64, 8);                   // 8 TS N=128
      if (PAT == 3) {                                 // v10 block: PV_A S_A PV_B S_B
        ts(256, 64, 8); ss(0, db, id128); ts(384, 192, 8); ss(128, db, id128);
      }
      if (PAT == 4) {                                 // v11 sub-block: PV_A S_A PV_B S_B (N=64, K=64 PV)
        ts(256, 32, 4); ss(0, db, id64); ts(384, 160, 4); ss(128, db_hi, id64);
      }
      if (PAT == 5) ss(0, db_hi, id64);               // 8 SS N=64 on the upper K rows
    }
    tc::mma_commit_ws(&bar);
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int PAT>
void run(const char* name, int per_rep, long long* d, int sms) {
  const int reps = 2000;
  const size_t smem = 4 * kPanel + 1024;
  cudaFuncSetAttribute(bench<PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bench<PAT><<<sms, 128, smem>>>(d, 10);
  bench<PAT><<<sms, 128, smem>>>(d, reps);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    return;
  }
  long long h[1024];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  printf("%-44s %8.1f clk per rep, %6.1f clk per MMA\n", name, avg / reps, avg / reps / per_rep);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, 1024 * sizeof(long long));
  run<0>("SS M128 N128 K16 x8", 8, d, sms);
  run<1>("SS M128 N64 K16 x8", 8, d, sms);
  run<5>("SS M128 N64 K16 x8 (B rows 64..127)", 8, d, sms);
  run<2>("TS M128 N128 K16 x8", 8, d, sms);
  run<3>("v10 block (8 TS, 8 SS128, 8 TS, 8 SS128)", 32, d, sms);
  run<4>("v11 sub-block (4 TS, 8 SS64, 4 TS, 8 SS64)", 24, d, sms);
  return 0;
}
