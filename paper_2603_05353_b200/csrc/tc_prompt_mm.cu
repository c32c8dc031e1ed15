// Prompt-row GEMM of the scoring pass on the tcgen05 tensor cores:
//   out[s][r][n] = sum_{p < P} sum_{k in split s} X[p][r][k] * W[k][n]
// X: the P (= 3) bf16 split terms of the fp32 activations of the R (= 32)
// prompt rows, W: a bf16 projection stored "out x in" ([N][K], K-major; the
// reference's x @ W with W^T stored, model.py:435-455).  With R*P <= 256 rows the product is a weight stream:
// 2 x 96 FLOP per weight byte, far below the tensor ridge, so the kernel is
// bound by HBM reading W once (selection.py:127-169 runs it for every layer
// below the capture layer: 8.3 GB of weights at C2).
//
// Transposed tile: D^T[n][p*R + r] = W^T[n][k] . X^T[k][p*R + r], so W is the
// A operand (M = 128 output columns, K-major rows of the stored W^T) and the
// P*R activation rows are the N of the MMA (K-major).  The split terms are summed in fp32 in the epilogue in a
// fixed order; K is split over gridDim.y so the grid covers the GPU, each
// split writing its own fp32 partial (out[s]) -- consumers sum the partials
// in a fixed order (n_parts), so results are deterministic.
// Warps: 0 TMA producer, 1 MMA issuer (+ TMEM alloc), 0-3 epilogue.
#include "tc_common.cuh"

namespace ifkv {
namespace {

constexpr int kN = 128;      // output columns per CTA (MMA M)
constexpr int kKStep = 64;   // K per stage (one 128-byte swizzle row of X)
constexpr int kWStage = 128 * 128;    // 16 KB: 128 n rows x 64 k (128 B)

template <int kStages>
__global__ void __launch_bounds__(128, 2)
    prompt_mm_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x, int P,
                     int R, int NR, int k_steps, int N, float* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int x_bytes = NR * 128;  // NR activation rows x 64 k (bf16)
  const int stage_bytes = kWStage + ((x_bytes + 1023) & ~1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + kStages * stage_bytes);
  uint64_t* empty = full + kStages;
  uint64_t* done = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * kN;
  const int s0 = (int)((int64_t)blockIdx.y * k_steps / gridDim.y);
  const int ns = (int)((int64_t)(blockIdx.y + 1) * k_steps / gridDim.y) - s0;

  pdl_trigger();
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    tc::mbar_init(done, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<256>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tm_w);
    tc::tma_prefetch(&tm_x);
    // the weights do not depend on the previous kernel: the first stages'
    // W tiles are requested before waiting for it (programmatic launch),
    // the activations after
    const int pre = ns < kStages ? ns : kStages;
    for (int i = 0; i < pre; ++i) {
      tc::mbar_arrive_expect_tx(&full[i], kWStage + x_bytes);
      tc::tma_load_2d(base + i * stage_bytes, &tm_w, &full[i], (s0 + i) * kKStep, n0);
    }
    pdl_wait();
    for (int i = 0; i < pre; ++i)
      tc::tma_load_2d(base + i * stage_bytes + kWStage, &tm_x, &full[i], (s0 + i) * kKStep, 0);
    for (int i = pre; i < ns; ++i) {
      const int s = i % kStages;
      const int k0 = (s0 + i) * kKStep;
      tc::mbar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
      uint8_t* st = base + s * stage_bytes;
      tc::mbar_arrive_expect_tx(&full[s], kWStage + x_bytes);
      tc::tma_load_2d(st, &tm_w, &full[s], k0, n0);
      tc::tma_load_2d(st + kWStage, &tm_x, &full[s], k0, 0);
    }
  } else if (warp == 1) {
    // A = W tile, B = X tile, both K-major: rows of 128 B (64 k), 8-row
    // swizzle atoms 1 KB apart, K = 16 per MMA = 32 B along the row.
    const uint32_t idesc = tc::idesc_bf16(kN, NR, 0, 0);
    for (int i = 0; i < ns; ++i) {
      const int s = i % kStages;
      tc::mbar_wait(&full[s], (i / kStages) & 1);
      tc::tc_fence_after();
      const uint32_t st = tc::smem_u32(base + s * stage_bytes);
      const uint64_t a = tc::smem_desc_sw128(st, 16, 1024);
      const uint64_t b = tc::smem_desc_sw128(st + kWStage, 16, 1024);
#pragma unroll
      for (int t = 0; t < kKStep / 16; ++t)
        tc::mma_bf16_ss_ws(tmem, a + (uint64_t)(t * 2), b + (uint64_t)(t * 2), idesc,
                           (i > 0 || t > 0) ? 1u : 0u);
      tc::mma_commit_ws(&empty[s]);
    }
    tc::mma_commit_ws(done);
  }
  __syncwarp();
  // epilogue: lane n of warp w holds output column n0 + 32 w + lane; sum the
  // P split terms of each row in a fixed order, store row-contiguous
  tc::mbar_wait(done, 0);
  tc::tc_fence_after();
  const uint32_t t_row = tmem + ((uint32_t)(warp * 32) << 16);
  float* dst = out + (int64_t)blockIdx.y * R * N + n0 + warp * 32 + lane;
  for (int r0 = 0; r0 < R; r0 += 32) {
    float acc[32];
    tc::tmem_ld32(t_row + r0, acc);
    tc::tmem_ld_wait();
    for (int p = 1; p < P; ++p) {
      float v[32];
      tc::tmem_ld32(t_row + p * R + r0, v);
      tc::tmem_ld_wait();
#pragma unroll
      for (int u = 0; u < 32; ++u) acc[u] += v[u];
    }
#pragma unroll
    for (int u = 0; u < 32; ++u) dst[(int64_t)(r0 + u) * N] = acc[u];
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<256>(tmem);
}

}  // namespace
}  // namespace ifkv

using namespace ifkv;

// x: bf16 [P][R][K] (contiguous), w: bf16 [N][K] ("out x in"), out: fp32
// [splits][R][N] (each K split's partial; the caller sums them).
extern "C" int ifkv_prompt_mm(const void* x, int P, int R, int K, const void* w, int N, int splits, float* out,
                              void* stream) {
  IFKV_CHECK_ARG(P >= 1 && R >= 32 && R % 32 == 0 && P * R <= 256 && K > 0 && K % kKStep == 0 && N > 0 &&
                     N % kN == 0,
                 "prompt_mm: needs R %% 32 == 0, P*R <= 256, K %% 64 == 0, N %% 128 == 0");
  const int k_steps = K / kKStep;
  IFKV_CHECK_ARG(splits >= 1 && splits <= k_steps, "prompt_mm: splits must be in [1, K/64]");
  IFKV_CHECK_ARG(((uintptr_t)x & 15) == 0 && ((uintptr_t)w & 15) == 0, "prompt_mm: operands must be 16-byte aligned");
  const int NR = P * R;  // MMA N
  CUtensorMap tw, tx;
  {
    uint64_t dims[2] = {(uint64_t)K, (uint64_t)N};
    uint64_t strides[1] = {(uint64_t)K * 2};
    uint32_t box[2] = {(uint32_t)kKStep, (uint32_t)kN};
    int rc = make_tmap_bf16(&tw, w, 2, dims, strides, box);
    if (rc) return rc;
  }
  {
    uint64_t dims[2] = {(uint64_t)K, (uint64_t)P * R};
    uint64_t strides[1] = {(uint64_t)K * 2};
    uint32_t box[2] = {(uint32_t)kKStep, (uint32_t)NR};
    int rc = make_tmap_bf16(&tx, x, 2, dims, strides, box);
    if (rc) return rc;
  }
#ifndef IFKV_PMM_STAGES
#define IFKV_PMM_STAGES 3
#endif
  constexpr int kStages = IFKV_PMM_STAGES;  // 3: 2 CTAs per SM at P*R = 96, 6 x 16 KB of W in flight per SM
  const int stage_bytes = kWStage + ((NR * 128 + 1023) & ~1023);
  const size_t smem = (size_t)kStages * stage_bytes + 1024 + 2 * kStages * 8 + 8 + 16;
  auto kern = prompt_mm_kernel<kStages>;
  IFKV_CUDA_CALL(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                 "prompt_mm: smem attribute");
  IFKV_CUDA_CALL(launch_pdl(kern, dim3(N / kN, splits), dim3(128), smem, as_stream(stream), tw, tx, P, R, NR, k_steps,
                            N, out),
                 "prompt_mm: launch");
  IFKV_LAUNCH_CHECK("prompt_mm");
  return IFKV_OK;
}
