// fp32-accurate prompt attention over bf16 context keys on the tcgen05 tensor
// cores: the attention-norm scorer and the prompt forward of layers below the
// capture layer (reference selection.py:127-169, model.py:297-315).
//
// Accuracy: the selected set must match the float64 reference exactly, so
// every product is exact and every sum fp32: queries are fp32 split into
// three bf16 terms (q = q_hi + q_mid + q_lo, |residual| <= 2^-24 |q|), keys
// are bf16 (exact), S = sum_t Q_t K^T accumulates in fp32 TMEM; the fp32
// probabilities are split the same way for O = sum_t P_t V.
//
// One CTA = one work item (<= 128 keys of one constant-delta run) x one kv
// head x one chunk of <= 128 / M query heads (rows = heads x prompt rows).
// 128 threads; thread 0 issues TMA and MMAs; thread r owns TMEM lane r.
//   mode 0 (partial): row max m, l = sum p, O = P V -> part_ml / part_o
//   mode 1 (score):   p = exp(s - m_final) / l_final; column sums over the
//                     tile's rows -> colsum[item][chunk][128] (deterministic)
// TMEM: S [0,128), P terms [128,320), O [384,512).
#include "tc_common.cuh"

namespace ifkv {
namespace {

constexpr int kPanel = 128 * 128;
constexpr int kTile = 2 * kPanel;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColS = 0, kColP = 128, kColO = 384;

struct PSmem {
  uint8_t q[3][kTile];  // split query terms; reused as the transposed P in mode 1
  uint8_t k[kTile];
  uint8_t v[kTile];
  uint64_t qk_full, v_full, s_full, p_full, o_full;
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(128, 1)
    prompt_attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, const ifkv_attn_item* __restrict__ items, int H,
                          int Hkv, int M, int hpt, int n_hchunks, float scale, int mode,
                          float* __restrict__ part_ml, float* __restrict__ part_o,
                          const float* __restrict__ ml_final, float* __restrict__ colsum) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  PSmem& sm = *reinterpret_cast<PSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const ifkv_attn_item it = items[blockIdx.x];
  const int g = blockIdx.y, hc = blockIdx.z;
  const int G = H / Hkv;
  const int h0 = g * G + hc * hpt;
  const int heads = min(hpt, G - hc * hpt);
  const int R = heads * M;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int box_rows = hpt * M;

  if (tid == 0) {
    tc::mbar_init(&sm.qk_full, 1);
    tc::mbar_init(&sm.v_full, 1);
    tc::mbar_init(&sm.s_full, 1);
    tc::mbar_init(&sm.p_full, 128);
    tc::mbar_init(&sm.o_full, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc<kTmemCols>(&sm.tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (tid == 0) {
    tc::tma_prefetch(&tm_q);
    tc::tma_prefetch(&tm_k);
    tc::mbar_arrive_expect_tx(&sm.qk_full, 3 * 2 * box_rows * 128 + kTile);
    for (int t = 0; t < 3; ++t) {
      const int y = ((it.qset * 3 + t) * H + h0) * M;
      tc::tma_load_2d(sm.q[t], &tm_q, &sm.qk_full, 0, y);
      tc::tma_load_2d(sm.q[t] + kPanel, &tm_q, &sm.qk_full, 64, y);
    }
    tc::tma_load_2d(sm.k, &tm_k, &sm.qk_full, g * 128, it.key_row0);
    tc::tma_load_2d(sm.k + kPanel, &tm_k, &sm.qk_full, g * 128 + 64, it.key_row0);
    if (mode == 0) {
      tc::mbar_arrive_expect_tx(&sm.v_full, kTile);
      tc::tma_load_2d(sm.v, &tm_v, &sm.v_full, g * 128, it.key_row0);
      tc::tma_load_2d(sm.v + kPanel, &tm_v, &sm.v_full, g * 128 + 64, it.key_row0);
    }
    constexpr uint32_t idesc_qk = tc::idesc_bf16(128, 128, 0, 0);
    tc::mbar_wait(&sm.qk_full, 0);
    tc::tc_fence_after();
    const uint32_t k_addr = tc::smem_u32(sm.k);
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const uint32_t q_addr = tc::smem_u32(sm.q[t]);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        uint64_t a = tc::smem_desc_sw128(q_addr + (kk >> 2) * kPanel + (kk & 3) * 32, 16, 1024);
        uint64_t b = tc::smem_desc_sw128(k_addr + (kk >> 2) * kPanel + (kk & 3) * 32, 16, 1024);
        tc::mma_bf16_ss(tmem + kColS, a, b, idesc_qk, (t > 0 || kk > 0) ? 1u : 0u);
      }
    }
    tc::mma_commit(&sm.s_full);
  }
  __syncwarp();

  // ---- softmax: thread tid owns row tid ------------------------------------
  const int row = tid;
  const bool valid = row < R;
  const int h = h0 + (valid ? row / M : 0);
  const int m = valid ? row % M : 0;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  float p[128];
  tc::mbar_wait(&sm.s_full, 0);
  tc::tc_fence_after();
#pragma unroll
  for (int c = 0; c < 4; ++c) tc::tmem_ld32(tmem + lane_off + kColS + c * 32, p + c * 32);
  tc::tmem_ld_wait();
  const int n = it.n_keys;
  float mx, l;
  if (mode == 0) {
    mx = -INFINITY;
#pragma unroll
    for (int c = 0; c < 128; ++c) {
      p[c] = c < n ? p[c] * scale : -INFINITY;
      mx = fmaxf(mx, p[c]);
    }
    l = 0.f;
#pragma unroll
    for (int c = 0; c < 128; ++c) {
      p[c] = c < n ? expf(p[c] - mx) : 0.f;
      l += p[c];
    }
  } else {
    const int64_t s = 2 * (((int64_t)it.group * H + h) * M + m);
    mx = valid ? ml_final[s] : 0.f;
    const float inv_l = valid ? 1.f / ml_final[s + 1] : 0.f;
    l = 0.f;
#pragma unroll
    for (int c = 0; c < 128; ++c) p[c] = (c < n && valid) ? expf(p[c] * scale - mx) * inv_l : 0.f;
  }

  if (mode == 0) {
    // P = hi + mid + lo (bf16) -> TMEM columns kColP + 64 t + c / 2
#pragma unroll
    for (int t = 0; t < 3; ++t) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float packed[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const int c = half * 64 + 2 * u;
          __nv_bfloat16 a0, a1, a2, b0, b1, b2;
          split3(p[c], a0, a1, a2);
          split3(p[c + 1], b0, b1, b2);
          __nv_bfloat16 lo = t == 0 ? a0 : (t == 1 ? a1 : a2);
          __nv_bfloat16 hi = t == 0 ? b0 : (t == 1 ? b1 : b2);
          __nv_bfloat162 pr;
          pr.x = lo;
          pr.y = hi;
          packed[u] = *reinterpret_cast<float*>(&pr);
        }
        tc::tmem_st32(tmem + lane_off + kColP + 64 * t + 32 * half, packed);
      }
    }
    tc::tmem_st_wait();
    tc::tc_fence_before();
    tc::mbar_arrive(&sm.p_full);
    if (tid == 0) {
      constexpr uint32_t idesc_pv = tc::idesc_bf16(128, 128, 0, 1);
      tc::mbar_wait(&sm.p_full, 0);
      tc::mbar_wait(&sm.v_full, 0);
      tc::tc_fence_after();
      const uint32_t v_addr = tc::smem_u32(sm.v);
#pragma unroll
      for (int t = 0; t < 3; ++t) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          uint64_t b = tc::smem_desc_sw128(v_addr + kk * 2048, kPanel, 1024);
          tc::mma_bf16_ts(tmem + kColO, tmem + kColP + 64 * t + 8 * kk, b, idesc_pv, (t > 0 || kk > 0) ? 1u : 0u);
        }
      }
      tc::mma_commit(&sm.o_full);
    }
    __syncwarp();
    tc::mbar_wait(&sm.o_full, 0);
    tc::tc_fence_after();
    const int64_t row_id = ((int64_t)blockIdx.x * H + h) * M + m;
    float* dst = part_o + row_id * 128;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float o[32];
      tc::tmem_ld32(tmem + lane_off + kColO + c * 32, o);
      tc::tmem_ld_wait();
      if (valid) {
#pragma unroll
        for (int u = 0; u < 32; u += 4)
          *reinterpret_cast<float4*>(dst + c * 32 + u) = make_float4(o[u], o[u + 1], o[u + 2], o[u + 3]);
      }
    }
    if (valid) {
      part_ml[2 * row_id] = mx;
      part_ml[2 * row_id + 1] = l;
    }
  } else {
    // column sums over the tile's rows via a transposed fp32 copy in smem
    float* T = reinterpret_cast<float*>(sm.q[0]);  // [128 keys][129]
#pragma unroll
    for (int c = 0; c < 128; ++c) T[c * 129 + row] = p[c];
    __syncthreads();
    const int c = tid;
    float acc = 0.f;
    for (int r = 0; r < R; ++r) acc += T[c * 129 + r];
    colsum[((int64_t)blockIdx.x * (Hkv * n_hchunks) + g * n_hchunks + hc) * 128 + c] = acc;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<kTmemCols>(tmem);
}

__global__ void colsum_finalize_kernel(const ifkv_attn_item* __restrict__ items, const float* __restrict__ colsum,
                                       int n_chunks, float inv_h, float* __restrict__ scores) {
  const ifkv_attn_item it = items[blockIdx.x];
  const int c = threadIdx.x;
  if (!it.score || it.prompt || c >= it.n_keys) return;
  const float* src = colsum + (int64_t)blockIdx.x * n_chunks * 128 + c;
  float acc = 0.f;
  for (int k = 0; k < n_chunks; ++k) acc += src[k * 128];
  scores[it.key_row0 + c] = acc * inv_h;
}

}  // namespace
}  // namespace ifkv

using namespace ifkv;

extern "C" int ifkv_prompt_attn_tc_supported(int kv_dtype, int H, int Hkv, int M, int Dh) {
  if (kv_dtype != IFKV_BF16 || Dh != 128 || Hkv <= 0 || H % Hkv || M <= 0 || M > 128) return 0;
  return 1;
}

static int launch_prompt_tc(int mode, const __nv_bfloat16* qd3, int n_qsets, const void* k_slab, const void* v_slab,
                            int n_rows, const ifkv_attn_item* items, int n_items, int H, int Hkv, int M, float scale,
                            float* part_ml, float* part_o, const float* ml_final, float* colsum, void* stream) {
  IFKV_CHECK_ARG(ifkv_prompt_attn_tc_supported(IFKV_BF16, H, Hkv, M, 128), "prompt_attn_tc: unsupported shape");
  if (n_items <= 0) return IFKV_OK;
  const int G = H / Hkv;
  const int hpt = (128 / M) < G ? (128 / M) : G;
  const int n_hchunks = (G + hpt - 1) / hpt;
  CUtensorMap tq, tk, tv;
  {
    uint64_t dims[2] = {128, (uint64_t)n_qsets * 3 * H * M};
    uint64_t strides[1] = {256};
    uint32_t box[2] = {64, (uint32_t)(hpt * M)};
    int rc = make_tmap_bf16(&tq, qd3, 2, dims, strides, box);
    if (rc) return rc;
  }
  {
    uint64_t dims[2] = {(uint64_t)Hkv * 128, (uint64_t)n_rows};
    uint64_t strides[1] = {(uint64_t)Hkv * 256};
    uint32_t box[2] = {64, 128};
    int rc = make_tmap_bf16(&tk, k_slab, 2, dims, strides, box);
    if (rc) return rc;
    rc = make_tmap_bf16(&tv, v_slab ? v_slab : k_slab, 2, dims, strides, box);
    if (rc) return rc;
  }
  const size_t smem = sizeof(PSmem) + 1024;
  IFKV_CUDA_CALL(cudaFuncSetAttribute(prompt_attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                 "prompt_attn_tc: smem attribute");
  dim3 grid(n_items, Hkv, n_hchunks);
  prompt_attn_tc_kernel<<<grid, 128, smem, as_stream(stream)>>>(tq, tk, tv, items, H, Hkv, M, hpt, n_hchunks, scale,
                                                               mode, part_ml, part_o, ml_final, colsum);
  IFKV_LAUNCH_CHECK("prompt_attn_tc");
  return IFKV_OK;
}

extern "C" int ifkv_prompt_attn_partial_tc(const void* qd3, int n_qsets, const void* k_slab, const void* v_slab,
                                           int n_rows, const ifkv_attn_item* items, int n_items, int H, int Hkv,
                                           int M, float scale, float* part_ml, float* part_o, void* stream) {
  return launch_prompt_tc(0, (const __nv_bfloat16*)qd3, n_qsets, k_slab, v_slab, n_rows, items, n_items, H, Hkv, M,
                          scale, part_ml, part_o, nullptr, nullptr, stream);
}

extern "C" int ifkv_score_columns_tc(const void* qd3, int n_qsets, const void* k_slab, int n_rows,
                                     const ifkv_attn_item* items, int n_items, const float* ml, int H, int Hkv, int M,
                                     float scale, float* colsum_ws, float* scores, void* stream) {
  int rc = launch_prompt_tc(1, (const __nv_bfloat16*)qd3, n_qsets, k_slab, nullptr, n_rows, items, n_items, H, Hkv,
                            M, scale, nullptr, nullptr, ml, colsum_ws, stream);
  if (rc) return rc;
  if (n_items <= 0) return IFKV_OK;
  const int G = H / Hkv;
  const int hpt = (128 / M) < G ? (128 / M) : G;
  const int n_chunks = Hkv * ((G + hpt - 1) / hpt);
  colsum_finalize_kernel<<<n_items, 128, 0, as_stream(stream)>>>(items, colsum_ws, n_chunks, 1.f / (float)H, scores);
  IFKV_LAUNCH_CHECK("colsum_finalize");
  return IFKV_OK;
}
