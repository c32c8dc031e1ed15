// fp32-accurate prompt attention over bf16 context keys on the tcgen05 tensor
// cores: the attention-norm scorer and the prompt forward of the layers below
// the capture layer (reference selection.py:127-169, model.py:297-315).
//
// Accuracy: the selected set must match the float64 reference exactly, so
// every product is exact and every sum fp32: queries are fp32 split into
// three bf16 terms (q = q_hi + q_mid + q_lo, |residual| <= 2^-24 |q|), keys
// are bf16 (exact), S = sum_t Q_t K^T accumulates in fp32 TMEM; the fp32
// probabilities are split the same way for O = sum_t P_t V.
//
// One CTA = one work item (a run of <= 128 * kMaxBlocks keys that share one
// rotation delta) x one kv head x one chunk of <= 128 / M query heads (tile
// rows = heads x prompt rows).  The item's 128-key blocks stream through a
// 2-stage TMA ring; online softmax across blocks (O rescaled in TMEM, fp32).
// Warps: 0 TMA producer, 1 MMA issuer (+ TMEM alloc), 2-5 softmax (thread =
// tile row; TMEM lane quarter = warp % 4).
//   mode 0 (partial): (m, l, O) of the item -> part_ml / part_o
//   mode 1 (score):   p = exp(s - m_final) / l_final per block, column sums
//                     over the tile rows via a swizzled smem transpose ->
//                     colsum[item][chunk][key] (deterministic order)
// TMEM: S [0,128), P terms [128,320), O [384,512).
#include "tc_common.cuh"

namespace ifkv {
namespace {

constexpr int kPanel = 128 * 128;
constexpr int kTile = 2 * kPanel;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColS = 0, kColP = 128, kColO = 384;
constexpr float kRescale = 10.0f;  // natural-log units; p <= e^10 stays exact in fp32

struct PSmem {
  uint8_t q[3][kTile];  // hi / mid / lo query terms
  uint8_t k[2][kTile];
  uint8_t v[2][kTile];  // mode 1: transposed probabilities [128][128] fp32 (64 KB)
  uint64_t q_full, k_full[2], k_empty[2], v_full[2], v_empty[2];
  uint64_t s_full, s_free, p_full[2], pv_done;  // p_full: P published by 64-key halves
  uint32_t tmem_base;
};

// kMode is a template parameter so each mode gets its own register
// allocation (one kernel for both modes needed 255 registers and spilled).
template <int kMode>
__global__ void __launch_bounds__(192, 1)
    prompt_attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, const ifkv_attn_item* __restrict__ items, int H,
                          int Hkv, int M, int hpt, int n_hchunks, int item_keys, float scale,
                          float* __restrict__ part_ml, float* __restrict__ part_o,
                          const float* __restrict__ ml_final, float* __restrict__ colsum) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  PSmem& sm = *reinterpret_cast<PSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const ifkv_attn_item it = items[blockIdx.x];
  const int g = blockIdx.y, hc = blockIdx.z;
  const int G = H / Hkv;
  const int h0 = g * G + hc * hpt;
  const int R = min(hpt, G - hc * hpt) * M;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int box_rows = hpt * M;
  const int nblk = (it.n_keys + 127) / 128;

  if (threadIdx.x == 0) {
    tc::mbar_init(&sm.q_full, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&sm.k_full[i], 1);
      tc::mbar_init(&sm.k_empty[i], 1);
      tc::mbar_init(&sm.v_full[i], 1);
      tc::mbar_init(&sm.v_empty[i], 1);
    }
    tc::mbar_init(&sm.s_full, 1);
    tc::mbar_init(&sm.s_free, 128);
    tc::mbar_init(&sm.p_full[0], 128);
    tc::mbar_init(&sm.p_full[1], 128);
    tc::mbar_init(&sm.pv_done, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<kTmemCols>(&sm.tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&tm_q);
      tc::tma_prefetch(&tm_k);
      tc::mbar_arrive_expect_tx(&sm.q_full, 3 * 2 * box_rows * 128);
      for (int t = 0; t < 3; ++t) {
        const int y = ((it.qset * 3 + t) * H + h0) * M;
        tc::tma_load_2d(sm.q[t], &tm_q, &sm.q_full, 0, y);
        tc::tma_load_2d(sm.q[t] + kPanel, &tm_q, &sm.q_full, 64, y);
      }
      for (int j = 0; j < nblk; ++j) {
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        const int row0 = it.key_row0 + j * 128;
        tc::mbar_wait(&sm.k_empty[s], ph ^ 1);
        tc::mbar_arrive_expect_tx(&sm.k_full[s], kTile);
        tc::tma_load_2d(sm.k[s], &tm_k, &sm.k_full[s], g * 128, row0);
        tc::tma_load_2d(sm.k[s] + kPanel, &tm_k, &sm.k_full[s], g * 128 + 64, row0);
        if constexpr (kMode == 0) {
          tc::mbar_wait(&sm.v_empty[s], ph ^ 1);
          tc::mbar_arrive_expect_tx(&sm.v_full[s], kTile);
          tc::tma_load_2d(sm.v[s], &tm_v, &sm.v_full[s], g * 128, row0);
          tc::tma_load_2d(sm.v[s] + kPanel, &tm_v, &sm.v_full[s], g * 128 + 64, row0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_qk = tc::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idesc_pv = tc::idesc_bf16(128, 128, 0, 1);
      tc::mbar_wait(&sm.q_full, 0);
      // S(j) = sum_t Q_t K_j^T; issued one block ahead so the tensor core
      // computes S(j+1) while the softmax warps turn S(j) into P(j).
      auto issue_s = [&](int j) {
        const int s = j & 1;
        tc::mbar_wait(&sm.k_full[s], (j >> 1) & 1);
        tc::mbar_wait(&sm.s_free, (j & 1) ^ 1);  // softmax has read S(j-1)
        tc::tc_fence_after();
        const uint32_t k_addr = tc::smem_u32(sm.k[s]);
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
        tc::mma_commit(&sm.k_empty[s]);
      };
      issue_s(0);
      for (int j = 0; j < nblk; ++j) {
        if (j + 1 < nblk) issue_s(j + 1);
        if constexpr (kMode == 0) {
          const int s = j & 1;
          tc::mbar_wait(&sm.v_full[s], (j >> 1) & 1);
          const uint32_t v_addr = tc::smem_u32(sm.v[s]);
          // PV by 64-key halves as the softmax publishes them (fixed order:
          // half, term, key step)
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            tc::mbar_wait(&sm.p_full[hf], j & 1);
            tc::tc_fence_after();
#pragma unroll
            for (int t = 0; t < 3; ++t) {
#pragma unroll
              for (int kk = 4 * hf; kk < 4 * hf + 4; ++kk) {
                uint64_t b = tc::smem_desc_sw128(v_addr + kk * 2048, kPanel, 1024);
                tc::mma_bf16_ts(tmem + kColO, tmem + kColP + 64 * t + 8 * kk, b, idesc_pv,
                                (j > 0 || t > 0 || kk > 0) ? 1u : 0u);
              }
            }
          }
          tc::mma_commit(&sm.pv_done);
          tc::mma_commit(&sm.v_empty[s]);
        }
      }
    }
  } else {
    // ---- softmax warps 2..5: thread owns tile row `row` -----------------------
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const bool valid = row < R;
    const int h = h0 + (valid ? row / M : 0);
    const int m = valid ? row % M : 0;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    // m_used: running max of the RAW scores; exponentials in log2 units
    const float sl2 = scale * 1.4426950408889634f;
    float m_used = -INFINITY, l = 0.f, mf2 = 0.f, inv_lf = 0.f;
    if (kMode == 1 && valid) {
      const int64_t s = 2 * (((int64_t)it.group * H + h) * M + m);
      mf2 = ml_final[s] * 1.4426950408889634f;  // natural-unit max of the scaled logits -> log2 units
      inv_lf = 1.f / ml_final[s + 1];
    }
    float* T = reinterpret_cast<float*>(sm.v[0]);  // mode 1 transpose, [key][row ^ (key & 31)]
    for (int j = 0; j < nblk; ++j) {
      const int nk = min(128, it.n_keys - j * 128);
      float v[128];
      tc::mbar_wait(&sm.s_full, j & 1);
      tc::tc_fence_after();
#pragma unroll
      for (int q = 0; q < 4; ++q) tc::tmem_ld32(tmem + lane_off + kColS + 32 * q, v + 32 * q);
      tc::tmem_ld_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&sm.s_free);  // S may be overwritten by S(j+1) from here on
      if (nk < 128) {  // last block of a run only
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (c >= nk) v[c] = -INFINITY;
      }
      if constexpr (kMode == 0) {
        // raw-score max (scale > 0 commutes with max), four FMNMX3 chains
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 128; c += 8) {
          m4[0] = tc::max3(m4[0], v[c], v[c + 1]);
          m4[1] = tc::max3(m4[1], v[c + 2], v[c + 3]);
          m4[2] = tc::max3(m4[2], v[c + 4], v[c + 5]);
          m4[3] = tc::max3(m4[3], v[c + 6], v[c + 7]);
        }
        const float mx = tc::max3(m4[0], m4[1], fmaxf(m4[2], m4[3]));
        float alpha = 1.f;
        bool need = false;
        if (m_used == -INFINITY || (mx - m_used) * scale > kRescale) {
          need = true;
          alpha = m_used == -INFINITY ? 0.f : tc::ex2((m_used - mx) * sl2);
          m_used = mx;
        }
        // p = 2^(s sl2 - m sl2): packed FFMA2 + MUFU ex2 (fp32 accurate to ~2 ulp)
        const float2 sc2 = make_float2(sl2, sl2), mb2 = make_float2(-m_used * sl2, -m_used * sl2);
        float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < 128; c += 2) {
          const float2 x = tc::ffma2(make_float2(v[c], v[c + 1]), sc2, mb2);
          const float2 e = make_float2(tc::ex2(x.x), tc::ex2(x.y));
          v[c] = e.x;
          v[c + 1] = e.y;
          sum2[(c >> 1) & 1] = tc::fadd2(sum2[(c >> 1) & 1], e);
        }
        const float sum = (sum2[0].x + sum2[1].x) + (sum2[0].y + sum2[1].y);
        // P(j-1) consumed and O = PV(0..j-1) complete
        if (j > 0) tc::mbar_wait(&sm.pv_done, (j - 1) & 1);
        tc::tc_fence_after();
        // P = hi + mid + lo (bf16 pairs), term t at TMEM cols kColP + 64 t + key / 2,
        // published by 64-key halves so PV on keys 0..63 overlaps the second half
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
          for (int q = 4 * hf; q < 4 * hf + 4; ++q) {  // 8-column stores keep the split terms' registers low
            uint32_t p0[8], p1[8], p2[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
              tc::split3_pair(v[16 * q + 2 * u], v[16 * q + 2 * u + 1], p0[u], p1[u], p2[u]);
            tc::tmem_st8(tmem + lane_off + kColP + 0 * 64 + 8 * q, p0);
            tc::tmem_st8(tmem + lane_off + kColP + 1 * 64 + 8 * q, p1);
            tc::tmem_st8(tmem + lane_off + kColP + 2 * 64 + 8 * q, p2);
          }
          // O rescale before the first PV of this block reads O
          if (hf == 0 && j > 0 && __any_sync(0xffffffffu, need)) {
            const float a = need ? alpha : 1.f;
#pragma unroll 1
            for (int c = 0; c < 8; ++c) {
              float o[16];
              tc::tmem_ld16(tmem + lane_off + kColO + c * 16, o);
              tc::tmem_ld_wait();
#pragma unroll
              for (int u = 0; u < 16; ++u) o[u] *= a;
              tc::tmem_st16(tmem + lane_off + kColO + c * 16, reinterpret_cast<const uint32_t*>(o));
            }
          }
          tc::tmem_st_wait();
          tc::tc_fence_before();
          tc::mbar_arrive(&sm.p_full[hf]);
        }
        l = l * alpha + sum;
      } else {
        // p = exp(s - m_final) / l_final -> transposed smem -> column sums
        asm volatile("bar.sync 1, 128;" ::: "memory");  // previous block's column reads done
#pragma unroll
        for (int c = 0; c < 128; ++c)
          T[c * 128 + (row ^ (c & 31))] = valid ? tc::ex2(fmaf(v[c], sl2, -mf2)) * inv_lf : 0.f;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const int c = row;  // this thread sums key column c over the tile rows
        float acc = 0.f;
        for (int r = 0; r < R; ++r) acc += T[c * 128 + (r ^ (c & 31))];
        if (c < nk)
          colsum[((int64_t)blockIdx.x * (Hkv * n_hchunks) + g * n_hchunks + hc) * item_keys + j * 128 + c] = acc;
      }
    }
    if constexpr (kMode == 0) {
      tc::mbar_wait(&sm.pv_done, (nblk - 1) & 1);
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
        part_ml[2 * row_id] = m_used * scale;  // natural units of the scaled logits
        part_ml[2 * row_id + 1] = l;
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<kTmemCols>(tmem);
}

__global__ void colsum_finalize_kernel(const ifkv_attn_item* __restrict__ items, const float* __restrict__ colsum,
                                       int n_chunks, int item_keys, float inv_h, float* __restrict__ scores) {
  const ifkv_attn_item it = items[blockIdx.x];
  if (!it.score || it.prompt) return;
  for (int c = threadIdx.x; c < it.n_keys; c += blockDim.x) {
    const float* src = colsum + (int64_t)blockIdx.x * n_chunks * item_keys + c;
    float acc = 0.f;
    for (int k = 0; k < n_chunks; ++k) acc += src[(int64_t)k * item_keys];
    scores[it.key_row0 + c] = acc * inv_h;
  }
}

}  // namespace
}  // namespace ifkv

using namespace ifkv;

extern "C" int ifkv_prompt_attn_tc_supported(int kv_dtype, int H, int Hkv, int M, int Dh) {
  if (kv_dtype != IFKV_BF16 || Dh != 128 || Hkv <= 0 || H % Hkv || M <= 0 || M > 128) return 0;
  return 1;
}

static int launch_prompt_tc(int mode, const __nv_bfloat16* qd3, int n_qsets, const void* k_slab, const void* v_slab,
                            int n_rows, const ifkv_attn_item* items, int n_items, int item_keys, int H, int Hkv,
                            int M, float scale, float* part_ml, float* part_o, const float* ml_final, float* colsum,
                            void* stream) {
  IFKV_CHECK_ARG(ifkv_prompt_attn_tc_supported(IFKV_BF16, H, Hkv, M, 128), "prompt_attn_tc: unsupported shape");
  IFKV_CHECK_ARG(item_keys >= 1 && item_keys % 128 == 0, "prompt_attn_tc: item_keys must be a multiple of 128");
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
  auto kern = mode == 0 ? prompt_attn_tc_kernel<0> : prompt_attn_tc_kernel<1>;
  IFKV_CUDA_CALL(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                 "prompt_attn_tc: smem attribute");
  dim3 grid(n_items, Hkv, n_hchunks);
  kern<<<grid, 192, smem, as_stream(stream)>>>(tq, tk, tv, items, H, Hkv, M, hpt, n_hchunks, item_keys, scale, part_ml,
                                               part_o, ml_final, colsum);
  IFKV_LAUNCH_CHECK("prompt_attn_tc");
  return IFKV_OK;
}

extern "C" int ifkv_prompt_attn_partial_tc(const void* qd3, int n_qsets, const void* k_slab, const void* v_slab,
                                           int n_rows, const ifkv_attn_item* items, int n_items, int item_keys, int H,
                                           int Hkv, int M, float scale, float* part_ml, float* part_o, void* stream) {
  return launch_prompt_tc(0, (const __nv_bfloat16*)qd3, n_qsets, k_slab, v_slab, n_rows, items, n_items, item_keys,
                          H, Hkv, M, scale, part_ml, part_o, nullptr, nullptr, stream);
}

extern "C" int ifkv_score_columns_tc(const void* qd3, int n_qsets, const void* k_slab, int n_rows,
                                     const ifkv_attn_item* items, int n_items, int item_keys, const float* ml, int H,
                                     int Hkv, int M, float scale, float* colsum_ws, float* scores, void* stream) {
  int rc = launch_prompt_tc(1, (const __nv_bfloat16*)qd3, n_qsets, k_slab, nullptr, n_rows, items, n_items,
                            item_keys, H, Hkv, M, scale, nullptr, nullptr, ml, colsum_ws, stream);
  if (rc) return rc;
  if (n_items <= 0) return IFKV_OK;
  const int G = H / Hkv;
  const int hpt = (128 / M) < G ? (128 / M) : G;
  const int n_chunks = Hkv * ((G + hpt - 1) / hpt);
  colsum_finalize_kernel<<<n_items, 256, 0, as_stream(stream)>>>(items, colsum_ws, n_chunks, item_keys,
                                                                 1.f / (float)H, scores);
  IFKV_LAUNCH_CHECK("colsum_finalize");
  return IFKV_OK;
}
