// Selective-recompute attention on the 5th-gen tensor cores (tcgen05 + TMEM
// + TMA), bf16 in / fp32 softmax / bf16 out, Dh = 128, any GQA ratio that is a
// multiple of ... 4 query heads per tile row group (H/Hkv = 4, Llama-3-8B) or
// 1/2/8 (tile rows = 128 = tokens x group heads).
//
// Reference: recompute.py:92-114 (selected queries vs all context keys,
// causal by global index) with masked_attention model.py:297-315.
//
// Tile: one CTA = 128 query rows = (128 / G) selected tokens x the G query
// heads of one kv head (GQA packing: the K/V tile loaded once serves all G
// heads).  Row r = token r / G, head r % G.  Key blocks of 128; the tile's key
// span ends at the horizon of its last token (selected tokens ascending).
//
// Warp roles (256 threads):
//   warp 0  TMA producer: Q once; K and V tiles, 2-stage rings
//   warp 1  MMA issuer (one thread): S = Q K^T into TMEM (double-buffered),
//           O += P V into TMEM
//   warp 2  TMEM allocator
//   warps 4-7 softmax: thread = one query row; S row via tcgen05.ld, causal
//           mask, online softmax with lazy rescale (only when the running max
//           grows by > 2^8), P -> bf16 -> 128B-swizzled smem (K-major A of the
//           PV MMA); epilogue O / l -> bf16 -> global.
// smem: Q 32 KB + K 2x32 KB + V 2x32 KB + P 2x32 KB = 224 KB.
// TMEM: S0 cols [0,128), S1 [128,256), O [256,384) of a 512-col allocation.
#include "tc_common.cuh"

namespace ifkv {
namespace {

constexpr int kRows = 128;        // query rows per tile
constexpr int kKeys = 128;        // keys per block
constexpr int kDh = 128;
constexpr int kPanel = 128 * 128;  // bytes of one 128-row x 64-col bf16 panel
constexpr int kTileBytes = 2 * kPanel;
constexpr uint32_t kTmemCols = 512;
constexpr float kRescaleLog2 = 8.0f;

struct Smem {
  uint8_t q[kTileBytes];
  uint8_t k[2][kTileBytes];
  uint8_t v[2][kTileBytes];
  uint8_t p[2][kTileBytes];
  uint64_t q_full;
  uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2];
  uint64_t s_full[2], s_free[2], p_full[2], pv_done[2];
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(256, 1)
    recompute_attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                             const __grid_constant__ CUtensorMap tm_v, const int64_t* __restrict__ horizon, int S,
                             int H, int Hkv, float scale_log2, __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = H / Hkv;                 // query heads per kv head
  const int tok_per_tile = kRows / G;
  const int g = blockIdx.x;              // kv head
  const int tile = gridDim.y - 1 - blockIdx.y;  // heaviest (latest) tiles first
  const int t0 = tile * tok_per_tile;
  const int t_last = min(t0 + tok_per_tile, S) - 1;
  const int64_t max_h = horizon[t_last];
  const int nblk = (int)((max_h + kKeys) / kKeys);

  if (threadIdx.x == 0) {
    tc::mbar_init(&sm.q_full, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&sm.k_full[i], 1);
      tc::mbar_init(&sm.k_empty[i], 1);
      tc::mbar_init(&sm.v_full[i], 1);
      tc::mbar_init(&sm.v_empty[i], 1);
      tc::mbar_init(&sm.s_full[i], 1);
      tc::mbar_init(&sm.s_free[i], 128);
      tc::mbar_init(&sm.p_full[i], 128);
      tc::mbar_init(&sm.pv_done[i], 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc<kTmemCols>(&sm.tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const uint32_t tm_s0 = tmem, tm_o = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&tm_q);
      tc::tma_prefetch(&tm_k);
      tc::tma_prefetch(&tm_v);
      tc::mbar_arrive_expect_tx(&sm.q_full, kTileBytes);
      tc::tma_load_3d(sm.q, &tm_q, &sm.q_full, 0, g * G, t0);
      tc::tma_load_3d(sm.q + kPanel, &tm_q, &sm.q_full, 64, g * G, t0);
      for (int j = 0; j < nblk; ++j) {
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        tc::mbar_wait(&sm.k_empty[s], ph ^ 1);
        tc::mbar_arrive_expect_tx(&sm.k_full[s], kTileBytes);
        tc::tma_load_2d(sm.k[s], &tm_k, &sm.k_full[s], g * kDh, j * kKeys);
        tc::tma_load_2d(sm.k[s] + kPanel, &tm_k, &sm.k_full[s], g * kDh + 64, j * kKeys);
        tc::mbar_wait(&sm.v_empty[s], ph ^ 1);
        tc::mbar_arrive_expect_tx(&sm.v_full[s], kTileBytes);
        tc::tma_load_2d(sm.v[s], &tm_v, &sm.v_full[s], g * kDh, j * kKeys);
        tc::tma_load_2d(sm.v[s] + kPanel, &tm_v, &sm.v_full[s], g * kDh + 64, j * kKeys);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_qk = tc::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idesc_pv = tc::idesc_bf16(128, 128, 0, 1);
      const uint32_t q_addr = tc::smem_u32(sm.q);
      tc::mbar_wait(&sm.q_full, 0);
      auto issue_pv = [&](int i) {
        const int s = i & 1;
        const uint32_t ph = (i >> 1) & 1;
        tc::mbar_wait(&sm.p_full[s], ph);
        tc::mbar_wait(&sm.v_full[s], ph);
        tc::tc_fence_after();
        const uint32_t p_addr = tc::smem_u32(sm.p[s]);
        const uint32_t v_addr = tc::smem_u32(sm.v[s]);
#pragma unroll
        for (int t = 0; t < kKeys / 16; ++t) {
          // A = P (K-major over keys): panel t/4, 32-byte step t%4
          uint64_t a = tc::smem_desc_sw128(p_addr + (t >> 2) * kPanel + (t & 3) * 32, 16, 1024);
          // B = V (MN-major over dims): 16 keys = 2 atoms of 8 rows, dims groups LBO apart
          uint64_t b = tc::smem_desc_sw128(v_addr + t * 2048, kPanel, 1024);
          tc::mma_bf16_ss(tm_o, a, b, idesc_pv, (i > 0 || t > 0) ? 1u : 0u);
        }
        tc::mma_commit(&sm.pv_done[s]);
        tc::mma_commit(&sm.v_empty[s]);
      };
      for (int j = 0; j < nblk; ++j) {
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        tc::mbar_wait(&sm.k_full[s], ph);
        tc::mbar_wait(&sm.s_free[s], ph ^ 1);
        tc::tc_fence_after();
        const uint32_t k_addr = tc::smem_u32(sm.k[s]);
#pragma unroll
        for (int t = 0; t < kDh / 16; ++t) {
          uint64_t a = tc::smem_desc_sw128(q_addr + (t >> 2) * kPanel + (t & 3) * 32, 16, 1024);
          uint64_t b = tc::smem_desc_sw128(k_addr + (t >> 2) * kPanel + (t & 3) * 32, 16, 1024);
          tc::mma_bf16_ss(tm_s0 + s * 128, a, b, idesc_qk, t > 0 ? 1u : 0u);
        }
        tc::mma_commit(&sm.s_full[s]);
        tc::mma_commit(&sm.k_empty[s]);
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(nblk - 1);
    }
  } else if (warp >= 4) {
    const int w = warp - 4;
    const int row = w * 32 + lane;
    const int tok = t0 + row / G;
    const bool valid = tok < S;
    const int hz = valid ? (int)horizon[tok] : 0;
    const uint32_t lane_off = (uint32_t)(w * 32) << 16;
    float m_used = -INFINITY, l = 0.f;
    float v[kKeys];
    for (int j = 0; j < nblk; ++j) {
      const int s = j & 1;
      const uint32_t ph = (j >> 1) & 1;
      tc::mbar_wait(&sm.s_full[s], ph);
      tc::tc_fence_after();
#pragma unroll
      for (int c = 0; c < kKeys / 32; ++c) tc::tmem_ld32(tm_s0 + lane_off + s * 128 + c * 32, v + c * 32);
      tc::tmem_ld_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&sm.s_free[s]);
      const int j0 = j * kKeys;
      // causal mask only where the block crosses this warp's horizons
      if (__any_sync(0xffffffffu, j0 + kKeys - 1 > hz)) {
#pragma unroll
        for (int c = 0; c < kKeys; ++c)
          if (j0 + c > hz) v[c] = -INFINITY;
      }
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < kKeys; c += 2) mx = tc::max3(mx, v[c], v[c + 1]);
      float alpha = 1.f;
      bool need = false;
      if (mx > -INFINITY && (m_used == -INFINITY || (mx - m_used) * scale_log2 > kRescaleLog2)) {
        need = true;
        alpha = m_used == -INFINITY ? 0.f : tc::ex2((m_used - mx) * scale_log2);
        m_used = mx;
      }
      const float mb = m_used == -INFINITY ? 0.f : m_used * scale_log2;
      float sum = 0.f;
      // P buffer s was last read by PV(j - 2)
      if (j >= 2) tc::mbar_wait(&sm.pv_done[s], ((j - 2) >> 1) & 1);
      uint8_t* prow = sm.p[s] + row * 128;
#pragma unroll
      for (int ch = 0; ch < kKeys / 8; ++ch) {
        float e[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          e[u] = tc::ex2(fmaf(v[ch * 8 + u], scale_log2, -mb));  // ex2.approx.ftz(-inf) = +0
          sum += e[u];
        }
        uint4 pk;
        pk.x = tc::pack_bf16(e[0], e[1]);
        pk.y = tc::pack_bf16(e[2], e[3]);
        pk.z = tc::pack_bf16(e[4], e[5]);
        pk.w = tc::pack_bf16(e[6], e[7]);
        const int panel = ch >> 3, c16 = ch & 7;
        *reinterpret_cast<uint4*>(prow + panel * kPanel + ((c16 ^ (row & 7)) << 4)) = pk;
      }
      l = l * alpha + sum;
      if (j > 0 && __any_sync(0xffffffffu, need)) {
        // O holds PV(0..j-1): wait for PV(j-1), rescale this warp's rows in TMEM
        tc::mbar_wait(&sm.pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
        tc::tc_fence_after();
        const float a = need ? alpha : 1.f;
#pragma unroll
        for (int c = 0; c < kDh / 32; ++c) {
          float o[32];
          tc::tmem_ld32(tm_o + lane_off + c * 32, o);
          tc::tmem_ld_wait();
#pragma unroll
          for (int u = 0; u < 32; ++u) o[u] *= a;
          tc::tmem_st32(tm_o + lane_off + c * 32, o);
        }
        tc::tmem_st_wait();
      }
      tc::fence_async_smem();
      tc::tc_fence_before();
      tc::mbar_arrive(&sm.p_full[s]);
    }
    // epilogue: O / l -> bf16 -> out[token][g*G + row%G][:]
    tc::mbar_wait(&sm.pv_done[(nblk - 1) & 1], ((nblk - 1) >> 1) & 1);
    tc::tc_fence_after();
    const float inv = 1.f / l;
    __nv_bfloat16* dst = out + ((int64_t)tok * H + g * G + row % G) * kDh;
#pragma unroll
    for (int c = 0; c < kDh / 32; ++c) {
      float o[32];
      tc::tmem_ld32(tm_o + lane_off + c * 32, o);
      tc::tmem_ld_wait();
      if (valid) {
#pragma unroll
        for (int u = 0; u < 32; u += 8) {
          uint4 pk;
          pk.x = tc::pack_bf16(o[u] * inv, o[u + 1] * inv);
          pk.y = tc::pack_bf16(o[u + 2] * inv, o[u + 3] * inv);
          pk.z = tc::pack_bf16(o[u + 4] * inv, o[u + 5] * inv);
          pk.w = tc::pack_bf16(o[u + 6] * inv, o[u + 7] * inv);
          *reinterpret_cast<uint4*>(dst + c * 32 + u) = pk;
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) tc::tmem_dealloc<kTmemCols>(tmem);
}

}  // namespace
}  // namespace ifkv

using namespace ifkv;

extern "C" int ifkv_recompute_attn_tc_supported(int dtype, int H, int Hkv, int Dh) {
  if (dtype != IFKV_BF16 || Dh != kDh || Hkv <= 0 || H % Hkv) return 0;
  int G = H / Hkv;
  return (G == 1 || G == 2 || G == 4 || G == 8) ? 1 : 0;
}

extern "C" int ifkv_recompute_attn_tc(const void* q, const void* k_layer, const void* v_layer, const int64_t* horizon,
                                      int S, int H, int Hkv, int Dh, int n_rows, float scale, void* out,
                                      void* stream) {
  IFKV_CHECK_ARG(ifkv_recompute_attn_tc_supported(IFKV_BF16, H, Hkv, Dh), "recompute_attn_tc: unsupported shape");
  if (S <= 0) return IFKV_OK;
  const int G = H / Hkv;
  CUtensorMap tq, tk, tv;
  {
    uint64_t dims[3] = {(uint64_t)Dh, (uint64_t)H, (uint64_t)S};
    uint64_t strides[2] = {(uint64_t)Dh * 2, (uint64_t)H * Dh * 2};
    uint32_t box[3] = {64, (uint32_t)G, (uint32_t)(kRows / G)};
    int rc = make_tmap_bf16(&tq, q, 3, dims, strides, box);
    if (rc) return rc;
  }
  {
    uint64_t dims[2] = {(uint64_t)Hkv * Dh, (uint64_t)n_rows};
    uint64_t strides[1] = {(uint64_t)Hkv * Dh * 2};
    uint32_t box[2] = {64, (uint32_t)kKeys};
    int rc = make_tmap_bf16(&tk, k_layer, 2, dims, strides, box);
    if (rc) return rc;
    rc = make_tmap_bf16(&tv, v_layer, 2, dims, strides, box);
    if (rc) return rc;
  }
  const size_t smem = sizeof(Smem) + 1024;
  IFKV_CUDA_CALL(cudaFuncSetAttribute(recompute_attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem),
                 "recompute_attn_tc: smem attribute");
  const int tok_per_tile = kRows / G;
  dim3 grid(Hkv, (S + tok_per_tile - 1) / tok_per_tile);
  const float scale_log2 = scale * 1.4426950408889634f;
  recompute_attn_tc_kernel<<<grid, 256, smem, as_stream(stream)>>>(tq, tk, tv, horizon, S, H, Hkv, scale_log2,
                                                                    (__nv_bfloat16*)out);
  IFKV_LAUNCH_CHECK("recompute_attn_tc");
  return IFKV_OK;
}
