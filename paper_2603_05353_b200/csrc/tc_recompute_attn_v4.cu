// Selective-recompute attention, v4: one 128-row tile per CTA, S
// double-buffered in TMEM, column-split softmax (8 warps).
//
// Reference: recompute.py:92-114 -- selected queries attend every context
// key up to their own global index (masked_attention model.py:297-315).
//
// v2 (tc_recompute_attn.cu) ping-pongs two tiles with one S buffer each, so a
// tile's S(j+1) waits for its own P(j): the MMA -> softmax -> MMA handshake
// sits on the critical path (profiles/r1_attn_ab.md).  Here a CTA owns one
// tile and two S buffers (TMEM: S0 [0,128), S1 [128,256), O [256,384)), so
//     S(0) S(1) | PV(j) S(j+2) ...
// keeps the next QK^T queued while the softmax of block j runs; the softmax
// warps run block after block without waiting for the MMA side.  Eight
// softmax warps, two per TMEM lane quarter: warp 4+q handles key columns
// [0,64) of rows 32q..32q+31, warp 8+q columns [64,128); the row max is
// exchanged through shared memory (named barrier of the warp pair, double-
// buffered by block parity), the row sums are combined in the epilogue.  P
// (bf16) of the left half goes to S columns [0,32) and of the right half to
// [64,96) -- each half overwrites only columns it has already read -- and the
// PV MMA takes its K-steps from those two column ranges.
// Warps: 0 Q + K-ring producer, 1 MMA issuer, 2 TMEM allocator, 3 n_blocks +
// V-ring producer, 4-11 softmax.  Key splits (gridDim.z) as in v2.
#include "tc_common.cuh"

namespace ifkv {
namespace {

constexpr int kRows = 128;
constexpr int kKeys = 128;
constexpr int kDh = 128;
constexpr int kPanel = 128 * 128;
constexpr int kTile = 2 * kPanel;  // 32 KB: 128 rows x 128 bf16
constexpr uint32_t kTmemCols = 512;
constexpr float kRescaleLog2 = 8.0f;
#ifndef IFKV_ATTN4_STAGES
#define IFKV_ATTN4_STAGES 2
#endif
constexpr int kStages = IFKV_ATTN4_STAGES;
// S buffers in TMEM (128 columns each) + O (128 columns): 3 buffers let S(j+3)
// follow PV(j), so the softmax of block j+1 never waits on the PV(j) handshake.
#ifndef IFKV_ATTN4_SBUF
#define IFKV_ATTN4_SBUF 3
#endif
constexpr int kSBuf = IFKV_ATTN4_SBUF;
constexpr uint32_t kColO = 128 * kSBuf;

struct Smem {
  uint8_t q[kTile];
  uint8_t k[kStages][kTile];
  uint8_t v[kStages][kTile];
  uint64_t q_full;
  uint64_t k_full[kStages], k_empty[kStages], v_full[kStages], v_empty[kStages];
  // p_full[S buffer][column half]; pv_done[i & 1] completes once per PV(i) of that parity
  uint64_t s_full[kSBuf], p_full[kSBuf][2], pv_done[2], o_final;
  uint32_t tmem_base;
  int n_blocks;
  // row-max exchange [buffer][column half][row]; double-buffered by block
  // parity with 2 stages, single-buffered (one extra pair barrier per block)
  // with 3 stages to fit 227 KB; reused for the final row-sum exchange
  float xmax[kStages >= 3 ? 1 : 2][2][128];
};

__device__ __forceinline__ int tile_blocks_warp(const int64_t* horizon, int t0, int tok, int S) {
  int64_t mx = -1;
  for (int t = t0 + (threadIdx.x & 31); t < min(t0 + tok, S); t += 32) mx = max(mx, horizon[t]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mx, o));
  return mx < 0 ? 0 : (int)((mx + kKeys) / kKeys);
}

__device__ __forceinline__ void pair_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

// One softmax warp: rows 32q..32q+31 of the tile, key columns [64 hf, 64 hf + 64).
__device__ __forceinline__ void softmax_half(Smem& sm, uint32_t tmem, int hf, int nblk, int b0, int t0, int S, int H,
                                             int G, int g, const int64_t* __restrict__ horizon, float scale_log2,
                                             __nv_bfloat16* __restrict__ out, float* __restrict__ ml_out) {
  const int q = (threadIdx.x >> 5) & 3;
  const int lane = threadIdx.x & 31;
  const int row = q * 32 + lane;
  const int tok = t0 + row / G;
  const bool valid = row < (kRows / G) * G && tok < S;
  const int hz = valid ? (int)horizon[tok] : INT_MAX;  // pad rows: never force the masked path
  const uint32_t lane_off = (uint32_t)(q * 32) << 16;
  const uint32_t t_o = tmem + kColO + lane_off + 64 * hf;
  const int bar_id = 1 + q;
  float m_used = -INFINITY, l = 0.f;
  for (int j = 0; j < nblk; ++j) {
    const int b = j % kSBuf, xb = j & 1;  // S buffer, exchange parity
    const uint32_t t_s = tmem + 128 * b + lane_off + 64 * hf;
    tc::mbar_wait(&sm.s_full[b], (j / kSBuf) & 1);
    tc::tc_fence_after();
#ifdef IFKV_ATTN_NOSOFTMAX  // experiment: MMA / TMA pipeline alone
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&sm.p_full[b][hf]);
    continue;
#endif
    const int j0 = (b0 + j) * kKeys + 64 * hf;  // absolute first key of this half
    const bool masked = __any_sync(0xffffffffu, j0 + 63 > hz);
    float v[64];
    tc::tmem_ld32(t_s, v);
#ifdef IFKV_ATTN4_HALFLD  // experiment: half the TMEM reads (wrong results), same MUFU work
#pragma unroll
    for (int c = 0; c < 32; ++c) v[32 + c] = v[c];
#else
    tc::tmem_ld32(t_s + 32, v + 32);
#endif
    tc::tmem_ld_wait();
    if (masked) {
#pragma unroll
      for (int c = 0; c < 64; ++c)
        if (j0 + c > hz) v[c] = -INFINITY;
    }
    float m2[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int c = 0; c < 64; c += 4) {
      m2[0] = tc::max3(m2[0], v[c], v[c + 1]);
      m2[1] = tc::max3(m2[1], v[c + 2], v[c + 3]);
    }
    float mx = fmaxf(m2[0], m2[1]);
    constexpr int kXb = kStages >= 3 ? 1 : 2;
    sm.xmax[xb % kXb][hf][row] = mx;
    pair_sync(bar_id);
    mx = fmaxf(mx, sm.xmax[xb % kXb][hf ^ 1][row]);
    if (kXb == 1) pair_sync(bar_id);  // partner has read before the next block overwrites
    float alpha = 1.f;
    bool need = false;
    if (mx > -INFINITY && (m_used == -INFINITY || (mx - m_used) * scale_log2 > kRescaleLog2)) {
      need = true;
      alpha = m_used == -INFINITY ? 0.f : tc::ex2((m_used - mx) * scale_log2);
      m_used = mx;
    }
    const float mb = m_used == -INFINITY ? 0.f : m_used * scale_log2;
    if (j > 0 && __any_sync(0xffffffffu, need)) {
      // O = PV(0..j-1): wait for PV(j-1) on the barrier of its parity.  PV(j-3)
      // is complete (S(j) was issued after it) and PV(j+1) cannot be (it needs
      // P(j+1)), so that barrier is on phase (j-1)/2 or just past it.
      tc::mbar_wait(&sm.pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
      tc::tc_fence_after();
      const float a = need ? alpha : 1.f;
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        float o[32];
        tc::tmem_ld32(t_o + c * 32, o);
        tc::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 32; ++u) o[u] *= a;
        tc::tmem_st32(t_o + c * 32, o);
      }
    }
    uint32_t pk[32];
    const float2 sc2 = make_float2(scale_log2, scale_log2), mb2 = make_float2(-mb, -mb);
    float2 sum2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c < 64; c += 2) {
      const float2 xx = tc::ffma2(make_float2(v[c], v[c + 1]), sc2, mb2);
      const float2 e = make_float2(tc::ex2(xx.x), tc::ex2(xx.y));  // ex2.approx.ftz(-inf) = +0
      sum2 = tc::fadd2(sum2, e);
      pk[c / 2] = tc::pack_bf16(e.x, e.y);
    }
    tc::tmem_st16(t_s, pk);  // P cols [64 hf, 64 hf + 32) of the buffer: already read by this warp
    tc::tmem_st16(t_s + 16, pk + 16);
    tc::tmem_st_wait();
    tc::tc_fence_before();
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&sm.p_full[b][hf]);
    l = l * alpha + (sum2.x + sum2.y);
  }
  if (nblk > 0) {
    tc::mbar_wait(&sm.o_final, 0);
    tc::tc_fence_after();
  }
  pair_sync(bar_id);  // (2-buffer mode) partner done reading the last block's max
  sm.xmax[0][hf][row] = l;
  pair_sync(bar_id);
  const float lt = l + sm.xmax[0][hf ^ 1][row];
  const float inv = lt > 0.f ? 1.f / lt : 0.f;
  const int64_t orow = (int64_t)tok * H + g * G + row % G;
  __nv_bfloat16* dst = out + orow * kDh + 64 * hf;
  if (ml_out && valid && hf == 0) {  // (max, sum) in natural units of the scaled logits
    ml_out[2 * orow] = m_used == -INFINITY ? -INFINITY : m_used * scale_log2 * 0.6931471805599453f;
    ml_out[2 * orow + 1] = lt;
  }
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float o[32];
    if (nblk > 0) {
      tc::tmem_ld32(t_o + c * 32, o);
      tc::tmem_ld_wait();
    } else {
#pragma unroll
      for (int u = 0; u < 32; ++u) o[u] = 0.f;
    }
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

__global__ void __launch_bounds__(384, 1)
    recompute_attn_v4_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                             const __grid_constant__ CUtensorMap tm_v, const int64_t* __restrict__ horizon, int S,
                             int H, int Hkv, float scale_log2, __nv_bfloat16* __restrict__ out,
                             float* __restrict__ ml_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = H / Hkv;
  const int tok = kRows / G;
  const int g = blockIdx.x;
  const int tile = gridDim.y - 1 - blockIdx.y;  // heaviest (latest) tiles first
  const int t0 = tile * tok;
  if (warp == 3) {
    const int n = t0 < S ? tile_blocks_warp(horizon, t0, tok, S) : 0;
    if (lane == 0) sm.n_blocks = n;
  }
  if (threadIdx.x == 0) {
    tc::mbar_init(&sm.q_full, 1);
    for (int i = 0; i < kStages; ++i) {
      tc::mbar_init(&sm.k_full[i], 1);
      tc::mbar_init(&sm.k_empty[i], 1);
      tc::mbar_init(&sm.v_full[i], 1);
      tc::mbar_init(&sm.v_empty[i], 1);
    }
    for (int b = 0; b < kSBuf; ++b) {
      tc::mbar_init(&sm.s_full[b], 1);
      tc::mbar_init(&sm.p_full[b][0], 4);  // one elected arrival per softmax warp of the half
      tc::mbar_init(&sm.p_full[b][1], 4);
    }
    tc::mbar_init(&sm.pv_done[0], 1);
    tc::mbar_init(&sm.pv_done[1], 1);
    tc::mbar_init(&sm.o_final, 1);
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc<kTmemCols>(&sm.tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const int n_full = sm.n_blocks;
  const int b0 = (int)((int64_t)blockIdx.z * n_full / gridDim.z);
  const int nblk = (int)((int64_t)(blockIdx.z + 1) * n_full / gridDim.z) - b0;
  out += (int64_t)blockIdx.z * S * H * kDh;
  if (ml_out) ml_out += (int64_t)blockIdx.z * S * H * 2;

  if (warp < 4) {
    if (warp == 0 && lane == 0 && nblk > 0) {  // Q, then the K ring (no TMA in flight at exit if keyless)
      tc::tma_prefetch(&tm_q);
      tc::tma_prefetch(&tm_k);
      tc::mbar_arrive_expect_tx(&sm.q_full, 2 * 128 * (tok * G));  // box = tok x G rows
      tc::tma_load_3d(sm.q, &tm_q, &sm.q_full, 0, g * G, t0);
      tc::tma_load_3d(sm.q + kPanel, &tm_q, &sm.q_full, 64, g * G, t0);
      for (int j = 0; j < nblk; ++j) {
        const int s = j % kStages;
        tc::mbar_wait(&sm.k_empty[s], ((j / kStages) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&sm.k_full[s], kTile);
        tc::tma_load_2d(sm.k[s], &tm_k, &sm.k_full[s], g * kDh, (b0 + j) * kKeys);
        tc::tma_load_2d(sm.k[s] + kPanel, &tm_k, &sm.k_full[s], g * kDh + 64, (b0 + j) * kKeys);
      }
    } else if (warp == 3 && lane == 0) {  // the V ring
      tc::tma_prefetch(&tm_v);
      for (int j = 0; j < nblk; ++j) {
        const int s = j % kStages;
        tc::mbar_wait(&sm.v_empty[s], ((j / kStages) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&sm.v_full[s], kTile);
        tc::tma_load_2d(sm.v[s], &tm_v, &sm.v_full[s], g * kDh, (b0 + j) * kKeys);
        tc::tma_load_2d(sm.v[s] + kPanel, &tm_v, &sm.v_full[s], g * kDh + 64, (b0 + j) * kKeys);
      }
    } else if (warp == 1 && lane == 0 && nblk > 0) {
      constexpr uint32_t idesc_qk = tc::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idesc_pv = tc::idesc_bf16(128, 128, 0, 1);
      tc::mbar_wait(&sm.q_full, 0);
      const uint32_t q_addr = tc::smem_u32(sm.q);
      auto issue_s = [&](int j) {  // S(j) = Q K_j^T into buffer j % kSBuf
        const int s = j % kStages;
        tc::mbar_wait(&sm.k_full[s], (j / kStages) & 1);
        tc::tc_fence_after();
        const uint32_t k_addr = tc::smem_u32(sm.k[s]);
#pragma unroll
        for (int t = 0; t < kDh / 16; ++t) {
          uint64_t a = tc::smem_desc_sw128(q_addr + (t >> 2) * kPanel + (t & 3) * 32, 16, 1024);
          uint64_t b = tc::smem_desc_sw128(k_addr + (t >> 2) * kPanel + (t & 3) * 32, 16, 1024);
          tc::mma_bf16_ss(tmem + 128 * (j % kSBuf), a, b, idesc_qk, t > 0 ? 1u : 0u);
        }
        tc::mma_commit(&sm.s_full[j % kSBuf]);
        tc::mma_commit(&sm.k_empty[s]);
      };
      issue_s(0);
      for (int j = 1; j < kSBuf && j < nblk; ++j) issue_s(j);
      for (int j = 0; j < nblk; ++j) {
        const int b = j % kSBuf, s = j % kStages;
        const uint32_t v_addr = tc::smem_u32(sm.v[s]);
        tc::mbar_wait(&sm.v_full[s], (j / kStages) & 1);
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {  // keys [64 hf, 64 hf + 64): P at buffer cols [64 hf, 64 hf + 32)
          tc::mbar_wait(&sm.p_full[b][hf], (j / kSBuf) & 1);
          tc::tc_fence_after();
#pragma unroll
          for (int t = 4 * hf; t < 4 * hf + 4; ++t) {
            uint64_t bd = tc::smem_desc_sw128(v_addr + t * 2048, kPanel, 1024);
            tc::mma_bf16_ts(tmem + kColO, tmem + 128 * b + 64 * hf + 8 * (t - 4 * hf), bd, idesc_pv,
                            (j > 0 || t > 0) ? 1u : 0u);
          }
        }
        tc::mma_commit(&sm.pv_done[j & 1]);
        tc::mma_commit(&sm.v_empty[s]);
        if (j == nblk - 1) tc::mma_commit(&sm.o_final);
        if (j + kSBuf < nblk) issue_s(j + kSBuf);  // buffer b again: PV(j) has read P(j) (in-order pipe)
      }
    }
  } else if (t0 < S) {
    const int hf = (warp - 4) >> 2;
    softmax_half(sm, tmem, hf, nblk, b0, t0, S, H, G, g, horizon, scale_log2, out, ml_out);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) tc::tmem_dealloc<kTmemCols>(tmem);
}

__global__ void attn_v4_merge_kernel(const __nv_bfloat16* __restrict__ part_o, const float* __restrict__ part_ml,
                                     int P, int64_t rows, __nv_bfloat16* __restrict__ out,
                                     float* __restrict__ ml_out) {
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  float M = -INFINITY;
  for (int p = 0; p < P; ++p) M = fmaxf(M, part_ml[2 * (p * rows + r)]);
  float L = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int p = 0; p < P; ++p) {
    const float m = part_ml[2 * (p * rows + r)];
    const float w = m == -INFINITY ? 0.f : part_ml[2 * (p * rows + r) + 1] * __expf(m - M);
    L += w;
    const uint2 u = *reinterpret_cast<const uint2*>(part_o + (p * rows + r) * kDh + lane * 4);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 c = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    acc[0] += w * a.x;
    acc[1] += w * a.y;
    acc[2] += w * c.x;
    acc[3] += w * c.y;
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  uint2 o;
  o.x = tc::pack_bf16(acc[0] * inv, acc[1] * inv);
  o.y = tc::pack_bf16(acc[2] * inv, acc[3] * inv);
  *reinterpret_cast<uint2*>(out + r * kDh + lane * 4) = o;
  if (ml_out && lane == 0) {
    ml_out[2 * r] = M;
    ml_out[2 * r + 1] = L;
  }
}

}  // namespace
}  // namespace ifkv

using namespace ifkv;

extern "C" int ifkv_recompute_attn_tc_v4(const void* q, const void* k_layer, const void* v_layer,
                                         const int64_t* horizon, int S, int H, int Hkv, int Dh, int n_rows,
                                         float scale, void* out, float* ml_out, void* stream) {
  IFKV_CHECK_ARG(Dh == kDh && Hkv > 0 && H % Hkv == 0 && H / Hkv <= 16, "recompute_attn_v4: unsupported shape");
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
  IFKV_CUDA_CALL(cudaFuncSetAttribute(recompute_attn_v4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem),
                 "recompute_attn_v4: smem attribute");
  const int tok = kRows / G;
  const int tiles = (S + tok - 1) / tok;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int P = 1;
  if (Hkv * tiles < 2 * sms) P = min(4, (2 * sms + Hkv * tiles - 1) / (Hkv * tiles));
  const float scale_log2 = scale * 1.4426950408889634f;
  cudaStream_t st = as_stream(stream);
  if (P == 1) {
    recompute_attn_v4_kernel<<<dim3(Hkv, tiles, 1), 384, smem, st>>>(tq, tk, tv, horizon, S, H, Hkv, scale_log2,
                                                                     (__nv_bfloat16*)out, ml_out);
    IFKV_LAUNCH_CHECK("recompute_attn_v4");
    return IFKV_OK;
  }
  const int64_t rows = (int64_t)S * H;
  void* ws = nullptr;
  const size_t o_bytes = (size_t)P * rows * kDh * 2, ml_bytes = (size_t)P * rows * 2 * 4;
  ws = workspace_alloc(o_bytes + ml_bytes, st);
  if (!ws) {
    set_error("recompute_attn_v4: split workspace (%zu bytes)", o_bytes + ml_bytes);
    return IFKV_ERR_CUDA;
  }
  auto* part_o = reinterpret_cast<__nv_bfloat16*>(ws);
  auto* part_ml = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + o_bytes);
  recompute_attn_v4_kernel<<<dim3(Hkv, tiles, P), 384, smem, st>>>(tq, tk, tv, horizon, S, H, Hkv, scale_log2,
                                                                   part_o, part_ml);
  IFKV_LAUNCH_CHECK("recompute_attn_v4 (split)");
  attn_v4_merge_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(part_o, part_ml, P, rows, (__nv_bfloat16*)out,
                                                                     ml_out);
  IFKV_LAUNCH_CHECK("recompute_attn_v4 (merge)");
  IFKV_CUDA_CALL(cudaFreeAsync(ws, st), "recompute_attn_v4: free split workspace");
  return IFKV_OK;
}
