// Selective-recompute attention on the 5th-gen tensor cores (tcgen05 + TMEM
// + TMA): bf16 Q/K/V, fp32 softmax, bf16 out, Dh = 128, GQA groups of
// G = H/Hkv <= 16 query heads per kv head (floor(128/G) tokens per tile).
//
// Reference: recompute.py:92-114 -- selected queries attend every context
// key up to their own global index (masked_attention model.py:297-315).
//
// Work decomposition.  A tile is 128 query rows = (128/G) selected tokens x
// the G query heads of one kv head (GQA packing: one K/V block feeds all G
// heads).  Selected tokens are ascending, so a tile's key span ends at its
// last token's horizon.  A CTA owns TWO consecutive tiles (A, B) of the same
// kv head and streams the K/V blocks once for both; the tensor core
// ping-pongs between them so one tile's softmax overlaps the other's MMAs
// (the FlashAttention-4 schedule):
//     S_A(0) S_B(0) | PV_A(j) S_A(j+1) PV_B(j) S_B(j+1) | ...
// Warp roles (384 threads):
//   warp 0        TMA producer: Q_A, Q_B once; K / V blocks, 2-stage rings
//   warp 1        MMA issuer (one thread)
//   warp 2        TMEM allocator
//   warps 4-7     softmax of tile A, warps 8-11 softmax of tile B: thread =
//                 one query row; S row via tcgen05.ld, causal mask only on
//                 blocks crossing the warp's horizons, online softmax with
//                 lazy rescale (O rescaled only when the running max grows by
//                 more than 2^8), P -> bf16 written back into TMEM over the
//                 consumed S columns (A operand of the PV MMA, TS form);
//                 epilogue O / l -> bf16 -> global.
// smem: Q 2 x 32 KB + K 2 x 32 KB + V 2 x 32 KB = 192 KB.
// TMEM: tile X in {A, B}: S/P at cols [256X, 256X+128), O at [256X+128, 256X+256).
#include "tc_common.cuh"

namespace ifkv {
namespace {

constexpr int kRows = 128;
constexpr int kKeys = 128;
constexpr int kDh = 128;
constexpr int kPanel = 128 * 128;
constexpr int kTile = 2 * kPanel;
constexpr uint32_t kTmemCols = 512;
constexpr float kRescaleLog2 = 8.0f;
// A/B switches (tools/attn_bench.py): register split between the producer /
// MMA warpgroup and the softmax warpgroups; which exp2 pairs go to the
// FMA-pipe polynomial instead of the MUFU: bit (pair index & 7) of the mask.
#ifndef IFKV_ATTN_SETMAXNREG
#define IFKV_ATTN_SETMAXNREG 0
#endif
// IFKV_ATTN_TRACE=1: CTA (0, 0) records globaltimer-free clock64 stamps of
// every phase into a device buffer (tools/attn_trace.py reads it).
#ifndef IFKV_ATTN_TRACE
#define IFKV_ATTN_TRACE 0
#endif
#if IFKV_ATTN_TRACE
__device__ long long g_attn_trace[12][4096];
__device__ int g_attn_trace_n[12];
#define TRACE(stream, val)                                                                          \
  do {                                                                                              \
    if (blockIdx.x == 0 && blockIdx.y == 0) {                                                       \
      int i_ = g_attn_trace_n[stream]++;                                                            \
      if (i_ < 4096) g_attn_trace[stream][i_] = (val);                                              \
    }                                                                                               \
  } while (0)
#else
#define TRACE(stream, val) \
  do {                     \
  } while (0)
#endif
#ifndef IFKV_ATTN_POLY_MASK
#define IFKV_ATTN_POLY_MASK 0x00
#endif

// P published in kPParts key parts per block (2: halves; 4: quarters, A/B):
// the PV MMA of a part starts while the next part is exponentiated.
#ifndef IFKV_ATTN_PPARTS
#define IFKV_ATTN_PPARTS 2
#endif
constexpr int kPParts = IFKV_ATTN_PPARTS;

struct Smem {
  uint8_t q[2][kTile];
  uint8_t k[2][kTile];
  uint8_t v[2][kTile];
  uint64_t q_full;
  uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2];
  uint64_t s_full[2], p_full[2][kPParts], o_final[2];  // p_full[tile][key part]
  uint32_t tmem_base;
  int n_blocks[2];
};

// Key blocks a tile needs: its largest horizon decides (horizons are
// ascending on the single-GPU path, but not across the rank-ordered query
// lists of the chunk-sharded path).  Computed by one warp, lane-strided.
__device__ __forceinline__ int tile_blocks_warp(const int64_t* horizon, int t0, int tok, int S) {
  int64_t mx = -1;
  for (int t = t0 + (threadIdx.x & 31); t < min(t0 + tok, S); t += 32) mx = max(mx, horizon[t]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mx, o));
  return mx < 0 ? 0 : (int)((mx + kKeys) / kKeys);
}

// Softmax + epilogue of one tile; `x` = 0 (A) or 1 (B).
__device__ __forceinline__ void softmax_tile(Smem& sm, uint32_t tmem, int x, int nblk, int b0, int t0, int S, int H,
                                             int G,
                                             int g, const int64_t* __restrict__ horizon, float scale_log2,
                                             __nv_bfloat16* __restrict__ out, float* __restrict__ ml_out) {
  const int w = (threadIdx.x >> 5) & 3;  // lane quarter of TMEM this warp may access
  const int lane = threadIdx.x & 31;
  const int row = w * 32 + lane;
  const int tok = t0 + row / G;
  const bool valid = row < (kRows / G) * G && tok < S;  // G not dividing 128 leaves pad rows
  const int hz = valid ? (int)horizon[tok] : INT_MAX;  // pad rows: never force the masked path
  const uint32_t lane_off = (uint32_t)(w * 32) << 16;
  const uint32_t t_s = tmem + 256 * x + lane_off;
  const uint32_t t_o = t_s + 128;
  float m_used = -INFINITY, l = 0.f;
#ifdef IFKV_ATTN_RAWMMA
  if (false)
#endif
  for (int j = 0; j < nblk; ++j) {
    if (lane == 0 && w == 0) TRACE(x * 3 + 0, clock64());  // softmax: start waiting S
    tc::mbar_wait(&sm.s_full[x], j & 1);
    tc::tc_fence_after();
    if (lane == 0 && w == 0) TRACE(x * 3 + 1, clock64());  // softmax: S ready
#ifdef IFKV_ATTN_NOSOFTMAX  // experiment: pure MMA / TMA pipeline throughput
    tc::tc_fence_before();
    for (int q = 0; q < kPParts; ++q) tc::mbar_arrive(&sm.p_full[x][q]);
    if (lane == 0 && w == 0) TRACE(x * 3 + 2, clock64());
    continue;
#endif
    const int j0 = (b0 + j) * kKeys;  // absolute first key of the block
    const bool masked = __any_sync(0xffffffffu, j0 + kKeys - 1 > hz);
    float v[64];
    // pass 1: row max over the block (two 64-column halves)
    float mx = -INFINITY;
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      tc::tmem_ld32(t_s + hf * 64, v);
      tc::tmem_ld32(t_s + hf * 64 + 32, v + 32);
      tc::tmem_ld_wait();
      if (masked) {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (j0 + hf * 64 + c > hz) v[c] = -INFINITY;
      }
#pragma unroll
      for (int c = 0; c < 64; c += 2) mx = tc::max3(mx, v[c], v[c + 1]);
    }
    float alpha = 1.f;
    bool need = false;
    if (mx > -INFINITY && (m_used == -INFINITY || (mx - m_used) * scale_log2 > kRescaleLog2)) {
      need = true;
      alpha = m_used == -INFINITY ? 0.f : tc::ex2((m_used - mx) * scale_log2);
      m_used = mx;
    }
    const float mb = m_used == -INFINITY ? 0.f : m_used * scale_log2;
    // O holds PV(0..j-1) and is idle: S(j) completing implies PV(j-1) did.
    if (j > 0 && __any_sync(0xffffffffu, need)) {
      const float a = need ? alpha : 1.f;
#pragma unroll
      for (int c = 0; c < kDh / 32; ++c) {
        tc::tmem_ld32(t_o + c * 32, v);
        tc::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 32; ++u) v[u] *= a;
        tc::tmem_st32(t_o + c * 32, v);
      }
    }
    // pass 2: p = exp2(s * log2e / sqrt(d) - m) -> bf16 pairs written over
    // the consumed S columns (P cols [32 hf, 32 hf + 32) <- S cols [64 hf, 64 hf + 64))
    float sum = 0.f;
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      tc::tmem_ld32(t_s + hf * 64, v);
      tc::tmem_ld32(t_s + hf * 64 + 32, v + 32);
      tc::tmem_ld_wait();
      if (masked) {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (j0 + hf * 64 + c > hz) v[c] = -INFINITY;
      }
      uint32_t pk[32];
      const float2 sc2 = make_float2(scale_log2, scale_log2), mb2 = make_float2(-mb, -mb);
      float2 sum2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < 64; c += 2) {
        if (kPParts == 4 && c == 32) {  // publish the first quarter of this half
          tc::tmem_st16(t_s + hf * 32, pk);
          tc::tmem_st_wait();
          tc::tc_fence_before();
          tc::mbar_arrive(&sm.p_full[x][2 * hf]);
        }
        // packed x = s * scale - m; exp2 on the MUFU, or on the FMA pipe for
        // the pairs selected by IFKV_ATTN_POLY_MASK in unmasked blocks
        // (ex2.approx.ftz(-inf) = +0 on the masked ones)
        const float2 xx = tc::ffma2(make_float2(v[c], v[c + 1]), sc2, mb2);
        float2 e;
        if (!masked && ((IFKV_ATTN_POLY_MASK >> ((c >> 1) & 7)) & 1)) {  // masked blocks keep exact zeros
          e = tc::ex2_poly2(xx);
        } else {
          e = make_float2(tc::ex2(xx.x), tc::ex2(xx.y));
        }
        sum2 = tc::fadd2(sum2, e);
        pk[c / 2] = tc::pack_bf16(e.x, e.y);
      }
      sum += sum2.x + sum2.y;
      if (kPParts == 2) tc::tmem_st16(t_s + hf * 32, pk);
      tc::tmem_st16(t_s + hf * 32 + 16, pk + 16);
      // publish this half of P: the PV MMA over keys [64 hf, 64 hf + 64)
      // starts while the next half is still being exponentiated
      tc::tmem_st_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&sm.p_full[x][kPParts == 4 ? 2 * hf + 1 : hf]);
    }
    l = l * alpha + sum;
    if (lane == 0 && w == 0) TRACE(x * 3 + 2, clock64());  // softmax: P published
  }
  // epilogue (a row that saw no key -- horizon -1 in partial mode -- writes 0)
  if (nblk > 0) {
    tc::mbar_wait(&sm.o_final[x], 0);
    tc::tc_fence_after();
  }
  const float inv = l > 0.f ? 1.f / l : 0.f;
  const int64_t orow = (int64_t)tok * H + g * G + row % G;
  __nv_bfloat16* dst = out + orow * kDh;
  if (ml_out && valid) {  // (max, sum) in natural units of the scaled logits, like the SIMT kernel
    ml_out[2 * orow] = m_used == -INFINITY ? -INFINITY : m_used * scale_log2 * 0.6931471805599453f;
    ml_out[2 * orow + 1] = l;
  }
#pragma unroll
  for (int c = 0; c < kDh / 32; ++c) {
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
    recompute_attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                             const __grid_constant__ CUtensorMap tm_v, const int64_t* __restrict__ horizon, int S,
                             int H, int Hkv, float scale_log2, __nv_bfloat16* __restrict__ out,
                             float* __restrict__ ml_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = H / Hkv;
  const int tok = kRows / G;  // tokens per tile
  const int g = blockIdx.x;
  const int pair = gridDim.y - 1 - blockIdx.y;  // heaviest (latest) tile pairs first
  const int tA = pair * 2 * tok, tB = tA + tok;
  if (warp == 3) {
    const int a = tA < S ? tile_blocks_warp(horizon, tA, tok, S) : 0;
    const int b = tB < S ? tile_blocks_warp(horizon, tB, tok, S) : 0;
    if (lane == 0) {
      sm.n_blocks[0] = a;
      sm.n_blocks[1] = b;
    }
  }

  if (threadIdx.x == 0) {
    tc::mbar_init(&sm.q_full, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&sm.k_full[i], 1);
      tc::mbar_init(&sm.k_empty[i], 1);
      tc::mbar_init(&sm.v_full[i], 1);
      tc::mbar_init(&sm.v_empty[i], 1);
      tc::mbar_init(&sm.s_full[i], 1);
      for (int q = 0; q < kPParts; ++q) tc::mbar_init(&sm.p_full[i][q], 128);
      tc::mbar_init(&sm.o_final[i], 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc<kTmemCols>(&sm.tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  // key split (gridDim.z > 1 when the grid alone would not fill the GPU):
  // split s takes blocks [b0, b1) of the pair's span; partial outputs
  const int n_full = max(sm.n_blocks[0], sm.n_blocks[1]);
  const int b0 = (int)((int64_t)blockIdx.z * n_full / gridDim.z);
  const int b1 = (int)((int64_t)(blockIdx.z + 1) * n_full / gridDim.z);
  const int nA = max(0, min(sm.n_blocks[0], b1) - b0), nB = max(0, min(sm.n_blocks[1], b1) - b0);
  const int nblk = max(nA, nB);
  out += (int64_t)blockIdx.z * S * H * kDh;
  if (ml_out) ml_out += (int64_t)blockIdx.z * S * H * 2;

  if (warp < 4) {
#if IFKV_ATTN_SETMAXNREG
    tc::reg_dealloc<96>();
#endif
    if (warp == 0 && lane == 0) {
      tc::tma_prefetch(&tm_q);
      tc::tma_prefetch(&tm_k);
      tc::tma_prefetch(&tm_v);
      tc::mbar_arrive_expect_tx(&sm.q_full, (nB > 0 ? 2 : 1) * 2 * 128 * (tok * G));  // box = tok x G rows
      tc::tma_load_3d(sm.q[0], &tm_q, &sm.q_full, 0, g * G, tA);
      tc::tma_load_3d(sm.q[0] + kPanel, &tm_q, &sm.q_full, 64, g * G, tA);
      if (nB > 0) {
        tc::tma_load_3d(sm.q[1], &tm_q, &sm.q_full, 0, g * G, tB);
        tc::tma_load_3d(sm.q[1] + kPanel, &tm_q, &sm.q_full, 64, g * G, tB);
      }
#ifdef IFKV_ATTN_RAWMMA
      if (false)
#endif
      for (int j = 0; j < nblk; ++j) {
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        tc::mbar_wait(&sm.k_empty[s], ph ^ 1);
#ifdef IFKV_ATTN_NOTMA_STEADY  // experiment: only the first two K/V blocks are loaded (stale data after)
        if (j >= 2) {
          tc::mbar_arrive(&sm.k_full[s]);
          tc::mbar_wait(&sm.v_empty[s], ph ^ 1);
          tc::mbar_arrive(&sm.v_full[s]);
          continue;
        }
#endif
        tc::mbar_arrive_expect_tx(&sm.k_full[s], kTile);
        tc::tma_load_2d(sm.k[s], &tm_k, &sm.k_full[s], g * kDh, (b0 + j) * kKeys);
        tc::tma_load_2d(sm.k[s] + kPanel, &tm_k, &sm.k_full[s], g * kDh + 64, (b0 + j) * kKeys);
        tc::mbar_wait(&sm.v_empty[s], ph ^ 1);
        tc::mbar_arrive_expect_tx(&sm.v_full[s], kTile);
        tc::tma_load_2d(sm.v[s], &tm_v, &sm.v_full[s], g * kDh, (b0 + j) * kKeys);
        tc::tma_load_2d(sm.v[s] + kPanel, &tm_v, &sm.v_full[s], g * kDh + 64, (b0 + j) * kKeys);
      }
    } else if (warp == 1) {  // MMA issuer: the whole warp runs this, one elected lane issues (tc::*_ws)
      constexpr uint32_t idesc_qk = tc::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idesc_pv = tc::idesc_bf16(128, 128, 0, 1);
      tc::mbar_wait(&sm.q_full, 0);
      // Descriptors: one base per operand buffer, built once; a K-step adds a
      // compile-time offset to the 14-bit address field (smem < 256 KB, no carry),
      // keeping the single-thread issue path short (it sits on the P -> PV chain).
      const uint64_t dq0 = tc::smem_desc_sw128(tc::smem_u32(sm.q[0]), 16, 1024);
      const uint64_t dq1 = tc::smem_desc_sw128(tc::smem_u32(sm.q[1]), 16, 1024);
      const uint64_t dk0 = tc::smem_desc_sw128(tc::smem_u32(sm.k[0]), 16, 1024);
      const uint64_t dk1 = tc::smem_desc_sw128(tc::smem_u32(sm.k[1]), 16, 1024);
      const uint64_t dv0 = tc::smem_desc_sw128(tc::smem_u32(sm.v[0]), kPanel, 1024);
      const uint64_t dv1 = tc::smem_desc_sw128(tc::smem_u32(sm.v[1]), kPanel, 1024);
      auto issue_s = [&](int x, int j) {  // S_x(j) = Q_x K_j^T
        const uint64_t qa = x == 0 ? dq0 : dq1, kb = (j & 1) ? dk1 : dk0;
#pragma unroll
        for (int t = 0; t < kDh / 16; ++t) {
          const uint64_t step = (uint64_t)((t >> 2) * (kPanel >> 4) + (t & 3) * 2);  // (bytes >> 4)
          tc::mma_bf16_ss_ws(tmem + 256 * x, qa + step, kb + step, idesc_qk, t > 0 ? 1u : 0u);
        }
        tc::mma_commit_ws(&sm.s_full[x]);
      };
      auto issue_pv = [&](int x, int j) {  // O_x += P_x(j) V_j, P from TMEM, one key half at a time
        const uint64_t vb = (j & 1) ? dv1 : dv0;
#pragma unroll
        for (int hf = 0; hf < kPParts; ++hf) {
#ifndef IFKV_ATTN_ONEPWAIT
          if (hf > 0) {
            tc::mbar_wait(&sm.p_full[x][hf], j & 1);
            tc::tc_fence_after();
          }
#endif
          constexpr int kT = 8 / kPParts;  // K-steps (16 keys) per part
#pragma unroll
          for (int t = kT * hf; t < kT * hf + kT; ++t)
            tc::mma_bf16_ts_ws(tmem + 256 * x + 128, tmem + 256 * x + 8 * t, vb + (uint64_t)(t * (2048 >> 4)), idesc_pv,
                            (j > 0 || t > 0) ? 1u : 0u);
        }
        if (j == (x == 0 ? nA : nB) - 1) tc::mma_commit_ws(&sm.o_final[x]);
      };
#ifdef IFKV_ATTN_RAWMMA  // experiment: the MMA stream alone, no waits (garbage operands)
      for (int j = 0; j < nblk; ++j) {
        for (int x = 0; x < 2; ++x) {
          const uint32_t q_addr = tc::smem_u32(sm.q[x]);
          const uint32_t k_addr = tc::smem_u32(sm.k[j & 1]);
#pragma unroll
          for (int t = 0; t < kDh / 16; ++t) {
            uint64_t a = tc::smem_desc_sw128(q_addr + (t >> 2) * kPanel + (t & 3) * 32, 16, 1024);
            uint64_t b = tc::smem_desc_sw128(k_addr + (t >> 2) * kPanel + (t & 3) * 32, 16, 1024);
            tc::mma_bf16_ss_ws(tmem + 256 * x, a, b, idesc_qk, t > 0 ? 1u : 0u);
          }
#ifdef IFKV_ATTN_RAWCOMMIT  // ... with the real kernel's commit cadence
          tc::mma_commit_ws(&sm.s_full[x]);
#endif
        }
        for (int x = 0; x < 2; ++x) {
          const uint32_t v_addr = tc::smem_u32(sm.v[j & 1]);
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            uint64_t b = tc::smem_desc_sw128(v_addr + t * 2048, kPanel, 1024);
            tc::mma_bf16_ts_ws(tmem + 256 * x + 128, tmem + 256 * x + 8 * t, b, idesc_pv, (j > 0 || t > 0) ? 1u : 0u);
          }
        }
#ifdef IFKV_ATTN_RAWCOMMIT
        tc::mma_commit_ws(&sm.v_empty[j & 1]);
        tc::mma_commit_ws(&sm.k_empty[j & 1]);
#endif
      }
      tc::mma_commit_ws(&sm.o_final[0]);
      tc::mma_commit_ws(&sm.o_final[1]);
      if (false) {
#else
      {
#endif
      // prologue: S_A(0), S_B(0).  A pair with no visible key at all (every
      // horizon -1: queries of other ranks' chunks in the sharded partial
      // mode) has nblk = 0 and no K block is ever loaded.
      if (nblk > 0) {
        tc::mbar_wait(&sm.k_full[0], 0);
        tc::tc_fence_after();
        for (int x = 0; x < 2; ++x)
          if ((x == 0 ? nA : nB) > 0) issue_s(x, 0);
        tc::mma_commit_ws(&sm.k_empty[0]);  // K_0 is only read by the prologue
      }
      for (int j = 0; j < nblk; ++j) {
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        bool v_ready = false;
        bool next_k = false;
        for (int x = 0; x < 2; ++x) {
          const int nx = x == 0 ? nA : nB;
          if (j >= nx) continue;
          if (lane == 0) TRACE(6, clock64());  // MMA: start waiting P_x
#ifdef IFKV_ATTN_ONEPWAIT  // experiment: one P wait per tile-block (the last part's)
          tc::mbar_wait(&sm.p_full[x][kPParts - 1], j & 1);
#else
          tc::mbar_wait(&sm.p_full[x][0], j & 1);
#endif
          if (lane == 0) TRACE(7, clock64());  // MMA: P_x ready
          if (!v_ready) {
            if (lane == 0) TRACE(8, clock64());  // MMA: start waiting V
            tc::mbar_wait(&sm.v_full[s], ph);
            if (lane == 0) TRACE(9, clock64());
            v_ready = true;
          }
          tc::tc_fence_after();
          issue_pv(x, j);
          if (j + 1 < nx) {
            if (!next_k) {
              if (lane == 0) TRACE(10, clock64());  // MMA: start waiting K
              tc::mbar_wait(&sm.k_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
              if (lane == 0) TRACE(11, clock64());
              tc::tc_fence_after();
              next_k = true;
            }
            issue_s(x, j + 1);
          }
        }
        tc::mma_commit_ws(&sm.v_empty[s]);
        if (next_k) tc::mma_commit_ws(&sm.k_empty[(j + 1) & 1]);
      }
      }
    }
  } else {
#if IFKV_ATTN_SETMAXNREG
    tc::reg_alloc<200>();
#endif
    const int x = (warp - 4) >> 2;  // 0: tile A (warps 4-7), 1: tile B (warps 8-11)
    const int nx = x == 0 ? nA : nB;
    const int tx = x == 0 ? tA : tB;
    if (tx < S) softmax_tile(sm, tmem, x, nx, b0, tx, S, H, G, g, horizon, scale_log2, out, ml_out);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) tc::tmem_dealloc<kTmemCols>(tmem);
}

// Combine P key-split partials (bf16 O/l normalised per split, (m, l) in
// natural units): one warp per (token, head) row, 4 dims per lane.
__global__ void attn_split_merge_kernel(const __nv_bfloat16* __restrict__ part_o, const float* __restrict__ part_ml,
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
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    acc[0] += w * a.x;
    acc[1] += w * a.y;
    acc[2] += w * b.x;
    acc[3] += w * b.y;
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

extern "C" int ifkv_recompute_attn_tc_supported(int dtype, int H, int Hkv, int Dh) {
  if (dtype != IFKV_BF16 || Dh != kDh || Hkv <= 0 || H % Hkv) return 0;
  return H / Hkv <= 16 ? 1 : 0;  // a tile holds floor(128 / G) tokens x G heads
}

// Key splits for a grid of `ctas` CTAs on `sms` SMs: none while the grid
// fills two waves, else enough (<= 4) to reach two waves.
static int attn_key_splits(int ctas, int sms) {
#ifdef IFKV_ATTN_SPLITS
  return IFKV_ATTN_SPLITS;
#else
  if (ctas >= 2 * sms) return 1;
  const int p = (2 * sms + ctas - 1) / ctas;
  return p < 4 ? p : 4;
#endif
}

extern "C" int ifkv_recompute_attn_tc(const void* q, const void* k_layer, const void* v_layer, const int64_t* horizon,
                                      int S, int H, int Hkv, int Dh, int n_rows, float scale, void* out, float* ml_out,
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
  const int tok_per_pair = 2 * (kRows / G);
  const int pairs = (S + tok_per_pair - 1) / tok_per_pair;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int P = attn_key_splits(Hkv * pairs, sms);
  const float scale_log2 = scale * 1.4426950408889634f;
  cudaStream_t st = as_stream(stream);
  if (P == 1) {
    recompute_attn_tc_kernel<<<dim3(Hkv, pairs, 1), 384, smem, st>>>(tq, tk, tv, horizon, S, H, Hkv, scale_log2,
                                                                     (__nv_bfloat16*)out, ml_out);
    IFKV_LAUNCH_CHECK("recompute_attn_tc");
    return IFKV_OK;
  }
  // key-split partials in a stream-ordered scratch allocation, then one merge
  const int64_t rows = (int64_t)S * H;
  void* ws = nullptr;
  const size_t o_bytes = (size_t)P * rows * kDh * 2, ml_bytes = (size_t)P * rows * 2 * 4;
  ws = workspace_alloc(o_bytes + ml_bytes, st);
  if (!ws) {
    set_error("recompute_attn_tc: split workspace (%zu bytes)", o_bytes + ml_bytes);
    return IFKV_ERR_CUDA;
  }
  auto* part_o = reinterpret_cast<__nv_bfloat16*>(ws);
  auto* part_ml = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + o_bytes);
  recompute_attn_tc_kernel<<<dim3(Hkv, pairs, P), 384, smem, st>>>(tq, tk, tv, horizon, S, H, Hkv, scale_log2,
                                                                   part_o, part_ml);
  IFKV_LAUNCH_CHECK("recompute_attn_tc (split)");
  attn_split_merge_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(part_o, part_ml, P, rows,
                                                                        (__nv_bfloat16*)out, ml_out);
  IFKV_LAUNCH_CHECK("recompute_attn_tc (merge)");
  IFKV_CUDA_CALL(cudaFreeAsync(ws, st), "recompute_attn_tc: free split workspace");
  return IFKV_OK;
}

// Debug: copy the phase trace of CTA (0, 0) out (IFKV_ATTN_TRACE builds only).
extern "C" int ifkv_attn_trace_read(long long* out, int* counts, int reset) {
#if IFKV_ATTN_TRACE
  IFKV_CUDA_CALL(cudaDeviceSynchronize(), "trace");
  IFKV_CUDA_CALL(cudaMemcpyFromSymbol(out, g_attn_trace, sizeof(g_attn_trace)), "trace");
  IFKV_CUDA_CALL(cudaMemcpyFromSymbol(counts, g_attn_trace_n, sizeof(g_attn_trace_n)), "trace");
  if (reset) {
    int zero[12] = {0};
    IFKV_CUDA_CALL(cudaMemcpyToSymbol(g_attn_trace_n, zero, sizeof(zero)), "trace");
  }
  return IFKV_OK;
#else
  (void)out;
  (void)counts;
  (void)reset;
  ifkv::set_error("library built without IFKV_ATTN_TRACE");
  return IFKV_ERR_ARG;
#endif
}
