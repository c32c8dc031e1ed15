// Selective-recompute attention, v10: P stays in tensor memory.
//
// Reference: recompute.py:92-114 (masked_attention model.py:297-315).
//
// Why (profiles/r2_attn.md, tools/fa4_compare.py): v5 stages P in shared
// memory, so per 128-key block and tile the SM's shared memory serves the
// S MMA's two operands (Q, K), the PV MMA's two operands (P, V), the P stores
// and the K/V TMA writes -- about 1.5x what one SM's shared memory delivers
// while the tensor pipe is busy.  Here P is written by the softmax warps into
// the TMEM columns of its own S tile (bf16 pairs over the upper 64 columns)
// and the PV MMA reads its A operand from TMEM (TS form): per block and tile
// the shared-memory traffic drops to Q + K + V reads plus the TMA writes.
//
// Schedule (per CTA: two tiles A, B of 128 rows = floor(128/G) tokens x G
// heads, sharing every K/V block): the MMA warp issues, for each key block j,
//   PV_A(j-1), S_A(j), PV_B(j-1), S_B(j)
// back to back.  tcgen05 MMAs of one thread execute in issue order, so
// S_x(j) overwrites the S/P columns of tile x only after PV_x(j-1) consumed
// P_x(j-1), and the completion of S_x(j) (mbarrier s_full) implies O_x is
// idle: the softmax warps of tile x then rescale O_x themselves when the row
// maximum grew (rare: > 2^8), with no extra handshake.  While the softmax of
// one tile runs, the tensor pipe works on the other tile.
//
// smem (224 KB): Q 2 x 32 KB, a kStages-deep ring of 32 KB K / V blocks in
// consumption order K0 V0 K1 V1 ...  TMEM: S_A | S_B | O_A | O_B (128 columns
// each), P_x aliased on columns 64..127 of S_x.
// Softmax per block: one 128-column TMEM read of S, row max, an optional O
// rescale (O_x is idle), then each 32-key quarter's exponentials -- an eighth
// of them on the FMA pipe (degree-3 polynomial), the rest on MUFU -- are
// packed, stored over S and published, so PV_x(j) on the first keys overlaps
// the exponentials of the later ones (profiles/r2_attn10.md: 5-15 % over the
// variant that publishes P after all 128 exponentials).
// Warps: 0-3 softmax A, 4-7 softmax B (TMEM lane quarter = warp % 4),
// 8 TMA producer, 9 MMA issuer (warp-synchronous, elected lane), 10 TMEM
// allocator + block counts, 11 idle.  Softmax warpgroups raise their register
// budget with setmaxnreg (the whole 128-column S row is held in registers).
// The variants measured and not kept (alternating exponential phases, MMAs
// issued by the softmax warpgroups, spin polling, two warps per row, ...)
// are in profiles/attic/tc_recompute_attn_v10_variants.cu.txt with their
// numbers in profiles/r2_attn10.md.
#include "tc_common.cuh"

namespace ifkv {
namespace {

constexpr int kRows = 128;
constexpr int kKeys = 128;
constexpr int kDh = 128;
constexpr int kPanel = 128 * 128;  // 128 rows x 128 B (64 bf16)
constexpr int kTile = 2 * kPanel;  // 32 KB
constexpr int kStages = 5;         // K/V ring (Q 64 KB + 5 x 32 KB = 224 KB)
constexpr uint32_t kTmemCols = 512;
constexpr float kRescaleLog2 = 8.0f;
constexpr int kThreads = 384;
constexpr int kWarpTma = 8, kWarpMma = 9, kWarpAlloc = 10;
constexpr int kSoftmaxRegs = 200, kOtherRegs = 96;  // setmaxnreg moves registers within the CTA:
                                                     // 256 x (200 - 168) <= 128 x (168 - 96)
// P is published in kParts parts of 128 / kParts keys as their exponentials finish
#ifndef IFKV_ATTN10_PARTS
#define IFKV_ATTN10_PARTS 4
#endif
constexpr int kParts = IFKV_ATTN10_PARTS;
constexpr int kPairs = 64 / kParts;  // column pairs (= TMEM columns of P) per part
// FMA-pipe exponentials: in each 32-key fragment selected by FRAGS, the last
// EMU of every 8 column pairs use the polynomial instead of MUFU (12.5 %;
// 0 / 25 / 37.5 / 50 % measured slower, profiles/r2_attn10.md section 5)
#ifndef IFKV_ATTN10_EMU
#define IFKV_ATTN10_EMU 1
#endif
#ifndef IFKV_ATTN10_FRAGS
#define IFKV_ATTN10_FRAGS 0xF
#endif
#ifndef IFKV_ATTN10_SPLIT_WAVES
#define IFKV_ATTN10_SPLIT_WAVES 2
#endif
#ifndef IFKV_ATTN10_SPLIT_MAX
#define IFKV_ATTN10_SPLIT_MAX 4
#endif

#ifndef IFKV_ATTN10_TRACE
#define IFKV_ATTN10_TRACE 0
#endif
#if IFKV_ATTN10_TRACE
// clock64 event trace of ONE CTA (blockIdx 0, 0, 0) for tools/attn10_trace.py:
// [event][tile][block]; events 0 S observed, 1 row max done, 2 exponentials
// done, 3 P published (softmax warp 0 of the tile), 4 PV issue (after the last
// P wait), 5 S issue (MMA warp)
constexpr int kTraceBlocks = 512;
__device__ long long g_attn10_trace[6][2][kTraceBlocks];
#define TRACE10(ev, x, j)                                                                                    \
  do {                                                                                                      \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (threadIdx.x & 127) == 0 && (j) < kTraceBlocks) \
      g_attn10_trace[ev][x][j] = clock64();                                                                 \
  } while (0)
#define TRACE10M(ev, x, j)                                                                                   \
  do {                                                                                                      \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (threadIdx.x & 31) == 0 && (j) < kTraceBlocks) \
      g_attn10_trace[ev][x][j] = clock64();                                                                 \
  } while (0)
#else
#define TRACE10(ev, x, j)
#define TRACE10M(ev, x, j)
#endif

struct Smem10 {
  uint8_t q[2][kTile];
  uint8_t kv[kStages][kTile];
  uint64_t q_full, full[kStages], empty[kStages];
  uint64_t s_full[2], p_part[2][kParts], o_final[2];
  uint32_t tmem_base;
  int n_blocks[2];
  int first_block;
};

// Key blocks a tile of tok tokens needs (its largest horizon), and the first
// block any of its tokens can see (key ranges key_start..horizon; key_start ==
// nullptr: every range starts at key 0).
__device__ __forceinline__ int tile_blocks_warp10(const int64_t* horizon, int t0, int tok, int S) {
  int64_t mx = -1;
  for (int t = t0 + (threadIdx.x & 31); t < min(t0 + tok, S); t += 32) mx = max(mx, horizon[t]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mx, o));
  return mx < 0 ? 0 : (int)((mx + kKeys) / kKeys);
}
__device__ __forceinline__ int tile_first_block_warp10(const int64_t* key_start, int t0, int tok, int S) {
  if (key_start == nullptr) return 0;
  int64_t mn = INT64_MAX;
  for (int t = t0 + (threadIdx.x & 31); t < min(t0 + tok, S); t += 32) mn = min(mn, key_start[t]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = min(mn, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mn, o));
  return mn == INT64_MAX ? 0 : (int)(mn / kKeys);
}

__device__ __forceinline__ void softmax_tile10(Smem10& sm, uint32_t tmem, int x, int nblk, int b0, int t0, int S,
                                               int H, int G, int g, const int64_t* __restrict__ horizon,
                                               const int64_t* __restrict__ key_start, float scale_log2,
                                               __nv_bfloat16* __restrict__ out, float* __restrict__ ml_out) {
  const int w = (threadIdx.x >> 5) & 3;
  const int lane = threadIdx.x & 31;
  const int row = w * 32 + lane;
  const int tok = t0 + row / G;
  const bool valid = row < (kRows / G) * G && tok < S;
  const int hz = valid ? (int)horizon[tok] : INT_MAX;  // pad rows never force the masked path
  const int ks = valid && key_start ? (int)key_start[tok] : 0;
  const uint32_t lane_off = (uint32_t)(w * 32) << 16;
  const uint32_t t_s = tmem + 128 * x + lane_off;
  const uint32_t t_p = t_s + 64;
  const uint32_t t_o = tmem + 256 + 128 * x + lane_off;
  float m_used = -INFINITY, l = 0.f;
  for (int j = 0; j < nblk; ++j) {
    tc::mbar_wait(&sm.s_full[x], j & 1);
    tc::tc_fence_after();
    TRACE10(0, x, j);
    const int j0 = (b0 + j) * kKeys;
    const bool masked = __any_sync(0xffffffffu, j0 + kKeys - 1 > hz || j0 < ks);
    // the whole 128-key S row in registers (one TMEM read)
    float v[128];
#pragma unroll
    for (int q = 0; q < 4; ++q) tc::tmem_ld32(t_s + 32 * q, v + 32 * q);
    tc::tmem_ld_wait();
    if (masked) {
#pragma unroll
      for (int c = 0; c < 128; ++c)
        if (j0 + c > hz || j0 + c < ks) v[c] = -INFINITY;
    }
    float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int c = 0; c < 128; c += 8) {
      m4[0] = tc::max3(m4[0], v[c], v[c + 1]);
      m4[1] = tc::max3(m4[1], v[c + 2], v[c + 3]);
      m4[2] = tc::max3(m4[2], v[c + 4], v[c + 5]);
      m4[3] = tc::max3(m4[3], v[c + 6], v[c + 7]);
    }
    const float mx = tc::max3(m4[0], m4[1], fmaxf(m4[2], m4[3]));
    TRACE10(1, x, j);
    float alpha = 1.f;
    bool need = false;
    if (mx > -INFINITY && (m_used == -INFINITY || (mx - m_used) * scale_log2 > kRescaleLog2)) {
      need = true;
      alpha = m_used == -INFINITY ? 0.f : tc::ex2((m_used - mx) * scale_log2);
      m_used = mx;
    }
    const float mb = m_used == -INFINITY ? 0.f : m_used * scale_log2;
    const float2 sc2 = make_float2(scale_log2, scale_log2), mb2 = make_float2(-mb, -mb);
    // S_x(j) complete => PV_x(j-1) complete (in-order MMAs): O_x is idle and
    // is rescaled before any part of P(j) is published
    if (j > 0 && __any_sync(0xffffffffu, need)) {
      const float a = need ? alpha : 1.f;
#pragma unroll 1
      for (int c = 0; c < kDh / 32; ++c) {
        float o[32];
        tc::tmem_ld32(t_o + c * 32, o);
        tc::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 32; ++u) o[u] *= a;
        tc::tmem_st32(t_o + c * 32, o);
      }
    }
    // P over the upper half of S (bf16 pairs, keys 2c, 2c+1 in column c; the
    // whole row was read above), each part published as soon as it is stored
    float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
    for (int hf = 0; hf < kParts; ++hf) {
      uint32_t p[kPairs];
#pragma unroll
      for (int u = 0; u < kPairs; ++u) {
        const int pu = hf * kPairs + u;  // column pair pu = keys 2pu, 2pu+1
        const float2 xx = tc::ffma2(make_float2(v[2 * pu], v[2 * pu + 1]), sc2, mb2);
        float2 e;
        if (((IFKV_ATTN10_FRAGS >> (pu >> 4)) & 1) && (pu & 7) >= 8 - IFKV_ATTN10_EMU)
          e = tc::ex2_poly2(xx);  // FMA pipe (exactly 0 for masked keys)
        else
          e = make_float2(tc::ex2(xx.x), tc::ex2(xx.y));
        sum2[u & 1] = tc::fadd2(sum2[u & 1], e);
        p[u] = tc::pack_bf16(e.x, e.y);
      }
      if constexpr (kPairs == 32)
        tc::tmem_st32(t_p + kPairs * hf, reinterpret_cast<const float*>(p));
      else if constexpr (kPairs == 16)
        tc::tmem_st16(t_p + kPairs * hf, p);
      else
        tc::tmem_st8(t_p + kPairs * hf, p);
      tc::tmem_st_wait();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&sm.p_part[x][hf]);
    }
    TRACE10(2, x, j);
    TRACE10(3, x, j);
    l = l * alpha + ((sum2[0].x + sum2[1].x) + (sum2[0].y + sum2[1].y));
  }
  if (nblk > 0) {
    tc::mbar_wait(&sm.o_final[x], 0);
    tc::tc_fence_after();
  }
  const float inv = l > 0.f ? 1.f / l : 0.f;
  const int64_t orow = (int64_t)tok * H + g * G + row % G;
  __nv_bfloat16* dst = out + orow * kDh;
  if (ml_out && valid) {
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

__global__ void __launch_bounds__(kThreads, 1)
    recompute_attn_v10_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                              const __grid_constant__ CUtensorMap tm_v, const int64_t* __restrict__ horizon,
                              const int64_t* __restrict__ key_start, int S, int H, int Hkv, float scale_log2,
                              __nv_bfloat16* __restrict__ out, float* __restrict__ ml_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem10& sm = *reinterpret_cast<Smem10*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = H / Hkv;
  const int tok = kRows / G;
  const int g = blockIdx.x;
  const int pair = gridDim.y - 1 - blockIdx.y;  // heaviest (latest) pairs first
  const int tA = pair * 2 * tok, tB = tA + tok;
  if (warp == kWarpAlloc) {
    const int a = tA < S ? tile_blocks_warp10(horizon, tA, tok, S) : 0;
    const int b = tB < S ? tile_blocks_warp10(horizon, tB, tok, S) : 0;
    const int fa = tA < S ? tile_first_block_warp10(key_start, tA, tok, S) : INT_MAX;
    const int fb = tB < S ? tile_first_block_warp10(key_start, tB, tok, S) : INT_MAX;
    if (lane == 0) {
      sm.n_blocks[0] = a;
      sm.n_blocks[1] = b;
      sm.first_block = min(min(fa, fb), max(a, b));  // blocks before it are masked for every row
    }
  }
  if (threadIdx.x == 0) {
    tc::mbar_init(&sm.q_full, 1);
    for (int i = 0; i < kStages; ++i) {
      tc::mbar_init(&sm.full[i], 1);
      tc::mbar_init(&sm.empty[i], 1);
    }
    for (int x = 0; x < 2; ++x) {
      tc::mbar_init(&sm.s_full[x], 1);
      for (int q = 0; q < kParts; ++q) tc::mbar_init(&sm.p_part[x][q], 4);  // one elected arrival per softmax warp
      tc::mbar_init(&sm.o_final[x], 1);
    }
    tc::fence_barrier_init();
  }
  {
    // G not dividing 128 (G = 7: 18 tokens x 7 heads = 126 rows): the Q rows
    // outside the TMA box are zeroed (generic stores -> async proxy fence)
    const int tile_rows = tok * G;
    for (int i = threadIdx.x; i < 2 * 2 * (kRows - tile_rows) * 8; i += blockDim.x) {
      const int c = i & 7, r = tile_rows + ((i >> 3) % (kRows - tile_rows)), pq = (i >> 3) / (kRows - tile_rows);
      *reinterpret_cast<uint4*>(sm.q[pq >> 1] + (pq & 1) * kPanel + r * 128 + c * 16) = make_uint4(0, 0, 0, 0);
    }
    tc::fence_async_smem();
  }
  if (warp == kWarpAlloc) tc::tmem_alloc<kTmemCols>(&sm.tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const int n_full = max(sm.n_blocks[0], sm.n_blocks[1]);
  const int kb0 = sm.first_block;  // key ranges: blocks [kb0, n_full)
  const int b0 = kb0 + (int)((int64_t)blockIdx.z * (n_full - kb0) / gridDim.z);
  const int b1 = kb0 + (int)((int64_t)(blockIdx.z + 1) * (n_full - kb0) / gridDim.z);
  const int nA = max(0, min(sm.n_blocks[0], b1) - b0), nB = max(0, min(sm.n_blocks[1], b1) - b0);
  const int nblk = max(nA, nB);
  out += (int64_t)blockIdx.z * S * H * kDh;
  if (ml_out) ml_out += (int64_t)blockIdx.z * S * H * 2;

  if (warp >= kWarpTma) {
    tc::reg_dealloc<kOtherRegs>();
    if (warp == kWarpTma && lane == 0 && nblk > 0) {  // TMA producer
      tc::tma_prefetch(&tm_q);
      tc::tma_prefetch(&tm_k);
      tc::tma_prefetch(&tm_v);
      pdl_wait();  // Q and the slab's fresh K/V rows come from the previous kernel
      tc::mbar_arrive_expect_tx(&sm.q_full, (nB > 0 ? 2 : 1) * 2 * tok * G * 128);
      tc::tma_load_4d(sm.q[0], &tm_q, &sm.q_full, 0, 0, g, tA);
      tc::tma_load_4d(sm.q[0] + kPanel, &tm_q, &sm.q_full, 64, 0, g, tA);
      if (nB > 0) {
        tc::tma_load_4d(sm.q[1], &tm_q, &sm.q_full, 0, 0, g, tB);
        tc::tma_load_4d(sm.q[1] + kPanel, &tm_q, &sm.q_full, 64, 0, g, tB);
      }
      for (int i = 0; i < 2 * nblk; ++i) {  // item 2j = K(j), 2j + 1 = V(j)
        const int s = i % kStages;
        tc::mbar_wait(&sm.empty[s], ((i / kStages) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&sm.full[s], kTile);
        const CUtensorMap* tm = (i & 1) ? &tm_v : &tm_k;
        const int row = (b0 + (i >> 1)) * kKeys;
        tc::tma_load_2d(sm.kv[s], tm, &sm.full[s], g * kDh, row);
        tc::tma_load_2d(sm.kv[s] + kPanel, tm, &sm.full[s], g * kDh + 64, row);
      }
    } else if (warp == kWarpMma && nblk > 0) {  // MMA issuer (converged warp, elected lane)
      constexpr uint32_t idesc_qk = tc::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idesc_pv = tc::idesc_bf16(128, 128, 0, 1);
      const int n_of[2] = {nA, nB};
      auto wait_item = [&](int i) {
        tc::mbar_wait(&sm.full[i % kStages], (i / kStages) & 1);
        tc::tc_fence_after();
      };
      auto issue_s = [&](int x, int j) {  // S_x(j) = Q_x K_j^T
        const uint64_t qa = tc::smem_desc_sw128(tc::smem_u32(sm.q[x]), 16, 1024);
        const uint64_t kb = tc::smem_desc_sw128(tc::smem_u32(sm.kv[(2 * j) % kStages]), 16, 1024);
#pragma unroll
        for (int t = 0; t < kDh / 16; ++t) {
          const uint64_t step = (uint64_t)((t >> 2) * (kPanel >> 4) + (t & 3) * 2);
          tc::mma_bf16_ss_ws(tmem + 128 * x, qa + step, kb + step, idesc_qk, t > 0 ? 1u : 0u);
        }
        tc::mma_commit_ws(&sm.s_full[x]);
      };
      auto issue_pv = [&](int x, int j) {  // O_x += P_x(j) V_j, P from TMEM, part by part as they land
        const uint64_t vb = tc::smem_desc_sw128(tc::smem_u32(sm.kv[(2 * j + 1) % kStages]), kPanel, 1024);
#pragma unroll
        for (int hf = 0; hf < kParts; ++hf) {
          tc::mbar_wait(&sm.p_part[x][hf], j & 1);
          tc::tc_fence_after();
          if (hf == kParts - 1) TRACE10M(4, x, j);
#pragma unroll
          for (int t = (8 / kParts) * hf; t < (8 / kParts) * (hf + 1); ++t)
            tc::mma_bf16_ts_ws(tmem + 256 + 128 * x, tmem + 128 * x + 64 + 8 * t, vb + (uint64_t)(t * (2048 >> 4)),
                               idesc_pv, (j > 0 || t > 0) ? 1u : 0u);
        }
        if (j == n_of[x] - 1) tc::mma_commit_ws(&sm.o_final[x]);
      };
      tc::mbar_wait(&sm.q_full, 0);
      wait_item(0);
      for (int x = 0; x < 2; ++x)
        if (n_of[x] > 0) issue_s(x, 0);
      tc::mma_commit_ws(&sm.empty[0]);
      for (int j = 1; j < nblk; ++j) {
        wait_item(2 * j - 1);  // V(j-1)
        for (int x = 0; x < 2; ++x) {
          if (j - 1 < n_of[x]) issue_pv(x, j - 1);
          if (x == 0) wait_item(2 * j);  // K(j)
          if (j < n_of[x]) {
            TRACE10M(5, x, j);
            issue_s(x, j);
          }
        }
        tc::mma_commit_ws(&sm.empty[(2 * j - 1) % kStages]);
        tc::mma_commit_ws(&sm.empty[(2 * j) % kStages]);
      }
      wait_item(2 * nblk - 1);
      for (int x = 0; x < 2; ++x)
        if (nblk - 1 < n_of[x]) issue_pv(x, nblk - 1);
      tc::mma_commit_ws(&sm.empty[(2 * nblk - 1) % kStages]);
    }
  } else {
    tc::reg_alloc<kSoftmaxRegs>();
    pdl_wait();  // (tiles without key blocks write their rows without any other wait)
    const int x = warp >> 2;
    const int nx = x == 0 ? nA : nB;
    const int tx = x == 0 ? tA : tB;
    if (tx < S) softmax_tile10(sm, tmem, x, nx, b0, tx, S, H, G, g, horizon, key_start, scale_log2, out, ml_out);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == kWarpAlloc) tc::tmem_dealloc<kTmemCols>(tmem);
}

// Key-split partials -> output, fixed split order (as v5's merge).
__global__ void attn_v10_merge_kernel(const __nv_bfloat16* __restrict__ part_o, const float* __restrict__ part_ml,
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

#if IFKV_ATTN10_TRACE
extern "C" int ifkv_attn10_trace_read(long long* dst) {
  return cudaMemcpyFromSymbol(dst, g_attn10_trace, sizeof(g_attn10_trace)) == cudaSuccess ? 0 : 1;
}
extern "C" int ifkv_attn10_trace_clear() {
  static long long z[6 * 2 * kTraceBlocks] = {};
  return cudaMemcpyToSymbol(g_attn10_trace, z, sizeof(z)) == cudaSuccess ? 0 : 1;
}
#endif

extern "C" int ifkv_recompute_attn_tc_supported(int dtype, int H, int Hkv, int Dh) {
  if (dtype != IFKV_BF16 || Dh != kDh || Hkv <= 0 || H % Hkv) return 0;
  return H / Hkv <= 16 ? 1 : 0;  // a tile holds floor(128 / G) tokens x G heads
}

extern "C" int ifkv_recompute_attn_tc_v10(const void* q, const void* k_layer, const void* v_layer,
                                          const int64_t* key_start, const int64_t* horizon, int S, int H, int Hkv,
                                          int Dh, int n_rows, float scale, void* out, float* ml_out, void* stream) {
  IFKV_CHECK_ARG(Dh == kDh && Hkv > 0 && H % Hkv == 0 && H / Hkv <= 16, "recompute_attn_v10: unsupported shape");
  if (S <= 0) return IFKV_OK;
  const int G = H / Hkv;
  CUtensorMap tq, tk, tv;
  {
    // q [S][Hkv][G][Dh] viewed 4-D; a box = floor(128 / G) tokens x G heads
    uint64_t dims[4] = {(uint64_t)Dh, (uint64_t)G, (uint64_t)Hkv, (uint64_t)S};
    uint64_t strides[3] = {(uint64_t)Dh * 2, (uint64_t)G * Dh * 2, (uint64_t)H * Dh * 2};
    uint32_t box[4] = {64, (uint32_t)G, 1, (uint32_t)(kRows / G)};
    int rc = make_tmap_bf16(&tq, q, 4, dims, strides, box);
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
  const size_t smem = sizeof(Smem10) + 1024;
  IFKV_CUDA_CALL(cudaFuncSetAttribute(recompute_attn_v10_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem),
                 "recompute_attn_v10: smem attribute");
  const int per_pair = 2 * (kRows / G);
  const int pairs = (S + per_pair - 1) / per_pair;
  const float scale_log2 = scale * 1.4426950408889634f;
  cudaStream_t st = as_stream(stream);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int P = 1;
  if (Hkv * pairs < IFKV_ATTN10_SPLIT_WAVES * sms)
    P = min(IFKV_ATTN10_SPLIT_MAX, (IFKV_ATTN10_SPLIT_WAVES * sms + Hkv * pairs - 1) / (Hkv * pairs));
  if (P == 1) {
    IFKV_CUDA_CALL(launch_pdl(recompute_attn_v10_kernel, dim3(Hkv, pairs, 1), dim3(kThreads), smem, st, tq, tk, tv,
                              horizon, key_start, S, H, Hkv, scale_log2, (__nv_bfloat16*)out, ml_out),
                   "recompute_attn_v10: launch");
    IFKV_LAUNCH_CHECK("recompute_attn_v10");
    return IFKV_OK;
  }
  const int64_t rows = (int64_t)S * H;
  const size_t o_bytes = (size_t)P * rows * kDh * 2, ml_bytes = (size_t)P * rows * 2 * 4;
  void* ws = workspace_alloc(o_bytes + ml_bytes, st);
  if (!ws) {
    set_error("recompute_attn_v10: split workspace (%zu bytes)", o_bytes + ml_bytes);
    return IFKV_ERR_CUDA;
  }
  auto* part_o = reinterpret_cast<__nv_bfloat16*>(ws);
  auto* part_ml = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + o_bytes);
  IFKV_CUDA_CALL(launch_pdl(recompute_attn_v10_kernel, dim3(Hkv, pairs, P), dim3(kThreads), smem, st, tq, tk, tv,
                            horizon, key_start, S, H, Hkv, scale_log2, part_o, part_ml),
                 "recompute_attn_v10: launch (split)");
  IFKV_LAUNCH_CHECK("recompute_attn_v10 (split)");
  attn_v10_merge_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(part_o, part_ml, P, rows, (__nv_bfloat16*)out,
                                                                      ml_out);
  IFKV_LAUNCH_CHECK("recompute_attn_v10 (merge)");
  IFKV_CUDA_CALL(cudaFreeAsync(ws, st), "recompute_attn_v10: free split workspace");
  return IFKV_OK;
}
