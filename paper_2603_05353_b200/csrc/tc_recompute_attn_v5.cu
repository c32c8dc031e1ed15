// Selective-recompute attention, v5: two ping-ponging tiles per CTA like v2,
// but P goes to shared memory (SS-form PV MMA) instead of back into TMEM over
// S.  S_x(j+1) can then be issued as soon as the softmax has *read* S_x(j)
// (mbarrier s_free) rather than after PV_x(j) consumed P_x(j) -- the
// MMA -> softmax -> PV -> S handshake that bounds v2 (profiles/r1_attn_ab.md)
// leaves the critical path; the softmax of block j+1 starts while P(j) is
// still being written.
//
// Reference: recompute.py:92-114 (masked_attention model.py:297-315).
//
// smem (224 KB): Q 2 x 32 KB, P 2 x 32 KB (bf16, 128-byte swizzled K-major
// like Q), a 3-slot ring of 32 KB K / V blocks in consumption order
// K0 K1 V0 K2 V1 K3 V2 ...  TMEM: S_A, O_A, S_B, O_B (128 columns each).
// Warps: 0 TMA producer, 1 MMA issuer (warp-synchronous, elected lane),
// 2 TMEM allocator, 3 n_blocks, 4-7 softmax tile A, 8-11 softmax tile B.
#include "tc_common.cuh"

namespace ifkv {
namespace {

constexpr int kRows = 128;
constexpr int kKeys = 128;
constexpr int kDh = 128;
constexpr int kPanel = 128 * 128;  // 128 rows x 128 B (64 bf16)
constexpr int kTile = 2 * kPanel;  // 32 KB
constexpr int kSlots = 3;
constexpr uint32_t kTmemCols = 512;
constexpr float kRescaleLog2 = 8.0f;
#ifndef IFKV_ATTN5_DYN
#define IFKV_ATTN5_DYN 0
#endif
#ifndef IFKV_ATTN5_XORDER
#define IFKV_ATTN5_XORDER 0
#endif
#ifndef IFKV_ATTN5_ONEPASS
#define IFKV_ATTN5_ONEPASS 0
#endif
#ifndef IFKV_ATTN5_SPLITS
#define IFKV_ATTN5_SPLITS 1
#endif
// key splits while the tile pairs fill fewer than this many waves (x SMs), up to SPLIT_MAX
#ifndef IFKV_ATTN5_SPLIT_WAVES
#define IFKV_ATTN5_SPLIT_WAVES 2
#endif
#ifndef IFKV_ATTN5_SPLIT_MAX
#define IFKV_ATTN5_SPLIT_MAX 4
#endif
// IFKV_ATTN5_SEQ (A/B): the exponential phases of the two tiles alternate
// per SM sub-partition (A(j), B(j), A(j+1), ...) through per-warp mbarriers
#ifndef IFKV_ATTN5_SEQ
#define IFKV_ATTN5_SEQ 0
#endif
#ifndef IFKV_ATTN5_EXACTG
#define IFKV_ATTN5_EXACTG 1
#endif

struct Smem {
  uint8_t q[2][kTile];
  uint8_t p[2][kTile];
  uint8_t kv[kSlots][kTile];
  uint64_t q_full, full[kSlots], empty[kSlots];
  uint64_t s_full[2], s_free[2], p_full[2][2], pv_done[2][2], o_final[2];
  uint64_t seq[2][4];
  uint32_t tmem_base;
  int n_blocks[2];
  int first_block;
};

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(tc::smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Load order of the K/V ring: K(0), then for j >= 0: K(j+1), V(j) (and finally
// V(n-1)).  Item i of that order occupies slot i % kSlots; the MMA warp frees
// slots in the same order.

__device__ __forceinline__ int tile_blocks_warp(const int64_t* horizon, int t0, int tok, int S) {
  int64_t mx = -1;
  for (int t = t0 + (threadIdx.x & 31); t < min(t0 + tok, S); t += 32) mx = max(mx, horizon[t]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mx, o));
  return mx < 0 ? 0 : (int)((mx + kKeys) / kKeys);
}
// First key block any token of the tile can see (key ranges key_start..horizon;
// key_start == nullptr: every range starts at key 0).
__device__ __forceinline__ int tile_first_block_warp(const int64_t* key_start, int t0, int tok, int S) {
  if (key_start == nullptr) return 0;
  int64_t mn = INT64_MAX;
  for (int t = t0 + (threadIdx.x & 31); t < min(t0 + tok, S); t += 32) mn = min(mn, key_start[t]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = min(mn, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mn, o));
  return mn == INT64_MAX ? 0 : (int)(mn / kKeys);
}

// 8 bf16 (16 B chunk c of a 64-key panel) of row r into the swizzled P tile.
__device__ __forceinline__ void st_p_chunk(uint8_t* p, int r, int panel, int c, uint4 v) {
  *reinterpret_cast<uint4*>(p + panel * kPanel + r * 128 + ((c ^ (r & 7)) << 4)) = v;
}

__device__ __forceinline__ void softmax_tile(Smem& sm, uint32_t tmem, int x, int nblk, int ny, int b0, int t0, int S, int H,
                                             int G, int Gp, int g, const int64_t* __restrict__ horizon,
                                             const int64_t* __restrict__ key_start, float scale_log2,
                                             __nv_bfloat16* __restrict__ out, float* __restrict__ ml_out) {
  const int w = (threadIdx.x >> 5) & 3;
  const int lane = threadIdx.x & 31;
  const int row = w * 32 + lane;
  // tile row = token (row / Gp) x head of the group (row % Gp); Gp is G rounded
  // up to a power of two -- the padded heads are zero query rows (TMA OOB fill)
  const int tok = t0 + row / Gp;
  const bool valid = row < (kRows / Gp) * Gp && row % Gp < G && tok < S;  // tile rows: tokens x Gp heads
  const int hz = valid ? (int)horizon[tok] : INT_MAX;  // pad rows: never force the masked path
  const int ks = valid && key_start ? (int)key_start[tok] : 0;  // first visible key (block-diagonal prefill)
  const uint32_t lane_off = (uint32_t)(w * 32) << 16;
  const uint32_t t_s = tmem + 256 * x + lane_off;
  const uint32_t t_o = t_s + 128;
  uint8_t* P = sm.p[x];
  float m_used = -INFINITY, l = 0.f;
  for (int j = 0; j < nblk; ++j) {
    tc::mbar_wait(&sm.s_full[x], j & 1);
    tc::tc_fence_after();
    const int j0 = (b0 + j) * kKeys;
    const bool masked = __any_sync(0xffffffffu, j0 + kKeys - 1 > hz || j0 < ks);
#if IFKV_ATTN5_ONEPASS
    // one TMEM read of the whole S row; S_x(j+1) may start right after it
    float v[128];
#pragma unroll
    for (int q = 0; q < 4; ++q) tc::tmem_ld32(t_s + 32 * q, v + 32 * q);
    tc::tmem_ld_wait();
    tc::tc_fence_before();
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&sm.s_free[x]);
    if (masked) {
#pragma unroll
      for (int c = 0; c < 128; ++c)
        if (j0 + c > hz) v[c] = -INFINITY;
    }
    float mx = -INFINITY;
#pragma unroll
    for (int c = 0; c < 128; c += 2) mx = tc::max3(mx, v[c], v[c + 1]);
    float alpha = 1.f;
    bool need = false;
    if (mx > -INFINITY && (m_used == -INFINITY || (mx - m_used) * scale_log2 > kRescaleLog2)) {
      need = true;
      alpha = m_used == -INFINITY ? 0.f : tc::ex2((m_used - mx) * scale_log2);
      m_used = mx;
    }
    const float mb = m_used == -INFINITY ? 0.f : m_used * scale_log2;
    if (j > 0) {
      tc::mbar_wait(&sm.pv_done[x][(j - 1) & 1], ((j - 1) >> 1) & 1);
      tc::tc_fence_after();
    }
    if (j > 0 && __any_sync(0xffffffffu, need)) {
      const float a = need ? alpha : 1.f;
#pragma unroll 1
      for (int c = 0; c < kDh / 16; ++c) {
        float o[16];
        tc::tmem_ld16(t_o + c * 16, o);
        tc::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 16; ++u) o[u] *= a;
        tc::tmem_st16(t_o + c * 16, reinterpret_cast<const uint32_t*>(o));
      }
      tc::tmem_st_wait();
    }
    float sum = 0.f;
    const float2 sc2 = make_float2(scale_log2, scale_log2), mb2 = make_float2(-mb, -mb);
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      float2 sum2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int c8 = 0; c8 < 8; ++c8) {
        uint4 pk;
        uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = hf * 64 + c8 * 8 + 2 * u;
          const float2 xx = tc::ffma2(make_float2(v[c], v[c + 1]), sc2, mb2);
          const float2 e = make_float2(tc::ex2(xx.x), tc::ex2(xx.y));
          sum2 = tc::fadd2(sum2, e);
          pw[u] = tc::pack_bf16(e.x, e.y);
        }
        st_p_chunk(P, row, hf, c8, pk);
      }
      sum += sum2.x + sum2.y;
      tc::fence_async_smem();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&sm.p_full[x][hf]);
    }
#else
    float v[64];
    float mx = -INFINITY;
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      tc::tmem_ld32(t_s + hf * 64, v);
      tc::tmem_ld32(t_s + hf * 64 + 32, v + 32);
      tc::tmem_ld_wait();
      if (masked) {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (j0 + hf * 64 + c > hz || j0 + hf * 64 + c < ks) v[c] = -INFINITY;
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
    // PV(j-1) done: O idle for the rescale and the P buffer free.  PV(j-2) is
    // complete (S(j) was issued after it) and PV(j) cannot be: the barrier of
    // PV(j-1)'s parity is on its phase (j-1)/2 or just past it.
    if (j > 0) {
      tc::mbar_wait(&sm.pv_done[x][(j - 1) & 1], ((j - 1) >> 1) & 1);
      tc::tc_fence_after();
    }
    if (j > 0 && __any_sync(0xffffffffu, need)) {
      const float a = need ? alpha : 1.f;
#pragma unroll 1
      for (int c = 0; c < kDh / 32; ++c) {
        tc::tmem_ld32(t_o + c * 32, v);
        tc::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 32; ++u) v[u] *= a;
        tc::tmem_st32(t_o + c * 32, v);
      }
      tc::tmem_st_wait();  // rescaled O complete before PV(j) (ordered by the p_full arrive below)
    }
    float sum = 0.f;
    const float2 sc2 = make_float2(scale_log2, scale_log2), mb2 = make_float2(-mb, -mb);
#if IFKV_ATTN5_SEQ
    if (x == 0 ? (j > 0 && j - 1 < ny) : (j < ny)) tc::mbar_wait(&sm.seq[x][w], (x == 0 ? j - 1 : j) & 1);
#endif
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      tc::tmem_ld32(t_s + hf * 64, v);
      tc::tmem_ld32(t_s + hf * 64 + 32, v + 32);
      tc::tmem_ld_wait();
      if (hf == 1) {  // all of S(j) is in registers: the MMA may overwrite it with S(j+1)
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&sm.s_free[x]);
      }
      if (masked) {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (j0 + hf * 64 + c > hz || j0 + hf * 64 + c < ks) v[c] = -INFINITY;
      }
      float2 sum2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int c8 = 0; c8 < 8; ++c8) {  // 8 chunks of 8 keys = this 64-key panel
        uint4 pk;
        uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c8 * 8 + 2 * u;
          const float2 xx = tc::ffma2(make_float2(v[c], v[c + 1]), sc2, mb2);
#ifndef IFKV_ATTN_POLY_MASK
#define IFKV_ATTN_POLY_MASK 0
#endif
          float2 e;
          if (!masked && ((IFKV_ATTN_POLY_MASK >> ((c8 * 4 + u) & 7)) & 1))
            e = tc::ex2_poly2(xx);  // FMA-pipe exp2 for a fraction of the pairs (A/B)
          else
            e = make_float2(tc::ex2(xx.x), tc::ex2(xx.y));
          sum2 = tc::fadd2(sum2, e);
          pw[u] = tc::pack_bf16(e.x, e.y);
        }
        st_p_chunk(P, row, hf, c8, pk);
      }
      sum += sum2.x + sum2.y;
      tc::fence_async_smem();  // generic-proxy P writes -> visible to the tensor core
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&sm.p_full[x][hf]);
    }
#if IFKV_ATTN5_SEQ
    if (lane == 0 && (x == 0 ? j < ny : j + 1 < ny)) tc::mbar_arrive(&sm.seq[x ^ 1][w]);
#endif
#endif
    l = l * alpha + sum;
  }
  if (nblk > 0) {
    tc::mbar_wait(&sm.o_final[x], 0);
    tc::tc_fence_after();
  }
  const float inv = l > 0.f ? 1.f / l : 0.f;
  const int64_t orow = (int64_t)tok * H + g * G + row % Gp;
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

__global__ void __launch_bounds__(384, 1)
    recompute_attn_v5_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                             const __grid_constant__ CUtensorMap tm_v, const int64_t* __restrict__ horizon,
                             const int64_t* __restrict__ key_start, int S,
                             int H, int Hkv, int Gp, float scale_log2, __nv_bfloat16* __restrict__ out,
                             float* __restrict__ ml_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = H / Hkv;
  const int tok = kRows / Gp;
  const int g = blockIdx.x;
  const int pair = gridDim.y - 1 - blockIdx.y;
  const int tA = pair * 2 * tok, tB = tA + tok;
  if (warp == 3) {
    const int a = tA < S ? tile_blocks_warp(horizon, tA, tok, S) : 0;
    const int b = tB < S ? tile_blocks_warp(horizon, tB, tok, S) : 0;
    const int fa = tA < S ? tile_first_block_warp(key_start, tA, tok, S) : INT_MAX;
    const int fb = tB < S ? tile_first_block_warp(key_start, tB, tok, S) : INT_MAX;
    if (lane == 0) {
      sm.n_blocks[0] = a;
      sm.n_blocks[1] = b;
      sm.first_block = min(min(fa, fb), max(a, b));  // blocks before it are masked for every row
    }
  }
  if (threadIdx.x == 0) {
    tc::mbar_init(&sm.q_full, 1);
    for (int i = 0; i < kSlots; ++i) {
      tc::mbar_init(&sm.full[i], 1);
      tc::mbar_init(&sm.empty[i], 1);
    }
    for (int x = 0; x < 2; ++x) {
      tc::mbar_init(&sm.s_full[x], 1);
      tc::mbar_init(&sm.s_free[x], 4);  // one elected arrival per softmax warp
      tc::mbar_init(&sm.p_full[x][0], 4);
      tc::mbar_init(&sm.p_full[x][1], 4);
      tc::mbar_init(&sm.pv_done[x][0], 1);
      tc::mbar_init(&sm.pv_done[x][1], 1);
      tc::mbar_init(&sm.o_final[x], 1);
      for (int w = 0; w < 4; ++w) tc::mbar_init(&sm.seq[x][w], 1);
    }
    tc::fence_barrier_init();
  }
  {
    // a group that does not divide 128 rows (G = 7: 18 tokens x 7 heads =
    // 126 rows) leaves the last rows of each Q tile outside the TMA box: zero
    // them (generic-proxy stores, made visible to the tensor core below)
    const int tile_rows = tok * Gp;
    for (int i = threadIdx.x; i < 2 * 2 * (kRows - tile_rows) * 8; i += blockDim.x) {
      const int c = i & 7, r = tile_rows + ((i >> 3) % (kRows - tile_rows)), pq = (i >> 3) / (kRows - tile_rows);
      *reinterpret_cast<uint4*>(sm.q[pq >> 1] + (pq & 1) * kPanel + r * 128 + c * 16) = make_uint4(0, 0, 0, 0);
    }
    tc::fence_async_smem();
  }
  if (warp == 2) tc::tmem_alloc<kTmemCols>(&sm.tmem_base);
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

  if (warp < 4) {
    if (warp == 0 && lane == 0 && nblk > 0) {
      tc::tma_prefetch(&tm_q);
      tc::tma_prefetch(&tm_k);
      tc::tma_prefetch(&tm_v);
      tc::mbar_arrive_expect_tx(&sm.q_full, (nB > 0 ? 2 : 1) * 2 * tok * Gp * 128);  // box = tok x Gp rows
      tc::tma_load_4d(sm.q[0], &tm_q, &sm.q_full, 0, 0, g, tA);
      tc::tma_load_4d(sm.q[0] + kPanel, &tm_q, &sm.q_full, 64, 0, g, tA);
      if (nB > 0) {
        tc::tma_load_4d(sm.q[1], &tm_q, &sm.q_full, 0, 0, g, tB);
        tc::tma_load_4d(sm.q[1] + kPanel, &tm_q, &sm.q_full, 64, 0, g, tB);
      }
      // items in order K0, K1, V0, K2, V1, ..., K(n-1), V(n-2), V(n-1)
      const int n_items = 2 * nblk;
      for (int i = 0; i < n_items; ++i) {
        bool is_k;
        int j;
        if (i == 0) {
          is_k = true, j = 0;
        } else if (i == n_items - 1) {
          is_k = false, j = nblk - 1;
        } else {
          is_k = (i & 1), j = is_k ? (i + 1) / 2 : (i / 2) - 1;
        }
        const int s = i % kSlots;
        tc::mbar_wait(&sm.empty[s], ((i / kSlots) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&sm.full[s], kTile);
        const CUtensorMap* tm = is_k ? &tm_k : &tm_v;
        tc::tma_load_2d(sm.kv[s], tm, &sm.full[s], g * kDh, (b0 + j) * kKeys);
        tc::tma_load_2d(sm.kv[s] + kPanel, tm, &sm.full[s], g * kDh + 64, (b0 + j) * kKeys);
      }
    } else if (warp == 1 && nblk > 0) {  // MMA issuer: the whole warp, one elected lane issues
      constexpr uint32_t idesc_qk = tc::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idesc_pv = tc::idesc_bf16(128, 128, 0, 1);
      tc::mbar_wait(&sm.q_full, 0);
      const int n_items = 2 * nblk;
      auto item_of_k = [&](int j) { return j == 0 ? 0 : 2 * j - 1; };
      auto item_of_v = [&](int j) { return j == nblk - 1 ? n_items - 1 : 2 * j + 2; };
      auto wait_item = [&](int i) {
        tc::mbar_wait(&sm.full[i % kSlots], (i / kSlots) & 1);
        tc::tc_fence_after();
      };
      auto issue_s = [&](int x, int j) {  // S_x(j) = Q_x K_j^T
        const uint64_t qa = tc::smem_desc_sw128(tc::smem_u32(sm.q[x]), 16, 1024);
        const uint64_t kb = tc::smem_desc_sw128(tc::smem_u32(sm.kv[item_of_k(j) % kSlots]), 16, 1024);
#pragma unroll
        for (int t = 0; t < kDh / 16; ++t) {
          const uint64_t step = (uint64_t)((t >> 2) * (kPanel >> 4) + (t & 3) * 2);
          tc::mma_bf16_ss_ws(tmem + 256 * x, qa + step, kb + step, idesc_qk, t > 0 ? 1u : 0u);
        }
        tc::mma_commit_ws(&sm.s_full[x]);
      };
      auto issue_pv_half = [&](int x, int j, int hf) {  // O_x += P_x(j)[keys 64hf..] V_j
        const uint64_t pa = tc::smem_desc_sw128(tc::smem_u32(sm.p[x]), 16, 1024);
        const uint64_t vb = tc::smem_desc_sw128(tc::smem_u32(sm.kv[item_of_v(j) % kSlots]), kPanel, 1024);
#pragma unroll
        for (int t = 4 * hf; t < 4 * hf + 4; ++t) {
          const uint64_t astep = (uint64_t)((t >> 2) * (kPanel >> 4) + (t & 3) * 2);
          tc::mma_bf16_ss_ws(tmem + 256 * x + 128, pa + astep, vb + (uint64_t)(t * (2048 >> 4)), idesc_pv,
                             (j > 0 || t > 0) ? 1u : 0u);
        }
      };
      // prologue: S_A(0), S_B(0)
      wait_item(item_of_k(0));
      for (int x = 0; x < 2; ++x)
        if ((x == 0 ? nA : nB) > 0) issue_s(x, 0);
      tc::mma_commit_ws(&sm.empty[item_of_k(0) % kSlots]);
#if IFKV_ATTN5_DYN  // A/B: event-driven issue -- whichever S / PV half of either tile is ready
      {
        const int n_of[2] = {nA, nB};
        int s_next[2] = {1, 1}, pv_next[2] = {0, 0}, half[2] = {0, 0};
        auto k_ready = [&](int j) {
          const int i = item_of_k(j);
          return mbar_test(&sm.full[i % kSlots], (i / kSlots) & 1);
        };
        auto v_ready = [&](int j) {
          const int i = item_of_v(j);
          return mbar_test(&sm.full[i % kSlots], (i / kSlots) & 1);
        };
        while (pv_next[0] < n_of[0] || pv_next[1] < n_of[1]) {
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            const int y = x ^ 1;
            if (s_next[x] < n_of[x]) {
              const int j = s_next[x];
              if (mbar_test(&sm.s_free[x], (j - 1) & 1) && k_ready(j)) {
                tc::tc_fence_after();
                issue_s(x, j);
                ++s_next[x];
                if (s_next[y] > j || n_of[y] <= j) tc::mma_commit_ws(&sm.empty[item_of_k(j) % kSlots]);
              }
            }
            if (pv_next[x] < n_of[x]) {
              const int j = pv_next[x];
              if (mbar_test(&sm.p_full[x][half[x]], j & 1) && v_ready(j)) {
                tc::tc_fence_after();
                issue_pv_half(x, j, half[x]);
                if (++half[x] == 2) {
                  half[x] = 0;
                  tc::mma_commit_ws(&sm.pv_done[x][j & 1]);
                  if (j == n_of[x] - 1) tc::mma_commit_ws(&sm.o_final[x]);
                  ++pv_next[x];
                  if (pv_next[y] > j || n_of[y] <= j) tc::mma_commit_ws(&sm.empty[item_of_v(j) % kSlots]);
                }
              }
            }
          }
        }
      }
#else
#if IFKV_ATTN5_XORDER  // A/B: per tile, S_x(j+1) then PV_x(j), tile A then tile B
      for (int j = 0; j < nblk; ++j) {
        if (j + 1 < nblk) wait_item(item_of_k(j + 1));
        wait_item(item_of_v(j));
        for (int x = 0; x < 2; ++x) {
          const int nx = x == 0 ? nA : nB;
          if (j + 1 < nx) {
            tc::mbar_wait(&sm.s_free[x], j & 1);
            tc::tc_fence_after();
            issue_s(x, j + 1);
          }
          if (j < nx) {
            for (int hf = 0; hf < 2; ++hf) {
              tc::mbar_wait(&sm.p_full[x][hf], j & 1);
              tc::tc_fence_after();
              issue_pv_half(x, j, hf);
            }
            tc::mma_commit_ws(&sm.pv_done[x][j & 1]);
            if (j == nx - 1) tc::mma_commit_ws(&sm.o_final[x]);
          }
        }
        if (j + 1 < nblk) tc::mma_commit_ws(&sm.empty[item_of_k(j + 1) % kSlots]);
#else
      for (int j = 0; j < nblk; ++j) {
        // S_x(j+1) as soon as the softmax has read S_x(j)
        if (j + 1 < nblk) {
          wait_item(item_of_k(j + 1));
          for (int x = 0; x < 2; ++x) {
            if (j + 1 >= (x == 0 ? nA : nB)) continue;
            tc::mbar_wait(&sm.s_free[x], j & 1);
            tc::tc_fence_after();
            issue_s(x, j + 1);
          }
          tc::mma_commit_ws(&sm.empty[item_of_k(j + 1) % kSlots]);
        }
        // PV_x(j) by key halves as P halves land in smem
        wait_item(item_of_v(j));
        for (int x = 0; x < 2; ++x) {
          const int nx = x == 0 ? nA : nB;
          if (j >= nx) continue;
          for (int hf = 0; hf < 2; ++hf) {
            tc::mbar_wait(&sm.p_full[x][hf], j & 1);
            tc::tc_fence_after();
            issue_pv_half(x, j, hf);
          }
          tc::mma_commit_ws(&sm.pv_done[x][j & 1]);
          if (j == nx - 1) tc::mma_commit_ws(&sm.o_final[x]);
        }
#endif
        tc::mma_commit_ws(&sm.empty[item_of_v(j) % kSlots]);
      }
#endif  // IFKV_ATTN5_DYN
    }
  } else {
    const int x = (warp - 4) >> 2;
    const int nx = x == 0 ? nA : nB;
    const int tx = x == 0 ? tA : tB;
    if (tx < S)
      softmax_tile(sm, tmem, x, nx, x == 0 ? nB : nA, b0, tx, S, H, G, Gp, g, horizon, key_start, scale_log2, out,
                   ml_out);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) tc::tmem_dealloc<kTmemCols>(tmem);
}

// Key-split partials -> output: per row, weights l_p e^(m_p - M) over the
// splits in a fixed order (one warp per row, 4 columns per lane).
__global__ void attn_v5_merge_kernel(const __nv_bfloat16* __restrict__ part_o, const float* __restrict__ part_ml,
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

extern "C" int ifkv_recompute_attn_tc_supported(int dtype, int H, int Hkv, int Dh) {
  if (dtype != IFKV_BF16 || Dh != kDh || Hkv <= 0 || H % Hkv) return 0;
  return H / Hkv <= 16 ? 1 : 0;  // a tile holds floor(128 / G) tokens x G heads
}

extern "C" int ifkv_recompute_attn_tc_v5(const void* q, const void* k_layer, const void* v_layer,
                                         const int64_t* key_start, const int64_t* horizon, int S, int H, int Hkv,
                                         int Dh, int n_rows, float scale, void* out, float* ml_out, void* stream) {
  IFKV_CHECK_ARG(Dh == kDh && Hkv > 0 && H % Hkv == 0 && H / Hkv <= 16, "recompute_attn_v5: unsupported shape");
  if (S <= 0) return IFKV_OK;
  const int G = H / Hkv;
  // heads per tile row group: G itself (tiles of floor(128/G) tokens x G heads,
  // the last 128 mod G rows zero), or G padded to a power of two (A/B)
  int Gp = 1;
  while (Gp < G) Gp *= 2;
  if (IFKV_ATTN5_EXACTG) Gp = G;
  CUtensorMap tq, tk, tv;
  {
    // q [S][Hkv][G][Dh] viewed 4-D; the box takes Gp >= G heads (padded
    // variant: rows of heads G..Gp-1 fall outside the tensor, zero-filled by TMA)
    uint64_t dims[4] = {(uint64_t)Dh, (uint64_t)G, (uint64_t)Hkv, (uint64_t)S};
    uint64_t strides[3] = {(uint64_t)Dh * 2, (uint64_t)G * Dh * 2, (uint64_t)H * Dh * 2};
    uint32_t box[4] = {64, (uint32_t)Gp, 1, (uint32_t)(kRows / Gp)};
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
  const size_t smem = sizeof(Smem) + 1024;
  IFKV_CUDA_CALL(cudaFuncSetAttribute(recompute_attn_v5_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem),
                 "recompute_attn_v5: smem attribute");
  const int per_pair = 2 * (kRows / Gp);
  const int pairs = (S + per_pair - 1) / per_pair;
  const float scale_log2 = scale * 1.4426950408889634f;
  cudaStream_t st = as_stream(stream);
  // key splits (gridDim.z) when the tile pairs alone leave the GPU under two
  // waves: the heaviest (latest) pairs are split first into equal key ranges
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int P = 1;
#if IFKV_ATTN5_SPLITS
  if (Hkv * pairs < IFKV_ATTN5_SPLIT_WAVES * sms)
    P = min(IFKV_ATTN5_SPLIT_MAX, (IFKV_ATTN5_SPLIT_WAVES * sms + Hkv * pairs - 1) / (Hkv * pairs));
#endif
  if (P == 1) {
    recompute_attn_v5_kernel<<<dim3(Hkv, pairs, 1), 384, smem, st>>>(tq, tk, tv, horizon, key_start, S, H, Hkv, Gp,
                                                                     scale_log2, (__nv_bfloat16*)out, ml_out);
    IFKV_LAUNCH_CHECK("recompute_attn_v5");
    return IFKV_OK;
  }
  const int64_t rows = (int64_t)S * H;
  void* ws = nullptr;
  const size_t o_bytes = (size_t)P * rows * kDh * 2, ml_bytes = (size_t)P * rows * 2 * 4;
  ws = workspace_alloc(o_bytes + ml_bytes, st);
  if (!ws) {
    set_error("recompute_attn_v5: split workspace (%zu bytes)", o_bytes + ml_bytes);
    return IFKV_ERR_CUDA;
  }
  auto* part_o = reinterpret_cast<__nv_bfloat16*>(ws);
  auto* part_ml = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + o_bytes);
  recompute_attn_v5_kernel<<<dim3(Hkv, pairs, P), 384, smem, st>>>(tq, tk, tv, horizon, key_start, S, H, Hkv, Gp, scale_log2,
                                                                   part_o, part_ml);
  IFKV_LAUNCH_CHECK("recompute_attn_v5 (split)");
  attn_v5_merge_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(part_o, part_ml, P, rows, (__nv_bfloat16*)out,
                                                                     ml_out);
  IFKV_LAUNCH_CHECK("recompute_attn_v5 (merge)");
  IFKV_CUDA_CALL(cudaFreeAsync(ws, st), "recompute_attn_v5: free split workspace");
  return IFKV_OK;
}
