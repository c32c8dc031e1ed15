// Projection GEMMs of the layer stack on tcgen05 CTA pairs, with the
// consumer of every projection fused into the epilogue:
//
//   C[M][N] = A[M][K] . W[N][K]^T     (A bf16 activations, W bf16 weights
//                                      stored "out x in", both K-major)
//
// Reference arithmetic: the x @ wq/wk/wv, ctx @ wo and the SwiGLU MLP of
// recompute.py:98-116 / model.py:433-455,293-294 (the same layer stack
// prefills chunks, cache.py:74-99).  Epilogues:
//   STORE_BF16  C -> bf16 [M][ldo]
//   STORE_F32   C -> fp32 [M][ldo]       (split-term GEMMs of the scoring pass)
//   RESIDUAL    h[M][ldo] += C (fp32)    (h += ctx Wo, h += a Wdown; deterministic:
//                                          each tile owns its outputs, no split-K)
//   QKV_ROPE    q = R(pos) C[:, :H Dh] -> q_out; k = R(pos) C[:, H Dh : (H+Hkv) Dh]
//               and v = C[:, (H+Hkv) Dh:] scattered to slab rows dst_rows[m]
//               (recompute.py:99-112 + replace_entries cache.py:354-363, in place)
//   SWIGLU      W rows interleaved in 64-blocks (gate 64 | up 64 | ...):
//               out[m][j] = silu(g_j) * u_j -> bf16 [M][N/2]  (model.py:283-294)
//
// Schedule: persistent, one CTA pair (cluster of 2, cta_group::2) per two
// SMs.  A pair computes a 256 x BN tile: each CTA TMA-loads its 128 rows of A
// and half (BN/2 rows) of the W tile per 64-wide K step into a multi-stage
// ring; the leader CTA's single MMA thread issues the M = 256 MMAs, which
// read both CTAs' shared memory, and accumulates in TMEM of both SMs (each
// SM holds its own 128 rows x BN fp32).  Accumulators are double-buffered in
// TMEM (2 x BN <= 512 columns), so the epilogue of tile i (4 warps per CTA,
// one output row per thread) overlaps the main loop of tile i+1.
// Warp roles per CTA: 0 TMA producer, 1 MMA issuer (leader only), 2 TMEM
// allocator, 4-7 epilogue.
#include <string.h>

#include <algorithm>

#include "tc_pair.cuh"

namespace ifkv {
namespace {

constexpr int kBK = 64;            // K per stage: one 128-byte swizzle row
constexpr int kSmemBudget = 227 * 1024;

enum Epi { EPI_STORE_BF16 = 0, EPI_STORE_F32 = 1, EPI_RESIDUAL = 2, EPI_QKV_ROPE = 3, EPI_SWIGLU = 4 };

struct EpiParams {
  void* out;                 // STORE_* / SWIGLU output, RESIDUAL in/out
  int64_t ldo;               // output row stride (elements)
  const float2* cs;          // QKV_ROPE: (cos, sin) per row, [M][64]
  __nv_bfloat16* q_out;      // QKV_ROPE: [M][H][128] (may be null: K/V only)
  __nv_bfloat16* k_dst;      // QKV_ROPE: slab [*][Hkv][128]
  __nv_bfloat16* v_dst;
  const int64_t* dst_rows;   // QKV_ROPE: slab row of every A row (null = m)
  int H, Hkv;                // QKV_ROPE: head counts (Dh = 128); W rows start at head q_head0
  int q_head0;               // first output column's head index (H when only K/V are projected)
};

__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Pair tile BM x BN: BM = 256 (one M = 256 MMA per K slice, accumulator
// double-buffered in TMEM so the epilogue overlaps the next tile) or
// BM = 512 (two M = 256 MMAs per K slice sharing the W operand: 25 % fewer
// operand bytes per FLOP through L2 -> SM, which is what bounds the 256-row
// tile; single accumulator, 8 epilogue warps drain it).
template <int BM, int BN>
struct Cfg {
  static constexpr int kBlocks = BM / 256;            // M = 256 MMAs per K slice
  static constexpr int kBufs = kBlocks == 1 ? 2 : 1;  // TMEM accumulator buffers
  static constexpr int kAStage = (BM / 2) * 128;      // this CTA's BM/2 A rows x 64 k
  static constexpr int kBStage = (BN / 2) * 128;      // BN/2 W rows x 64 k
  static constexpr int kStage = kAStage + kBStage;
  static constexpr int kEpiWarps = 4 * kBlocks;
  static constexpr int kStaging = kEpiWarps * 2 * 2048;  // per epilogue warp: two 32-row x 64-byte store tiles
  static constexpr int kStageRoom = kSmemBudget - 2048 - kStaging;
  static constexpr int kStages = kStageRoom / kStage > 8 ? 8 : kStageRoom / kStage;
  static constexpr int kSmem = kStages * kStage + kStaging + 1024 /*align*/ + 512 /*barriers*/;
  static constexpr int kThreads = 128 + 32 * kEpiWarps;
};

// ---- epilogue output paths ----------------------------------------------------
// TMA store of a 32-row x 64-byte smem tile (SWIZZLE_64B layout), plain or
// with an fp32 add-reduction into global memory (the residual h += C: every
// element receives exactly one add, so the result is the fp32 sum h + C).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(tc::smem_u32(src)), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(tc::smem_u32(src)), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// One warp's staged store of 32 rows x 64 bytes (lane = row): row r's 16-byte
// chunk c lives at chunk c ^ ((r >> 1) & 3) (the TMA SWIZZLE_64B pattern,
// which also makes the 16-byte smem writes of a quarter-warp conflict-free).
struct Stager {
  uint8_t* buf;  // 2 x 2 KB, 1024-aligned
  int n = 0;     // tiles issued by this warp
  __device__ __forceinline__ void put(const uint4 (&row)[4], const CUtensorMap* map, int x, int y, bool reduce,
                                      int lane) {
    uint8_t* b = buf + (n & 1) * 2048;
    if (lane == 0 && n >= 2) bulk_wait_read1();  // the store issued 2 tiles ago has read its buffer
    __syncwarp();
    const int sw = (lane >> 1) & 3;
#pragma unroll
    for (int c = 0; c < 4; ++c) *reinterpret_cast<uint4*>(b + lane * 64 + ((c ^ sw) << 4)) = row[c];
    tc::fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      if (reduce)
        tma_reduce_add_2d(map, b, x, y);
      else
        tma_store_2d(map, b, x, y);
      bulk_commit();
    }
    ++n;
  }
};

__device__ __forceinline__ void pack8(const float* v, uint4& w) {
  w.x = tc::pack_bf16(v[0], v[1]);
  w.y = tc::pack_bf16(v[2], v[3]);
  w.z = tc::pack_bf16(v[4], v[5]);
  w.w = tc::pack_bf16(v[6], v[7]);
}

// QKV_ROPE: 32 accumulator columns (tile column col, a multiple of 32) of one
// row -> rotated q / k, or v, written straight to the q buffer or the slab row.
__device__ __forceinline__ void qkv_chunk(const EpiParams& p, const float (&v)[32], int64_t row, int col) {
  const int head = p.q_head0 + (col >> 7), e0 = col & 127;
  float r[32];
  if (head < p.H + p.Hkv) {
    const float4* c4 = reinterpret_cast<const float4*>(p.cs + row * 64 + (e0 >> 1));
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float4 a = __ldg(c4 + u);  // (cos, sin) of pairs 2u, 2u+1
      r[4 * u + 0] = v[4 * u + 0] * a.x - v[4 * u + 1] * a.y;
      r[4 * u + 1] = v[4 * u + 0] * a.y + v[4 * u + 1] * a.x;
      r[4 * u + 2] = v[4 * u + 2] * a.z - v[4 * u + 3] * a.w;
      r[4 * u + 3] = v[4 * u + 2] * a.w + v[4 * u + 3] * a.z;
    }
  } else {
#pragma unroll
    for (int u = 0; u < 32; ++u) r[u] = v[u];
  }
  __nv_bfloat16* d;
  if (head < p.H) {
    if (p.q_out == nullptr) return;
    d = p.q_out + (row * p.H + head) * 128 + e0;
  } else {
    const int64_t drow = p.dst_rows ? __ldg(p.dst_rows + row) : row;
    d = head < p.H + p.Hkv ? p.k_dst + (drow * p.Hkv + (head - p.H)) * 128 + e0
                           : p.v_dst + (drow * p.Hkv + (head - p.H - p.Hkv)) * 128 + e0;
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    uint4 w;
    pack8(r + 8 * u, w);
    reinterpret_cast<uint4*>(d)[u] = w;
  }
}

// Tile order: bands of `band` m-tiles, each band swept over every n-tile
// (m fastest inside the band).  The pairs resident at once then share a few W
// tiles and one band of A rows that fits L2: a large-M GEMM (the batched chunk
// prefill, M = 32768) reads A once per band instead of once per n-tile.  With
// band >= m_tiles this is the plain m-fastest order.
__device__ __forceinline__ void tile_mn(int t, int m_tiles, int n_tiles, int band, int& mt, int& nt) {
  const int per_band = band * n_tiles;
  const int b = t / per_band, r = t - b * per_band;
  const int bm = min(band, m_tiles - b * band);
  nt = r / bm;
  mt = b * band + (r - nt * bm);
}

template <int BM, int BN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cfg<BM, BN>::kThreads, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_w,
                     const __grid_constant__ CUtensorMap tm_out, int M, int N, int K, int m_tiles, int n_tiles, int band,
                     EpiParams p) {
  using C = Cfg<BM, BN>;
  constexpr int S = C::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = base + S * C::kStage;  // kEpiWarps x 2 x 2 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + C::kStaging);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;   // [kBufs] accumulator ready (both CTAs)
  uint64_t* tempty = tfull + 2;  // [kBufs] accumulator drained (leader; every epilogue warp of both CTAs arrives)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  pdl_trigger();
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int k_steps = (K + kBK - 1) / kBK;
  const int n_tile_total = m_tiles * n_tiles;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < C::kBufs; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], 2 * C::kEpiWarps);
    }
    tc::fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot);
  tc::tc_fence_before();
  cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- TMA producer (both CTAs: own BM/2 A rows, own half of the W tile) ----
    if (threadIdx.x == 0) {
      tc::tma_prefetch(&tm_a);
      tc::tma_prefetch(&tm_w);
      const uint32_t full0 = map_to_rank(full, 0);
      int it = 0;
      // programmatic launch: the weights of the first stages do not depend on
      // the previous kernel and are requested before waiting for it; the
      // activations (its output) after
      int pre = 0;
      if (pair < n_tile_total) {
        int mt, nt;
        tile_mn(pair, m_tiles, n_tiles, band, mt, nt);
        const int w0 = nt * BN + (int)rank * (BN / 2);
        pre = k_steps < S ? k_steps : S;
        for (int ks = 0; ks < pre; ++ks) {
          if (rank == 0) tc::mbar_arrive_expect_tx(&full[ks], 2 * C::kStage);
          tma_load_2d_pair(base + ks * C::kStage + C::kAStage, &tm_w, full0 + (uint32_t)(ks * 8), ks * kBK, w0);
        }
      }
      pdl_wait();
      for (int t = pair; t < n_tile_total; t += n_pairs) {
        int mt, nt;
        tile_mn(t, m_tiles, n_tiles, band, mt, nt);
        const int m0 = mt * BM + (int)rank * (BM / 2);
        const int w0 = nt * BN + (int)rank * (BN / 2);
        for (int ks = 0; ks < k_steps; ++ks, ++it) {
          const int s = it % S;
          const uint32_t bar = full0 + (uint32_t)(s * 8);
          uint8_t* st = base + s * C::kStage;
          if (it < pre) {  // W already requested
            tma_load_2d_pair(st, &tm_a, bar, ks * kBK, m0);
            continue;
          }
          tc::mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          if (rank == 0) tc::mbar_arrive_expect_tx(&full[s], 2 * C::kStage);
          tma_load_2d_pair(st, &tm_a, bar, ks * kBK, m0);
          tma_load_2d_pair(st + C::kAStage, &tm_w, bar, ks * kBK, w0);
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer (leader CTA, one elected lane) ----
    if (rank == 0) {
      const uint32_t idesc = tc::idesc_bf16(256, BN, 0, 0);
      int it = 0, local = 0;
      for (int t = pair; t < n_tile_total; t += n_pairs, ++local) {
        const int buf = local % C::kBufs;
        tc::mbar_wait(&tempty[buf], ((local / C::kBufs) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(buf * 256);
        for (int ks = 0; ks < k_steps; ++ks, ++it) {
          const int s = it % S;
          tc::mbar_wait(&full[s], (it / S) & 1);
          tc::tc_fence_after();
          const uint32_t st = tc::smem_u32(base + s * C::kStage);
          const uint64_t b = tc::smem_desc_sw128(st + C::kAStage, 16, 1024);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
#pragma unroll
            for (int blk = 0; blk < C::kBlocks; ++blk) {
              const uint64_t a = tc::smem_desc_sw128(st + blk * 16384, 16, 1024);
              mma_pair(d + (uint32_t)(blk * 256), a + (uint64_t)(2 * k), b + (uint64_t)(2 * k), idesc,
                       (ks | k) ? 1u : 0u);
            }
          commit_pair(&empty[s]);
        }
        commit_pair(&tfull[buf]);
      }
    }
  } else if (warp >= 4) {
    // ---- epilogue: thread = one output row of one 128-row block of this CTA ----
    const int ew = warp & 3;             // TMEM lane quadrant (warp id % 4)
    const int blk = (warp - 4) >> 2;     // accumulator block (BM = 512: two)
    const int lane = threadIdx.x & 31;
    const uint32_t tempty0 = map_to_rank(tempty, 0);
    Stager stg{staging + (warp - 4) * 4096};
    if (lane == 0 && EPI != EPI_QKV_ROPE) tc::tma_prefetch(&tm_out);
    int local = 0;
    for (int t = pair; t < n_tile_total; t += n_pairs, ++local) {
      const int buf = local % C::kBufs;
      tc::mbar_wait(&tfull[buf], (local / C::kBufs) & 1);
      tc::tc_fence_after();
      int mt, nt;
      tile_mn(t, m_tiles, n_tiles, band, mt, nt);
      const int row0 = mt * BM + (int)rank * (BM / 2) + blk * 128 + ew * 32;  // this warp's rows
      const int n0 = nt * BN;
      const uint32_t tbase = tmem + ((uint32_t)(ew * 32) << 16) + (uint32_t)((buf + blk) * 256);
      if (EPI == EPI_SWIGLU) {
        // tile columns [128 b, 128 b + 64) gate, [128 b + 64, 128 b + 128) up
#pragma unroll 1
        for (int c = 0; c < BN / 2; c += 32) {
          const int tc0 = (c / 64) * 128 + (c % 64);
          float g[32], u[32];
          tc::tmem_ld32(tbase + tc0, g);
          tc::tmem_ld32(tbase + tc0 + 64, u);
          tc::tmem_ld_wait();
          float y[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) y[e] = 0.5f * g[e] * (1.f + tanh_fast(0.5f * g[e])) * u[e];
          uint4 w[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) pack8(y + 8 * q, w[q]);
          if (n0 / 2 + c < N / 2) stg.put(w, &tm_out, n0 / 2 + c, row0, false, lane);
        }
      } else if (EPI == EPI_QKV_ROPE) {
        const int64_t row = row0 + lane;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          float v[32];
          tc::tmem_ld32(tbase + c, v);
          tc::tmem_ld_wait();
          if (row < M && n0 + c < N) qkv_chunk(p, v, row, n0 + c);
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          float v[32];
          tc::tmem_ld32(tbase + c, v);
          tc::tmem_ld_wait();
          if (n0 + c >= N) continue;
          if (EPI == EPI_STORE_BF16) {
            uint4 w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) pack8(v + 8 * q, w[q]);
            stg.put(w, &tm_out, n0 + c, row0, false, lane);
          } else {  // fp32 store / residual add: two 16-column tiles
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint4 w[4];
#pragma unroll
              for (int q = 0; q < 4; ++q)
                w[q] = make_uint4(__float_as_uint(v[16 * h + 4 * q]), __float_as_uint(v[16 * h + 4 * q + 1]),
                                  __float_as_uint(v[16 * h + 4 * q + 2]), __float_as_uint(v[16 * h + 4 * q + 3]));
              if (n0 + c + 16 * h < N) stg.put(w, &tm_out, n0 + c + 16 * h, row0, EPI == EPI_RESIDUAL, lane);
            }
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty0 + (uint32_t)(buf * 8));
    }
    if (lane == 0) bulk_wait_all();  // staged stores have left shared memory
    __syncwarp();
  }
  tc::tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc::tc_fence_after();
    tmem_dealloc_pair(tmem);
  }
}

int make_kmajor_map(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  uint64_t dims[2] = {(uint64_t)cols, (uint64_t)rows};
  uint64_t strides[1] = {(uint64_t)ld * 2};
  uint32_t box[2] = {(uint32_t)kBK, (uint32_t)box_rows};
  return make_tmap_bf16(m, ptr, 2, dims, strides, box);
}

int g_sms = 0;
int sm_count() {
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms < 2) g_sms = 148;
  }
  return g_sms;
}

template <int BM, int BN, int EPI>
int launch_tile(const void* a, int64_t lda, int M, int K, const void* w, int N, const EpiParams& p, cudaStream_t st) {
  using C = Cfg<BM, BN>;
  CUtensorMap ta, tw;
  int rc = make_kmajor_map(&ta, a, M, K, lda, BM / 2);
  if (rc) return rc;
  rc = make_kmajor_map(&tw, w, N, K, K, BN / 2);
  if (rc) return rc;
  CUtensorMap to;
  memset(&to, 0, sizeof(to));
  if (EPI != EPI_QKV_ROPE) {  // 32 rows x 64 bytes per TMA store
    const bool f32 = EPI == EPI_STORE_F32 || EPI == EPI_RESIDUAL;
    const int cols = EPI == EPI_SWIGLU ? N / 2 : N;
    uint64_t dims[2] = {(uint64_t)cols, (uint64_t)M};
    uint64_t strides[1] = {(uint64_t)p.ldo * (f32 ? 4 : 2)};
    uint32_t box[2] = {f32 ? 16u : 32u, 32u};
    rc = make_tmap(&to, p.out, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dims,
                   strides, box, CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
  }
  const int m_tiles = (M + BM - 1) / BM, n_tiles = (N + BN - 1) / BN;
  // a band of A rows of <= ~40 MB (a third of L2) per n-tile sweep
  const int64_t band_rows = (int64_t)40 * 1024 * 1024 / ((int64_t)K * 2);
  const int band = (int)std::max<int64_t>(1, std::min<int64_t>(m_tiles, band_rows / BM));
  const int pairs = std::min(m_tiles * n_tiles, sm_count() / 2);
  auto kern = gemm_pair_kernel<BM, BN, EPI>;
  IFKV_CUDA_CALL(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem), "gemm: smem");
  IFKV_CUDA_CALL(launch_pdl(kern, dim3(2 * pairs), dim3(C::kThreads), C::kSmem, st, ta, tw, to, M, N, K, m_tiles,
                            n_tiles, band, p),
                 "gemm: launch");
  IFKV_LAUNCH_CHECK("gemm");
  return IFKV_OK;
}

// Tile shape: the BN with the fewest "rounds x per-tile cost" over the
// persistent grid (a round = one tile per CTA pair; per-tile cost ~ BN + a
// fixed ~24-column overhead).  BM = 512 tiles (two M = 256 MMAs sharing the W
// operand, 25 % fewer L2 -> SM bytes per FLOP) measured 15-25 % slower than
// BM = 256 with a double-buffered accumulator (their epilogue cannot overlap
// the next main loop; profiles/r2_gemm.md), so they are not instantiated.
// tile code = BM / 256 * 1000 + BN.
int pick_tile(int M, int N, int K, bool swiglu) {
  static const int bns[] = {256, 224, 192, 160, 128};
  const int pairs = sm_count() / 2;
  int best = 1256;
  double best_cost = 1e30;
  for (int bn : bns) {
    if (swiglu && bn % 128) continue;
    const int tiles = ((M + 255) / 256) * ((N + bn - 1) / bn);
    const int rounds = (tiles + pairs - 1) / pairs;
    const double cost = rounds * (double)(bn + 24);
    if (cost < best_cost * (1 - 1e-9)) {
      best_cost = cost;
      best = 1000 + bn;
    }
  }
  (void)K;
  return best;
}

template <int EPI>
int launch(const void* a, int64_t lda, int M, int K, const void* w, int N, const EpiParams& p, int tile,
           cudaStream_t st) {
  switch (tile) {
    case 1256: return launch_tile<256, 256, EPI>(a, lda, M, K, w, N, p, st);
    case 1224: return launch_tile<256, 224, EPI>(a, lda, M, K, w, N, p, st);
    case 1192: return launch_tile<256, 192, EPI>(a, lda, M, K, w, N, p, st);
    case 1160: return launch_tile<256, 160, EPI>(a, lda, M, K, w, N, p, st);
    case 1128: return launch_tile<256, 128, EPI>(a, lda, M, K, w, N, p, st);
  }
  set_error("gemm: unsupported tile code %d (1000 + BN, BN in 256/224/192/160/128)", tile);
  return IFKV_ERR_ARG;
}

int check_common(const void* a, int64_t lda, int M, int K, const void* w, int N) {
  IFKV_CHECK_ARG(M >= 0 && K > 0 && N > 0, "gemm: bad shape M=%d K=%d N=%d", M, K, N);
  IFKV_CHECK_ARG(K % 8 == 0 && lda % 8 == 0 && lda >= K, "gemm: K and lda must be multiples of 8 (16-byte rows)");
  IFKV_CHECK_ARG(((uintptr_t)a & 15) == 0 && ((uintptr_t)w & 15) == 0, "gemm: operands must be 16-byte aligned");
  return IFKV_OK;
}

}  // namespace
}  // namespace ifkv

using namespace ifkv;

extern "C" int ifkv_gemm(const void* a, int64_t lda, int M, int K, const void* w, int N, int out_dtype, void* out,
                         int64_t ldo, int accumulate, int tile_n, void* stream) {
  int rc = check_common(a, lda, M, K, w, N);
  if (rc) return rc;
  IFKV_CHECK_ARG(out_dtype == IFKV_F32 || (out_dtype == IFKV_BF16 && !accumulate),
                 "gemm: output must be fp32, or bf16 without accumulation");
  IFKV_CHECK_ARG(out != nullptr && ldo >= N && ((uintptr_t)out & 15) == 0 && ldo % 8 == 0,
                 "gemm: output must be 16-byte aligned with ldo >= N, ldo %% 8 == 0");
  if (M == 0) return IFKV_OK;
  EpiParams p{};
  p.out = out;
  p.ldo = ldo;
  const int bn = tile_n > 0 ? tile_n : pick_tile(M, N, K, false);
  cudaStream_t st = as_stream(stream);
  if (accumulate) return launch<EPI_RESIDUAL>(a, lda, M, K, w, N, p, bn, st);
  if (out_dtype == IFKV_F32) return launch<EPI_STORE_F32>(a, lda, M, K, w, N, p, bn, st);
  return launch<EPI_STORE_BF16>(a, lda, M, K, w, N, p, bn, st);
}

extern "C" int ifkv_gemm_qkv_rope_scatter(const void* a, int64_t lda, int M, int K, const void* w, int H, int Hkv,
                                          int kv_only, const float* cs, void* q_out, void* k_dst, void* v_dst,
                                          const int64_t* dst_rows, int tile_n, void* stream) {
  const int heads = (kv_only ? 0 : H) + 2 * Hkv;
  const int N = heads * 128;
  int rc = check_common(a, lda, M, K, w, N);
  if (rc) return rc;
  IFKV_CHECK_ARG(H > 0 && Hkv > 0 && cs != nullptr && k_dst != nullptr && v_dst != nullptr &&
                     (kv_only || q_out != nullptr),
                 "gemm_qkv_rope_scatter: bad heads or null pointers");
  IFKV_CHECK_ARG(((uintptr_t)k_dst & 15) == 0 && ((uintptr_t)v_dst & 15) == 0 && ((uintptr_t)q_out & 15) == 0,
                 "gemm_qkv_rope_scatter: outputs must be 16-byte aligned");
  if (M == 0) return IFKV_OK;
  EpiParams p{};
  p.cs = reinterpret_cast<const float2*>(cs);
  p.q_out = kv_only ? nullptr : reinterpret_cast<__nv_bfloat16*>(q_out);
  p.k_dst = reinterpret_cast<__nv_bfloat16*>(k_dst);
  p.v_dst = reinterpret_cast<__nv_bfloat16*>(v_dst);
  p.dst_rows = dst_rows;
  p.H = H;
  p.Hkv = Hkv;
  p.q_head0 = kv_only ? H : 0;
  const int bn = tile_n > 0 ? tile_n : pick_tile(M, N, K, false);
  IFKV_CHECK_ARG(bn % 1000 % 32 == 0, "gemm_qkv_rope_scatter: tile width must be a multiple of 32");
  return launch<EPI_QKV_ROPE>(a, lda, M, K, w, N, p, bn, as_stream(stream));
}

extern "C" int ifkv_gemm_swiglu(const void* a, int64_t lda, int M, int K, const void* w, int d_ff, void* out,
                                int tile_n, void* stream) {
  const int N = 2 * d_ff;
  int rc = check_common(a, lda, M, K, w, N);
  if (rc) return rc;
  IFKV_CHECK_ARG(d_ff % 64 == 0, "gemm_swiglu: d_ff must be a multiple of 64 (64-blocks of gate|up)");
  IFKV_CHECK_ARG(out != nullptr && ((uintptr_t)out & 15) == 0, "gemm_swiglu: output must be 16-byte aligned");
  if (M == 0) return IFKV_OK;
  EpiParams p{};
  p.out = out;
  p.ldo = d_ff;
  const int bn = tile_n > 0 ? tile_n : pick_tile(M, N, K, true);  // BN 256 or 128: whole gate|up block pairs
  IFKV_CHECK_ARG(bn % 1000 % 128 == 0, "gemm_swiglu: tile width must be a multiple of 128");
  return launch<EPI_SWIGLU>(a, lda, M, K, w, N, p, bn, as_stream(stream));
}
