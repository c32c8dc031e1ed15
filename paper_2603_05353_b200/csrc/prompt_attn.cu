// Prompt attention over an injected KV prefix, split into <=128-key work
// items (flash-decoding style), plus the capture-layer column scorer.
// Generic SIMT fp32 path: any even Dh <= 256, any GQA ratio, fp32 or bf16
// K/V.  Arithmetic is fp32 throughout (fp32-accurate scoring, SURVEY §7 hard
// part 1); reference: selection.py:127-169, model.py:297-315, 352-360.
#include "common.cuh"

namespace ifkv {

constexpr int kItemKeysMax = 128;

// K/V element of the item's key j (kv head g), as fp32.
__device__ __forceinline__ const void* item_kv_base(const ifkv_attn_item& it, int kv_dtype, const void* slab,
                                                    const float* prompt, int M, int Hkv, int Dh, int g, int j,
                                                    bool& is_f32, int64_t& idx) {
  if (it.prompt) {
    is_f32 = true;
    idx = (((int64_t)it.group * M + it.key_row0 + j) * Hkv + g) * Dh;
    return prompt;
  }
  is_f32 = kv_dtype == IFKV_F32;
  idx = ((int64_t)(it.key_row0 + j) * Hkv + g) * Dh;
  return slab;
}

// Stage the item's keys (and values) of kv head g into shared memory as fp32.
// Ks has row stride Dh + 1 (conflict-free per-key dot products).
__device__ void stage_item(const ifkv_attn_item& it, int kv_dtype, const void* k_slab, const void* v_slab,
                           const float* k_prompt, const float* v_prompt, int M, int Hkv, int Dh, int g, float* Ks,
                           float* Vs) {
  const int n = it.n_keys;
  for (int t = threadIdx.x; t < n * Dh; t += blockDim.x) {
    int j = t / Dh, d = t - j * Dh;
    bool f32;
    int64_t idx;
    const void* kb = item_kv_base(it, kv_dtype, k_slab, k_prompt, M, Hkv, Dh, g, j, f32, idx);
    Ks[j * (Dh + 1) + d] = f32 ? reinterpret_cast<const float*>(kb)[idx + d] : load_as_f32(kb, IFKV_BF16, idx + d);
    if (Vs) {
      const void* vb = item_kv_base(it, kv_dtype, v_slab, v_prompt, M, Hkv, Dh, g, j, f32, idx);
      Vs[j * Dh + d] = f32 ? reinterpret_cast<const float*>(vb)[idx + d] : load_as_f32(vb, IFKV_BF16, idx + d);
    }
  }
}

// grid (n_items, Hkv, row_splits), 256 threads.  Warp w of split z handles
// query rows 8z + w, 8z + w + 8*row_splits, ... of the item's group restricted
// to kv head g (grp heads x M rows).
__global__ void __launch_bounds__(256) prompt_attn_partial_kernel(
    int kv_dtype, const float* __restrict__ qd, const void* __restrict__ k_slab, const void* __restrict__ v_slab,
    const float* __restrict__ k_prompt, const float* __restrict__ v_prompt, const ifkv_attn_item* __restrict__ items,
    int kmax, int H, int Hkv, int M, int Dh, float scale, float* __restrict__ part_ml, float* __restrict__ part_o) {
  extern __shared__ float smem[];
  const ifkv_attn_item it = items[blockIdx.x];
  const int g = blockIdx.y;
  const int grp = H / Hkv;
  const int n = it.n_keys;
  float* Ks = smem;                  // [n][Dh+1]
  float* Vs = Ks + kmax * (Dh + 1);  // [n][Dh]
  float* Qs = Vs + kmax * Dh;        // [8][Dh]
  stage_item(it, kv_dtype, k_slab, v_slab, k_prompt, v_prompt, M, Hkv, Dh, g, Ks, Vs);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* q = Qs + warp * Dh;
  const int rows = grp * M;
  for (int r = blockIdx.z * 8 + warp; r < rows; r += 8 * gridDim.z) {
    const int h = g * grp + r / M, m = r % M;
    const float* qsrc = qd + (((int64_t)it.qset * H + h) * M + m) * Dh;
    for (int d = lane; d < Dh; d += 32) q[d] = qsrc[d];
    __syncwarp();
    float logit[4];
    float mx = -INFINITY;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      int j = lane + 32 * t;
      logit[t] = -INFINITY;
      if (j < n && (!it.prompt || it.key_row0 + j <= m)) {
        const float* kr = Ks + j * (Dh + 1);
        float acc = 0.f;
        for (int d = 0; d < Dh; ++d) acc = fmaf(q[d], kr[d], acc);
        logit[t] = acc * scale;
      }
      mx = fmaxf(mx, logit[t]);
    }
    mx = warp_max(mx);
    float p[4], l = 0.f;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      p[t] = logit[t] == -INFINITY ? 0.f : expf(logit[t] - mx);
      l += p[t];
    }
    l = warp_sum(l);
    float o[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) o[u] = 0.f;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (32 * t >= n) break;
      for (int jj = 0; jj < 32; ++jj) {
        float pj = __shfl_sync(0xffffffffu, p[t], jj);
        int j = 32 * t + jj;
        if (j >= n) break;
        const float* vr = Vs + j * Dh;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          int d = lane + 32 * u;
          if (d < Dh) o[u] = fmaf(pj, vr[d], o[u]);
        }
      }
    }
    const int64_t row_id = ((int64_t)blockIdx.x * H + h) * M + m;
    if (lane == 0) {
      part_ml[2 * row_id] = mx;
      part_ml[2 * row_id + 1] = l;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      int d = lane + 32 * u;
      if (d < Dh) part_o[row_id * Dh + d] = o[u];
    }
    __syncwarp();
  }
}

// The same partial for Dh = 128 with 16-byte shared-memory traffic: keys staged
// with float4 / 8 x bf16 copies (K rows padded to 132 floats: conflict-free
// LDS.128 per 8-lane phase), each lane's key dot product in float4 steps over
// 4 accumulators, and the lane's 4 output dims read as one float4 per key in
// P V.  (The generic kernel reads everything as scalars: ~2.5x the
// instructions; the reorder first pass runs it for 16 prompt groups.)
constexpr int kD128 = 128, kKStride = 132;
__global__ void __launch_bounds__(256) prompt_attn_partial_d128_kernel(
    int kv_dtype, const float* __restrict__ qd, const void* __restrict__ k_slab, const void* __restrict__ v_slab,
    const float* __restrict__ k_prompt, const float* __restrict__ v_prompt, const ifkv_attn_item* __restrict__ items,
    int kmax, int H, int Hkv, int M, float scale, float* __restrict__ part_ml, float* __restrict__ part_o) {
  extern __shared__ __align__(16) float smem[];
  const ifkv_attn_item it = items[blockIdx.x];
  const int g = blockIdx.y;
  const int grp = H / Hkv;
  const int n = it.n_keys;
  float* Ks = smem;                    // [n][132]
  float* Vs = Ks + kmax * kKStride;    // [n][128]
  float* Qs = Vs + kmax * kD128;       // [8][128]
  for (int t = threadIdx.x; t < n * (kD128 / 4); t += blockDim.x) {  // one float4 of K and of V per step
    const int j = t / (kD128 / 4), c = (t % (kD128 / 4)) * 4;
    float4 kv4, vv4;
    if (it.prompt) {
      const int64_t idx = (((int64_t)it.group * M + it.key_row0 + j) * Hkv + g) * kD128 + c;
      kv4 = *reinterpret_cast<const float4*>(k_prompt + idx);
      vv4 = *reinterpret_cast<const float4*>(v_prompt + idx);
    } else {
      const int64_t idx = ((int64_t)(it.key_row0 + j) * Hkv + g) * kD128 + c;
      if (kv_dtype == IFKV_F32) {
        kv4 = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(k_slab) + idx);
        vv4 = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(v_slab) + idx);
      } else {
        const uint2 ku = *reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(k_slab) + idx);
        const uint2 vu = *reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(v_slab) + idx);
        const float2 k0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ku.x));
        const float2 k1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ku.y));
        const float2 v0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vu.x));
        const float2 v1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vu.y));
        kv4 = make_float4(k0.x, k0.y, k1.x, k1.y);
        vv4 = make_float4(v0.x, v0.y, v1.x, v1.y);
      }
    }
    *reinterpret_cast<float4*>(Ks + j * kKStride + c) = kv4;
    *reinterpret_cast<float4*>(Vs + j * kD128 + c) = vv4;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* q = Qs + warp * kD128;
  const int rows = grp * M;
  for (int r = blockIdx.z * 8 + warp; r < rows; r += 8 * gridDim.z) {
    const int h = g * grp + r / M, m = r % M;
    const float* qsrc = qd + (((int64_t)it.qset * H + h) * M + m) * kD128;
    *reinterpret_cast<float4*>(q + 4 * lane) = *reinterpret_cast<const float4*>(qsrc + 4 * lane);
    __syncwarp();
    float logit[4];
    float mx = -INFINITY;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int j = lane + 32 * t;
      logit[t] = -INFINITY;
      if (32 * t < n && j < n && (!it.prompt || it.key_row0 + j <= m)) {
        const float* kr = Ks + j * kKStride;
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 8
        for (int d = 0; d < kD128; d += 4) {
          const float4 qv = *reinterpret_cast<const float4*>(q + d);
          const float4 kv = *reinterpret_cast<const float4*>(kr + d);
          a0 = fmaf(qv.x, kv.x, a0);
          a1 = fmaf(qv.y, kv.y, a1);
          a2 = fmaf(qv.z, kv.z, a2);
          a3 = fmaf(qv.w, kv.w, a3);
        }
        logit[t] = ((a0 + a1) + (a2 + a3)) * scale;
      }
      mx = fmaxf(mx, logit[t]);
    }
    mx = warp_max(mx);
    float p[4], l = 0.f;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      p[t] = logit[t] == -INFINITY ? 0.f : expf(logit[t] - mx);
      l += p[t];
    }
    l = warp_sum(l);
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (32 * t >= n) break;
      const int jn = min(32, n - 32 * t);
      for (int jj = 0; jj < jn; ++jj) {
        const float pj = __shfl_sync(0xffffffffu, p[t], jj);
        const float4 v = *reinterpret_cast<const float4*>(Vs + (32 * t + jj) * kD128 + 4 * lane);
        o.x = fmaf(pj, v.x, o.x);
        o.y = fmaf(pj, v.y, o.y);
        o.z = fmaf(pj, v.z, o.z);
        o.w = fmaf(pj, v.w, o.w);
      }
    }
    const int64_t row_id = ((int64_t)blockIdx.x * H + h) * M + m;
    if (lane == 0) {
      part_ml[2 * row_id] = mx;
      part_ml[2 * row_id + 1] = l;
    }
    *reinterpret_cast<float4*>(part_o + row_id * kD128 + 4 * lane) = o;
    __syncwarp();
  }
}

// grid (G * H * M), 256 threads = 8 warps: merge the group's items.
// Items of group g: [item_begin[g], item_begin[g+1]) then, if
// prompt_item0 >= 0, items prompt_item0 + g * n_prompt + [0, n_prompt) (the
// group's causal prompt items: its prompt keys in blocks of <= 128).
// Warp w takes items k = w, w + 8, ...; lane owns Dh/32 (<= 4) consecutive
// dims as one vector load.  Warp partials combine in warp order through smem
// (fixed order -> deterministic).
__global__ void __launch_bounds__(256) prompt_attn_merge_kernel(
    const float* __restrict__ part_ml, const float* __restrict__ part_o, const int32_t* __restrict__ item_begin,
    int prompt_item0, int n_prompt, int H, int M, int Dh, float* __restrict__ ctx, float* __restrict__ ml,
    __nv_bfloat16* __restrict__ ctx3, int64_t plane) {
  __shared__ float s_m[8], s_l[8];
  __shared__ float s_o[8][256];
  pdl_trigger();  // the next projection (programmatic launch) may start streaming its weights
  pdl_wait();
  const int r = blockIdx.x;  // (g, h, m)
  const int m = r % M, h = (r / M) % H, g = r / (M * H);
  const int b = item_begin[g], e = item_begin[g + 1];
  const int n = e - b + (prompt_item0 >= 0 ? n_prompt : 0);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int per = (Dh + 31) / 32;  // dims per lane (<= 8)
  auto row_of = [&](int k) -> int64_t {
    const int it = k < e - b ? b + k : prompt_item0 + g * n_prompt + (k - (e - b));
    return ((int64_t)it * H + h) * M + m;
  };
  // pass 1: max over all items (every warp computes it redundantly -> no sync)
  float mx = -INFINITY;
  for (int k = lane; k < n; k += 32) mx = fmaxf(mx, part_ml[2 * row_of(k)]);
  mx = warp_max(mx);
  // pass 2: this warp's items, weighted
  float l = 0.f, o[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) o[u] = 0.f;
  const int d0 = lane * per;
  for (int k = w; k < n; k += 8) {
    const int64_t row = row_of(k);
    const float mi = part_ml[2 * row];
    const float a = mi == -INFINITY ? 0.f : expf(mi - mx);
    l += part_ml[2 * row + 1] * a;
    const float* src = part_o + row * Dh + d0;
    if (per == 4 && d0 < Dh) {
      const float4 v = *reinterpret_cast<const float4*>(src);
      o[0] += v.x * a; o[1] += v.y * a; o[2] += v.z * a; o[3] += v.w * a;
    } else {
      for (int u = 0; u < per; ++u)
        if (d0 + u < Dh) o[u] += src[u] * a;
    }
  }
  if (lane == 0) s_l[w] = l;
  for (int u = 0; u < per; ++u)
    if (d0 + u < Dh) s_o[w][d0 + u] = o[u];
  __syncthreads();
  float lt = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) lt += s_l[k];
  for (int d = threadIdx.x; d < Dh; d += blockDim.x) {
    float ot = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) ot += s_o[k][d];
    const float c = lt > 0.f ? ot / lt : 0.f;  // no item: empty shard
    const int64_t ci = (((int64_t)g * M + m) * H + h) * Dh + d;
    ctx[ci] = c;
    if (ctx3) {  // fused hi/mid/lo split of the next GEMM's operand
      __nv_bfloat16 a0, a1, a2;
      split3(c, a0, a1, a2);
      ctx3[ci] = a0;
      ctx3[plane + ci] = a1;
      ctx3[2 * plane + ci] = a2;
    }
  }
  if (threadIdx.x == 0) {
    ml[2 * (((int64_t)g * H + h) * M + m)] = mx;
    ml[2 * (((int64_t)g * H + h) * M + m) + 1] = lt;
  }
  (void)s_m;
}

// grid (n_items), 128 threads: thread j owns key column j of the item and
// sums p over all heads and prompt rows in a fixed order (deterministic).
// The same merge with one warp per (g, h, m) row (8 rows per CTA): for
// groups of few items (the reorder first pass: K groups, a chunk's items each),
// where a CTA per row is launch-bound.  Lane owns Dh/32 (<= 8) dims; items in
// order.
__global__ void __launch_bounds__(256) prompt_attn_merge_rows_kernel(
    const float* __restrict__ part_ml, const float* __restrict__ part_o, const int32_t* __restrict__ item_begin,
    int prompt_item0, int n_prompt, int G, int H, int M, int Dh, float* __restrict__ ctx, float* __restrict__ ml,
    __nv_bfloat16* __restrict__ ctx3, int64_t plane) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);  // (g, h, m)
  if (r >= G * H * M) return;
  const int lane = threadIdx.x & 31;
  const int m = r % M, h = (r / M) % H, g = r / (M * H);
  const int b = item_begin[g], e = item_begin[g + 1];
  const int n = e - b + (prompt_item0 >= 0 ? n_prompt : 0);
  auto row_of = [&](int k) -> int64_t {
    const int it = k < e - b ? b + k : prompt_item0 + g * n_prompt + (k - (e - b));
    return ((int64_t)it * H + h) * M + m;
  };
  float mx = -INFINITY;
  for (int k = lane; k < n; k += 32) mx = fmaxf(mx, part_ml[2 * row_of(k)]);
  mx = warp_max(mx);
  const int per = (Dh + 31) / 32;
  const int d0 = lane * per;
  float l = 0.f, o[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) o[u] = 0.f;
  for (int k = 0; k < n; ++k) {
    const int64_t row = row_of(k);
    const float mi = part_ml[2 * row];
    const float a = mi == -INFINITY ? 0.f : expf(mi - mx);
    l += part_ml[2 * row + 1] * a;
    const float* src = part_o + row * Dh + d0;
    if (per == 4 && d0 < Dh) {
      const float4 v = *reinterpret_cast<const float4*>(src);
      o[0] += v.x * a; o[1] += v.y * a; o[2] += v.z * a; o[3] += v.w * a;
    } else {
      for (int u = 0; u < per; ++u)
        if (d0 + u < Dh) o[u] += src[u] * a;
    }
  }
  for (int u = 0; u < per; ++u) {
    const int d = d0 + u;
    if (d >= Dh) break;
    const float c = l > 0.f ? o[u] / l : 0.f;
    const int64_t ci = (((int64_t)g * M + m) * H + h) * Dh + d;
    ctx[ci] = c;
    if (ctx3) {
      __nv_bfloat16 a0, a1, a2;
      split3(c, a0, a1, a2);
      ctx3[ci] = a0;
      ctx3[plane + ci] = a1;
      ctx3[2 * plane + ci] = a2;
    }
  }
  if (lane == 0) {
    ml[2 * (((int64_t)g * H + h) * M + m)] = mx;
    ml[2 * (((int64_t)g * H + h) * M + m) + 1] = l;
  }
}

__global__ void __launch_bounds__(128) score_columns_kernel(int kv_dtype, const float* __restrict__ qd,
                                                            const void* __restrict__ k_slab,
                                                            const ifkv_attn_item* __restrict__ items,
                                                            const float* __restrict__ ml, int H, int Hkv, int M,
                                                            int Dh, float scale, float* __restrict__ scores) {
  extern __shared__ float smem[];
  const ifkv_attn_item it = items[blockIdx.x];
  if (!it.score || it.prompt) return;
  float* Ks = smem;                          // [n][Dh+1]
  float* Qs = Ks + kItemKeysMax * (Dh + 1);  // [M][Dh] for one head
  const int grp = H / Hkv;
  const int j = threadIdx.x;
  float colsum = 0.f;
  for (int g = 0; g < Hkv; ++g) {
    __syncthreads();
    stage_item(it, kv_dtype, k_slab, nullptr, nullptr, nullptr, M, Hkv, Dh, g, Ks, nullptr);
    for (int hh = 0; hh < grp; ++hh) {
      const int h = g * grp + hh;
      __syncthreads();
      const float* qsrc = qd + ((int64_t)it.qset * H + h) * M * Dh;
      for (int t = threadIdx.x; t < M * Dh; t += blockDim.x) Qs[t] = qsrc[t];
      __syncthreads();
      if (j < it.n_keys) {
        const float* kr = Ks + j * (Dh + 1);
        for (int m = 0; m < M; ++m) {
          const float* q = Qs + m * Dh;
          float acc = 0.f;
          for (int d = 0; d < Dh; ++d) acc = fmaf(q[d], kr[d], acc);
          int64_t s = 2 * (((int64_t)it.group * H + h) * M + m);
          colsum += expf(acc * scale - ml[s]) / ml[s + 1];
        }
      }
    }
  }
  if (j < it.n_keys) scores[it.key_row0 + j] = colsum / (float)H;
}

}  // namespace ifkv

using namespace ifkv;

#ifndef IFKV_PARTIAL_D128
#define IFKV_PARTIAL_D128 1
#endif
static size_t partial_smem(int Dh, int kmax) { return (size_t)(kmax * (Dh + 1) + kmax * Dh + 8 * Dh) * 4; }
static size_t partial_d128_smem(int kmax) { return (size_t)(kmax * kKStride + kmax * kD128 + 8 * kD128) * 4; }
static size_t score_smem(int Dh, int M) { return (size_t)(kItemKeysMax * (Dh + 1) + M * Dh) * 4; }

extern "C" int ifkv_prompt_attn_partial(int kv_dtype, const float* qd, const void* k_slab, const void* v_slab,
                                        const float* k_prompt, const float* v_prompt, const ifkv_attn_item* items,
                                        int n_items, int max_keys, int H, int Hkv, int M, int Dh, float scale,
                                        float* part_ml, float* part_o, void* stream) {
  IFKV_CHECK_ARG(kv_dtype == IFKV_F32 || kv_dtype == IFKV_BF16, "prompt_attn_partial: bad dtype");
  IFKV_CHECK_ARG(Dh % 2 == 0 && Dh <= 256 && H % Hkv == 0 && M > 0, "prompt_attn_partial: bad shape");
  IFKV_CHECK_ARG(max_keys >= 1 && max_keys <= kItemKeysMax, "prompt_attn_partial: max_keys must be in [1, 128]");
  if (n_items <= 0) return IFKV_OK;
  const bool d128 = Dh == kD128 && IFKV_PARTIAL_D128;
  size_t sm = d128 ? partial_d128_smem(max_keys) : partial_smem(Dh, max_keys);
  if (d128)
    IFKV_CUDA_CALL(cudaFuncSetAttribute(prompt_attn_partial_d128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)sm),
                   "prompt_attn_partial: smem attribute");
  else
    IFKV_CUDA_CALL(cudaFuncSetAttribute(prompt_attn_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)sm),
                   "prompt_attn_partial: smem attribute");
  const int rows = (H / Hkv) * M;
  int splits = (rows + 7) / 8;
  const int64_t ctas = (int64_t)n_items * Hkv;
  while (splits > 1 && ctas * splits > 4 * 148) splits = (splits + 1) / 2;  // enough CTAs, bounded restaging
  dim3 grid(n_items, Hkv, splits);
  if (d128)
    prompt_attn_partial_d128_kernel<<<grid, 256, sm, as_stream(stream)>>>(
        kv_dtype, qd, k_slab, v_slab, k_prompt, v_prompt, items, max_keys, H, Hkv, M, scale, part_ml, part_o);
  else
    prompt_attn_partial_kernel<<<grid, 256, sm, as_stream(stream)>>>(kv_dtype, qd, k_slab, v_slab, k_prompt,
                                                                       v_prompt, items, max_keys, H, Hkv, M, Dh, scale,
                                                                       part_ml, part_o);
  IFKV_LAUNCH_CHECK("prompt_attn_partial");
  return IFKV_OK;
}

extern "C" int ifkv_prompt_attn_merge(const float* part_ml, const float* part_o, const int32_t* item_begin,
                                      int prompt_item0, int n_prompt_items, int G, int H, int M, int Dh, float* ctx,
                                      float* ml, void* ctx_split3, void* stream) {
  IFKV_CHECK_ARG(Dh <= 256 && G > 0, "prompt_attn_merge: bad shape");
  IFKV_CHECK_ARG(prompt_item0 < 0 || n_prompt_items >= 1, "prompt_attn_merge: n_prompt_items must be >= 1");
  prompt_attn_merge_kernel<<<G * H * M, 256, 0, as_stream(stream)>>>(
      part_ml, part_o, item_begin, prompt_item0, n_prompt_items, H, M, Dh, ctx, ml, (__nv_bfloat16*)ctx_split3,
      (int64_t)G * M * H * Dh);
  IFKV_LAUNCH_CHECK("prompt_attn_merge");
  return IFKV_OK;
}

extern "C" int ifkv_prompt_attn_merge_rows(const float* part_ml, const float* part_o, const int32_t* item_begin,
                                           int prompt_item0, int n_prompt_items, int G, int H, int M, int Dh,
                                           float* ctx, float* ml, void* ctx_split3, void* stream) {
  IFKV_CHECK_ARG(Dh <= 256 && G > 0, "prompt_attn_merge_rows: bad shape");
  IFKV_CHECK_ARG(prompt_item0 < 0 || n_prompt_items >= 1, "prompt_attn_merge_rows: n_prompt_items must be >= 1");
  const int64_t rows = (int64_t)G * H * M;
  IFKV_CUDA_CALL(launch_pdl(prompt_attn_merge_rows_kernel, dim3((unsigned)((rows + 7) / 8)), dim3(256), 0,
                            as_stream(stream), part_ml, part_o, item_begin, prompt_item0, n_prompt_items, G, H, M, Dh,
                            ctx, ml, (__nv_bfloat16*)ctx_split3, (int64_t)G * M * H * Dh),
                 "prompt_attn_merge_rows: launch");
  IFKV_LAUNCH_CHECK("prompt_attn_merge_rows");
  return IFKV_OK;
}

extern "C" int ifkv_score_columns(int kv_dtype, const float* qd, const void* k_slab, const ifkv_attn_item* items,
                                  int n_items, const float* ml, int H, int Hkv, int M, int Dh, float scale,
                                  float* scores, void* stream) {
  IFKV_CHECK_ARG(kv_dtype == IFKV_F32 || kv_dtype == IFKV_BF16, "score_columns: bad dtype");
  IFKV_CHECK_ARG(Dh % 2 == 0 && Dh <= 256 && H % Hkv == 0, "score_columns: bad shape");
  if (n_items <= 0) return IFKV_OK;
  size_t sm = score_smem(Dh, M);
  IFKV_CHECK_ARG(sm <= 220 * 1024, "score_columns: M*Dh too large for shared memory");
  IFKV_CUDA_CALL(cudaFuncSetAttribute(score_columns_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
                 "score_columns: smem attribute");
  score_columns_kernel<<<n_items, 128, sm, as_stream(stream)>>>(kv_dtype, qd, k_slab, items, ml, H, Hkv, M, Dh,
                                                                 scale, scores);
  IFKV_LAUNCH_CHECK("score_columns");
  return IFKV_OK;
}
