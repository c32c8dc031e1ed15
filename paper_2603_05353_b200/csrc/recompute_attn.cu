// Selective-recompute attention, generic SIMT path (fp32 mode, any even
// Dh <= 256, any GQA ratio).  Query row i attends keys 0..horizon[i]
// (recompute.py:92-93, 114; masked_attention model.py:297-315) with an
// online fp32 softmax.  The bf16 / Dh=128 hot path is the tcgen05 kernel in
// tc_recompute_attn.cu; this kernel is its numerical cross-check.
#include "common.cuh"

namespace ifkv {

constexpr int kRaTokens = 16;  // query rows (tokens) per CTA, one head
constexpr int kRaKeys = 32;    // keys per smem block

template <typename T>
__global__ void __launch_bounds__(128) recompute_attn_simt_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                                  const T* __restrict__ v,
                                                                  const int64_t* __restrict__ key_start,
                                                                  const int64_t* __restrict__ horizon, int S, int H,
                                                                  int Hkv, int Dh, float scale, T* __restrict__ out,
                                                                  float* __restrict__ ml_out) {
  extern __shared__ float smem[];
  float* Ks = smem;                          // [32][Dh+1]
  float* Vs = Ks + kRaKeys * (Dh + 1);       // [32][Dh]
  float* Qs = Vs + kRaKeys * Dh;             // [16][Dh]
  const int t0 = blockIdx.x * kRaTokens;
  const int h = blockIdx.y;
  const int g = h / (H / Hkv);
  const int nt = min(kRaTokens, S - t0);
  for (int t = threadIdx.x; t < nt * Dh; t += blockDim.x) {
    int r = t / Dh, d = t - r * Dh;
    Qs[t] = to_f32(q[((int64_t)(t0 + r) * H + h) * Dh + d]);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t hz[4], ks[4];
  float m[4], l[4], o[4][8];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    int row = warp * 4 + r;
    hz[r] = row < nt ? horizon[t0 + row] : -1;
    ks[r] = row < nt && key_start ? key_start[t0 + row] : 0;
    m[r] = -INFINITY;
    l[r] = 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) o[r][u] = 0.f;
  }
  int64_t kmax = -1;  // largest horizon of the tile (-1 in partial mode: no local key visible)
  int64_t kmin = INT64_MAX;  // smallest first key of the tile (block-diagonal prefill)
  for (int r = 0; r < nt; ++r) {
    kmax = max(kmax, horizon[t0 + r]);
    kmin = min(kmin, key_start ? key_start[t0 + r] : (int64_t)0);
  }
  for (int64_t k0 = kmin == INT64_MAX ? 0 : kmin / kRaKeys * kRaKeys; k0 <= kmax; k0 += kRaKeys) {
    __syncthreads();
    const int nk = (int)(kmax + 1 - k0 < kRaKeys ? kmax + 1 - k0 : kRaKeys);
    for (int t = threadIdx.x; t < nk * Dh; t += blockDim.x) {
      int j = t / Dh, d = t - j * Dh;
      int64_t src = ((k0 + j) * Hkv + g) * Dh + d;
      Ks[j * (Dh + 1) + d] = to_f32(k[src]);
      Vs[j * Dh + d] = to_f32(v[src]);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (hz[r] < k0 || k0 + kRaKeys <= ks[r]) continue;  // warp-uniform
      const float* qr = Qs + (warp * 4 + r) * Dh;
      float s = -INFINITY;
      if (lane < nk && k0 + lane <= hz[r] && k0 + lane >= ks[r]) {
        const float* kr = Ks + lane * (Dh + 1);
        float acc = 0.f;
        for (int d = 0; d < Dh; ++d) acc = fmaf(qr[d], kr[d], acc);
        s = acc * scale;
      }
      float mb = warp_max(s);
      float mn = fmaxf(m[r], mb);
      float p = s == -INFINITY ? 0.f : expf(s - mn);
      float alpha = m[r] == -INFINITY ? 0.f : expf(m[r] - mn);
      l[r] = l[r] * alpha + warp_sum(p);
      m[r] = mn;
#pragma unroll
      for (int u = 0; u < 8; ++u) o[r][u] *= alpha;
      for (int j = 0; j < nk; ++j) {
        float pj = __shfl_sync(0xffffffffu, p, j);
        const float* vr = Vs + j * Dh;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          int d = lane + 32 * u;
          if (d < Dh) o[r][u] = fmaf(pj, vr[d], o[r][u]);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    int row = warp * 4 + r;
    if (row >= nt) continue;
    const int64_t orow = (int64_t)(t0 + row) * H + h;
    const float inv = l[r] > 0.f ? 1.f / l[r] : 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      int d = lane + 32 * u;
      if (d < Dh) out[orow * Dh + d] = from_f32<T>(o[r][u] * inv);
    }
    if (ml_out && lane == 0) {
      ml_out[2 * orow] = m[r];
      ml_out[2 * orow + 1] = l[r];
    }
  }
}

}  // namespace ifkv

using namespace ifkv;

extern "C" int ifkv_recompute_attn_tc_v10(const void* q, const void* k_layer, const void* v_layer,
                                          const int64_t* key_start, const int64_t* horizon, int S, int H, int Hkv,
                                          int Dh, int n_rows, float scale, void* out, float* ml_out, void* stream);
// The tcgen05 kernel (tc_recompute_attn_v10.cu): two tiles of floor(128/G)
// tokens x G heads per CTA, P written into the TMEM columns of its own S tile
// and read by a TS-form PV MMA part by part, an eighth of the exponentials on
// the FMA pipe, key splits below two waves.  The generations it replaced (v2,
// v4, v5, the CTA-pair kernels v7-v9) were measured slower and moved out of
// the library (profiles/r1_attn_ab.md, r2_attn.md, r2_attn10.md; sources in
// profiles/attic/).
static int recompute_attn_tc_any(const void* q, const void* k_layer, const void* v_layer, const int64_t* horizon,
                                 int S, int H, int Hkv, int Dh, int n_rows, float scale, void* out, float* ml_out,
                                 void* stream, const int64_t* key_start = nullptr) {
  return ifkv_recompute_attn_tc_v10(q, k_layer, v_layer, key_start, horizon, S, H, Hkv, Dh, n_rows, scale, out,
                                    ml_out, stream);
}

static int recompute_attn_simt_impl(int dtype, const void* q, const void* k_layer, const void* v_layer,
                                    const int64_t* horizon, int S, int H, int Hkv, int Dh, float scale, void* out,
                                    float* ml_out, void* stream, const int64_t* key_start = nullptr) {
  IFKV_CHECK_ARG(dtype == IFKV_F32 || dtype == IFKV_BF16, "recompute_attn: bad dtype");
  IFKV_CHECK_ARG(Dh % 2 == 0 && Dh <= 256 && Hkv > 0 && H % Hkv == 0, "recompute_attn: bad shape");
  if (S <= 0) return IFKV_OK;
  size_t sm = (size_t)(kRaKeys * (Dh + 1) + kRaKeys * Dh + kRaTokens * Dh) * 4;
  dim3 grid((S + kRaTokens - 1) / kRaTokens, H);
  if (dtype == IFKV_BF16) {
    auto kern = recompute_attn_simt_kernel<__nv_bfloat16>;
    IFKV_CUDA_CALL(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm), "recompute_attn");
    kern<<<grid, 128, sm, as_stream(stream)>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k_layer,
                                               (const __nv_bfloat16*)v_layer, key_start, horizon, S, H, Hkv, Dh, scale,
                                               (__nv_bfloat16*)out, ml_out);
  } else {
    auto kern = recompute_attn_simt_kernel<float>;
    IFKV_CUDA_CALL(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm), "recompute_attn");
    kern<<<grid, 128, sm, as_stream(stream)>>>((const float*)q, (const float*)k_layer, (const float*)v_layer, key_start,
                                               horizon, S, H, Hkv, Dh, scale, (float*)out, ml_out);
  }
  IFKV_LAUNCH_CHECK("recompute_attn_simt");
  return IFKV_OK;
}

extern "C" int ifkv_recompute_attn_simt(int dtype, const void* q, const void* k_layer, const void* v_layer,
                                        const int64_t* horizon, int S, int H, int Hkv, int Dh, int n_rows, float scale,
                                        void* out, void* stream) {
  return recompute_attn_simt_impl(dtype, q, k_layer, v_layer, horizon, S, H, Hkv, Dh, scale, out, nullptr, stream);
}

extern "C" int ifkv_recompute_attn_range(int dtype, const void* q, const void* k_layer, const void* v_layer,
                                         const int64_t* key_start, const int64_t* horizon, int S, int H, int Hkv,
                                         int Dh, int n_rows, float scale, void* out, void* stream) {
  IFKV_CHECK_ARG(key_start != nullptr, "recompute_attn_range: key_start required");
  if (ifkv_recompute_attn_tc_supported(dtype, H, Hkv, Dh))
    return recompute_attn_tc_any(q, k_layer, v_layer, horizon, S, H, Hkv, Dh, n_rows, scale, out, nullptr, stream,
                                 key_start);
  return recompute_attn_simt_impl(dtype, q, k_layer, v_layer, horizon, S, H, Hkv, Dh, scale, out, nullptr, stream,
                                  key_start);
}

extern "C" int ifkv_recompute_attn(int dtype, const void* q, const void* k_layer, const void* v_layer,
                                   const int64_t* horizon, int S, int H, int Hkv, int Dh, int n_rows, float scale,
                                   void* out, void* stream) {
  if (ifkv_recompute_attn_tc_supported(dtype, H, Hkv, Dh))
    return recompute_attn_tc_any(q, k_layer, v_layer, horizon, S, H, Hkv, Dh, n_rows, scale, out, nullptr, stream);
  return recompute_attn_simt_impl(dtype, q, k_layer, v_layer, horizon, S, H, Hkv, Dh, scale, out, nullptr, stream);
}

namespace ifkv {
// Softmax-state merge of P partial attentions of the same queries over
// disjoint key sets (chunk sharding: recompute.py:114 and model.py:297-315
// over every rank's keys):
//   out[r] = sum_p l_p e^(m_p - M) o_p / sum_p l_p e^(m_p - M), fixed p order.
// One warp per context row r (Dh columns, 4 per lane per 128); parts_o
// [P][rows][Dh] each normalised by its own l.  The (m, l) pairs may be laid
// out in another row order: context row r = (g, m, h) of [G][M][H] reads ml
// row (g, h, m) of [G][H][M] (the prompt states); M = 1 makes them the same
// order (the query states).  m in natural-log units.
template <typename TC>
__global__ void merge_states_kernel(const TC* __restrict__ part_o, const float* __restrict__ part_ml, int P,
                                    int64_t rows, int Dh, int H, int M, TC* __restrict__ out,
                                    float* __restrict__ ml_out) {
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int64_t g = r / ((int64_t)M * H), mi = (r / H) % M, h = r % H;
  const int64_t rm = (g * H + h) * M + mi;
  float Mx = -INFINITY;
  for (int p = 0; p < P; ++p) Mx = fmaxf(Mx, part_ml[2 * (p * rows + rm)]);
  float L = 0.f;
  for (int c0 = 0; c0 < Dh; c0 += 128) {
    const int c = c0 + lane * 4;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    float Lc = 0.f;
    for (int p = 0; p < P; ++p) {
      const float m = part_ml[2 * (p * rows + rm)];
      const float w = m == -INFINITY ? 0.f : part_ml[2 * (p * rows + rm) + 1] * expf(m - Mx);
      Lc += w;
      if (c < Dh) {
        const TC* src = part_o + (p * rows + r) * Dh + c;
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] += w * to_f32(src[u]);
      }
    }
    L = Lc;
    if (c < Dh) {
      const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
      for (int u = 0; u < 4; ++u) out[r * Dh + c + u] = from_f32<TC>(acc[u] * inv);
    }
  }
  if (ml_out && lane == 0) {
    ml_out[2 * rm] = Mx;
    ml_out[2 * rm + 1] = L;
  }
}
}  // namespace ifkv

extern "C" int ifkv_merge_partials(const void* part_o, const float* part_ml, int P, int64_t rows, int Dh, void* out,
                                   float* ml_out, void* stream) {
  IFKV_CHECK_ARG(P >= 1 && rows >= 0 && Dh > 0 && Dh % 4 == 0, "merge_partials: bad shape");
  if (rows == 0) return IFKV_OK;
  merge_states_kernel<__nv_bfloat16><<<(unsigned)((rows + 7) / 8), 256, 0, as_stream(stream)>>>(
      (const __nv_bfloat16*)part_o, part_ml, P, rows, Dh, 1, 1, (__nv_bfloat16*)out, ml_out);
  IFKV_LAUNCH_CHECK("merge_partials");
  return IFKV_OK;
}

extern "C" int ifkv_merge_prompt_states(const float* part_ctx, const float* part_ml, int P, int G, int M, int H,
                                        int Dh, float* out_ctx, float* out_ml, void* stream) {
  IFKV_CHECK_ARG(P >= 1 && G >= 0 && M > 0 && H > 0 && Dh > 0 && Dh % 4 == 0, "merge_prompt_states: bad shape");
  const int64_t rows = (int64_t)G * M * H;
  if (rows == 0) return IFKV_OK;
  merge_states_kernel<float><<<(unsigned)((rows + 7) / 8), 256, 0, as_stream(stream)>>>(
      part_ctx, part_ml, P, rows, Dh, H, M, out_ctx, out_ml);
  IFKV_LAUNCH_CHECK("merge_prompt_states");
  return IFKV_OK;
}

extern "C" int ifkv_recompute_attn_partial(int dtype, const void* q, const void* k_layer, const void* v_layer,
                                           const int64_t* horizon, int S, int H, int Hkv, int Dh, int n_rows,
                                           float scale, void* out, float* ml_out, void* stream) {
  IFKV_CHECK_ARG(ml_out != nullptr, "recompute_attn_partial: ml_out required");
  IFKV_CHECK_ARG(n_rows > 0, "recompute_attn_partial: the shard holds no key rows (n_rows = %d)", n_rows);
  if (ifkv_recompute_attn_tc_supported(dtype, H, Hkv, Dh))
    return recompute_attn_tc_any(q, k_layer, v_layer, horizon, S, H, Hkv, Dh, n_rows, scale, out, ml_out, stream);
  return recompute_attn_simt_impl(dtype, q, k_layer, v_layer, horizon, S, H, Hkv, Dh, scale, out, ml_out, stream);
}
