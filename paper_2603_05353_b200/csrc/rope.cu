// RoPE tables, Kernel 1 (in-place / out-of-place key re-rotation), rotated
// query sets and the fused fresh-q/k/v rope + scatter epilogue.
//
// Pair convention: interleaved (x[2i], x[2i+1]) rotated by theta_i * p,
// theta_i = base^(-2i/Dh) (reference model.py:226-270).
#include "common.cuh"

namespace ifkv {

__global__ void rope_table_kernel(const int64_t* __restrict__ pos, int n, int half, double base,
                                  float2* __restrict__ cs) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * half) return;
  int i = (int)(t / half), j = (int)(t % half);
  double theta = pow(base, (-2.0 * (double)j) / (double)(2 * half));
  double ang = (double)pos[i] * theta;
  double s, c;
  sincos(ang, &s, &c);
  cs[t] = make_float2((float)c, (float)s);
}

// ---- Kernel 1 -----------------------------------------------------------
// One thread moves one 16-byte vector (8 bf16 / 4 fp32 = 4 / 2 pairs) and
// handles kUnroll vectors with all loads issued before any store.  Rows whose
// table entry is negative are skipped (in place) or copied bit-exactly.
template <typename T, int kUnroll>
__global__ void __launch_bounds__(256) rotate_rows_kernel(const T* __restrict__ src, T* __restrict__ dst,
                                                          int64_t layer_stride, int64_t n_rows,
                                                          int vecs_per_row, int vecs_per_head,
                                                          int64_t total_vecs, const int32_t* __restrict__ row_table,
                                                          const float2* __restrict__ cs, int half, bool in_place) {
  constexpr int kVec = 16 / sizeof(T);
  constexpr int kPairs = kVec / 2;
  using V = uint4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < total_vecs;
       base += stride * kUnroll) {
    V val[kUnroll];
    int tab[kUnroll];
    bool live[kUnroll];
    int64_t off[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      int64_t g = base + (int64_t)u * stride;
      live[u] = g < total_vecs;
      tab[u] = -1;
      off[u] = 0;
      if (live[u]) {
        int64_t row_all = g / vecs_per_row;  // (layer, row)
        int vin = (int)(g - row_all * vecs_per_row);
        int64_t layer = row_all / n_rows;
        int64_t row = row_all - layer * n_rows;
        int t = row_table[row];
        off[u] = layer * layer_stride + row * (int64_t)vecs_per_row * kVec + (int64_t)vin * kVec;
        if (t >= 0 || !in_place) val[u] = *reinterpret_cast<const V*>(src + off[u]);
        // table offset of this vector's first pair
        tab[u] = t >= 0 ? (t * half + (vin % vecs_per_head) * kPairs) : -1;
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (!live[u]) continue;
      if (tab[u] >= 0) {
        T* e = reinterpret_cast<T*>(&val[u]);
#pragma unroll
        for (int p = 0; p < kPairs; ++p) {
          float2 c = __ldg(cs + tab[u] + p);
          float x0 = to_f32(e[2 * p]), x1 = to_f32(e[2 * p + 1]);
          e[2 * p] = from_f32<T>(x0 * c.x - x1 * c.y);
          e[2 * p + 1] = from_f32<T>(x0 * c.y + x1 * c.x);
        }
        *reinterpret_cast<V*>(dst + off[u]) = val[u];
      } else if (!in_place) {
        *reinterpret_cast<V*>(dst + off[u]) = val[u];
      }
    }
  }
}

// Rotated query sets: qd[s][h][m][:] = R(-angle) q[g][m][h][:].
__global__ void rotate_queries_kernel(const float* __restrict__ q, int M, int H, int Dh,
                                      const int32_t* __restrict__ qset_group, const int32_t* __restrict__ qset_cs,
                                      int n_qsets, const float2* __restrict__ cs, float* __restrict__ qd,
                                      __nv_bfloat16* __restrict__ qd3) {
  int half = Dh / 2;
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)n_qsets * H * M * half;
  if (t >= total) return;
  int p = (int)(t % half);
  int64_t r = t / half;
  int m = (int)(r % M);
  r /= M;
  int h = (int)(r % H);
  int s = (int)(r / H);
  int g = qset_group[s];
  const float* src = q + (((int64_t)g * M + m) * H + h) * Dh + 2 * p;
  float x0 = src[0], x1 = src[1];
  int ci = qset_cs[s];
  float y0 = x0, y1 = x1;
  if (ci >= 0) {
    float2 c = cs[(int64_t)ci * half + p];
    y0 = x0 * c.x + x1 * c.y;   // rotation by -angle
    y1 = -x0 * c.y + x1 * c.x;
  }
  const int64_t o = (((int64_t)s * H + h) * M + m) * Dh + 2 * p;
  qd[o] = y0;
  qd[o + 1] = y1;
  if (qd3) {  // [n_qsets][3][H][M][Dh] split terms for the tensor-core scorer
    const int64_t plane = (int64_t)H * M * Dh;
    const int64_t o3 = ((int64_t)s * 3) * plane + (o - (int64_t)s * plane);
    __nv_bfloat16 a0, a1, a2, b0, b1, b2;
    split3(y0, a0, a1, a2);
    split3(y1, b0, b1, b2);
    qd3[o3] = a0;
    qd3[o3 + 1] = b0;
    qd3[o3 + plane] = a1;
    qd3[o3 + plane + 1] = b1;
    qd3[o3 + 2 * plane] = a2;
    qd3[o3 + 2 * plane + 1] = b2;
  }
}

// Fresh q/k/v epilogue: rope q and k at the rows' positions, write q
// compact, scatter k and v into the destination rows.
template <typename TIn, typename TOut>
__global__ void qkv_rope_scatter_kernel(const TIn* __restrict__ qkv, int n_parts, int64_t part_stride, int rows,
                                        int H, int Hkv, int Dh, const float2* __restrict__ cs,
                                        TOut* __restrict__ q_out, TOut* __restrict__ k_dst,
                                        TOut* __restrict__ v_dst, const int64_t* __restrict__ dst_rows) {
  const int half = Dh / 2;
  const int width_pairs = (H + 2 * Hkv) * half;
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)rows * width_pairs) return;
  int r = (int)(t / width_pairs);
  int c = (int)(t % width_pairs);  // pair column
  const TIn* src = qkv + (int64_t)r * (H + 2 * Hkv) * Dh + 2 * c;
  float x0 = 0.f, x1 = 0.f;
  for (int p = 0; p < n_parts; ++p) {
    x0 += to_f32(src[p * part_stride]);
    x1 += to_f32(src[p * part_stride + 1]);
  }
  int head = c / half, pi = c % half;
  if (head < H + Hkv) {  // q or k: rotate
    float2 a = cs[(int64_t)r * half + pi];
    float y0 = x0 * a.x - x1 * a.y;
    float y1 = x0 * a.y + x1 * a.x;
    x0 = y0;
    x1 = y1;
  }
  int64_t drow = dst_rows ? dst_rows[r] : r;
  TOut* d;
  if (head < H) {
    if (!q_out) return;
    d = q_out + ((int64_t)r * H + head) * Dh + 2 * pi;
  } else if (head < H + Hkv) {
    d = k_dst + (drow * Hkv + (head - H)) * Dh + 2 * pi;
  } else {
    d = v_dst + (drow * Hkv + (head - H - Hkv)) * Dh + 2 * pi;
  }
  d[0] = from_f32<TOut>(x0);
  d[1] = from_f32<TOut>(x1);
}

// Vectorised variant (Dh % 8 == 0): one thread = 8 consecutive elements
// (4 pairs) of one head row.
template <typename TIn, typename TOut>
__global__ void qkv_rope_scatter_vec_kernel(const TIn* __restrict__ qkv, int n_parts, int64_t part_stride, int rows,
                                            int H, int Hkv, int Dh, const float2* __restrict__ cs,
                                            TOut* __restrict__ q_out, TOut* __restrict__ k_dst,
                                            TOut* __restrict__ v_dst, const int64_t* __restrict__ dst_rows) {
  const int half = Dh / 2;
  const int vpr = (H + 2 * Hkv) * Dh / 8;  // vectors per row
  const int64_t total = (int64_t)rows * vpr;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(t / vpr);
    const int c8 = (int)(t - (int64_t)r * vpr) * 8;  // element column
    const int head = c8 / Dh, e0 = c8 % Dh;
    if (head < H && !q_out) continue;
    float x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = 0.f;
    const TIn* src = qkv + (int64_t)r * (H + 2 * Hkv) * Dh + c8;
    for (int p = 0; p < n_parts; ++p) {
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] += to_f32(src[p * part_stride + u]);
    }
    if (head < H + Hkv) {
      const float2* c = cs + (int64_t)r * half + e0 / 2;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float2 a = c[u];
        float y0 = x[2 * u] * a.x - x[2 * u + 1] * a.y;
        float y1 = x[2 * u] * a.y + x[2 * u + 1] * a.x;
        x[2 * u] = y0;
        x[2 * u + 1] = y1;
      }
    }
    const int64_t drow = dst_rows ? dst_rows[r] : r;
    TOut* d;
    if (head < H) d = q_out + ((int64_t)r * H + head) * Dh + e0;
    else if (head < H + Hkv) d = k_dst + (drow * Hkv + (head - H)) * Dh + e0;
    else d = v_dst + (drow * Hkv + (head - H - Hkv)) * Dh + e0;
#pragma unroll
    for (int u = 0; u < 8; ++u) d[u] = from_f32<TOut>(x[u]);
  }
}

}  // namespace ifkv

using namespace ifkv;

extern "C" int ifkv_rope_table(const int64_t* pos, int n, int d_head, double rope_base, float* cs, void* stream) {
  IFKV_CHECK_ARG(d_head >= 2 && d_head % 2 == 0, "rope_table: d_head must be even, got %d", d_head);
  IFKV_CHECK_ARG(n >= 0 && rope_base > 0, "rope_table: bad n=%d / base", n);
  if (n == 0) return IFKV_OK;
  int half = d_head / 2;
  int64_t total = (int64_t)n * half;
  rope_table_kernel<<<(unsigned)((total + 255) / 256), 256, 0, as_stream(stream)>>>(pos, n, half, rope_base,
                                                                                   reinterpret_cast<float2*>(cs));
  IFKV_LAUNCH_CHECK("rope_table");
  return IFKV_OK;
}

extern "C" int ifkv_rotate_rows(int dtype, const void* src, void* dst, int64_t layer_stride, int n_layers,
                                int n_rows, int heads, int d_head, const int32_t* row_table, const float* cs,
                                void* stream) {
  IFKV_CHECK_ARG(dtype == IFKV_F32 || dtype == IFKV_BF16, "rotate_rows: bad dtype %d", dtype);
  IFKV_CHECK_ARG(d_head % 2 == 0 && heads > 0, "rotate_rows: bad head shape");
  if (n_layers <= 0 || n_rows <= 0) return IFKV_OK;
  const int vec = dtype == IFKV_F32 ? 4 : 8;
  IFKV_CHECK_ARG(d_head % vec == 0, "rotate_rows: d_head %d must be a multiple of %d", d_head, vec);
  IFKV_CHECK_ARG(((uintptr_t)src % 16 == 0) && ((uintptr_t)dst % 16 == 0) && layer_stride % vec == 0,
                 "rotate_rows: slab must be 16-byte aligned");
  int vecs_per_head = d_head / vec;
  int vecs_per_row = heads * vecs_per_head;
  int64_t total = (int64_t)n_layers * n_rows * vecs_per_row;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  constexpr int kUnroll = 4;
  int64_t want = (total + 256 * kUnroll - 1) / (256 * kUnroll);
  int64_t cap = (int64_t)sms * 8;  // 8 x 256-thread CTAs resident per SM
  unsigned grid = (unsigned)(want < cap ? want : cap);
  if (grid == 0) grid = 1;
  bool in_place = src == dst;
  auto tab = reinterpret_cast<const float2*>(cs);
  if (dtype == IFKV_BF16)
    rotate_rows_kernel<__nv_bfloat16, kUnroll><<<grid, 256, 0, as_stream(stream)>>>(
        (const __nv_bfloat16*)src, (__nv_bfloat16*)dst, layer_stride, n_rows, vecs_per_row, vecs_per_head, total,
        row_table, tab, d_head / 2, in_place);
  else
    rotate_rows_kernel<float, kUnroll><<<grid, 256, 0, as_stream(stream)>>>(
        (const float*)src, (float*)dst, layer_stride, n_rows, vecs_per_row, vecs_per_head, total, row_table, tab,
        d_head / 2, in_place);
  IFKV_LAUNCH_CHECK("rotate_rows");
  return IFKV_OK;
}

extern "C" int ifkv_rotate_queries(const float* q, int G, int M, int H, int Dh, const int32_t* qset_group,
                                   const int32_t* qset_cs, int n_qsets, const float* cs, float* qd, void* qd3,
                                   void* stream) {
  IFKV_CHECK_ARG(Dh % 2 == 0 && G > 0 && M > 0 && H > 0, "rotate_queries: bad shape");
  if (n_qsets <= 0) return IFKV_OK;
  int64_t total = (int64_t)n_qsets * H * M * (Dh / 2);
  rotate_queries_kernel<<<(unsigned)((total + 255) / 256), 256, 0, as_stream(stream)>>>(
      q, M, H, Dh, qset_group, qset_cs, n_qsets, reinterpret_cast<const float2*>(cs), qd,
      reinterpret_cast<__nv_bfloat16*>(qd3));
  IFKV_LAUNCH_CHECK("rotate_queries");
  return IFKV_OK;
}

extern "C" int ifkv_qkv_rope_scatter(const void* qkv, int qkv_dtype, int n_parts, int rows, int H, int Hkv, int Dh,
                                     const float* cs, int out_dtype, void* q_out, void* k_dst, void* v_dst,
                                     const int64_t* dst_rows, void* stream) {
  IFKV_CHECK_ARG(Dh % 2 == 0 && H % Hkv == 0 && n_parts >= 1, "qkv_rope_scatter: bad shape");
  IFKV_CHECK_ARG(qkv_dtype == IFKV_F32 || qkv_dtype == IFKV_BF16, "qkv_rope_scatter: bad qkv dtype");
  IFKV_CHECK_ARG(out_dtype == IFKV_F32 || out_dtype == IFKV_BF16, "qkv_rope_scatter: bad out dtype");
  if (rows <= 0) return IFKV_OK;
  int64_t total = (int64_t)rows * (H + 2 * Hkv) * (Dh / 2);
  int64_t part_stride = (int64_t)rows * (H + 2 * Hkv) * Dh;
  unsigned grid = (unsigned)((total + 255) / 256);
  auto c = reinterpret_cast<const float2*>(cs);
  cudaStream_t s = as_stream(stream);
  const bool vec = Dh % 8 == 0;
  if (vec) {
    int64_t nv = (int64_t)rows * (H + 2 * Hkv) * Dh / 8;
    int64_t want = (nv + 255) / 256;
    grid = (unsigned)(want < 148 * 16 ? want : 148 * 16);
  }
#define IFKV_QKV_LAUNCH(TI, TO)                                                                                   \
  if (vec)                                                                                                        \
    qkv_rope_scatter_vec_kernel<TI, TO><<<grid, 256, 0, s>>>((const TI*)qkv, n_parts, part_stride, rows, H, Hkv,   \
                                                             Dh, c, (TO*)q_out, (TO*)k_dst, (TO*)v_dst, dst_rows); \
  else                                                                                                            \
    qkv_rope_scatter_kernel<TI, TO><<<grid, 256, 0, s>>>((const TI*)qkv, n_parts, part_stride, rows, H, Hkv, Dh, c, \
                                                         (TO*)q_out, (TO*)k_dst, (TO*)v_dst, dst_rows)
  if (qkv_dtype == IFKV_F32 && out_dtype == IFKV_F32) IFKV_QKV_LAUNCH(float, float);
  else if (qkv_dtype == IFKV_F32) IFKV_QKV_LAUNCH(float, __nv_bfloat16);
  else if (out_dtype == IFKV_F32) IFKV_QKV_LAUNCH(__nv_bfloat16, float);
  else IFKV_QKV_LAUNCH(__nv_bfloat16, __nv_bfloat16);
#undef IFKV_QKV_LAUNCH
  IFKV_LAUNCH_CHECK("qkv_rope_scatter");
  return IFKV_OK;
}
