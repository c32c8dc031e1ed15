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
// One warp per (layer, row) pair, two rows in flight per warp: every lane
// issues all its 16-byte loads (8 bf16 / 4 fp32 = 4 / 2 RoPE pairs per
// vector) before rotating and storing.  The row's cos/sin come from a small
// fp64-derived table (one entry per distinct delta) that stays in L1.  Rows
// whose table entry is negative (delta 0) are skipped in place or copied
// bit-exactly out of place.
template <typename T, int kVpl>
__global__ void __launch_bounds__(256) rotate_rows_kernel(const T* __restrict__ src, T* __restrict__ dst,
                                                          int64_t layer_stride, int n_rows, int n_layers,
                                                          int vecs_per_head, const int32_t* __restrict__ row_table,
                                                          const float2* __restrict__ cs, int half, bool in_place) {
  constexpr int kVec = 16 / sizeof(T);
  constexpr int kPairs = kVec / 2;
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  const int64_t total = (int64_t)n_layers * n_rows;
  const int64_t row_elems = (int64_t)kVpl * 32 * kVec;
  // pair offset of this lane's vectors inside the head (same for all kVpl)
  const int pair0 = (lane % vecs_per_head) * kPairs;
  for (int64_t r0 = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r0 < total; r0 += 2 * (int64_t)warps) {
    uint4 val[2][kVpl];
    int tab[2];
    int64_t base[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int64_t r = r0 + (int64_t)q * warps;
      tab[q] = -2;
      if (r < total) {
        const int layer = (int)(r / n_rows);
        const int row = (int)(r - (int64_t)layer * n_rows);
        tab[q] = row_table[row];
        base[q] = layer * layer_stride + row * row_elems;
        if (tab[q] >= 0 || !in_place) {
#pragma unroll
          for (int u = 0; u < kVpl; ++u)
            val[q][u] = *reinterpret_cast<const uint4*>(src + base[q] + (int64_t)(lane + 32 * u) * kVec);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (tab[q] == -2 || (tab[q] < 0 && in_place)) continue;
      if (tab[q] >= 0) {
        float2 c[kPairs];
#pragma unroll
        for (int p = 0; p < kPairs; ++p) c[p] = __ldg(cs + (int64_t)tab[q] * half + pair0 + p);
#pragma unroll
        for (int u = 0; u < kVpl; ++u) {
          T* e = reinterpret_cast<T*>(&val[q][u]);
#pragma unroll
          for (int p = 0; p < kPairs; ++p) {
            const float2 y = rot_pair(to_f32(e[2 * p]), to_f32(e[2 * p + 1]), c[p]);
            e[2 * p] = from_f32<T>(y.x);
            e[2 * p + 1] = from_f32<T>(y.y);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kVpl; ++u)
        *reinterpret_cast<uint4*>(dst + base[q] + (int64_t)(lane + 32 * u) * kVec) = val[q][u];
    }
  }
}

// Generic fallback: one thread per 16-byte vector (rows not a multiple of
// 32 vectors, e.g. the tiny parity configs).
template <typename T>
__global__ void rotate_rows_generic_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t layer_stride,
                                           int64_t n_rows, int vecs_per_row, int vecs_per_head, int64_t total_vecs,
                                           const int32_t* __restrict__ row_table, const float2* __restrict__ cs,
                                           int half, bool in_place) {
  constexpr int kVec = 16 / sizeof(T);
  constexpr int kPairs = kVec / 2;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total_vecs;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row_all = g / vecs_per_row;
    const int vin = (int)(g - row_all * vecs_per_row);
    const int64_t layer = row_all / n_rows;
    const int64_t row = row_all - layer * n_rows;
    const int t = row_table[row];
    if (t < 0 && in_place) continue;
    const int64_t off = layer * layer_stride + row * (int64_t)vecs_per_row * kVec + (int64_t)vin * kVec;
    uint4 val = *reinterpret_cast<const uint4*>(src + off);
    if (t >= 0) {
      T* e = reinterpret_cast<T*>(&val);
      const int p0 = t * half + (vin % vecs_per_head) * kPairs;
#pragma unroll
      for (int p = 0; p < kPairs; ++p) {
        float2 c = __ldg(cs + p0 + p);
        float x0 = to_f32(e[2 * p]), x1 = to_f32(e[2 * p + 1]);
        e[2 * p] = from_f32<T>(x0 * c.x - x1 * c.y);
        e[2 * p + 1] = from_f32<T>(x0 * c.y + x1 * c.x);
      }
    }
    *reinterpret_cast<uint4*>(dst + off) = val;
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

// Prompt-row q/k/v of the scoring pass in one pass (replaces
// qkv_rope_scatter + rotate_queries there): the n_parts fp32 GEMM partials
// summed in a fixed order, q and k rotated to the prompt positions (cs), k/v
// written compact fp32 [rows][Hkv][Dh], and q rotated once more by -delta for
// each of its group's query sets (q . R(d) k == (R(-d) q) . k, the context
// keys stay as stored) into qd [s][H][M][Dh] (+ the bf16 split terms qd3).
// Group g's query sets: qs_list[qs_begin[g] .. qs_begin[g+1]).
constexpr int kQsetsPerThread = 4;
__global__ void prompt_qkv_kernel(const float* __restrict__ qkv, int n_parts, int64_t part_stride, int G, int M,
                                  int H, int Hkv, int Dh, const float2* __restrict__ cs,
                                  const int32_t* __restrict__ qs_begin, const int32_t* __restrict__ qs_list,
                                  const int32_t* __restrict__ qset_cs, const float2* __restrict__ cs_delta,
                                  float* __restrict__ kp, float* __restrict__ vp, float* __restrict__ qd,
                                  __nv_bfloat16* __restrict__ qd3) {
  pdl_trigger();
  pdl_wait();
  const int half = Dh / 2;
  const int width_pairs = (H + 2 * Hkv) * half;
  const int rows = G * M;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)rows * width_pairs) return;
  const int r = (int)(t / width_pairs), c = (int)(t % width_pairs);
  const int head = c / half, pi = c % half;
  const int g = r / M, m = r % M;
  // blockIdx.y: this thread's slab of kQsetsPerThread of the group's query sets
  const int k0 = qs_begin[g] + blockIdx.y * kQsetsPerThread;
  const int k1 = min(qs_begin[g + 1], k0 + kQsetsPerThread);
  if (head >= H ? blockIdx.y != 0 : k0 >= k1) return;  // nothing to write: skip the loads
  const float* src = qkv + (int64_t)r * (H + 2 * Hkv) * Dh + 2 * c;
  float x0 = 0.f, x1 = 0.f;
  for (int p = 0; p < n_parts; ++p) {
    x0 += src[p * part_stride];
    x1 += src[p * part_stride + 1];
  }
  if (head < H + Hkv) {
    const float2 a = cs[(int64_t)r * half + pi];
    const float y0 = x0 * a.x - x1 * a.y, y1 = x0 * a.y + x1 * a.x;
    x0 = y0;
    x1 = y1;
  }
  if (head >= H) {
    float* d = (head < H + Hkv ? kp + ((int64_t)r * Hkv + (head - H)) * Dh
                               : vp + ((int64_t)r * Hkv + (head - H - Hkv)) * Dh) + 2 * pi;
    d[0] = x0;
    d[1] = x1;
    return;
  }
  const int64_t plane = (int64_t)H * M * Dh;
  for (int k = k0; k < k1; ++k) {
    const int s = qs_list[k], ci = qset_cs[s];
    float y0 = x0, y1 = x1;
    if (ci >= 0) {
      const float2 a = cs_delta[(int64_t)ci * half + pi];
      y0 = x0 * a.x + x1 * a.y;  // rotation by -angle
      y1 = -x0 * a.y + x1 * a.x;
    }
    const int64_t o = (((int64_t)s * H + head) * M + m) * Dh + 2 * pi;
    if (!qd3 || ci < 0) {  // fp32 sets: the SIMT kernels' input (tensor-core path: only the prompt's own, delta 0)
      qd[o] = y0;
      qd[o + 1] = y1;
    }
    if (qd3) {  // [n_qsets][3][H][M][Dh]
      const int64_t o3 = ((int64_t)s * 3) * plane + (o - (int64_t)s * plane);
      __nv_bfloat16 a0, a1, a2, b0, b1, b2;
      split3(y0, a0, a1, a2);
      split3(y1, b0, b1, b2);
      reinterpret_cast<__nv_bfloat162*>(qd3 + o3)[0] = __halves2bfloat162(a0, b0);
      reinterpret_cast<__nv_bfloat162*>(qd3 + o3 + plane)[0] = __halves2bfloat162(a1, b1);
      reinterpret_cast<__nv_bfloat162*>(qd3 + o3 + 2 * plane)[0] = __halves2bfloat162(a2, b2);
    }
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

__device__ __forceinline__ void load8_add(const float* p, float* x) {
  float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  x[0] += a.x; x[1] += a.y; x[2] += a.z; x[3] += a.w; x[4] += b.x; x[5] += b.y; x[6] += b.z; x[7] += b.w;
}
__device__ __forceinline__ void load8_add(const __nv_bfloat16* p, float* x) {
  uint4 v = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float2 f = __bfloat1622float2(h[k]);
    x[2 * k] += f.x;
    x[2 * k + 1] += f.y;
  }
}
__device__ __forceinline__ void store8(float* d, const float* x) {
  *reinterpret_cast<float4*>(d) = make_float4(x[0], x[1], x[2], x[3]);
  *reinterpret_cast<float4*>(d + 4) = make_float4(x[4], x[5], x[6], x[7]);
}
__device__ __forceinline__ void store8(__nv_bfloat16* d, const float* x) {
  uint4 v;
  uint32_t* o = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    __nv_bfloat162 y = __floats2bfloat162_rn(x[2 * k], x[2 * k + 1]);
    o[k] = *reinterpret_cast<uint32_t*>(&y);
  }
  *reinterpret_cast<uint4*>(d) = v;
}

// Vectorised variant (Dh % 8 == 0): one CTA per row (no index division);
// thread = 8 consecutive elements (4 pairs) of one head row, up to kU such
// vectors per thread with all loads issued before any store.
template <typename TIn, typename TOut, int kU>
__global__ void __launch_bounds__(256) qkv_rope_scatter_vec_kernel(
    const TIn* __restrict__ qkv, int n_parts, int64_t part_stride, int rows, int H, int Hkv, int Dh,
    const float2* __restrict__ cs, TOut* __restrict__ q_out, TOut* __restrict__ k_dst, TOut* __restrict__ v_dst,
    const int64_t* __restrict__ dst_rows) {
  const int half = Dh / 2;
  const int vpr = (H + 2 * Hkv) * Dh / 8;  // vectors per row
  const int r = blockIdx.x;
  const int64_t drow = dst_rows ? dst_rows[r] : r;
  const TIn* src = qkv + (int64_t)r * (H + 2 * Hkv) * Dh;
  const float2* csr = cs + (int64_t)r * half;
  const int q_end = q_out ? 0 : H * Dh / 8;  // vectors below q_end are skipped (no q output)
  for (int v0 = q_end + threadIdx.x; v0 < vpr; v0 += kU * blockDim.x) {
    float x[kU][8];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int v = v0 + u * blockDim.x;
#pragma unroll
      for (int e = 0; e < 8; ++e) x[u][e] = 0.f;
      if (v < vpr)
        for (int p = 0; p < n_parts; ++p) load8_add(src + p * part_stride + v * 8, x[u]);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int v = v0 + u * blockDim.x;
      if (v >= vpr) break;
      const int c8 = v * 8, head = c8 / Dh, e0 = c8 - head * Dh;
      if (head < H + Hkv) {
        const float4* c4 = reinterpret_cast<const float4*>(csr + e0 / 2);
        const float4 ab = __ldg(c4), cd = __ldg(c4 + 1);
        const float2 a[4] = {make_float2(ab.x, ab.y), make_float2(ab.z, ab.w), make_float2(cd.x, cd.y),
                             make_float2(cd.z, cd.w)};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float y0 = x[u][2 * q] * a[q].x - x[u][2 * q + 1] * a[q].y;
          const float y1 = x[u][2 * q] * a[q].y + x[u][2 * q + 1] * a[q].x;
          x[u][2 * q] = y0;
          x[u][2 * q + 1] = y1;
        }
      }
      TOut* d;
      if (head < H)
        d = q_out + ((int64_t)r * H + head) * Dh + e0;
      else if (head < H + Hkv)
        d = k_dst + (drow * Hkv + (head - H)) * Dh + e0;
      else
        d = v_dst + (drow * Hkv + (head - H - Hkv)) * Dh + e0;
      store8(d, x[u]);
    }
  }
}

// Grid-stride variant (A/B, IFKV_SCATTER_ROW=0): one thread = 8 consecutive
// elements (4 pairs) of one head row per iteration.
template <typename TIn, typename TOut>
__global__ void qkv_rope_scatter_strided_kernel(const TIn* __restrict__ qkv, int n_parts, int64_t part_stride, int rows,
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
    for (int p = 0; p < n_parts; ++p) load8_add(src + p * part_stride, x);
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
    store8(d, x);
  }
}

// bf16 -> bf16, one part, Dh = 128 (the recompute loop): one pass, two
// 16-byte vectors per thread (both loads issued first), 32-bit indexing,
// cos/sin as two 16-byte loads.
__global__ void __launch_bounds__(256) qkv_rope_scatter_bf16_kernel(
    const __nv_bfloat16* __restrict__ qkv, int total, int H, int Hkv, const float2* __restrict__ cs,
    __nv_bfloat16* __restrict__ q_out, __nv_bfloat16* __restrict__ k_dst, __nv_bfloat16* __restrict__ v_dst,
    const int64_t* __restrict__ dst_rows) {
  const int vpr = (H + 2 * Hkv) * 16;  // 16-byte vectors per row (Dh = 128: 16 per head)
  const int t0 = blockIdx.x * 512 + threadIdx.x;
  uint4 val[2];
  int r[2], c[2];
  bool on[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int t = t0 + u * 256;
    r[u] = t / vpr;
    c[u] = t - r[u] * vpr;
    on[u] = t < total && (q_out || c[u] >= H * 16);
    if (on[u]) val[u] = *reinterpret_cast<const uint4*>(qkv + (int64_t)t * 8);
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    if (!on[u]) continue;
    const int head = c[u] >> 4, e0 = (c[u] & 15) * 8;
    if (head < H + Hkv) {
      const float4* c4 = reinterpret_cast<const float4*>(cs + (int64_t)r[u] * 64 + e0 / 2);
      const float4 ab = __ldg(c4), cd = __ldg(c4 + 1);
      const float2 a[4] = {make_float2(ab.x, ab.y), make_float2(ab.z, ab.w), make_float2(cd.x, cd.y),
                           make_float2(cd.z, cd.w)};
      __nv_bfloat162* e = reinterpret_cast<__nv_bfloat162*>(&val[u]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 x = __bfloat1622float2(e[q]);
        e[q] = __floats2bfloat162_rn(x.x * a[q].x - x.y * a[q].y, x.x * a[q].y + x.y * a[q].x);
      }
    }
    __nv_bfloat16* d;
    if (head < H) {
      d = q_out + ((int64_t)r[u] * H + head) * 128 + e0;
    } else {
      const int64_t drow = dst_rows ? dst_rows[r[u]] : r[u];
      d = head < H + Hkv ? k_dst + (drow * Hkv + (head - H)) * 128 + e0
                         : v_dst + (drow * Hkv + (head - H - Hkv)) * 128 + e0;
    }
    *reinterpret_cast<uint4*>(d) = val[u];
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
  const int vecs_per_head = d_head / vec;
  const int vecs_per_row = heads * vecs_per_head;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool in_place = src == dst;
  auto tab = reinterpret_cast<const float2*>(cs);
  cudaStream_t st = as_stream(stream);
  const int64_t rows = (int64_t)n_layers * n_rows;
  const bool warp_rows = vecs_per_row % 32 == 0 && 32 % vecs_per_head == 0 && vecs_per_row / 32 <= 8;
  if (warp_rows) {
    const int64_t want = (rows + 15) / 16;  // 8 warps x 2 rows per CTA iteration
    const unsigned grid = (unsigned)(want < (int64_t)sms * 8 ? (want > 0 ? want : 1) : (int64_t)sms * 8);
    const int vpl = vecs_per_row / 32;
#define IFKV_ROT(T, V)                                                                                     \
  rotate_rows_kernel<T, V><<<grid, 256, 0, st>>>((const T*)src, (T*)dst, layer_stride, n_rows, n_layers, \
                                                  vecs_per_head, row_table, tab, d_head / 2, in_place)
    if (dtype == IFKV_BF16) {
      if (vpl == 4) IFKV_ROT(__nv_bfloat16, 4);
      else if (vpl == 2) IFKV_ROT(__nv_bfloat16, 2);
      else if (vpl == 1) IFKV_ROT(__nv_bfloat16, 1);
      else if (vpl == 8) IFKV_ROT(__nv_bfloat16, 8);
      else goto generic;
    } else {
      if (vpl == 8) IFKV_ROT(float, 8);
      else if (vpl == 4) IFKV_ROT(float, 4);
      else if (vpl == 2) IFKV_ROT(float, 2);
      else if (vpl == 1) IFKV_ROT(float, 1);
      else goto generic;
    }
#undef IFKV_ROT
    IFKV_LAUNCH_CHECK("rotate_rows");
    return IFKV_OK;
  }
generic : {
  const int64_t total = rows * vecs_per_row;
  const int64_t want = (total + 255) / 256;
  const unsigned grid = (unsigned)(want < (int64_t)sms * 8 ? want : (int64_t)sms * 8);
  if (dtype == IFKV_BF16)
    rotate_rows_generic_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)src, (__nv_bfloat16*)dst,
                                                                    layer_stride, n_rows, vecs_per_row, vecs_per_head,
                                                                    total, row_table, tab, d_head / 2, in_place);
  else
    rotate_rows_generic_kernel<float><<<grid, 256, 0, st>>>((const float*)src, (float*)dst, layer_stride, n_rows,
                                                            vecs_per_row, vecs_per_head, total, row_table, tab,
                                                            d_head / 2, in_place);
  IFKV_LAUNCH_CHECK("rotate_rows");
  return IFKV_OK;
}
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

extern "C" int ifkv_prompt_qkv(const float* qkv, int n_parts, int G, int M, int H, int Hkv, int Dh, const float* cs,
                               const int32_t* qs_begin, const int32_t* qs_list, const int32_t* qset_cs,
                               int max_group_qsets, const float* cs_delta, float* kp, float* vp, float* qd, void* qd3,
                               void* stream) {
  IFKV_CHECK_ARG(Dh % 2 == 0 && Hkv > 0 && H > 0 && H % Hkv == 0 && n_parts >= 1 && G > 0 && M > 0,
                 "prompt_qkv: bad shape");
  IFKV_CHECK_ARG(max_group_qsets >= 1, "prompt_qkv: max_group_qsets must be >= 1");
  const int64_t total = (int64_t)G * M * (H + 2 * Hkv) * (Dh / 2);
  const int64_t part_stride = (int64_t)G * M * (H + 2 * Hkv) * Dh;
  // grid.y: slabs of kQsetsPerThread query sets (max_group_qsets bounds every
  // group's count; slabs past a group's end return before loading)
  const dim3 grid((unsigned)((total + 255) / 256),
                  (unsigned)((max_group_qsets + kQsetsPerThread - 1) / kQsetsPerThread));
  IFKV_CUDA_CALL(launch_pdl(prompt_qkv_kernel, grid, dim3(256), 0, as_stream(stream), qkv, n_parts, part_stride, G, M,
                            H, Hkv, Dh, reinterpret_cast<const float2*>(cs), qs_begin, qs_list, qset_cs,
                            reinterpret_cast<const float2*>(cs_delta), kp, vp, qd,
                            reinterpret_cast<__nv_bfloat16*>(qd3)),
                 "prompt_qkv: launch");
  IFKV_LAUNCH_CHECK("prompt_qkv");
  return IFKV_OK;
}

extern "C" int ifkv_qkv_rope_scatter(const void* qkv, int qkv_dtype, int n_parts, int rows, int H, int Hkv, int Dh,
                                     const float* cs, int out_dtype, void* q_out, void* k_dst, void* v_dst,
                                     const int64_t* dst_rows, void* stream) {
  IFKV_CHECK_ARG(Dh % 2 == 0 && Hkv > 0 && H >= 0 && H % Hkv == 0 && n_parts >= 1, "qkv_rope_scatter: bad shape");
  IFKV_CHECK_ARG(qkv_dtype == IFKV_F32 || qkv_dtype == IFKV_BF16, "qkv_rope_scatter: bad qkv dtype");
  IFKV_CHECK_ARG(out_dtype == IFKV_F32 || out_dtype == IFKV_BF16, "qkv_rope_scatter: bad out dtype");
  if (rows <= 0) return IFKV_OK;
  int64_t total = (int64_t)rows * (H + 2 * Hkv) * (Dh / 2);
  int64_t part_stride = (int64_t)rows * (H + 2 * Hkv) * Dh;
  unsigned grid = (unsigned)((total + 255) / 256);
  auto c = reinterpret_cast<const float2*>(cs);
  cudaStream_t s = as_stream(stream);
#ifndef IFKV_SCATTER_ROW
#define IFKV_SCATTER_ROW 0
#endif
  const bool row_kernel = IFKV_SCATTER_ROW && Dh % 8 == 0 && (H + 2 * Hkv) * Dh / 8 <= 4 * 256;
  const bool strided = !row_kernel && Dh % 8 == 0;
  if (row_kernel) {
    grid = (unsigned)rows;
  } else if (strided) {
    int64_t nv = (int64_t)rows * (H + 2 * Hkv) * Dh / 8;
    int64_t want = (nv + 255) / 256;
    grid = (unsigned)(want < 148 * 16 ? want : 148 * 16);
  }
#define IFKV_QKV_LAUNCH(TI, TO)                                                                                     \
  if (row_kernel)                                                                                                   \
    qkv_rope_scatter_vec_kernel<TI, TO, 4><<<grid, 256, 0, s>>>((const TI*)qkv, n_parts, part_stride, rows, H, Hkv, \
                                                                Dh, c, (TO*)q_out, (TO*)k_dst, (TO*)v_dst, dst_rows); \
  else if (strided)                                                                                                 \
    qkv_rope_scatter_strided_kernel<TI, TO><<<grid, 256, 0, s>>>((const TI*)qkv, n_parts, part_stride, rows, H, Hkv, \
                                                                 Dh, c, (TO*)q_out, (TO*)k_dst, (TO*)v_dst,        \
                                                                 dst_rows);                                        \
  else                                                                                                              \
    qkv_rope_scatter_kernel<TI, TO><<<grid, 256, 0, s>>>((const TI*)qkv, n_parts, part_stride, rows, H, Hkv, Dh, c,  \
                                                         (TO*)q_out, (TO*)k_dst, (TO*)v_dst, dst_rows)
#ifndef IFKV_SCATTER_BF16
#define IFKV_SCATTER_BF16 1
#endif
  const int64_t total16 = (int64_t)rows * (H + 2 * Hkv) * Dh / 8;
  if (IFKV_SCATTER_BF16 && qkv_dtype == IFKV_BF16 && out_dtype == IFKV_BF16 && n_parts == 1 && Dh == 128 &&
      total16 + 512 < (int64_t)INT32_MAX) {
    qkv_rope_scatter_bf16_kernel<<<(unsigned)((total16 + 511) / 512), 256, 0, s>>>(
        (const __nv_bfloat16*)qkv, (int)total16, H, Hkv, c, (__nv_bfloat16*)q_out, (__nv_bfloat16*)k_dst,
        (__nv_bfloat16*)v_dst, dst_rows);
    IFKV_LAUNCH_CHECK("qkv_rope_scatter");
    return IFKV_OK;
  }
  if (qkv_dtype == IFKV_F32 && out_dtype == IFKV_F32) IFKV_QKV_LAUNCH(float, float);
  else if (qkv_dtype == IFKV_F32) IFKV_QKV_LAUNCH(float, __nv_bfloat16);
  else if (out_dtype == IFKV_F32) IFKV_QKV_LAUNCH(__nv_bfloat16, float);
  else IFKV_QKV_LAUNCH(__nv_bfloat16, __nv_bfloat16);
#undef IFKV_QKV_LAUNCH
  IFKV_LAUNCH_CHECK("qkv_rope_scatter");
  return IFKV_OK;
}
