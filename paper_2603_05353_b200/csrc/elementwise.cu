// Fused elementwise kernels of the decoder block (reference model.py:278-294):
// residual add + RMSNorm with the GEMM-operand conversion fused in, SiLU-gate,
// embedding gather, fp32 -> 3 x bf16 operand split.
#include "common.cuh"

namespace ifkv {

template <typename TD>
__device__ __forceinline__ float sum_parts(const TD* p, int n_parts, int64_t part_stride, int64_t i) {
  float s = 0.f;
  for (int q = 0; q < n_parts; ++q) s += to_f32(p[q * part_stride + i]);
  return s;
}

__device__ __forceinline__ void store_mode(void* out, int mode, int64_t part_stride, int64_t i, float x) {
  if (mode == IFKV_OUT_F32) {
    reinterpret_cast<float*>(out)[i] = x;
  } else if (mode == IFKV_OUT_BF16) {
    reinterpret_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(x);
  } else {
    __nv_bfloat16 a, b, c;
    split3(x, a, b, c);
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(out);
    o[i] = a;
    o[part_stride + i] = b;
    o[2 * part_stride + i] = c;
  }
}

// Block-wide deterministic sum (fixed tree) for blockDim.x == kThreads.
template <int kThreads>
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = l < kThreads / 32 ? red[l] : 0.f;
  t = warp_sum(t);
  __syncthreads();
  return t;
}

// Vector helpers: 4 consecutive elements as fp32.
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ld4(const __nv_bfloat16* p) {
  uint2 u = *reinterpret_cast<const uint2*>(p);
  __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&u.x), b = *reinterpret_cast<__nv_bfloat162*>(&u.y);
  return make_float4(__low2float(a), __high2float(a), __low2float(b), __high2float(b));
}
__device__ __forceinline__ void add4(float4& a, const float4& b) {
  a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
}
__device__ __forceinline__ void store4_mode(void* out, int mode, int64_t part_stride, int64_t i, float4 x) {
  if (mode == IFKV_OUT_F32) {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + i) = x;
  } else if (mode == IFKV_OUT_BF16) {
    __nv_bfloat162 a = __floats2bfloat162_rn(x.x, x.y), b = __floats2bfloat162_rn(x.z, x.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + i) = u;
  } else {
    __nv_bfloat16 t[3][4];
    split3(x.x, t[0][0], t[1][0], t[2][0]);
    split3(x.y, t[0][1], t[1][1], t[2][1]);
    split3(x.z, t[0][2], t[1][2], t[2][2]);
    split3(x.w, t[0][3], t[1][3], t[2][3]);
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(out);
#pragma unroll
    for (int k = 0; k < 3; ++k) *reinterpret_cast<uint2*>(o + k * part_stride + i) = *reinterpret_cast<uint2*>(t[k]);
  }
}

// One CTA per row; each thread owns 4-wide vectors (d % 4 == 0), kept in
// registers between the residual add and the normalisation
// (d <= 8 * 4 * kThreads).  128-thread CTAs for d <= 4096: 16 rows in flight
// per SM instead of 8 (the kernel is load-latency bound).
template <typename TD, int kThreads, int kMaxVec = 8>
__global__ void __launch_bounds__(kThreads) add_rmsnorm_kernel(float* __restrict__ h, const TD* __restrict__ delta,
                                                               int n_parts, const float* __restrict__ gain, int rows,
                                                               int d, int mode, void* __restrict__ out) {
  __shared__ float red[kThreads / 32];
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  float* hr = h + (int64_t)r * d;
  const int64_t pstride = (int64_t)rows * d;
  float4 x[kMaxVec];
  float ss = 0.f;
#pragma unroll
  for (int u = 0; u < kMaxVec; ++u) {
    const int i = (u * kThreads + threadIdx.x) * 4;
    if (i < d) x[u] = ld4(hr + i);
  }
  if (n_parts > 0) {
#pragma unroll
    for (int u = 0; u < kMaxVec; ++u) {
      const int i = (u * kThreads + threadIdx.x) * 4;
      if (i < d) {
        for (int q = 0; q < n_parts; ++q) add4(x[u], ld4(delta + q * pstride + (int64_t)r * d + i));
        *reinterpret_cast<float4*>(hr + i) = x[u];
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kMaxVec; ++u) {
    const int i = (u * kThreads + threadIdx.x) * 4;
    if (i < d) ss += x[u].x * x[u].x + x[u].y * x[u].y + x[u].z * x[u].z + x[u].w * x[u].w;
  }
  if (!out) return;
  float ms = block_sum<kThreads>(ss, red) / (float)d;
  float den = sqrtf(ms + 1e-6f);
#pragma unroll
  for (int u = 0; u < kMaxVec; ++u) {
    const int i = (u * kThreads + threadIdx.x) * 4;
    if (i < d) {
      float4 g = ld4(gain + i);
      float4 y = make_float4(x[u].x / den * g.x, x[u].y / den * g.y, x[u].z / den * g.z, x[u].w / den * g.w);
      store4_mode(out, mode, pstride, (int64_t)r * d + i, y);
    }
  }
}

// Persistent variant for d == 4 * 4 * 256 = 4096 rows (the Llama-width
// recompute loop): a CTA walks rows r, r + grid, ... and issues the loads of
// its next row before reducing and storing the current one, so HBM reads stay
// in flight across the reduction barrier.
template <typename TD>
__global__ void __launch_bounds__(256) add_rmsnorm_pf_kernel(float* __restrict__ h, const TD* __restrict__ delta,
                                                             int n_parts, const float* __restrict__ gain, int rows,
                                                             int mode, void* __restrict__ out) {
  constexpr int d = 4096, kV = 4;
  __shared__ float red[2][8];
  pdl_trigger();
  pdl_wait();
  const int64_t pstride = (int64_t)rows * d;
  float4 g[kV];
#pragma unroll
  for (int u = 0; u < kV; ++u) g[u] = ld4(gain + (u * 256 + threadIdx.x) * 4);
  auto load = [&](int r, float4* x) {
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const int i = (u * 256 + threadIdx.x) * 4;
      x[u] = ld4(h + (int64_t)r * d + i);
      for (int q = 0; q < n_parts; ++q) add4(x[u], ld4(delta + q * pstride + (int64_t)r * d + i));
    }
  };
  float4 cur[kV], nxt[kV];
  int r = blockIdx.x;
  if (r < rows) load(r, cur);
  for (int it = 0; r < rows; r += gridDim.x, ++it) {
    const int rn = r + gridDim.x;
    if (rn < rows) load(rn, nxt);
    float ss = 0.f;
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const int i = (u * 256 + threadIdx.x) * 4;
      if (n_parts > 0) *reinterpret_cast<float4*>(h + (int64_t)r * d + i) = cur[u];
      ss += cur[u].x * cur[u].x + cur[u].y * cur[u].y + cur[u].z * cur[u].z + cur[u].w * cur[u].w;
    }
    if (out) {
      // block sum, double-buffered scratch: one barrier per row
      ss = warp_sum(ss);
      if ((threadIdx.x & 31) == 0) red[it & 1][threadIdx.x >> 5] = ss;
      __syncthreads();
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += red[it & 1][w];
      const float den = sqrtf(t / (float)d + 1e-6f);
#pragma unroll
      for (int u = 0; u < kV; ++u) {
        const int i = (u * 256 + threadIdx.x) * 4;
        float4 y = make_float4(cur[u].x / den * g[u].x, cur[u].y / den * g[u].y, cur[u].z / den * g[u].z,
                               cur[u].w / den * g[u].w);
        store4_mode(out, mode, pstride, (int64_t)r * d + i, y);
      }
    }
#pragma unroll
    for (int u = 0; u < kV; ++u) cur[u] = nxt[u];
  }
}

__device__ __forceinline__ float silu_f(float g) {
  if (g >= 0.f) return g / (1.f + expf(-g));
  float e = expf(g);
  return g * e / (1.f + e);
}

// 4-wide vectors over [rows][d_ff] (d_ff % 4 == 0).
template <typename T>
__global__ void silu_mul_kernel(const T* __restrict__ gu, int n_parts, int rows, int d_ff, int blk, int mode,
                                void* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int vpr = d_ff / 4;
  const int64_t nv = (int64_t)rows * vpr;
  const int64_t pstride = (int64_t)rows * 2 * d_ff;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nv; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / vpr;
    const int c = (int)(t - r * vpr) * 4;
    const T* base = gu + r * 2 * d_ff + (c / blk) * 2 * blk + c % blk;  // gate; up is blk further
    float4 g = ld4(base), u = ld4(base + blk);
    for (int q = 1; q < n_parts; ++q) {
      add4(g, ld4(base + q * pstride));
      add4(u, ld4(base + q * pstride + blk));
    }
    float4 y = make_float4(silu_f(g.x) * u.x, silu_f(g.y) * u.y, silu_f(g.z) * u.z, silu_f(g.w) * u.w);
    store4_mode(out, mode, (int64_t)rows * d_ff, r * d_ff + c, y);
  }
}

// silu for bf16 outputs: MUFU exp + reciprocal (the bf16 rounding of the
// product dominates their ~1e-7 relative error).
__device__ __forceinline__ float silu_fast(float g) { return g * __frcp_rn(1.f + __expf(-g)); }

// bf16 -> bf16 fast path (single part): 8 elements per thread-iteration,
// 16-byte loads of gate and up, 16-byte store.
__global__ void silu_mul_bf16x8_kernel(const __nv_bfloat16* __restrict__ gu, int rows, int d_ff, int blk,
                                       __nv_bfloat16* __restrict__ out) {
  const int vpr = d_ff / 8;
  const int64_t nv = (int64_t)rows * vpr;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nv; t += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(t / vpr);
    const int c = (int)(t - (int64_t)r * vpr) * 8;
    const __nv_bfloat16* base = gu + (int64_t)r * 2 * d_ff + (c / blk) * 2 * blk + c % blk;
    uint4 gv = *reinterpret_cast<const uint4*>(base);
    uint4 uv = *reinterpret_cast<const uint4*>(base + blk);
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gv);
    const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&uv);
    uint4 ov;
    uint32_t* o = reinterpret_cast<uint32_t*>(&ov);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 gf = __bfloat1622float2(g2[k]), uf = __bfloat1622float2(u2[k]);
      __nv_bfloat162 y = __floats2bfloat162_rn(silu_fast(gf.x) * uf.x, silu_fast(gf.y) * uf.y);
      o[k] = *reinterpret_cast<uint32_t*>(&y);
    }
    *reinterpret_cast<uint4*>(out + (int64_t)r * d_ff + c) = ov;
  }
}

// silu(g) = g * sigmoid(g) = 0.5 g (1 + tanh(g / 2)): one MUFU.TANH per
// element (tanh.approx.f32, rel. error ~2^-11, below the bf16 output rounding).
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// bf16 -> bf16, one part: one pass (no grid-stride loop), two 8-element
// vectors per thread with all four 16-byte loads issued first, 32-bit indexing.
__global__ void __launch_bounds__(256) silu_mul_bf16_fast_kernel(const __nv_bfloat16* __restrict__ gu, int total,
                                                                 int vpr, int blk, __nv_bfloat16* __restrict__ out) {
  const int t0 = blockIdx.x * 512 + threadIdx.x;
  uint4 gv[2], uv[2];
  int r[2], c[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int t = t0 + u * 256;
    r[u] = t / vpr;
    c[u] = t - r[u] * vpr;
    if (t < total) {
      const int e = c[u] * 8;
      const __nv_bfloat16* base = gu + (int64_t)r[u] * 16 * vpr + (e / blk) * 2 * blk + e % blk;
      gv[u] = *reinterpret_cast<const uint4*>(base);
      uv[u] = *reinterpret_cast<const uint4*>(base + blk);
    }
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    if (t0 + u * 256 >= total) continue;
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gv[u]);
    const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&uv[u]);
    uint4 ov;
    uint32_t* o = reinterpret_cast<uint32_t*>(&ov);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 g = __bfloat1622float2(g2[k]), up = __bfloat1622float2(u2[k]);
      const float s0 = 0.5f * g.x * (1.f + tanh_approx(0.5f * g.x));
      const float s1 = 0.5f * g.y * (1.f + tanh_approx(0.5f * g.y));
      __nv_bfloat162 y = __floats2bfloat162_rn(s0 * up.x, s1 * up.y);
      o[k] = *reinterpret_cast<uint32_t*>(&y);
    }
    *reinterpret_cast<uint4*>(out + (int64_t)r[u] * 8 * vpr + c[u] * 8) = ov;
  }
}

template <typename T>
__global__ void embed_rows_kernel(const T* __restrict__ table, const int64_t* __restrict__ ids, int rows, int d,
                                  float* __restrict__ h) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)rows * d) return;
  int64_t r = t / d, c = t - r * d;
  h[t] = to_f32(table[ids[r] * d + c]);
}

__global__ void split3_kernel(const float* __restrict__ x, int64_t n, __nv_bfloat16* __restrict__ out) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  __nv_bfloat16 a, b, c;
  split3(x[t], a, b, c);
  out[t] = a;
  out[n + t] = b;
  out[2 * n + t] = c;
}

// One warp per row: acc[r] += sqrt(sum_c (a - b)^2), fp32 lane partials,
// fp64 cross-lane sum (CacheBlend hidden-state deviation, selection.py:219-222).
__global__ void __launch_bounds__(256) row_dist_accum_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                             int rows, int d, double* __restrict__ acc) {
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* pa = a + (int64_t)r * d;
  const float* pb = b + (int64_t)r * d;
  float s = 0.f;
  if (d % 4 == 0) {
    for (int c = lane * 4; c < d; c += 128) {
      const float4 x = *reinterpret_cast<const float4*>(pa + c), y = *reinterpret_cast<const float4*>(pb + c);
      const float e0 = x.x - y.x, e1 = x.y - y.y, e2 = x.z - y.z, e3 = x.w - y.w;
      s += (e0 * e0 + e1 * e1) + (e2 * e2 + e3 * e3);
    }
  } else {
    for (int c = lane; c < d; c += 32) {
      const float e = pa[c] - pb[c];
      s += e * e;
    }
  }
  double t = s;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) acc[r] += sqrt(t);
}

}  // namespace ifkv

using namespace ifkv;

extern "C" int ifkv_row_dist_accum(const float* a, const float* b, int rows, int d, double* acc, void* stream) {
  IFKV_CHECK_ARG(rows >= 0 && d > 0, "row_dist_accum: bad shape");
  if (rows == 0) return IFKV_OK;
  IFKV_CHECK_ARG(d % 4 != 0 || ((uintptr_t)a % 16 == 0 && (uintptr_t)b % 16 == 0), "row_dist_accum: misaligned rows");
  row_dist_accum_kernel<<<(rows + 7) / 8, 256, 0, as_stream(stream)>>>(a, b, rows, d, acc);
  IFKV_LAUNCH_CHECK("row_dist_accum");
  return IFKV_OK;
}

extern "C" int ifkv_add_rmsnorm(float* h, const void* delta, int delta_dtype, int n_parts, const float* gain,
                                int rows, int d, int out_mode, void* out, void* stream) {
  IFKV_CHECK_ARG(rows >= 0 && d > 0 && d % 4 == 0 && d <= 8192, "add_rmsnorm: d must be a multiple of 4, <= 8192");
  IFKV_CHECK_ARG(out_mode >= IFKV_OUT_F32 && out_mode <= IFKV_OUT_SPLIT3, "add_rmsnorm: bad out mode");
  IFKV_CHECK_ARG(n_parts == 0 || delta_dtype == IFKV_F32 || delta_dtype == IFKV_BF16, "add_rmsnorm: bad dtype");
  if (rows == 0) return IFKV_OK;
  cudaStream_t s = as_stream(stream);
  const bool bf = n_parts > 0 && delta_dtype == IFKV_BF16;
#ifndef IFKV_RMS_PERSIST
#define IFKV_RMS_PERSIST 1
#endif
#ifndef IFKV_RMS_PERSIST_CTAS
#define IFKV_RMS_PERSIST_CTAS 3
#endif
  if (IFKV_RMS_PERSIST && d == 4096 && rows >= 148 * 4) {
    const unsigned grid = 148 * IFKV_RMS_PERSIST_CTAS;
    if (bf)
      IFKV_CUDA_CALL(launch_pdl(add_rmsnorm_pf_kernel<__nv_bfloat16>, dim3(grid), dim3(256), 0, s, h,
                                (const __nv_bfloat16*)delta, n_parts, gain, rows, out_mode, out),
                     "add_rmsnorm: launch");
    else
      IFKV_CUDA_CALL(launch_pdl(add_rmsnorm_pf_kernel<float>, dim3(grid), dim3(256), 0, s, h, (const float*)delta,
                                n_parts, gain, rows, out_mode, out),
                     "add_rmsnorm: launch");
  } else if (rows < 2 * 148 && d <= 4 * 2 * 1024) {  // few rows (prompt forward): spread each row over 1024 threads
    if (bf)
      add_rmsnorm_kernel<__nv_bfloat16, 1024, 2><<<rows, 1024, 0, s>>>(h, (const __nv_bfloat16*)delta, n_parts, gain,
                                                                      rows, d, out_mode, out);
    else
      IFKV_CUDA_CALL(launch_pdl(add_rmsnorm_kernel<float, 1024, 2>, dim3(rows), dim3(1024), 0, s, h,
                                (const float*)delta, n_parts, gain, rows, d, out_mode, out),
                     "add_rmsnorm: launch");
  } else if (d <= 4096) {
    if (bf)
      add_rmsnorm_kernel<__nv_bfloat16, 128><<<rows, 128, 0, s>>>(h, (const __nv_bfloat16*)delta, n_parts, gain, rows,
                                                                 d, out_mode, out);
    else
      add_rmsnorm_kernel<float, 128><<<rows, 128, 0, s>>>(h, (const float*)delta, n_parts, gain, rows, d, out_mode,
                                                         out);
  } else {
    if (bf)
      add_rmsnorm_kernel<__nv_bfloat16, 256><<<rows, 256, 0, s>>>(h, (const __nv_bfloat16*)delta, n_parts, gain, rows,
                                                                 d, out_mode, out);
    else
      add_rmsnorm_kernel<float, 256><<<rows, 256, 0, s>>>(h, (const float*)delta, n_parts, gain, rows, d, out_mode,
                                                         out);
  }
  IFKV_LAUNCH_CHECK("add_rmsnorm");
  return IFKV_OK;
}

extern "C" int ifkv_silu_mul(const void* gu, int gu_dtype, int n_parts, int rows, int d_ff, int gu_block,
                             int out_mode, void* out, void* stream) {
  IFKV_CHECK_ARG(rows >= 0 && d_ff > 0 && d_ff % 4 == 0 && n_parts >= 1, "silu_mul: d_ff must be a multiple of 4");
  IFKV_CHECK_ARG(gu_block > 0 && gu_block % 4 == 0 && d_ff % gu_block == 0,
                 "silu_mul: gu_block must divide d_ff and be a multiple of 4");
  IFKV_CHECK_ARG(out_mode >= IFKV_OUT_F32 && out_mode <= IFKV_OUT_SPLIT3, "silu_mul: bad out mode");
  int64_t n = (int64_t)rows * d_ff / 4;
  if (n == 0) return IFKV_OK;
  int64_t want = (n + 255) / 256;
  unsigned grid = (unsigned)(want < 148 * 16 ? want : 148 * 16);
#ifndef IFKV_SILU_FAST
#define IFKV_SILU_FAST 1
#endif
  if (IFKV_SILU_FAST && gu_dtype == IFKV_BF16 && n_parts == 1 && out_mode == IFKV_OUT_BF16 && gu_block % 8 == 0 &&
      (int64_t)rows * d_ff / 8 + 512 < (int64_t)INT32_MAX) {
    const int total = (int)((int64_t)rows * d_ff / 8);
    silu_mul_bf16_fast_kernel<<<(unsigned)((total + 511) / 512), 256, 0, as_stream(stream)>>>(
        (const __nv_bfloat16*)gu, total, d_ff / 8, gu_block, (__nv_bfloat16*)out);
  } else if (gu_dtype == IFKV_BF16 && n_parts == 1 && out_mode == IFKV_OUT_BF16 && gu_block % 8 == 0) {
    const int64_t nv = (int64_t)rows * d_ff / 8;
    const int64_t w8 = (nv + 255) / 256;
    silu_mul_bf16x8_kernel<<<(unsigned)(w8 < 148 * 16 ? w8 : 148 * 16), 256, 0, as_stream(stream)>>>(
        (const __nv_bfloat16*)gu, rows, d_ff, gu_block, (__nv_bfloat16*)out);
  } else if (gu_dtype == IFKV_BF16)
    silu_mul_kernel<__nv_bfloat16><<<grid, 256, 0, as_stream(stream)>>>((const __nv_bfloat16*)gu, n_parts, rows,
                                                                       d_ff, gu_block, out_mode, out);
  else
    IFKV_CUDA_CALL(launch_pdl(silu_mul_kernel<float>, dim3(grid), dim3(256), 0, as_stream(stream), (const float*)gu,
                              n_parts, rows, d_ff, gu_block, out_mode, out),
                   "silu_mul: launch");
  IFKV_LAUNCH_CHECK("silu_mul");
  return IFKV_OK;
}

extern "C" int ifkv_embed_rows(const void* table, int dtype, const int64_t* ids, int rows, int d, float* h,
                               void* stream) {
  IFKV_CHECK_ARG(dtype == IFKV_F32 || dtype == IFKV_BF16, "embed_rows: bad dtype");
  int64_t n = (int64_t)rows * d;
  if (n <= 0) return IFKV_OK;
  unsigned grid = (unsigned)((n + 255) / 256);
  if (dtype == IFKV_BF16)
    embed_rows_kernel<__nv_bfloat16><<<grid, 256, 0, as_stream(stream)>>>((const __nv_bfloat16*)table, ids, rows, d, h);
  else
    embed_rows_kernel<float><<<grid, 256, 0, as_stream(stream)>>>((const float*)table, ids, rows, d, h);
  IFKV_LAUNCH_CHECK("embed_rows");
  return IFKV_OK;
}

extern "C" int ifkv_split3(const float* x, int64_t n, void* out, void* stream) {
  if (n <= 0) return IFKV_OK;
  split3_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(x, n, (__nv_bfloat16*)out);
  IFKV_LAUNCH_CHECK("split3");
  return IFKV_OK;
}
