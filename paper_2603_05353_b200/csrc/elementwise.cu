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

// Block-wide deterministic sum (fixed tree) for blockDim.x == 256.
__device__ __forceinline__ float block_sum_256(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = l < 8 ? red[l] : 0.f;
  t = warp_sum(t);
  __syncthreads();
  return t;
}

template <typename TD>
__global__ void __launch_bounds__(256) add_rmsnorm_kernel(float* __restrict__ h, const TD* __restrict__ delta,
                                                          int n_parts, const float* __restrict__ gain, int rows,
                                                          int d, int mode, void* __restrict__ out) {
  __shared__ float red[8];
  const int r = blockIdx.x;
  float* hr = h + (int64_t)r * d;
  const int64_t pstride = (int64_t)rows * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += 256) {
    float x = hr[i];
    if (n_parts > 0) {
      x += sum_parts(delta, n_parts, pstride, (int64_t)r * d + i);
      hr[i] = x;
    }
    ss += x * x;
  }
  if (!out) return;
  float ms = block_sum_256(ss, red) / (float)d;
  float den = sqrtf(ms + 1e-6f);
  for (int i = threadIdx.x; i < d; i += 256) {
    store_mode(out, mode, pstride, (int64_t)r * d + i, hr[i] / den * gain[i]);
  }
}

template <typename T>
__global__ void silu_mul_kernel(const T* __restrict__ gu, int n_parts, int rows, int d_ff, int mode,
                                void* __restrict__ out) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)rows * d_ff;
  if (t >= n) return;
  int64_t r = t / d_ff, c = t - r * d_ff;
  const int64_t pstride = (int64_t)rows * 2 * d_ff;
  float g = sum_parts(gu, n_parts, pstride, r * 2 * d_ff + c);
  float u = sum_parts(gu, n_parts, pstride, r * 2 * d_ff + d_ff + c);
  float s;
  if (g >= 0.f) {
    s = g / (1.f + expf(-g));
  } else {
    float e = expf(g);
    s = g * e / (1.f + e);
  }
  store_mode(out, mode, n, t, s * u);
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

}  // namespace ifkv

using namespace ifkv;

extern "C" int ifkv_add_rmsnorm(float* h, const void* delta, int delta_dtype, int n_parts, const float* gain,
                                int rows, int d, int out_mode, void* out, void* stream) {
  IFKV_CHECK_ARG(rows >= 0 && d > 0, "add_rmsnorm: bad shape");
  IFKV_CHECK_ARG(out_mode >= IFKV_OUT_F32 && out_mode <= IFKV_OUT_SPLIT3, "add_rmsnorm: bad out mode");
  IFKV_CHECK_ARG(n_parts == 0 || delta_dtype == IFKV_F32 || delta_dtype == IFKV_BF16, "add_rmsnorm: bad dtype");
  if (rows == 0) return IFKV_OK;
  cudaStream_t s = as_stream(stream);
  if (n_parts > 0 && delta_dtype == IFKV_BF16)
    add_rmsnorm_kernel<__nv_bfloat16><<<rows, 256, 0, s>>>(h, (const __nv_bfloat16*)delta, n_parts, gain, rows, d,
                                                           out_mode, out);
  else
    add_rmsnorm_kernel<float><<<rows, 256, 0, s>>>(h, (const float*)delta, n_parts, gain, rows, d, out_mode, out);
  IFKV_LAUNCH_CHECK("add_rmsnorm");
  return IFKV_OK;
}

extern "C" int ifkv_silu_mul(const void* gu, int gu_dtype, int n_parts, int rows, int d_ff, int out_mode, void* out,
                             void* stream) {
  IFKV_CHECK_ARG(rows >= 0 && d_ff > 0 && n_parts >= 1, "silu_mul: bad shape");
  IFKV_CHECK_ARG(out_mode >= IFKV_OUT_F32 && out_mode <= IFKV_OUT_SPLIT3, "silu_mul: bad out mode");
  int64_t n = (int64_t)rows * d_ff;
  if (n == 0) return IFKV_OK;
  unsigned grid = (unsigned)((n + 255) / 256);
  if (gu_dtype == IFKV_BF16)
    silu_mul_kernel<__nv_bfloat16><<<grid, 256, 0, as_stream(stream)>>>((const __nv_bfloat16*)gu, n_parts, rows,
                                                                       d_ff, out_mode, out);
  else
    silu_mul_kernel<float><<<grid, 256, 0, as_stream(stream)>>>((const float*)gu, n_parts, rows, d_ff, out_mode, out);
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
