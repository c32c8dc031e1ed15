// assemble (reference cache.py:259-322): gather chunk KV caches into the
// per-query layer-major slab.  Pure HBM->HBM copy with 128-bit vectors; one
// launch covers up to kMaxChunks chunks (grid.y = chunk).
//
// The rotating variant also moves every key to its assembled (global)
// position while copying -- rotate_heads by the chunk's delta
// (model.py:254-270, as recompute.py:106-109 / decode_view cache.py:382-403
// apply it) -- so the per-query slab comes out in the decode layout in ONE
// pass over K instead of a gather followed by Kernel 1 in place.
#include <stdlib.h>

#include "common.cuh"

namespace ifkv {

constexpr int kMaxChunks = 256;

struct GatherParams {
  const uint4* src_k[kMaxChunks];
  const uint4* src_v[kMaxChunks];
  int64_t src_layer_stride[kMaxChunks];  // in 16-byte vectors
  int32_t len[kMaxChunks];
  int32_t row0[kMaxChunks];
  int32_t cs_row[kMaxChunks];  // rotating variant: row of the (cos, sin) table, -1 = delta 0
};

// Rotate the interleaved pairs of one 16-byte key vector (element e0 of its
// head onward) by the angles cs[e0/2 ..]: 8 bf16 = 4 pairs or 4 fp32 = 2 pairs.
template <bool kBf16>
__device__ __forceinline__ uint4 rotate_vec(uint4 v, const float2* __restrict__ cs, int e0) {
  if (kBf16) {
    __nv_bfloat162* e = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 x = __bfloat1622float2(e[q]);
      const float2 y = rot_pair(x.x, x.y, __ldg(cs + e0 / 2 + q));
      e[q] = __floats2bfloat162_rn(y.x, y.y);
    }
  } else {
    float* f = reinterpret_cast<float*>(&v);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float2 y = rot_pair(f[2 * q], f[2 * q + 1], __ldg(cs + e0 / 2 + q));
      f[2 * q] = y.x;
      f[2 * q + 1] = y.y;
    }
  }
  return v;
}

template <bool kBf16>
__global__ void __launch_bounds__(256) assemble_gather_rotate_kernel(const __grid_constant__ GatherParams p,
                                                                     const float2* __restrict__ cs, int half,
                                                                     int vecs_per_head, uint4* __restrict__ dst_k,
                                                                     uint4* __restrict__ dst_v,
                                                                     int64_t dst_layer_stride, int n_layers,
                                                                     int vecs_per_row) {
  const int c = blockIdx.y;
  const int per_layer = p.len[c] * vecs_per_row;
  const int64_t total = (int64_t)per_layer * n_layers;
  const uint4* sk = p.src_k[c];
  const uint4* sv = p.src_v[c];
  const int64_t ss = p.src_layer_stride[c];
  const int64_t drow0 = (int64_t)p.row0[c] * vecs_per_row;
  const float2* tab = p.cs_row[c] >= 0 ? cs + (int64_t)p.cs_row[c] * half : nullptr;
  constexpr int kElems = kBf16 ? 8 : 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += 2 * stride) {
    const int64_t g2 = g + stride;
    const bool two = g2 < total;
    const int64_t l = g / per_layer, r = g - l * per_layer;
    const int64_t l2 = two ? g2 / per_layer : 0, r2 = two ? g2 - l2 * per_layer : 0;
    uint4 k0 = sk[l * ss + r], v0 = sv[l * ss + r], k1, v1;
    if (two) {
      k1 = sk[l2 * ss + r2];
      v1 = sv[l2 * ss + r2];
    }
    if (tab) {
      k0 = rotate_vec<kBf16>(k0, tab, (int)((r % vecs_per_row) % vecs_per_head) * kElems);
      if (two) k1 = rotate_vec<kBf16>(k1, tab, (int)((r2 % vecs_per_row) % vecs_per_head) * kElems);
    }
    dst_k[l * dst_layer_stride + drow0 + r] = k0;
    dst_v[l * dst_layer_stride + drow0 + r] = v0;
    if (two) {
      dst_k[l2 * dst_layer_stride + drow0 + r2] = k1;
      dst_v[l2 * dst_layer_stride + drow0 + r2] = v1;
    }
  }
}

__global__ void __launch_bounds__(256) assemble_gather_kernel(const __grid_constant__ GatherParams p,
                                                              uint4* __restrict__ dst_k, uint4* __restrict__ dst_v,
                                                              int64_t dst_layer_stride, int n_layers,
                                                              int vecs_per_row) {
  const int c = blockIdx.y;
  const int64_t per_layer = (int64_t)p.len[c] * vecs_per_row;
  const int64_t total = per_layer * n_layers;
  const uint4* sk = p.src_k[c];
  const uint4* sv = p.src_v[c];
  const int64_t ss = p.src_layer_stride[c];
  const int64_t drow0 = (int64_t)p.row0[c] * vecs_per_row;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += 2 * stride) {
    int64_t g2 = g + stride;
    int64_t l = g / per_layer, r = g - l * per_layer;
    uint4 k0 = sk[l * ss + r], v0 = sv[l * ss + r];
    uint4 k1, v1;
    int64_t l2 = 0, r2 = 0;
    bool two = g2 < total;
    if (two) {
      l2 = g2 / per_layer;
      r2 = g2 - l2 * per_layer;
      k1 = sk[l2 * ss + r2];
      v1 = sv[l2 * ss + r2];
    }
    dst_k[l * dst_layer_stride + drow0 + r] = k0;
    dst_v[l * dst_layer_stride + drow0 + r] = v0;
    if (two) {
      dst_k[l2 * dst_layer_stride + drow0 + r2] = k1;
      dst_v[l2 * dst_layer_stride + drow0 + r2] = v1;
    }
  }
}

}  // namespace ifkv

using namespace ifkv;

static int gather_launch(int dtype, int n_chunks, const void* const* src_k, const void* const* src_v,
                         const int64_t* src_layer_stride, const int32_t* chunk_len, const int32_t* dst_row0,
                         const int32_t* cs_row, const float* cs, int d_head, void* dst_k, void* dst_v,
                         int64_t dst_layer_stride, int n_layers, int row_elems, void* stream) {
  IFKV_CHECK_ARG(dtype == IFKV_F32 || dtype == IFKV_BF16, "assemble_gather: bad dtype %d", dtype);
  const int esz = dtype == IFKV_F32 ? 4 : 2;
  IFKV_CHECK_ARG((row_elems * esz) % 16 == 0, "assemble_gather: row bytes must be a multiple of 16");
  IFKV_CHECK_ARG((dst_layer_stride * esz) % 16 == 0, "assemble_gather: dst layer stride misaligned");
  IFKV_CHECK_ARG((uintptr_t)dst_k % 16 == 0 && (uintptr_t)dst_v % 16 == 0, "assemble_gather: dst misaligned");
  const bool rotate = cs_row != nullptr;
  if (rotate)
    IFKV_CHECK_ARG(cs != nullptr && d_head > 0 && (d_head * esz) % 16 == 0 && row_elems % d_head == 0,
                   "assemble_gather_rotate: d_head must divide the row and be a multiple of 16 bytes");
  if (n_chunks <= 0 || n_layers <= 0) return IFKV_OK;
  const int vpr = row_elems * esz / 16;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int c0 = 0; c0 < n_chunks; c0 += kMaxChunks) {
    int nc = n_chunks - c0 < kMaxChunks ? n_chunks - c0 : kMaxChunks;
    GatherParams p;
    int64_t max_work = 0;
    for (int i = 0; i < nc; ++i) {
      int c = c0 + i;
      IFKV_CHECK_ARG(chunk_len[c] >= 0, "assemble_gather: negative chunk length");
      IFKV_CHECK_ARG((uintptr_t)src_k[c] % 16 == 0 && (uintptr_t)src_v[c] % 16 == 0 &&
                         (src_layer_stride[c] * esz) % 16 == 0,
                     "assemble_gather: chunk %d misaligned", c);
      p.src_k[i] = reinterpret_cast<const uint4*>(src_k[c]);
      p.src_v[i] = reinterpret_cast<const uint4*>(src_v[c]);
      p.src_layer_stride[i] = src_layer_stride[c] * esz / 16;
      p.len[i] = chunk_len[c];
      p.row0[i] = dst_row0[c];
      p.cs_row[i] = rotate ? cs_row[c] : -1;
      int64_t w = (int64_t)chunk_len[c] * vpr * n_layers;
      if (w > max_work) max_work = w;
    }
    // enough CTAs per chunk that all chunks together fill ~16 CTAs per SM
    // (C2 in-step A/B, profiles/r2_session3/cps_ab/: 16 per SM 2.06-2.09 ms vs
    // 8 2.25-2.63, 4 2.16-2.24, 32 2.14-2.23; IFKV_GATHER_CPS overrides)
    int cps = 16;
    if (const char* e = getenv("IFKV_GATHER_CPS")) cps = atoi(e) > 0 ? atoi(e) : 16;
    int64_t per_chunk = ((int64_t)sms * cps + nc - 1) / nc;
    int64_t need = (max_work + 511) / 512;
    unsigned gx = (unsigned)(need < per_chunk ? (need > 0 ? need : 1) : per_chunk);
#ifdef IFKV_GATHER_SHORT_CTAS
    // A/B: one pass of short CTAs (512 vectors each, no grid-stride loop), so
    // that a higher-priority stream's kernels are scheduled between them
    if (rotate) gx = (unsigned)(need > 0 ? need : 1);
#endif
    dim3 grid(gx, nc);
    if (!rotate)
      assemble_gather_kernel<<<grid, 256, 0, as_stream(stream)>>>(p, reinterpret_cast<uint4*>(dst_k),
                                                                 reinterpret_cast<uint4*>(dst_v),
                                                                 dst_layer_stride * esz / 16, n_layers, vpr);
    else if (dtype == IFKV_BF16)
      assemble_gather_rotate_kernel<true><<<grid, 256, 0, as_stream(stream)>>>(
          p, reinterpret_cast<const float2*>(cs), d_head / 2, d_head * esz / 16, reinterpret_cast<uint4*>(dst_k),
          reinterpret_cast<uint4*>(dst_v), dst_layer_stride * esz / 16, n_layers, vpr);
    else
      assemble_gather_rotate_kernel<false><<<grid, 256, 0, as_stream(stream)>>>(
          p, reinterpret_cast<const float2*>(cs), d_head / 2, d_head * esz / 16, reinterpret_cast<uint4*>(dst_k),
          reinterpret_cast<uint4*>(dst_v), dst_layer_stride * esz / 16, n_layers, vpr);
    IFKV_LAUNCH_CHECK("assemble_gather");
  }
  return IFKV_OK;
}

extern "C" int ifkv_assemble_gather(int dtype, int n_chunks, const void* const* src_k, const void* const* src_v,
                                    const int64_t* src_layer_stride, const int32_t* chunk_len,
                                    const int32_t* dst_row0, void* dst_k, void* dst_v, int64_t dst_layer_stride,
                                    int n_layers, int row_elems, void* stream) {
  return gather_launch(dtype, n_chunks, src_k, src_v, src_layer_stride, chunk_len, dst_row0, nullptr, nullptr, 0,
                       dst_k, dst_v, dst_layer_stride, n_layers, row_elems, stream);
}

extern "C" int ifkv_assemble_gather_rotate(int dtype, int n_chunks, const void* const* src_k,
                                           const void* const* src_v, const int64_t* src_layer_stride,
                                           const int32_t* chunk_len, const int32_t* dst_row0,
                                           const int32_t* cs_row, const float* cs, int d_head, void* dst_k,
                                           void* dst_v, int64_t dst_layer_stride, int n_layers, int row_elems,
                                           void* stream) {
  IFKV_CHECK_ARG(cs_row != nullptr, "assemble_gather_rotate: cs_row required");
  return gather_launch(dtype, n_chunks, src_k, src_v, src_layer_stride, chunk_len, dst_row0, cs_row, cs, d_head,
                       dst_k, dst_v, dst_layer_stride, n_layers, row_elems, stream);
}
