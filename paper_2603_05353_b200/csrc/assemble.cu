// assemble (reference cache.py:259-322): gather chunk KV caches into the
// per-query layer-major slab.  Pure HBM->HBM copy with 128-bit vectors; one
// launch covers up to kMaxChunks chunks (grid.y = chunk).
#include "common.cuh"

namespace ifkv {

constexpr int kMaxChunks = 256;

struct GatherParams {
  const uint4* src_k[kMaxChunks];
  const uint4* src_v[kMaxChunks];
  int64_t src_layer_stride[kMaxChunks];  // in 16-byte vectors
  int32_t len[kMaxChunks];
  int32_t row0[kMaxChunks];
};

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

extern "C" int ifkv_assemble_gather(int dtype, int n_chunks, const void* const* src_k, const void* const* src_v,
                                    const int64_t* src_layer_stride, const int32_t* chunk_len,
                                    const int32_t* dst_row0, void* dst_k, void* dst_v, int64_t dst_layer_stride,
                                    int n_layers, int row_elems, void* stream) {
  IFKV_CHECK_ARG(dtype == IFKV_F32 || dtype == IFKV_BF16, "assemble_gather: bad dtype %d", dtype);
  const int esz = dtype == IFKV_F32 ? 4 : 2;
  IFKV_CHECK_ARG((row_elems * esz) % 16 == 0, "assemble_gather: row bytes must be a multiple of 16");
  IFKV_CHECK_ARG((dst_layer_stride * esz) % 16 == 0, "assemble_gather: dst layer stride misaligned");
  IFKV_CHECK_ARG((uintptr_t)dst_k % 16 == 0 && (uintptr_t)dst_v % 16 == 0, "assemble_gather: dst misaligned");
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
      int64_t w = (int64_t)chunk_len[c] * vpr * n_layers;
      if (w > max_work) max_work = w;
    }
    // enough CTAs per chunk that all chunks together fill ~8 CTAs per SM
    int64_t per_chunk = ((int64_t)sms * 8 + nc - 1) / nc;
    int64_t need = (max_work + 511) / 512;
    unsigned gx = (unsigned)(need < per_chunk ? (need > 0 ? need : 1) : per_chunk);
    dim3 grid(gx, nc);
    assemble_gather_kernel<<<grid, 256, 0, as_stream(stream)>>>(p, reinterpret_cast<uint4*>(dst_k),
                                                               reinterpret_cast<uint4*>(dst_v),
                                                               dst_layer_stride * esz / 16, n_layers, vpr);
    IFKV_LAUNCH_CHECK("assemble_gather");
  }
  return IFKV_OK;
}
