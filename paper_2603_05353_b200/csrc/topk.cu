// Exact top-k with the reference tie rule (selection.py:172-183: stable
// argsort of -scores, i.e. score desc then index asc; output ascending) and
// the per-chunk importance aggregation of the reorder first pass
// (reorder.py:84-112, 45-54).
//
// One 1024-thread CTA per segment.  Radix select over order-preserving
// uint32 keys finds the k-th largest score T exactly (4 passes x 256-bin
// shared histograms, integer counts -> deterministic); a block scan in index
// order then emits every index with score > T plus the lowest-index
// (k - #greater) entries equal to T, already ascending.
#include "common.cuh"

namespace ifkv {

constexpr int kTopkThreads = 1024;

__device__ __forceinline__ uint32_t order_key(float f) {
  if (f == 0.f) f = 0.f;  // -0 == +0 in the reference's comparisons
  uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// Inclusive block scan of 0/1 flags for 1024 threads; returns the inclusive
// prefix and writes the block total into *total.
__device__ __forceinline__ int block_scan_1024(int v, int* warp_tot, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;  // inclusive warp prefix
  }
  __syncthreads();
  int res = x + (w > 0 ? warp_tot[w - 1] : 0);
  *total = warp_tot[31];
  __syncthreads();
  return res;
}

__global__ void __launch_bounds__(kTopkThreads) topk_segments_kernel(const float* __restrict__ scores,
                                                                   const int32_t* __restrict__ seg_begin,
                                                                   const int32_t* __restrict__ seg_k,
                                                                   const int32_t* __restrict__ out_begin,
                                                                   int64_t* __restrict__ out_idx, int agg_mode,
                                                                   double* __restrict__ agg) {
  __shared__ int hist[256];
  __shared__ int warp_tot[32];
  __shared__ uint32_t s_prefix;
  __shared__ int s_remaining;
  __shared__ double red[32];
  const int s = blockIdx.x;
  const int b = seg_begin[s], e = seg_begin[s + 1], n = e - b;
  const int k = seg_k[s];
  const float* sc = scores + b;

  uint32_t prefix = 0, mask = 0;
  int remaining = k;
  if (k > 0 && k < n) {
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += kTopkThreads) hist[i] = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += kTopkThreads) {
        uint32_t u = order_key(sc[i]);
        if ((u & mask) == prefix) atomicAdd(&hist[(u >> shift) & 0xFF], 1);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int cum = 0, d = 255;
        for (; d > 0; --d) {
          if (cum + hist[d] >= remaining) break;
          cum += hist[d];
        }
        s_prefix = prefix | ((uint32_t)d << shift);
        s_remaining = remaining - cum;
      }
      __syncthreads();
      prefix = s_prefix;
      remaining = s_remaining;
      mask |= 0xFFu << shift;
      __syncthreads();
    }
  }
  // prefix = T (k-th largest key); take all > T and the first `remaining` == T.
  const bool take_all = k >= n;
  int written = 0, eq_seen = 0;
  double acc = 0.0;
  double mx = -INFINITY;
  const int ob = out_begin[s];
  for (int base = 0; base < n && k > 0; base += kTopkThreads) {
    int i = base + threadIdx.x;
    int gt = 0, eq = 0;
    float v = 0.f;
    if (i < n) {
      v = sc[i];
      uint32_t u = order_key(v);
      gt = take_all || u > prefix;
      eq = !take_all && u == prefix;
    }
    int eq_tot;
    int eq_incl = block_scan_1024(eq, warp_tot, &eq_tot);
    int take = gt || (eq && (eq_seen + eq_incl - 1) < remaining);
    int tot;
    int pos = block_scan_1024(take, warp_tot, &tot) - 1;
    if (take) {
      out_idx[ob + written + pos] = (int64_t)(b + i);
      acc += (double)v;
      mx = fmax(mx, (double)v);
    }
    written += tot;
    eq_seen += eq_tot;
  }
  if (agg_mode != IFKV_AGG_NONE) {
    // deterministic fixed-tree reduction of the per-thread partials
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double val = agg_mode == IFKV_AGG_MAX ? mx : acc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double y = __shfl_xor_sync(0xffffffffu, val, o);
      val = agg_mode == IFKV_AGG_MAX ? fmax(val, y) : val + y;
    }
    if (lane == 0) red[w] = val;
    __syncthreads();
    if (w == 0) {
      val = red[lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double y = __shfl_xor_sync(0xffffffffu, val, o);
        val = agg_mode == IFKV_AGG_MAX ? fmax(val, y) : val + y;
      }
      if (lane == 0) {
        if (k == 0) val = 0.0;
        else if (agg_mode == IFKV_AGG_MEAN) val /= (double)k;
        agg[s] = val;
      }
    }
  }
}

}  // namespace ifkv

using namespace ifkv;

extern "C" int ifkv_topk_segments(const float* scores, const int32_t* seg_begin, const int32_t* seg_k,
                                  const int32_t* out_begin, int n_seg, int64_t* out_idx, int agg_mode, double* agg,
                                  void* stream) {
  IFKV_CHECK_ARG(agg_mode >= IFKV_AGG_NONE && agg_mode <= IFKV_AGG_MAX, "topk_segments: bad agg mode %d", agg_mode);
  IFKV_CHECK_ARG(agg_mode == IFKV_AGG_NONE || agg != nullptr, "topk_segments: agg output missing");
  if (n_seg <= 0) return IFKV_OK;
  topk_segments_kernel<<<n_seg, kTopkThreads, 0, as_stream(stream)>>>(scores, seg_begin, seg_k, out_begin, out_idx,
                                                                      agg_mode, agg);
  IFKV_LAUNCH_CHECK("topk_segments");
  return IFKV_OK;
}
