// Shared helpers for the ifkv sm_100a kernels: error reporting, dtype
// conversion, warp reductions.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/ifkv.h"

namespace ifkv {

void set_error(const char* fmt, ...);

#define IFKV_CHECK_ARG(cond, ...)          \
  do {                                     \
    if (!(cond)) {                         \
      ::ifkv::set_error(__VA_ARGS__);      \
      return IFKV_ERR_ARG;                 \
    }                                      \
  } while (0)

#define IFKV_LAUNCH_CHECK(name)                                                         \
  do {                                                                                  \
    cudaError_t e_ = cudaGetLastError();                                                \
    if (e_ != cudaSuccess) {                                                            \
      ::ifkv::set_error("%s: CUDA launch failed: %s", name, cudaGetErrorString(e_));    \
      return IFKV_ERR_CUDA;                                                             \
    }                                                                                   \
  } while (0)

#define IFKV_CUDA_CALL(expr, name)                                                      \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      ::ifkv::set_error("%s: %s", name, cudaGetErrorString(e_));                        \
      return IFKV_ERR_CUDA;                                                             \
    }                                                                                   \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- programmatic dependent launch (the scoring pass's kernel chain) ---------
// A kernel launched with launch_pdl may start while its stream predecessor is
// still running (once every CTA of the predecessor has executed pdl_trigger
// or exited); it must call pdl_wait before it reads anything the predecessor
// wrote and before its first global write.  Both are no-ops for a normal
// launch.  IFKV_PDL=0 turns the attribute off (A/B).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Stream-ordered workspace (cudaMallocAsync) for the attention key splits.
// The device's default memory pool returns freed memory to the driver at
// every synchronize (release threshold 0), so the first split launch after
// each query's host sync re-mapped its workspace -- tens of ms in a step
// (C4 at 5 % recompute).  Keep it in the pool instead.
void* workspace_alloc(size_t bytes, cudaStream_t st);


__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T>
__device__ __forceinline__ T from_f32(float x);
template <>
__device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

__device__ __forceinline__ float load_as_f32(const void* p, int dtype, int64_t i) {
  return dtype == IFKV_F32 ? reinterpret_cast<const float*>(p)[i]
                           : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// RoPE rotation of one interleaved pair by (cos, sin) = c, with a fixed
// rounding sequence (x0 c - x1 s as fmul + fma) so that every kernel that moves
// a stored key (Kernel 1, the rotating gather) produces identical bits.
__device__ __forceinline__ float2 rot_pair(float x0, float x1, float2 c) {
  return make_float2(__fmaf_rn(x0, c.x, -__fmul_rn(x1, c.y)), __fmaf_rn(x0, c.y, __fmul_rn(x1, c.x)));
}

// Split an fp32 value into three bf16 terms whose sum reproduces it to
// ~2^-24 relative: hi = rn(x), mid = rn(x - hi), lo = rn(x - hi - mid).
__device__ __forceinline__ void split3(float x, __nv_bfloat16& hi, __nv_bfloat16& mid, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(x);
  float r = x - __bfloat162float(hi);
  mid = __float2bfloat16_rn(r);
  r -= __bfloat162float(mid);
  lo = __float2bfloat16_rn(r);
}

}  // namespace ifkv
