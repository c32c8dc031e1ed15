// ABI bookkeeping: thread-local error message and version.
#include <stdarg.h>
#include <stdlib.h>

#include <mutex>

#include "common.cuh"

namespace ifkv {
static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("IFKV_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

void* workspace_alloc(size_t bytes, cudaStream_t st) {
  static std::once_flag once[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::call_once(once[dev & 63], [dev] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;  // never trim at synchronize: split workspaces are reused per query
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  });
  void* p = nullptr;
  return cudaMallocAsync(&p, bytes, st) == cudaSuccess ? p : nullptr;
}
}  // namespace ifkv

extern "C" const char* ifkv_last_error(void) { return ifkv::g_err; }
extern "C" int ifkv_abi_version(void) { return 1; }
