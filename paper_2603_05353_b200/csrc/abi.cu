// ABI bookkeeping: thread-local error message and version.
#include <stdarg.h>

#include "common.cuh"

namespace ifkv {
static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace ifkv

extern "C" const char* ifkv_last_error(void) { return ifkv::g_err; }
extern "C" int ifkv_abi_version(void) { return 1; }
