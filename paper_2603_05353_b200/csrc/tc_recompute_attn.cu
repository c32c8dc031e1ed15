// placeholder: replaced by the tcgen05 kernel
#include "common.cuh"
extern "C" int ifkv_recompute_attn_tc_supported(int dtype, int H, int Hkv, int Dh) { return 0; }
extern "C" int ifkv_recompute_attn_tc(const void*, const void*, const void*, const int64_t*, int, int, int, int, float,
                                      void*, void*) {
  ifkv::set_error("tcgen05 recompute attention not built");
  return IFKV_ERR_ARG;
}
