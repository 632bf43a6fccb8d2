// tc_gemm.cuh — tcgen05 / TMA tensor-core products (placeholder until the
// sm_100a kernels land; every entry returns GEIG_ERR_UNSUPPORTED).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../../include/geig.h"

namespace geig { namespace tc {

struct TcPlan { int ready = 0; };

inline const char* last_error() { return "tcgen05 products not built in this version"; }

inline geig_status plan_create(TcPlan&, int, int64_t, int64_t, int, int, int64_t, int) {
  return GEIG_ERR_UNSUPPORTED;
}
inline void plan_destroy(TcPlan&) {}
inline geig_status products_cca(TcPlan&, const void*, const void*, int64_t, float, const __nv_bfloat16*,
                                const float*, __nv_bfloat16*, __nv_bfloat16*, float*, float*,
                                cudaStream_t, int64_t*) {
  return GEIG_ERR_UNSUPPORTED;
}
inline geig_status products_dense(TcPlan&, const void*, const void*, int64_t, int64_t, const __nv_bfloat16*,
                                  const float*, float*, float*, cudaStream_t, int64_t*) {
  return GEIG_ERR_UNSUPPORTED;
}

}}  // namespace geig::tc
