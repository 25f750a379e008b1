// tcgen05 / TMEM / TMA bf16 contractions for sm_100a (placeholder until the tensor-core kernels land).
#include "pfc_internal.cuh"

namespace pfc {
bool tc_available() { return false; }
int launch_logits_tc(const Sizes&, const __nv_bfloat16*, const __nv_bfloat16*, const int32_t*, const float*,
                     const SamplerState*, MarginParams, __half*, float2*, cudaStream_t) { return 0; }
int launch_dx_tc(const Sizes&, const __nv_bfloat16*, const __nv_bfloat16*, const SamplerState*, float*, float*,
                 cudaStream_t) { return 0; }
int launch_dw_tc(const Sizes&, const __nv_bfloat16*, const __nv_bfloat16*, const SamplerState*, float*,
                 cudaStream_t) { return 0; }
}  // namespace pfc
