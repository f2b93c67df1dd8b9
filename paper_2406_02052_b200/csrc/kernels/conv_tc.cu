// conv_tc.cu -- tcgen05 (5th-gen tensor core) bf16 implicit-GEMM convolutions.
// Placeholder until the sm_100a kernels land: reports "unsupported" so the
// engine routes to the SIMT kernels.
#include "../kernels.h"

namespace petra {
bool conv_tc_supported(const ConvGeom &, int) { return false; }
size_t conv_tc_workspace(const ConvGeom &, int) { return 0; }
void conv_fwd_tc(const ConvGeom &, const __nv_bfloat16 *, const __nv_bfloat16 *, float *, __nv_bfloat16 *,
                 cudaStream_t) {}
void conv_dgrad_tc(const ConvGeom &, const __nv_bfloat16 *, const __nv_bfloat16 *, const float *, float *,
                   cudaStream_t) {}
void conv_wgrad_tc(const ConvGeom &, const __nv_bfloat16 *, const __nv_bfloat16 *, float *, float *,
                   cudaStream_t) {}
}  // namespace petra
