// conv_tc.cu -- tcgen05 TF32 implicit-GEMM convolution (placeholder until bring-up).
#include "common.cuh"
#include "kernels.cuh"

namespace sysml {
bool tc_fwd_supported(const ConvArgs &, const PoolArgs *) { return false; }
size_t tc_fwd_ws(const ConvArgs &) { return 0; }
sysml_status tc_conv_fwd(const ConvArgs &, const float *, const float *, const float *, float *,
                         const PoolArgs *, float *, int32_t *, void *, cudaStream_t) {
  set_error("tcgen05 forward kernel not available");
  return SYSML_ERR_UNSUPPORTED;
}
bool tc_bwd_data_supported(const ConvArgs &) { return false; }
size_t tc_bwd_data_ws(const ConvArgs &) { return 0; }
sysml_status tc_conv_bwd_data(const ConvArgs &, const float *, const float *, float *, void *,
                              cudaStream_t) {
  set_error("tcgen05 bwd_data kernel not available");
  return SYSML_ERR_UNSUPPORTED;
}
bool tc_bwd_filter_supported(const ConvArgs &) { return false; }
size_t tc_bwd_filter_ws(const ConvArgs &) { return 0; }
sysml_status tc_conv_bwd_filter(const ConvArgs &, const float *, const float *, float *, float *,
                                void *, cudaStream_t) {
  set_error("tcgen05 bwd_filter kernel not available");
  return SYSML_ERR_UNSUPPORTED;
}
}  // namespace sysml
