// fused_h16_c256.cu -- instantiations of the fused tile-decode kernel (fused_kernel.cuh),
// one translation unit per group so the build compiles them in parallel
#include "fused_kernel.cuh"

namespace ndgi {
template cudaError_t launch_fused_t<16, FMT_BC7, 256>(const KParams& p, int num_sms, cudaStream_t s);
template cudaError_t launch_fused_t<16, FMT_BC7_TEX, 256>(const KParams& p, int num_sms, cudaStream_t s);
template cudaError_t launch_fused_t<16, FMT_U8, 256>(const KParams& p, int num_sms, cudaStream_t s);
template cudaError_t launch_fused_t<16, FMT_F16, 256>(const KParams& p, int num_sms, cudaStream_t s);
template cudaError_t launch_fused_t<16, FMT_BC1, 256>(const KParams& p, int num_sms, cudaStream_t s);
template cudaError_t launch_fused_t<16, FMT_BC3, 256>(const KParams& p, int num_sms, cudaStream_t s);
}  // namespace ndgi
