// fused_h16_c128_bc7.cu -- instantiations of the fused tile-decode kernel (fused_kernel.cuh),
// one translation unit per group so the build compiles them in parallel
#include "fused_kernel.cuh"

namespace ndgi {
template cudaError_t launch_fused_t<16, FMT_BC7, 128>(const KParams& p, int num_sms, cudaStream_t s);
template cudaError_t launch_fused_t<16, FMT_BC7_TEX, 128>(const KParams& p, int num_sms, cudaStream_t s);
}  // namespace ndgi

#if NDGI_TIMELINE
// diagnostic builds only: the block-0 stage stamps of the last launch of a
// (h = 16, C = 128, BC7) fused kernel
extern "C" __attribute__((visibility("default"))) int ndgi_debug_timeline(unsigned long long* out16) {
    return (int)cudaMemcpyFromSymbol(out16, ndgi::g_ndgi_timeline, 16 * sizeof(unsigned long long));
}
#endif

#if NDGI_RESIDENCY
// diagnostic builds only: per-CTA (SM id, entry, after TMEM allocation, exit) of
// the last (h = 16, C = 128, BC7) fused launch
extern "C" __attribute__((visibility("default"))) int ndgi_debug_residency(unsigned long long* out, int nblocks) {
    return (int)cudaMemcpyFromSymbol(out, ndgi::g_ndgi_res, (size_t)(nblocks < 4096 ? nblocks : 4096) * 4 * sizeof(unsigned long long));
}
#endif
