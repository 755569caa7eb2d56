// fused_kernel.cu -- host side of the fused tile-decode kernel: the load-time
// weight prepack and the dispatch to the per-(h, C) instantiations
// (fused_h16_c128.cu, fused_h16_c256.cu, fused_h64.cu).
#include <cuda_runtime.h>

#include "fused_common.cuh"

namespace ndgi {

// per-format instantiations live in fused_h*_*.cu (parallel compilation)
template <int H, int FMT_UV, int CT>
cudaError_t launch_fused_t(const KParams& p, int num_sms, cudaStream_t s);

template <int H, int CT>
static cudaError_t launch_fused_fmt(const KParams& p, int num_sms, cudaStream_t s) {
    if (p.fmt_uv == FMT_BC7_TEX) return launch_fused_t<H, FMT_BC7_TEX, CT>(p, num_sms, s);
    if (p.fmt_uv == FMT_BC7) return launch_fused_t<H, FMT_BC7, CT>(p, num_sms, s);
    if (p.fmt_uv == FMT_U8) return launch_fused_t<H, FMT_U8, CT>(p, num_sms, s);
    if (p.fmt_uv == FMT_BC1) return launch_fused_t<H, FMT_BC1, CT>(p, num_sms, s);
    if (p.fmt_uv == FMT_BC3) return launch_fused_t<H, FMT_BC3, CT>(p, num_sms, s);
    return launch_fused_t<H, FMT_F16, CT>(p, num_sms, s);
}

size_t wpack_tile_bytes(int H) { return H == 16 ? WPack<16>::BYTES : WPack<64>::BYTES; }

cudaError_t prep_weights(const uint16_t* mlp, size_t tile_elems, int H, int fmt_uv, uint8_t* out, int num_tiles,
                         cudaStream_t s) {
    const float s_uv = fmt_uv == FMT_F16 ? kGeluA : kGeluA / 255.0f;   // F_uv enters in q units (R8)
    const int grid = num_tiles < 4096 ? num_tiles : 4096;
    if (H == 16) prep_weights_kernel<16><<<grid, 256, 0, s>>>(mlp, tile_elems, s_uv, out, num_tiles);
    else prep_weights_kernel<64><<<grid, 256, 0, s>>>(mlp, tile_elems, s_uv, out, num_tiles);
    return cudaGetLastError();
}

// the GELU split compiled into the epilogues: MUFU pairs of every 16 (h = 16:
// a step's two items take NDGI_POLY_PAIRS_ITEM0 + NDGI_POLY_PAIRS polynomial
// pairs of their 2 x 8; h = 64: NDGI_POLY_PAIRS64 of every 8)
int fused_gelu_mufu_pairs(int H) {
    return H == 16 ? 16 - NDGI_POLY_PAIRS_ITEM0 - NDGI_POLY_PAIRS : 16 - 2 * NDGI_POLY_PAIRS64;
}
int fused_f16acc() { return NDGI_F16ACC; }

int fused_ctas_per_sm(int H) { return H == 16 ? FusedCfg<16>::MIN_CTAS : FusedCfg<64>::MIN_CTAS; }

cudaError_t launch_fused(const KParams& p, int num_sms, cudaStream_t s) {
    if (p.H == 16) return p.C == 128 ? launch_fused_fmt<16, 128>(p, num_sms, s) : launch_fused_fmt<16, 256>(p, num_sms, s);
    return p.C == 128 ? launch_fused_fmt<64, 128>(p, num_sms, s) : launch_fused_fmt<64, 256>(p, num_sms, s);
}

}  // namespace ndgi
