// ref_common.cuh -- scalar fp32 sampling helpers shared by the reference
// decode kernel (ref_kernel.cu) and the fine-tuning kernels (train_kernel.cu):
// texel fetch from a stored map (BC7 / BC1 / BC3 / BC5 decoded per tap, R8
// dequantisation),
// texel-centre bilinear with clamp (R1), accurate GELU (R7).
#pragma once
#include "bc7_device.cuh"
#include "bcn_device.cuh"
#include "ndgi_common.cuh"

namespace ndgi {

struct Map2D {
    const uint8_t* base;
    int fmt, rx, ry, nc;
};

// packed texel of the other block formats (BC1 / BC3 / BC5), out of line so
// the taps that inline fetch_texel do not each carry these decoders
static __device__ __noinline__ uint32_t bcn_texel(const uint8_t* base, int fmt, size_t bi, int i) {
    if (fmt == FMT_BC1) return bc1_texel(__ldg(reinterpret_cast<const uint2*>(base) + bi), i, false);
    const uint4 raw = __ldg(reinterpret_cast<const uint4*>(base) + bi);
    if (fmt == FMT_BC3)
        return (bc1_texel(make_uint2(raw.z, raw.w), i, true) & 0x00ffffffu) | bc4_texel(make_uint2(raw.x, raw.y), i) << 24;
    return bc4_texel(make_uint2(raw.x, raw.y), i) | bc4_texel(make_uint2(raw.z, raw.w), i) << 8;   // BC5
}

// all channels of texel (a, b), dequantised (R8)
__device__ __forceinline__ void fetch_texel(const Map2D& m, int a, int b, float* out) {
    if (m.fmt == FMT_BC7) {
        const uint4 raw = __ldg(reinterpret_cast<const uint4*>(m.base) + (b >> 2) * (m.rx >> 2) + (a >> 2));
        const uint32_t v = bc7_texel(raw, 4 * (b & 3) + (a & 3));
        for (int c = 0; c < m.nc; ++c) out[c] = (float)((v >> (8 * c)) & 0xffu) / 255.0f;
    } else if (m.fmt == FMT_U8) {
        if (m.nc == 4) {   // one 32-bit load (U8 maps are 4-byte aligned, include/ndgi.h)
            const uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(m.base) + ((size_t)b * m.rx + a));
            for (int c = 0; c < 4; ++c) out[c] = (float)((v >> (8 * c)) & 0xffu) / 255.0f;
        } else {
            const uint8_t* p = m.base + ((size_t)b * m.rx + a) * m.nc;
            for (int c = 0; c < m.nc; ++c) out[c] = (float)p[c] / 255.0f;
        }
    } else if (m.fmt == FMT_F16) {
        const uint16_t* p = reinterpret_cast<const uint16_t*>(m.base) + ((size_t)b * m.rx + a) * m.nc;
        for (int c = 0; c < m.nc; ++c) out[c] = half_bits_to_float(p[c]);
    } else {   // BC1 / BC3 / BC5
        const uint32_t v = bcn_texel(m.base, m.fmt, (size_t)(b >> 2) * (m.rx >> 2) + (a >> 2), 4 * (b & 3) + (a & 3));
        for (int c = 0; c < m.nc; ++c) out[c] = (float)((v >> (8 * c)) & 0xffu) / 255.0f;
    }
}

// texel-centre bilinear with clamp (R1)
__device__ __forceinline__ void bilinear(const Map2D& m, float a, float b, float* out) {
    const float sx = a * (float)m.rx - 0.5f, sy = b * (float)m.ry - 0.5f;
    const float fx0 = floorf(sx), fy0 = floorf(sy);
    const float fx = sx - fx0, fy = sy - fy0;
    const int x0 = clampi((int)fx0, 0, m.rx - 1), x1 = clampi((int)fx0 + 1, 0, m.rx - 1);
    const int y0 = clampi((int)fy0, 0, m.ry - 1), y1 = clampi((int)fy0 + 1, 0, m.ry - 1);
    float t00[4], t10[4], t01[4], t11[4];
    fetch_texel(m, x0, y0, t00);
    fetch_texel(m, x1, y0, t10);
    fetch_texel(m, x0, y1, t01);
    fetch_texel(m, x1, y1, t11);
    const float w00 = (1.f - fx) * (1.f - fy), w10 = fx * (1.f - fy), w01 = (1.f - fx) * fy, w11 = fx * fy;
    for (int c = 0; c < m.nc; ++c) out[c] = w00 * t00[c] + w10 * t10[c] + w01 * t01[c] + w11 * t11[c];
}

__device__ __forceinline__ float gelu_ref(float z, int variant) {
    if (variant == GELU_TANH) return 0.5f * z * (1.0f + tanhf(0.7978845608028654f * (z + 0.044715f * z * z * z)));
    return 0.5f * z * (1.0f + erff(z * 0.7071067811865476f));
}

}  // namespace ndgi
