// sample_kernel.cu -- shading-side sampling of the page cache (SURVEY.md §8(f)
// NEXT 1): page-table lookup, bilinear filtering of the RGBA8 physical
// texture with the tile border serving the out-of-core taps, and the HDR
// restore x^g * mu_hat(t, c).
//
// P:229  "During shading, we first sample the page table to locate each tile
//        within the physical texture, then sample the physical texture"
// P:232  gamma correction and per-channel mean normalisation before training;
//        the means "are later used during rendering to restore the original
//        lightmap data"; outputs stored as 8-bit 4-channel
// P:526  "To support hardware texture filtering, each tile is stored with a
//        small border"
// Readings R21-R25.  One thread per sample, grid-stride; the
// sample position and owning-tile decision are taken in fp64 (exact for fp32
// u, v and power-of-two or small atlas widths, and identical to the oracle's),
// the filter and the restore in fp32.  The path is bandwidth/latency bound:
// 8 B (u, v) + 4 B (atlas id) in, 12 B out, 16 B of cache taps (L1/L2-hot for
// coherent samples).
#include <cuda_runtime.h>

#include <cstdint>

#include "ndgi_common.cuh"

namespace ndgi {

struct SParams {
    const int32_t* pt;      // [tiles][2] (slot, bucket)
    const uint8_t* cache;   // [slots][P][P][4] RGBA8
    const float2* uv;       // [n]
    const uint32_t* atlas;  // [n] or nullptr (atlas 0)
    float* out;             // [n][3]
    uint32_t* err;
    uint32_t n, num_slots;
    int32_t bucket;
    int C, B, P, tiles_x, tiles_y, atlases;
    float g;
    float mu[kMaxSampleAtlases][3];
};

__global__ void __launch_bounds__(256) ndgi_sample_kernel(const __grid_constant__ SParams p) {
    const double W = (double)p.tiles_x * p.C, H = (double)p.tiles_y * p.C;
    const size_t slot_bytes = (size_t)p.P * p.P * 4;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += gridDim.x * blockDim.x) {
        const float2 q = __ldg(p.uv + i);
        const uint32_t a = p.atlas ? __ldg(p.atlas + i) : 0u;
        const double u = fmin(fmax((double)q.x, 0.0), 1.0);   // NaN -> 0 (fmax)
        const double v = fmin(fmax((double)q.y, 0.0), 1.0);
        int tx = (int)floor(u * p.tiles_x), ty = (int)floor(v * p.tiles_y);
        tx = tx > p.tiles_x - 1 ? p.tiles_x - 1 : tx;
        ty = ty > p.tiles_y - 1 ? p.tiles_y - 1 : ty;
        bool ok = a < (uint32_t)p.atlases;
        int slot = -1;
        if (ok) {
            const size_t id = ((size_t)a * p.tiles_y + ty) * p.tiles_x + tx;
            const int2 e = __ldg(reinterpret_cast<const int2*>(p.pt) + id);
            slot = e.x;
            ok = slot >= 0 && (uint32_t)slot < p.num_slots && e.y == p.bucket;
        }
        float* o = p.out + (size_t)3 * i;
        if (!ok) {
            o[0] = o[1] = o[2] = __int_as_float(0x7fc00000);   // NaN: not resident (counted)
            atomicAdd(p.err, 1u);
            continue;
        }
        const double lx = u * W - 0.5 - (double)tx * p.C;   // [-0.5, C - 0.5]
        const double ly = v * H - 0.5 - (double)ty * p.C;
        const double x0 = floor(lx), y0 = floor(ly);
        const float fx = (float)(lx - x0), fy = (float)(ly - y0);
        const uint32_t* s = reinterpret_cast<const uint32_t*>(p.cache + (size_t)slot * slot_bytes);
        const int px = (int)x0 + p.B, py = (int)y0 + p.B;
        const uint32_t* r0 = s + (size_t)py * p.P + px;
        const uint32_t t00 = __ldg(r0), t10 = __ldg(r0 + 1), t01 = __ldg(r0 + p.P), t11 = __ldg(r0 + p.P + 1);
        const float w00 = (1.f - fx) * (1.f - fy), w10 = fx * (1.f - fy), w01 = (1.f - fx) * fy, w11 = fx * fy;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int sh = 8 * c;
            const float val = (w00 * (float)((t00 >> sh) & 0xffu) + w10 * (float)((t10 >> sh) & 0xffu) +
                               w01 * (float)((t01 >> sh) & 0xffu) + w11 * (float)((t11 >> sh) & 0xffu)) *
                              (1.0f / 255.0f);
            o[c] = powf(val, p.g) * p.mu[a][c];
        }
    }
}

cudaError_t launch_sample(const SampleArgs& a, cudaStream_t s) {
    SParams p;
    p.pt = a.pt;
    p.cache = a.cache;
    p.uv = reinterpret_cast<const float2*>(a.uv);
    p.atlas = a.atlas;
    p.out = a.out;
    p.err = a.err;
    p.n = a.n;
    p.num_slots = a.num_slots;
    p.bucket = a.bucket;
    p.C = a.C;
    p.B = a.B;
    p.P = a.C + 2 * a.B;
    p.tiles_x = a.tiles_x;
    p.tiles_y = a.tiles_y;
    p.atlases = a.atlases;
    p.g = a.g;
    for (int k = 0; k < a.atlases && k < kMaxSampleAtlases; ++k)
        for (int c = 0; c < 3; ++c) p.mu[k][c] = a.mu[3 * k + c];
    const uint32_t per = 256u;
    uint32_t grid = (a.n + per - 1) / per;
    const uint32_t cap = (uint32_t)a.num_sms * 16u;   // grid-stride beyond 16 CTAs per SM
    if (grid > cap) grid = cap;
    if (grid == 0) grid = 1;
    ndgi_sample_kernel<<<grid, per, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace ndgi
