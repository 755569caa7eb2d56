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
#include <type_traits>

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

// byte c of an RGBA8 word as an exact float (0x4B000000 | b = 2^23 + b), no I2F
__device__ __forceinline__ float byte_to_float(uint32_t w, int c) {
    return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7650u + (uint32_t)c) ) - 8388608.0f;
}
__device__ __forceinline__ float log2f_fast(float x) {
    float r;
    asm("lg2.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float exp2f_fast(float x) {
    float r;
    asm("ex2.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// K samples per thread, strided by the grid width (coalesced per batch), with
// the three dependent loads of each sample (uv -> page table -> 4 taps) issued
// for all K before any is consumed: the chain is latency-, not issue-bound
constexpr int kSampleK = 4;

// POW2: atlas width and height are powers of two, so the tile decision
// floor(u * tiles_x) and u * W are exact in fp32 too and the position math
// runs in fp32 (the fractional weights then differ from fp64 by < 2^-24);
// otherwise fp64 (the oracle's decisions exactly)
template <bool POW2>
__global__ void __launch_bounds__(256) ndgi_sample_kernel(const __grid_constant__ SParams p) {
    using Pos = typename std::conditional<POW2, float, double>::type;
    const Pos W = (Pos)p.tiles_x * (Pos)p.C, H = (Pos)p.tiles_y * (Pos)p.C;
    const size_t slot_bytes = (size_t)p.P * p.P * 4;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x; base < p.n; base += stride * kSampleK) {
        float2 q[kSampleK];
        uint32_t a[kSampleK];
#pragma unroll
        for (int k = 0; k < kSampleK; ++k) {
            const uint32_t i = base + k * stride;
            q[k] = i < p.n ? __ldg(p.uv + i) : make_float2(0.f, 0.f);
            a[k] = (i < p.n && p.atlas) ? __ldg(p.atlas + i) : 0u;
        }
        int2 e[kSampleK];
        Pos lx[kSampleK], ly[kSampleK];
#pragma unroll
        for (int k = 0; k < kSampleK; ++k) {
            const Pos u = fmin(fmax((Pos)q[k].x, (Pos)0), (Pos)1);   // NaN -> 0 (fmax)
            const Pos v = fmin(fmax((Pos)q[k].y, (Pos)0), (Pos)1);
            int tx = (int)floor(u * (Pos)p.tiles_x), ty = (int)floor(v * (Pos)p.tiles_y);
            tx = tx > p.tiles_x - 1 ? p.tiles_x - 1 : tx;
            ty = ty > p.tiles_y - 1 ? p.tiles_y - 1 : ty;
            lx[k] = u * W - (Pos)0.5 - (Pos)tx * (Pos)p.C;   // [-0.5, C - 0.5]
            ly[k] = v * H - (Pos)0.5 - (Pos)ty * (Pos)p.C;
            const size_t id = ((size_t)(a[k] < (uint32_t)p.atlases ? a[k] : 0u) * p.tiles_y + ty) * p.tiles_x + tx;
            e[k] = __ldg(reinterpret_cast<const int2*>(p.pt) + id);
        }
        uint32_t t[kSampleK][4];
        bool ok[kSampleK];
#pragma unroll
        for (int k = 0; k < kSampleK; ++k) {
            ok[k] = base + k * stride < p.n && a[k] < (uint32_t)p.atlases && e[k].x >= 0 &&
                    (uint32_t)e[k].x < p.num_slots && e[k].y == p.bucket;
            const int slot = ok[k] ? e[k].x : 0;
            const uint32_t* s = reinterpret_cast<const uint32_t*>(p.cache + (size_t)slot * slot_bytes);
            const int px = (int)floor(lx[k]) + p.B, py = (int)floor(ly[k]) + p.B;
            const uint32_t* r0 = s + (size_t)py * p.P + px;
            if (ok[k]) {
                t[k][0] = __ldg(r0);
                t[k][1] = __ldg(r0 + 1);
                t[k][2] = __ldg(r0 + p.P);
                t[k][3] = __ldg(r0 + p.P + 1);
            } else {
                t[k][0] = t[k][1] = t[k][2] = t[k][3] = 0u;
            }
        }
#pragma unroll
        for (int k = 0; k < kSampleK; ++k) {
            const uint32_t i = base + k * stride;
            if (i >= p.n) break;
            float* o = p.out + (size_t)3 * i;
            if (!ok[k]) {
                o[0] = o[1] = o[2] = __int_as_float(0x7fc00000);   // NaN: not resident (counted)
                atomicAdd(p.err, 1u);
                continue;
            }
            const float fx = (float)(lx[k] - floor(lx[k])), fy = (float)(ly[k] - floor(ly[k]));
            const float w00 = (1.f - fx) * (1.f - fy), w10 = fx * (1.f - fy), w01 = (1.f - fx) * fy, w11 = fx * fy;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float val = (w00 * byte_to_float(t[k][0], c) + w10 * byte_to_float(t[k][1], c) +
                                   w01 * byte_to_float(t[k][2], c) + w11 * byte_to_float(t[k][3], c)) *
                                  (1.0f / 255.0f);
                // x^g = 2^(g log2 x) on the MUFU (rel. error ~1e-6 for x >= 1/255; 0 -> 0)
                o[c] = exp2f_fast(p.g * log2f_fast(val)) * p.mu[a[k]][c];
            }
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
    uint32_t grid = (a.n + per * kSampleK - 1) / (per * kSampleK);
    const uint32_t cap = (uint32_t)a.num_sms * 8u;   // grid-stride beyond 8 CTAs (2048 threads) per SM
    if (grid > cap) grid = cap;
    if (grid == 0) grid = 1;
    const uint32_t Wt = (uint32_t)(a.tiles_x * a.C), Ht = (uint32_t)(a.tiles_y * a.C);
    const bool pow2 = (Wt & (Wt - 1)) == 0 && (Ht & (Ht - 1)) == 0 && Wt <= (1u << 20) && Ht <= (1u << 20);
    if (pow2) ndgi_sample_kernel<true><<<grid, per, 0, s>>>(p);
    else ndgi_sample_kernel<false><<<grid, per, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace ndgi
