// fused_common.cuh -- pieces of the fused tile-decode kernel (fused_kernel.cu)
// and the reference/training kernels that share the prologue:
// TMEM/smem layouts, the GELU epilogue, the per-unit parameter prologue.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "bc7_device.cuh"
#include "bcn_device.cuh"
#include "ndgi_common.cuh"
#include "tc_ptx.cuh"

namespace ndgi {

constexpr int kChunkTexels = 2048;             // F_uv texels decoded per chunk (4 warps x 32 blocks x 16)

#ifndef NDGI_MIN_CTAS16
#define NDGI_MIN_CTAS16 8
#endif
#ifndef NDGI_SLOTS16
#define NDGI_SLOTS16 2
#endif

template <int H>
struct FusedCfg {
    static constexpr int K2 = H + 16;                    // layer 2/3 K incl. bias chunk
    // TMEM columns of one slot (32-bit columns, two f16 per column for A):
    //   [0, H/2)          GELU outputs = A of layers 2 and 3 (K = 0 .. H-1)
    //   [H/2, H/2 + 8)    the "feature chunk", K = H .. H+15 of layers 2/3 and
    //                     the whole A of layer 1 (K = 16), in the order
    //                     [1, 0 | V_ut | V_vt | 0, 0 | V_uvt (2 cols) | F_uv (2 cols)]
    //                     -- B2/B3 are zero past K = H (the bias row), so the
    //                     features ride along in layers 2/3 at no cost, and the
    //                     constant columns are written once per work unit
    //   [TM_D, TM_D + H)  fp32 accumulators
    static constexpr uint32_t TM_A23 = 0;
    static constexpr uint32_t TM_A1 = H / 2;
    static constexpr uint32_t TM_UVT = TM_A1 + 4;        // V_uvt, F_uv: per item
    static constexpr uint32_t TM_VT = TM_A1 + 2;         // V_vt: per row
    static constexpr uint32_t TM_D = H == 16 ? 16 : 64;  // H columns (fp32 accumulators)
    static constexpr uint32_t SLOT_COLS = H == 16 ? 32 : 128;
    static constexpr int SLOTS = H == 16 ? NDGI_SLOTS16 : 1;   // 128-texel items per MMA step (one TMEM slot each)
    static constexpr uint32_t TM_COLS = SLOTS * SLOT_COLS < 32 ? 32 : SLOTS * SLOT_COLS;
    static constexpr int MIN_CTAS = H == 16 ? NDGI_MIN_CTAS16 : 4;   // register budget: 64 / 128 per thread
    static constexpr int B1_BYTES = H * 16 * 2;
    static constexpr int B2_BYTES = H * K2 * 2;
    static constexpr int B3_BYTES = 16 * K2 * 2;
    static_assert(TM_A1 + 8 <= TM_D, "TMEM layout");
    static_assert(TM_D + H <= SLOT_COLS, "TMEM layout");
};

// layer-1 K position of Eq. 4 input j (R6: x = [V_uvt 0..3 | V_uv 4..7 | V_ut
// 8..9 | V_vt 10..11 | gamma 12..15]) in the TMEM feature chunk above; the
// bias (with gamma(t) folded) sits at K = 0, K = 1, 6, 7 hold zeros
__host__ __device__ constexpr int a1_k_of_input(int j) {
    return j < 4 ? 8 + j : (j < 8 ? 12 + (j - 4) : (j < 10 ? 2 + (j - 8) : 4 + (j - 10)));
}

// element (n, k) of a K-major no-swizzle operand with Kt columns:
// [n/8][k/8][n%8][k%8] halves -> LBO = 128 B, SBO = Kt/8 * 128 B
__device__ __forceinline__ int bofs(int n, int k, int Kt) {
    return (((n >> 3) * (Kt >> 3) + (k >> 3)) << 6) + ((n & 7) << 3) + (k & 7);
}

__device__ __forceinline__ uint32_t hsub2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t hfma2(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ uint32_t hmul2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
// a + f (b - a), packed
__device__ __forceinline__ uint32_t hlerp2(uint32_t a, uint32_t b, uint32_t f2) { return hfma2(f2, hsub2(b, a), a); }

// 4 u8 channels -> two f16x2 holding the integers 0..255 exactly
__device__ __forceinline__ void u8x4_to_h2(uint32_t q, uint32_t& rg, uint32_t& ba) {
    const uint32_t k1024 = 0x64006400u;  // f16x2(1024, 1024); 0x64XX = 1024 + XX
    rg = hsub2(__byte_perm(q, 0x64646464u, 0x5140u), k1024);
    ba = hsub2(__byte_perm(q, 0x64646464u, 0x7362u), k1024);
}

struct FusedSmem {
    // byte offsets from the dynamic smem base
    uint32_t b1, b2, b3, uvt, uvc, utcol, rowtab, colc, cnt, bars, tmem_slot, total;
};

template <int H>
__host__ __device__ inline FusedSmem fused_smem_layout(int C, int R3) {
    using Cfg = FusedCfg<H>;
    FusedSmem s{};
    uint32_t o = 0;
    // every offset but the total is a compile-time constant (H, C template
    // parameters): the R3-sized slice goes last
    s.b1 = o; o += Cfg::B1_BYTES;
    s.b2 = o; o += Cfg::B2_BYTES;
    s.b3 = o; o += Cfg::B3_BYTES;
    o = (o + 127) & ~127u;
    s.uvc = o; o += kChunkTexels * 4;                 // decoded F_uv chunk, RGBA8 (4 per-warp parts)
    s.utcol = o; o += (uint32_t)(C * 4);              // V_ut per column, f16x2
    o = (o + 15) & ~15u;
    s.rowtab = o; o += (uint32_t)(C * 16);            // per core row: y0*R3, y1*R3, fy (f16x2), V_vt (f16x2)
    s.colc = o; o += (uint32_t)(C * 16);              // per core column: x0 / x1 slice byte offsets, fx (f16x2), V_ut
    s.cnt = o; o += 8 * 4;                            // [0]: the CTA's claimed next unit (KParams::sched)
    s.bars = o; o += 8 * 8;                           // d_ready
    s.tmem_slot = o; o += 8;
    o = (o + 127) & ~127u;
    s.uvt = o; o += (uint32_t)(R3 * R3 * 8);         // blended slice, f16x4 per texel
    s.total = o;
    return s;
}

// ---- GELU epilogue of one layer: D (fp32) -> f16x2 GELU~ -> A23 ---------------
// Some of every 8 f16x2 GELU pairs run on the FMA pipe
// (gelu_poly_f16x2) instead of MUFU.TANH: the MUFU queue (mio_throttle) is the
// hot loop's main stall; 2 + 1 of the step's 16 measured best
#ifndef NDGI_POLY_PAIRS         // h = 16, the second item of a step: 3 of 8 (measured)
#define NDGI_POLY_PAIRS 3
#endif
#ifndef NDGI_POLY_PAIRS_ITEM0   // h = 16, the first item of a step: 3 of 8
#define NDGI_POLY_PAIRS_ITEM0 3
#endif
#ifndef NDGI_POLY_PAIRS64       // h = 64: 3 of every 8 (measured)
#define NDGI_POLY_PAIRS64 3
#endif
template <int H>
__device__ __forceinline__ void gelu_epilogue(uint32_t d_addr, uint32_t a_addr) {
#pragma unroll
    for (int c0 = 0; c0 < H; c0 += 16) {
        uint32_t d[16], g[8];
        ptx::tmem_ld_x16(d_addr + c0, d);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t x = pack_f16x2(__uint_as_float(d[2 * q]), __uint_as_float(d[2 * q + 1]));
            g[q] = q < 8 - NDGI_POLY_PAIRS64 ? gelu_scaled_f16x2(x) : gelu_poly_f16x2(x);
        }
        ptx::tmem_st_x8(a_addr + c0 / 2, g);
    }
}

// h = 16, S items: all accumulators loaded before one wait, 8*S independent
// GELU pairs in flight.  Layers 1-2 accumulate in fp32 (north_star: "fp16 in,
// fp32 accumulate"); NDGI_F16ACC=1 is an opt-in build with f16 accumulators
// read back packed (tcgen05.ld .pack::16b), kept only as a measured variant.
#ifndef NDGI_F16ACC
#define NDGI_F16ACC 0
#endif

// h = 16, S items with f16 accumulators (layers 1, 2): tcgen05.ld .pack::16b
// delivers the 16 pre-activations as 8 f16x2 words -- no fp32 -> f16 packing
template <int S>
__device__ __forceinline__ void gelu_epilogue_h16_f16acc(uint32_t d0, uint32_t a0, uint32_t stride) {
    uint32_t x[S][8];
#pragma unroll
    for (int s = 0; s < S; ++s) ptx::tmem_ld_x8_pack16(d0 + s * stride, x[s]);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int s = 0; s < S; ++s) {
        uint32_t g[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
            g[q] = q < 8 - (s == 0 ? NDGI_POLY_PAIRS_ITEM0 : NDGI_POLY_PAIRS) ? gelu_scaled_f16x2(x[s][q])
                                                                            : gelu_poly_f16x2(x[s][q]);
        ptx::tmem_st_x8(a0 + s * stride, g);
    }
}

// h = 16, S items with fp32 accumulators: one cvt.rn.f16x2.f32 per pair, then
// the same GELU split as above
template <int S>
__device__ __forceinline__ void gelu_epilogue_h16(uint32_t d0, uint32_t a0, uint32_t stride) {
    uint32_t x[S][16];
#pragma unroll
    for (int s = 0; s < S; ++s) ptx::tmem_ld_x16(d0 + s * stride, x[s]);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int s = 0; s < S; ++s) {
        uint32_t g[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t h = pack_f16x2(__uint_as_float(x[s][2 * q]), __uint_as_float(x[s][2 * q + 1]));
            g[q] = q < 8 - (s == 0 ? NDGI_POLY_PAIRS_ITEM0 : NDGI_POLY_PAIRS) ? gelu_scaled_f16x2(h)
                                                                            : gelu_poly_f16x2(h);
        }
        ptx::tmem_st_x8(a0 + s * stride, g);
    }
}

// ---- F_uvt ring (large R3, C = 128): instead of the whole tau-blended slice
// (R3^2 x 8 B = 32 KB for the H profile, which would halve residency), the CTA
// keeps a ring of `rows` F_uvt rows (all R3 columns; row y in ring row
// y mod rows) covering the rows one F_uv chunk samples, and stages the new
// block rows at each chunk start with all 128 threads (one block row of one
// 4x4 block of both slices per thread).
struct UvtRing {
    int rows;          // ring rows: a power of two, 4 x the block rows a chunk can span
    uint32_t pitch;    // bytes per ring row (R3 x f16x4)
    uint32_t bytes;
};
__host__ __device__ inline UvtRing uvt_ring(int R3, int C, int chunk_rows) {
    UvtRing w;
    int brows = (chunk_rows * R3 / C + 2 + 3) / 4 + 1;   // F_uvt rows of a chunk (+ bilinear, misalignment)
    while (brows & (brows - 1)) ++brows;
    w.rows = 4 * brows;
    w.pitch = (uint32_t)R3 * 8u;
    w.bytes = (uint32_t)w.rows * w.pitch;
    return w;
}

// ---- load-time weight prepack ------------------------------------------------
// Per tile, the t-independent part of the three tcgen05 B operands with the
// GELU folds of DESIGN.md §6.1, already in the smem layout (bofs), followed by
// [b1[n], W1[n][12..15]] as fp32 for the per-call gamma(t) fold into layer-1's
// bias column (k = 12, left 0 here).  Built once by ndgi_load; a work unit
// then moves it to smem with one coalesced 16-B copy per thread.
template <int H>
struct WPack {
    using Cfg = FusedCfg<H>;
    static constexpr uint32_t B_BYTES = Cfg::B1_BYTES + Cfg::B2_BYTES + Cfg::B3_BYTES;
    static constexpr uint32_t G_BYTES = ((uint32_t)H * 5 * 4 + 15u) & ~15u;
    static constexpr uint32_t BYTES = B_BYTES + G_BYTES;
};

template <int H>
__global__ void prep_weights_kernel(const uint16_t* __restrict__ mlp, size_t tile_elems, float s_uv,
                                    uint8_t* __restrict__ out, int num_tiles) {
    using Cfg = FusedCfg<H>;
    const float a = kGeluA;
    for (int k = blockIdx.x; k < num_tiles; k += gridDim.x) {
        const uint16_t* w = mlp + tile_elems * k;
        const uint16_t *W1 = w, *b1 = W1 + 16 * H, *W2 = b1 + H, *b2 = W2 + H * H, *W3 = b2 + H, *b3 = W3 + 3 * H;
        uint8_t* o = out + (size_t)WPack<H>::BYTES * k;
        __half* B1 = reinterpret_cast<__half*>(o);
        __half* B2 = reinterpret_cast<__half*>(o + Cfg::B1_BYTES);
        __half* B3 = reinterpret_cast<__half*>(o + Cfg::B1_BYTES + Cfg::B2_BYTES);
        float* G = reinterpret_cast<float*>(o + WPack<H>::B_BYTES);
        for (int e = threadIdx.x; e < H * 16; e += blockDim.x) {
            const int n = e >> 4, j = e & 15;   // Eq. 4 input j; gamma (j >= 12) and b1 go to K = 0 per call
            if (j < 12) B1[bofs(n, a1_k_of_input(j), 16)] = __float2half_rn(half_bits_to_float(W1[n * 16 + j]) * ((j >= 4 && j < 8) ? s_uv : a));
            else B1[bofs(n, j == 12 ? 0 : (j == 13 ? 1 : j - 8), 16)] = __float2half_rn(0.f);   // K = 0, 1, 6, 7
        }
        for (int e = threadIdx.x; e < H * Cfg::K2; e += blockDim.x) {
            const int n = e / Cfg::K2, kk = e % Cfg::K2;
            float v = 0.f;
            if (kk < H) v = 0.5f * half_bits_to_float(W2[n * H + kk]);
            else if (kk == H) v = a * half_bits_to_float(b2[n]);
            B2[bofs(n, kk, Cfg::K2)] = __float2half_rn(v);
        }
        for (int e = threadIdx.x; e < 16 * Cfg::K2; e += blockDim.x) {
            const int n = e / Cfg::K2, kk = e % Cfg::K2;
            float v = 0.f;
            if (n < 3) {
                if (kk < H) v = half_bits_to_float(W3[n * H + kk]) * (0.5f / a);
                else if (kk == H) v = half_bits_to_float(b3[n]);
            }
            B3[bofs(n, kk, Cfg::K2)] = __float2half_rn(v);
        }
        for (int e = threadIdx.x; e < H * 5; e += blockDim.x) {
            const int n = e / 5, g = e % 5;
            G[e] = half_bits_to_float(g == 0 ? b1[n] : W1[n * 16 + 11 + g]);
        }
    }
}

// the prepacked B operands of tile k -> smem (L.b1, L.b2, L.b3 are contiguous),
// patching layer-1's bias column (K = 0) with a (b1 + W1_gamma gamma(t)) (R6) on the way
template <int H>
__device__ __forceinline__ void copy_prepacked_weights(const KParams& p, const TConst& tc, int k, uint8_t* smem,
                                                       const FusedSmem& L, int tid, int nthr) {
    using Cfg = FusedCfg<H>;
    const uint8_t* base = p.wpack + (size_t)WPack<H>::BYTES * k;
    const uint4* src = reinterpret_cast<const uint4*>(base);
    const float* G = reinterpret_cast<const float*>(base + WPack<H>::B_BYTES);
    uint4* dst = reinterpret_cast<uint4*>(smem + L.b1);
    for (int c = tid; c < (int)(WPack<H>::B_BYTES / 16); c += nthr) {
        uint4 v = __ldg(src + c);
        if (c < Cfg::B1_BYTES / 16 && !((c >> 3) & 1)) {
            // this chunk is k = 0..7 of B1 row n: element k = 0 is v.x's low half
            const int n = (c >> 4) * 8 + (c & 7);
            float acc = __ldg(G + n * 5);
#pragma unroll
            for (int g = 0; g < 4; ++g) acc = fmaf(__ldg(G + n * 5 + 1 + g), tc.gamma[g], acc);
            const uint32_t hb = (uint32_t)__half_as_ushort(__float2half_rn(kGeluA * acc));
            v.x = (v.x & 0xffff0000u) | hb;
        }
        dst[c] = v;
    }
}

// a2 for decode_tiles (VT): the same results as copy_prepacked_weights +
// unit_prologue for BC7 F_uvt (R3 <= 32) and u8 line maps, restructured for
// latency -- a small VT batch runs one unit per CTA and waits on it.  Every
// global read of the unit (weights, both slices' F_uvt blocks, the line-map
// taps) is issued before any is consumed (one HBM latency instead of three),
// and the F_uvt blocks are decoded one per thread (both slices over all 128
// threads) into `scratch` (>= 2 * (R3/4)^2 * 64 B: the F_uv chunk buffer, free
// here), then blended 8 texels per thread after a CTA barrier.
template <int H, int C>
__device__ __forceinline__ void unit_prologue_vt(const KParams& p, const TConst& tc, int k, uint8_t* smem,
                                                 const FusedSmem& L, int tid, uint8_t* scratch) {
    using Cfg = FusedCfg<H>;
    constexpr int NW = (int)(WPack<H>::B_BYTES / 16);   // 16-B chunks of the B operands
    static_assert(NW <= 2 * 128 && Cfg::B1_BYTES / 16 <= 128, "two chunks per thread, B1 in the first");
    const int R3 = p.R3, nbx = R3 >> 2, nb = nbx * nbx;
    // ---- issue every load of the unit
    const uint8_t* wbase = p.wpack + (size_t)WPack<H>::BYTES * k;
    const uint4* wsrc = reinterpret_cast<const uint4*>(wbase);
    const uint4 w0 = tid < NW ? __ldg(wsrc + tid) : make_uint4(0u, 0u, 0u, 0u);
    const uint4 w1 = tid + 128 < NW ? __ldg(wsrc + tid + 128) : make_uint4(0u, 0u, 0u, 0u);
    // the threads that patch layer 1's bias column (chunk tid holds K = 0 of B1
    // row n) fetch [b1[n], W1[n][12..15]] now as well
    const float* G = reinterpret_cast<const float*>(wbase + WPack<H>::B_BYTES);
    const bool patch = tid < Cfg::B1_BYTES / 16 && !((tid >> 3) & 1);
    const int pn = (tid >> 4) * 8 + (tid & 7);
    float g5[5];
#pragma unroll
    for (int g = 0; g < 5; ++g) g5[g] = patch ? __ldg(G + pn * 5 + g) : 0.f;
    const int sl = tid >= nb, bi = tid - (sl ? nb : 0);   // this thread's F_uvt item (slice, block)
    const bool fitem = tid < 2 * nb;
    const uint8_t* vol = p.uvt + p.uvt_tile_bytes * k;
    const uint4 fblk = fitem ? __ldg(reinterpret_cast<const uint4*>(vol + p.uvt_slice_bytes * (sl ? tc.k1 : tc.k0)) + bi)
                             : make_uint4(0u, 0u, 0u, 0u);
    const float scu = (float)p.U * (1.0f / (float)C);
    const uint8_t* ut = p.ut + p.line_tile_bytes * k;
    const uint8_t* vt = p.vt + p.line_tile_bytes * k;
    uint32_t lt[2][4];   // per line entry e = tid, tid + 128: (x0, r0), (x1, r0), (x0, r1), (x1, r1) as u8 pairs
    float lfx[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int e = tid + 128 * h, i = e % C;
        const uint8_t* m = e < C ? ut : vt;
        const float sx = fmaf((float)i + 0.5f, scu, -0.5f);
        const float fl = floorf(sx);
        lfx[h] = sx - fl;
        const int x0 = clampi((int)fl, 0, p.U - 1), x1 = clampi((int)fl + 1, 0, p.U - 1);
        const uint16_t* mh = reinterpret_cast<const uint16_t*>(m);
        lt[h][0] = __ldg(mh + tc.r0 * p.U + x0);
        lt[h][1] = __ldg(mh + tc.r0 * p.U + x1);
        lt[h][2] = __ldg(mh + tc.r1 * p.U + x0);
        lt[h][3] = __ldg(mh + tc.r1 * p.U + x1);
    }
    // ---- weights -> smem (gamma(t) folded into layer 1's bias, as copy_prepacked_weights)
    {
        uint4* dst = reinterpret_cast<uint4*>(smem + L.b1);
        if (tid < NW) {
            uint4 v = w0;
            if (patch) {
                float acc = g5[0];
#pragma unroll
                for (int g = 0; g < 4; ++g) acc = fmaf(g5[1 + g], tc.gamma[g], acc);
                const uint32_t hb = (uint32_t)__half_as_ushort(__float2half_rn(kGeluA * acc));
                v.x = (v.x & 0xffff0000u) | hb;
            }
            dst[tid] = v;
        }
        if (tid + 128 < NW) dst[tid + 128] = w1;   // chunks >= 128 are past B1 (no patch)
    }
    // ---- F_uvt: one block per thread -> scratch (raw RGBA8, 64 B per item)
    if (fitem) {
        uint32_t t16[16];
        bc7_decode(fblk, [&](int i, uint32_t v) { t16[i] = v; });
        uint4* d = reinterpret_cast<uint4*>(scratch + (size_t)tid * 64);
#pragma unroll
        for (int r = 0; r < 4; ++r) d[r] = make_uint4(t16[4 * r], t16[4 * r + 1], t16[4 * r + 2], t16[4 * r + 3]);
    }
    // ---- line maps (R5) from the preloaded taps
    {
        uint32_t* sUt = reinterpret_cast<uint32_t*>(smem + L.utcol);
        uint4* sRow = reinterpret_cast<uint4*>(smem + L.rowtab);
        const float rho = tc.rho, omr = 1.0f - rho;
        const float sc3 = (float)R3 * (1.0f / (float)C);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = tid + 128 * h, i = e % C;
            const float fx = lfx[h];
            float c[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const float v00 = u8f(lt[h][0], q), v10 = u8f(lt[h][1], q), v01 = u8f(lt[h][2], q),
                            v11 = u8f(lt[h][3], q);
                const float v = (1.f - fx) * omr * v00 + fx * omr * v10 + (1.f - fx) * rho * v01 + fx * rho * v11;
                c[q] = v * (1.0f / 255.0f);
            }
            if (e < C) {
                sUt[i] = pack_f16x2(c[0], c[1]);
            } else {
                const float sy = fmaf((float)i + 0.5f, sc3, -0.5f);
                const float fly = floorf(sy);
                const int y0 = clampi((int)fly, 0, R3 - 1), y1 = clampi((int)fly + 1, 0, R3 - 1);
                sRow[i] = make_uint4((uint32_t)y0 * R3 * 8u, (uint32_t)y1 * R3 * 8u, pack_f16x2(sy - fly, sy - fly),
                                     pack_f16x2(c[0], c[1]));
            }
        }
    }
    ndgi_jitter(9u);
    __syncthreads();   // scratch complete
    // ---- tau-blend both slices -> the f16x4 slice (R4, R17), same arithmetic as unit_prologue
    {
        uint2* sUvt = reinterpret_cast<uint2*>(smem + L.uvt);
        const float tau = tc.tau, omt = 1.0f - tau;
        const uint32_t* sc = reinterpret_cast<const uint32_t*>(scratch);
        for (int e = tid; e < R3 * R3; e += 128) {
            const int y = e / R3, x = e % R3;
            const int b = (y >> 2) * nbx + (x >> 2), i = (y & 3) * 4 + (x & 3);
            const uint32_t q0 = sc[b * 16 + i], q1 = sc[(nb + b) * 16 + i];
            float c[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) c[q] = (omt * u8f(q0, q) + tau * u8f(q1, q)) * (1.0f / 255.0f);
            sUvt[e] = make_uint2(pack_f16x2(c[0], c[1]), pack_f16x2(c[2], c[3]));
        }
    }
}

// a2: one unit's feature parameters -> shared memory: the tau-blended F_uvt
// slice, V_ut per column and the per-row gather table (F_uvt y taps, V_vt)
// (the MLP's B operands come prepacked: copy_prepacked_weights).
// Executed by threads tid = 0 .. nthr-1 of the CTA.
// win_pitch == 0: the whole tau-blended F_uvt slice goes to smem (row offsets
// y * R3 * 8); > 0: the kernel stages a ring of win_rows (a power of two)
// F_uvt rows itself (UvtRing) and the row table holds ring-row offsets
template <int H, int FMT_UV, int C>
__device__ __forceinline__ void unit_prologue(const KParams& p, const TConst& tc, int k, uint8_t* smem,
                                              const FusedSmem& L, int tid, int nthr, uint32_t win_pitch = 0,
                                              int win_rows = 0) {
    const int R3 = p.R3;
    const float sc3 = (float)R3 * (1.0f / (float)C);
    uint2* sUvt = reinterpret_cast<uint2*>(smem + L.uvt);
    uint32_t* sUt = reinterpret_cast<uint32_t*>(smem + L.utcol);
    uint4* sRow = reinterpret_cast<uint4*>(smem + L.rowtab);
        {
            // F_uvt slices k0, k1 blended with tau (R4, R17) -> f16x4 [R3][R3], values in [0,1]
            const uint8_t* vol = p.uvt + p.uvt_tile_bytes * k;
            const float tau = tc.tau, omt = 1.0f - tau;
            if (win_pitch) {
                // windowed: staged per chunk by the kernel
            } else if (fmt_block4(p.fmt_uvt)) {
                const int nbx = R3 >> 2, nb = nbx * nbx;
                const uint8_t* s0 = vol + p.uvt_slice_bytes * tc.k0;
                const uint8_t* s1 = vol + p.uvt_slice_bytes * tc.k1;
                for (int bi = tid; bi < nb; bi += nthr) {
                    uint32_t t0[16], t1[16];
                    block4_decode(p.fmt_uvt, s0, bi, [&](int i, uint32_t v) { t0[i] = v; });
                    block4_decode(p.fmt_uvt, s1, bi, [&](int i, uint32_t v) { t1[i] = v; });
                    const int bx = bi % nbx, by = bi / nbx;
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        float c[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            c[q] = (omt * u8f(t0[i], q) + tau * u8f(t1[i], q)) *
                                   (1.0f / 255.0f);
                        NDGI_CHECK((by * 4 + (i >> 2)) * R3 + bx * 4 + (i & 3) < R3 * R3);
                        sUvt[(by * 4 + (i >> 2)) * R3 + bx * 4 + (i & 3)] = make_uint2(pack_f16x2(c[0], c[1]), pack_f16x2(c[2], c[3]));
                    }
                }
            } else {
                const int ntex = R3 * R3;
                for (int e = tid; e < ntex; e += nthr) {
                    float c[4];
                    if (p.fmt_uvt == FMT_U8) {
                        const uint32_t q0 = __ldg(reinterpret_cast<const uint32_t*>(vol + p.uvt_slice_bytes * tc.k0) + e);
                        const uint32_t q1 = __ldg(reinterpret_cast<const uint32_t*>(vol + p.uvt_slice_bytes * tc.k1) + e);
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            c[q] = (omt * u8f(q0, q) + tau * u8f(q1, q)) * (1.0f / 255.0f);
                    } else {
                        const uint16_t* h0 = reinterpret_cast<const uint16_t*>(vol + p.uvt_slice_bytes * tc.k0) + 4 * e;
                        const uint16_t* h1 = reinterpret_cast<const uint16_t*>(vol + p.uvt_slice_bytes * tc.k1) + 4 * e;
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            c[q] = omt * half_bits_to_float(__ldg(h0 + q)) + tau * half_bits_to_float(__ldg(h1 + q));
                    }
                    sUvt[e] = make_uint2(pack_f16x2(c[0], c[1]), pack_f16x2(c[2], c[3]));
                }
            }
            // line maps (R5): V_ut(u_i) per core column i, V_vt(v_j) per core row j
            const uint8_t* ut = p.ut + p.line_tile_bytes * k;
            const uint8_t* vt = p.vt + p.line_tile_bytes * k;
            const float rho = tc.rho, omr = 1.0f - rho;
            const float scu = (float)p.U * (1.0f / (float)C);
            for (int e = tid; e < 2 * C; e += nthr) {
                const int i = e % C;
                const uint8_t* m = e < C ? ut : vt;
                const float sx = fmaf((float)i + 0.5f, scu, -0.5f);
                const float fl = floorf(sx), fx = sx - fl;
                const int x0 = clampi((int)fl, 0, p.U - 1), x1 = clampi((int)fl + 1, 0, p.U - 1);
                NDGI_CHECK(tc.r0 >= 0 && tc.r1 < p.T && tc.k0 >= 0 && tc.k1 < p.D);
                float c[2];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    float v00, v10, v01, v11;
                    if (p.fmt_line == FMT_U8) {
                        v00 = u8f(__ldg(m + (tc.r0 * p.U + x0) * 2 + q), 0);
                        v10 = u8f(__ldg(m + (tc.r0 * p.U + x1) * 2 + q), 0);
                        v01 = u8f(__ldg(m + (tc.r1 * p.U + x0) * 2 + q), 0);
                        v11 = u8f(__ldg(m + (tc.r1 * p.U + x1) * 2 + q), 0);
                    } else if (p.fmt_line == FMT_BC5) {
                        v00 = u8f(bc5_texel_at(m, p.U, x0, tc.r0), q);
                        v10 = u8f(bc5_texel_at(m, p.U, x1, tc.r0), q);
                        v01 = u8f(bc5_texel_at(m, p.U, x0, tc.r1), q);
                        v11 = u8f(bc5_texel_at(m, p.U, x1, tc.r1), q);
                    } else {
                        const uint16_t* mh = reinterpret_cast<const uint16_t*>(m);
                        v00 = half_bits_to_float(__ldg(mh + (tc.r0 * p.U + x0) * 2 + q));
                        v10 = half_bits_to_float(__ldg(mh + (tc.r0 * p.U + x1) * 2 + q));
                        v01 = half_bits_to_float(__ldg(mh + (tc.r1 * p.U + x0) * 2 + q));
                        v11 = half_bits_to_float(__ldg(mh + (tc.r1 * p.U + x1) * 2 + q));
                    }
                    float v = (1.f - fx) * omr * v00 + fx * omr * v10 + (1.f - fx) * rho * v01 + fx * rho * v11;
                    c[q] = p.fmt_line != FMT_F16 ? v * (1.0f / 255.0f) : v;   // U8, BC5: q/255 (R8)
                }
                if (e < C) {
                    sUt[i] = pack_f16x2(c[0], c[1]);
                } else {
                    // per-row gather table: F_uvt y taps and weight, V_vt
                    const float sy = fmaf((float)i + 0.5f, sc3, -0.5f);
                    const float fly = floorf(sy);
                    const int y0 = clampi((int)fly, 0, R3 - 1), y1 = clampi((int)fly + 1, 0, R3 - 1);
                    // whole slice: row y at y * R3 * 8; window: ring row y mod (win_rows)
                    const uint32_t r0 = win_pitch ? (uint32_t)(y0 & (win_rows - 1)) * win_pitch : (uint32_t)y0 * R3 * 8u;
                    const uint32_t r1 = win_pitch ? (uint32_t)(y1 & (win_rows - 1)) * win_pitch : (uint32_t)y1 * R3 * 8u;
                    sRow[i] = make_uint4(r0, r1, pack_f16x2(sy - fly, sy - fly), pack_f16x2(c[0], c[1]));
                }
            }
        }
}

}  // namespace ndgi
