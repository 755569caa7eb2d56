// ndgi_common.cuh -- kernel-side parameter block and small helpers shared by
// the CUDA kernels of libndgi.so (never by the oracle).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_fp16.h>

namespace ndgi {

enum : int { FMT_BC7 = 0, FMT_U8 = 1, FMT_F16 = 2, FMT_BC1 = 3, FMT_BC3 = 4, FMT_BC5 = 5 };
// kernel-internal: BC7 F_uv fetched through the texture unit (NDGI_MODE_FAST_TEXUNIT)
constexpr int FMT_BC7_TEX = 16;
constexpr int kMaxTexAtlases = 64;
enum : int { OUT_RGBA8 = 0, OUT_RGBA16F = 1, OUT_RGBA32F = 2 };
enum : int { GELU_ERF = 0, GELU_TANH = 1 };
enum : int { BORDER_MIRROR = 0, BORDER_EVAL_CLAMP = 1 };

constexpr int kMaxT = 32;   // query times per launch
constexpr uint32_t kSchedSlots = 1024;   // dynamic-scheduling counters per context (KParams::sched)

struct TConst {
    float t;
    float gamma[4];      // Eq. 4: sin(pi t), cos(pi t), sin(2 pi t), cos(2 pi t)
    int k0, k1;          // F_uvt slices (R4)
    float tau;
    int r0, r1;          // F_ut/F_vt rows (R5)
    float rho;
};

// Everything a decode launch needs, passed by value (__grid_constant__).
struct KParams {
    // layout (include/ndgi.h)
    int C, B, P, R_uv, R3, D, U, T, H;
    int fmt_uv, fmt_uvt, fmt_line, gelu, border_mode;
    int atlases, tiles_x, tiles_y, num_tiles;
    // Theta, device, tile-major
    const uint8_t* uv;
    const uint8_t* uvt;
    const uint8_t* ut;
    const uint8_t* vt;
    const uint16_t* mlp;
    const uint8_t* wpack;       // per-tile prepacked tcgen05 B operands (ndgi_load), or nullptr
    unsigned long long uvtex[kMaxTexAtlases];   // NDGI_MODE_FAST_TEXUNIT: BC7 F_uv texture per atlas
    size_t uv_tile_bytes, uvt_tile_bytes, uvt_slice_bytes, line_tile_bytes, mlp_tile_elems;
    // per-call constants (call setup), one set per query time,
    // computed on the host in fp64
    int nt;
    TConst tc[kMaxT];
    size_t out_t_stride;        // decode_full: texels per atlas set (one t)
    // requests
    const uint32_t* tile_ids;   // decode_tiles; nullptr for decode_full
    const uint32_t* slots;      // nullptr -> slot = request index
    uint32_t n_req, num_slots;
    int full;                   // 1: decode_full (atlas addressing, core only)
    // output
    void* out;
    int out_fmt;
    uint32_t* err;              // device error counter
    // work decomposition of the fused kernel
    int strip_rows;             // rows of core per work unit
    int strips_per_tile;
    uint32_t units;             // tail_from + tail_strips * (requests past it)
    // the launch's last requests are split finer (tail_strips strips each) so
    // the final dynamically claimed units are short: units >= tail_from are
    // (request tail_req0 + v / tail_strips, strip v % tail_strips), v = unit - tail_from
    uint32_t tail_from;
    int tail_strips;
    // dynamic unit scheduling (fused kernel, units > grid): a zeroed counter of
    // this launch; CTA b takes unit b, then gridDim.x + atomicAdd(sched, 1)
    // until the units run out -- co-resident CTAs progress at different rates
    // (warp-scheduler priority), so a static unit += gridDim.x split leaves the
    // SMs half-occupied for the second half of the launch
    uint32_t* sched;
};

// shading-side sampling (sample_kernel.cu)
constexpr int kMaxSampleAtlases = 64;
struct SampleArgs {
    const int32_t* pt;
    const uint8_t* cache;
    const float* uv;
    const uint32_t* atlas;
    float* out;
    uint32_t* err;
    uint32_t n, num_slots;
    int32_t bucket;
    int C, B, tiles_x, tiles_y, atlases, num_sms;
    float g;
    const float* mu;   // host [atlases][3], mu_hat at the call's t
};

// fine-tuning step (train_kernel.cu)
struct TrainArgs {
    // maps (as KParams)
    const uint8_t *uv, *uvt, *ut, *vt;
    size_t uv_tile_bytes, uvt_tile_bytes, uvt_slice_bytes, line_tile_bytes;
    int fmt_uv, fmt_uvt, fmt_line, R_uv, R3, D, U, T, gelu, num_tiles;
    // batch
    const uint32_t* tile_ids;   // [n]
    const float* samples;       // [n][S][3] (u, v, t)
    const float* targets;       // [n][S][3]
    int n, S, chunks;
    // state
    float* theta;               // [num_tiles][P] fp32 master weights (FULL: [num_tiles][P_full])
    // FULL (R28): BC-simulated maps + line grids in theta after the MLP; noise [n][S][12]
    const float* noise;
    size_t pfull, off_uv, off_uvt, off_ut, off_vt;
    // FULL: per batch row, dL/d(texel) of each map, vector atomics:
    // [R_uv^2][4] | [D][R3^2][4] | [T][U][2] (ut) | [T][U][2] (vt)
    float* dtex;
    size_t dtex_stride;
    float* grad;                // [n][P] (zeroed by the host)
    float* loss;                // [n] (zeroed by the host), mean squared error
    uint32_t* err;
};

__device__ __forceinline__ int clampi(int x, int lo, int hi) { return x < lo ? lo : (x > hi ? hi : x); }

// ---- self-checking builds (compute-sanitizer is not available on this pool) --
// NDGI_CHECKED=1: every shared-memory index and every global read / write
// offset of the fused kernel is checked against its buffer; a violation traps
// (the launch then fails with cudaErrorLaunchFailure / illegal instruction).
// NDGI_JITTER=1: pseudo-random per-warp delays (0..~2 us) at every
// synchronisation point, so a missing barrier or an aliasing race shows up as
// a nondeterministic output; tests require bit-equality with the product build.
#ifndef NDGI_CHECKED
#define NDGI_CHECKED 0
#endif
#ifndef NDGI_JITTER
#define NDGI_JITTER 0
#endif
#if NDGI_CHECKED
#define NDGI_CHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define NDGI_CHECK(cond) do {} while (0)
#endif
__device__ __forceinline__ void ndgi_jitter(uint32_t salt) {
#if NDGI_JITTER
    uint32_t h = (uint32_t)clock() * 0x9E3779B1u ^ (salt * 0x85EBCA6Bu) ^ ((threadIdx.x >> 5) * 0xC2B2AE35u) ^
                 (blockIdx.x * 0x27D4EB2Fu);
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    if (h & 1u) __nanosleep(h >> 21);   // 0 .. ~2 us
#else
    (void)salt;
#endif
}

__device__ __forceinline__ float half_bits_to_float(uint16_t h) {
    return __half2float(__ushort_as_half(h));
}

// byte c of `word` as an exact fp32 without I2F (which issues on the XU/MUFU
// pipe the GELUs saturate): the bits 0x4B0000qq are 2^23 + q, minus 2^23
__device__ __forceinline__ float u8f(uint32_t word, int c) {
    return __int_as_float(__byte_perm(word, 0x4B000000u, 0x7540u | (uint32_t)c)) - 8388608.0f;
}

// mirror a core coordinate, reflect without repeating the edge (R3)
__device__ __forceinline__ int mirror_core(int i, int C) {
    if (i < 0) i = -i;
    if (i >= C) i = 2 * (C - 1) - i;
    return i;
}

// RGBA8 texel on the FMA pipe (no F2I on the XU/MUFU pipe): clamp to [0,1],
// then t*255 + 1.5*2^23 rounds the exact product to the nearest integer, ties
// to even, into the low mantissa bits (R12); A = 255.
__device__ __forceinline__ uint32_t rgba8_fma(float r, float g, float b) {
    const uint32_t qr = __float_as_uint(fmaf(__saturatef(r), 255.0f, 12582912.0f));
    const uint32_t qg = __float_as_uint(fmaf(__saturatef(g), 255.0f, 12582912.0f));
    // blue on the negative side: -(1.5 * 2^23 + RN-even(255 b)) has the same low
    // byte (round-to-nearest-even is symmetric) and a sign byte 0xCB, whose
    // replicated MSB is A = 255 -- two PRMTs, no constant
    const uint32_t qb = __float_as_uint(fmaf(__saturatef(b), -255.0f, -12582912.0f));
    // (prmt's sign-replicating selector bit; __byte_perm masks selectors to 3 bits)
    uint32_t v;
    asm("prmt.b32 %0, %1, %2, 0xF410;" : "=r"(v) : "r"(__byte_perm(qr, qg, 0x0040u)), "r"(qb));
    return v;
}

__device__ __forceinline__ void store_texel(void* out, size_t idx, int fmt, float r, float g, float b) {
    if (fmt == OUT_RGBA8) {
        reinterpret_cast<uint32_t*>(out)[idx] = rgba8_fma(r, g, b);
    } else if (fmt == OUT_RGBA16F) {
        __half2 rg = __floats2half2_rn(r, g), ba = __floats2half2_rn(b, 1.0f);
        uint2 v;
        v.x = *reinterpret_cast<uint32_t*>(&rg);
        v.y = *reinterpret_cast<uint32_t*>(&ba);
        reinterpret_cast<uint2*>(out)[idx] = v;
    } else {
        reinterpret_cast<float4*>(out)[idx] = make_float4(r, g, b, 1.0f);
    }
}

}  // namespace ndgi

namespace ndgi {

// ---------------------------------------------------------------------------
// GELU in the fused kernel (FAST mode, reading R7): tanh form on packed f16x2
// with the constants folded into the neighbouring layers' weights.
//   With a = sqrt(2/pi) and z~ = a z (the layer's MMA produces z~ directly):
//   tanh-GELU(z) = 0.5 z (1 + tanh(a (z + 0.044715 z^3)))
//                = g~ / (2a),   g~ = z~ (1 + tanh(z~ (1 + c z~^2))),  c = 0.044715/a^2
//   so each hidden activation costs HMUL2, HFMA2, HMUL2, MUFU.TANH, HFMA2
//   per two values, and 1/(2a) moves into the next layer's weights.
// ---------------------------------------------------------------------------
constexpr float kGeluA = 0.7978845608028654f;        // sqrt(2/pi)
constexpr float kGeluC = 0.044715f / (0.7978845608028654f * 0.7978845608028654f);

__device__ __forceinline__ uint32_t gelu_scaled_f16x2(uint32_t h) {
    const uint32_t c2 = 0x2C7F2C7Fu;   // f16x2(c), c = 0.0702382 -> f16 0.07025
    const uint32_t one2 = 0x3C003C00u; // f16x2(1.0)
    uint32_t s, p, u, t, g;
    asm("mul.rn.f16x2 %0, %1, %1;" : "=r"(s) : "r"(h));
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(p) : "r"(s), "r"(c2), "r"(one2));
    asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(u) : "r"(h), "r"(p));
    asm("tanh.approx.f16x2 %0, %1;" : "=r"(t) : "r"(u));
    asm("fma.rn.f16x2 %0, %1, %2, %1;" : "=r"(g) : "r"(h), "r"(t));
    return g;
}

// GELU~ on the FMA pipe (NDGI_POLY_PAIRS): g = h + (h hc) Q(hc^2),
// hc = clamp(h, +-2.5), h Q(h^2) an odd near-minimax fit of tanh(h (1 + c h^2))
// on [0, 2.5] with f16 coefficients: degree 9 (Q of degree 4, max error 9.3e-4
// over all h including the clamped tail, the size of tanh.approx.f16's own
// error) -- no MUFU, 9 HFMA2-pipe instructions; NDGI_POLY_DEG4=0 gives the
// earlier degree-11 fit (1.2e-3 on [0, 2.5], 2.7e-3 in the tail, 10 instructions)
#ifndef NDGI_POLY_DEG4   // 1: degree-4 Q (measured 97.7 -> 99.3 Gtexel/s); 0: degree 5
#define NDGI_POLY_DEG4 1
#endif
__device__ __forceinline__ uint32_t gelu_poly_f16x2(uint32_t h) {
    uint32_t hc, s, q, hh, g;
    asm("min.f16x2 %0, %1, %2;" : "=r"(hc) : "r"(h), "r"(0x41004100u));
    asm("max.f16x2 %0, %1, %2;" : "=r"(hc) : "r"(hc), "r"(0xC100C100u));
    asm("mul.rn.f16x2 %0, %1, %1;" : "=r"(s) : "r"(hc));
#if NDGI_POLY_DEG4
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(q) : "r"(s), "r"(0x0C540C54u), "r"(0x9DAE9DAEu));
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(q) : "r"(q), "r"(s), "r"(0x2A472A47u));
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(q) : "r"(q), "r"(s), "r"(0xB3FEB3FEu));
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(q) : "r"(q), "r"(s), "r"(0x3BF83BF8u));
#else
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(q) : "r"(s), "r"(0x82428242u), "r"(0x12EB12EBu));
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(q) : "r"(q), "r"(s), "r"(0xA0A7A0A7u));
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(q) : "r"(q), "r"(s), "r"(0x2B7B2B7Bu));
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(q) : "r"(q), "r"(s), "r"(0xB429B429u));
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(q) : "r"(q), "r"(s), "r"(0x3BFF3BFFu));
#endif
    asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(hh) : "r"(h), "r"(hc));
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(g) : "r"(hh), "r"(q), "r"(h));
    return g;
}

__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

}  // namespace ndgi
