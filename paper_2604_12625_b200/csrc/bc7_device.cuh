// bc7_device.cuh -- BC7 (BPTC) block decoder for sm_100a, integer and bit-exact.
//
// The paper stores F_uv and each t-slice of F_uvt as BC7 and
// decodes it with the texture unit; this build decodes the blocks in
// the fused kernel itself.  Format definition: D3D11
// functional specification, BC7 section (modes 0..7; reserved mode 8 decodes
// to zero, reading R9 in DESIGN.md).  Per-texel interpolation is Eq. bc_interp
// in the spec's integer form c = ((64-w) e0 + w e1 + 32) >> 6.
//
// Structure (not a translation of any reference decoder):
//  * the 128-bit block is held as two u64 and consumed by a branch-free
//    bit stream (`take(n)`, n may be 0), so every mode runs the SAME
//    instruction sequence with per-mode field widths looked up from packed
//    nibble immediates -> no divergence between modes 0..7 inside a warp;
//  * R|B and G|A are interpolated as packed 16-bit lanes of one 32-bit word
//    (all intermediates < 2^16), two IMADs per channel pair;
//  * partition / anchor tables live in global memory behind the read-only
//    path (divergent partition indices would serialise on __constant__);
//  * a specialised mode-6 path (the smooth payload BC simulation trains for,
//    P:203-222) is used when a whole warp holds mode-6 blocks.
//
// Output: 16 texels, texel = 4*row + col, packed RGBA8 (R in bits 0..7).
#pragma once
#include <cstdint>

namespace ndgi {

// ---- tables (D3D11 BC7 partition sets and anchor indices) -----------------
// 2-subset partitions: bit i set <=> texel i belongs to subset 1.
__device__ const uint16_t kBc7Part2[64] = {
    0xcccc, 0x8888, 0xeeee, 0xecc8, 0xc880, 0xfeec, 0xfec8, 0xec80, 0xc800, 0xffec, 0xfe80, 0xe800, 0xffe8, 0xff00, 0xfff0, 0xf000,
    0xf710, 0x008e, 0x7100, 0x08ce, 0x008c, 0x7310, 0x3100, 0x8cce, 0x088c, 0x3110, 0x6666, 0x366c, 0x17e8, 0x0ff0, 0x718e, 0x399c,
    0xaaaa, 0xf0f0, 0x5a5a, 0x33cc, 0x3c3c, 0x55aa, 0x9696, 0xa55a, 0x73ce, 0x13c8, 0x324c, 0x3bdc, 0x6996, 0xc33c, 0x9966, 0x0660,
    0x0272, 0x04e4, 0x4e40, 0x2720, 0xc936, 0x936c, 0x39c6, 0x639c, 0x9336, 0x9cc6, 0x817e, 0xe718, 0xccf0, 0x0fcc, 0x7744, 0xee22};

// 3-subset partitions: 2 bits per texel, texel 0 in bits 0..1.
__device__ const uint32_t kBc7Part3[64] = {
    0xaa685050u, 0x6a5a5040u, 0x5a5a4200u, 0x5450a0a8u, 0xa5a50000u, 0xa0a05050u, 0x5555a0a0u, 0x5a5a5050u,
    0xaa550000u, 0xaa555500u, 0xaaaa5500u, 0x90909090u, 0x94949494u, 0xa4a4a4a4u, 0xa9a59450u, 0x2a0a4250u,
    0xa5945040u, 0x0a425054u, 0xa5a5a500u, 0x55a0a0a0u, 0xa8a85454u, 0x6a6a4040u, 0xa4a45000u, 0x1a1a0500u,
    0x0050a4a4u, 0xaaa59090u, 0x14696914u, 0x69691400u, 0xa08585a0u, 0xaa821414u, 0x50a4a450u, 0x6a5a0200u,
    0xa9a58000u, 0x5090a0a8u, 0xa8a09050u, 0x24242424u, 0x00aa5500u, 0x24924924u, 0x24499224u, 0x50a50a50u,
    0x500aa550u, 0xaaaa4444u, 0x66660000u, 0xa5a0a5a0u, 0x50a050a0u, 0x69286928u, 0x44aaaa44u, 0x66666600u,
    0xaa444444u, 0x54a854a8u, 0x95809580u, 0x96969600u, 0xa85454a8u, 0x80959580u, 0xaa141414u, 0x96960000u,
    0xaaaa1414u, 0xa05050a0u, 0xa0a5a5a0u, 0x96000000u, 0x40804080u, 0xa9a8a9a8u, 0xaaaaaa44u, 0x2a4a5254u};

// Anchor texels, packed: bits 0..7 = 2-subset anchor of subset 1,
// bits 8..15 = 3-subset anchor of subset 1, bits 16..23 = of subset 2.
#define NDGI_A(a2, a31, a32) ((uint32_t)(a2) | ((uint32_t)(a31) << 8) | ((uint32_t)(a32) << 16))
__device__ const uint32_t kBc7Anchors[64] = {
    NDGI_A(15, 3, 15), NDGI_A(15, 3, 8),  NDGI_A(15, 15, 8), NDGI_A(15, 15, 3), NDGI_A(15, 8, 15), NDGI_A(15, 3, 15),
    NDGI_A(15, 15, 3), NDGI_A(15, 15, 8), NDGI_A(15, 8, 15), NDGI_A(15, 8, 15), NDGI_A(15, 6, 15), NDGI_A(15, 6, 15),
    NDGI_A(15, 6, 15), NDGI_A(15, 5, 15), NDGI_A(15, 3, 15), NDGI_A(15, 3, 8),  NDGI_A(15, 3, 15), NDGI_A(2, 3, 8),
    NDGI_A(8, 8, 15),  NDGI_A(2, 15, 3),  NDGI_A(2, 3, 15),  NDGI_A(8, 3, 8),   NDGI_A(8, 6, 15),  NDGI_A(15, 10, 8),
    NDGI_A(2, 5, 3),   NDGI_A(8, 8, 15),  NDGI_A(2, 8, 6),   NDGI_A(2, 6, 10),  NDGI_A(8, 8, 15),  NDGI_A(8, 5, 15),
    NDGI_A(2, 15, 10), NDGI_A(2, 15, 8),  NDGI_A(15, 8, 15), NDGI_A(15, 15, 3), NDGI_A(6, 3, 15),  NDGI_A(8, 5, 10),
    NDGI_A(2, 6, 10),  NDGI_A(8, 10, 8),  NDGI_A(15, 8, 9),  NDGI_A(15, 15, 10), NDGI_A(2, 15, 6), NDGI_A(8, 3, 15),
    NDGI_A(2, 15, 8),  NDGI_A(2, 5, 15),  NDGI_A(2, 15, 3),  NDGI_A(15, 15, 6), NDGI_A(15, 15, 6), NDGI_A(6, 15, 8),
    NDGI_A(6, 3, 15),  NDGI_A(2, 15, 3),  NDGI_A(6, 5, 15),  NDGI_A(8, 5, 15),  NDGI_A(15, 5, 15), NDGI_A(15, 8, 15),
    NDGI_A(2, 5, 15),  NDGI_A(2, 10, 15), NDGI_A(15, 5, 15), NDGI_A(15, 10, 15), NDGI_A(15, 8, 15), NDGI_A(15, 13, 15),
    NDGI_A(15, 15, 3), NDGI_A(2, 12, 15), NDGI_A(2, 3, 15),  NDGI_A(15, 3, 8)};
#undef NDGI_A

// ---- per-mode field widths, one nibble per mode (mode 0 in bits 0..3) -----
constexpr uint32_t kNS  = 0x21112323u;  // subsets
constexpr uint32_t kPB  = 0x60006664u;  // partition bits
constexpr uint32_t kRB  = 0x00220000u;  // rotation bits
constexpr uint32_t kISB = 0x00010000u;  // index-selection bit
constexpr uint32_t kCB  = 0x57757564u;  // colour bits per channel
constexpr uint32_t kAB  = 0x57860000u;  // alpha bits
constexpr uint32_t kEPB = 0x11001001u;  // one p-bit per endpoint
constexpr uint32_t kSPB = 0x00000010u;  // one p-bit per subset
constexpr uint32_t kIB  = 0x24222233u;  // primary index bits
constexpr uint32_t kIB2 = 0x00230000u;  // secondary index bits

__device__ __forceinline__ uint32_t nib(uint32_t table, uint32_t mode) { return (table >> (4u * mode)) & 15u; }

// branch-free LSB-first reader over a 128-bit value
struct Bits128 {
    uint64_t lo, hi;
    // n in [0, 8]
    __device__ __forceinline__ uint32_t take(uint32_t n) {
        uint32_t v = (uint32_t)lo & ((1u << n) - 1u);
        uint64_t carry = n ? (hi << (64u - n)) : 0ull;
        lo = (lo >> n) | carry;
        hi >>= n;
        return v;
    }
    // n in [0, 63]
    __device__ __forceinline__ void skip(uint32_t n) {
        uint64_t carry = n ? (hi << (64u - n)) : 0ull;
        lo = (lo >> n) | carry;
        hi >>= n;
    }
};

// weight tables as byte lanes: W2 in bytes 0..3 of w2; W3 in w3; W4 in (w4lo, w4hi)
constexpr uint32_t kW2 = 0x402b1500u;                 // 0, 21, 43, 64
constexpr uint64_t kW3 = 0x40372e251b120900ull;       // 0, 9, 18, 27, 37, 46, 55, 64
constexpr uint64_t kW4lo = 0x1e1a15110d090400ull;     // 0, 4, 9, 13, 17, 21, 26, 30
constexpr uint64_t kW4hi = 0x403c37332f2b2622ull;     // 34, 38, 43, 47, 51, 55, 60, 64

// weight-table handle for `bits` index bits
struct WTab {
    uint64_t lo, hi;
    __device__ __forceinline__ void set(uint32_t bits) {
        lo = bits == 4u ? kW4lo : (bits == 3u ? kW3 : (uint64_t)kW2);
        hi = kW4hi;
    }
    __device__ __forceinline__ uint32_t w(uint32_t idx) const {
        uint64_t t = (idx & 8u) ? hi : lo;
        return (uint32_t)(t >> ((idx & 7u) * 8u)) & 0xffu;
    }
};

// expand an n-bit value (n in 4..8) to 8 bits by bit replication
__device__ __forceinline__ uint32_t expand8(uint32_t v, uint32_t n) {
    v <<= (8u - n);
    return (v | (v >> n)) & 0xffu;
}

// packed interpolation of two channels held in 16-bit lanes of e0/e1
__device__ __forceinline__ uint32_t lerp2(uint32_t e0, uint32_t e1, uint32_t w) {
    uint32_t v = (64u - w) * e0 + w * e1 + 0x00200020u;
    return (v >> 6) & 0x00ff00ffu;
}

// ---------------------------------------------------------------------------
// Generic decoder: every mode 0..7 (+ reserved 8) through one code path.
// sink(i, rgba) receives texel i (= 4*row + col) as packed RGBA8.
// ---------------------------------------------------------------------------
template <class Sink>
__device__ __forceinline__ void bc7_decode_generic(uint4 raw, Sink&& sink) {
    Bits128 s;
    s.lo = (uint64_t)raw.x | ((uint64_t)raw.y << 32);
    s.hi = (uint64_t)raw.z | ((uint64_t)raw.w << 32);
    const uint32_t byte0 = raw.x & 0xffu;
    const bool reserved = byte0 == 0u;
    const uint32_t mode = reserved ? 0u : (uint32_t)(__ffs(byte0) - 1);
    s.take(mode + 1u);

    const uint32_t ns = nib(kNS, mode), cb = nib(kCB, mode), ab = nib(kAB, mode);
    const uint32_t part = s.take(nib(kPB, mode));
    const uint32_t rot = s.take(nib(kRB, mode));
    const uint32_t isel = s.take(nib(kISB, mode));
    const uint32_t ne = 2u * ns;

    // endpoint fields, channel-major then endpoint (s0e0, s0e1, s1e0, ...)
    uint32_t ep[6][4];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int e = 0; e < 6; ++e) ep[e][c] = s.take((uint32_t)e < ne ? cb : 0u);
#pragma unroll
    for (int e = 0; e < 6; ++e) ep[e][3] = s.take((uint32_t)e < ne ? ab : 0u);

    // p-bits: one per endpoint (modes 0,3,6,7) or one per subset (mode 1)
    const uint32_t epb = nib(kEPB, mode), spb = nib(kSPB, mode);
    uint32_t pb[6];
#pragma unroll
    for (int e = 0; e < 6; ++e) pb[e] = s.take(((uint32_t)e < ne) ? epb : 0u);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const uint32_t p = s.take(((uint32_t)q < ns) ? spb : 0u);
        if (spb) { pb[2 * q] = p; pb[2 * q + 1] = p; }
    }
    const uint32_t hasp = epb | spb;

    // expanded 8-bit endpoints packed as R|B<<16 and G|A<<16
    uint32_t rb[6], ga[6];
    const uint32_t nc = cb + hasp, na = ab + hasp;
#pragma unroll
    for (int e = 0; e < 6; ++e) {
        const uint32_t p = pb[e] & hasp;
        const uint32_t r = expand8((ep[e][0] << hasp) | p, nc);
        const uint32_t g = expand8((ep[e][1] << hasp) | p, nc);
        const uint32_t b = expand8((ep[e][2] << hasp) | p, nc);
        const uint32_t a = ab ? expand8((ep[e][3] << hasp) | p, na) : 255u;
        rb[e] = r | (b << 16);
        ga[e] = g | (a << 16);
    }

    // subset map (2 bits per texel) and anchors
    const uint32_t pi = part & 63u;
    uint32_t smap = 0u;
    if (ns == 2u) {
        uint32_t x = __ldg(&kBc7Part2[pi]);
        x = (x | (x << 8)) & 0x00ff00ffu;
        x = (x | (x << 4)) & 0x0f0f0f0fu;
        x = (x | (x << 2)) & 0x33333333u;
        smap = (x | (x << 1)) & 0x55555555u;
    } else if (ns == 3u) {
        smap = __ldg(&kBc7Part3[pi]);
    }
    const uint32_t anc = __ldg(&kBc7Anchors[pi]);
    const uint32_t a1 = ns == 2u ? (anc & 0xffu) : (ns == 3u ? ((anc >> 8) & 0xffu) : 16u);
    const uint32_t a2 = ns == 3u ? ((anc >> 16) & 0xffu) : 16u;

    // primary indices start here; secondary indices (modes 4,5) follow them
    const uint32_t ib = nib(kIB, mode), ib2 = nib(kIB2, mode);
    Bits128 s2 = s;
    s2.skip(16u * ib - ns);

    // mode 4: index selection swaps which array drives colour and alpha
    const bool swap = isel && ib2;
    WTab wc, wa;
    wc.set(swap ? ib2 : ib);
    wa.set(ib2 ? (isel ? ib : ib2) : ib);
    // rotation (modes 4,5): swap A with channel rot-1
    const uint32_t sel = rot == 0u ? 0x3210u : (rot == 1u ? 0x0213u : (rot == 2u ? 0x1230u : 0x2310u));

#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const bool anchor = (i == 0) || ((uint32_t)i == a1) || ((uint32_t)i == a2);
        const uint32_t i1 = s.take(ib - (anchor ? 1u : 0u));
        const uint32_t i2 = s2.take(ib2 ? ib2 - (i == 0 ? 1u : 0u) : 0u);
        const uint32_t ci = swap ? i2 : i1;
        const uint32_t ai = ib2 ? (isel ? i1 : i2) : i1;
        const uint32_t w = wc.w(ci), wA = wa.w(ai);
        const uint32_t sub = (smap >> (2 * i)) & 3u;
        const uint32_t e0rb = sub == 0u ? rb[0] : (sub == 1u ? rb[2] : rb[4]);
        const uint32_t e1rb = sub == 0u ? rb[1] : (sub == 1u ? rb[3] : rb[5]);
        const uint32_t e0ga = sub == 0u ? ga[0] : (sub == 1u ? ga[2] : ga[4]);
        const uint32_t e1ga = sub == 0u ? ga[1] : (sub == 1u ? ga[3] : ga[5]);
        const uint32_t RB = lerp2(e0rb, e1rb, w);
        const uint32_t G = ((64u - w) * (e0ga & 0xffu) + w * (e1ga & 0xffu) + 32u) >> 6;
        const uint32_t A = ((64u - wA) * (e0ga >> 16) + wA * (e1ga >> 16) + 32u) >> 6;
        const uint32_t rgba = __byte_perm(RB | (G << 8) | (A << 24), 0u, sel);
        sink(i, reserved ? 0u : rgba);
    }
}

// ---------------------------------------------------------------------------
// Mode-6 decoder (valid only when (byte0 & 0x7f) == 0x40).
// Layout: mode(7) R0 R1 G0 G1 B0 B1 A0 A1 (7 each) P0 P1 idx0(3) idx1..15(4)
// ---------------------------------------------------------------------------
//
// Per texel the interpolation ((64 - w) e0 + w e1 + 32) >> 6 runs on two
// channels at once in 16-bit lanes, rewritten as w (e1 - e0) + (64 e0 + 32):
// with D = rb1 - rb0 taken as a plain 32-bit difference of the packed words
// (R + 2^16 B), w D + E = L + 2^16 H exactly, where L and H are the two lanes'
// non-negative sums (< 2^14), so the lanes separate without borrows -- one
// IMAD per channel pair.  The 4-bit weights round(64 i / 15) are
// 4 i + ((i + 2) >> 2) (exact for i = 0..15), evaluated for four texels at
// once on bytes.
struct Bc7Mode6 {
    uint32_t drb, dga, erb, ega, iw0, iw1;
    __device__ __forceinline__ explicit Bc7Mode6(uint4 raw) {
        const uint64_t lo = (uint64_t)raw.x | ((uint64_t)raw.y << 32);
        const uint32_t p0 = raw.y >> 31, p1 = raw.z & 1u;
        auto f = [&](int k) { return (uint32_t)(lo >> (7 + 7 * k)) & 0x7fu; };
        const uint32_t rb0 = ((f(0) << 1) | p0) | (((f(4) << 1) | p0) << 16);
        const uint32_t rb1 = ((f(1) << 1) | p1) | (((f(5) << 1) | p1) << 16);
        const uint32_t ga0 = ((f(2) << 1) | p0) | (((f(6) << 1) | p0) << 16);
        const uint32_t ga1 = ((f(3) << 1) | p1) | (((f(7) << 1) | p1) << 16);
        drb = rb1 - rb0;
        dga = ga1 - ga0;
        erb = (rb0 << 6) + 0x00200020u;
        ega = (ga0 << 6) + 0x00200020u;
        // texel i's index: bits 64 + 4i (i >= 1); texel 0: 3 bits at 65 (anchor)
        iw0 = (raw.z & ~0xfu) | ((raw.z >> 1) & 7u);
        iw1 = raw.w;
    }
    // texels 4g .. 4g+3 (block row g) as packed RGBA8
    template <class Sink>
    __device__ __forceinline__ void row(int g, Sink&& sink) const {
        const uint32_t nib = (g < 2 ? iw0 : iw1) >> (16 * (g & 1));
        // indices -> bytes, then their weights
        const uint32_t ib = __byte_perm(nib & 0x0f0fu, (nib >> 4) & 0x0f0fu, 0x5140u);
        const uint32_t wb = (ib << 2) + (((ib + 0x02020202u) >> 2) & 0x3f3f3f3fu);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t w = (wb >> (8 * k)) & 0xffu;
            const uint32_t vrb = w * drb + erb, vga = w * dga + ega;
            sink(k, ((vrb >> 6) & 0x00ff00ffu) | ((vga << 2) & 0xff00ff00u));
        }
    }
};

template <class Sink>
__device__ __forceinline__ void bc7_decode_mode6(uint4 raw, Sink&& sink) {
    const Bc7Mode6 m(raw);
#pragma unroll
    for (int g = 0; g < 4; ++g) m.row(g, [&](int k, uint32_t v) { sink(4 * g + k, v); });
}

__device__ __forceinline__ bool bc7_is_mode6(uint4 raw) { return (raw.x & 0x7fu) == 0x40u; }

// the all-mode decoder out of line (into a 16-word array), NDGI_BC7_OOL=1: halves
// the fused kernel's code (10.7 K -> 6.0 K SASS instructions) but measured 1 %
// slower on config 2 (register allocation of the step loop) and no faster for
// small VT batches, so the default build keeps it inline
static __device__ __noinline__ void bc7_decode_generic16(uint4 raw, uint32_t* out) {
    bc7_decode_generic(raw, [&](int i, uint32_t v) { out[i] = v; });
}

// Decodes one block; uses the mode-6 path when every active lane holds mode 6.
#ifndef NDGI_BC7_OOL
#define NDGI_BC7_OOL 0
#endif
template <class Sink>
__device__ __forceinline__ void bc7_decode(uint4 raw, Sink&& sink) {
    if (__all_sync(__activemask(), bc7_is_mode6(raw))) {
        bc7_decode_mode6(raw, sink);
    } else if (!NDGI_BC7_OOL) {
        bc7_decode_generic(raw, sink);
    } else {
        uint32_t t[16];
        bc7_decode_generic16(raw, t);
#pragma unroll
        for (int i = 0; i < 16; ++i) sink(i, t[i]);
    }
}

// Row r (texels 4r .. 4r+3) of one block: the mode-6 path when every active
// lane holds mode 6, else the full decode
__device__ __forceinline__ void bc7_decode_row(uint4 raw, int r, uint32_t (&out)[4]) {
    if (__all_sync(__activemask(), bc7_is_mode6(raw))) {
        Bc7Mode6(raw).row(r, [&](int k, uint32_t v) { out[k] = v; });
    } else {
        bc7_decode_generic(raw, [&](int i, uint32_t v) {
            if ((i >> 2) == r) out[i & 3] = v;
        });
    }
}

// Single texel of a mode-6 block: RGBA 7-bit endpoints at bits 7..62, p-bits
// at 63 and 64, texel 0's 3-bit index at 65, texel i's 4-bit index at 64 + 4i.
__device__ __forceinline__ uint32_t bc7_texel_mode6(uint4 raw, int texel) {
    const uint64_t lo = (uint64_t)raw.x | ((uint64_t)raw.y << 32);
    const uint64_t hi = (uint64_t)raw.z | ((uint64_t)raw.w << 32);
    const uint32_t p0 = (uint32_t)(lo >> 63), p1 = (uint32_t)hi & 1u;
    const uint32_t idx = texel == 0 ? (uint32_t)(hi >> 1) & 7u : (uint32_t)(hi >> (4 * texel)) & 15u;
    const uint32_t w = (uint32_t)((idx < 8u ? kW4lo : kW4hi) >> (8u * (idx & 7u))) & 0xffu;
    uint32_t v = 0u;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const uint32_t e0 = ((uint32_t)(lo >> (7 + 14 * c)) & 127u) << 1 | p0;
        const uint32_t e1 = ((uint32_t)(lo >> (14 + 14 * c)) & 127u) << 1 | p1;
        v |= (((64u - w) * e0 + w * e1 + 32u) >> 6) << (8 * c);
    }
    return v;
}

// Single-texel decode (texel = 4*row + col): the mode-6 path for mode-6 blocks,
// else the generic decoder; used by the scalar fp32 reference and fine-tuning
// kernels.
// the all-mode decoder as an out-of-line call: inlined at every tap of a
// bilinear/trilinear sampler it would multiply the code size (instruction-cache
// misses), and mode-6 payloads never reach it
static __device__ __noinline__ uint32_t bc7_texel_generic(uint4 raw, int texel) {
    uint32_t v = 0u;
    bc7_decode_generic(raw, [&](int i, uint32_t rgba) { if (i == texel) v = rgba; });
    return v;
}

__device__ __forceinline__ uint32_t bc7_texel(uint4 raw, int texel) {
    if (bc7_is_mode6(raw)) return bc7_texel_mode6(raw, texel);
    return bc7_texel_generic(raw, texel);
}

}  // namespace ndgi
