// bcn_device.cuh -- BC1 / BC4 block decoders and their combinations BC3 and
// BC5 for sm_100a, integer and bit-exact (the other
// points of config 5's "BC format" axis; "DXTC spans BC1
// through BC7 ... BC5 for normal maps"; reading R29 in DESIGN.md).
//
// Layouts (little-endian, texel i = 4*row + col), as include/ndgi.h states:
//  * BC1 (8 B): c0, c1 RGB565 in the low word, 2-bit indices in the high
//    word (texel i at bits 2i).  565 -> 888 by bit replication.  Palette:
//    c0 > c1 (or always, for BC3's colour half): c0, c1, (2c0+c1)/3,
//    (c0+2c1)/3; else c0, c1, (c0+c1)/2, transparent black (A = 0).
//  * BC4 (8 B): a0, a1 in bytes 0, 1, 3-bit indices in the 48 bits above
//    (texel i at bit 16 + 3i).  a0 > a1: a0, a1, ((8-j) a0 + (j-1) a1)/7,
//    j = 2..7; else a0, a1, ((6-j) a0 + (j-1) a1)/5, j = 2..5, 0, 255.
//  * BC3 (16 B) = BC4 for A, then BC1 for RGB (four-colour mode always).
//  * BC5 (16 B) = BC4 for channel 0, then BC4 for channel 1.
// The interpolated entries use integer division (truncation) -- the reading
// the oracle takes from Pillow's decoder (R29).
//
// Palettes are built once per block (packed RGBA8 words) and indexed with
// selects, never with dynamic register indexing.
#pragma once
#include <cstdint>

#include "bc7_device.cuh"
#include "ndgi_common.cuh"

namespace ndgi {

__device__ __forceinline__ bool fmt_block4(int f) { return f == FMT_BC7 || f == FMT_BC1 || f == FMT_BC3; }
__device__ __host__ __forceinline__ int fmt_block_bytes(int f) { return f == FMT_BC1 ? 8 : 16; }

// packed RGBA8 palette of a BC1 colour block (ep = c0 | c1 << 16)
__device__ __forceinline__ void bc1_palette(uint32_t ep, bool always4, uint32_t pal[4]) {
    const uint32_t c0 = ep & 0xffffu, c1 = ep >> 16;
    const uint32_t r0 = (c0 >> 11) << 3 | (c0 >> 13), g0 = ((c0 >> 5) & 63u) << 2 | ((c0 >> 9) & 3u),
                   b0 = (c0 & 31u) << 3 | ((c0 >> 2) & 7u);
    const uint32_t r1 = (c1 >> 11) << 3 | (c1 >> 13), g1 = ((c1 >> 5) & 63u) << 2 | ((c1 >> 9) & 3u),
                   b1 = (c1 & 31u) << 3 | ((c1 >> 2) & 7u);
    pal[0] = r0 | g0 << 8 | b0 << 16 | 0xff000000u;
    pal[1] = r1 | g1 << 8 | b1 << 16 | 0xff000000u;
    if (always4 || c0 > c1) {
        pal[2] = (2 * r0 + r1) / 3 | ((2 * g0 + g1) / 3) << 8 | ((2 * b0 + b1) / 3) << 16 | 0xff000000u;
        pal[3] = (r0 + 2 * r1) / 3 | ((g0 + 2 * g1) / 3) << 8 | ((b0 + 2 * b1) / 3) << 16 | 0xff000000u;
    } else {
        pal[2] = (r0 + r1) / 2 | ((g0 + g1) / 2) << 8 | ((b0 + b1) / 2) << 16 | 0xff000000u;
        pal[3] = 0u;
    }
}

__device__ __forceinline__ uint32_t sel4(const uint32_t p[4], uint32_t q) {
    const uint32_t lo = (q & 1u) ? p[1] : p[0], hi = (q & 1u) ? p[3] : p[2];
    return (q & 2u) ? hi : lo;
}

// BC4 palette of a block whose low word is lo (a0 = byte 0, a1 = byte 1)
__device__ __forceinline__ void bc4_palette(uint32_t lo, uint32_t pal[8]) {
    const uint32_t a0 = lo & 0xffu, a1 = (lo >> 8) & 0xffu;
    pal[0] = a0;
    pal[1] = a1;
    if (a0 > a1) {
#pragma unroll
        for (int j = 2; j < 8; ++j) pal[j] = ((8 - j) * a0 + (j - 1) * a1) / 7;
    } else {
#pragma unroll
        for (int j = 2; j < 6; ++j) pal[j] = ((6 - j) * a0 + (j - 1) * a1) / 5;
        pal[6] = 0u;
        pal[7] = 255u;
    }
}

__device__ __forceinline__ uint32_t sel8(const uint32_t p[8], uint32_t q) {
    const uint32_t a = (q & 1u) ? p[1] : p[0], b = (q & 1u) ? p[3] : p[2];
    const uint32_t c = (q & 1u) ? p[5] : p[4], d = (q & 1u) ? p[7] : p[6];
    const uint32_t lo = (q & 2u) ? b : a, hi = (q & 2u) ? d : c;
    return (q & 4u) ? hi : lo;
}

// the 8 BC4 palette bytes packed into two words: entry q = byte q of {hi:lo},
// so a lookup is one PRMT (byte_perm selects by a 3-bit index)
__device__ __forceinline__ void bc4_palette_packed(uint32_t lo, uint32_t& plo, uint32_t& phi) {
    uint32_t p[8];
    bc4_palette(lo, p);
    plo = p[0] | p[1] << 8 | p[2] << 16 | p[3] << 24;
    phi = p[4] | p[5] << 8 | p[6] << 16 | p[7] << 24;
}

__device__ __forceinline__ uint32_t bc4_index(uint2 w, int i) {
    const uint64_t v = (uint64_t)w.y << 32 | w.x;
    return (uint32_t)(v >> (16 + 3 * i)) & 7u;
}

// whole-block decoders: sink(texel, packed RGBA8)
template <class Sink>
__device__ __forceinline__ void bc1_decode(uint2 w, bool always4, Sink&& sink) {
    uint32_t pal[4];
    bc1_palette(w.x, always4, pal);
#pragma unroll
    for (int i = 0; i < 16; ++i) sink(i, sel4(pal, (w.y >> (2 * i)) & 3u));
}

template <class Sink>
__device__ __forceinline__ void bc3_decode(uint4 raw, Sink&& sink) {
    uint32_t pal[4], alo, ahi;
    bc1_palette(raw.z, true, pal);
    bc4_palette_packed(raw.x, alo, ahi);
    const uint2 aw = make_uint2(raw.x, raw.y);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        // colour bytes 0..2, then palette byte q of {ahi:alo} as byte 3
        const uint32_t a = __byte_perm(alo, ahi, bc4_index(aw, i));
        sink(i, __byte_perm(sel4(pal, (raw.w >> (2 * i)) & 3u), a, 0x4210u));
    }
}

// single texels (reference / training paths)
__device__ __forceinline__ uint32_t bc1_texel(uint2 w, int i, bool always4) {
    uint32_t pal[4];
    bc1_palette(w.x, always4, pal);
    return sel4(pal, (w.y >> (2 * i)) & 3u);
}

__device__ __forceinline__ uint32_t bc4_texel(uint2 w, int i) {
    uint32_t pal[8];
    bc4_palette(w.x, pal);
    return sel8(pal, bc4_index(w, i));
}

// one 4-channel block (BC7 / BC1 / BC3) of a map at block index bi; fmt is
// warp-uniform (bc7_decode votes across the warp)
static __device__ __noinline__ void bcn_decode16(int fmt, const uint8_t* base, size_t bi, uint32_t* out) {
    auto sink = [&](int i, uint32_t v) { out[i] = v; };
    if (fmt == FMT_BC1) bc1_decode(__ldg(reinterpret_cast<const uint2*>(base) + bi), false, sink);
    else bc3_decode(__ldg(reinterpret_cast<const uint4*>(base) + bi), sink);
}

template <class Sink>
__device__ __forceinline__ void block4_decode(int fmt, const uint8_t* base, size_t bi, Sink&& sink) {
    if (fmt == FMT_BC1 || fmt == FMT_BC3) {   // the other formats' decoders out of line (code size)
        uint32_t t[16];
        bcn_decode16(fmt, base, bi, t);
#pragma unroll
        for (int i = 0; i < 16; ++i) sink(i, t[i]);
    } else {
        bc7_decode(__ldg(reinterpret_cast<const uint4*>(base) + bi), sink);
    }
}

// row r (texels 4r .. 4r+3) of block bi of a BC7 / BC1 / BC3 map (the F_uvt
// ring's staging: one block row per thread, so all 128 threads take part; the
// BC1 / BC3 palettes are rebuilt per row -- their cost is small next to a
// chunk start with three of four warps idle at the barrier)
template <int FMT>
__device__ __forceinline__ void block4_decode_row(const uint8_t* base, size_t bi, int r, uint32_t (&out)[4]) {
    static_assert(FMT == FMT_BC7 || FMT == FMT_BC1 || FMT == FMT_BC3, "4x4 block formats");
    if constexpr (FMT == FMT_BC1) {
        const uint2 w = __ldg(reinterpret_cast<const uint2*>(base) + bi);
        uint32_t pal[4];
        bc1_palette(w.x, false, pal);
#pragma unroll
        for (int x = 0; x < 4; ++x) out[x] = sel4(pal, (w.y >> (8 * r + 2 * x)) & 3u);
    } else if constexpr (FMT == FMT_BC3) {
        const uint4 raw = __ldg(reinterpret_cast<const uint4*>(base) + bi);
        uint32_t pal[4], alo, ahi;
        bc1_palette(raw.z, true, pal);
        bc4_palette_packed(raw.x, alo, ahi);
        const uint32_t aidx = (uint32_t)((((uint64_t)raw.y << 32) | raw.x) >> (16 + 12 * r));   // 4 x 3 bits
#pragma unroll
        for (int x = 0; x < 4; ++x)
            out[x] = __byte_perm(sel4(pal, (raw.w >> (8 * r + 2 * x)) & 3u), __byte_perm(alo, ahi, (aidx >> (3 * x)) & 7u),
                                 0x4210u);
    } else {
        bc7_decode_row(__ldg(reinterpret_cast<const uint4*>(base) + bi), r, out);
    }
}

// BC5 texel (x, y) of a [ry][rx] 2-channel map: packed c0 | c1 << 8
__device__ __forceinline__ uint32_t bc5_texel_at(const uint8_t* base, int rx, int x, int y) {
    const uint4 raw = __ldg(reinterpret_cast<const uint4*>(base) + (size_t)(y >> 2) * (rx >> 2) + (x >> 2));
    const int i = 4 * (y & 3) + (x & 3);
    return bc4_texel(make_uint2(raw.x, raw.y), i) | bc4_texel(make_uint2(raw.z, raw.w), i) << 8;
}

}  // namespace ndgi
