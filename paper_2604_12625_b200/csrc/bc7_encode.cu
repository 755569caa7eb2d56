// bc7_encode.cu -- BC7 mode-6 encoder on the GPU (the
// step before the path, turning 8-bit feature maps into BC7 payloads).
//
// P:180 "after training, we not only quantize them to 8-bit, but also apply the
// BC7 compression algorithm, which encodes each 4x4 texel block"
// "followed by quantization and BC7 compression to produce the final compressed
// results".  Reading R26 defines the encoder in exact integer
// arithmetic (principal axis by shifted power iteration, extreme texels as
// endpoints, best p-bits, nearest indices, anchor swap), so this kernel matches
// oracle_bc7_encode_mode6 bit for bit.
//
// One thread per 4x4 block, grid-stride.  A warp reads 32 adjacent blocks = 4
// rows of 512 contiguous bytes (16-B loads) and writes 512 contiguous bytes.
// The nearest-index search uses |a - b|^2 = |a|^2 + |b|^2 - 2 a.b with a.b as
// one dp4a per palette entry: |b|^2 is the same for every candidate, so the
// argmin (and its ties) are those of the squared error itself.
#include <cuda_runtime.h>

#include <cstdint>

#include "bc7_device.cuh"

namespace ndgi {

__constant__ int kW4[16] = {0, 4, 9, 13, 17, 21, 26, 30, 34, 38, 43, 47, 51, 55, 60, 64};

__device__ __forceinline__ int ch(uint32_t t, int c) { return (int)((t >> (8 * c)) & 0xffu); }

// 7 bits + p-bit for one endpoint (R26 step 3)
__device__ __forceinline__ void quant_m6(uint32_t e, int (&val)[4], int& pbit) {
    int best = -1;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        int v[4], err = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            int q = (ch(e, c) - p + 1) >> 1;
            q = q < 0 ? 0 : (q > 127 ? 127 : q);
            v[c] = 2 * q + p;
            const int d = v[c] - ch(e, c);
            err += d * d;
        }
        if (best < 0 || err < best) {
            best = err;
            pbit = p;
#pragma unroll
            for (int c = 0; c < 4; ++c) val[c] = v[c];
        }
    }
}

// floor((2 n + det) / (2 det)) clamped to [0, 255], det > 0, without a 64-bit
// division: a float estimate (accurate to << 1 inside [-1, 256], where the
// clamp does not decide) corrected by one exact integer comparison each way
__device__ __forceinline__ int round_div_clamp255(long long n, long long det) {
    const float q = __ll2float_rn(n) / __ll2float_rn(det);
    if (q < -1.0f) return 0;
    if (q > 256.0f) return 255;
    long long k = (long long)floorf(q + 0.5f);
    const long long x = 2 * n + det, y = 2 * det;
    if (y * k > x) --k;
    else if (y * (k + 1) <= x) ++k;
    return k < 0 ? 0 : (k > 255 ? 255 : (int)k);
}

// LSB-first write of n bits of v at bit position pos into 4 words
__device__ __forceinline__ void put_bits(uint32_t (&w)[4], int& pos, uint32_t v, int n) {
    const int i = pos >> 5, o = pos & 31;
    w[i] |= v << o;
    if (o + n > 32) w[i + 1] |= v >> (32 - o);
    pos += n;
}

__device__ __forceinline__ void load_block(const uint8_t* __restrict__ rgba, int w, int bx, int by, uint32_t (&t)[16]) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(rgba + ((size_t)(4 * by + r) * w + 4 * bx) * 4));
        t[4 * r] = q.x;
        t[4 * r + 1] = q.y;
        t[4 * r + 2] = q.z;
        t[4 * r + 3] = q.w;
    }
}

// R26 mode-6 encode of one block of 16 packed RGBA8 texels; *sse (optional)
// receives the block's squared error against the input
__device__ __forceinline__ uint4 encode_mode6_block(const uint32_t (&t)[16], int* sse) {
    // 1. 16 * covariance, exact (|entries| < 2^25)
    int S[4] = {0, 0, 0, 0}, Q[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int r = ch(t[i], 0), g = ch(t[i], 1), bl = ch(t[i], 2), a = ch(t[i], 3);
        S[0] += r; S[1] += g; S[2] += bl; S[3] += a;
        Q[0] += r * r; Q[1] += r * g; Q[2] += r * bl; Q[3] += r * a;
        Q[4] += g * g; Q[5] += g * bl; Q[6] += g * a;
        Q[7] += bl * bl; Q[8] += bl * a; Q[9] += a * a;
    }
    int M[4][4];
    {
        int k = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int d = c; d < 4; ++d) {
                M[c][d] = 16 * Q[k++] - S[c] * S[d];
                M[d][c] = M[c][d];
            }
    }
    // 2. principal axis: 4 power iterations from the largest-variance column,
    // magnitudes shifted below 2^20 at every step (sign kept)
    int cs = 0;
#pragma unroll
    for (int c = 1; c < 4; ++c)
        if (M[c][c] > M[cs][cs]) cs = c;
    long long v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = M[c][cs];
#pragma unroll 1
    for (int it = 0; it <= 4; ++it) {
        long long wv[4];
        if (it == 0) {
#pragma unroll
            for (int c = 0; c < 4; ++c) wv[c] = v[c];
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                wv[c] = 0;
#pragma unroll
                for (int d = 0; d < 4; ++d) wv[c] += (long long)M[c][d] * v[d];
            }
        }
        unsigned long long mx = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const unsigned long long a = (unsigned long long)(wv[c] < 0 ? -wv[c] : wv[c]);
            mx = a > mx ? a : mx;
        }
        if (mx == 0) {
            if (it == 0)
#pragma unroll
                for (int c = 0; c < 4; ++c) v[c] = 1;
            break;
        }
        const int bl = 64 - __clzll((long long)mx);
        const int s = bl > 20 ? bl - 20 : 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const unsigned long long a = (unsigned long long)(wv[c] < 0 ? -wv[c] : wv[c]) >> s;
            v[c] = wv[c] < 0 ? -(long long)a : (long long)a;
        }
    }
    // 3. extreme texels along the axis (|p.v| < 2^30), first index on ties
    const int v0 = (int)v[0], v1 = (int)v[1], v2 = (int)v[2], v3 = (int)v[3];
    int imin = 0, imax = 0, dmin = 0, dmax = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int d = ch(t[i], 0) * v0 + ch(t[i], 1) * v1 + ch(t[i], 2) * v2 + ch(t[i], 3) * v3;
        if (i == 0 || d < dmin) { dmin = d; imin = i; }
        if (i == 0 || d > dmax) { dmax = d; imax = i; }
    }
    uint32_t emin = t[0], emax = t[0];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        emin = i == imin ? t[i] : emin;
        emax = i == imax ? t[i] : emax;
    }
    int E0[4], E1[4], p0, p1;
    quant_m6(emin, E0, p0);
    quant_m6(emax, E1, p1);
    // 4. palette (the decoder's own interpolation) and nearest index per texel
    // key_k(texel) = 16 * (|a_k|^2 - 2 a_k.b) + k: its minimum over k is the
    // smallest squared error, ties to the smallest index (|key| < 2^24)
    uint32_t pal[16];
    int key0[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        uint32_t pw = 0;
        int n2 = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int x = ((64 - kW4[k]) * E0[c] + kW4[k] * E1[c] + 32) >> 6;
            pw |= (uint32_t)x << (8 * c);
            n2 += x * x;
        }
        pal[k] = pw;
        key0[k] = 16 * n2 + k;
    }
    int idx[16];
    int err_old = 0;   // sum over texels of (squared error - |texel|^2)
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        int best = 0x7fffffff;
#pragma unroll
        for (int k = 0; k < 16; ++k) best = min(best, key0[k] - 32 * (int)__dp4a(pal[k], t[i], 0u));
        idx[i] = best & 15;
        err_old += best >> 4;
    }
    int err_final = err_old;
    // 4b. one least-squares refit of the endpoints for these indices (R26),
    // exact integers; kept only if the total squared error drops
    {
        int isaa = 0, isab = 0, isbb = 0;   // < 2^17
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int a = 64 - kW4[idx[i]], b = kW4[idx[i]];
            isaa += a * a;
            isab += a * b;
            isbb += b * b;
        }
        const long long saa = isaa, sab = isab, sbb = isbb;
        const long long det = saa * sbb - sab * sab;
        if (det > 0) {
            uint32_t fpk0 = 0u, fpk1 = 0u;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                int r0 = 0, r1 = 0;   // < 2^24
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    r0 += (64 - kW4[idx[i]]) * ch(t[i], c);
                    r1 += kW4[idx[i]] * ch(t[i], c);
                }
                const long long n0 = sbb * (64LL * r0) - sab * (64LL * r1), n1 = saa * (64LL * r1) - sab * (64LL * r0);
                fpk0 |= (uint32_t)round_div_clamp255(n0, det) << (8 * c);
                fpk1 |= (uint32_t)round_div_clamp255(n1, det) << (8 * c);
            }
            int F0[4], F1[4], q0, q1;
            quant_m6(fpk0, F0, q0);
            quant_m6(fpk1, F1, q1);
            uint32_t pal2[16];
            int kk0[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                uint32_t pw = 0;
                int n2 = 0;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int x = ((64 - kW4[k]) * F0[c] + kW4[k] * F1[c] + 32) >> 6;
                    pw |= (uint32_t)x << (8 * c);
                    n2 += x * x;
                }
                pal2[k] = pw;
                kk0[k] = 16 * n2 + k;
            }
            int jdx[16], err_new = 0;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                int best = 0x7fffffff;
#pragma unroll
                for (int k = 0; k < 16; ++k) best = min(best, kk0[k] - 32 * (int)__dp4a(pal2[k], t[i], 0u));
                jdx[i] = best & 15;
                err_new += best >> 4;
            }
            if (err_new < err_old) {
                err_final = err_new;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    E0[c] = F0[c];
                    E1[c] = F1[c];
                }
                p0 = q0;
                p1 = q1;
#pragma unroll
                for (int i = 0; i < 16; ++i) idx[i] = jdx[i];
            }
        }
    }
    // 5. anchor: texel 0's index must fit in 3 bits
    if (idx[0] >= 8) {
#pragma unroll
        for (int c = 0; c < 4; ++c) { const int x = E0[c]; E0[c] = E1[c]; E1[c] = x; }
        const int x = p0; p0 = p1; p1 = x;
#pragma unroll
        for (int i = 0; i < 16; ++i) idx[i] = 15 - idx[i];
    }
    // 6. pack
    uint32_t wd[4] = {0u, 0u, 0u, 0u};
    int pos = 0;
    put_bits(wd, pos, 1u << 6, 7);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        put_bits(wd, pos, (uint32_t)(E0[c] >> 1), 7);
        put_bits(wd, pos, (uint32_t)(E1[c] >> 1), 7);
    }
    put_bits(wd, pos, (uint32_t)p0, 1);
    put_bits(wd, pos, (uint32_t)p1, 1);
    put_bits(wd, pos, (uint32_t)idx[0], 3);
#pragma unroll
    for (int i = 1; i < 16; ++i) put_bits(wd, pos, (uint32_t)idx[i], 4);
    if (sse) {
        int n2 = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) n2 += (int)__dp4a(t[i], t[i], 0u);
        *sse = n2 + err_final;
    }
    return make_uint4(wd[0], wd[1], wd[2], wd[3]);
}

__global__ void __launch_bounds__(256) bc7_encode_mode6_kernel(const uint8_t* __restrict__ rgba, int w, int h,
                                                              uint4* __restrict__ out) {
    const int wb = w >> 2;
    const size_t nb = (size_t)wb * (h >> 2);
    for (size_t b = blockIdx.x * (size_t)blockDim.x + threadIdx.x; b < nb; b += (size_t)gridDim.x * blockDim.x) {
        const int bx = (int)(b % wb), by = (int)(b / wb);
        uint32_t t[16];
        load_block(rgba, w, bx, by, t);
        out[b] = encode_mode6_block(t, nullptr);
    }
}

// ---- R31: multi-mode search (mode 6, mode 5 x 4 rotations, mode 7 x 64
// partitions), the oracle's algorithm and candidate order; each candidate's
// squared error is computed from its own palette (the decoder's arithmetic)
__constant__ int kW2e[4] = {0, 21, 43, 64};

__device__ __forceinline__ int expand_bits(int v, int n) {
    v <<= 8 - n;
    return v | (v >> n);
}

// R26 step 2/3 over the texels of `mask` and channels 0..NC-1
template <int NC>
__device__ __forceinline__ void axis_extremes(const uint32_t (&t)[16], uint32_t mask, int& imin, int& imax) {
    int S[NC], Q[NC][NC], n = 0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        S[c] = 0;
#pragma unroll
        for (int d = 0; d < NC; ++d) Q[c][d] = 0;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        if (!((mask >> i) & 1u)) continue;
        ++n;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            S[c] += ch(t[i], c);
#pragma unroll
            for (int d = 0; d < NC; ++d) Q[c][d] += ch(t[i], c) * ch(t[i], d);
        }
    }
    int M[NC][NC];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int d = 0; d < NC; ++d) M[c][d] = n * Q[c][d] - S[c] * S[d];
    int cs = 0;
#pragma unroll
    for (int c = 1; c < NC; ++c)
        if (M[c][c] > M[cs][cs]) cs = c;
    long long v[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) v[c] = M[c][cs];
#pragma unroll 1
    for (int it = 0; it <= 4; ++it) {
        long long wv[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            if (it == 0) {
                wv[c] = v[c];
            } else {
                wv[c] = 0;
#pragma unroll
                for (int d = 0; d < NC; ++d) wv[c] += (long long)M[c][d] * v[d];
            }
        }
        unsigned long long mx = 0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const unsigned long long a = (unsigned long long)(wv[c] < 0 ? -wv[c] : wv[c]);
            mx = a > mx ? a : mx;
        }
        if (mx == 0) {
            if (it == 0)
#pragma unroll
                for (int c = 0; c < NC; ++c) v[c] = 1;
            break;
        }
        const int bl = 64 - __clzll((long long)mx);
        const int sh = bl > 20 ? bl - 20 : 0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const unsigned long long a = (unsigned long long)(wv[c] < 0 ? -wv[c] : wv[c]) >> sh;
            v[c] = wv[c] < 0 ? -(long long)a : (long long)a;
        }
    }
    bool first = true;
    int dmin = 0, dmax = 0;
    imin = imax = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        if (!((mask >> i) & 1u)) continue;
        int d = 0;
#pragma unroll
        for (int c = 0; c < NC; ++c) d += ch(t[i], c) * (int)v[c];
        if (first || d < dmin) { dmin = d; imin = i; }
        if (first || d > dmax) { dmax = d; imax = i; }
        first = false;
    }
}

// nearest 7-bit code (no p-bit) / 5-bit code with p-bit p to the 8-bit e;
// the window provably holds the exhaustive argmin (ties to the lower code)
__device__ __forceinline__ int nearest7(int e) {
    int bk = 0, bd = 1 << 30;
#pragma unroll
    for (int j = -1; j <= 1; ++j) {
        const int k = min(max((e >> 1) + j, 0), 127);
        const int d = abs(expand_bits(k, 7) - e);
        if (d < bd || (d == bd && k < bk)) { bd = d; bk = k; }
    }
    return bk;
}
__device__ __forceinline__ int nearest5p(int e, int p) {
    const int k0 = ((e >> 2) - p) >> 1;
    int bk = 0, bd = 1 << 30;
#pragma unroll
    for (int j = -1; j <= 2; ++j) {
        const int k = min(max(k0 + j, 0), 31);
        const int d = abs(expand_bits((k << 1) | p, 6) - e);
        if (d < bd || (d == bd && k < bk)) { bd = d; bk = k; }
    }
    return bk;
}

__device__ __forceinline__ int lerp6(int e0, int e1, int w) { return ((64 - w) * e0 + w * e1 + 32) >> 6; }

// mode 5, rotation rot: A swapped with channel rot - 1 before encoding
__device__ __noinline__ uint4 encode_mode5_block(const uint32_t (&tin)[16], int rot, int& sse) {
    const uint32_t sel = rot == 0 ? 0x3210u : (rot == 1 ? 0x0213u : (rot == 2 ? 0x1230u : 0x2310u));
    uint32_t t[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = __byte_perm(tin[i], 0u, sel);
    int imin, imax;
    axis_extremes<3>(t, 0xffffu, imin, imax);
    uint32_t emin = t[0], emax = t[0];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        emin = i == imin ? t[i] : emin;
        emax = i == imax ? t[i] : emax;
    }
    int C0[3], C1[3], V0[3], V1[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        C0[c] = nearest7(ch(emin, c));
        C1[c] = nearest7(ch(emax, c));
        V0[c] = expand_bits(C0[c], 7);
        V1[c] = expand_bits(C1[c], 7);
    }
    int A0 = 255, A1 = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        A0 = min(A0, ch(t[i], 3));
        A1 = max(A1, ch(t[i], 3));
    }
    int ci[16], ai[16];
    sse = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        int bc = 1 << 30, ba = 1 << 30;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            int err = 0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int d = lerp6(V0[c], V1[c], kW2e[w]) - ch(t[i], c);
                err += d * d;
            }
            if (err < bc) { bc = err; ci[i] = w; }
            const int da = lerp6(A0, A1, kW2e[w]) - ch(t[i], 3);
            if (da * da < ba) { ba = da * da; ai[i] = w; }
        }
        sse += bc + ba;
    }
    if (ci[0] >= 2) {
#pragma unroll
        for (int c = 0; c < 3; ++c) { const int x = C0[c]; C0[c] = C1[c]; C1[c] = x; }
#pragma unroll
        for (int i = 0; i < 16; ++i) ci[i] = 3 - ci[i];
    }
    if (ai[0] >= 2) {
        const int x = A0; A0 = A1; A1 = x;
#pragma unroll
        for (int i = 0; i < 16; ++i) ai[i] = 3 - ai[i];
    }
    uint32_t wd[4] = {0u, 0u, 0u, 0u};
    int pos = 0;
    put_bits(wd, pos, 1u << 5, 6);
    put_bits(wd, pos, (uint32_t)rot, 2);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        put_bits(wd, pos, (uint32_t)C0[c], 7);
        put_bits(wd, pos, (uint32_t)C1[c], 7);
    }
    put_bits(wd, pos, (uint32_t)A0, 8);
    put_bits(wd, pos, (uint32_t)A1, 8);
    put_bits(wd, pos, (uint32_t)ci[0], 1);
#pragma unroll
    for (int i = 1; i < 16; ++i) put_bits(wd, pos, (uint32_t)ci[i], 2);
    put_bits(wd, pos, (uint32_t)ai[0], 1);
#pragma unroll
    for (int i = 1; i < 16; ++i) put_bits(wd, pos, (uint32_t)ai[i], 2);
    return make_uint4(wd[0], wd[1], wd[2], wd[3]);
}

// mode 7, partition part (kBc7Part2 bit i set <=> texel i in subset 1)
__device__ __noinline__ uint4 encode_mode7_block(const uint32_t (&t)[16], int part, int& sse) {
    const uint32_t m1 = kBc7Part2[part], m0 = ~m1 & 0xffffu;
    int code[2][2][4], pb[2][2], val[2][2][4];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        int ie[2];
        axis_extremes<4>(t, s ? m1 : m0, ie[0], ie[1]);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            uint32_t px = t[0];
#pragma unroll
            for (int i = 0; i < 16; ++i) px = i == ie[e] ? t[i] : px;
            int best = 1 << 30;
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                int k[4], err = 0;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    k[c] = nearest5p(ch(px, c), p);
                    const int d = expand_bits((k[c] << 1) | p, 6) - ch(px, c);
                    err += d * d;
                }
                if (err < best) {
                    best = err;
                    pb[s][e] = p;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        code[s][e][c] = k[c];
                        val[s][e][c] = expand_bits((k[c] << 1) | p, 6);
                    }
                }
            }
        }
    }
    int idx[16];
    sse = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int s = (m1 >> i) & 1u;
        int best = 1 << 30;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            int err = 0;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int d = lerp6(s ? val[1][0][c] : val[0][0][c], s ? val[1][1][c] : val[0][1][c], kW2e[w]) - ch(t[i], c);
                err += d * d;
            }
            if (err < best) { best = err; idx[i] = w; }
        }
        sse += best;
    }
    const int a1 = (int)(kBc7Anchors[part] & 0xffu);
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const int a = s ? a1 : 0;
        int ia = idx[0];
#pragma unroll
        for (int i = 0; i < 16; ++i) ia = i == a ? idx[i] : ia;
        if (ia >= 2) {
#pragma unroll
            for (int c = 0; c < 4; ++c) { const int x = code[s][0][c]; code[s][0][c] = code[s][1][c]; code[s][1][c] = x; }
            const int x = pb[s][0]; pb[s][0] = pb[s][1]; pb[s][1] = x;
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if ((int)((m1 >> i) & 1u) == s) idx[i] = 3 - idx[i];
        }
    }
    uint32_t wd[4] = {0u, 0u, 0u, 0u};
    int pos = 0;
    put_bits(wd, pos, 1u << 7, 8);
    put_bits(wd, pos, (uint32_t)part, 6);
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int e = 0; e < 2; ++e) put_bits(wd, pos, (uint32_t)code[s][e][c], 5);
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int e = 0; e < 2; ++e) put_bits(wd, pos, (uint32_t)pb[s][e], 1);
#pragma unroll
    for (int i = 0; i < 16; ++i) put_bits(wd, pos, (uint32_t)idx[i], (i == 0 || i == a1) ? 1 : 2);
    return make_uint4(wd[0], wd[1], wd[2], wd[3]);
}

__global__ void __launch_bounds__(128) bc7_encode_multi_kernel(const uint8_t* __restrict__ rgba, int w, int h,
                                                              uint4* __restrict__ out) {
    const int wb = w >> 2;
    const size_t nb = (size_t)wb * (h >> 2);
    for (size_t b = blockIdx.x * (size_t)blockDim.x + threadIdx.x; b < nb; b += (size_t)gridDim.x * blockDim.x) {
        const int bx = (int)(b % wb), by = (int)(b / wb);
        uint32_t t[16];
        load_block(rgba, w, bx, by, t);
        int best;
        uint4 blk = encode_mode6_block(t, &best);
        for (int r = 0; r < 4 && best > 0; ++r) {
            int e;
            const uint4 c = encode_mode5_block(t, r, e);
            if (e < best) { best = e; blk = c; }
        }
        for (int p = 0; p < 64 && best > 0; ++p) {
            int e;
            const uint4 c = encode_mode7_block(t, p, e);
            if (e < best) { best = e; blk = c; }
        }
        out[b] = blk;
    }
}

cudaError_t launch_bc7_encode_multi(const void* rgba, int w, int h, void* blocks, int num_sms, cudaStream_t s) {
    const size_t nb = (size_t)(w / 4) * (h / 4);
    size_t grid = (nb + 127) / 128;
    const size_t cap = (size_t)num_sms * 16;
    if (grid > cap) grid = cap;
    if (grid == 0) grid = 1;
    bc7_encode_multi_kernel<<<(unsigned)grid, 128, 0, s>>>(static_cast<const uint8_t*>(rgba), w, h,
                                                          static_cast<uint4*>(blocks));
    return cudaGetLastError();
}

cudaError_t launch_bc7_encode_mode6(const void* rgba, int w, int h, void* blocks, int num_sms, cudaStream_t s) {
    const size_t nb = (size_t)(w / 4) * (h / 4);
    size_t grid = (nb + 255) / 256;
    const size_t cap = (size_t)num_sms * 8;
    if (grid > cap) grid = cap;
    if (grid == 0) grid = 1;
    bc7_encode_mode6_kernel<<<(unsigned)grid, 256, 0, s>>>(static_cast<const uint8_t*>(rgba), w, h,
                                                          static_cast<uint4*>(blocks));
    return cudaGetLastError();
}

}  // namespace ndgi
