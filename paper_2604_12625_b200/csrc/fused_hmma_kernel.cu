// fused_hmma_kernel.cu -- NDGI_MODE_FAST for h = 16 with a register-resident
// tensor-core chain (mma.sync.m16n8k16, f16 in / fp32 accumulate).
//
// Same hot path and arithmetic as fused_kernel.cu (
// DESIGN.md §6.1) -- BC7 decode, sampling, Eq. 4 input row, G_Phi with the
// tanh-form f16x2 GELU, RGBA8 writer -- but G_Phi runs per warp: the fp32
// accumulator fragment of one m16n8k16 MMA is exactly (after GELU and f16x2
// packing) the A fragment of the next layer's MMA, so the three layers never
// leave registers, biases enter as the fp32 C operand (exact, no K padding),
// and warps never synchronise with each other inside a tile: for h = 16 the
// path is bound by the MUFU pipe (2h tanh per texel), and what costs time in
// the TMEM design is the CTA-wide barrier + MMA round trip per layer, not
// tensor throughput (the tensor pipe is ~9% busy there).
//
// CTA = 4 warps; warp w owns core columns [32w, 32w+32) of every row (C = 128)
// or those columns in both 128-halves (C = 256).  Per warp-row (32 texels =
// two m16 tiles): gather (one texel per lane) -> 2 x STS.128 -> 2 x LDSM.x4
// -> 4 + 4 + 2 HMMA with GELU in between -> RGBA8 of 4 texels per quad-leader
// lane, 8-lane coalesced 32-B stores.
#include <cstdio>
#include <cstdlib>

#include "fused_common.cuh"

namespace ndgi {

constexpr int kHmThreads = 128;
#ifndef NDGI_HM_MIN_CTAS
#define NDGI_HM_MIN_CTAS 8
#endif

struct HmSmem {
    FusedSmem base;        // common layout (B1..B3 regions unused)
    uint32_t w1, w2, w3;   // f16 [n][16] row-major (k contiguous): 16, 16, 8 rows
    uint32_t bias;         // fp32 b1'[16], b2'[16], b3[8]
    uint32_t frag;         // per lane: 10 B-fragment words + 10 C floats (+4 pad) = 96 B
    uint32_t stage;        // per-warp 1 KB A-row staging for ldmatrix
    uint32_t total;
};

__host__ __device__ inline HmSmem hm_smem_layout(int C, int R3) {
    HmSmem s;
    s.base = fused_smem_layout<16>(C, R3);
    uint32_t o = (s.base.total + 127u) & ~127u;
    s.w1 = o; o += 16 * 16 * 2;
    s.w2 = o; o += 16 * 16 * 2;
    s.w3 = o; o += 8 * 16 * 2;
    s.bias = o; o += 40 * 4;
    o = (o + 127u) & ~127u;
    s.frag = o; o += 32 * 96;
    s.stage = o; o += 4 * 1024;
    s.total = o;
    return s;
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1, float c0,
                                         float c1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%11,%12,%13};"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(c0), "f"(c1), "f"(c0), "f"(c1));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}

// 16 fp32 accumulators of one m16 tile (two n8 tiles) -> GELU~ -> A fragment
__device__ __forceinline__ void gelu_frag(const float (&d0)[4], const float (&d1)[4], uint32_t (&a)[4]) {
    a[0] = gelu_scaled_f16x2(pack_f16x2(d0[0], d0[1]));   // row r,   k 2q..2q+1
    a[1] = gelu_scaled_f16x2(pack_f16x2(d0[2], d0[3]));   // row r+8, k 2q..2q+1
    a[2] = gelu_scaled_f16x2(pack_f16x2(d1[0], d1[1]));   // row r,   k 8+2q..
    a[3] = gelu_scaled_f16x2(pack_f16x2(d1[2], d1[3]));   // row r+8, k 8+2q..
}

template <int FMT_UV, int CT>
__global__ void __launch_bounds__(kHmThreads, NDGI_HM_MIN_CTAS) ndgi_fused_hmma_kernel(const __grid_constant__ KParams p) {
    constexpr int H = 16;
    constexpr int C = CT;
    constexpr int BPR = CT / 128;
    constexpr int chunk_rows = kChunkTexels / CT;
    extern __shared__ __align__(1024) uint8_t smem[];
    const HmSmem L = hm_smem_layout(C, p.R3);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, q = lane & 3, r8 = lane >> 2;
    const uint2* sUvt = reinterpret_cast<const uint2*>(smem + L.base.uvt);
    const uint32_t* sUt = reinterpret_cast<const uint32_t*>(smem + L.base.utcol);
    const uint4* sRow = reinterpret_cast<const uint4*>(smem + L.base.rowtab);
    __half* sW1 = reinterpret_cast<__half*>(smem + L.w1);
    __half* sW2 = reinterpret_cast<__half*>(smem + L.w2);
    __half* sW3 = reinterpret_cast<__half*>(smem + L.w3);
    float* sBias = reinterpret_cast<float*>(smem + L.bias);
    uint8_t* stage = smem + L.stage + warp * 1024;
    const uint32_t stage_s = ptx::smem_addr(stage);

    const int B = p.B, P = p.P, R3 = p.R3;
    const float sc3 = (float)R3 * (1.0f / (float)C);

    for (uint32_t unit = blockIdx.x; unit < p.units; unit += gridDim.x) {
        const int strip = (int)(unit % (uint32_t)p.strips_per_tile);
        const uint32_t rq = unit / (uint32_t)p.strips_per_tile;
        const int ti = (int)(rq / p.n_req);
        const uint32_t r = rq % p.n_req;
        const TConst& tc = p.tc[ti];
        int k;
        size_t out_base, row_pitch;
        if (p.full) {
            k = (int)r;
            const int tx = k % p.tiles_x, ty = (k / p.tiles_x) % p.tiles_y, a = k / (p.tiles_x * p.tiles_y);
            row_pitch = (size_t)p.tiles_x * C;
            out_base = (size_t)ti * p.out_t_stride + (size_t)a * p.tiles_y * C * row_pitch +
                       (size_t)ty * C * row_pitch + (size_t)tx * C;
        } else {
            const uint32_t id = __ldg(p.tile_ids + r);
            const uint32_t slot = p.slots ? __ldg(p.slots + r) : r;
            if (id >= (uint32_t)p.num_tiles || slot >= p.num_slots) {
                if (strip == 0 && tid == 0) atomicAdd(p.err, 1u);
                continue;  // uniform across the CTA
            }
            k = (int)id;
            row_pitch = (size_t)P;
            out_base = ((size_t)slot * P + B) * P + B;
        }

        // ---- a2: unit parameters -> smem ------------------------------------------
        __syncthreads();
        unit_prologue<H, FMT_UV, C, false>(p, tc, k, smem, L.base, tid, kHmThreads);
        {
            // MLP with the same folds as the TMEM kernel, B operands
            // as f16 [n][k] (= PyTorch [out][in]), biases fp32 (enter as the C operand)
            const uint16_t* w = p.mlp + p.mlp_tile_elems * k;
            const uint16_t *W1 = w, *b1 = W1 + 16 * H, *W2 = b1 + H, *b2 = W2 + H * H, *W3 = b2 + H, *b3 = W3 + 3 * H;
            const float a = kGeluA;
            const float s_uv = FMT_UV == FMT_F16 ? a : a / 255.0f;
            for (int e = tid; e < 16 * 16; e += kHmThreads) {
                const int n = e >> 4, kk = e & 15;
                // layer 1: k 0..11 features, 12..15 zero (gamma(t) is in the bias)
                const float v1 = kk < 12 ? half_bits_to_float(__ldg(W1 + n * 16 + kk)) * ((kk >= 4 && kk < 8) ? s_uv : a) : 0.f;
                sW1[e] = __float2half_rn(v1);
                sW2[e] = __float2half_rn(0.5f * half_bits_to_float(__ldg(W2 + e)));
                if (n < 8) sW3[e] = __float2half_rn(n < 3 ? half_bits_to_float(__ldg(W3 + n * 16 + kk)) * (0.5f / a) : 0.f);
            }
            if (tid < 16) {
                float acc = half_bits_to_float(__ldg(b1 + tid));
                for (int g = 0; g < 4; ++g) acc = fmaf(half_bits_to_float(__ldg(W1 + tid * 16 + 12 + g)), tc.gamma[g], acc);
                sBias[tid] = a * acc;
                sBias[16 + tid] = a * half_bits_to_float(__ldg(b2 + tid));
                if (tid < 8) sBias[32 + tid] = tid < 3 ? half_bits_to_float(__ldg(b3 + tid)) : 0.f;
            }
        }
        __syncthreads();

        // per-lane fragment table: B fragments (b0 = W[n = nt*8 + lane/4][k = 2q..2q+1],
        // b1 = same at k + 8) and C fragments (bias of columns 2q, 2q+1 of each n8 tile)
        if (tid < 32) {
            const uint32_t* w1u = reinterpret_cast<const uint32_t*>(sW1);
            const uint32_t* w2u = reinterpret_cast<const uint32_t*>(sW2);
            const uint32_t* w3u = reinterpret_cast<const uint32_t*>(sW3);
            uint32_t* f = reinterpret_cast<uint32_t*>(smem + L.frag) + tid * 24;
            const int fq = tid & 3, fr = tid >> 2;
            for (int nt = 0; nt < 2; ++nt) {
                const int n = nt * 8 + fr;
                f[0 + 2 * nt] = w1u[n * 8 + fq];
                f[1 + 2 * nt] = w1u[n * 8 + 4 + fq];
                f[4 + 2 * nt] = w2u[n * 8 + fq];
                f[5 + 2 * nt] = w2u[n * 8 + 4 + fq];
                f[12 + 2 * nt] = __float_as_uint(sBias[nt * 8 + 2 * fq]);
                f[13 + 2 * nt] = __float_as_uint(sBias[nt * 8 + 2 * fq + 1]);
                f[16 + 2 * nt] = __float_as_uint(sBias[16 + nt * 8 + 2 * fq]);
                f[17 + 2 * nt] = __float_as_uint(sBias[16 + nt * 8 + 2 * fq + 1]);
            }
            f[8] = w3u[fr * 8 + fq];
            f[9] = w3u[fr * 8 + 4 + fq];
            f[20] = __float_as_uint(sBias[32 + 2 * fq]);
            f[21] = __float_as_uint(sBias[32 + 2 * fq + 1]);
        }
        __syncthreads();
        const uint4* fragq = reinterpret_cast<const uint4*>(smem + L.frag) + lane * 6;

        // gather-side per-thread column constants (thread owns column b*128 + tid)
        uint32_t cxb0[BPR], cxb1[BPR], cfx[BPR], cut[BPR];
#pragma unroll
        for (int b = 0; b < BPR; ++b) {
            const int i = b * 128 + tid;
            const float sx = fmaf((float)i + 0.5f, sc3, -0.5f);
            const float flx = floorf(sx);
            cxb0[b] = (uint32_t)clampi((int)flx, 0, R3 - 1) * 8u;
            cxb1[b] = (uint32_t)clampi((int)flx + 1, 0, R3 - 1) * 8u;
            cfx[b] = pack_f16x2(sx - flx, sx - flx);
            cut[b] = sUt[i];
        }
        const uint8_t* uvmap = p.uv + p.uv_tile_bytes * k;
        const uint8_t* sUvtB = reinterpret_cast<const uint8_t*>(sUvt);
        uint32_t* sUvw = reinterpret_cast<uint32_t*>(smem + L.base.uvc) + warp * (chunk_rows * BPR * 32);
        const int out_fmt = p.out_fmt;
        const bool tiles_border = !p.full && B > 0;
        // ldmatrix row address of this lane within an m16 tile (XOR-swizzled halves)
        const int lrow = (lane & 7) + ((lane >> 3) & 1) * 8, lhalf = lane >> 4;

        const int j_begin = strip * p.strip_rows, j_end = j_begin + p.strip_rows;
        for (int row = j_begin; row < j_end; ++row) {
            const int jr = row % chunk_rows;
            if (FMT_UV == FMT_BC7 && jr == 0) {
                // a3: this warp's 32 BC7 blocks of the chunk (one per lane)
                constexpr int bpw = 8 * BPR;
                const int br = lane / bpw, qq = lane % bpw, bb = qq >> 3, bc = qq & 7;
                const int gbc = 32 * bb + 8 * warp + bc;
                const uint4 raw = __ldg(reinterpret_cast<const uint4*>(uvmap) + ((row >> 2) + br) * (C >> 2) + gbc);
                uint32_t* dst = sUvw + ((4 * br) * BPR + bb) * 32 + 4 * bc;
                uint32_t rowv[4];
                __syncwarp();
                bc7_decode(raw, [&](int t, uint32_t v) {
                    rowv[t & 3] = v;
                    if ((t & 3) == 3)
                        *reinterpret_cast<uint4*>(dst + (t >> 2) * BPR * 32) = make_uint4(rowv[0], rowv[1], rowv[2], rowv[3]);
                });
                __syncwarp();
            }
            const uint4 rt = sRow[row];
#pragma unroll
            for (int blk = 0; blk < BPR; ++blk) {
                // ---- a4/a6: this lane's texel -> 16 f16 (Eq. 4 order, bias column 12 = 0) ----
                const uint2 t00 = *reinterpret_cast<const uint2*>(sUvtB + rt.x + cxb0[blk]);
                const uint2 t10 = *reinterpret_cast<const uint2*>(sUvtB + rt.x + cxb1[blk]);
                const uint2 t01 = *reinterpret_cast<const uint2*>(sUvtB + rt.y + cxb0[blk]);
                const uint2 t11 = *reinterpret_cast<const uint2*>(sUvtB + rt.y + cxb1[blk]);
                const uint32_t fx2 = cfx[blk];
                uint4 lo, hi;
                lo.x = hlerp2(hlerp2(t00.x, t10.x, fx2), hlerp2(t01.x, t11.x, fx2), rt.z);
                lo.y = hlerp2(hlerp2(t00.y, t10.y, fx2), hlerp2(t01.y, t11.y, fx2), rt.z);
                if (FMT_UV == FMT_BC7) {
                    u8x4_to_h2(sUvw[(jr * BPR + blk) * 32 + lane], lo.z, lo.w);
                } else if (FMT_UV == FMT_U8) {
                    u8x4_to_h2(__ldg(reinterpret_cast<const uint32_t*>(uvmap) + (size_t)row * C + blk * 128 + tid), lo.z, lo.w);
                } else {
                    const uint2 hv = __ldg(reinterpret_cast<const uint2*>(uvmap) + (size_t)row * C + blk * 128 + tid);
                    lo.z = hv.x;
                    lo.w = hv.y;
                }
                hi = make_uint4(cut[blk], rt.w, 0u, 0u);
                const int sw = (lane >> 2) & 1;
                __syncwarp();   // previous warp-row's ldmatrix reads done
                *reinterpret_cast<uint4*>(stage + lane * 32 + (sw << 4)) = lo;
                *reinterpret_cast<uint4*>(stage + lane * 32 + ((1 - sw) << 4)) = hi;
                __syncwarp();
                // ---- a7: three layers in registers, two m16 tiles ----
                uint32_t A0[4], A1[4];
                {
                    const int t0 = lrow, t1 = 16 + lrow;
                    ldsm_x4(stage_s + t0 * 32 + ((lhalf ^ ((t0 >> 2) & 1)) << 4), A0);
                    ldsm_x4(stage_s + t1 * 32 + ((lhalf ^ ((t1 >> 2) & 1)) << 4), A1);
                }
                float D0[2][4], D1[2][4];
                {
                    const uint4 f0 = fragq[0], f3 = fragq[3];   // W1 b-frags, b1' c-frags
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt) {
                        const uint32_t b0 = nt ? f0.z : f0.x, b1 = nt ? f0.w : f0.y;
                        const float c0 = __uint_as_float(nt ? f3.z : f3.x), c1 = __uint_as_float(nt ? f3.w : f3.y);
                        mma16816(D0[nt], A0, b0, b1, c0, c1);
                        mma16816(D1[nt], A1, b0, b1, c0, c1);
                    }
                }
                gelu_frag(D0[0], D0[1], A0);
                gelu_frag(D1[0], D1[1], A1);
                {
                    const uint4 f1 = fragq[1], f4 = fragq[4];   // W2 b-frags, b2' c-frags
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt) {
                        const uint32_t b0 = nt ? f1.z : f1.x, b1 = nt ? f1.w : f1.y;
                        const float c0 = __uint_as_float(nt ? f4.z : f4.x), c1 = __uint_as_float(nt ? f4.w : f4.y);
                        mma16816(D0[nt], A0, b0, b1, c0, c1);
                        mma16816(D1[nt], A1, b0, b1, c0, c1);
                    }
                }
                gelu_frag(D0[0], D0[1], A0);
                gelu_frag(D1[0], D1[1], A1);
                float Y0[4], Y1[4];
                {
                    const uint4 f2 = fragq[2], f5 = fragq[5];   // W3 b-frags, b3 c-frags
                    mma16816(Y0, A0, f2.x, f2.y, __uint_as_float(f5.x), __uint_as_float(f5.y));
                    mma16816(Y1, A1, f2.x, f2.y, __uint_as_float(f5.x), __uint_as_float(f5.y));
                }
                // ---- a8: lanes q = 0 (R,G) and q = 1 (B,-) hold rows r, r+8 of each m16 tile ->
                // transpose through the staging buffer so lane L writes texel L ----
                __syncwarp();   // ldmatrix reads of the staging buffer are done
                if (q < 2) {
                    float2* st2 = reinterpret_cast<float2*>(stage);
                    st2[(r8) * 2 + q] = make_float2(Y0[0], Y0[1]);
                    st2[(r8 + 8) * 2 + q] = make_float2(Y0[2], Y0[3]);
                    st2[(16 + r8) * 2 + q] = make_float2(Y1[0], Y1[1]);
                    st2[(24 + r8) * 2 + q] = make_float2(Y1[2], Y1[3]);
                }
                __syncwarp();
                const float4 yv = reinterpret_cast<const float4*>(stage)[lane];
                {
                    const int i = blk * 128 + tid;
                    const size_t o = out_base + (size_t)row * row_pitch + i;
                    if (out_fmt == OUT_RGBA8) reinterpret_cast<uint32_t*>(p.out)[o] = rgba8_fma(yv.x, yv.y, yv.z);
                    else store_texel(p.out, o, out_fmt, yv.x, yv.y, yv.z);
                    if (tiles_border) {
                        const int j = row;
                        const bool bx = (i >= 1 && i <= B) || (i >= C - 1 - B && i <= C - 2);
                        const bool by = (j >= 1 && j <= B) || (j >= C - 1 - B && j <= C - 2);
                        if (bx || by) {
                            const int xm = i <= B ? -i : 2 * (C - 1) - i;
                            const int ym = j <= B ? -j : 2 * (C - 1) - j;
                            const ptrdiff_t bs = (ptrdiff_t)out_base, rp = (ptrdiff_t)row_pitch;
                            if (bx) store_texel(p.out, (size_t)(bs + (ptrdiff_t)j * rp + xm), out_fmt, yv.x, yv.y, yv.z);
                            if (by) store_texel(p.out, (size_t)(bs + (ptrdiff_t)ym * rp + i), out_fmt, yv.x, yv.y, yv.z);
                            if (bx && by) store_texel(p.out, (size_t)(bs + (ptrdiff_t)ym * rp + xm), out_fmt, yv.x, yv.y, yv.z);
                        }
                    }
                }
            }
        }
    }
}

template <int FMT_UV, int CT>
static cudaError_t launch_hmma_t(const KParams& p, int num_sms, cudaStream_t s) {
    const HmSmem L = hm_smem_layout(CT, p.R3);
    auto kern = ndgi_fused_hmma_kernel<FMT_UV, CT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kHmThreads, L.total);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    const uint32_t cap = (uint32_t)(num_sms * occ);
    const uint32_t grid = p.units < cap ? p.units : cap;
    if (getenv("NDGI_VERBOSE"))
        fprintf(stderr, "[ndgi] fused_hmma<uv=%d,C=%d> occ=%d grid=%u units=%u strips=%d smem=%u\n", FMT_UV, CT, occ, grid,
                p.units, p.strips_per_tile, L.total);
    kern<<<grid, kHmThreads, L.total, s>>>(p);
    return cudaGetLastError();
}

int fused_hmma_ctas_per_sm() { return NDGI_HM_MIN_CTAS; }

// h = 16 only
cudaError_t launch_fused_hmma(const KParams& p, int num_sms, cudaStream_t s) {
    if (p.H != 16) return cudaErrorNotSupported;
    if (p.C == 128) {
        if (p.fmt_uv == FMT_BC7) return launch_hmma_t<FMT_BC7, 128>(p, num_sms, s);
        if (p.fmt_uv == FMT_U8) return launch_hmma_t<FMT_U8, 128>(p, num_sms, s);
        return launch_hmma_t<FMT_F16, 128>(p, num_sms, s);
    }
    if (p.fmt_uv == FMT_BC7) return launch_hmma_t<FMT_BC7, 256>(p, num_sms, s);
    if (p.fmt_uv == FMT_U8) return launch_hmma_t<FMT_U8, 256>(p, num_sms, s);
    return launch_hmma_t<FMT_F16, 256>(p, num_sms, s);
}

}  // namespace ndgi
