// fused_pipe_kernel.cu -- NDGI_MODE_FAST for h = 16: the software-pipelined
// variant of the fused tile-decode kernel (default for h = 16).
//
// Same hot path and arithmetic as fused_kernel.cu (SURVEY.md §8(a) a1-a8,
// DESIGN.md §6.1): BC7 decode, sampling, Eq. 4 input row, G_Phi on tcgen05
// (A in TMEM, B in smem, f16 accumulators for the hidden layers), tanh-form
// f16x2 GELU, RGBA8 writer.  What changes is the schedule.  Measured on the
// CTA-synchronous kernel, a warp spends ~30-40 % of a step waiting for the
// three MMA round trips of the step (CTA barrier skew + tcgen05 latency); here
// the work that does not depend on the in-flight MMA fills those waits:
//
//   step n:  wait L0(n) -> GELU -> A            | barrier, issue L1(n)
//            gather(n+1) -> A0                   (overlaps the L1 round trip)
//            wait L1(n) -> GELU -> A             | barrier, issue L2(n)
//            wait L2(n) -> y(n) to registers     | barrier, issue L0(n+1)
//            RGBA8 quantise + store y(n)         (overlaps the L0 round trip)
//
// To hold the next step's layer-1 input while the current step is in flight
// each 32-column TMEM slot is [A 8 | A0 8 | D 16]; the bias K chunk of the
// hidden layers is gone: b2 is preloaded into D (tcgen05.st .unpack::16b)
// and layer 2 accumulates onto it, b3 is added in the fp32 output epilogue.
// Layer 1's bias (with gamma(t), R6) stays in A0's ones column (k = 12).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "fused_common.cuh"

namespace ndgi {

constexpr int kPipeThreads = 128;
#ifndef NDGI_PIPE_MIN_CTAS
#define NDGI_PIPE_MIN_CTAS 8
#endif
#ifndef NDGI_PIPE_BIAS_ST
#define NDGI_PIPE_BIAS_ST 1   // 1: b2 preloaded into D; 0: added in the GELU epilogue (HADD2)
#endif

namespace pipe {
constexpr int S = 2;                 // 128-texel items per step
constexpr uint32_t SLOT = 32;        // TMEM columns per item
constexpr uint32_t TA = 0;           // hidden-layer A operand (K = 16 f16 = 8 columns)
constexpr uint32_t TA0 = 8;          // layer-1 A operand of the next step
constexpr uint32_t TD = 16;          // accumulators (16 f16, or 16 fp32 for the output layer)
constexpr uint32_t COLS = S * SLOT;  // 64
}  // namespace pipe

// RGBA8 / 16F / 32F writer of one core texel (+ its mirrored border copies, R3)
__device__ __forceinline__ void pipe_store(const KParams& p, size_t out_base, size_t row_pitch, int j, int i, int C,
                                           int B, bool tiles_border, int out_fmt, float y0, float y1, float y2) {
    const size_t o = out_base + (size_t)j * row_pitch + i;
    if (out_fmt == OUT_RGBA8) {
        const uint32_t v = rgba8_fma(y0, y1, y2);
        uint32_t* out = reinterpret_cast<uint32_t*>(p.out);
        out[o] = v;
        if (tiles_border) {
            const bool bx = (i >= 1 && i <= B) || (i >= C - 1 - B && i <= C - 2);
            const bool by = (j >= 1 && j <= B) || (j >= C - 1 - B && j <= C - 2);
            if (bx || by) {
                const ptrdiff_t xm = i <= B ? -i : 2 * (C - 1) - i;
                const ptrdiff_t ym = j <= B ? -j : 2 * (C - 1) - j;
                const ptrdiff_t base = (ptrdiff_t)out_base, rp = (ptrdiff_t)row_pitch;
                if (bx) out[base + j * rp + xm] = v;
                if (by) out[base + ym * rp + i] = v;
                if (bx && by) out[base + ym * rp + xm] = v;
            }
        }
        return;
    }
    store_texel(p.out, o, out_fmt, y0, y1, y2);
    if (tiles_border) {
        const bool bx = (i >= 1 && i <= B) || (i >= C - 1 - B && i <= C - 2);
        const bool by = (j >= 1 && j <= B) || (j >= C - 1 - B && j <= C - 2);
        if (bx || by) {
            const int xm = i <= B ? -i : 2 * (C - 1) - i;
            const int ym = j <= B ? -j : 2 * (C - 1) - j;
            const ptrdiff_t base = (ptrdiff_t)out_base, rp = (ptrdiff_t)row_pitch;
            if (bx) store_texel(p.out, (size_t)(base + (ptrdiff_t)j * rp + xm), out_fmt, y0, y1, y2);
            if (by) store_texel(p.out, (size_t)(base + (ptrdiff_t)ym * rp + i), out_fmt, y0, y1, y2);
            if (bx && by) store_texel(p.out, (size_t)(base + (ptrdiff_t)ym * rp + xm), out_fmt, y0, y1, y2);
        }
    }
}

template <int FMT_UV, int CT, bool FULL8>
__global__ void __launch_bounds__(kPipeThreads, NDGI_PIPE_MIN_CTAS)
    ndgi_fused_pipe_kernel(const __grid_constant__ KParams p) {
    using namespace pipe;
    constexpr int H = 16;
    constexpr int C = CT;
    constexpr int BPR = CT / kPipeThreads;
    constexpr int chunk_rows = kChunkTexels / CT;
    constexpr int chunk_steps = chunk_rows * BPR / S;
    extern __shared__ __align__(1024) uint8_t smem[];
    const FusedSmem L = fused_smem_layout<H>(C, p.R3);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t bars = ptx::smem_addr(smem + L.bars);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem_slot);
    // B operands, K-major no-swizzle [n/8][k/8][n%8][k%8], K = 16 for all three layers
    __half* sB1 = reinterpret_cast<__half*>(smem + L.b1);
    __half* sB2 = reinterpret_cast<__half*>(smem + L.b2);
    __half* sB3 = reinterpret_cast<__half*>(smem + L.b3);
    uint32_t* sBias2 = reinterpret_cast<uint32_t*>(smem + L.b2 + 512);   // a*b2 as 8 f16x2
    float* sBias3 = reinterpret_cast<float*>(smem + L.b3 + 512);         // b3 (fp32, exact)
    const uint32_t* sUt = reinterpret_cast<const uint32_t*>(smem + L.utcol);
    const uint4* sRow = reinterpret_cast<const uint4*>(smem + L.rowtab);
    uint4* sCol = reinterpret_cast<uint4*>(smem + L.colc);
    uint32_t* sUv = reinterpret_cast<uint32_t*>(smem + L.uvc);   // decoded F_uv chunk [chunk_rows][C]

    if (tid == 0) {
        ptx::mbar_init(bars, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc<COLS>(ptx::smem_addr(tmem_slot));
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tm_lane = tmem + ((uint32_t)(warp * 32) << 16);   // this warp's TMEM lane quarter

    const int B = p.B, P = p.P, R3 = p.R3;
    const float sc3 = (float)R3 * (1.0f / (float)C);
    const uint32_t idesc_h = ptx::idesc_f16_f16(128, 16);   // hidden layers: f16 accumulators
    const uint32_t idesc_y = ptx::idesc_f16_f32(128, 16);   // output layer: fp32
    const uint64_t bd1 = ptx::smem_desc_kmajor(ptx::smem_addr(sB1), 128u, 256u);
    const uint64_t bd2 = ptx::smem_desc_kmajor(ptx::smem_addr(sB2), 128u, 256u);
    const uint64_t bd3 = ptx::smem_desc_kmajor(ptx::smem_addr(sB3), 128u, 256u);
    uint32_t dph = 0u;

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
        const int nsteps = p.strip_rows * BPR / S;
        const int j_begin = strip * p.strip_rows;

        // ---- a2: tile parameters -> shared memory --------------------------------
        __syncthreads();   // previous unit: all MMAs complete, all smem readers done
        unit_prologue<H, FMT_UV, C, false>(p, tc, k, smem, L, tid, kPipeThreads);
        {
            // G_Phi with the GELU folds of DESIGN.md §6.1 (a = sqrt(2/pi)):
            // B1 = a W1 (F_uv columns /255, R8), k = 12 <- a (b1 + W1_gamma gamma(t));
            // B2 = W2 / 2, bias a b2 (preloaded into D); B3 = W3 / (2a), bias b3
            const uint16_t* w = p.mlp + p.mlp_tile_elems * k;
            const uint16_t *W1 = w, *b1 = W1 + 16 * H, *W2 = b1 + H, *b2 = W2 + H * H, *W3 = b2 + H, *b3 = W3 + 3 * H;
            const float a = kGeluA;
            const float s_uv = FMT_UV == FMT_F16 ? a : a / 255.0f;
            for (int e = tid; e < 16 * 16; e += kPipeThreads) {
                const int n = e >> 4, kk = e & 15;
                float v1 = 0.f;
                if (kk < 12) {
                    v1 = half_bits_to_float(__ldg(W1 + n * 16 + kk)) * ((kk >= 4 && kk < 8) ? s_uv : a);
                } else if (kk == 12) {
                    float acc = half_bits_to_float(__ldg(b1 + n));
                    for (int g = 0; g < 4; ++g) acc = fmaf(half_bits_to_float(__ldg(W1 + n * 16 + 12 + g)), tc.gamma[g], acc);
                    v1 = a * acc;
                }
                sB1[bofs(n, kk, 16)] = __float2half_rn(v1);
                sB2[bofs(n, kk, 16)] = __float2half_rn(0.5f * half_bits_to_float(__ldg(W2 + n * H + kk)));
                sB3[bofs(n, kk, 16)] =
                    __float2half_rn(n < 3 ? half_bits_to_float(__ldg(W3 + n * H + kk)) * (0.5f / a) : 0.f);
            }
            if (tid < 8)
                sBias2[tid] = pack_f16x2(a * half_bits_to_float(__ldg(b2 + 2 * tid)),
                                         a * half_bits_to_float(__ldg(b2 + 2 * tid + 1)));
            if (tid < 4) sBias3[tid] = tid < 3 ? half_bits_to_float(__ldg(b3 + tid)) : 0.f;
        }
        ptx::fence_proxy_async_smem();   // B operands: generic-proxy writes -> tensor core
        __syncthreads();

        // per-column gather constants (written and read by the same thread)
#pragma unroll
        for (int b = 0; b < BPR; ++b) {
            const int i = b * kPipeThreads + tid;
            const float sx = fmaf((float)i + 0.5f, sc3, -0.5f);
            const float flx = floorf(sx);
            sCol[i] = make_uint4(L.uvt + (uint32_t)clampi((int)flx, 0, R3 - 1) * 8u,
                                 L.uvt + (uint32_t)clampi((int)flx + 1, 0, R3 - 1) * 8u, pack_f16x2(sx - flx, sx - flx),
                                 sUt[i]);
        }
        const uint8_t* uvmap = p.uv + p.uv_tile_bytes * k;

        // a3: this warp's 32 BC7 blocks of the chunk starting at core row jc
        auto decode_chunk = [&](int jc) {
            constexpr int bpw = 8 * BPR;
            const int br = lane / bpw, q = lane % bpw, blk = q >> 3, bc = q & 7;
            const int gbc = 32 * blk + 8 * warp + bc;
            const uint4 raw = __ldg(reinterpret_cast<const uint4*>(uvmap) + ((jc >> 2) + br) * (C >> 2) + gbc);
            uint32_t* dst = sUv + (4 * br) * C + 4 * gbc;
            uint32_t rowv[4];
            __syncwarp();
            bc7_decode(raw, [&](int i, uint32_t v) {
                rowv[i & 3] = v;
                if ((i & 3) == 3)
                    *reinterpret_cast<uint4*>(dst + (i >> 2) * C) = make_uint4(rowv[0], rowv[1], rowv[2], rowv[3]);
            });
            __syncwarp();
        };

        // a4/a6: Eq. 4 input rows of step n -> A0 of both slots
        auto xlerp = [&](uint32_t yoff, const uint4& cc, uint32_t& lo, uint32_t& hi) {
            const uint2 a = *reinterpret_cast<const uint2*>(smem + yoff + cc.x);
            const uint2 b = *reinterpret_cast<const uint2*>(smem + yoff + cc.y);
            lo = hlerp2(a.x, b.x, cc.z);
            hi = hlerp2(a.y, b.y, cc.z);
        };
        auto finish_row = [&](int row, int jr, int blk, const uint4& rt, const uint4& cc, uint32_t y0lo, uint32_t y0hi,
                              uint32_t y1lo, uint32_t y1hi, int s) {
            uint32_t a1[8];
            a1[0] = hlerp2(y0lo, y1lo, rt.z);
            a1[1] = hlerp2(y0hi, y1hi, rt.z);
            if (FMT_UV == FMT_BC7) {
                u8x4_to_h2(sUv[jr * C + blk * kPipeThreads + tid], a1[2], a1[3]);
            } else if (FMT_UV == FMT_U8) {
                u8x4_to_h2(__ldg(reinterpret_cast<const uint32_t*>(uvmap) + (size_t)row * C + blk * kPipeThreads + tid),
                           a1[2], a1[3]);
            } else {
                const uint2 hv = __ldg(reinterpret_cast<const uint2*>(uvmap) + (size_t)row * C + blk * kPipeThreads + tid);
                a1[2] = hv.x;
                a1[3] = hv.y;
            }
            a1[4] = cc.w;
            a1[5] = rt.w;
            a1[6] = 0x00003C00u;   // k = 12: 1.0 (layer-1 bias column), k = 13: 0
            a1[7] = 0u;
            ptx::tmem_st_x8(tm_lane + s * SLOT + TA0, a1);
        };
        auto gather_step = [&](int n) {
            const int it = n * S;   // first item of the step
            const int c0 = (n / chunk_steps) * chunk_steps * S;
            if (FMT_UV == FMT_BC7 && it == c0) decode_chunk(j_begin + c0 / BPR);
            if constexpr (BPR == 1) {
                // two consecutive rows, usually between the same two F_uvt rows
                const int row = j_begin + it, jr = it - c0;
                const uint4 rt0 = sRow[row], rt1 = sRow[row + 1];
                const uint4 cc = sCol[tid];
                uint32_t y0lo, y0hi, y1lo, y1hi;
                xlerp(rt0.x, cc, y0lo, y0hi);
                xlerp(rt0.y, cc, y1lo, y1hi);
                finish_row(row, jr, 0, rt0, cc, y0lo, y0hi, y1lo, y1hi, 0);
                if (rt1.x != rt0.x || rt1.y != rt0.y) {
                    xlerp(rt1.x, cc, y0lo, y0hi);
                    xlerp(rt1.y, cc, y1lo, y1hi);
                }
                finish_row(row + 1, jr + 1, 0, rt1, cc, y0lo, y0hi, y1lo, y1hi, 1);
            } else {
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const int row = j_begin + (it + s) / BPR, jr = (it + s - c0) / BPR, blk = (it + s) % BPR;
                    const uint4 rt = sRow[row];
                    const uint4 cc = sCol[blk * kPipeThreads + tid];
                    uint32_t y0lo, y0hi, y1lo, y1hi;
                    xlerp(rt.x, cc, y0lo, y0hi);
                    xlerp(rt.y, cc, y1lo, y1hi);
                    finish_row(row, jr, blk, rt, cc, y0lo, y0hi, y1lo, y1hi, s);
                }
            }
        };

        // a8: page-cache writes of step n from registers
        uint32_t* const orow = reinterpret_cast<uint32_t*>(p.out) + out_base + (size_t)j_begin * row_pitch + tid;
        const uint32_t rp32 = (uint32_t)row_pitch;
        auto output_step = [&](int n, const float (&y)[S][3]) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const int it = n * S + s, jo = it / BPR, i = (it % BPR) * kPipeThreads + tid;
                if constexpr (FULL8) {
                    orow[(size_t)((uint32_t)jo * rp32) + (it % BPR) * kPipeThreads] = rgba8_fma(y[s][0], y[s][1], y[s][2]);
                } else {
                    pipe_store(p, out_base, row_pitch, j_begin + jo, i, C, B, !p.full && B > 0, p.out_fmt, y[s][0], y[s][1],
                               y[s][2]);
                }
            }
        };

        // all A/D TMEM traffic of this thread done -> CTA barrier -> one lane
        // of warp 0 issues layer l of both items and commits to d_ready
        auto sync_issue = [&](int l) {
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncthreads();
            if (warp == 0) {
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        const uint32_t slot = tmem + s * SLOT;
                        if (l == 0) ptx::mma_f16_ts(slot + TD, slot + TA0, bd1, idesc_h, 0u);
                        else if (l == 1) ptx::mma_f16_ts(slot + TD, slot + TA, bd2, idesc_h, NDGI_PIPE_BIAS_ST);
                        else ptx::mma_f16_ts(slot + TD, slot + TA, bd3, idesc_y, 0u);
                    }
                    ptx::mma_commit(bars);
                }
                __syncwarp();
            }
        };
        auto wait_d = [&]() {
            ptx::mbar_wait_spin(bars, dph);
            dph ^= 1u;
            ptx::tc_fence_after();
        };
        auto gelu_to_a = [&](uint32_t (&x)[S][8]) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
                uint32_t g[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) g[q] = gelu_scaled_f16x2(x[s][q]);
                ptx::tmem_st_x8(tm_lane + s * SLOT + TA, g);
            }
        };

        // ---- a7/a8: the pipelined step loop ----------------------------------------
        gather_step(0);
        sync_issue(0);
        float y[S][3];
        for (int step = 0; step < nsteps; ++step) {
            // layer 1 done: D <- a*b2, GELU -> A; previous step's page-cache writes
            wait_d();
            {
                uint32_t x[S][8];
#pragma unroll
                for (int s = 0; s < S; ++s) ptx::tmem_ld_x8_pack16(tm_lane + s * SLOT + TD, x[s]);
                ptx::tmem_wait_ld();
#if NDGI_PIPE_BIAS_ST
                {
                    const uint4 bl = reinterpret_cast<const uint4*>(sBias2)[0];
                    const uint4 bh = reinterpret_cast<const uint4*>(sBias2)[1];
                    const uint32_t bb[8] = {bl.x, bl.y, bl.z, bl.w, bh.x, bh.y, bh.z, bh.w};
#pragma unroll
                    for (int s = 0; s < S; ++s) ptx::tmem_st_x8_unpack16(tm_lane + s * SLOT + TD, bb);
                }
#endif
                if (step > 0) output_step(step - 1, y);
                gelu_to_a(x);
            }
            sync_issue(1);
            // layer 2 done: (+ a*b2) GELU -> A; next step's inputs -> A0
            wait_d();
            {
                uint32_t x[S][8];
#pragma unroll
                for (int s = 0; s < S; ++s) ptx::tmem_ld_x8_pack16(tm_lane + s * SLOT + TD, x[s]);
                ptx::tmem_wait_ld();
#if !NDGI_PIPE_BIAS_ST
                {
                    const uint4 bl = reinterpret_cast<const uint4*>(sBias2)[0];
                    const uint4 bh = reinterpret_cast<const uint4*>(sBias2)[1];
                    const uint32_t bb[8] = {bl.x, bl.y, bl.z, bl.w, bh.x, bh.y, bh.z, bh.w};
#pragma unroll
                    for (int s = 0; s < S; ++s)
#pragma unroll
                        for (int q = 0; q < 8; ++q) asm("add.rn.f16x2 %0, %0, %1;" : "+r"(x[s][q]) : "r"(bb[q]));
                }
#endif
                if (step + 1 < nsteps) gather_step(step + 1);
                gelu_to_a(x);
            }
            sync_issue(2);
            // output layer done: y -> registers, release D, start the next step
            wait_d();
            {
                uint32_t yv[S][4];
#pragma unroll
                for (int s = 0; s < S; ++s) ptx::tmem_ld_x4(tm_lane + s * SLOT + TD, yv[s]);
                ptx::tmem_wait_ld();
                const float4 b3 = *reinterpret_cast<const float4*>(sBias3);
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    y[s][0] = __uint_as_float(yv[s][0]) + b3.x;
                    y[s][1] = __uint_as_float(yv[s][1]) + b3.y;
                    y[s][2] = __uint_as_float(yv[s][2]) + b3.z;
                }
            }
            if (step + 1 < nsteps) sync_issue(0);
        }
        output_step(nsteps - 1, y);
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<COLS>(tmem);
}

template <int FMT_UV, int CT>
static cudaError_t launch_pipe_t(const KParams& p, int num_sms, cudaStream_t s) {
    const FusedSmem L = fused_smem_layout<16>(CT, p.R3);
    auto kern = (p.full && p.out_fmt == OUT_RGBA8) ? ndgi_fused_pipe_kernel<FMT_UV, CT, true>
                                                   : ndgi_fused_pipe_kernel<FMT_UV, CT, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    // resident CTAs per SM from the kernel's own resource use (the runtime's
    // occupancy query reports 1 for tcgen05 kernels on driver 580)
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    int dev = 0, smem_sm = 0, regs_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    const int regs_cta = ((fa.numRegs * 32 + 255) / 256) * 256 * (kPipeThreads / 32);
    const int smem_cta = (int)L.total + (int)fa.sharedSizeBytes + 1024;
    int occ = regs_sm / regs_cta;
    if (smem_sm / smem_cta < occ) occ = smem_sm / smem_cta;
    const int tmem_cap = 512 / (int)pipe::COLS;
    if (occ > tmem_cap) occ = tmem_cap;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    const uint32_t cap = (uint32_t)(num_sms * occ);
    const uint32_t grid = p.units < cap ? p.units : cap;
    if (getenv("NDGI_VERBOSE"))
        fprintf(stderr, "[ndgi] fused_pipe<uv=%d,C=%d> occ=%d (regs %d, local %zu) grid=%u units=%u strips=%d smem=%u\n",
                FMT_UV, CT, occ, fa.numRegs, fa.localSizeBytes, grid, p.units, p.strips_per_tile, L.total);
    kern<<<grid, kPipeThreads, L.total, s>>>(p);
    return cudaGetLastError();
}

// h = 16 only
cudaError_t launch_fused_pipe(const KParams& p, int num_sms, cudaStream_t s) {
    if (p.H != 16) return cudaErrorNotSupported;
    if (p.C == 128) {
        if (p.fmt_uv == FMT_BC7) return launch_pipe_t<FMT_BC7, 128>(p, num_sms, s);
        if (p.fmt_uv == FMT_U8) return launch_pipe_t<FMT_U8, 128>(p, num_sms, s);
        return launch_pipe_t<FMT_F16, 128>(p, num_sms, s);
    }
    if (p.fmt_uv == FMT_BC7) return launch_pipe_t<FMT_BC7, 256>(p, num_sms, s);
    if (p.fmt_uv == FMT_U8) return launch_pipe_t<FMT_U8, 256>(p, num_sms, s);
    return launch_pipe_t<FMT_F16, 256>(p, num_sms, s);
}

}  // namespace ndgi
