// fused_ws_kernel.cu -- NDGI_MODE_FAST, warp-specialised variant (h = 16).
//
// Same hot path and arithmetic as fused_kernel.cu (SURVEY.md §8(a) a1-a8,
// DESIGN.md §6.1); only the schedule differs.  A CTA has 9 warps:
//   warps 0-3  "epi" warps: the GELU epilogues (the MUFU-bound part)
//   warps 4-7  "io" warps : BC7 decode, gather of the Eq. 4 input row (a3-a6)
//                           and the page-cache writer (a8)
//   warp 8     "mma" warp : one elected lane issues every tcgen05.mma
// Warp w in 0-3 and 4-7 owns TMEM lane quarter w % 4.  NS = 8 TMEM slots of
// 32 columns carry 8 items (128-texel blocks) through the three layers at
// once; per slot s and item, mbarriers hand over
//   io  --a1[s]--> mma --d1[s]--> epi --a2[s]--> mma --d2[s]--> epi
//       --a3[s]--> mma --d3[s]--> io (output, then gather the next item into s).
// The epi warps interleave the layer-1 epilogue of item i with the layer-2
// epilogue of item i-D, so the MUFU pipe always has independent work while
// the tensor core runs the other layer; the mma warp issues layer 1 A items
// ahead.  No CTA barrier in the steady state.
#include <cstdio>
#include <cstdlib>

#include "fused_common.cuh"

namespace ndgi {

constexpr int kWsWarps = 9;
constexpr int kWsThreads = kWsWarps * 32;
constexpr int kWsNS = 8;    // TMEM slots per CTA (h = 16: 8 x 32 = 256 columns -> 2 CTAs per SM)
constexpr int kWsD = 4;     // layer-2 epilogues lag layer-1 epilogues by D items
constexpr int kWsA = 2;     // the mma warp issues layer 1 A items ahead of the epi warps
static_assert(kWsA + 1 + kWsD < kWsNS, "pipeline depth: slot reuse would deadlock");

struct WsBars {
    // mbarrier byte offsets (in a region after the common smem layout)
    uint32_t base;
    __device__ __forceinline__ uint32_t a1(int s) const { return base + 8u * s; }
    __device__ __forceinline__ uint32_t a2(int s) const { return base + 8u * (kWsNS + s); }
    __device__ __forceinline__ uint32_t a3(int s) const { return base + 8u * (2 * kWsNS + s); }
    __device__ __forceinline__ uint32_t d1(int s) const { return base + 8u * (3 * kWsNS + s); }
    __device__ __forceinline__ uint32_t d2(int s) const { return base + 8u * (4 * kWsNS + s); }
    __device__ __forceinline__ uint32_t d3(int s) const { return base + 8u * (5 * kWsNS + s); }
};

__host__ __device__ inline uint32_t ws_bars_offset(const FusedSmem& L) { return (L.total + 15u) & ~15u; }
__host__ __device__ inline uint32_t ws_smem_total(const FusedSmem& L) { return ws_bars_offset(L) + 6u * kWsNS * 8u; }

template <int FMT_UV, int CT>
__global__ void __launch_bounds__(kWsThreads, 2) ndgi_fused_ws_kernel(const __grid_constant__ KParams p) {
    constexpr int H = 16;
    using Cfg = FusedCfg<H>;
    constexpr int NS = kWsNS;
    constexpr int C = CT;
    constexpr int BPR = CT / 128;
    constexpr int chunk_rows = kChunkTexels / CT;
    extern __shared__ __align__(1024) uint8_t smem[];
    const FusedSmem L = fused_smem_layout<H>(C, p.R3);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const WsBars bar{ptx::smem_addr(smem) + ws_bars_offset(L)};
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem_slot);
    const uint2* sUvt = reinterpret_cast<const uint2*>(smem + L.uvt);
    const uint32_t* sUt = reinterpret_cast<const uint32_t*>(smem + L.utcol);
    const uint4* sRow = reinterpret_cast<const uint4*>(smem + L.rowtab);

    // ---- one-time setup ------------------------------------------------------------
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            ptx::mbar_init(bar.a1(s), 128);
            ptx::mbar_init(bar.a2(s), 128);
            ptx::mbar_init(bar.a3(s), 128);
            ptx::mbar_init(bar.d1(s), 1);
            ptx::mbar_init(bar.d2(s), 1);
            ptx::mbar_init(bar.d3(s), 1);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc<NS * Cfg::SLOT_COLS>(ptx::smem_addr(tmem_slot));
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tm_lane = tmem + ((uint32_t)((warp & 3) * 32) << 16);

    if (warp >= 4 && warp < 8) {   // bias chunk [1, 0, ..., 0] of every slot's layer-2/3 A operand
        uint32_t c[8] = {0x00003C00u, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int s = 0; s < NS; ++s) ptx::tmem_st_x8(tm_lane + s * Cfg::SLOT_COLS + Cfg::TM_A23 + H / 2, c);
        ptx::tmem_wait_st();
    }

    const int B = p.B, P = p.P, R3 = p.R3;
    const float sc3 = (float)R3 * (1.0f / (float)C);
    uint32_t base = 0;   // items processed by this CTA before the current unit (slot/phase origin)

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
        const int N = p.strip_rows * BPR;
        const int j_begin = strip * p.strip_rows;

        __syncthreads();   // every role finished the previous unit
        unit_prologue<H, FMT_UV, C>(p, tc, k, smem, L, tid, kWsThreads);
        ptx::fence_proxy_async_smem();
        __syncthreads();

        if (warp == 8) {
            // ============================ mma warp ============================
            const uint32_t idesc1 = ptx::idesc_f16_f32(128, H), idesc3 = ptx::idesc_f16_f32(128, 16);
            constexpr uint32_t sbo2 = (uint32_t)(Cfg::K2 / 8) * 128u;
            const uint64_t bd1 = ptx::smem_desc_kmajor(ptx::smem_addr(smem + L.b1), 128u, 256u);
            const uint64_t bd2 = ptx::smem_desc_kmajor(ptx::smem_addr(smem + L.b2), 128u, sbo2);
            const uint64_t bd3 = ptx::smem_desc_kmajor(ptx::smem_addr(smem + L.b3), 128u, sbo2);
            for (int i = -kWsA; i <= N + kWsD; ++i) {
                const int l1 = i + kWsA, l2 = i - 1, l3 = i - 1 - kWsD;
                if (l1 >= 0 && l1 < N) {
                    const uint32_t g = base + l1, s = g % NS;
                    ptx::mbar_wait_fast(bar.a1(s), (g / NS) & 1u);
                    ptx::tc_fence_after();
                    if (ptx::elect_one()) {
                        const uint32_t sl = tmem + s * Cfg::SLOT_COLS;
                        ptx::mma_f16_ts(sl + Cfg::TM_D, sl + Cfg::TM_A1, bd1, idesc1, 0u);
                        ptx::mma_commit(bar.d1(s));
                    }
                    __syncwarp();
                }
                if (l2 >= 0 && l2 < N) {
                    const uint32_t g = base + l2, s = g % NS;
                    ptx::mbar_wait_fast(bar.a2(s), (g / NS) & 1u);
                    ptx::tc_fence_after();
                    if (ptx::elect_one()) {
                        const uint32_t sl = tmem + s * Cfg::SLOT_COLS;
                        ptx::mma_f16_ts(sl + Cfg::TM_D, sl + Cfg::TM_A23, bd2, idesc1, 0u);
                        ptx::mma_f16_ts(sl + Cfg::TM_D, sl + Cfg::TM_A23 + 8u, bd2 + 16u, idesc1, 1u);
                        ptx::mma_commit(bar.d2(s));
                    }
                    __syncwarp();
                }
                if (l3 >= 0 && l3 < N) {
                    const uint32_t g = base + l3, s = g % NS;
                    ptx::mbar_wait_fast(bar.a3(s), (g / NS) & 1u);
                    ptx::tc_fence_after();
                    if (ptx::elect_one()) {
                        const uint32_t sl = tmem + s * Cfg::SLOT_COLS;
                        ptx::mma_f16_ts(sl + Cfg::TM_D, sl + Cfg::TM_A23, bd3, idesc3, 0u);
                        ptx::mma_f16_ts(sl + Cfg::TM_D, sl + Cfg::TM_A23 + 8u, bd3 + 16u, idesc3, 1u);
                        ptx::mma_commit(bar.d3(s));
                    }
                    __syncwarp();
                }
            }
        } else if (warp < 4) {
            // ============================ epi warps ===========================
            // iteration i: layer-1 epilogue of item i and layer-2 epilogue of item i-D
            for (int i = 0; i < N + kWsD; ++i) {
                const int j = i - kWsD;
                const bool e1 = i < N, e2 = j >= 0;
                const uint32_t g1 = base + i, s1 = g1 % NS;
                const uint32_t g2 = base + j, s2 = g2 % NS;
                uint32_t x[16], y[16];
                if (e1) {
                    ptx::mbar_wait_fast(bar.d1(s1), (g1 / NS) & 1u);
                    ptx::tc_fence_after();
                    ptx::tmem_ld_x16(tm_lane + s1 * Cfg::SLOT_COLS + Cfg::TM_D, x);
                }
                if (e2) {
                    ptx::mbar_wait_fast(bar.d2(s2), (g2 / NS) & 1u);
                    ptx::tc_fence_after();
                    ptx::tmem_ld_x16(tm_lane + s2 * Cfg::SLOT_COLS + Cfg::TM_D, y);
                }
                ptx::tmem_wait_ld();
                uint32_t gx[8], gy[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    gx[q] = gelu_scaled_f16x2(pack_f16x2(__uint_as_float(x[2 * q]), __uint_as_float(x[2 * q + 1])));
                    gy[q] = gelu_scaled_f16x2(pack_f16x2(__uint_as_float(y[2 * q]), __uint_as_float(y[2 * q + 1])));
                }
                if (e1) ptx::tmem_st_x8(tm_lane + s1 * Cfg::SLOT_COLS + Cfg::TM_A23, gx);
                if (e2) ptx::tmem_st_x8(tm_lane + s2 * Cfg::SLOT_COLS + Cfg::TM_A23, gy);
                ptx::tmem_wait_st();
                ptx::tc_fence_before();
                if (e1) ptx::mbar_arrive(bar.a2(s1));
                if (e2) ptx::mbar_arrive(bar.a3(s2));
            }
        } else {
            // ============================ io warps ============================
            const int q = warp - 4;                  // TMEM lane quarter / column group
            const int tq = q * 32 + lane;            // column within a 128-texel block
            uint32_t cxb0[BPR], cxb1[BPR], cfx[BPR], cut[BPR];
#pragma unroll
            for (int b = 0; b < BPR; ++b) {
                const int i = b * 128 + tq;
                const float sx = fmaf((float)i + 0.5f, sc3, -0.5f);
                const float flx = floorf(sx);
                cxb0[b] = (uint32_t)clampi((int)flx, 0, R3 - 1) * 8u;
                cxb1[b] = (uint32_t)clampi((int)flx + 1, 0, R3 - 1) * 8u;
                cfx[b] = pack_f16x2(sx - flx, sx - flx);
                cut[b] = sUt[i];
            }
            const uint8_t* uvmap = p.uv + p.uv_tile_bytes * k;
            const uint8_t* sUvtB = reinterpret_cast<const uint8_t*>(sUvt);
            uint32_t* sUvw = reinterpret_cast<uint32_t*>(smem + L.uvc) + q * (chunk_rows * BPR * 32);
            const int out_fmt = p.out_fmt;
            const bool tiles_border = !p.full && B > 0;
            for (int i = 0; i < N + NS; ++i) {
                const int j = i - NS;
                if (j >= 0) {
                    // a8: y of item j -> page cache
                    const uint32_t g = base + j, s = g % NS;
                    ptx::mbar_wait_fast(bar.d3(s), (g / NS) & 1u);
                    ptx::tc_fence_after();
                    uint32_t yv[4];
                    ptx::tmem_ld_x4(tm_lane + s * Cfg::SLOT_COLS + Cfg::TM_D, yv);
                    ptx::tmem_wait_ld();
                    const int row = j_begin + j / BPR, col = (j % BPR) * 128 + tq;
                    const float y0f = __uint_as_float(yv[0]), y1f = __uint_as_float(yv[1]), y2f = __uint_as_float(yv[2]);
                    const size_t o = out_base + (size_t)row * row_pitch + col;
                    if (out_fmt == OUT_RGBA8) reinterpret_cast<uint32_t*>(p.out)[o] = rgba8_fma(y0f, y1f, y2f);
                    else store_texel(p.out, o, out_fmt, y0f, y1f, y2f);
                    if (tiles_border) {
                        const bool bx = (col >= 1 && col <= B) || (col >= C - 1 - B && col <= C - 2);
                        const bool by = (row >= 1 && row <= B) || (row >= C - 1 - B && row <= C - 2);
                        if (bx || by) {
                            const int xm = col <= B ? -col : 2 * (C - 1) - col;
                            const int ym = row <= B ? -row : 2 * (C - 1) - row;
                            const ptrdiff_t bs = (ptrdiff_t)out_base, rp = (ptrdiff_t)row_pitch;
                            if (bx) store_texel(p.out, (size_t)(bs + (ptrdiff_t)row * rp + xm), out_fmt, y0f, y1f, y2f);
                            if (by) store_texel(p.out, (size_t)(bs + (ptrdiff_t)ym * rp + col), out_fmt, y0f, y1f, y2f);
                            if (bx && by) store_texel(p.out, (size_t)(bs + (ptrdiff_t)ym * rp + xm), out_fmt, y0f, y1f, y2f);
                        }
                    }
                }
                if (i < N) {
                    // a3/a4/a6: Eq. 4 input row of item i -> A1 of its slot
                    const uint32_t g = base + i, s = g % NS;
                    const int row = j_begin + i / BPR, blk = i % BPR;
                    const int jr = row % chunk_rows;
                    if (FMT_UV == FMT_BC7 && jr == 0 && blk == 0) {
                        // this warp's 32 BC7 blocks of the chunk (one per lane)
                        constexpr int bpw = 8 * BPR;
                        const int br = lane / bpw, qq = lane % bpw, bb = qq >> 3, bc = qq & 7;
                        const int gbc = 32 * bb + 8 * q + bc;
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
                    const uint2 t00 = *reinterpret_cast<const uint2*>(sUvtB + rt.x + cxb0[blk]);
                    const uint2 t10 = *reinterpret_cast<const uint2*>(sUvtB + rt.x + cxb1[blk]);
                    const uint2 t01 = *reinterpret_cast<const uint2*>(sUvtB + rt.y + cxb0[blk]);
                    const uint2 t11 = *reinterpret_cast<const uint2*>(sUvtB + rt.y + cxb1[blk]);
                    const uint32_t fx2 = cfx[blk];
                    uint32_t a1[8];
                    a1[0] = hlerp2(hlerp2(t00.x, t10.x, fx2), hlerp2(t01.x, t11.x, fx2), rt.z);
                    a1[1] = hlerp2(hlerp2(t00.y, t10.y, fx2), hlerp2(t01.y, t11.y, fx2), rt.z);
                    if (FMT_UV == FMT_BC7) {
                        u8x4_to_h2(sUvw[(jr * BPR + blk) * 32 + lane], a1[2], a1[3]);
                    } else if (FMT_UV == FMT_U8) {
                        u8x4_to_h2(__ldg(reinterpret_cast<const uint32_t*>(uvmap) + (size_t)row * C + blk * 128 + tq), a1[2], a1[3]);
                    } else {
                        const uint2 hv = __ldg(reinterpret_cast<const uint2*>(uvmap) + (size_t)row * C + blk * 128 + tq);
                        a1[2] = hv.x;
                        a1[3] = hv.y;
                    }
                    a1[4] = cut[blk];
                    a1[5] = rt.w;
                    a1[6] = 0x00003C00u;
                    a1[7] = 0u;
                    ptx::tmem_st_x8(tm_lane + s * Cfg::SLOT_COLS + Cfg::TM_A1, a1);
                    ptx::tmem_wait_st();
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(bar.a1(s));
                }
            }
        }
        base += (uint32_t)N;
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<NS * Cfg::SLOT_COLS>(tmem);
}

template <int FMT_UV, int CT>
static cudaError_t launch_ws_t(const KParams& p, int num_sms, cudaStream_t s) {
    const FusedSmem L = fused_smem_layout<16>(CT, p.R3);
    const uint32_t smem = ws_smem_total(L);
    auto kern = ndgi_fused_ws_kernel<FMT_UV, CT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int occ = 2;   // TMEM: 2 x 256 columns
    const uint32_t cap = (uint32_t)(num_sms * occ);
    const uint32_t grid = p.units < cap ? p.units : cap;
    if (getenv("NDGI_VERBOSE"))
        fprintf(stderr, "[ndgi] fused_ws<uv=%d,C=%d> grid=%u units=%u strips=%d smem=%u\n", FMT_UV, CT, grid, p.units,
                p.strips_per_tile, smem);
    kern<<<grid, kWsThreads, smem, s>>>(p);
    return cudaGetLastError();
}

// h = 16 only; returns cudaErrorNotSupported for other widths
cudaError_t launch_fused_ws(const KParams& p, int num_sms, cudaStream_t s) {
    if (p.H != 16) return cudaErrorNotSupported;
    if (p.C == 128) {
        if (p.fmt_uv == FMT_BC7) return launch_ws_t<FMT_BC7, 128>(p, num_sms, s);
        if (p.fmt_uv == FMT_U8) return launch_ws_t<FMT_U8, 128>(p, num_sms, s);
        return launch_ws_t<FMT_F16, 128>(p, num_sms, s);
    }
    if (p.fmt_uv == FMT_BC7) return launch_ws_t<FMT_BC7, 256>(p, num_sms, s);
    if (p.fmt_uv == FMT_U8) return launch_ws_t<FMT_U8, 256>(p, num_sms, s);
    return launch_ws_t<FMT_F16, 256>(p, num_sms, s);
}

}  // namespace ndgi
