// host.cu -- the C ABI of libndgi.so (include/ndgi.h): validation, context,
// call setup and kernel launches.  No torch types cross
// this boundary; every entry point returns an ndgi_status and never throws.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/ndgi.h"
#include "ndgi_common.cuh"

namespace ndgi {
cudaError_t launch_ref(const KParams& p, cudaStream_t stream);
cudaError_t launch_fused(const KParams& p, int num_sms, cudaStream_t s);
int fused_ctas_per_sm(int H);
cudaError_t launch_sample(const SampleArgs& a, cudaStream_t s);
cudaError_t launch_bc7_encode_mode6(const void* rgba, int w, int h, void* blocks, int num_sms, cudaStream_t s);
cudaError_t launch_train_grad(const TrainArgs& a, int H, cudaStream_t s);
cudaError_t launch_convert_f32_f16_2d(const float* in, size_t in_stride, uint16_t* out, size_t out_stride, size_t rows,
                                      size_t cols, cudaStream_t s);
cudaError_t launch_bc7_encode_multi(const void* rgba, int w, int h, void* blocks, int num_sms, cudaStream_t s);
cudaError_t launch_full_ptq(const float* theta, size_t P, size_t off_uv, size_t off_uvt, size_t off_ut, size_t off_vt,
                            int num_tiles, int R, int R3, int D, int nline, uint32_t* uv_img, uint32_t* uvt_img,
                            uint8_t* ut, uint8_t* vt, int num_sms, cudaStream_t s);
cudaError_t launch_bc7_encode_mode6(const void* rgba, int w, int h, void* blocks, int num_sms, cudaStream_t s);
cudaError_t launch_adam(float* theta, float* m, float* v, int* steps, const float* grad, const uint32_t* tile_ids,
                        int n, size_t P, int num_tiles, float lr, float b1, float b2, float eps, size_t proj,
                        cudaStream_t s);
cudaError_t launch_convert_f16_f32(const uint16_t* in, float* out, size_t n, cudaStream_t s);
cudaError_t launch_convert_f32_f16(const float* in, uint16_t* out, size_t n, cudaStream_t s);
cudaError_t uv_textures_build(const void* uv, int atlases, int tiles_x, int tiles_y, int C, cudaArray_t* arrays,
                              unsigned long long* texs);
void uv_textures_free(int atlases, cudaArray_t* arrays, unsigned long long* texs);
size_t wpack_tile_bytes(int H);
cudaError_t prep_weights(const uint16_t* mlp, size_t tile_elems, int H, int fmt_uv, uint8_t* out, int num_tiles,
                         cudaStream_t s);
cudaError_t launch_bc7_map(const void* blocks, uint32_t w, uint32_t h, uint8_t* rgba, cudaStream_t s);
cudaError_t bc7_decode_hw(const void* blocks, uint32_t w, uint32_t h, uint8_t* rgba);
cudaError_t gelu_rate(uint32_t iters, uint32_t mufu_pairs, int pack, float* ms, double* acts);
int fused_gelu_mufu_pairs(int H);
cudaError_t null_launch(cudaStream_t s, int kind);
int fused_f16acc();
cudaError_t mma_latency(uint32_t iters, double* cycles_per_iter);
cudaError_t tmem_f16_probe(uint32_t* host_out);
cudaError_t f16d_probe(uint32_t seed, uint32_t iters, uint32_t ctas, unsigned long long* mism,
                       unsigned long long* total);
}  // namespace ndgi

struct ndgi_ctx {
    ndgi_layout L;
    ndgi_params P;
    int device;
    int num_sms;
    uint32_t* d_err;
    // dynamic-scheduling counters of the fused kernel (KParams::sched): a ring
    // of kSchedSlots, one per launch, so launches in flight on different
    // streams do not share one (each is zeroed on the launch's stream first)
    uint32_t* d_sched;
    mutable std::atomic<uint32_t> sched_seq;
    uint8_t* wpack;   // prepacked tcgen05 B operands per tile (FAST layouts), owned
    // NDGI_MODE_FAST_TEXUNIT: per-atlas BC7 F_uv textures, built on first use
    std::mutex tex_mu;
    bool tex_ready;
    cudaArray_t uvarr[ndgi::kMaxTexAtlases];
    unsigned long long uvtex[ndgi::kMaxTexAtlases];
    // host-buffer path (ndgi_decode_full_host): staging buffers and streams
    // shared by every caller of the context, so the whole call holds host_mu
    std::mutex host_mu;
    cudaStream_t hstream[2];
    cudaEvent_t hevent[2];
    void* stage[2];
    size_t stage_bytes;
};

namespace {

// NVTX range per C-ABI call (SURVEY §5 tracing): visible in nsys / ncu timelines;
// a no-op (one predictable branch) when no tool is attached
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

thread_local std::string g_last_error;

ndgi_status fail(ndgi_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

ndgi_status cuda_fail(cudaError_t e, const char* where) {
    g_last_error = std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return NDGI_ERR_CUDA;
}

// restores the caller's current device on scope exit
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

size_t map2d_bytes(uint32_t fmt, uint32_t rx, uint32_t ry, uint32_t nc) {
    if (fmt == NDGI_FMT_BC7 || fmt == NDGI_FMT_BC3 || fmt == NDGI_FMT_BC5) return (size_t)(rx / 4) * (ry / 4) * 16;
    if (fmt == NDGI_FMT_BC1) return (size_t)(rx / 4) * (ry / 4) * 8;
    return (size_t)rx * ry * nc * (fmt == NDGI_FMT_U8 ? 1 : 2);
}

size_t mlp_elems(uint32_t h) { return (size_t)16 * h + h + (size_t)h * h + h + 3 * (size_t)h + 3; }

// 4-channel maps: BC7, U8, F16, BC1, BC3; 2-channel line maps: U8, F16, BC5
bool fmt_ok(uint32_t f) { return f <= NDGI_FMT_BC3; }
bool fmt_block(uint32_t f) { return f == NDGI_FMT_BC7 || f == NDGI_FMT_BC1 || f == NDGI_FMT_BC3 || f == NDGI_FMT_BC5; }

ndgi_status validate(const ndgi_layout* L, int* fast) {
    if (!L) return fail(NDGI_ERR_ARG, "layout is NULL");
    if (L->abi_version != NDGI_ABI_VERSION) return fail(NDGI_ERR_ARG, "abi_version mismatch");
    if (L->num_tiles == 0) return fail(NDGI_ERR_ARG, "num_tiles == 0");
    if ((uint64_t)L->atlases * L->tiles_x * L->tiles_y != L->num_tiles)
        return fail(NDGI_ERR_ARG, "num_tiles != atlases*tiles_y*tiles_x");
    if (L->core < 4 || L->core % 4 != 0) return fail(NDGI_ERR_ARG, "core must be a multiple of 4, >= 4");
    if (L->border >= L->core) return fail(NDGI_ERR_ARG, "border must be < core");
    if (L->uv_res == 0 || L->uvt_res == 0 || L->uvt_depth == 0 || L->line_res == 0 || L->line_t == 0)
        return fail(NDGI_ERR_ARG, "zero resolution");
    if (!fmt_ok(L->fmt_uv) || !fmt_ok(L->fmt_uvt)) return fail(NDGI_ERR_ARG, "bad feature format");
    if (L->fmt_line != NDGI_FMT_U8 && L->fmt_line != NDGI_FMT_F16 && L->fmt_line != NDGI_FMT_BC5)
        return fail(NDGI_ERR_ARG, "fmt_line must be U8, F16 or BC5");
    if (fmt_block(L->fmt_uv) && L->uv_res % 4) return fail(NDGI_ERR_ARG, "block-compressed F_uv resolution must be a multiple of 4");
    if (fmt_block(L->fmt_uvt) && L->uvt_res % 4) return fail(NDGI_ERR_ARG, "block-compressed F_uvt resolution must be a multiple of 4");
    if (L->fmt_line == NDGI_FMT_BC5 && (L->line_res % 4 || L->line_t % 4))
        return fail(NDGI_ERR_ARG, "BC5 line maps need line_res and line_t multiples of 4");
    if (L->hidden < 1 || L->hidden > 256) return fail(NDGI_ERR_ARG, "hidden must be in [1, 256]");
    if (L->gelu > NDGI_GELU_TANH) return fail(NDGI_ERR_ARG, "bad gelu");
    if (L->border_mode > NDGI_BORDER_EVAL_CLAMP) return fail(NDGI_ERR_ARG, "bad border_mode");
    if (fast) {
        *fast = (L->core == 128 || L->core == 256) && L->uv_res == L->core && (L->hidden == 16 || L->hidden == 64) &&
                L->border_mode == NDGI_BORDER_MIRROR && L->uvt_res <= 64 && L->line_res <= 256 &&
                L->uvt_res >= 4;
    }
    return NDGI_OK;
}

// call setup (a1): gamma(t), slice and row indices, in fp64 (R4, R5, Eq. 4)
ndgi::TConst make_tconst(const ndgi_layout& L, double t) {
    ndgi::TConst c{};
    c.t = (float)t;
    c.gamma[0] = (float)std::sin(M_PI * t);
    c.gamma[1] = (float)std::cos(M_PI * t);
    c.gamma[2] = (float)std::sin(2.0 * M_PI * t);
    c.gamma[3] = (float)std::cos(2.0 * M_PI * t);
    auto axis = [](double s, int n, int& i0, int& i1, float& f) {
        const double fl = std::floor(s);
        f = (float)(s - fl);
        const int a = (int)fl;
        i0 = a < 0 ? 0 : (a > n - 1 ? n - 1 : a);
        i1 = a + 1 < 0 ? 0 : (a + 1 > n - 1 ? n - 1 : a + 1);
    };
    axis(t * L.uvt_depth - 0.5, (int)L.uvt_depth, c.k0, c.k1, c.tau);
    axis(t * L.line_t - 0.5, (int)L.line_t, c.r0, c.r1, c.rho);
    return c;
}

void fill_common(const ndgi_ctx* ctx, ndgi::KParams& p) {
    const ndgi_layout& L = ctx->L;
    memset(&p, 0, sizeof(p));
    p.C = (int)L.core;
    p.B = (int)L.border;
    p.P = (int)(L.core + 2 * L.border);
    p.R_uv = (int)L.uv_res;
    p.R3 = (int)L.uvt_res;
    p.D = (int)L.uvt_depth;
    p.U = (int)L.line_res;
    p.T = (int)L.line_t;
    p.H = (int)L.hidden;
    p.fmt_uv = (int)L.fmt_uv;
    p.fmt_uvt = (int)L.fmt_uvt;
    p.fmt_line = (int)L.fmt_line;
    p.gelu = (int)L.gelu;
    p.border_mode = (int)L.border_mode;
    p.atlases = (int)L.atlases;
    p.tiles_x = (int)L.tiles_x;
    p.tiles_y = (int)L.tiles_y;
    p.num_tiles = (int)L.num_tiles;
    p.uv = static_cast<const uint8_t*>(ctx->P.uv);
    p.uvt = static_cast<const uint8_t*>(ctx->P.uvt);
    p.ut = static_cast<const uint8_t*>(ctx->P.ut);
    p.vt = static_cast<const uint8_t*>(ctx->P.vt);
    p.mlp = ctx->P.mlp;
    p.wpack = ctx->wpack;
    p.uv_tile_bytes = map2d_bytes(L.fmt_uv, L.uv_res, L.uv_res, 4);
    p.uvt_slice_bytes = map2d_bytes(L.fmt_uvt, L.uvt_res, L.uvt_res, 4);
    p.uvt_tile_bytes = p.uvt_slice_bytes * L.uvt_depth;
    p.line_tile_bytes = map2d_bytes(L.fmt_line, L.line_res, L.line_t, 2);
    p.mlp_tile_elems = mlp_elems(L.hidden);
    p.err = ctx->d_err;
    p.sched = ctx->d_sched + (ctx->sched_seq.fetch_add(1, std::memory_order_relaxed) % ndgi::kSchedSlots);
}

ndgi_status check_t(float t) {
    if (!std::isfinite(t) || t < 0.0f || t > 1.0f) return fail(NDGI_ERR_RANGE, "t must be finite and in [0, 1]");
    return NDGI_OK;
}

// work decomposition of the fused kernel (strips of core rows per tile).
// Strips are whole 2048-texel F_uv chunks, or -- default kernel -- down to
// min_rows = 4 rows (one BC7 block row).  More strips mean more parallel
// units but one tile prologue per unit; the measured VT optimum (config 3,
// scripts/strip_sweep.py: n = 8/32/128/512 -> 32/16/8/4 strips) follows
// s^2 * requests >= 8192.  Kernels without short strips: >= 2 waves.
void choose_strips(ndgi::KParams& p, int num_sms, int min_rows) {
    const int C = p.C;
    const int chunk_rows = 2048 / C;
    const int max_strips = C / (min_rows < chunk_rows ? min_rows : chunk_rows);
    const uint64_t req = (uint64_t)p.nt * p.n_req;
    int s = 1;
    if (min_rows < chunk_rows) {
        while (s < max_strips && (uint64_t)s * s * req < 8192u) s *= 2;
    } else {
        const uint64_t target = 2ull * num_sms * ndgi::fused_ctas_per_sm(p.H);
        while (s < max_strips && req * s < target) s *= 2;
    }
    p.strips_per_tile = s;
    p.strip_rows = C / s;
    p.units = (uint32_t)((uint64_t)p.nt * p.n_req * s);
    p.tail_from = p.units;
    p.tail_strips = 1;
    // whole-tile units over several rounds of resident CTAs (decode_full, large
    // batches): the last ~one round of requests as 4 strips each, so the final
    // dynamically claimed units (KParams::sched) are a quarter as long and the
    // SMs stay full until closer to the end
    const uint64_t resident = (uint64_t)num_sms * ndgi::fused_ctas_per_sm(p.H);
#ifndef NDGI_TAIL_STRIPS   // experiment builds: 1 = no finer tail
#define NDGI_TAIL_STRIPS 4
#endif
    constexpr int kTail = NDGI_TAIL_STRIPS;
    if (kTail > 1 && s == 1 && req > 2 * resident && (C / kTail) % chunk_rows == 0) {
        const uint64_t tail = resident;
        p.tail_from = (uint32_t)(req - tail);
        p.tail_strips = kTail;
        p.units = (uint32_t)(req - tail + kTail * tail);
    }
}

ndgi_status launch(ndgi_ctx* ctx, ndgi::KParams& p, ndgi_mode mode, cudaStream_t s) {
    int fast = 0;
    validate(&ctx->L, &fast);
    cudaError_t e;
    if (mode == NDGI_MODE_FAST_TEXUNIT) {
        if (!fast) return fail(NDGI_ERR_UNSUPPORTED, "layout not supported by NDGI_MODE_FAST (see ndgi.h)");
        if (ctx->L.fmt_uv != NDGI_FMT_BC7 || ctx->L.atlases > (uint32_t)ndgi::kMaxTexAtlases)
            return fail(NDGI_ERR_UNSUPPORTED, "NDGI_MODE_FAST_TEXUNIT needs BC7 F_uv and <= 64 atlases");
        {
            std::lock_guard<std::mutex> lock(ctx->tex_mu);
            if (!ctx->tex_ready) {
                e = ndgi::uv_textures_build(ctx->P.uv, (int)ctx->L.atlases, (int)ctx->L.tiles_x, (int)ctx->L.tiles_y,
                                            (int)ctx->L.core, ctx->uvarr, ctx->uvtex);
                if (e != cudaSuccess) {
                    ndgi::uv_textures_free((int)ctx->L.atlases, ctx->uvarr, ctx->uvtex);
                    return cuda_fail(e, "building the BC7 F_uv textures");
                }
                ctx->tex_ready = true;
            }
        }
        for (uint32_t a = 0; a < ctx->L.atlases; ++a) p.uvtex[a] = ctx->uvtex[a];
        p.fmt_uv = ndgi::FMT_BC7_TEX;
        choose_strips(p, ctx->num_sms, 4);
        e = ndgi::launch_fused(p, ctx->num_sms, s);
    } else if (mode == NDGI_MODE_FAST) {
        if (!fast) return fail(NDGI_ERR_UNSUPPORTED, "layout not supported by NDGI_MODE_FAST (see ndgi.h)");
        choose_strips(p, ctx->num_sms, 4);
        e = ndgi::launch_fused(p, ctx->num_sms, s);
    } else {
        e = ndgi::launch_ref(p, s);
    }
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    return NDGI_OK;
}

bool mode_ok(int m) { return m == NDGI_MODE_FAST || m == NDGI_MODE_REF_FP32 || m == NDGI_MODE_FAST_TEXUNIT; }
bool out_ok(int f) { return f >= NDGI_OUT_RGBA8 && f <= NDGI_OUT_RGBA32F; }

ndgi_status decode_full_async(ndgi_ctx* ctx, const float* ts, uint32_t nt, void* out, ndgi_out_fmt fmt,
                              ndgi_mode mode, cudaStream_t stream) {
    const size_t per_t = ndgi_full_texels(&ctx->L);
    for (uint32_t t0 = 0; t0 < nt; t0 += ndgi::kMaxT) {
        const uint32_t n = nt - t0 < (uint32_t)ndgi::kMaxT ? nt - t0 : (uint32_t)ndgi::kMaxT;
        ndgi::KParams p;
        fill_common(ctx, p);
        p.nt = (int)n;
        for (uint32_t i = 0; i < n; ++i) p.tc[i] = make_tconst(ctx->L, (double)ts[t0 + i]);
        p.out_t_stride = per_t;
        p.full = 1;
        p.n_req = ctx->L.num_tiles;
        p.num_slots = 0;
        p.out = static_cast<uint8_t*>(out) + (size_t)t0 * per_t * ndgi_texel_bytes(fmt);
        p.out_fmt = (int)fmt;
        ndgi_status st = launch(ctx, p, mode, stream);
        if (st != NDGI_OK) return st;
    }
    return NDGI_OK;
}

}  // namespace

namespace ndgi {
// for the other translation units of the C ABI (vt_cache.cu)
ndgi_status set_error(ndgi_status s, const char* msg) {
    g_last_error = msg;
    return s;
}
}  // namespace ndgi

extern "C" {

const char* ndgi_status_string(ndgi_status s) {
    switch (s) {
        case NDGI_OK: return "NDGI_OK";
        case NDGI_ERR_ARG: return "NDGI_ERR_ARG";
        case NDGI_ERR_RANGE: return "NDGI_ERR_RANGE";
        case NDGI_ERR_UNSUPPORTED: return "NDGI_ERR_UNSUPPORTED";
        case NDGI_ERR_CUDA: return "NDGI_ERR_CUDA";
        case NDGI_ERR_NOMEM: return "NDGI_ERR_NOMEM";
        case NDGI_ERR_DEVICE: return "NDGI_ERR_DEVICE";
    }
    return "NDGI_ERR_UNKNOWN";
}

const char* ndgi_last_error(void) { return g_last_error.c_str(); }

ndgi_status ndgi_validate_layout(const ndgi_layout* layout, int* fast_supported) {
    return validate(layout, fast_supported);
}

uint64_t ndgi_full_texels(const ndgi_layout* L) {
    return L ? (uint64_t)L->num_tiles * L->core * L->core : 0;
}

size_t ndgi_texel_bytes(ndgi_out_fmt fmt) {
    return fmt == NDGI_OUT_RGBA8 ? 4 : (fmt == NDGI_OUT_RGBA16F ? 8 : (fmt == NDGI_OUT_RGBA32F ? 16 : 0));
}

ndgi_status ndgi_load(const ndgi_layout* layout, const ndgi_params* params, int device, ndgi_ctx** out) {
    NvtxRange nvtx_("ndgi_load");
    if (!out) return fail(NDGI_ERR_ARG, "out is NULL");
    ndgi_status st = validate(layout, nullptr);
    if (st != NDGI_OK) return st;
    if (!params || !params->uv || !params->uvt || !params->ut || !params->vt || !params->mlp)
        return fail(NDGI_ERR_ARG, "params or one of its pointers is NULL");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || device < 0 || device >= ndev) return fail(NDGI_ERR_DEVICE, "no such CUDA device");
    cudaDeviceProp prop;
    e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0)
        return fail(NDGI_ERR_DEVICE, "libndgi.so is built for sm_100a (B200); device is sm_" +
                                         std::to_string(prop.major) + std::to_string(prop.minor));
    DeviceGuard g(device);
    ndgi_ctx* c = new (std::nothrow) ndgi_ctx();
    if (!c) return fail(NDGI_ERR_NOMEM, "host allocation");
    c->L = *layout;
    c->P = *params;
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    e = cudaMalloc(&c->d_err, sizeof(uint32_t));
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "cudaMalloc(error counter)");
    }
    cudaMemset(c->d_err, 0, sizeof(uint32_t));
    e = cudaMalloc(&c->d_sched, ndgi::kSchedSlots * sizeof(uint32_t));
    if (e != cudaSuccess) {
        cudaFree(c->d_err);
        delete c;
        return cuda_fail(e, "cudaMalloc(scheduling counters)");
    }
    cudaMemset(c->d_sched, 0, ndgi::kSchedSlots * sizeof(uint32_t));
    int fast = 0;
    validate(layout, &fast);
    if (fast) {
        // G_Phi's folded B operands, once per context
        const size_t tb = ndgi::wpack_tile_bytes((int)layout->hidden);
        e = cudaMalloc(&c->wpack, tb * layout->num_tiles);
        if (e != cudaSuccess) {
            cudaFree(c->d_err);
            cudaFree(c->d_sched);
            delete c;
            return cuda_fail(e, "cudaMalloc(prepacked weights)");
        }
        e = ndgi::prep_weights(params->mlp, mlp_elems(layout->hidden), (int)layout->hidden, (int)layout->fmt_uv,
                               c->wpack, (int)layout->num_tiles, 0);
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaFree(c->d_err);
        cudaFree(c->d_sched);
        if (c->wpack) cudaFree(c->wpack);
        delete c;
        return cuda_fail(e, "ndgi_load prepack / sync");
    }
    *out = c;
    return NDGI_OK;
}

ndgi_status ndgi_decode_tiles(ndgi_ctx* ctx, const uint32_t* tile_ids, const uint32_t* slots, uint32_t n,
                              uint32_t num_slots, float t, void* out_cache, ndgi_out_fmt fmt, ndgi_mode mode,
                              void* stream) {
    NvtxRange nvtx_("ndgi_decode_tiles");
    if (!ctx || !tile_ids || !out_cache) return fail(NDGI_ERR_ARG, "NULL ctx, tile_ids or out_cache");
    if (!out_ok(fmt) || !mode_ok(mode)) return fail(NDGI_ERR_ARG, "bad fmt or mode");
    if (n == 0) return fail(NDGI_ERR_ARG, "n == 0");
    if (n > (1u << 24)) return fail(NDGI_ERR_RANGE, "n > 2^24");
    if (num_slots == 0) return fail(NDGI_ERR_ARG, "num_slots == 0");
    ndgi_status st = check_t(t);
    if (st != NDGI_OK) return st;
    DeviceGuard g(ctx->device);
    ndgi::KParams p;
    fill_common(ctx, p);
    p.nt = 1;
    p.tc[0] = make_tconst(ctx->L, (double)t);
    p.full = 0;
    p.tile_ids = tile_ids;
    p.slots = slots;
    p.n_req = n;
    p.num_slots = num_slots;
    p.out = out_cache;
    p.out_fmt = (int)fmt;
    return launch(ctx, p, mode, static_cast<cudaStream_t>(stream));
}

ndgi_status ndgi_decode_full(ndgi_ctx* ctx, float t, void* out, ndgi_out_fmt fmt, ndgi_mode mode, void* stream) {
    NvtxRange nvtx_("ndgi_decode_full");
    if (!ctx || !out) return fail(NDGI_ERR_ARG, "NULL ctx or out");
    if (!out_ok(fmt) || !mode_ok(mode)) return fail(NDGI_ERR_ARG, "bad fmt or mode");
    ndgi_status st = check_t(t);
    if (st != NDGI_OK) return st;
    DeviceGuard g(ctx->device);
    return decode_full_async(ctx, &t, 1, out, fmt, mode, static_cast<cudaStream_t>(stream));
}

ndgi_status ndgi_decode_full_batch(ndgi_ctx* ctx, const float* t, uint32_t n_t, void* out, ndgi_out_fmt fmt,
                                   ndgi_mode mode, void* stream) {
    NvtxRange nvtx_("ndgi_decode_full_batch");
    if (!ctx || !out || !t) return fail(NDGI_ERR_ARG, "NULL ctx, t or out");
    if (!out_ok(fmt) || !mode_ok(mode)) return fail(NDGI_ERR_ARG, "bad fmt or mode");
    if (n_t == 0) return fail(NDGI_ERR_ARG, "n_t == 0");
    for (uint32_t i = 0; i < n_t; ++i) {
        ndgi_status st = check_t(t[i]);
        if (st != NDGI_OK) return st;
    }
    DeviceGuard g(ctx->device);
    return decode_full_async(ctx, t, n_t, out, fmt, mode, static_cast<cudaStream_t>(stream));
}

ndgi_status ndgi_decode_full_host(ndgi_ctx* ctx, const float* t, uint32_t n_t, void* out_host, ndgi_out_fmt fmt,
                                  ndgi_mode mode) {
    NvtxRange nvtx_("ndgi_decode_full_host");
    if (!ctx || !out_host || !t) return fail(NDGI_ERR_ARG, "NULL ctx, t or out_host");
    if (!out_ok(fmt) || !mode_ok(mode)) return fail(NDGI_ERR_ARG, "bad fmt or mode");
    if (n_t == 0) return fail(NDGI_ERR_ARG, "n_t == 0");
    for (uint32_t i = 0; i < n_t; ++i) {
        ndgi_status st = check_t(t[i]);
        if (st != NDGI_OK) return st;
    }
    DeviceGuard g(ctx->device);
    std::lock_guard<std::mutex> lock(ctx->host_mu);
    const size_t bytes = ndgi_full_texels(&ctx->L) * ndgi_texel_bytes(fmt);
    cudaError_t e;
    if (ctx->stage_bytes < bytes) {
        for (int i = 0; i < 2; ++i) {
            if (ctx->stage[i]) cudaFree(ctx->stage[i]);
            ctx->stage[i] = nullptr;
        }
        ctx->stage_bytes = 0;
        for (int i = 0; i < 2; ++i) {
            e = cudaMalloc(&ctx->stage[i], bytes);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(staging)");
            if (!ctx->hstream[i]) {
                cudaStreamCreateWithFlags(&ctx->hstream[i], cudaStreamNonBlocking);
                cudaEventCreateWithFlags(&ctx->hevent[i], cudaEventDisableTiming);
            }
        }
        ctx->stage_bytes = bytes;
    }
    // time i decodes into stage[i%2] on stream i%2 and is copied out on the same
    // stream, so decode of i+1 overlaps the copy of i
    for (uint32_t i = 0; i < n_t; ++i) {
        const int b = (int)(i & 1u);
        ndgi_status st = decode_full_async(ctx, t + i, 1, ctx->stage[b], fmt, mode, ctx->hstream[b]);
        if (st != NDGI_OK) return st;
        e = cudaMemcpyAsync(static_cast<uint8_t*>(out_host) + (size_t)i * bytes, ctx->stage[b], bytes,
                            cudaMemcpyDeviceToHost, ctx->hstream[b]);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(D2H)");
    }
    for (int b = 0; b < 2; ++b) {
        e = cudaStreamSynchronize(ctx->hstream[b]);
        if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    }
    return NDGI_OK;
}

ndgi_status ndgi_device_error(ndgi_ctx* ctx, uint32_t* bad_requests, int reset) {
    if (!ctx || !bad_requests) return fail(NDGI_ERR_ARG, "NULL ctx or bad_requests");
    DeviceGuard g(ctx->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceSynchronize");
    e = cudaMemcpy(bad_requests, ctx->d_err, sizeof(uint32_t), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(error counter)");
    if (reset) cudaMemset(ctx->d_err, 0, sizeof(uint32_t));
    return NDGI_OK;
}

ndgi_status ndgi_sample_lighting(ndgi_ctx* ctx, const int32_t* page_table, int32_t bucket, const void* cache,
                                 uint32_t num_slots, const float* uv, const uint32_t* atlas, uint32_t n, float t,
                                 const ndgi_hdr* hdr, float* out_rgb, void* stream) {
    NvtxRange nvtx_("ndgi_sample_lighting");
    if (!ctx || !page_table || !cache || !uv || !out_rgb || !hdr || !hdr->frame_times || !hdr->means)
        return fail(NDGI_ERR_ARG, "NULL argument");
    if (num_slots == 0) return fail(NDGI_ERR_ARG, "num_slots == 0");
    if (!std::isfinite(hdr->gamma) || hdr->gamma <= 0.0f) return fail(NDGI_ERR_ARG, "gamma must be finite and > 0");
    if (hdr->n_frames == 0) return fail(NDGI_ERR_ARG, "n_frames == 0");
    const ndgi_layout& L = ctx->L;
    if (L.atlases > (uint32_t)ndgi::kMaxSampleAtlases) return fail(NDGI_ERR_UNSUPPORTED, "more than 64 atlases");
    if (L.border < 1) return fail(NDGI_ERR_UNSUPPORTED, "sampling needs a tile border >= 1 (P:526)");
    const float* tm = hdr->frame_times;
    for (uint32_t i = 0; i < hdr->n_frames; ++i) {
        if (!std::isfinite(tm[i]) || (i && !(tm[i] > tm[i - 1])))
            return fail(NDGI_ERR_ARG, "frame_times must be finite and increasing");
    }
    if (!std::isfinite(t) || t < tm[0] || t > tm[hdr->n_frames - 1])
        return fail(NDGI_ERR_RANGE, "t outside [frame_times[0], frame_times[n_frames-1]] (R22)");
    if (n == 0) return NDGI_OK;
    // R22: per-atlas, per-channel mean at t, linear between the bracketing bake times (fp64)
    uint32_t i0 = 0;
    while (hdr->n_frames > 1 && i0 < hdr->n_frames - 2 && t > tm[i0 + 1]) ++i0;
    const double lam = hdr->n_frames > 1 ? ((double)t - tm[i0]) / ((double)tm[i0 + 1] - tm[i0]) : 0.0;
    const uint32_t i1 = hdr->n_frames > 1 ? i0 + 1 : i0;
    std::vector<float> mu((size_t)L.atlases * 3);
    for (uint32_t a = 0; a < L.atlases; ++a)
        for (int c = 0; c < 3; ++c) {
            const double m0 = hdr->means[((size_t)a * hdr->n_frames + i0) * 3 + c];
            const double m1 = hdr->means[((size_t)a * hdr->n_frames + i1) * 3 + c];
            if (!std::isfinite(m0) || !std::isfinite(m1)) return fail(NDGI_ERR_ARG, "means must be finite");
            mu[(size_t)a * 3 + c] = (float)((1.0 - lam) * m0 + lam * m1);
        }
    DeviceGuard g(ctx->device);
    ndgi::SampleArgs A;
    A.pt = page_table;
    A.cache = static_cast<const uint8_t*>(cache);
    A.uv = uv;
    A.atlas = atlas;
    A.out = out_rgb;
    A.err = ctx->d_err;
    A.n = n;
    A.num_slots = num_slots;
    A.bucket = bucket;
    A.C = (int)L.core;
    A.B = (int)L.border;
    A.tiles_x = (int)L.tiles_x;
    A.tiles_y = (int)L.tiles_y;
    A.atlases = (int)L.atlases;
    A.num_sms = ctx->num_sms;
    A.g = hdr->gamma;
    A.mu = mu.data();
    const cudaError_t e = ndgi::launch_sample(A, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "sample launch");
    return NDGI_OK;
}

ndgi_status ndgi_bc7_encode_mode6(const void* rgba, uint32_t w, uint32_t h, void* blocks, void* stream) {
    NvtxRange nvtx_("ndgi_bc7_encode_mode6");
    if (!rgba || !blocks) return fail(NDGI_ERR_ARG, "NULL rgba or blocks");
    if (w == 0 || h == 0 || w % 4 || h % 4) return fail(NDGI_ERR_ARG, "w and h must be positive multiples of 4");
    if (w > (1u << 16) || h > (1u << 16)) return fail(NDGI_ERR_RANGE, "w or h > 65536");
    int dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(e, "device query");
    e = ndgi::launch_bc7_encode_mode6(rgba, (int)w, (int)h, blocks, sms, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? NDGI_OK : cuda_fail(e, "bc7 encode launch");
}

ndgi_status ndgi_bc7_encode_multi(const void* rgba, uint32_t w, uint32_t h, void* blocks, void* stream) {
    NvtxRange nvtx_("ndgi_bc7_encode_multi");
    if (!rgba || !blocks) return fail(NDGI_ERR_ARG, "NULL rgba or blocks");
    if (w == 0 || h == 0 || w % 4 || h % 4) return fail(NDGI_ERR_ARG, "w and h must be positive multiples of 4");
    if (w > (1u << 16) || h > (1u << 16)) return fail(NDGI_ERR_RANGE, "w or h > 65536");
    int dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(e, "device query");
    e = ndgi::launch_bc7_encode_multi(rgba, (int)w, (int)h, blocks, sms, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? NDGI_OK : cuda_fail(e, "bc7 encode launch");
}

// ---- training ----------------------------------------------
// One trainer type for both stages: fine-tuning (R27, parameters = the MLP) and
// the full step (R28, parameters = MLP + BC-simulated maps + line grids).
struct ndgi_train {
    ndgi_ctx* ctx;
    bool full;
    size_t P;                      // parameters per tile
    size_t off_uv, off_uvt, off_ut, off_vt;
    float *theta, *m, *v, *grad, *loss;
    float* dtex;                   // full: per-row texel gradients [cap][dtex_stride]
    size_t dtex_stride;
    int* steps;
    uint32_t cap;                  // batch capacity of grad / loss / dtex
    uint32_t last_n;               // batch of the last step (ndgi_train_last_grad)
    // fine-tuning: the frozen BC7 feature maps decoded once (bit-exact) into
    // owned u8 copies, [tile][R][R][4] and [tile][D][R3][R3][4], so a step's
    // taps are plain loads instead of a BC7 block decode each (same values:
    // both paths dequantise q / 255, R8); nullptr for other formats
    uint8_t *uv8, *uvt8;
};

namespace {

size_t full_params(const ndgi_layout& L, size_t* off) {
    const size_t mlp = mlp_elems(L.hidden);
    const size_t uv = mlp, uvt = uv + (size_t)(L.uv_res / 4) * (L.uv_res / 4) * 24;
    const size_t ut = uvt + (size_t)L.uvt_depth * (L.uvt_res / 4) * (L.uvt_res / 4) * 24;
    const size_t vt = ut + (size_t)L.line_t * L.line_res * 2;
    const size_t total = vt + (size_t)L.line_t * L.line_res * 2;
    if (off) {
        off[0] = uv;
        off[1] = uvt;
        off[2] = ut;
        off[3] = vt;
    }
    return total;
}

ndgi_status train_create(ndgi_ctx* ctx, bool full, const float* init, ndgi_train** out) {
    if (!ctx || !out || (full && !init)) return fail(NDGI_ERR_ARG, "NULL ctx, out or init");
    if (ctx->L.hidden != 16) return fail(NDGI_ERR_UNSUPPORTED, "training is built for h = 16");
    if (full && (ctx->L.uv_res % 4 || ctx->L.uvt_res % 4))
        return fail(NDGI_ERR_UNSUPPORTED, "BC-simulated maps need resolutions that are multiples of 4");
    DeviceGuard g(ctx->device);
    ndgi_train* t = new (std::nothrow) ndgi_train();
    if (!t) return fail(NDGI_ERR_NOMEM, "host allocation");
    t->ctx = ctx;
    t->full = full;
    size_t off[4] = {0, 0, 0, 0};
    t->P = full ? full_params(ctx->L, off) : mlp_elems(ctx->L.hidden);
    t->off_uv = off[0];
    t->off_uvt = off[1];
    t->off_ut = off[2];
    t->off_vt = off[3];
    t->dtex_stride = full ? (size_t)ctx->L.uv_res * ctx->L.uv_res * 4 +
                                (size_t)ctx->L.uvt_depth * ctx->L.uvt_res * ctx->L.uvt_res * 4 +
                                (size_t)ctx->L.line_t * ctx->L.line_res * 4
                          : 0;
    t->dtex_stride = (t->dtex_stride + 3) & ~(size_t)3;
    const size_t n = (size_t)ctx->L.num_tiles * t->P;
    cudaError_t e = cudaMalloc(&t->theta, n * 4);
    if (e == cudaSuccess) e = cudaMalloc(&t->m, n * 4);
    if (e == cudaSuccess) e = cudaMalloc(&t->v, n * 4);
    if (e == cudaSuccess) e = cudaMalloc(&t->steps, (size_t)ctx->L.num_tiles * sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(t->m, 0, n * 4);
    if (e == cudaSuccess) e = cudaMemset(t->v, 0, n * 4);
    if (e == cudaSuccess) e = cudaMemset(t->steps, 0, (size_t)ctx->L.num_tiles * sizeof(int));
    if (e == cudaSuccess) {
        if (full) e = cudaMemcpy(t->theta, init, n * 4, cudaMemcpyDeviceToDevice);
        else e = ndgi::launch_convert_f16_f32(ctx->P.mlp, t->theta, n, 0);   // fp32 master copy
    }
    const ndgi_layout& L = ctx->L;
    if (e == cudaSuccess && !full && L.fmt_uv == NDGI_FMT_BC7) {
        // tile-major blocks = one image of R_uv x (R_uv * tiles) in block row-major order
        e = cudaMalloc(&t->uv8, (size_t)L.num_tiles * L.uv_res * L.uv_res * 4);
        if (e == cudaSuccess) e = ndgi::launch_bc7_map(ctx->P.uv, L.uv_res, L.uv_res * L.num_tiles, t->uv8, 0);
    }
    if (e == cudaSuccess && !full && L.fmt_uvt == NDGI_FMT_BC7) {
        e = cudaMalloc(&t->uvt8, (size_t)L.num_tiles * L.uvt_depth * L.uvt_res * L.uvt_res * 4);
        if (e == cudaSuccess)
            e = ndgi::launch_bc7_map(ctx->P.uvt, L.uvt_res, L.uvt_res * L.uvt_depth * L.num_tiles, t->uvt8, 0);
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaFree(t->theta);
        cudaFree(t->m);
        cudaFree(t->v);
        cudaFree(t->steps);
        cudaFree(t->uv8);
        cudaFree(t->uvt8);
        delete t;
        return cuda_fail(e, "training state allocation");
    }
    *out = t;
    return NDGI_OK;
}

ndgi_status train_step(ndgi_train* t, const uint32_t* tile_ids, uint32_t n, const float* samples, const float* targets,
                       const float* noise, uint32_t S, float lr, float* loss, void* stream) {
    if (!t || !tile_ids || !samples || !targets || (t->full && !noise)) return fail(NDGI_ERR_ARG, "NULL argument");
    if (n == 0 || S == 0) return fail(NDGI_ERR_ARG, "n == 0 or S == 0");
    if (n > (1u << 20) || S > (1u << 24)) return fail(NDGI_ERR_RANGE, "n > 2^20 or S > 2^24");
    if (!std::isfinite(lr) || lr < 0.0f) return fail(NDGI_ERR_ARG, "lr must be finite and >= 0");
    ndgi_ctx* ctx = t->ctx;
    DeviceGuard g(ctx->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaSuccess;
    if (n > t->cap) {
        cudaFree(t->grad);
        cudaFree(t->loss);
        cudaFree(t->dtex);
        t->grad = nullptr;
        t->loss = nullptr;
        t->dtex = nullptr;
        t->cap = 0;
        e = cudaMalloc(&t->grad, (size_t)n * t->P * 4);
        if (e == cudaSuccess) e = cudaMalloc(&t->loss, (size_t)n * 4);
        if (e == cudaSuccess && t->full) e = cudaMalloc(&t->dtex, (size_t)n * t->dtex_stride * 4);
        if (e != cudaSuccess) return cuda_fail(e, "train scratch");
        t->cap = n;
    }
    if (t->full) {   // the MLP part takes atomics; ndgi_bc_grad_kernel writes the rest
        const size_t pm = mlp_elems(ctx->L.hidden);
        e = cudaMemset2DAsync(t->grad, t->P * 4, 0, pm * 4, n, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(t->dtex, 0, (size_t)n * t->dtex_stride * 4, s);
    } else {
        e = cudaMemsetAsync(t->grad, 0, (size_t)n * t->P * 4, s);
    }
    if (e == cudaSuccess) e = cudaMemsetAsync(t->loss, 0, (size_t)n * 4, s);
    if (e != cudaSuccess) return cuda_fail(e, "train scratch clear");
    const ndgi_layout& L = ctx->L;
    ndgi::TrainArgs a{};
    a.uv = static_cast<const uint8_t*>(ctx->P.uv);
    a.uvt = static_cast<const uint8_t*>(ctx->P.uvt);
    a.ut = static_cast<const uint8_t*>(ctx->P.ut);
    a.vt = static_cast<const uint8_t*>(ctx->P.vt);
    a.uv_tile_bytes = map2d_bytes(L.fmt_uv, L.uv_res, L.uv_res, 4);
    a.uvt_slice_bytes = map2d_bytes(L.fmt_uvt, L.uvt_res, L.uvt_res, 4);
    a.uvt_tile_bytes = a.uvt_slice_bytes * L.uvt_depth;
    a.line_tile_bytes = map2d_bytes(L.fmt_line, L.line_res, L.line_t, 2);
    a.fmt_uv = (int)L.fmt_uv;
    a.fmt_uvt = (int)L.fmt_uvt;
    if (t->uv8) {   // the decoded copies (train_create)
        a.uv = t->uv8;
        a.fmt_uv = NDGI_FMT_U8;
        a.uv_tile_bytes = (size_t)L.uv_res * L.uv_res * 4;
    }
    if (t->uvt8) {
        a.uvt = t->uvt8;
        a.fmt_uvt = NDGI_FMT_U8;
        a.uvt_slice_bytes = (size_t)L.uvt_res * L.uvt_res * 4;
        a.uvt_tile_bytes = a.uvt_slice_bytes * L.uvt_depth;
    }
    a.fmt_line = (int)L.fmt_line;
    a.R_uv = (int)L.uv_res;
    a.R3 = (int)L.uvt_res;
    a.D = (int)L.uvt_depth;
    a.U = (int)L.line_res;
    a.T = (int)L.line_t;
    a.gelu = (int)L.gelu;
    a.num_tiles = (int)L.num_tiles;
    a.tile_ids = tile_ids;
    a.samples = samples;
    a.targets = targets;
    a.n = (int)n;
    a.S = (int)S;
    // enough CTAs for two waves at 128 threads, >= 128 samples per CTA
    const uint32_t want = (2u * (uint32_t)ctx->num_sms * 8u + n - 1) / n;
    const uint32_t maxc = S / 128 > 0 ? S / 128 : 1;
    a.chunks = (int)(want < 1 ? 1 : (want > maxc ? maxc : want));
    a.theta = t->theta;
    a.grad = t->grad;
    a.loss = t->loss;
    a.err = ctx->d_err;
    a.noise = t->full ? noise : nullptr;
    a.pfull = t->P;
    a.off_uv = t->off_uv;
    a.off_uvt = t->off_uvt;
    a.off_ut = t->off_ut;
    a.off_vt = t->off_vt;
    a.dtex = t->dtex;
    a.dtex_stride = t->dtex_stride;
    t->last_n = n;
    e = ndgi::launch_train_grad(a, (int)L.hidden, s);
    if (e == cudaSuccess)
        e = ndgi::launch_adam(t->theta, t->m, t->v, t->steps, t->grad, tile_ids, (int)n, t->P, (int)L.num_tiles, lr,
                              0.9f, 0.999f, 1e-8f, t->full ? t->off_uv : t->P, s);
    if (e == cudaSuccess && loss) e = cudaMemcpyAsync(loss, t->loss, (size_t)n * 4, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "train step");
    return NDGI_OK;
}

}  // namespace

ndgi_status ndgi_train_create(ndgi_ctx* ctx, ndgi_train** out) { return train_create(ctx, false, nullptr, out); }

ndgi_status ndgi_train_full_create(ndgi_ctx* ctx, const float* init, ndgi_train** out) {
    return train_create(ctx, true, init, out);
}

size_t ndgi_train_full_params(const ndgi_layout* layout) { return layout ? full_params(*layout, nullptr) : 0; }

ndgi_status ndgi_train_step(ndgi_train* t, const uint32_t* tile_ids, uint32_t n, const float* samples,
                            const float* targets, uint32_t S, float lr, float* loss, void* stream) {
    NvtxRange nvtx_("ndgi_train_step");
    if (t && t->full) return fail(NDGI_ERR_ARG, "a full trainer steps with ndgi_train_full_step");
    return train_step(t, tile_ids, n, samples, targets, nullptr, S, lr, loss, stream);
}

ndgi_status ndgi_train_full_step(ndgi_train* t, const uint32_t* tile_ids, uint32_t n, const float* samples,
                                 const float* targets, const float* noise, uint32_t S, float lr, float* loss,
                                 void* stream) {
    NvtxRange nvtx_("ndgi_train_full_step");
    if (t && !t->full) return fail(NDGI_ERR_ARG, "a fine-tuning trainer steps with ndgi_train_step");
    return train_step(t, tile_ids, n, samples, targets, noise, S, lr, loss, stream);
}

ndgi_status ndgi_train_last_grad(ndgi_train* t, float* out, uint32_t n, void* stream) {
    if (!t || !out) return fail(NDGI_ERR_ARG, "NULL argument");
    if (n == 0 || n > t->last_n) return fail(NDGI_ERR_RANGE, "n must be in [1, the last step's batch]");
    DeviceGuard g(t->ctx->device);
    const cudaError_t e = cudaMemcpyAsync(out, t->grad, (size_t)n * t->P * 4, cudaMemcpyDeviceToDevice,
                                          static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? NDGI_OK : cuda_fail(e, "train grad copy");
}

ndgi_status ndgi_train_weights(ndgi_train* t, float* out, void* stream) {
    if (!t || !out) return fail(NDGI_ERR_ARG, "NULL argument");
    DeviceGuard g(t->ctx->device);
    const cudaError_t e = cudaMemcpyAsync(out, t->theta, (size_t)t->ctx->L.num_tiles * t->P * 4,
                                          cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? NDGI_OK : cuda_fail(e, "train weights copy");
}

ndgi_status ndgi_train_export_f16(ndgi_train* t, uint16_t* mlp, void* stream) {
    if (!t || !mlp) return fail(NDGI_ERR_ARG, "NULL argument");
    DeviceGuard g(t->ctx->device);
    const size_t pm = mlp_elems(t->ctx->L.hidden);
    cudaError_t e = cudaSuccess;
    if (!t->full) {
        e = ndgi::launch_convert_f32_f16(t->theta, mlp, (size_t)t->ctx->L.num_tiles * pm, static_cast<cudaStream_t>(stream));
    } else {
        e = ndgi::launch_convert_f32_f16_2d(t->theta, t->P, mlp, pm, t->ctx->L.num_tiles, pm,   // the MLP part
                                            static_cast<cudaStream_t>(stream));
    }
    return e == cudaSuccess ? NDGI_OK : cuda_fail(e, "train export");
}

ndgi_status ndgi_train_full_export(ndgi_train* t, void* uv, void* uvt, void* ut, void* vt, uint16_t* mlp,
                                   void* stream) {
    NvtxRange nvtx_("ndgi_train_full_export");
    if (!t || !uv || !uvt || !ut || !vt || !mlp) return fail(NDGI_ERR_ARG, "NULL argument");
    if (!t->full) return fail(NDGI_ERR_ARG, "export needs a full trainer");
    ndgi_ctx* ctx = t->ctx;
    const ndgi_layout& L = ctx->L;
    DeviceGuard g(ctx->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t n_uv = (size_t)L.num_tiles * L.uv_res * L.uv_res * 4,
                 n_uvt = (size_t)L.num_tiles * L.uvt_depth * L.uvt_res * L.uvt_res * 4;
    uint8_t* img = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&img), n_uv + n_uvt, s);
    if (e != cudaSuccess) return cuda_fail(e, "export scratch");
    e = ndgi::launch_full_ptq(t->theta, t->P, t->off_uv, t->off_uvt, t->off_ut, t->off_vt, (int)L.num_tiles,
                              (int)L.uv_res, (int)L.uvt_res, (int)L.uvt_depth, (int)(L.line_t * L.line_res * 2),
                              reinterpret_cast<uint32_t*>(img), reinterpret_cast<uint32_t*>(img + n_uv),
                              static_cast<uint8_t*>(ut), static_cast<uint8_t*>(vt), ctx->num_sms, s);
    if (e == cudaSuccess)   // the tile-major image stack encodes straight into [tile][by][bx] blocks
        e = ndgi::launch_bc7_encode_mode6(img, (int)L.uv_res, (int)(L.num_tiles * L.uv_res), uv, ctx->num_sms, s);
    if (e == cudaSuccess)
        e = ndgi::launch_bc7_encode_mode6(img + n_uv, (int)L.uvt_res, (int)(L.num_tiles * L.uvt_depth * L.uvt_res), uvt,
                                          ctx->num_sms, s);
    cudaFreeAsync(img, s);
    if (e != cudaSuccess) return cuda_fail(e, "export");
    return ndgi_train_export_f16(t, mlp, stream);
}

ndgi_status ndgi_train_free(ndgi_train* t) {
    if (!t) return fail(NDGI_ERR_ARG, "NULL argument");
    DeviceGuard g(t->ctx->device);
    cudaDeviceSynchronize();
    cudaFree(t->theta);
    cudaFree(t->m);
    cudaFree(t->v);
    cudaFree(t->steps);
    cudaFree(t->grad);
    cudaFree(t->loss);
    cudaFree(t->dtex);
    cudaFree(t->uv8);
    cudaFree(t->uvt8);
    delete t;
    return NDGI_OK;
}

ndgi_status ndgi_free(ndgi_ctx* ctx) {
    if (!ctx) return fail(NDGI_ERR_ARG, "NULL ctx");
    DeviceGuard g(ctx->device);
    cudaDeviceSynchronize();
    cudaFree(ctx->d_err);
    cudaFree(ctx->d_sched);
    if (ctx->wpack) cudaFree(ctx->wpack);
    if (ctx->tex_ready) ndgi::uv_textures_free((int)ctx->L.atlases, ctx->uvarr, ctx->uvtex);
    for (int i = 0; i < 2; ++i) {
        if (ctx->stage[i]) cudaFree(ctx->stage[i]);
        if (ctx->hstream[i]) cudaStreamDestroy(ctx->hstream[i]);
        if (ctx->hevent[i]) cudaEventDestroy(ctx->hevent[i]);
    }
    delete ctx;
    return NDGI_OK;
}

ndgi_status ndgi_debug_bc7_decode(const void* blocks, uint32_t w, uint32_t h, uint8_t* rgba, void* stream) {
    if (!blocks || !rgba || w % 4 || h % 4 || !w || !h) return fail(NDGI_ERR_ARG, "bad arguments");
    cudaError_t e = ndgi::launch_bc7_map(blocks, w, h, rgba, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? NDGI_OK : cuda_fail(e, "bc7 map decode");
}

ndgi_status ndgi_debug_bc7_decode_hw(const void* blocks, uint32_t w, uint32_t h, uint8_t* rgba) {
    if (!blocks || !rgba || w % 4 || h % 4 || !w || !h) return fail(NDGI_ERR_ARG, "bad arguments");
    cudaError_t e = ndgi::bc7_decode_hw(blocks, w, h, rgba);
    return e == cudaSuccess ? NDGI_OK : cuda_fail(e, "bc7 texture decode");
}

ndgi_status ndgi_debug_gelu_rate(uint32_t iters, uint32_t mufu_pairs, int pack_f32, float* ms, double* activations) {
    if (!ms || !activations || !iters) return fail(NDGI_ERR_ARG, "bad arguments");
    if (mufu_pairs > 16) return fail(NDGI_ERR_RANGE, "mufu_pairs must be in [0, 16]");
    cudaError_t e = ndgi::gelu_rate(iters, mufu_pairs, pack_f32, ms, activations);
    return e == cudaSuccess ? NDGI_OK : cuda_fail(e, "gelu rate");
}

ndgi_status ndgi_debug_gelu_split(uint32_t hidden, uint32_t* mufu_pairs_of_16, int* fp32_acc) {
    if (!mufu_pairs_of_16 || !fp32_acc) return fail(NDGI_ERR_ARG, "bad arguments");
    if (hidden != 16 && hidden != 64) return fail(NDGI_ERR_UNSUPPORTED, "the fused kernel is built for h = 16 / 64");
    *mufu_pairs_of_16 = (uint32_t)ndgi::fused_gelu_mufu_pairs((int)hidden);
    *fp32_acc = hidden == 64 ? 1 : !ndgi::fused_f16acc();
    return NDGI_OK;
}

ndgi_status ndgi_debug_null_launch(void* stream) {
    const cudaError_t e = ndgi::null_launch(static_cast<cudaStream_t>(stream), 0);
    return e == cudaSuccess ? NDGI_OK : cuda_fail(e, "null launch");
}

ndgi_status ndgi_debug_launch_probe(int kind, void* stream) {
    if (kind < 0 || kind > 3) return fail(NDGI_ERR_ARG, "kind must be 0..3");
    const cudaError_t e = ndgi::null_launch(static_cast<cudaStream_t>(stream), kind);
    return e == cudaSuccess ? NDGI_OK : cuda_fail(e, "null launch");
}

ndgi_status ndgi_debug_mma_latency(uint32_t iters, double* cycles_per_iter) {
    if (!cycles_per_iter || !iters) return fail(NDGI_ERR_ARG, "bad arguments");
    cudaError_t e = ndgi::mma_latency(iters, cycles_per_iter);
    return e == cudaSuccess ? NDGI_OK : cuda_fail(e, "mma latency");
}

ndgi_status ndgi_debug_f16d_probe(uint32_t seed, uint32_t iters, uint32_t ctas, uint64_t* mismatches,
                                  uint64_t* pairs) {
    if (!mismatches || !pairs || !iters || !ctas) return fail(NDGI_ERR_ARG, "bad arguments");
    unsigned long long m = 0, t = 0;
    cudaError_t e = ndgi::f16d_probe(seed, iters, ctas, &m, &t);
    *mismatches = m;
    *pairs = t;
    return e == cudaSuccess ? NDGI_OK : cuda_fail(e, "f16-D probe");
}

ndgi_status ndgi_debug_tmem_f16_probe(uint32_t* host_out) {
    if (!host_out) return fail(NDGI_ERR_ARG, "bad arguments");
    cudaError_t e = ndgi::tmem_f16_probe(host_out);
    return e == cudaSuccess ? NDGI_OK : cuda_fail(e, "tmem f16 probe");
}

}  // extern "C"
