/*
 * ndgi.h -- C ABI of the B200-native NDGI tile decoder (libndgi.so).
 *
 * Operation (Neural Dynamic GI, arXiv 2604.12625; "P:n" = PAPER.md line n):
 *   I(u, v, t) = H_Theta(u, v, t)                                  Eq. 3
 *   I(u, v, t) = G_Phi(V_uvt, V_uv, V_ut, V_vt, gamma(t)),
 *   gamma(t)   = [sin(pi t), cos(pi t), sin(2 pi t), cos(2 pi t)]  Eq. 4
 *   Theta = {F3D_uvt, F2D_uv, F2D_ut, F2D_vt, Phi}, one per tile   Eq. 5
 * F_uv and every t-slice of F_uvt are BC7; F_ut/F_vt are 8-bit;
 * G_Phi is 16 -> h -> h -> 3 with GELU on the hidden layers (Table 3).
 * The decoded tiles are written into a virtual-texturing page cache as
 * 8-bit RGBA with a mirrored border.
 * Every reading the paper leaves open (R1..R20) is listed in DESIGN.md.
 *
 * Conventions
 * -----------
 * - Every call returns an ndgi_status; nothing aborts or throws.
 * - Pointers documented "device" are CUDA device pointers on the context's
 *   device; "host" pointers are CPU memory.  Input buffers are BORROWED: the
 *   caller keeps them alive (and unchanged) for the context's lifetime.
 * - Decode calls are stream-ordered and asynchronous on the given
 *   cudaStream_t (passed as void*; NULL = legacy default stream) unless
 *   documented otherwise.  They never synchronise.
 * - Outputs are bit-deterministic for identical inputs (no atomics on data).
 * - Host-detectable argument errors are reported synchronously; a tile id
 *   >= num_tiles or a slot >= num_slots is detected on the device: that
 *   request is skipped and the context's error counter is incremented
 *   (read it with ndgi_device_error).
 * - Thread safety: one context may be used from several host threads on
 *   different streams; the context is read-only after ndgi_load except for
 *   its device error counter and its work-scheduling counters: a FAST decode
 *   launch with more work units than resident CTAs takes the next of 1,024
 *   per-context counters (zeroed by a cudaMemsetAsync on the call's stream
 *   before the kernel; the CTAs claim units from it with atomics -- the
 *   claimed order never changes the output).  More than 1,024 such launches
 *   in flight at once on different streams of one context, or concurrent
 *   replays of one captured CUDA graph, would share a counter: unsupported.
 */
#ifndef NDGI_H
#define NDGI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NDGI_ABI_VERSION 1u

#if defined(__GNUC__)
#define NDGI_API __attribute__((visibility("default")))
#else
#define NDGI_API
#endif

typedef struct ndgi_ctx ndgi_ctx; /* opaque; one per device */

typedef enum {
    NDGI_OK = 0,
    NDGI_ERR_ARG = 1,         /* null pointer, malformed layout, bad enum       */
    NDGI_ERR_RANGE = 2,       /* t not finite or outside [0,1]; n too large     */
    NDGI_ERR_UNSUPPORTED = 3, /* valid layout the chosen mode does not support  */
    NDGI_ERR_CUDA = 4,        /* CUDA runtime error; see ndgi_last_error        */
    NDGI_ERR_NOMEM = 5,       /* device or host allocation failed               */
    NDGI_ERR_DEVICE = 6       /* device is not an sm_100 part / not present     */
} ndgi_status;

/* storage format of a feature map (reading R8) */
typedef enum {
    NDGI_FMT_BC7 = 0, /* 16-byte BC7 blocks, UNORM, value = q/255            */
    NDGI_FMT_U8 = 1,  /* raw 8-bit texels, value = q/255                     */
    NDGI_FMT_F16 = 2, /* IEEE binary16 texels, value as stored               */
    /* The other DXTC formats ("BC1 through BC7 ... BC5 for normal maps";
     * SURVEY.md §8(f) NEXT 2, config 5's BC-format axis; reading R29).
     * Blocks row-major, texel i = 4*row + col, little-endian fields, UNORM
     * value = q/255; interpolated palette entries use integer division.   */
    NDGI_FMT_BC1 = 3, /* 8-byte blocks, 4-channel maps (F_uv, F_uvt): c0, c1
                         RGB565, 2-bit indices; c0 > c1: 4 colours, else 3 +
                         transparent black; A = 255 / 0 (4 bpp)            */
    NDGI_FMT_BC3 = 4, /* 16-byte blocks, 4-channel maps: BC4 block for A, then
                         a BC1 colour block decoded with 4 colours (8 bpp)  */
    NDGI_FMT_BC5 = 5  /* 16-byte blocks, 2-channel line maps (F_ut, F_vt):
                         BC4 blocks for channel 0 then channel 1 (8 bpp);
                         BC4 = a0, a1, 3-bit indices, 8 or 6+{0,255} values */
} ndgi_feat_fmt;

/* page-cache texel format (reading R12) */
typedef enum {
    NDGI_OUT_RGBA8 = 0,   /* RN-even(clamp(y,0,1)*255), A = 255 (4 B/texel)  */
    NDGI_OUT_RGBA16F = 1, /* (fp16(y), 1.0)                       (8 B/texel)  */
    NDGI_OUT_RGBA32F = 2  /* (y, 1.0)                            (16 B/texel) */
} ndgi_out_fmt;

typedef enum { NDGI_GELU_ERF = 0, NDGI_GELU_TANH = 1 } ndgi_gelu;           /* R7 */
typedef enum { NDGI_BORDER_MIRROR = 0, NDGI_BORDER_EVAL_CLAMP = 1 } ndgi_border; /* R3 */

typedef enum {
    /* fused tensor-core kernel: BC7 -> smem, fp16 MMA operands (tcgen05, fp32
     * accumulation in TMEM), tanh-form GELU.  Parity bar vs the fp64 oracle:
     * max-abs <= 2e-2, mean-abs <= 2e-3 (BASELINE.json north_star).          */
    NDGI_MODE_FAST = 0,
    /* scalar fp32 reference kernel, accurate erff/tanhf GELU per layout.gelu;
     * parity bar: max-abs <= 1e-5.                                            */
    NDGI_MODE_REF_FP32 = 1,
    /* NDGI_MODE_FAST with F_uv fetched through the B200 texture unit's BC7
     * decoder -- the paper's runtime mechanism -- instead of the
     * kernel's software decoder (an in-box comparator).
     * Needs a FAST layout with fmt_uv == BC7 and <= 64 atlases (UNSUPPORTED
     * otherwise).  The first call builds one BC7 texture per atlas (a second,
     * context-owned copy of F_uv: 16 KB per C = 128 tile).  The hardware
     * decode is bit-exact, so the output equals NDGI_MODE_FAST's bit for bit. */
    NDGI_MODE_FAST_TEXUNIT = 2
} ndgi_mode;

/*
 * Layout of every tile's Theta (the "BC layout" of ndgi_load).
 * C = core, B = border, P = C + 2B (padded tile side).
 * Tile id k <-> atlas placement for decode_full:
 *   k = (a * tiles_y + ty) * tiles_x + tx,  num_tiles = atlases*tiles_y*tiles_x.
 * Constraints (NDGI_ERR_ARG otherwise): abi_version == NDGI_ABI_VERSION;
 *   num_tiles >= 1; core >= 4, core % 4 == 0; border < core;
 *   block-compressed maps need resolutions that are multiples of 4 (BC5 line
 *   maps: line_res and line_t); all resolutions >= 1; uvt_depth, line_t >= 1;
 *   1 <= hidden <= 256; fmt_uv / fmt_uvt in {BC7, U8, F16, BC1, BC3};
 *   fmt_line in {U8, F16, BC5}.
 * NDGI_MODE_FAST additionally needs (NDGI_ERR_UNSUPPORTED otherwise):
 *   core in {128, 256}, uv_res == core (R2), hidden in {16, 64}
 *   (Table 3), border_mode == MIRROR, uvt_res <= 64, line_res <= 256.
 */
typedef struct ndgi_layout {
    uint32_t abi_version;            /* = NDGI_ABI_VERSION                     */
    uint32_t num_tiles;
    uint32_t atlases, tiles_x, tiles_y;
    uint32_t core;                   /* C: core texels per tile side (128)     */
    uint32_t border;                 /* B: border texels per edge (4)          */
    uint32_t uv_res;                 /* R_uv: F_uv side (= C, R2)              */
    uint32_t uvt_res;                /* R3: F_uvt side (16/32/64, Table 3)     */
    uint32_t uvt_depth;              /* D: F_uvt slices along t (12, Table 1)  */
    uint32_t line_res;               /* U: spatial texels of F_ut/F_vt (64)    */
    uint32_t line_t;                 /* T: temporal rows of F_ut/F_vt (24)     */
    uint32_t hidden;                 /* h: MLP width (16 or 64, Table 3)       */
    uint32_t fmt_uv, fmt_uvt, fmt_line; /* ndgi_feat_fmt                       */
    uint32_t gelu;                   /* ndgi_gelu                              */
    uint32_t border_mode;            /* ndgi_border                            */
} ndgi_layout;

/*
 * Theta buffers, DEVICE pointers, dense, tile-major (tile k's data at
 * k * per_tile_bytes), borrowed for the context's lifetime:
 *   uv : BC7 [tile][R_uv/4][R_uv/4][16 B]  |  U8/F16 [tile][R_uv][R_uv][4]
 *   uvt: BC7 [tile][D][R3/4][R3/4][16 B]   |  U8/F16 [tile][D][R3][R3][4]
 *   ut, vt: [tile][T][U][2] (U8 or F16; row = time, reading R5)
 *   mlp: [tile][W1 h*16 | b1 h | W2 h*h | b2 h | W3 3*h | b3 3] binary16,
 *        PyTorch [out][in] order (R11)
 * BC7 block (bx, by) of a map is at (by * (R/4) + bx) * 16; texel (x, y) of a
 * block is texel 4*y + x of the BC7 block.  All pointers 16-byte aligned.
 */
typedef struct ndgi_params {
    const void* uv;
    const void* uvt;
    const void* ut;
    const void* vt;
    const uint16_t* mlp;
} ndgi_params;

/*
 * Creates a context on CUDA device `device` for the given layout and Theta.
 * Validates the layout (synchronously), queries the device (must be an
 * sm_100 part for decode), keeps the feature maps zero-copy (borrowed), and
 * for layouts NDGI_MODE_FAST takes derives the per-tile tensor-core weight
 * operands from `mlp` once (context-owned device memory: 2,880 B per tile
 * for h = 16, 16,128 B for h = 64; the MLP weights must therefore not change
 * after this call -- create a new context instead), then synchronises once.
 * *out is set only on NDGI_OK.  Errors: ARG (null/invalid layout), DEVICE,
 * CUDA, NOMEM.
 */
NDGI_API ndgi_status ndgi_load(const ndgi_layout* layout, const ndgi_params* params, int device, ndgi_ctx** out);

/*
 * Decodes n requested tiles at time t into the page cache.
 *   tile_ids : DEVICE u32[n], tile id per request
 *   slots    : DEVICE u32[n], destination slot per request, or NULL (slot = i)
 *   out_cache: DEVICE [num_slots][P][P][texel], texel per `fmt`; slot s holds
 *              the padded tile, core at rows/cols [B, B+C), border = mirror
 *              of the core (R3).  Written texels: n * P * P.
 * Errors (synchronous): ARG (null ctx/tile_ids/out_cache, bad enum, n == 0),
 *   RANGE (t not finite or outside [0,1]; n > 2^24), UNSUPPORTED (mode/layout),
 *   CUDA (launch failure).  Invalid ids/slots: device error counter.
 */
NDGI_API ndgi_status ndgi_decode_tiles(ndgi_ctx* ctx, const uint32_t* tile_ids, const uint32_t* slots, uint32_t n,
                              uint32_t num_slots, float t, void* out_cache, ndgi_out_fmt fmt, ndgi_mode mode,
                              void* stream);

/*
 * Decodes every tile's core at time t into atlas images:
 *   out: DEVICE [atlases][tiles_y*C][tiles_x*C][texel]; tile k's core texel
 *        (i, j) lands at row ty*C + j, column tx*C + i of atlas a.
 * Written texels: num_tiles * C * C.  Errors as ndgi_decode_tiles.
 */
NDGI_API ndgi_status ndgi_decode_full(ndgi_ctx* ctx, float t, void* out, ndgi_out_fmt fmt, ndgi_mode mode, void* stream);

/*
 * Batched ndgi_decode_full over n_t query times t[0..n_t) (HOST array of
 * floats, read during the call): out receives n_t consecutive atlas sets
 * (n_t * num_tiles * C * C texels).  One launch per 32 times, so small
 * lightmaps and many times still fill the GPU.  Errors as ndgi_decode_tiles.
 */
NDGI_API ndgi_status ndgi_decode_full_batch(ndgi_ctx* ctx, const float* t, uint32_t n_t, void* out, ndgi_out_fmt fmt,
                                   ndgi_mode mode, void* stream);

/*
 * Host-buffer variant of ndgi_decode_full for end-to-end use: decodes the
 * n_t times t[0..n_t) (HOST array) into out_host (HOST memory, ideally
 * pinned), n_t consecutive atlas images.  Device staging buffers are owned by
 * the context; decode of time i+1 overlaps the device->host copy of time i.
 * SYNCHRONOUS: returns when out_host holds every result.
 */
NDGI_API ndgi_status ndgi_decode_full_host(ndgi_ctx* ctx, const float* t, uint32_t n_t, void* out_host, ndgi_out_fmt fmt,
                                  ndgi_mode mode);

/* Written-texel and byte sizes helpers (host, no CUDA). */
NDGI_API uint64_t ndgi_full_texels(const ndgi_layout* layout);
NDGI_API size_t ndgi_texel_bytes(ndgi_out_fmt fmt);

/*
 * Synchronises the context's device and returns the number of rejected
 * requests (bad tile id or slot) and non-resident shading samples
 * (ndgi_sample_lighting) since load or the last reset; resets the counter
 * when `reset` != 0.
 */
NDGI_API ndgi_status ndgi_device_error(ndgi_ctx* ctx, uint32_t* bad_requests, int reset);

NDGI_API const char* ndgi_status_string(ndgi_status s);
/* detail of the last failing call on this host thread ("" if none) */
NDGI_API const char* ndgi_last_error(void);
NDGI_API ndgi_status ndgi_free(ndgi_ctx* ctx);

/* Validates a layout without touching CUDA (same rules as ndgi_load; FAST-mode
 * support reported through *fast_supported if non-NULL). */
NDGI_API ndgi_status ndgi_validate_layout(const ndgi_layout* layout, int* fast_supported);

/* ------------------------------------------------------------------------
 * Shading side of the page cache
 *
 * P:229 "During shading, we first sample the page table to locate each tile
 * within the physical texture, then sample the physical texture to obtain the
 * final lighting. For tiles already resident ... we can reuse the cached
 * content for a period"; P:521 (page table), P:524 (missing tiles, eviction),
 * P:526 (border for filtering), P:232 (gamma + per-time channel means,
 * restored during rendering).  Readings R21-R25 in DESIGN.md.
 * ------------------------------------------------------------------------ */

/* Page table + strict-LRU residency of `capacity` page-cache slots, host
 * side.  `num_buckets` time buckets over t in [0,1] (SPEC's default 96, i.e.
 * 15 minutes of a day): a tile resident for bucket b = floor(t * num_buckets)
 * (t = 1 -> last bucket) is reused for any t in that bucket and
 * re-decoded in place otherwise.  Not thread-safe: one host thread per
 * ndgi_vt.  Errors: ARG (0 tiles/slots/buckets, > 2^20 buckets), NOMEM. */
typedef struct ndgi_vt ndgi_vt;
NDGI_API ndgi_status ndgi_vt_create(uint32_t num_tiles, uint32_t capacity, uint32_t num_buckets, ndgi_vt** out);
NDGI_API ndgi_status ndgi_vt_free(ndgi_vt* vt);

/*
 * One frame's tile requests ("identifies missing tiles"): ids = HOST
 * u32[n] (duplicates allowed); for every distinct id that is not resident
 * for bucket(t) a decode job (job_ids[j], job_slots[j]), j < *n_jobs <= n,
 * HOST arrays with room for n entries.  Slots: never-used slots first (in
 * increasing order), then the least recently requested slot not requested in
 * this frame; the evicted tile becomes absent.  The page table is updated as
 * if the jobs had run: decode them (ndgi_decode_tiles(ctx, job ids, job
 * slots, *n_jobs, capacity, *t_decode, cache, ...) with *t_decode = the
 * bucket centre) and upload the table on the same stream before sampling.
 * *bucket receives bucket(t) (optional).  Errors: ARG (NULL, id >=
 * num_tiles: no state change), RANGE (t outside [0,1], or more distinct ids
 * than slots: no state change).
 */
NDGI_API ndgi_status ndgi_vt_request(ndgi_vt* vt, const uint32_t* ids, uint32_t n, float t, uint32_t* job_ids,
                                     uint32_t* job_slots, uint32_t* n_jobs, float* t_decode, int32_t* bucket);
/* bucket(t) and its decode time (b + 1/2) / num_buckets, without touching residency */
NDGI_API ndgi_status ndgi_vt_bucket(const ndgi_vt* vt, float t, int32_t* bucket, float* t_decode);
/* HOST copy of the page table: int32 [num_tiles][2] = (slot, bucket), slot -1 = absent */
NDGI_API ndgi_status ndgi_vt_page_table(const ndgi_vt* vt, int32_t* out_host);
/* the page table -> DEVICE int32 [num_tiles][2], stream-ordered (returns once
 * staged); skipped when the table is unchanged since the last upload to the
 * same buffer (the caller must not write that buffer in between) */
NDGI_API ndgi_status ndgi_vt_upload(ndgi_vt* vt, int32_t* page_table_dev, void* stream);
/* counters: [distinct tile requests, hits, decode jobs, evictions] */
NDGI_API ndgi_status ndgi_vt_stats(const ndgi_vt* vt, uint64_t out[4]);

/* HDR restore parameters of the lightmap sets: the decoder output is
 * gamma-corrected and normalised by per-channel means at each bake time. */
typedef struct ndgi_hdr {
    float gamma;               /* g > 0: stored value x -> x^g (R23)                    */
    uint32_t n_frames;         /* bake times                                            */
    const float* frame_times;  /* HOST [n_frames], strictly increasing                  */
    const float* means;        /* HOST [atlases][n_frames][3] per-channel means (R22)   */
} ndgi_hdr;

/*
 * Shading samples of the page cache: for sample i at
 * (u, v) = uv[i] in [0,1]^2 (clamped) of atlas atlas[i] (NULL: atlas 0), the
 * owning tile is the one whose core contains the point on the atlas texel grid
 * (centres at ((x + 0.5)/W, (y + 0.5)/H), W = tiles_x*C, H = tiles_y*C); its
 * page-table entry must be (slot < num_slots, bucket); the RGBA8 slot is
 * filtered bilinearly, the border supplying taps outside the core (R25),
 * and restored: out = (filtered/255)^g * mu_hat(t, c) (R21), mu_hat linear
 * between the bracketing bake times (R22).
 *   page_table: DEVICE int32 [num_tiles][2] (ndgi_vt_upload)
 *   cache     : DEVICE [num_slots][P][P][4] RGBA8 (ndgi_decode_tiles output)
 *   uv        : DEVICE float [n][2];  atlas: DEVICE u32 [n] or NULL
 *   out_rgb   : DEVICE float [n][3], linear HDR
 * Non-resident samples (absent tile, other bucket, bad atlas/slot) get NaN
 * and count in ndgi_device_error.  Position math in fp64, filter and restore
 * in fp32.  Errors (synchronous): ARG (NULL, gamma <= 0, frame times not
 * increasing, means not finite), RANGE (t outside the bake times),
 * UNSUPPORTED (border 0 or > 64 atlases), CUDA.  n == 0 is a no-op.
 */
NDGI_API ndgi_status ndgi_sample_lighting(ndgi_ctx* ctx, const int32_t* page_table, int32_t bucket,
                                          const void* cache, uint32_t num_slots, const float* uv,
                                          const uint32_t* atlas, uint32_t n, float t, const ndgi_hdr* hdr,
                                          float* out_rgb, void* stream);

/* ------------------------------------------------------------------------
 * BC7 encoder: the step before the path, turning
 * 8-bit feature maps into the BC7 payloads ndgi_load takes ("apply the
 * BC7 compression algorithm, which encodes each 4x4 texel block").
 * Mode 6 (single subset, RGBA, 7-bit endpoints + p-bits, 4-bit indices),
 * defined in exact integer arithmetic by reading R26, so the
 * result is deterministic and equal to the oracle's encoder bit for bit.
 *   rgba  : DEVICE [h][w][4] u8, row-major (16-byte aligned)
 *   blocks: DEVICE [h/4][w/4][16 B], block (bx, by) at (by * w/4 + bx) * 16
 * Errors: ARG (NULL, w or h not a positive multiple of 4), RANGE (> 65536),
 * CUDA.  Asynchronous on `stream`.
 * ------------------------------------------------------------------------ */
NDGI_API ndgi_status ndgi_bc7_encode_mode6(const void* rgba, uint32_t w, uint32_t h, void* blocks, void* stream);

/* Multi-mode search (SURVEY.md §8(f) NEXT 3 "then multi-mode search";
 * reading R31): per block the mode-6 result above, then mode 5 with each of
 * the 4 rotations (7-bit RGB endpoints along the RGB principal axis, 8-bit
 * alpha endpoints min/max, 2-bit indices), then mode 7 with each of the 64
 * two-subset partitions (per-subset principal-axis endpoints, 5-bit + p-bit,
 * 2-bit indices); a candidate replaces the best only if its squared error
 * is strictly smaller.  Same arguments, layout and errors as
 * ndgi_bc7_encode_mode6; equal to the oracle's search bit for bit.        */
NDGI_API ndgi_status ndgi_bc7_encode_multi(const void* rgba, uint32_t w, uint32_t h, void* blocks, void* stream);

/* ------------------------------------------------------------------------
 * Fine-tuning of the per-tile decoders: the paper's
 * last training stage, "we freeze the feature maps and fine-tune the MLP
 * under simulated quantization and BC compression" with Adam and an L2 loss
 * (P:234); reading R27.  The features are the context's stored (quantized /
 * BC7) maps sampled at (u, v, t) like the decode samples them; the trainer
 * owns an fp32 master copy of every tile's MLP (initialised from the
 * context's f16 weights) and the Adam state (beta 0.9 / 0.999, eps 1e-8,
 * bias correction with each tile's own step count).  h = 16 only
 * (UNSUPPORTED otherwise).  The context's own f16 weights and prepacked
 * operands are not changed: export and create a new context to decode with
 * the fine-tuned weights.
 * ------------------------------------------------------------------------ */
typedef struct ndgi_train ndgi_train;
NDGI_API ndgi_status ndgi_train_create(ndgi_ctx* ctx, ndgi_train** out);
/* One step for n tiles: DEVICE tile_ids u32[n], samples float[n][S][3]
 * (u, v, t in [0,1]), targets float[n][S][3] (RGB); loss: DEVICE float[n]
 * (mean squared error of each tile before the update) or NULL.  Tiles with
 * an id >= num_tiles are skipped and counted (ndgi_device_error); a tile may
 * appear once per step.  Errors: ARG, RANGE (n > 2^20, S > 2^24), CUDA. */
NDGI_API ndgi_status ndgi_train_step(ndgi_train* tr, const uint32_t* tile_ids, uint32_t n, const float* samples,
                                     const float* targets, uint32_t S, float lr, float* loss, void* stream);
/*
 * Full training step (reading R28): the BC-simulated
 * feature maps of Eq. 6-7 (per 4x4 block endpoints e1, e2 and 16 weights;
 * texel p = (1 - w_p) e1 + w_p e2), the plain line grids and the MLP are all
 * trained; the sampled vectors get uniform noise alpha * n (Eq. 5, alpha =
 * 1/256); after each Adam step the map parameters are projected onto [0,1].
 * Parameters per tile (ndgi_train_full_params(layout) floats, fp32):
 *   [MLP blob (as ndgi_params.mlp) | F_uv blocks [(R_uv/4)^2][24] |
 *    F_uvt blocks [D][(R3/4)^2][24] | F_ut [T][U][2] | F_vt [T][U][2]],
 *   block = [e1 RGBA | e2 RGBA | w_0 .. w_15] (texel p = 4 * row + col).
 * init: DEVICE float [num_tiles][P], copied.  The context supplies the layout
 * (its feature maps are not used).  Steps take DEVICE noise float[n][S][12]
 * (draws in [-0.5, 0.5): V_uvt 0..3, V_uv 4..7, V_ut 8..9, V_vt 10..11).
 * ndgi_train_weights / _last_grad then move P floats per tile;
 * ndgi_train_export_f16 exports the MLP part.  Errors as the fine-tuning calls.
 */
NDGI_API size_t ndgi_train_full_params(const ndgi_layout* layout);
NDGI_API ndgi_status ndgi_train_full_create(ndgi_ctx* ctx, const float* init, ndgi_train** out);
NDGI_API ndgi_status ndgi_train_full_step(ndgi_train* tr, const uint32_t* tile_ids, uint32_t n, const float* samples,
                                          const float* targets, const float* noise, uint32_t S, float lr, float* loss,
                                          void* stream);

/*
 * Export of a full trainer's tiles to a deployable Theta (SURVEY.md §8(f)
 * NEXT 3 "u8 PTQ plus a BC7 encoder"; "BC compression on the final
 * generated feature maps"; reading R30).  Per tile: every BC-simulated
 * block's 16 texels by Eq. 7 in fp32 (each operation rounded, no FMA),
 * post-training quantisation q = RN-even(clamp(x, 0, 1) * 255), BC7 mode 6
 * (as ndgi_bc7_encode_mode6) for F_uv and each F_uvt slice; line grids by
 * the same PTQ to u8; the MLP to f16 (RN-even).  All outputs DEVICE, in
 * ndgi_load's dense per-tile layouts for fmt_uv = fmt_uvt = NDGI_FMT_BC7,
 * fmt_line = NDGI_FMT_U8: uv [num_tiles][R_uv/4][R_uv/4][16] B,
 * uvt [num_tiles][D][R3/4][R3/4][16] B, ut / vt [num_tiles][T][U][2] B,
 * mlp [num_tiles][P_mlp] f16.  Needs a full trainer (NDGI_ERR_ARG otherwise);
 * stream-ordered; uses stream-ordered scratch of 4 B per map texel.
 */
NDGI_API ndgi_status ndgi_train_full_export(ndgi_train* tr, void* uv, void* uvt, void* ut, void* vt, uint16_t* mlp,
                                            void* stream);

/* the last step's gradients (mean-loss gradient of each batch tile, before
 * Adam) -> DEVICE float[n][P]; n <= that step's batch (RANGE otherwise) */
NDGI_API ndgi_status ndgi_train_last_grad(ndgi_train* tr, float* out, uint32_t n, void* stream);
/* fp32 master weights -> DEVICE float[num_tiles][P] (P = 595 for h = 16, blob order) */
NDGI_API ndgi_status ndgi_train_weights(ndgi_train* tr, float* out, void* stream);
/* master weights rounded to f16 -> DEVICE [num_tiles][P] (an ndgi_params.mlp buffer) */
NDGI_API ndgi_status ndgi_train_export_f16(ndgi_train* tr, uint16_t* mlp, void* stream);
NDGI_API ndgi_status ndgi_train_free(ndgi_train* tr);

/* ---------------- test hooks (not the product path) ---------------- */

/* Bit-exact BC7 map decode: blocks (DEVICE, (w/4)*(h/4) blocks row-major) ->
 * rgba (DEVICE, [h][w][4] u8).  w, h multiples of 4.  Same device decoder as
 * the fused kernel. */
NDGI_API ndgi_status ndgi_debug_bc7_decode(const void* blocks, uint32_t w, uint32_t h, uint8_t* rgba, void* stream);

/* Same map decoded by the GPU texture unit (cudaArray of BC7 with
 * cudaChannelFormatKindUnsignedBlockCompressed7, point sampling): an
 * independent hardware decoder for the cross-check.  Synchronous. */
NDGI_API ndgi_status ndgi_debug_bc7_decode_hw(const void* blocks, uint32_t w, uint32_t h, uint8_t* rgba);

/* GELU-rate microbenchmark for the ALU roofline (SURVEY.md §8(d) T_alu):
 * the fused kernel's own f16x2 GELU epilogue functions on 148 x 2048 threads,
 * 16 independent chains of GELU pairs per thread, `mufu_pairs` of every 16
 * pairs through MUFU.TANH (tanh.approx.f16x2) and the rest through the
 * FMA-pipe polynomial; pack_f32 != 0 first packs each pair from two fp32
 * values (cvt.rn.f16x2.f32) as the fp32-accumulator epilogue does.  Returns
 * the elapsed device milliseconds and activations evaluated (2 per pair).
 * Errors: ARG, RANGE (mufu_pairs > 16), CUDA.  Synchronous. */
NDGI_API ndgi_status ndgi_debug_gelu_rate(uint32_t iters, uint32_t mufu_pairs, int pack_f32, float* ms,
                                          double* activations);

/* The GELU formulation compiled into the fused kernel for hidden width h (16
 * or 64): MUFU pairs of every 16 GELU pairs (the rest on the FMA pipe) and
 * whether the hidden layers accumulate in fp32 (1) or f16 (0). */
NDGI_API ndgi_status ndgi_debug_gelu_split(uint32_t hidden, uint32_t* mufu_pairs_of_16, int* fp32_acc);

/* Launch-latency floor of the VT path: one empty kernel launched on `stream`
 * through the C ABI (bench.py times it beside ndgi_decode_tiles). */
NDGI_API ndgi_status ndgi_debug_null_launch(void* stream);

/* Launch-cost probes beside the floor: kind 0 = the empty kernel above, 1 = an
 * empty kernel with the fused kernel's parameter block, 2 = an empty 256-CTA
 * grid with 24 KB of dynamic smem, 3 = 256 CTAs allocating and freeing 64
 * TMEM columns.  Errors: ARG, CUDA. */
NDGI_API ndgi_status ndgi_debug_launch_probe(int kind, void* stream);

/* tcgen05 round-trip microbenchmark (st A, barrier, MMA M128N16K16, commit,
 * mbarrier wait, ld D) on one CTA: SM cycles per iteration.  Synchronous. */
NDGI_API ndgi_status ndgi_debug_mma_latency(uint32_t iters, double* cycles_per_iter);

/* TMEM layout probe of an f16-accumulator MMA (M128 N16 K16, B = identity):
 * host_out[128][24] receives columns 0..15 of every lane, then the same columns
 * read with .pack::16b (8 words).  Synchronous. */
NDGI_API ndgi_status ndgi_debug_tmem_f16_probe(uint32_t* host_out);

/* Rounding probe of the f16-accumulator MMA: `ctas` CTAs x `iters` random
 * M128 N16 K16 problems (A in TMEM, B in smem; f16 operands up to |x| 256),
 * each issued once with an fp32 D and once with an f16 D; *mismatches counts
 * the f16x2 output pairs where the f16 D differs from cvt.rn.f16x2 of the
 * fp32 D, *pairs the pairs compared.  Synchronous.  Errors: ARG, CUDA. */
NDGI_API ndgi_status ndgi_debug_f16d_probe(uint32_t seed, uint32_t iters, uint32_t ctas, uint64_t* mismatches,
                                           uint64_t* pairs);

#ifdef __cplusplus
}
#endif
#endif /* NDGI_H */
