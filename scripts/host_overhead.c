/* Host-side cost of one ndgi_decode_tiles call (VT batch of 8) measured in C,
 * without the Python binding: many calls back to back, then one sync.
 * build: gcc -O2 scripts/host_overhead.c -Iinclude -I/usr/local/cuda/include \
 *        -Lpaper_2604_12625_b200 -lndgi -L/usr/local/cuda/lib64 -lcudart -o /tmp/host_overhead */
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>
#include <time.h>

#include "ndgi.h"

static double now(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

int main(void) {
    ndgi_layout L;
    memset(&L, 0, sizeof(L));
    L.abi_version = NDGI_ABI_VERSION;
    L.num_tiles = 64; L.atlases = 1; L.tiles_x = 8; L.tiles_y = 8;
    L.core = 128; L.border = 4; L.uv_res = 128; L.uvt_res = 32; L.uvt_depth = 12;
    L.line_res = 64; L.line_t = 24; L.hidden = 16;
    L.fmt_uv = NDGI_FMT_BC7; L.fmt_uvt = NDGI_FMT_BC7; L.fmt_line = NDGI_FMT_U8;
    L.gelu = NDGI_GELU_ERF; L.border_mode = NDGI_BORDER_MIRROR;
    void *uv, *uvt, *ut, *vt, *mlp, *cache, *ids;
    cudaMalloc(&uv, 64 * 16384); cudaMemset(uv, 0, 64 * 16384);
    cudaMalloc(&uvt, 64 * 12288); cudaMemset(uvt, 0, 64 * 12288);
    cudaMalloc(&ut, 64 * 3072); cudaMemset(ut, 0, 64 * 3072);
    cudaMalloc(&vt, 64 * 3072); cudaMemset(vt, 0, 64 * 3072);
    cudaMalloc(&mlp, 64 * 1190); cudaMemset(mlp, 0, 64 * 1190);
    cudaMalloc(&cache, 8 * 136 * 136 * 4);
    unsigned hid[8] = {0, 9, 18, 27, 36, 45, 54, 63};
    cudaMalloc(&ids, sizeof(hid)); cudaMemcpy(ids, hid, sizeof(hid), cudaMemcpyHostToDevice);
    ndgi_params P = {uv, uvt, ut, vt, (const uint16_t*)mlp};
    ndgi_ctx* ctx = 0;
    if (ndgi_load(&L, &P, 0, &ctx) != NDGI_OK) { printf("load failed: %s\n", ndgi_last_error()); return 1; }
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (int i = 0; i < 100; ++i) ndgi_decode_tiles(ctx, ids, 0, 8, 8, 0.3f, cache, NDGI_OUT_RGBA8, NDGI_MODE_FAST, s);
    cudaStreamSynchronize(s);
    const int N = 5000;
    double host = 0.0, all = 0.0;
    for (int i = 0; i < N; ++i) {   /* idle GPU at every call: the call's own host cost */
        const double t0 = now();
        ndgi_decode_tiles(ctx, ids, 0, 8, 8, 0.3f, cache, NDGI_OUT_RGBA8, NDGI_MODE_FAST, s);
        const double t1 = now();
        cudaStreamSynchronize(s);
        const double t2 = now();
        host += t1 - t0;
        all += t2 - t0;
    }
    printf("{\"c_host_us_per_call\": %.3f, \"c_call_to_done_us\": %.3f}\n", host / N * 1e6, all / N * 1e6);
    ndgi_free(ctx);
    return 0;
}
