// ref_kernel.cu -- NDGI_MODE_REF_FP32: scalar fp32 reference decode.
//
// One thread per written texel, every step in fp32 on the CUDA cores, accurate
// erff/tanhf GELU per the layout flag (reading R7).  It shares the BC7 device
// decoder with the fused kernel (bc7_device.cuh) and nothing else; its job is
// the <= 1e-5 parity mode of BASELINE.json's north_star, not speed.
//
// Per texel (Eq. 3/4):
//   (i, j) = mirror(x - B, y - B)            R3 (or unreflected: EVAL_CLAMP)
//   u = (i + 0.5)/C, v = (j + 0.5)/C         R1, R2
//   V_uvt = (1-tau) S(slice k0) + tau S(slice k1)   R4 (4-tap bilinear each)
//   V_uv = S(F_uv; u, v), V_ut = S(F_ut; u, t), V_vt = S(F_vt; v, t)   R5
//   x = [V_uvt, V_uv, V_ut, V_vt, gamma(t)]  R6
//   y = W3 gelu(W2 gelu(W1 x + b1) + b2) + b3
#include "ref_common.cuh"

namespace ndgi {

__device__ void eval_texel(const KParams& p, const TConst& tc, int k, int i, int j, float* y) {
    const float u = ((float)i + 0.5f) / (float)p.C, v = ((float)j + 0.5f) / (float)p.C;
    float x[16];
    // V_uvt (trilinear = tau-blend of two bilinear slice samples)
    const uint8_t* vol = p.uvt + p.uvt_tile_bytes * k;
    Map2D s0{vol + p.uvt_slice_bytes * tc.k0, p.fmt_uvt, p.R3, p.R3, 4};
    Map2D s1{vol + p.uvt_slice_bytes * tc.k1, p.fmt_uvt, p.R3, p.R3, 4};
    float a[4], b[4];
    bilinear(s0, u, v, a);
    bilinear(s1, u, v, b);
    for (int c = 0; c < 4; ++c) x[c] = (1.0f - tc.tau) * a[c] + tc.tau * b[c];
    Map2D uvm{p.uv + p.uv_tile_bytes * k, p.fmt_uv, p.R_uv, p.R_uv, 4};
    bilinear(uvm, u, v, x + 4);
    Map2D utm{p.ut + p.line_tile_bytes * k, p.fmt_line, p.U, p.T, 2};
    Map2D vtm{p.vt + p.line_tile_bytes * k, p.fmt_line, p.U, p.T, 2};
    bilinear(utm, u, tc.t, x + 8);
    bilinear(vtm, v, tc.t, x + 10);
    for (int g = 0; g < 4; ++g) x[12 + g] = tc.gamma[g];

    const int h = p.H;
    const uint16_t* w = p.mlp + p.mlp_tile_elems * k;
    const uint16_t *W1 = w, *b1 = W1 + 16 * h, *W2 = b1 + h, *b2 = W2 + h * h, *W3 = b2 + h, *b3 = W3 + 3 * h;
    float h1[256], h2[256];
    for (int o = 0; o < h; ++o) {
        float acc = half_bits_to_float(b1[o]);
        for (int q = 0; q < 16; ++q) acc = fmaf(half_bits_to_float(W1[o * 16 + q]), x[q], acc);
        h1[o] = gelu_ref(acc, p.gelu);
    }
    for (int o = 0; o < h; ++o) {
        float acc = half_bits_to_float(b2[o]);
        for (int q = 0; q < h; ++q) acc = fmaf(half_bits_to_float(W2[o * h + q]), h1[q], acc);
        h2[o] = gelu_ref(acc, p.gelu);
    }
    for (int o = 0; o < 3; ++o) {
        float acc = half_bits_to_float(b3[o]);
        for (int q = 0; q < h; ++q) acc = fmaf(half_bits_to_float(W3[o * h + q]), h2[q], acc);
        y[o] = acc;
    }
}

// grid.x = output rows: n_req * P (decode_tiles) or num_tiles * C (decode_full); grid.y = query time
__global__ void __launch_bounds__(128) ndgi_ref_kernel(const __grid_constant__ KParams p) {
    const int row = blockIdx.x;
    const TConst& tc = p.tc[blockIdx.y];
    int k, y, width;
    size_t out_row;
    if (p.full) {
        k = row / p.C;
        y = row % p.C + p.B;
        width = p.C;
        const int tx = k % p.tiles_x, ty = (k / p.tiles_x) % p.tiles_y, a = k / (p.tiles_x * p.tiles_y);
        const size_t W = (size_t)p.tiles_x * p.C, Hh = (size_t)p.tiles_y * p.C;
        out_row = (size_t)blockIdx.y * p.out_t_stride + (size_t)a * Hh * W + ((size_t)ty * p.C + (y - p.B)) * W + (size_t)tx * p.C;
    } else {
        const int r = row / p.P;
        y = row % p.P;
        width = p.P;
        const uint32_t tid = p.tile_ids[r];
        const uint32_t slot = p.slots ? p.slots[r] : (uint32_t)r;
        if (tid >= (uint32_t)p.num_tiles || slot >= p.num_slots) {
            if (y == 0 && threadIdx.x == 0 && blockIdx.y == 0) atomicAdd(p.err, 1u);
            return;
        }
        k = (int)tid;
        out_row = ((size_t)slot * p.P + y) * p.P;
    }
    for (int x = threadIdx.x; x < width; x += blockDim.x) {
        const int xx = p.full ? x + p.B : x;
        int i = xx - p.B, j = y - p.B;
        if (p.border_mode == BORDER_MIRROR) {
            i = mirror_core(i, p.C);
            j = mirror_core(j, p.C);
        }
        float yv[3];
        eval_texel(p, tc, k, i, j, yv);
        store_texel(p.out, out_row + x, p.out_fmt, yv[0], yv[1], yv[2]);
    }
}

cudaError_t launch_ref(const KParams& p, cudaStream_t stream) {
    const unsigned rows = p.full ? (unsigned)(p.num_tiles * p.C) : (unsigned)(p.n_req * p.P);
    ndgi_ref_kernel<<<dim3(rows, p.nt), 128, 0, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace ndgi
