// tex_uv.cu -- NDGI_MODE_FAST_TEXUNIT: F_uv through
// the B200 texture unit's BC7 decoder, the paper's own runtime mechanism
// ("hardware-accelerated ... decoding is performed entirely in hardware during
// texture sampling"), as an in-box comparator for the kernel's
// software decoder.
//
// Per atlas, one 2D BC7 texture over the atlas's F_uv maps (tile (tx, ty)'s
// map at texels [tx*C, (tx+1)*C) x [ty*C, (ty+1)*C); R_uv == C, R2): the
// context copies the tile-major BC7 blocks of Theta into atlas block order
// once (a scatter kernel + one 2D copy into a cudaArray), the fused kernel
// fetches texel centres with point sampling (tex2D) and no smem chunk decode.
#include <cuda_runtime.h>

#include <cstdint>

#include "ndgi_common.cuh"

namespace ndgi {

// tile-major [tile][C/4][C/4] blocks -> block-row-major image of one atlas
__global__ void scatter_uv_blocks(const uint4* __restrict__ src, uint4* __restrict__ dst, int tiles_x, int tiles_y,
                                  int bpt /* blocks per tile side */, size_t tile0) {
    const size_t nb = (size_t)tiles_x * tiles_y * bpt * bpt;
    const int wb = tiles_x * bpt;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < nb; e += (size_t)gridDim.x * blockDim.x) {
        const int bx = (int)(e % wb), by = (int)(e / wb);
        const int tx = bx / bpt, ty = by / bpt;
        const size_t tile = tile0 + (size_t)ty * tiles_x + tx;
        dst[e] = src[(tile * bpt + (by % bpt)) * bpt + (bx % bpt)];
    }
}

// builds the per-atlas BC7 textures; arrays/textures are returned for the
// context to own (destroy with uv_textures_free)
cudaError_t uv_textures_build(const void* uv, int atlases, int tiles_x, int tiles_y, int C, cudaArray_t* arrays,
                              unsigned long long* texs) {
    const int bpt = C / 4;
    const int wb = tiles_x * bpt, hb = tiles_y * bpt;
    uint4* staging = nullptr;
    cudaError_t e = cudaMalloc(&staging, (size_t)wb * hb * 16);
    if (e != cudaSuccess) return e;
    for (int a = 0; a < atlases && e == cudaSuccess; ++a) {
        arrays[a] = nullptr;
        texs[a] = 0;
        const size_t tile0 = (size_t)a * tiles_x * tiles_y;
        scatter_uv_blocks<<<1024, 256>>>(reinterpret_cast<const uint4*>(uv), staging, tiles_x, tiles_y, bpt, tile0);
        e = cudaGetLastError();
        if (e != cudaSuccess) break;
        const cudaChannelFormatDesc cd = cudaCreateChannelDesc(32, 32, 32, 32, cudaChannelFormatKindUnsigned);
        e = cudaMallocArray(&arrays[a], &cd, wb, hb);
        if (e != cudaSuccess) break;
        e = cudaMemcpy2DToArray(arrays[a], 0, 0, staging, (size_t)wb * 16, (size_t)wb * 16, hb, cudaMemcpyDeviceToDevice);
        if (e != cudaSuccess) break;
        cudaResourceDesc rd = {};
        rd.resType = cudaResourceTypeArray;
        rd.res.array.array = arrays[a];
        cudaTextureDesc td = {};
        td.addressMode[0] = td.addressMode[1] = cudaAddressModeClamp;
        td.filterMode = cudaFilterModePoint;
        td.readMode = cudaReadModeElementType;   // BC7 views return UNORM floats
        td.normalizedCoords = 0;
        cudaResourceViewDesc vd = {};
        vd.format = cudaResViewFormatUnsignedBlockCompressed7;
        vd.width = (size_t)wb * 4;
        vd.height = (size_t)hb * 4;
        cudaTextureObject_t t = 0;
        e = cudaCreateTextureObject(&t, &rd, &td, &vd);
        texs[a] = t;
    }
    cudaError_t e2 = cudaDeviceSynchronize();   // staging is freed below
    cudaFree(staging);
    return e != cudaSuccess ? e : e2;
}

void uv_textures_free(int atlases, cudaArray_t* arrays, unsigned long long* texs) {
    for (int a = 0; a < atlases; ++a) {
        if (texs[a]) cudaDestroyTextureObject(texs[a]);
        if (arrays[a]) cudaFreeArray(arrays[a]);
        texs[a] = 0;
        arrays[a] = nullptr;
    }
}

}  // namespace ndgi
