// launch_util.cuh -- host helpers shared by the fused codec kernels' launchers
// (tensor maps for the TMA loads / stores, persistent launch shapes).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

namespace fntrs_gpu {
namespace fast {
namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 2-D map over a packet-major uint16 buffer [rows][L], box [box_rows][wt].
cudaError_t make_map(CUtensorMap* map, const void* base, uint64_t rows, uint32_t L, uint32_t wt, uint32_t box_rows) {
    EncodeTiledFn fn = encode_tiled();
    if (!fn) return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {L, rows};
    const cuuint64_t strides[1] = {cuuint64_t(L) * 2};
    const cuuint32_t box[2] = {wt, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// 3-D map over packet-major uint16 stripes [stripes][rows][L], box [1][box_rows][wt]:
// a box never crosses into the next stripe (rows beyond `rows` are clipped).
cudaError_t make_map3(CUtensorMap* map, const void* base, uint64_t stripes, uint32_t rows, uint32_t L, uint32_t wt,
                      uint32_t box_rows) {
    EncodeTiledFn fn = encode_tiled();
    if (!fn) return cudaErrorNotSupported;
    const cuuint64_t dims[3] = {L, rows, stripes};
    const cuuint64_t strides[2] = {cuuint64_t(L) * 2, cuuint64_t(L) * rows * 2};
    const cuuint32_t box[3] = {wt, box_rows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

struct LaunchShape {
    uint32_t tps, tiles, nbox, box_rows, grid;
    size_t smem;
};

template <class K>
cudaError_t shape_for(K kernel, int E, int wt, int nt, uint32_t k, uint32_t stripes, uint32_t L, LaunchShape& sh,
                      size_t extra = 0, int stages = 2) {
    sh.tps = L / wt;
    const uint64_t tiles = uint64_t(stripes) * sh.tps;
    if (tiles > 0xFFFFFFFFull) return cudaErrorInvalidConfiguration;
    sh.tiles = uint32_t(tiles);
    sh.box_rows = k < 256 ? k : 256;
    sh.nbox = (k + sh.box_rows - 1) / sh.box_rows;
    sh.smem = (size_t(1) << E) * wt * 4 + size_t(stages) * sh.nbox * sh.box_rows * wt * 2 + extra;
    cudaError_t err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sh.smem));
    if (err) return err;
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if ((err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, nt, sh.smem))) return err;
    if (per < 1) return cudaErrorInvalidConfiguration;
    const uint64_t g = uint64_t(sms) * per;
    sh.grid = uint32_t(g < tiles ? g : tiles);
    return cudaSuccess;
}

}  // namespace
}  // namespace fast
}  // namespace fntrs_gpu
