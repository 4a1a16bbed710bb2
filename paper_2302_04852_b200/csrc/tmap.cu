// tmap.cu -- host-side TMA tensor maps (cuTensorMapEncodeTiled through the
// runtime's driver entry point, so the library links only cudart).
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>

#include "sp_internal.cuh"

namespace sp {
namespace {

using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

}  // namespace

bool make_tmap_2d(CUtensorMap *map, const float *base, int64_t rows, int64_t B, int box_cols, int box_rows) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)B, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)B * sizeof(float)};
    const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 4-D map of a conv product's input for the tap tiles of cc: CHWN [C][H][W][B]
// (dims innermost first B, W, H, C; box bs x nq x 1 x kc) or NCHW [B][C][H][W]
// (dims W, H, C, B; box nq x np x kc x 1).  One box is a [kc][128] tile of the
// slice's exact output positions; coordinates may be negative or past the edge
// (the conv halo), which the hardware zero-fills.
bool make_tmap_conv(CUtensorMap *map, const float *base, const ConvCols &cc, int64_t C, int64_t H, int64_t W,
                    int kc) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    const int64_t B = cc.B;
    cuuint64_t dims[4], strides[3];
    cuuint32_t box[4];
    if (cc.nchw) {
        dims[0] = (cuuint64_t)W, dims[1] = (cuuint64_t)H, dims[2] = (cuuint64_t)C, dims[3] = (cuuint64_t)B;
        strides[0] = (cuuint64_t)W * sizeof(float);
        strides[1] = (cuuint64_t)(H * W) * sizeof(float);
        strides[2] = (cuuint64_t)(C * H * W) * sizeof(float);
        box[0] = (cuuint32_t)cc.nq, box[1] = (cuuint32_t)cc.np, box[2] = (cuuint32_t)kc, box[3] = 1u;
    } else {
        dims[0] = (cuuint64_t)B, dims[1] = (cuuint64_t)W, dims[2] = (cuuint64_t)H, dims[3] = (cuuint64_t)C;
        strides[0] = (cuuint64_t)B * sizeof(float);
        strides[1] = (cuuint64_t)(W * B) * sizeof(float);
        strides[2] = (cuuint64_t)(H * W * B) * sizeof(float);
        box[0] = (cuuint32_t)(1 << cc.bsh), box[1] = (cuuint32_t)cc.nq, box[2] = 1u, box[3] = (cuuint32_t)kc;
    }
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace sp
