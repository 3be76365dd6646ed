// tmap.cu -- host-side TMA tensor-map encoding, resolved through the runtime's
// driver entry point so libsqz has no link-time libcuda dependency.
#include <cuda.h>
#include <cuda_runtime.h>

#include "internal.h"

namespace sqz {

namespace {
using encode_fn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                               const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                               const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
encode_fn resolve() {
    static encode_fn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<encode_fn>(p);
    }();
    return fn;
}
}  // namespace

// Contiguous bf16 tensor [dims[2]][dims[1]][dims[0]] (dims[0] innermost), boxes of
// box[0] x box[1] x box[2] elements, 128-byte swizzle, out-of-bounds reads = 0.
int encode_tmap_bf16_3d(CUtensorMap *m, const void *ptr, const uint64_t dims[3], const uint32_t box[3]) {
    encode_fn fn = resolve();
    if (!fn) return -1;
    const cuuint64_t d[3] = {dims[0], dims[1], dims[2]};
    const cuuint64_t strides[2] = {dims[0] * 2, dims[0] * dims[1] * 2};
    const cuuint32_t b[3] = {box[0], box[1], box[2]};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(ptr), d, strides, b, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : (int)r;
}

}  // namespace sqz
