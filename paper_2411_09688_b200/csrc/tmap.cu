// tmap.cu -- host-side TMA tensor-map encoding, resolved through the runtime's
// driver entry point so libsqz has no link-time libcuda dependency.
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>
#include <vector>

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

// Contiguous bf16 matrix [rows][cols], boxes of box_rows x box_cols, 128-byte
// swizzle (box_cols * 2 = 128 for the swizzle span), out-of-bounds reads = 0.
int encode_tmap_bf16_2d(CUtensorMap *m, const void *ptr, uint64_t cols, uint64_t rows, uint32_t box_cols,
                        uint32_t box_rows) {
    encode_fn fn = resolve();
    if (!fn) return -1;
    const cuuint64_t d[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t b[2] = {box_cols, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), d, strides, b, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : (int)r;
}

}  // namespace sqz

// ---------------------------------------------------------------------------
// Per-device launch-configuration caches.  Function attributes (the opt-in
// dynamic shared memory size, non-portable cluster sizes) belong to each
// device's context, and SM counts / occupancies differ by device, so every
// cached value is keyed by (device ordinal, kernel) and guarded by a mutex:
// a process may drive several GPUs from several threads.
// ---------------------------------------------------------------------------
namespace sqz {
namespace {
struct AttrEntry {
    int dev;
    const void *kern;
    int attr;   // cudaFuncAttribute, or -1 for an occupancy entry
    long long key;  // occupancy: threads << 32 | smem
    int value;
};
std::mutex g_cache_mu;
std::vector<AttrEntry> g_cache;
int g_sm_count[64];
}  // namespace

int device_sm_count() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    std::lock_guard<std::mutex> lk(g_cache_mu);
    if (!g_sm_count[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        g_sm_count[dev] = n > 0 ? n : 148;
    }
    return g_sm_count[dev];
}

cudaError_t ensure_func_attr(const void *kern, cudaFuncAttribute attr, int value) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (AttrEntry &x : g_cache)
        if (x.dev == dev && x.kern == kern && x.attr == (int)attr) {
            if (x.value >= value) return cudaSuccess;  // a larger opt-in covers this one
            e = cudaFuncSetAttribute(kern, attr, value);
            if (e == cudaSuccess) x.value = value;
            return e;
        }
    e = cudaFuncSetAttribute(kern, attr, value);
    if (e == cudaSuccess) g_cache.push_back({dev, kern, (int)attr, 0, value});
    return e;
}

int occupancy_blocks(const void *kern, int threads, size_t smem) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 1;
    const long long key = ((long long)threads << 32) | (long long)smem;
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (const AttrEntry &x : g_cache)
        if (x.dev == dev && x.kern == kern && x.attr == -1 && x.key == key) return x.value;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess) occ = 1;
    occ = occ > 0 ? occ : 1;
    g_cache.push_back({dev, kern, -1, key, occ});
    return occ;
}

}  // namespace sqz
