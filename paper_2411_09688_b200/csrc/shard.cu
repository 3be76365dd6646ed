// shard.cu -- fixed-context sharding by cluster across GPUs.
//
// The paper runs on one GPU; this build partitions the fixed context
// of a layer across the ranks by cluster: Level-1 cluster p (single level:
// cluster i) lives on rank p mod world together with its children and their
// keys.  The plan is computed on the host from the integer tables; the rows
// (centroids, perm, cluster-major K/V) are gathered on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace sqz {

// dst[h][j] = src[h][map[h][j]] for rows of `row_bytes` (multiple of 16);
// map value < 0 -> zero row.
__global__ void k_gather_rows(const uint4 *__restrict__ src, int64_t src_rows, uint4 *__restrict__ dst,
                              int64_t dst_rows, const int32_t *__restrict__ map, int row_vec) {
    const int h = blockIdx.y;
    const int64_t n = dst_rows * row_vec;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / row_vec;
        const int v = (int)(e % row_vec);
        const int32_t r = map[(size_t)h * dst_rows + j];
        uint4 val = make_uint4(0, 0, 0, 0);
        if (r >= 0) val = src[((size_t)h * src_rows + r) * row_vec + v];
        dst[((size_t)h * dst_rows + j) * row_vec + v] = val;
    }
}

// perm_loc[h][j] = perm[h][key_src[h][j]] or -1
__global__ void k_gather_perm(const int32_t *__restrict__ perm, int64_t L, int32_t *__restrict__ out,
                              int64_t Lloc, const int32_t *__restrict__ key_src) {
    const int h = blockIdx.y;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < Lloc;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = key_src[(size_t)h * Lloc + j];
        out[(size_t)h * Lloc + j] = r >= 0 ? perm[(size_t)h * L + r] : -1;
    }
}

static cudaError_t gather(const void *src, int64_t src_rows, void *dst, int64_t dst_rows,
                          const int32_t *map, int H, size_t row_bytes, cudaStream_t st) {
    if (dst_rows == 0) return cudaSuccess;
    const int row_vec = (int)(row_bytes / 16);
    const int64_t n = dst_rows * row_vec;
    dim3 g((unsigned)std::min<int64_t>(4096, (n + 255) / 256), H);
    k_gather_rows<<<g, 256, 0, st>>>(reinterpret_cast<const uint4 *>(src), src_rows,
                                     reinterpret_cast<uint4 *>(dst), dst_rows, map, row_vec);
    return cudaGetLastError();
}

cudaError_t launch_shard_gather(const sqz_index &full, const void *Kp, const void *Vp,
                                const int32_t *c1_src, const int32_t *c2_src,
                                const int32_t *key_src, const sqz_index &local, void *Kp_loc,
                                void *Vp_loc, cudaStream_t st) {
    const size_t esz = full.dtype == SQZ_BF16 ? 2 : 4;
    const size_t row = esz * full.d;
    const int H = full.H;
    cudaError_t e = gather(full.C2, full.c2, local.C2, local.c2, c2_src, H, row, st);
    if (e == cudaSuccess && full.levels == 2)
        e = gather(full.C1, full.c1, local.C1, local.c1, c1_src, H, row, st);
    if (e == cudaSuccess) e = gather(Kp, full.L, Kp_loc, local.L, key_src, H, row, st);
    if (e == cudaSuccess) e = gather(Vp, full.L, Vp_loc, local.L, key_src, H, row, st);
    if (e == cudaSuccess && full.perm && local.perm) {
        dim3 g((unsigned)std::min<int64_t>(4096, (local.L + 255) / 256), H);
        k_gather_perm<<<g, 256, 0, st>>>(full.perm, full.L, local.perm, local.L, key_src);
        e = cudaGetLastError();
    }
    return e;
}

}  // namespace sqz
