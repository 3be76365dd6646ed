// Two 16 KB tile streams per CTA (like K and V), each with an NS-stage ring,
// source 64 MB (L2-resident after warm-up) or 1 GB (DRAM), runs of 32 rows:
//   mode 0: both streams by cp.async (64 threads each)
//   mode 1: stream A by cp.async, stream B by TMA boxes of 32 rows
//   mode 2: both by TMA boxes of 32 rows
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include "../paper_2411_09688_b200/csrc/tma.cuh"
#include "../paper_2411_09688_b200/csrc/tcgen05.cuh"
using namespace sqz;
constexpr int NTILE = 256, NS = 5;

__device__ void stream_cp(uint32_t ring, uint64_t *full, const __nv_bfloat16 *src, const int *rw, int lt) {
    for (int t = 0; t < NTILE; ++t) {
        const int st = t % NS;
        if (t >= NS) mbar_wait(&full[st], ((t / NS) - 1) & 1);
        const uint32_t dst = ring + st * 16384;
        for (int j = 0; j < 16; ++j) {
            const int row = 2 * ((lt >> 5) + 2 * j) + ((lt & 31) >> 4), c = lt & 15;
            cp_async16_zfill(dst + (c >> 3) * 8192 + sw128_off(row, c & 7), src + (size_t)rw[t * 64 + row] * 128 + c * 8, true);
        }
        cp_async_mbar_arrive(&full[st]);
    }
}
__device__ void stream_tma(uint32_t ring, uint64_t *full, const CUtensorMap *m, const int *rw, int lane) {
    for (int t = 0; t < NTILE; ++t) {
        const int st = t % NS;
        if (t >= NS) mbar_wait(&full[st], ((t / NS) - 1) & 1);
        if (lane == 0) mbar_arrive_expect_tx(&full[st], 16384);
        __syncwarp();
        if (lane < 4) tma_load_2d(ring + st * 16384 + (lane >> 1) * 8192 + (lane & 1) * 32 * 128, m, (lane >> 1) * 64, rw[t * 64 + (lane & 1) * 32], &full[st]);
        __syncwarp();
    }
}
__global__ void __launch_bounds__(128, 1) kmix(const __nv_bfloat16 *src, const int *rows, int mode, const __grid_constant__ CUtensorMap m32, int *sink) {
    extern __shared__ unsigned char smraw[];
    unsigned char *sm = (unsigned char *)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
    uint64_t *fa = (uint64_t *)(sm + 2 * NS * 16384), *fb = fa + NS;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool a_tma = mode == 2, b_tma = mode >= 1;
    if (tid == 0) { for (int s = 0; s < NS; ++s) { mbar_init(&fa[s], a_tma ? 1 : 64); mbar_init(&fb[s], b_tma ? 1 : 64); } mbar_fence_init(); }
    __syncthreads();
    const int *rw = rows + (size_t)blockIdx.x * NTILE * 64;
    const uint32_t base = smem_u32(sm);
    if (warp < 2) { if (a_tma) { if (warp == 0) stream_tma(base, fa, &m32, rw, lane); } else stream_cp(base, fa, src, rw, tid); }
    else { const int lt = tid - 64; if (b_tma) { if (warp == 2) stream_tma(base + NS * 16384, fb, &m32, rw + 32, lane); } else stream_cp(base + NS * 16384, fb, src, rw + 32, lt); }
    __syncthreads();
    for (int t = NTILE - NS; t < NTILE; ++t) { mbar_wait(&fa[t % NS], (t / NS) & 1); mbar_wait(&fb[t % NS], (t / NS) & 1); }
    if (tid == 0) sink[blockIdx.x] = sm[5];
}
static CUtensorMap mk(const void *p, uint64_t rows, uint32_t br) {
    CUtensorMap m;
    cuuint64_t dims[2] = {128, rows}; cuuint64_t str[1] = {256}; cuuint32_t box[2] = {64, br}, es[2] = {1, 1};
    if (cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void *)p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) printf("encode failed\n");
    return m;
}
int main() {
    const int G = 148;
    for (uint64_t NR : {(uint64_t)1 << 18, (uint64_t)1 << 22}) {
        __nv_bfloat16 *src; int *rows, *sink;
        cudaMalloc(&src, NR * 256); cudaMemset(src, 0, NR * 256); cudaMalloc(&sink, G * 4);
        std::vector<int> hr((size_t)G * NTILE * 64 + 64);
        std::mt19937 rng(1);
        for (size_t i = 0; i < hr.size(); i += 32) { int r0 = (int)(rng() % (NR - 64)); for (int j = 0; j < 32 && i + j < hr.size(); ++j) hr[i + j] = r0 + j; }
        cudaMalloc(&rows, hr.size() * 4); cudaMemcpy(rows, hr.data(), hr.size() * 4, cudaMemcpyHostToDevice);
        CUtensorMap m32 = mk(src, NR, 32);
        cudaFuncSetAttribute(kmix, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * NS * 16384 + 2048);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        const char *nm[3] = {"cp.async + cp.async", "cp.async + TMA box32", "TMA box32 + TMA box32"};
        for (int mode = 0; mode < 3; ++mode) {
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(e0);
                kmix<<<G, 128, 2 * NS * 16384 + 2048>>>(src, rows, mode, m32, sink);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                if (rep == 2) printf("%s %-24s %8.1f us  %6.1f GB/s/SM (both streams)  %s\n", NR < (1u << 20) ? "L2  " : "DRAM", nm[mode], ms * 1e3,
                                     2.0 * NTILE * 16384 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
            }
        }
        cudaFree(src); cudaFree(rows); cudaFree(sink);
    }
    return 0;
}
