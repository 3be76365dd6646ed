// Microbenchmark: ways to gather 128 rows x 256 B (a K tile) into swizzled smem,
// 148 CTAs, each loading NT tiles into a 2-stage ring (no consumer compute).
//   mode 0: cp.async 16 B by 64 threads (2 warps), random rows
//   mode 1: TMA tile::gather4 (box {64,1}), random rows, 1 warp issuing
//   mode 2: TMA 2-D boxes of R rows (R = 32) at random starts (runs), 1 warp
//   mode 3: TMA 2-D boxes of 128 rows (contiguous tile)
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

struct Maps { CUtensorMap g4, r32, r128; };
constexpr int NTILE = 64;

__global__ void __launch_bounds__(128, 1) kbench(const __nv_bfloat16 *src, const int *rows, int mode, const __grid_constant__ Maps maps, int *sink) {
    extern __shared__ unsigned char smraw[];
    unsigned char *sm = (unsigned char *)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = (uint64_t *)(sm + 4 * 32768);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) { for (int s = 0; s < 4; ++s) mbar_init(&full[s], mode == 0 ? 64 : 1); mbar_fence_init(); }
    __syncthreads();
    const int *rw = rows + (size_t)blockIdx.x * NTILE * 128;
    const uint32_t base = smem_u32(sm);
    for (int t = 0; t < NTILE; ++t) {
        const int st = t & 3;
        if (t >= 4) mbar_wait(&full[st], ((t >> 2) - 1) & 1);  // "consume" stage t-4
        __syncthreads();
        const uint32_t dst = base + st * 32768;
        if (mode == 0) {
            if (tid < 64) {
                for (int j = 0; j < 32; ++j) {
                    const int row = 2 * ((tid >> 5) + 2 * j) + ((tid & 31) >> 4), c = tid & 15;
                    const __nv_bfloat16 *s = src + (size_t)rw[t * 128 + row] * 128 + c * 8;
                    cp_async16_zfill(dst + (c >> 3) * 16384 + sw128_off(row, c & 7), s, true);
                }
                cp_async_mbar_arrive(&full[st]);
            }
        } else if (warp == 0) {
            if (lane == 0) mbar_arrive_expect_tx(&full[st], 32768);
            __syncwarp();
            if (mode == 1) {
                const int *r = rw + t * 128 + 4 * lane;
                for (int hf = 0; hf < 2; ++hf)
                    tma_gather4(dst + hf * 16384 + lane * 512, &maps.g4, hf * 64, r[0], r[1], r[2], r[3], &full[st]);
            } else if (mode == 2) {
                if (lane < 4) {
                    const int r0 = rw[t * 128 + 32 * lane];
                    for (int hf = 0; hf < 2; ++hf)
                        tma_load_2d(dst + hf * 16384 + lane * 32 * 128, &maps.r32, hf * 64, r0, &full[st]);
                }
            } else {
                if (lane == 0) {
                    const int r0 = rw[t * 128];
                    for (int hf = 0; hf < 2; ++hf)
                        tma_load_2d(dst + hf * 16384, &maps.r128, hf * 64, r0, &full[st]);
                }
            }
        }
    }
    for (int t = NTILE - 4; t < NTILE; ++t) mbar_wait(&full[t & 3], (t >> 2) & 1);
    if (tid == 0) sink[blockIdx.x] = sm[5];
}

static CUtensorMap mk(const void *p, uint64_t rows, uint32_t br) {
    CUtensorMap m;
    cuuint64_t dims[2] = {128, rows}; cuuint64_t str[1] = {256}; cuuint32_t box[2] = {64, br}, es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void *)p, dims, str, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", r);
    return m;
}

int main() {
    const int G = 148; const uint64_t NR = 1 << 22;  // 4M rows x 256 B = 1 GB (no L2 reuse)
    __nv_bfloat16 *src; int *rows, *sink;
    cudaMalloc(&src, NR * 256); cudaMemset(src, 0, NR * 256);
    cudaMalloc(&sink, G * 4);
    std::vector<int> hr((size_t)G * NTILE * 128);
    std::mt19937 rng(1);
    for (auto &p : std::vector<int>(1)) (void)p;
    cudaMalloc(&rows, hr.size() * 4);
    Maps maps{mk(src, NR, 1), mk(src, NR, 32), mk(src, NR, 128)};
    cudaFuncSetAttribute(kbench, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768 + 2048);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char *names[4] = {"cp.async 16B x64thr, random rows", "TMA gather4, random rows", "TMA box 32 rows (runs)", "TMA box 128 rows"};
    for (int pattern = 0; pattern < 2; ++pattern) {
        // pattern 0: random rows (each 32-row run random start for mode 2); pattern 1: runs of 32 contiguous rows
        for (size_t i = 0; i < hr.size(); i += 32) {
            int r0 = (int)(rng() % (NR - 256));
            for (int j = 0; j < 32; ++j) hr[i + j] = pattern ? r0 + j : (int)(rng() % NR);
        }
        for (size_t i = 0; i < hr.size(); i += 128) {  // mode 3 needs the tile's first row
            (void)i;
        }
        cudaMemcpy(rows, hr.data(), hr.size() * 4, cudaMemcpyHostToDevice);
        for (int mode = 0; mode < 4; ++mode) {
            if (pattern == 0 && mode >= 2) continue;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(e0);
                kbench<<<G, 128, 4 * 32768 + 2048>>>(src, rows, mode, maps, sink);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                cudaError_t err = cudaGetLastError();
                if (rep == 2) printf("pattern %s mode %d %-36s %8.1f us  %7.1f GB/s total  %5.1f GB/s/SM %s\n",
                    pattern ? "runs32" : "random", mode, names[mode], ms * 1e3, (double)G * NTILE * 32768 / (ms * 1e-3) / 1e9,
                    (double)NTILE * 32768 / (ms * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
            }
        }
    }
    return 0;
}
