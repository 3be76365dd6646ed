// (1) Does a SWIZZLE_128B TMA box written at a smem row offset that is not a
//     multiple of 8 rows land in the address-based swizzle (chunk ^ (row % 8))?
// (2) L2-resident throughput: cp.async 64 thr vs TMA boxes of 8/16/32 rows.
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

__global__ void kalign(const CUtensorMap *mp, int row_off, int src_row, int nrows, uint16_t *out) {
    __shared__ __align__(1024) unsigned char sm[16384];
    __shared__ uint64_t bar;
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) sm[i] = 0xEE;
    __syncthreads();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar, nrows * 128);
        tma_load_2d(smem_u32(sm) + row_off * 128, mp, 0, src_row, &bar);
    }
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) out[i] = reinterpret_cast<uint16_t *>(sm)[i];
}

struct Maps { CUtensorMap m[6]; };  // box rows 1,2,4,8,16,32
constexpr int NTILE = 256;
__global__ void __launch_bounds__(128, 1) kthru(const __nv_bfloat16 *src, const int *rows, int mode, int br, int nrows_src, const __grid_constant__ Maps maps, int *sink) {
    extern __shared__ unsigned char smraw[];
    unsigned char *sm = (unsigned char *)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = (uint64_t *)(sm + 4 * 16384);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) { for (int s = 0; s < 4; ++s) mbar_init(&full[s], mode == 0 ? 64 : 1); mbar_fence_init(); }
    __syncthreads();
    const int *rw = rows + (size_t)blockIdx.x * NTILE * 64;
    const uint32_t base = smem_u32(sm);
    int lg = 0; while ((1 << lg) < br) ++lg;
    for (int t = 0; t < NTILE; ++t) {
        const int st = t & 3;
        if (t >= 4) mbar_wait(&full[st], ((t >> 2) - 1) & 1);
        __syncthreads();
        const uint32_t dst = base + st * 16384;   // 64 rows x 256 B
        if (mode == 0) {
            if (tid < 64) {
                for (int j = 0; j < 16; ++j) {
                    const int row = 2 * ((tid >> 5) + 2 * j) + ((tid & 31) >> 4), c = tid & 15;
                    const __nv_bfloat16 *s = src + (size_t)rw[t * 64 + row] * 128 + c * 8;
                    cp_async16_zfill(dst + (c >> 3) * 8192 + sw128_off(row, c & 7), s, true);
                }
                cp_async_mbar_arrive(&full[st]);
            }
        } else if (warp == 0) {
            if (lane == 0) mbar_arrive_expect_tx(&full[st], 16384);
            __syncwarp();
            const int nb = 64 / br;  // boxes per half
            for (int b = lane; b < 2 * nb; b += 32) {
                const int hf = b / nb, bi = b % nb;
                tma_load_2d(dst + hf * 8192 + bi * br * 128, &maps.m[lg], hf * 64, rw[t * 64 + bi * br], &full[st]);
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
    // ---- (1) alignment semantics ----
    const int NR = 1024;
    std::vector<uint16_t> h(NR * 128);
    for (int r = 0; r < NR; ++r) for (int k = 0; k < 128; ++k) h[r * 128 + k] = (uint16_t)(r * 128 + k);
    uint16_t *d, *out; cudaMalloc(&d, h.size() * 2); cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    cudaMalloc(&out, 16384);
    for (int br : {8, 32}) {
        CUtensorMap m = mk(d, NR, br), *dm; cudaMalloc(&dm, sizeof(m)); cudaMemcpy(dm, &m, sizeof(m), cudaMemcpyHostToDevice);
        for (int off : {0, 3, 8, 13}) {
            kalign<<<1, 128>>>(dm, off, 100, br, out);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<uint16_t> o(8192); cudaMemcpy(o.data(), out, 16384, cudaMemcpyDeviceToHost);
            int bad_abs = 0, bad_rel = 0;
            for (int r = 0; r < br; ++r) for (int c = 0; c < 8; ++c) for (int e2 = 0; e2 < 8; ++e2) {
                const int R = off + r;  // absolute smem row
                const uint16_t want = (uint16_t)((100 + r) * 128 + c * 8 + e2);
                if (o[R * 64 + ((c ^ (R & 7)) * 8) + e2] != want) ++bad_abs;
                if (o[R * 64 + ((c ^ (r & 7)) * 8) + e2] != want) ++bad_rel;
            }
            printf("box %2d rows at row offset %2d: %s  mismatches vs address-swizzle %d, vs box-relative swizzle %d\n",
                   br, off, e ? cudaGetErrorString(e) : "ok", bad_abs, bad_rel);
            if (e) return 1;
        }
    }
    // ---- (2) throughput from L2 (64 MB source) ----
    const int G = 148; const uint64_t NS = 1 << 18;  // 256K rows x 256 B = 64 MB
    __nv_bfloat16 *src; int *rows, *sink;
    cudaMalloc(&src, NS * 256); cudaMemset(src, 0, NS * 256); cudaMalloc(&sink, G * 4);
    std::vector<int> hr((size_t)G * NTILE * 64);
    std::mt19937 rng(1);
    for (size_t i = 0; i < hr.size(); i += 32) { int r0 = (int)(rng() % (NS - 64)); for (int j = 0; j < 32; ++j) hr[i + j] = r0 + j; }
    cudaMalloc(&rows, hr.size() * 4); cudaMemcpy(rows, hr.data(), hr.size() * 4, cudaMemcpyHostToDevice);
    Maps maps; for (int i = 0; i < 6; ++i) maps.m[i] = mk(src, NS, 1u << i);
    cudaFuncSetAttribute(kthru, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384 + 2048);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    struct { int mode, br; const char *name; } cfgs[] = {{0, 1, "cp.async 64 thr"}, {1, 1, "TMA box 1"}, {1, 4, "TMA box 4"}, {1, 8, "TMA box 8"}, {1, 16, "TMA box 16"}, {1, 32, "TMA box 32"}};
    for (auto c : cfgs) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            kthru<<<G, 128, 4 * 16384 + 2048>>>(src, rows, c.mode, c.br, NS, maps, sink);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (rep == 2) printf("L2 %-18s %8.1f us  %6.1f GB/s/SM  %s\n", c.name, ms * 1e3, (double)NTILE * 16384 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
