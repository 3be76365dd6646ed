// tcgen05.mma issue/execution rate per SM for kind::f16 (bf16 -> f32), M = 128,
// cta_group::1, N in {64, 128, 256}, A from SMEM (SS) or TMEM (TS); one thread
// issues NI MMAs back to back (accumulating into one TMEM tile), 148 CTAs.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2411_09688_b200/csrc/tma.cuh"
#include "../paper_2411_09688_b200/csrc/tcgen05.cuh"
using namespace sqz;
constexpr int NI = 4096;

template <int N, bool TS, int UNROLL>
__global__ void __launch_bounds__(128, 1) krate(int *sink, long long *cyc) {
    extern __shared__ unsigned char smraw[];
    unsigned char *sm = (unsigned char *)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t taddr;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 65536; i += blockDim.x) sm[i] = 0;
    if (warp == 0) tmem_alloc(&taddr, 512);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = taddr;
    constexpr uint32_t idesc = idesc_bf16(128, N, false);
    long long t0 = clock64();
    if (warp == 0) {
        const uint64_t ad = sdesc_sw128(smem_u32(sm), 16, 1024), bd = sdesc_sw128(smem_u32(sm) + 32768, 16, 1024);
        for (int i = 0; i < NI; i += UNROLL) {
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                if (TS) umma_bf16_ts_w(tm, tm + 256, bd + 2 * (u & 3), idesc, 1);
                else umma_bf16_w(tm, ad + 2 * (u & 3), bd + 2 * (u & 3), idesc, 1);
            }
        }
        umma_commit_w(&bar);
        mbar_wait(&bar, 0);
    }
    long long t1 = clock64();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(tm, 512);
    if (threadIdx.x == 0) { sink[blockIdx.x] = 1; cyc[blockIdx.x] = t1 - t0; }
}

template <int N, bool TS>
void run(const char *nm) {
    int *sink; long long *cyc; cudaMalloc(&sink, 148 * 4); cudaMalloc(&cyc, 148 * 8);
    auto k = krate<N, TS, 8>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k<<<148, 128, 65536 + 1024>>>(sink, cyc);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        long long hc[148]; cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
        const double flops = 2.0 * 128 * N * 16 * NI * 148;
        if (rep == 2) printf("%-10s N=%3d: %.1f us, %.1f clk/MMA (SM clock), %.0f TFLOP/s  %s\n", nm, N, ms * 1e3,
                             (double)hc[0] / NI, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
}
int main() {
    run<64, false>("SS"); run<128, false>("SS"); run<256, false>("SS");
    run<64, true>("TS"); run<128, true>("TS"); run<256, true>("TS");
    return 0;
}
