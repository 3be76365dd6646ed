// Microbenchmark: the decode lookup's scan pattern alone -- each warp loads U
// centroid rows (256 B, 8 B per lane) per batch, dot products with one query,
// 8 warps per CTA, 2 CTAs/SM -- over an 89 MB table (cfg5 Level 1).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/scb experiments/scan_bench.cu && /tmp/scb
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
template <int U, int CLUSTER>
__global__ void __launch_bounds__(256, 2) kscan(const uint2 *C, long rows_per_cta, float *out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long r0 = blockIdx.x * rows_per_cta;
    float acc = 0.f;
    for (long rr = warp * U; rr < rows_per_cta; rr += 8 * U) {
        uint2 raw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) raw[u] = __ldg(C + (r0 + rr + u) * 32 + lane);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += __uint_as_float(raw[u].x << 16) * __uint_as_float(raw[u].y & 0xffff0000u);
    }
    if (acc == 1234.5f) out[0] = acc;
}
// 16-byte loads: lanes 0-15 read row 2m, lanes 16-31 row 2m+1 (U rows per batch)
template <int U>
__global__ void __launch_bounds__(256, 2) kscan16(const uint4 *C, long rows_per_cta, float *out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long r0 = blockIdx.x * rows_per_cta;
    float acc = 0.f;
    for (long rr = warp * U; rr < rows_per_cta; rr += 8 * U) {
        uint4 raw[U / 2];
#pragma unroll
        for (int u = 0; u < U / 2; ++u) raw[u] = __ldg(C + (r0 + rr + 2 * u + (lane >> 4)) * 16 + (lane & 15));
#pragma unroll
        for (int u = 0; u < U / 2; ++u) acc += __uint_as_float(raw[u].x << 16) * __uint_as_float(raw[u].w & 0xffff0000u);
    }
    if (acc == 1234.5f) out[0] = acc;
}
int main() {
    const long rows = 10486L * 32;  // cfg5 Level 1: 89 MB
    uint2 *C;
    float *out;
    cudaMalloc(&C, rows * 256);
    cudaMalloc(&out, 4);
    cudaMemset(C, 0, rows * 256);
    char *flush;
    cudaMalloc(&flush, 512 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int ctas : {256, 296, 592}) {
        const long rpc = rows / ctas;
        for (int U : {16, 32, 64}) {
            float best = 1e9;
            for (int it = 0; it < 5; ++it) {
                cudaMemsetAsync(flush, it, 512 << 20);
                cudaEventRecord(a);
                if (U == 16) kscan<16, 1><<<ctas, 256>>>(C, rpc, out);
                else if (U == 32) kscan<32, 1><<<ctas, 256>>>(C, rpc, out);
                else kscan<64, 1><<<ctas, 256>>>(C, rpc, out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                best = ms < best ? ms : best;
            }
            printf("ctas %d U %d: %.1f us  %.2f TB/s\n", ctas, U, best * 1e3, rows * 256 / (best * 1e-3) / 1e12);
            best = 1e9;
            for (int it = 0; it < 5; ++it) {
                cudaMemsetAsync(flush, it, 512 << 20);
                cudaEventRecord(a);
                if (U == 16) kscan16<16><<<ctas, 256>>>((const uint4 *)C, rpc, out);
                else if (U == 32) kscan16<32><<<ctas, 256>>>((const uint4 *)C, rpc, out);
                else kscan16<64><<<ctas, 256>>>((const uint4 *)C, rpc, out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                best = ms < best ? ms : best;
            }
            printf("ctas %d U %d 16B: %.1f us  %.2f TB/s\n", ctas, U, best * 1e3, rows * 256 / (best * 1e-3) / 1e12);
        }
    }
    return 0;
}
