// Microbenchmark for the cfg2 decode lookup (32 heads x 1024 centroid rows x
// 256 B = 8.4 MB): how fast can G CTAs of T threads scan the table after the
// bench's 512 MB write flush, and what do cluster barriers / DSMEM reads cost.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/scs experiments/scan_small.cu && /tmp/scs
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

// each warp loads U rows (8 B per lane) per batch, dots with q, writes logits
template <int U>
__global__ void kscan(const uint2 *C, int rows_per_cta, float *out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const long r0 = (long)blockIdx.x * rows_per_cta;
    for (int rr = warp * U; rr < rows_per_cta; rr += nw * U) {
        uint2 raw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) raw[u] = __ldg(C + (r0 + rr + u) * 32 + lane);
        float acc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            acc[u] = __uint_as_float(raw[u].x << 16) * 0.5f + __uint_as_float(raw[u].y & 0xffff0000u);
#pragma unroll
            for (int o = 16; o; o >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
        }
        if (lane < U) out[r0 + rr + lane] = acc[lane & (U - 1)];
    }
}
// TMA-style bulk copy of the CTA's rows into smem, then one pass
__global__ void kbulk(const uint2 *C, int rows_per_cta, float *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    const long r0 = (long)blockIdx.x * rows_per_cta;
    const unsigned bytes = rows_per_cta * 256;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(sm), mb = (unsigned)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(mb));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes));
        for (unsigned off = 0; off < bytes; off += 32768) {
            const unsigned n = bytes - off < 32768 ? bytes - off : 32768;
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(sb + off), "l"((const char *)(C + r0 * 32) + off), "r"(n), "r"(mb) : "memory");
        }
    }
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(mb));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const uint2 *S = reinterpret_cast<const uint2 *>(sm);
    for (int rr = warp; rr < rows_per_cta; rr += nw) {
        uint2 v = S[rr * 32 + lane];
        float a = __uint_as_float(v.x << 16) * 0.5f + __uint_as_float(v.y & 0xffff0000u);
#pragma unroll
        for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) out[r0 + rr] = a;
    }
}
// cost of NS cluster barriers (+ a DSMEM read each)
template <int NC>
__global__ void __cluster_dims__(NC, 1, 1) kbar(int ns, float *out) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ float v;
    if (threadIdx.x == 0) v = blockIdx.x;
    float acc = 0.f;
    for (int i = 0; i < ns; ++i) {
        cl.sync();
        if (threadIdx.x < NC) acc += *cl.map_shared_rank(&v, threadIdx.x);
    }
    cl.sync();
    if (acc == -1.f) out[0] = acc;
}
__global__ void kempty(float *out) { if (threadIdx.x == 1234567) out[0] = 1.f; }

int main() {
    const long rows = 32L * 1024;
    uint2 *C;
    float *out;
    cudaMalloc(&C, rows * 256);
    cudaMalloc(&out, rows * 4);
    cudaMemset(C, 0, rows * 256);
    char *flush;
    cudaMalloc(&flush, 512 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto launch, bool fl) {
        float best = 1e9, sum = 0;
        for (int it = 0; it < 12; ++it) {
            if (fl) cudaMemsetAsync(flush, it, 512 << 20);
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (it >= 2) { best = ms < best ? ms : best; sum += ms; }
        }
        return std::make_pair(best * 1e3f, sum / 10 * 1e3f);
    };
    auto e = timeit([&] { kempty<<<1, 32>>>(out); }, true);
    printf("empty kernel: best %.2f mean %.2f us\n", e.first, e.second);
    for (int g : {32, 64, 128, 256, 512}) {
        for (int t : {256, 512, 1024}) {
            const int rpc = rows / g;
            if (rpc < t / 32 * 16) continue;
            auto r = timeit([&] { kscan<16><<<g, t>>>(C, rpc, out); }, true);
            auto r2 = timeit([&] { kscan<16><<<g, t>>>(C, rpc, out); }, false);
            printf("LDG  ctas %4d thr %4d rows/cta %5d: flushed best %.2f mean %.2f | warm %.2f us\n", g, t, rpc,
                   r.first, r.second, r2.first);
        }
    }
    for (int g : {64, 128, 256}) {
        const int rpc = rows / g;
        const int smem = rpc * 256;
        cudaFuncSetAttribute(kbulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        auto r = timeit([&] { kbulk<<<g, 256, smem>>>(C, rpc, out); }, true);
        printf("BULK ctas %4d rows/cta %5d: flushed best %.2f mean %.2f us (err %s)\n", g, rpc, r.first, r.second,
               cudaGetErrorString(cudaGetLastError()));
    }
    for (int ns : {1, 2, 4, 16}) {
        auto r8 = timeit([&] { kbar<8><<<256, 256>>>(ns, out); }, false);
        auto r2 = timeit([&] { kbar<2><<<64, 512>>>(ns, out); }, false);
        printf("cluster barriers %2d: NC=8 x256 ctas %.2f us | NC=2 x64 ctas %.2f us\n", ns, r8.first, r2.first);
    }
    return 0;
}
