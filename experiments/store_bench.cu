// Microbenchmark: the lookup's range-expansion store pattern (warp per range of
// ~20 consecutive int32 at arbitrary offsets) vs sector-aligned stores, with the
// destination cold (after a 512 MB L2 flush) or warm.  Build+run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sb experiments/store_bench.cu && /tmp/sb
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <random>

// ranges: st[j], n[j], kp[j] for j < R per CTA (contiguous output kp)
__global__ void k_ranges(const int *st, const int *n, const int *kp, int R, int *out, int mode) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int base = blockIdx.x * R;
    __shared__ int s_st[2048], s_n[2048], s_kp[2048];
    if (mode == 0 || mode == 2) {  // warp per range, range table staged in smem first
        for (int j = threadIdx.x; j < R; j += blockDim.x) {
            s_st[j] = st[base + j]; s_n[j] = n[base + j]; s_kp[j] = kp[base + j];
        }
        __syncthreads();
        for (int j = warp; j < R; j += blockDim.x / 32) {
            const int s = s_st[j], c = s_n[j], k = s_kp[j];
            if (mode == 0)
                for (int t = lane; t < c; t += 32) out[k + t] = s + t;
            else
                for (int t = lane; t < c; t += 32) __stcs(out + k + t, s + t);
        }
    } else {  // thread per output element, contiguous: out[k0 + e] = e (same bytes, aligned)
        const int k0 = kp[base], k1 = kp[base + R - 1] + n[base + R - 1];
        for (int e = k0 + threadIdx.x; e < k1; e += blockDim.x) out[e] = e;
    }
}

int main() {
    const int CTAS = 256, R = 340;  // ~ cfg5 L2: 16 CTAs x 32 heads, ~340 selected ranges each
    std::mt19937 rng(1);
    std::vector<int> st(CTAS * R), n(CTAS * R), kp(CTAS * R);
    long k = 0;
    for (int i = 0; i < CTAS * R; ++i) {
        n[i] = 1 + rng() % 40;
        st[i] = rng() % 1000000;
        kp[i] = (int)k;
        k += n[i];
    }
    int *dst, *dn, *dkp, *out;
    char *flush;
    cudaMalloc(&dst, 4 * st.size()); cudaMalloc(&dn, 4 * n.size()); cudaMalloc(&dkp, 4 * kp.size());
    cudaMalloc(&out, 4 * (k + 64)); cudaMalloc(&flush, 512 << 20);
    cudaMemcpy(dst, st.data(), 4 * st.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dn, n.data(), 4 * n.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dkp, kp.data(), 4 * kp.size(), cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 3; ++mode)
        for (int cold = 0; cold < 2; ++cold) {
            float best = 1e9;
            for (int it = 0; it < 10; ++it) {
                if (cold) cudaMemsetAsync(flush, it, 512 << 20);
                else k_ranges<<<CTAS, 256>>>(dst, dn, dkp, R, out, mode);
                cudaEventRecord(a);
                k_ranges<<<CTAS, 256>>>(dst, dn, dkp, R, out, mode);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf("mode %s dest %s: %.2f us for %ld ints (%.1f GB/s)\n", mode == 1 ? "aligned-contiguous" : mode == 2 ? "warp-per-range .cs" : "warp-per-range",
                   cold ? "cold(flushed)" : "warm", best * 1e3, k, 4.0 * k / (best * 1e-3) / 1e9);
        }
    // single CTA, as in the prefill finalize
    for (int mode = 0; mode < 3; ++mode) {
        float best = 1e9;
        for (int it = 0; it < 10; ++it) {
            cudaMemsetAsync(flush, it, 512 << 20);
            cudaEventRecord(a);
            k_ranges<<<1, 256>>>(dst, dn, dkp, R * 4, out, mode);  // R*4 <= 2048
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("1 CTA, %d ranges, mode %d, cold: %.2f us\n", R * 4, mode, best * 1e3);
    }
    return 0;
}
