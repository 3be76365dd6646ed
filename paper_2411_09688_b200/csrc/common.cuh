// common.cuh -- device helpers shared by the libsqz kernels (sm_100a only).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "../../include/sqz.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libsqz is built for sm_100a only"
#endif

namespace sqz {

constexpr unsigned FULL = 0xffffffffu;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

// ---- storage loads: 8 consecutive elements -> fp32 ------------------------
__device__ __forceinline__ void load8(const __nv_bfloat16 *p, float (&f)[8]) {
    uint4 u = __ldg(reinterpret_cast<const uint4 *>(p));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
}
__device__ __forceinline__ void load8(const float *p, float (&f)[8]) {
    float4 a = __ldg(reinterpret_cast<const float4 *>(p));
    float4 b = __ldg(reinterpret_cast<const float4 *>(p) + 1);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}
// streaming (no L1 allocate) variant for the KV stream
__device__ __forceinline__ void load8_stream(const __nv_bfloat16 *p, float (&f)[8]) {
    uint4 u;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
                 : "l"(p));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
}
__device__ __forceinline__ void load8_stream(const float *p, float (&f)[8]) { load8(p, f); }

__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ float to_f32(float x) { return x; }
template <typename T> __device__ __forceinline__ T from_f32(float x);
template <> __device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) {
    return __float2bfloat16_rn(x);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULL, v, o));
    return v;
}
__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// e^x as ex2.approx.ftz(x log2 e): one FMUL + one MUFU op (relative error ~2e-7
// for the O(1) arguments it is used on)
__device__ __forceinline__ float exp_fast(float x) { return fast_exp2(x * LOG2E); }

// ld.global that bypasses L1 (data written by other CTAs of this launch).
template <typename T> __device__ __forceinline__ T ldcg(const T *p) { return __ldcg(p); }

}  // namespace sqz

// ---- optional device-side timeline tracing (experiments only: -DSQZ_TRACE) ----
#ifdef SQZ_TRACE
#define SQZ_TRACE_DECL(name) __device__ unsigned long long name[2048 * 8];
#define SQZ_TRACE_AT(name, slot)                                                          \
    do {                                                                                  \
        const unsigned lin_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z); \
        if (threadIdx.x == 0 && lin_ < 2048) {                                            \
            unsigned long long t_;                                                        \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                       \
            name[lin_ * 8 + (slot)] = t_;                                                 \
        }                                                                                 \
    } while (0)
#define SQZ_TRACE_EXPORT(name, fn)                                                        \
    extern "C" int fn(void *host, size_t bytes) {                                         \
        return (int)cudaMemcpyFromSymbol(host, name, bytes < sizeof(name) ? bytes : sizeof(name)); \
    }
#else
#define SQZ_TRACE_DECL(name)
#define SQZ_TRACE_AT(name, slot) do { } while (0)
#define SQZ_TRACE_EXPORT(name, fn)
#endif
