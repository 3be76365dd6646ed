// scan.cuh -- centroid-row scan helpers shared by the decode lookup kernels
// (lookup.cu, decode_step.cu): lane-slice row loads, the transposed butterfly
// that reduces 16 partial dot products per warp, and the (m, D) combine of
// Eq. 1's denominator.
#pragma once
#include "common.cuh"

namespace sqz {

// lane-slice loads: lane holds D/32 consecutive elements of a row.  `Raw` is the
// stored form (bf16 stays packed in registers until used, so a warp can keep
// twice as many rows in flight), `cvt` widens it to fp32 exactly.
template <typename T, int D> struct Lane;
template <> struct Lane<__nv_bfloat16, 128> {
    using Raw = uint2;
    static __device__ __forceinline__ Raw load_raw(const __nv_bfloat16 *row, int lane) {
        return __ldg(reinterpret_cast<const uint2 *>(row) + lane);
    }
    // a load the compiler keeps where it is written (not hoisted out of a loop)
    static __device__ __forceinline__ Raw load_raw_pinned(const __nv_bfloat16 *row, int lane) {
        Raw u;
        asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(u.x), "=r"(u.y)
                     : "l"(reinterpret_cast<const uint2 *>(row) + lane));
        return u;
    }
    static __device__ __forceinline__ void cvt(const Raw &u, float (&f)[4]) {
        f[0] = __uint_as_float(u.x << 16); f[1] = __uint_as_float(u.x & 0xffff0000u);
        f[2] = __uint_as_float(u.y << 16); f[3] = __uint_as_float(u.y & 0xffff0000u);
    }
    static __device__ __forceinline__ void load(const __nv_bfloat16 *row, int lane, float (&f)[4]) {
        cvt(load_raw(row, lane), f);
    }
};
template <> struct Lane<__nv_bfloat16, 64> {
    using Raw = uint32_t;
    static __device__ __forceinline__ Raw load_raw(const __nv_bfloat16 *row, int lane) {
        return __ldg(reinterpret_cast<const uint32_t *>(row) + lane);
    }
    static __device__ __forceinline__ Raw load_raw_pinned(const __nv_bfloat16 *row, int lane) {
        Raw u;
        asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(u)
                     : "l"(reinterpret_cast<const uint32_t *>(row) + lane));
        return u;
    }
    static __device__ __forceinline__ void cvt(const Raw &u, float (&f)[2]) {
        f[0] = __uint_as_float(u << 16); f[1] = __uint_as_float(u & 0xffff0000u);
    }
    static __device__ __forceinline__ void load(const __nv_bfloat16 *row, int lane, float (&f)[2]) {
        cvt(load_raw(row, lane), f);
    }
};
template <> struct Lane<float, 128> {
    using Raw = float4;
    static __device__ __forceinline__ Raw load_raw(const float *row, int lane) {
        return __ldg(reinterpret_cast<const float4 *>(row) + lane);
    }
    static __device__ __forceinline__ Raw load_raw_pinned(const float *row, int lane) {
        Raw u;
        asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(u.x), "=f"(u.y), "=f"(u.z), "=f"(u.w)
                     : "l"(reinterpret_cast<const float4 *>(row) + lane));
        return u;
    }
    static __device__ __forceinline__ void cvt(const Raw &u, float (&f)[4]) {
        f[0] = u.x; f[1] = u.y; f[2] = u.z; f[3] = u.w;
    }
    static __device__ __forceinline__ void load(const float *row, int lane, float (&f)[4]) {
        cvt(load_raw(row, lane), f);
    }
};
template <> struct Lane<float, 64> {
    using Raw = float2;
    static __device__ __forceinline__ Raw load_raw(const float *row, int lane) {
        return __ldg(reinterpret_cast<const float2 *>(row) + lane);
    }
    static __device__ __forceinline__ Raw load_raw_pinned(const float *row, int lane) {
        Raw u;
        asm volatile("ld.global.nc.v2.f32 {%0,%1}, [%2];" : "=f"(u.x), "=f"(u.y)
                     : "l"(reinterpret_cast<const float2 *>(row) + lane));
        return u;
    }
    static __device__ __forceinline__ void cvt(const Raw &u, float (&f)[2]) {
        f[0] = u.x; f[1] = u.y;
    }
    static __device__ __forceinline__ void load(const float *row, int lane, float (&f)[2]) {
        cvt(load_raw(row, lane), f);
    }
};

// Transposed butterfly: NV per-lane partial dot products -> each lane ends
// with the full 32-lane sum of value index (lane >> (5 - log2 NV)) & (NV-1).
template <int NV>
__device__ __forceinline__ float transpose_reduce(float (&v)[NV], int lane) {
    int stride = 16;
#pragma unroll
    for (int w = NV; w > 1; w >>= 1) {
        const bool hi = lane & stride;
#pragma unroll
        for (int k = 0; k < w / 2; ++k) {
            float keep = hi ? v[k + w / 2] : v[k];
            float send = hi ? v[k] : v[k + w / 2];
            v[k] = keep + __shfl_xor_sync(FULL, send, stride);
        }
        stride >>= 1;
    }
#pragma unroll
    for (; stride >= 1; stride >>= 1) v[0] += __shfl_xor_sync(FULL, v[0], stride);
    return v[0];
}
template <int NV> __device__ __forceinline__ int transpose_index(int lane) {
    static_assert(NV == 1 || NV == 2 || NV == 4 || NV == 8 || NV == 16, "NV");
    constexpr int lg = NV == 1 ? 0 : NV == 2 ? 1 : NV == 4 ? 2 : NV == 8 ? 3 : 4;
    return (lane >> (5 - lg)) & (NV - 1);
}

// (m, D) online combine with N weights: D = sum N_j exp(s_j - m)
__device__ __forceinline__ void md_combine(float &m, float &D, float m2, float D2) {
    float mn = fmaxf(m, m2);
    if (mn == -INFINITY) return;
    D = D * expf(m - mn) + D2 * expf(m2 - mn);
    m = mn;
}
// the same with ex2.approx (relative error ~2e-7, far inside the 1e-5 band)
__device__ __forceinline__ void md_combine_fast(float &m, float &D, float m2, float D2) {
    float mn = fmaxf(m, m2);
    if (mn == -INFINITY) return;
    D = D * exp_fast(m - mn) + D2 * exp_fast(m2 - mn);
    m = mn;
}


}  // namespace sqz
