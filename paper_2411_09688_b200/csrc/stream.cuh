// stream.cuh -- KV-row streaming helpers shared by the decode attention kernels
// (attention.cu, decode_step.cu): non-allocating 16-byte row loads kept packed
// until use, their fp32 widening, and the grouped transposed butterfly that
// reduces the partial dot products of the keys a warp holds.
#pragma once
#include "common.cuh"

namespace sqz {

#ifndef SQZ_ATT_L2PF  // L2::256B prefetch hint on the K/V row loads (tuning knob)
#define SQZ_ATT_L2PF 0
#endif
#ifndef SQZ_ATT_KR_BF16
#define SQZ_ATT_KR_BF16 16
#endif
// keys per warp round (bf16 rows: tuning knob; fp32 rows take twice the registers)
template <typename T> constexpr int keys_per_round() { return sizeof(T) == 2 ? SQZ_ATT_KR_BF16 : 16; }
template <typename T> struct Raw { uint4 v[sizeof(T) == 2 ? 1 : 2]; };
__device__ __forceinline__ uint4 ld_nc_v4(const void *p) {
    uint4 u;
#if SQZ_ATT_L2PF
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
                 : "l"(p));
#else
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
                 : "l"(p));
#endif
    return u;
}
template <typename T> __device__ __forceinline__ void ld_raw(Raw<T> &r, const T *p) {
#pragma unroll
    for (int i = 0; i < (int)(sizeof(r.v) / sizeof(uint4)); ++i)
        r.v[i] = ld_nc_v4(reinterpret_cast<const uint4 *>(p) + i);
}
__device__ __forceinline__ void cvt(const Raw<__nv_bfloat16> &r, float (&f)[8]) {
    const uint32_t w[4] = {r.v[0].x, r.v[0].y, r.v[0].z, r.v[0].w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
}
__device__ __forceinline__ void cvt(const Raw<float> &r, float (&f)[8]) {
    f[0] = __uint_as_float(r.v[0].x); f[1] = __uint_as_float(r.v[0].y);
    f[2] = __uint_as_float(r.v[0].z); f[3] = __uint_as_float(r.v[0].w);
    f[4] = __uint_as_float(r.v[1].x); f[5] = __uint_as_float(r.v[1].y);
    f[6] = __uint_as_float(r.v[1].z); f[7] = __uint_as_float(r.v[1].w);
}

// NV values per lane, reduced over aligned groups of G lanes; lane ends with
// the group sum of value index (sub >> (log2 G - log2 NV)) & (NV - 1).
template <int NV, int G>
__device__ __forceinline__ float group_transpose_reduce(float (&v)[NV], int lane) {
    int stride = G / 2;
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

}  // namespace sqz
