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

// ---- run-length selection streams (sqz_selection.key_pref) ------------------
// The selected keys of one (b,h) are the runs j < n: stream keys
// [pref[j], pref[j+1]) (pref[n] = nkf) at cluster-major positions
// key_off[cl[j]] + (k - pref[j]).
struct RunList {
    const int32_t *cl, *pref, *koff;
    int n, nkf;
};
// A warp's window of 64 consecutive runs [J, J + 64): lane m holds runs J + m
// and J + 32 + m (first stream key, cluster-major start); `end` is the first
// stream key past the window.  Locating a key is a 6-step shuffle search.
struct RunWin {
    int J, end;
    int p0, p1, s0, s1;
};
__device__ __forceinline__ void runwin_load(RunWin &w, const RunList &r, int J, int lane) {
    w.J = J;
    const int j0 = J + lane, j1 = J + 32 + lane;
    w.p0 = j0 < r.n ? ldcg(r.pref + j0) : 0x7fffffff;
    w.p1 = j1 < r.n ? ldcg(r.pref + j1) : 0x7fffffff;
    const int c0 = j0 < r.n ? ldcg(r.cl + j0) : 0, c1 = j1 < r.n ? ldcg(r.cl + j1) : 0;
    w.end = J + 64 < r.n ? ldcg(r.pref + J + 64) : r.nkf;
    w.s0 = j0 < r.n ? __ldg(r.koff + c0) : 0;
    w.s1 = j1 < r.n ? __ldg(r.koff + c1) : 0;
}
// run index (absolute) of stream key k < nkf, by binary search over the list
__device__ __forceinline__ int run_of(const RunList &r, int k) {
    int lo = 0, hi = r.n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (ldcg(r.pref + mid) <= k) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}
// make the window hold the runs of stream keys [kmin, kmax] (warp-uniform,
// kmin <= kmax < nkf; at most 64 runs apart)
__device__ __forceinline__ void runwin_cover(RunWin &w, const RunList &r, int kmin, int kmax, int lane) {
    int first = __shfl_sync(FULL, w.p0, 0);
    if (kmin >= first && kmax < w.end) return;
    // a warp advances by a fixed stride, so the next key usually lies just past the
    // window: try the following 64 runs (one round trip) before a full search
    if (w.end >= 0 && kmin >= w.end && w.J + 64 < r.n) {
        runwin_load(w, r, w.J + 64, lane);
        first = __shfl_sync(FULL, w.p0, 0);
        if (kmax < w.end) return;
    }
    int J;
    if (kmin >= first && kmin < w.end) {  // slide: the run of kmin is in the window
        const unsigned b0 = __ballot_sync(FULL, w.p0 <= kmin), b1 = __ballot_sync(FULL, w.p1 <= kmin);
        J = w.J + __popc(b0) + __popc(b1) - 1;
    } else {
        J = run_of(r, kmin);
    }
    runwin_load(w, r, J, lane);
}
// cluster-major position of stream key k (the window must cover k)
__device__ __forceinline__ int runwin_pos(const RunWin &w, int k) {
    int m = 0;  // last window slot with first key <= k
#pragma unroll
    for (int step = 32; step >= 1; step >>= 1) {
        const int cand = m + step;
        const int v0 = __shfl_sync(FULL, w.p0, cand & 31), v1 = __shfl_sync(FULL, w.p1, cand & 31);
        const int v = cand < 32 ? v0 : v1;
        if (cand < 64 && v <= k) m = cand;
    }
    const int q0 = __shfl_sync(FULL, w.p0, m & 31), q1 = __shfl_sync(FULL, w.p1, m & 31);
    const int t0 = __shfl_sync(FULL, w.s0, m & 31), t1 = __shfl_sync(FULL, w.s1, m & 31);
    return (m < 32 ? t0 : t1) + (k - (m < 32 ? q0 : q1));
}

// Ticket of a "last CTA finishes the job" reduction, taken by ONE thread after a
// block barrier: the acquire-release atomic publishes the CTA's earlier global
// writes (ordered before it by the barrier) and, for the last CTA, makes every
// other CTA's writes visible to the reads that follow the next barrier.
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(int *p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// spin (one thread) until *p >= v, acquiring what the releasing writers published
__device__ __forceinline__ void spin_until_geq(const int *p, int v) {
    while (ld_acquire(p) < v) __nanosleep(32);
}
__device__ __forceinline__ int ticket_acq_rel(int *p) {
    int t;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(p) : "memory");
    return t;
}

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
#define SQZ_TRACE_VAL(name, slot, val)                                                    \
    do {                                                                                  \
        const unsigned lin_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z); \
        if (threadIdx.x == 0 && lin_ < 2048) name[lin_ * 8 + (slot)] = (unsigned long long)(val); \
    } while (0)
#define SQZ_TRACE_EXPORT(name, fn)                                                        \
    extern "C" int fn(void *host, size_t bytes) {                                         \
        return (int)cudaMemcpyFromSymbol(host, name, bytes < sizeof(name) ? bytes : sizeof(name)); \
    }
#else
#define SQZ_TRACE_DECL(name)
#define SQZ_TRACE_AT(name, slot) do { } while (0)
#define SQZ_TRACE_VAL(name, slot, val) do { } while (0)
#define SQZ_TRACE_EXPORT(name, fn)
#endif
