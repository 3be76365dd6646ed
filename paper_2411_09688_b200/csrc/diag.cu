// diag.cu -- selection diagnostics on the GPU (
// sqz_selection_diagnostics in include/sqz.h).
//
// App. A: the "cumulative attention scores for the top 1% highest
// scoring attention values" of each head -- the softmax over ALL fixed keys,
// a_j = exp(z_j - LSE) with z_j = scale q.k_j, summed over its n_top largest
// entries.  App. D: the "Ideal" lookup computes "attention from the
// ... query tokens to all of the fixed context keys" and keeps "the keys whose
// attention scores are above the configured threshold"; it is compared with
// the centroid selection at matched budget (the k largest a_j, k = the
// selection's key count): index-set recall, retrieved attention mass.
//
// Three launches per call, none on the online path:
//   k_diag_flags   per (b,h): a bitmap of the selected finest-level clusters;
//   k_diag_logits  per key position: z_j (fp32 dot product over bf16/fp32
//                  inputs, the logits attention uses) and its selected flag
//                  (cluster of the position by binary search in key_off);
//   k_diag_row     per (b,h), one 1024-thread CTA: LSE, then two exact radix
//                  selects (4 passes of 8 bits over the order-preserving
//                  uint32 image of z) for the n_top-th and k-th largest
//                  logits, then one pass that sums the masses and counts the
//                  overlap.  Ties at a select boundary are resolved by count
//                  (the oracle breaks them by key index; for the mass sums the
//                  two agree, for the recall a tie of two fp32 logits is the
//                  only place they can differ).
// Deterministic: fixed per-thread strides and a fixed-order block reduction.
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace sqz {

namespace {
constexpr int DG_NT = 1024;

__device__ __forceinline__ uint32_t ord_key(float z) {  // order-preserving image
    const uint32_t b = __float_as_uint(z);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord_val(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__global__ void k_diag_flags(const int32_t *clusters, const int32_t *n_clusters, int c2, int words,
                             uint32_t *flags) {
    const int bh = blockIdx.x;
    uint32_t *f = flags + (size_t)bh * words;
    for (int w = threadIdx.x; w < words; w += blockDim.x) f[w] = 0u;
    __syncthreads();
    const int n = n_clusters[bh];
    const int32_t *cl = clusters + (size_t)bh * c2;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int i = cl[e];
        atomicOr(f + (i >> 5), 1u << (i & 31));
    }
}

template <typename T, int D>
__global__ void __launch_bounds__(256) k_diag_logits(const T *Q, const T *Kp, const int32_t *key_off,
                                                     const uint32_t *flags, int H, int c2, int words,
                                                     int64_t L, float scale, float *z, uint8_t *selm) {
    __shared__ float qs[D];
    const int bh = blockIdx.y, h = bh % H;
    for (int k = threadIdx.x; k < D; k += blockDim.x) qs[k] = to_f32(Q[(size_t)bh * D + k]);
    __syncthreads();
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= L) return;
    const T *kr = Kp + ((size_t)h * L + p) * D;
    float acc = 0.f;
#pragma unroll 4
    for (int k = 0; k < D; k += 8) {
        float f[8];
        load8(kr + k, f);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc = fmaf(qs[k + i], f[i], acc);
    }
    // cluster of position p: the last i with key_off[i] <= p
    const int32_t *ko = key_off + (size_t)h * (c2 + 1);
    int lo = 0, hi = c2 - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(ko + mid) <= p) lo = mid;
        else hi = mid - 1;
    }
    const uint32_t fw = __ldg(flags + (size_t)bh * words + (lo >> 5));
    z[(size_t)bh * L + p] = acc * scale;
    selm[(size_t)bh * L + p] = (fw >> (lo & 31)) & 1u;
}

// block-wide fixed-order sums (double accumulators for the masses)
__device__ __forceinline__ double block_sum_d(double v, double *red) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < DG_NT / 32; ++w) t += red[w];
    return t;
}

// exact k-th largest (1-based) of the row: returns its key, and the number of
// entries strictly greater in *gt
__device__ uint32_t radix_select(const float *zr, int64_t L, long long kth, long long *gt,
                                 unsigned *hist, long long *s_out) {
    uint32_t prefix = 0u, mask = 0u;
    long long want = kth, above = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0u;
        __syncthreads();
        for (int64_t p = threadIdx.x; p < L; p += blockDim.x) {
            const uint32_t u = ord_key(zr[p]);
            if ((u & mask) == prefix) atomicAdd(hist + ((u >> shift) & 255u), 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            long long cum = 0;
            int b = 255;
            for (; b > 0; --b) {
                if (cum + hist[b] >= want) break;
                cum += hist[b];
            }
            s_out[0] = b;
            s_out[1] = cum;
        }
        __syncthreads();
        const uint32_t b = (uint32_t)s_out[0];
        want -= s_out[1];
        above += s_out[1];
        prefix |= b << shift;
        mask |= 255u << shift;
        __syncthreads();
    }
    *gt = above;
    return prefix;
}

__global__ void __launch_bounds__(DG_NT) k_diag_row(const float *z, const uint8_t *selm,
                                                    const int32_t *n_keys, int64_t L, long long n_top,
                                                    float logT, int all_T, float *skew, float *mass_sel,
                                                    float *mass_ideal, float *recall, int32_t *n_T,
                                                    float *mass_T) {
    __shared__ unsigned hist[256];
    __shared__ double red[DG_NT / 32];
    __shared__ float redf[DG_NT / 32];
    __shared__ long long s_sel[2];
    const int bh = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float *zr = z + (size_t)bh * L;
    const uint8_t *sr = selm + (size_t)bh * L;
    // LSE over all L fixed keys
    float m = -INFINITY;
    for (int64_t p = tid; p < L; p += DG_NT) m = fmaxf(m, zr[p]);
    m = warp_max(m);
    if (lane == 0) redf[warp] = m;
    __syncthreads();
    m = -INFINITY;
    for (int w = 0; w < DG_NT / 32; ++w) m = fmaxf(m, redf[w]);
    double l = 0.0;
    for (int64_t p = tid; p < L; p += DG_NT) l += (double)expf(zr[p] - m);
    l = block_sum_d(l, red);
    const float lse = m + (float)log(l);
    const long long k = n_keys[bh];
    long long gt_n, gt_k = 0;
    const uint32_t un = radix_select(zr, L, n_top, &gt_n, hist, s_sel);
    uint32_t uk = 0xffffffffu;
    if (k > 0) uk = radix_select(zr, L, k, &gt_k, hist, s_sel);
    // one pass: masses above the boundaries, the selection's mass and overlap,
    // the ideal lookup at threshold T (log domain: z - LSE > log T, R19)
    double a_gn = 0.0, a_gk = 0.0, a_sel = 0.0, a_T = 0.0;
    double c_hit = 0.0, c_tie = 0.0, c_T = 0.0;
    for (int64_t p = tid; p < L; p += DG_NT) {
        const float zz = zr[p];
        const uint32_t u = ord_key(zz);
        const double a = (double)expf(zz - lse);
        const bool s = sr[p] != 0;
        if (u > un) a_gn += a;
        if (u > uk) a_gk += a;
        if (s) {
            a_sel += a;
            if (u > uk) c_hit += 1.0;
            else if (u == uk) c_tie += 1.0;
        }
        if (all_T || zz - lse > logT) {
            a_T += a;
            c_T += 1.0;
        }
    }
    a_gn = block_sum_d(a_gn, red);
    a_gk = block_sum_d(a_gk, red);
    a_sel = block_sum_d(a_sel, red);
    a_T = block_sum_d(a_T, red);
    c_hit = block_sum_d(c_hit, red);
    c_tie = block_sum_d(c_tie, red);
    c_T = block_sum_d(c_T, red);
    if (tid == 0) {
        skew[bh] = (float)(a_gn + (double)(n_top - gt_n) * (double)expf(ord_val(un) - lse));
        mass_sel[bh] = (float)a_sel;
        if (k > 0) {
            const double rest = (double)(k - gt_k);
            mass_ideal[bh] = (float)(a_gk + rest * (double)expf(ord_val(uk) - lse));
            recall[bh] = (float)((c_hit + fmin(c_tie, rest)) / (double)k);
        } else {
            mass_ideal[bh] = 0.f;
            recall[bh] = 1.f;
        }
        n_T[bh] = (int32_t)c_T;
        mass_T[bh] = (float)a_T;
    }
}
}  // namespace

size_t diag_ws_bytes(int B, int H, int c2, int64_t L) {
    const size_t BH = (size_t)B * H;
    const size_t words = ((size_t)c2 + 31) / 32;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    return al(BH * L * 4) + al(BH * L) + al(BH * words * 4) + 256;
}

cudaError_t launch_diagnostics(const DiagLaunch &a, cudaStream_t st) {
    const int BH = a.B * a.H;
    const int words = (a.c2 + 31) / 32;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    char *p = reinterpret_cast<char *>(((uintptr_t)a.ws + 255) & ~(uintptr_t)255);
    float *z = reinterpret_cast<float *>(p);
    p += al((size_t)BH * a.L * 4);
    uint8_t *selm = reinterpret_cast<uint8_t *>(p);
    p += al((size_t)BH * a.L);
    uint32_t *flags = reinterpret_cast<uint32_t *>(p);
    k_diag_flags<<<BH, 256, 0, st>>>(a.clusters, a.n_clusters, a.c2, words, flags);
    const dim3 g((unsigned)((a.L + 255) / 256), (unsigned)BH);
    if (a.dtype == SQZ_BF16) {
        auto Q = reinterpret_cast<const __nv_bfloat16 *>(a.Q);
        auto K = reinterpret_cast<const __nv_bfloat16 *>(a.Kp);
        if (a.d == 128)
            k_diag_logits<__nv_bfloat16, 128><<<g, 256, 0, st>>>(Q, K, a.key_off, flags, a.H, a.c2, words,
                                                                 a.L, a.scale, z, selm);
        else
            k_diag_logits<__nv_bfloat16, 64><<<g, 256, 0, st>>>(Q, K, a.key_off, flags, a.H, a.c2, words,
                                                                a.L, a.scale, z, selm);
    } else {
        auto Q = reinterpret_cast<const float *>(a.Q);
        auto K = reinterpret_cast<const float *>(a.Kp);
        if (a.d == 128)
            k_diag_logits<float, 128><<<g, 256, 0, st>>>(Q, K, a.key_off, flags, a.H, a.c2, words, a.L,
                                                         a.scale, z, selm);
        else
            k_diag_logits<float, 64><<<g, 256, 0, st>>>(Q, K, a.key_off, flags, a.H, a.c2, words, a.L,
                                                        a.scale, z, selm);
    }
    const int all_T = !(a.T > 0.f);
    k_diag_row<<<BH, DG_NT, 0, st>>>(z, selm, a.n_keys, a.L, a.n_top, all_T ? 0.f : logf(a.T), all_T,
                                     a.skew, a.mass_sel, a.mass_ideal, a.recall, a.n_T, a.mass_T);
    return cudaGetLastError();
}

}  // namespace sqz
