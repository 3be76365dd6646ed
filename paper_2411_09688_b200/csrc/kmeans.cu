// kmeans.cu -- offline key clustering and index construction
// (section 3.1, section 3.3, Fig. 2).
//
// Lloyd's algorithm on unit-normalised keys, all heads at once:
//   k_normalize     x^ = x / ||x|| (fp32 working copy)
//   k_assign        a_j = argmin_i ||x^_j - mu_i||^2 (= argmin ||mu_i||^2 - 2 x^.mu_i),
//                   ties to the lowest i; 64x64 register-tiled FFMA
//   k_counts/k_repair  empty clusters take the farthest point (deterministic)
//   k_accumulate    member sums in 2^-32 fixed point with 64-bit integer atomics:
//                   exact and order-independent, so every build is bit-reproducible
//   k_update        mu = sum / count, max centroid shift per head
// One 8-byte-per-head readback per iteration decides convergence ("no
// assignment changed, or max shift < tol"), per head.
// Then C = mean of the RAW members, accumulated in fp64 over the members in
// increasing key index (the sum order of the definition, so the result is the
// oracle's bit for bit) and rounded once to the storage dtype (R2, R18); the
// Level-1 pass on the stored C2 rows (R5); the cluster-major reordering with
// stable radix sorts (CUB) and a K/V gather.
#include <cub/device/device_radix_sort.cuh>

#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace sqz {

constexpr double FIX_SCALE = 4294967296.0;  // 2^32

template <typename T>
__global__ void k_normalize(const T *__restrict__ X, int64_t n, int d, float *__restrict__ Xh) {
    // one warp per row
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const T *x = X + row * d;
    float ss = 0.f;
    for (int k = lane; k < d; k += 32) {
        const float v = to_f32(x[k]);
        ss = fmaf(v, v, ss);
    }
    ss = warp_sum(ss);
    const float inv = ss > 0.f ? 1.0f / sqrtf(ss) : 0.f;
    for (int k = lane; k < d; k += 32) Xh[row * d + k] = to_f32(x[k]) * inv;
}

__global__ void k_init(const float *__restrict__ Xh, const int64_t *__restrict__ init, int n, int c,
                       int d, float *__restrict__ mu) {
    const int i = blockIdx.x, h = blockIdx.y;
    const int64_t j = init[(size_t)h * c + i];
    for (int k = threadIdx.x; k < d; k += blockDim.x)
        mu[((size_t)h * c + i) * d + k] = Xh[((size_t)h * n + j) * d + k];
}

__global__ void k_musq(const float *__restrict__ mu, int c, int d, const int *__restrict__ done,
                       float *__restrict__ musq) {
    const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), h = blockIdx.y;
    const int lane = threadIdx.x & 31;
    if (i >= c || done[h]) return;
    const float *m = mu + ((size_t)h * c + i) * d;
    float s = 0.f;
    for (int k = lane; k < d; k += 32) s = fmaf(m[k], m[k], s);
    s = warp_sum(s);
    if (lane == 0) musq[(size_t)h * c + i] = s;
}

// 64 points x 64 centroids per tile, 256 threads, 4x4 register micro-tile.
constexpr int KT = 64;
__global__ void __launch_bounds__(256) k_assign(const float *__restrict__ Xh, int n, int c, int d,
                                                const float *__restrict__ mu,
                                                const float *__restrict__ musq,
                                                const int *__restrict__ done,
                                                int32_t *__restrict__ assign,
                                                float *__restrict__ pdist,
                                                int *__restrict__ changed) {
    extern __shared__ float sm[];
    const int h = blockIdx.y;
    if (done[h]) return;
    const int ld = d + 1;
    float *xs = sm;            // [64][d+1]
    float *ms = sm + KT * ld;  // [64][d+1]
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int p0 = blockIdx.x * KT;
    const float *X = Xh + (size_t)h * n * d;
    for (int e = tid; e < KT * d; e += 256) {
        const int p = e / d, k = e % d;
        xs[p * ld + k] = (p0 + p < n) ? X[(size_t)(p0 + p) * d + k] : 0.f;
    }
    float best[4];
    int bidx[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) { best[i] = INFINITY; bidx[i] = 0; }
    const float *M = mu + (size_t)h * c * d;
    const float *MS = musq + (size_t)h * c;
    for (int c0 = 0; c0 < c; c0 += KT) {
        __syncthreads();
        for (int e = tid; e < KT * d; e += 256) {
            const int i = e / d, k = e % d;
            ms[i * ld + k] = (c0 + i < c) ? M[(size_t)(c0 + i) * d + k] : 0.f;
        }
        __syncthreads();
        float acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
        for (int k = 0; k < d; ++k) {
            float xv[4], mv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) xv[a] = xs[(ty + 16 * a) * ld + k];
#pragma unroll
            for (int b = 0; b < 4; ++b) mv[b] = ms[(tx + 16 * b) * ld + k];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(xv[a], mv[b], acc[a][b]);
        }
        // centroids tx + 16b scanned in increasing id per thread
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int ci = c0 + tx + 16 * b;
            if (ci < c) {
                const float m2 = MS[ci];
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const float e = fmaf(-2.f, acc[a][b], m2);
                    if (e < best[a] || (e == best[a] && ci < bidx[a])) { best[a] = e; bidx[a] = ci; }
                }
            }
        }
    }
    // lexicographic (value, index) min over the 16 tx lanes
#pragma unroll
    for (int a = 0; a < 4; ++a) {
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(FULL, best[a], o);
            const int oi = __shfl_xor_sync(FULL, bidx[a], o);
            if (ov < best[a] || (ov == best[a] && oi < bidx[a])) { best[a] = ov; bidx[a] = oi; }
        }
    }
    if (tx == 0) {
        int ch = 0;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int p = p0 + ty + 16 * a;
            if (p < n) {
                float xx = 0.f;
                for (int k = 0; k < d; ++k) xx = fmaf(xs[(ty + 16 * a) * ld + k], xs[(ty + 16 * a) * ld + k], xx);
                int32_t *ap = assign + (size_t)h * n + p;
                if (*ap != bidx[a]) ++ch;
                *ap = bidx[a];
                pdist[(size_t)h * n + p] = fmaxf(xx + best[a], 0.f);
            }
        }
        if (ch) atomicAdd(changed + h, ch);
    }
}

__global__ void k_counts(const int32_t *__restrict__ assign, int n, int c,
                         const int *__restrict__ done, int *__restrict__ counts) {
    const int h = blockIdx.y;
    if (done[h]) return;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        atomicAdd(counts + (size_t)h * c + assign[(size_t)h * n + j], 1);
}

// Empty-cluster repair, one CTA per head: empty clusters in increasing id take
// the point farthest from its centroid among clusters with > 1 member (ties to
// the lowest point index).
__global__ void __launch_bounds__(1024) k_repair(int32_t *__restrict__ assign,
                                                 float *__restrict__ pdist, int n, int c,
                                                 const int *__restrict__ done,
                                                 int *__restrict__ counts,
                                                 int *__restrict__ changed) {
    const int h = blockIdx.x;
    if (done[h]) return;
    int *cnt = counts + (size_t)h * c;
    int32_t *A = assign + (size_t)h * n;
    float *P = pdist + (size_t)h * n;
    __shared__ float sv[32];
    __shared__ int si[32];
    __shared__ int s_any;
    if (threadIdx.x == 0) s_any = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < c; i += blockDim.x)
        if (cnt[i] == 0) s_any = 1;
    __syncthreads();
    if (!s_any) return;
    for (int i = 0; i < c; ++i) {
        if (threadIdx.x == 0) s_any = cnt[i] == 0;
        __syncthreads();
        if (!s_any) { __syncthreads(); continue; }
        float bv = -1.f;
        int bj = n;
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            if (cnt[A[j]] > 1 && P[j] > bv) { bv = P[j]; bj = j; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(FULL, bv, o);
            const int oj = __shfl_xor_sync(FULL, bj, o);
            if (ov > bv || (ov == bv && oj < bj)) { bv = ov; bj = oj; }
        }
        if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = bv; si[threadIdx.x >> 5] = bj; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < (int)(blockDim.x / 32); ++w)
                if (sv[w] > bv || (sv[w] == bv && si[w] < bj)) { bv = sv[w]; bj = si[w]; }
            if (bj < n) {
                cnt[A[bj]] -= 1;
                A[bj] = i;
                cnt[i] = 1;
                P[bj] = 0.f;
                changed[h] += 1;
            }
        }
        __syncthreads();
    }
}

template <typename T>
__global__ void k_accumulate(const T *__restrict__ X, const int32_t *__restrict__ assign, int n,
                             int c, int d, const int *__restrict__ done,
                             unsigned long long *__restrict__ sums) {
    const int h = blockIdx.y;
    if (done && done[h]) return;
    const int64_t total = (int64_t)n * d;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / d;
        const int k = (int)(e % d);
        const float v = to_f32(X[(size_t)h * total + e]);
        const long long q = __double2ll_rn((double)v * FIX_SCALE);
        atomicAdd(sums + ((size_t)h * c + assign[(size_t)h * n + j]) * d + k,
                  (unsigned long long)q);
    }
}

__global__ void k_update(const unsigned long long *__restrict__ sums, const int *__restrict__ counts,
                         int c, int d, const int *__restrict__ done, float *__restrict__ mu,
                         unsigned *__restrict__ shift) {
    const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), h = blockIdx.y;
    const int lane = threadIdx.x & 31;
    if (i >= c || done[h]) return;
    const int cn = counts[(size_t)h * c + i];
    float *m = mu + ((size_t)h * c + i) * d;
    float s2 = 0.f;
    for (int k = lane; k < d; k += 32) {
        if (cn > 0) {
            const long long q = (long long)sums[((size_t)h * c + i) * d + k];
            const float v = (float)((double)q / FIX_SCALE / (double)cn);
            const float t = v - m[k];
            s2 = fmaf(t, t, s2);
            m[k] = v;
        }
    }
    s2 = warp_sum(s2);
    if (lane == 0) atomicMax(shift + h, __float_as_uint(sqrtf(s2)));
}

// C[h][i] = round(mean of X[h][rows[h][pos]] for pos in [off[h][i], off[h][i+1])),
// accumulated in fp64 in list order (one warp per segment); N[h][i] = count.
template <typename T>
__global__ void k_segment_means(const T *__restrict__ X, int n, const int32_t *__restrict__ rows,
                                const int32_t *__restrict__ off, int c, int d, T *__restrict__ C,
                                int32_t *__restrict__ Nout) {
    const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), h = blockIdx.y;
    const int lane = threadIdx.x & 31;
    if (i >= c) return;
    const int32_t *o = off + (size_t)h * (c + 1);
    const int s = o[i], e = o[i + 1];
    const T *Xh = X + (size_t)h * n * d;
    const int32_t *R = rows + (size_t)h * n;
    for (int k0 = 0; k0 < d; k0 += 32) {
        const int k = k0 + lane;
        double acc = 0.0;
        for (int pos = s; pos < e; ++pos) acc += (double)to_f32(Xh[(size_t)R[pos] * d + k]);
        const double v = e > s ? acc / (double)(e - s) : 0.0;
        if constexpr (sizeof(T) == 2) C[((size_t)h * c + i) * d + k] = __double2bfloat16(v);
        else C[((size_t)h * c + i) * d + k] = (float)v;
    }
    if (lane == 0 && Nout) Nout[(size_t)h * c + i] = e - s;
}

__global__ void k_invert(const int32_t *__restrict__ order, int n, int32_t *__restrict__ inv) {
    const int h = blockIdx.y;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
        inv[(size_t)h * n + order[(size_t)h * n + p]] = p;
}

// key = h * kmul + keyfn, value = h * n + j
__global__ void k_make_keys(const int32_t *__restrict__ lab, const int32_t *__restrict__ remap,
                            int n, int kmul, int rmul, int32_t *__restrict__ keys,
                            int32_t *__restrict__ vals) {
    const int h = blockIdx.y;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        int l = lab[(size_t)h * n + j];
        if (remap) l = remap[(size_t)h * rmul + l];
        keys[(size_t)h * n + j] = h * kmul + l;
        vals[(size_t)h * n + j] = (int32_t)((size_t)h * n + j);
    }
}

__global__ void k_iota(int n, int32_t *__restrict__ a, int32_t *__restrict__ b) {
    const int h = blockIdx.y;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        a[(size_t)h * n + p] = p;
        b[(size_t)h * n + p] = p;
    }
}

// sorted values -> per-head position tables
__global__ void k_positions(const int32_t *__restrict__ sorted_vals, int n, int32_t *__restrict__ out_order,
                            int32_t *__restrict__ inv) {
    const int h = blockIdx.y;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const int v = sorted_vals[(size_t)h * n + p] - h * n;
        if (out_order) out_order[(size_t)h * n + p] = v;
        if (inv) inv[(size_t)h * n + v] = p;
    }
}

// offsets[h][0..m] = exclusive scan of cnt[h][0..m), one CTA per head
__global__ void k_exscan(const int32_t *__restrict__ cnt, int m, int32_t *__restrict__ off) {
    const int h = blockIdx.x;
    __shared__ int s_tot[33];
    __shared__ int s_run;
    if (threadIdx.x == 0) s_run = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int base = 0; base < m; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const int v = i < m ? cnt[(size_t)h * m + i] : 0;
        int inc = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) s_tot[warp] = inc;
        __syncthreads();
        int wb = 0;
        for (int w = 0; w < warp; ++w) wb += s_tot[w];
        if (i < m) off[(size_t)h * (m + 1) + i] = s_run + wb + inc - v;
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = 0;
            for (int w = 0; w < (int)(blockDim.x / 32); ++w) t += s_tot[w];
            s_run += t;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) off[(size_t)h * (m + 1) + m] = s_run;
}

// dst[h][new] = src[h][order[h][new]] for rows of `w` elements of type T
template <typename T>
__global__ void k_gather_rows(const T *__restrict__ src, const int32_t *__restrict__ order, int n,
                              int w, T *__restrict__ dst) {
    const int h = blockIdx.y;
    const int64_t total = (int64_t)n * w;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = e / w;
        const int k = (int)(e % w);
        dst[(size_t)h * total + e] = src[(size_t)h * total + (size_t)order[(size_t)h * n + p] * w + k];
    }
}

// 16-byte row gather for K/V (row = d elements)
__global__ void k_gather_kv(const uint4 *__restrict__ src, const int32_t *__restrict__ perm,
                            int64_t L, int vec_per_row, uint4 *__restrict__ dst) {
    const int h = blockIdx.y;
    const int64_t total = L * vec_per_row;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = e / vec_per_row;
        const int k = (int)(e % vec_per_row);
        dst[(size_t)h * total + e] = src[(size_t)h * total + (size_t)perm[(size_t)h * L + p] * vec_per_row + k];
    }
}

// N1[h][p] += N2[h][o] for parent[h][o] = p
__global__ void k_parent_weights(const int32_t *__restrict__ parent, const int32_t *__restrict__ N2,
                                 int c2, int c1, int32_t *__restrict__ N1) {
    const int h = blockIdx.y;
    for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < c2; o += gridDim.x * blockDim.x)
        atomicAdd(N1 + (size_t)h * c1 + parent[(size_t)h * c2 + o], N2[(size_t)h * c2 + o]);
}

// lab[h, j] <- map[h, lab[h, j]] (labels renumbered)
__global__ void k_remap(int32_t *__restrict__ lab, const int32_t *__restrict__ map, int n, int m) {
    const int h = blockIdx.y;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        lab[(size_t)h * n + j] = map[(size_t)h * m + lab[(size_t)h * n + j]];
}

// --------------------------------------------------------------------------
// host orchestration
// --------------------------------------------------------------------------
namespace {
struct Carve {
    char *p;
    size_t used = 0;
    template <typename X> X *take(size_t n) {
        used = (used + 255) & ~(size_t)255;
        X *r = reinterpret_cast<X *>(p ? p + used : nullptr);
        used += n * sizeof(X);
        return r;
    }
};

size_t cub_bytes(int64_t n) {
    size_t b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, (int32_t *)nullptr, (int32_t *)nullptr,
                                    (int32_t *)nullptr, (int32_t *)nullptr, (int)n, 0, 32);
    return b;
}

struct Ws {
    float *Xh, *mu, *musq, *pdist;
    int32_t *assign, *counts, *done, *changed;
    unsigned *shift;
    unsigned long long *sums;
    int32_t *keys_in, *keys_out, *vals_in, *vals_out, *inv, *order;
    int32_t *assign2, *rowbuf, *segoff;
    void *C2old;
    int32_t *N2old, *parent;
    void *cub;
    size_t cub_b;
    void *tc;  // tensor-core assignment region (kmeans_tc.cu)
    // levels == 3: Level-1 tables in K-means id order, Level-0 labels and order
    void *C1old;
    int32_t *N1old, *coff1, *parent0, *order1, *inv1;
};

Ws carve(const sqz_index &idx, char *base, size_t *total) {
    const int64_t H = idx.H, L = idx.L, d = idx.d;
    const int64_t c = idx.c2, n = L;
    const int64_t esz = idx.dtype == SQZ_BF16 ? 2 : 4;
    Carve cv{base};
    Ws w;
    w.Xh = cv.take<float>(H * n * d);
    w.mu = cv.take<float>(H * c * d);
    w.musq = cv.take<float>(H * c);
    w.pdist = cv.take<float>(H * n);
    w.assign = cv.take<int32_t>(H * n);
    w.counts = cv.take<int32_t>(H * c);
    w.done = cv.take<int32_t>(H);
    w.changed = cv.take<int32_t>(H);
    w.shift = cv.take<unsigned>(H);
    w.sums = cv.take<unsigned long long>(H * c * d);
    w.keys_in = cv.take<int32_t>(H * n);
    w.keys_out = cv.take<int32_t>(H * n);
    w.vals_in = cv.take<int32_t>(H * n);
    w.vals_out = cv.take<int32_t>(H * n);
    w.inv = cv.take<int32_t>(H * c);
    w.order = cv.take<int32_t>(H * c);
    w.assign2 = cv.take<int32_t>(H * n);
    w.rowbuf = cv.take<int32_t>(H * n);
    w.segoff = cv.take<int32_t>(H * (c + 1));
    w.C2old = cv.take<char>(H * c * d * esz);
    w.N2old = cv.take<int32_t>(H * c);
    w.parent = cv.take<int32_t>(H * c);
    w.cub_b = cub_bytes(H * n);
    w.cub = cv.take<char>(w.cub_b);
    w.tc = cv.take<char>(kmeans_tc_ws_bytes((int)H, n, c, (int)d));
    const int64_t c1 = idx.levels == 3 ? idx.c1 : 0;
    w.C1old = cv.take<char>(H * c1 * d * esz);
    w.N1old = cv.take<int32_t>(H * c1);
    w.coff1 = cv.take<int32_t>(H * (c1 + 1));
    w.parent0 = cv.take<int32_t>(H * c1);
    w.order1 = cv.take<int32_t>(H * c1);
    w.inv1 = cv.take<int32_t>(H * c1);
    *total = cv.used + 256;
    return w;
}

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess) {                                                         \
            snprintf(err, errlen, "%s: %s", #x, cudaGetErrorString(e_));                \
            return SQZ_ERR_CUDA;                                                         \
        }                                                                                \
    } while (0)

// Lloyd iterations for all heads on Xh[H,n,d] with c clusters. Leaves assign.
int lloyd(Ws &w, int H, int n, int c, int d, const int64_t *init, const sqz_kmeans_params &p,
          int32_t *iters, cudaStream_t st, char *err, size_t errlen) {
    CK(cudaMemsetAsync(w.done, 0, sizeof(int32_t) * H, st));
    CK(cudaMemsetAsync(w.assign, 0xff, sizeof(int32_t) * (size_t)H * n, st));  // -1
    k_init<<<dim3(c, H), 128, 0, st>>>(w.Xh, init, n, c, d, w.mu);
    CK(cudaGetLastError());
    const size_t smem = (size_t)2 * KT * (d + 1) * sizeof(float);
    CK(cudaFuncSetAttribute(k_assign, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // the tensor-core assignment (NEXT-3): split the normalised keys once per run
    const bool tc = kmeans_tc_applies(p.assign_mode, d, n, c);
    KmeansTc ktc;
    if (tc) {
        ktc.H = H; ktc.n = n; ktc.c = c; ktc.d = d;
        ktc.Xh = w.Xh; ktc.mu = w.mu; ktc.musq = w.musq; ktc.done = w.done;
        ktc.assign = w.assign; ktc.pdist = w.pdist; ktc.changed = w.changed;
        ktc.margin = 2e-4f;
        ktc.w = kmeans_tc_carve(w.tc, H, n, d);
        CK(kmeans_tc_split_x(w.Xh, H, n, d, ktc.w, st));
    }
    std::vector<int32_t> changed(H), done(H, 0);
    std::vector<unsigned> shift(H);
    *iters = 0;
    for (int it = 0; it < p.max_iters; ++it) {
        CK(cudaMemsetAsync(w.changed, 0, sizeof(int32_t) * H, st));
        CK(cudaMemsetAsync(w.shift, 0, sizeof(unsigned) * H, st));
        CK(cudaMemsetAsync(w.counts, 0, sizeof(int32_t) * (size_t)H * c, st));
        CK(cudaMemsetAsync(w.sums, 0, sizeof(unsigned long long) * (size_t)H * c * d, st));
        k_musq<<<dim3((c + 7) / 8, H), 256, 0, st>>>(w.mu, c, d, w.done, w.musq);
        if (tc)
            CK(kmeans_tc_assign(ktc, st));
        else
            k_assign<<<dim3((n + KT - 1) / KT, H), 256, smem, st>>>(w.Xh, n, c, d, w.mu, w.musq, w.done,
                                                                   w.assign, w.pdist, w.changed);
        k_counts<<<dim3(std::min(1024, (n + 255) / 256), H), 256, 0, st>>>(w.assign, n, c, w.done,
                                                                          w.counts);
        k_repair<<<H, 1024, 0, st>>>(w.assign, w.pdist, n, c, w.done, w.counts, w.changed);
        const int64_t tot = (int64_t)n * d;
        k_accumulate<float><<<dim3((unsigned)std::min<int64_t>(4096, (tot + 255) / 256), H), 256, 0,
                              st>>>(w.Xh, w.assign, n, c, d, w.done, w.sums);
        k_update<<<dim3((c + 7) / 8, H), 256, 0, st>>>(w.sums, w.counts, c, d, w.done, w.mu,
                                                       w.shift);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(changed.data(), w.changed, sizeof(int32_t) * H, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(shift.data(), w.shift, sizeof(unsigned) * H, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        bool all = true;
        for (int h = 0; h < H; ++h) {
            if (done[h]) continue;
            float sh;
            std::memcpy(&sh, &shift[h], 4);
            if (changed[h] == 0 || sh < p.tol) done[h] = 1;
            all = all && done[h];
        }
        *iters = it + 1;
        CK(cudaMemcpyAsync(w.done, done.data(), sizeof(int32_t) * H, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));  // `done` is a stack vector
        if (all) break;
    }
    return SQZ_OK;
}

// Stable radix sort of (h * kmul + label) keys; returns, per head, the sorted
// local row order in `order_out` ([H, n]) so that rows with equal label keep
// increasing index order.
int sort_by_label(Ws &w, const int32_t *lab, const int32_t *remap, int H, int n, int kmul,
                  int rmul, int32_t *order_out, cudaStream_t st, char *err, size_t errlen) {
    k_make_keys<<<dim3(std::max(1, std::min(4096, (n + 255) / 256)), H), 256, 0, st>>>(
        lab, remap, n, kmul, rmul, w.keys_in, w.vals_in);
    size_t cb = w.cub_b;
    CK(cub::DeviceRadixSort::SortPairs(w.cub, cb, w.keys_in, w.keys_out, w.vals_in, w.vals_out,
                                       (int)((int64_t)H * n), 0, 32, st));
    k_positions<<<dim3(std::max(1, std::min(4096, (n + 255) / 256)), H), 256, 0, st>>>(
        w.vals_out, n, order_out, nullptr);
    CK(cudaGetLastError());
    return SQZ_OK;
}

template <typename T>
int cluster_keys_t(const T *K, const T *V, const int64_t *init2, const int64_t *init1,
                   sqz_index *idx, T *Kp, T *Vp, const sqz_kmeans_params &p, Ws &w,
                   int32_t *iters_out, cudaStream_t st, char *err, size_t errlen) {
    const int H = idx->H, d = idx->d, c2 = idx->c2, c1 = idx->c1;
    const int64_t L = idx->L;
    const int n = (int)L;
    const int wpb = 8;  // warps per 256-thread block
    // ---- Level 2: K-means on the normalised keys ----
    k_normalize<T><<<dim3((unsigned)((H * L + wpb - 1) / wpb)), 256, 0, st>>>(K, (int64_t)H * L, d,
                                                                             w.Xh);
    CK(cudaGetLastError());
    int32_t it2 = 0, it1 = 0;
    int rc = lloyd(w, H, n, c2, d, init2, p, &it2, st, err, errlen);
    if (rc) return rc;
    int32_t *assign2 = w.assign2;
    CK(cudaMemcpyAsync(assign2, w.assign, sizeof(int32_t) * (size_t)H * n, cudaMemcpyDeviceToDevice,
                       st));
    // members of each (old) Level-2 cluster in increasing key index
    rc = sort_by_label(w, assign2, nullptr, H, n, c2, 0, w.rowbuf, st, err, errlen);
    if (rc) return rc;
    CK(cudaMemsetAsync(w.done, 0, sizeof(int32_t) * H, st));
    CK(cudaMemsetAsync(w.counts, 0, sizeof(int32_t) * (size_t)H * c2, st));
    k_counts<<<dim3(std::max(1, std::min(1024, (n + 255) / 256)), H), 256, 0, st>>>(
        assign2, n, c2, w.done, w.counts);
    k_exscan<<<H, 1024, 0, st>>>(w.counts, c2, w.segoff);
    // C2 = raw member mean in fp64, summed in increasing key order (R2, R18)
    T *C2old = reinterpret_cast<T *>(w.C2old);
    k_segment_means<T><<<dim3((c2 + wpb - 1) / wpb, H), 256, 0, st>>>(K, n, w.rowbuf, w.segoff, c2, d,
                                                                     C2old, w.N2old);
    CK(cudaGetLastError());

    int32_t it0 = 0;
    if (idx->levels >= 2) {
        // ---- Level 1: K-means on the stored Level-2 centroids (R5) ----
        k_normalize<T><<<dim3((unsigned)((H * c2 + wpb - 1) / wpb)), 256, 0, st>>>(
            C2old, (int64_t)H * c2, d, w.Xh);
        rc = lloyd(w, H, c2, c1, d, init1, p, &it1, st, err, errlen);
        if (rc) return rc;
        CK(cudaMemcpyAsync(w.parent, w.assign, sizeof(int32_t) * (size_t)H * c2,
                           cudaMemcpyDeviceToDevice, st));
    }
    if (idx->levels == 3) {
        // ---- Level 0: the Level-1 tables in K-means id order first ----
        const int c0 = idx->c0;
        T *C1old = reinterpret_cast<T *>(w.C1old);
        rc = sort_by_label(w, w.parent, nullptr, H, c2, c1, 0, w.order, st, err, errlen);
        if (rc) return rc;
        CK(cudaMemsetAsync(w.done, 0, sizeof(int32_t) * H, st));
        CK(cudaMemsetAsync(w.counts, 0, sizeof(int32_t) * (size_t)H * c1, st));
        k_counts<<<dim3((c2 + 255) / 256, H), 256, 0, st>>>(w.parent, c2, c1, w.done, w.counts);
        k_exscan<<<H, 1024, 0, st>>>(w.counts, c1, w.coff1);
        k_segment_means<T><<<dim3((c1 + wpb - 1) / wpb, H), 256, 0, st>>>(C2old, c2, w.order, w.coff1, c1,
                                                                         d, C1old, nullptr);
        CK(cudaMemsetAsync(w.N1old, 0, sizeof(int32_t) * (size_t)H * c1, st));
        k_parent_weights<<<dim3((c2 + 255) / 256, H), 256, 0, st>>>(w.parent, w.N2old, c2, c1, w.N1old);
        CK(cudaGetLastError());
        // K-means on the stored Level-1 rows -> Level-0 labels
        k_normalize<T><<<dim3((unsigned)((H * c1 + wpb - 1) / wpb)), 256, 0, st>>>(
            C1old, (int64_t)H * c1, d, w.Xh);
        rc = lloyd(w, H, c1, c0, d, p.init0, p, &it0, st, err, errlen);
        if (rc) return rc;
        CK(cudaMemcpyAsync(w.parent0, w.assign, sizeof(int32_t) * (size_t)H * c1,
                           cudaMemcpyDeviceToDevice, st));
        // Level-1 ids grouped by Level-0 parent, stable in K-means id: order1[new] = old
        rc = sort_by_label(w, w.parent0, nullptr, H, c1, c0, 0, w.order1, st, err, errlen);
        if (rc) return rc;
        k_invert<<<dim3((c1 + 255) / 256, H), 256, 0, st>>>(w.order1, c1, w.inv1);
        CK(cudaMemsetAsync(w.done, 0, sizeof(int32_t) * H, st));
        CK(cudaMemsetAsync(w.counts, 0, sizeof(int32_t) * (size_t)H * c0, st));
        k_counts<<<dim3((c1 + 255) / 256, H), 256, 0, st>>>(w.parent0, c1, c0, w.done, w.counts);
        k_exscan<<<H, 1024, 0, st>>>(w.counts, c0, idx->child_off0);
        // C0 = unweighted mean of the child Level-1 rows (R5 one level up), N0 = descendant keys
        k_segment_means<T><<<dim3((c0 + wpb - 1) / wpb, H), 256, 0, st>>>(
            C1old, c1, w.order1, idx->child_off0, c0, d, (T *)idx->C0, nullptr);
        CK(cudaMemsetAsync(idx->N0, 0, sizeof(int32_t) * (size_t)H * c0, st));
        k_parent_weights<<<dim3((c1 + 255) / 256, H), 256, 0, st>>>(w.parent0, w.N1old, c1, c0, idx->N0);
        // Level-1 tables in the new order; Level-2 parents renumbered
        k_gather_rows<T><<<dim3(std::max(1, std::min(4096, (c1 * d + 255) / 256)), H), 256, 0, st>>>(
            C1old, w.order1, c1, d, (T *)idx->C1);
        k_gather_rows<int32_t><<<dim3(std::max(1, (c1 + 255) / 256), H), 256, 0, st>>>(w.N1old, w.order1,
                                                                                     c1, 1, idx->N1);
        k_remap<<<dim3((c2 + 255) / 256, H), 256, 0, st>>>(w.parent, w.inv1, c2, c1);
        CK(cudaGetLastError());
    }
    if (idx->levels >= 2) {
        // Level-2 clusters grouped by parent, stable in old id: order[new] = old
        rc = sort_by_label(w, w.parent, nullptr, H, c2, c1, 0, w.order, st, err, errlen);
        if (rc) return rc;
        k_invert<<<dim3((c2 + 255) / 256, H), 256, 0, st>>>(w.order, c2, w.inv);
        CK(cudaMemsetAsync(w.done, 0, sizeof(int32_t) * H, st));
        CK(cudaMemsetAsync(w.counts, 0, sizeof(int32_t) * (size_t)H * c1, st));
        k_counts<<<dim3((c2 + 255) / 256, H), 256, 0, st>>>(w.parent, c2, c1, w.done, w.counts);
        k_exscan<<<H, 1024, 0, st>>>(w.counts, c1, idx->child_off);
        if (idx->levels == 2) {
            // C1 = unweighted mean of the child rows, summed in increasing old id
            k_segment_means<T><<<dim3((c1 + wpb - 1) / wpb, H), 256, 0, st>>>(
                C2old, c2, w.order, idx->child_off, c1, d, (T *)idx->C1, nullptr);
            CK(cudaMemsetAsync(idx->N1, 0, sizeof(int32_t) * (size_t)H * c1, st));
            k_parent_weights<<<dim3((c2 + 255) / 256, H), 256, 0, st>>>(w.parent, w.N2old, c2, c1,
                                                                        idx->N1);
        }
        CK(cudaGetLastError());
    } else {
        k_iota<<<dim3((c2 + 255) / 256, H), 256, 0, st>>>(c2, w.order, w.inv);
        CK(cudaGetLastError());
    }
    // C2, N2 in the new order; key_off
    k_gather_rows<T><<<dim3(std::max(1, std::min(4096, (c2 * d + 255) / 256)), H), 256, 0, st>>>(
        C2old, w.order, c2, d, (T *)idx->C2);
    k_gather_rows<int32_t><<<dim3(std::max(1, (c2 + 255) / 256), H), 256, 0, st>>>(w.N2old, w.order,
                                                                                 c2, 1, idx->N2);
    k_exscan<<<H, 1024, 0, st>>>(idx->N2, c2, idx->key_off);
    // keys grouped by new Level-2 id, stable in original index -> perm
    rc = sort_by_label(w, assign2, w.inv, H, n, c2, c2, idx->perm, st, err, errlen);
    if (rc) return rc;
    const int vpr = d * (int)sizeof(T) / 16;
    const int64_t tot = L * vpr;
    dim3 gg((unsigned)std::min<int64_t>(8192, (tot + 255) / 256), H);
    k_gather_kv<<<gg, 256, 0, st>>>((const uint4 *)K, idx->perm, L, vpr, (uint4 *)Kp);
    k_gather_kv<<<gg, 256, 0, st>>>((const uint4 *)V, idx->perm, L, vpr, (uint4 *)Vp);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    if (iters_out) {
        iters_out[0] = it2;
        iters_out[1] = it1;
        if (idx->levels == 3) iters_out[2] = it0;
    }
    return SQZ_OK;
}
}  // namespace

size_t kmeans_workspace_bytes(const sqz_index &idx) {
    size_t t = 0;
    carve(idx, nullptr, &t);
    return t;
}

int cluster_keys(const void *K, const void *V, const int64_t *init2, const int64_t *init1,
                 sqz_index *idx, void *Kp, void *Vp, const sqz_kmeans_params &p, void *ws,
                 size_t ws_bytes, int32_t *iters_out, cudaStream_t st, char *err, size_t errlen) {
    size_t need = 0;
    char *base = reinterpret_cast<char *>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    Ws w = carve(*idx, base, &need);
    if (ws_bytes < need) {
        snprintf(err, errlen, "ws_bytes %zu < required %zu", ws_bytes, need);
        return SQZ_ERR_INVALID_ARG;
    }
    if (idx->dtype == SQZ_BF16)
        return cluster_keys_t<__nv_bfloat16>((const __nv_bfloat16 *)K, (const __nv_bfloat16 *)V, init2,
                                             init1, idx, (__nv_bfloat16 *)Kp, (__nv_bfloat16 *)Vp, p,
                                             w, iters_out, st, err, errlen);
    return cluster_keys_t<float>((const float *)K, (const float *)V, init2, init1, idx, (float *)Kp,
                                 (float *)Vp, p, w, iters_out, st, err, errlen);
}

// --------------------------------------------------------------------------
// index validation
// --------------------------------------------------------------------------
__global__ void k_validate(sqz_index idx, int32_t *__restrict__ hist, int *__restrict__ bad) {
    const int h = blockIdx.y;
    const int c2 = idx.c2;
    const int64_t L = idx.L;
    // a shard (L_total > 0) holds key_off[c2] <= L keys of the L_total original ones
    const int64_t Lt = idx.L_total > 0 ? idx.L_total : L;
    const int32_t *N2 = idx.N2 + (size_t)h * c2;
    const int32_t *ko = idx.key_off + (size_t)h * (c2 + 1);
    const int64_t nkeys = min((int64_t)ko[c2], L);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < c2; i += gridDim.x * blockDim.x) {
        if (N2[i] < 0 || ko[i + 1] - ko[i] != N2[i]) atomicOr(bad, 1);
        if (i == 0 && ko[0] != 0) atomicOr(bad, 1);
        if (i == c2 - 1 && (idx.L_total > 0 ? ko[c2] > L : ko[c2] != L)) atomicOr(bad, 1);
    }
    const int32_t *pm = idx.perm + (size_t)h * L;
    for (int64_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nkeys; j += gridDim.x * blockDim.x) {
        const int32_t v = pm[j];
        if (v < 0 || v >= Lt) atomicOr(bad, 2);
        else atomicAdd(hist + (size_t)h * Lt + v, 1);
    }
    if (idx.levels == 3) {  // Level 0 over Level 1: contiguous, non-empty, N0 = descendant keys
        const int c0 = idx.c0, c1 = idx.c1;
        const int32_t *co = idx.child_off0 + (size_t)h * (c0 + 1);
        const int32_t *N0 = idx.N0 + (size_t)h * c0;
        const int32_t *N1 = idx.N1 + (size_t)h * c1;
        for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < c0; g += gridDim.x * blockDim.x) {
            if (co[g + 1] <= co[g] || co[g] < 0 || co[g + 1] > c1) { atomicOr(bad, 16); continue; }
            if (g == 0 && co[0] != 0) atomicOr(bad, 16);
            if (g == c0 - 1 && co[c0] != c1) atomicOr(bad, 16);
            long long t = 0;
            for (int p = co[g]; p < co[g + 1]; ++p) t += N1[p];
            if (t != N0[g]) atomicOr(bad, 16);
        }
    }
    if (idx.levels >= 2) {
        const int c1 = idx.c1;
        const int32_t *co = idx.child_off + (size_t)h * (c1 + 1);
        const int32_t *N1 = idx.N1 + (size_t)h * c1;
        for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < c1; p += gridDim.x * blockDim.x) {
            // an unsharded index has no empty Level-1 cluster (K-means repairs empty
            // clusters; the decode Level-2 lookup relies on >= 1 child per survivor);
            // shard padding rows (L_total > 0) have empty ranges
            if (co[p + 1] < co[p] || co[p] < 0 || co[p + 1] > c2 ||
                (idx.L_total == 0 && co[p + 1] == co[p])) { atomicOr(bad, 4); continue; }
            if (p == 0 && co[0] != 0) atomicOr(bad, 4);
            if (p == c1 - 1 && (idx.L_total > 0 ? co[c1] > c2 : co[c1] != c2)) atomicOr(bad, 4);
            long long s = 0;
            for (int l = co[p]; l < co[p + 1]; ++l) s += N2[l];
            if (s != N1[p]) atomicOr(bad, 8);
        }
    }
}
// every original key exactly once (a shard: at most once)
__global__ void k_validate_hist(const int32_t *__restrict__ hist, int64_t n, int shard,
                                int *__restrict__ bad) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        if (shard ? hist[j] > 1 : hist[j] != 1) atomicOr(bad, 2);
}

size_t validate_workspace_bytes(const sqz_index &idx) {
    return sizeof(int32_t) * ((size_t)idx.H * (idx.L_total > 0 ? idx.L_total : idx.L) + 64);
}

int index_validate(const sqz_index &idx, void *ws, size_t ws_bytes, cudaStream_t st, char *err,
                   size_t errlen) {
    if (ws_bytes < validate_workspace_bytes(idx)) {
        snprintf(err, errlen, "ws_bytes too small");
        return SQZ_ERR_INVALID_ARG;
    }
    int *bad = reinterpret_cast<int *>(ws);
    int32_t *hist = reinterpret_cast<int32_t *>(ws) + 64;
    CK(cudaMemsetAsync(ws, 0, validate_workspace_bytes(idx), st));
    dim3 g(std::max(1, (int)std::min<int64_t>(1024, (idx.L + 255) / 256)), idx.H);
    k_validate<<<g, 256, 0, st>>>(idx, hist, bad);
    k_validate_hist<<<1024, 256, 0, st>>>(hist, (int64_t)idx.H * (idx.L_total > 0 ? idx.L_total : idx.L),
                                          idx.L_total > 0, bad);
    CK(cudaGetLastError());
    int hb = 0;
    CK(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hb) {
        snprintf(err, errlen, "index invariant violated:%s%s%s%s%s", (hb & 1) ? " key_off/N2" : "",
                 (hb & 2) ? " perm" : "", (hb & 4) ? " child_off" : "", (hb & 8) ? " N1" : "",
                 (hb & 16) ? " child_off0/N0" : "");
        return SQZ_ERR_INVARIANT;
    }
    return SQZ_OK;
}

}  // namespace sqz
