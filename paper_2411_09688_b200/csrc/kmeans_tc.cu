// kmeans_tc.cu -- the K-means assignment step of sqz_cluster_keys on the 5th-gen
// tensor cores ("Fast GPU K-means ... tcgen05 assignment
// GEMM fused with argmax"; the paper names faster offline clustering as future
// work, and clustered its 1M-token contexts with offloading).
//
// a_j = argmin_i ||x^_j - mu_i||^2 = argmin_i (||mu_i||^2 - 2 x^_j . mu_i) is a
// GEMM (keys x centroids, K = d) with an argmin epilogue.  bf16 operands alone
// would perturb the scores by ~2^-8 and flip many assignments, so both sides
// are split, x = x_h + x_l and mu = mu_h + mu_l with x_h = bf16(x),
// x_l = bf16(x - x_h), and the tensor cores accumulate (in fp32)
//     x_h.mu_h + x_h.mu_l + x_l.mu_h
// (the dropped x_l.mu_l term and the rounding of x_l, mu_l are ~2^-17 of
// |x||mu|, the size of fp32 FFMA rounding).  One CTA holds 128 keys of a head
// (A = [x_h | x_l], 2d bf16 per row, loaded once by TMA) and sweeps all
// centroids in 256-column tiles (B = [mu_h | mu_l] halves streamed by TMA
// through a 4-stage ring; tcgen05.mma M128 N256 K16; double-buffered TMEM
// accumulators, 2 x 256 columns).  Four epilogue warps (thread = key row) read
// the accumulator with tcgen05.ld, form e = ||mu||^2 - 2 s and keep the two
// best (e, id) per key (ids ascend, so strict '<' keeps the lowest id on ties).
// A key whose two best scores are closer than `margin` is re-ranked exactly by
// k_rerank (fp32 FFMA over the two candidates, in the same order and with the
// same tie rule as the exact kernel k_assign); every other key takes the best
// tensor-core candidate.
#include <cstring>

#include "common.cuh"
#include "internal.h"
#include "tcgen05.cuh"

namespace sqz {

namespace kmt {
constexpr int BM = 128;                 // keys per CTA
constexpr int BN = 256;                 // centroids per tile
constexpr int A_HB = BM * 128;          // 16 KB: one 64-element half of 128 rows
constexpr int B_HB = BN * 128;          // 32 KB: one half of 256 rows
constexpr int NST = 4;                  // B ring stages
constexpr int NT = 192;                 // 4 epilogue warps + producer + MMA warp
}  // namespace kmt

template <int D>
struct KmtSmem {
    static constexpr int NH = D / 64;                   // halves per split part
    static constexpr int A = 0;                         // 2*NH A halves
    static constexpr int B = A + 2 * NH * kmt::A_HB;    // ring
    static constexpr int MS = B + kmt::NST * kmt::B_HB; // musq slices [4][256] fp32
    static constexpr int BAR = MS + 4 * kmt::BN * 4;
    static constexpr int BYTES = BAR + 256 + 1024;      // + barriers, 1024 alignment slack
};

template <int D>
__global__ void __launch_bounds__(kmt::NT, 1)
    k_assign_tc(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmM, int n,
                int c, const float *__restrict__ musq, const float *__restrict__ xx,
                const int *__restrict__ done, int32_t *__restrict__ assign, float *__restrict__ pdist,
                int *__restrict__ changed, int4 *__restrict__ amb, int *__restrict__ amb_n, float margin) {
    using S = KmtSmem<D>;
    constexpr int NH = S::NH;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int h = blockIdx.y;
    if (done[h]) return;
    unsigned char *sm = reinterpret_cast<unsigned char *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const uint32_t sbase = smem_u32(sm);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + S::BAR);
    uint64_t *a_full = bar, *b_full = bar + 1, *b_empty = bar + 1 + kmt::NST;
    uint64_t *acc_full = bar + 1 + 2 * kmt::NST, *acc_empty = acc_full + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = (c + kmt::BN - 1) / kmt::BN;
    if (threadIdx.x == 0) {
        mbar_init(a_full, 1);
        for (int s = 0; s < kmt::NST; ++s) {
            mbar_init(&b_full[s], 1);
            mbar_init(&b_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 4);
        }
        mbar_fence_init();
    }
    if (warp == 5) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int row0 = blockIdx.x * kmt::BM;
    if (warp == 4) {
        // ======================= TMA producer =======================
        if (lane == 0) {
            mbar_arrive_expect_tx(a_full, 2 * NH * kmt::A_HB);
            for (int q = 0; q < 2 * NH; ++q)
                tma_load_3d(sbase + S::A + q * kmt::A_HB, &tmX, q * 64, h * n + row0, 0, a_full);
            int t = 0;
            for (int j = 0; j < ntiles; ++j)
                for (int q = 0; q < 2 * NH; ++q, ++t) {
                    const int st = t % kmt::NST;
                    mbar_wait(&b_empty[st], ((t / kmt::NST) & 1) ^ 1);
                    mbar_arrive_expect_tx(&b_full[st], kmt::B_HB);
                    tma_load_3d(sbase + S::B + st * kmt::B_HB, &tmM, q * 64, h * c + j * kmt::BN, 0,
                                &b_full[st]);
                }
        }
    } else if (warp == 5) {
        // ======================= MMA issuer (whole warp, one elected lane) =======================
        constexpr uint32_t IDESC = idesc_bf16(kmt::BM, kmt::BN, false);
        mbar_wait(a_full, 0);
        tc_fence_after();
        int t = 0;
        for (int j = 0; j < ntiles; ++j) {
            const int buf = j & 1;
            mbar_wait(&acc_empty[buf], ((j >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t dt = tmem + buf * kmt::BN;
            uint32_t acc = 0;
            for (int q = 0; q < 2 * NH; ++q, ++t) {
                const int st = t % kmt::NST;
                mbar_wait(&b_full[st], (t / kmt::NST) & 1);
                tc_fence_after();
                const uint64_t bd = sdesc_sw128(sbase + S::B + st * kmt::B_HB, 16, 1024);
                // B half q: mu_h half q (q < NH) pairs with x_h half q and x_l half q;
                // mu_l half q - NH pairs with x_h half q - NH
                const int np = q < NH ? 2 : 1;
                for (int pi = 0; pi < np; ++pi) {
                    const int ah = q < NH ? (pi == 0 ? q : NH + q) : q - NH;
                    const uint64_t ad = sdesc_sw128(sbase + S::A + ah * kmt::A_HB, 16, 1024);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        umma_bf16_w(dt, ad + 2 * k, bd + 2 * k, IDESC, acc);
                        acc = 1;
                    }
                }
                umma_commit_w(&b_empty[st]);
            }
            umma_commit_w(&acc_full[buf]);
        }
    } else {
        // ======================= epilogue: thread = key row =======================
        float *ms = reinterpret_cast<float *>(sm + S::MS) + warp * kmt::BN;
        float b1 = INFINITY, b2 = INFINITY;
        int i1 = 0, i2 = -1;
        const float *mq = musq + (size_t)h * c;
        for (int j = 0; j < ntiles; ++j) {
            const int buf = j & 1;
            for (int e = lane; e < kmt::BN; e += 32) {
                const int col = j * kmt::BN + e;
                ms[e] = col < c ? __ldg(mq + col) : INFINITY;  // columns past c never win
            }
            __syncwarp();
            mbar_wait(&acc_full[buf], (j >> 1) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int cc = 0; cc < kmt::BN / 32; ++cc) {
                float v[32];
                tmem_ld32(tmem + buf * kmt::BN + cc * 32 + ((uint32_t)(warp * 32) << 16), v);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const float e = fmaf(-2.f, v[i], ms[cc * 32 + i]);
                    const int col = j * kmt::BN + cc * 32 + i;
                    if (e < b1) {
                        b2 = b1;
                        i2 = i1;
                        b1 = e;
                        i1 = col;
                    } else if (e < b2) {
                        b2 = e;
                        i2 = col;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[buf]);
        }
        const int p = row0 + warp * 32 + lane;
        int ch = 0;
        if (p < n) {
            const size_t r = (size_t)h * n + p;
            if (i2 < 0 || b2 - b1 >= margin) {
                if (assign[r] != i1) ch = 1;
                assign[r] = i1;
                pdist[r] = fmaxf(xx[r] + b1, 0.f);
            } else {
                const int slot = atomicAdd(amb_n, 1);
                amb[slot] = make_int4(h, p, i1, i2);
            }
        }
        ch = __reduce_add_sync(FULL, ch);
        if (lane == 0 && ch) atomicAdd(changed + h, ch);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 5) tmem_dealloc(tmem, 512);
}

// exact fp32 re-rank of the ambiguous keys over their two candidates, with the
// arithmetic of k_assign (sequential FMA over k; e = ||mu||^2 - 2 s; lowest id on ties)
__global__ void k_rerank(const float *__restrict__ Xh, const float *__restrict__ mu,
                         const float *__restrict__ musq, int n, int c, int d, const int4 *__restrict__ amb,
                         const int *__restrict__ amb_n, int32_t *__restrict__ assign,
                         float *__restrict__ pdist, int *__restrict__ changed) {
    const int tot = *amb_n;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += gridDim.x * blockDim.x) {
        const int4 a = amb[e];
        const int h = a.x, p = a.y;
        const float *x = Xh + ((size_t)h * n + p) * d;
        const float *m1 = mu + ((size_t)h * c + a.z) * d, *m2 = mu + ((size_t)h * c + a.w) * d;
        float s1 = 0.f, s2 = 0.f, xs = 0.f;
        for (int k = 0; k < d; ++k) {
            const float xv = x[k];
            s1 = fmaf(xv, m1[k], s1);
            s2 = fmaf(xv, m2[k], s2);
            xs = fmaf(xv, xv, xs);
        }
        const float e1 = fmaf(-2.f, s1, musq[(size_t)h * c + a.z]);
        const float e2 = fmaf(-2.f, s2, musq[(size_t)h * c + a.w]);
        const bool first = e1 < e2 || (e1 == e2 && a.z < a.w);
        const int best = first ? a.z : a.w;
        const float be = first ? e1 : e2;
        const size_t r = (size_t)h * n + p;
        if (assign[r] != best) atomicAdd(changed + h, 1);
        assign[r] = best;
        pdist[r] = fmaxf(xs + be, 0.f);
    }
}

// rows of X [R, d] fp32 -> S [R, 2d] bf16 = [bf16(x) | bf16(x - bf16(x))]; optional
// sq[r] = sum_k x_k^2 by sequential FMA (the order k_assign uses)
__global__ void k_split_rows(const float *__restrict__ X, int64_t R, int d, __nv_bfloat16 *__restrict__ S,
                             float *__restrict__ sq) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= R) return;
    const float *x = X + row * d;
    __nv_bfloat16 *s = S + row * 2 * d;
    for (int k = lane; k < d; k += 32) {
        const float v = x[k];
        const __nv_bfloat16 hi = __float2bfloat16_rn(v);
        s[k] = hi;
        s[d + k] = __float2bfloat16_rn(v - __bfloat162float(hi));
    }
    if (sq && lane == 0) {
        float a = 0.f;
        for (int k = 0; k < d; ++k) a = fmaf(x[k], x[k], a);
        sq[row] = a;
    }
}

size_t kmeans_tc_ws_bytes(int H, int64_t n, int64_t c, int d) {
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    return al(256) + al((size_t)H * n * 4) + al((size_t)H * n * 16) + al((size_t)H * n * 2 * d * 2) +
           al((size_t)H * c * 2 * d * 2) + 512;
}

bool kmeans_tc_applies(int mode, int d, int64_t n, int64_t c) {
    if (mode == SQZ_KMEANS_EXACT || (d != 64 && d != 128) || c < 2) return false;
    if (mode == SQZ_KMEANS_TENSOR) return true;
    return n * c >= (int64_t)1 << 26;  // auto: the large problems
}

KmeansTcWs kmeans_tc_carve(void *ws, int H, int64_t n, int d) {
    KmeansTcWs w;
    char *p = reinterpret_cast<char *>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    w.amb_n = reinterpret_cast<int *>(p);
    p += al(256);
    w.xx = reinterpret_cast<float *>(p);
    p += al((size_t)H * n * 4);
    w.amb = reinterpret_cast<int4 *>(p);
    p += al((size_t)H * n * 16);
    w.Xs = p;
    p += al((size_t)H * n * 2 * d * 2);
    w.Ms = p;
    return w;
}

cudaError_t kmeans_tc_split_x(const float *Xh, int H, int n, int d, const KmeansTcWs &w, cudaStream_t st) {
    const int64_t R = (int64_t)H * n;
    k_split_rows<<<(unsigned)((R + 7) / 8), 256, 0, st>>>(Xh, R, d, reinterpret_cast<__nv_bfloat16 *>(w.Xs),
                                                         w.xx);
    return cudaGetLastError();
}

namespace {
template <int D>
cudaError_t launch_tc_t(const KmeansTc &k, const CUtensorMap &mx, const CUtensorMap &mm, cudaStream_t st) {
    using S = KmtSmem<D>;
    auto kern = k_assign_tc<D>;
    cudaError_t e = ensure_func_attr((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::BYTES);
    if (e != cudaSuccess) return e;
    const dim3 grid((unsigned)((k.n + kmt::BM - 1) / kmt::BM), (unsigned)k.H);
    kern<<<grid, kmt::NT, S::BYTES, st>>>(mx, mm, k.n, k.c, k.musq, k.w.xx, k.done, k.assign, k.pdist,
                                           k.changed, k.w.amb, k.w.amb_n, k.margin);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_rerank<<<592, 128, 0, st>>>(k.Xh, k.mu, k.musq, k.n, k.c, D, k.w.amb, k.w.amb_n, k.assign, k.pdist,
                                  k.changed);
    return cudaGetLastError();
}
}  // namespace

cudaError_t kmeans_tc_assign(const KmeansTc &k, cudaStream_t st) {
    // per iteration: split the centroids, encode the maps, clear the ambiguous list
    const int64_t R = (int64_t)k.H * k.c;
    k_split_rows<<<(unsigned)((R + 7) / 8), 256, 0, st>>>(k.mu, R, k.d,
                                                         reinterpret_cast<__nv_bfloat16 *>(k.w.Ms), nullptr);
    cudaError_t e = cudaMemsetAsync(k.w.amb_n, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    const uint32_t boxA[3] = {64, (uint32_t)kmt::BM, 1}, boxB[3] = {64, (uint32_t)kmt::BN, 1};
    const uint64_t dX[3] = {(uint64_t)2 * k.d, (uint64_t)k.H * k.n, 1};
    const uint64_t dM[3] = {(uint64_t)2 * k.d, (uint64_t)k.H * k.c, 1};
    CUtensorMap mx, mm;
    if (encode_tmap_bf16_3d(&mx, k.w.Xs, dX, boxA) != 0 || encode_tmap_bf16_3d(&mm, k.w.Ms, dM, boxB) != 0)
        return cudaErrorInvalidValue;
    if (k.d == 128) return launch_tc_t<128>(k, mx, mm, st);
    return launch_tc_t<64>(k, mx, mm, st);
}

}  // namespace sqz
