// shared_attn.cu -- batch-shared decode attention.
//
// The paper's serving scenario is many sequences sharing ONE fixed context
// (P:45-50): B decode queries per head attend to their own selections of the
// same cluster-major Kp/Vp.  The per-row kernel (attention.cu) streams every
// (b,h) selection separately, so a cluster selected by several queries is read
// several times.  Here each head streams the UNION of its B selections once:
//   k_union        per head: the B ascending cluster lists -> one ascending
//                  union list with a B-bit mask per cluster (which queries
//                  selected it) and the key prefix of the union;
//   k_attend_shared persistent CTAs over equal-cost ranges of the per-head
//                  streams [union fixed keys | user KV of b = 0 .. B-1] (the
//                  user keys of b carry the mask {b}); a warp takes 32-key
//                  tiles (cp.async, 3-stage ring per warp, XOR-swizzled rows)
//                  and runs S^T = K Q^T and O^T += V^T P^T on the tensor cores
//                  (mma.sync m16n8k16 bf16: M = 16 keys / 16 head dims, N =
//                  8 queries per tile) with the per-key query mask applied to
//                  S before the online softmax (log2 domain);
//                  each (segment, query) yields a normalised partial, and the
//                  CTA completing a row's last partial merges it.
// Every query attends exactly the keys of its own selection plus all n_u of
// its user keys: the result is the per-(b,h) attention of P:347-363, read
// with one pass over the union instead of B passes.  mma.sync (not tcgen05):
// the contraction per key is 16 x 128 -- tcgen05 tiles start at M = 64 -- and
// the pass is HBM-bound; the tensor cores only keep the ALU off the critical
// path (a CUDA-core version needs ~2000 FMA per key for B = 8).
#include <cstring>

#include "common.cuh"
#include "internal.h"
#include "tma.cuh"

namespace sqz {

namespace shd {
constexpr int D = 128;
// measured on cfg4 (same box): 32-key tiles x 4 warps 240 us, 16 x 8 warps 245 us,
// 16 x 6 warps x 4 stages 254 us, 16 x 4 warps x 6 stages 291 us; 32 x 6 x 2
// stages 248 us, 32 x 5 x 2 stages 241 us
#ifndef SQZ_SHD_NW
#define SQZ_SHD_NW 4
#endif
#ifndef SQZ_SHD_TK
#define SQZ_SHD_TK 32
#endif
#ifndef SQZ_SHD_NST
#define SQZ_SHD_NST 3
#endif
constexpr int NW = SQZ_SHD_NW;     // warps per CTA (one CTA per SM)
constexpr int NT = NW * 32;
static_assert(NT >= D, "the row merge gives one thread per head-dim column");
constexpr int TK = SQZ_SHD_TK;     // keys per warp tile (16 or 32)
constexpr int NST = SQZ_SHD_NST;   // ring stages per warp
// K/V tiles by TMA row gathers (tile::gather4, 4 rows x 128 B per op) instead of
// cp.async: correct, but measured 321 vs 239 us on cfg4 (32 small TMA ops per tile
// per warp; the engine's per-op cost dominates at 128-B rows) -- off
#ifndef SQZ_SHD_TMA
#define SQZ_SHD_TMA 0
#endif
static_assert(TK == 16 || TK == 32, "tile of 16 or 32 keys");
constexpr int ROWB = D * 2;        // 256 B per bf16 row
constexpr int TILEB = TK * ROWB;   // 4 KB: one K or V tile
constexpr int STAGEB = 2 * TILEB;  // K then V
constexpr int WARPB = NST * STAGEB;
constexpr int SMEM = NW * WARPB + 1024;  // 192 KB by default (+ 1 KB: SW128 tiles need 1024-B alignment)
static_assert(SMEM <= 200 * 1024 && SMEM >= NW * 16 * 128 * 4, "ring holds the merge buffer");
constexpr int SEG_KW = 256;        // partition cost of a segment's setup
constexpr int MIN_KEYS = 1024;     // minimum cost units per CTA
constexpr int MAXB = 16;
}  // namespace shd

struct ShdMaps {  // [rows][D] bf16 row tensors, box {64 cols, 1 row}, 128-B swizzle
    CUtensorMap kp, vp, ku, vu;
};

struct SharedArgs {
    const __nv_bfloat16 *Q, *Kp, *Vp, *Ku, *Vu;
    const int32_t *key_off;
    const int32_t *u_cl, *u_mask, *u_pref, *u_n, *u_keys;
    int32_t B, H, c2, n_u, partial, out_dtype, maxp;
    int64_t L;
    float scale;
    float *part_o, *part_lse;
    int32_t *row_cnt, *status;
    void *O;
    float *LSE;
};

namespace {
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
// D = A B + D, m16n8k16, bf16 inputs, fp32 accumulators
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// 8x8 b16 matrix transpose across the warp (lane l holds row l/4, elements 2(l%4), +1)
__device__ __forceinline__ uint32_t movmatrix_t(uint32_t x) {
    uint32_t y;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t *>(&v);
}
// byte offset of 16-byte chunk c (0..15) of row r of a K or V tile.  cp.async:
// 256-B rows, chunk XOR (row & 7).  TMA: two 64-column halves of 128-B rows with
// the hardware's 128-B swizzle (chunk XOR (row & 7) within each half).
__device__ __forceinline__ uint32_t swz(int r, int c) {
#if SQZ_SHD_TMA
    return (uint32_t)((c >> 3) * (shd::TK * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4));
#else
    return (uint32_t)(r * shd::ROWB + ((c ^ (r & 7)) << 4));
#endif
}

// warp window of 64 consecutive union runs with their query masks (cf. RunWin)
struct MWin {
    int J, end, p0, p1, s0, s1, m0, m1;
};
struct UList {
    const int32_t *cl, *pref, *koff, *mask;
    int n, nkf;
};
__device__ __forceinline__ void mwin_load(MWin &w, const UList &r, int J, int lane) {
    w.J = J;
    const int j0 = J + lane, j1 = J + 32 + lane;
    w.p0 = j0 < r.n ? ldcg(r.pref + j0) : 0x7fffffff;
    w.p1 = j1 < r.n ? ldcg(r.pref + j1) : 0x7fffffff;
    const int c0 = j0 < r.n ? ldcg(r.cl + j0) : 0, c1 = j1 < r.n ? ldcg(r.cl + j1) : 0;
    w.m0 = j0 < r.n ? ldcg(r.mask + j0) : 0;
    w.m1 = j1 < r.n ? ldcg(r.mask + j1) : 0;
    w.end = J + 64 < r.n ? ldcg(r.pref + J + 64) : r.nkf;
    w.s0 = j0 < r.n ? __ldg(r.koff + c0) : 0;
    w.s1 = j1 < r.n ? __ldg(r.koff + c1) : 0;
}
__device__ __forceinline__ void mwin_cover(MWin &w, const UList &r, int kmin, int kmax, int lane) {
    int first = __shfl_sync(FULL, w.p0, 0);
    if (kmin >= first && kmax < w.end) return;
    // a warp's tiles advance by NW * TK keys, so the next key usually lies just past
    // the window: try the following 64 runs (one round trip) before a full search
    if (w.end >= 0 && kmin >= w.end && w.J + 64 < r.n) {
        mwin_load(w, r, w.J + 64, lane);
        first = __shfl_sync(FULL, w.p0, 0);
        if (kmax < w.end) return;
    }
    int J;
    if (kmin >= first && kmin < w.end) {
        const unsigned b0 = __ballot_sync(FULL, w.p0 <= kmin), b1 = __ballot_sync(FULL, w.p1 <= kmin);
        J = w.J + __popc(b0) + __popc(b1) - 1;
    } else {
        int lo = 0, hi = r.n - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (ldcg(r.pref + mid) <= kmin) lo = mid;
            else hi = mid - 1;
        }
        J = lo;
    }
    mwin_load(w, r, J, lane);
}
// cluster-major position and query mask of stream key k (window covers k)
__device__ __forceinline__ void mwin_get(const MWin &w, int k, int &pos, int &msk) {
    int m = 0;
#pragma unroll
    for (int step = 32; step >= 1; step >>= 1) {
        const int cand = m + step;
        const int v0 = __shfl_sync(FULL, w.p0, cand & 31), v1 = __shfl_sync(FULL, w.p1, cand & 31);
        const int v = cand < 32 ? v0 : v1;
        if (cand < 64 && v <= k) m = cand;
    }
    const int q0 = __shfl_sync(FULL, w.p0, m & 31), q1 = __shfl_sync(FULL, w.p1, m & 31);
    const int t0 = __shfl_sync(FULL, w.s0, m & 31), t1 = __shfl_sync(FULL, w.s1, m & 31);
    const int k0 = __shfl_sync(FULL, w.m0, m & 31), k1 = __shfl_sync(FULL, w.m1, m & 31);
    pos = (m < 32 ? t0 : t1) + (k - (m < 32 ? q0 : q1));
    msk = m < 32 ? k0 : k1;
}
}  // namespace

// ---------------------------------------------------------------- union
// grid = H, block = 1024, dynamic smem = c2 * 4 bytes (the per-cluster masks)
__global__ void __launch_bounds__(1024) k_union(const int32_t *clusters, const int32_t *n_clusters,
                                                const int32_t *N2, int B, int H, int c2, int32_t *u_cl,
                                                int32_t *u_mask, int32_t *u_pref, int32_t *u_n,
                                                int32_t *u_keys) {
    extern __shared__ uint32_t s_mask[];
    __shared__ int s_w[32], s_wk[32], s_carry, s_carryk;
    griddep_wait();  // the lookup's selection
    const int h = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < c2; i += blockDim.x) s_mask[i] = 0u;
    if (tid == 0) s_carry = s_carryk = 0;
    __syncthreads();
    for (int b = 0; b < B; ++b) {
        const int bh = b * H + h, n = n_clusters[bh];
        const int32_t *cl = clusters + (size_t)bh * c2;
        for (int e = tid; e < n; e += blockDim.x) atomicOr(s_mask + cl[e], 1u << b);
    }
    __syncthreads();
    const int32_t *N = N2 + (size_t)h * c2;
    int32_t *ocl = u_cl + (size_t)h * c2, *omk = u_mask + (size_t)h * c2, *opr = u_pref + (size_t)h * c2;
    const int nwarps = blockDim.x >> 5;
    for (int base = 0; base < c2; base += blockDim.x) {
        const int i = base + tid;
        const uint32_t m = i < c2 ? s_mask[i] : 0u;
        const bool sel = m != 0u;
        const int nk = sel ? N[i] : 0;
        const unsigned bal = __ballot_sync(FULL, sel);
        int inc = nk;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) {
            s_w[warp] = __popc(bal);
            s_wk[warp] = inc;
        }
        __syncthreads();
        int wb = 0, kb = 0, tc = 0, tk = 0;
        for (int w = 0; w < nwarps; ++w) {
            if (w < warp) {
                wb += s_w[w];
                kb += s_wk[w];
            }
            tc += s_w[w];
            tk += s_wk[w];
        }
        const int cb = s_carry, ckb = s_carryk;
        if (sel) {
            const int pos = cb + wb + __popc(bal & ((1u << lane) - 1u));
            ocl[pos] = i;
            omk[pos] = (int32_t)m;
            opr[pos] = ckb + kb + inc - nk;
        }
        __syncthreads();
        if (tid == 0) {
            s_carry = cb + tc;
            s_carryk = ckb + tk;
        }
        __syncthreads();
    }
    if (tid == 0) {
        u_n[h] = s_carry;
        u_keys[h] = s_carryk;
    }
}

// --------------------------------------------------------- merge helpers
// Merge of a row's P partials into O / LSE; thread k < D owns column k.
__device__ void shd_merge_row(const SharedArgs &a, int row, int P) {
    constexpr int MB = 16;
    const int tid = threadIdx.x;
    if (tid >= shd::D) return;
    const float *lse = a.part_lse + (size_t)row * a.maxp;
    const float *op = a.part_o + (size_t)row * a.maxp * shd::D + tid;
    float M = -INFINITY, L = 0.f, acc = 0.f;
    for (int p0 = 0; p0 < P; p0 += MB) {
        float lv[MB], ov[MB];
#pragma unroll
        for (int j = 0; j < MB; ++j) {
            const bool in = p0 + j < P;
            lv[j] = in ? ldcg(lse + p0 + j) : -INFINITY;
            ov[j] = in ? ldcg(op + (size_t)(p0 + j) * shd::D) : 0.f;
        }
        float mt = M;
#pragma unroll
        for (int j = 0; j < MB; ++j) mt = fmaxf(mt, lv[j]);
        if (mt == -INFINITY) continue;
        const float corr = expf(M - mt);
        L *= corr;
        acc *= corr;
#pragma unroll
        for (int j = 0; j < MB; ++j) {
            const float w = expf(lv[j] - mt);
            L += w;
            acc = fmaf(w, ov[j], acc);
        }
        M = mt;
    }
    const float v = (M == -INFINITY) ? 0.f : acc / L;
    if (a.out_dtype == SQZ_BF16)
        reinterpret_cast<__nv_bfloat16 *>(a.O)[(size_t)row * shd::D + tid] = __float2bfloat16_rn(v);
    else
        reinterpret_cast<float *>(a.O)[(size_t)row * shd::D + tid] = v;
    if (tid == 0) {
        a.LSE[row] = (M == -INFINITY) ? -INFINITY : M + logf(L);
        if (M == -INFINITY && !a.partial) atomicOr(a.status, 1);
    }
}

// ------------------------------------------------------------- attention
// NQ8 = query tiles of 8 (B <= 8: 1, B <= 16: 2).  The contractions run
// TRANSPOSED -- S^T = K Q^T (M = 16 keys, N = 8 queries) and O^T += V^T P^T
// (M = 16 head dims) -- so no MMA row is padding when B <= 8 and the
// accumulators are 32 registers per query tile; P^T is formed from the S^T
// fragment with movmatrix (an 8x8 b16 transpose in registers).
template <int NQ8>
__global__ void __launch_bounds__(shd::NT, 1) k_attend_shared(SharedArgs a, const __grid_constant__ ShdMaps maps) {
    using namespace shd;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ long long s_pref[1025];  // per-head cost prefix
    __shared__ float s_m[NW][MAXB], s_l[NW][MAXB];
    __shared__ int s_last[MAXB];
    __shared__ int s_tm[NW][NST][TK];  // query mask of each key of each stage's tile
    __shared__ __align__(8) uint64_t s_bar[NW][NST];  // TMA: stage landed (bytes counted)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const int B = a.B, H = a.H;
#if SQZ_SHD_TMA
    if (lane == 0) {
        for (int st = 0; st < NST; ++st) mbar_init(&s_bar[warp][st], 1);
        mbar_fence_init();
    }
    __syncwarp();
    int tiles_done = 0;  // this warp's tiles so far (stage / phase of its ring)
#endif
    griddep_wait();  // the union lists
    const long long ucost = (long long)B * a.n_u;
    if (tid == 0) s_pref[0] = 0;
    // per-head cost: union keys + B * n_u user keys + the segment setup allowance
    for (int base = 0; base < H; base += NT) {
        __syncthreads();
        if (tid == 0) {
            long long c = s_pref[base];
            for (int h = base; h < min(H, base + NT); ++h) {
                const long long nk = (long long)ldcg(a.u_keys + h) + ucost;
                c += nk > 0 ? nk + SEG_KW : 0;
                s_pref[h + 1] = c;
            }
        }
    }
    __syncthreads();
    const long long K = s_pref[H];
    const int G = gridDim.x, j = blockIdx.x;
    const int Gp = (int)min((long long)G, max(1LL, (K + MIN_KEYS - 1) / MIN_KEYS));
    auto cta_of = [&](long long x) { return (int)(((x + 1) * (long long)Gp - 1) / K); };
    auto nparts = [&](int h) {
        const long long cs = s_pref[h], re = s_pref[h + 1];
        if (re == cs) return 1;
        return cta_of(re - 1) - cta_of(cs + SEG_KW) + 1;
    };
    // heads without any key: an identity partial per row (one per head, CTA h mod G)
    for (int h = j; h < H; h += G)
        if (s_pref[h + 1] == s_pref[h]) {
            for (int b = 0; b < B; ++b) {
                const int row = b * H + h;
                const size_t sl = (size_t)row * a.maxp;
                for (int k = tid; k < D; k += NT) a.part_o[sl * D + k] = 0.f;
                if (tid == 0) a.part_lse[sl] = -INFINITY;
            }
            __syncthreads();
            if (tid < B) {
                const int row = tid * H + h;
                s_last[tid] = ticket_acq_rel(a.row_cnt + row) == 0;
                if (s_last[tid]) a.row_cnt[row] = 0;
            }
            __syncthreads();
            for (int b = 0; b < B; ++b)
                if (s_last[b]) shd_merge_row(a, b * H + h, 1);
            __syncthreads();
        }
    if (j >= Gp || K == 0) return;
    const long long ks = (long long)j * K / Gp, ke = (long long)(j + 1) * K / Gp;
    int lo = 0, hi = H - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_pref[mid] <= ks) lo = mid;
        else hi = mid - 1;
    }
    const float sl2 = a.scale * LOG2E;
    unsigned char *wsm = reinterpret_cast<unsigned char *>(((uintptr_t)smem + 1023) & ~(uintptr_t)1023) +
                         warp * WARPB;
    const uint32_t wbase = smem_addr(wsm);
    for (int h = lo; h < H && s_pref[h] < ke; ++h) {
        const long long cs = s_pref[h], re = s_pref[h + 1], rs = cs + SEG_KW;
        if (re <= ks || re == cs || ke <= rs) continue;
        const int a0 = (int)(max(ks, rs) - rs), a1 = (int)(min(ke, re) - rs);
        const int slot = j - cta_of(rs);
        UList ul;
        ul.cl = a.u_cl + (size_t)h * a.c2;
        ul.pref = a.u_pref + (size_t)h * a.c2;
        ul.mask = a.u_mask + (size_t)h * a.c2;
        ul.koff = a.key_off + (size_t)h * (a.c2 + 1);
        ul.n = ldcg(a.u_n + h);
        ul.nkf = ldcg(a.u_keys + h);
        const int KU = ul.nkf;
        const __nv_bfloat16 *Kf = a.Kp + (size_t)h * a.L * D, *Vf = a.Vp + (size_t)h * a.L * D;
        // Q^T fragments (B operand of S^T = K Q^T): query nq*8 + g, dims kk*16 + 2t4 (+8)
        uint32_t qb[NQ8][8][2];
#pragma unroll
        for (int nq = 0; nq < NQ8; ++nq) {
            const int q = nq * 8 + g;
            const bool ok = q < B;
            const uint32_t *qp = reinterpret_cast<const uint32_t *>(a.Q + ((size_t)q * H + h) * D);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                qb[nq][kk][0] = ok ? __ldg(qp + kk * 8 + t4) : 0u;
                qb[nq][kk][1] = ok ? __ldg(qp + kk * 8 + 4 + t4) : 0u;
            }
        }
        // O^T accumulators: dim tile n (dims 16n + g, 16n + g + 8) x queries nq*8 + 2t4 + {0,1}
        float o[NQ8][8][4];
#pragma unroll
        for (int nq = 0; nq < NQ8; ++nq)
#pragma unroll
            for (int n = 0; n < 8; ++n) o[nq][n][0] = o[nq][n][1] = o[nq][n][2] = o[nq][n][3] = 0.f;
        float m_r[NQ8][2], l_r[NQ8][2];
#pragma unroll
        for (int nq = 0; nq < NQ8; ++nq) m_r[nq][0] = m_r[nq][1] = -INFINITY, l_r[nq][0] = l_r[nq][1] = 0.f;
        MWin win;
        win.J = 0;
        win.end = -1;
        win.p0 = win.p1 = 0x7fffffff;
        win.m0 = win.m1 = 0;
        const int ntile = (a1 - a0 + TK - 1) / TK;
        // issue the cp.async copies of warp-tile i (tile a0 + (warp + i * NW) * TK) into stage st
        auto issue = [&](int i, int st) {
            const int k0 = a0 + (warp + i * NW) * TK;
            const int kl = min(k0 + TK, a1) - 1;  // last valid key of the tile
            const int myk = min(k0 + (lane & (TK - 1)), kl);
            if (k0 < KU) mwin_cover(win, ul, k0, min(kl, KU - 1), lane);
            int pos = 0, msk = 0;
            if (k0 < KU) mwin_get(win, min(myk, KU - 1), pos, msk);
#if SQZ_SHD_TMA
            // row of the key in the fixed [H*L] or the user [B*H*n_u] row tensor
            int row, usr;
            if (myk < KU) {
                row = h * (int)a.L + pos;
                usr = 0;
            } else {
                const int u = myk - KU, b = u / a.n_u, uu = u - b * a.n_u;
                msk = 1 << b;
                row = (b * H + h) * a.n_u + uu;
                usr = 1;
            }
            if (k0 + (lane & (TK - 1)) > kl) msk = 0;  // past the segment end: masked for every query
            if (lane < TK) s_tm[warp][st][lane] = msk;
            const uint32_t sK = wbase + st * STAGEB, sV = sK + TILEB;
            uint64_t *bar = &s_bar[warp][st];
            if (lane == 0) mbar_arrive_expect_tx(bar, STAGEB);
            // lane l < TK/4 gathers keys 4l .. 4l+3 (both halves of K and V rows)
            int rr[4], us[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                rr[j] = __shfl_sync(FULL, row, (4 * lane + j) & (TK - 1));
                us[j] = __shfl_sync(FULL, usr, (4 * lane + j) & (TK - 1));
            }
            if (lane < TK / 4) {
                const int u0 = us[0] + us[1] + us[2] + us[3];
                const uint32_t ro = (uint32_t)(4 * lane) * 128;
                if (u0 == 0 || u0 == 4) {
                    const void *mk = u0 ? (const void *)&maps.ku : (const void *)&maps.kp;
                    const void *mv = u0 ? (const void *)&maps.vu : (const void *)&maps.vp;
#pragma unroll
                    for (int hb = 0; hb < 2; ++hb) {
                        tma_gather4(sK + hb * (TK * 128) + ro, mk, hb * 64, rr[0], rr[1], rr[2], rr[3], bar);
                        tma_gather4(sV + hb * (TK * 128) + ro, mv, hb * 64, rr[0], rr[1], rr[2], rr[3], bar);
                    }
                } else {  // fixed and user rows in one group: one row per load
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const void *mk = us[j] ? (const void *)&maps.ku : (const void *)&maps.kp;
                        const void *mv = us[j] ? (const void *)&maps.vu : (const void *)&maps.vp;
#pragma unroll
                        for (int hb = 0; hb < 2; ++hb) {
                            tma_load_2d(sK + hb * (TK * 128) + ro + j * 128, mk, hb * 64, rr[j], bar);
                            tma_load_2d(sV + hb * (TK * 128) + ro + j * 128, mv, hb * 64, rr[j], bar);
                        }
                    }
                }
            }
#else
            const __nv_bfloat16 *kr, *vr;
            if (myk < KU) {
                kr = Kf + (size_t)pos * D;
                vr = Vf + (size_t)pos * D;
            } else {
                const int u = myk - KU, b = u / a.n_u, uu = u - b * a.n_u;
                msk = 1 << b;
                kr = a.Ku + (((size_t)b * H + h) * a.n_u + uu) * D;
                vr = a.Vu + (((size_t)b * H + h) * a.n_u + uu) * D;
            }
            if (k0 + (lane & (TK - 1)) > kl) msk = 0;  // past the segment end: masked for every query
            if (lane < TK) s_tm[warp][st][lane] = msk;
            const uint32_t sK = wbase + st * STAGEB, sV = sK + TILEB;
            const int c = lane & 15;
#pragma unroll
            for (int it = 0; it < TK / 2; ++it) {
                const int r = it * 2 + (lane >> 4);
                const uint64_t kp = __shfl_sync(FULL, (uint64_t)kr, r);
                const uint64_t vp = __shfl_sync(FULL, (uint64_t)vr, r);
                cp16(sK + swz(r, c), reinterpret_cast<const char *>(kp) + c * 16);
                cp16(sV + swz(r, c), reinterpret_cast<const char *>(vp) + c * 16);
            }
#endif
        };
        const int my_tiles = ntile > warp ? (ntile - warp + NW - 1) / NW : 0;
#if SQZ_SHD_TMA
        // stage of this warp's tile i: its ring continues across segments
        const int tb = tiles_done;
        tiles_done += my_tiles;
#pragma unroll
        for (int i = 0; i < NST - 1; ++i)
            if (i < my_tiles) issue(i, (tb + i) % NST);
        for (int i = 0; i < my_tiles; ++i) {
            const int st = (tb + i) % NST;
            if (i + NST - 1 < my_tiles) issue(i + NST - 1, (tb + i + NST - 1) % NST);
            mbar_wait(&s_bar[warp][st], ((tb + i) / NST) & 1);
#else
        // prologue: the first NST - 1 tiles of this warp
#pragma unroll
        for (int i = 0; i < NST - 1; ++i) {
            if (i < my_tiles) issue(i, i);
            cp_commit();
        }
        for (int i = 0; i < my_tiles; ++i) {
            const int st = i % NST;
            if (i + NST - 1 < my_tiles) issue(i + NST - 1, (i + NST - 1) % NST);
            cp_commit();
            cp_wait<NST - 1>();
            __syncwarp();
#endif
            const uint32_t sK = wbase + st * STAGEB, sV = sK + TILEB;
            // ---- S^T = K Q^T: NMT m-tiles of 16 keys ----
            constexpr int NMT = TK / 16;
            float sv[NMT][NQ8][4];
#pragma unroll
            for (int mt = 0; mt < NMT; ++mt)
#pragma unroll
                for (int nq = 0; nq < NQ8; ++nq) sv[mt][nq][0] = sv[mt][nq][1] = sv[mt][nq][2] = sv[mt][nq][3] = 0.f;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
                for (int mt = 0; mt < NMT; ++mt) {
                    // A = K rows: (keys 0-7, k lo), (keys 8-15, k lo), (0-7, k hi), (8-15, k hi)
                    const int mi = lane >> 3, r = mt * 16 + (mi & 1) * 8 + (lane & 7), c = kk * 2 + (mi >> 1);
                    uint32_t a0, a1, a2, a3;
                    ldsm_x4(sK + swz(r, c), a0, a1, a2, a3);
#pragma unroll
                    for (int nq = 0; nq < NQ8; ++nq)
                        mma16816(sv[mt][nq], a0, a1, a2, a3, qb[nq][kk][0], qb[nq][kk][1]);
                }
            }
            // ---- query mask, online softmax per query column (keys g, g + 8 of each m-tile) ----
            int km[NMT][2];
#pragma unroll
            for (int mt = 0; mt < NMT; ++mt) {
                km[mt][0] = s_tm[warp][st][mt * 16 + g];
                km[mt][1] = s_tm[warp][st][mt * 16 + g + 8];
            }
            uint32_t pb[NMT][NQ8][2];  // P^T fragments (B operand of O^T += V^T P^T)
#pragma unroll
            for (int nq = 0; nq < NQ8; ++nq) {
                float pv[NMT][4];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int q = nq * 8 + 2 * t4 + e;
                    float v[NMT][2];
                    float mx = -INFINITY;
#pragma unroll
                    for (int mt = 0; mt < NMT; ++mt) {
                        v[mt][0] = ((km[mt][0] >> q) & 1) ? sv[mt][nq][e] * sl2 : -INFINITY;
                        v[mt][1] = ((km[mt][1] >> q) & 1) ? sv[mt][nq][2 + e] * sl2 : -INFINITY;
                        mx = fmaxf(mx, fmaxf(v[mt][0], v[mt][1]));
                    }
                    mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, 4));
                    mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, 8));
                    mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, 16));
                    const float mn = fmaxf(m_r[nq][e], mx);
                    float alpha = 1.f, ps = 0.f;
#pragma unroll
                    for (int mt = 0; mt < NMT; ++mt) {
                        const float p0 = mn == -INFINITY ? 0.f : fast_exp2(v[mt][0] - mn);
                        const float p1 = mn == -INFINITY ? 0.f : fast_exp2(v[mt][1] - mn);
                        pv[mt][e] = p0;
                        pv[mt][2 + e] = p1;
                        ps += p0 + p1;
                    }
                    if (mn != -INFINITY) alpha = fast_exp2(m_r[nq][e] - mn);  // exp2(-inf) = 0
                    l_r[nq][e] = l_r[nq][e] * alpha + ps;
                    m_r[nq][e] = mn;
#pragma unroll
                    for (int n = 0; n < 8; ++n) {
                        o[nq][n][e] *= alpha;
                        o[nq][n][2 + e] *= alpha;
                    }
                }
#pragma unroll
                for (int mt = 0; mt < NMT; ++mt) {
                    // (key g, queries 2t4..) -> transpose -> (query g, keys 2t4..)
                    pb[mt][nq][0] = movmatrix_t(pack_bf16(pv[mt][0], pv[mt][1]));
                    pb[mt][nq][1] = movmatrix_t(pack_bf16(pv[mt][2], pv[mt][3]));
                }
            }
            // ---- O^T += V^T P^T: A = V^T via ldmatrix.trans, per 16-dim tile and 16-key step ----
#pragma unroll
            for (int mt = 0; mt < NMT; ++mt) {
#pragma unroll
                for (int n = 0; n < 8; ++n) {
                    // matrices: (keys 0-7, dims lo), (keys 0-7, dims hi), (keys 8-15, lo), (8-15, hi)
                    const int mi = lane >> 3, r = mt * 16 + (mi >> 1) * 8 + (lane & 7), c = n * 2 + (mi & 1);
                    uint32_t a0, a1, a2, a3;
                    ldsm_x4_t(sV + swz(r, c), a0, a1, a2, a3);
#pragma unroll
                    for (int nq = 0; nq < NQ8; ++nq)
                        mma16816(o[nq][n], a0, a1, a2, a3, pb[mt][nq][0], pb[mt][nq][1]);
                }
            }
            __syncwarp();  // the stage is refilled by the next issue
        }
#if !SQZ_SHD_TMA
        cp_wait<0>();
#endif
        // ---- combine the warps' states; one partial per query row ----
        float lr[NQ8][2];
#pragma unroll
        for (int nq = 0; nq < NQ8; ++nq)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                float v = l_r[nq][e];
                v += __shfl_xor_sync(FULL, v, 4);
                v += __shfl_xor_sync(FULL, v, 8);
                v += __shfl_xor_sync(FULL, v, 16);
                lr[nq][e] = v;
            }
        __syncthreads();  // every warp is done with its ring: reuse it for the states
        float *so = reinterpret_cast<float *>(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);  // [NW][MAXB][D]
#pragma unroll
        for (int nq = 0; nq < NQ8; ++nq)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int q = nq * 8 + 2 * t4 + e;
                if (g == 0) {
                    s_m[warp][q] = m_r[nq][e];
                    s_l[warp][q] = lr[nq][e];
                }
#pragma unroll
                for (int n = 0; n < 8; ++n) {
                    so[(warp * MAXB + q) * D + n * 16 + g] = o[nq][n][e];
                    so[(warp * MAXB + q) * D + n * 16 + g + 8] = o[nq][n][2 + e];
                }
            }
        __syncthreads();
        for (int e = tid; e < B * D; e += NT) {
            const int b = e / D, col = e - b * D;
            float M = -INFINITY;
#pragma unroll
            for (int w = 0; w < NW; ++w) M = fmaxf(M, s_m[w][b]);
            float L = 0.f, O = 0.f;
            if (M != -INFINITY) {
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    const float ew = s_m[w][b] == -INFINITY ? 0.f : fast_exp2(s_m[w][b] - M);
                    L += s_l[w][b] * ew;
                    O += so[(w * MAXB + b) * D + col] * ew;
                }
            }
            const size_t sl = (size_t)(b * H + h) * a.maxp + slot;
            a.part_o[sl * D + col] = L > 0.f ? O / L : 0.f;
            if (col == 0) a.part_lse[sl] = L > 0.f ? (M + log2f(L)) * LN2 : -INFINITY;
        }
        __syncthreads();
        const int total = nparts(h);
        if (tid < B) {
            const int row = tid * H + h;
            const int tk = ticket_acq_rel(a.row_cnt + row);
            s_last[tid] = tk == total - 1;
            if (s_last[tid]) a.row_cnt[row] = 0;
        }
        __syncthreads();
        for (int b = 0; b < B; ++b)
            if (s_last[b]) shd_merge_row(a, b * H + h, total);
        __syncthreads();
#if SQZ_SHD_TMA
        // the ring held the merge buffer (generic stores): order them before the
        // next segment's TMA writes (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
    }
}

// ---------------------------------------------------------------- host
size_t shared_attn_ws_bytes(int B, int H, int c2) {
    const size_t G = 1184;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t rows = (size_t)B * H, maxp = G + 1;
    return 3 * al((size_t)H * c2 * 4) + 2 * al((size_t)H * 4) + al(rows * 4) + al(rows * maxp * 4) +
           al(rows * maxp * shd::D * 4) + 512;
}

bool shared_attn_applies(int B, int n_q, int d, int dtype, int c2) {
    return n_q == 1 && B >= 2 && B <= shd::MAXB && d == 128 && dtype == SQZ_BF16 && c2 <= 56 * 1024;
}

cudaError_t launch_attention_shared(const AttnArgs &x, cudaStream_t st) {
    SharedArgs a;
    std::memset(&a, 0, sizeof(a));
    auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
    char *p = reinterpret_cast<char *>(x.shared_ws);
    const size_t H = x.H, c2 = x.c2, rows = (size_t)x.B * x.H;
    int32_t *u_cl = reinterpret_cast<int32_t *>(p); p += al(H * c2 * 4);
    int32_t *u_mask = reinterpret_cast<int32_t *>(p); p += al(H * c2 * 4);
    int32_t *u_pref = reinterpret_cast<int32_t *>(p); p += al(H * c2 * 4);
    int32_t *u_n = reinterpret_cast<int32_t *>(p); p += al(H * 4);
    int32_t *u_keys = reinterpret_cast<int32_t *>(p); p += al(H * 4);
    int32_t *row_cnt = reinterpret_cast<int32_t *>(p); p += al(rows * 4);
    const int G = std::min(device_sm_count(), 1184);
    a.maxp = G + 1;
    float *part_lse = reinterpret_cast<float *>(p); p += al(rows * 1185 * 4);
    float *part_o = reinterpret_cast<float *>(p);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(x.H);
        cfg.blockDim = dim3(1024);
        cfg.dynamicSmemBytes = c2 * 4;
        cfg.stream = st;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (cfg.dynamicSmemBytes > 48 * 1024) {
            cudaError_t e = ensure_func_attr((const void *)k_union, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)cfg.dynamicSmemBytes);
            if (e != cudaSuccess) return e;
        }
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_union, x.sel_cl, x.sel_n, x.N2, x.B, x.H, x.c2, u_cl,
                                           u_mask, u_pref, u_n, u_keys);
        if (e != cudaSuccess) return e;
    }
    a.Q = reinterpret_cast<const __nv_bfloat16 *>(x.Q);
    a.Kp = reinterpret_cast<const __nv_bfloat16 *>(x.Kp);
    a.Vp = reinterpret_cast<const __nv_bfloat16 *>(x.Vp);
    a.Ku = reinterpret_cast<const __nv_bfloat16 *>(x.Ku);
    a.Vu = reinterpret_cast<const __nv_bfloat16 *>(x.Vu);
    a.key_off = x.key_off;
    a.u_cl = u_cl; a.u_mask = u_mask; a.u_pref = u_pref; a.u_n = u_n; a.u_keys = u_keys;
    a.B = x.B; a.H = x.H; a.c2 = x.c2; a.n_u = x.Ku ? x.n_u : 0; a.partial = x.partial;
    a.out_dtype = x.out_dtype; a.L = x.L; a.scale = x.scale;
    a.part_o = part_o; a.part_lse = part_lse; a.row_cnt = row_cnt; a.status = x.status;
    a.O = x.O; a.LSE = x.LSE;
    ShdMaps maps;
    std::memset(&maps, 0, sizeof(maps));
#if SQZ_SHD_TMA
    {
        const uint64_t rf = (uint64_t)x.H * x.L, ru = (uint64_t)x.B * x.H * (x.n_u > 0 ? x.n_u : 1);
        if (encode_tmap_bf16_2d(&maps.kp, x.Kp, shd::D, rf, 64, 1) != 0 ||
            encode_tmap_bf16_2d(&maps.vp, x.Vp, shd::D, rf, 64, 1) != 0)
            return cudaErrorInvalidValue;
        const void *ku = x.Ku && x.n_u > 0 ? x.Ku : x.Kp, *vu = x.Vu && x.n_u > 0 ? x.Vu : x.Vp;
        if (encode_tmap_bf16_2d(&maps.ku, ku, shd::D, x.Ku && x.n_u > 0 ? ru : rf, 64, 1) != 0 ||
            encode_tmap_bf16_2d(&maps.vu, vu, shd::D, x.Vu && x.n_u > 0 ? ru : rf, 64, 1) != 0)
            return cudaErrorInvalidValue;
    }
#endif
    auto kern = x.B <= 8 ? k_attend_shared<1> : k_attend_shared<2>;
    cudaError_t e = ensure_func_attr((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, shd::SMEM);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(shd::NT);
    cfg.dynamicSmemBytes = shd::SMEM;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a, maps);
}

}  // namespace sqz
