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
//                  and runs S = Q K^T and O += P V on the tensor cores
//                  (mma.sync m16n8k16 bf16: M = the up-to-16 queries of the
//                  head, N = keys / head dims) with the per-key query mask
//                  applied to S before the online softmax (log2 domain);
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

namespace sqz {

namespace shd {
constexpr int D = 128;
// measured on cfg4 (same box): 32-key tiles x 4 warps 240 us, 16 x 8 warps 245 us,
// 16 x 6 warps x 4 stages 254 us, 16 x 4 warps x 6 stages 291 us
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
constexpr int TK = SQZ_SHD_TK;     // keys per warp tile (16 or 32)
constexpr int NST = SQZ_SHD_NST;   // ring stages per warp
constexpr int NB8 = TK / 8;        // n8 key tiles of S per warp tile
static_assert(TK == 16 || TK == 32, "tile of 16 or 32 keys");
constexpr int ROWB = D * 2;        // 256 B per bf16 row
constexpr int TILEB = TK * ROWB;   // 4 KB: one K or V tile
constexpr int STAGEB = 2 * TILEB;  // K then V
constexpr int WARPB = NST * STAGEB;
constexpr int SMEM = NW * WARPB;   // 192 KB by default
static_assert(SMEM <= 200 * 1024 && SMEM >= NW * 16 * 128 * 4, "ring holds the merge buffer");
constexpr int SEG_KW = 256;        // partition cost of a segment's setup
constexpr int MIN_KEYS = 1024;     // minimum cost units per CTA
constexpr int MAXB = 16;
}  // namespace shd

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
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t *>(&v);
}
// byte offset of 16-byte chunk c (0..15) of row r in a swizzled 256-byte-row tile
__device__ __forceinline__ uint32_t swz(int r, int c) { return (uint32_t)(r * shd::ROWB + ((c ^ (r & 7)) << 4)); }

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
__global__ void __launch_bounds__(shd::NT, 1) k_attend_shared(SharedArgs a) {
    using namespace shd;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ long long s_pref[1025];  // per-head cost prefix
    __shared__ float s_m[NW][MAXB], s_l[NW][MAXB];
    __shared__ int s_last[MAXB];
    __shared__ int s_tm[NW][NST][TK];  // query mask of each key of each stage's tile
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const int B = a.B, H = a.H;
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
    unsigned char *wsm = smem + warp * WARPB;
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
        // Q fragments (A operand of S = Q K^T): rows g and g + 8 are queries b = g, g + 8
        uint32_t qa[8][4];
        {
            const bool r0 = g < B, r1 = g + 8 < B;
            const uint32_t *q0 = reinterpret_cast<const uint32_t *>(a.Q + ((size_t)g * H + h) * D);
            const uint32_t *q1 = reinterpret_cast<const uint32_t *>(a.Q + ((size_t)(g + 8) * H + h) * D);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                qa[kk][0] = r0 ? __ldg(q0 + kk * 8 + t4) : 0u;
                qa[kk][1] = r1 ? __ldg(q1 + kk * 8 + t4) : 0u;
                qa[kk][2] = r0 ? __ldg(q0 + kk * 8 + 4 + t4) : 0u;
                qa[kk][3] = r1 ? __ldg(q1 + kk * 8 + 4 + t4) : 0u;
            }
        }
        float o[16][4];
#pragma unroll
        for (int n = 0; n < 16; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
        float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
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
        };
        const int my_tiles = ntile > warp ? (ntile - warp + NW - 1) / NW : 0;
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
            const uint32_t sK = wbase + st * STAGEB, sV = sK + TILEB;
            // ---- S = Q K^T: NB8 n8 tiles of keys ----
            // two accumulator sets (even / odd k-steps) halve the dependent HMMA chain
            float s[NB8][4], s2[NB8][4];
#pragma unroll
            for (int nt = 0; nt < NB8; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) s[nt][e] = s2[nt][e] = 0.f;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
                for (int pr = 0; pr < NB8 / 2; ++pr) {
                    // matrices: (keys 16pr+0-7, dims lo), (same keys, dims hi), (keys 16pr+8-15, lo), (hi)
                    const int mi = lane >> 3, r = pr * 16 + (mi >> 1) * 8 + (lane & 7), c = kk * 2 + (mi & 1);
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4(sK + swz(r, c), b0, b1, b2, b3);
                    float(&d0)[4] = (kk & 1) ? s2[2 * pr] : s[2 * pr];
                    float(&d1)[4] = (kk & 1) ? s2[2 * pr + 1] : s[2 * pr + 1];
                    mma16816(d0, qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b0, b1);
                    mma16816(d1, qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b2, b3);
                }
            }
#pragma unroll
            for (int nt = 0; nt < NB8; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) s[nt][e] += s2[nt][e];
            // ---- mask, online softmax (rows g, g + 8; keys 8j + 2t4, 8j + 2t4 + 1) ----
            int mk[NB8][2];
#pragma unroll
            for (int jt = 0; jt < NB8; ++jt) {
                mk[jt][0] = s_tm[warp][st][jt * 8 + 2 * t4];
                mk[jt][1] = s_tm[warp][st][jt * 8 + 2 * t4 + 1];
            }
            float p[NB8][4];
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const int q = g + rr * 8;
                float v[NB8][2];
                float mx = -INFINITY;
#pragma unroll
                for (int jt = 0; jt < NB8; ++jt) {
                    v[jt][0] = ((mk[jt][0] >> q) & 1) ? s[jt][rr * 2] * sl2 : -INFINITY;
                    v[jt][1] = ((mk[jt][1] >> q) & 1) ? s[jt][rr * 2 + 1] * sl2 : -INFINITY;
                    mx = fmaxf(mx, fmaxf(v[jt][0], v[jt][1]));
                }
                mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, 1));
                mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, 2));
                const float mn = fmaxf(m_r[rr], mx);
                float alpha = 1.f, ps = 0.f;
#pragma unroll
                for (int jt = 0; jt < NB8; ++jt) {
                    if (mn == -INFINITY) {
                        p[jt][rr * 2] = p[jt][rr * 2 + 1] = 0.f;
                    } else {
                        p[jt][rr * 2] = fast_exp2(v[jt][0] - mn);
                        p[jt][rr * 2 + 1] = fast_exp2(v[jt][1] - mn);
                    }
                    ps += p[jt][rr * 2] + p[jt][rr * 2 + 1];
                }
                if (mn != -INFINITY) alpha = fast_exp2(m_r[rr] - mn);  // exp2(-inf) = 0 for a first key
                l_r[rr] = l_r[rr] * alpha + ps;
                m_r[rr] = mn;
#pragma unroll
                for (int n = 0; n < 16; ++n) {
                    o[n][rr * 2] *= alpha;
                    o[n][rr * 2 + 1] *= alpha;
                }
            }
            // ---- O += P V: A = P (rows g, g+8; 16 keys per k-step), B = V via ldmatrix.trans ----
#pragma unroll
            for (int kc = 0; kc < TK / 16; ++kc) {
                const uint32_t pa0 = pack_bf16(p[2 * kc][0], p[2 * kc][1]);
                const uint32_t pa1 = pack_bf16(p[2 * kc][2], p[2 * kc][3]);
                const uint32_t pa2 = pack_bf16(p[2 * kc + 1][0], p[2 * kc + 1][1]);
                const uint32_t pa3 = pack_bf16(p[2 * kc + 1][2], p[2 * kc + 1][3]);
#pragma unroll
                for (int n2 = 0; n2 < 8; ++n2) {
                    // matrices: (keys 16kc+0-7, dims 16n2..+7), (keys +8-15, same), (0-7, +8..), (8-15, +8..)
                    const int mi = lane >> 3, r = kc * 16 + (mi & 1) * 8 + (lane & 7), c = n2 * 2 + (mi >> 1);
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4_t(sV + swz(r, c), b0, b1, b2, b3);
                    mma16816(o[2 * n2], pa0, pa1, pa2, pa3, b0, b1);
                    mma16816(o[2 * n2 + 1], pa0, pa1, pa2, pa3, b2, b3);
                }
            }
            __syncwarp();  // the stage is refilled by the next issue
        }
        cp_wait<0>();
        // ---- combine the warps' states; one partial per query row ----
        float lr[2];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            float v = l_r[rr];
            v += __shfl_xor_sync(FULL, v, 1);
            v += __shfl_xor_sync(FULL, v, 2);
            lr[rr] = v;
        }
        __syncthreads();  // every warp is done with its ring: reuse it for the states
        float *so = reinterpret_cast<float *>(smem);  // [NW][MAXB][D]
        if (t4 == 0) {
            s_m[warp][g] = m_r[0];
            s_l[warp][g] = lr[0];
            s_m[warp][g + 8] = m_r[1];
            s_l[warp][g + 8] = lr[1];
        }
#pragma unroll
        for (int n = 0; n < 16; ++n) {
            const int col = n * 8 + 2 * t4;
            so[(warp * MAXB + g) * D + col] = o[n][0];
            so[(warp * MAXB + g) * D + col + 1] = o[n][1];
            so[(warp * MAXB + g + 8) * D + col] = o[n][2];
            so[(warp * MAXB + g + 8) * D + col + 1] = o[n][3];
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
    cudaError_t e = ensure_func_attr((const void *)k_attend_shared, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     shd::SMEM);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(shd::NT);
    cfg.dynamicSmemBytes = shd::SMEM;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_attend_shared, a);
}

}  // namespace sqz
