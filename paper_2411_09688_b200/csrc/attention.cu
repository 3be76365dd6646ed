// attention.cu -- sparse attention over the selected fixed-context keys plus
// the user KV (section 4.2), split-KV + merge, one kernel launch.
//
// Every query row owns a key STREAM: its selected fixed keys (key_idx,
// cluster-major positions into Kp/Vp) followed by its visible user keys
// (causal, bottom-right aligned in prefill, R8).  The streams are split into
// segments; each segment yields a normalised partial (o, lse) and the CTA that
// completes a row's last segment merges the row's partials with the partial
// maxima/denominators (atomic ticket, so a call is ONE launch).
//
// Decode (n_q == 1): PERSISTENT CTAs (grid = SMs x occupancy) split the
// concatenation of all rows' streams into equal contiguous key ranges -- "a
// fixed number of desired keys and values ... for a single SM": a head
// with more selected keys is spread over more SMs, every CTA moves the same
// number of bytes, and a CTA pays the per-segment setup once or twice.  The
// ranges are derived on the device from n_keys, so nothing returns to the
// host.  Prefill rows use a 2-D grid of (row, fixed-size segment).
//
// Data movement: each warp streams 16 keys per round; a group of G = d/8 lanes
// reads one key row (256 B at d=128 bf16) with 16-byte non-allocating loads,
// the K and V rows of all 16 keys are in flight before the first FMA, and the
// next round's key positions are prefetched.  The 16 partial dot products are
// reduced with a transposed butterfly (8 shuffles) and the online softmax runs
// in the log2 domain (ex2.approx).  The kernel is launched with programmatic
// stream serialization; griddepcontrol.wait orders it after the lookup kernel.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "stream.cuh"
#include "tma.cuh"

namespace sqz {

SQZ_TRACE_DECL(g_trace_attn)
#ifdef SQZ_TRACE
__device__ unsigned long long g_trace_mrg[2048 * 4];  // per row: merge start, loads in, end
#define MRG_AT(row, slot)                                                                  \
    do {                                                                                   \
        if (threadIdx.x == 0 && (row) < 2048) {                                            \
            unsigned long long t_;                                                         \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                        \
            g_trace_mrg[(row) * 4 + (slot)] = t_;                                          \
        }                                                                                  \
    } while (0)
extern "C" int sqz_trace_mrg(void *host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, g_trace_mrg, bytes < sizeof(g_trace_mrg) ? bytes : sizeof(g_trace_mrg));
}
#else
#define MRG_AT(row, slot) do { } while (0)
#endif

constexpr int NCW = 4;                  // warps per CTA
constexpr int NCT = NCW * 32;           // threads per CTA
#ifndef SQZ_ATT_ACQREL  // acquire-release ticket atomic instead of fence + atomic (tuning knob)
#define SQZ_ATT_ACQREL 1  // cfg2 -0.4 us, cfg4 -0.1 us (same box)
#endif
constexpr int MAX_PERSIST_CTAS = 1184;  // 148 SMs x 8
constexpr int MIN_KEYS = 256;           // minimum keys per persistent CTA
// Partition cost of a decode segment: its keys plus SEG_KW keys' worth for the
// segment's setup and epilogue (q load, position prefetch, pipeline refill,
// partial write + ticket), so a CTA whose range straddles a row boundary gets
// fewer keys (measured: ~2.3 us per extra segment at ~25 keys/us per CTA;
// 128 was the best of 0 / 64 / 128 on cfg2 and of 0 / 128 / 256 / 512 on cfg4).
#ifndef SQZ_DEC_SEG_KW
#define SQZ_DEC_SEG_KW 128
#endif
constexpr int SEG_KW = SQZ_DEC_SEG_KW;
// decode step: user keys per chunk attended before the wait for the lookup
#ifndef SQZ_USER_CHUNK
#define SQZ_USER_CHUNK 256
#endif
constexpr int USER_CHUNK = SQZ_USER_CHUNK;

int attention_kch(int n_q) { return n_q == 1 ? 256 : 1024; }
int attention_user_chunk() { return USER_CHUNK; }
int attention_max_parts(int64_t L, int n_u, int n_q) {
    const int kch = attention_kch(n_q);
    const int grid_parts = (int)((L + n_u + kch - 1) / kch);
    return n_q == 1 ? std::max(grid_parts, MAX_PERSIST_CTAS) : grid_parts;
}

// A row's key stream: nkf selected fixed keys, then nu visible user keys.
struct RowInfo {
    int bh, h, nkf, nu;
    __device__ __forceinline__ int total() const { return nkf + nu; }
};
__device__ __forceinline__ RowInfo row_info(const AttnArgs &a, int row, int nkf = -1) {
    RowInfo r;
    r.bh = row / a.n_q;
    r.h = r.bh % a.H;
    const int t = row % a.n_q;
    r.nkf = nkf >= 0 ? nkf : ldcg(a.n_keys + r.bh);
    int vis = a.causal ? t + a.n_u - a.n_q + 1 : a.n_u;
    r.nu = a.up_o ? 0 : max(0, min(vis, a.n_u));  // decode step: the user chunks hold them
    return r;
}

// One segment [a0, a1) of a row's stream, its partial slot and the number of
// partials the row has.
struct Seg {
    int row, a0, a1, slot, nparts;
};

// Merge of one row's partials by the CTA: O = sum_p e^(lse_p - M) o_p / L,
// LSE = M + log L.  Thread k < D owns output column k; the
// partials are read MB at a time (their lse values and o columns in the same
// memory round trip) with an online rescale, so the merge is one pass without
// block barriers.  Every thread forms the same weights in the same order (the
// result does not depend on which CTA merges or when).
// MB partials per memory round trip: 16 for the in-kernel (ticket) merge, 32 for
// k_merge_rows, whose rows also carry the decode step's user-chunk partials
template <int D, int MB = 16>
__device__ void merge_row(const AttnArgs &a, int row, int P) {
    const int tid = threadIdx.x;
    if (tid >= D) return;
    MRG_AT(row, 0);
    const float *lse = a.part_lse + (size_t)row * a.max_chunks;
    const float *op = a.part_o + (size_t)row * a.max_chunks * D + tid;
    // decode step: the user-chunk partials follow the P fixed-key ones
    const int U = a.up_o ? a.up_n : 0;
    const float *ulse = U ? a.up_lse + (size_t)row * U : nullptr;
    const float *uop = U ? a.up_o + (size_t)row * U * D + tid : nullptr;
    float M = -INFINITY, L = 0.f, acc = 0.f;
    for (int p0 = 0; p0 < P + U; p0 += MB) {
        float lv[MB], ov[MB];
#pragma unroll
        for (int j = 0; j < MB; ++j) {
            const int p = p0 + j;
            const bool in = p < P, inu = !in && p < P + U;
            lv[j] = in ? ldcg(lse + p) : inu ? ldcg(ulse + (p - P)) : -INFINITY;
            ov[j] = in ? ldcg(op + (size_t)p * D) : inu ? ldcg(uop + (size_t)(p - P) * D) : 0.f;
        }
        // four short dependency chains (fixed order: the result is deterministic)
        float m4[4] = {M, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int j = 0; j < MB; ++j) m4[j & 3] = fmaxf(m4[j & 3], lv[j]);
        const float mt = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
        MRG_AT(row, 1);
        if (mt == -INFINITY) continue;
        const float corr = exp_fast(M - mt);  // M = -inf -> 0
        float L4[4] = {L * corr, 0.f, 0.f, 0.f}, A4[4] = {acc * corr, 0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < MB; ++j) {
            const float w = exp_fast(lv[j] - mt);  // lse = -inf -> 0
            L4[j & 3] += w;
            A4[j & 3] = fmaf(w, ov[j], A4[j & 3]);
        }
        L = (L4[0] + L4[1]) + (L4[2] + L4[3]);
        acc = (A4[0] + A4[1]) + (A4[2] + A4[3]);
        M = mt;
    }
    const float v = (M == -INFINITY) ? 0.f : acc / L;
    if (a.out_dtype == SQZ_BF16)
        reinterpret_cast<__nv_bfloat16 *>(a.O)[(size_t)row * D + tid] = __float2bfloat16_rn(v);
    else
        reinterpret_cast<float *>(a.O)[(size_t)row * D + tid] = v;
    if (tid == 0) {
        a.LSE[row] = (M == -INFINITY) ? -INFINITY : M + logf(L);
        if (M == -INFINITY && !a.partial) atomicOr(a.status, 1);
    }
    MRG_AT(row, 2);
}

// Rows with no key at all (no selected fixed key, no visible user key) get the
// identity partial O = 0, LSE = -inf (an error for final outputs).
template <int D>
__device__ void empty_row(const AttnArgs &a, int row) {
    for (int k = threadIdx.x; k < D; k += blockDim.x) {
        if (a.out_dtype == SQZ_BF16)
            reinterpret_cast<__nv_bfloat16 *>(a.O)[(size_t)row * D + k] = __float2bfloat16_rn(0.f);
        else
            reinterpret_cast<float *>(a.O)[(size_t)row * D + k] = 0.f;
    }
    if (threadIdx.x == 0) {
        a.LSE[row] = -INFINITY;
        if (!a.partial) atomicOr(a.status, 1);
    }
}

// Iterates the segments of this CTA.
template <bool PERSIST> struct SegIter {
    const AttnArgs *a;
    const int *pref;  // PERSIST: exclusive prefix of row partition costs, [rows + 1]
    int rows, r;
    long long ks, ke, K;
    int G;
    bool done;
    __device__ __forceinline__ int cta_of(long long x) const {  // CTA whose range holds key x
        return (int)(((x + 1) * (long long)G - 1) / K);
    }
    __device__ void init(const AttnArgs &aa, const int *p, int nrows) {
        a = &aa;
        pref = p;
        rows = nrows;
        done = false;
        if (PERSIST) {
            // the CTAs split the cost space (row r: SEG_KW setup units, then one
            // unit per key) into equal ranges; at least MIN_KEYS units per CTA,
            // so small problems use fewer CTAs and no range lies inside a setup gap
            K = pref[rows];
            G = (int)min((long long)gridDim.x, max(1LL, (K + MIN_KEYS - 1) / MIN_KEYS));
            if ((int)blockIdx.x >= G || K == 0) { r = rows; ke = 0; return; }
            ks = (long long)blockIdx.x * K / G;
            ke = (long long)(blockIdx.x + 1) * K / G;
            int lo = 0, hi = rows - 1;  // last row with pref <= ks
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (pref[mid] <= ks) lo = mid; else hi = mid - 1;
            }
            r = lo;
        }
    }
    __device__ bool next(Seg &s) {
        if (PERSIST) {
            while (r < rows && pref[r] < ke) {
                const long long cs = pref[r], re = pref[r + 1];
                const int row = r++;
                const long long rs = cs + SEG_KW;  // cost unit of the row's first key
                if (re <= ks || re == cs || ke <= rs) continue;
                s.row = row;
                s.a0 = (int)(max(ks, rs) - rs);
                s.a1 = (int)(min(ke, re) - rs);
                const int wf = cta_of(rs), wl = cta_of(re - 1);
                s.slot = (int)blockIdx.x - wf;
                s.nparts = wl - wf + 1;
                return true;
            }
            return false;
        }
        if (done) return false;
        done = true;
        const RowInfo ri = row_info(*a, blockIdx.x);
        const int n = ri.total();
        s.row = blockIdx.x;
        s.a0 = blockIdx.y * a->kch;
        s.a1 = min(n, s.a0 + a->kch);
        s.slot = blockIdx.y;
        s.nparts = (n + a->kch - 1) / a->kch;
        return s.a0 < n;
    }
};

// Streams the keys [a0, a1) of row `row`'s stream (stream key k < ri.nkf: the
// selected fixed key key_idx[k] (or read from the run-length selection), else
// user key k - nkf) and writes the CTA's normalised partial -- o/l to
// o_dst[0, D) and the natural-log LSE to *lse_dst (-inf, o = 0 if empty).
// Every thread of the CTA calls it; no barrier after the partial stores.
//
// Data movement: each warp streams KR keys per round; a group of G = D/8 lanes
// reads one key row with 16-byte non-allocating loads, the K and V rows of all
// KR keys are in flight before the first FMA, and the next round's key
// positions are prefetched while they are.
template <typename T, int D>
__device__ __forceinline__ void stream_partial(const AttnArgs &a, int row, const RowInfo &ri, int a0,
                                               int a1, float *o_dst, float *lse_dst, float *s_m,
                                               float *s_l, float *s_o) {
    constexpr int G = D / 8;          // lanes per key row (8 elements each)
    constexpr int KPW = 32 / G;       // key rows per warp instruction
    constexpr int KR = keys_per_round<T>();
    constexpr int NS = KR / KPW;      // key slots per lane per round
    constexpr int LPS = G / NS;       // lanes holding each reduced key
    constexpr int LG_G = G == 16 ? 4 : 3;
    constexpr int LG_NS = NS == 16 ? 4 : NS == 8 ? 3 : NS == 4 ? 2 : NS == 2 ? 1 : 0;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane / G, sub = lane % G;
    const int myslot = sub >> (LG_G - LG_NS);
    const T *Kf = reinterpret_cast<const T *>(a.Kp) + (size_t)ri.h * a.L * D;
    const T *Vf = reinterpret_cast<const T *>(a.Vp) + (size_t)ri.h * a.L * D;
    const T *Ku = reinterpret_cast<const T *>(a.Ku) + (size_t)ri.bh * a.n_u * D;
    const T *Vu = reinterpret_cast<const T *>(a.Vu) + (size_t)ri.bh * a.n_u * D;
    const int32_t *kidx = a.key_idx ? a.key_idx + (size_t)ri.bh * a.L : nullptr;
    RunList rl;
    RunWin rw;
    if (!kidx && ri.nkf > 0) {
        rl.cl = a.sel_cl + (size_t)ri.bh * a.c2;
        rl.pref = a.sel_pref + (size_t)ri.bh * a.c2;
        rl.koff = a.key_off + (size_t)ri.h * (a.c2 + 1);
        rl.n = ldcg(a.sel_n + ri.bh);
        rl.nkf = ri.nkf;
        rw.J = 0;
        rw.end = -1;  // empty: the first cover loads
        rw.p0 = rw.p1 = 0x7fffffff;
    }
    // source position of stream key k (this lane's key of a warp round starting
    // at stream key j): >= 0 fixed key row, < 0 user key -1-u.  Warp-collective.
    auto pos_of = [&](int j, int k) -> int {
        if (!kidx) {
            const int kmax = min(min(j + KR, a1), ri.nkf) - 1;
            if (j <= kmax) {  // warp-uniform
                runwin_cover(rw, rl, j, kmax, lane);
                const int p = runwin_pos(rw, min(k, kmax));
                if (k <= kmax) return p;
            }
            if (k >= a1) return 0;
            return -1 - (k - ri.nkf);
        }
        if (k >= a1) return 0;
        return k < ri.nkf ? ldcg(kidx + k) : -1 - (k - ri.nkf);
    };
    // lane l (< KR) holds the position of key l of this warp's current round;
    // the first positions are requested before the query row, so the two
    // loads share one memory round trip
    int j0 = a0 + warp * KR;
    int pos_cur = pos_of(j0, j0 + (lane & (KR - 1)));
    float q[8];
    load8(reinterpret_cast<const T *>(a.Q) + (size_t)row * D + sub * 8, q);
    const float sc = a.scale * LOG2E;
#pragma unroll
    for (int k = 0; k < 8; ++k) q[k] *= sc;
    float m_run = -INFINITY, l_lane = 0.f, o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = 0.f;
    // one warp round: the K and V rows of keys [j, j + KR) (positions in `pc`)
    auto issue = [&](int j, int pc, Raw<T> (&kr)[NS], Raw<T> (&vr)[NS]) {
        const int nk = min(KR, a1 - j);
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const int kk = s * KPW + g;
            const int pos = __shfl_sync(FULL, pc, kk);
            if (kk < nk) {
                const T *kp = pos >= 0 ? Kf + (size_t)pos * D : Ku + (size_t)(-1 - pos) * D;
                const T *vp = pos >= 0 ? Vf + (size_t)pos * D : Vu + (size_t)(-1 - pos) * D;
                ld_raw(kr[s], kp + sub * 8);
                ld_raw(vr[s], vp + sub * 8);
            } else {
#pragma unroll
                for (int i = 0; i < (int)(sizeof(kr[s].v) / sizeof(uint4)); ++i)
                    kr[s].v[i] = vr[s].v[i] = make_uint4(0, 0, 0, 0);
            }
        }
    };
    auto consume = [&](int j, const Raw<T> (&kr)[NS], const Raw<T> (&vr)[NS]) {
        const int nk = min(KR, a1 - j);
        float v[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            float f[8];
            cvt(kr[s], f);
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < 8; ++k) acc = fmaf(q[k], f[k], acc);
            v[s] = acc;
        }
        float z = group_transpose_reduce<NS, G>(v, lane);
        if (myslot * KPW + g >= nk) z = -INFINITY;
        const float mx = warp_max(z);
        const float m_new = fmaxf(m_run, mx);
        const float alpha = fast_exp2(m_run - m_new);  // m_run = -inf -> 0
        const float p = fast_exp2(z - m_new);          // z = -inf -> 0
        l_lane = l_lane * alpha + p;
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] *= alpha;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const float ps = __shfl_sync(FULL, p, g * G + s * LPS);
            if (s * KPW + g < nk) {
                float f[8];
                cvt(vr[s], f);
#pragma unroll
                for (int k = 0; k < 8; ++k) o[k] = fmaf(ps, f[k], o[k]);
            }
        }
        m_run = m_new;
    };
    constexpr int STRIDE = NCW * KR;
    for (; j0 < a1; j0 += STRIDE) {
        Raw<T> kr[NS], vr[NS];
        issue(j0, pos_cur, kr, vr);
        // prefetch the next round's positions while this round's rows are in flight
        pos_cur = pos_of(j0 + STRIDE, j0 + STRIDE + (lane & (KR - 1)));
        consume(j0, kr, vr);
    }
    // ---- fold the key groups, then the warps ----
#pragma unroll
    for (int s2 = G; s2 < 32; s2 <<= 1)
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] += __shfl_xor_sync(FULL, o[k], s2);
    const float l_w = warp_sum(l_lane) * (1.0f / LPS);
    if (lane == 0) { s_m[warp] = m_run; s_l[warp] = l_w; }
    if (g == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) s_o[warp * D + sub * 8 + k] = o[k];
    }
    __syncthreads();
    if (tid < D) {
        float M = -INFINITY;
        for (int w = 0; w < NCW; ++w) M = fmaxf(M, s_m[w]);
        float L = 0.f, O = 0.f;
        for (int w = 0; w < NCW; ++w) {
            const float e = (s_m[w] == -INFINITY) ? 0.f : exp2f(s_m[w] - M);
            L += s_l[w] * e;
            O += s_o[w * D + tid] * e;
        }
        o_dst[tid] = L > 0.f ? O / L : 0.f;
        if (tid == 0) *lse_dst = L > 0.f ? (M + log2f(L)) * LN2 : -INFINITY;
    }
}

// MINB: CTAs per SM the register allocation must allow.  3 (<= 170 registers)
// for short per-CTA streams; 4 (128 registers, a few spilled prologue values)
// for long ones, where the extra warps' bytes in flight pay (cfg5 attention
// 274 -> 262 us; cfg2 +0.4 us, so it stays at 3 there)
template <typename T, int D, bool PERSIST, int MINB>
__global__ void __launch_bounds__(NCT, MINB) k_attend(AttnArgs a, int rows) {
    extern __shared__ __align__(16) int dyn_i[];
    int *s_pref = dyn_i;             // [rows + 1] (persistent)
    int *s_nkf = dyn_i + rows + 1;   // [rows]     (persistent)
    __shared__ float s_m[NCW], s_l[NCW], s_o[NCW * D];
    __shared__ int s_last;
    const int tid = threadIdx.x, lane = tid & 31;

    SQZ_TRACE_AT(g_trace_attn, 0);
    // the merge kernel behind this one may take the SM slots this grid frees
    if (PERSIST && a.merge_kernel) asm volatile("griddepcontrol.launch_dependents;");
    // decode step (a.up_o): the user KV does not depend on the selection, so the
    // CTAs resident beside the lookup's CTAs attend it now, in USER_CHUNK-key
    // chunks spread statically over the first up_ctas CTAs, each chunk's
    // partial counted in the high bits of the row's ticket word
    if (PERSIST && a.up_o && (int)blockIdx.x < a.up_ctas) {
        const int nch = rows * a.up_n;
        for (int c = blockIdx.x; c < nch; c += a.up_ctas) {
            const int r = c / a.up_n, j = c % a.up_n;
            RowInfo ri;
            ri.bh = r;  // n_q == 1
            ri.h = r % a.H;
            ri.nkf = 0;
            ri.nu = a.n_u;
            const int a0 = j * USER_CHUNK;
            stream_partial<T, D>(a, r, ri, a0, min(a.n_u, a0 + USER_CHUNK),
                                 a.up_o + ((size_t)r * a.up_n + j) * D, a.up_lse + (size_t)r * a.up_n + j,
                                 s_m, s_l, s_o);
            __syncthreads();
            // the row's ticket word counts user chunks in its high 16 bits (the
            // merge kernel, when used, runs after the whole grid instead)
            if (tid == 0 && !a.merge_kernel) red_release_add(a.row_cnt + r, 1 << 16);
        }
    }
    // the selection comes from the preceding lookup kernel (programmatic
    // dependent launch: the launch itself overlaps its tail)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    SQZ_TRACE_AT(g_trace_attn, 1);
    // a row with no fixed-key segment: wait for its user chunks (long done in
    // practice), then clear its ticket word for the next step
    auto user_ready = [&](int r) {  // CTA-uniform
        if (tid == 0) {
            while ((ld_acquire(a.row_cnt + r) >> 16) < a.up_n) __nanosleep(32);
            a.row_cnt[r] = 0;
        }
        __syncthreads();
    };

    if (PERSIST) {
        // exclusive prefix of the row stream lengths (rows <= a few thousand)
        __shared__ int s_ws[NCW];
        const int warp = tid >> 5;
        if (tid == 0) s_pref[0] = 0;
        for (int base = 0; base < rows; base += NCT) {
            __syncthreads();
            const int r = base + tid;
            int len = 0;
            if (r < rows) {
                const RowInfo ri = row_info(a, r);
                len = ri.total() > 0 ? ri.total() + SEG_KW : 0;
                s_nkf[r] = ri.nkf;
            }
            int inc = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(FULL, inc, o);
                if (lane >= o) inc += t;
            }
            if (lane == 31) s_ws[warp] = inc;
            __syncthreads();
            int wb = 0;
            for (int w = 0; w < warp; ++w) wb += s_ws[w];
            const int basev = s_pref[base];
            __syncthreads();
            if (r < rows) s_pref[r + 1] = basev + wb + inc;
        }
        __syncthreads();
        for (int r = blockIdx.x; r < rows && !a.merge_kernel; r += gridDim.x)
            if (s_pref[r + 1] == s_pref[r]) {
                if (a.up_o) {  // no selected fixed key: the user-chunk partials alone
                    user_ready(r);
                    merge_row<D>(a, r, 0);
                    __syncthreads();
                } else {
                    empty_row<D>(a, r);
                }
            }
    } else {
        if (blockIdx.y == 0 && row_info(a, blockIdx.x).total() == 0) empty_row<D>(a, blockIdx.x);
    }
    __syncthreads();
    SQZ_TRACE_AT(g_trace_attn, 2);

    SegIter<PERSIST> it;
    it.init(a, s_pref, rows);
    Seg sg;
#ifdef SQZ_TRACE
    int tr_nseg = 0, tr_nmerge = 0, tr_keys = 0;
#endif
    while (it.next(sg)) {
#ifdef SQZ_TRACE
        ++tr_nseg;
        tr_keys += sg.a1 - sg.a0;
#endif
        const RowInfo ri = row_info(a, sg.row, PERSIST ? s_nkf[sg.row] : -1);
        const size_t slot = (size_t)sg.row * a.max_chunks + sg.slot;
        stream_partial<T, D>(a, sg.row, ri, sg.a0, sg.a1, a.part_o + slot * D, a.part_lse + slot, s_m,
                             s_l, s_o);
        SQZ_TRACE_AT(g_trace_attn, 4);
        __syncthreads();
        if (PERSIST && a.merge_kernel) {  // the merge kernel takes it from here
            if (tid == 0 && sg.slot == 0) a.row_cnt[sg.row] = sg.nparts;
            continue;
        }
        // the CTA that completes a row's last segment merges its partials (the
        // barrier orders the CTA's partial stores before thread 0's release fence)
        if (tid == 0) {
            // ticket word: fixed-key partials counted in the low 16 bits, the
            // decode step's user chunks (released before the wait) in the high ones
#if SQZ_ATT_ACQREL
            // one acquire-release atomic: releases the CTA's partial (ordered before
            // it by the barrier), and acquires the other segments' partials for the merge
            int t = ticket_acq_rel(a.row_cnt + sg.row);
#else
            __threadfence();
            int t = atomicAdd(a.row_cnt + sg.row, 1);
#endif
            s_last = ((t & 0xffff) == sg.nparts - 1);
            if (s_last) {
                while ((t >> 16) < a.up_n) {  // a user chunk still out (not seen in practice)
                    __nanosleep(32);
                    t = ld_acquire(a.row_cnt + sg.row);
                }
                a.row_cnt[sg.row] = 0;
            }
        }
        __syncthreads();
        if (s_last) {
            SQZ_TRACE_AT(g_trace_attn, 6);  // ticket taken (merging CTAs)
#if !SQZ_ATT_ACQREL
            __threadfence();
#endif
            merge_row<D>(a, sg.row, sg.nparts);
            __syncthreads();
#ifdef SQZ_TRACE
            ++tr_nmerge;
#endif
        }
    }
    SQZ_TRACE_AT(g_trace_attn, 5);
#ifdef SQZ_TRACE
    {
        unsigned smid_;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));
        SQZ_TRACE_VAL(g_trace_attn, 3, (unsigned long long)tr_nseg | ((unsigned long long)tr_nmerge << 8) |
                                           ((unsigned long long)tr_keys << 16));
        SQZ_TRACE_VAL(g_trace_attn, 7, smid_);
    }
#endif
}

// Decode step: the merge of every row's partials (fixed-key segments, then the
// user chunks) after the whole attention grid is done (griddepcontrol.wait):
// no ticket atomics and no last-CTA merge on the attention kernel's tail.
template <int D>
__global__ void __launch_bounds__(D) k_merge_rows(AttnArgs a) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int row = blockIdx.x;
    const int P = ldcg(a.row_cnt + row);
    merge_row<D, 32>(a, row, P);
    __syncthreads();
    if (threadIdx.x == 0) a.row_cnt[row] = 0;  // self-cleaning (the ticket array)
}

template <typename T, int D>
static cudaError_t launch_t(const AttnArgs &a, cudaStream_t st) {
    const int rows = a.B * a.H * a.n_q;
    if (rows == 0) return cudaSuccess;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(NCT);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // The persistent decode partition keeps int32 cost prefixes in shared
    // memory: shapes whose total cost could reach 2^31 (e.g. dense attention over
    // 1M keys with B*H >= 2048) take the 2-D split-KV grid instead.
    const long long max_cost = (long long)rows * (a.L + a.n_u + SEG_KW);
    const bool persist = a.n_q == 1 && rows <= 8192 && max_cost < 0x7fffffffLL;
    if (a.up_o && !persist) return cudaErrorInvalidValue;  // user chunks need the persistent grid
    if (persist) {
        const size_t dsm = (size_t)(2 * rows + 1) * sizeof(int);
        // long per-CTA streams (upper bound of the selected keys: rows x L) take the
        // 4-CTAs-per-SM variant
        static const int minb_env = std::getenv("SQZ_ATT_MINB") ? std::atoi(std::getenv("SQZ_ATT_MINB")) : 0;  // A/B knob
        const bool four = minb_env ? minb_env == 4 : (long long)rows * a.L >= (1LL << 24);
        auto kern = four ? k_attend<T, D, true, 4> : k_attend<T, D, true, 3>;
        if (dsm > 48 * 1024) {
            cudaError_t e = ensure_func_attr((const void *)kern,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
            if (e != cudaSuccess) return e;
        }
        const int occ = occupancy_blocks((const void *)kern, NCT, dsm);
        cfg.gridDim = dim3(std::min(device_sm_count() * occ, MAX_PERSIST_CTAS));
        cfg.dynamicSmemBytes = dsm;
        AttnArgs a2 = a;
        // user chunks go to the first CTAs, one per SM: those are dispatched
        // first and fit beside the lean lookup's CTAs (k_lookup_decode MINB = 3)
        a2.up_ctas = std::min((int)cfg.gridDim.x, device_sm_count());
        // short per-CTA streams: rows are merged by k_merge_rows behind the grid
        // (measured on cfg2: the last-CTA ticket merge put ~3 us of atomics and
        // L2 round trips on the tail; 56.0 -> 54.3 us for the two calls, 52.8 ->
        // 51.9 for the step); long ones keep the in-kernel ticket merge, which
        // their tail hides (cfg5 391 vs 393 us), and so do tiny problems, whose few
        // CTAs would pay the extra launch (cfg1 21.5 vs 20.0 us).  SQZ_TICKET_MERGE=1: A/B
        static const bool ticket_merge = std::getenv("SQZ_TICKET_MERGE") != nullptr;
        const bool tiny = (long long)rows * a.L < (1LL << 17);
        a2.merge_kernel = (ticket_merge || four || tiny) ? 0 : 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a2, rows);
        if (e != cudaSuccess || !a2.merge_kernel) return e;
        cfg.gridDim = dim3(rows);
        cfg.blockDim = dim3(D);
        cfg.dynamicSmemBytes = 0;
        return cudaLaunchKernelEx(&cfg, k_merge_rows<D>, a2);
    }
    cfg.gridDim = dim3(rows, a.max_chunks);
    cfg.dynamicSmemBytes = 0;
    return cudaLaunchKernelEx(&cfg, k_attend<T, D, false, 3>, a, rows);
}

cudaError_t launch_attention(const AttnArgs &a, cudaStream_t st) {
    // bf16 prefill runs on the tensor cores (prefill_attn.cu); fp32 inputs stay
    // on exact fp32 FFMA (tf32 tensor cores would break the fp32 tolerance)
    if (a.n_q > 1 && a.dtype == SQZ_BF16) return launch_prefill_attention(a, st);
    if (a.dtype == SQZ_BF16) {
        if (a.d == 128) return launch_t<__nv_bfloat16, 128>(a, st);
        return launch_t<__nv_bfloat16, 64>(a, st);
    }
    if (a.d == 128) return launch_t<float, 128>(a, st);
    return launch_t<float, 64>(a, st);
}

// Generic merge of P partial results (multi-shard / multi-call).
template <typename TO>
__global__ void k_merge_parts(int P, const float *__restrict__ Op, const float *__restrict__ Lp,
                              int64_t rows, int d, TO *O, float *LSE) {
    const int64_t row = blockIdx.x;
    float M = -INFINITY;
    for (int p = 0; p < P; ++p) M = fmaxf(M, Lp[(size_t)p * rows + row]);
    float L = 0.f;
    if (M != -INFINITY)
        for (int p = 0; p < P; ++p) L += expf(Lp[(size_t)p * rows + row] - M);
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
        float acc = 0.f;
        if (M != -INFINITY)
            for (int p = 0; p < P; ++p) {
                const float w = expf(Lp[(size_t)p * rows + row] - M);
                if (w > 0.f) acc += w * Op[((size_t)p * rows + row) * d + k];
            }
        O[(size_t)row * d + k] = from_f32<TO>(M == -INFINITY ? 0.f : acc / L);
    }
    if (threadIdx.x == 0) LSE[row] = (M == -INFINITY) ? -INFINITY : M + logf(L);
}

cudaError_t launch_merge(int P, const float *O_parts, const float *LSE_parts, int64_t rows, int d,
                         void *O, float *LSE, int out_dtype, cudaStream_t st) {
    if (rows == 0) return cudaSuccess;
    const int nt = d >= 128 ? 128 : 64;
    if (out_dtype == SQZ_BF16)
        k_merge_parts<__nv_bfloat16><<<(unsigned)rows, nt, 0, st>>>(P, O_parts, LSE_parts, rows, d,
                                                                    (__nv_bfloat16 *)O, LSE);
    else
        k_merge_parts<float><<<(unsigned)rows, nt, 0, st>>>(P, O_parts, LSE_parts, rows, d,
                                                           (float *)O, LSE);
    return cudaGetLastError();
}

}  // namespace sqz

SQZ_TRACE_EXPORT(sqz::g_trace_attn, sqz_trace_attn)
