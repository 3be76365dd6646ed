// decode_step.cu -- the fused single-level decode step (sqz_decode_step): the
// centroid lookup (Eq. 1 with the single-pass threshold of the generation
// stage) and the exact sparse attention over the
// selected fixed-context keys plus the user KV, in ONE persistent,
// cooperatively launched kernel.
//
// Why fused: at decode sizes the two-launch path spends most of its non-
// streaming time in dependent latency -- the lookup's scan, reductions and
// compaction, the launch hand-off, and the attention prologue -- while the
// selection-independent user-KV stream waits behind all of it.  Here every CTA
// of the persistent grid takes part in every phase, separated by two software
// grid barriers (all CTAs are co-resident: cooperative launch):
//   A  scan: the CTAs split each (b,h)'s centroid rows into S equal parts
//      (S = grid / (B*H)); logits s_i = scale q.C_i stay in shared memory, the
//      part's (m, D = sum_i N_i e^(s_i - m)) goes to global memory;
//   -- barrier 1 --
//   B  every CTA folds its (b,h)'s S partials in one fixed order (identical bits
//      in every CTA), thresholds its own rows with the log-domain single-pass
//      test (s_i - m) > log D + log T (App. C) and compacts
//      them into a local ascending list with local key offsets;
//   -- barrier 2 --
//   C  every CTA scans the parts' (count, keys) into the (b,h) offsets, writes
//      its own entries of the ABI selection outputs, and derives the equal-cost
//      partition of the selected-key streams ("a fixed number of ... keys for a
//      single SM");
//   D  the CTA streams its key range (selected clusters are contiguous runs of
//      the cluster-major Kp/Vp, read through the parts' local lists), writes a
//      normalised partial (o, lse) per segment, and the CTA completing a row's
//      last partial merges it (atomic ticket).
// The user KV does not depend on the selection: it is cut into 64-key chunks
// that CTAs take dynamically (atomic counter) while they wait at a barrier,
// and after their fixed range; its partials join the row's merge.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "internal.h"
#include "scan.cuh"
#include "stream.cuh"

namespace sqz {

SQZ_TRACE_DECL(g_trace_step)

namespace dstep {
constexpr int NW = 4;          // warps per CTA
constexpr int NT = NW * 32;    // threads per CTA
constexpr int UCH = 64;        // user keys per dynamic chunk (one CTA round)
constexpr int SEG_KW = 128;    // partition cost of a fixed-stream segment's setup
constexpr int MIN_KEYS = 256;  // minimum cost units per CTA in the partition
constexpr int MAX_GRID = 1184;
}  // namespace dstep

struct StepArgs {
    const void *Q, *C, *Kp, *Vp, *Ku, *Vu;
    const int32_t *N, *koff;
    int32_t B, H, c, n_u, out_dtype, partial, all;
    int64_t L;
    float scale, logT;
    int32_t G, S, rpp, rmax;  // grid, scan parts per (b,h), rows per part, rows per CTA
    int32_t nuc, maxp;        // user chunks per row, partial slots per row
    int32_t umode;            // bit b: take user chunks while waiting at barrier b+1
    // workspace
    float2 *md;               // [BH * S] part statistics (m, D)
    int2 *cntk;               // [BH * S] part (selected clusters, selected keys)
    int32_t *loc_cl, *loc_pref;  // [BH, c] parts' local lists (at the part's first row)
    float *part_o, *part_lse;    // [rows, maxp, D], [rows, maxp]
    int32_t *row_cnt;         // [rows] self-cleaning merge tickets
    int32_t *ctl;             // [0] grid barrier, [1] user-chunk counter, [2] exit ticket
    int32_t *status;          // set when a final row attended no key
    // outputs
    int32_t *clusters, *key_pref, *n_clusters, *n_keys, *key_idx;
    void *O;
    float *LSE;
};

// ---- virtual run list of one (b,h): the concatenation of its S parts' local
// lists (part k's entries sit at loc_cl[bh*c + k*rpp + e], e < cnt_k, with key
// offsets local to the part); FC/FK are the flat exclusive prefixes of the
// parts' counts / keys (shared memory) ------------------------------------
struct VRun {
    const int32_t *lcl, *lpref, *koff;
    const int *FC, *FK;
    int s0, S, rpp, n, nkf, c0, k0;  // c0 = FC[s0], k0 = FK[s0]
};
__device__ __forceinline__ int vrun_part_by_count(const VRun &r, int v) {
    int lo = 0, hi = r.S - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (r.FC[r.s0 + mid] - r.c0 <= v) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}
__device__ __forceinline__ void vrun_get(const VRun &r, int v, int &cl, int &pref) {
    const int k = vrun_part_by_count(r, v);
    const int idx = k * r.rpp + (v - (r.FC[r.s0 + k] - r.c0));
    cl = ldcg(r.lcl + idx);
    pref = (r.FK[r.s0 + k] - r.k0) + ldcg(r.lpref + idx);
}
// run index of stream key k < nkf
__device__ __forceinline__ int vrun_of(const VRun &r, int key) {
    int lo = 0, hi = r.S - 1;  // last part whose first key <= key (lands on a non-empty part)
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (r.FK[r.s0 + mid] - r.k0 <= key) lo = mid;
        else hi = mid - 1;
    }
    const int part = lo;
    const int kb = r.FK[r.s0 + part] - r.k0;
    const int cnt = r.FC[r.s0 + part + 1] - r.FC[r.s0 + part];
    const int32_t *lp = r.lpref + part * r.rpp;
    int a = 0, b = cnt - 1;
    while (a < b) {
        const int mid = (a + b + 1) >> 1;
        if (kb + ldcg(lp + mid) <= key) a = mid;
        else b = mid - 1;
    }
    return (r.FC[r.s0 + part] - r.c0) + a;
}
// a warp's window of 64 consecutive runs [J, J + 64) (as RunWin in common.cuh)
__device__ __forceinline__ void vwin_load(RunWin &w, const VRun &r, int J, int lane) {
    w.J = J;
    const int j0 = J + lane, j1 = J + 32 + lane;
    int c0 = 0, c1 = 0;
    w.p0 = w.p1 = 0x7fffffff;
    if (j0 < r.n) vrun_get(r, j0, c0, w.p0);
    if (j1 < r.n) vrun_get(r, j1, c1, w.p1);
    w.s0 = j0 < r.n ? __ldg(r.koff + c0) : 0;
    w.s1 = j1 < r.n ? __ldg(r.koff + c1) : 0;
    if (J + 64 < r.n) {
        int cc;
        vrun_get(r, J + 64, cc, w.end);
    } else {
        w.end = r.nkf;
    }
}
__device__ __forceinline__ void vwin_cover(RunWin &w, const VRun &r, int kmin, int kmax, int lane) {
    int first = __shfl_sync(FULL, w.p0, 0);
    if (kmin >= first && kmax < w.end) return;
    if (w.end >= 0 && kmin >= w.end && w.J + 64 < r.n) {  // usually just past the window
        vwin_load(w, r, w.J + 64, lane);
        first = __shfl_sync(FULL, w.p0, 0);
        if (kmax < w.end) return;
    }
    int J;
    if (kmin >= first && kmin < w.end) {
        const unsigned b0 = __ballot_sync(FULL, w.p0 <= kmin), b1 = __ballot_sync(FULL, w.p1 <= kmin);
        J = w.J + __popc(b0) + __popc(b1) - 1;
    } else {
        J = vrun_of(r, kmin);
    }
    vwin_load(w, r, J, lane);
}

// ---- the partial of one segment of a row's stream --------------------------
// FIXED: stream keys [a0, a1) of the row's selected-key stream (through `vr`);
// else user keys [a0, a1).  Writes the normalised partial (o / l, lse) to
// `slot` of the row.  Block-collective (all NT threads).
template <typename T, int D, bool FIXED>
__device__ void stream_part(const StepArgs &a, int row, int a0, int a1, const VRun &vr, int slot) {
    using namespace dstep;
    constexpr int G = D / 8;
    constexpr int KPW = 32 / G;
    constexpr int KR = keys_per_round<T>();
    constexpr int NS = KR / KPW;
    constexpr int LPS = G / NS;
    constexpr int LG_G = G == 16 ? 4 : 3;
    constexpr int LG_NS = NS == 16 ? 4 : NS == 8 ? 3 : NS == 4 ? 2 : NS == 2 ? 1 : 0;
    __shared__ float s_m[NW], s_l[NW], s_o[NW * D];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane / G, sub = lane % G;
    const int myslot = sub >> (LG_G - LG_NS);
    const int h = row % a.H;
    const T *Kf = reinterpret_cast<const T *>(a.Kp) + (size_t)h * a.L * D;
    const T *Vf = reinterpret_cast<const T *>(a.Vp) + (size_t)h * a.L * D;
    const T *Ku = reinterpret_cast<const T *>(a.Ku) + (size_t)row * a.n_u * D;
    const T *Vu = reinterpret_cast<const T *>(a.Vu) + (size_t)row * a.n_u * D;
    RunWin rw;
    rw.J = 0;
    rw.end = -1;
    rw.p0 = rw.p1 = 0x7fffffff;
    // position of stream key k of a round starting at j: >= 0 a Kp/Vp row,
    // < 0 user key -1-u (warp-collective for FIXED)
    auto pos_of = [&](int j, int k) -> int {
        if (FIXED) {
            const int kmax = min(j + KR, a1) - 1;
            if (j <= kmax) {
                vwin_cover(rw, vr, j, kmax, lane);
                return runwin_pos(rw, min(k, kmax));
            }
            return 0;
        }
        return k < a1 ? -1 - k : 0;
    };
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
    for (; j0 < a1; j0 += NW * KR) {
        const int nk = min(KR, a1 - j0);
        Raw<T> kr[NS], vrr[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const int kk = s * KPW + g;
            const int pos = __shfl_sync(FULL, pos_cur, kk);
            if (kk < nk) {
                const T *kp = pos >= 0 ? Kf + (size_t)pos * D : Ku + (size_t)(-1 - pos) * D;
                const T *vp = pos >= 0 ? Vf + (size_t)pos * D : Vu + (size_t)(-1 - pos) * D;
                ld_raw(kr[s], kp + sub * 8);
                ld_raw(vrr[s], vp + sub * 8);
            } else {
#pragma unroll
                for (int i = 0; i < (int)(sizeof(kr[s].v) / sizeof(uint4)); ++i)
                    kr[s].v[i] = vrr[s].v[i] = make_uint4(0, 0, 0, 0);
            }
        }
        pos_cur = pos_of(j0 + NW * KR, j0 + NW * KR + (lane & (KR - 1)));
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
        const float alpha = fast_exp2(m_run - m_new);
        const float p = fast_exp2(z - m_new);
        l_lane = l_lane * alpha + p;
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] *= alpha;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const float ps = __shfl_sync(FULL, p, g * G + s * LPS);
            if (s * KPW + g < nk) {
                float f[8];
                cvt(vrr[s], f);
#pragma unroll
                for (int k = 0; k < 8; ++k) o[k] = fmaf(ps, f[k], o[k]);
            }
        }
        m_run = m_new;
    }
#pragma unroll
    for (int s2 = G; s2 < 32; s2 <<= 1)
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] += __shfl_xor_sync(FULL, o[k], s2);
    const float l_w = warp_sum(l_lane) * (1.0f / LPS);
    __syncthreads();  // the previous segment's readers of s_m / s_o are done
    if (lane == 0) {
        s_m[warp] = m_run;
        s_l[warp] = l_w;
    }
    if (g == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) s_o[warp * D + sub * 8 + k] = o[k];
    }
    __syncthreads();
    if (tid < D) {
        float M = -INFINITY;
        for (int w = 0; w < NW; ++w) M = fmaxf(M, s_m[w]);
        float L = 0.f, O = 0.f;
        for (int w = 0; w < NW; ++w) {
            const float e = (s_m[w] == -INFINITY) ? 0.f : exp2f(s_m[w] - M);
            L += s_l[w] * e;
            O += s_o[w * D + tid] * e;
        }
        const size_t sl = (size_t)row * a.maxp + slot;
        a.part_o[sl * D + tid] = L > 0.f ? O / L : 0.f;
        if (tid == 0) a.part_lse[sl] = L > 0.f ? (M + log2f(L)) * LN2 : -INFINITY;
    }
}

// identity partial (no key): O = 0, lse = -inf
template <int D>
__device__ void identity_part(const StepArgs &a, int row, int slot) {
    const size_t sl = (size_t)row * a.maxp + slot;
    for (int k = threadIdx.x; k < D; k += blockDim.x) a.part_o[sl * D + k] = 0.f;
    if (threadIdx.x == 0) a.part_lse[sl] = -INFINITY;
}

// Merge of a row's P partials (slots [0, P)) into O / LSE, thread
// k < D owns column k; every merger forms the same weights in the same order.
template <int D>
__device__ void merge_slots(const StepArgs &a, int row, int P) {
    constexpr int MB = 16;
    const int tid = threadIdx.x;
    if (tid >= D) return;
    const float *lse = a.part_lse + (size_t)row * a.maxp;
    const float *op = a.part_o + (size_t)row * a.maxp * D + tid;
    float M = -INFINITY, L = 0.f, acc = 0.f;
    for (int p0 = 0; p0 < P; p0 += MB) {
        float lv[MB], ov[MB];
#pragma unroll
        for (int j = 0; j < MB; ++j) {
            const bool in = p0 + j < P;
            lv[j] = in ? ldcg(lse + p0 + j) : -INFINITY;
            ov[j] = in ? ldcg(op + (size_t)(p0 + j) * D) : 0.f;
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
        reinterpret_cast<__nv_bfloat16 *>(a.O)[(size_t)row * D + tid] = __float2bfloat16_rn(v);
    else
        reinterpret_cast<float *>(a.O)[(size_t)row * D + tid] = v;
    if (tid == 0) {
        a.LSE[row] = (M == -INFINITY) ? -INFINITY : M + logf(L);
        if (M == -INFINITY && !a.partial) atomicOr(a.status, 1);
    }
}

// Ticket after a partial was written (block-collective); the CTA that brings
// the row's count to `total` merges.  total < 0: not known yet (never last).
template <int D>
__device__ void finish_part(const StepArgs &a, int row, int total) {
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        const int t = ticket_acq_rel(a.row_cnt + row);
        s_last = total > 0 && t == total - 1;
        if (s_last) a.row_cnt[row] = 0;
    }
    __syncthreads();
    if (s_last) {
        merge_slots<D>(a, row, total);
        __syncthreads();
    }
}

// Block-wide ordered compaction of one tile of NT rows (cf. lookup.cu tile_scan).
__device__ __forceinline__ void step_tile_scan(bool sel, int n, int &pos, int &kpre, int &tot_c,
                                               int &tot_k) {
    using namespace dstep;
    __shared__ int s_wc[NW], s_wk[NW];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned bal = __ballot_sync(FULL, sel);
    const int wpre = __popc(bal & ((1u << lane) - 1u));
    int inc = sel ? n : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) {
        s_wc[warp] = __popc(bal);
        s_wk[warp] = inc;
    }
    __syncthreads();
    int wb = 0, kb = 0, tc = 0, tk = 0;
    for (int w = 0; w < NW; ++w) {
        if (w < warp) {
            wb += s_wc[w];
            kb += s_wk[w];
        }
        tc += s_wc[w];
        tk += s_wk[w];
    }
    pos = wb + wpre;
    kpre = kb + inc - (sel ? n : 0);
    tot_c = tc;
    tot_k = tk;
    __syncthreads();
}

// Block-wide exclusive scan of x[0..n) in shared memory (in place), x[n] = total.
__device__ void block_exscan(int *x, int n) {
    using namespace dstep;
    __shared__ int s_w[NW], s_carry;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += NT) {
        const int i = base + tid;
        const int v = i < n ? x[i] : 0;
        int inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) s_w[warp] = inc;
        __syncthreads();
        int wb = 0, tot = 0;
        for (int w = 0; w < NW; ++w) {
            if (w < warp) wb += s_w[w];
            tot += s_w[w];
        }
        const int carry = s_carry;
        if (i < n) x[i] = carry + wb + inc - v;
        __syncthreads();
        if (tid == 0) s_carry = carry + tot;
        __syncthreads();
    }
    if (tid == 0) x[n] = s_carry;
    __syncthreads();
}

template <typename T, int D>
__global__ void __launch_bounds__(dstep::NT) k_decode_step(StepArgs a) {
    using namespace dstep;
    constexpr int U = sizeof(T) == 2 ? 32 : 16;  // centroid rows per warp batch
    constexpr int RPT = 16;                      // rows per 16-value transpose
    using LaneT = Lane<T, D>;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int j = blockIdx.x, G = a.G;
    const int BH = a.B * a.H, S = a.S, c = a.c;
    const int nslot = BH * S;
    extern __shared__ __align__(16) int dyn[];
    float *s_log = reinterpret_cast<float *>(dyn);      // [rmax]
    int *s_N = dyn + a.rmax;                            // [rmax]
    int *FC = s_N + a.rmax;                             // [nslot + 1]
    int *FK = FC + nslot + 1;                           // [nslot + 1]
    int *s_pref = FK + nslot + 1;                       // [BH + 1] partition cost prefix
    __shared__ float s_red_m[NW], s_red_d[NW];
    __shared__ float s_M, s_lD;
    __shared__ int s_u;

    // this CTA's scan parts: (bh, k) with rows [k*rpp, min(c, (k+1)*rpp)) of bh
    const bool multi = BH > G;  // then S = 1 and CTA j owns bh = j, j + G, ...
    const int nparts = multi ? (BH - j + G - 1) / G : (j < S * BH ? 1 : 0);
    auto part_bh = [&](int m) { return multi ? j + m * G : j / S; };
    auto part_k = [&](int m) { return multi ? 0 : j % S; };

    SQZ_TRACE_AT(g_trace_step, 0);
    // ------------------------------------------------------------ A: scan
    int sbase = 0;
    for (int m = 0; m < nparts; ++m) {
        const int bh = part_bh(m), k = part_k(m), h = bh % a.H;
        const int i0 = min(c, k * a.rpp), n = min(c, i0 + a.rpp) - i0;
        const T *C = reinterpret_cast<const T *>(a.C) + ((size_t)h * c + i0) * D;
        const int32_t *N = a.N + (size_t)h * c + i0;
        const T *qp = reinterpret_cast<const T *>(a.Q) + (size_t)bh * D;
        for (int rr0 = warp * U; rr0 < n; rr0 += NW * U) {
            // the rows, their N and the query: one memory round trip
            const int myrr = rr0 + lane;
            const bool mine = lane < U && myrr < n;
            const int myN = mine ? __ldg(N + myrr) : 0;
            typename LaneT::Raw raw[U];
#pragma unroll
            for (int u = 0; u < U; ++u) raw[u] = LaneT::load_raw(C + (size_t)min(rr0 + u, n - 1) * D, lane);
            float q[D / 32];
            LaneT::cvt(LaneT::load_raw_pinned(qp, lane), q);
            if (mine) s_N[sbase + myrr] = myN;
#pragma unroll
            for (int gq = 0; gq < U / RPT; ++gq) {
                float v[16];
#pragma unroll
                for (int u = 0; u < RPT; ++u) {
                    float cf[D / 32];
                    LaneT::cvt(raw[gq * RPT + u], cf);
                    float acc = 0.f;
#pragma unroll
                    for (int kk = 0; kk < D / 32; ++kk) acc = fmaf(q[kk], cf[kk], acc);
                    v[u] = acc;
                }
                const float sv = transpose_reduce<16>(v, lane) * a.scale;
                const int rr = rr0 + gq * RPT + transpose_index<16>(lane);
                if ((lane & 1) == 0 && rr < n) s_log[sbase + rr] = sv;
            }
        }
        __syncthreads();
        // the part's (m, D): per-thread online, then warps, then the CTA
        float pm = -INFINITY, pd = 0.f;
        for (int rr = tid; rr < n; rr += NT) md_combine(pm, pd, s_log[sbase + rr], (float)s_N[sbase + rr]);
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const float m2 = __shfl_xor_sync(FULL, pm, o), d2 = __shfl_xor_sync(FULL, pd, o);
            md_combine(pm, pd, m2, d2);
        }
        if (lane == 0) {
            s_red_m[warp] = pm;
            s_red_d[warp] = pd;
        }
        __syncthreads();
        if (tid == 0) {
            float mm = -INFINITY, dd = 0.f;
            for (int w = 0; w < NW; ++w) md_combine(mm, dd, s_red_m[w], s_red_d[w]);
            a.md[bh * S + k] = make_float2(mm, dd);
        }
        sbase += n;
    }

    // user-KV chunks taken dynamically while waiting at a barrier.  Their
    // partials are written at once, their merge tickets deferred until the
    // row's partial count is known (after barrier 2), so whichever partial of
    // a row is last always knows it is last.
    constexpr int MAXDEF = 32;
    __shared__ int s_def[MAXDEF], s_ndef;
    if (tid == 0) s_ndef = 0;
    const int nuch = a.nuc * BH;
    auto user_chunks_until = [&](int target) {
        while (true) {
            if (tid == 0) {
                int u = -1;
                if (s_ndef < MAXDEF && ld_acquire(a.ctl) < target) u = atomicAdd(a.ctl + 1, 1);
                s_u = u;
            }
            __syncthreads();
            const int u = s_u;
            if (u < 0 || u >= nuch) {
                __syncthreads();
                return;
            }
            const int row = u / a.nuc, part = u % a.nuc;
            VRun dummy;
            stream_part<T, D, false>(a, row, part * UCH, min(a.n_u, (part + 1) * UCH), dummy, part);
            __syncthreads();
            if (tid == 0) s_def[s_ndef++] = row;
        }
    };
    auto grid_barrier = [&](int target, bool take) {
        __syncthreads();
        if (tid == 0) red_release_add(a.ctl, 1);
        if (take) user_chunks_until(target);
        if (tid == 0)
            while (ld_acquire(a.ctl) < target) {
            }
        __syncthreads();
    };
    SQZ_TRACE_AT(g_trace_step, 1);
    grid_barrier(G, a.umode & 1);
    SQZ_TRACE_AT(g_trace_step, 2);

    // ------------------------------------------- B: fold, threshold, compact
    sbase = 0;
    for (int m = 0; m < nparts; ++m) {
        const int bh = part_bh(m), k = part_k(m);
        const int i0 = min(c, k * a.rpp), n = min(c, i0 + a.rpp) - i0;
        if (warp == 0) {  // fixed-order fold of the S parts: lane l takes l, l + 32, ...
            float mm = -INFINITY, dd = 0.f;
            for (int p = lane; p < S; p += 32) {
                const float2 v = ldcg(a.md + (size_t)bh * S + p);
                md_combine(mm, dd, v.x, v.y);
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const float m2 = __shfl_xor_sync(FULL, mm, o), d2 = __shfl_xor_sync(FULL, dd, o);
                md_combine(mm, dd, m2, d2);
            }
            if (lane == 0) {
                s_M = mm;
                s_lD = logf(dd);
            }
        }
        __syncthreads();
        const float M = s_M, thr = s_lD + a.logT;
        int run = 0, runk = 0;
        int32_t *lcl = a.loc_cl + (size_t)bh * c + i0, *lpr = a.loc_pref + (size_t)bh * c + i0;
        for (int base = 0; base < n; base += NT) {
            const int rr = base + tid;
            const bool sel = rr < n && (a.all || (s_log[sbase + rr] - M) > thr);
            const int nk = rr < n ? s_N[sbase + rr] : 0;
            int pos, kpre, tc, tk;
            step_tile_scan(sel, nk, pos, kpre, tc, tk);
            if (sel) {
                lcl[run + pos] = i0 + rr;
                lpr[run + pos] = runk + kpre;
            }
            run += tc;
            runk += tk;
        }
        if (tid == 0) a.cntk[bh * S + k] = make_int2(run, runk);
        sbase += n;
    }
    SQZ_TRACE_AT(g_trace_step, 3);
    grid_barrier(2 * G, a.umode & 2);
    SQZ_TRACE_AT(g_trace_step, 4);

    // ---------------------------------- C: offsets, outputs, partition
    for (int s = tid; s < nslot; s += NT) {
        const int2 v = ldcg(a.cntk + s);
        FC[s] = v.x;
        FK[s] = v.y;
    }
    __syncthreads();
    block_exscan(FC, nslot);
    block_exscan(FK, nslot);
    for (int r = tid; r < BH; r += NT) {
        const int nkf = FK[(r + 1) * S] - FK[r * S];
        s_pref[r] = nkf > 0 ? nkf + SEG_KW : 0;
    }
    __syncthreads();
    block_exscan(s_pref, BH);
    // equal split of the cost space (row r: SEG_KW setup units, then one per key)
    const long long K = s_pref[BH];
    const int Gp = (int)min((long long)G, max(1LL, (K + MIN_KEYS - 1) / MIN_KEYS));
    auto cta_of = [&](long long x) { return (int)(((x + 1) * (long long)Gp - 1) / K); };
    auto fixed_parts = [&](int r) {  // partials of row r's fixed stream (1 identity if none)
        const long long cs = s_pref[r], re = s_pref[r + 1];
        if (re == cs) return 1;
        return cta_of(re - 1) - cta_of(cs + SEG_KW) + 1;
    };
    SQZ_TRACE_AT(g_trace_step, 5);
    SQZ_TRACE_VAL(g_trace_step, 7, s_ndef);
    // ------------------------------------------------------ D: attention
    if (j < Gp && K > 0) {
        const long long ks = (long long)j * K / Gp, ke = (long long)(j + 1) * K / Gp;
        int lo = 0, hi = BH - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_pref[mid] <= ks) lo = mid;
            else hi = mid - 1;
        }
        for (int r = lo; r < BH && s_pref[r] < ke; ++r) {
            const long long cs = s_pref[r], re = s_pref[r + 1], rs = cs + SEG_KW;
            if (re <= ks || re == cs || ke <= rs) continue;
            const int a0 = (int)(max(ks, rs) - rs), a1 = (int)(min(ke, re) - rs);
            const int slot = j - cta_of(rs);
            VRun vr;
            vr.lcl = a.loc_cl + (size_t)r * c;
            vr.lpref = a.loc_pref + (size_t)r * c;
            vr.koff = a.koff + (size_t)(r % a.H) * (c + 1);
            vr.FC = FC;
            vr.FK = FK;
            vr.s0 = r * S;
            vr.S = S;
            vr.rpp = a.rpp;
            vr.c0 = FC[r * S];
            vr.k0 = FK[r * S];
            vr.n = FC[(r + 1) * S] - vr.c0;
            vr.nkf = FK[(r + 1) * S] - vr.k0;
            stream_part<T, D, true>(a, r, a0, a1, vr, a.nuc + slot);
            finish_part<D>(a, r, a.nuc + fixed_parts(r));
        }
    }
    SQZ_TRACE_AT(g_trace_step, 6);
    // user chunks nobody took while waiting
    {
        while (true) {
            if (tid == 0) s_u = atomicAdd(a.ctl + 1, 1);
            __syncthreads();
            const int u = s_u;
            __syncthreads();
            if (u >= nuch) break;
            const int row = u / a.nuc, part = u % a.nuc;
            VRun dummy;
            stream_part<T, D, false>(a, row, part * UCH, min(a.n_u, (part + 1) * UCH), dummy, part);
            finish_part<D>(a, row, a.nuc + fixed_parts(row));
        }
    }
    // the deferred tickets of the user chunks taken at the barriers
    for (int i = 0; i < s_ndef; ++i) finish_part<D>(a, s_def[i], a.nuc + fixed_parts(s_def[i]));
    // rows without a selected key: an identity partial stands in for the fixed part
    for (int r = j; r < BH; r += G)
        if (s_pref[r + 1] == s_pref[r]) {
            identity_part<D>(a, r, a.nuc);
            finish_part<D>(a, r, a.nuc + 1);
        }

    // ------------------------------------------------ E: selection outputs
    // (after the streams: nothing on the step's critical path reads them).  The
    // part's entries are fetched in one parallel pass into shared memory (the
    // scan's logit / N arrays are free now), then written: clusters / key_pref
    // coalesced, the key-index tensor one warp per run.
    __syncthreads();
    sbase = 0;
    for (int m = 0; m < nparts; ++m) {
        const int bh = part_bh(m), k = part_k(m), sl = bh * S + k;
        const int i0 = min(c, k * a.rpp), n = min(c, i0 + a.rpp) - i0;
        const int cnt = FC[sl + 1] - FC[sl], cb = FC[sl] - FC[bh * S], kb = FK[sl] - FK[bh * S];
        const int32_t *lcl = a.loc_cl + (size_t)bh * c + i0, *lpr = a.loc_pref + (size_t)bh * c + i0;
        const int32_t *ko = a.koff + (size_t)(bh % a.H) * (c + 1);
        int *e_st = reinterpret_cast<int *>(s_log) + sbase, *e_kp = s_N + sbase;
        for (int e = tid; e < cnt; e += NT) {
            const int cl = ldcg(lcl + e), kp = kb + ldcg(lpr + e);
            a.clusters[(size_t)bh * c + cb + e] = cl;
            a.key_pref[(size_t)bh * c + cb + e] = kp;
            e_st[e] = __ldg(ko + cl);
            e_kp[e] = kp;
        }
        if (k == 0 && tid == 0) {
            a.n_clusters[bh] = FC[(bh + 1) * S] - FC[bh * S];
            a.n_keys[bh] = FK[(bh + 1) * S] - FK[bh * S];
        }
        __syncthreads();
        if (a.key_idx) {  // the expanded key-index tensor, one warp per run
            int32_t *ki = a.key_idx + (size_t)bh * a.L;
            const int kend = FK[sl + 1] - FK[bh * S];
            for (int e = warp; e < cnt; e += NW) {
                const int st = e_st[e], kp = e_kp[e];
                const int len = (e + 1 < cnt ? e_kp[e + 1] : kend) - kp;
                for (int t = lane; t < len; t += 32) ki[kp + t] = st + t;
            }
        }
        sbase += n;
    }
    // the last CTA out resets the barrier and chunk counters (self-cleaning workspace)
    __syncthreads();
    if (tid == 0) {
        const int t = ticket_acq_rel(a.ctl + 2);
        if (t == G - 1) {
            a.ctl[0] = 0;
            a.ctl[1] = 0;
            a.ctl[2] = 0;
        }
    }
}

// ---------------------------------------------------------------- host side
namespace {
template <typename T, int D>
cudaError_t launch_step_t(StepArgs a, cudaStream_t st) {
    auto kern = k_decode_step<T, D>;
    const int BH = a.B * a.H;
    // grid: co-resident persistent CTAs (occupancy with the dynamic shared
    // memory, which grows as the grid shrinks: iterate to a fixed point)
    int G = std::min(device_sm_count() * 4, dstep::MAX_GRID);
    size_t dsm = 0;
    for (int it = 0; it < 6; ++it) {
        a.S = BH > G ? 1 : G / BH;
        a.rpp = (a.c + a.S - 1) / a.S;
        a.rmax = BH > G ? ((BH + G - 1) / G) * a.c : a.rpp;
        const int nslot = BH * a.S;
        dsm = (size_t)(2 * a.rmax + 2 * (nslot + 1) + BH + 1) * sizeof(int);
        if (dsm > 48 * 1024) {
            cudaError_t e = ensure_func_attr((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)dsm);
            if (e != cudaSuccess) return e;
        }
        const int occ = occupancy_blocks((const void *)kern, dstep::NT, dsm);
        const int Gn = std::min(device_sm_count() * occ, dstep::MAX_GRID);
        if (Gn >= G) break;
        G = Gn;
    }
    a.G = G;
    a.maxp = a.nuc + a.G + 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.G);
    cfg.blockDim = dim3(dstep::NT);
    cfg.dynamicSmemBytes = dsm;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;  // the grid barriers need co-residency
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}
}  // namespace

size_t decode_step_ws_bytes(int B, int H, int c, int n_u, int d) {
    const size_t BH = (size_t)B * H;
    const size_t G = dstep::MAX_GRID;
    const size_t nuc = (size_t)(n_u + dstep::UCH - 1) / dstep::UCH;
    const size_t maxp = nuc + G + 1;
    const size_t nslot = BH > G ? BH : G;  // BH * S <= max(G, BH)
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    return al(16 * 4) + al(BH * 4) + al(nslot * 8) + al(nslot * 8) + 2 * al(BH * c * 4) +
           al(BH * maxp * 4) + al(BH * maxp * d * 4) + 256;
}

int decode_step_rows_ok(int B, int H, int c, long long L) {
    const long long BH = (long long)B * H;
    return c >= 16 && BH <= 8192 && (long long)c * ((BH + 147) / 148 + 1) <= 16384 &&
           BH * (L + dstep::SEG_KW) < 0x7fffffffLL;
}

cudaError_t launch_decode_step(const StepLaunch &l, cudaStream_t st) {
    StepArgs a;
    std::memset(&a, 0, sizeof(a));
    a.Q = l.Q; a.C = l.C; a.Kp = l.Kp; a.Vp = l.Vp; a.Ku = l.Ku; a.Vu = l.Vu;
    a.N = l.N; a.koff = l.koff;
    a.B = l.B; a.H = l.H; a.c = l.c; a.n_u = l.n_u; a.out_dtype = l.out_dtype; a.partial = l.partial;
    a.L = l.L; a.scale = l.scale;
    a.all = !(l.T > 0.f);
    a.logT = a.all ? 0.f : logf(l.T);
    a.nuc = (l.n_u + dstep::UCH - 1) / dstep::UCH;
    static const int umode = [] {
        const char *e = getenv("SQZ_STEP_UMODE");  // tuning experiments only
        return e ? atoi(e) : 3;
    }();
    a.umode = umode;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    char *p = reinterpret_cast<char *>(((uintptr_t)l.ws + 255) & ~(uintptr_t)255);
    const size_t BH = (size_t)l.B * l.H;
    const size_t G = dstep::MAX_GRID;
    const size_t maxp = a.nuc + G + 1;
    const size_t nslot = BH > G ? BH : G;
    a.ctl = reinterpret_cast<int32_t *>(p); p += al(16 * 4);
    a.row_cnt = reinterpret_cast<int32_t *>(p); p += al(BH * 4);
    a.md = reinterpret_cast<float2 *>(p); p += al(nslot * 8);
    a.cntk = reinterpret_cast<int2 *>(p); p += al(nslot * 8);
    a.loc_cl = reinterpret_cast<int32_t *>(p); p += al(BH * l.c * 4);
    a.loc_pref = reinterpret_cast<int32_t *>(p); p += al(BH * l.c * 4);
    a.part_lse = reinterpret_cast<float *>(p); p += al(BH * maxp * 4);
    a.part_o = reinterpret_cast<float *>(p);
    a.clusters = l.clusters; a.key_pref = l.key_pref; a.n_clusters = l.n_clusters; a.n_keys = l.n_keys;
    a.key_idx = l.key_idx; a.O = l.O; a.LSE = l.LSE; a.status = l.status;
    if (l.dtype == SQZ_BF16) {
        if (l.d == 128) return launch_step_t<__nv_bfloat16, 128>(a, st);
        return launch_step_t<__nv_bfloat16, 64>(a, st);
    }
    if (l.d == 128) return launch_step_t<float, 128>(a, st);
    return launch_step_t<float, 64>(a, st);
}

}  // namespace sqz

SQZ_TRACE_EXPORT(sqz::g_trace_step, sqz_trace_step)
