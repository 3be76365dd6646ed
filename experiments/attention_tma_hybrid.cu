// attention.cu -- sparse attention over the selected fixed-context keys plus
// the user KV (section 4.2), split-KV + merge, one kernel launch.
//
// Every query row owns a key STREAM: its selected fixed keys (key_idx,
// cluster-major positions into Kp/Vp) followed by its visible user keys
// (causal, bottom-right aligned in prefill, R8).  Streams are cut into TILES
// of `kch` keys ("a fixed number of desired keys and values ... for a single
// SM"): a head with more selected keys owns more tiles and is spread
// over more SMs.  Each tile yields a normalised partial (o, lse); the CTA that
// completes a row's last tile merges the row's partials with the partial
// maxima/denominators (atomic ticket, so a call is ONE launch).
//
// Decode (n_q == 1): PERSISTENT CTAs (grid = SMs x occupancy).  The tile space
// is derived on the device from n_keys (shared-memory prefix, nothing returns
// to the host) and handed out dynamically: a CTA's first tile is static, later
// ones come from an atomic counter fetched one tile ahead, so CTAs that see
// more bandwidth take more tiles and all finish together.  Prefill rows use a
// 2-D grid of (row, tile).
//
// Data movement is TMA-staged: a producer warp turns each 32-key slice of a
// tile into runs of consecutive positions (selected clusters are contiguous in
// the cluster-major layout, so a slice is usually 1-2 runs) and issues one
// cp.async.bulk per run for K and for V into a NSTAGE-deep shared-memory ring,
// completing on an mbarrier (bytes-counted); the slice's metadata (row, count,
// tile boundaries) and, on a tile's first slice, the query row travel in the
// same stage.  Four consumer warps read the stage from shared memory (a
// G = d/8 lane group per key row, conflict-free 16-byte reads), reduce the
// partial dot products with a transposed butterfly, run the online softmax in
// the log2 domain and release the stage with an mbarrier arrive.  The kernel
// is launched with programmatic stream serialization; griddepcontrol.wait
// orders it after the lookup kernel that produced the selection.
#include "common.cuh"
#include "internal.h"
#include "tma.cuh"

namespace sqz {

SQZ_TRACE_DECL(g_trace_attn)

constexpr int NCW = 4;                  // consumer warps
constexpr int NCT = NCW * 32;           // consumer threads
constexpr int AT_NT = NCT + 32;         // + one producer warp
constexpr int AT_NW = AT_NT / 32;
constexpr int KS = 32;                  // keys per pipeline stage
constexpr int NSTAGE = 4;               // ring depth
constexpr int KPWS = KS / NCW;          // keys per consumer warp per stage
constexpr int MAX_PERSIST_CTAS = 1184;  // 148 SMs x 8

int attention_kch(int n_q) { return n_q == 1 ? 256 : 1024; }
// partial slots per row: prefill = tiles of kch keys; decode = the static CTAs
// that overlap the row plus the 128-key tail tiles
int attention_max_parts(int64_t L, int n_u, int n_q) {
    if (n_q == 1) return MAX_PERSIST_CTAS + (int)((L + n_u + 127) / 128) + 1;
    const int kch = attention_kch(n_q);
    return (int)((L + n_u + kch - 1) / kch);
}

enum { META_FIRST = 1, META_LAST = 2, META_END = 4 };
struct StageMeta {
    int row, nk, flags, tile, ntiles;
};

template <typename T, int D> struct Ring {
    static constexpr int ROWB = D * (int)sizeof(T);
    static constexpr int STAGE_ELEMS = 2 * KS * D;  // K then V
    static constexpr size_t KV_BYTES = (size_t)NSTAGE * STAGE_ELEMS * sizeof(T);
    static constexpr size_t Q_BYTES = (size_t)NSTAGE * D * sizeof(T);
    static constexpr size_t BYTES = KV_BYTES + Q_BYTES + NSTAGE * (2 * sizeof(uint64_t) + sizeof(StageMeta));
};

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

__device__ __forceinline__ void lds8(const __nv_bfloat16 *p, float (&f)[8]) {
    const uint4 u = *reinterpret_cast<const uint4 *>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
}
__device__ __forceinline__ void lds8(const float *p, float (&f)[8]) {
    const float4 a = reinterpret_cast<const float4 *>(p)[0];
    const float4 b = reinterpret_cast<const float4 *>(p)[1];
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
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
    r.nu = max(0, min(vis, a.n_u));
    return r;
}

// Merge of one row's partials by the NCT consumer threads:
// O = sum_p e^(lse_p - M) o_p / L, LSE = M + log L.
template <int D>
__device__ void merge_row(const AttnArgs &a, int row, int P, float *s_w, float *s_red) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const float *lse = a.part_lse + (size_t)row * a.max_chunks;
    float acc = 0.f, lsum = 0.f;
    float M = -INFINITY;
    for (int p0 = 0; p0 < P; p0 += NCT) {
        // one tile of <= NCT partials: lse values once, block max, weights in
        // smem, then the o rows with independent (unrolled) loads
        const int p = p0 + tid;
        const float lv = p < P ? ldcg(lse + p) : -INFINITY;
        float mx = warp_max(lv);
        if (lane == 0) s_red[warp] = mx;
        named_bar(1, NCT);
        float Mt = -INFINITY;
        for (int w = 0; w < NCW; ++w) Mt = fmaxf(Mt, s_red[w]);
        const float Mn = fmaxf(M, Mt);
        const float corr = (M == -INFINITY) ? 0.f : expf(M - Mn);  // rescale earlier tiles
        acc *= corr;
        lsum *= corr;
        M = Mn;
        const float w = (lv == -INFINITY) ? 0.f : expf(lv - M);
        s_w[tid] = w;
        lsum += w;
        named_bar(1, NCT);
        const int np = min(NCT, P - p0);
        if (tid < D) {
            const float *op = a.part_o + ((size_t)row * a.max_chunks + p0) * D + tid;
#pragma unroll 16
            for (int j = 0; j < np; ++j) acc = fmaf(s_w[j], ldcg(op + (size_t)j * D), acc);
        }
        named_bar(1, NCT);
    }
    lsum = warp_sum(lsum);
    if (lane == 0) s_red[warp] = lsum;
    named_bar(1, NCT);
    float L = 0.f;
    for (int w = 0; w < NCW; ++w) L += s_red[w];
    if (tid < D) {
        const float v = (M == -INFINITY) ? 0.f : acc / L;
        if (a.out_dtype == SQZ_BF16)
            reinterpret_cast<__nv_bfloat16 *>(a.O)[(size_t)row * D + tid] = __float2bfloat16_rn(v);
        else
            reinterpret_cast<float *>(a.O)[(size_t)row * D + tid] = v;
    }
    if (tid == 0) {
        a.LSE[row] = (M == -INFINITY) ? -INFINITY : M + logf(L);
        if (M == -INFINITY && !a.partial) atomicOr(a.status, 1);
    }
    named_bar(1, NCT);
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

template <typename T, int D, bool PERSIST>
__global__ void __launch_bounds__(AT_NT) k_attend(AttnArgs a, int rows) {
    using R = Ring<T, D>;
    constexpr int G = D / 8;            // lanes per key row (8 elements each)
    constexpr int KPW = 32 / G;         // key rows per warp instruction
    constexpr int NS = KPWS / KPW;      // key slots per lane per stage
    constexpr int LPS = G / NS;         // lanes holding each reduced key
    constexpr int LG_G = G == 16 ? 4 : 3;
    constexpr int LG_NS = NS == 4 ? 2 : NS == 2 ? 1 : 0;

    extern __shared__ __align__(128) unsigned char dyn[];
    T *ring = reinterpret_cast<T *>(dyn);
    T *s_q = reinterpret_cast<T *>(dyn + R::KV_BYTES);  // [NSTAGE][D]
    uint64_t *full = reinterpret_cast<uint64_t *>(dyn + R::KV_BYTES + R::Q_BYTES);
    uint64_t *empty = full + NSTAGE;
    StageMeta *s_meta = reinterpret_cast<StageMeta *>(empty + NSTAGE);
    int *s_tpref = reinterpret_cast<int *>(dyn + R::BYTES);  // [rows + 1] tile prefix (persistent)
    int *s_nkf = s_tpref + rows + 1;                         // [rows]     (persistent)
    __shared__ float s_m[NCW], s_l[NCW], s_o[NCW * D], s_w[NCT], s_red[NCW];
    __shared__ int s_last;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < NSTAGE; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        mbar_fence_init();
    }
    SQZ_TRACE_AT(g_trace_attn, 0);
    // the selection comes from the preceding lookup kernel (programmatic
    // dependent launch: the launch and the lines above overlap its tail)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    SQZ_TRACE_AT(g_trace_attn, 1);

    if (PERSIST) {
        // exclusive prefix of the row stream lengths (rows <= a few thousand)
        __shared__ int s_ws[AT_NW];
        if (tid == 0) s_tpref[0] = 0;
        for (int base = 0; base < rows; base += AT_NT) {
            __syncthreads();
            const int r = base + tid;
            int nt = 0;
            if (r < rows) {
                const RowInfo ri = row_info(a, r);
                nt = ri.total();
                s_nkf[r] = ri.nkf;
            }
            int inc = nt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(FULL, inc, o);
                if (lane >= o) inc += t;
            }
            if (lane == 31) s_ws[warp] = inc;
            __syncthreads();
            int wb = 0;
            for (int w = 0; w < warp; ++w) wb += s_ws[w];
            const int basev = s_tpref[base];
            __syncthreads();
            if (r < rows) s_tpref[r + 1] = basev + wb + inc;
        }
        __syncthreads();
        for (int r = blockIdx.x; r < rows; r += gridDim.x)
            if (s_tpref[r + 1] == s_tpref[r]) empty_row<D>(a, r);
    } else {
        if (blockIdx.y == 0 && row_info(a, blockIdx.x).total() == 0) empty_row<D>(a, blockIdx.x);
    }
    __syncthreads();
    SQZ_TRACE_AT(g_trace_attn, 2);

    if (warp == NCW) {
        // ================= producer warp: tiles -> TMA bulk copies =================
        const uint64_t pol = policy_evict_first();
        int st = 0;
        uint32_t ph = 0;
        // Issues the stages of stream range [a0, a1) of `row` (partial `slot` of `nparts`).
        auto emit = [&](int row, const RowInfo &ri, int a0, int a1, int slot, int nparts) {
            const T *Kf = reinterpret_cast<const T *>(a.Kp) + (size_t)ri.h * a.L * D;
            const T *Vf = reinterpret_cast<const T *>(a.Vp) + (size_t)ri.h * a.L * D;
            const T *Ku = reinterpret_cast<const T *>(a.Ku) + (size_t)ri.bh * a.n_u * D;
            const T *Vu = reinterpret_cast<const T *>(a.Vu) + (size_t)ri.bh * a.n_u * D;
            const int32_t *kidx = a.key_idx + (size_t)ri.bh * a.L;
            for (int g0 = a0; g0 < a1; g0 += 8 * KS) {
                // stream positions of the next 8 stages: one load latency per 8 stages
                int posr[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int k = g0 + u * KS + lane;
                    posr[u] = k < a1 ? (k < ri.nkf ? ldcg(kidx + k) : k - ri.nkf) : 0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int j0 = g0 + u * KS;
                    if (j0 >= a1) break;
                    mbar_wait(&empty[st], ph ^ 1);
                    const int nk = min(KS, a1 - j0);
                    const bool first = j0 == a0, last = j0 + KS >= a1;
                    const int k = j0 + lane;
                    const bool user = k >= ri.nkf;
                    const int pos = posr[u];
                    const int prev = __shfl_up_sync(FULL, pos, 1);
                    const bool prev_user = __shfl_up_sync(FULL, (int)user, 1);
                    const bool start = lane < nk && (lane == 0 || pos != prev + 1 || user != prev_user);
                    const unsigned starts = __ballot_sync(FULL, start);
                    if (lane == 0) {
                        StageMeta m;
                        m.row = row;
                        m.nk = nk;
                        m.flags = (first ? META_FIRST : 0) | (last ? META_LAST : 0);
                        m.tile = slot;
                        m.ntiles = nparts;
                        s_meta[st] = m;
                        mbar_arrive_expect_tx(&full[st], (uint32_t)(2 * nk * R::ROWB +
                                                                    (first ? R::ROWB : 0)));
                        if (first)
                            bulk_g2s(s_q + (size_t)st * D,
                                     reinterpret_cast<const T *>(a.Q) + (size_t)row * D, R::ROWB,
                                     &full[st], pol);
                    }
                    __syncwarp();
                    if (start) {
                        const unsigned later = starts & ~((2u << lane) - 1u);
                        const int end = later ? __ffs(later) - 1 : nk;
                        const uint32_t bytes = (uint32_t)((end - lane) * R::ROWB);
                        T *sK = ring + (size_t)st * R::STAGE_ELEMS + (size_t)lane * D;
                        T *sV = sK + KS * D;
                        bulk_g2s(sK, (user ? Ku : Kf) + (size_t)pos * D, bytes, &full[st], pol);
                        bulk_g2s(sV, (user ? Vu : Vf) + (size_t)pos * D, bytes, &full[st], pol);
                    }
                    if (++st == NSTAGE) { st = 0; ph ^= 1; }
                }
            }
        };

        if (PERSIST) {
            // Work = a static contiguous range of the first 7/8 of the concatenated
            // key streams (equal bytes per CTA, streams of all rows in flight at
            // once), then dynamically claimed 128-key tiles of the last 1/8, so
            // CTAs that see more bandwidth take more and all finish together.
            const long long K = s_tpref[rows];
            const long long Ks = K * 7 / 8;
            const int G = (int)min((long long)gridDim.x, max(1LL, (Ks + 255) / 256));
            constexpr int TT = 4 * KS;
            auto cta_of = [&](long long x) { return (int)(((x + 1) * G - 1) / Ks); };
            auto tile_of = [&](long long x) { return (int)((x - Ks) / TT); };
            // Emits every row segment of key range [x0, x1); `src` = static CTA or tail tile.
            auto emit_range = [&](long long x0, long long x1, bool is_static, int src) {
                int lo = 0, hi = rows - 1;  // last row with pref <= x0
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (s_tpref[mid] <= x0) lo = mid; else hi = mid - 1;
                }
                for (int r = lo; r < rows && s_tpref[r] < x1; ++r) {
                    const long long rs = s_tpref[r], re = s_tpref[r + 1];
                    if (re <= x0 || re == rs) continue;
                    int n_static = 0, wf = 0, n_tail = 0, tf = 0;
                    if (rs < Ks) {
                        wf = cta_of(rs);
                        n_static = cta_of(min(re, Ks) - 1) - wf + 1;
                    }
                    if (re > Ks) {
                        tf = tile_of(max(rs, Ks));
                        n_tail = tile_of(re - 1) - tf + 1;
                    }
                    const int slot = is_static ? src - wf : n_static + src - tf;
                    emit(r, row_info(a, r, s_nkf[r]), (int)(max(x0, rs) - rs),
                         (int)(min(x1, re) - rs), slot, n_static + n_tail);
                }
            };
            int t_next = 0;
            if (lane == 0) t_next = atomicAdd(a.sched, 1);
            if (Ks > 0 && (int)blockIdx.x < G)
                emit_range((long long)blockIdx.x * Ks / G, (long long)(blockIdx.x + 1) * Ks / G, true,
                           blockIdx.x);
            while (true) {
                const int t = __shfl_sync(FULL, t_next, 0);
                const long long x0 = Ks + (long long)t * TT;
                if (x0 >= K) break;
                if (lane == 0) t_next = atomicAdd(a.sched, 1);
                emit_range(x0, min(K, x0 + TT), false, t);
            }
        } else {
            const int row = blockIdx.x, tile = blockIdx.y;
            const RowInfo ri = row_info(a, row);
            const int ntiles = (ri.total() + a.kch - 1) / a.kch;
            if (tile < ntiles)
                emit(row, ri, tile * a.kch, min(ri.total(), (tile + 1) * a.kch), tile, ntiles);
        }
        // end-of-work sentinel for the consumers
        mbar_wait(&empty[st], ph ^ 1);
        if (lane == 0) {
            s_meta[st].flags = META_END;
            mbar_arrive(&full[st]);
            if (PERSIST) {
                // the last CTA to finish re-arms the tile scheduler for the next call
                __threadfence();
                if (atomicAdd(a.sched + 1, 1) == (int)gridDim.x - 1) {
                    a.sched[0] = 0;
                    a.sched[1] = 0;
                }
            }
        }
        return;
    }

    // ================= consumer warps =================
    const int g = lane / G, sub = lane % G;
    const int myslot = sub >> (LG_G - LG_NS);
    int st = 0;
    uint32_t ph = 0;
    float q[8], m_run = -INFINITY, l_lane = 0.f, o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { q[k] = 0.f; o[k] = 0.f; }
    bool traced = false;
    while (true) {
        mbar_wait(&full[st], ph);
        const StageMeta m = s_meta[st];
        if (m.flags & META_END) break;
#ifdef SQZ_TRACE
        if (!traced) { SQZ_TRACE_AT(g_trace_attn, 3); traced = true; }
#endif
        (void)traced;
        if (m.flags & META_FIRST) {
            lds8(s_q + (size_t)st * D + sub * 8, q);
            const float sc = a.scale * LOG2E;
#pragma unroll
            for (int k = 0; k < 8; ++k) { q[k] *= sc; o[k] = 0.f; }
            m_run = -INFINITY;
            l_lane = 0.f;
        }
        const int nk = m.nk;
        const T *sK = ring + (size_t)st * R::STAGE_ELEMS;
        const T *sV = sK + KS * D;
        const int kb = warp * KPWS;  // this warp's keys in the stage
        if (kb < nk) {
            float v[NS];
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                const int kk = kb + s * KPW + g;
                float f[8];
                lds8(sK + kk * D + sub * 8, f);
                float acc = 0.f;
#pragma unroll
                for (int k = 0; k < 8; ++k) acc = fmaf(q[k], f[k], acc);
                v[s] = acc;
            }
            float z = group_transpose_reduce<NS, G>(v, lane);
            if (kb + myslot * KPW + g >= nk) z = -INFINITY;
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
                const int kk = kb + s * KPW + g;
                if (kk < nk) {
                    float f[8];
                    lds8(sV + kk * D + sub * 8, f);
#pragma unroll
                    for (int k = 0; k < 8; ++k) o[k] = fmaf(ps, f[k], o[k]);
                }
            }
            m_run = m_new;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (++st == NSTAGE) { st = 0; ph ^= 1; }
        if (!(m.flags & META_LAST)) continue;

        // ---- tile epilogue: fold key groups, then the consumer warps ----
        float oo[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) oo[k] = o[k];
#pragma unroll
        for (int s2 = G; s2 < 32; s2 <<= 1)
#pragma unroll
            for (int k = 0; k < 8; ++k) oo[k] += __shfl_xor_sync(FULL, oo[k], s2);
        const float l_w = warp_sum(l_lane) * (1.0f / LPS);
        if (lane == 0) { s_m[warp] = m_run; s_l[warp] = l_w; }
        if (g == 0) {
#pragma unroll
            for (int k = 0; k < 8; ++k) s_o[warp * D + sub * 8 + k] = oo[k];
        }
        named_bar(1, NCT);
        if (tid < D) {
            float M = -INFINITY;
            for (int w = 0; w < NCW; ++w) M = fmaxf(M, s_m[w]);
            float L = 0.f, O = 0.f;
            for (int w = 0; w < NCW; ++w) {
                const float e = (s_m[w] == -INFINITY) ? 0.f : exp2f(s_m[w] - M);
                L += s_l[w] * e;
                O += s_o[w * D + tid] * e;
            }
            const size_t slot = (size_t)m.row * a.max_chunks + m.tile;
            a.part_o[slot * D + tid] = L > 0.f ? O / L : 0.f;
            if (tid == 0) a.part_lse[slot] = L > 0.f ? (M + log2f(L)) * LN2 : -INFINITY;
        }
        // the CTA that completes a row's last tile merges its partials
        __threadfence();
        named_bar(1, NCT);
        if (tid == 0) {
            const int t = atomicAdd(a.row_cnt + m.row, 1);
            s_last = (t == m.ntiles - 1);
            if (s_last) a.row_cnt[m.row] = 0;
        }
        named_bar(1, NCT);
        if (s_last) {
            __threadfence();
            merge_row<D>(a, m.row, m.ntiles, s_w, s_red);
        }
    }
    SQZ_TRACE_AT(g_trace_attn, 5);
}

template <typename T, int D>
static cudaError_t launch_t(const AttnArgs &a, cudaStream_t st) {
    const int rows = a.B * a.H * a.n_q;
    if (rows == 0) return cudaSuccess;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(AT_NT);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const size_t ring = Ring<T, D>::BYTES;
    // Host-side launch cost matters at decode sizes (a few microseconds per
    // runtime query): attributes are set once and the persistent grid size is
    // cached per row count (one device per process).
    if (a.n_q == 1 && rows <= 8192) {
        const size_t dsm = ring + (size_t)(2 * rows + 1) * sizeof(int);
        auto kern = k_attend<T, D, true>;
        static size_t attr_bytes = 0;
        static int cached_rows = -1, cached_grid = 0;
        if (dsm > attr_bytes) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)dsm);
            if (e != cudaSuccess) return e;
            attr_bytes = dsm;
        }
        if (rows != cached_rows) {
            int dev = 0, nsm = 0, occ = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, AT_NT, dsm);
            cached_grid = std::min(nsm * std::max(occ, 1), MAX_PERSIST_CTAS);
            cached_rows = rows;
        }
        cfg.gridDim = dim3(cached_grid);
        cfg.dynamicSmemBytes = dsm;
        return cudaLaunchKernelEx(&cfg, kern, a, rows);
    }
    auto kern = k_attend<T, D, false>;
    static bool attr_set_g = false;
    if (!attr_set_g) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ring);
        if (e != cudaSuccess) return e;
        attr_set_g = true;
    }
    cfg.gridDim = dim3(rows, a.max_chunks);
    cfg.dynamicSmemBytes = ring;
    return cudaLaunchKernelEx(&cfg, kern, a, rows);
}

cudaError_t launch_attention(const AttnArgs &a, cudaStream_t st) {
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
