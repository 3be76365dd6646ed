// lookup.cu -- centroid lookup kernels (section 4.1).
//
// Decode (n_q == 1, "generation stage"):
//   k_lookup_decode: one 8-CTA thread-block cluster per (group of NB queries,
//   head).  Centroid rows are read once per head for the whole query group
//   (the batch shares the fixed context) with 8/16-byte coalesced
//   loads; logits s_i = scale*q.C_i are fp32 FFMA over exact bf16->fp32
//   products and stay in shared memory ("cache exp(qC) during the first pass",
//   P:342, kept as logits).  The per-CTA (m, D = sum N e^(s-m)) partials are
//   folded through distributed shared memory, then every CTA thresholds its
//   own rows in parallel ("the second pass can be parallelized across the
//   cluster dimension"):
//   select i  <=>  (s_i - m) > log D + log T      (single-pass form, P:343,
//   max folded into the threshold as in App. C; no second exp).
// Prefill (n_q > 1):
//   k_prefill_rowlse: LSE_t = log sum_j N_j exp(s_tj) for every query row.
//   k_prefill_colsum: S-bar partials sum_t exp(s_ti - LSE_t) per 64-query
//   tile, fixed-order (butterfly + sequential) fp32 reductions, no atomics on
//   floats; the last CTA per (b,h) reduces the tiles and thresholds S-bar > T.
// Both run on an explicit row list for the Level-2 pass of the hierarchy
// (Eq. 3: only the children of the Level-1 survivors).
#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"
#include "scan.cuh"
#include "tcgen05.cuh"
#include "tma.cuh"
#include <cuda.h>

namespace sqz {

SQZ_TRACE_DECL(g_trace_look)
SQZ_TRACE_DECL(g_trace_pl)
#ifdef SQZ_TRACE
__device__ unsigned long long g_trace_pl_it[64 * 4];
#define PL_IT(it, slot)                                                                    \
    do {                                                                                   \
        if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && (it) < 64) {         \
            unsigned long long t_;                                                         \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                        \
            g_trace_pl_it[(it) * 4 + (slot)] = t_;                                         \
        }                                                                                  \
    } while (0)
extern "C" int sqz_trace_pl_it(void *host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, g_trace_pl_it, bytes < sizeof(g_trace_pl_it) ? bytes : sizeof(g_trace_pl_it));
}
__device__ unsigned long long g_trace_fin[64 * 8];
#define PL_FIN(bh, slot)                                                                   \
    do {                                                                                   \
        if (threadIdx.x == 0 && (bh) < 64) {                                               \
            unsigned long long t_;                                                         \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                        \
            g_trace_fin[(bh) * 8 + (slot)] = t_;                                           \
        }                                                                                  \
    } while (0)
extern "C" int sqz_trace_fin(void *host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, g_trace_fin, bytes < sizeof(g_trace_fin) ? bytes : sizeof(g_trace_fin));
}
#else
#define PL_IT(it, slot) do { } while (0)
#define PL_FIN(bh, slot) do { } while (0)
#endif

constexpr int CH = 128;     // centroid rows per CTA
constexpr int NT = 256;     // threads per CTA
constexpr int NW = NT / 32;
#ifndef SQZ_L2_LATE_DEP
#define SQZ_L2_LATE_DEP 1
#endif
#ifndef SQZ_L2_PDL  // programmatic launch of the Level-2 (candidate-list) lookup
#define SQZ_L2_PDL 0  // measured: cfg4 -2.5 us, cfg5 +50 us (the attention grid floods in)
#endif
constexpr int QT = 64;      // prefill queries per tile (8 warps x 8 queries)

int lookup_chunk_rows() { return CH; }
int lookup_qtile() { return QT; }

// --------------------------------------------------------------------------
// Block-wide ordered compaction of one tile of NT rows: every thread brings
// (sel, n = expanded count); returns its position among the tile's selected rows,
// its exclusive prefix of n, and the tile totals.
// --------------------------------------------------------------------------
__device__ __forceinline__ void tile_scan(bool sel, int n, int &pos, int &kpre, int &tot_c,
                                          int &tot_k) {
    __shared__ int s_wc[32], s_wk[32];  // up to 32 warps (blockDim.x / 32)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned bal = __ballot_sync(FULL, sel);
    const int wpre = __popc(bal & ((1u << lane) - 1u));
    int inc = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) { s_wc[warp] = __popc(bal); s_wk[warp] = inc; }
    __syncthreads();
    int wb = 0, kb = 0, tc = 0, tk = 0;
    const int nw = blockDim.x >> 5;  // 4 or 8 warps
    for (int w = 0; w < nw; ++w) {
        if (w < warp) { wb += s_wc[w]; kb += s_wk[w]; }
        tc += s_wc[w];
        tk += s_wk[w];
    }
    pos = wb + wpre;
    kpre = kb + inc - n;
    tot_c = tc;
    tot_k = tk;
    __syncthreads();
}

// Prefill epilogue (the last CTA of a (b,h)): S-bar_i = (1/n_q) sum over the
// q-tile partials (fixed tile order), threshold, ascending compaction and
// range expansion.  Rows are processed R per thread per pass with every
// partial load issued before the first use, so the pass costs one or two L2
// round trips instead of one per row tile.
template <bool ROWLIST, int R = 4>
__device__ void finalize_colpart(const LevelArgs &lv, int bh, int h, int nrows, int nqt, int BH,
                                 float inv_nq) {
    const int tid = threadIdx.x;
    const int nt = blockDim.x;
    const int32_t *off = lv.off + (size_t)h * (lv.c + 1);
    int32_t *list = lv.list + (size_t)bh * lv.c;
    const int32_t *rows = ROWLIST ? lv.rows + (size_t)bh * lv.row_stride : nullptr;
    const bool all = !(lv.T > 0.f);
    PL_FIN(bh, 0);
    if (ROWLIST && (lv.dbg_S || lv.bitmap))  // rows outside the candidate list: not scanned
        for (int r = tid; r < lv.c; r += nt) {
            if (lv.dbg_S) lv.dbg_S[(size_t)bh * lv.c + r] = NAN;
            if (lv.bitmap) lv.bitmap[(size_t)bh * lv.c + r] = 0;
        }
    __syncthreads();
    const float *cp = lv.colpart + (size_t)bh * lv.c;
    const size_t stride = (size_t)BH * lv.c;
    int run = 0, runk = 0;
    for (int sb = 0; sb < nrows; sb += nt * R) {
        int row[R], st[R], n[R];
        bool sel[R];
        float acc[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int r = sb + i * nt + tid;
            row[i] = r < nrows ? (ROWLIST ? ldcg(rows + r) : r) : -1;
            acc[i] = 0.f;
        }
        int t = 0;
        for (; t + 4 <= nqt; t += 4) {
            float x[4][R];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int i = 0; i < R; ++i) x[u][i] = row[i] >= 0 ? ldcg(cp + (t + u) * stride + row[i]) : 0.f;
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int i = 0; i < R; ++i) acc[i] += x[u][i];
        }
        for (; t < nqt; ++t)
#pragma unroll
            for (int i = 0; i < R; ++i) acc[i] += row[i] >= 0 ? ldcg(cp + t * stride + row[i]) : 0.f;
        PL_FIN(bh, 1);
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const float Sbar = acc[i] * inv_nq;
            sel[i] = row[i] >= 0 && (all || Sbar > lv.T);
            st[i] = 0;
            n[i] = 0;
            if (sel[i]) {
                st[i] = __ldg(off + row[i]);
                n[i] = __ldg(off + row[i] + 1) - st[i];
            }
            if (row[i] >= 0 && lv.dbg_S) lv.dbg_S[(size_t)bh * lv.c + row[i]] = Sbar;
            if (row[i] >= 0 && lv.bitmap) lv.bitmap[(size_t)bh * lv.c + row[i]] = sel[i] ? 1 : 0;
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
            if (sb + i * nt >= nrows) break;  // uniform
            int pos, kpre, tc, tk;
            PL_FIN(bh, 2 + i);
            tile_scan(sel[i], n[i], pos, kpre, tc, tk);
            if (sel[i]) {  // the keys are expanded by k_expand_ranges (many CTAs)
                list[run + pos] = row[i];
                lv.sel_pref[(size_t)bh * lv.c + run + pos] = runk + kpre;
            }
            if (i == 0) PL_FIN(bh, 7);
            run += tc;
            runk += tk;
        }
    }
    if (tid == 0) {
        lv.n_list[bh] = run;
        lv.n_exp[bh] = runk;
    }
    PL_FIN(bh, 6);
}

// Range expansion of a finished selection, spread over many CTAs: list entry j
// of (b,h) (row id, key offset sel_pref[j]) becomes the positions
// [off[row], off[row + 1]) at exp_list[sel_pref[j] ...].  One warp per list
// entry; grid (ceil(c / EXP_ROWS), B*H).
constexpr int EXP_ROWS = 32;
__global__ void __launch_bounds__(NT) k_expand_ranges(LevelArgs lv, int H) {
    asm volatile("griddepcontrol.launch_dependents;");
    // launched programmatically behind the lookup: its CTAs start during the
    // lookup's tail and wait here for the finished selection
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int bh = blockIdx.y, h = bh % H;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = ldcg(lv.n_list + bh);
    const int32_t *off = lv.off + (size_t)h * (lv.c + 1);
    int32_t *exp_list = lv.exp_list + (size_t)bh * lv.exp_stride;
    for (int j = blockIdx.x * EXP_ROWS + warp; j < min(n, (blockIdx.x + 1) * EXP_ROWS); j += NW) {
        const int row = ldcg(lv.list + (size_t)bh * lv.c + j);
        const int kp = ldcg(lv.sel_pref + (size_t)bh * lv.c + j);
        const int st = __ldg(off + row), cnt = __ldg(off + row + 1) - st;
        for (int q = lane; q < cnt; q += 32) exp_list[kp + q] = st + q;
    }
}

static cudaError_t launch_expand(const LookupShape &s, const LevelArgs &lv, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((lv.c + EXP_ROWS - 1) / EXP_ROWS, s.B * s.H);
    cfg.blockDim = dim3(NT);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_expand_ranges, lv, s.H);
}

// --------------------------------------------------------------------------
// Decode lookup: one thread-block CLUSTER of NC CTAs per (query group, head).
// Each CTA scans a contiguous slice of the row space (logits kept in smem),
// the per-query (m, D) partials are combined through distributed shared
// memory in rank order (deterministic, identical in every CTA), each CTA
// thresholds and compacts its own rows, and the cluster-wide output offsets
// come from a DSMEM prefix over the ranks.  No global scratch round trip, no
// serial last-CTA epilogue.
// --------------------------------------------------------------------------
// CTAs per cluster: 8 (portable maximum), or 16 (non-portable, B200) when the
// row space is too large for 8 CTAs' shared memory (e.g. 52K Level-2 rows at 1M)

template <int NB> struct DecodeSmem {
    float2 md[NB];
    int cnt[NB], keys[NB];
};

// rows per warp batch: 32 for packed bf16 rows with one or two queries (their
// raw rows take the registers 16 fp32 rows would), else 16; a CTA whose rows all
// fit one 16-row batch per warp takes U = 16 (every warp loads, fewer registers)
template <typename T, int NB> constexpr int decode_u_max() { return (sizeof(T) == 2 && NB <= 2) ? 32 : 16; }

// MINB = 3 (decode step, at most 84 registers): two lookup CTAs leave room on
// the SM for one persistent attention CTA, which attends the user KV meanwhile
template <typename T, int D, int NB, bool ROWLIST, int NC, bool SLIM, int U, int MINB = 2>
__global__ void __launch_bounds__(NT, MINB) k_lookup_decode(LookupShape s, const T *__restrict__ Q,
                                                      LevelArgs lv, int rpc) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    // let the dependent attention grid launch now: its CTAs become resident and
    // park at griddepcontrol.wait until this grid has completed.  A Level-2
    // lookup that may run in more than one wave leaves the trigger to its CTAs'
    // exits (parked attention CTAs would take the slots its later clusters need)
    if (!ROWLIST || !SQZ_L2_LATE_DEP) asm volatile("griddepcontrol.launch_dependents;");
    // a candidate-list (Level-2) lookup is launched programmatically behind the
    // kernel that wrote its candidates: it becomes resident as that grid drains
    // and waits here for its completion
    if (ROWLIST) asm volatile("griddepcontrol.wait;" ::: "memory");
    SQZ_TRACE_AT(g_trace_look, 0);
    const int rank = (int)cluster.block_rank();
    const int h = blockIdx.y, g = blockIdx.z;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int H = s.H, c = lv.c;
    const int b0 = g * NB;
    const int nb = min(NB, s.B - b0);
    const T *C = reinterpret_cast<const T *>(lv.C) + (size_t)h * c * D;
    const int32_t *N = lv.N + (size_t)h * c;
    const int32_t *off = lv.off + (size_t)h * (c + 1);

    extern __shared__ __align__(16) unsigned char dyn[];
    // per-row arrays.  With one query (NB == 1) the compaction writes its output
    // in place over them (output position <= input position, and a tile's reads
    // precede its writes), 20 B per row.  SLIM (one query, large row spaces)
    // keeps only the logit, row id and off[row] (12 B per row; N and
    // off[row + 1] are re-read from the tables where needed): selected row ->
    // s_row, range start -> s_o0, key offset -> s_log, range length =
    // difference of consecutive key offsets.
    static_assert(!SLIM || NB == 1, "SLIM layout is for one query");
    constexpr bool ONEQ = SLIM;
    constexpr int NCMP = NB == 1 ? 0 : NB;                         // separate compaction arrays
    float *s_log = reinterpret_cast<float *>(dyn);                 // [NB][rpc]
    int *s_row = reinterpret_cast<int *>(s_log + NB * rpc);        // [rpc] (ROWLIST)
    int *s_o0 = s_row + rpc;                                       // [rpc] off[row]
    float *s_Nw = reinterpret_cast<float *>(s_o0 + rpc);           // [rpc] N of the row (NB > 1)
    int *s_o1 = reinterpret_cast<int *>(s_Nw + rpc);               // [rpc] off[row + 1] (NB > 1)
    int *s_cmp = s_o1 + rpc;                                       // [4][NCMP][rpc]
    int *s_sel = NB == 1 ? s_row : s_cmp;                          // [NB][rpc] selected row ids
    int *s_st = NB == 1 ? s_o0 : s_cmp + NCMP * rpc;               // [NB][rpc] range starts
    int *s_n = ONEQ ? nullptr : NB == 1 ? s_o1 : s_cmp + 2 * NCMP * rpc;  // range lengths
    int *s_kp = ONEQ ? reinterpret_cast<int *>(s_log)
                     : NB == 1 ? reinterpret_cast<int *>(s_Nw) : s_cmp + 3 * NCMP * rpc;  // key offsets
    __shared__ DecodeSmem<NB> sh;
    __shared__ float s_M[NB], s_lD[NB];
    __shared__ float s_wm[NW][NB], s_wd[NW][NB];
    // Point-to-point exchange (phase 0): every CTA pushes its per-query (m, D)
    // and later its (count, keys) into every peer's shared memory (st.async,
    // counted in bytes on the receiver's mbarrier) instead of a cluster barrier
    // followed by remote reads: a CTA waits only for the messages it needs.
    __shared__ uint64_t s_xbar[2];
    __shared__ float2 s_xmd[NC][NB];
    __shared__ int2 s_xck[NC][NB];
    const bool push = lv.phase == 0;
    if (push) {
        if (tid == 0) {
            mbar_init(&s_xbar[0], 1);
            mbar_init(&s_xbar[1], 1);
            mbar_fence_init();
            mbar_arrive_expect_tx(&s_xbar[0], (NC - 1) * NB * 8);
            mbar_arrive_expect_tx(&s_xbar[1], (NC - 1) * NB * 8);
        }
        // a peer may push only after every CTA's barriers exist: arrive now,
        // wait just before the first push (long after every CTA arrived)
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    }
    const int nrows = ROWLIST ? ldcg(lv.n_rows + (size_t)b0 * H + h) : c;
    // a candidate list is split evenly over the cluster by its actual length
    // (the smem is sized for the capacity rpc >= that share)
    const int per = ROWLIST ? (nrows + NC - 1) / NC : rpc;
    const int r0 = rank * per;
    const int nloc = max(0, min(per, nrows - r0));
    const int32_t *rows = ROWLIST ? lv.rows + ((size_t)b0 * H + h) * lv.row_stride : nullptr;
    if (ROWLIST && (lv.dbg_S || lv.bitmap)) {  // rows outside the candidate list: not scanned
        const int per = (c + NC - 1) / NC;
        for (int r = rank * per + tid; r < min(c, (rank + 1) * per); r += NT) {
            if (lv.dbg_S) lv.dbg_S[((size_t)b0 * H + h) * c + r] = NAN;
            if (lv.bitmap) lv.bitmap[((size_t)b0 * H + h) * c + r] = 0;
        }
    }

    const int phase = lv.phase;
    // the staged select (phase 2) has no scan barrier: order this CTA's NaN fill
    // before any peer writes a real score to the same rows (uniform branch)
    if (ROWLIST && (lv.dbg_S || lv.bitmap) && phase == 2) cluster.sync();
    if (phase == 2) {
        // ---- staged select: the logits and row metadata phase 1 stored, and the
        // (M, log D) folded over every shard ----
        for (int rr = tid; rr < nloc; rr += NT) {
            const int row = ROWLIST ? ldcg(rows + r0 + rr) : r0 + rr;
            s_row[rr] = row;
            s_o0[rr] = __ldg(off + row);
            if (!ONEQ) {
                s_Nw[rr] = (float)__ldg(N + row);
                s_o1[rr] = __ldg(off + row + 1);
            }
            for (int i = 0; i < nb; ++i)
                s_log[i * rpc + rr] = ldcg(lv.logits + ((size_t)(b0 + i) * H + h) * c + r0 + rr);
        }
        if (tid < nb) {
            const float2 g2 = ldcg(lv.gstat + (size_t)(b0 + tid) * H + h);
            s_M[tid] = g2.x;
            s_lD[tid] = g2.y;
            if (rank == 0 && lv.dbg_lse) lv.dbg_lse[(size_t)(b0 + tid) * H + h] = g2.x + g2.y;
        }
    } else {
    // ---- scan: logits of the CTA's rows for the NB queries ----
    if (ROWLIST && lv.rl_list) {
        // candidate q = r0 + rr is child (q - pref[j]) of survivor j, pref[j] <= q <
        // pref[j+1]: the slice's survivors (at most nloc, each has >= 1 child) are
        // staged in s_o0 / s_log (free until the scan), then a search per row
        int *s_sp = reinterpret_cast<int *>(s_log);
        const size_t pb = ((size_t)b0 * H + h) * lv.rl_c;
        __shared__ int s_ja, s_ns, s_smp;
        // last survivor with pref <= r0: 256 samples, then a warp scans the gap
        // (two memory round trips instead of a serial binary search)
        const int n = ldcg(lv.rl_n + (size_t)b0 * H + h);
        if (tid == 0) s_smp = -1;
        __syncthreads();
        if (n > 0) {
            const int ik = (int)((long long)tid * n / NT);
            if (ldcg(lv.rl_pref + pb + ik) <= r0) atomicMax(&s_smp, tid);
        }
        __syncthreads();
        if (warp == 0) {
            const int k = max(s_smp, 0);
            const int lo = (int)((long long)k * n / NT), hi = (int)((long long)(k + 1) * n / NT);
            int best = lo;
            for (int base = lo + 1; base < hi; base += 32) {
                const int j = base + lane;
                const bool le = j < hi && ldcg(lv.rl_pref + pb + j) <= r0;
                const unsigned bal = __ballot_sync(FULL, le);
                if (bal) best = base + 31 - __clz(bal);
            }
            if (lane == 0) {
                s_ja = best;
                s_ns = max(0, min(n - best, nloc));
            }
        }
        __syncthreads();
        const int ja = s_ja, ns = s_ns;
        const int32_t *po = lv.rl_off + (size_t)h * (lv.rl_c + 1);
        for (int m = tid; m < ns; m += NT) {
            s_o0[m] = __ldg(po + ldcg(lv.rl_list + pb + ja + m));  // first child row
            s_sp[m] = ldcg(lv.rl_pref + pb + ja + m);              // its candidate index
        }
        __syncthreads();
        for (int rr = tid; rr < nloc; rr += NT) {
            const int q = r0 + rr;
            int lo = 0, hi = ns - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_sp[mid] <= q) lo = mid;
                else hi = mid - 1;
            }
            s_row[rr] = s_o0[lo] + (q - s_sp[lo]);
        }
        __syncthreads();
        SQZ_TRACE_AT(g_trace_look, 6);
    } else if (ROWLIST) {  // the CTA's row ids in one coalesced pass (not one round trip per batch)
        for (int rr = tid; rr < nloc; rr += NT) s_row[rr] = ldcg(rows + r0 + rr);
        __syncthreads();
    }
    // A warp loads U rows at once (one memory round trip), forms the U x NB
    // partial dot products, and reduces them 16 at a time with the transposed
    // butterfly: value v = row_local * NB + query.  The row metadata, the
    // centroid rows and the query of a warp's first batch are all in flight
    // before any of them is used (one round trip, not three).
    using LaneT = Lane<T, D>;
    constexpr int RPT = 16 / NB;  // rows per 16-value transpose
    for (int rr0 = warp * U; rr0 < nloc; rr0 += NW * U) {
        // lane l < U owns row rr0 + l: its id and its N / key-range metadata are
        // fetched now, in the same memory round trip as the centroid rows, and
        // reach shared memory after the row loads are issued
        const int myrr = rr0 + lane;
        const bool mine = lane < U && myrr < nloc;
        int myrow = -1, m_o0 = 0, m_N = 0, m_o1 = 0;
        if (mine) {
            myrow = ROWLIST ? s_row[myrr] : r0 + myrr;
            m_o0 = __ldg(off + myrow);
            if (!ONEQ) {
                m_N = __ldg(N + myrow);
                m_o1 = __ldg(off + myrow + 1);
            }
        }
        typename LaneT::Raw raw[U];
        bool have[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            // every slot loads (a missing row reads row 0 and is zeroed at use):
            // a conditional load would be a predicated move that waits for it
            const int rid = __shfl_sync(FULL, myrow, u);
            have[u] = rid >= 0;
            raw[u] = LaneT::load_raw(C + (size_t)max(rid, 0) * D, lane);
        }
        if (mine) {
            s_o0[myrr] = m_o0;
            if (!ONEQ) {
                s_Nw[myrr] = (float)m_N;
                s_o1[myrr] = m_o1;
            }
        }
        // the query row, (re)loaded in the batch's own block (a cache hit after
        // the first batch) so the compiler does not hoist it, and its wait,
        // ahead of the row loads
        float q[NB][D / 32];
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            if (i < nb) {
                LaneT::cvt(LaneT::load_raw_pinned(Q + ((size_t)(b0 + i) * H + h) * D, lane), q[i]);
            } else {
#pragma unroll
                for (int k = 0; k < D / 32; ++k) q[i][k] = 0.f;
            }
        }
#pragma unroll
        for (int gq = 0; gq < U / RPT; ++gq) {
            float v[16];
#pragma unroll
            for (int u = 0; u < RPT; ++u) {
                float cf[D / 32];
                if (have[gq * RPT + u]) {
                    LaneT::cvt(raw[gq * RPT + u], cf);
                } else {
#pragma unroll
                    for (int k = 0; k < D / 32; ++k) cf[k] = 0.f;
                }
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    float acc = 0.f;
#pragma unroll
                    for (int k = 0; k < D / 32; ++k) acc = fmaf(q[i][k], cf[k], acc);
                    v[u * NB + i] = acc;
                }
            }
            const float sv = transpose_reduce<16>(v, lane) * s.scale;
            const int vi = transpose_index<16>(lane);
            const int rr = rr0 + gq * RPT + vi / NB;
            if ((lane & 1) == 0 && rr < nloc) s_log[(vi % NB) * rpc + rr] = sv;
        }
    }
    __syncthreads();
    if (phase == 1)  // keep the logits for the phase-2 threshold
        for (int i = 0; i < nb; ++i)
            for (int rr = tid; rr < nloc; rr += NT)
                lv.logits[((size_t)(b0 + i) * H + h) * c + r0 + rr] = s_log[i * rpc + rr];
    SQZ_TRACE_AT(g_trace_look, 1);
    // (m, D) of the CTA's rows per query: block max, then one exp per row.
    for (int i = 0; i < nb; ++i) {
        float mx = -INFINITY;
        for (int rr = tid; rr < nloc; rr += NT) mx = fmaxf(mx, s_log[i * rpc + rr]);
        mx = warp_max(mx);
        if (lane == 0) s_wm[warp][i] = mx;
        __syncthreads();
        float M = -INFINITY;
        for (int w = 0; w < NW; ++w) M = fmaxf(M, s_wm[w][i]);
        float e = 0.f;
        if (M != -INFINITY)
            for (int rb = tid; rb < nloc; rb += 4 * NT) {
                // 4 rows per thread per trip, their cluster sizes loaded together
                float nw[4], lg[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int rr = rb + u * NT;
                    const bool in = rr < nloc;
                    nw[u] = !in ? 0.f : ONEQ ? (float)__ldg(N + (ROWLIST ? s_row[rr] : r0 + rr)) : s_Nw[rr];
                    lg[u] = in ? s_log[i * rpc + rr] : M;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) e += nw[u] * exp_fast(lg[u] - M);  // O(1) arguments
            }
        e = warp_sum(e);
        if (lane == 0) s_wd[warp][i] = e;
        __syncthreads();
        if (tid == 0) {
            float dd = 0.f;
            for (int w = 0; w < NW; ++w) dd += s_wd[w][i];
            sh.md[i] = make_float2(M, dd);
        }
    }
    if (push) {
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (warp == 0) {  // lane r sends this CTA's partials to rank r
            __syncwarp();  // sh.md was written by thread 0
            if (lane < NC)
                for (int i = 0; i < NB; ++i) {
                    const float2 v = i < nb ? sh.md[i] : make_float2(-INFINITY, 0.f);
                    if (lane == rank)
                        s_xmd[rank][i] = v;
                    else
                        st_async_b64(&s_xmd[rank][i],
                                     ((uint64_t)__float_as_uint(v.y) << 32) | __float_as_uint(v.x),
                                     &s_xbar[0], lane);
                }
        }
        __syncthreads();
        if (warp < nb) mbar_wait_cluster(&s_xbar[0], 0);
    } else {
        cluster.sync();
    }
    SQZ_TRACE_AT(g_trace_look, 2);
    // ---- global (m, D) per query: warp i reads the NC ranks' partials in
    // parallel (one DSMEM load per lane) and folds them with a butterfly, so
    // every CTA of the cluster computes bit-identical values ----
    if (warp < nb) {
        const int i = warp;
        float mm = -INFINITY, dd = 0.f;
        if (lane < NC) {
            const float2 v = push ? s_xmd[lane][i] : cluster.map_shared_rank(&sh, lane)->md[i];
            mm = v.x;
            dd = v.y;
        }
#pragma unroll
        for (int o = 1; o < NC; o <<= 1) {
            const float m2 = __shfl_xor_sync(FULL, mm, o), d2 = __shfl_xor_sync(FULL, dd, o);
            md_combine_fast(mm, dd, m2, d2);
        }
        if (lane == 0) {
            s_M[i] = mm;
            s_lD[i] = logf(dd);
            if (phase == 1) {
                if (rank == 0) lv.stats_out[(size_t)(b0 + i) * H + h] = make_float2(mm, dd);
            } else if (rank == 0 && lv.dbg_lse) {
                lv.dbg_lse[(size_t)(b0 + i) * H + h] = mm + logf(dd);
            }
        }
    }
    if (phase == 1) {  // statistics only; keep smem alive for the other ranks' reads
        cluster.sync();
        return;
    }
    }  // phase != 2
    __syncthreads();
    // ---- threshold + ordered compaction of the CTA's rows ----
    const bool all = !(lv.T > 0.f);
    const float logT = all ? 0.f : logf(lv.T);
    for (int i = 0; i < nb; ++i) {
        const int bh = (b0 + i) * H + h;
        const float M = s_M[i], lD = s_lD[i], thr = lD + logT;
        int run = 0, runk = 0;
        if constexpr (ONEQ) {
            // the selection and the range lengths of all the CTA's rows first, in
            // one pass of independent loads of off[row + 1] (one memory round trip,
            // not one per tile): s_log[rr] becomes the length, or -1 if unselected
            int *s_len = reinterpret_cast<int *>(s_log);
            for (int rr = tid; rr < nloc; rr += NT) {
                const int row = ROWLIST ? s_row[rr] : r0 + rr;
                const float x = s_log[rr] - M;
                const bool sel = all || x > thr;
                if (lv.dbg_S) lv.dbg_S[(size_t)bh * c + row] = expf(x - lD);
                if (lv.bitmap) lv.bitmap[(size_t)bh * c + row] = sel ? 1 : 0;
                s_len[rr] = sel ? __ldg(off + row + 1) - s_o0[rr] : -1;
            }
            __syncthreads();
            SQZ_TRACE_AT(g_trace_look, 7);
        }
        for (int base = 0; base < nloc; base += NT) {
            const int rr = base + tid;
            const bool valid = rr < nloc;
            const int row = valid ? (ROWLIST ? s_row[rr] : r0 + rr) : 0;
            bool sel;
            int st = 0, n = 0;
            if constexpr (ONEQ) {
                const int len = valid ? reinterpret_cast<const int *>(s_log)[rr] : -1;
                sel = len >= 0;
                if (sel) {
                    st = s_o0[rr];
                    n = len;
                }
            } else {
                const float x = valid ? s_log[i * rpc + rr] - M : 0.f;
                sel = valid && (all || x > thr);
                if (valid && lv.dbg_S) lv.dbg_S[(size_t)bh * c + row] = expf(x - lD);
                if (valid && lv.bitmap) lv.bitmap[(size_t)bh * c + row] = sel ? 1 : 0;
                if (sel) {
                    st = s_o0[rr];
                    n = s_o1[rr] - st;
                }
            }
            int pos, kpre, tc, tk;
            tile_scan(sel, n, pos, kpre, tc, tk);
            if (sel) {
                s_sel[i * rpc + run + pos] = row;
                s_st[i * rpc + run + pos] = st;
                if (!ONEQ) s_n[i * rpc + run + pos] = n;
                s_kp[i * rpc + run + pos] = runk + kpre;
            }
            run += tc;
            runk += tk;
        }
        if (tid == 0) { sh.cnt[i] = run; sh.keys[i] = runk; }
    }
    SQZ_TRACE_AT(g_trace_look, 2);  // (overwrites the fold time: compaction done, before the barrier)
    if (push) {
        if (warp == 0) {
            __syncwarp();  // sh.cnt / sh.keys were written by thread 0
            if (lane < NC)
                for (int i = 0; i < NB; ++i) {
                    const int2 v = i < nb ? make_int2(sh.cnt[i], sh.keys[i]) : make_int2(0, 0);
                    if (lane == rank)
                        s_xck[rank][i] = v;
                    else
                        st_async_b64(&s_xck[rank][i], ((uint64_t)(uint32_t)v.y << 32) | (uint32_t)v.x,
                                     &s_xbar[1], lane);
                }
        }
        __syncthreads();
        if (warp < nb) mbar_wait_cluster(&s_xbar[1], 0);
    } else {
        cluster.sync();
    }
    SQZ_TRACE_AT(g_trace_look, 3);
    // ---- cluster-wide offsets, then write the lists and expand the ranges ----
    __shared__ int s_oc[NB], s_ok[NB];
    if (warp < nb) {  // warp i: lane r reads rank r's counts, prefix by shuffles
        const int i = warp;
        int cr = 0, kr = 0;
        if (lane < NC) {
            if (push) {
                const int2 v = s_xck[lane][i];
                cr = v.x;
                kr = v.y;
            } else {
                const DecodeSmem<NB> *o = cluster.map_shared_rank(&sh, lane);
                cr = o->cnt[i];
                kr = o->keys[i];
            }
        }
        int ic = cr, ik = kr;
#pragma unroll
        for (int o = 1; o < NC; o <<= 1) {
            const int tc_ = __shfl_up_sync(FULL, ic, o), tk_ = __shfl_up_sync(FULL, ik, o);
            if (lane >= o) { ic += tc_; ik += tk_; }
        }
        const int exc = __shfl_sync(FULL, ic - cr, rank), exk = __shfl_sync(FULL, ik - kr, rank);
        const int totc = __shfl_sync(FULL, ic, NC - 1), totk = __shfl_sync(FULL, ik, NC - 1);
        if (lane == 0) {
            s_oc[i] = exc;
            s_ok[i] = exk;
            if (rank == 0) {
                const int bh = (b0 + i) * H + h;
                lv.n_list[bh] = totc;
                lv.n_exp[bh] = totk;
            }
        }
    }
    __syncthreads();
    if (!ROWLIST && !ONEQ) SQZ_TRACE_AT(g_trace_look, 6);
    // this CTA is done reading its peers' shared memory: arrive now, wait (so
    // that its own stays alive for the peers' reads) only before exiting.  (The
    // push exchange reads no remote memory, and every message addressed to this
    // CTA has arrived: no barrier.)
    if (!push) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    for (int i = 0; i < nb; ++i) {
        const int bh = (b0 + i) * H + h;
        const int oc = s_oc[i], ok = s_ok[i];
        const int mine = sh.cnt[i];
        int32_t *list = lv.list + (size_t)bh * c + oc;
        int32_t *exp_list = lv.exp_list ? lv.exp_list + (size_t)bh * lv.exp_stride + ok : nullptr;
        int32_t *kpref = lv.sel_pref + (size_t)bh * c + oc;  // run-length key offsets
        for (int j = tid; j < mine; j += NT) {
            list[j] = s_sel[i * rpc + j];
            kpref[j] = ok + s_kp[i * rpc + j];
        }
        if (!ROWLIST && !ONEQ) SQZ_TRACE_AT(g_trace_look, 7);
        if (exp_list)
        for (int j = warp; j < mine; j += NW) {
            const int st = s_st[i * rpc + j], kp = s_kp[i * rpc + j];
            const int n = ONEQ ? (j + 1 < mine ? s_kp[i * rpc + j + 1] : sh.keys[i]) - kp : s_n[i * rpc + j];
            for (int t = lane; t < n; t += 32) exp_list[kp + t] = st + t;
        }
    }
    SQZ_TRACE_AT(g_trace_look, 4);
    if (!push) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    SQZ_TRACE_AT(g_trace_look, 5);
}

SQZ_TRACE_EXPORT(g_trace_look, sqz_trace_look)
SQZ_TRACE_EXPORT(g_trace_pl, sqz_trace_pl)

// --------------------------------------------------------------------------
// Fold of the shards' (m, D) statistics, sequentially in rank order (every
// rank folds the same gathered array, so all ranks get identical bits).
// --------------------------------------------------------------------------
__global__ void k_fold_stats(int P, const float2 *__restrict__ in, int64_t n, float2 *__restrict__ g,
                             float *__restrict__ rowlse) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        float m = -INFINITY, D = 0.f;
        for (int p = 0; p < P; ++p) {
            const float2 v = in[(size_t)p * n + j];
            md_combine(m, D, v.x, v.y);
        }
        const float lD = logf(D);  // -inf when no shard scanned a row
        g[j] = make_float2(m, lD);
        if (rowlse) rowlse[j] = m + lD;
    }
}

cudaError_t launch_fold_stats(int P, const float2 *stats_in, int64_t n, float2 *gstat, float *rowlse,
                              cudaStream_t st) {
    const int blocks = (int)std::min<int64_t>(1024, (n + 255) / 256);
    k_fold_stats<<<std::max(blocks, 1), 256, 0, st>>>(P, stats_in, n, gstat, rowlse);
    return cudaGetLastError();
}

static size_t decode_smem_bytes(int NB, int rpc, bool slim = false) {
    return (size_t)rpc * 4 * (slim ? 3 : NB == 1 ? 5 : NB + 4 + 4 * NB) + 16;
}

// --------------------------------------------------------------------------
// Prefill pass 1: LSE_t over the row space for every query row.
// grid (ceil(n_q/QT), B*H); warp w handles queries [tile*QT + 8w, +8).
// --------------------------------------------------------------------------
template <typename T, int D, bool ROWLIST>
__global__ void __launch_bounds__(NT) k_prefill_rowlse(LookupShape s, const T *__restrict__ Q,
                                                       LevelArgs lv) {
    const int tile = blockIdx.x, bh = blockIdx.y;
    const int h = bh % s.H;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = lv.c;
    const T *C = reinterpret_cast<const T *>(lv.C) + (size_t)h * c * D;
    const int32_t *N = lv.N + (size_t)h * c;
    const int nrows = ROWLIST ? ldcg(lv.n_rows + bh) : c;
    const int32_t *rows = ROWLIST ? lv.rows + (size_t)bh * lv.row_stride : nullptr;
    const int t0 = tile * QT + warp * 8;
    float q[8][D / 32];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int t = min(t0 + i, s.n_q - 1);
        Lane<T, D>::load(Q + ((size_t)bh * s.n_q + t) * D, lane, q[i]);
    }
    const int myq = transpose_index<8>(lane);
    float m = -INFINITY, Dsum = 0.f;
    for (int r = 0; r < nrows; ++r) {
        const int row = ROWLIST ? ldcg(rows + r) : r;
        float cf[D / 32];
        Lane<T, D>::load(C + (size_t)row * D, lane, cf);
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < D / 32; ++k) acc = fmaf(q[i][k], cf[k], acc);
            v[i] = acc;
        }
        const float sv = transpose_reduce<8>(v, lane) * s.scale;
        md_combine(m, Dsum, sv, (float)N[row]);
    }
    const int t = t0 + myq;
    if ((lane & 3) == 0 && t < s.n_q && lv.phase == 1) {
        lv.stats_out[(size_t)bh * s.n_q + t] = make_float2(m, Dsum);
    } else if ((lane & 3) == 0 && t < s.n_q) {
        const float lse = m + logf(Dsum);  // -inf when no row
        lv.rowlse[(size_t)bh * s.n_q + t] = lse;
        if (lv.dbg_lse) lv.dbg_lse[(size_t)bh * s.n_q + t] = lse;
    }
}

// --------------------------------------------------------------------------
// Prefill pass 2: S-bar tile partials; last CTA per (b,h) thresholds.
// grid (row chunks, q tiles, B*H).
// --------------------------------------------------------------------------
template <typename T, int D, bool ROWLIST>
__global__ void __launch_bounds__(NT) k_prefill_colsum(LookupShape s, const T *__restrict__ Q,
                                                       LevelArgs lv) {
    const int chunk = blockIdx.x, tile = blockIdx.y, bh = blockIdx.z;
    asm volatile("griddepcontrol.launch_dependents;");
    const int h = bh % s.H;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = lv.c;
    const int nqt = gridDim.y;
    const T *C = reinterpret_cast<const T *>(lv.C) + (size_t)h * c * D;
    const int nrows = ROWLIST ? ldcg(lv.n_rows + bh) : c;
    const int32_t *rows = ROWLIST ? lv.rows + (size_t)bh * lv.row_stride : nullptr;
    const int t0 = tile * QT + warp * 8;
    float q[8][D / 32];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int t = min(t0 + i, s.n_q - 1);
        Lane<T, D>::load(Q + ((size_t)bh * s.n_q + t) * D, lane, q[i]);
    }
    const int myq = transpose_index<8>(lane);
    const int tq = t0 + myq;
    const float lse = tq < s.n_q ? ldcg(lv.rowlse + (size_t)bh * s.n_q + tq) : INFINITY;
    __shared__ float s_part[NW][CH];
    const int r0 = chunk * CH;
    for (int rr = 0; rr < CH; ++rr) {
        const int r = r0 + rr;
        float colv = 0.f;
        if (r < nrows) {
            const int row = ROWLIST ? ldcg(rows + r) : r;
            float cf[D / 32];
            Lane<T, D>::load(C + (size_t)row * D, lane, cf);
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                float acc = 0.f;
#pragma unroll
                for (int k = 0; k < D / 32; ++k) acc = fmaf(q[i][k], cf[k], acc);
                v[i] = acc;
            }
            const float sv = transpose_reduce<8>(v, lane) * s.scale;
            float p = (lse == INFINITY || lse == -INFINITY) ? 0.f : expf(sv - lse);
            // sum over the 8 distinct queries (lanes differing in bits 2..4)
            p += __shfl_xor_sync(FULL, p, 4);
            p += __shfl_xor_sync(FULL, p, 8);
            p += __shfl_xor_sync(FULL, p, 16);
            colv = p;
        }
        if (lane == 0) s_part[warp][rr] = colv;
    }
    __syncthreads();
    for (int rr = threadIdx.x; rr < CH; rr += NT) {
        const int r = r0 + rr;
        if (r < nrows) {
            float acc = 0.f;
            for (int w = 0; w < NW; ++w) acc += s_part[w][rr];
            const int row = ROWLIST ? ldcg(rows + r) : r;
            lv.colpart[((size_t)tile * s.B * s.H + bh) * c + row] = acc;
        }
    }
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        const int t = ticket_acq_rel(lv.tick + bh);
        s_last = (t == (int)(gridDim.x * gridDim.y) - 1);
        if (s_last) lv.tick[bh] = 0;
    }
    __syncthreads();
    if (!s_last) return;
    finalize_colpart<ROWLIST>(lv, bh, h, nrows, nqt, s.B * s.H, 1.0f / (float)s.n_q);
}

// --------------------------------------------------------------------------
constexpr size_t DECODE_SMEM_MAX = 200 * 1024;
static bool decode_fits(int NB, int rowspace, int nc) {
    return decode_smem_bytes(NB, (rowspace + nc - 1) / nc) <= DECODE_SMEM_MAX;
}

template <typename T, int D, int NB, bool RL, int NC, bool SLIM = false>
static cudaError_t launch_decode_nc(const LookupShape &s, const T *Q, const LevelArgs &lv, int rowspace,
                                    int groups, cudaStream_t st) {
    const int rpc = (rowspace + NC - 1) / NC;
    const size_t smem = decode_smem_bytes(NB, rpc, SLIM);
    if (smem > DECODE_SMEM_MAX) return cudaErrorInvalidValue;
    constexpr int UMAX = decode_u_max<T, NB>();
    auto kern = k_lookup_decode<T, D, NB, RL, NC, SLIM, UMAX>;
    if constexpr (UMAX == 32 && !RL)
        if (rpc <= NW * 16) kern = k_lookup_decode<T, D, NB, RL, NC, SLIM, 16>;
    if constexpr (NB == 1 && !RL && !SLIM)
        if (lv.lean && rpc <= NW * 16) kern = k_lookup_decode<T, D, NB, RL, NC, SLIM, 16, 3>;
    if (smem > 48 * 1024) {
        cudaError_t e = ensure_func_attr((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    if (NC > 8) {
        cudaError_t e = ensure_func_attr((const void *)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(NC, s.H, groups);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = NC;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = RL && SQZ_L2_PDL ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, s, Q, lv, rpc);
}

#ifndef SQZ_LOOKUP_MIN_CTAS
#define SQZ_LOOKUP_MIN_CTAS 256
#endif
// the smallest cluster whose CTAs' rows fit 110 KB (2 CTAs per SM, which is
// also the register limit) while the grid keeps >= 256 CTAs (one wave):
// fewer, longer CTAs amortise the per-CTA phases (fold, compaction, cluster
// exchanges), e.g. 2-CTA clusters for batched Level-2 lookups.  Returns NC;
// slim = the 12 B/row layout (one query, large row space: keeps 8-CTA clusters).
static int pick_nc(int NB, int rowspace, int units, bool &slim) {
    slim = false;
    const int min_ctas = SQZ_LOOKUP_MIN_CTAS;
    auto ok = [&](int nc) {
        return decode_smem_bytes(NB, (rowspace + nc - 1) / nc) <= 110 * 1024 && nc * units >= min_ctas;
    };
    if (ok(2)) return 2;
    if (ok(4)) return 4;
    if (ok(8) || decode_smem_bytes(NB, (rowspace + 7) / 8) <= 110 * 1024) return 8;
    if (NB == 1 && decode_smem_bytes(1, (rowspace + 7) / 8, true) <= 110 * 1024) {
        slim = true;
        return 8;
    }
    return 16;
}

template <typename T, int D, int NB, bool RL>
static cudaError_t launch_decode(const LookupShape &s, const T *Q, const LevelArgs &lv, int rowspace,
                                 int groups, cudaStream_t st) {
    bool slim;
    switch (pick_nc(NB, rowspace, s.H * groups, slim)) {
        case 2: return launch_decode_nc<T, D, NB, RL, 2>(s, Q, lv, rowspace, groups, st);
        case 4: return launch_decode_nc<T, D, NB, RL, 4>(s, Q, lv, rowspace, groups, st);
        case 8:
            if constexpr (NB == 1)
                if (slim) return launch_decode_nc<T, D, NB, RL, 8, true>(s, Q, lv, rowspace, groups, st);
            return launch_decode_nc<T, D, NB, RL, 8>(s, Q, lv, rowspace, groups, st);
        default: return launch_decode_nc<T, D, NB, RL, 16>(s, Q, lv, rowspace, groups, st);
    }
}

// --------------------------------------------------------------------------
// Prefill lookup on the 5th-generation tensor cores (bf16): one CTA of 8 warps
// per (128-query tile, b*h).  The centroid rows of the (candidate) row space
// are streamed in 128-row tiles (cp.async gather into the 128B-swizzled
// operand layout, double-buffered), and every tile is multiplied twice
// (the paper's kernel also recomputes the scores):
//   pass 1: S = Q C^T (M = queries): thread = query row, the online
//           (m, D = sum N e^(s-m)) over its half of the columns, the two halves
//           folded in fixed order -> LSE_t;
//   pass 2: S^T = C Q^T (M = centroids): thread = centroid row, so the column
//           sum S-bar_i = sum_t e^(s_ti - LSE_t) is a per-thread sum over its
//           half of the queries (4 interleaved fp32 accumulators, fixed order)
//           -- no shuffles, no float atomics, deterministic (numerics rule 4).
// Both MMAs read the same two K-major smem tiles; only the operand roles swap.
// Exponentials are ex2.approx(x log2 e) (relative error ~2e-7, inside the
// 1e-5 selection band; the arguments are O(1) differences, never raw logits).
// The last CTA of each (b,h) averages the q-tile partials and thresholds.
// --------------------------------------------------------------------------
constexpr int PL_T = 128;   // query rows per CTA = centroid rows per tile
constexpr int PL_NT = 256;  // 8 warps: (TMEM lane quarter) x (column half)

struct PlMaps {
    CUtensorMap c;  // centroids [H][c][D] bf16, box {64, 128, 1}, 128B swizzle
    CUtensorMap q;  // queries [B*H][n_q][D] bf16, same box
};

template <int D> struct PlSmem {
    static constexpr int TILE = PL_T * D * 2;
    static constexpr int Q = 0;
    static constexpr int C0 = Q + TILE;              // 2 buffers
    static constexpr int MISC = C0 + 2 * TILE;  // 5 mbarriers + TMEM address
    static constexpr int BYTES = MISC + 64 + 1024;
};

// GATHERED (with ROWLIST): the candidate rows were first copied, per (b,h) and in
// list order, into the contiguous buffer lv.cgather [B*H][c][D] (k_gather_cand),
// so every query tile loads them with TMA boxes like a full table: the copy is
// read once, the n_q / 128 query tiles of the (b,h) reuse it from L2.
template <int D, bool ROWLIST, bool GATHERED>
__global__ void __launch_bounds__(PL_NT, 2) k_prefill_lookup_tc(LookupShape s,
                                                                 const __nv_bfloat16 *__restrict__ Q,
                                                                 LevelArgs lv,
                                                                 const __grid_constant__ PlMaps maps) {
    using SM = PlSmem<D>;
    constexpr int CPR = D * 2 / 16;
    constexpr int HB = PL_T * 128;
    constexpr uint32_t IDESC = idesc_bf16(128, PL_T, false);
    extern __shared__ unsigned char smem_raw[];
    unsigned char *sm = reinterpret_cast<unsigned char *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const uint32_t sbase = smem_u32(sm);
    // small per-tile metadata in static shared memory (plain LDS/STS)
    __shared__ __align__(16) float s_nw[4 * PL_T];
    __shared__ int s_rid[4 * PL_T];
    __shared__ __align__(16) float s_lse[PL_T];
    __shared__ float2 s_half[2 * PL_T];
    uint64_t *mbar = reinterpret_cast<uint64_t *>(sm + SM::MISC);     // [2] MMA done
    uint64_t *tbar = mbar + 2;                                           // [2] C tile landed (TMA)
    uint64_t *qbar = mbar + 4;                                           // Q tile landed (TMA)
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(sm + SM::MISC + 48);
    constexpr uint32_t TILE_BYTES = PL_T * D * 2;
    __shared__ int s_last;

    asm volatile("griddepcontrol.launch_dependents;");
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int quarter = warp & 3, hf = warp >> 2;  // TMEM lanes [32q, +32), columns [64hf, +64)
    const int r = quarter * 32 + lane;              // TMEM lane = M row of this thread
    const int qt = blockIdx.x, bh = blockIdx.y, h = bh % s.H;
    const int t0 = qt * PL_T, c = lv.c;
    const __nv_bfloat16 *C = reinterpret_cast<const __nv_bfloat16 *>(lv.C) + (size_t)h * c * D;
    const int32_t *N = lv.N + (size_t)h * c;
    const int nrows = ROWLIST ? ldcg(lv.n_rows + bh) : c;
    const int32_t *rows = ROWLIST ? lv.rows + (size_t)bh * lv.row_stride : nullptr;
    const int ntile = (nrows + PL_T - 1) / PL_T;

    if (warp == 0) tmem_alloc(s_tmem, 256);
    if (tid == 0) {
        for (int i = 0; i < 5; ++i) mbar_init(&mbar[i], 1);
        mbar_fence_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    SQZ_TRACE_AT(g_trace_pl, 0);

    // Q tile (rows beyond n_q are zero): TMA for contiguous tables, else cp.async
    if constexpr (!ROWLIST || GATHERED) {
        if (tid == 0) {
            mbar_arrive_expect_tx(qbar, TILE_BYTES);
#pragma unroll
            for (int hb = 0; hb < D / 64; ++hb) tma_load_3d(sbase + SM::Q + hb * HB, &maps.q, hb * 64, t0, bh, qbar);
        }
    } else {
        const __nv_bfloat16 *Qb = Q + ((size_t)bh * s.n_q + t0) * D;
        for (int e = tid; e < PL_T * CPR; e += PL_NT) {
            const int rr = e / CPR, cc = e % CPR;
            const bool valid = t0 + rr < s.n_q;
            cp_async16_zfill(sbase + SM::Q + (cc >> 3) * HB + sw128_off(rr, cc & 7),
                             Qb + (size_t)(valid ? rr : 0) * D + cc * 8, valid);
        }
    }
    // pass 1 then pass 2 over the same tiles; the staged lookup runs them as
    // separate launches (phase 1: pass 1 only; phase 2: pass 2 only, with the
    // LSE folded over the shards)
    const int first = lv.phase == 2 ? ntile : 0;
    const int total = lv.phase == 1 ? ntile : 2 * ntile;
    // Tile j (iteration k = j - first) lives in C buffer k & 1, TMEM buffer
    // k & 1 and metadata slot k & 3.  Thread t gathers row t & 127 of a tile
    // (8 of its 16-byte chunks), computing that row's id itself, so a tile
    // load needs no barrier; slot writes by threads < 128.
    auto tile_meta = [&](int j, int &rid, float &nw) {
        rid = -1;
        nw = 0.f;
        if (j < total) {  // (ntile > 0 here: no j % 0, which would let the compiler assume it away)
            const int jj = (j % ntile) * PL_T + (tid & (PL_T - 1));
            if (jj < nrows) {
                rid = ROWLIST ? ldcg(rows + jj) : jj;
                nw = (float)__ldg(N + rid);
            }
        }
    };
    auto load_tile = [&](int j, int rid, float nw) {
        const int k = j - first, rr = tid & (PL_T - 1);
        if (tid < PL_T) {
            s_rid[(k & 3) * PL_T + rr] = rid;
            s_nw[(k & 3) * PL_T + rr] = nw;
        }
        const uint32_t dst = sbase + SM::C0 + (k & 1) * SM::TILE;
        if constexpr (!ROWLIST || GATHERED) {  // one thread: two 64-column boxes, rows past c zero-filled
            if (tid == 0) {
                mbar_arrive_expect_tx(&tbar[k & 1], TILE_BYTES);
#pragma unroll
                for (int hb = 0; hb < D / 64; ++hb)
                    tma_load_3d(dst + hb * HB, &maps.c, hb * 64, (j % ntile) * PL_T, GATHERED ? bh : h,
                                &tbar[k & 1]);
            }
        } else {
            for (int cc = (tid / PL_T) * (CPR / 2); cc < (tid / PL_T + 1) * (CPR / 2); ++cc)
                cp_async16_zfill(dst + (cc >> 3) * HB + sw128_off(rr, cc & 7),
                                 C + (size_t)(rid >= 0 ? rid : 0) * D + cc * 8, rid >= 0);
            cp_async_commit_grp();
        }
    };
    // thread 0, before issuing MMA(j): the TMA loads of its operands have landed
    auto wait_tile = [&](int j) {
        if constexpr (!ROWLIST || GATHERED) {
            const int k = j - first;
            if (k == 0) mbar_wait(qbar, 0);
            mbar_wait(&tbar[k & 1], (k >> 1) & 1);
        }
    };
    auto issue_mma = [&](int j) {  // one elected thread
        const int k = j - first;
        const bool p0 = j < ntile;  // pass 1: S = Q C^T; pass 2: S^T = C Q^T
        const uint32_t qa = sbase + SM::Q, ca = sbase + SM::C0 + (k & 1) * SM::TILE;
        const uint32_t a_base = p0 ? qa : ca, b_base = p0 ? ca : qa;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t off = (ks >> 2) * HB + (ks & 3) * 32;
            umma_bf16(tmem + (k & 1) * 128, sdesc_sw128(a_base + off, 16, 1024),
                      sdesc_sw128(b_base + off, 16, 1024), IDESC, ks > 0);
        }
        umma_commit(&mbar[k & 1]);
    };
    const bool row_ok = t0 + r < s.n_q;  // pass 1: this thread's query row
    if (tid < PL_T) {
        float lse = INFINITY;
        if (lv.phase == 2 && t0 + tid < s.n_q) {
            const float2 g2 = ldcg(lv.gstat + (size_t)bh * s.n_q + t0 + tid);
            lse = g2.x + g2.y;
            if (lv.dbg_lse) lv.dbg_lse[(size_t)bh * s.n_q + t0 + tid] = lse;
            if (!(lse < INFINITY) || lse == -INFINITY) lse = INFINITY;  // no row: p = 0
        }
        s_lse[tid] = lse * LOG2E;  // log2 units (pass 2 works in the log2 domain)
    }
    cp_async_commit_grp();  // the Q tile
    int rid_pf;
    float nw_pf;
    tile_meta(first, rid_pf, nw_pf);
    if (first < total) load_tile(first, rid_pf, nw_pf);
    tile_meta(first + 1, rid_pf, nw_pf);
    if (first + 1 < total) load_tile(first + 1, rid_pf, nw_pf);
    else cp_async_commit_grp();  // keep one group per slot so the wait below covers `first`
    tile_meta(first + 2, rid_pf, nw_pf);  // prefetched: consumed by load_tile(first + 2)
    cp_async_wait_grp<1>();  // Q and tile `first` landed (tile first+1 may be in flight)
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0 && first < total) {
        wait_tile(first);
        tc_fence_after();
        issue_mma(first);
    }

    SQZ_TRACE_AT(g_trace_pl, 1);
    // both passes work in the log2 domain: s2 = scale log2(e) q.c, m and LSE in
    // log2 units, exponentials ex2.approx (one multiply fewer per element)
    const float sl2 = s.scale * LOG2E;
    float m = -INFINITY, Dsum = 0.f;
    for (int it = first; it < total; ++it) {
        if (it == ntile) SQZ_TRACE_AT(g_trace_pl, 2);
        const int k = it - first, buf = k & 1, tl = it % ntile, pass = it / ntile;
        // MMA of the next tile into the other TMEM buffer, overlapping this epilogue
        cp_async_wait_all();
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0 && it + 1 < total) {
            wait_tile(it + 1);
            tc_fence_after();
            issue_mma(it + 1);
        }
        PL_IT(k, 0);
        mbar_wait(&mbar[buf], (k >> 1) & 1);
        tc_fence_after();
        PL_IT(k, 1);
        if (it + 2 < total) load_tile(it + 2, rid_pf, nw_pf);  // MMA(it) no longer reads buffer `buf`
        tile_meta(it + 3, rid_pf, nw_pf);  // latency hidden behind this epilogue
        const float *nwb = s_nw + (k & 3) * PL_T;
        if (pass == 0) {
            // thread = query row r; columns = centroids hf*64 + [0, 64) of tile tl
            float v0[32], v1[32];
            tmem_ld32(tmem + buf * 128 + lane_off + hf * 64, v0);
            tmem_ld32(tmem + buf * 128 + lane_off + hf * 64 + 32, v1);
            tmem_wait_ld();
            const int lim = nrows - tl * PL_T - hf * 64;  // valid columns of this half
            float cmx = -INFINITY;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                v0[j] = j < lim ? v0[j] * sl2 : -INFINITY;
                v1[j] = j + 32 < lim ? v1[j] * sl2 : -INFINITY;
                cmx = fmaxf(cmx, fmaxf(v0[j], v1[j]));
            }
            const float mn = fmaxf(m, cmx);
            if (mn != -INFINITY) {
                const float4 *nw4 = reinterpret_cast<const float4 *>(nwb + hf * 64);
                float a[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) a[u] = 0.f;
#pragma unroll
                for (int j = 0; j < 32; j += 4) {
                    const float4 w0 = nw4[j / 4], w1 = nw4[8 + j / 4];
                    a[0] = fmaf(w0.x, fast_exp2(v0[j] - mn), a[0]);
                    a[1] = fmaf(w0.y, fast_exp2(v0[j + 1] - mn), a[1]);
                    a[2] = fmaf(w0.z, fast_exp2(v0[j + 2] - mn), a[2]);
                    a[3] = fmaf(w0.w, fast_exp2(v0[j + 3] - mn), a[3]);
                    a[4] = fmaf(w1.x, fast_exp2(v1[j] - mn), a[4]);
                    a[5] = fmaf(w1.y, fast_exp2(v1[j + 1] - mn), a[5]);
                    a[6] = fmaf(w1.z, fast_exp2(v1[j + 2] - mn), a[6]);
                    a[7] = fmaf(w1.w, fast_exp2(v1[j + 3] - mn), a[7]);
                }
                Dsum = Dsum * exp2f(m - mn) + (((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7])));
                m = mn;
            }
            if (tl == ntile - 1) {  // fold the two column halves of each query row
                s_half[hf * PL_T + r] = make_float2(m * LN2, Dsum);  // natural units for the fold
                __syncthreads();
                if (tid < PL_T) {
                    const float2 h0 = s_half[tid], h1 = s_half[PL_T + tid];
                    float mm = h0.x, dd = h0.y;
                    md_combine(mm, dd, h1.x, h1.y);
                    const bool ok = t0 + tid < s.n_q;
                    if (lv.phase == 1) {
                        if (ok) lv.stats_out[(size_t)bh * s.n_q + t0 + tid] = make_float2(mm, dd);
                    } else {
                        float lse = mm + logf(dd);  // -inf when no row
                        if (ok) {
                            lv.rowlse[(size_t)bh * s.n_q + t0 + tid] = lse;
                            if (lv.dbg_lse) lv.dbg_lse[(size_t)bh * s.n_q + t0 + tid] = lse;
                        }
                        if (!ok || !(lse < INFINITY) || lse == -INFINITY) lse = INFINITY;
                        s_lse[tid] = lse * LOG2E;
                    }
                }
                // s_lse is read after the next iteration's __syncthreads
            }
        } else {
            // S^T: thread = centroid row r of tile tl; columns = queries hf*64 + [0, 64)
            float v0[32], v1[32];
            tmem_ld32(tmem + buf * 128 + lane_off + hf * 64, v0);
            tmem_ld32(tmem + buf * 128 + lane_off + hf * 64 + 32, v1);
            tmem_wait_ld();
            const float4 *l4 = reinterpret_cast<const float4 *>(s_lse + hf * 64);
            float a[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = 0.f;
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
                const float4 e0 = l4[j / 4], e1 = l4[8 + j / 4];
                a[0] += fast_exp2(fmaf(v0[j], sl2, -e0.x));
                a[1] += fast_exp2(fmaf(v0[j + 1], sl2, -e0.y));
                a[2] += fast_exp2(fmaf(v0[j + 2], sl2, -e0.z));
                a[3] += fast_exp2(fmaf(v0[j + 3], sl2, -e0.w));
                a[4] += fast_exp2(fmaf(v1[j], sl2, -e1.x));
                a[5] += fast_exp2(fmaf(v1[j + 1], sl2, -e1.y));
                a[6] += fast_exp2(fmaf(v1[j + 2], sl2, -e1.z));
                a[7] += fast_exp2(fmaf(v1[j + 3], sl2, -e1.w));
            }
            const float a0 = a[0] + a[1], a1 = a[2] + a[3], a2 = a[4] + a[5], a3 = a[6] + a[7];
            s_half[hf * PL_T + r].x = (a0 + a1) + (a2 + a3);
            __syncthreads();
            if (tid < PL_T) {
                const int rid = s_rid[(k & 3) * PL_T + tid];
                if (rid >= 0)
                    lv.colpart[((size_t)qt * s.B * s.H + bh) * c + rid] = s_half[tid].x + s_half[PL_T + tid].x;
            }
        }
        PL_IT(k, 2);
        tc_fence_before();
    }
    __syncthreads();
    SQZ_TRACE_AT(g_trace_pl, 3);
    if (warp == 0) tmem_dealloc(tmem, 256);
    if (lv.phase == 1) {
        if (ntile == 0 && tid < PL_T && t0 + tid < s.n_q)  // no rows: the identity statistics
            lv.stats_out[(size_t)bh * s.n_q + t0 + tid] = make_float2(-INFINITY, 0.f);
        return;
    }
    // ---- the last CTA of this (b,h) averages the tiles and thresholds ----
    __syncthreads();
    if (tid == 0) {
        const int t = ticket_acq_rel(lv.tick + bh);
        s_last = (t == (int)gridDim.x - 1);
        if (s_last) lv.tick[bh] = 0;
    }
    __syncthreads();
    if (!s_last) return;
    SQZ_TRACE_AT(g_trace_pl, 4);
    finalize_colpart<ROWLIST>(lv, bh, h, nrows, gridDim.x, s.B * s.H, 1.0f / (float)s.n_q);
    SQZ_TRACE_AT(g_trace_pl, 5);
}

// --------------------------------------------------------------------------
// Warp-specialised prefill lookup (TMA tables: full tables or gathered candidate
// lists).  Same arithmetic and outputs as k_prefill_lookup_tc; the roles:
//   warp 8      TMA producer: the Q tile once, then the C tiles of pass 1 and
//               pass 2 through a 3-stage ring;
//   warp 9      MMA issuer: tile t (S = Q C^T in pass 1, S^T = C Q^T in pass 2)
//               into TMEM buffer t % 4 (4 x 128 columns);
//   warps 0-3   epilogue group 0 (even tiles), warps 4-7 group 1 (odd tiles):
//               a thread owns a whole TMEM lane (128 columns) of its tiles, so
//               the two groups' exponentials overlap each other and the MMAs
//               without a CTA-wide barrier per tile.
// Pass 1 leaves each group a partial (m, D) per query row; they are folded
// (group 0 tiles then group 1 -- a fixed order) before pass 2 needs the LSE.
// --------------------------------------------------------------------------
constexpr int PW_NT = 320;

template <int D, bool GATHERED>
__global__ void __launch_bounds__(PW_NT, 1) k_prefill_lookup_ws(LookupShape s, LevelArgs lv,
                                                                const __grid_constant__ PlMaps maps) {
    constexpr int HB = PL_T * 128;                 // one 64-column half of a 128-row tile
    constexpr uint32_t TILE = PL_T * D * 2;        // 32 KB at d = 128
    constexpr int NST = 3;                         // C ring stages
    constexpr uint32_t IDESC = idesc_bf16(128, PL_T, false);
    extern __shared__ unsigned char smem_raw[];
    unsigned char *sm = reinterpret_cast<unsigned char *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const uint32_t sQ = smem_u32(sm), sC = sQ + TILE;
    __shared__ __align__(8) uint64_t c_full[NST], c_empty[NST], acc_full[4], acc_empty[4], q_full;
    __shared__ uint32_t s_tmem;
    __shared__ __align__(16) float s_nw[2][2][PL_T];  // per group, double-buffered tile weights
    __shared__ int s_rid[2][2][PL_T];
    __shared__ float2 s_md[2][PL_T];
    __shared__ __align__(16) float s_lse[PL_T];
    __shared__ int s_last;

    asm volatile("griddepcontrol.launch_dependents;");
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int qt = blockIdx.x, bh = blockIdx.y, h = bh % s.H;
    const int t0 = qt * PL_T, c = lv.c;
    const int32_t *N = lv.N + (size_t)h * c;
    const int nrows = GATHERED ? ldcg(lv.n_rows + bh) : c;
    const int32_t *rows = GATHERED ? lv.rows + (size_t)bh * lv.row_stride : nullptr;
    const int ntile = (nrows + PL_T - 1) / PL_T;
    const int total = 2 * ntile;
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(&c_full[i], 1);
            mbar_init(&c_empty[i], 1);
        }
        for (int i = 0; i < 4; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], 4);
        }
        mbar_init(&q_full, 1);
        mbar_fence_init();
    }
    if (warp == 9) tmem_alloc(&s_tmem, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    if (warp == 8) {
        // ======================= TMA producer =======================
        if (lane == 0) {
            mbar_arrive_expect_tx(&q_full, TILE);
#pragma unroll
            for (int hb = 0; hb < D / 64; ++hb) tma_load_3d(sQ + hb * HB, &maps.q, hb * 64, t0, bh, &q_full);
            for (int t = 0; t < total; ++t) {
                const int st = t % NST;
                mbar_wait(&c_empty[st], ((t / NST) & 1) ^ 1);
                mbar_arrive_expect_tx(&c_full[st], TILE);
#pragma unroll
                for (int hb = 0; hb < D / 64; ++hb)
                    tma_load_3d(sC + st * TILE + hb * HB, &maps.c, hb * 64, (t % ntile) * PL_T,
                                GATHERED ? bh : h, &c_full[st]);
            }
        }
    } else if (warp == 9) {
        // ======================= MMA issuer =======================
        mbar_wait(&q_full, 0);
        tc_fence_after();
        for (int t = 0; t < total; ++t) {
            const int st = t % NST, buf = t & 3;
            mbar_wait(&c_full[st], (t / NST) & 1);
            mbar_wait(&acc_empty[buf], ((t >> 2) & 1) ^ 1);
            tc_fence_after();
            const bool p0 = t < ntile;  // pass 1: S = Q C^T; pass 2: S^T = C Q^T
            const uint32_t ca = sC + st * TILE;
            const uint32_t a_base = p0 ? sQ : ca, b_base = p0 ? ca : sQ;
            if (lane == 0) {
#pragma unroll
                for (int ks = 0; ks < D / 16; ++ks) {
                    const uint32_t off = (ks >> 2) * HB + (ks & 3) * 32;
                    umma_bf16(tmem + buf * 128, sdesc_sw128(a_base + off, 16, 1024),
                              sdesc_sw128(b_base + off, 16, 1024), IDESC, ks > 0);
                }
                umma_commit(&c_empty[st]);
                umma_commit(&acc_full[buf]);
            }
            __syncwarp();
        }
    } else {
        // ======================= epilogue groups =======================
        const int grp = warp >> 2, quarter = warp & 3;
        const int r = quarter * 32 + lane;              // TMEM lane = M row of this thread
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        const int gtid = tid & 127, bar_id = 1 + grp;   // named barrier of the group (128 threads)
        // this group's tiles: t = grp, grp + 2, ...; prefetch the first tile's metadata
        auto meta = [&](int t, int &rid, float &nw) {
            rid = -1;
            nw = 0.f;
            if (t < total) {
                const int jj = (t % ntile) * PL_T + gtid;
                if (jj < nrows) {
                    rid = GATHERED ? ldcg(rows + jj) : jj;
                    nw = (float)__ldg(N + rid);
                }
            }
        };
        int rid_pf;
        float nw_pf;
        meta(grp, rid_pf, nw_pf);
        float m = -INFINITY, Dsum = 0.f;
        bool lse_ready = false;
        int k = 0;  // this group's tile count (metadata slot k & 1)
        for (int t = grp; t < total; t += 2, ++k) {
            const int buf = t & 3, tl = t % ntile, slot = k & 1;
            s_nw[grp][slot][gtid] = nw_pf;
            s_rid[grp][slot][gtid] = rid_pf;
            named_bar(bar_id, 128);  // this tile's metadata visible; slot k - 2 readers done
            meta(t + 2, rid_pf, nw_pf);
            if (t >= ntile && !lse_ready) {
                // pass 1 complete in both groups: fold the two groups' (m, D), fixed order
                s_md[grp][r] = make_float2(m, Dsum);
                named_bar(3, 256);
                if (grp == 0) {
                    float mm = s_md[0][r].x, dd = s_md[0][r].y;
                    md_combine(mm, dd, s_md[1][r].x, s_md[1][r].y);
                    const bool ok = t0 + r < s.n_q;
                    float lse = mm + logf(dd);  // -inf when no row
                    if (ok) {
                        lv.rowlse[(size_t)bh * s.n_q + t0 + r] = lse;
                        if (lv.dbg_lse) lv.dbg_lse[(size_t)bh * s.n_q + t0 + r] = lse;
                    }
                    if (!ok || !(lse < INFINITY) || lse == -INFINITY) lse = INFINITY;  // p = 0
                    s_lse[r] = lse;
                }
                named_bar(3, 256);
                lse_ready = true;
            }
            mbar_wait(&acc_full[buf], (t >> 2) & 1);
            tc_fence_after();
            const float *nwb = s_nw[grp][slot];
            if (t < ntile) {
                // pass 1: thread = query row r; the 128 centroid columns of tile tl
#pragma unroll 1
                for (int hf = 0; hf < 2; ++hf) {
                    float v0[32], v1[32];
                    tmem_ld32(tmem + buf * 128 + lane_off + hf * 64, v0);
                    tmem_ld32(tmem + buf * 128 + lane_off + hf * 64 + 32, v1);
                    tmem_wait_ld();
                    const int lim = nrows - tl * PL_T - hf * 64;
                    float cmx = -INFINITY;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        v0[j] = j < lim ? v0[j] * s.scale : -INFINITY;
                        v1[j] = j + 32 < lim ? v1[j] * s.scale : -INFINITY;
                        cmx = fmaxf(cmx, fmaxf(v0[j], v1[j]));
                    }
                    const float mn = fmaxf(m, cmx);
                    if (mn != -INFINITY) {
                        const float4 *nw4 = reinterpret_cast<const float4 *>(nwb + hf * 64);
                        float a[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) a[u] = 0.f;
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
                            const float4 w0 = nw4[j / 4], w1 = nw4[8 + j / 4];
                            a[0] = fmaf(w0.x, exp_fast(v0[j] - mn), a[0]);
                            a[1] = fmaf(w0.y, exp_fast(v0[j + 1] - mn), a[1]);
                            a[2] = fmaf(w0.z, exp_fast(v0[j + 2] - mn), a[2]);
                            a[3] = fmaf(w0.w, exp_fast(v0[j + 3] - mn), a[3]);
                            a[4] = fmaf(w1.x, exp_fast(v1[j] - mn), a[4]);
                            a[5] = fmaf(w1.y, exp_fast(v1[j + 1] - mn), a[5]);
                            a[6] = fmaf(w1.z, exp_fast(v1[j + 2] - mn), a[6]);
                            a[7] = fmaf(w1.w, exp_fast(v1[j + 3] - mn), a[7]);
                        }
                        Dsum = Dsum * expf(m - mn) + (((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7])));
                        m = mn;
                    }
                }
            } else {
                // pass 2: thread = centroid row r of tile tl; the 128 query columns
                float tot = 0.f;
#pragma unroll 1
                for (int hf = 0; hf < 2; ++hf) {
                    float v0[32], v1[32];
                    tmem_ld32(tmem + buf * 128 + lane_off + hf * 64, v0);
                    tmem_ld32(tmem + buf * 128 + lane_off + hf * 64 + 32, v1);
                    tmem_wait_ld();
                    const float4 *l4 = reinterpret_cast<const float4 *>(s_lse + hf * 64);
                    float a[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) a[u] = 0.f;
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        const float4 e0 = l4[j / 4], e1 = l4[8 + j / 4];
                        a[0] += exp_fast(fmaf(v0[j], s.scale, -e0.x));
                        a[1] += exp_fast(fmaf(v0[j + 1], s.scale, -e0.y));
                        a[2] += exp_fast(fmaf(v0[j + 2], s.scale, -e0.z));
                        a[3] += exp_fast(fmaf(v0[j + 3], s.scale, -e0.w));
                        a[4] += exp_fast(fmaf(v1[j], s.scale, -e1.x));
                        a[5] += exp_fast(fmaf(v1[j + 1], s.scale, -e1.y));
                        a[6] += exp_fast(fmaf(v1[j + 2], s.scale, -e1.z));
                        a[7] += exp_fast(fmaf(v1[j + 3], s.scale, -e1.w));
                    }
                    tot += ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
                }
                const int rid = s_rid[grp][slot][r];
                if (rid >= 0) lv.colpart[((size_t)qt * s.B * s.H + bh) * c + rid] = tot;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[buf]);
        }
        if (!lse_ready) {  // a group without pass-2 tiles still takes part in the fold
            s_md[grp][r] = make_float2(m, Dsum);
            named_bar(3, 256);
            if (grp == 0) {
                float mm = s_md[0][r].x, dd = s_md[0][r].y;
                md_combine(mm, dd, s_md[1][r].x, s_md[1][r].y);
                const bool ok = t0 + r < s.n_q;
                float lse = mm + logf(dd);
                if (ok) {
                    lv.rowlse[(size_t)bh * s.n_q + t0 + r] = lse;
                    if (lv.dbg_lse) lv.dbg_lse[(size_t)bh * s.n_q + t0 + r] = lse;
                }
                if (!ok || !(lse < INFINITY) || lse == -INFINITY) lse = INFINITY;
                s_lse[r] = lse;  // the other group's pass-2 tiles read it
            }
            named_bar(3, 256);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) tmem_dealloc(tmem, 512);
    // ---- the last CTA of this (b,h) averages the tiles and thresholds ----
    if (tid == 0) {
        const int tk = ticket_acq_rel(lv.tick + bh);
        s_last = (tk == (int)gridDim.x - 1);
        if (s_last) lv.tick[bh] = 0;
    }
    __syncthreads();
    if (!s_last) return;
    finalize_colpart<GATHERED>(lv, bh, h, nrows, gridDim.x, s.B * s.H, 1.0f / (float)s.n_q);
}

// the candidate rows of every (b,h), in list order, into a contiguous copy
template <int D>
__global__ void k_gather_cand(const __nv_bfloat16 *__restrict__ C, const int32_t *__restrict__ rows,
                              const int32_t *__restrict__ n_rows, int row_stride, int c, int H,
                              __nv_bfloat16 *__restrict__ out) {
    constexpr int V = D * 2 / 16;  // 16-byte chunks per row
    const int bh = blockIdx.y, h = bh % H;
    const int n = ldcg(n_rows + bh);
    const int32_t *rl = rows + (size_t)bh * row_stride;
    const uint4 *src = reinterpret_cast<const uint4 *>(C + (size_t)h * c * D);
    uint4 *dst = reinterpret_cast<uint4 *>(out + (size_t)bh * c * D);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * V; e += gridDim.x * blockDim.x) {
        const int rr = e / V, ch = e - rr * V;
        dst[(size_t)rr * V + ch] = __ldg(src + (size_t)ldcg(rl + rr) * V + ch);
    }
}

template <int D, bool RL, bool GATHERED = false>
static cudaError_t launch_prefill_tc(const LookupShape &s, const __nv_bfloat16 *Q, const LevelArgs &lv,
                                     cudaStream_t st) {
    auto kern = k_prefill_lookup_tc<D, RL, GATHERED>;
    {
        cudaError_t e = ensure_func_attr((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         PlSmem<D>::BYTES);
        if (e != cudaSuccess) return e;
    }
    PlMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    if (GATHERED) {
        k_gather_cand<D><<<dim3(64, s.B * s.H), 256, 0, st>>>(
            reinterpret_cast<const __nv_bfloat16 *>(lv.C), lv.rows, lv.n_rows, lv.row_stride, lv.c, s.H,
            reinterpret_cast<__nv_bfloat16 *>(lv.cgather));
        const uint64_t dc[3] = {(uint64_t)D, (uint64_t)lv.c, (uint64_t)s.B * s.H};
        const uint64_t dq[3] = {(uint64_t)D, (uint64_t)s.n_q, (uint64_t)s.B * s.H};
        const uint32_t box[3] = {64, PL_T, 1};
        if (encode_tmap_bf16_3d(&maps.c, lv.cgather, dc, box) != 0 ||
            encode_tmap_bf16_3d(&maps.q, Q, dq, box) != 0)
            return cudaErrorInvalidValue;
    } else if (!RL) {
        const uint64_t dc[3] = {(uint64_t)D, (uint64_t)lv.c, (uint64_t)s.H};
        const uint64_t dq[3] = {(uint64_t)D, (uint64_t)s.n_q, (uint64_t)s.B * s.H};
        const uint32_t box[3] = {64, PL_T, 1};
        if (encode_tmap_bf16_3d(&maps.c, lv.C, dc, box) != 0 ||
            encode_tmap_bf16_3d(&maps.q, Q, dq, box) != 0)
            return cudaErrorInvalidValue;
    }
    dim3 grid((s.n_q + PL_T - 1) / PL_T, s.B * s.H);
    cudaError_t e;
// warp-specialised kernel for TMA-fed unstaged lookups: correct, but measured
// slower (cfg3 62.3 vs 58.8 us, cfg5p 6.18 vs 5.90 ms): with one CTA per SM the
// 8 epilogue warps leave the xu pipe at 43% like the two-CTA kernel, and the
// second wave of CTAs (256 on 148 SMs) costs more than the overlap gains -- off
#ifndef SQZ_PL_WS
#define SQZ_PL_WS 0
#endif
    if (SQZ_PL_WS && (!RL || GATHERED) && lv.phase == 0) {
        auto kw = k_prefill_lookup_ws<D, GATHERED>;
        constexpr int WBYTES = 4 * PL_T * D * 2 + 1024;  // Q + 3 C stages + alignment
        e = ensure_func_attr((const void *)kw, cudaFuncAttributeMaxDynamicSharedMemorySize, WBYTES);
        if (e != cudaSuccess) return e;
        kw<<<grid, PW_NT, WBYTES, st>>>(s, lv, maps);
    } else {
        kern<<<grid, PL_NT, PlSmem<D>::BYTES, st>>>(s, Q, lv, maps);
    }
    e = cudaGetLastError();
    if (e == cudaSuccess && lv.phase != 1 && lv.exp_list) e = launch_expand(s, lv, st);
    return e;
}

template <typename T, int D>
static cudaError_t launch_level_t(const LookupShape &s, const T *Q, const LevelArgs &lv,
                                  cudaStream_t st) {
    if constexpr (sizeof(T) == 2) {
        // bf16 prefill: tensor-core lookup (fp32 inputs keep the exact FFMA path)
        if (s.n_q > 1) {
            // many query tiles: gather the candidates once, then TMA tiles (4+ tiles)
            if (lv.rows && lv.cgather && s.n_q >= 4 * PL_T) return launch_prefill_tc<D, true, true>(s, Q, lv, st);
            if (lv.rows) return launch_prefill_tc<D, true>(s, Q, lv, st);
            return launch_prefill_tc<D, false>(s, Q, lv, st);
        }
    }
    const bool rl = lv.rows != nullptr;
    const int rowspace = rl ? lv.row_stride : lv.c;
    const int nch = (rowspace + CH - 1) / CH;
    if (s.n_q == 1) {
        // queries per cluster: the largest NB <= B whose logits fit a 16-CTA cluster
        if (rl) return launch_decode<T, D, 1, true>(s, Q, lv, rowspace, s.B, st);
        if (s.B >= 8 && decode_fits(8, rowspace, 16))
            return launch_decode<T, D, 8, false>(s, Q, lv, rowspace, (s.B + 7) / 8, st);
        if (s.B >= 4 && decode_fits(4, rowspace, 16))
            return launch_decode<T, D, 4, false>(s, Q, lv, rowspace, (s.B + 3) / 4, st);
        if (s.B >= 2 && decode_fits(2, rowspace, 16))
            return launch_decode<T, D, 2, false>(s, Q, lv, rowspace, (s.B + 1) / 2, st);
        return launch_decode<T, D, 1, false>(s, Q, lv, rowspace, s.B, st);
    }
    const int nqt = (s.n_q + QT - 1) / QT;
    dim3 g1(nqt, s.B * s.H);
    dim3 g2(nch, nqt, s.B * s.H);
    // staged: phase 1 = row statistics only, phase 2 = column sums against the
    // folded LSE (written into lv.rowlse by the fold)
    if (rl) {
        if (lv.phase != 2) k_prefill_rowlse<T, D, true><<<g1, NT, 0, st>>>(s, Q, lv);
        if (lv.phase != 1) k_prefill_colsum<T, D, true><<<g2, NT, 0, st>>>(s, Q, lv);
    } else {
        if (lv.phase != 2) k_prefill_rowlse<T, D, false><<<g1, NT, 0, st>>>(s, Q, lv);
        if (lv.phase != 1) k_prefill_colsum<T, D, false><<<g2, NT, 0, st>>>(s, Q, lv);
    }
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && lv.phase != 1 && lv.exp_list) e = launch_expand(s, lv, st);
    return e;
}

cudaError_t launch_lookup_level(const LookupShape &s, const void *Q, const LevelArgs &lv,
                                cudaStream_t st) {
    if (s.dtype == SQZ_BF16) {
        if (s.d == 128) return launch_level_t<__nv_bfloat16, 128>(s, (const __nv_bfloat16 *)Q, lv, st);
        return launch_level_t<__nv_bfloat16, 64>(s, (const __nv_bfloat16 *)Q, lv, st);
    }
    if (s.d == 128) return launch_level_t<float, 128>(s, (const float *)Q, lv, st);
    return launch_level_t<float, 64>(s, (const float *)Q, lv, st);
}

}  // namespace sqz
