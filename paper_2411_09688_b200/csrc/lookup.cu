// lookup.cu -- centroid lookup kernels (section 4.1).
//
// Decode (n_q == 1, "generation stage"):
//   k_scan_decode: one CTA per (chunk of CH centroid rows, head, group of NB
//   queries).  Centroid rows are read once per head for the whole query group
//   (the batch shares the fixed context) with 8/16-byte coalesced
//   loads; logits s_i = scale*q.C_i are fp32 FFMA over exact bf16->fp32
//   products.  Each CTA stores its logits and a per-query (m, D = sum N e^(s-m))
//   partial; the LAST CTA of each (group, head) (atomic ticket) folds the
//   partials in a fixed order and runs the threshold + compaction epilogue:
//   select i  <=>  (s_i - m) > log D + log T      (single-pass form, P:343,
//   max folded into the threshold as in App. C; no second exp).
// Prefill (n_q > 1):
//   k_prefill_rowlse: LSE_t = log sum_j N_j exp(s_tj) for every query row.
//   k_prefill_colsum: S-bar partials sum_t exp(s_ti - LSE_t) per 64-query
//   tile, fixed-order (butterfly + sequential) fp32 reductions, no atomics on
//   floats; the last CTA per (b,h) reduces the tiles and thresholds S-bar > T.
// Both run on an explicit row list for the Level-2 pass of the hierarchy
// (Eq. 3: only the children of the Level-1 survivors).
#include "common.cuh"
#include "internal.h"

namespace sqz {

constexpr int CH = 128;     // centroid rows per CTA
constexpr int NT = 256;     // threads per CTA
constexpr int NW = NT / 32;
constexpr int QT = 64;      // prefill queries per tile (8 warps x 8 queries)

int lookup_chunk_rows() { return CH; }
int lookup_qtile() { return QT; }

// lane-slice loads: lane holds D/32 consecutive elements of a row
template <typename T, int D> struct Lane;
template <> struct Lane<__nv_bfloat16, 128> {
    static __device__ __forceinline__ void load(const __nv_bfloat16 *row, int lane, float (&f)[4]) {
        uint2 u = __ldg(reinterpret_cast<const uint2 *>(row) + lane);
        f[0] = __uint_as_float(u.x << 16); f[1] = __uint_as_float(u.x & 0xffff0000u);
        f[2] = __uint_as_float(u.y << 16); f[3] = __uint_as_float(u.y & 0xffff0000u);
    }
};
template <> struct Lane<__nv_bfloat16, 64> {
    static __device__ __forceinline__ void load(const __nv_bfloat16 *row, int lane, float (&f)[2]) {
        uint32_t u = __ldg(reinterpret_cast<const uint32_t *>(row) + lane);
        f[0] = __uint_as_float(u << 16); f[1] = __uint_as_float(u & 0xffff0000u);
    }
};
template <> struct Lane<float, 128> {
    static __device__ __forceinline__ void load(const float *row, int lane, float (&f)[4]) {
        float4 u = __ldg(reinterpret_cast<const float4 *>(row) + lane);
        f[0] = u.x; f[1] = u.y; f[2] = u.z; f[3] = u.w;
    }
};
template <> struct Lane<float, 64> {
    static __device__ __forceinline__ void load(const float *row, int lane, float (&f)[2]) {
        float2 u = __ldg(reinterpret_cast<const float2 *>(row) + lane);
        f[0] = u.x; f[1] = u.y;
    }
};

// Transposed butterfly: NV per-lane partial dot products -> each lane ends
// with the full 32-lane sum of value index (lane >> (5 - log2 NV)) & (NV-1).
template <int NV>
__device__ __forceinline__ float transpose_reduce(float (&v)[NV], int lane) {
    int stride = 16;
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
template <int NV> __device__ __forceinline__ int transpose_index(int lane) {
    constexpr int lg = NV == 1 ? 0 : NV == 2 ? 1 : NV == 4 ? 2 : 3;
    return (lane >> (5 - lg)) & (NV - 1);
}

// (m, D) online combine with N weights: D = sum N_j exp(s_j - m)
__device__ __forceinline__ void md_combine(float &m, float &D, float m2, float D2) {
    float mn = fmaxf(m, m2);
    if (mn == -INFINITY) return;
    D = D * expf(m - mn) + D2 * expf(m2 - mn);
    m = mn;
}

// --------------------------------------------------------------------------
// Epilogue: threshold + ascending compaction + range expansion, one CTA.
// sel(row) is given by the functor; every selected row's range
// [off[row], off[row+1]) is expanded into exp_list (keys or Level-2 rows).
// --------------------------------------------------------------------------
template <bool ROWLIST, typename SelFn>
__device__ void finalize_rows(const LevelArgs &lv, int bh, int h, int nrows, SelFn selfn) {
    __shared__ int s_wcnt[NW], s_wsum[NW];
    __shared__ int s_run, s_runN;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int32_t *off = lv.off + (size_t)h * (lv.c + 1);
    int32_t *list = lv.list + (size_t)bh * lv.c;
    int32_t *pref = lv.sel_pref + (size_t)bh * lv.c;
    const int32_t *rows = ROWLIST ? lv.rows + (size_t)bh * lv.row_stride : nullptr;
    if (lv.dbg_S && ROWLIST) {
        for (int r = tid; r < lv.c; r += NT) lv.dbg_S[(size_t)bh * lv.c + r] = NAN;
    }
    if (tid == 0) { s_run = 0; s_runN = 0; }
    __syncthreads();
    for (int base = 0; base < nrows; base += NT) {
        const int r = base + tid;
        const bool valid = r < nrows;
        const int row = valid ? (ROWLIST ? ldcg(rows + r) : r) : 0;
        float dbg = 0.f;
        const bool sel = valid && selfn(row, dbg);
        if (valid && lv.dbg_S) lv.dbg_S[(size_t)bh * lv.c + row] = dbg;
        if (valid && lv.bitmap) lv.bitmap[(size_t)bh * lv.c + row] = sel ? 1 : 0;
        const int cnt = sel ? (off[row + 1] - off[row]) : 0;
        const unsigned bal = __ballot_sync(FULL, sel);
        const int wpre = __popc(bal & ((1u << lane) - 1u));
        int inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) { s_wcnt[warp] = __popc(bal); s_wsum[warp] = inc; }
        __syncthreads();
        int wb = 0, nb = 0;
        for (int w = 0; w < warp; ++w) { wb += s_wcnt[w]; nb += s_wsum[w]; }
        if (sel) {
            const int pos = s_run + wb + wpre;
            list[pos] = row;
            pref[pos] = s_runN + nb + inc - cnt;
        }
        __syncthreads();
        if (tid == 0) {
            int tc = 0, tn = 0;
            for (int w = 0; w < NW; ++w) { tc += s_wcnt[w]; tn += s_wsum[w]; }
            s_run += tc;
            s_runN += tn;
        }
        __syncthreads();
    }
    const int nsel = s_run;
    if (tid == 0) {
        lv.n_list[bh] = nsel;
        lv.n_exp[bh] = s_runN;
    }
    int32_t *exp_list = lv.exp_list + (size_t)bh * lv.exp_stride;
    for (int j = warp; j < nsel; j += NW) {
        const int i = list[j];
        const int st = off[i], n = off[i + 1] - st, b0 = pref[j];
        for (int t = lane; t < n; t += 32) exp_list[b0 + t] = st + t;
    }
}

// --------------------------------------------------------------------------
// Decode scan: logits + (m, D) partials, last CTA thresholds.
// --------------------------------------------------------------------------
template <typename T, int D, int NB, bool ROWLIST>
__global__ void __launch_bounds__(NT) k_scan_decode(LookupShape s, const T *__restrict__ Q,
                                                    LevelArgs lv) {
    const int chunk = blockIdx.x, h = blockIdx.y, g = blockIdx.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int H = s.H, c = lv.c;
    const int b0 = g * NB;
    const int nb = min(NB, s.B - b0);
    const T *C = reinterpret_cast<const T *>(lv.C) + (size_t)h * c * D;
    const int32_t *N = lv.N + (size_t)h * c;
    const int nrows = ROWLIST ? ldcg(lv.n_rows + (size_t)b0 * H + h) : c;
    const int32_t *rows = ROWLIST ? lv.rows + ((size_t)b0 * H + h) * lv.row_stride : nullptr;

    float q[NB][D / 32];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        if (i < nb) Lane<T, D>::load(Q + ((size_t)(b0 + i) * H + h) * D, lane, q[i]);
        else
#pragma unroll
            for (int k = 0; k < D / 32; ++k) q[i][k] = 0.f;
    }
    const int myq = transpose_index<NB>(lane);
    float m = -INFINITY, Dsum = 0.f;  // for query myq (lanes sharing myq hold equal values)
    const int r0 = chunk * CH;
    for (int rr = warp; rr < CH; rr += NW) {
        const int r = r0 + rr;
        if (r >= nrows) break;
        const int row = ROWLIST ? ldcg(rows + r) : r;
        float cf[D / 32];
        Lane<T, D>::load(C + (size_t)row * D, lane, cf);
        float v[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < D / 32; ++k) acc = fmaf(q[i][k], cf[k], acc);
            v[i] = acc;
        }
        const float sv = transpose_reduce<NB>(v, lane) * s.scale;
        if (myq < nb) {
            if ((lane & ((32 / NB) - 1)) == 0)
                lv.logits[((size_t)(b0 + myq) * H + h) * c + row] = sv;
            md_combine(m, Dsum, sv, (float)N[row]);
        }
    }
    // fold the 8 warps in fixed order
    __shared__ float s_m[NW][NB], s_d[NW][NB];
    __shared__ int s_last;
    if ((lane & ((32 / NB) - 1)) == 0) { s_m[warp][myq] = m; s_d[warp][myq] = Dsum; }
    __syncthreads();
    if (threadIdx.x < nb) {
        const int i = threadIdx.x;
        float mm = -INFINITY, dd = 0.f;
        for (int w = 0; w < NW; ++w) md_combine(mm, dd, s_m[w][i], s_d[w][i]);
        lv.part[((size_t)(b0 + i) * H + h) * gridDim.x + chunk] = make_float2(mm, dd);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int t = atomicAdd(lv.tick + (size_t)g * H + h, 1);
        s_last = (t == (int)gridDim.x - 1);
        if (s_last) lv.tick[(size_t)g * H + h] = 0;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();

    for (int i = 0; i < nb; ++i) {
        const int bh = (b0 + i) * H + h;
        __shared__ float s_M, s_lD;
        if (warp == 0) {
            float mm = -INFINITY, dd = 0.f;
            for (int j = lane; j < (int)gridDim.x; j += 32) {
                float2 p = ldcg(lv.part + (size_t)bh * gridDim.x + j);
                md_combine(mm, dd, p.x, p.y);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                float m2 = __shfl_xor_sync(FULL, mm, o), d2 = __shfl_xor_sync(FULL, dd, o);
                md_combine(mm, dd, m2, d2);
            }
            if (lane == 0) { s_M = mm; s_lD = logf(dd); }
        }
        __syncthreads();
        const float M = s_M, lD = s_lD;
        const bool all = !(lv.T > 0.f);
        const float thr = all ? -INFINITY : lD + logf(lv.T);
        if (threadIdx.x == 0 && lv.dbg_lse) lv.dbg_lse[bh] = M + lD;
        const float *lg = lv.logits + (size_t)bh * c;
        const int nr = ROWLIST ? ldcg(lv.n_rows + bh) : c;
        finalize_rows<ROWLIST>(lv, bh, h, nr, [&](int row, float &dbg) {
            const float x = ldcg(lg + row) - M;
            dbg = expf(x - lD);
            return all || (x > thr);
        });
        __syncthreads();
    }
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
    if ((lane & 3) == 0 && t < s.n_q) {
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
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int t = atomicAdd(lv.tick + bh, 1);
        s_last = (t == (int)(gridDim.x * gridDim.y) - 1);
        if (s_last) lv.tick[bh] = 0;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const bool all = !(lv.T > 0.f);
    const float inv_nq = 1.0f / (float)s.n_q;
    finalize_rows<ROWLIST>(lv, bh, h, nrows, [&](int row, float &dbg) {
        float acc = 0.f;
        for (int t = 0; t < nqt; ++t) acc += ldcg(lv.colpart + ((size_t)t * s.B * s.H + bh) * c + row);
        const float Sbar = acc * inv_nq;
        dbg = Sbar;
        return all || (Sbar > lv.T);
    });
}

// --------------------------------------------------------------------------
template <typename T, int D>
static cudaError_t launch_level_t(const LookupShape &s, const T *Q, const LevelArgs &lv,
                                  cudaStream_t st) {
    const bool rl = lv.rows != nullptr;
    const int rowspace = rl ? lv.row_stride : lv.c;
    const int nch = (rowspace + CH - 1) / CH;
    if (s.n_q == 1) {
        if (rl) {
            dim3 grid(nch, s.H, s.B);
            k_scan_decode<T, D, 1, true><<<grid, NT, 0, st>>>(s, Q, lv);
        } else if (s.B >= 8) {
            dim3 grid(nch, s.H, (s.B + 7) / 8);
            k_scan_decode<T, D, 8, false><<<grid, NT, 0, st>>>(s, Q, lv);
        } else if (s.B >= 4) {
            dim3 grid(nch, s.H, (s.B + 3) / 4);
            k_scan_decode<T, D, 4, false><<<grid, NT, 0, st>>>(s, Q, lv);
        } else if (s.B >= 2) {
            dim3 grid(nch, s.H, (s.B + 1) / 2);
            k_scan_decode<T, D, 2, false><<<grid, NT, 0, st>>>(s, Q, lv);
        } else {
            dim3 grid(nch, s.H, s.B);
            k_scan_decode<T, D, 1, false><<<grid, NT, 0, st>>>(s, Q, lv);
        }
    } else {
        const int nqt = (s.n_q + QT - 1) / QT;
        dim3 g1(nqt, s.B * s.H);
        dim3 g2(nch, nqt, s.B * s.H);
        if (rl) {
            k_prefill_rowlse<T, D, true><<<g1, NT, 0, st>>>(s, Q, lv);
            k_prefill_colsum<T, D, true><<<g2, NT, 0, st>>>(s, Q, lv);
        } else {
            k_prefill_rowlse<T, D, false><<<g1, NT, 0, st>>>(s, Q, lv);
            k_prefill_colsum<T, D, false><<<g2, NT, 0, st>>>(s, Q, lv);
        }
    }
    return cudaGetLastError();
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
