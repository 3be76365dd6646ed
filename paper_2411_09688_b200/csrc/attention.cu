// attention.cu -- sparse attention over the selected fixed-context keys plus
// the user KV (section 4.2), split-KV + merge.
//
// Work unit = (query row, key chunk of `kch` keys).  A row's chunks are its
// selected fixed keys (key_idx, cluster-major positions into Kp/Vp) followed by
// its visible user keys (causal, bottom-right aligned in prefill, R8).  A head
// with more selected keys simply owns more chunks ("parallelized across a
// greater number of SMs").  Phase 1 writes a normalised partial
// (o, lse) per chunk; phase 2 (k_merge) combines them with the partial
// maxima/denominators.
//
// Decode (n_q == 1) runs PERSISTENT CTAs (grid = SMs x occupancy) that walk a
// device-resident chunk space: each CTA derives the per-row chunk prefix from
// n_keys in shared memory, so nothing returns to the host.
//
// Per chunk, 4 warps stream 16 keys per round each: a group of G = d/8 lanes
// reads one 256-B (d=128 bf16) key row with 16-B non-allocating loads (K and V
// rows of all 16 keys are in flight before the first FMA), the 16 partial dot
// products are reduced with a transposed butterfly (8 shuffles for 16 keys),
// and the online softmax runs in the log2 domain with ex2.approx.
#include "common.cuh"
#include "internal.h"

namespace sqz {

constexpr int AT_NT = 128;  // threads per CTA (4 warps)
constexpr int AT_NW = AT_NT / 32;
constexpr int KEYS_PER_ROUND = 16;

int attention_kch(int n_q) { return n_q == 1 ? 256 : 1024; }

template <typename T> struct Raw { uint4 v[sizeof(T) == 2 ? 1 : 2]; };
__device__ __forceinline__ uint4 ld_nc_v4(const void *p) {
    uint4 u;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
                 : "l"(p));
    return u;
}
template <typename T> __device__ __forceinline__ void ld_raw(Raw<T> &r, const T *p) {
#pragma unroll
    for (int i = 0; i < (int)(sizeof(r.v) / sizeof(uint4)); ++i)
        r.v[i] = ld_nc_v4(reinterpret_cast<const uint4 *>(p) + i);
}
__device__ __forceinline__ void cvt(const Raw<__nv_bfloat16> &r, float (&f)[8]) {
    const uint32_t w[4] = {r.v[0].x, r.v[0].y, r.v[0].z, r.v[0].w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
}
__device__ __forceinline__ void cvt(const Raw<float> &r, float (&f)[8]) {
    f[0] = __uint_as_float(r.v[0].x); f[1] = __uint_as_float(r.v[0].y);
    f[2] = __uint_as_float(r.v[0].z); f[3] = __uint_as_float(r.v[0].w);
    f[4] = __uint_as_float(r.v[1].x); f[5] = __uint_as_float(r.v[1].y);
    f[6] = __uint_as_float(r.v[1].z); f[7] = __uint_as_float(r.v[1].w);
}

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

struct RowInfo {
    int bh, t, nf, nuc, nu_vis;
};

__device__ __forceinline__ RowInfo row_info(const AttnArgs &a, int row) {
    RowInfo r;
    r.bh = row / a.n_q;
    r.t = row % a.n_q;
    const int nk = ldcg(a.n_keys + r.bh);
    r.nf = (nk + a.kch - 1) / a.kch;
    int vis = a.causal ? r.t + a.n_u - a.n_q + 1 : a.n_u;
    vis = max(0, min(vis, a.n_u));
    r.nu_vis = vis;
    r.nuc = (vis + a.kch - 1) / a.kch;
    return r;
}

template <typename T, int D>
__device__ void attend_chunk(const AttnArgs &a, int row, const RowInfo &ri, int chunk,
                             int *s_idx, float *s_m, float *s_l, float *s_o) {
    constexpr int G = D / 8;             // lanes per key row
    constexpr int KPW = 32 / G;          // keys per warp instruction
    constexpr int NS = KEYS_PER_ROUND / KPW;  // key slots per lane per round
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane / G, sub = lane % G;
    const int h = ri.bh % a.H;

    const T *Kb, *Vb;
    int cnt;
    if (chunk < ri.nf) {
        const int nk = ldcg(a.n_keys + ri.bh);
        const int k0 = chunk * a.kch;
        cnt = min(a.kch, nk - k0);
        const int32_t *ki = a.key_idx + (size_t)ri.bh * a.L + k0;
        for (int j = tid; j < cnt; j += AT_NT) s_idx[j] = ldcg(ki + j);
        Kb = reinterpret_cast<const T *>(a.Kp) + (size_t)h * a.L * D;
        Vb = reinterpret_cast<const T *>(a.Vp) + (size_t)h * a.L * D;
    } else {
        const int u0 = (chunk - ri.nf) * a.kch;
        cnt = min(a.kch, ri.nu_vis - u0);
        for (int j = tid; j < cnt; j += AT_NT) s_idx[j] = u0 + j;
        Kb = reinterpret_cast<const T *>(a.Ku) + (size_t)ri.bh * a.n_u * D;
        Vb = reinterpret_cast<const T *>(a.Vu) + (size_t)ri.bh * a.n_u * D;
    }
    // query slice, pre-scaled into the log2 domain
    float q[8];
    {
        const T *qp = reinterpret_cast<const T *>(a.Q) + (size_t)row * D + sub * 8;
        load8(qp, q);
        const float sc = a.scale * LOG2E;
#pragma unroll
        for (int k = 0; k < 8; ++k) q[k] *= sc;
    }
    __syncthreads();

    float m_run = -INFINITY, l_lane = 0.f, o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = 0.f;
    const int myslot = (sub >> 1) & (NS - 1);

    for (int j0 = warp * KEYS_PER_ROUND; j0 < cnt; j0 += AT_NW * KEYS_PER_ROUND) {
        Raw<T> kr[NS], vr[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const int kl = j0 + s * KPW + g;
            if (kl < cnt) {
                const size_t r = (size_t)s_idx[kl] * D + sub * 8;
                ld_raw(kr[s], Kb + r);
                ld_raw(vr[s], Vb + r);
            } else {
#pragma unroll
                for (int i = 0; i < (int)(sizeof(kr[s].v) / sizeof(uint4)); ++i)
                    kr[s].v[i] = vr[s].v[i] = make_uint4(0, 0, 0, 0);
            }
        }
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
        if (j0 + myslot * KPW + g >= cnt) z = -INFINITY;
        const float mx = warp_max(z);
        const float m_new = fmaxf(m_run, mx);
        const float alpha = fast_exp2(m_run - m_new);  // m_run = -inf -> 0
        const float p = fast_exp2(z - m_new);          // z = -inf -> 0
        l_lane = l_lane * alpha + p;
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] *= alpha;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const float ps = __shfl_sync(FULL, p, g * G + 2 * s);
            if (j0 + s * KPW + g < cnt) {
                float f[8];
                cvt(vr[s], f);
#pragma unroll
                for (int k = 0; k < 8; ++k) o[k] = fmaf(ps, f[k], o[k]);
            }
        }
        m_run = m_new;
    }
    // fold the key groups of the warp, then the warps of the CTA
#pragma unroll
    for (int st = G; st < 32; st <<= 1)
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] += __shfl_xor_sync(FULL, o[k], st);
    const float l_w = warp_sum(l_lane) * 0.5f;  // each key is held by two lanes
    if (lane == 0) { s_m[warp] = m_run; s_l[warp] = l_w; }
    if (g == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) s_o[warp * D + sub * 8 + k] = o[k];
    }
    __syncthreads();
    if (tid < D) {
        float M = -INFINITY;
        for (int w = 0; w < AT_NW; ++w) M = fmaxf(M, s_m[w]);
        float L = 0.f, O = 0.f;
        for (int w = 0; w < AT_NW; ++w) {
            const float e = (s_m[w] == -INFINITY) ? 0.f : exp2f(s_m[w] - M);
            L += s_l[w] * e;
            O += s_o[w * D + tid] * e;
        }
        const size_t slot = (size_t)row * a.max_chunks + chunk;
        a.part_o[slot * D + tid] = O / L;
        if (tid == 0) a.part_lse[slot] = (M + log2f(L)) * LN2;
    }
    __syncthreads();
}

// Persistent kernel: chunk space derived on the device from n_keys.
template <typename T, int D>
__global__ void __launch_bounds__(AT_NT) k_attend_persistent(AttnArgs a, int rows) {
    extern __shared__ int s_pref[];  // [rows + 1]
    __shared__ int s_idx[1024];
    __shared__ float s_m[AT_NW], s_l[AT_NW], s_o[AT_NW * D];
    const int tid = threadIdx.x;
    // exclusive prefix of per-row chunk counts (rows <= a few thousand)
    if (tid == 0) s_pref[0] = 0;
    for (int base = 0; base < rows; base += AT_NT) {
        __syncthreads();
        const int r = base + tid;
        int cntc = 0;
        if (r < rows) {
            RowInfo ri = row_info(a, r);
            cntc = ri.nf + ri.nuc;
        }
        // block inclusive scan (simple two-level)
        __shared__ int s_ws[AT_NW];
        int inc = cntc;
        const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(FULL, inc, o);
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
    const int total = s_pref[rows];
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
        // row = last r with s_pref[r] <= w
        int lo = 0, hi = rows - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_pref[mid] <= w) lo = mid; else hi = mid - 1;
        }
        const RowInfo ri = row_info(a, lo);
        attend_chunk<T, D>(a, lo, ri, w - s_pref[lo], s_idx, s_m, s_l, s_o);
    }
}

// Grid kernel (prefill rows): blockIdx.x = row, blockIdx.y = chunk.
template <typename T, int D>
__global__ void __launch_bounds__(AT_NT) k_attend_grid(AttnArgs a) {
    __shared__ int s_idx[1024];
    __shared__ float s_m[AT_NW], s_l[AT_NW], s_o[AT_NW * D];
    const int row = blockIdx.x, chunk = blockIdx.y;
    const RowInfo ri = row_info(a, row);
    if (chunk >= ri.nf + ri.nuc) return;
    attend_chunk<T, D>(a, row, ri, chunk, s_idx, s_m, s_l, s_o);
}

// Merge the chunk partials of each row.
template <int D, typename TO>
__global__ void k_merge_rows(AttnArgs a) {
    const int row = blockIdx.x, tid = threadIdx.x;
    const RowInfo ri = row_info(a, row);
    const int P = ri.nf + ri.nuc;
    const float *lse = a.part_lse + (size_t)row * a.max_chunks;
    float M = -INFINITY;
    for (int p = 0; p < P; ++p) M = fmaxf(M, ldcg(lse + p));
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
        for (int p = 0; p < P; ++p) {
            const float w = expf(ldcg(lse + p) - M);
            L += w;
            O += w * ldcg(a.part_o + ((size_t)row * a.max_chunks + p) * D + tid);
        }
        O /= L;
    }
    reinterpret_cast<TO *>(a.O)[(size_t)row * D + tid] = from_f32<TO>(O);
    if (tid == 0) {
        a.LSE[row] = (M == -INFINITY) ? -INFINITY : M + logf(L);
        if (M == -INFINITY && !a.partial) atomicOr(a.status, 1);
    }
}

template <typename T, int D>
static cudaError_t launch_t(const AttnArgs &a, cudaStream_t st) {
    const int rows = a.B * a.H * a.n_q;
    if (rows == 0) return cudaSuccess;
    if (a.n_q == 1 && rows <= 8192) {
        static int nsm = 0, occ = 0;
        const size_t dsm = (size_t)(rows + 1) * sizeof(int);
        if (dsm > 48 * 1024)
            cudaFuncSetAttribute(k_attend_persistent<T, D>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_attend_persistent<T, D>, AT_NT, dsm);
        if (occ < 1) occ = 1;
        k_attend_persistent<T, D><<<nsm * occ, AT_NT, dsm, st>>>(a, rows);
    } else {
        dim3 grid(rows, a.max_chunks);
        k_attend_grid<T, D><<<grid, AT_NT, 0, st>>>(a);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (a.out_dtype == SQZ_BF16) k_merge_rows<D, __nv_bfloat16><<<rows, D, 0, st>>>(a);
    else k_merge_rows<D, float><<<rows, D, 0, st>>>(a);
    return cudaGetLastError();
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
