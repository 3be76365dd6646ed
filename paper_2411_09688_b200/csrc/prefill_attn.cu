// prefill_attn.cu -- prefill sparse attention on the 5th-generation tensor cores
// (section 4.2; prefill = many query rows).
//
// This split-KV kernel serves d = 64 bf16 prefill; d = 128 runs on the persistent
// warp-specialised kernel of prefill_attn_ws.cu.
// CTA = one 128-row query tile of one (b,h) and one split of its key stream
// (selected fixed keys, then the user keys visible to the tile, R8).  Per
// 128-key tile:
//   * the K and V rows are gathered by key position with 16-byte cp.async
//     straight into the 128B-swizzled shared-memory layout tcgen05 reads
//     (double-buffered: tile t+1 streams in while tile t is computed);
//   * S = Q K^T: 8 x tcgen05.mma (M=128, N=128, K=16, bf16 -> fp32) issued by
//     one thread, accumulator in TMEM (128 columns);
//   * softmax: thread = query row reads its S row from TMEM (tcgen05.ld
//     32x32b), applies the causal user mask, keeps a lazily rescaled running
//     max (O in TMEM is rescaled only when the max grows by more than 2^8,
//     as in FA4), writes P as bf16 into shared memory (swizzled K-major);
//   * O += P V: 8 x tcgen05.mma (M=128, N=d, K=16, V read as an MN-major
//     operand), O stays in TMEM across the whole split.
// The split's normalised partial (O/l, lse) goes to the workspace; the CTA
// that completes the tile's last split merges them.
#include "common.cuh"
#include "internal.h"
#include "tcgen05.cuh"

namespace sqz {

#ifdef SQZ_TRACE
__device__ unsigned long long g_trace_pf[64 * 8];
#define PF_TRACE(it, slot)                                                                   \
    do {                                                                                      \
        if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 &&      \
            (it) < 64) {                                                                      \
            unsigned long long t_;                                                            \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
            g_trace_pf[(it) * 8 + (slot)] = t_;                                               \
        }                                                                                     \
    } while (0)
#else
#define PF_TRACE(it, slot) do { } while (0)
#endif

constexpr int PF_NT = 128;         // threads: 4 warps, thread = query row
constexpr int PF_QT = 128;         // query rows per CTA
constexpr int PF_KT = 128;         // keys per tile
constexpr int PF_SPLIT = 4096;     // keys per CTA (32 tiles)

int prefill_split_keys() { return PF_SPLIT; }

template <int D> struct PfSmem {
    static constexpr int TILE = PF_QT * D * 2;  // 128 rows x D bf16 (Q, K or V tile)
    static constexpr int Q = 0;
    static constexpr int K0 = Q + TILE;         // 2 buffers
    static constexpr int V0 = K0 + 2 * TILE;    // 2 buffers
    static constexpr int P = V0 + 2 * TILE;     // 128 rows x 128 keys bf16
    static constexpr int PB = PF_QT * PF_KT * 2;
    static constexpr int MISC = P + PB;          // 2 mbarriers + tmem base
    static constexpr int POS = MISC + 64;        // int[128]
    static constexpr int BYTES = POS + PF_KT * 4 + 1024;  // + alignment slack
};

template <int D>
__global__ void __launch_bounds__(PF_NT, 1) k_prefill_attend(AttnArgs a, int qtiles) {
    using S = PfSmem<D>;
    constexpr int CPR = D * 2 / 16;  // 16-byte chunks per row
    constexpr int HB = PF_QT * 128;  // bytes per 64-element half of a tile
    constexpr uint32_t IDESC_S = idesc_bf16(128, PF_KT, false);
    constexpr uint32_t IDESC_O = idesc_bf16(128, D, true);

    extern __shared__ unsigned char smem_raw[];
    unsigned char *sm = reinterpret_cast<unsigned char *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const uint32_t sbase = smem_u32(sm);
    uint64_t *mbar = reinterpret_cast<uint64_t *>(sm + S::MISC);
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(sm + S::MISC + 16);
    int *s_pos = reinterpret_cast<int *>(sm + S::POS);
    __shared__ int s_flag;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int qt = blockIdx.x, split = blockIdx.y, bh = blockIdx.z;
    const int h = bh % a.H;
    const int t0 = qt * PF_QT;

    asm volatile("griddepcontrol.wait;" ::: "memory");
    // stream of this (b,h) for this query tile: fixed keys, then the user keys
    // visible to at least one of its rows
    const int nkf = ldcg(a.n_keys + bh);
    int nuv = a.causal ? (t0 + PF_QT - 1) + a.n_u - a.n_q + 1 : a.n_u;
    nuv = max(0, min(nuv, a.n_u));
    const int len = nkf + nuv;
    const int nsplit = (len + PF_SPLIT - 1) / PF_SPLIT;
    const size_t row0 = (size_t)bh * a.n_q + t0;  // first output row of the tile
    if (nsplit == 0) {
        // no key at all for this tile: identity outputs (an error when final)
        if (split == 0 && t0 + tid < a.n_q) {
            for (int k = 0; k < D; ++k) {
                if (a.out_dtype == SQZ_BF16)
                    reinterpret_cast<__nv_bfloat16 *>(a.O)[(row0 + tid) * D + k] = __float2bfloat16_rn(0.f);
                else
                    reinterpret_cast<float *>(a.O)[(row0 + tid) * D + k] = 0.f;
            }
            a.LSE[row0 + tid] = -INFINITY;
            if (!a.partial) atomicOr(a.status, 1);
        }
        return;
    }
    if (split >= nsplit) return;

    if (warp == 0) tmem_alloc(s_tmem, 256);
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        mbar_fence_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;
    const uint32_t tS = tmem, tO = tmem + 128;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;

    const __nv_bfloat16 *Qb = reinterpret_cast<const __nv_bfloat16 *>(a.Q) + row0 * D;
    const __nv_bfloat16 *Kf = reinterpret_cast<const __nv_bfloat16 *>(a.Kp) + (size_t)h * a.L * D;
    const __nv_bfloat16 *Vf = reinterpret_cast<const __nv_bfloat16 *>(a.Vp) + (size_t)h * a.L * D;
    const __nv_bfloat16 *Ku = reinterpret_cast<const __nv_bfloat16 *>(a.Ku) + (size_t)bh * a.n_u * D;
    const __nv_bfloat16 *Vu = reinterpret_cast<const __nv_bfloat16 *>(a.Vu) + (size_t)bh * a.n_u * D;
    const int32_t *kidx = a.key_idx ? a.key_idx + (size_t)bh * a.L : nullptr;
    RunList rl;  // run-length selection when key_idx is not materialised
    if (!kidx) {
        rl.cl = a.sel_cl + (size_t)bh * a.c2;
        rl.pref = a.sel_pref + (size_t)bh * a.c2;
        rl.koff = a.key_off + (size_t)h * (a.c2 + 1);
        rl.n = ldcg(a.sel_n + bh);
        rl.nkf = nkf;
    }
    const int k_begin = split * PF_SPLIT, k_end = min(len, k_begin + PF_SPLIT);
    const int ntile = (k_end - k_begin + PF_KT - 1) / PF_KT;
    auto pos_of = [&](int k) -> int {
        if (k >= nkf) return -1 - (k - nkf);
        if (kidx) return ldcg(kidx + k);
        const int j = run_of(rl, k);  // (d = 64 path: a plain search per key)
        return __ldg(rl.koff + ldcg(rl.cl + j)) + (k - ldcg(rl.pref + j));
    };

    // Q tile (rows beyond n_q zero-filled)
    for (int e = tid; e < PF_QT * CPR; e += PF_NT) {
        const int r = e / CPR, c = e % CPR;
        const bool valid = t0 + r < a.n_q;
        const uint32_t dst = sbase + S::Q + (c >> 3) * HB + sw128_off(r, c & 7);
        cp_async16_zfill(dst, Qb + (size_t)(valid ? r : 0) * D + c * 8, valid);
    }
    auto issue_tile = [&](int k0, int buf) {
        for (int e = tid; e < PF_KT * CPR; e += PF_NT) {
            const int key = e / CPR, c = e % CPR;
            const bool valid = k0 + key < k_end;
            const int pos = s_pos[key];
            const __nv_bfloat16 *ks = pos >= 0 ? Kf + (size_t)pos * D : Ku + (size_t)(-1 - pos) * D;
            const __nv_bfloat16 *vs = pos >= 0 ? Vf + (size_t)pos * D : Vu + (size_t)(-1 - pos) * D;
            const uint32_t off = (c >> 3) * HB + sw128_off(key, c & 7);
            cp_async16_zfill(sbase + S::K0 + buf * S::TILE + off, valid ? ks + c * 8 : Kf, valid);
            cp_async16_zfill(sbase + S::V0 + buf * S::TILE + off, valid ? vs + c * 8 : Vf, valid);
        }
    };
    s_pos[tid] = k_begin + tid < k_end ? pos_of(k_begin + tid) : 0;
    __syncthreads();
    issue_tile(k_begin, 0);
    cp_async_commit_grp();

    const float sl2 = a.scale * LOG2E;
    const int trow = t0 + tid;                   // query index of this thread's row
    const bool row_ok = trow < a.n_q;
    const int ulim = a.causal ? trow + a.n_u - a.n_q : a.n_u;  // user key u visible iff u <= ulim
    float m_used = -INFINITY, l = 0.f;

    for (int it = 0; it < ntile; ++it) {
        const int buf = it & 1;
        const int k0 = k_begin + it * PF_KT;
        const int k0n = k0 + PF_KT;
        PF_TRACE(it, 0);
        const int pos_next = (it + 1 < ntile && k0n + tid < k_end) ? pos_of(k0n + tid) : 0;
        cp_async_wait_all();  // tile `it` (and Q) are in shared memory
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        PF_TRACE(it, 1);
        if (tid == 0) {  // S = Q K^T
            tc_fence_after();
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks) {
                const uint32_t off = (ks >> 2) * HB + (ks & 3) * 32;
                umma_bf16(tS, sdesc_sw128(sbase + S::Q + off, 16, 1024),
                          sdesc_sw128(sbase + S::K0 + buf * S::TILE + off, 16, 1024), IDESC_S,
                          ks > 0);
            }
            umma_commit(&mbar[0]);
        }
        // the other buffer and P are free once O(it-1) = P V(it-1) has completed
        if (it > 0) mbar_wait(&mbar[1], (it - 1) & 1);
        if (it + 1 < ntile) s_pos[tid] = pos_next;
        __syncthreads();
        if (it + 1 < ntile) issue_tile(k0n, buf ^ 1);
        cp_async_commit_grp();

        // ---- softmax on this thread's row ----
        mbar_wait(&mbar[0], it & 1);
        PF_TRACE(it, 2);
        tc_fence_after();
        // the row's 128 logits stay in registers for both passes
        float sv[PF_KT];
#pragma unroll
        for (int c = 0; c < PF_KT / 32; ++c)
            tmem_ld32(tS + lane_off + c * 32, *reinterpret_cast<float(*)[32]>(sv + c * 32));
        tmem_wait_ld();
        // masks only where needed: ragged rows, the stream tail, the causal diagonal
        const bool full = row_ok && k0 + PF_KT <= k_end &&
                          (k0 + PF_KT <= nkf || k0 + PF_KT - 1 - nkf <= ulim);
        if (!full) {
#pragma unroll
            for (int j = 0; j < PF_KT; ++j) {
                const int k = k0 + j;
                const bool vis = row_ok && k < k_end && (k < nkf || k - nkf <= ulim);
                if (!vis) sv[j] = -INFINITY;
            }
        }
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int j = 0; j < PF_KT; j += 4) {
            mx4[0] = fmaxf(mx4[0], sv[j]);
            mx4[1] = fmaxf(mx4[1], sv[j + 1]);
            mx4[2] = fmaxf(mx4[2], sv[j + 2]);
            mx4[3] = fmaxf(mx4[3], sv[j + 3]);
        }
        const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * sl2;
        float v[32];
        // lazy rescale: only when a row's max grew by more than 2^8 (FA4); the
        // TMEM accesses are warp-collective, so the warp rescales together
        const bool need = mx > m_used + 8.f;
        const float alpha = need ? ((m_used == -INFINITY) ? 0.f : exp2f(m_used - mx)) : 1.f;
        if (it > 0 && __any_sync(FULL, need)) {
#pragma unroll 1
            for (int c = 0; c < D / 32; ++c) {
                tmem_ld32(tO + lane_off + c * 32, v);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] *= alpha;
                tmem_st32(tO + lane_off + c * 32, v);
            }
            tmem_wait_st();
        }
        l *= alpha;
        if (need) m_used = mx;
        // p = 2^(s*scale*log2e - m) (ex2.approx), bf16, into the swizzled P tile
        const float moff = (m_used == -INFINITY) ? 0.f : m_used;  // masked row: all p = 0
        float ls[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int ch = 0; ch < PF_KT / 8; ++ch) {  // 16 chunks of 8 keys
            uint32_t pk[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float p0 = fast_exp2(fmaf(sv[ch * 8 + 2 * q], sl2, -moff));
                const float p1 = fast_exp2(fmaf(sv[ch * 8 + 2 * q + 1], sl2, -moff));
                ls[q] += p0 + p1;
                const __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
                pk[q] = *reinterpret_cast<const uint32_t *>(&b2);
            }
            const uint32_t addr = sbase + S::P + (ch >> 3) * HB + sw128_off(tid, ch & 7);
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(pk[0]), "r"(pk[1]),
                         "r"(pk[2]), "r"(pk[3])
                         : "memory");
        }
        l += (ls[0] + ls[1]) + (ls[2] + ls[3]);
        PF_TRACE(it, 3);
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {  // O += P V
            tc_fence_after();
#pragma unroll
            for (int ks = 0; ks < PF_KT / 16; ++ks) {
                umma_bf16(tO, sdesc_sw128(sbase + S::P + (ks >> 2) * HB + (ks & 3) * 32, 16, 1024),
                          sdesc_sw128(sbase + S::V0 + buf * S::TILE + ks * 2048, HB, 1024), IDESC_O,
                          (it > 0 || ks > 0) ? 1u : 0u);
            }
            umma_commit(&mbar[1]);
            PF_TRACE(it, 4);
        }
    }
    // ---- split partial: O / l and lse for every row of the tile ----
    mbar_wait(&mbar[1], (ntile - 1) & 1);
    tc_fence_after();
    const size_t slot = (row0 + tid) * a.max_chunks + split;
    const bool have = row_ok && l > 0.f;
    const float inv_l = have ? 1.0f / l : 0.f;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
        float v[32];
        tmem_ld32(tO + lane_off + c * 32, v);
        tmem_wait_ld();
        if (row_ok) {
            float4 *dst = reinterpret_cast<float4 *>(a.part_o + slot * D + c * 32);
#pragma unroll
            for (int j = 0; j < 32; j += 4)
                dst[j / 4] = make_float4(v[j] * inv_l, v[j + 1] * inv_l, v[j + 2] * inv_l, v[j + 3] * inv_l);
        }
    }
    if (row_ok) a.part_lse[slot] = have ? (m_used + log2f(l)) * LN2 : -INFINITY;
    tc_fence_before();
    __threadfence();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 256);
    // ---- the CTA completing the tile's last split merges ----
    if (tid == 0) {
        int *cnt = a.row_cnt + (size_t)bh * qtiles + qt;
        const int t = atomicAdd(cnt, 1);
        s_flag = (t == nsplit - 1);
        if (s_flag) *cnt = 0;
    }
    __syncthreads();
    if (!s_flag) return;
    __threadfence();
    for (int r = warp; r < PF_QT; r += PF_NT / 32) {
        if (t0 + r >= a.n_q) break;
        const size_t row = row0 + r;
        float M = -INFINITY;
        for (int p = 0; p < nsplit; ++p) M = fmaxf(M, ldcg(a.part_lse + row * a.max_chunks + p));
        float L = 0.f;
        float acc[D / 32];
#pragma unroll
        for (int k = 0; k < D / 32; ++k) acc[k] = 0.f;
        if (M != -INFINITY) {
            for (int p = 0; p < nsplit; ++p) {
                const float w = expf(ldcg(a.part_lse + row * a.max_chunks + p) - M);
                L += w;
                const float *op = a.part_o + (row * a.max_chunks + p) * D;
#pragma unroll
                for (int k = 0; k < D / 32; ++k) acc[k] = fmaf(w, ldcg(op + lane + 32 * k), acc[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < D / 32; ++k) {
            const float o = M == -INFINITY ? 0.f : acc[k] / L;
            if (a.out_dtype == SQZ_BF16)
                reinterpret_cast<__nv_bfloat16 *>(a.O)[row * D + lane + 32 * k] = __float2bfloat16_rn(o);
            else
                reinterpret_cast<float *>(a.O)[row * D + lane + 32 * k] = o;
        }
        if (lane == 0) {
            a.LSE[row] = M == -INFINITY ? -INFINITY : M + logf(L);
            if (M == -INFINITY && !a.partial) atomicOr(a.status, 1);
        }
    }
}

cudaError_t launch_prefill_attention(const AttnArgs &a, cudaStream_t st) {
    const int qtiles = (a.n_q + PF_QT - 1) / PF_QT;
    const int nsplit_max = (int)((a.L + a.n_u + PF_SPLIT - 1) / PF_SPLIT);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(qtiles, nsplit_max, a.B * a.H);
    cfg.blockDim = dim3(PF_NT);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (prefill_ws_applies(a.d, a.dtype, a.n_q)) return launch_prefill_attention_ws(a, st);
    if (a.d != 64) return cudaErrorInvalidValue;  // d = 128 bf16 prefill is the persistent kernel
    {
        cudaError_t e = ensure_func_attr((const void *)k_prefill_attend<64>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, PfSmem<64>::BYTES);
        if (e != cudaSuccess) return e;
    }
    cfg.dynamicSmemBytes = PfSmem<64>::BYTES;
    return cudaLaunchKernelEx(&cfg, k_prefill_attend<64>, a, qtiles);
}

}  // namespace sqz

#ifdef SQZ_TRACE
extern "C" int sqz_trace_pf(void *host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, sqz::g_trace_pf, bytes < sizeof(sqz::g_trace_pf) ? bytes : sizeof(sqz::g_trace_pf));
}
#endif
