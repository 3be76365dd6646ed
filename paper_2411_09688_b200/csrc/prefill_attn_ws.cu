// prefill_attn_ws.cu -- warp-specialised prefill sparse attention on tcgen05
// (section 4.2), d = 128, bf16.  FA4-style ping-pong:
//
//   CTA = two 128-row query tiles (Q0, Q1) of one (b,h) x one 4096-key split of
//   its key stream (selected fixed keys, then the visible user keys, R8).
//   warps 0-3  softmax group 0 (rows of Q0)    warps 4-7  softmax group 1 (Q1)
//   warp  8    MMA issuer (one lane)          warps 9-11 loaders (cp.async)
//   TMEM: S0 | S1 | O0 | O1 (4 x 128 columns); P_g (bf16) is written by the
//   softmax group into the first 64 columns of S_g and consumed from TMEM by the
//   PV MMA (A operand in tensor memory), so shared memory holds only Q0, Q1 and
//   a 2-stage K/V ring (192 KB).
//   Order on the tensor core per key tile t: PV0(t), S0(t+1), PV1(t), S1(t+1):
//   while group 0 runs the softmax of tile t+1, the tensor core computes
//   group 1's PV(t) and S(t+1), and vice versa.
//   Loaders gather the K/V rows by key position with 16-byte cp.async into the
//   128B-swizzled operand layout; cp.async.mbarrier.arrive signals a stage.
// Softmax: thread = query row, logits in registers, lazy O rescale (only when
// the row max grows by > 2^8, FA4), ex2.approx, masks only on ragged / causal
// diagonal tiles.  Each split writes (O/l, lse) partials; the CTA that
// completes a pair's last split merges them.
#include "common.cuh"
#include "internal.h"
#include "tcgen05.cuh"

namespace sqz {

namespace ws {
constexpr int D = 128;
constexpr int MMAW = 8;               // MMA warp index
constexpr int LD0 = 9, NLDW = 3;      // loader warps
constexpr int NLD = NLDW * 32;        // loader threads
constexpr int NT = 32 * (LD0 + NLDW); // 384
constexpr int QT = 128;               // rows per query tile
constexpr int KT = 128;               // keys per key tile
constexpr int NST = 2;                // K/V stages
constexpr int SPLIT = 4096;           // keys per CTA
constexpr int HB = 128 * 128;         // bytes of one 64-element half of a 128-row tile
constexpr int TILE = 2 * HB;          // 128 rows x 128 bf16
constexpr int OFF_Q = 0;              // Q0, Q1
constexpr int OFF_KV = 2 * TILE;      // stage s: K at OFF_KV + s*2*TILE, V right after
constexpr int OFF_POS = OFF_KV + NST * 2 * TILE;  // int [NST][128]
constexpr int OFF_BAR = OFF_POS + NST * KT * 4;    // mbarriers
constexpr int NBAR = 2 * NST + 2 + 2 + 2 + 1;
constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
constexpr int BYTES = OFF_TMEM + 16 + 1024;
}  // namespace ws

__device__ __forceinline__ void tmem_st32f(uint32_t taddr, const float *v) {
    uint32_t u[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(v[i]);
    tmem_st32u(taddr, u);
}

__global__ void __launch_bounds__(ws::NT, 1) k_prefill_attend_ws(AttnArgs a, int npairs) {
    using namespace ws;
    constexpr uint32_t IDESC_S = idesc_bf16(128, KT, false);
    constexpr uint32_t IDESC_O = idesc_bf16(128, D, true);
    extern __shared__ unsigned char smem_raw[];
    unsigned char *sm = reinterpret_cast<unsigned char *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const uint32_t sbase = smem_u32(sm);
    int *s_pos = reinterpret_cast<int *>(sm + OFF_POS);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + OFF_BAR);
    uint64_t *kv_full = bar, *kv_empty = bar + NST, *s_full = bar + 2 * NST,
             *p_full = bar + 2 * NST + 2, *o_done = bar + 2 * NST + 4, *q_full = bar + 2 * NST + 6;
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(sm + OFF_TMEM);
    __shared__ int s_flag;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int pair = blockIdx.x, split = blockIdx.y, bh = blockIdx.z;
    const int h = bh % a.H;
    const int t0 = pair * 2 * QT;

    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int nkf = ldcg(a.n_keys + bh);
    int nuv = a.causal ? (t0 + 2 * QT - 1) + a.n_u - a.n_q + 1 : a.n_u;
    nuv = max(0, min(nuv, a.n_u));
    const int len = nkf + nuv;
    const int nsplit = (len + SPLIT - 1) / SPLIT;
    const size_t row0 = (size_t)bh * a.n_q + t0;
    if (nsplit == 0) {  // no key at all: identity outputs (an error when final)
        if (split == 0 && tid < 2 * QT && t0 + tid < a.n_q) {
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
    const int k_begin = split * SPLIT, k_end = min(len, k_begin + SPLIT);
    const int ntile = (k_end - k_begin + KT - 1) / KT;

    if (warp == 0) tmem_alloc(s_tmem, 512);
    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&kv_full[s], NLD);
            mbar_init(&kv_empty[s], 1);
        }
        for (int g = 0; g < 2; ++g) {
            mbar_init(&s_full[g], 1);
            mbar_init(&p_full[g], 128);
            mbar_init(&o_done[g], 1);
        }
        mbar_init(q_full, NLD);
        mbar_fence_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;

    if (warp >= LD0) {
        // ======================= loaders =======================
        const int li = tid - LD0 * 32;
        const __nv_bfloat16 *Qb = reinterpret_cast<const __nv_bfloat16 *>(a.Q) + row0 * D;
        for (int e = li; e < 2 * QT * 16; e += NLD) {
            const int r = e >> 4, c = e & 15, g = r >> 7, rr = r & 127;
            const bool valid = t0 + r < a.n_q;
            cp_async16_zfill(sbase + OFF_Q + g * TILE + (c >> 3) * HB + sw128_off(rr, c & 7),
                             Qb + (size_t)(valid ? r : 0) * D + c * 8, valid);
        }
        cp_async_mbar_arrive(q_full);
        const __nv_bfloat16 *Kf = reinterpret_cast<const __nv_bfloat16 *>(a.Kp) + (size_t)h * a.L * D;
        const __nv_bfloat16 *Vf = reinterpret_cast<const __nv_bfloat16 *>(a.Vp) + (size_t)h * a.L * D;
        const __nv_bfloat16 *Ku = reinterpret_cast<const __nv_bfloat16 *>(a.Ku) + (size_t)bh * a.n_u * D;
        const __nv_bfloat16 *Vu = reinterpret_cast<const __nv_bfloat16 *>(a.Vu) + (size_t)bh * a.n_u * D;
        const int32_t *kidx = a.key_idx + (size_t)bh * a.L;
        auto pos_of = [&](int k) -> int {
            if (k >= k_end) return 0;
            return k < nkf ? ldcg(kidx + k) : -1 - (k - nkf);
        };
        for (int t = 0; t < ntile; ++t) {
            const int st = t % NST, k0 = k_begin + t * KT;
            const int p0 = pos_of(k0 + li);
            const int p1 = li + NLD < KT ? pos_of(k0 + li + NLD) : 0;
            if (t >= NST) mbar_wait(&kv_empty[st], ((t / NST) - 1) & 1);
            s_pos[st * KT + li] = p0;
            if (li + NLD < KT) s_pos[st * KT + li + NLD] = p1;
            named_bar(2, NLD);
            const uint32_t kb = sbase + OFF_KV + st * 2 * TILE, vb = kb + TILE;
            for (int e = li; e < KT * 16; e += NLD) {
                const int key = e >> 4, c = e & 15;
                const bool valid = k0 + key < k_end;
                const int pos = s_pos[st * KT + key];
                const __nv_bfloat16 *ks = pos >= 0 ? Kf + (size_t)pos * D : Ku + (size_t)(-1 - pos) * D;
                const __nv_bfloat16 *vs = pos >= 0 ? Vf + (size_t)pos * D : Vu + (size_t)(-1 - pos) * D;
                const uint32_t off = (c >> 3) * HB + sw128_off(key, c & 7);
                cp_async16_zfill(kb + off, valid ? ks + c * 8 : Kf, valid);
                cp_async16_zfill(vb + off, valid ? vs + c * 8 : Vf, valid);
            }
            cp_async_mbar_arrive(&kv_full[st]);
            // s_pos[st] may be rewritten only after every loader has issued from it
            named_bar(2, NLD);
        }
    } else if (warp == MMAW) {
        // ======================= MMA issuer =======================
        if (lane == 0) {
            auto wait_kv = [&](int t) {
                mbar_wait(&kv_full[t % NST], (t / NST) & 1);
                fence_async_smem();
                tc_fence_after();
            };
            auto issue_S = [&](int g, int t) {
                const uint32_t qb = sbase + OFF_Q + g * TILE;
                const uint32_t kb = sbase + OFF_KV + (t % NST) * 2 * TILE;
#pragma unroll
                for (int ks = 0; ks < D / 16; ++ks) {
                    const uint32_t off = (ks >> 2) * HB + (ks & 3) * 32;
                    umma_bf16(tmem + g * 128, sdesc_sw128(qb + off, 16, 1024),
                              sdesc_sw128(kb + off, 16, 1024), IDESC_S, ks > 0);
                }
                umma_commit(&s_full[g]);
            };
            auto issue_PV = [&](int g, int t) {
                const uint32_t vb = sbase + OFF_KV + (t % NST) * 2 * TILE + TILE;
#pragma unroll
                for (int ks = 0; ks < KT / 16; ++ks)
                    umma_bf16_ts(tmem + 256 + g * 128, tmem + g * 128 + ks * 8,
                                 sdesc_sw128(vb + ks * 2048, HB, 1024), IDESC_O, (t > 0 || ks > 0));
                umma_commit(&o_done[g]);
            };
            mbar_wait(q_full, 0);
            wait_kv(0);
            issue_S(0, 0);
            issue_S(1, 0);
            for (int t = 0; t < ntile; ++t) {
                mbar_wait(&p_full[0], t & 1);
                tc_fence_after();
                issue_PV(0, t);
                if (t + 1 < ntile) {
                    wait_kv(t + 1);
                    issue_S(0, t + 1);
                }
                mbar_wait(&p_full[1], t & 1);
                tc_fence_after();
                issue_PV(1, t);
                umma_commit(&kv_empty[t % NST]);  // stage t free once its MMAs complete
                if (t + 1 < ntile) issue_S(1, t + 1);
            }
        }
        __syncwarp();
    } else {
        // ======================= softmax groups =======================
        const int g = warp >> 2, r = tid & 127;  // TMEM lane = r
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tS = tmem + g * 128 + lane_off, tO = tmem + 256 + g * 128 + lane_off;
        const int trow = t0 + g * QT + r;
        const bool row_ok = trow < a.n_q;
        const int ulim = trow + a.n_u - a.n_q;
        const float sl2 = a.scale * LOG2E;
        float m_used = -INFINITY, l = 0.f;
        for (int t = 0; t < ntile; ++t) {
            const int k0 = k_begin + t * KT;
            mbar_wait(&s_full[g], t & 1);
            tc_fence_after();
            float sv[KT];
#pragma unroll
            for (int c = 0; c < KT / 32; ++c)
                tmem_ld32(tS + c * 32, *reinterpret_cast<float(*)[32]>(sv + c * 32));
            tmem_wait_ld();
            const bool full = row_ok && k0 + KT <= k_end && (k0 + KT <= nkf || k0 + KT - 1 - nkf <= ulim);
            if (!full) {
#pragma unroll
                for (int j = 0; j < KT; ++j) {
                    const int k = k0 + j;
                    const bool vis = row_ok && k < k_end && (k < nkf || k - nkf <= ulim);
                    if (!vis) sv[j] = -INFINITY;
                }
            }
            float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int j = 0; j < KT; j += 4) {
                mx4[0] = fmaxf(mx4[0], sv[j]);
                mx4[1] = fmaxf(mx4[1], sv[j + 1]);
                mx4[2] = fmaxf(mx4[2], sv[j + 2]);
                mx4[3] = fmaxf(mx4[3], sv[j + 3]);
            }
            const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * sl2;
            const bool need = mx > m_used + 8.f;
            const float alpha = need ? ((m_used == -INFINITY) ? 0.f : exp2f(m_used - mx)) : 1.f;
            if (t > 0 && __any_sync(FULL, need)) {
                // O_g must be stable: PV_g(t-1) has completed
                mbar_wait(&o_done[g], (t - 1) & 1);
                tc_fence_after();
#pragma unroll 1
                for (int c = 0; c < D / 32; ++c) {
                    float v[32];
                    tmem_ld32(tO + c * 32, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] *= alpha;
                    tmem_st32(tO + c * 32, v);
                }
                tmem_wait_st();
            }
            l *= alpha;
            if (need) m_used = mx;
            const float moff = (m_used == -INFINITY) ? 0.f : m_used;
            float ls[4] = {0.f, 0.f, 0.f, 0.f};
            // p packed in place: bf16x2 of keys (2j, 2j+1) into sv[j] (slot j <= 2j is consumed)
#pragma unroll
            for (int j = 0; j < KT / 2; ++j) {
                const float p0 = fast_exp2(fmaf(sv[2 * j], sl2, -moff));
                const float p1 = fast_exp2(fmaf(sv[2 * j + 1], sl2, -moff));
                ls[j & 3] += p0 + p1;
                const __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
                sv[j] = __uint_as_float(*reinterpret_cast<const uint32_t *>(&b2));
            }
            l += (ls[0] + ls[1]) + (ls[2] + ls[3]);
            tmem_st32f(tS, sv);        // P columns 0..31
            tmem_st32f(tS + 32, sv + 32);  // P columns 32..63
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&p_full[g]);
        }
        // ---- this split's partial for the row ----
        mbar_wait(&o_done[g], (ntile - 1) & 1);
        tc_fence_after();
        const size_t slot = ((size_t)row0 + g * QT + r) * a.max_chunks + split;
        const bool have = row_ok && l > 0.f;
        const float inv_l = have ? 1.0f / l : 0.f;
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
            float v[32];
            tmem_ld32(tO + c * 32, v);
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
    }
    __threadfence();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
    // ---- the CTA completing the pair's last split merges ----
    if (tid == 0) {
        int *cnt = a.row_cnt + (size_t)bh * npairs + pair;
        const int t = atomicAdd(cnt, 1);
        s_flag = (t == nsplit - 1);
        if (s_flag) *cnt = 0;
    }
    __syncthreads();
    if (!s_flag) return;
    __threadfence();
    for (int r = warp; r < 2 * QT; r += NT / 32) {
        if (t0 + r >= a.n_q) break;
        const size_t row = row0 + r;
        float M = -INFINITY;
        for (int p = 0; p < nsplit; ++p) M = fmaxf(M, ldcg(a.part_lse + row * a.max_chunks + p));
        float L = 0.f, acc[D / 32];
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

cudaError_t launch_prefill_attention_ws(const AttnArgs &a, cudaStream_t st) {
    const int npairs = (a.n_q + 2 * ws::QT - 1) / (2 * ws::QT);
    const int nsplit_max = (int)((a.L + a.n_u + ws::SPLIT - 1) / ws::SPLIT);
    static bool set = false;
    if (!set) {
        cudaError_t e = cudaFuncSetAttribute(k_prefill_attend_ws,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, ws::BYTES);
        if (e != cudaSuccess) return e;
        set = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(npairs, nsplit_max, a.B * a.H);
    cfg.blockDim = dim3(ws::NT);
    cfg.dynamicSmemBytes = ws::BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_prefill_attend_ws, a, npairs);
}

}  // namespace sqz
