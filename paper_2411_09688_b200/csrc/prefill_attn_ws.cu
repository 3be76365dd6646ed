// prefill_attn_ws.cu -- warp-specialised, persistent prefill sparse attention on
// tcgen05 (section 4.2), d = 128, bf16.
//
// Work decomposition.  A "segment" is one (b,h) x one pair of 128-row query
// tiles (256 rows) with its key stream: the selected fixed keys of (b,h), then
// the user keys visible to the pair's last row (R8).  The segments' 128-key
// tiles are laid end to end (segment s = pair * B*H + bh, see seg_ids) and the grid --
// one CTA per SM -- cuts that list into equal contiguous ranges, so every CTA
// does the same number of tiles whatever the per-head selection sizes are (the
// decode kernel's equal-key-range idea).  A CTA walks the
// "pieces" (segment x its range) in order; a segment cut by a CTA boundary
// writes (O/l, lse) partials per piece, and the CTA that completes its last
// piece merges them at its end.  Unsplit segments are written
// directly.
//
// Inside a CTA (FA4-style):
//   warps 0-3  softmax group 0 (query tile 0)   warps 4-7  softmax group 1 (tile 1)
//   warp  8    MMA issuer (one lane)            warps 12-13 K loaders, 14-15 V loaders
//   (setmaxnreg moves registers from warpgroups 2-3 to the softmax groups)
//   TMEM: S0 | S1 | O0 | O1 (4 x 128 columns); P_g (bf16) is written by the
//   softmax group into the first 64 columns of S_g and consumed from TMEM by the
//   PV MMA (A operand in tensor memory), so shared memory holds Q0, Q1, a
//   3-stage K ring and a 2-stage V ring (224 KB).  K(t) is released as soon as
//   S1(t) completes, V(t) after PV1(t), Q after the piece's last S.
//   Tensor-core order per key tile t: PV0(t), S0(t+1), PV1(t), S1(t+1).
//   Loaders gather the K/V rows by key position with 16-byte cp.async into the
//   128B-swizzled operand layout; cp.async.mbarrier.arrive signals a stage.
// Softmax: thread = query row, logits in registers, lazy O rescale (only when
// the row max grows by > 2^8, FA4), FFMA2/FADD2 packed arithmetic, ex2.approx,
// masks only on ragged / causal-diagonal tiles.
#include <cuda.h>

#include "common.cuh"
#include "internal.h"
#include "tcgen05.cuh"

namespace sqz {

namespace ws {
constexpr int D = 128;
constexpr int MMAW = 8;               // MMA warp index
constexpr int NWK = 4, NWV = 3;       // K loader warps 9, 10, 12, 13; V loader warps 11, 14, 15
constexpr int NT = 512;               // 16 warps = 4 warpgroups
constexpr int QT = 128;               // rows per query tile
constexpr int PR = 2 * QT;            // rows per segment (query-tile pair)
constexpr int KT = 64;                // keys per key tile
constexpr int NKS = 6, NVS = 4;       // K / V ring stages
constexpr int HBQ = 128 * 128;        // bytes of one 64-element half of a 128-row Q tile
constexpr int QTILE = 2 * HBQ;        // 128 rows x 128 bf16 = 32 KB
constexpr int HBK = KT * 128;         // half of a K/V tile (64 rows x 128 B)
constexpr int KTILE = 2 * HBK;        // 64 keys x 128 bf16 = 16 KB
constexpr int OFF_Q = 0;              // Q0, Q1
constexpr int OFF_K = 2 * QTILE;
constexpr int OFF_V = OFF_K + NKS * KTILE;
constexpr int OFF_BAR = OFF_V + NVS * KTILE;
constexpr int NBAR = 2 * NKS + 2 * NVS + 4 + 4 + 2 + 2 + 2;
constexpr int OFF_MISC = OFF_BAR + NBAR * 8;  // tmem addr, first segment, merges
constexpr int BYTES = OFF_MISC + 64 + 1024;   // + alignment slack
static_assert(BYTES <= 232448, "shared memory budget");
constexpr int INVALID = (int)0x80000000;      // key position of a masked (past-the-end) slot
}  // namespace ws

#ifdef SQZ_TRACE
#ifndef SQZ_TRACE_CTA
#define SQZ_TRACE_CTA 0
#endif
__device__ unsigned long long g_trace_ws[128 * 24];
__device__ unsigned long long g_cta_ws[1024 * 4];  // per CTA: entry, loop end, exit (globaltimer)
#define WS_CTA_T(slot)                                                                        \
    do {                                                                                      \
        if (threadIdx.x == 0 && blockIdx.x < 1024) {                                          \
            unsigned long long t_;                                                            \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
            g_cta_ws[blockIdx.x * 4 + (slot)] = t_;                                           \
        }                                                                                     \
    } while (0)
#define WS_TRACE(cond, it, slot)                                                              \
    do {                                                                                      \
        if ((cond) && blockIdx.x == SQZ_TRACE_CTA && (it) < 128) {                                       \
            unsigned long long t_;                                                            \
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_));                                \
            g_trace_ws[(it) * 24 + (slot)] = t_;                                              \
        }                                                                                     \
    } while (0)
#else
#define WS_TRACE(cond, it, slot) do { } while (0)
#define WS_CTA_T(slot) do { } while (0)
#endif

// ---- packed fp32x2 arithmetic (FFMA2 / FADD2, sm_100) and the FMA-pipe exp2 ----
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(d)
        : "l"(*reinterpret_cast<const uint64_t *>(&a)), "l"(*reinterpret_cast<const uint64_t *>(&b)),
          "l"(*reinterpret_cast<const uint64_t *>(&c)));
    return *reinterpret_cast<float2 *>(&d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;"
        : "=l"(d)
        : "l"(*reinterpret_cast<const uint64_t *>(&a)), "l"(*reinterpret_cast<const uint64_t *>(&b)));
    return *reinterpret_cast<float2 *>(&d);
}
// 2^x for a pair without the MUFU: x = j + f (j = rint(x) by the 1.5*2^23 trick,
// f in [-1/2, 1/2]), 2^f by a degree-3 polynomial (max relative error 7.5e-5,
// far below the bf16 rounding of P), 2^j added into the exponent field.
// x is clamped at -125 so 2^j stays a normal number (smaller p are irrelevant
// next to the row maximum's p >= 2^-8).
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
    constexpr float MAGIC = 12582912.0f;  // 1.5 * 2^23
    x.x = fmaxf(x.x, -125.f);
    x.y = fmaxf(x.y, -125.f);
    const float2 t = fadd2(x, make_float2(MAGIC, MAGIC));
    const float2 jf = fadd2(t, make_float2(-MAGIC, -MAGIC));
    const float2 f = ffma2(jf, make_float2(-1.f, -1.f), x);
    float2 p = ffma2(f, make_float2(0.05517121f, 0.05517121f), make_float2(0.24261023f, 0.24261023f));
    p = ffma2(p, f, make_float2(0.69326103f, 0.69326103f));
    p = ffma2(p, f, make_float2(0.99992818f, 0.99992818f));
    return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                       __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}
// which key pairs of a 128-key tile take the polynomial (the rest use MUFU.EX2);
// measured on cfg3: every step towards the polynomial was slower, so 0.
#ifndef SQZ_PF_EMU_MASK
#define SQZ_PF_EMU_MASK 0x00u
#endif

// bits j of a 32-bit word (slots base + j) that fall in [lo, hi)
__device__ __forceinline__ uint32_t range_bits(int lo, int hi, int base) {
    const int l = min(max(lo - base, 0), 32), h = min(max(hi - base, 0), 32);
    const uint32_t below_h = h >= 32 ? 0xffffffffu : (1u << h) - 1u;
    const uint32_t below_l = l >= 32 ? 0xffffffffu : (1u << l) - 1u;
    return below_h & ~below_l;
}

__device__ __forceinline__ void tmem_st32f(uint32_t taddr, const float *v) {
    uint32_t u[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(v[i]);
    tmem_st32u(taddr, u);
}

// NW warps gather a 64-row K/V tile into the SW128 layout.  Warp w (0..NW-1)
// copies row pairs w + NW j (< KT/2), rows 2(w + NW j) + (lane/16), 16-byte
// chunk lane%16; the row's key position is held by lane 2j + (lane/16) of the
// same warp and broadcast by shuffle.
template <int NW>
__device__ __forceinline__ void gather_rows(uint32_t dst, const __nv_bfloat16 *fixed,
                                            const __nv_bfloat16 *user, int pos_mine, int w, int lane) {
    using namespace ws;
    const int hh = lane >> 4, c = lane & 15;
    const uint32_t coff = (uint32_t)((c >> 3) * HBK);
#pragma unroll
    for (int j = 0; j < (KT / 2 + NW - 1) / NW; ++j) {
        const int pos = __shfl_sync(FULL, pos_mine, 2 * j + hh);
        const int row = 2 * (w + NW * j) + hh;
        if (w + NW * j >= KT / 2) break;  // (NW not dividing 32: the last round is partial)
        const bool valid = pos != INVALID;
        const __nv_bfloat16 *src = pos >= 0 ? fixed + (size_t)pos * D : user + (size_t)(-1 - pos) * D;
        cp_async16_zfill(dst + coff + sw128_off(row, c & 7), valid ? src + c * 8 : fixed, valid);
    }
}

// TMA descriptor of Q (2-D [B*H*n_q, 128] bf16, box {64, 128}, 128B swizzle)
struct TmaMaps {
    CUtensorMap q;
};

// ---- the segment list ----
// key stream of a segment: selected fixed keys [0, nkf), padding [nkf, nkf4)
// (masked; nkf4 = nkf rounded up to 4 when user keys follow, so that every TMA
// gather4 group of 4 stream slots reads from one tensor), user keys
// [nkf4, nkf4 + nuv)
// Partition cost of a segment: its tiles plus SEG_W tiles' worth for the
// per-piece setup/drain (Q load, pipeline fill, epilogue; fitted ~6 tiles on cfg3;
// 3 and 8 were slower),
// so CTAs holding many short segments are not the stragglers.
constexpr int SEG_W = 6;
struct Seg {
    int bh, pair, nkf, nkf4, len, tiles, cost;
};
// Segment order: PAIR-major (s = pair * B*H + bh) by default.  The equal-cost
// ranges then put the npairs query pairs of one head on CTAs G/npairs apart that
// start at (nearly) the same key of that head's stream and advance at the same
// rate, so the head's selected K/V tiles are read from DRAM once and served from
// L2 to the other pairs; with head-major order (s = bh * npairs + pair) the
// pairs of a head run on neighbouring CTAs at different offsets of the stream
// and every pair re-reads it from DRAM once it exceeds the L2 window.
#ifndef SQZ_PF_PAIR_MAJOR
#define SQZ_PF_PAIR_MAJOR 1
#endif
__device__ __forceinline__ void seg_ids(const AttnArgs &a, int npairs, int s, int &bh, int &pair) {
#if SQZ_PF_PAIR_MAJOR
    const int BH = a.B * a.H;
    pair = s / BH;
    bh = s - pair * BH;
#else
    bh = s / npairs;
    pair = s - bh * npairs;
#endif
}
__device__ __forceinline__ Seg seg_of(const AttnArgs &a, int npairs, int s) {
    Seg g;
    seg_ids(a, npairs, s, g.bh, g.pair);
    g.nkf = ldcg(a.n_keys + g.bh);
    const int last_row = min(g.pair * ws::PR + ws::PR, a.n_q) - 1;
    int nuv = a.causal ? last_row + a.n_u - a.n_q + 1 : a.n_u;
    nuv = max(0, min(nuv, a.n_u));
    g.nkf4 = nuv > 0 ? (g.nkf + 3) & ~3 : g.nkf;
    g.len = g.nkf4 + nuv;
    g.tiles = (g.len + ws::KT - 1) / ws::KT;
    g.cost = g.tiles > 0 ? g.tiles + SEG_W : 0;
    return g;
}
// CTA owning global tile x when T tiles are cut into G equal ranges
// [floor(T c / G), floor(T (c+1) / G))
__device__ __forceinline__ int owner_of(long long x, long long T, int G) {
    const long long c = ((x + 1) * G + T - 1) / T - 1;
    return (int)(c < 0 ? 0 : (c > G - 1 ? G - 1 : c));
}

// Iterates the pieces of CTA c: all roles walk the identical sequence.
struct PieceWalk {
    int s, nseg, npairs, c, G;
    long long st, lo, hi, T;
    long long seg_st;  // start tile of the segment last returned
    // next piece; false when done.  Fills seg, [pb, pe) tile range within the segment.
    __device__ __forceinline__ bool next(const AttnArgs &a, Seg &g, int &pb, int &pe, int &seg_id) {
        while (s < nseg) {
            const bool last_cta = c == G - 1;
            if (st > hi || (st == hi && !last_cta)) return false;
            g = seg_of(a, npairs, s);
            // cost units [st0, en): SEG_W setup units, then one unit per tile
            const long long st0 = st, en = st + g.cost;
            const long long b = max(st0, lo), e = min(en, hi);
            seg_id = s;
            seg_st = st0;
            ++s;
            st = en;
            if (g.tiles == 0) {
                if (st0 >= lo && (st0 < hi || last_cta)) {
                    pb = pe = 0;
                    return true;
                }
                continue;
            }
            if (e > b) {
                pb = (int)max(0LL, b - st0 - SEG_W);
                pe = (int)max(0LL, e - st0 - SEG_W);
                if (pe > pb) return true;  // (a range holding only setup units skips it)
            }
        }
        return false;
    }
};

__global__ void __launch_bounds__(ws::NT, 1)
    k_prefill_attend_ws(AttnArgs a, int npairs, const __grid_constant__ TmaMaps maps) {
    using namespace ws;
    constexpr uint32_t IDESC_S = idesc_bf16(128, KT, false);
    constexpr uint32_t IDESC_O = idesc_bf16(128, D, true);
    extern __shared__ unsigned char smem_raw[];
    unsigned char *sm = reinterpret_cast<unsigned char *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const uint32_t sbase = smem_u32(sm);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + OFF_BAR);
    // s_full / p_full[2 * g + b]: S / P of group g in TMEM buffer b (tiles with
    // tau & 1 == b).  Per buffer, so no waiter is ever two phases behind (a
    // softmax group may finish P(t+1) before the MMA warp consumed P(t)).
    uint64_t *k_full = bar, *k_empty = bar + NKS, *v_full = bar + 2 * NKS,
             *v_empty = bar + 2 * NKS + NVS, *s_full = bar + 2 * NKS + 2 * NVS,
             *p_full = s_full + 4, *o_done = s_full + 8, *q_full = s_full + 10, *q_empty = s_full + 11,
             *o_fin = s_full + 12;  // o_fin[g]: the piece's last PV_g is complete (one phase per piece)
    // misc ints: [0] tmem addr, [1] first segment, [6..7] segments to merge,
    // [8..9] merge flags, [10..13] their CTA ranges; misc64[0] (bytes 48..55) start
    // tile of the first segment
    int *misc = reinterpret_cast<int *>(sm + OFF_MISC);
    long long *misc64 = reinterpret_cast<long long *>(sm + OFF_MISC + 56);

    const int tid = threadIdx.x, warp = tid >> 5;
    const int c = blockIdx.x;
    const int nseg = a.B * a.H * npairs;

    asm volatile("griddepcontrol.wait;" ::: "memory");
    WS_TRACE(tid == 0, 0, 19);
    WS_CTA_T(0);

    // ---- segment prefix (in tiles): per-thread runs + block scan in the K ring ----
    long long *scan = reinterpret_cast<long long *>(sm + OFF_K);
    const int R = (nseg + NT - 1) / NT;
    const int sb = min(nseg, tid * R), se = min(nseg, sb + R);
    long long run = 0;
    for (int s = sb; s < se; ++s) run += seg_of(a, npairs, s).cost;
    scan[tid] = run;
    if (tid == 0) {
        misc[1] = nseg;
        misc64[0] = 0;
    }
    __syncthreads();
    for (int off = 1; off < NT; off <<= 1) {  // Hillis-Steele inclusive scan
        const long long v = tid >= off ? scan[tid - off] : 0;
        __syncthreads();
        scan[tid] += v;
        __syncthreads();
    }
    const long long T = scan[NT - 1];
    // at most one CTA per tile, so every CTA range is non-empty and the owners of
    // a segment's tiles are consecutive CTAs each holding one piece of it
    // (>= SEG_W + 1 units per CTA, so a CTA range never lies inside one segment's setup units)
    const long long Gmax = T / (SEG_W + 1);
    const int G = (int)(Gmax < 1 ? 1 : (Gmax < (long long)gridDim.x ? Gmax : (long long)gridDim.x));
    if (c >= G) {
        if (tid == 0) a.cut[3 * c] = -1;
        return;
    }
    const long long lo = T * c / G, hi = T * (c + 1) / G;
    {
        // first segment of this CTA: the first s that is not (entirely before lo)
        long long st = scan[tid] - run;
        for (int s = sb; s < se; ++s) {
            const long long en = st + seg_of(a, npairs, s).cost;
            if (!(en <= lo && st < lo)) {
                atomicMin(&misc[1], s);
                break;
            }
            st = en;
        }
    }
    __syncthreads();
    {
        const int s0 = misc[1];
        if (s0 >= sb && s0 < se) {
            long long st = scan[tid] - run;
            for (int s = sb; s < s0; ++s) st += seg_of(a, npairs, s).cost;
            misc64[0] = st;
        }
    }
    if (warp == 0) tmem_alloc(reinterpret_cast<uint32_t *>(&misc[0]), 512);
    if (tid == 0) {
        for (int s = 0; s < NKS; ++s) {
            mbar_init(&k_full[s], 32 * NWK);
            mbar_init(&k_empty[s], 1);
        }
        for (int s = 0; s < NVS; ++s) {
            mbar_init(&v_full[s], 32 * NWV);
            mbar_init(&v_empty[s], 1);
        }
        for (int g = 0; g < 4; ++g) {
            mbar_init(&s_full[g], 1);
            mbar_init(&p_full[g], 128);
        }
        for (int g = 0; g < 2; ++g) {
            mbar_init(&o_done[g], 1);
            mbar_init(&o_fin[g], 1);
        }
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        misc[6] = misc[7] = -1;
        mbar_fence_init();
    }
    tc_fence_before();
    __syncthreads();  // also: the scan scratch in the K ring is dead before any cp.async
    tc_fence_after();
    const uint32_t tmem = static_cast<uint32_t>(misc[0]);
    PieceWalk walk{misc[1], nseg, npairs, c, G, misc64[0], lo, hi, T, 0};
    WS_TRACE(tid == 0, 0, 20);

    const int kw = warp == 9 ? 0 : warp == 10 ? 1 : (warp == 12 || warp == 13) ? warp - 10 : -1;
    const int vw = warp == 11 ? 0 : warp >= 14 ? warp - 13 : -1;
    if (kw >= 0 || vw >= 0) {
        // ======================= loaders =======================
        // K/V rows gathered by key position with 16-byte cp.async (a TMA gather4
        // moves only 512 B per instruction and measured ~3x slower here; LDGSTS
        // issue is per-warp latency bound, hence 4 K warps); the Q pair is two
        // contiguous 128-row tiles and comes by TMA
        asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
        const int lane = tid & 31;
        const bool isK = kw >= 0;
        const int w = isK ? kw : vw, nwl = isK ? NWK : NWV;
        const int rA = 2 * (w + nwl * (lane >> 1)) + (lane & 1);  // the row whose position this lane holds
        const int nst = isK ? NKS : NVS;
        uint64_t *full = isK ? k_full : v_full, *empty = isK ? k_empty : v_empty;
        const uint32_t ring = sbase + (isK ? OFF_K : OFF_V);
        Seg g;
        int pb, pe, s_id, tau = 0, piece = 0;
        while (walk.next(a, g, pb, pe, s_id)) {
            if (pe == pb) continue;
            const int h = g.bh % a.H;
            const __nv_bfloat16 *Fx = reinterpret_cast<const __nv_bfloat16 *>(isK ? a.Kp : a.Vp) + (size_t)h * a.L * D;
            const __nv_bfloat16 *Us = reinterpret_cast<const __nv_bfloat16 *>(isK ? a.Ku : a.Vu) + (size_t)g.bh * a.n_u * D;
            const int32_t *kidx = a.key_idx ? a.key_idx + (size_t)g.bh * a.L : nullptr;
            RunList rl;
            RunWin rw;
            if (!kidx) {
                rl.cl = a.sel_cl + (size_t)g.bh * a.c2;
                rl.pref = a.sel_pref + (size_t)g.bh * a.c2;
                rl.koff = a.key_off + (size_t)h * (a.c2 + 1);
                rl.n = ldcg(a.sel_n + g.bh);
                rl.nkf = g.nkf;
                rw.J = 0;
                rw.end = -1;
                rw.p0 = rw.p1 = 0x7fffffff;
            }
            // stream slot -> key position (>= 0 fixed, < 0 user), INVALID when masked;
            // warp-collective (k0 uniform: the tile's first slot)
            auto pos_of = [&](int k0, int k) -> int {
                int p = INVALID;
                if (!kidx) {
                    const int kmax = min(k0 + KT, g.nkf) - 1;
                    if (k0 <= kmax) {  // warp-uniform
                        runwin_cover(rw, rl, k0, kmax, lane);
                        p = runwin_pos(rw, min(k, kmax));
                    }
                } else if (k < g.nkf) {
                    p = ldcg(kidx + k);
                }
                if (k >= g.len || (k >= g.nkf && k < g.nkf4)) return INVALID;
                return k < g.nkf ? p : -1 - (k - g.nkf4);
            };
            for (int tt = pb; tt < pe; ++tt, ++tau) {
                const int st = tau % nst, k0 = tt * KT;
                const int pA = pos_of(k0, k0 + rA);
                if (tau >= nst) mbar_wait(&empty[st], ((tau / nst) - 1) & 1);
                WS_TRACE(w == 0 && lane == 0, tau, isK ? 10 : 11);
                if (isK)
                    gather_rows<NWK>(ring + st * KTILE, Fx, Us, pA, w, lane);
                else
                    gather_rows<NWV>(ring + st * KTILE, Fx, Us, pA, w, lane);
                cp_async_mbar_arrive(&full[st]);
                WS_TRACE(w == 0 && lane == 0, tau, isK ? 8 : 9);
                if (isK && tt == pb && w == 0 && lane == 0) {
                    // the piece's Q pair once the previous piece's S are done (after the
                    // first K tile is in flight, so a piece switch costs one Q latency)
                    if (piece > 0) mbar_wait(q_empty, (piece - 1) & 1);
                    mbar_arrive_expect_tx(q_full, 2 * QTILE);
                    WS_TRACE(true, tau, 23);
                    const int y0 = g.bh * a.n_q + g.pair * PR;
#pragma unroll
                    for (int qg = 0; qg < 2; ++qg)
#pragma unroll
                        for (int hf = 0; hf < 2; ++hf)
                            tma_load_2d(sbase + OFF_Q + qg * QTILE + hf * HBQ, &maps.q, hf * 64, y0 + qg * QT, q_full);
                }
            }
            ++piece;
        }
    } else if (warp == MMAW) {
        // ======================= MMA issuer =======================
        asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
        {  // whole warp, converged; one elected lane issues
            auto wait_full = [&](uint64_t *b, int t, int nst) {
                mbar_wait(&b[t % nst], (t / nst) & 1);
                fence_async_smem();
                tc_fence_after();
            };
            // descriptors: base + (byte offset >> 4) (the start-address field is the low bits)
            const uint64_t dQ = sdesc_sw128(sbase + OFF_Q, 16, 1024);
            const uint64_t dK = sdesc_sw128(sbase + OFF_K, 16, 1024);
            const uint64_t dV = sdesc_sw128(sbase + OFF_V, HBK, 1024);
            // S_g(t) -> TMEM buffer t & 1 of group g (columns g*128 + (t&1)*64)
            auto issue_S = [&](int g, int t) {
                const uint64_t qd = dQ + (uint64_t)((g * QTILE) >> 4);
                const uint64_t kd = dK + (uint64_t)(((t % NKS) * KTILE) >> 4);
                umma_S8_w<(HBQ >> 4), (HBK >> 4)>(tmem + g * 128 + (t & 1) * 64, qd, kd, IDESC_S);
                umma_commit_w(&s_full[2 * g + (t & 1)]);
            };
            // O_g += P_g(t) V(t), P_g(t) bf16 in the first 32 columns of S buffer t & 1
            static_assert(KT == 64, "umma_PV4_w covers 4 K16 steps");
            auto issue_PV = [&](int g, int t, bool first) {
                const uint64_t vd = dV + (uint64_t)(((t % NVS) * KTILE) >> 4);
                umma_PV4_w(tmem + 256 + g * 128, tmem + g * 128 + (t & 1) * 64, vd, IDESC_O, !first);
                umma_commit_w(&o_done[g]);
            };
            Seg g;
            int pb, pe, s_id, tau = 0, piece = 0;
            while (walk.next(a, g, pb, pe, s_id)) {
                const int n = pe - pb;
                if (n == 0) continue;
                mbar_wait(q_full, piece & 1);
                WS_TRACE((tid & 31) == 0, tau, 15);
                // S of the piece's first two tiles; afterwards S(t + 2) follows PV(t),
                // which frees its buffer, so each softmax group always has the next S
                // ready when it finishes a tile
                for (int j2 = 0; j2 < 2 && j2 < n; ++j2) {
                    wait_full(k_full, tau + j2, NKS);
                    issue_S(0, tau + j2);
                    issue_S(1, tau + j2);
                    umma_commit_w(&k_empty[(tau + j2) % NKS]);
                }
                if (n <= 2) umma_commit_w(q_empty);
                for (int i = 0; i < n; ++i, ++tau) {
                    mbar_wait(&p_full[tau & 1], (tau >> 1) & 1);
                    tc_fence_after();
                    WS_TRACE((tid & 31) == 0, tau, 4);
                    wait_full(v_full, tau, NVS);
                    WS_TRACE((tid & 31) == 0, tau, 5);
                    issue_PV(0, tau, i == 0);
                    if (i + 1 == n) umma_commit_w(&o_fin[0]);
                    WS_TRACE((tid & 31) == 0, tau, 12);
                    if (i + 2 < n) {
                        wait_full(k_full, tau + 2, NKS);
                        WS_TRACE((tid & 31) == 0, tau, 6);
                        issue_S(0, tau + 2);
                        WS_TRACE((tid & 31) == 0, tau, 13);
                    }
                    mbar_wait(&p_full[2 + (tau & 1)], (tau >> 1) & 1);
                    tc_fence_after();
                    WS_TRACE((tid & 31) == 0, tau, 7);
                    issue_PV(1, tau, i == 0);
                    if (i + 1 == n) umma_commit_w(&o_fin[1]);
                    umma_commit_w(&v_empty[tau % NVS]);
                    if (i + 2 < n) {
                        issue_S(1, tau + 2);
                        umma_commit_w(&k_empty[(tau + 2) % NKS]);
                        if (i + 3 == n) umma_commit_w(q_empty);
                    }
                }
                ++piece;
            }
        }
        __syncwarp();
    } else {
        // ======================= softmax groups =======================
        asm volatile("setmaxnreg.inc.sync.aligned.u32 184;");
        const int g = warp >> 2, r = tid & 127;  // TMEM lane = r
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tS0 = tmem + g * 128 + lane_off, tO = tmem + 256 + g * 128 + lane_off;
        const float sl2 = a.scale * LOG2E;
        Seg sg;
        int pb, pe, s_id, tau = 0, piece = 0;
        while (walk.next(a, sg, pb, pe, s_id)) {
            const int trow = sg.pair * PR + g * QT + r;
            const bool row_ok = trow < a.n_q;
            const size_t orow = (size_t)sg.bh * a.n_q + trow;
            if (pe == pb) {  // no key at all: identity outputs (an error when final)
                if (row_ok) {
                    for (int k = 0; k < D; ++k) {
                        if (a.out_dtype == SQZ_BF16)
                            reinterpret_cast<__nv_bfloat16 *>(a.O)[orow * D + k] = __float2bfloat16_rn(0.f);
                        else
                            reinterpret_cast<float *>(a.O)[orow * D + k] = 0.f;
                    }
                    a.LSE[orow] = -INFINITY;
                    if (!a.partial) atomicOr(a.status, 1);
                }
                continue;
            }
            // visible keys of the row form a prefix of the segment's stream: all fixed
            // keys, then user keys u <= trow + n_u - n_q (causal, R8) or all of them
            // visible stream slots: [0, a_end) fixed keys and [nkf4, b_end) user keys
            // u <= trow + n_u - n_q (causal, R8) or all of them
            const int uvis = a.causal ? max(0, trow + a.n_u - a.n_q + 1) : a.n_u;
            const int a_end = row_ok ? sg.nkf : 0;
            const int b_end = row_ok ? min(sg.len, sg.nkf4 + uvis) : 0;
            float m_used = -INFINITY, l = 0.f;
            for (int tt = pb; tt < pe; ++tt, ++tau) {
                const int k0 = tt * KT;
                mbar_wait(&s_full[2 * g + (tau & 1)], (tau >> 1) & 1);
                tc_fence_after();
                WS_TRACE(r == 0, tau, 2 * g);
                const uint32_t tS = tS0 + (tau & 1) * 64;
                float sv[KT];
#pragma unroll
                for (int cc = 0; cc < KT / 32; ++cc)
                    tmem_ld32(tS + cc * 32, *reinterpret_cast<float(*)[32]>(sv + cc * 32));
                tmem_wait_ld();
                WS_TRACE(r == 0 && g == 0, tau, 16);
                const int na = a_end - k0, nb0 = sg.nkf4 - k0, nb1 = b_end - k0;
                if (na < KT && (nb0 > 0 || nb1 < KT)) {
                    // visible slots [0, na) u [nb0, nb1) as a 128-bit mask, then one
                    // bit test + select per logit
#pragma unroll
                    for (int w = 0; w < KT / 32; ++w) {
                        const uint32_t vm = range_bits(0, na, 32 * w) | range_bits(nb0, nb1, 32 * w);
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            sv[32 * w + j] = (vm >> j) & 1u ? sv[32 * w + j] : -INFINITY;
                    }
                }
                float mx8[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) mx8[j] = sv[j];
#pragma unroll
                for (int j = 8; j < KT; j += 8) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) mx8[q] = fmaxf(mx8[q], sv[j + q]);
                }
                const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                       fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * sl2;
                const bool need = mx > m_used + 8.f;
                const float alpha = need ? ((m_used == -INFINITY) ? 0.f : exp2f(m_used - mx)) : 1.f;
                if (tt > pb && __any_sync(FULL, need)) {
                    // O_g must be stable: PV_g(tau-1) has completed
                    mbar_wait(&o_done[g], (tau - 1) & 1);
                    tc_fence_after();
#pragma unroll 1
                    for (int cc = 0; cc < D / 32; ++cc) {
                        float v[32];
                        tmem_ld32(tO + cc * 32, v);
                        tmem_wait_ld();
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] *= alpha;
                        tmem_st32(tO + cc * 32, v);
                    }
                    tmem_wait_st();
                }
                l *= alpha;
                if (need) m_used = mx;
                const float moff = (m_used == -INFINITY) ? 0.f : m_used;
                WS_TRACE(r == 0 && g == 0, tau, 14);
                // p = 2^(s*scale*log2e - m): FFMA2 for the pair, MUFU.EX2 (or the
                // FMA-pipe polynomial), bf16x2 packed in place into sv[j] (slot j <= 2j
                // is already consumed), row sum by FADD2
                const float2 sc2 = make_float2(sl2, sl2), mo2 = make_float2(-moff, -moff);
                float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
                for (int j = 0; j < KT / 2; ++j) {
                    const float2 x = ffma2(make_float2(sv[2 * j], sv[2 * j + 1]), sc2, mo2);
                    float2 p;
                    if ((SQZ_PF_EMU_MASK >> (j & 7)) & 1u) {
                        p = exp2_poly2(x);
                    } else {
                        p.x = fast_exp2(x.x);
                        p.y = fast_exp2(x.y);
                    }
                    acc2[j & 1] = fadd2(acc2[j & 1], p);
                    const __nv_bfloat162 b2 = __floats2bfloat162_rn(p.x, p.y);
                    sv[j] = __uint_as_float(*reinterpret_cast<const uint32_t *>(&b2));
                }
                const float2 accs = fadd2(acc2[0], acc2[1]);
                l += accs.x + accs.y;
                WS_TRACE(r == 0 && g == 0, tau, 17);
                tmem_st32f(tS, sv);            // P: columns 0..31 of the S buffer
                tmem_wait_st();
                WS_TRACE(r == 0 && g == 0, tau, 18);
                tc_fence_before();
                mbar_arrive(&p_full[2 * g + (tau & 1)]);
                WS_TRACE(r == 0, tau, 2 * g + 1);
            }
            // ---- the piece's result for the row: final, or a partial to merge ----
            // (o_done alone is ambiguous here: with S issued two tiles ahead, PV(last-1)
            // may still be pending, two phases behind)
            mbar_wait(&o_fin[g], piece & 1);
            ++piece;
            tc_fence_after();
            const int c0 = owner_of(walk.seg_st + SEG_W, T, G),
                      c1 = owner_of(walk.seg_st + SEG_W + sg.tiles - 1, T, G);
            const bool have = row_ok && l > 0.f;
            const float inv_l = have ? 1.0f / l : 0.f;
            const float lse = have ? (m_used + log2f(l)) * LN2 : -INFINITY;
            if (c0 == c1) {
#pragma unroll 1
                for (int cc = 0; cc < D / 32; ++cc) {
                    float v[32];
                    tmem_ld32(tO + cc * 32, v);
                    tmem_wait_ld();
                    if (row_ok) {
                        if (a.out_dtype == SQZ_BF16) {
                            uint4 *dst = reinterpret_cast<uint4 *>(reinterpret_cast<__nv_bfloat16 *>(a.O) + orow * D + cc * 32);
#pragma unroll
                            for (int j = 0; j < 32; j += 8) {
                                uint32_t u[4];
#pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    const __nv_bfloat162 b = __floats2bfloat162_rn(v[j + 2 * q] * inv_l, v[j + 2 * q + 1] * inv_l);
                                    u[q] = *reinterpret_cast<const uint32_t *>(&b);
                                }
                                dst[j / 8] = make_uint4(u[0], u[1], u[2], u[3]);
                            }
                        } else {
                            float4 *dst = reinterpret_cast<float4 *>(reinterpret_cast<float *>(a.O) + orow * D + cc * 32);
#pragma unroll
                            for (int j = 0; j < 32; j += 4)
                                dst[j / 4] = make_float4(v[j] * inv_l, v[j + 1] * inv_l, v[j + 2] * inv_l, v[j + 3] * inv_l);
                        }
                    }
                }
                if (row_ok) {
                    a.LSE[orow] = lse;
                    if (!have && !a.partial) atomicOr(a.status, 1);
                }
            } else {
                const size_t slot = (size_t)(s_id + c) * PR + g * QT + r;  // piece id = segment + CTA
#pragma unroll 1
                for (int cc = 0; cc < D / 32; ++cc) {
                    float v[32];
                    tmem_ld32(tO + cc * 32, v);
                    tmem_wait_ld();
                    if (row_ok) {
                        float4 *dst = reinterpret_cast<float4 *>(a.part_o + slot * D + cc * 32);
#pragma unroll
                        for (int j = 0; j < 32; j += 4)
                            dst[j / 4] = make_float4(v[j] * inv_l, v[j + 1] * inv_l, v[j + 2] * inv_l, v[j + 3] * inv_l);
                    }
                }
                if (row_ok) a.part_lse[slot] = lse;
                WS_TRACE(r == 0 && g == 0, tau - 1, 19);
                // only a CTA's first and last pieces can be cut
                if (tid == 0) {
                    if (misc[6] < 0) misc[6] = s_id;
                    else if (misc[6] != s_id) misc[7] = s_id;
                    misc[10 + 2 * (misc[7] == s_id ? 1 : 0)] = c0;
                    misc[11 + 2 * (misc[7] == s_id ? 1 : 0)] = c1;
                }
            }
        }
        tc_fence_before();
    }
    __threadfence();
    __syncthreads();
    WS_TRACE(tid == 0, 0, 21);
    WS_CTA_T(1);
    if (warp == 0) tmem_dealloc(tmem, 512);
    // ---- cut segments are merged by k_merge_cut (next launch, all SMs): the
    // first piece's owner c0 lists (segment, c0, c1) ----
    // (slot c: the cut segment whose first piece this CTA holds, or -1; every slot
    // is rewritten by every call, so the list needs no counter or reset)
    if (tid == 0) {
        asm volatile("griddepcontrol.launch_dependents;");
        int seg = -1, k1 = -1;
        for (int k = 0; k < 2; ++k)
            if (misc[6 + k] >= 0 && misc[10 + 2 * k] == c) { seg = misc[6 + k]; k1 = misc[11 + 2 * k]; }
        a.cut[3 * c] = seg;
        a.cut[3 * c + 1] = c;
        a.cut[3 * c + 2] = k1;
    }
    WS_TRACE(tid == 0, 0, 22);
    WS_CTA_T(2);
}

// Merge of the cut segments' pieces: CTA (k, slice) merges rows
// [slice * MERGE_ROWS, +MERGE_ROWS) of the segment whose first piece main-kernel
// CTA k holds (slot k; -1: none) from its pieces' (O/l, lse) partials.
// Launched with programmatic stream serialization after the main kernel.
#ifndef SQZ_MERGE_ROWS
#define SQZ_MERGE_ROWS 64
#endif
constexpr int MERGE_ROWS = SQZ_MERGE_ROWS;  // rows per merge CTA
__global__ void __launch_bounds__(256) k_merge_cut(AttnArgs a, int npairs) {
    using namespace ws;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ float wgt[8][MERGE_ROWS];  // up to 8 pieces in registers' worth of weights
    const int tid = threadIdx.x;
    const int k = blockIdx.x;
    const int s = ldcg(a.cut + 3 * k);
    if (s >= 0) {
        const int c0 = ldcg(a.cut + 3 * k + 1), c1 = ldcg(a.cut + 3 * k + 2);
        const int np = c1 - c0 + 1;
        int bh, pair;
        seg_ids(a, npairs, s, bh, pair);
        const int nrow_seg = min(PR, a.n_q - pair * PR);
        const int r_lo = blockIdx.y * MERGE_ROWS, nrow = min(MERGE_ROWS, nrow_seg - r_lo);
        if (nrow > 0) {
            const float *lse_p = a.part_lse + (size_t)(s + c0) * PR + r_lo;
            const float *o_p = a.part_o + ((size_t)(s + c0) * PR + r_lo) * D;
            const int row0 = pair * PR + r_lo;
            float *wg = &wgt[0][0];
            const bool small = np <= 8;
            if (tid < nrow) {
                const int rr = tid;
                float M = -INFINITY;
                for (int p = 0; p < np; ++p) M = fmaxf(M, ldcg(lse_p + (size_t)p * PR + rr));
                float L = 0.f;
                for (int p = 0; p < np; ++p) {
                    const float w = M == -INFINITY ? 0.f : expf(ldcg(lse_p + (size_t)p * PR + rr) - M);
                    if (small) wg[p * MERGE_ROWS + rr] = w;
                    L += w;
                }
                const float inv = M == -INFINITY ? 0.f : 1.f / L;
                if (small)
                    for (int p = 0; p < np; ++p) wg[p * MERGE_ROWS + rr] *= inv;
                const size_t orow = (size_t)bh * a.n_q + row0 + rr;
                a.LSE[orow] = M == -INFINITY ? -INFINITY : M + logf(L);
                if (M == -INFINITY && !a.partial) atomicOr(a.status, 1);
            }
            __syncthreads();
            for (int it = tid; it < nrow * (D / 4); it += blockDim.x) {
                const int rr = it / (D / 4), ch = it % (D / 4);
                float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
                float4 o[8];
#pragma unroll
                for (int p = 0; p < 8; ++p)
                    if (p < np) o[p] = __ldcg(reinterpret_cast<const float4 *>(o_p + ((size_t)p * PR + rr) * D) + ch);
                float wsum_inv = 1.f;
                if (!small) {  // > 8 pieces (never at the configured sizes): recompute the weights
                    float M = -INFINITY;
                    for (int p = 0; p < np; ++p) M = fmaxf(M, ldcg(lse_p + (size_t)p * PR + rr));
                    float L = 0.f;
                    for (int p = 0; p < np; ++p) {
                        const float w = M == -INFINITY ? 0.f : expf(ldcg(lse_p + (size_t)p * PR + rr) - M);
                        L += w;
                        const float4 op = __ldcg(reinterpret_cast<const float4 *>(o_p + ((size_t)p * PR + rr) * D) + ch);
                        acc.x = fmaf(w, op.x, acc.x);
                        acc.y = fmaf(w, op.y, acc.y);
                        acc.z = fmaf(w, op.z, acc.z);
                        acc.w = fmaf(w, op.w, acc.w);
                    }
                    wsum_inv = L > 0.f ? 1.f / L : 0.f;
                } else {
#pragma unroll
                    for (int p = 0; p < 8; ++p)
                        if (p < np) {
                            const float w = wg[p * MERGE_ROWS + rr];
                            acc.x = fmaf(w, o[p].x, acc.x);
                            acc.y = fmaf(w, o[p].y, acc.y);
                            acc.z = fmaf(w, o[p].z, acc.z);
                            acc.w = fmaf(w, o[p].w, acc.w);
                        }
                }
                acc.x *= wsum_inv; acc.y *= wsum_inv; acc.z *= wsum_inv; acc.w *= wsum_inv;
                const size_t orow = (size_t)bh * a.n_q + row0 + rr;
                if (a.out_dtype == SQZ_BF16) {
                    __nv_bfloat162 *dst = reinterpret_cast<__nv_bfloat162 *>(reinterpret_cast<__nv_bfloat16 *>(a.O) + orow * D + ch * 4);
                    dst[0] = __floats2bfloat162_rn(acc.x, acc.y);
                    dst[1] = __floats2bfloat162_rn(acc.z, acc.w);
                } else {
                    reinterpret_cast<float4 *>(reinterpret_cast<float *>(a.O) + orow * D)[ch] = acc;
                }
            }
        }
    }
}

namespace {
int ws_grid() { return device_sm_count(); }
}  // namespace

bool prefill_ws_applies(int d, int dtype, int n_q) {
    return n_q > 1 && d == 128 && dtype == SQZ_BF16;
}
// rows of the partial buffers: one 256-row slot per piece, piece id = segment + CTA
size_t prefill_ws_part_rows(int B, int H, int n_q) {
    const size_t npairs = (size_t)(n_q + ws::PR - 1) / ws::PR;
    return ((size_t)B * H * npairs + ws_grid()) * ws::PR;
}

namespace {
CUresult encode_map(CUtensorMap *m, const void *ptr, uint64_t rows, uint32_t box_rows) {
    cuuint64_t dims[2] = {(cuuint64_t)ws::D, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ws::D * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t estr[2] = {1, 1};
    // resolved through the runtime so libsqz has no link-time libcuda dependency
    using encode_fn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                   const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                   const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static encode_fn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess || q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<encode_fn>(p);
    }();
    if (!fn) return CUDA_ERROR_NOT_FOUND;
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims,
                                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}
}  // namespace

cudaError_t launch_prefill_attention_ws(const AttnArgs &a, cudaStream_t st) {
    const int npairs = (a.n_q + ws::PR - 1) / ws::PR;
    TmaMaps maps;
    if (encode_map(&maps.q, a.Q, (uint64_t)a.B * a.H * a.n_q, 128) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    {
        cudaError_t e = ensure_func_attr((const void *)k_prefill_attend_ws,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, ws::BYTES);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ws_grid());
    cfg.blockDim = dim3(ws::NT);
    cfg.dynamicSmemBytes = ws::BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_prefill_attend_ws, a, npairs, maps);
    if (e != cudaSuccess) return e;
    // merge of the cut segments on all SMs (at most one cut per CTA boundary)
    cudaLaunchConfig_t mc = cfg;
    mc.gridDim = dim3(ws_grid(), ws::PR / MERGE_ROWS);
    mc.blockDim = dim3(256);
    mc.dynamicSmemBytes = 0;
    return cudaLaunchKernelEx(&mc, k_merge_cut, a, npairs);
}

}  // namespace sqz

#ifdef SQZ_TRACE
extern "C" int sqz_trace_ws_cta(void *host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, sqz::g_cta_ws, bytes < sizeof(sqz::g_cta_ws) ? bytes : sizeof(sqz::g_cta_ws));
}
extern "C" int sqz_trace_ws(void *host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, sqz::g_trace_ws, bytes < sizeof(sqz::g_trace_ws) ? bytes : sizeof(sqz::g_trace_ws));
}
#endif
