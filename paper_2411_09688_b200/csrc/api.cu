// api.cu -- the C ABI of libsqz.so (include/sqz.h): argument validation,
// workspace carving and kernel launches.  No device allocation, no host
// synchronisation on the online path.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/sqz.h"
#include "internal.h"

using namespace sqz;

namespace {
thread_local char g_err[512] = "";

int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}
}  // namespace

int sqz::set_error(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

namespace {
int cuda_fail(cudaError_t e, const char *what) {
    return fail(SQZ_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}
bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

struct Carve {
    char *p;
    size_t used = 0;
    template <typename X> X *take(size_t n) {
        used = (used + 255) & ~(size_t)255;
        X *r = reinterpret_cast<X *>(p ? p + used : nullptr);
        used += n * sizeof(X);
        return r;
    }
};

int check_index(const sqz_index *idx, bool need_tables) {
    if (!idx) return fail(SQZ_ERR_INVALID_ARG, "idx is NULL");
    if (idx->H < 1) return fail(SQZ_ERR_INVALID_ARG, "idx->H = %d must be >= 1", idx->H);
    if (idx->d != 64 && idx->d != 128)
        return fail(SQZ_ERR_UNSUPPORTED, "idx->d = %d: head dimension must be 64 or 128", idx->d);
    if (idx->L < 1 || idx->L > 0x7fffffffLL)
        return fail(SQZ_ERR_INVALID_ARG, "idx->L = %lld out of range [1, 2^31)", (long long)idx->L);
    if (idx->levels < 1 || idx->levels > 3)
        return fail(SQZ_ERR_INVALID_ARG, "idx->levels = %d must be 1, 2 or 3", idx->levels);
    if (idx->dtype != SQZ_F32 && idx->dtype != SQZ_BF16)
        return fail(SQZ_ERR_INVALID_ARG, "idx->dtype = %d is not a sqz_dtype", idx->dtype);
    if (idx->c2 < 1 || (int64_t)idx->c2 > idx->L)
        return fail(SQZ_ERR_INVALID_ARG, "idx->c2 = %d must be in [1, L=%lld]", idx->c2,
                    (long long)idx->L);
    if (idx->levels >= 2 && (idx->c1 < 1 || idx->c1 > idx->c2))
        return fail(SQZ_ERR_INVALID_ARG, "idx->c1 = %d must be in [1, c2=%d]", idx->c1, idx->c2);
    if (idx->levels == 3 && (idx->c0 < 1 || idx->c0 > idx->c1))
        return fail(SQZ_ERR_INVALID_ARG, "idx->c0 = %d must be in [1, c1=%d]", idx->c0, idx->c1);
    if (idx->levels == 3 && idx->L_total != 0)
        return fail(SQZ_ERR_UNSUPPORTED, "three-level indexes cannot be sharded");
    if (idx->L_total < 0 || idx->L_total > 0x7fffffffLL)
        return fail(SQZ_ERR_INVALID_ARG, "idx->L_total = %lld out of range [0, 2^31)",
                    (long long)idx->L_total);
    if (need_tables) {
        if (!idx->C2 || !idx->N2 || !idx->key_off)
            return fail(SQZ_ERR_INVALID_ARG, "idx->C2 / N2 / key_off must be non-NULL");
        if (!aligned16(idx->C2)) return fail(SQZ_ERR_INVALID_ARG, "idx->C2 must be 16-byte aligned");
        if (idx->levels >= 2) {
            if (!idx->C1 || !idx->N1 || !idx->child_off)
                return fail(SQZ_ERR_INVALID_ARG, "idx->C1 / N1 / child_off must be non-NULL (levels>=2)");
            if (!aligned16(idx->C1)) return fail(SQZ_ERR_INVALID_ARG, "idx->C1 must be 16-byte aligned");
        }
        if (idx->levels == 3) {
            if (!idx->C0 || !idx->N0 || !idx->child_off0)
                return fail(SQZ_ERR_INVALID_ARG, "idx->C0 / N0 / child_off0 must be non-NULL (levels=3)");
            if (!aligned16(idx->C0)) return fail(SQZ_ERR_INVALID_ARG, "idx->C0 must be 16-byte aligned");
        }
    }
    return SQZ_OK;
}

// ---------------- lookup workspace ----------------
struct LookupWs {
    LevelArgs l0, l1, l2;  // l0: levels == 3 only
    float2 *send, *recv;  // comm mode: this rank's statistics, the gathered [world] ones
    size_t bytes;
};

LookupWs lookup_carve(const sqz_index *idx, int B, int n_q, char *base, int world = 0) {
    Carve cv{base};
    const int64_t BH = (int64_t)B * idx->H;
    const int CHR = lookup_chunk_rows();
    const int nqt = (n_q + lookup_qtile() - 1) / lookup_qtile();
    const bool prefill = n_q > 1;
    LookupWs w;
    std::memset(&w.l0, 0, sizeof(w.l0));
    std::memset(&w.l1, 0, sizeof(w.l1));
    std::memset(&w.l2, 0, sizeof(w.l2));
    auto level = [&](LevelArgs &lv, int c) {
        const int nch = (c + CHR - 1) / CHR;
        lv.tick = cv.take<int32_t>(BH);
        lv.sel_pref = cv.take<int32_t>(BH * c);
        lv.gstat = cv.take<float2>(BH * n_q);
        if (prefill) {
            lv.rowlse = cv.take<float>(BH * n_q);
            lv.colpart = cv.take<float>((size_t)nqt * BH * c);
        } else {
            lv.logits = cv.take<float>(BH * c);
            lv.part = cv.take<float2>(BH * nch);
        }
    };
    level(w.l2, idx->c2);
    // candidate-list levels of a bf16 prefill with 4+ query tiles: gathered rows
    const bool gat = prefill && idx->dtype == SQZ_BF16 && n_q >= 4 * 128;
    if (gat && idx->levels >= 2) w.l2.cgather = cv.take<char>((size_t)BH * idx->c2 * idx->d * 2);
    if (idx->levels >= 2) {
        level(w.l1, idx->c1);
        w.l1.list = cv.take<int32_t>(BH * idx->c1);
        w.l1.n_list = cv.take<int32_t>(BH);
        w.l1.exp_list = cv.take<int32_t>(BH * idx->c2);
        w.l1.n_exp = cv.take<int32_t>(BH);
    }
    if (gat && idx->levels == 3) w.l1.cgather = cv.take<char>((size_t)BH * idx->c1 * idx->d * 2);
    if (idx->levels == 3) {
        level(w.l0, idx->c0);
        w.l0.list = cv.take<int32_t>(BH * idx->c0);
        w.l0.n_list = cv.take<int32_t>(BH);
        w.l0.exp_list = cv.take<int32_t>(BH * idx->c1);
        w.l0.n_exp = cv.take<int32_t>(BH);
    }
    w.send = w.recv = nullptr;
    if (world > 0) {
        w.send = cv.take<float2>(BH * n_q);
        w.recv = cv.take<float2>((size_t)world * BH * n_q);
    }
    w.bytes = cv.used + 256;
    return w;
}

// ---------------- attention workspace ----------------
struct AttnWs {
    float *part_o, *part_lse;
    int32_t *status, *row_cnt, *cut;
    int32_t kch, max_chunks;
    char *shared;  // batch-shared decode region (B >= 2, n_q == 1)
    size_t bytes;
};
AttnWs attn_carve(const sqz_index *idx, int B, int n_q, int n_u, char *base) {
    Carve cv{base};
    AttnWs w;
    w.kch = attention_kch(n_q);
    w.max_chunks = attention_max_parts(idx->L, n_u, n_q);
    const size_t rows = (size_t)B * idx->H * n_q;
    w.status = cv.take<int32_t>(64);
    w.row_cnt = cv.take<int32_t>(rows);
    w.cut = cv.take<int32_t>(3 * 1024);  // one (segment, c0, c1) slot per persistent CTA
    // partial rows: [rows, max_chunks] for the split-KV kernels, one 256-row slot
    // per piece for the persistent prefill kernel
    // (the persistent prefill kernel indexes its partials by piece, never by chunk)
    const size_t prow = prefill_ws_applies(idx->d, idx->dtype, n_q)
                            ? prefill_ws_part_rows(B, idx->H, n_q)
                            : rows * w.max_chunks;
    w.part_lse = cv.take<float>(prow);
    w.part_o = cv.take<float>(prow * idx->d);
    w.shared = shared_attn_applies(B, n_q, idx->d, idx->dtype, idx->c2)
                   ? cv.take<char>(shared_attn_ws_bytes(B, idx->H, idx->c2))
                   : nullptr;
    w.bytes = cv.used + 256;
    return w;
}
char *align_ws(void *ws) { return reinterpret_cast<char *>(((uintptr_t)ws + 255) & ~(uintptr_t)255); }
}  // namespace

extern "C" {

const char *sqz_last_error(void) { return g_err; }
int sqz_abi_version(void) { return SQZ_ABI_VERSION; }

int sqz_device_check(void) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    cudaDeviceProp p;
    e = cudaGetDeviceProperties(&p, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
    if (p.major != 10 || p.minor != 0)
        return fail(SQZ_ERR_UNSUPPORTED, "device %s is sm_%d%d; libsqz is built for sm_100a", p.name,
                    p.major, p.minor);
    return SQZ_OK;
}

int sqz_workspace_init(void *ws, size_t ws_bytes, void *stream) {
    if (!ws && ws_bytes) return fail(SQZ_ERR_INVALID_ARG, "ws is NULL");
    cudaError_t e = cudaMemsetAsync(ws, 0, ws_bytes, (cudaStream_t)stream);
    return e == cudaSuccess ? SQZ_OK : cuda_fail(e, "cudaMemsetAsync(ws)");
}

// ------------------------------------------------------------------ offline
int sqz_cluster_keys_workspace(const sqz_index *idx, size_t *ws_bytes) {
    int rc = check_index(idx, false);
    if (rc) return rc;
    if (!ws_bytes) return fail(SQZ_ERR_INVALID_ARG, "ws_bytes is NULL");
    *ws_bytes = kmeans_workspace_bytes(*idx) + 256;
    return SQZ_OK;
}

int sqz_cluster_keys(const void *K, const void *V, const int64_t *init2, const int64_t *init1,
                     sqz_index *idx, void *Kp, void *Vp, const sqz_kmeans_params *p, void *ws,
                     size_t ws_bytes, int32_t *iters_out, void *stream) {
    int rc = check_index(idx, true);
    if (rc) return rc;
    if (!K || !V || !Kp || !Vp) return fail(SQZ_ERR_INVALID_ARG, "K, V, Kp, Vp must be non-NULL");
    if (!aligned16(K) || !aligned16(V) || !aligned16(Kp) || !aligned16(Vp))
        return fail(SQZ_ERR_INVALID_ARG, "K, V, Kp, Vp must be 16-byte aligned");
    if (idx->L_total != 0)
        return fail(SQZ_ERR_INVALID_ARG, "sqz_cluster_keys builds a full index: L_total must be 0");
    if (!init2) return fail(SQZ_ERR_INVALID_ARG, "init2 is NULL");
    if (idx->levels >= 2 && !init1) return fail(SQZ_ERR_INVALID_ARG, "init1 is NULL (levels>=2)");
    if (idx->levels == 3 && (!p || !p->init0))
        return fail(SQZ_ERR_INVALID_ARG, "p->init0 is NULL (levels=3)");
    if (!idx->perm) return fail(SQZ_ERR_INVALID_ARG, "idx->perm is NULL");
    if (!p || p->max_iters < 1 || !(p->tol >= 0.f))
        return fail(SQZ_ERR_INVALID_ARG, "kmeans params: max_iters >= 1 and tol >= 0 required");
    if (!ws) return fail(SQZ_ERR_INVALID_ARG, "ws is NULL");
    char err[400] = "";
    rc = cluster_keys(K, V, init2, init1, idx, Kp, Vp, *p, ws, ws_bytes, iters_out,
                      (cudaStream_t)stream, err, sizeof(err));
    if (rc) return fail(rc, "sqz_cluster_keys: %s", err);
    return SQZ_OK;
}

int sqz_index_validate_workspace(const sqz_index *idx, size_t *ws_bytes) {
    int rc = check_index(idx, false);
    if (rc) return rc;
    if (!ws_bytes) return fail(SQZ_ERR_INVALID_ARG, "ws_bytes is NULL");
    *ws_bytes = validate_workspace_bytes(*idx);
    return SQZ_OK;
}

int sqz_index_validate(const sqz_index *idx, void *ws, size_t ws_bytes, void *stream) {
    int rc = check_index(idx, true);
    if (rc) return rc;
    if (!idx->perm) return fail(SQZ_ERR_INVALID_ARG, "idx->perm is NULL");
    char err[400] = "";
    rc = index_validate(*idx, ws, ws_bytes, (cudaStream_t)stream, err, sizeof(err));
    if (rc) return fail(rc, "%s", err);
    return SQZ_OK;
}

// ------------------------------------------------------------------ lookup
int sqz_lookup_workspace(const sqz_index *idx, int32_t B, int32_t n_q, size_t *ws_bytes) {
    int rc = check_index(idx, false);
    if (rc) return rc;
    if (B < 1 || n_q < 1) return fail(SQZ_ERR_INVALID_ARG, "B = %d and n_q = %d must be >= 1", B, n_q);
    if (!ws_bytes) return fail(SQZ_ERR_INVALID_ARG, "ws_bytes is NULL");
    *ws_bytes = lookup_carve(idx, B, n_q, nullptr).bytes + 256;
    return SQZ_OK;
}

static int lookup_check(const sqz_index *idx, const void *Q, int32_t B, int32_t n_q,
                        const sqz_lookup_params *p, const sqz_selection *out, const void *ws) {
    int rc = check_index(idx, true);
    if (rc) return rc;
    if (!Q) return fail(SQZ_ERR_INVALID_ARG, "Q is NULL");
    if (!aligned16(Q)) return fail(SQZ_ERR_INVALID_ARG, "Q must be 16-byte aligned");
    if (B < 1 || n_q < 1) return fail(SQZ_ERR_INVALID_ARG, "B = %d and n_q = %d must be >= 1", B, n_q);
    if (!p) return fail(SQZ_ERR_INVALID_ARG, "params is NULL");
    if (!(p->T >= 0.f) || std::isinf(p->T))
        return fail(SQZ_ERR_INVALID_ARG, "T = %g must be finite and >= 0", (double)p->T);
    if (idx->levels >= 2 && (!(p->T1 >= 0.f) || std::isinf(p->T1)))
        return fail(SQZ_ERR_INVALID_ARG, "T1 = %g must be finite and >= 0", (double)p->T1);
    if (idx->levels == 3 && (!(p->T0 >= 0.f) || std::isinf(p->T0)))
        return fail(SQZ_ERR_INVALID_ARG, "T0 = %g must be finite and >= 0", (double)p->T0);
    if (idx->levels == 3 && p->comm)
        return fail(SQZ_ERR_UNSUPPORTED, "sharded lookup of a three-level index");
    if (!std::isfinite(p->scale)) return fail(SQZ_ERR_INVALID_ARG, "scale must be finite");
    if (!out || !out->clusters || !out->n_clusters || !out->n_keys || !out->key_pref)
        return fail(SQZ_ERR_INVALID_ARG, "selection outputs clusters/n_clusters/n_keys/key_pref required");
    if (!ws) return fail(SQZ_ERR_INVALID_ARG, "ws is NULL");
    return SQZ_OK;
}

// wires the level arguments of the carved workspace to the index and outputs
static void lookup_levels(const sqz_index *idx, const sqz_lookup_params *p, const sqz_selection *out,
                          LookupWs &w) {
    LevelArgs &l2 = w.l2;
    l2.C = idx->C2;
    l2.N = idx->N2;
    l2.off = idx->key_off;
    l2.c = idx->c2;
    l2.T = p->T;
    l2.list = out->clusters;
    l2.n_list = out->n_clusters;
    l2.exp_list = out->key_idx;  // optional expansion
    l2.sel_pref = out->key_pref;
    l2.n_exp = out->n_keys;
    l2.exp_stride = idx->L;
    l2.dbg_S = out->dbg_S;
    l2.dbg_lse = out->dbg_lse;
    if (idx->levels >= 2) {
        LevelArgs &l1 = w.l1;
        l1.C = idx->C1;
        l1.N = idx->N1;
        l1.off = idx->child_off;
        l1.c = idx->c1;
        l1.T = p->T1;
        l1.exp_stride = idx->c2;
        l1.bitmap = out->l1_surv;
        l1.dbg_S = out->dbg_S1;
        l2.rows = l1.exp_list;
        l2.n_rows = l1.n_exp;
        l2.row_stride = idx->c2;
    }
    if (idx->levels == 3) {
        LevelArgs &l0 = w.l0;
        l0.C = idx->C0;
        l0.N = idx->N0;
        l0.off = idx->child_off0;
        l0.c = idx->c0;
        l0.T = p->T0;
        l0.exp_stride = idx->c1;
        l0.bitmap = out->l0_surv;
        l0.dbg_S = out->dbg_S0;
        w.l1.rows = l0.exp_list;
        w.l1.n_rows = l0.n_exp;
        w.l1.row_stride = idx->c1;
    }
}

// one stage of the staged lookup (see sqz_centroid_lookup_stage)
static int run_stage(const sqz_index *idx, const LookupShape &s, const void *Q, LookupWs &w, int stage,
                     int P, const float2 *stats_in, float2 *stats_out, cudaStream_t st) {
    const int levels = idx->levels;
    const int64_t n = (int64_t)s.B * s.H * s.n_q;
    const bool prefill = s.n_q > 1;
    auto level = [&](int k) -> LevelArgs & { return (levels == 2 && k == 1) ? w.l1 : w.l2; };
    cudaError_t e;
    if (stage > 0) {
        LevelArgs &lv = level(stage);
        e = launch_fold_stats(P, stats_in, n, const_cast<float2 *>(lv.gstat),
                              prefill ? lv.rowlse : nullptr, st);
        if (e != cudaSuccess) return cuda_fail(e, "stats fold");
        if (prefill && lv.dbg_lse) {
            e = cudaMemcpyAsync(lv.dbg_lse, lv.rowlse, n * sizeof(float), cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return cuda_fail(e, "dbg_lse copy");
        }
        lv.phase = 2;
        e = launch_lookup_level(s, Q, lv, st);
        if (e != cudaSuccess) return cuda_fail(e, "lookup select");
    }
    if (stage < levels) {
        LevelArgs &nx = level(stage + 1);
        nx.phase = 1;
        nx.stats_out = stats_out;
        e = launch_lookup_level(s, Q, nx, st);
        if (e != cudaSuccess) return cuda_fail(e, "lookup statistics");
    }
    return SQZ_OK;
}

int sqz_lookup_workspace_comm(const sqz_index *idx, int32_t B, int32_t n_q, int32_t world,
                              size_t *ws_bytes) {
    int rc = check_index(idx, false);
    if (rc) return rc;
    if (B < 1 || n_q < 1 || world < 1)
        return fail(SQZ_ERR_INVALID_ARG, "B = %d, n_q = %d, world = %d must be >= 1", B, n_q, world);
    if (!ws_bytes) return fail(SQZ_ERR_INVALID_ARG, "ws_bytes is NULL");
    *ws_bytes = lookup_carve(idx, B, n_q, nullptr, world).bytes + 256;
    return SQZ_OK;
}

int sqz_centroid_lookup(const sqz_index *idx, const void *Q, int32_t B, int32_t n_q,
                        const sqz_lookup_params *p, const sqz_selection *out, void *ws,
                        size_t ws_bytes, void *stream) {
    int rc = lookup_check(idx, Q, B, n_q, p, out, ws);
    if (rc) return rc;
    const int world = p->comm ? comm_world(p->comm) : 0;
    LookupWs w = lookup_carve(idx, B, n_q, align_ws(ws), world);
    if (ws_bytes < w.bytes + 256)
        return fail(SQZ_ERR_INVALID_ARG, "ws_bytes = %zu < required %zu%s", ws_bytes, w.bytes + 256,
                    world ? " (size it with sqz_lookup_workspace_comm)" : "");
    LookupShape s{B, idx->H, n_q, idx->d, idx->dtype, p->scale};
    cudaStream_t st = (cudaStream_t)stream;
    lookup_levels(idx, p, out, w);
    if (world) {
        // sharded: stats -> all-gather -> fold + select, once per level
        const size_t cnt = (size_t)B * idx->H * n_q * 2;
        for (int stage = 0; stage <= idx->levels; ++stage) {
            rc = run_stage(idx, s, Q, w, stage, world, w.recv, w.send, st);
            if (rc) return rc;
            if (stage < idx->levels) {
                rc = comm_allgather_f32(p->comm, reinterpret_cast<const float *>(w.send),
                                        reinterpret_cast<float *>(w.recv), cnt, st);
                if (rc) return rc;
            }
        }
        return SQZ_OK;
    }
    if (idx->levels == 2 && n_q == 1) {
        // decode: Level 2 expands its slice of the candidate rows from the Level-1
        // survivors (run-length) in shared memory; no candidate list is written
        w.l1.exp_list = nullptr;
        w.l2.rl_list = w.l1.list;
        w.l2.rl_pref = w.l1.sel_pref;
        w.l2.rl_off = idx->child_off;
        w.l2.rl_n = w.l1.n_list;
        w.l2.rl_c = idx->c1;
    }
    if (idx->levels == 3) {
        cudaError_t e = launch_lookup_level(s, Q, w.l0, st);
        if (e != cudaSuccess) return cuda_fail(e, "lookup level 0");
    }
    if (idx->levels >= 2) {
        cudaError_t e = launch_lookup_level(s, Q, w.l1, st);
        if (e != cudaSuccess) return cuda_fail(e, "lookup level 1");
    }
    cudaError_t e = launch_lookup_level(s, Q, w.l2, st);
    if (e != cudaSuccess) return cuda_fail(e, "lookup level 2");
    return SQZ_OK;
}

int sqz_centroid_lookup_stage(const sqz_index *idx, const void *Q, int32_t B, int32_t n_q,
                              const sqz_lookup_params *p, int32_t stage, int32_t P,
                              const float *stats_in, float *stats_out, const sqz_selection *out,
                              void *ws, size_t ws_bytes, void *stream) {
    int rc = lookup_check(idx, Q, B, n_q, p, out, ws);
    if (rc) return rc;
    if (idx->levels == 3) return fail(SQZ_ERR_UNSUPPORTED, "staged lookup of a three-level index");
    if (stage < 0 || stage > idx->levels)
        return fail(SQZ_ERR_INVALID_ARG, "stage = %d must be in [0, levels=%d]", stage, idx->levels);
    if (stage > 0 && (P < 1 || !stats_in))
        return fail(SQZ_ERR_INVALID_ARG, "stage %d needs P >= 1 and stats_in", stage);
    if (stage < idx->levels && !stats_out)
        return fail(SQZ_ERR_INVALID_ARG, "stage %d needs stats_out", stage);
    LookupWs w = lookup_carve(idx, B, n_q, align_ws(ws));
    if (ws_bytes < w.bytes + 256)
        return fail(SQZ_ERR_INVALID_ARG, "ws_bytes = %zu < required %zu", ws_bytes, w.bytes + 256);
    LookupShape s{B, idx->H, n_q, idx->d, idx->dtype, p->scale};
    lookup_levels(idx, p, out, w);
    return run_stage(idx, s, Q, w, stage, P, reinterpret_cast<const float2 *>(stats_in),
                     reinterpret_cast<float2 *>(stats_out), (cudaStream_t)stream);
}

// ------------------------------------------------------------------ attention
int sqz_attention_workspace(const sqz_index *idx, int32_t B, int32_t n_q, int32_t n_u,
                            size_t *ws_bytes) {
    int rc = check_index(idx, false);
    if (rc) return rc;
    if (B < 1 || n_q < 1 || n_u < 0)
        return fail(SQZ_ERR_INVALID_ARG, "B=%d, n_q=%d must be >= 1 and n_u=%d >= 0", B, n_q, n_u);
    if (!ws_bytes) return fail(SQZ_ERR_INVALID_ARG, "ws_bytes is NULL");
    *ws_bytes = attn_carve(idx, B, n_q, n_u, nullptr).bytes + 256;
    return SQZ_OK;
}

int sqz_sparse_attention(const void *Q, int32_t B, int32_t n_q, const void *Kp, const void *Vp,
                         const sqz_index *idx, const sqz_selection *sel, const void *Ku,
                         const void *Vu, int32_t n_u, const sqz_attn_params *p, void *O,
                         float *LSE, void *ws, size_t ws_bytes, void *stream) {
    int rc = check_index(idx, false);
    if (rc) return rc;
    if (!Q || !Kp || !Vp) return fail(SQZ_ERR_INVALID_ARG, "Q, Kp, Vp must be non-NULL");
    if (!aligned16(Q) || !aligned16(Kp) || !aligned16(Vp))
        return fail(SQZ_ERR_INVALID_ARG, "Q, Kp, Vp must be 16-byte aligned");
    if (B < 1 || n_q < 1 || n_u < 0)
        return fail(SQZ_ERR_INVALID_ARG, "B=%d, n_q=%d must be >= 1 and n_u=%d >= 0", B, n_q, n_u);
    if (n_u > 0 && (!Ku || !Vu)) return fail(SQZ_ERR_INVALID_ARG, "Ku, Vu required when n_u > 0");
    if (n_u > 0 && (!aligned16(Ku) || !aligned16(Vu)))
        return fail(SQZ_ERR_INVALID_ARG, "Ku, Vu must be 16-byte aligned");
    if (!sel || !sel->n_keys ||
        (!sel->key_idx && (!sel->clusters || !sel->n_clusters || !sel->key_pref || !idx->key_off)))
        return fail(SQZ_ERR_INVALID_ARG,
                    "sel->n_keys and either sel->key_idx or (sel->clusters, n_clusters, key_pref, "
                    "idx->key_off) are required");
    if (!p) return fail(SQZ_ERR_INVALID_ARG, "params is NULL");
    if (p->out_dtype != SQZ_F32 && p->out_dtype != SQZ_BF16)
        return fail(SQZ_ERR_INVALID_ARG, "out_dtype = %d is not a sqz_dtype", p->out_dtype);
    if (!std::isfinite(p->scale)) return fail(SQZ_ERR_INVALID_ARG, "scale must be finite");
    if (!O || !LSE) return fail(SQZ_ERR_INVALID_ARG, "O and LSE must be non-NULL");
    if (!ws) return fail(SQZ_ERR_INVALID_ARG, "ws is NULL");
    AttnWs w = attn_carve(idx, B, n_q, n_u, align_ws(ws));
    if (ws_bytes < w.bytes + 256)
        return fail(SQZ_ERR_INVALID_ARG, "ws_bytes = %zu < required %zu", ws_bytes, w.bytes + 256);
    AttnArgs a;
    std::memset(&a, 0, sizeof(a));
    a.Q = Q; a.Kp = Kp; a.Vp = Vp; a.Ku = Ku; a.Vu = Vu;
    a.n_keys = sel->n_keys; a.key_idx = sel->key_idx;
    a.sel_cl = sel->clusters; a.sel_pref = sel->key_pref; a.sel_n = sel->n_clusters;
    a.key_off = idx->key_off; a.c2 = idx->c2;
    a.B = B; a.H = idx->H; a.n_q = n_q; a.n_u = n_u; a.d = idx->d; a.dtype = idx->dtype;
    a.causal = p->causal ? 1 : 0; a.partial = p->partial ? 1 : 0; a.out_dtype = p->out_dtype;
    a.L = idx->L; a.scale = p->scale;
    a.kch = w.kch; a.max_chunks = w.max_chunks;
    a.part_o = w.part_o; a.part_lse = w.part_lse; a.status = w.status; a.row_cnt = w.row_cnt;
    a.sched = w.status + 1;
    a.cut = w.cut;
    a.O = O; a.LSE = LSE;
    a.shared_ws = w.shared;
    a.N2 = idx->N2;
    cudaError_t e;
    if (w.shared && !p->per_row && sel->clusters && sel->n_clusters && idx->N2 && idx->key_off)
        e = launch_attention_shared(a, (cudaStream_t)stream);
    else
        e = launch_attention(a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "sparse attention launch");
    return SQZ_OK;
}

// ------------------------------------------------------------------ decode step
// workspace regions: [attention | user chunks | lookup].  The attention region
// comes first so that its status word sits where sqz_attention_status(ws)
// reads it.  The user-chunk region holds the partials of the user KV the
// attention kernel attends before it waits for the lookup ([B*H, n_chunks, d]
// + [B*H, n_chunks] fp32).
static int user_chunks(int n_u) { return (n_u + attention_user_chunk() - 1) / attention_user_chunk(); }
static size_t user_region_bytes(const sqz_index *idx, int B, int n_u) {
    const size_t BH = (size_t)B * idx->H, nch = (size_t)user_chunks(n_u);
    return (BH * nch * (idx->d + 1) * sizeof(float) + 255) & ~(size_t)255;
}

int sqz_decode_step_workspace(const sqz_index *idx, int32_t B, int32_t n_u, size_t *ws_bytes) {
    int rc = check_index(idx, false);
    if (rc) return rc;
    if (B < 1 || n_u < 0) return fail(SQZ_ERR_INVALID_ARG, "B = %d must be >= 1 and n_u = %d >= 0", B, n_u);
    if (!ws_bytes) return fail(SQZ_ERR_INVALID_ARG, "ws_bytes is NULL");
    *ws_bytes = 256 + ((attn_carve(idx, B, 1, n_u, nullptr).bytes + 511) & ~(size_t)255) +
                user_region_bytes(idx, B, n_u) + ((lookup_carve(idx, B, 1, nullptr).bytes + 511) & ~(size_t)255);
    return SQZ_OK;
}

int sqz_decode_step(const sqz_index *idx, const void *Q, int32_t B, const void *Kp, const void *Vp,
                    const void *Ku, const void *Vu, int32_t n_u, const sqz_lookup_params *lp,
                    const sqz_attn_params *ap, const sqz_selection *sel, void *O, float *LSE,
                    void *ws, size_t ws_bytes, void *stream) {
    int rc = lookup_check(idx, Q, B, 1, lp, sel, ws);
    if (rc) return rc;
    if (lp->comm) return fail(SQZ_ERR_INVALID_ARG, "sqz_decode_step: lp->comm must be NULL (use the two calls)");
    if (!ap) return fail(SQZ_ERR_INVALID_ARG, "attention params is NULL");
    if (!Kp || !Vp || !aligned16(Kp) || !aligned16(Vp))
        return fail(SQZ_ERR_INVALID_ARG, "Kp, Vp must be non-NULL and 16-byte aligned");
    if (n_u < 0 || (n_u > 0 && (!Ku || !Vu || !aligned16(Ku) || !aligned16(Vu))))
        return fail(SQZ_ERR_INVALID_ARG, "n_u = %d: Ku, Vu must be non-NULL and 16-byte aligned", n_u);
    if (ap->out_dtype != SQZ_F32 && ap->out_dtype != SQZ_BF16)
        return fail(SQZ_ERR_INVALID_ARG, "out_dtype = %d is not a sqz_dtype", ap->out_dtype);
    if (!O || !LSE) return fail(SQZ_ERR_INVALID_ARG, "O and LSE must be non-NULL");
    if (!sel->n_keys || !sel->clusters || !sel->n_clusters || !sel->key_pref)
        return fail(SQZ_ERR_INVALID_ARG, "sel->clusters, n_clusters, n_keys, key_pref are required");
    size_t need = 0;
    sqz_decode_step_workspace(idx, B, n_u, &need);
    if (ws_bytes < need) return fail(SQZ_ERR_INVALID_ARG, "ws_bytes = %zu < required %zu", ws_bytes, need);
    char *base = align_ws(ws);
    const size_t attn_b = (attn_carve(idx, B, 1, n_u, nullptr).bytes + 511) & ~(size_t)255;
    char *user_ws = base + attn_b;
    char *look_ws = user_ws + user_region_bytes(idx, B, n_u);
    const size_t look_b = (lookup_carve(idx, B, 1, nullptr).bytes + 511) & ~(size_t)255;
    const bool debug = sel->dbg_S || sel->dbg_S1 || sel->dbg_lse || sel->l1_surv || sel->dbg_S0 ||
                       sel->l0_surv;
    cudaStream_t st = (cudaStream_t)stream;
    const long long H = idx->H;
    // One query row, single level, unsharded: the lookup kernel is limited to
    // 84 registers (two of its CTAs leave room for an attention CTA on the SM),
    // and the attention kernel -- launched behind it -- attends the
    // selection-independent user KV in chunks on those early CTAs before it
    // waits for the lookup; the chunks' partials join each row's merge.
    if (idx->levels == 1 && B == 1 && !debug && idx->L_total == 0 && n_u > 0 &&
        H * (idx->L + n_u + 1024) < 0x7fffffffLL && H <= 8192) {
        static const bool no_user = std::getenv("SQZ_STEP_NO_USER") != nullptr;  // A/B knob
        const size_t BH = (size_t)B * H;
        const int nch = no_user ? 0 : user_chunks(n_u);
        float *up_o = reinterpret_cast<float *>(user_ws);
        float *up_lse = up_o + BH * nch * idx->d;
        LookupWs w = lookup_carve(idx, B, 1, look_ws);
        LookupShape s{B, idx->H, 1, idx->d, idx->dtype, lp->scale};
        lookup_levels(idx, lp, sel, w);
        w.l2.lean = 1;
        cudaError_t e = launch_lookup_level(s, Q, w.l2, st);
        if (e != cudaSuccess) return cuda_fail(e, "decode step lookup");
        AttnWs aw = attn_carve(idx, B, 1, n_u, base);
        AttnArgs a;
        std::memset(&a, 0, sizeof(a));
        a.Q = Q; a.Kp = Kp; a.Vp = Vp; a.Ku = Ku; a.Vu = Vu;
        a.n_keys = sel->n_keys; a.key_idx = sel->key_idx;
        a.sel_cl = sel->clusters; a.sel_pref = sel->key_pref; a.sel_n = sel->n_clusters;
        a.key_off = idx->key_off; a.c2 = idx->c2;
        a.B = B; a.H = idx->H; a.n_q = 1; a.n_u = n_u; a.d = idx->d; a.dtype = idx->dtype;
        a.causal = 0; a.partial = ap->partial ? 1 : 0; a.out_dtype = ap->out_dtype;
        a.L = idx->L; a.scale = ap->scale;
        a.kch = aw.kch; a.max_chunks = aw.max_chunks;
        a.part_o = aw.part_o; a.part_lse = aw.part_lse; a.status = aw.status; a.row_cnt = aw.row_cnt;
        a.sched = aw.status + 1;
        a.cut = aw.cut;
        a.O = O; a.LSE = LSE;
        if (nch > 0) {
            a.up_o = up_o; a.up_lse = up_lse;
            a.up_n = nch;
        }
        e = launch_attention(a, st);
        if (e != cudaSuccess) return cuda_fail(e, "decode step attention");
        return SQZ_OK;
    }
    // the two calls, on sub-workspaces of this one
    rc = sqz_centroid_lookup(idx, Q, B, 1, lp, sel, look_ws, look_b, stream);
    if (rc) return rc;
    return sqz_sparse_attention(Q, B, 1, Kp, Vp, idx, sel, Ku, Vu, n_u, ap, O, LSE, base, attn_b, stream);
}

int sqz_attention_status(void *ws, size_t ws_bytes, void *stream) {
    if (!ws || ws_bytes < 512) return fail(SQZ_ERR_INVALID_ARG, "ws too small");
    int32_t *status = reinterpret_cast<int32_t *>(align_ws(ws));
    int32_t h = 0;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemcpyAsync(&h, status, sizeof(h), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(status, 0, sizeof(h), st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "attention status");
    if (h) return fail(SQZ_ERR_EMPTY, "a final output row attended no key (S:351-353)");
    return SQZ_OK;
}

int sqz_merge_partials(int32_t P, const float *O_parts, const float *LSE_parts, int64_t rows,
                       int32_t d, void *O, float *LSE, int32_t out_dtype, void *stream) {
    if (P < 1 || rows < 0 || d < 1)
        return fail(SQZ_ERR_INVALID_ARG, "P=%d >= 1, rows=%lld >= 0, d=%d >= 1 required", P,
                    (long long)rows, d);
    if (!O_parts || !LSE_parts || !O || !LSE)
        return fail(SQZ_ERR_INVALID_ARG, "O_parts, LSE_parts, O, LSE must be non-NULL");
    if (out_dtype != SQZ_F32 && out_dtype != SQZ_BF16)
        return fail(SQZ_ERR_INVALID_ARG, "out_dtype = %d is not a sqz_dtype", out_dtype);
    if (rows > 0x7fffffffLL) return fail(SQZ_ERR_UNSUPPORTED, "rows must be < 2^31");
    cudaError_t e = launch_merge(P, O_parts, LSE_parts, rows, d, O, LSE, out_dtype, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "merge launch");
    return SQZ_OK;
}

// ------------------------------------------------------------------ diagnostics
int sqz_selection_diagnostics_workspace(const sqz_index *idx, int32_t B, size_t *ws_bytes) {
    int rc = check_index(idx, false);
    if (rc) return rc;
    if (B < 1) return fail(SQZ_ERR_INVALID_ARG, "B = %d must be >= 1", B);
    if (!ws_bytes) return fail(SQZ_ERR_INVALID_ARG, "ws_bytes is NULL");
    *ws_bytes = diag_ws_bytes(B, idx->H, idx->c2, idx->L) + 256;
    return SQZ_OK;
}

int sqz_selection_diagnostics(const sqz_index *idx, const void *Q, int32_t B, const void *Kp,
                              const sqz_selection *sel, float scale, double top_frac, float T,
                              const sqz_diagnostics *out, void *ws, size_t ws_bytes, void *stream) {
    int rc = check_index(idx, true);
    if (rc) return rc;
    if (idx->L_total != 0) return fail(SQZ_ERR_INVALID_ARG, "diagnostics need an unsharded index");
    if (!Q || !Kp) return fail(SQZ_ERR_INVALID_ARG, "Q and Kp must be non-NULL");
    if (!aligned16(Q) || !aligned16(Kp)) return fail(SQZ_ERR_INVALID_ARG, "Q, Kp must be 16-byte aligned");
    if (B < 1) return fail(SQZ_ERR_INVALID_ARG, "B = %d must be >= 1", B);
    if (!sel || !sel->clusters || !sel->n_clusters || !sel->n_keys)
        return fail(SQZ_ERR_INVALID_ARG, "sel->clusters / n_clusters / n_keys required");
    if (!(top_frac > 0.0 && top_frac <= 1.0))
        return fail(SQZ_ERR_INVALID_ARG, "top_frac = %g must be in (0, 1]", top_frac);
    if (!(T >= 0.f) || std::isinf(T))
        return fail(SQZ_ERR_INVALID_ARG, "T = %g must be finite and >= 0", (double)T);
    if (!std::isfinite(scale)) return fail(SQZ_ERR_INVALID_ARG, "scale must be finite");
    if (!out || !out->skew || !out->mass_sel || !out->mass_ideal || !out->recall || !out->n_T ||
        !out->mass_T)
        return fail(SQZ_ERR_INVALID_ARG, "every sqz_diagnostics output is required");
    const size_t need = diag_ws_bytes(B, idx->H, idx->c2, idx->L);
    if (!ws || ws_bytes < need) return fail(SQZ_ERR_INVALID_ARG, "ws too small (need %zu bytes)", need);
    DiagLaunch a;
    std::memset(&a, 0, sizeof(a));
    a.Q = Q;
    a.Kp = Kp;
    a.key_off = idx->key_off;
    a.clusters = sel->clusters;
    a.n_clusters = sel->n_clusters;
    a.n_keys = sel->n_keys;
    a.B = B;
    a.H = idx->H;
    a.c2 = idx->c2;
    a.d = idx->d;
    a.dtype = idx->dtype;
    a.L = idx->L;
    a.scale = scale;
    a.T = T;
    const long long nt = (long long)std::ceil(top_frac * (double)idx->L);
    a.n_top = nt < 1 ? 1 : (nt > idx->L ? idx->L : nt);
    a.ws = ws;
    a.skew = out->skew;
    a.mass_sel = out->mass_sel;
    a.mass_ideal = out->mass_ideal;
    a.recall = out->recall;
    a.n_T = out->n_T;
    a.mass_T = out->mass_T;
    cudaError_t e = launch_diagnostics(a, (cudaStream_t)stream);
    return e == cudaSuccess ? SQZ_OK : cuda_fail(e, "diagnostics launch");
}


}  // extern "C"
