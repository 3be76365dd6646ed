// internal.h -- launcher interfaces between the C-ABI layer (api.cu) and the
// kernel translation units.  Not part of the public ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sqz.h"

namespace sqz {

// api.cu: records the thread-local sqz_last_error() message; returns `code`
int set_error(int code, const char *fmt, ...);
// dist.cu: communicator helpers (comm = sqz_comm_init handle)
int comm_world(void *comm);
int comm_allgather_f32(void *comm, const float *send, float *recv, size_t count, cudaStream_t st);

// One lookup level (Eq. 1 single level, or Eq. 2 / Eq. 3 of the hierarchy).
struct LevelArgs {
    const void *C;        // [H, c, d] centroid table of this level
    const int32_t *N;     // [H, c] Eq.1 weights N_i (descendant keys for Level 1, R4)
    const int32_t *off;   // [H, c+1] expansion ranges (key_off or child_off)
    int32_t c;            // rows in this level's table
    float T;              // threshold for this level
    // row space: all c rows, or the per-(b,h) candidate list rows[b,h,0..n_rows)
    const int32_t *rows;  // [B,H,row_stride] or null
    const int32_t *n_rows;
    int32_t row_stride;
    // scratch
    float *logits;        // [B,H,c]           (decode)
    float2 *part;         // [B,H,nch] (m, D)  (decode)
    int32_t *tick;        // [B*H] self-cleaning tickets
    int32_t *sel_pref;    // [B,H,c] prefix of expanded counts over the selected list
    float *rowlse;        // [B,H,n_q]         (prefill)
    float *colpart;       // [nqt,B,H,c]       (prefill)
    // outputs
    int32_t *list;        // [B,H,c] ascending selected row ids
    int32_t *n_list;      // [B,H]
    int32_t *exp_list;    // [B,H,exp_stride] expanded positions (keys or Level-2 rows)
    int32_t *n_exp;       // [B,H]
    int64_t exp_stride;
    uint8_t *bitmap;      // optional [B,H,c]
    float *dbg_S;         // optional [B,H,c]
    float *dbg_lse;       // optional [B,H,n_q]
    // staged lookup over fixed-context shards (sqz_centroid_lookup_stage)
    int32_t phase;        // 0: scan + threshold; 1: scan -> stats_out only; 2: threshold
                          //    with the folded global statistics gstat (decode reuses the
                          //    logits phase 1 stored, prefill recomputes them)
    float2 *stats_out;    // [B,H,n_q] (m, D) of this shard's rows        (phase 1)
    const float2 *gstat;  // [B,H,n_q] (M, log D) folded over the shards  (phase 2)
    // decode Level 2: the candidate rows in run-length form (the parent level's
    // ascending survivor list and its child-count prefix) instead of a
    // materialised list; the kernel expands its own slice in shared memory
    const int32_t *rl_list, *rl_pref, *rl_off;  // [B,H,rl_c], [B,H,rl_c], [H,rl_c+1]
    const int32_t *rl_n;                        // [B,H] survivors
    int32_t rl_c;
    // bf16 prefill with a candidate list and many query tiles: the candidate
    // rows gathered contiguously per (b,h), [B*H][c][d] (TMA-loaded)
    void *cgather;
    // decode step (sqz_decode_step): the kernel variant limited to 84 registers
    // (3 CTAs' worth per SM), so that an attention CTA fits beside two of them
    int32_t lean;
};

struct LookupShape {
    int32_t B, H, n_q, d, dtype;
    float scale;
};

// lookup.cu
cudaError_t launch_lookup_level(const LookupShape &s, const void *Q, const LevelArgs &lv,
                                cudaStream_t st);
// fold of P shards' (m, D) statistics in rank order -> (M, log D); also
// M + log D into rowlse when non-null (prefill)
cudaError_t launch_fold_stats(int P, const float2 *stats_in, int64_t n, float2 *gstat,
                              float *rowlse, cudaStream_t st);
int lookup_chunk_rows();
int lookup_qtile();

// attention.cu
struct AttnArgs {
    const void *Q, *Kp, *Vp, *Ku, *Vu;
    const int32_t *n_keys, *key_idx;
    // run-length selection (sqz_selection.key_pref): used when key_idx is null
    const int32_t *sel_cl, *sel_pref, *sel_n, *key_off;
    int32_t c2;
    int32_t B, H, n_q, n_u, d, dtype, causal, partial, out_dtype;
    int64_t L;
    float scale;
    int32_t kch, max_chunks;
    float *part_o;    // [rows, max_chunks, d]
    float *part_lse;  // [rows, max_chunks]
    int32_t *status;  // [1]
    int32_t *row_cnt; // [rows] self-cleaning tile tickets
    int32_t *sched;   // [2] dynamic tile counter + finished-CTA counter (self-cleaning)
    int32_t *cut;     // [3 * 1024] cut-segment slots of the persistent prefill kernel (one per CTA)
    void *O;
    float *LSE;
    // batch-shared decode (shared_attn.cu): its workspace region and the N2 table
    void *shared_ws;
    const int32_t *N2;
    // decode step (sqz_decode_step): the user KV is attended BEFORE the wait for
    // the lookup, in USER_CHUNK-key chunks spread statically over the first
    // up_ctas CTAs (resident beside the lookup's CTAs); chunk j of row r leaves
    // its partial at up_o [rows, up_n, d] / up_lse [rows, up_n] and adds 1 << 16
    // to the row's ticket word row_cnt[r] (its merger waits for up_n of them).
    // Null up_o: the user keys are part of the rows' streams.
    float *up_o, *up_lse;
    int32_t up_n, up_ctas;
    // persistent decode grid: no tickets -- the CTA holding a row's first segment
    // stores the row's partial count in row_cnt[r], and k_merge_rows (launched
    // behind the attention kernel) merges every row after the whole grid is done
    // (set by the launcher)
    int32_t merge_kernel;
};
cudaError_t launch_attention(const AttnArgs &a, cudaStream_t st);
// shared_attn.cu: batch-shared decode attention over the per-head union of the
// B selections (NEXT-1)
bool shared_attn_applies(int B, int n_q, int d, int dtype, int c2);
size_t shared_attn_ws_bytes(int B, int H, int c2);
cudaError_t launch_attention_shared(const AttnArgs &a, cudaStream_t st);
// prefill_attn.cu: tcgen05 path for bf16 prefill (n_q > 1)
cudaError_t launch_prefill_attention(const AttnArgs &a, cudaStream_t st);
cudaError_t launch_prefill_attention_ws(const AttnArgs &a, cudaStream_t st);  // d = 128
bool prefill_ws_applies(int d, int dtype, int n_q);       // routes to the persistent kernel
size_t prefill_ws_part_rows(int B, int H, int n_q);       // its partial-buffer rows
int prefill_split_keys();
int attention_kch(int n_q);
int attention_user_chunk();  // decode step: user keys per pre-wait chunk
int attention_max_parts(int64_t L, int n_u, int n_q);
cudaError_t launch_merge(int P, const float *O_parts, const float *LSE_parts, int64_t rows, int d,
                         void *O, float *LSE, int out_dtype, cudaStream_t st);

// diag.cu: App. A skewness + App. D ideal-lookup diagnostics (NEXT-4)
struct DiagLaunch {
    const void *Q, *Kp;
    const int32_t *key_off, *clusters, *n_clusters, *n_keys;
    int32_t B, H, c2, d, dtype;
    int64_t L;
    float scale, T;
    long long n_top;
    void *ws;
    float *skew, *mass_sel, *mass_ideal, *recall, *mass_T;
    int32_t *n_T;
};
size_t diag_ws_bytes(int B, int H, int c2, int64_t L);
cudaError_t launch_diagnostics(const DiagLaunch &a, cudaStream_t st);

// kmeans_tc.cu: tensor-core assignment step of the Lloyd iterations (NEXT-3)
struct KmeansTcWs {
    int *amb_n;     // ambiguous-key count
    float *xx;      // [H, n] ||x^||^2 (sequential FMA)
    int4 *amb;      // [H * n] (h, key, best, second) of the keys re-ranked exactly
    void *Xs, *Ms;  // [H, n, 2d], [H, c, 2d] bf16 splits [hi | lo]
};
struct KmeansTc {
    int H, n, c, d;
    const float *Xh, *mu, *musq;
    const int *done;
    int32_t *assign;
    float *pdist;
    int *changed;
    float margin;
    KmeansTcWs w;
};
size_t kmeans_tc_ws_bytes(int H, int64_t n, int64_t c, int d);
bool kmeans_tc_applies(int mode, int d, int64_t n, int64_t c);
KmeansTcWs kmeans_tc_carve(void *ws, int H, int64_t n, int d);
cudaError_t kmeans_tc_split_x(const float *Xh, int H, int n, int d, const KmeansTcWs &w, cudaStream_t st);
cudaError_t kmeans_tc_assign(const KmeansTc &k, cudaStream_t st);

// kmeans.cu
struct KmeansWs;
size_t kmeans_workspace_bytes(const sqz_index &idx);
int cluster_keys(const void *K, const void *V, const int64_t *init2, const int64_t *init1,
                 sqz_index *idx, void *Kp, void *Vp, const sqz_kmeans_params &p, void *ws,
                 size_t ws_bytes, int32_t *iters_out, cudaStream_t st, char *err, size_t errlen);
size_t validate_workspace_bytes(const sqz_index &idx);
int index_validate(const sqz_index &idx, void *ws, size_t ws_bytes, cudaStream_t st, char *err,
                   size_t errlen);

// tmap.cu: TMA tensor map of a contiguous bf16 [dims2][dims1][dims0] tensor
// (128-byte swizzle, zero out-of-bounds fill); 0 on success
int encode_tmap_bf16_3d(CUtensorMap *m, const void *ptr, const uint64_t dims[3], const uint32_t box[3]);
int encode_tmap_bf16_2d(CUtensorMap *m, const void *ptr, uint64_t cols, uint64_t rows, uint32_t box_cols,
                        uint32_t box_rows);
// tmap.cu: per-device launch caches (keyed by device ordinal and kernel, mutex
// guarded): SM count of the current device; sets a function attribute once per
// (device, kernel) -- for cudaFuncAttributeMaxDynamicSharedMemorySize only when
// `value` exceeds the largest opt-in set so far; cached occupancy.
int device_sm_count();
cudaError_t ensure_func_attr(const void *kern, cudaFuncAttribute attr, int value);
int occupancy_blocks(const void *kern, int threads, size_t smem);

// shard.cu: gathers of the shard index rows
cudaError_t launch_shard_gather(const sqz_index &full, const void *Kp, const void *Vp,
                                const int32_t *c1_src, const int32_t *c2_src,
                                const int32_t *key_src, const sqz_index &local, void *Kp_loc,
                                void *Vp_loc, cudaStream_t st);

}  // namespace sqz
