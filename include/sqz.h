/*
 * sqz.h -- C ABI of libsqz.so, the B200-native (sm_100a) hot path of
 * Squeezed Attention (Hooper et al., arXiv 2411.09688).
 *
 * Citations: "P:n" = line n of the paper's LaTeX source; readings R<k> are
 * listed in DESIGN.md.  The online path is two steps:
 *   1. sqz_centroid_lookup  -- Eq. 1-3 centroid scoring + global threshold
 *       -> per-(b,h) selected clusters and the "tensor
 *      of key indices that need to be selectively loaded";
 *   2. sqz_sparse_attention -- exact attention over the selected fixed-context
 *      keys plus the dense user KV, split-KV with a merge.
 * sqz_cluster_keys is the offline step.
 *
 * Conventions (all entry points)
 *   - Every tensor argument is CALLER-OWNED DEVICE memory (cudaMalloc /
 *     torch), row-major with the last dimension contiguous; strides are
 *     implied by the shapes given.  The library never allocates device memory
 *     and never copies to the host on the online path.
 *   - Per-head tables are laid out [H, ...]; queries and user KV [B, H, ...].
 *   - "stream" is a cudaStream_t passed as void*; every online call only
 *     enqueues work on it (no host synchronisation).
 *   - Scratch: every call that needs scratch takes (ws, ws_bytes); the size is
 *     given by the matching *_workspace() query.  Workspaces must be zeroed
 *     ONCE before first use (sqz_workspace_init); the library leaves its
 *     counters zeroed again when each call completes, so a workspace can be
 *     reused by consecutive calls with the SAME geometry (B, n_q, n_u and
 *     index shape) on the same stream (not concurrently); re-zero it before
 *     using it with another geometry.
 *   - Return codes: SQZ_OK, or an error code; sqz_last_error() returns a
 *     thread-local message naming the offending argument.  Argument errors
 *     are detected on the host before anything is enqueued.
 */
#ifndef SQZ_H
#define SQZ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SQZ_ABI_VERSION 6

enum {
    SQZ_OK = 0,
    SQZ_ERR_INVALID_ARG = 2, /* shape / dtype / nullptr / T < 0 or NaN / c > L          */
    SQZ_ERR_FORMAT = 3,      /* malformed index tables                                   */
    SQZ_ERR_INVARIANT = 4,   /* tables violate sum N = L, perm not a permutation, ...    */
    SQZ_ERR_CUDA = 5,        /* a CUDA runtime call failed (message has the CUDA error)  */
    SQZ_ERR_NCCL = 6,        /* NCCL missing or a collective failed (message has why)     */
    SQZ_ERR_EMPTY = 7,       /* a final (non-partial) output row attended no key         */
    SQZ_ERR_UNSUPPORTED = 8  /* valid but not supported by this build (e.g. d not 64/128) */
};

typedef enum { SQZ_F32 = 0, SQZ_BF16 = 1 } sqz_dtype;

/* ---------------------------------------------------------------------- */
/* Index: per-head centroid tables and the cluster-major key layout (D1-D4) */
/* ---------------------------------------------------------------------- */
/* The fixed-context K/V are stored permuted into cluster-major order: the
 * keys of Level-2 cluster i occupy positions [key_off[h][i], key_off[h][i+1])
 * of Kp[h] / Vp[h], and perm[h][pos] is the original key index of position
 * pos.  This is legal because fixed-context keys are all visible to every
 * query (no causal mask within the fixed context), so attention is
 * permutation-invariant over them.  With two levels, Level-2 clusters are
 * numbered grouped by their Level-1 parent: the children of Level-1 cluster p
 * are Level-2 ids [child_off[h][p], child_off[h][p+1]).
 *
 *   field      shape        type              meaning
 *   C2         [H, c2, d]   dtype             Level-2 (finest) centroids C_i (R2)
 *   N2         [H, c2]      int32             keys per Level-2 cluster, N_i (Eq. 1)
 *   key_off    [H, c2 + 1]  int32             cluster-major key ranges
 *   perm       [H, L]       int32             position -> original key index
 *   C1         [H, c1, d]   dtype             Level-1 centroids (levels == 2)
 *   N1         [H, c1]      int32             descendant keys of each Level-1 cluster (R4)
 *   child_off  [H, c1 + 1]  int32             Level-2 children ranges (levels == 2)
 * Single level: levels = 1, c1 = 0, C1/N1/child_off = NULL.  Three levels
 * (levels = 3) add Level 0 above Level 1 (fields c0, C0, N0, child_off0).
 *
 * Fixed-context shards (cluster sharding across GPUs): a shard
 * index (sqz_shard_plan + sqz_index_shard) holds a subset of the clusters of
 * every head.  Then L_total = the global keys per head (perm values index the
 * ORIGINAL key space [0, L_total)), L = the shard's row capacity of Kp/Vp/perm
 * (>= its keys in every head), and sum_i N2[h][i] = key_off[h][c2] <= L; rows
 * past key_off[h][c2] are padding that no call reads.  L_total = 0 means an
 * unsharded index (L_total == L, sum N2 = L). */
typedef struct {
    int32_t H;       /* heads                                  */
    int32_t d;       /* head dimension: 64 or 128              */
    int64_t L;       /* fixed-context keys per head            */
    int32_t levels;  /* 1, 2 or 3                              */
    int32_t c1;      /* Level-1 clusters (0 when levels == 1)  */
    int32_t c2;      /* Level-2 / single-level clusters        */
    int32_t dtype;   /* sqz_dtype of C1, C2 (and of K, V, Q)   */
    void *C1;
    int32_t *N1;
    int32_t *child_off;
    void *C2;
    int32_t *N2;
    int32_t *key_off;
    int32_t *perm;
    int64_t L_total; /* 0: unsharded; else global keys per head (see above) */
    /* levels == 3 ("extended to multiple levels"): Level 0 above Level 1,
     * its children contiguous Level-1 ids (Level-1 ids are grouped by parent):
     *   C0 [H, c0, d] dtype, N0 [H, c0] descendant keys, child_off0 [H, c0 + 1] */
    int32_t c0;
    void *C0;
    int32_t *N0;
    int32_t *child_off0;
} sqz_index;

/* ---------------------------------------------------------------------- */
/* Offline: K-means key clustering (section 3.1; section 3.3       */
/* P:244-247; Fig. 2)                                            */
/* ---------------------------------------------------------------------- */
enum { SQZ_KMEANS_AUTO = 0, SQZ_KMEANS_EXACT = 1, SQZ_KMEANS_TENSOR = 2 };
typedef struct {
    int32_t max_iters;   /* Lloyd iterations per level (e.g. 50)                       */
    float tol;           /* stop when the max centroid shift < tol (e.g. 1e-4)         */
    int32_t assign_mode; /* assignment step: SQZ_KMEANS_EXACT = fp32 FFMA scores;       */
                         /* SQZ_KMEANS_TENSOR = tcgen05 GEMM on split-bf16 operands     */
                         /* (x_h.mu_h + x_h.mu_l + x_l.mu_h, fp32 accumulation, ~fp32   */
                         /* FFMA accuracy) with an exact fp32 re-rank of every key     */
                         /* whose two best scores are within 2e-4; SQZ_KMEANS_AUTO (0) */
                         /* = TENSOR when keys x clusters >= 2^26 (d = 64 or 128)      */
    const int64_t *init0; /* levels == 3: [H, c0] device, the seeded initial subset  */
                          /* of the Level-1 centroids (K-means id order) for Level 0 */
} sqz_kmeans_params;

/* Workspace bytes for sqz_cluster_keys with the index geometry in *idx. */
int sqz_cluster_keys_workspace(const sqz_index *idx, size_t *ws_bytes);

/* Clusters the keys of every head and writes the index tables and the
 * cluster-major copies of K and V.
 *   K, V   [H, L, d] dtype, ORIGINAL key order (read only)
 *   init2  [H, c2] int64 device: seeded initial subset for Level 2 (R3)
 *   init1  [H, c1] int64 device: initial subset of the Level-2 centroids for
 *          Level 1 (levels == 2), else NULL
 *   idx    geometry fields (H, d, L, levels, c1, c2, dtype) set by the caller;
 *          every table pointer must point to caller-allocated device memory of
 *          the shape above; all tables are written.
 *   Kp, Vp [H, L, d] dtype outputs (cluster-major copies)
 *   iters_out optional HOST int32[2] (int32[3] when levels == 3): max Lloyd
 *          iterations over heads used by Level 2, Level 1 (and Level 0).
 * Algorithm: Lloyd on unit-normalised keys (assignment argmin ||x^ - mu||^2,
 * ties to the lowest id; farthest-point repair of empty clusters; update =
 * mean of member x^), then C_i = mean of the RAW member keys rounded once to
 * dtype; Level 1 clusters the stored C2 rows, C1 = unweighted mean of child
 * rows, N1 = descendant keys; levels == 3: Level 0 clusters the stored C1 rows
 * (init p->init0) the same way, and the Level-1 ids are renumbered grouped by
 * their Level-0 parent (stable) before the Level-2 ids are grouped by Level-1
 * parent.  This is the only call that synchronises the stream (once per Lloyd
 * iteration, to test convergence). */
int sqz_cluster_keys(const void *K, const void *V, const int64_t *init2, const int64_t *init1,
                     sqz_index *idx, void *Kp, void *Vp, const sqz_kmeans_params *p, void *ws,
                     size_t ws_bytes, int32_t *iters_out, void *stream);

/* Checks the index invariants on the device (sum N2 = L, key_off consistent
 * with N2, perm a permutation of [0, L), child_off a partition of [0, c2)
 * into NON-EMPTY child ranges for an unsharded index (K-means leaves no
 * cluster empty; the decode Level-2 lookup relies on it), N1 = descendant
 * keys).  Indexes built outside sqz_cluster_keys should be validated once.  Synchronises the stream.  SQZ_ERR_INVARIANT on
 * failure.  ws: sqz_index_validate_workspace() bytes. */
int sqz_index_validate_workspace(const sqz_index *idx, size_t *ws_bytes);
int sqz_index_validate(const sqz_index *idx, void *ws, size_t ws_bytes, void *stream);

/* Index persistence (ABI v6).  The offline clustering output is the artefact
 * built once per fixed context and reused online (S:100-103, S:115-123
 * name the magic and the round-trip property).  File: the 8 bytes "SQZIDX1\0",
 * u32 version = 1, nine little-endian i64 {H, d, L, levels, c0, c1, c2, dtype,
 * L_total}, then the tables' raw little-endian bytes in the device layout above,
 * in the order [C0, N0, child_off0] (levels 3), [C1, N1, child_off] (levels >= 2),
 * C2, N2, key_off, perm.  load(save(x)) == x bit for bit.
 *   sqz_index_save      copies the tables device -> host and writes `path`
 *                       (synchronises the stream).  SQZ_ERR_FORMAT: invalid
 *                       geometry; SQZ_ERR_INVALID_ARG: NULL table, I/O failure.
 *   sqz_index_file_info host only: reads and checks the header (magic, version,
 *                       geometry, payload size == the geometry's tables) and
 *                       fills the geometry fields of *geom (pointers NULL), so the
 *                       caller can allocate.  SQZ_ERR_FORMAT on any mismatch.
 *   sqz_index_load      copies the file's tables into the caller-allocated device
 *                       tables of *dst, whose geometry must equal the file's
 *                       (synchronises).  Run sqz_index_validate on the result
 *                       before trusting a file from elsewhere. */
int sqz_index_save(const sqz_index *idx, const char *path, void *stream);
int sqz_index_file_info(const char *path, sqz_index *geom);
int sqz_index_load(const char *path, const sqz_index *dst, void *stream);

/* ---------------------------------------------------------------------- */
/* Online step 1: centroid lookup (Eq. 1-3; section 4.1)          */
/* ---------------------------------------------------------------------- */
typedef struct {
    float scale; /* logit scale s_i = scale * q.C_i; 1/sqrt(d) default (R1)          */
    float T;     /* global threshold (finest level), T >= 0; T == 0 selects all (R6)  */
    float T1;    /* Level-1 threshold (levels == 2), T1 >= 0                         */
    void *comm;  /* NULL: idx is the whole fixed context.  Else an sqz_comm (see    */
                 /* "Multi-GPU") whose ranks each hold one shard of it: the lookup  */
                 /* exchanges the per-query (m, D) statistics of every level with   */
                 /* an all-gather so each rank thresholds against the GLOBAL Eq. 1  */
                 /* / Eq. 3 denominator and selects exactly the clusters the        */
                 /* unsharded lookup selects among its own (the workspace must then */
                 /* be sized by sqz_lookup_workspace_comm).                         */
    float T0;    /* Level-0 threshold (levels == 3), T0 >= 0                        */
} sqz_lookup_params;

/* Outputs of the lookup, caller-allocated device memory.
 *   clusters   [B, H, c2] int32: ascending selected finest-level cluster ids;
 *              the first n_clusters[b,h] entries are valid
 *   n_clusters [B, H] int32
 *   n_keys     [B, H] int32: k = sum of N_i over the selected clusters
 *   key_pref   [B, H, c2] int32: the key-index tensor of P:354 in run-length
 *              form: the selected keys are the runs [key_off[h][clusters[j]],
 *              + N) of Kp/Vp, and key_pref[j] = sum of N over clusters[0..j) is
 *              the first key of run j in the (b,h)'s selection stream.
 *              sqz_sparse_attention reads the runs (no O(k) index tensor).
 *   key_idx    optional [B, H, L] int32: the same selection expanded, one
 *              cluster-major position (into Kp/Vp) per selected key, ascending;
 *              the first n_keys[b,h] are valid.  NULL: not materialised.
 *   l1_surv    optional [B, H, c1] uint8: Level-1 survivors (levels == 2)
 *   dbg_S      optional [B, H, c2] fp32: finest-level S_i (decode) or S-bar_i
 *              (prefill) as the kernel evaluated it, NaN for rows not scanned
 *   dbg_S1     optional [B, H, c1] fp32: Level-1 S^(1) / S-bar^(1)
 *   dbg_lse    optional [B, H, n_q] fp32: finest-level log denominator per query
 *              (log sum_j N_j exp(s_j) over the scanned rows; -inf if none) */
typedef struct {
    int32_t *clusters;
    int32_t *n_clusters;
    int32_t *n_keys;
    int32_t *key_idx;
    uint8_t *l1_surv;
    float *dbg_S;
    float *dbg_S1;
    float *dbg_lse;
    int32_t *key_pref;
    uint8_t *l0_surv; /* optional [B, H, c0] Level-0 survivors (levels == 3) */
    float *dbg_S0;    /* optional [B, H, c0] Level-0 S^(0) / S-bar^(0)       */
} sqz_selection;

int sqz_lookup_workspace(const sqz_index *idx, int32_t B, int32_t n_q, size_t *ws_bytes);

/* Q [B, H, n_q, d] dtype.  n_q == 1 is the generation stage: per
 * (b,h) the cluster i is selected iff S_i > T, evaluated as
 * (s_i - m) > log D + log T with m = max_j s_j, D = sum_j N_j exp(s_j - m)
 * (the paper's single-pass form with the max folded into the threshold,
 * P:775-776).  n_q > 1 is the prefill stage: S-bar_i =
 * (1/n_q) sum_t S_{t,i}, selected iff S-bar_i > T, one selection per (b,h)
 * shared by its n_q queries (R7).  levels == 2: Level-1 scores with N1 against
 * T1, survivors expanded to their children, Level-2 scores with the
 * denominator restricted to those children (Eq. 3), against T.
 * levels == 3: Level 0 (N0, T0) first, then Level 1 restricted to the
 * children of the Level-0 survivors (Eq. 3 one level up), then Level 2 as
 * above (O(c' log L + k)).  Sharded (p->comm) and staged
 * lookups support levels 1 and 2. */
int sqz_centroid_lookup(const sqz_index *idx, const void *Q, int32_t B, int32_t n_q,
                        const sqz_lookup_params *p, const sqz_selection *out, void *ws,
                        size_t ws_bytes, void *stream);

/* Staged form of the lookup, for fixed-context shards with a caller-driven
 * exchange (what sqz_centroid_lookup runs internally when p->comm is set).
 * A level's statistics are, per query row (b, h, t), the pair (m, D) with
 * m = max_i s_i and D = sum_i N_i exp(s_i - m) over the rows this shard scans
 * at that level (m = -inf, D = 0 if none); the global denominator of Eq. 1 /
 * Eq. 3 is the fold of the shards' pairs, LSE_w = log sum_r D_r e^{m_r}.
 *   stage 0:        scan the first level (Level 1, or the single level),
 *                   write its statistics to stats_out [B, H, n_q, 2] fp32.
 *   stage k >= 1:   stats_in [P, B, H, n_q, 2] = the statistics of level k
 *                   from all P shards in rank order (P = 1: this shard only,
 *                   equal to the unsharded lookup); fold them in rank order,
 *                   threshold level k (writing `out` when k == levels), and if
 *                   k < levels scan level k + 1 over the children of the
 *                   surviving clusters, writing its statistics to stats_out.
 * Stages 0 .. levels must run in order on one workspace (p->comm ignored);
 * the exchange between them is the caller's (sqz_comm_allgather_stats, NCCL,
 * or, in tests, a device copy). */
int sqz_centroid_lookup_stage(const sqz_index *idx, const void *Q, int32_t B, int32_t n_q,
                              const sqz_lookup_params *p, int32_t stage, int32_t P,
                              const float *stats_in, float *stats_out, const sqz_selection *out,
                              void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------- */
/* Online step 2: sparse attention (section 4.2)                  */
/* ---------------------------------------------------------------------- */
typedef struct {
    float scale;       /* z = scale * q.k (1/sqrt(d))                                      */
    int32_t causal;    /* 1: user key u visible to query t iff u <= t + n_u - n_q (R8)       */
    int32_t partial;   /* 1: rows with no attended key give O = 0, LSE = -inf (identity     */
                       /*    partial for a later merge); 0: such rows are an error,          */
                       /*    reported by sqz_attention_status()                              */
    int32_t out_dtype; /* sqz_dtype of O                                                     */
    int32_t per_row;   /* decode (n_q == 1) with B >= 2: 0 (default) = the B sequences share  */
                       /*    the fixed context, so each head streams the UNION of   */
                       /*    its B selections once, every key applied to the queries whose    */
                       /*    selection holds it (bf16, d = 128, B <= 16); 1 = one key stream  */
                       /*    per (b,h).  Same result either way (each query attends exactly   */
                       /*    its own selection plus its own user KV).                         */
} sqz_attn_params;

int sqz_attention_workspace(const sqz_index *idx, int32_t B, int32_t n_q, int32_t n_u,
                            size_t *ws_bytes);

/* Q [B,H,n_q,d] dtype; Kp, Vp [H,L,d] dtype (cluster-major); sel: output of
 * sqz_centroid_lookup (n_keys, n_clusters, clusters and key_pref are read, with
 * idx->key_off; key_idx is not needed); Ku, Vu [B,H,n_u,d] dtype
 * (may be NULL when n_u == 0).  Outputs: O [B,H,n_q,d] out_dtype and
 * LSE [B,H,n_q] fp32 = natural-log sum of exp(z) over the attended keys.
 * For each query row the attended set is the selected fixed keys of its (b,h)
 * plus the visible user keys; O is the exact softmax-weighted sum of their
 * values.  Work is split into fixed-size key chunks ("a fixed number of ...
 * keys ... for a single SM") whose partials are merged. */
int sqz_sparse_attention(const void *Q, int32_t B, int32_t n_q, const void *Kp, const void *Vp,
                         const sqz_index *idx, const sqz_selection *sel, const void *Ku,
                         const void *Vu, int32_t n_u, const sqz_attn_params *p, void *O,
                         float *LSE, void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------- */
/* One decode step: lookup + sparse attention in one call                    */
/* ---------------------------------------------------------------------- */
/* sqz_decode_step(Q [B,H,1,d]) computes exactly what sqz_centroid_lookup
 * (n_q = 1) followed by sqz_sparse_attention computes -- the same selection
 * rule and the same attended set (selected fixed keys + all n_u
 * user keys) -- and writes the same outputs: `sel` (clusters,
 * n_clusters, n_keys, key_pref required; key_idx optional) and O, LSE.
 * For B = 1, a single-level unsharded index, n_u > 0 and no debug outputs the
 * two kernels are arranged for decode latency: the user KV does not depend on
 * the selection (the user input follows the fixed context), so the
 * attention kernel -- launched behind the lookup -- attends it in 256-key
 * chunks on CTAs that run beside the lookup's CTAs (a lookup variant limited to
 * 84 registers leaves them room) BEFORE it waits for the selection; the chunk
 * partials join each row's split-KV merge.  Other shapes run the
 * two calls internally.  The selection is identical to the two-call path's
 * (same lookup arithmetic); O/LSE differ only in summation order.
 * ap->causal is ignored (decode sees all n_u user keys, R8).  ws:
 * sqz_decode_step_workspace bytes, zeroed once (sqz_workspace_init), then
 * self-cleaning for a fixed (idx, B, n_u); empty rows with ap->partial == 0
 * are reported by sqz_attention_status(ws) as for sqz_sparse_attention. */
int sqz_decode_step_workspace(const sqz_index *idx, int32_t B, int32_t n_u, size_t *ws_bytes);
int sqz_decode_step(const sqz_index *idx, const void *Q, int32_t B, const void *Kp, const void *Vp,
                    const void *Ku, const void *Vu, int32_t n_u, const sqz_lookup_params *lp,
                    const sqz_attn_params *ap, const sqz_selection *sel, void *O, float *LSE,
                    void *ws, size_t ws_bytes, void *stream);

/* Synchronises the stream and returns SQZ_ERR_EMPTY if the last non-partial
 * sqz_sparse_attention on this workspace produced a row with no attended key
 * (and clears the flag), else SQZ_OK. */
int sqz_attention_status(void *ws, size_t ws_bytes, void *stream);

/* Merge of P partial results:
 *   O_parts [P, rows, d] fp32, LSE_parts [P, rows] fp32 (natural log; -inf =
 *   identity partial)  ->  O [rows, d] out_dtype, LSE [rows] fp32 with
 *   LSE = log sum_p exp(LSE_p), O = sum_p exp(LSE_p - LSE) O_p. */
int sqz_merge_partials(int32_t P, const float *O_parts, const float *LSE_parts, int64_t rows,
                       int32_t d, void *O, float *LSE, int32_t out_dtype, void *stream);

/* ---------------------------------------------------------------------- */
/* Selection diagnostics (App. A; App. D; NEXT-4)        */
/* ---------------------------------------------------------------------- */
/* For ONE decode query per (b,h) (Q [B,H,1,d]) and the selection `sel` the
 * lookup produced for it (clusters, n_clusters, n_keys read), with
 * a_j = exp(z_j - LSE) the softmax of z_j = scale q.k_j over ALL L fixed keys
 * of the head (Kp, cluster-major; attention is permutation-invariant):
 *   skew       [B,H] fp32  sum of the n_top largest a_j, n_top = max(1,
 *                          ceil(top_frac * L)) -- App. A's "cumulative
 *                          attention scores for the top 1%" (1 = skewed head,
 *                          ~top_frac = flat head)
 *   n_T, mass_T [B,H]      App. D's ideal lookup at threshold T: the keys with
 *                          a_j > T (T == 0: all), their count and mass
 *   mass_sel   [B,H] fp32  sum of a_j over the selected keys (the attention
 *                          mass the centroid lookup retrieves)
 *   mass_ideal [B,H] fp32  sum of the k largest a_j, k = n_keys[b,h] (the
 *                          ideal selection at MATCHED budget; >= mass_sel)
 *   recall     [B,H] fp32  |selected n ideal k-set| / k (1 when k = 0)
 * Logits are fp32 dot products of the stored bits (the logits attention
 * uses); the oracle ranks fp64 logits, so results can differ only through
 * fp32 rounding of near-equal logits.  Not an online-path call: three
 * launches, the last with one CTA per (b,h).  Unsharded indexes only
 * (L_total == 0).  ws: sqz_selection_diagnostics_workspace bytes (about
 * 5 B per (b,h) and key; no zeroing needed).  Errors: SQZ_ERR_INVALID_ARG
 * (NULL pointers, top_frac not in (0, 1], T < 0 or NaN, sharded index). */
typedef struct {
    float *skew;
    float *mass_sel;
    float *mass_ideal;
    float *recall;
    int32_t *n_T;
    float *mass_T;
} sqz_diagnostics;

int sqz_selection_diagnostics_workspace(const sqz_index *idx, int32_t B, size_t *ws_bytes);
int sqz_selection_diagnostics(const sqz_index *idx, const void *Q, int32_t B, const void *Kp,
                              const sqz_selection *sel, float scale, double top_frac, float T,
                              const sqz_diagnostics *out, void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------- */
/* Multi-GPU: fixed-context sharding by cluster (the paper is    */
/* single-GPU, so this is this build's addition)                     */
/* ---------------------------------------------------------------------- */
/* Plan of one rank's shard, computed on the HOST from host copies of the
 * index's integer tables (no GPU needed).  Ownership: Level-1 cluster p (or,
 * single level, cluster i) belongs to rank p mod world ("interleaved", so
 * jointly selected neighbouring clusters spread over the ranks); a Level-1
 * cluster's children and every cluster's keys stay with it.  Local ids keep
 * the global order.
 *   key_off   [H, c2 + 1] host int32 of the full index; child_off [H, c1 + 1]
 *             host int32 (levels == 2) else NULL.
 *   plan->c1, c2, L   out: local table rows / key row capacity (max over
 *             heads; padding rows have N = 0 and empty ranges)
 *   The array fields are optional HOST outputs (NULL = skip; call once with
 *   all NULL to size them):
 *   c1_src [H, c1] global Level-1 id of local row      N1 [H, c1], child_off [H, c1 + 1]
 *   c2_src [H, c2] global Level-2 id, -1 = padding     N2 [H, c2], key_off [H, c2 + 1]
 *   key_src [H, L] global cluster-major position of local key row, -1 = padding
 * Errors: SQZ_ERR_INVALID_ARG (world < 1, rank out of range, fewer clusters
 * than ranks at the sharded level, inconsistent tables). */
typedef struct {
    int32_t c1, c2;
    int64_t L;
    int32_t *c1_src, *c2_src, *key_src;
    int32_t *N1, *child_off, *N2, *key_off;
} sqz_shard_plan;

int sqz_shard_plan_compute(int32_t H, int32_t levels, int32_t c1, int32_t c2, int64_t L,
                           const int32_t *key_off, const int32_t *child_off, int32_t rank,
                           int32_t world, sqz_shard_plan *plan);

/* Builds the shard index on the device from the full one:
 *   full, Kp, Vp: the full index and its cluster-major K/V (device)
 *   c1_src, c2_src, key_src: the plan's arrays copied to the DEVICE
 *   local: geometry (H, d, levels, dtype, c1, c2, L = plan's, L_total =
 *          full->L) and device tables; the caller uploads N1, child_off, N2,
 *          key_off from the plan; this call writes C1, C2 (rows gathered,
 *          padding = 0), perm (gathered, padding = -1), Kp_local, Vp_local
 *          [H, L, d] (padding rows = 0).  Asynchronous on `stream`. */
int sqz_index_shard(const sqz_index *full, const void *Kp, const void *Vp, const int32_t *c1_src,
                    const int32_t *c2_src, const int32_t *key_src, const sqz_index *local,
                    void *Kp_local, void *Vp_local, void *stream);

/* Communicator over the ranks holding the shards (one process per GPU).  The
 * library resolves NCCL at run time (the copy already loaded in the process,
 * e.g. torch's, else libnccl.so.2); without it these calls return
 * SQZ_ERR_NCCL.  Rank 0 creates the id and the caller broadcasts its 128
 * bytes (e.g. with torch.distributed); every rank then calls sqz_comm_init
 * with the CUDA device it will use current.  Blocking (collective). */
int sqz_comm_unique_id(uint8_t id[128]);
int sqz_comm_init(const uint8_t id[128], int32_t rank, int32_t world, void **comm);
int sqz_comm_destroy(void *comm);

/* Workspace of sqz_centroid_lookup with p->comm set (world ranks). */
int sqz_lookup_workspace_comm(const sqz_index *idx, int32_t B, int32_t n_q, int32_t world,
                              size_t *ws_bytes);

/* Output exchange (P:361-363 across GPUs): every rank passes its partial
 * (O_part [rows, d] fp32, LSE_part [rows] fp32; -inf = identity) from
 * sqz_sparse_attention(partial = 1, out_dtype = SQZ_F32); the partials are
 * all-gathered over NVLink (NCCL) into ws and merged in rank order, so every
 * rank ends with the same O [rows, d] out_dtype and LSE [rows].  ws:
 * sqz_comm_merge_workspace bytes.  Asynchronous on `stream`. */
int sqz_comm_merge_workspace(int32_t world, int64_t rows, int32_t d, size_t *ws_bytes);
int sqz_comm_allgather_merge(void *comm, const float *O_part, const float *LSE_part, int64_t rows,
                             int32_t d, void *O, float *LSE, int32_t out_dtype, void *ws,
                             size_t ws_bytes, void *stream);

/* Output exchange by HEAD SLICE (the prefill form): a 4K-token
 * prefill partial is [B, H, n_q, d] fp32 per rank, and all-gathering it would
 * land world x that on every rank.  Here rank r receives from every rank only
 * the partial rows of its heads [r H/world, (r+1) H/world) (grouped
 * ncclSend/ncclRecv) and merges them in rank order:
 *   O_part [B, H, n_q, d] fp32, LSE_part [B, H, n_q] fp32 (this rank's partial;
 *   -inf = identity) -> O_slice [B, H/world, n_q, d] out_dtype, LSE_slice
 *   [B, H/world, n_q] fp32: the exact output of this rank's heads (what a
 *   head-parallel o_proj consumes).  H must be a multiple of world.  ws:
 *   sqz_comm_alltoall_merge_workspace bytes.  Asynchronous on `stream`. */
int sqz_comm_alltoall_merge_workspace(int32_t world, int32_t B, int32_t H, int32_t n_q, int32_t d,
                                      size_t *ws_bytes);
int sqz_comm_alltoall_merge(void *comm, const float *O_part, const float *LSE_part, int32_t B, int32_t H,
                            int32_t n_q, int32_t d, void *O_slice, float *LSE_slice, int32_t out_dtype,
                            void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------- */
/* Misc                                                                      */
/* ---------------------------------------------------------------------- */
/* Zero a workspace (cudaMemsetAsync) before its first use. */
int sqz_workspace_init(void *ws, size_t ws_bytes, void *stream);
/* Thread-local message describing the last error returned on this thread. */
const char *sqz_last_error(void);
/* SQZ_ABI_VERSION of the loaded library. */
int sqz_abi_version(void);
/* SQZ_OK iff the current device is an sm_100 part the library was built for. */
int sqz_device_check(void);

#ifdef __cplusplus
}
#endif
#endif /* SQZ_H */
