/*
 * sqzref.c -- CPU ORACLE for Squeezed Attention (arXiv 2411.09688).
 *
 * TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2411_09688_b200/csrc) and neither side includes the other.
 *
 * Conventions
 *   - Every floating-point operation is IEEE fp64; exp/log are libm exp/log.
 *     No -ffast-math.  Inputs are the stored (bf16 / fp32) bits converted
 *     exactly to fp64 by the Python wrapper (oracle/__init__.py).
 *   - Citations: "P:n" = line n of the paper's LaTeX source;
 *     "S:n" = line n of SPEC.md.  Readings where the paper is silent are
 *     labelled R<k> and listed in DESIGN.md section "Readings".
 *   - The loops are written out literally, in the order the paper states the
 *     computation.  The only parallelism is "#pragma omp parallel for" over
 *     mutually independent outer units (points, (b,h) rows, query rows); it
 *     does not change any arithmetic.
 */
#include "sqzref.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Storage rounding (R18): fp64 -> bf16 / fp32, round-to-nearest-even, once. */
/* ------------------------------------------------------------------------ */

double sqzref_round_bf16(double x)
{
    /* bf16 keeps 8 significant bits.  frexp gives x = m * 2^e, 0.5 <= |m| < 1;
     * nearbyint under the default FE_TONEAREST mode rounds half to even. */
    if (x == 0.0 || !isfinite(x)) return x;
    int e;
    double m = frexp(x, &e);
    double r = nearbyint(ldexp(m, 8));
    return ldexp(r, e - 8);
}

void sqzref_round_array(double *x, int64_t n, int dtype)
{
    for (int64_t i = 0; i < n; ++i) {
        if (dtype == SQZREF_BF16) x[i] = sqzref_round_bf16(x[i]);
        else x[i] = (double)(float)x[i]; /* C conversion rounds to nearest-even */
    }
}

/* ------------------------------------------------------------------------ */
/* Offline K-means (section 3.1):                                 */
/*   "we use K-means clustering with normalized key vectors to group similar */
/*    keys together" -- Lloyd's algorithm on unit-normalised vectors (R3).   */
/* ------------------------------------------------------------------------ */

static double sqdist(const double *a, const double *b, int d)
{
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
        double t = a[k] - b[k];
        s += t * t;
    }
    return s;
}

int sqzref_kmeans(const double *X, int64_t n, int d, int c, const int64_t *init,
                  int max_iters, double tol, int32_t *assign, double *mu,
                  int *iters_out, double *objective)
{
    if (c < 1 || (int64_t)c > n || d < 1) return SQZREF_ERR_INVALID;
    for (int i = 0; i < c; ++i)
        if (init[i] < 0 || init[i] >= n) return SQZREF_ERR_INVALID;

    /* Step 1: X^_j = X_j / ||X_j||; a zero vector stays zero. */
    double *Xh = (double *)malloc(sizeof(double) * (size_t)n * d);
    double *mu_new = (double *)malloc(sizeof(double) * (size_t)c * d);
    int64_t *count = (int64_t *)malloc(sizeof(int64_t) * (size_t)c);
    double *pdist = (double *)malloc(sizeof(double) * (size_t)n);
    if (!Xh || !mu_new || !count || !pdist) {
        free(Xh); free(mu_new); free(count); free(pdist);
        return SQZREF_ERR_INVALID;
    }
    for (int64_t j = 0; j < n; ++j) {
        double nrm = 0.0;
        for (int k = 0; k < d; ++k) nrm += X[j * d + k] * X[j * d + k];
        nrm = sqrt(nrm);
        for (int k = 0; k < d; ++k) Xh[j * d + k] = nrm > 0.0 ? X[j * d + k] / nrm : 0.0;
    }

    /* Step 2: mu_i = X^_{init[i]} (seeded subset drawn by the harness, R3). */
    for (int i = 0; i < c; ++i)
        memcpy(mu + (size_t)i * d, Xh + (size_t)init[i] * d, sizeof(double) * d);
    for (int64_t j = 0; j < n; ++j) assign[j] = -1;

    int it = 0;
    for (it = 0; it < max_iters; ++it) {
        /* Step 3a: assignment a_j = argmin_i ||X^_j - mu_i||^2, ties -> lowest i. */
        int64_t changed = 0;
#pragma omp parallel for reduction(+ : changed) schedule(static)
        for (int64_t j = 0; j < n; ++j) {
            double best = INFINITY;
            int bi = 0;
            for (int i = 0; i < c; ++i) {
                double dist = sqdist(Xh + j * d, mu + (size_t)i * d, d);
                if (dist < best) { best = dist; bi = i; }
            }
            if (assign[j] != bi) changed += 1;
            assign[j] = bi;
            pdist[j] = best;
        }

        /* Step 3b: empty-cluster repair: each empty cluster, in
         * increasing id, takes the point farthest from its own centroid among
         * clusters with more than one member (ties -> lowest point index). */
        for (int i = 0; i < c; ++i) count[i] = 0;
        for (int64_t j = 0; j < n; ++j) count[assign[j]] += 1;
        for (int i = 0; i < c; ++i) {
            if (count[i] != 0) continue;
            int64_t bj = -1;
            double bd = -1.0;
            for (int64_t j = 0; j < n; ++j) {
                if (count[assign[j]] > 1 && pdist[j] > bd) { bd = pdist[j]; bj = j; }
            }
            if (bj < 0) break; /* cannot happen when c <= n */
            count[assign[bj]] -= 1;
            assign[bj] = i;
            count[i] = 1;
            pdist[bj] = 0.0;
            changed += 1;
        }

        /* Step 3c: update mu_i = mean of member X^ (P:173 applied in the
         * normalised space used for the assignment). */
        for (size_t t = 0; t < (size_t)c * d; ++t) mu_new[t] = 0.0;
        for (int64_t j = 0; j < n; ++j)
            for (int k = 0; k < d; ++k) mu_new[(size_t)assign[j] * d + k] += Xh[j * d + k];
        double shift = 0.0;
        for (int i = 0; i < c; ++i) {
            double s2 = 0.0;
            for (int k = 0; k < d; ++k) {
                double v = count[i] > 0 ? mu_new[(size_t)i * d + k] / (double)count[i]
                                        : mu[(size_t)i * d + k];
                double t = v - mu[(size_t)i * d + k];
                s2 += t * t;
                mu_new[(size_t)i * d + k] = v;
            }
            if (sqrt(s2) > shift) shift = sqrt(s2);
        }
        memcpy(mu, mu_new, sizeof(double) * (size_t)c * d);

        if (objective) {
            double J = 0.0;
            for (int64_t j = 0; j < n; ++j) J += sqdist(Xh + j * d, mu + (size_t)assign[j] * d, d);
            objective[it] = J;
        }
        /* Step 3d: stop when no assignment changed or max shift < tol. */
        if (changed == 0 || shift < tol) { it += 1; break; }
    }
    if (iters_out) *iters_out = it;
    free(Xh); free(mu_new); free(count); free(pdist);
    return SQZREF_OK;
}

/* Step 4: C_i = mean of the RAW member vectors (reading R2); N_i = |members|. */
void sqzref_cluster_means(const double *X, int64_t n, int d, int c, const int32_t *assign,
                          double *C, int32_t *N)
{
    for (size_t t = 0; t < (size_t)c * d; ++t) C[t] = 0.0;
    for (int i = 0; i < c; ++i) N[i] = 0;
    for (int64_t j = 0; j < n; ++j) {
        N[assign[j]] += 1;
        for (int k = 0; k < d; ++k) C[(size_t)assign[j] * d + k] += X[j * d + k];
    }
    for (int i = 0; i < c; ++i)
        for (int k = 0; k < d; ++k)
            C[(size_t)i * d + k] = N[i] > 0 ? C[(size_t)i * d + k] / (double)N[i] : 0.0;
}

/* Cluster-major ordering of the index (section 3.3 / Fig. 2).
 * Level-2 clusters are grouped by their Level-1 parent (stable in old id) and
 * keys are grouped by Level-2 cluster (stable in original key index).
 *   l2_order[new] = old level-2 id; perm[pos] = original key index;
 *   key_off[new .. new+1) = key positions of level-2 cluster `new`;
 *   child_off[p .. p+1)   = new level-2 ids whose parent is p. */
int sqzref_build_order(int64_t L, int c2, const int32_t *assign2, int c1, const int32_t *parent,
                       int32_t *l2_order, int32_t *perm, int32_t *key_off, int32_t *child_off)
{
    int32_t *new_of_old = (int32_t *)malloc(sizeof(int32_t) * (size_t)c2);
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(c2 + 1));
    if (!new_of_old || !fill) { free(new_of_old); free(fill); return SQZREF_ERR_INVALID; }

    int pos = 0;
    if (parent && c1 > 0) {
        for (int p = 0; p < c1; ++p) {
            child_off[p] = pos;
            for (int o = 0; o < c2; ++o)
                if (parent[o] == p) l2_order[pos++] = o;
        }
        child_off[c1] = pos;
    } else {
        for (int o = 0; o < c2; ++o) l2_order[pos++] = o;
    }
    if (pos != c2) { free(new_of_old); free(fill); return SQZREF_ERR_INVARIANT; }
    for (int i = 0; i < c2; ++i) new_of_old[l2_order[i]] = i;

    /* counting sort of keys by new level-2 id; scanning j upward keeps it stable */
    for (int i = 0; i <= c2; ++i) fill[i] = 0;
    for (int64_t j = 0; j < L; ++j) fill[new_of_old[assign2[j]] + 1] += 1;
    for (int i = 0; i < c2; ++i) fill[i + 1] += fill[i];
    for (int i = 0; i <= c2; ++i) key_off[i] = (int32_t)fill[i];
    for (int64_t j = 0; j < L; ++j) {
        int i = new_of_old[assign2[j]];
        perm[fill[i]++] = (int32_t)j;
    }
    free(new_of_old); free(fill);
    return SQZREF_OK;
}

/* ------------------------------------------------------------------------ */
/* Online centroid lookup (section 3.2 Eq. 1; section 3.3          */
/* Eq. 2-3; prefill averaging P:330-335).                         */
/* ------------------------------------------------------------------------ */

/* Eq. 1 for one query over the rows listed in `rows` (all c rows when
 * rows == NULL):  s_i = scale * q.C_i   (R1: scale = 1/sqrt(d) by default)
 *                 S_i = exp(s_i) / sum_j N_j exp(s_j)
 * evaluated with the max subtracted: lse = m + log(sum_j N_j exp(s_j - m)),
 * S_i = exp(s_i - lse).  Eq. 3 is the same formula with `rows` = the children
 * of the surviving Level-1 clusters ("the denominator is also calculated based
 * on these selected centroids"). */
void sqzref_scores(const double *q, const double *C, const int32_t *N, int d, int c,
                   int n_rows, const int32_t *rows, double scale,
                   double *s, double *S, double *lse_out)
{
    int nr = rows ? n_rows : c;
    double m = -INFINITY;
    for (int r = 0; r < nr; ++r) {
        int i = rows ? rows[r] : r;
        double dot = 0.0;
        for (int k = 0; k < d; ++k) dot += q[k] * C[(size_t)i * d + k];
        s[i] = scale * dot;
        if (s[i] > m) m = s[i];
    }
    double D = 0.0;
    for (int r = 0; r < nr; ++r) {
        int i = rows ? rows[r] : r;
        D += (double)N[i] * exp(s[i] - m);
    }
    double lse = m + log(D);
    for (int r = 0; r < nr; ++r) {
        int i = rows ? rows[r] : r;
        S[i] = exp(s[i] - lse);
    }
    if (lse_out) *lse_out = lse;
}

/* Generation-stage single-pass selection (P:339-345 and App. C):
 * pass 1 computes m = max s_j and D = sum_j N_j exp(s_j - m) while caching
 * e_i = exp(s_i - m); pass 2 selects i iff e_i > D * T.  The max correction is
 * folded into the threshold rather than into e_i. */
void sqzref_select_singlepass(const double *s, const int32_t *N, int c, double T, uint8_t *sel)
{
    double m = -INFINITY;
    for (int i = 0; i < c; ++i) if (s[i] > m) m = s[i];
    double *e = (double *)malloc(sizeof(double) * (size_t)c);
    double D = 0.0;
    for (int i = 0; i < c; ++i) { e[i] = exp(s[i] - m); D += (double)N[i] * e[i]; }
    for (int i = 0; i < c; ++i) sel[i] = (T == 0.0) ? 1 : (e[i] > D * T);
    free(e);
}

/* Full lookup for B x H query blocks of n_q rows each (decode: n_q = 1).
 *   Single level (levels == 1): S_bar_i = (1/n_q) sum_t S_{t,i};
 *     cluster i selected iff S_bar_i > T (strict, R6);
 *     T == 0 selects every cluster (R6).
 *   Two levels (levels == 2): Level-1 S_bar^(1) with N^(1) = descendant keys
 *     (R4) against T1; survivors expand to their children via
 *     child_off; Level-2 scores use the denominator restricted to those
 *     children (Eq. 3), averaged over queries, against T (= T2).
 *     forced_l1 (optional [B,H,c1]) replaces the Level-1 decision: the
 *     conditional-parity rule of DESIGN.md.
 * Outputs (all [B,H,...]): sel2[c2], Sbar2[c2] (NaN for unscanned rows),
 *   surv1[c1], Sbar1[c1] (levels==2 only), lse[n_q] = finest-level log
 *   denominator per query (-inf when no row was scanned). */
int sqzref_lookup(int B, int H, int n_q, int d, const double *Q,
                  int levels, int c1, const double *C1, const int32_t *N1, const int32_t *child_off,
                  int c2, const double *C2, const int32_t *N2,
                  double scale, double T, double T1, const uint8_t *forced_l1,
                  uint8_t *sel2, double *Sbar2, uint8_t *surv1, double *Sbar1, double *lse)
{
    if (B < 1 || H < 1 || n_q < 1 || d < 1 || c2 < 1) return SQZREF_ERR_INVALID;
    if (!(T >= 0.0) || (levels == 2 && !(T1 >= 0.0))) return SQZREF_ERR_INVALID;
    if (levels == 2 && (c1 < 1 || !C1 || !N1 || !child_off)) return SQZREF_ERR_INVALID;

#pragma omp parallel for schedule(dynamic)
    for (int bh = 0; bh < B * H; ++bh) {
        int h = bh % H;
        const double *Qbh = Q + (size_t)bh * n_q * d;
        const double *C2h = C2 + (size_t)h * c2 * d;
        const int32_t *N2h = N2 + (size_t)h * c2;
        uint8_t *sel = sel2 + (size_t)bh * c2;
        double *Sb2 = Sbar2 + (size_t)bh * c2;
        double *lse_bh = lse ? lse + (size_t)bh * n_q : NULL;
        double *s = (double *)malloc(sizeof(double) * (size_t)(c2 > c1 ? c2 : c1));
        double *S = (double *)malloc(sizeof(double) * (size_t)(c2 > c1 ? c2 : c1));
        int32_t *rows = (int32_t *)malloc(sizeof(int32_t) * (size_t)c2);
        int n_rows = 0;

        if (levels == 2) {
            const double *C1h = C1 + (size_t)h * c1 * d;
            const int32_t *N1h = N1 + (size_t)h * c1;
            const int32_t *coff = child_off + (size_t)h * (c1 + 1);
            double *Sb1 = Sbar1 + (size_t)bh * c1;
            uint8_t *sv1 = surv1 + (size_t)bh * c1;
            /* Eq. 2 per query, averaged over the n_q queries (R7). */
            for (int p = 0; p < c1; ++p) Sb1[p] = 0.0;
            for (int t = 0; t < n_q; ++t) {
                sqzref_scores(Qbh + (size_t)t * d, C1h, N1h, d, c1, 0, NULL, scale, s, S, NULL);
                for (int p = 0; p < c1; ++p) Sb1[p] += S[p];
            }
            for (int p = 0; p < c1; ++p) Sb1[p] /= (double)n_q;
            for (int p = 0; p < c1; ++p) {
                if (forced_l1) sv1[p] = forced_l1[(size_t)bh * c1 + p] ? 1 : 0;
                else sv1[p] = (T1 == 0.0) ? 1 : (Sb1[p] > T1);
            }
            /* expand survivors to their Level-2 children */
            for (int p = 0; p < c1; ++p)
                if (sv1[p])
                    for (int l = coff[p]; l < coff[p + 1]; ++l) rows[n_rows++] = l;
        } else {
            for (int l = 0; l < c2; ++l) rows[n_rows++] = l;
        }

        for (int l = 0; l < c2; ++l) { Sb2[l] = NAN; sel[l] = 0; }
        if (n_rows == 0) {
            if (lse_bh) for (int t = 0; t < n_q; ++t) lse_bh[t] = -INFINITY;
        } else {
            for (int r = 0; r < n_rows; ++r) Sb2[rows[r]] = 0.0;
            for (int t = 0; t < n_q; ++t) {
                double l_t;
                sqzref_scores(Qbh + (size_t)t * d, C2h, N2h, d, c2, n_rows, rows, scale, s, S, &l_t);
                for (int r = 0; r < n_rows; ++r) Sb2[rows[r]] += S[rows[r]];
                if (lse_bh) lse_bh[t] = l_t;
            }
            for (int r = 0; r < n_rows; ++r) {
                int l = rows[r];
                Sb2[l] /= (double)n_q;
                sel[l] = (T == 0.0) ? 1 : (Sb2[l] > T);
            }
        }
        free(s); free(S); free(rows);
    }
    return SQZREF_OK;
}

/* Multi-level lookup (section 3.3: "this method can be extended to multiple
 * levels of hierarchy"; complexity O(c' log L + k)).
 * Lv levels, 0 = coarsest ... Lv-1 = finest (the key clusters).  Level l has
 * the table C[l] [H, c[l], d] and N[l] [H, c[l]] (descendant keys, R4); for
 * l < Lv-1, child_off[l] [H, c[l]+1] gives the contiguous level-(l+1) children
 * of each cluster.  Level 0 scores all its rows with Eq. 2; level l > 0 scores
 * the children of the level-(l-1) survivors with the denominator restricted to
 * them (Eq. 3 applied level by level).  Scores are averaged over the n_q queries
 * of a (b,h) (R7), survivors are S_bar > T[l] (strict; T[l] = 0 keeps all, R6);
 * forced[l] (optional [B,H,c[l]]) replaces the decision at level l < Lv-1 (the
 * conditional-parity rule).  Outputs per level: surv[l] [B,H,c[l]], Sbar[l]
 * [B,H,c[l]] (NaN for rows not scanned); lse [B,H,n_q] of the finest level. */
int sqzref_lookup_ml(int B, int H, int n_q, int d, const double *Q, int Lv, const int32_t *c,
                     const double *const *C, const int32_t *const *N,
                     const int32_t *const *child_off, double scale, const double *T,
                     const uint8_t *const *forced, uint8_t *const *surv, double *const *Sbar,
                     double *lse)
{
    if (B < 1 || H < 1 || n_q < 1 || d < 1 || Lv < 1) return SQZREF_ERR_INVALID;
    int cmax = 1;
    for (int l = 0; l < Lv; ++l) {
        if (c[l] < 1 || !(T[l] >= 0.0)) return SQZREF_ERR_INVALID;
        if (c[l] > cmax) cmax = c[l];
    }
#pragma omp parallel for schedule(dynamic)
    for (int bh = 0; bh < B * H; ++bh) {
        int h = bh % H;
        const double *Qbh = Q + (size_t)bh * n_q * d;
        double *s = (double *)malloc(sizeof(double) * (size_t)cmax);
        double *S = (double *)malloc(sizeof(double) * (size_t)cmax);
        int32_t *rows = (int32_t *)malloc(sizeof(int32_t) * (size_t)cmax);
        int32_t *next = (int32_t *)malloc(sizeof(int32_t) * (size_t)cmax);
        int n_rows = c[0];
        for (int r = 0; r < n_rows; ++r) rows[r] = r;
        for (int l = 0; l < Lv; ++l) {
            const double *Ch = C[l] + (size_t)h * c[l] * d;
            const int32_t *Nh = N[l] + (size_t)h * c[l];
            double *Sb = Sbar[l] + (size_t)bh * c[l];
            uint8_t *sv = surv[l] + (size_t)bh * c[l];
            for (int i = 0; i < c[l]; ++i) { Sb[i] = NAN; sv[i] = 0; }
            if (n_rows == 0) {
                if (l == Lv - 1 && lse) for (int t = 0; t < n_q; ++t) lse[(size_t)bh * n_q + t] = -INFINITY;
                continue;
            }
            for (int r = 0; r < n_rows; ++r) Sb[rows[r]] = 0.0;
            for (int t = 0; t < n_q; ++t) {
                double l_t;
                sqzref_scores(Qbh + (size_t)t * d, Ch, Nh, d, c[l], n_rows, rows, scale, s, S, &l_t);
                for (int r = 0; r < n_rows; ++r) Sb[rows[r]] += S[rows[r]];
                if (l == Lv - 1 && lse) lse[(size_t)bh * n_q + t] = l_t;
            }
            for (int r = 0; r < n_rows; ++r) {
                int i = rows[r];
                Sb[i] /= (double)n_q;
                if (l < Lv - 1 && forced && forced[l]) sv[i] = forced[l][(size_t)bh * c[l] + i] ? 1 : 0;
                else sv[i] = (T[l] == 0.0) ? 1 : (Sb[i] > T[l]);
            }
            if (l < Lv - 1) {
                /* expand the survivors, in increasing id, to their children */
                const int32_t *co = child_off[l] + (size_t)h * (c[l] + 1);
                int nn = 0;
                for (int i = 0; i < c[l]; ++i)
                    if (sv[i])
                        for (int ch = co[i]; ch < co[i + 1]; ++ch) next[nn++] = ch;
                for (int r = 0; r < nn; ++r) rows[r] = next[r];
                n_rows = nn;
            }
        }
        free(s); free(S); free(rows); free(next);
    }
    return SQZREF_OK;
}

/* ------------------------------------------------------------------------ */
/* Exact attention over the selected fixed keys plus the user KV            */
/* (section 4.2; separate fixed / user caches P:312; R8).        */
/* ------------------------------------------------------------------------ */

/* For every (b, h, query t):
 *   A_t = {fixed key j : keymask[b,h,j]} U {user key u : !causal or
 *          u <= qpos[t] + n_u - n_q_total}   (user input follows the fixed
 *          context; bottom-right-aligned causal mask, R8)
 *   z_j = scale * q_t . k_j
 *   LSE_t = log sum_{j in A_t} exp(z_j)      (evaluated as m + log sum exp(z - m))
 *   O_t = sum_{j in A_t} exp(z_j - LSE_t) v_j
 * K, V: [H, L, d] in ORIGINAL key order; keymask: [B, H, L] or NULL (= all);
 * Ku, Vu: [B, H, n_u, d]; qpos: [n_q] query positions in 0..n_q_total-1 (NULL =
 * 0..n_q-1).  An empty A_t gives O_t = 0, LSE_t = -inf and the return value
 * SQZREF_ERR_EMPTY. */
int sqzref_attention(int B, int H, int n_q, int d, int64_t L, int n_u,
                     const double *Q, const double *K, const double *V, const uint8_t *keymask,
                     const double *Ku, const double *Vu, int causal, int n_q_total,
                     const int32_t *qpos, double scale, double *O, double *LSE)
{
    if (B < 1 || H < 1 || n_q < 1 || d < 1 || L < 0 || n_u < 0) return SQZREF_ERR_INVALID;
    int empty = 0;
#pragma omp parallel for schedule(dynamic) reduction(| : empty)
    for (int64_t row = 0; row < (int64_t)B * H * n_q; ++row) {
        int t = (int)(row % n_q);
        int64_t bh = row / n_q;
        int h = (int)(bh % H);
        const double *q = Q + (size_t)row * d;
        const double *Kh = K + (size_t)h * L * d;
        const double *Vh = V + (size_t)h * L * d;
        const uint8_t *mk = keymask ? keymask + (size_t)bh * L : NULL;
        const double *Kub = Ku ? Ku + (size_t)bh * n_u * d : NULL;
        const double *Vub = Vu ? Vu + (size_t)bh * n_u * d : NULL;
        int64_t tpos = qpos ? qpos[t] : t;
        int64_t u_last = causal ? tpos + n_u - n_q_total : (int64_t)n_u - 1; /* inclusive */
        if (u_last > (int64_t)n_u - 1) u_last = (int64_t)n_u - 1;

        /* pass 1: logits and max */
        double m = -INFINITY;
        for (int64_t j = 0; j < L; ++j) {
            if (mk && !mk[j]) continue;
            double z = 0.0;
            for (int k = 0; k < d; ++k) z += q[k] * Kh[(size_t)j * d + k];
            z *= scale;
            if (z > m) m = z;
        }
        for (int64_t u = 0; u <= u_last; ++u) {
            double z = 0.0;
            for (int k = 0; k < d; ++k) z += q[k] * Kub[(size_t)u * d + k];
            z *= scale;
            if (z > m) m = z;
        }
        double *o = O + (size_t)row * d;
        for (int k = 0; k < d; ++k) o[k] = 0.0;
        if (m == -INFINITY) { LSE[row] = -INFINITY; empty |= 1; continue; }

        /* pass 2: denominator */
        double l = 0.0;
        for (int64_t j = 0; j < L; ++j) {
            if (mk && !mk[j]) continue;
            double z = 0.0;
            for (int k = 0; k < d; ++k) z += q[k] * Kh[(size_t)j * d + k];
            l += exp(scale * z - m);
        }
        for (int64_t u = 0; u <= u_last; ++u) {
            double z = 0.0;
            for (int k = 0; k < d; ++k) z += q[k] * Kub[(size_t)u * d + k];
            l += exp(scale * z - m);
        }
        double lse = m + log(l);
        LSE[row] = lse;

        /* pass 3: O = sum softmax * v */
        for (int64_t j = 0; j < L; ++j) {
            if (mk && !mk[j]) continue;
            double z = 0.0;
            for (int k = 0; k < d; ++k) z += q[k] * Kh[(size_t)j * d + k];
            double p = exp(scale * z - lse);
            for (int k = 0; k < d; ++k) o[k] += p * Vh[(size_t)j * d + k];
        }
        for (int64_t u = 0; u <= u_last; ++u) {
            double z = 0.0;
            for (int k = 0; k < d; ++k) z += q[k] * Kub[(size_t)u * d + k];
            double p = exp(scale * z - lse);
            for (int k = 0; k < d; ++k) o[k] += p * Vub[(size_t)u * d + k];
        }
    }
    return empty ? SQZREF_ERR_EMPTY : SQZREF_OK;
}

/* Merge of partial results ("merges the partial attention outputs,
 * while correcting the outputs using the partial Softmax denominators and max
 * values").  With LSE_p = m_p + log l_p each partial is already normalised:
 *   LSE = log sum_p exp(LSE_p),  O = sum_p exp(LSE_p - LSE) O_p.
 * A partial with LSE_p = -inf is the identity. */
void sqzref_merge(int P, int64_t rows, int d, const double *O_parts, const double *LSE_parts,
                  double *O, double *LSE)
{
    for (int64_t r = 0; r < rows; ++r) {
        double m = -INFINITY;
        for (int p = 0; p < P; ++p)
            if (LSE_parts[(size_t)p * rows + r] > m) m = LSE_parts[(size_t)p * rows + r];
        double *o = O + (size_t)r * d;
        for (int k = 0; k < d; ++k) o[k] = 0.0;
        if (m == -INFINITY) { LSE[r] = -INFINITY; continue; }
        double l = 0.0;
        for (int p = 0; p < P; ++p) l += exp(LSE_parts[(size_t)p * rows + r] - m);
        double lse = m + log(l);
        LSE[r] = lse;
        for (int p = 0; p < P; ++p) {
            double w = exp(LSE_parts[(size_t)p * rows + r] - lse);
            if (w == 0.0) continue;
            for (int k = 0; k < d; ++k) o[k] += w * O_parts[((size_t)p * rows + r) * d + k];
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Selection diagnostics.                               */
/*                                                                           */
/* App. A ("cumulative attention scores for the top 1% highest    */
/* scoring attention values"): per query row, the softmax over ALL fixed     */
/* keys a_j = exp(z_j - LSE), z_j = scale q.k_j, sorted descending; skew =   */
/* the sum of the n_top largest a_j ("up to a maximum of 1 ... sharper,      */
/* more skewed"; n_top = ceil(top_frac L)).                       */
/*                                                                           */
/* App. D (the "Ideal" lookup): "compute attention from the ...  */
/* query tokens to all of the fixed context keys", then "select the keys     */
/* whose attention scores are above the configured threshold": n_T = #{a_j > */
/* T}, mass_T = sum of those a_j.  Compared with the centroid selection      */
/* `sel` (k keys) at MATCHED budget: the ideal k-set = the k largest */
/* a_j (ties: lower key index first); recall = |sel n ideal_k| / k (1 when   */
/* k = 0); mass_sel = sum_{j in sel} a_j (the attention mass the centroid    */
/* selection retrieves); mass_ideal = sum of the k largest a_j (its upper    */
/* bound, "an upper bound on the attainable accuracy").                */
/* Q [B,H,d] (one decode query per (b,h)); K [H,L,d] original order; sel     */
/* [B,H,L] uint8 in original key order.  Outputs are [B,H].                  */
/* ------------------------------------------------------------------------ */
typedef struct { double a; int64_t j; } sqzref_rank_t;

static int rank_desc(const void *x, const void *y)
{
    const sqzref_rank_t *p = (const sqzref_rank_t *)x, *q = (const sqzref_rank_t *)y;
    if (p->a > q->a) return -1;
    if (p->a < q->a) return 1;
    return (p->j > q->j) - (p->j < q->j);
}

int sqzref_diagnostics(int B, int H, int d, int64_t L, const double *Q, const double *K,
                       const uint8_t *sel, double scale, int64_t n_top, double T,
                       double *skew, double *mass_sel, double *mass_ideal, double *recall,
                       int64_t *k_out, int64_t *n_T, double *mass_T)
{
    if (B < 1 || H < 1 || d < 1 || L < 1 || n_top < 1 || n_top > L || !(T >= 0.0))
        return SQZREF_ERR_INVALID;
#pragma omp parallel for schedule(dynamic)
    for (int64_t bh = 0; bh < (int64_t)B * H; ++bh) {
        const int h = (int)(bh % H);
        const double *q = Q + (size_t)bh * d;
        const double *Kh = K + (size_t)h * L * d;
        const uint8_t *sl = sel + (size_t)bh * L;
        sqzref_rank_t *r = (sqzref_rank_t *)malloc((size_t)L * sizeof(sqzref_rank_t));
        /* z_j and the softmax over all L fixed keys */
        double m = -INFINITY;
        for (int64_t j = 0; j < L; ++j) {
            double z = 0.0;
            for (int k = 0; k < d; ++k) z += q[k] * Kh[(size_t)j * d + k];
            r[j].a = scale * z;
            r[j].j = j;
            if (r[j].a > m) m = r[j].a;
        }
        double l = 0.0;
        for (int64_t j = 0; j < L; ++j) l += exp(r[j].a - m);
        const double lse = m + log(l);
        int64_t k = 0, nt = 0;
        double ms = 0.0, mt = 0.0;
        for (int64_t j = 0; j < L; ++j) {
            r[j].a = exp(r[j].a - lse);
            if (sl[j]) { ++k; ms += r[j].a; }
            if (T == 0.0 || r[j].a > T) { ++nt; mt += r[j].a; }   /* T = 0 selects all (R6) */
        }
        qsort(r, (size_t)L, sizeof(sqzref_rank_t), rank_desc);
        double sk = 0.0, mi = 0.0;
        int64_t hit = 0;
        for (int64_t t = 0; t < n_top; ++t) sk += r[t].a;
        for (int64_t t = 0; t < k; ++t) {
            mi += r[t].a;
            if (sl[r[t].j]) ++hit;
        }
        skew[bh] = sk;
        mass_sel[bh] = ms;
        mass_ideal[bh] = mi;
        recall[bh] = k ? (double)hit / (double)k : 1.0;
        k_out[bh] = k;
        n_T[bh] = nt;
        mass_T[bh] = mt;
        free(r);
    }
    return SQZREF_OK;
}

int sqzref_version(void) { return 1; }
