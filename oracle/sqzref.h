/*
 * sqzref.h -- CPU ORACLE for Squeezed Attention (arXiv 2411.09688).
 * TEST INFRASTRUCTURE ONLY (see sqzref.c).  Independent of include/sqz.h.
 */
#ifndef SQZREF_H
#define SQZREF_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { SQZREF_OK = 0, SQZREF_ERR_INVALID = 2, SQZREF_ERR_INVARIANT = 4, SQZREF_ERR_EMPTY = 7 };
enum { SQZREF_F32 = 0, SQZREF_BF16 = 1 };

double sqzref_round_bf16(double x);
void sqzref_round_array(double *x, int64_t n, int dtype);

int sqzref_kmeans(const double *X, int64_t n, int d, int c, const int64_t *init,
                  int max_iters, double tol, int32_t *assign, double *mu,
                  int *iters_out, double *objective);
void sqzref_cluster_means(const double *X, int64_t n, int d, int c, const int32_t *assign,
                          double *C, int32_t *N);
int sqzref_build_order(int64_t L, int c2, const int32_t *assign2, int c1, const int32_t *parent,
                       int32_t *l2_order, int32_t *perm, int32_t *key_off, int32_t *child_off);

void sqzref_scores(const double *q, const double *C, const int32_t *N, int d, int c,
                   int n_rows, const int32_t *rows, double scale,
                   double *s, double *S, double *lse_out);
void sqzref_select_singlepass(const double *s, const int32_t *N, int c, double T, uint8_t *sel);
int sqzref_lookup(int B, int H, int n_q, int d, const double *Q,
                  int levels, int c1, const double *C1, const int32_t *N1, const int32_t *child_off,
                  int c2, const double *C2, const int32_t *N2,
                  double scale, double T, double T1, const uint8_t *forced_l1,
                  uint8_t *sel2, double *Sbar2, uint8_t *surv1, double *Sbar1, double *lse);

int sqzref_lookup_ml(int B, int H, int n_q, int d, const double *Q, int Lv, const int32_t *c,
                     const double *const *C, const int32_t *const *N,
                     const int32_t *const *child_off, double scale, const double *T,
                     const uint8_t *const *forced, uint8_t *const *surv, double *const *Sbar,
                     double *lse);

int sqzref_attention(int B, int H, int n_q, int d, int64_t L, int n_u,
                     const double *Q, const double *K, const double *V, const uint8_t *keymask,
                     const double *Ku, const double *Vu, int causal, int n_q_total,
                     const int32_t *qpos, double scale, double *O, double *LSE);
void sqzref_merge(int P, int64_t rows, int d, const double *O_parts, const double *LSE_parts,
                  double *O, double *LSE);
int sqzref_diagnostics(int B, int H, int d, int64_t L, const double *Q, const double *K,
                       const uint8_t *sel, double scale, int64_t n_top, double T,
                       double *skew, double *mass_sel, double *mass_ideal, double *recall,
                       int64_t *k_out, int64_t *n_T, double *mass_T);
int sqzref_version(void);

#ifdef __cplusplus
}
#endif
#endif
