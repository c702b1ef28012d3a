/*
 * CPU ORACLE -- test infrastructure only.  Nothing in the product path
 * (paper_1108_2580_b200/) may link, load or call this file; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * use it, as the checker and as the reported CPU baseline.
 *
 * A float64 C restatement of the reference's ALS hot path
 * (/root/reference/pkg/src/multicf, Python + numba):
 *
 *   oracle_side_csr       <- factor._side_csr            factor.py:493-509
 *                            (stable argsort by key == counting sort)
 *   oracle_als_solve_rows <- _kernels.als_solve_rows     _kernels.py:151-215
 *   oracle_als_half_step  <- factor.als_half_step        factor.py:512-538
 *                            + parallel.run_blocks / even_bounds
 *                                                         parallel.py:134-145
 *   oracle_predict        <- _kernels.mf_predict_batch   _kernels.py:331-375
 *                            (ALS and MFITR branches: no time, no implicit)
 *   oracle_ac_pair        <- _kernels.ac_pair            _kernels.py:218-244
 *
 * Arithmetic is written in the reference's operation order and compiled with
 * -ffp-contract=off, so for plain lambda (lam_n = 0, no taxonomy terms) it is
 * bit-identical to the numba kernel (pinned by tests/test_oracle.py against
 * fixtures produced by the reference itself, tests/golden/make_golden.py).
 *
 * Generalisation used by the device path:
 *   A_r = sum_k w_k x_k x_k^T + (lam_c + lam_n * n_r + tau * S_r) I
 *   b_r = sum_k w_k y_k x_k + tau * T_r
 * With lam_n = tau = 0 the diagonal seed is exactly lam_c, as in the
 * reference (`A[i, i] = lam` before accumulation, _kernels.py:172-176).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Stable counting sort of records by key: ptr[n+1], and the gathered cols /
 * vals / wts in (key, record) order -- identical to
 * order = argsort(keys, kind="stable"); cols[order] ... (factor.py:502-509). */
int oracle_side_csr(const int64_t *keys, const int64_t *cols, const double *vals,
                    const double *wts, int64_t nnz, int64_t n_rows, int64_t *ptr,
                    int64_t *idx_out, double *val_out, double *wts_out,
                    int64_t *perm_out) {
    int64_t *cur = (int64_t *)calloc((size_t)n_rows + 1, sizeof(int64_t));
    if (!cur) return -1;
    for (int64_t k = 0; k < nnz; ++k) {
        if (keys[k] < 0 || keys[k] >= n_rows) { free(cur); return -2; }
        cur[keys[k] + 1]++;
    }
    for (int64_t r = 0; r < n_rows; ++r) cur[r + 1] += cur[r];
    memcpy(ptr, cur, sizeof(int64_t) * ((size_t)n_rows + 1));
    for (int64_t k = 0; k < nnz; ++k) {
        int64_t dst = cur[keys[k]]++;
        idx_out[dst] = cols[k];
        val_out[dst] = vals[k];
        if (wts_out) wts_out[dst] = wts ? wts[k] : 1.0;
        if (perm_out) perm_out[dst] = k;
    }
    free(cur);
    return 0;
}

/* One block of rows [lo, hi).  Returns -1, or the first failing row of the
 * block (the block stops there, like the reference, _kernels.py:197-203). */
int64_t oracle_als_solve_rows(int64_t lo, int64_t hi, const int64_t *ptr,
                              const int64_t *idx, const double *val, const double *wts,
                              const double *fixed, int64_t D, double *out, double lam_c,
                              double lam_n, const double *tax_S, const double *tax_T,
                              double tau) {
    double *A = (double *)malloc(sizeof(double) * (size_t)(D * D));
    double *b = (double *)malloc(sizeof(double) * (size_t)D);
    int64_t failed = -1;
    for (int64_t r = lo; r < hi && failed < 0; ++r) {
        const int64_t n = ptr[r + 1] - ptr[r];
        const double S = tax_S ? tax_S[r] : 0.0;
        if (n == 0 && S == 0.0) {
            /* empty row: zero when regularised, singular otherwise (:164-171) */
            if (lam_c > 0.0 || lam_n > 0.0) {
                for (int64_t d = 0; d < D; ++d) out[r * D + d] = 0.0;
                continue;
            }
            failed = r;
            break;
        }
        double diag = lam_c;
        if (lam_n != 0.0) diag = diag + lam_n * (double)n;
        if (tax_S) diag = diag + tau * S;
        for (int64_t i = 0; i < D; ++i) {
            b[i] = tax_T ? tau * tax_T[r * D + i] : 0.0;
            for (int64_t j = 0; j <= i; ++j) A[i * D + j] = 0.0;
            A[i * D + i] = diag;
        }
        for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) {
            const double *f = fixed + idx[k] * D;
            const double wv = wts ? wts[k] : 1.0;
            const double v = wv * val[k];
            for (int64_t i = 0; i < D; ++i) {
                const double fi = f[i];
                b[i] += v * fi;
                const double wfi = wv * fi;
                for (int64_t j = 0; j <= i; ++j) A[i * D + j] += wfi * f[j];
            }
        }
        /* row-oriented in-place Cholesky, lower triangle (:187-200) */
        int ok = 1;
        for (int64_t i = 0; i < D && ok; ++i) {
            for (int64_t j = 0; j < i; ++j) {
                double s = A[i * D + j];
                for (int64_t k2 = 0; k2 < j; ++k2) s -= A[i * D + k2] * A[j * D + k2];
                A[i * D + j] = s / A[j * D + j];
            }
            double s = A[i * D + i];
            for (int64_t k2 = 0; k2 < i; ++k2) s -= A[i * D + k2] * A[i * D + k2];
            if (!(s > 0.0) || !isfinite(s)) { ok = 0; break; }
            A[i * D + i] = sqrt(s);
        }
        if (!ok) { failed = r; break; }
        for (int64_t i = 0; i < D; ++i) {                 /* L y = b  (:204-208) */
            double s = b[i];
            for (int64_t k2 = 0; k2 < i; ++k2) s -= A[i * D + k2] * b[k2];
            b[i] = s / A[i * D + i];
        }
        for (int64_t i = D - 1; i >= 0; --i) {            /* L^T x = y (:209-213) */
            double s = b[i];
            for (int64_t k2 = i + 1; k2 < D; ++k2) s -= A[k2 * D + i] * b[k2];
            b[i] = s / A[i * D + i];
        }
        for (int64_t d = 0; d < D; ++d) out[r * D + d] = b[d];
    }
    free(A);
    free(b);
    return failed;
}

typedef struct {
    int64_t lo, hi;
    const int64_t *ptr, *idx;
    const double *val, *wts, *fixed, *tax_S, *tax_T;
    int64_t D;
    double *out;
    double lam_c, lam_n, tau;
    int64_t failed;
} block_arg;

static void *block_main(void *p) {
    block_arg *a = (block_arg *)p;
    a->failed = oracle_als_solve_rows(a->lo, a->hi, a->ptr, a->idx, a->val, a->wts, a->fixed,
                                      a->D, a->out, a->lam_c, a->lam_n, a->tax_S, a->tax_T,
                                      a->tau);
    return NULL;
}

/* Rows [row_lo, row_hi) split into `threads` equal-row static blocks
 * (even_bounds, parallel.py:144-145), one pthread per block.  Output is
 * independent of the thread count.  Returns the minimum failing row or -1
 * (factor.py:535-537). */
int64_t oracle_als_half_step(int64_t row_lo, int64_t row_hi, const int64_t *ptr,
                             const int64_t *idx, const double *val, const double *wts,
                             const double *fixed, int64_t D, double *out, double lam_c,
                             double lam_n, const double *tax_S, const double *tax_T,
                             double tau, int threads) {
    if (threads < 1) threads = 1;
    const int64_t n = row_hi - row_lo;
    block_arg *args = (block_arg *)calloc((size_t)threads, sizeof(block_arg));
    pthread_t *tid = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) {
        /* np.linspace(0, n, threads + 1).astype(int64) */
        const int64_t lo = row_lo + (int64_t)((double)n * t / threads);
        const int64_t hi = row_lo + (t + 1 == threads ? n : (int64_t)((double)n * (t + 1) / threads));
        block_arg a = {lo, hi, ptr, idx, val, wts, fixed, tax_S, tax_T, D, out,
                       lam_c, lam_n, tau, -1};
        args[t] = a;
        if (threads == 1) block_main(&args[t]);
        else pthread_create(&tid[t], NULL, block_main, &args[t]);
    }
    int64_t failed = -1;
    for (int t = 0; t < threads; ++t) {
        if (threads > 1) pthread_join(tid[t], NULL);
        if (args[t].failed >= 0 && (failed < 0 || args[t].failed < failed)) failed = args[t].failed;
    }
    free(args);
    free(tid);
    return failed;
}

/* The same half-step with rows handed out dynamically (an atomic counter,
 * 16 rows at a time) instead of static blocks: rows are independent, so the
 * output is bit-identical to oracle_als_half_step; used to check full-size
 * configurations, whose Zipf-hot rows serialise static blocks.  The minimum
 * failing row is returned, but a failing row does not stop other rows. */
typedef struct {
    block_arg base;
    int64_t *next;
} dyn_arg;

static void *dyn_main(void *p) {
    dyn_arg *a = (dyn_arg *)p;
    block_arg *b = &a->base;
    for (;;) {
        const int64_t lo = __atomic_fetch_add(a->next, 16, __ATOMIC_RELAXED);
        if (lo >= b->hi) break;
        const int64_t hi = lo + 16 < b->hi ? lo + 16 : b->hi;
        for (int64_t r = lo; r < hi; ++r) {
            int64_t f = oracle_als_solve_rows(r, r + 1, b->ptr, b->idx, b->val, b->wts, b->fixed,
                                              b->D, b->out, b->lam_c, b->lam_n, b->tax_S,
                                              b->tax_T, b->tau);
            if (f >= 0 && (b->failed < 0 || f < b->failed)) b->failed = f;
        }
    }
    return NULL;
}

int64_t oracle_als_half_step_dynamic(int64_t row_lo, int64_t row_hi, const int64_t *ptr,
                                     const int64_t *idx, const double *val, const double *wts,
                                     const double *fixed, int64_t D, double *out, double lam_c,
                                     double lam_n, const double *tax_S, const double *tax_T,
                                     double tau, int threads) {
    if (threads < 1) threads = 1;
    int64_t next = row_lo;
    dyn_arg *args = (dyn_arg *)calloc((size_t)threads, sizeof(dyn_arg));
    pthread_t *tid = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) {
        block_arg a = {row_lo, row_hi, ptr, idx, val, wts, fixed, tax_S, tax_T, D, out,
                       lam_c, lam_n, tau, -1};
        args[t].base = a;
        args[t].next = &next;
        pthread_create(&tid[t], NULL, dyn_main, &args[t]);
    }
    int64_t failed = -1;
    for (int t = 0; t < threads; ++t) {
        pthread_join(tid[t], NULL);
        const int64_t f = args[t].base.failed;
        if (f >= 0 && (failed < 0 || f < failed)) failed = f;
    }
    free(args);
    free(tid);
    return failed;
}

/* mu + b_u + b_i (+ b_a) + (q_i (+ q_a)) . p_u with the reference's
 * cold-start rules (_kernels.py:344-375); arts may be NULL (ALS). */
void oracle_predict(const int64_t *qu, const int64_t *qi, int64_t n, double mu,
                    const double *b_u, int64_t n_users, const double *b_i, int64_t n_items,
                    const double *P, const double *Q, int64_t D, const int64_t *arts,
                    const double *b_a, const double *Q_a, double *out) {
    for (int64_t t = 0; t < n; ++t) {
        const int64_t u = qu[t], i = qi[t];
        const int know_u = u >= 0 && u < n_users, know_i = i >= 0 && i < n_items;
        const int64_t a = arts ? arts[t] : -1;
        double pred = mu;
        if (know_u) pred += b_u ? b_u[u] : 0.0;
        if (know_i) {
            pred += b_i ? b_i[i] : 0.0;
            if (a >= 0) pred += b_a[a];
        }
        if (know_u && know_i) {
            double dot = 0.0;
            for (int64_t d = 0; d < D; ++d) {
                double qe = Q[i * D + d];
                if (a >= 0) qe += Q_a[a * D + d];
                dot += qe * P[u * D + d];
            }
            pred += dot;
        }
        out[t] = pred;
    }
}

/* Adjusted cosine of two user-sorted centred rating lists, merged in
 * ascending user order (_kernels.py:218-244). */
double oracle_ac_pair(const int64_t *ui, const double *ci, int64_t ni, const int64_t *uj,
                      const double *cj, int64_t nj) {
    int64_t a = 0, b = 0, n = 0;
    double num = 0.0, di = 0.0, dj = 0.0;
    while (a < ni && b < nj) {
        if (ui[a] < uj[b]) ++a;
        else if (ui[a] > uj[b]) ++b;
        else {
            const double x = ci[a], y = cj[b];
            num += x * y;
            di += x * x;
            dj += y * y;
            ++n; ++a; ++b;
        }
    }
    if (n == 0 || di == 0.0 || dj == 0.0) return 0.0;
    return num / sqrt(di * dj);
}

/* Edge weights max(0, AC(child, parent)) over a prebuilt item CSR of
 * (user ascending, centred rating) -- mfitr.edge_weights (mfitr.py:78-89)
 * evaluated with one cached _item_csr (neighborhood.py:46-55). */
void oracle_edge_weights(const int64_t *ec, const int64_t *ep, int64_t E, const int64_t *iptr,
                         const int64_t *iusers, const double *icv, int64_t n_items,
                         double *w) {
    for (int64_t e = 0; e < E; ++e) {
        const int64_t c = ec[e], p = ep[e];
        double s = 0.0;
        if (c >= 0 && c < n_items && p >= 0 && p < n_items)
            s = oracle_ac_pair(iusers + iptr[c], icv + iptr[c], iptr[c + 1] - iptr[c],
                               iusers + iptr[p], icv + iptr[p], iptr[p + 1] - iptr[p]);
        w[e] = s > 0.0 ? s : 0.0;
    }
}
