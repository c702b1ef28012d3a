/*
 * libmcf -- C-ABI of the B200-native ALS / MFITR sweep (sm_100a).
 *
 * The drop-in boundary for the reference's numba operators.  Every pointer
 * is caller-owned CUDA device memory (the Python host passes
 * torch.Tensor.data_ptr()), `stream` is a cudaStream_t passed as void*, no
 * call allocates device memory, and every call returns 0 on success or a
 * negative MCF_E* code with a message readable through mcf_last_error().
 * Calls are safe from any host thread on their own stream with disjoint
 * outputs.  Factor matrices are row-major [rows][ld] float32 with
 * ld = mcf_factor_ld(D) = round_up(D, 4) for D <= 4, else round_up(D, 8)
 * (whole 32-byte sectors), and zero padding columns.
 *
 * Reference operator each entry point replaces (paths relative to
 * /root/reference/pkg/src/multicf):
 *   mcf_csr_build      factor._side_csr                 factor.py:493-509
 *                      (+ np.bincount degrees, data.Dataset.by_user data.py:132-142)
 *   mcf_als_plan       parallel.run_blocks/even_bounds   parallel.py:134-145
 *   mcf_als_half_step  _kernels.als_solve_rows           _kernels.py:151-215
 *                      driven as factor.als_half_step    factor.py:512-538
 *   mcf_taxonomy_terms the graph term of mfitr.grad_mfitr mfitr.py:269-273
 *                      (ALS form of _kernels.edge_pass_range _kernels.py:128-148)
 *   mcf_edge_weights   mfitr.edge_weights / _kernels.ac_pair mfitr.py:78-89,
 *                      _kernels.py:218-244, neighborhood.py:37-89
 *   mcf_predict_sse    _kernels.mf_predict_batch         _kernels.py:331-375
 *                      + clip + squared error (factor.py:613-616, evaluation.py:11-18)
 *   mcf_sq_norms       the regulariser of factor.als_objective factor.py:541-547
 *                      / factor.loss_mf (factor.py:270-278)
 *   mcf_add_gathered   q_i + q_a[artist(i)] of mfitr._rating_terms mfitr.py:203-216
 *   mcf_als_half_step_peers the half-step + the replica all-gather of the
 *                      multi-GPU sweep (the reference is single-process)
 *   mcf_als_half_step_bias  the lam1 (bias) / lam2 (factor) regularisers of
 *                      mfitr.loss_mfitr for augmented [f | b] blocks  mfitr.py:226-242
 *   mcf_mfitr_sgd_epoch  mfitr.sgd_epoch_mfitr (the reference's SGD trainer) mfitr.py:323-336
 *   mcf_mfitr_fixed, mcf_mfitr_targets  the block terms of mfitr._rating_terms
 *                      (prediction mu + b_u + b_i + b_a + (q_i + q_a).p_u)  mfitr.py:203-216
 *   mcf_als_half_step_multicast  the half-step + the replica all-gather through
 *                      one NVLS multicast store per element
 *   mcf_comm_*, mcf_allgather_rows  the exchange of the row-sharded sweep
 *                      (SURVEY §8(b)); the reference's worker layer that hands
 *                      row blocks to threads, parallel.py:101-145
 */
#ifndef MCF_H
#define MCF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    MCF_OK = 0,
    MCF_E_ARG = -1,        /* invalid argument (null pointer, bad size, bad D) */
    MCF_E_WORKSPACE = -2,  /* workspace smaller than *_workspace_bytes()      */
    MCF_E_RANGE = -3,      /* a key / id outside its declared range            */
    MCF_E_CUDA = -4,       /* a CUDA runtime error (message has the details)   */
    MCF_E_UNSUPPORTED = -5 /* D outside the compiled range (1..128)            */
};

int mcf_version(void);
const char *mcf_last_error(void);
int mcf_factor_ld(int D);
int mcf_max_dim(void);

/* ---- rating layout: stable CSR (by user) / CSC (by item) build ----------
 * Rows keyed by keys[k] in [0, n_rows); in-row order == record order (the
 * reference's argsort(kind="stable")).  ptr_out[n_rows+1] int64,
 * idx_out[nnz] = cols in that order, val_out[nnz] = vals in that order,
 * perm_out[nnz] (nullable) = the record index of each CSR slot.
 * Synchronises `stream` once to report out-of-range keys (MCF_E_RANGE). */
size_t mcf_csr_workspace_bytes(int64_t nnz, int32_t n_rows);
int mcf_csr_build(const int32_t *keys, const int32_t *cols, const float *vals, int64_t nnz,
                  int32_t n_rows, int64_t *ptr_out, int32_t *idx_out, float *val_out,
                  int32_t *perm_out, void *ws, size_t ws_bytes, void *stream);

/* ---- ALS half-step --------------------------------------------------------
 * Work plan for a set of rows of one layout: the rows row_list[0..n_list)
 * (or, when row_list is NULL, rows row_lo .. row_lo + n_list), each cut into
 * chunks of at most `chunk` ratings and (D <= 20 path) sorted by length,
 * hot-row chunks first.  Built once per (layout, row set) and reused by
 * every half-step.  Synchronises `stream` once and fills the HOST array
 * totals[MCF_PLAN_INFO_LEN], which mcf_als_half_step takes as plan_info:
 *   [0] work items (D > 20 paths)   [1] partial slots (D > 20 paths)
 *   [2] tasks (D <= 20 path)        [3] partial slots (D <= 20 path)
 *   [4] hot rows (D <= 20 path)     [5] nnz the plan was sized for */
#define MCF_PLAN_INFO_LEN 6
size_t mcf_als_plan_bytes(int32_t n_list, int64_t nnz, int32_t chunk);
int mcf_als_plan(const int64_t *ptr, const int32_t *row_list, int32_t n_list, int32_t row_lo,
                 int32_t chunk, int64_t nnz, void *plan, size_t plan_bytes, int64_t *totals,
                 void *stream);
/* Bytes of half-step workspace: n_list row counters + `slots` partial
 * Grams at dimension D (slots = max(plan_info[3], plan_info[1])).
 * _fixed: also room for the tensor-core path (64 <= D <= 128, no
 * observation weights) -- its fp16 split tables of the n_fixed-row fixed
 * side and the split ratings of the layout's nnz (plan_info[5]); with the
 * plain query that path falls back to the CUDA-core kernels. */
size_t mcf_als_workspace_bytes(int32_t n_list, int64_t slots, int32_t D);
size_t mcf_als_workspace_bytes_fixed(int32_t n_list, int64_t slots, int32_t D, int64_t n_fixed,
                                     int64_t nnz);

/* Solve every planned row r exactly (Cholesky of the D x D system):
 *   A_r = sum_k w_k x_k x_k^T + (lam_c + lam_n * n_r + tau * S_r) I
 *   b_r = sum_k w_k (val_k - y_shift) x_k + tau * T_r
 *   out[r] = A_r^{-1} b_r
 * with x_k = fixed[idx[k]] (fixed: n_fixed rows), w_k = wts[k] (wts NULL -> 1),
 * n_r = ptr[r+1]-ptr[r],
 * S/T (nullable) the taxonomy terms of mcf_taxonomy_terms (T row-major, ld).
 * Plain ALS: lam_c = lam, lam_n = 0.  Weighted-lambda: lam_c = 0, lam_n = lam.
 * A row with no ratings and no taxonomy mass becomes 0 when lam_c > 0 or
 * lam_n > 0.  A row whose pivot is <= 0 or non-finite is left untouched and
 * *fail_row (device int64) receives the minimum such row (-1 = none); all
 * other rows still complete (the reference's failing block stops early,
 * _kernels.py:197-203).
 * obj_out (nullable, device double[2], D <= 20): the fused objective of the
 * solved rows, obj_out[0] = sum_r sum_k w_k (y_k - x_k^T out_r)^2 and
 * obj_out[1] = sum_r (lam_c + lam_n n_r) |out_r|^2, evaluated in the solve
 * epilogue from the Gram (sum w y^2 - b^T x - lam |x|^2) and summed in a fixed
 * order; exact for tau = 0 (the taxonomy term is not included). */
int mcf_als_half_step(const int64_t *ptr, const int32_t *idx, const float *val,
                      const float *wts, const float *fixed, int64_t n_fixed, float *out, int32_t D,
                      float lam_c, float lam_n, float y_shift, const float *tax_S,
                      const float *tax_T, float tau, const int32_t *row_list, int32_t n_list,
                      int32_t row_lo, int32_t chunk, const void *plan, const int64_t *plan_info,
                      int64_t *fail_row, double *obj_out, void *ws, size_t ws_bytes,
                      void *stream);

/* mcf_als_half_step with one "bias" coordinate (MFITR full blocks,
 * SURVEY §8(f)): coordinate bias_dim (0 <= bias_dim < D) of every row system
 * gets the regulariser bias_lam_c + bias_lam_n * n_r instead of
 * lam_c + lam_n * n_r + tau * S_r, and no taxonomy T term.  This is the
 * per-observation lam1 (biases) vs lam2 (factors) split of the reference's
 * loss_mfitr (mfitr.py:226-242) for the augmented unknowns [f | b].  No fused
 * objective.  Other arguments as mcf_als_half_step. */
int mcf_als_half_step_bias(const int64_t *ptr, const int32_t *idx, const float *val,
                           const float *wts, const float *fixed, int64_t n_fixed, float *out,
                           int32_t D, float lam_c, float lam_n, float y_shift,
                           const float *tax_S, const float *tax_T, float tau,
                           const int32_t *row_list, int32_t n_list, int32_t row_lo,
                           int32_t chunk, const void *plan, const int64_t *plan_info,
                           int64_t *fail_row, void *ws, size_t ws_bytes, int32_t bias_dim,
                           float bias_lam_c, float bias_lam_n, void *stream);

/* mcf_als_half_step fused with the all-gather of the row-sharded multi-GPU
 * sweep: every solved row of `out` (this rank's shard) is also
 * stored, by the solve kernel itself, at the same row offset of each of the
 * n_peers replicas in peer_out (a DEVICE array of n_peers float* -- NVLink
 * peer / symmetric-memory pointers to the peers' tables, already offset to
 * this rank's shard).  The caller orders the next half-step after every
 * rank's stores (a device barrier over the peers).  Other arguments as
 * mcf_als_half_step. */
int mcf_als_half_step_peers(const int64_t *ptr, const int32_t *idx, const float *val,
                            const float *wts, const float *fixed, int64_t n_fixed, float *out,
                            int32_t D, float lam_c, float lam_n, float y_shift,
                            const float *tax_S, const float *tax_T, float tau,
                            const int32_t *row_list, int32_t n_list, int32_t row_lo,
                            int32_t chunk, const void *plan, const int64_t *plan_info,
                            int64_t *fail_row, double *obj_out, void *ws, size_t ws_bytes,
                            float *const *peer_out, int32_t n_peers, void *stream);

/* mcf_als_half_step fused with the all-gather through NVLS multicast: every
 * solved row of this rank's shard is written with one multimem store to
 * mc_out, the multicast address of the replicated table (e.g. torch symmetric
 * memory's multicast_ptr, offset to this rank's shard), which reaches every
 * GPU's replica, this one's included -- `out` is not written separately.  The
 * caller orders the next half-step after every rank's stores (a device
 * barrier).  Other arguments as mcf_als_half_step. */
int mcf_als_half_step_multicast(const int64_t *ptr, const int32_t *idx, const float *val,
                                const float *wts, const float *fixed, int64_t n_fixed, float *out,
                                int32_t D, float lam_c, float lam_n, float y_shift,
                                const float *tax_S, const float *tax_T, float tau,
                                const int32_t *row_list, int32_t n_list, int32_t row_lo,
                                int32_t chunk, const void *plan, const int64_t *plan_info,
                                int64_t *fail_row, double *obj_out, void *ws, size_t ws_bytes,
                                float *mc_out, void *stream);

/* ---- multi-GPU exchange: libmcf's own NCCL communicator -------------------
 * For a C caller that shards the half-step over the GPUs of one node without
 * torch.distributed.  NCCL is loaded at run time (the copy already in the
 * process, else libnccl.so.2; MCF_NCCL_LIB overrides).  Rank 0 creates a
 * unique id (mcf_comm_id_bytes() bytes) and ships it to the other ranks by
 * any channel; every rank then calls mcf_comm_init on its own device.
 * mcf_allgather_rows: rows [offsets[k], offsets[k] + counts[k]) of the
 * [rows][ld] float table belong to rank k; afterwards every rank holds every
 * rank's rows (one grouped ncclBroadcast per rank, in place, exact sizes). */
size_t mcf_comm_id_bytes(void);
int mcf_comm_get_unique_id(void *id_out, size_t id_bytes);
int mcf_comm_init(const void *id, size_t id_bytes, int32_t nranks, int32_t rank,
                  void **comm_out);
int mcf_comm_destroy(void *comm);
int mcf_allgather_rows(void *comm, float *table, int32_t ld, const int64_t *offsets,
                       const int64_t *counts, void *stream);

/* ---- MFITR full-model blocks (mfitr.py:203-216 prediction) -----------------
 * Tables are [rows][mcf_factor_ld(D + 1)] with the factor in columns 0..D-1
 * and the bias in column D.
 * mcf_mfitr_fixed: the gather table of an augmented solve,
 *   out[r] = [main[r][:D] + (art && art[r] >= 0 ? add[art[r]][:D] : 0) | 1 | 0..]
 * (users step: main = Q, add = artist table; items / artists steps: main = P).
 * mcf_mfitr_targets: per-rating targets of one layout in CSR order,
 *   mode 0 (users layout, partner = item i):  r - mu - b_i - b_a[art(i)]
 *   mode 1 (items layout, row = item i, partner = user u, aux = i per rating):
 *                       r - mu - b_u - [art(i) >= 0] (b_a + q_a . p_u)
 *   mode 2 (artists layout, row = artist, partner = user u, aux = item i):
 *                       r - mu - b_u - b_i - q_i . p_u
 *   mode 3 (items layout, the artist terms left to the solve epilogue,
 *           mcf_als_half_step_mfitr_items): r - mu - b_u
 * (Pa = [p | b_u], Qa = [q | b_i], Aa = [q_a | b_a] indexed by artist id). */
int mcf_mfitr_fixed(const float *main_t, const float *add_t, const int32_t *art, int64_t n,
                    int32_t D, float *out, void *stream);

/* The reference's own MFITR trainer, one epoch of mfitr.sgd_epoch_mfitr
 * (mfitr.py:323-336; time / implicit terms off): users in order[0..n_order)
 * (the seeded shuffle), each user's ratings in the by-user layout's order
 * through _kernels.rate_update (_kernels.py:21-77), then the taxonomy edges
 * through _kernels.edge_pass_range (_kernels.py:129-148).  This entry:
 * Hogwild (a warp per user, item-side state updated without locks, atomic
 * adds in the edge pass), not bit-reproducible; mcf_mfitr_sgd_epoch_locked
 * below keeps the reference's per-item locking.  Tables [rows][ld(D)];
 * b_u/b_i/b_a float; art nullable (no artist terms); counter: one device
 * int32 of scratch.  workers: concurrent user warps (and edge warps) --
 * 1 reproduces the reference's single-thread order (strictly sequential),
 * <= 0 uses the whole GPU. */
int mcf_mfitr_sgd_epoch(const int64_t *uptr, const int32_t *uidx, const float *uval,
                        const int32_t *order, int32_t n_order, int32_t *counter, float *P,
                        float *Q, float *b_u, float *b_i, const int32_t *art, float *b_a,
                        float *Q_a, float mu, int32_t D, float gamma, float lam_bias,
                        float lam_fac, const int64_t *ec, const int64_t *ep, const double *w,
                        int64_t E, float lam3, float lam4, int32_t workers, void *stream);
/* The same epoch under the reference's LockTable contract (parallel.py:21-49,
 * factor.py:430-444, mfitr.py:298-320): every rating's
 * item-side update (q_i, b_i, q_a, b_a) holds one spin lock per item id --
 * the (item, artist) pair acquired in ascending id order, released after
 * the update -- and every edge update locks both endpoints, so no update is
 * lost for any worker count.  locks: int32[num_items], zeroed by the caller
 * (left zeroed). */
int mcf_mfitr_sgd_epoch_locked(const int64_t *uptr, const int32_t *uidx, const float *uval,
                               const int32_t *order, int32_t n_order, int32_t *counter, float *P,
                               float *Q, float *b_u, float *b_i, const int32_t *art, float *b_a,
                               float *Q_a, float mu, int32_t D, float gamma, float lam_bias,
                               float lam_fac, const int64_t *ec, const int64_t *ep,
                               const double *w, int64_t E, float lam3, float lam4,
                               int32_t workers, int32_t *locks, void *stream);
/* Stress test of that lock table: `workers` warps each take
 * `iters` ascending-order lock pairs over n_items ids and add 1 to both
 * locked accumulators acc[] non-atomically; afterwards sum(acc) must be
 * exactly 2 * workers * iters. */
int mcf_lock_stress(int32_t *locks, float *acc, int32_t n_items, int32_t workers, int32_t iters,
                    void *stream);
/* ALS-MFITR every-block sweep without per-rating target passes (D = factor
 * dimension + 1 bias, D <= 21: the Schur pair path).
 * mcf_als_half_step_mfitr = mcf_als_half_step_bias (bias in column D-1,
 * lam_c = 0) plus
 *  - ysub != 0: the partner rows are [x | 1 | t] (mcf_mfitr_fixed_bsub) and
 *    each rating's target is val - y_shift - t (items: t = b_u; users:
 *    t = b_i + b_a[art(i)]; val = the raw ratings, y_shift = mu);
 *  - emit (nullable): every row's augmented system [A | c | u | d | n]
 *    (packed lower A of the D-1 factor coordinates, rhs c, u = sum x,
 *    d = sum y, n; stride 256 floats, row r at emit + 256 r), stored before
 *  - corr_idx (nullable): the row's artist terms removed from its rhs through
 *    its own Gram: c -= A q_a + u b_a, d -= u.q_a + n b_a, [q_a | b_a] =
 *    corr_tab[corr_idx[r]] (corr_idx[r] < 0: none).
 * mcf_mfitr_artist_step then solves every artist's [q_a | b_a] from those
 * systems: A_a = sum_i A_i, rhs_a = sum_i (c_i - G_i [q_i | b_i]) over the
 * artist's items (art_ptr / art_items CSR, fixed order), regularised
 * lam_n n_a (factors) and bias_lam_n n_a (bias), n_a = cnt_ptr[r+1] -
 * cnt_ptr[r] for the artist's row r = artist_row[j]; results into Aa. */
int mcf_mfitr_fixed_bsub(const float *main_t, const float *add_t, const int32_t *art, int64_t n,
                         int32_t D, float *out, void *stream);
int mcf_als_half_step_mfitr(const int64_t *ptr, const int32_t *idx, const float *val,
                            const float *fixed, int64_t n_fixed, float *out, int32_t D,
                            float lam_n, float y_shift, const float *tax_S, const float *tax_T,
                            float tau, const int32_t *row_list, int32_t n_list, int32_t chunk,
                            const void *plan, const int64_t *plan_info, int64_t *fail_row,
                            void *ws, size_t ws_bytes, float bias_lam_n, float *emit,
                            const float *corr_tab, const int32_t *corr_idx, int32_t ysub,
                            void *stream);
size_t mcf_mfitr_artist_workspace_bytes(int32_t n_artists);
int mcf_mfitr_artist_step(const int64_t *art_ptr, const int32_t *art_items,
                          const int32_t *artist_row, int32_t n_artists, const int64_t *cnt_ptr,
                          const float *emit, const float *Qa, float *Aa, int32_t D, float lam_n,
                          float bias_lam_n, int64_t *fail_row, void *ws, size_t ws_bytes,
                          void *stream);
int mcf_mfitr_targets(int32_t mode, const int64_t *ptr, const int32_t *idx, const float *val,
                      const int32_t *aux, int32_t n_rows, const float *Pa, const float *Qa,
                      const float *Aa, const int32_t *art, float mu, int32_t D, float *out,
                      void *stream);

/* ---- MFITR taxonomy term (segmented reduction) ---------------------------
 * For each listed item i (row_list NULL -> all n_items):
 *   S[i] = sum_{e incident to i} w_e,   T[i] = sum_e w_e * q[other(e)]
 * over the incident-edge CSR (inc_ptr[n_items+1], inc_edge, inc_other),
 * summed in CSR order.  Only listed items are written. */
int mcf_taxonomy_terms(const int64_t *inc_ptr, const int32_t *inc_edge,
                       const int32_t *inc_other, const float *edge_w, const float *q,
                       int32_t n_items, int32_t D, const int32_t *row_list, int32_t n_list,
                       float *S_out, float *T_out, void *stream);

/* Edge weights w_e = max(0, adjusted cosine(child_e, parent_e)) over
 * co-raters, float64, bit-identical to the reference's mfitr.edge_weights
 * (ac_pair merge in ascending user order over ratings centred by the user
 * mean).  Input: the by-user layout (uptr[n_users+1], uidx = item, uval =
 * rating; in-row order = record order).  Synchronises `stream` once.
 * ws: mcf_edge_weights_workspace_bytes(nnz, n_users, n_items). */
size_t mcf_edge_weights_workspace_bytes(int64_t nnz, int32_t n_users, int32_t n_items);
int mcf_edge_weights(const int64_t *uptr, const int32_t *uidx, const float *uval,
                     int32_t n_users, int32_t n_items, const int32_t *ec, const int32_t *ep,
                     int64_t E, double *w_out, void *ws, size_t ws_bytes, void *stream);

/* ---- prediction / RMSE ----------------------------------------------------
 * pred = mu + b_u[u] + b_i[i] + b_a[a] + (q_i + q_a[a]) . p_u with the
 * reference's cold-start rules (unknown user or item keeps only the known
 * terms); a = art_of_item[i] (nullable -> no artist terms).  b_u/b_i/b_a
 * nullable (zeros).  pred_out (nullable) gets the unclipped prediction; when
 * truth is non-NULL, *sse_out (device double) = sum (clip(pred,lo,hi) -
 * truth)^2, reduced in a fixed order (deterministic).  ws:
 * mcf_predict_workspace_bytes(n). */
size_t mcf_predict_workspace_bytes(int64_t n);
int mcf_predict_sse(const int32_t *users, const int32_t *items, const float *truth, int64_t n,
                    const float *P, int32_t n_users, const float *Q, int32_t n_items, int32_t D,
                    float mu, const float *b_u, const float *b_i, const int32_t *art_of_item,
                    const float *b_a, const float *Q_a, float clip_lo, float clip_hi,
                    float *pred_out, double *sse_out, void *ws, size_t ws_bytes, void *stream);

/* *out (device double) = sum_r c_r |F_r|^2 with c_r = ptr[r+1]-ptr[r]
 * (ptr non-NULL: the per-observation regulariser) or 1.  Deterministic. */
int mcf_sq_norms(const float *F, int32_t n, int32_t D, const int64_t *ptr, double *out,
                 void *ws, size_t ws_bytes, void *stream);

/* out[i] = A[i] + B[map[i]] (map[i] < 0 -> A[i]); out may alias A. */
int mcf_add_gathered(const float *A, const float *B, const int32_t *map, int32_t n, int32_t D,
                     float *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MCF_H */
