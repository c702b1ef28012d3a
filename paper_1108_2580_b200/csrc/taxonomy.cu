// MFITR taxonomy term as a segmented reduction (sm_100a).
//
// The reference applies its graph regulariser by SGD over the sorted edge
// list (_kernels.edge_pass_range, reference _kernels.py:128-148); its exact
// gradient (mfitr.grad_mfitr, mfitr.py:269-273) is 2 (l3 + l4) w_e (q_c - q_p)
// on the child and the negative on the parent.  In an exact block solve of
// item i that term contributes tau * S_i * q_i to the normal matrix and
// tau * T_i to the right-hand side, tau = l3 + l4, with
//     S_i = sum_{e incident to i} w_e,   T_i = sum_{e incident} w_e q_other(e).
// A team of lanes per item walks the item's incident edges in CSR (= edge-list)
// order, lanes own float4 column blocks of q, so the sums have a fixed order.
#include "common.cuh"
#include "../../include/mcf.h"

namespace mcf {
namespace {

// A team of TL lanes per item (TL = the power of two >= ld/4, so D = 20
// packs 4 items into a warp instead of leaving 26 lanes idle); lane sub of
// the team owns float4 column block sub of T_i.  Per item and column the
// sums run in edge order exactly as before.
__global__ void __launch_bounds__(256) k_tax_terms(const int64_t *inc_ptr, const int32_t *inc_edge,
                                                   const int32_t *inc_other, const float *w,
                                                   const float *q, int32_t n_items, int ld,
                                                   const int32_t *row_list, int32_t n_list,
                                                   float *S, float *T, int TL) {
    const int lane = threadIdx.x & 31;
    const int team = lane / TL, sub = lane % TL;
    const int64_t j = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * (32 / TL) +
                      team;
    if (j >= n_list) return;
    const int i = row_list ? row_list[j] : (int)j;
    const int nq = ld / 4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float s = 0.f;
    for (int64_t e = inc_ptr[i]; e < inc_ptr[i + 1]; ++e) {
        const float we = w[inc_edge[e]];
        const int o = inc_other[e];
        s += we;
        if (sub < nq) {
            const float4 v = reinterpret_cast<const float4 *>(q + (size_t)o * ld)[sub];
            acc.x = fmaf(we, v.x, acc.x);
            acc.y = fmaf(we, v.y, acc.y);
            acc.z = fmaf(we, v.z, acc.z);
            acc.w = fmaf(we, v.w, acc.w);
        }
    }
    if (sub == 0) S[i] = s;
    if (sub < nq) reinterpret_cast<float4 *>(T + (size_t)i * ld)[sub] = acc;
}

}  // namespace
}  // namespace mcf

using namespace mcf;

extern "C" int mcf_taxonomy_terms(const int64_t *inc_ptr, const int32_t *inc_edge,
                                  const int32_t *inc_other, const float *edge_w, const float *q,
                                  int32_t n_items, int32_t D, const int32_t *row_list,
                                  int32_t n_list, float *S_out, float *T_out, void *stream) {
    if (D < 1 || D > mcf_max_dim() || n_items < 0 || !inc_ptr || !q || !S_out || !T_out) {
        set_error("mcf_taxonomy_terms: invalid arguments");
        return MCF_E_ARG;
    }
    const int32_t n = row_list ? n_list : n_items;
    if (n <= 0) return MCF_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int ld = mcf_factor_ld(D);
    int TL = 1;
    while (TL < ld / 4) TL <<= 1;          // ld <= 128 -> TL <= 32
    const int64_t per_block = 8 * (32 / TL);
    k_tax_terms<<<(unsigned)ceil_div(n, per_block), 256, 0, s>>>(inc_ptr, inc_edge, inc_other,
                                                                 edge_w, q, n_items, ld, row_list,
                                                                 n, S_out, T_out, TL);
    return check_launch("mcf_taxonomy_terms");
}

// ---------------------------------------------------------------------------
// Edge weights w_e = max(0, adjusted_cosine(child, parent)) on device.
//
// Reference: mfitr.edge_weights (mfitr.py:78-89) -> neighborhood.adjusted_cosine
// / _kernels.ac_pair (neighborhood.py:58-89, _kernels.py:218-244) over the
// item lists of (user ascending, rating - user mean) (neighborhood.py:37-55).
// All float64, in the reference's order, so the weights are bit-identical:
//   * user means: each user's ratings summed sequentially in record order
//     (np.bincount(users, weights=scores) accumulates in record order);
//   * per-item lists ordered by user: the item CSC is built (stable) from the
//     records in by-user order, so inside an item users ascend;
//   * one thread per edge walks the SHORTER list in ascending user order and
//     finds each user in the longer list by galloping search, so co-raters
//     are visited in ascending user order -- the same sequence of f64 adds
//     as the reference's two-pointer merge.
namespace mcf {
namespace {

__global__ void k_user_means(const int64_t *uptr, const float *uval, int32_t n_users,
                             double *mean) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n_users) return;
    double s = 0.0;
    const int64_t a = uptr[u], b = uptr[u + 1];
    for (int64_t k = a; k < b; ++k) s = __dadd_rn(s, (double)uval[k]);
    mean[u] = b > a ? __ddiv_rn(s, (double)(b - a)) : 0.0;
}

__global__ void k_rows_of(const int64_t *ptr, int32_t n_rows, int32_t *row_of) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rows) return;
    for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) row_of[k] = (int32_t)r;
}

__global__ void k_centered(const int32_t *perm, const float *uval, const int32_t *users_sorted,
                           const double *mean, int64_t nnz, double *cv) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
         k += (int64_t)gridDim.x * blockDim.x)
        cv[k] = __dsub_rn((double)uval[perm[k]], mean[users_sorted[k]]);
}

__device__ __forceinline__ int64_t gallop(const int32_t *a, int64_t lo, int64_t hi, int32_t x) {
    // first position in [lo, hi) with a[pos] >= x
    int64_t step = 1, prev = lo;
    while (lo < hi && a[lo] < x) {
        prev = lo;
        lo = min(hi, lo + step);
        step <<= 1;
    }
    int64_t l = prev, h = lo;
    while (l < h) {
        const int64_t m = (l + h) >> 1;
        if (a[m] < x) l = m + 1;
        else h = m;
    }
    return l;
}

__global__ void k_edge_ac(const int32_t *ec, const int32_t *ep, int64_t E, const int64_t *iptr,
                          const int32_t *iuser, const double *cv, int32_t n_items, double *w) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    const int c = ec[e], p = ep[e];
    double out = 0.0;
    if (c >= 0 && c < n_items && p >= 0 && p < n_items) {
        int64_t a0 = iptr[c], a1 = iptr[c + 1], b0 = iptr[p], b1 = iptr[p + 1];
        const bool swap = (a1 - a0) > (b1 - b0);  // walk the shorter list
        double num = 0.0, di = 0.0, dj = 0.0;
        int64_t n = 0;
        int64_t s0 = swap ? b0 : a0, s1 = swap ? b1 : a1, l0 = swap ? a0 : b0, l1 = swap ? a1 : b1;
        for (int64_t k = s0; k < s1 && l0 < l1; ++k) {
            const int32_t uk = iuser[k];
            l0 = gallop(iuser, l0, l1, uk);
            if (l0 < l1 && iuser[l0] == uk) {
                const double x = swap ? cv[l0] : cv[k];   // child's value
                const double y = swap ? cv[k] : cv[l0];   // parent's value
                // explicit roundings: no FMA contraction, the reference
                // (numba, no fastmath) rounds every product and sum
                num = __dadd_rn(num, __dmul_rn(x, y));
                di = __dadd_rn(di, __dmul_rn(x, x));
                dj = __dadd_rn(dj, __dmul_rn(y, y));
                ++n;
                ++l0;
            }
        }
        if (n > 0 && di != 0.0 && dj != 0.0) {
            const double s = __ddiv_rn(num, __dsqrt_rn(__dmul_rn(di, dj)));
            out = s > 0.0 ? s : 0.0;
        }
    }
    w[e] = out;
}

}  // namespace
}  // namespace mcf

extern "C" size_t mcf_edge_weights_workspace_bytes(int64_t nnz, int32_t n_users, int32_t n_items) {
    size_t b = 0;
    b += align_up(sizeof(double) * (size_t)n_users, 256);          // means
    b += align_up(sizeof(int32_t) * (size_t)nnz, 256) * 3;         // user_of, iuser, perm
    b += align_up(sizeof(int64_t) * ((size_t)n_items + 1), 256);   // iptr
    b += align_up(sizeof(float) * (size_t)nnz, 256);               // dummy vals out
    b += align_up(sizeof(double) * (size_t)nnz, 256);              // cv
    b += mcf_csr_workspace_bytes(nnz, n_items) + 256;
    return b;
}

extern "C" int mcf_edge_weights(const int64_t *uptr, const int32_t *uidx, const float *uval,
                                int32_t n_users, int32_t n_items, const int32_t *ec,
                                const int32_t *ep, int64_t E, double *w_out, void *ws,
                                size_t ws_bytes, void *stream) {
    if (n_users < 0 || n_items < 0 || E < 0 || !uptr || (E > 0 && (!ec || !ep || !w_out))) {
        set_error("mcf_edge_weights: invalid arguments");
        return MCF_E_ARG;
    }
    if (E == 0) return MCF_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int64_t nnz = 0;
    int rc;
    if ((rc = cuda_status(cudaMemcpyAsync(&nnz, uptr + n_users, sizeof(int64_t),
                                          cudaMemcpyDeviceToHost, s), "memcpy")))
        return rc;
    if ((rc = cuda_status(cudaStreamSynchronize(s), "sync"))) return rc;
    if (!ws || ws_bytes < mcf_edge_weights_workspace_bytes(nnz, n_users, n_items)) {
        set_error("mcf_edge_weights: workspace too small");
        return MCF_E_WORKSPACE;
    }
    Carve c(ws, ws_bytes);
    double *mean = c.take<double>((size_t)n_users);
    int32_t *user_of = c.take<int32_t>((size_t)nnz);
    int32_t *iuser = c.take<int32_t>((size_t)nnz);
    int32_t *perm = c.take<int32_t>((size_t)nnz);
    int64_t *iptr = c.take<int64_t>((size_t)n_items + 1);
    float *dummy = c.take<float>((size_t)nnz);
    double *cv = c.take<double>((size_t)nnz);
    const size_t csr_need = mcf_csr_workspace_bytes(nnz, n_items);
    void *csr_ws = c.take<char>(csr_need);
    if (!c.ok()) {
        set_error("mcf_edge_weights: workspace too small");
        return MCF_E_WORKSPACE;
    }
    if (n_users > 0) {
        k_user_means<<<(unsigned)ceil_div(n_users, 256), 256, 0, s>>>(uptr, uval, n_users, mean);
        k_rows_of<<<(unsigned)ceil_div(n_users, 256), 256, 0, s>>>(uptr, n_users, user_of);
    }
    // items keyed CSC of the by-user records: users ascend inside an item
    if ((rc = mcf_csr_build(uidx, user_of, uval, nnz, n_items, iptr, iuser, dummy, perm, csr_ws,
                            csr_need, stream)))
        return rc;
    if (nnz > 0) k_centered<<<148 * 8, 256, 0, s>>>(perm, uval, iuser, mean, nnz, cv);
    k_edge_ac<<<(unsigned)ceil_div(E, 128), 128, 0, s>>>(ec, ep, E, iptr, iuser, cv, n_items,
                                                          w_out);
    return check_launch("mcf_edge_weights");
}
