// MFITR full-model blocks (sm_100a): the two gathers that turn the
// reference's MFITR prediction (mfitr.py:203-216, _rating_terms)
//     pred = mu + b_u + b_i + b_a[art(i)] + (q_i + q_a[art(i)]) . p_u
// into per-block least-squares problems for mcf_als_half_step_bias.  Every
// block solve is over an augmented unknown [f | b] (D factor columns, the
// bias in column D):
//   users   [p_u | b_u]: x = [q_i + q_a[art(i)] | 1], y = r - mu - b_i - b_a[art(i)]
//   items   [q_i | b_i]: x = [p_u | 1],                y = r - mu - b_u - b_a - q_a . p_u
//   artists [q_a | b_a]: x = [p_u | 1],                y = r - mu - b_u - b_i - q_i . p_u
// (the artist terms apply only when art(i) >= 0; q_a / b_a are indexed by the
// artist's item id, mfitr.py:92-149).  Factor tables are [rows][ld] with the
// bias in column D.
#include <cuda_runtime.h>
#include <algorithm>
#include <stdint.h>

#include "common.cuh"
#include "../../include/mcf.h"

namespace mcf {
namespace {

// out[r] = [main[r][:D] + (art[r] >= 0 ? add[art[r]][:D] : 0) | 1 | t | 0 ...] with
// t = main[r][D] + (art[r] >= 0 ? add[art[r]][D] : 0) when bsub (the block's
// per-rating bias subtrahend, read by the pair kernel's YSUB gather), else 0
__global__ void k_mfitr_fixed(const float *main_t, const float *add_t, const int32_t *art,
                              int64_t n, int D, int ld, float *out, int bsub) {
    const int64_t total = n * ld;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / ld;
        const int c = (int)(e - r * ld);
        float v = 0.f;
        if (c < D) {
            v = main_t[e];
            if (add_t && art) {
                const int a = art[r];
                if (a >= 0) v += add_t[(size_t)a * ld + c];
            }
        } else if (c == D) {
            v = 1.f;
        } else if (c == D + 1 && bsub) {
            v = main_t[r * ld + D];
            if (add_t && art) {
                const int a = art[r];
                if (a >= 0) v += add_t[(size_t)a * ld + D];
            }
        }
        out[e] = v;
    }
}

// dot of the first D floats of two 16-byte aligned rows (column D onwards
// holds the bias / padding and is excluded), float4 loads
__device__ __forceinline__ float dot_d(const float *a, const float *b, int D) {
    const float4 *a4 = reinterpret_cast<const float4 *>(a);
    const float4 *b4 = reinterpret_cast<const float4 *>(b);
    float d = 0.f;
    const int nf = D >> 2;
    for (int c = 0; c < nf; ++c) {
        const float4 x = a4[c], y = b4[c];
        d = fmaf(x.x, y.x, d);
        d = fmaf(x.y, y.y, d);
        d = fmaf(x.z, y.z, d);
        d = fmaf(x.w, y.w, d);
    }
    const int rem = D & 3;
    if (rem) {
        const float4 x = a4[nf], y = b4[nf];
        d = fmaf(x.x, y.x, d);
        if (rem > 1) d = fmaf(x.y, y.y, d);
        if (rem > 2) d = fmaf(x.z, y.z, d);
    }
    return d;
}

// per-rating targets of one layout, thread per rating (a warp per row
// serialised the Zipf-hot rows), ratings in CSR order.
// mode 0 users (partner i), 1 items (partner u, aux = row item),
// 2 artists (partner u, aux = item), 3 items without the artist terms (those
// are applied per row from the Gram in the solve epilogue: y - mu - b_u).
__global__ void k_mfitr_targets(int mode, const int64_t *ptr, const int32_t *idx,
                                const float *val, const int32_t *aux, int32_t n_rows,
                                const float *Pa, const float *Qa, const float *Aa,
                                const int32_t *art, float mu, int D, int ld, float *out) {
    const int64_t nnz = ptr[n_rows];
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int j = idx[k];
        float t = val[k] - mu;
        if (mode == 0) {            // j = item
            t -= Qa[(size_t)j * ld + D];
            const int aj = art[j];
            if (aj >= 0) t -= Aa[(size_t)aj * ld + D];
        } else if (mode == 1) {     // j = user, aux = the row's item
            const float *pu = Pa + (size_t)j * ld;
            t -= pu[D];
            const int ar = art[aux[k]];
            if (ar >= 0) {
                const float *qa = Aa + (size_t)ar * ld;
                t -= qa[D] + dot_d(qa, pu, D);
            }
        } else if (mode == 3) {     // j = user
            t -= Pa[(size_t)j * ld + D];
        } else {                    // j = user, aux = item
            const float *qi = Qa + (size_t)aux[k] * ld;
            const float *pu = Pa + (size_t)j * ld;
            t -= pu[D] + qi[D] + dot_d(qi, pu, D);
        }
        out[k] = t;
    }
}

}  // namespace
}  // namespace mcf

using namespace mcf;

extern "C" int mcf_mfitr_fixed(const float *main_t, const float *add_t, const int32_t *art,
                               int64_t n, int32_t D, float *out, void *stream) {
    if (!main_t || !out || n < 0 || D < 1 || D + 1 > 128) {
        set_error("mcf_mfitr_fixed: invalid arguments");
        return MCF_E_ARG;
    }
    const int ld = mcf_factor_ld(D + 1);
    const int64_t total = n * ld;
    if (total == 0) return MCF_OK;
    const int grid = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 32);
    k_mfitr_fixed<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(main_t, add_t, art, n, D,
                                                                       ld, out, 0);
    return check_launch("mcf_mfitr_fixed");
}

extern "C" int mcf_mfitr_fixed_bsub(const float *main_t, const float *add_t, const int32_t *art,
                                    int64_t n, int32_t D, float *out, void *stream) {
    if (!main_t || !out || n < 0 || D < 1 || D + 2 > mcf_factor_ld(D + 1)) {
        set_error("mcf_mfitr_fixed_bsub: invalid arguments (needs a spare column D + 1)");
        return MCF_E_ARG;
    }
    const int ld = mcf_factor_ld(D + 1);
    const int64_t total = n * ld;
    if (total == 0) return MCF_OK;
    const int grid = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 32);
    k_mfitr_fixed<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(main_t, add_t, art, n, D,
                                                                       ld, out, 1);
    return check_launch("mcf_mfitr_fixed_bsub");
}

extern "C" int mcf_mfitr_targets(int32_t mode, const int64_t *ptr, const int32_t *idx,
                                 const float *val, const int32_t *aux, int32_t n_rows,
                                 const float *Pa, const float *Qa, const float *Aa,
                                 const int32_t *art, float mu, int32_t D, float *out,
                                 void *stream) {
    if (mode < 0 || mode > 3 || !ptr || !out || n_rows < 0 || D < 1 || D + 1 > 128 ||
        (mode == 0 && (!Qa || !Aa || !art)) || (mode == 1 && (!Pa || !Aa || !art || !aux)) ||
        (mode == 3 && !Pa) ||
        (mode == 2 && (!Pa || !Qa || !aux))) {
        set_error("mcf_mfitr_targets: invalid arguments");
        return MCF_E_ARG;
    }
    if (n_rows == 0) return MCF_OK;
    const int ld = mcf_factor_ld(D + 1);
    const int grid = 148 * 16;   // grid-stride over the layout's ratings
    k_mfitr_targets<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        mode, ptr, idx, val, aux, n_rows, Pa, Qa, Aa, art, mu, D, ld, out);
    return check_launch("mcf_mfitr_targets");
}

// ---------------------------------------------------------------------------
// The reference's own MFITR trainer (SGD), SURVEY §8(f)3:
// mfitr.sgd_epoch_mfitr (mfitr.py:323-336) = factor._sgd_pass (users in a
// seeded shuffle, each user's ratings in record order through
// _kernels.rate_update, _kernels.py:21-77) + _kernels.edge_pass_range
// (_kernels.py:129-148).  Device form: a warp per user -- warps take users
// in shuffle order -- walks that user's ratings sequentially with the
// reference's update order (item side sees the pre-update user factor, the
// user side the pre-update effective item factor).
// Conflict handling, the reference's LockTable contract (parallel.py:21-49,
// factor.py:430-444): with `locks` every rating's
// item-side read-modify-write (q_i, b_i and the artist's q_a, b_a) runs
// under one spin lock per item id, the (item, artist) pair acquired in
// ascending id order and released right after the update; user state is
// warp-private.  The edge pass then locks both endpoints of each edge
// (mfitr.py:298-320) and applies the reference's two directed updates.
// Locked item data is read through L2 (ld.global.cg), so a warp never sees
// a stale L1 line of another SM's update.  Without locks: Hogwild.
namespace mcf {
namespace {

__device__ __forceinline__ void lock_ids(int32_t *locks, int a, int b) {
    // ascending id order, a pair or a single id (a == b or b < 0)
    const int lo = b < 0 ? a : min(a, b), hi = b < 0 ? a : max(a, b);
    while (atomicCAS(locks + lo, 0, 1) != 0) __nanosleep(32);
    if (hi != lo)
        while (atomicCAS(locks + hi, 0, 1) != 0) __nanosleep(32);
    __threadfence();
}
__device__ __forceinline__ void unlock_ids(int32_t *locks, int a, int b) {
    const int lo = b < 0 ? a : min(a, b), hi = b < 0 ? a : max(a, b);
    __threadfence();
    if (hi != lo) atomicExch(locks + hi, 0);
    atomicExch(locks + lo, 0);
}
template <bool LOCK>
__device__ __forceinline__ float ld_item(const float *p) {
    return LOCK ? __ldcg(p) : *p;
}

template <bool LOCK>
__global__ void k_sgd_users(const int64_t *uptr, const int32_t *uidx, const float *uval,
                            const int32_t *order, int32_t n_order, int32_t *counter, float *P,
                            float *Q, float *bu, float *bi, const int32_t *art, float *ba,
                            float *Qa, float mu, int D, int ld, float gamma, float lam_b,
                            float lam_f, int32_t *locks) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(counter, 1);
        t = __shfl_sync(FULL, t, 0);
        if (t >= n_order) break;
        const int u = order[t];
        float *pu = P + (size_t)u * ld;
        for (int64_t k = uptr[u]; k < uptr[u + 1]; ++k) {
            const int i = uidx[k];
            const float r = uval[k];
            const int a = art ? art[i] : -1;
            const int la = (a >= 0 && a != i) ? a : -1;
            if (LOCK) {
                if (lane == 0) lock_ids(locks, i, la);
                __syncwarp();
            }
            float *qi = Q + (size_t)i * ld;
            float *qa = a >= 0 ? Qa + (size_t)a * ld : nullptr;
            float dot = 0.f;
            float qe[4], pe[4], qiv[4], qav[4];
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const int d = lane + 32 * s;
                qe[s] = pe[s] = qiv[s] = qav[s] = 0.f;
                if (d < D) {
                    qiv[s] = ld_item<LOCK>(qi + d);
                    qav[s] = qa ? ld_item<LOCK>(qa + d) : 0.f;
                    qe[s] = qiv[s] + qav[s];
                    pe[s] = pu[d];
                    dot = fmaf(qe[s], pe[s], dot);
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(FULL, dot, o);
            const float bi0 = ld_item<LOCK>(bi + i), ba0 = a >= 0 ? ld_item<LOCK>(ba + a) : 0.f;
            float pred = mu + bu[u] + bi0 + ba0 + dot;
            const float e = r - pred;
            __syncwarp();
            if (lane == 0) {
                bu[u] += gamma * (e - lam_b * bu[u]);
                bi[i] = bi0 + gamma * (e - lam_b * bi0);
                if (a >= 0) ba[a] = ba0 + gamma * (e - lam_b * ba0);
            }
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const int d = lane + 32 * s;
                if (d < D) {
                    qi[d] = qiv[s] + gamma * (e * pe[s] - lam_f * qiv[s]);
                    if (qa) qa[d] = qav[s] + gamma * (e * pe[s] - lam_f * qav[s]);
                    pu[d] += gamma * (e * qe[s] - lam_f * pe[s]);
                }
            }
            __syncwarp();
            if (LOCK && lane == 0) unlock_ids(locks, i, la);
        }
    }
}

template <bool LOCK>
__global__ void k_sgd_edges(const int64_t *ec, const int64_t *ep, const double *w, int64_t E,
                            float *Q, int D, int ld, float gamma, float lam3, float lam4,
                            int32_t *locks) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < E; k += warps) {
        const int64_t c = ec[k], p = ep[k];
        const float wk = (float)w[k];
        if (LOCK) {   // both endpoints, ascending (mfitr.py:298-320)
            if (lane == 0) lock_ids(locks, (int)c, (int)p);
            __syncwarp();
        }
        for (int d = lane; d < D; d += 32) {
            float *pc = Q + (size_t)c * ld + d, *pp = Q + (size_t)p * ld + d;
            float qc = ld_item<LOCK>(pc), qp = ld_item<LOCK>(pp);
            const float d1 = -2.f * gamma * lam3 * wk * (qc - qp);
            qc += d1;
            qp -= d1;
            const float d2 = -2.f * gamma * lam4 * wk * (qp - qc);
            if (LOCK) {   // the reference's exact sequence under the locks
                *pc = qc - d2;
                *pp = qp + d2;
            } else {      // Hogwild: concurrent edges of one node add up
                const float dc = d1 - d2, dp = d2 - d1;
                atomicAdd(pc, dc);
                atomicAdd(pp, dp);
            }
        }
        if (LOCK) {
            __syncwarp();
            if (lane == 0) unlock_ids(locks, (int)c, (int)p);
        }
    }
}

// the LockTable contract itself: `workers` warps each
// take `iters` ascending-order lock pairs over n_items ids and increment the
// locked accumulators non-atomically; no update may be lost, no deadlock
__global__ void k_lock_stress(int32_t *locks, float *acc, int32_t n_items, int32_t workers,
                              int32_t iters) {
    const int lane = threadIdx.x & 31;
    const int wid = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (wid >= workers) return;
    for (int it = 0; it < iters; ++it) {
        const int a = (wid + it) % n_items, b = (wid * 7 + it * 3 + 1) % n_items;
        if (lane == 0) {
            lock_ids(locks, b, a == b ? -1 : a);
            const float va = __ldcg(acc + a);
            __stcg(acc + a, va + 1.f);
            const float vb = __ldcg(acc + b);
            __stcg(acc + b, vb + 1.f);
            unlock_ids(locks, b, a == b ? -1 : a);
        }
        __syncwarp();
    }
}

}  // namespace
}  // namespace mcf

static int sgd_epoch_impl(const int64_t *uptr, const int32_t *uidx, const float *uval,
                          const int32_t *order, int32_t n_order, int32_t *counter, float *P,
                          float *Q, float *b_u, float *b_i, const int32_t *art, float *b_a,
                          float *Q_a, float mu, int32_t D, float gamma, float lam_bias,
                          float lam_fac, const int64_t *ec, const int64_t *ep, const double *w,
                          int64_t E, float lam3, float lam4, int32_t workers, int32_t *locks,
                          void *stream) {
    if (!uptr || !order || !counter || !P || !Q || !b_u || !b_i || D < 1 || D > 128 ||
        n_order < 0 || (art && (!b_a || !Q_a)) || E < 0 || (E > 0 && (!ec || !ep || !w))) {
        set_error("mcf_mfitr_sgd_epoch: invalid arguments");
        return MCF_E_ARG;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int ld = mcf_factor_ld(D);
    int rc;
    if ((rc = cuda_status(cudaMemsetAsync(counter, 0, sizeof(int32_t), s), "memset"))) return rc;
    // workers = concurrent user warps; 1 = the reference's single-thread order
    // (users and ratings strictly sequential), <= 0 = the whole GPU
    const int warps = workers > 0 ? std::min(workers, 148 * 64) : 148 * 64;
    const unsigned grid = (warps + 7) / 8, block = std::min(warps, 8) * 32;
    if (n_order > 0) {
        if (locks)
            k_sgd_users<true><<<grid, block, 0, s>>>(uptr, uidx, uval, order, n_order, counter, P,
                                                     Q, b_u, b_i, art, b_a, Q_a, mu, D, ld, gamma,
                                                     lam_bias, lam_fac, locks);
        else
            k_sgd_users<false><<<grid, block, 0, s>>>(uptr, uidx, uval, order, n_order, counter,
                                                      P, Q, b_u, b_i, art, b_a, Q_a, mu, D, ld,
                                                      gamma, lam_bias, lam_fac, nullptr);
    }
    if (E > 0 && (lam3 != 0.f || lam4 != 0.f)) {
        if (locks)
            k_sgd_edges<true><<<grid, block, 0, s>>>(ec, ep, w, E, Q, D, ld, gamma, lam3, lam4,
                                                     locks);
        else
            k_sgd_edges<false><<<grid, block, 0, s>>>(ec, ep, w, E, Q, D, ld, gamma, lam3, lam4,
                                                      nullptr);
    }
    return check_launch("mcf_mfitr_sgd_epoch");
}

extern "C" int mcf_mfitr_sgd_epoch(const int64_t *uptr, const int32_t *uidx, const float *uval,
                                   const int32_t *order, int32_t n_order, int32_t *counter,
                                   float *P, float *Q, float *b_u, float *b_i,
                                   const int32_t *art, float *b_a, float *Q_a, float mu,
                                   int32_t D, float gamma, float lam_bias, float lam_fac,
                                   const int64_t *ec, const int64_t *ep, const double *w,
                                   int64_t E, float lam3, float lam4, int32_t workers,
                                   void *stream) {
    return sgd_epoch_impl(uptr, uidx, uval, order, n_order, counter, P, Q, b_u, b_i, art, b_a,
                          Q_a, mu, D, gamma, lam_bias, lam_fac, ec, ep, w, E, lam3, lam4, workers,
                          nullptr, stream);
}

extern "C" int mcf_mfitr_sgd_epoch_locked(const int64_t *uptr, const int32_t *uidx,
                                          const float *uval, const int32_t *order,
                                          int32_t n_order, int32_t *counter, float *P, float *Q,
                                          float *b_u, float *b_i, const int32_t *art, float *b_a,
                                          float *Q_a, float mu, int32_t D, float gamma,
                                          float lam_bias, float lam_fac, const int64_t *ec,
                                          const int64_t *ep, const double *w, int64_t E,
                                          float lam3, float lam4, int32_t workers, int32_t *locks,
                                          void *stream) {
    if (!locks) {
        set_error("mcf_mfitr_sgd_epoch_locked: locks (int32[num_items], zeroed) is required");
        return MCF_E_ARG;
    }
    return sgd_epoch_impl(uptr, uidx, uval, order, n_order, counter, P, Q, b_u, b_i, art, b_a,
                          Q_a, mu, D, gamma, lam_bias, lam_fac, ec, ep, w, E, lam3, lam4, workers,
                          locks, stream);
}

extern "C" int mcf_lock_stress(int32_t *locks, float *acc, int32_t n_items, int32_t workers,
                               int32_t iters, void *stream) {
    if (!locks || !acc || n_items < 1 || workers < 1 || iters < 0) {
        set_error("mcf_lock_stress: invalid arguments");
        return MCF_E_ARG;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    k_lock_stress<<<(unsigned)((workers + 7) / 8), 256, 0, s>>>(locks, acc, n_items, workers, iters);
    return check_launch("mcf_lock_stress");
}
