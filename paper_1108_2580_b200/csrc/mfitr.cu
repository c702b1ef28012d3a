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

// out[r] = [main[r][:D] + (art[r] >= 0 ? add[art[r]][:D] : 0) | 1 | 0 ...]
__global__ void k_mfitr_fixed(const float *main_t, const float *add_t, const int32_t *art,
                              int64_t n, int D, int ld, float *out) {
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
// 2 artists (partner u, aux = item).
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
                                                                       ld, out);
    return check_launch("mcf_mfitr_fixed");
}

extern "C" int mcf_mfitr_targets(int32_t mode, const int64_t *ptr, const int32_t *idx,
                                 const float *val, const int32_t *aux, int32_t n_rows,
                                 const float *Pa, const float *Qa, const float *Aa,
                                 const int32_t *art, float mu, int32_t D, float *out,
                                 void *stream) {
    if (mode < 0 || mode > 2 || !ptr || !out || n_rows < 0 || D < 1 || D + 1 > 128 ||
        (mode == 0 && (!Qa || !Aa || !art)) || (mode == 1 && (!Pa || !Aa || !art || !aux)) ||
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
// (_kernels.py:129-148).  Device form (Hogwild, as GPU SGD trainers do): a
// warp per user -- warps take users in shuffle order -- walks that user's
// ratings sequentially with the reference's update order (item side sees
// the pre-update user factor, the user side the pre-update effective item
// factor); item / artist state shared between concurrent users is updated
// without locks.  The edge pass runs a warp per edge with atomic adds.  Not
// bit-reproducible (neither is the reference's threaded path);
// parity is the loss trajectory (tests/test_gpu_mfitr.py).
namespace mcf {
namespace {

__global__ void k_sgd_users(const int64_t *uptr, const int32_t *uidx, const float *uval,
                            const int32_t *order, int32_t n_order, int32_t *counter, float *P,
                            float *Q, float *bu, float *bi, const int32_t *art, float *ba,
                            float *Qa, float mu, int D, int ld, float gamma, float lam_b,
                            float lam_f) {
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
            float *qi = Q + (size_t)i * ld;
            float *qa = a >= 0 ? Qa + (size_t)a * ld : nullptr;
            float dot = 0.f;
            float qe[4], pe[4];
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const int d = lane + 32 * s;
                qe[s] = pe[s] = 0.f;
                if (d < D) {
                    qe[s] = qi[d] + (qa ? qa[d] : 0.f);
                    pe[s] = pu[d];
                    dot = fmaf(qe[s], pe[s], dot);
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(FULL, dot, o);
            float pred = mu + bu[u] + bi[i] + (a >= 0 ? ba[a] : 0.f) + dot;
            const float e = r - pred;
            __syncwarp();
            if (lane == 0) {
                bu[u] += gamma * (e - lam_b * bu[u]);
                bi[i] += gamma * (e - lam_b * bi[i]);
                if (a >= 0) ba[a] += gamma * (e - lam_b * ba[a]);
            }
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const int d = lane + 32 * s;
                if (d < D) {
                    qi[d] += gamma * (e * pe[s] - lam_f * qi[d]);
                    if (qa) qa[d] += gamma * (e * pe[s] - lam_f * qa[d]);
                    pu[d] += gamma * (e * qe[s] - lam_f * pe[s]);
                }
            }
            __syncwarp();
        }
    }
}

__global__ void k_sgd_edges(const int64_t *ec, const int64_t *ep, const double *w, int64_t E,
                            float *Q, int D, int ld, float gamma, float lam3, float lam4) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < E; k += warps) {
        const int64_t c = ec[k], p = ep[k];
        const float wk = (float)w[k];
        for (int d = lane; d < D; d += 32) {
            float qc = Q[(size_t)c * ld + d], qp = Q[(size_t)p * ld + d];
            const float d1 = -2.f * gamma * lam3 * wk * (qc - qp);
            qc += d1;
            qp -= d1;
            const float d2 = -2.f * gamma * lam4 * wk * (qp - qc);
            const float dc = d1 - d2, dp = d2 - d1;
            atomicAdd(Q + (size_t)c * ld + d, dc);
            atomicAdd(Q + (size_t)p * ld + d, dp);
        }
    }
}

}  // namespace
}  // namespace mcf

extern "C" int mcf_mfitr_sgd_epoch(const int64_t *uptr, const int32_t *uidx, const float *uval,
                                   const int32_t *order, int32_t n_order, int32_t *counter,
                                   float *P, float *Q, float *b_u, float *b_i,
                                   const int32_t *art, float *b_a, float *Q_a, float mu,
                                   int32_t D, float gamma, float lam_bias, float lam_fac,
                                   const int64_t *ec, const int64_t *ep, const double *w,
                                   int64_t E, float lam3, float lam4, int32_t workers,
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
    if (n_order > 0)
        k_sgd_users<<<(warps + 7) / 8, std::min(warps, 8) * 32, 0, s>>>(uptr, uidx, uval, order, n_order, counter, P, Q, b_u,
                                            b_i, art, b_a, Q_a, mu, D, ld, gamma, lam_bias,
                                            lam_fac);
    if (E > 0 && (lam3 != 0.f || lam4 != 0.f))
        k_sgd_edges<<<(warps + 7) / 8, std::min(warps, 8) * 32, 0, s>>>(ec, ep, w, E, Q, D, ld,
                                                                         gamma, lam3, lam4);
    return check_launch("mcf_mfitr_sgd_epoch");
}
