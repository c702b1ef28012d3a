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
