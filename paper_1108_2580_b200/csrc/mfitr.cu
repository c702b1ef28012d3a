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

// per-rating targets of one layout, warp per row, ratings in CSR order.
// mode 0 users (row u, partner i), 1 items (row i, partner u),
// 2 artists (row a, partner u, item = aux[k]).
__global__ void k_mfitr_targets(int mode, const int64_t *ptr, const int32_t *idx,
                                const float *val, const int32_t *aux, int32_t n_rows,
                                const float *Pa, const float *Qa, const float *Aa,
                                const int32_t *art, float mu, int D, int ld, float *out) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_rows;
         r += warps) {
        const int64_t a = ptr[r], b = ptr[r + 1];
        const int ar = mode == 1 ? art[r] : -1;   // items: the row's artist
        for (int64_t k = a + lane; k < b; k += 32) {
            const int j = idx[k];
            float t = val[k] - mu;
            if (mode == 0) {            // j = item
                t -= Qa[(size_t)j * ld + D];
                const int aj = art[j];
                if (aj >= 0) t -= Aa[(size_t)aj * ld + D];
            } else if (mode == 1) {     // j = user, row = item
                t -= Pa[(size_t)j * ld + D];
                if (ar >= 0) {
                    const float *qa = Aa + (size_t)ar * ld;
                    const float *pu = Pa + (size_t)j * ld;
                    float d = qa[D];
                    for (int c = 0; c < D; ++c) d = fmaf(qa[c], pu[c], d);
                    t -= d;
                }
            } else {                    // j = user, row = artist, aux = item
                const int i = aux[k];
                const float *qi = Qa + (size_t)i * ld;
                const float *pu = Pa + (size_t)j * ld;
                float d = pu[D] + qi[D];
                for (int c = 0; c < D; ++c) d = fmaf(qi[c], pu[c], d);
                t -= d;
            }
            out[k] = t;
        }
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
        (mode == 0 && (!Qa || !Aa || !art)) || (mode == 1 && (!Pa || !Aa || !art)) ||
        (mode == 2 && (!Pa || !Qa || !aux))) {
        set_error("mcf_mfitr_targets: invalid arguments");
        return MCF_E_ARG;
    }
    if (n_rows == 0) return MCF_OK;
    const int ld = mcf_factor_ld(D + 1);
    const int grid = (int)std::min<int64_t>(ceil_div((int64_t)n_rows, 8), 148 * 16);
    k_mfitr_targets<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        mode, ptr, idx, val, aux, n_rows, Pa, Qa, Aa, art, mu, D, ld, out);
    return check_launch("mcf_mfitr_targets");
}
