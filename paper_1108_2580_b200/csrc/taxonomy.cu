// MFITR taxonomy term as a segmented reduction (sm_100a).
//
// The reference applies its graph regulariser by SGD over the sorted edge
// list (_kernels.edge_pass_range, reference _kernels.py:128-148); its exact
// gradient (mfitr.grad_mfitr, mfitr.py:269-273) is 2 (l3 + l4) w_e (q_c - q_p)
// on the child and the negative on the parent.  In an exact block solve of
// item i that term contributes tau * S_i * q_i to the normal matrix and
// tau * T_i to the right-hand side, tau = l3 + l4, with
//     S_i = sum_{e incident to i} w_e,   T_i = sum_{e incident} w_e q_other(e).
// One warp per item walks the item's incident edges in CSR (= edge-list)
// order, lanes own float4 column blocks of q, so the sums have a fixed order.
#include "common.cuh"
#include "../../include/mcf.h"

namespace mcf {
namespace {

__global__ void __launch_bounds__(256) k_tax_terms(const int64_t *inc_ptr, const int32_t *inc_edge,
                                                   const int32_t *inc_other, const float *w,
                                                   const float *q, int32_t n_items, int ld,
                                                   const int32_t *row_list, int32_t n_list,
                                                   float *S, float *T) {
    const int lane = threadIdx.x & 31;
    const int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (j >= n_list) return;
    const int i = row_list ? row_list[j] : (int)j;
    const int nq = ld / 4;
    float4 acc[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    float s = 0.f;
    for (int64_t e = inc_ptr[i]; e < inc_ptr[i + 1]; ++e) {
        const float we = w[inc_edge[e]];
        const int o = inc_other[e];
        s += we;
        const float4 *q4 = reinterpret_cast<const float4 *>(q + (size_t)o * ld);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int blk = lane + 32 * c;
            if (blk < nq) {
                const float4 v = q4[blk];
                acc[c].x = fmaf(we, v.x, acc[c].x);
                acc[c].y = fmaf(we, v.y, acc[c].y);
                acc[c].z = fmaf(we, v.z, acc[c].z);
                acc[c].w = fmaf(we, v.w, acc[c].w);
            }
        }
    }
    if (lane == 0) S[i] = s;
    float4 *t4 = reinterpret_cast<float4 *>(T + (size_t)i * ld);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int blk = lane + 32 * c;
        if (blk < nq) t4[blk] = acc[c];
    }
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
    k_tax_terms<<<(unsigned)ceil_div(n, 8), 256, 0, s>>>(inc_ptr, inc_edge, inc_other, edge_w, q,
                                                         n_items, mcf_factor_ld(D), row_list, n,
                                                         S_out, T_out);
    return check_launch("mcf_taxonomy_terms");
}
