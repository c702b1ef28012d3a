// Prediction, squared error and small reductions (sm_100a).
//
// mcf_predict_sse replaces _kernels.mf_predict_batch (reference
// _kernels.py:331-375; ALS branch via factor.predict_batch factor.py:222-242,
// MFITR branch via mfitr.predict_batch mfitr.py:181-197) fused with the
// clip + squared error of the held-out RMSE (factor.py:613-616,
// evaluation.py:11-18).  One thread per query, float4 row loads; the error
// sum is a double tree reduction in a fixed order (per-block partials, then
// one block), so the RMSE is bit-reproducible.
#include "common.cuh"
#include "../../include/mcf.h"

namespace mcf {
namespace {

constexpr int RT = 256;  // threads per reduction block

__device__ __forceinline__ double block_sum(double v, double *sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULL, v, o);
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (warp == 0) {
        t = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(FULL, t, o);
    }
    return t;  // valid in thread 0
}

__global__ void __launch_bounds__(RT) k_predict(const int32_t *users, const int32_t *items,
                                                const float *truth, int64_t n, const float *P,
                                                int32_t n_users, const float *Q, int32_t n_items,
                                                int D, int ld, float mu, const float *b_u,
                                                const float *b_i, const int32_t *art,
                                                const float *b_a, const float *Q_a, float lo,
                                                float hi, float *pred_out, double *partial) {
    __shared__ double sh[RT / 32];
    const int64_t t = (int64_t)blockIdx.x * RT + threadIdx.x;
    double se = 0.0;
    if (t < n) {
        const int u = users[t], i = items[t];
        const bool ku = u >= 0 && u < n_users, ki = i >= 0 && i < n_items;
        const int a = (ki && art) ? art[i] : -1;
        float pred = mu;
        if (ku && b_u) pred += b_u[u];
        if (ki) {
            if (b_i) pred += b_i[i];
            if (a >= 0 && b_a) pred += b_a[a];
        }
        if (ku && ki) {
            const float4 *q4 = reinterpret_cast<const float4 *>(Q + (size_t)i * ld);
            const float4 *p4 = reinterpret_cast<const float4 *>(P + (size_t)u * ld);
            const float4 *a4 = a >= 0 ? reinterpret_cast<const float4 *>(Q_a + (size_t)a * ld)
                                      : nullptr;
            float dot = 0.f;
            for (int d = 0; d < ld / 4; ++d) {
                float4 q = q4[d];
                const float4 pp = p4[d];
                if (a4) {
                    const float4 qa = a4[d];
                    q.x += qa.x; q.y += qa.y; q.z += qa.z; q.w += qa.w;
                }
                dot = fmaf(q.x, pp.x, dot);
                dot = fmaf(q.y, pp.y, dot);
                dot = fmaf(q.z, pp.z, dot);
                dot = fmaf(q.w, pp.w, dot);
            }
            pred += dot;
        }
        if (pred_out) pred_out[t] = pred;
        if (truth) {
            const double e = (double)fminf(fmaxf(pred, lo), hi) - (double)truth[t];
            se = e * e;
        }
    }
    if (partial) {
        const double b = block_sum(se, sh);
        if (threadIdx.x == 0) partial[blockIdx.x] = b;
    }
}

__global__ void __launch_bounds__(RT) k_sum(const double *partial, int64_t n, double *out) {
    __shared__ double sh[RT / 32];
    double v = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += RT) v += partial[i];
    const double t = block_sum(v, sh);
    if (threadIdx.x == 0) *out = t;
}

__global__ void __launch_bounds__(RT) k_sq_norms(const float *F, int32_t n, int D, int ld,
                                                 const int64_t *ptr, double *partial) {
    __shared__ double sh[RT / 32];
    const int64_t r = (int64_t)blockIdx.x * RT + threadIdx.x;
    double v = 0.0;
    if (r < n) {
        float s = 0.f;
        for (int d = 0; d < D; ++d) {
            const float f = F[(size_t)r * ld + d];
            s = fmaf(f, f, s);
        }
        const double c = ptr ? (double)(ptr[r + 1] - ptr[r]) : 1.0;
        v = c * (double)s;
    }
    const double t = block_sum(v, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

__global__ void k_add_gathered(const float *A, const float *B, const int32_t *map, int32_t n,
                               int ld, float *out) {
    const int64_t total = (int64_t)n * ld;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / ld;
        const int m = map[r];
        out[e] = m >= 0 ? A[e] + B[(size_t)m * ld + (e - r * ld)] : A[e];
    }
}

}  // namespace
}  // namespace mcf

using namespace mcf;

extern "C" size_t mcf_predict_workspace_bytes(int64_t n) {
    return sizeof(double) * (size_t)(ceil_div(n, RT) + 1);
}

extern "C" int mcf_predict_sse(const int32_t *users, const int32_t *items, const float *truth,
                               int64_t n, const float *P, int32_t n_users, const float *Q,
                               int32_t n_items, int32_t D, float mu, const float *b_u,
                               const float *b_i, const int32_t *art_of_item, const float *b_a,
                               const float *Q_a, float clip_lo, float clip_hi, float *pred_out,
                               double *sse_out, void *ws, size_t ws_bytes, void *stream) {
    if (n < 0 || D < 1 || D > mcf_max_dim() || (n > 0 && (!users || !items || !P || !Q)) ||
        (truth && !sse_out) || (art_of_item && !Q_a)) {
        set_error("mcf_predict_sse: invalid arguments");
        return MCF_E_ARG;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t nb = ceil_div(n, RT);
    if (truth && (!ws || ws_bytes < mcf_predict_workspace_bytes(n))) {
        set_error("mcf_predict_sse: workspace too small");
        return MCF_E_WORKSPACE;
    }
    double *partial = truth ? static_cast<double *>(ws) : nullptr;
    if (nb > 0)
        k_predict<<<(unsigned)nb, RT, 0, s>>>(users, items, truth, n, P, n_users, Q, n_items, D,
                                              mcf_factor_ld(D), mu, b_u, b_i, art_of_item, b_a,
                                              Q_a, clip_lo, clip_hi, pred_out, partial);
    if (truth) k_sum<<<1, RT, 0, s>>>(partial, nb, sse_out);
    return check_launch("mcf_predict_sse");
}

extern "C" int mcf_sq_norms(const float *F, int32_t n, int32_t D, const int64_t *ptr,
                            double *out, void *ws, size_t ws_bytes, void *stream) {
    if (n < 0 || D < 1 || D > mcf_max_dim() || !out || (n > 0 && !F)) {
        set_error("mcf_sq_norms: invalid arguments");
        return MCF_E_ARG;
    }
    const int64_t nb = ceil_div(n, RT);
    if (!ws || ws_bytes < mcf_predict_workspace_bytes(n)) {
        set_error("mcf_sq_norms: workspace too small (mcf_predict_workspace_bytes(n))");
        return MCF_E_WORKSPACE;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    double *partial = static_cast<double *>(ws);
    if (nb > 0) k_sq_norms<<<(unsigned)nb, RT, 0, s>>>(F, n, D, mcf_factor_ld(D), ptr, partial);
    k_sum<<<1, RT, 0, s>>>(partial, nb, out);
    return check_launch("mcf_sq_norms");
}

extern "C" int mcf_add_gathered(const float *A, const float *B, const int32_t *map, int32_t n,
                                int32_t D, float *out, void *stream) {
    if (n < 0 || D < 1 || D > mcf_max_dim() || (n > 0 && (!A || !B || !map || !out))) {
        set_error("mcf_add_gathered: invalid arguments");
        return MCF_E_ARG;
    }
    if (n == 0) return MCF_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    k_add_gathered<<<148 * 8, 256, 0, s>>>(A, B, map, n, mcf_factor_ld(D), out);
    return check_launch("mcf_add_gathered");
}
