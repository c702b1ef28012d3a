// ALS half-step, short rows of the wide path in the dual form (CUDA cores).
//
// A row with n ratings and n < D has a rank-n Gram: by the push-through
// identity the reference's solve (reference _kernels.py:151-215)
//     x = (X^T X + lam I)^{-1} X^T y
// equals x = X^T alpha with (X X^T + lam I) alpha = y, an n x n system
// instead of D x D.  The tensor-core kernel (als_tc.cu) runs this form for
// n <= 64, but a 128-thread team per row is latency-bound there (~50 k cycles
// per row at D = 100, 4 rows per SM in flight).  This kernel takes the rows
// with n <= DN = 32 -- the tail of the plan's length-sorted task list: one
// WARP per row, the gathered partner rows transposed into shared memory,
// K = X X^T accumulated with lane i owning row i of K in registers (FFMA2),
// Cholesky by shuffles (right-looking, the reference's > 0 and finite pivot
// test), both substitutions, x = X^T alpha and one refinement step in the
// dual space (rho = y - X x - lam alpha; the rank-deficient short-row systems
// have cond ~ 5e3, fp32 rounding of K alone exceeds the 1e-4 budget).
//
// Eligible calls: no taxonomy terms, no bias coordinate, no observation
// weights, D > DN (so n < D for every row taken).  Tasks are taken from the
// END of the task list (shortest first) until one is longer than the cut; the
// tensor-core kernel stops at the first light task within the cut.

#include <algorithm>

#include "als_params.cuh"
#include "../../include/mcf.h"

namespace mcf {
namespace {

constexpr int DN = 32;     // longest row on this path (one rating per lane)
constexpr int XS = 36;     // Xt row stride: 16-byte aligned rows, an odd number of 16-byte units
constexpr int LSTR = 33;   // L row stride (conflict-free rows and columns)

__device__ __forceinline__ void ffma2d(float &x, float &y, float a, float bx, float by) {
    unsigned long long A, B, C;
    asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a));
    asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(bx), "f"(by));
    asm("mov.b64 %0, {%1, %2};" : "=l"(C) : "f"(x), "f"(y));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C) : "l"(A), "l"(B));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(C));
}

// K[lane][0 .. 4 NB4) += sum_f Xt[f][lane] * Xt[f][j]
template <int NB4>
__device__ __forceinline__ void dual_gram(const float *Xt, int D, int lane, float (&kr)[DN]) {
#pragma unroll 2
    for (int f = 0; f < D; ++f) {
        const float a = Xt[f * XS + lane];
        const float4 *b = reinterpret_cast<const float4 *>(Xt + f * XS);
#pragma unroll
        for (int j4 = 0; j4 < NB4; ++j4) {
            const float4 bv = b[j4];
            ffma2d(kr[4 * j4], kr[4 * j4 + 1], a, bv.x, bv.y);
            ffma2d(kr[4 * j4 + 2], kr[4 * j4 + 3], a, bv.z, bv.w);
        }
    }
}

// L^T a = z, column-oriented from the packed rows in shared memory
__device__ __forceinline__ float dual_back(float z, const float *Ls, float myinv, int n, int lane) {
    float a = z;
    for (int k = n - 1; k >= 0; --k) {
        const float ak = __shfl_sync(FULL, a, k) * __shfl_sync(FULL, myinv, k);
        if (lane == k) a = ak;
        else if (lane < k) a = fmaf(-Ls[k * LSTR + lane], ak, a);
    }
    return a;
}

// x[lane + 32 c] = sum_j Xt[lane + 32 c][j] * al[j]   (c < 4; rows >= ld read as 0)
template <bool ADD>
__device__ __forceinline__ void dual_xt(const float *Xt, const float *al, int nb4, int ld, int lane,
                                        float (&x)[4]) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int f = lane + 32 * c;
        float s0 = 0.f, s1 = 0.f;
        if (f < ld) {
            const float4 *xr = reinterpret_cast<const float4 *>(Xt + f * XS);
            for (int j4 = 0; j4 < nb4; ++j4) {
                const float4 xv = xr[j4];
                const float4 av = reinterpret_cast<const float4 *>(al)[j4];
                s0 = fmaf(xv.x, av.x, s0); s1 = fmaf(xv.y, av.y, s1);
                s0 = fmaf(xv.z, av.z, s0); s1 = fmaf(xv.w, av.w, s1);
            }
        }
        x[c] = ADD ? x[c] + (s0 + s1) : s0 + s1;
    }
}

// one warp per CTA: ~20 KB of shared memory per row in flight at D = 100, 11 rows per SM
__global__ void __launch_bounds__(32) k_als_dual(AlsParams p, PairPlan q, int *counter, int cut) {
    extern __shared__ __align__(16) float dsm[];
    const int lane = threadIdx.x & 31;
    const int D = p.D, ld = p.ld;
    float *Xt = dsm;   // [ld][XS]: Xt[f][j] = feature f of rating j
    float *Ls = Xt + ld * XS;                   // [DN][LSTR]: L rows
    float *al = Ls + DN * LSTR;                 // [DN] alpha / its correction (16-byte aligned)
    float *xs = al + DN;                        // [128] x
    for (;;) {
        int i = 0;
        if (lane == 0) i = atomicAdd(counter, 1);
        i = __shfl_sync(FULL, i, 0);
        const int64_t t = q.n_tasks - 1 - (int64_t)i;
        if (t < 0) break;
        const int n = q.task_n[t];
        if (n > cut || q.task_slot[t] >= 0) break;   // the list is sorted: nothing shorter is left
        const int row = q.task_row[t];
        const int64_t k0 = q.task_k0[t];
        if (n == 0) {   // empty row: 0 with a regulariser, else singular (factor.py:535-537)
            if (p.lam_c > 0.f || p.lam_n > 0.f) {
                for (int f = lane; f < ld; f += 32) put_out(p, row, f, 0.f);
            } else if (lane == 0) {
                report_fail(p.fail, row);
            }
            continue;
        }
        const float lam_row = p.lam_c + p.lam_n * (float)n;
        int id = 0;
        float y = 0.f;
        if (lane < n) {
            id = __ldg(p.idx + k0 + lane);
            y = __ldg(p.val + k0 + lane) - p.y_shift;
        }
        // gather: lane j reads its partner row in 16-byte pieces (8 in flight) and
        // stores them transposed (conflict-free: the lanes are consecutive columns)
        {
            const float4 *src = reinterpret_cast<const float4 *>(p.fixed + (size_t)id * ld);
            const int nc4 = ld >> 2;
            __syncwarp();
            for (int c = 0; c < nc4; c += 8) {
                float4 v[8];
#pragma unroll
                for (int q4 = 0; q4 < 8; ++q4)
                    v[q4] = (lane < n && c + q4 < nc4) ? __ldg(src + c + q4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int q4 = 0; q4 < 8; ++q4) {
                    if (c + q4 < nc4) {
                        float *d = Xt + 4 * (c + q4) * XS + lane;
                        d[0] = v[q4].x;
                        d[XS] = v[q4].y;
                        d[2 * XS] = v[q4].z;
                        d[3 * XS] = v[q4].w;
                    }
                }
            }
            __syncwarp();
        }
        // K = X X^T: lane i holds row i
        const int nb4 = (n + 3) >> 2;
        float kr[DN];
#pragma unroll
        for (int j = 0; j < DN; ++j) kr[j] = 0.f;
        if (nb4 <= 2) dual_gram<2>(Xt, D, lane, kr);
        else if (nb4 <= 4) dual_gram<4>(Xt, D, lane, kr);
        else if (nb4 <= 6) dual_gram<6>(Xt, D, lane, kr);
        else dual_gram<8>(Xt, D, lane, kr);
        // Cholesky of K + lam I (right-looking; column k of L ends up in kr[k] of the
        // lanes below k), forward substitution fused
        float r = y, myinv = 0.f;
        bool ok = true;
#pragma unroll
        for (int k = 0; k < DN; ++k) {
            if (k < n) {
                const float d = __shfl_sync(FULL, kr[k], k) + lam_row;
                ok = ok && d > 0.f && d < INFINITY;
                const float inv = rsqrtf(d);
                const float lik = kr[k] * inv;
                if (lane == k) myinv = inv;
                const float zk = __shfl_sync(FULL, r, k) * inv;
                if (lane == k) r = zk;
                else if (lane > k) r = fmaf(-lik, zk, r);
                kr[k] = lik;
#pragma unroll
                for (int jb = 0; jb < DN / 8; ++jb) {
                    if (8 * jb + 7 > k && 8 * jb < n) {
#pragma unroll
                        for (int j = 8 * jb; j < 8 * jb + 8; ++j) {
                            if (j > k) kr[j] = fmaf(-lik, __shfl_sync(FULL, lik, j), kr[j]);
                        }
                    }
                }
            }
        }
        if (!ok) {
            if (lane == 0) report_fail(p.fail, row);
            continue;
        }
#pragma unroll
        for (int k = 0; k < DN; ++k) Ls[lane * LSTR + k] = kr[k];
        __syncwarp();
        float a_sol = dual_back(r, Ls, myinv, n, lane);
        al[lane] = a_sol;
        __syncwarp();
        float x[4];
        dual_xt<false>(Xt, al, nb4, ld, lane, x);
        // one refinement step in the dual space
#pragma unroll
        for (int c = 0; c < 4; ++c) xs[lane + 32 * c] = x[c];
        __syncwarp();
        float dot0 = 0.f, dot1 = 0.f;
        for (int f = 0; f < D; f += 4) {   // D <= ld, ld a multiple of 4; rows D.. of Xt are zero
            const float4 xv = *reinterpret_cast<const float4 *>(xs + f);
            dot0 = fmaf(Xt[f * XS + lane], xv.x, dot0);
            dot1 = fmaf(Xt[(f + 1) * XS + lane], xv.y, dot1);
            dot0 = fmaf(Xt[(f + 2) * XS + lane], xv.z, dot0);
            dot1 = fmaf(Xt[(f + 3) * XS + lane], xv.w, dot1);
        }
        float rr = lane < n ? y - (dot0 + dot1) - lam_row * a_sol : 0.f;
        for (int k = 0; k < n; ++k) {   // L w = rho
            const float wk = __shfl_sync(FULL, rr, k) * __shfl_sync(FULL, myinv, k);
            if (lane == k) rr = wk;
            else if (lane > k) rr = fmaf(-Ls[lane * LSTR + k], wk, rr);
        }
        const float da = dual_back(rr, Ls, myinv, n, lane);
        __syncwarp();
        al[lane] = da;
        __syncwarp();
        dual_xt<true>(Xt, al, nb4, ld, lane, x);
        bool fin = true;
#pragma unroll
        for (int c = 0; c < 4; ++c) fin = fin && isfinite(x[c]);
        if (!__all_sync(FULL, fin)) {
            if (lane == 0) report_fail(p.fail, row);
            continue;
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int f = lane + 32 * c;
            if (f < ld) put_out(p, row, f, f < D ? x[c] : 0.f);
        }
    }
}

}  // namespace

// rows with at most this many ratings leave the tensor-core kernel for
// k_als_dual (0: the call is not eligible)
int als_dual_cut(const AlsParams &p, bool weighted) {
    if (weighted || p.tax_T || p.tax_S || p.bias_dim >= 0 || p.schur || p.D <= DN || p.D > 128 ||
        getenv("MCF_NO_DUAL_WARP"))
        return 0;
    return DN;
}

int launch_als_dual(const AlsParams &p, const PairPlan &q, int *counter, int cut, cudaStream_t s) {
    if (cut <= 0 || q.n_tasks == 0) return MCF_OK;
    const size_t smem = sizeof(float) * (size_t)(p.ld * XS + DN * LSTR + DN + 128);
    static size_t attr = 0;
    if (smem > attr) {
        cudaFuncSetAttribute(k_als_dual, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = smem;
    }
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_als_dual, 32, smem);
    const int64_t grid = std::min<int64_t>(q.n_tasks, (int64_t)sms * std::max(per_sm, 1));
    k_als_dual<<<(unsigned)grid, 32, smem, s>>>(p, q, counter, cut);
    return check_launch("mcf_als_half_step(dual rows)");
}

}  // namespace mcf
