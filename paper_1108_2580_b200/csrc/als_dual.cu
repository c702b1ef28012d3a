// ALS half-step, short rows of the wide path in the dual form (CUDA cores).
//
// A row with n ratings and n < D has a rank-n Gram: by the push-through
// identity the reference's solve (reference _kernels.py:151-215)
//     x = (X^T X + lam I)^{-1} X^T y
// equals x = X^T alpha with (X X^T + lam I) alpha = y, an n x n system
// instead of D x D.  The tensor-core kernel (als_tc.cu) has this form too,
// but a 128-thread team per row is latency-bound there (~50-60 k cycles per
// row at D = 100, 4 rows per SM in flight).  These kernels take the rows with
// n <= 64 -- the tail of the plan's length-sorted task list: one WARP per
// row, the gathered partner rows transposed into shared memory, K = X X^T
// accumulated with lane i owning rows i (and i + 32) of K in registers
// (FFMA2), Cholesky by shuffles (right-looking, the reference's > 0 and
// finite pivot test) with the forward substitution fused, back substitution,
// x = X^T alpha and one refinement step in the dual space (rho = y - X x -
// lam alpha: the rank-deficient short-row systems have cond ~ 5e3, fp32
// rounding of K alone exceeds the 1e-4 budget).
//
// k_als_dual<1, N> takes n <= 32 in four length classes (N = 8, 16, 24, 32;
// 11 rows per SM in flight at D = 100 for the longest, ~40 for the shortest);
// k_als_dual<2> (33 <= n <= 64, two row sets per lane, 4 rows per SM) is
// built but off by default (MCF_DUAL_WARP_MAX=64): at 4 warps per SM it is
// latency-bound and slower than the tensor-core kernel's dual form.
//
// Eligible calls: no taxonomy terms, no bias coordinate, no observation
// weights, every row taken has n < D.  The light tasks are sorted by length:
// each kernel bisects for its first task and walks towards the tail; the
// tensor-core kernel stops at the first light task within the cut.

#include <algorithm>

#include "als_params.cuh"
#include "../../include/mcf.h"

namespace mcf {
namespace {

// S row sets per lane (row i = lane + 32 s), rows of at most N ratings
// (N = 8, 16, 24, 32 for S = 1: the shared-memory footprint, and with it the
// number of rows in flight per SM, follows the row length; N = 64 for S = 2)
template <int S, int N_>
struct DualCfg {
    static constexpr int N = N_;
    static constexpr int XS = N + 4;       // Xt row stride: 16-byte rows, an odd number of 16-byte units
    static constexpr int LSTR = N + 1;     // L row stride (conflict-free rows and columns)
    static_assert(N % 8 == 0 && N <= 32 * S && N > 32 * (S - 1), "row cap");
    // columns of K kept by row set s (lower triangle)
    static constexpr int cols(int s) { return 32 * (s + 1) < N ? 32 * (s + 1) : N; }
    static size_t smem_bytes(int ld) { return sizeof(float) * (size_t)(ld * XS + N * LSTR + N + 128); }
};

__device__ __forceinline__ void ffma2d(float &x, float &y, float a, float bx, float by) {
    unsigned long long A, B, C;
    asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a));
    asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(bx), "f"(by));
    asm("mov.b64 %0, {%1, %2};" : "=l"(C) : "f"(x), "f"(y));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C) : "l"(A), "l"(B));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(C));
}

// kr[s][0 .. 4 NB4) += sum_f Xt[f][lane + 32 s] * Xt[f][j]; only the lower
// triangle is used, so row set s stops at column 32 (s + 1)
template <int S, int N, int NB4>
__device__ __forceinline__ void dual_gram(const float *Xt, int D, int lane, float (&kr)[S][N]) {
    constexpr int XS = DualCfg<S, N>::XS;
#pragma unroll 4
    for (int f = 0; f < D; ++f) {
        float a[S];
#pragma unroll
        for (int s = 0; s < S; ++s) a[s] = Xt[f * XS + lane + 32 * s];
        const float4 *b = reinterpret_cast<const float4 *>(Xt + f * XS);
#pragma unroll
        for (int j4 = 0; j4 < NB4; ++j4) {
            const float4 bv = b[j4];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (4 * j4 < DualCfg<S, N>::cols(s)) {
                    ffma2d(kr[s][4 * j4], kr[s][4 * j4 + 1], a[s], bv.x, bv.y);
                    ffma2d(kr[s][4 * j4 + 2], kr[s][4 * j4 + 3], a[s], bv.z, bv.w);
                }
            }
        }
    }
}

// value of row k of a lane-distributed vector v[s] (row i = lane + 32 s)
template <int S>
__device__ __forceinline__ float row_bcast(const float (&v)[S], int k) {
    float r = __shfl_sync(FULL, v[0], k & 31);
#pragma unroll
    for (int s = 1; s < S; ++s) {
        const float t = __shfl_sync(FULL, v[s], k & 31);
        if ((k >> 5) == s) r = t;
    }
    return r;
}

// L^T a = z, column-oriented from the L rows in shared memory
template <int S, int N>
__device__ __forceinline__ void dual_back(float (&a)[S], const float *Ls, const float (&myinv)[S], int n,
                                          int lane) {
    constexpr int LSTR = DualCfg<S, N>::LSTR;
    for (int k = n - 1; k >= 0; --k) {
        const float ak = row_bcast<S>(a, k) * row_bcast<S>(myinv, k);
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int i = lane + 32 * s;
            if (i == k) a[s] = ak;
            else if (i < k) a[s] = fmaf(-Ls[k * LSTR + i], ak, a[s]);
        }
    }
}

// L w = r, column-oriented
template <int S, int N>
__device__ __forceinline__ void dual_fwd(float (&r)[S], const float *Ls, const float (&myinv)[S], int n,
                                         int lane) {
    constexpr int LSTR = DualCfg<S, N>::LSTR;
    for (int k = 0; k < n; ++k) {
        const float wk = row_bcast<S>(r, k) * row_bcast<S>(myinv, k);
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int i = lane + 32 * s;
            if (i == k) r[s] = wk;
            else if (i > k && i < N) r[s] = fmaf(-Ls[i * LSTR + k], wk, r[s]);   // (lanes >= N hold no row)
        }
    }
}

// x[lane + 32 c] (+)= sum_j Xt[lane + 32 c][j] * al[j]   (c < 4; rows >= ld read as 0)
template <int S, int N, bool ADD>
__device__ __forceinline__ void dual_xt(const float *Xt, const float *al, int nb4, int ld, int lane,
                                        float (&x)[4]) {
    constexpr int XS = DualCfg<S, N>::XS;
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

// One warp per CTA (shared memory per row in flight: ~20 KB for S = 1, ~44 KB
// for S = 2 at D = 100).  Light tasks are sorted by length, longest first:
// the warp finds the first task with n <= hi by bisection and takes tasks
// from there while n > lo.
template <int S, int N>
__global__ void __launch_bounds__(32) k_als_dual(AlsParams p, PairPlan q, int64_t first_light,
                                                 int *counter, int lo, int hi) {
    using C = DualCfg<S, N>;
    constexpr int XS = C::XS, LSTR = C::LSTR;
    extern __shared__ __align__(16) float dsm[];
    const int lane = threadIdx.x & 31;
    const int D = p.D, ld = p.ld;
    float *Xt = dsm;                  // [ld][XS]: Xt[f][j] = feature f of rating j
    float *Ls = Xt + ld * XS;         // [N][LSTR]: L rows
    float *al = Ls + N * LSTR;        // [N] alpha / its correction (16-byte aligned)
    float *xs = al + N;               // [128] x
    int64_t t0 = first_light, t1 = q.n_tasks;   // first light task with n <= hi
    while (t0 < t1) {
        const int64_t mid = (t0 + t1) >> 1;
        if (q.task_n[mid] <= hi) t1 = mid;
        else t0 = mid + 1;
    }
    for (;;) {
        int i = 0;
        if (lane == 0) i = atomicAdd(counter, 1);
        i = __shfl_sync(FULL, i, 0);
        const int64_t t = t0 + (int64_t)i;
        if (t >= q.n_tasks) break;
        const int n = q.task_n[t];
        if (n <= lo) break;   // sorted: only shorter rows follow
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
        float y[S];
        // gather: lane j reads its partner rows in 16-byte pieces (8 in flight) and
        // stores them transposed (conflict-free: the lanes are consecutive columns)
        __syncwarp();
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int j = lane + 32 * s;
            int id = 0;
            y[s] = 0.f;
            if (j < n) {
                id = __ldg(p.idx + k0 + j);
                y[s] = __ldg(p.val + k0 + j) - p.y_shift;
            }
            const float4 *src = reinterpret_cast<const float4 *>(p.fixed + (size_t)id * ld);
            const int nc4 = ld >> 2;
            for (int c = 0; c < nc4; c += 8) {
                float4 v[8];
#pragma unroll
                for (int q4 = 0; q4 < 8; ++q4)
                    v[q4] = (j < n && c + q4 < nc4) ? __ldg(src + c + q4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int q4 = 0; q4 < 8; ++q4) {
                    if (c + q4 < nc4 && j < N) {
                        float *d = Xt + 4 * (c + q4) * XS + j;
                        d[0] = v[q4].x;
                        d[XS] = v[q4].y;
                        d[2 * XS] = v[q4].z;
                        d[3 * XS] = v[q4].w;
                    }
                }
            }
        }
        __syncwarp();
        // K = X X^T: lane i holds rows i + 32 s
        const int nb4 = (n + 3) >> 2;
        float kr[S][N];
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int j = 0; j < N; ++j) kr[s][j] = 0.f;
        if (N <= 8) {
            dual_gram<S, N, 2>(Xt, D, lane, kr);
        } else if (N <= 16) {
            dual_gram<S, N, 4>(Xt, D, lane, kr);
        } else if (N <= 32) {
            if (nb4 <= 6) dual_gram<S, N, 6>(Xt, D, lane, kr);
            else dual_gram<S, N, 8>(Xt, D, lane, kr);
        } else {
            if (nb4 <= 10) dual_gram<S, N, 10>(Xt, D, lane, kr);
            else if (nb4 <= 12) dual_gram<S, N, 12>(Xt, D, lane, kr);
            else if (nb4 <= 14) dual_gram<S, N, 14>(Xt, D, lane, kr);
            else dual_gram<S, N, 16>(Xt, D, lane, kr);
        }
        // Cholesky of K + lam I (right-looking; column k of L ends up in kr[.][k] of
        // the rows below k), forward substitution fused
        float r[S], myinv[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            r[s] = y[s];
            myinv[s] = 0.f;
        }
        bool ok = true;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            if (k < n) {
                const int ks = k >> 5, kl = k & 31;
                const float d = __shfl_sync(FULL, kr[ks][k], kl) + lam_row;
                ok = ok && d > 0.f && d < INFINITY;
                const float inv = rsqrtf(d);
                if (lane == kl) myinv[ks] = inv;
                const float zk = __shfl_sync(FULL, r[ks], kl) * inv;
                float lik[S];
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    if (C::cols(s) > k) {   // row set s still has rows at or below k
                        const int i = lane + 32 * s;
                        lik[s] = kr[s][k] * inv;
                        if (i == k) r[s] = zk;
                        else if (i > k) r[s] = fmaf(-lik[s], zk, r[s]);
                        kr[s][k] = lik[s];
                    } else {
                        lik[s] = 0.f;
                    }
                }
#pragma unroll
                for (int jb = 0; jb < N / 8; ++jb) {
                    if (8 * jb + 7 > k && 8 * jb < n) {
#pragma unroll
                        for (int j = 8 * jb; j < 8 * jb + 8; ++j) {
                            if (j > k) {
                                const float ljk = __shfl_sync(FULL, lik[j >> 5], j & 31);
#pragma unroll
                                for (int s = 0; s < S; ++s)
                                    if (C::cols(s) > j) kr[s][j] = fmaf(-lik[s], ljk, kr[s][j]);
                            }
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
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int k = 0; k < C::cols(s); ++k)
                if (lane + 32 * s < N) Ls[(lane + 32 * s) * LSTR + k] = kr[s][k];
        __syncwarp();
        float a_sol[S];
#pragma unroll
        for (int s = 0; s < S; ++s) a_sol[s] = r[s];
        dual_back<S, N>(a_sol, Ls, myinv, n, lane);
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (lane + 32 * s < N) al[lane + 32 * s] = a_sol[s];
        __syncwarp();
        float x[4];
        dual_xt<S, N, false>(Xt, al, nb4, ld, lane, x);
        // one refinement step in the dual space
#pragma unroll
        for (int c = 0; c < 4; ++c) xs[lane + 32 * c] = x[c];
        __syncwarp();
        float rr[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int j = lane + 32 * s;
            float dot0 = 0.f, dot1 = 0.f;
            for (int f = 0; f < D; f += 4) {   // D <= ld, ld a multiple of 4; rows D.. of Xt are zero
                const float4 xv = *reinterpret_cast<const float4 *>(xs + f);
                dot0 = fmaf(Xt[f * XS + j], xv.x, dot0);
                dot1 = fmaf(Xt[(f + 1) * XS + j], xv.y, dot1);
                dot0 = fmaf(Xt[(f + 2) * XS + j], xv.z, dot0);
                dot1 = fmaf(Xt[(f + 3) * XS + j], xv.w, dot1);
            }
            rr[s] = j < n ? y[s] - (dot0 + dot1) - lam_row * a_sol[s] : 0.f;
        }
        dual_fwd<S, N>(rr, Ls, myinv, n, lane);
        dual_back<S, N>(rr, Ls, myinv, n, lane);
        __syncwarp();
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (lane + 32 * s < N) al[lane + 32 * s] = rr[s];
        __syncwarp();
        dual_xt<S, N, true>(Xt, al, nb4, ld, lane, x);
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

template <int S, int N>
int launch_dual(const AlsParams &p, const PairPlan &q, int64_t first_light, int *counter, int lo, int hi,
                cudaStream_t s) {
    const size_t smem = DualCfg<S, N>::smem_bytes(p.ld);
    static size_t attr = 0;
    if (smem > attr) {
        cudaFuncSetAttribute(k_als_dual<S, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = smem;
    }
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_als_dual<S, N>, 32, smem);
    const int64_t grid = std::min<int64_t>(q.n_tasks - first_light, (int64_t)sms * std::max(per_sm, 1));
    if (grid > 0) k_als_dual<S, N><<<(unsigned)grid, 32, smem, s>>>(p, q, first_light, counter, lo, hi);
    return check_launch("mcf_als_half_step(dual rows)");
}

}  // namespace

// rows with at most this many ratings leave the tensor-core kernel for
// k_als_dual (0: the call is not eligible).  MCF_DUAL_WARP_MAX: 0 / 32 / 64.
int als_dual_cut(const AlsParams &p, bool weighted) {
    // default 32: k_als_dual<2> fits 4 warps per SM (44 KB of shared memory per
    // row) and is latency-bound there -- config 3: 17 ms per half-step for the
    // 33..64 rows against ~9 ms on the tensor-core kernel's dual form
    const char *e = getenv("MCF_DUAL_WARP_MAX");
    int mx = e ? atoi(e) : 32;
    if (p.D <= 64) mx = std::min(mx, 32);   // every row taken must have n < D
    if (weighted || p.tax_T || p.tax_S || p.bias_dim >= 0 || p.schur || p.D <= 32 || p.D > 128 ||
        getenv("MCF_NO_DUAL_WARP") || mx < 32)
        return 0;
    return mx >= 64 ? 64 : 32;
}

// counters: five zeroed ints (one per kernel); first_light: index of the
// first light task (= number of hot-row chunks)
int launch_als_dual(const AlsParams &p, const PairPlan &q, int64_t first_light, int *counters, int cut,
                    cudaStream_t s) {
    if (cut <= 0 || q.n_tasks <= first_light) return MCF_OK;
    int rc = MCF_OK;
    // the longer rows first; one kernel per length class (its own counter each)
    if (cut > 32 && (rc = launch_dual<2, 64>(p, q, first_light, counters + 4, 32, 64, s))) return rc;
    if ((rc = launch_dual<1, 32>(p, q, first_light, counters, 24, 32, s))) return rc;
    if ((rc = launch_dual<1, 24>(p, q, first_light, counters + 1, 16, 24, s))) return rc;
    if ((rc = launch_dual<1, 16>(p, q, first_light, counters + 2, 8, 16, s))) return rc;
    return launch_dual<1, 8>(p, q, first_light, counters + 3, -1, 8, s);
}

}  // namespace mcf
