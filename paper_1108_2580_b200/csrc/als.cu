// ALS half-step: fused ragged Gram + regulariser + Cholesky solve (sm_100a).
//
// Replaces _kernels.als_solve_rows (reference _kernels.py:151-215) driven by
// factor.als_half_step / parallel.run_blocks (factor.py:512-538,
// parallel.py:134-145).  For every planned row r:
//
//     A_r = sum_k w_k x_k x_k^T + (lam_c + lam_n n_r + tau S_r) I
//     b_r = sum_k w_k (y_k - y_shift) x_k + tau T_r,     out_r = A_r^{-1} b_r
//
// Work decomposition (the "plan"): every row is cut into chunks of at most
// CHUNK ratings; one warp owns one chunk (a work item).  Single-chunk rows
// (all users at cfg1) are solved by the same warp that built their Gram.
// Rows spanning several chunks (Zipf-hot items, up to ~1 M ratings) write
// partial Grams to a workspace slot; the last chunk to finish (atomic
// counter) sums the partials in chunk order -- a fixed order, so results are
// deterministic and independent of scheduling -- and solves.
//
// Gram formation for D <= 28 (NB = ceil(D/4) <= 7 4-wide blocks): a team of
// TS lanes owns the NB(NB+1)/2 lower-triangle 4x4 tiles of A, one tile per
// lane, held in registers; 32/TS teams split the ratings of a batch.  Each
// batch of 32 partner rows is gathered HBM/L2 -> shared memory with 16-byte
// cp.async (zero-fill past the chunk end), double buffered so the gather of
// batch j+1 overlaps the FMAs of batch j.  Per rating a lane issues two
// LDS.128 (its row block and column block) and 16 + 4 FFMA (the diagonal
// tiles' lanes keep the right-hand side; off-diagonal lanes compute the same
// 4 rhs FMAs redundantly so the warp never diverges).
//
// Solve for D <= 28: the reduced Gram is staged in shared memory, lane i
// holds row i of A in registers, right-looking Cholesky with shuffles,
// forward substitution with shuffles, backward substitution reading L^T
// from shared memory.  fp32 throughout; the pivot test matches the
// reference (s > 0 and finite, _kernels.py:197).
//
// D in 29..128: one CTA per work item, Gram tiles spread over the CTA's
// threads, CTA-cooperative Cholesky (correctness path for configs 3/4; the
// tensor-core path for D >= 64 replaces it).
#include <algorithm>

#include "common.cuh"
#include "../../include/mcf.h"

namespace mcf {
namespace {

constexpr int BATCH = 32;

struct AlsParams {
    const int64_t *ptr;
    const int32_t *idx;
    const float *val;
    const float *wts;
    const float *fixed;
    float *out;
    int D, ld;
    float lam_c, lam_n, y_shift, tau;
    const float *tax_S, *tax_T;
    const int32_t *row_list;
    int32_t n_list, row_lo, chunk;
    const int32_t *item_off;   // [n_list + 1]
    const int32_t *slot_off;   // [n_list + 1]
    const int32_t *item_row;   // [total_items] -> list index
    int64_t total_items;
    float *partials;           // [slots][pstride]
    int32_t *counters;         // [n_list]
    unsigned long long *fail;  // min failing row (as unsigned; ~0 = none)
};

// ---------------------------------------------------------------------------
// plan
__global__ void k_plan_count(const int64_t *ptr, const int32_t *row_list, int32_t n_list,
                             int32_t row_lo, int32_t chunk, int32_t *items, int32_t *slots) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= n_list;
         j += gridDim.x * blockDim.x) {
        if (j == n_list) {
            items[j] = 0;
            slots[j] = 0;
            continue;
        }
        const int r = row_list ? row_list[j] : row_lo + j;
        const int64_t n = ptr[r + 1] - ptr[r];
        const int nch = n <= chunk ? 1 : (int)((n + chunk - 1) / chunk);
        items[j] = nch;
        slots[j] = nch > 1 ? nch : 0;
    }
}

__global__ void k_plan_fill(const int32_t *item_off, int32_t n_list, int32_t *item_row) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_list;
         j += gridDim.x * blockDim.x)
        for (int32_t t = item_off[j]; t < item_off[j + 1]; ++t) item_row[t] = j;
}

// ---------------------------------------------------------------------------
// shared pieces

__device__ __forceinline__ void report_fail(unsigned long long *fail, int r) {
    atomicMin(fail, static_cast<unsigned long long>(r));
}

struct ItemInfo {
    int j, r, c, nch;
    int64_t k0, k1, n;
};

__device__ __forceinline__ ItemInfo item_info(const AlsParams &p, int64_t item) {
    ItemInfo it;
    it.j = p.item_row[item];
    it.r = p.row_list ? p.row_list[it.j] : p.row_lo + it.j;
    const int32_t first = p.item_off[it.j];
    it.nch = p.item_off[it.j + 1] - first;
    it.c = (int)(item - first);
    const int64_t a = p.ptr[it.r], b = p.ptr[it.r + 1];
    it.n = b - a;
    it.k0 = a + (int64_t)it.c * p.chunk;
    it.k1 = min(b, it.k0 + p.chunk);
    return it;
}

// ---------------------------------------------------------------------------
// warp path, D <= 28

template <int NB>
struct WarpCfg {
    static constexpr int T = NB * (NB + 1) / 2;                 // tiles per Gram
    static constexpr int TS = T <= 1 ? 1 : T <= 2 ? 2 : T <= 4 ? 4 : T <= 8 ? 8 : T <= 16 ? 16 : 32;
    static constexpr int TPW = 32 / TS;                          // teams per warp
    static constexpr int LD = 4 * NB;                            // floats per gathered row
    static constexpr int PSTRIDE = T * 20;                       // floats per partial slot
    static constexpr int STAGE_FLOATS = BATCH * LD + 2 * BATCH;  // rows + y + w
    static constexpr int WARP_FLOATS = 2 * STAGE_FLOATS;
    static_assert(LD * (LD + 1) <= WARP_FLOATS, "solve matrix must fit in the stage buffers");
};

template <int NB, bool HAS_W>
__device__ __forceinline__ void issue_batch(const AlsParams &p, float *stage, int64_t k,
                                            int64_t k1, int lane) {
    using C = WarpCfg<NB>;
    const int64_t kk = k + lane;
    const bool ok = kk < k1;
    const int col = ok ? p.idx[kk] : -1;
    float y = 0.f, w = 0.f;
    if (ok) {
        y = p.val[kk] - p.y_shift;
        w = HAS_W ? p.wts[kk] : 1.f;
    }
    float *rows = stage;
    float *ys = stage + BATCH * C::LD;
    ys[lane] = y;
    ys[BATCH + lane] = w;
#pragma unroll
    for (int m = 0; m < NB; ++m) {
        const int e = lane + 32 * m;
        const int rr = e / NB, part = e - rr * NB;
        const int src = __shfl_sync(FULL, col, rr);
        const float *g = src >= 0 ? p.fixed + (size_t)src * p.ld + part * 4 : p.fixed;
        cp_async16(rows + rr * C::LD + part * 4, g, src >= 0 ? 16 : 0);
    }
    cp_async_commit();
}

template <int NB, bool HAS_W>
__device__ __forceinline__ void accumulate(const float *stage, int team, int bi, int bj,
                                           float (&acc)[4][4], float (&rhs)[4]) {
    using C = WarpCfg<NB>;
    const float *rows = stage;
    const float *ys = stage + BATCH * C::LD;
#pragma unroll
    for (int q = 0; q < BATCH / C::TPW; ++q) {
        const int k = q * C::TPW + team;
        float4 a = *reinterpret_cast<const float4 *>(rows + k * C::LD + 4 * bi);
        const float4 b = *reinterpret_cast<const float4 *>(rows + k * C::LD + 4 * bj);
        const float y = ys[k];
        if (HAS_W) {
            const float w = ys[BATCH + k];
            a.x *= w; a.y *= w; a.z *= w; a.w *= w;
        }
        const float av[4] = {a.x, a.y, a.z, a.w};
        const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int m = 0; m < 4; ++m) {
#pragma unroll
            for (int n = 0; n < 4; ++n) acc[m][n] = fmaf(av[m], bv[n], acc[m][n]);
            rhs[m] = fmaf(y, av[m], rhs[m]);
        }
    }
}

template <int NB, bool HAS_W>
__global__ void __launch_bounds__(256) k_als_warp(AlsParams p) {
    using C = WarpCfg<NB>;
    extern __shared__ float4 smem4[];
    float *smem = reinterpret_cast<float *>(smem4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (item >= p.total_items) return;
    float *wbuf = smem + warp * C::WARP_FLOATS;
    float *stage[2] = {wbuf, wbuf + C::STAGE_FLOATS};

    const ItemInfo it = item_info(p, item);
    const int team = lane / C::TS, t = lane % C::TS;
    int bi = 0, bj = 0;
    {
        int id = 0;
#pragma unroll
        for (int i = 0; i < NB; ++i)
#pragma unroll
            for (int j2 = 0; j2 <= i; ++j2, ++id)
                if (id == t) { bi = i; bj = j2; }
    }
    const bool tile_ok = t < C::T;

    float acc[4][4], rhs[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        rhs[m] = 0.f;
#pragma unroll
        for (int n = 0; n < 4; ++n) acc[m][n] = 0.f;
    }
    // --- Gram over this chunk, double-buffered gathers
    const int64_t nb = (it.k1 - it.k0 + BATCH - 1) / BATCH;
    if (nb > 0) issue_batch<NB, HAS_W>(p, stage[0], it.k0, it.k1, lane);
    for (int64_t s = 0; s < nb; ++s) {
        if (s + 1 < nb) {
            issue_batch<NB, HAS_W>(p, stage[(s + 1) & 1], it.k0 + (s + 1) * BATCH, it.k1, lane);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        accumulate<NB, HAS_W>(stage[s & 1], team, bi, bj, acc, rhs);
        __syncwarp();
    }
#pragma unroll
    for (int off = C::TS; off < 32; off <<= 1) {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            rhs[m] += __shfl_xor_sync(FULL, rhs[m], off);
#pragma unroll
            for (int n = 0; n < 4; ++n) acc[m][n] += __shfl_xor_sync(FULL, acc[m][n], off);
        }
    }

    // --- multi-chunk rows: publish the partial, last finisher reduces
    if (it.nch > 1) {
        float *slot0 = p.partials + (size_t)p.slot_off[it.j] * C::PSTRIDE;
        if (team == 0 && tile_ok) {
            float *dst = slot0 + (size_t)it.c * C::PSTRIDE + t * 20;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
#pragma unroll
                for (int n = 0; n < 4; ++n) dst[m * 4 + n] = acc[m][n];
                dst[16 + m] = rhs[m];
            }
        }
        __threadfence();
        __syncwarp();
        int prev = 0;
        if (lane == 0) prev = atomicAdd(p.counters + it.j, 1);
        prev = __shfl_sync(FULL, prev, 0);
        if (prev != it.nch - 1) return;
        __threadfence();
        if (lane == 0) p.counters[it.j] = 0;  // ready for the next half-step
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            rhs[m] = 0.f;
#pragma unroll
            for (int n = 0; n < 4; ++n) acc[m][n] = 0.f;
        }
        if (tile_ok) {
            for (int c = team; c < it.nch; c += C::TPW) {
                const float *src = slot0 + (size_t)c * C::PSTRIDE + t * 20;
#pragma unroll
                for (int m = 0; m < 4; ++m) {
#pragma unroll
                    for (int n = 0; n < 4; ++n) acc[m][n] += __ldcg(src + m * 4 + n);
                    rhs[m] += __ldcg(src + 16 + m);
                }
            }
        }
#pragma unroll
        for (int off = C::TS; off < 32; off <<= 1) {
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                rhs[m] += __shfl_xor_sync(FULL, rhs[m], off);
#pragma unroll
                for (int n = 0; n < 4; ++n) acc[m][n] += __shfl_xor_sync(FULL, acc[m][n], off);
            }
        }
    }

    // --- regulariser, empty rows
    const int D = p.D, r = it.r;
    const float S = p.tax_S ? p.tax_S[r] : 0.f;
    if (it.n == 0 && S == 0.f) {
        if (p.lam_c > 0.f || p.lam_n > 0.f) {
            if (lane < p.ld) p.out[(size_t)r * p.ld + lane] = 0.f;
        } else if (lane == 0) {
            report_fail(p.fail, r);
        }
        return;
    }
    const float diag = p.lam_c + p.lam_n * (float)it.n + p.tau * S;

    // --- stage A (lower) and b in shared memory: M[i][0..LD-1], b in M[i][LD]
    float *M = wbuf;  // stage buffers are free now
    constexpr int MS = C::LD + 1;
    __syncwarp();
    if (team == 0 && tile_ok) {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int row = 4 * bi + m;
#pragma unroll
            for (int n = 0; n < 4; ++n) {
                const int col = 4 * bj + n;
                float v = acc[m][n];
                if (row == col) v += diag;
                if (col <= row) M[row * MS + col] = v;
            }
            if (bi == bj) {
                float bv = rhs[m];
                if (p.tax_T && row < D) bv = fmaf(p.tau, p.tax_T[(size_t)r * p.ld + row], bv);
                M[row * MS + C::LD] = bv;
            }
        }
    }
    __syncwarp();
    float a[C::LD];
#pragma unroll
    for (int j2 = 0; j2 < C::LD; ++j2) a[j2] = (lane < D && j2 <= lane) ? M[lane * MS + j2] : 0.f;
    float b = lane < D ? M[lane * MS + C::LD] : 0.f;

    // --- right-looking Cholesky, lane i owns row i
    bool bad = false;
#pragma unroll
    for (int j2 = 0; j2 < C::LD; ++j2) {
        if (j2 < D) {
            const float piv = __shfl_sync(FULL, a[j2], j2);
            bad |= !(piv > 0.f) || !isfinite(piv);
            const float l = sqrtf(piv);
            const float inv = 1.f / l;
            if (lane == j2) a[j2] = l;
            else if (lane > j2) a[j2] *= inv;
#pragma unroll
            for (int k2 = j2 + 1; k2 < C::LD; ++k2) {
                if (k2 < D) {
                    const float lk = __shfl_sync(FULL, a[j2], k2);
                    if (lane >= k2) a[k2] = fmaf(-a[j2], lk, a[k2]);
                }
            }
        }
    }
    if (bad) {
        if (lane == 0) report_fail(p.fail, r);
        return;
    }
    // forward: L y = b
#pragma unroll
    for (int j2 = 0; j2 < C::LD; ++j2) {
        if (j2 < D) {
            if (lane == j2) b = b / a[j2];
            const float yj = __shfl_sync(FULL, b, j2);
            if (lane > j2) b = fmaf(-a[j2], yj, b);
        }
    }
    // backward: L^T x = y, column j of L^T is row j of L (from shared memory)
    __syncwarp();
    if (lane < D) {
#pragma unroll
        for (int j2 = 0; j2 < C::LD; ++j2)
            if (j2 <= lane) M[lane * MS + j2] = a[j2];
    }
    __syncwarp();
    for (int j2 = D - 1; j2 >= 0; --j2) {
        if (lane == j2) b = b / M[j2 * MS + j2];
        const float xj = __shfl_sync(FULL, b, j2);
        if (lane < j2) b = fmaf(-M[j2 * MS + lane], xj, b);
    }
    if (lane < p.ld) p.out[(size_t)r * p.ld + lane] = lane < D ? b : 0.f;
}

// ---------------------------------------------------------------------------
// CTA path, 28 < D <= 128 (one CTA per work item)

constexpr int CTA_THREADS = 256;
constexpr int CTA_MAXNB = 32;

template <int NB, bool HAS_W>
__global__ void __launch_bounds__(CTA_THREADS) k_als_cta(AlsParams p) {
    constexpr int T = NB * (NB + 1) / 2;
    constexpr int TPT = (T + CTA_THREADS - 1) / CTA_THREADS;  // tiles per thread
    constexpr int LD = 4 * NB;
    constexpr int PSTRIDE = T * 20;
    extern __shared__ float4 smem4[];
    float *xs = reinterpret_cast<float *>(smem4);   // [BATCH][LD]
    float *ys = xs + BATCH * LD;                     // [BATCH] y, [BATCH] w
    float *M = ys + 2 * BATCH;                       // [LD][LD + 1]
    __shared__ int s_flag;
    const int tid = threadIdx.x;
    const int64_t item = blockIdx.x;
    if (item >= p.total_items) return;
    const ItemInfo it = item_info(p, item);
    const int D = p.D;

    int bi[TPT], bj[TPT];
#pragma unroll
    for (int q = 0; q < TPT; ++q) {
        int t = tid + q * CTA_THREADS, i = 0;
        if (t >= T) t = -1;
        bi[q] = bj[q] = 0;
        if (t >= 0) {
            while ((i + 1) * (i + 2) / 2 <= t) ++i;
            bi[q] = i;
            bj[q] = t - i * (i + 1) / 2;
        }
    }
    float acc[TPT][4][4], rhs[TPT][4];
#pragma unroll
    for (int q = 0; q < TPT; ++q)
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            rhs[q][m] = 0.f;
#pragma unroll
            for (int n = 0; n < 4; ++n) acc[q][m][n] = 0.f;
        }
    for (int64_t k = it.k0; k < it.k1; k += BATCH) {
        __syncthreads();
        for (int e = tid; e < BATCH * NB; e += CTA_THREADS) {
            const int rr = e / NB, part = e - rr * NB;
            const int64_t kk = k + rr;
            const bool ok = kk < it.k1;
            const float *g = ok ? p.fixed + (size_t)p.idx[kk] * p.ld + part * 4 : p.fixed;
            cp_async16(xs + rr * LD + part * 4, g, ok ? 16 : 0);
        }
        cp_async_commit();
        if (tid < BATCH) {
            const int64_t kk = k + tid;
            const bool ok = kk < it.k1;
            ys[tid] = ok ? p.val[kk] - p.y_shift : 0.f;
            ys[BATCH + tid] = ok ? (HAS_W ? p.wts[kk] : 1.f) : 0.f;
        }
        cp_async_wait<0>();
        __syncthreads();
#pragma unroll
        for (int q = 0; q < TPT; ++q) {
            if (tid + q * CTA_THREADS >= T) continue;
            for (int kb = 0; kb < BATCH; ++kb) {
                float4 a = *reinterpret_cast<const float4 *>(xs + kb * LD + 4 * bi[q]);
                const float4 b = *reinterpret_cast<const float4 *>(xs + kb * LD + 4 * bj[q]);
                const float y = ys[kb];
                if (HAS_W) {
                    const float w = ys[BATCH + kb];
                    a.x *= w; a.y *= w; a.z *= w; a.w *= w;
                }
                const float av[4] = {a.x, a.y, a.z, a.w};
                const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                for (int m = 0; m < 4; ++m) {
#pragma unroll
                    for (int n = 0; n < 4; ++n) acc[q][m][n] = fmaf(av[m], bv[n], acc[q][m][n]);
                    rhs[q][m] = fmaf(y, av[m], rhs[q][m]);
                }
            }
        }
    }
    if (it.nch > 1) {
        float *slot0 = p.partials + (size_t)p.slot_off[it.j] * PSTRIDE;
#pragma unroll
        for (int q = 0; q < TPT; ++q) {
            const int t = tid + q * CTA_THREADS;
            if (t >= T) continue;
            float *dst = slot0 + (size_t)it.c * PSTRIDE + t * 20;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
#pragma unroll
                for (int n = 0; n < 4; ++n) dst[m * 4 + n] = acc[q][m][n];
                dst[16 + m] = rhs[q][m];
            }
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) s_flag = atomicAdd(p.counters + it.j, 1);
        __syncthreads();
        if (s_flag != it.nch - 1) return;
        __threadfence();
        if (tid == 0) p.counters[it.j] = 0;
#pragma unroll
        for (int q = 0; q < TPT; ++q) {
            const int t = tid + q * CTA_THREADS;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                rhs[q][m] = 0.f;
#pragma unroll
                for (int n = 0; n < 4; ++n) acc[q][m][n] = 0.f;
            }
            if (t >= T) continue;
            for (int c = 0; c < it.nch; ++c) {
                const float *src = slot0 + (size_t)c * PSTRIDE + t * 20;
#pragma unroll
                for (int m = 0; m < 4; ++m) {
#pragma unroll
                    for (int n = 0; n < 4; ++n) acc[q][m][n] += __ldcg(src + m * 4 + n);
                    rhs[q][m] += __ldcg(src + 16 + m);
                }
            }
        }
    }
    const int r = it.r;
    const float S = p.tax_S ? p.tax_S[r] : 0.f;
    if (it.n == 0 && S == 0.f) {
        if (p.lam_c > 0.f || p.lam_n > 0.f) {
            for (int i = tid; i < p.ld; i += CTA_THREADS) p.out[(size_t)r * p.ld + i] = 0.f;
        } else if (tid == 0) {
            report_fail(p.fail, r);
        }
        return;
    }
    const float diag = p.lam_c + p.lam_n * (float)it.n + p.tau * S;
    constexpr int MS = LD + 1;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < TPT; ++q) {
        if (tid + q * CTA_THREADS >= T) continue;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int row = 4 * bi[q] + m;
#pragma unroll
            for (int n = 0; n < 4; ++n) {
                const int col = 4 * bj[q] + n;
                float v = acc[q][m][n];
                if (row == col) v += diag;
                if (col <= row) M[row * MS + col] = v;
            }
            if (bi[q] == bj[q]) {
                float bv = rhs[q][m];
                if (p.tax_T && row < D) bv = fmaf(p.tau, p.tax_T[(size_t)r * p.ld + row], bv);
                M[row * MS + LD] = bv;
            }
        }
    }
    if (tid == 0) s_flag = 0;
    __syncthreads();
    // right-looking Cholesky, one column per step
    for (int j = 0; j < D; ++j) {
        const float piv = M[j * MS + j];
        if (!(piv > 0.f) || !isfinite(piv)) {
            if (tid == 0) report_fail(p.fail, r);
            return;  // uniform: every thread read the same pivot
        }
        const float l = sqrtf(piv), inv = 1.f / l;
        __syncthreads();
        if (tid == 0) M[j * MS + j] = l;
        for (int i = j + 1 + tid; i < D; i += CTA_THREADS) M[i * MS + j] *= inv;
        __syncthreads();
        const int w = D - j - 1;
        for (int e = tid; e < w * w; e += CTA_THREADS) {
            const int i = j + 1 + e / w, k2 = j + 1 + e % w;
            if (k2 <= i) M[i * MS + k2] = fmaf(-M[i * MS + j], M[k2 * MS + j], M[i * MS + k2]);
        }
        __syncthreads();
    }
    // triangular solves by one warp (D <= 128: 4 rows per lane)
    if (tid < 32) {
        for (int j = 0; j < D; ++j) {
            if (tid == 0) M[j * MS + LD] /= M[j * MS + j];
            __syncwarp();
            const float yj = M[j * MS + LD];
            for (int i = j + 1 + tid; i < D; i += 32) M[i * MS + LD] -= M[i * MS + j] * yj;
            __syncwarp();
        }
        for (int j = D - 1; j >= 0; --j) {
            if (tid == 0) M[j * MS + LD] /= M[j * MS + j];
            __syncwarp();
            const float xj = M[j * MS + LD];
            for (int i = tid; i < j; i += 32) M[i * MS + LD] -= M[j * MS + i] * xj;
            __syncwarp();
        }
        for (int i = tid; i < p.ld; i += 32)
            p.out[(size_t)r * p.ld + i] = i < D ? M[i * MS + LD] : 0.f;
    }
}

// ---------------------------------------------------------------------------
// dispatch

template <int NB, bool W>
int launch_warp(const AlsParams &p, cudaStream_t s) {
    using C = WarpCfg<NB>;
    constexpr int warps = 8;
    const size_t smem = sizeof(float) * C::WARP_FLOATS * warps;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_als_warp<NB, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attr = true;
    }
    const int64_t grid = ceil_div(p.total_items, warps);
    if (grid > 0) k_als_warp<NB, W><<<(unsigned)grid, warps * 32, smem, s>>>(p);
    return check_launch("mcf_als_half_step(warp)");
}

template <int NB, bool W>
int launch_cta(const AlsParams &p, cudaStream_t s) {
    constexpr int LD = 4 * NB;
    const size_t smem = sizeof(float) * (BATCH * LD + 2 * BATCH + LD * (LD + 1));
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_als_cta<NB, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attr = true;
    }
    if (p.total_items > 0) k_als_cta<NB, W><<<(unsigned)p.total_items, CTA_THREADS, smem, s>>>(p);
    return check_launch("mcf_als_half_step(cta)");
}

template <bool W>
int dispatch(const AlsParams &p, cudaStream_t s) {
    const int nb = (p.D + 3) / 4;
    switch (nb) {
        case 1: return launch_warp<1, W>(p, s);
        case 2: return launch_warp<2, W>(p, s);
        case 3: return launch_warp<3, W>(p, s);
        case 4: return launch_warp<4, W>(p, s);
        case 5: return launch_warp<5, W>(p, s);
        case 6: return launch_warp<6, W>(p, s);
        case 7: return launch_warp<7, W>(p, s);
        default: break;
    }
    if (nb <= 9) return launch_cta<9, W>(p, s);
    if (nb <= 13) return launch_cta<13, W>(p, s);
    if (nb <= 16) return launch_cta<16, W>(p, s);
    if (nb <= 25) return launch_cta<25, W>(p, s);
    return launch_cta<32, W>(p, s);
}

size_t pstride_of(int D) {
    const int nb = (D + 3) / 4;
    const int T = nb * (nb + 1) / 2;
    return (size_t)T * 20;
}

struct PlanLayout {
    int32_t *items, *slots, *item_row;
    void *scan_tmp;
    size_t scan_bytes;
};

PlanLayout carve_plan(void *buf, size_t cap, int32_t n_list, int64_t nnz, int32_t chunk,
                      size_t *need) {
    Carve c(buf, cap);
    PlanLayout L;
    L.items = c.take<int32_t>((size_t)n_list + 1);
    L.slots = c.take<int32_t>((size_t)n_list + 1);
    const int64_t max_items = (int64_t)n_list + ceil_div(nnz, chunk) + 1;
    L.item_row = c.take<int32_t>((size_t)max_items);
    L.scan_bytes = scan_exclusive<int32_t>(nullptr, nullptr, (int64_t)n_list + 1, nullptr, 0,
                                           nullptr, nullptr);
    L.scan_tmp = c.take<char>(L.scan_bytes + 256);
    *need = c.used;
    return L;
}

}  // namespace
}  // namespace mcf

using namespace mcf;

extern "C" size_t mcf_als_plan_bytes(int32_t n_list, int64_t nnz, int32_t chunk) {
    size_t need = 0;
    if (chunk < 1) chunk = 1;
    carve_plan(nullptr, 0, n_list, nnz, chunk, &need);
    return need;
}

extern "C" int mcf_als_plan(const int64_t *ptr, const int32_t *row_list, int32_t n_list,
                            int32_t row_lo, int32_t chunk, int64_t nnz, void *plan,
                            size_t plan_bytes, int64_t *totals, void *stream) {
    if (!ptr || n_list < 0 || chunk < BATCH || chunk % BATCH || !totals || nnz < 0) {
        set_error("mcf_als_plan: invalid arguments (chunk must be a positive multiple of 32)");
        return MCF_E_ARG;
    }
    size_t need = 0;
    PlanLayout L = carve_plan(plan, plan_bytes, n_list, nnz, chunk, &need);
    if (!plan || plan_bytes < need) {
        set_error("mcf_als_plan: plan buffer too small");
        return MCF_E_WORKSPACE;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int grid = (int)std::min<int64_t>(ceil_div((int64_t)n_list + 1, 256), 148 * 16);
    k_plan_count<<<grid, 256, 0, s>>>(ptr, row_list, n_list, row_lo, chunk, L.items, L.slots);
    int err = 0;
    scan_exclusive<int32_t>(L.items, L.items, (int64_t)n_list + 1, L.scan_tmp, L.scan_bytes, s,
                            &err);
    scan_exclusive<int32_t>(L.slots, L.slots, (int64_t)n_list + 1, L.scan_tmp, L.scan_bytes, s,
                            &err);
    if (err) {
        set_error("mcf_als_plan: scan workspace");
        return MCF_E_WORKSPACE;
    }
    if (n_list > 0) k_plan_fill<<<grid, 256, 0, s>>>(L.items, n_list, L.item_row);
    int32_t tot[2];
    int rc;
    if ((rc = cuda_status(cudaMemcpyAsync(&tot[0], L.items + n_list, sizeof(int32_t),
                                          cudaMemcpyDeviceToHost, s), "memcpy")))
        return rc;
    if ((rc = cuda_status(cudaMemcpyAsync(&tot[1], L.slots + n_list, sizeof(int32_t),
                                          cudaMemcpyDeviceToHost, s), "memcpy")))
        return rc;
    if ((rc = cuda_status(cudaStreamSynchronize(s), "sync"))) return rc;
    totals[0] = tot[0];
    totals[1] = tot[1];
    return check_launch("mcf_als_plan");
}

extern "C" size_t mcf_als_workspace_bytes(int32_t n_list, int64_t slots, int32_t D) {
    if (D < 1 || n_list < 0 || slots < 0) return 0;
    return align_up(sizeof(int32_t) * (size_t)n_list, 256) +
           sizeof(float) * (size_t)slots * pstride_of(D);
}

extern "C" int mcf_als_half_step(const int64_t *ptr, const int32_t *idx, const float *val,
                                 const float *wts, const float *fixed, float *out, int32_t D,
                                 float lam_c, float lam_n, float y_shift, const float *tax_S,
                                 const float *tax_T, float tau, const int32_t *row_list,
                                 int32_t n_list, int32_t row_lo, int32_t chunk, const void *plan,
                                 int64_t total_items, int64_t *fail_row, void *ws,
                                 size_t ws_bytes, void *stream) {
    if (D < 1 || D > 128) {
        set_error("mcf_als_half_step: D must be in [1, 128]");
        return MCF_E_UNSUPPORTED;
    }
    if (!ptr || !fixed || !out || !plan || !fail_row || n_list < 0 || total_items < 0 ||
        chunk < BATCH || chunk % BATCH) {
        set_error("mcf_als_half_step: invalid arguments");
        return MCF_E_ARG;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int rc;
    if ((rc = cuda_status(cudaMemsetAsync(fail_row, 0xff, sizeof(int64_t), s), "memset")))
        return rc;
    if (n_list == 0 || total_items == 0) return MCF_OK;
    size_t need_plan = 0;
    PlanLayout L = carve_plan(const_cast<void *>(plan), SIZE_MAX, n_list, 0, chunk, &need_plan);
    AlsParams p{};
    p.ptr = ptr; p.idx = idx; p.val = val; p.wts = wts; p.fixed = fixed; p.out = out;
    p.D = D; p.ld = mcf_factor_ld(D);
    p.lam_c = lam_c; p.lam_n = lam_n; p.y_shift = y_shift; p.tau = tau;
    p.tax_S = tax_S; p.tax_T = tax_T;
    p.row_list = row_list; p.n_list = n_list; p.row_lo = row_lo; p.chunk = chunk;
    p.item_off = L.items; p.slot_off = L.slots;
    // item_row sits after items/slots; its offset does not depend on nnz
    p.item_row = L.item_row;
    p.total_items = total_items;
    p.fail = reinterpret_cast<unsigned long long *>(fail_row);
    // workspace: counters [n_list] + partial slots
    Carve c(ws, ws_bytes);
    p.counters = c.take<int32_t>((size_t)n_list);
    p.partials = c.take<float>(0);
    const size_t fixed_part = c.used;
    if (!ws || ws_bytes < fixed_part) {
        set_error("mcf_als_half_step: workspace too small");
        return MCF_E_WORKSPACE;
    }
    p.partials = reinterpret_cast<float *>(static_cast<char *>(ws) + fixed_part);
    if ((rc = cuda_status(cudaMemsetAsync(p.counters, 0, sizeof(int32_t) * (size_t)n_list, s),
                          "memset")))
        return rc;
    return wts ? dispatch<true>(p, s) : dispatch<false>(p, s);
}
