// ALS half-step: fused ragged Gram + regulariser + Cholesky solve (sm_100a).
//
// Replaces _kernels.als_solve_rows (reference _kernels.py:151-215) driven by
// factor.als_half_step / parallel.run_blocks (factor.py:512-538,
// parallel.py:134-145).  For every planned row r:
//
//     A_r = sum_k w_k x_k x_k^T + (lam_c + lam_n n_r + tau S_r) I
//     b_r = sum_k w_k (y_k - y_shift) x_k + tau T_r,     out_r = A_r^{-1} b_r
//
// Kernel per factor dimension (dispatch / dispatch_pair below):
//   D <= 20      k_als_pair: row-parallel lane pairs, FFMA2 Gram over a
//                4-rating cp.async + mbarrier ring, one-lane Cholesky;
//                hot rows as chunk partials summed by k_als_heavy.  Also the
//                bias-last D + 1 systems of MFITR (Schur-complement bias).
//   D 21..28     k_als_warp: 4x4 register tiles, one tile per lane of a team,
//                shuffle Cholesky.
//   D 29..103    k_als_tile_warp: warp per work item, 8x8 register tiles,
//                augmented Gram (rating in column D), blocked register
//                Cholesky, persistent warps.
//   D 104..128   k_als_cta: CTA per work item, CTA Cholesky.
// Work decomposition (the "plan"): every row is cut into chunks of at most
// CHUNK ratings (on the pair path CHUNK follows the layout size).  Rows
// spanning several chunks (Zipf-hot items, up to ~1 M ratings) write partial
// Grams to a workspace slot and are summed in chunk order -- a fixed order,
// so results are deterministic and independent of scheduling -- then solved.
// fp32 throughout; the pivot test matches the reference (s > 0 and finite,
// _kernels.py:197).  Every solved row can also be stored into peer replicas
// (the fused all-gather of the sharded sweep, put_out).

#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "als_params.cuh"
#include "../../include/mcf.h"

namespace mcf {
namespace {


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
            if (lane < p.ld) put_out(p, r, lane, 0.f);
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
                if (row == col) v += diag_at(p, row, diag, (float)it.n);
                if (col <= row) M[row * MS + col] = v;
            }
            if (bi == bj) {
                float bv = rhs[m];
                if (row < D) bv = tax_rhs(p, r, row, bv);
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
            const float inv = rsqrtf(piv), l = piv * inv;   // MUFU.RSQ (~2 ulp)
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
    if (lane < p.ld) put_out(p, r, lane, lane < D ? b : 0.f);
}

// Paired FP32 FMA (sm_100 FFMA2): acc.{x,y} += a * b.{x,y}; the scalar a is
// a broadcast operand of the instruction (no register moves).
__device__ __forceinline__ void ffma2(float2 &acc, float a, float bx, float by) {
    unsigned long long A, B, C;
    asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a));
    asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(bx), "f"(by));
    asm("mov.b64 %0, {%1, %2};" : "=l"(C) : "f"(acc.x), "f"(acc.y));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C) : "l"(A), "l"(B));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(acc.x), "=f"(acc.y) : "l"(C));
}

// ---------------------------------------------------------------------------
// wide path, 28 < D <= 128 (configs 3 and 4): one CTA per work item
//
// The lower triangle of A is cut into 8x8 tiles (NB8 = ceil(D/8) blocks,
// T8 = NB8(NB8+1)/2 tiles) listed row-block by row-block, so the lanes of a
// warp share few row blocks and their row-operand loads are shared-memory
// broadcasts.  A team of TEAM threads owns all tiles (TPT per thread);
// 128/TEAM teams split each 32-rating batch (k-split) and are reduced in a
// fixed order.  Per rating a thread loads 2 x 8 floats (4 LDS.128) and issues
// 32 FFMA2 + 4 FFMA2 (rhs): 4 FMA per loaded float.  Partner rows are
// gathered by cp.async, double buffered.  Hot rows: chunks publish their
// partial tiles, the last chunk to finish sums them in chunk order.  The
// solve is a CTA-cooperative right-looking Cholesky on the staged matrix.

constexpr int CTA_THREADS = 128;

template <int NB8>
struct WideCfg {
    static constexpr int LDK = 8 * NB8;
    static constexpr int T8 = NB8 * (NB8 + 1) / 2;
    static constexpr int TEAM = T8 <= 32 ? 32 : T8 <= 64 ? 64 : 128;
    static constexpr int TEAMS = CTA_THREADS / TEAM;
    static constexpr int TPT = (T8 + TEAM - 1) / TEAM;
    static constexpr int ROWS = LDK + 4;                // smem row stride (floats)
    static constexpr int STAGE = BATCH * ROWS + 2 * BATCH;
    static constexpr int MS = LDK + 1;                  // solve matrix stride
    static constexpr int SMEM_FLOATS =
        (2 * STAGE > LDK * MS ? 2 * STAGE : LDK * MS);
    static constexpr int PSTRIDE = T8 * 72;             // 64 tile + 8 rhs floats per tile
};

__device__ __forceinline__ void tile_of(int t, int &I, int &J) {
    int i = 0;
    while ((i + 1) * (i + 2) / 2 <= t) ++i;
    I = i;
    J = t - i * (i + 1) / 2;
}

template <int NB8, bool HAS_W>
__global__ void __launch_bounds__(CTA_THREADS) k_als_cta(AlsParams p) {
    using C = WideCfg<NB8>;
    extern __shared__ float4 smem4[];
    float *sm = reinterpret_cast<float *>(smem4);
    float *M = sm;   // aliases the stages once the Gram is done
    __shared__ int s_flag;
    const int tid = threadIdx.x;
    const int team = tid / C::TEAM, tt = tid % C::TEAM;
    const int64_t item = blockIdx.x;
    if (item >= p.total_items) return;
    const ItemInfo it = item_info(p, item);
    const int D = p.D;
    const int nb4_real = (D + 3) / 4;   // 16 B blocks present in `fixed`

    int tI[C::TPT], tJ[C::TPT];
    bool tok[C::TPT];
#pragma unroll
    for (int q = 0; q < C::TPT; ++q) {
        const int t = tt + q * C::TEAM;
        tok[q] = t < C::T8;
        tile_of(tok[q] ? t : 0, tI[q], tJ[q]);
    }
    float2 acc[C::TPT][8][4];
    float2 rhs[C::TPT][4];
#pragma unroll
    for (int q = 0; q < C::TPT; ++q) {
#pragma unroll
        for (int m = 0; m < 8; ++m)
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[q][m][k] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < 4; ++k) rhs[q][k] = make_float2(0.f, 0.f);
    }

    // Per-batch operands (partner ids, ratings, weights) are loaded by warp 0
    // one batch ahead into a 3-slot ring; the partner-row gathers of batch
    // b+1 (cp.async) overlap the FMAs of batch b.
    __shared__ int ring_id[3][BATCH];
    __shared__ float ring_y[3][BATCH], ring_w[3][BATCH];
    auto load_ops = [&](int64_t b) {   // warp 0: batch b -> ring slot b % 3
        if (tid < BATCH) {
            const int64_t kk = it.k0 + b * BATCH + tid;
            const bool ok = kk < it.k1;
            ring_id[b % 3][tid] = ok ? p.idx[kk] : -1;
            ring_y[b % 3][tid] = ok ? p.val[kk] - p.y_shift : 0.f;
            ring_w[b % 3][tid] = ok ? (HAS_W ? p.wts[kk] : 1.f) : 0.f;
        }
    };
    auto issue = [&](int64_t b, float *stage) {
        const int *ids = ring_id[b % 3];
        for (int e = tid; e < BATCH * (C::LDK / 4); e += CTA_THREADS) {
            const int rr = e / (C::LDK / 4), part = e - rr * (C::LDK / 4);
            const int id = ids[rr];
            const bool ok = id >= 0 && part < nb4_real;
            const float *g = ok ? p.fixed + (size_t)id * p.ld + part * 4 : p.fixed;
            cp_async16(stage + rr * C::ROWS + part * 4, g, ok ? 16 : 0);
        }
        cp_async_commit();
    };
    const int64_t nbatch = (it.k1 - it.k0 + BATCH - 1) / BATCH;
    if (nbatch > 0) {
        load_ops(0);
        if (nbatch > 1) load_ops(1);
        __syncthreads();
        issue(0, sm);
    }
    for (int64_t bt = 0; bt < nbatch; ++bt) {
        float *cur = sm + (bt & 1) * C::STAGE;
        if (bt + 1 < nbatch) {
            issue(bt + 1, sm + ((bt + 1) & 1) * C::STAGE);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        if (bt + 2 < nbatch) load_ops(bt + 2);   // consumed after the next barrier
        __syncthreads();
        const float *xs = cur;
        const float *ys = ring_y[bt % 3];
        const float *wsv = ring_w[bt % 3];
        for (int kb = team; kb < BATCH; kb += C::TEAMS) {
            const float *xr = xs + kb * C::ROWS;
            const float y = ys[kb];
            const float w = HAS_W ? wsv[kb] : 1.f;
#pragma unroll
            for (int q = 0; q < C::TPT; ++q) {
                if (!tok[q]) continue;
                const float4 a0 = *reinterpret_cast<const float4 *>(xr + 8 * tI[q]);
                const float4 a1 = *reinterpret_cast<const float4 *>(xr + 8 * tI[q] + 4);
                const float4 b0 = *reinterpret_cast<const float4 *>(xr + 8 * tJ[q]);
                const float4 b1 = *reinterpret_cast<const float4 *>(xr + 8 * tJ[q] + 4);
                float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                if (HAS_W) {
#pragma unroll
                    for (int m = 0; m < 8; ++m) a[m] *= w;
                }
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    ffma2(acc[q][m][0], a[m], b0.x, b0.y);
                    ffma2(acc[q][m][1], a[m], b0.z, b0.w);
                    ffma2(acc[q][m][2], a[m], b1.x, b1.y);
                    ffma2(acc[q][m][3], a[m], b1.z, b1.w);
                }
#pragma unroll
                for (int m = 0; m < 4; ++m) ffma2(rhs[q][m], y, a[2 * m], a[2 * m + 1]);
            }
        }
        __syncthreads();   // this stage is refilled two iterations later
    }

    // multi-chunk rows: publish this chunk's partial tiles, last finisher sums
    if (it.nch > 1) {
        float *slot0 = p.partials + (size_t)p.slot_off[it.j] * C::PSTRIDE;
        // team-reduce into the partial: teams write in turn (fixed order)
        for (int tm = 0; tm < C::TEAMS; ++tm) {
            if (team == tm) {
#pragma unroll
                for (int q = 0; q < C::TPT; ++q) {
                    const int t = tt + q * C::TEAM;
                    if (!tok[q]) continue;
                    float *dst = slot0 + (size_t)it.c * C::PSTRIDE + t * 72;
#pragma unroll
                    for (int m = 0; m < 8; ++m)
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            float2 v = acc[q][m][k];
                            if (tm > 0) {
                                v.x += dst[m * 8 + 2 * k];
                                v.y += dst[m * 8 + 2 * k + 1];
                            }
                            dst[m * 8 + 2 * k] = v.x;
                            dst[m * 8 + 2 * k + 1] = v.y;
                        }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        float2 v = rhs[q][k];
                        if (tm > 0) {
                            v.x += dst[64 + 2 * k];
                            v.y += dst[64 + 2 * k + 1];
                        }
                        dst[64 + 2 * k] = v.x;
                        dst[64 + 2 * k + 1] = v.y;
                    }
                }
            }
            __syncthreads();
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) s_flag = atomicAdd(p.counters + it.j, 1);
        __syncthreads();
        if (s_flag != it.nch - 1) return;
        __threadfence();
        if (tid == 0) p.counters[it.j] = 0;
        // last finisher: team 0 sums all chunks' tiles in chunk order
#pragma unroll
        for (int q = 0; q < C::TPT; ++q) {
#pragma unroll
            for (int m = 0; m < 8; ++m)
#pragma unroll
                for (int k = 0; k < 4; ++k) acc[q][m][k] = make_float2(0.f, 0.f);
#pragma unroll
            for (int k = 0; k < 4; ++k) rhs[q][k] = make_float2(0.f, 0.f);
            const int t = tt + q * C::TEAM;
            if (team != 0 || !tok[q]) continue;
            for (int c = 0; c < it.nch; ++c) {
                const float *src = slot0 + (size_t)c * C::PSTRIDE + t * 72;
#pragma unroll
                for (int m = 0; m < 8; ++m)
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        acc[q][m][k].x += __ldcg(src + m * 8 + 2 * k);
                        acc[q][m][k].y += __ldcg(src + m * 8 + 2 * k + 1);
                    }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    rhs[q][k].x += __ldcg(src + 64 + 2 * k);
                    rhs[q][k].y += __ldcg(src + 64 + 2 * k + 1);
                }
            }
        }
    }

    const int r = it.r;
    const float S = p.tax_S ? p.tax_S[r] : 0.f;
    if (it.n == 0 && S == 0.f) {
        if (p.lam_c > 0.f || p.lam_n > 0.f) {
            for (int i = tid; i < p.ld; i += CTA_THREADS) put_out(p, r, i, 0.f);
        } else if (tid == 0) {
            report_fail(p.fail, r);
        }
        return;
    }
    const float diag = p.lam_c + p.lam_n * (float)it.n + p.tau * S;
    constexpr int MS = C::MS;
    // stage A (lower) + b into M; teams fold in turn (fixed order)
    __syncthreads();
    const bool single = it.nch > 1;   // after the chunk sum only team 0 holds data
    for (int tm = 0; tm < (single ? 1 : C::TEAMS); ++tm) {
        if (team == tm) {
#pragma unroll
            for (int q = 0; q < C::TPT; ++q) {
                if (!tok[q]) continue;
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    const int row = 8 * tI[q] + m;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            const int col = 8 * tJ[q] + 2 * k + hh;
                            if (col <= row) {
                                const float v = hh ? acc[q][m][k].y : acc[q][m][k].x;
                                M[row * MS + col] = tm == 0 ? v : M[row * MS + col] + v;
                            }
                        }
                    }
                }
                if (tI[q] == tJ[q]) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            const int row = 8 * tI[q] + 2 * k + hh;
                            const float v = hh ? rhs[q][k].y : rhs[q][k].x;
                            M[row * MS + C::LDK] = tm == 0 ? v : M[row * MS + C::LDK] + v;
                        }
                    }
                }
            }
        }
        __syncthreads();
    }
    for (int i = tid; i < C::LDK; i += CTA_THREADS) {
        if (i < D) {
            M[i * MS + i] += diag_at(p, i, diag, (float)it.n);
            M[i * MS + C::LDK] = tax_rhs(p, r, i, M[i * MS + C::LDK]);
        } else {   // padding rows: identity, zero rhs (their solution is 0)
            M[i * MS + i] = 1.f;
            M[i * MS + C::LDK] = 0.f;
        }
    }
    __syncthreads();

    // ---- blocked right-looking Cholesky on the 8x8 tiles (team-0 threads own
    // their tiles in registers; the current panel lives in shared memory):
    // per block column J: factor the diagonal tile (+ its inverse), form the
    // panel L_IJ = A_IJ L_JJ^{-T}, update the trailing tiles A_IK -= L_IJ L_KJ^T.
    float t[C::TPT][8][8];
    const bool own = team == 0;
#pragma unroll
    for (int q = 0; q < C::TPT; ++q) {
#pragma unroll
        for (int m = 0; m < 8; ++m)
#pragma unroll
            for (int n = 0; n < 8; ++n) {
                const int row = 8 * tI[q] + m, col = 8 * tJ[q] + n;
                t[q][m][n] = (own && tok[q] && col <= row) ? M[row * MS + col]
                           : (own && tok[q] && tI[q] == tJ[q]) ? M[col * MS + row] : 0.f;
            }
    }
    float bvec = tid < C::LDK ? M[tid * MS + C::LDK] : 0.f;
    __syncthreads();
    float *PAN = M;                          // [NB8][64] current panel
    float *LINV = M + NB8 * 64;              // [64] inverse of the diagonal tile
    if (tid == 0) s_flag = 0;
    __syncthreads();
    for (int J = 0; J < NB8; ++J) {
        // (a) diagonal tile
#pragma unroll
        for (int q = 0; q < C::TPT; ++q) {
            if (!(own && tok[q] && tI[q] == J && tJ[q] == J)) continue;
            bool bad = false;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                float d = t[q][c][c];
#pragma unroll
                for (int k = 0; k < c; ++k) d = fmaf(-t[q][c][k], t[q][c][k], d);
                bad |= !(d > 0.f) || !isfinite(d);
                const float inv = rsqrtf(d), l = d * inv;   // MUFU.RSQ (~2 ulp)
                t[q][c][c] = l;
#pragma unroll
                for (int r2 = c + 1; r2 < 8; ++r2) {
                    float v = t[q][r2][c];
#pragma unroll
                    for (int k = 0; k < c; ++k) v = fmaf(-t[q][r2][k], t[q][c][k], v);
                    t[q][r2][c] = v * inv;
                }
            }
            // inverse of the lower-triangular tile
            float li[8][8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
#pragma unroll
                for (int r2 = 0; r2 < 8; ++r2) li[r2][c] = 0.f;
                li[c][c] = 1.f / t[q][c][c];
#pragma unroll
                for (int r2 = c + 1; r2 < 8; ++r2) {
                    float v = 0.f;
#pragma unroll
                    for (int k = c; k < r2; ++k) v = fmaf(t[q][r2][k], li[k][c], v);
                    li[r2][c] = -v / t[q][r2][r2];
                }
            }
#pragma unroll
            for (int m = 0; m < 8; ++m)
#pragma unroll
                for (int n = 0; n < 8; ++n) {
                    LINV[m * 8 + n] = li[m][n];
                    PAN[J * 64 + m * 8 + n] = n <= m ? t[q][m][n] : 0.f;
                }
            if (bad) s_flag = 1;
        }
        __syncthreads();
        if (s_flag) {
            if (tid == 0) report_fail(p.fail, r);
            return;
        }
        // (b) panel tiles below the diagonal
#pragma unroll
        for (int q = 0; q < C::TPT; ++q) {
            if (!(own && tok[q] && tJ[q] == J && tI[q] > J)) continue;
            float l2[8][8];
#pragma unroll
            for (int m = 0; m < 8; ++m)
#pragma unroll
                for (int n = 0; n < 8; ++n) {
                    float v = 0.f;
#pragma unroll
                    for (int k = 0; k <= n; ++k) v = fmaf(t[q][m][k], LINV[n * 8 + k], v);
                    l2[m][n] = v;
                }
#pragma unroll
            for (int m = 0; m < 8; ++m)
#pragma unroll
                for (int n = 0; n < 8; ++n) {
                    t[q][m][n] = l2[m][n];
                    PAN[tI[q] * 64 + m * 8 + n] = l2[m][n];
                }
        }
        __syncthreads();
        // (c) trailing update
#pragma unroll
        for (int q = 0; q < C::TPT; ++q) {
            if (!(own && tok[q] && tJ[q] > J)) continue;
            const float *pi = PAN + tI[q] * 64, *pk = PAN + tJ[q] * 64;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                float ci[8], ck[8];
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    ci[m] = pi[m * 8 + k];
                    ck[m] = pk[m * 8 + k];
                }
#pragma unroll
                for (int m = 0; m < 8; ++m)
#pragma unroll
                    for (int n = 0; n < 8; ++n) t[q][m][n] = fmaf(-ci[m], ck[n], t[q][m][n]);
            }
        }
        __syncthreads();
    }
    // ---- triangular solves: the L tiles go to shared memory, one warp solves
    float *LT = M;                           // [T8][64] tile-major
    float *vb = M + C::T8 * 64;              // [LDK] rhs -> solution
#pragma unroll
    for (int q = 0; q < C::TPT; ++q) {
        if (!(own && tok[q])) continue;
        const int tix = tI[q] * (tI[q] + 1) / 2 + tJ[q];
#pragma unroll
        for (int m = 0; m < 8; ++m)
#pragma unroll
            for (int n = 0; n < 8; ++n) LT[tix * 64 + m * 8 + n] = t[q][m][n];
    }
    if (tid < C::LDK) vb[tid] = bvec;
    __syncthreads();
    auto Lat = [&](int i, int k) {   // L[i][k], k <= i
        const int I = i >> 3, K = k >> 3;
        return LT[(I * (I + 1) / 2 + K) * 64 + (i & 7) * 8 + (k & 7)];
    };
    if (tid < 32) {
        for (int j = 0; j < C::LDK; ++j) {
            if (tid == 0) vb[j] /= Lat(j, j);
            __syncwarp();
            const float yj = vb[j];
            for (int i = j + 1 + tid; i < C::LDK; i += 32) vb[i] = fmaf(-Lat(i, j), yj, vb[i]);
            __syncwarp();
        }
        for (int j = C::LDK - 1; j >= 0; --j) {
            if (tid == 0) vb[j] /= Lat(j, j);
            __syncwarp();
            const float xj = vb[j];
            for (int i = tid; i < j; i += 32) vb[i] = fmaf(-Lat(j, i), xj, vb[i]);
            __syncwarp();
        }
        for (int i = tid; i < p.ld; i += 32) put_out(p, r, i, i < D ? vb[i] : 0.f);
    }
}

// ---------------------------------------------------------------------------
// tile-warp path, 28 < D <= 104 (configs 3 and 4): one WARP per work item,
// the whole [A | b] system in the warp's registers
//
// The lower triangle of A is cut into 8x8 tiles (NB8 blocks, T8 tiles);
// tile t lives in lane t % 32, register slot t / 32 (S <= 3 slots).
//   Gram:  per rating a lane loads its tiles' two 8-float row pieces from
//          the gathered partner row (4 LDS.128 per tile) and issues 32 FFMA2
//          per tile; the lane holding a diagonal tile also accumulates that
//          block of b.  Partner rows are gathered with 16-byte cp.async into
//          a per-warp double buffer, partner ids are staged one batch ahead
//          in registers and broadcast with shuffles.
//   Solve: blocked right-looking Cholesky in registers (same algorithm as
//          the reference's row-oriented one, _kernels.py:187-203, reordered
//          by 8x8 blocks).  Block column J: the diagonal lane factors its
//          tile; panel lanes solve their tile against it and publish it
//          transposed to shared memory; every lane then updates its trailing
//          tiles with 32 FFMA2 per panel column.  Forward substitution rides
//          along (b in shared memory, one writer per block per step); the
//          back substitution walks block rows bottom-up (_kernels.py:204-213).
//          Only __syncwarp: rows never wait on other warps, so a handful of
//          warps per SM keep the FMA pipe busy while others are on barriers.
// Hot rows are split into chunks whose partial tiles are summed in chunk
// order by the last chunk to finish (deterministic).

template <int NB8>
struct TileWarpCfg {
    static constexpr int LDK = 8 * NB8;
    static constexpr int T8 = NB8 * (NB8 + 1) / 2;
    static constexpr int S = (T8 + 31) / 32;         // register tiles per lane
    static constexpr int BT = 16;                    // ratings per stage
    static constexpr int ROWS = LDK + 4;             // smem row stride (floats)
    static constexpr int STAGE = BT * ROWS + 2 * BT;
    // solve scratch: PT [8][LDK], L_JJ [64], inverse diagonal [LDK], b [LDK],
    // back-substitution flag
    static constexpr int SOLVE = 8 * LDK + 64 + LDK + LDK + 4;
    static constexpr int WARP_FLOATS = ((2 * STAGE > SOLVE ? 2 * STAGE : SOLVE) + 3) / 4 * 4;
    static constexpr int WARPS = 4;
    static constexpr int PSTRIDE = T8 * 72;           // 64 tile + 8 rhs floats per tile
    static_assert(S <= 3, "at most 3 register tiles per lane");
};

// Tile order: by block column, last column first (q = 0 is (NB-1, NB-1)),
// rows ascending inside a column.  Tile q lives in lane q % 32, slot q / 32,
// so slot 0 holds the columns the right-looking update touches longest and
// the later slots go idle early (the update of slot s runs only while one of
// its tiles is still trailing).
template <int NB>
__device__ __forceinline__ void tile_of_by_col(int q, int &I, int &K) {
    int k = NB - 1;
    while (q >= NB - k) {
        q -= NB - k;
        --k;
    }
    K = k;
    I = k + q;
}

// Every lane must hold at most one diagonal tile (one rhs block per lane).
constexpr bool diag_lanes_distinct(int nb) {
    int pos[16] = {};
    int q = 0;
    for (int k = nb - 1; k >= 0; --k) {
        pos[k] = q;
        q += nb - k;
    }
    for (int a = 0; a < nb; ++a)
        for (int b = a + 1; b < nb; ++b)
            if (pos[a] % 32 == pos[b] % 32) return false;
    return true;
}
static_assert(diag_lanes_distinct(4) && diag_lanes_distinct(6) && diag_lanes_distinct(7) &&
                  diag_lanes_distinct(8) && diag_lanes_distinct(10) && diag_lanes_distinct(13),
              "diagonal tiles share a lane");

__device__ __forceinline__ float &tel(float2 (&t)[8][4], int m, int n) {
    return (n & 1) ? t[m][n >> 1].y : t[m][n >> 1].x;
}

template <int NB8, bool HAS_W>
__device__ __forceinline__ void tile_warp_item(const AlsParams &p, int64_t item, float *sm,
                                               int lane) {
    using C = TileWarpCfg<NB8>;
    constexpr int S = C::S, LDK = C::LDK, BT = C::BT;
    const ItemInfo it = item_info(p, item);
    if (p.skip_min_n > 0 && it.n >= p.skip_min_n) return;   // the tensor-core kernel's row
    const int D = p.D;
    const int nb4_real = (D + 3) / 4;

    int tI[S], tJ[S];
    bool tok[S];
    int dslot = -1;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int t = lane + 32 * s;
        tok[s] = t < C::T8;
        tile_of_by_col<NB8>(tok[s] ? t : 0, tI[s], tJ[s]);
        if (tok[s] && tI[s] == tJ[s]) dslot = s;
    }

    // augmented Gram: the rating y rides in column D of every staged row, so
    // sum w [x|y][x|y]^T carries b = sum w y x in row D (no separate rhs FMAs)
    float2 acc[S][8][4];
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
        for (int m = 0; m < 8; ++m)
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[s][m][k] = make_float2(0.f, 0.f);

    // ---- Gram ---------------------------------------------------------------
    // raw loads only (consumed one stage later by issue(), so their latency
    // hides behind a stage of FMAs); the streams are L2-prefetched 4 stages ahead
    auto ld = [&](int64_t b, int &id, float &y, float &w) {
        const int64_t kk = it.k0 + b * BT + lane;
        const bool ok = lane < BT && kk < it.k1;
        id = ok ? p.idx[kk] : -1;
        y = ok ? p.val[kk] : 0.f;
        w = ok ? (HAS_W ? p.wts[kk] : 1.f) : 0.f;
        const int64_t pf = it.k0 + (b + 4) * BT;
        if (lane < 2 && pf < it.k1 && ((b & 1) == 0))
            prefetch_l2(lane ? (const void *)(p.val + pf) : (const void *)(p.idx + pf));
    };
    // staged row layout, "split halves": the low 4 floats of 8-block I sit
    // in 16-byte unit I, the high 4 in unit NB8 + I, so the a-side loads of
    // 8 lanes holding consecutive block rows I hit 8 distinct bank groups
    // lane pair (2 rr, 2 rr + 1) copies row rr: lane h takes the 16-byte
    // parts h, h+2, ... (adjacent parts in one instruction -> one 32-byte
    // sector), i.e. unit j (h = 0) or NB8 + j (h = 1) of the split halves
    static_assert(BT == 16, "one lane pair per staged row");
    auto issue = [&](int id, float y, float w, float *stage) {
        float *ys = stage + BT * C::ROWS;
        {
            const int rr = lane >> 1, h = lane & 1;
            const int rid = __shfl_sync(FULL, id, rr);
            const float *g = p.fixed + (size_t)(rid >= 0 ? rid : 0) * p.ld + 4 * h;
            float *dst = stage + rr * C::ROWS + 4 * NB8 * h;
#pragma unroll
            for (int j = 0; j < NB8; ++j) {
                const bool ok = rid >= 0 && 2 * j + h < nb4_real;
                cp_async16(dst + 4 * j, g + 8 * j, ok ? 16 : 0);
            }
        }
        if (lane < BT) {
            ys[lane] = id >= 0 ? y - p.y_shift : 0.f;
            ys[BT + lane] = w;
        }
        cp_async_commit();
    };
    const int64_t nbatch = (it.k1 - it.k0 + BT - 1) / BT;
    int nid = -1;
    float ny = 0.f, nw = 0.f;
    if (nbatch > 0) {
        int id0;
        float y0, w0;
        ld(0, id0, y0, w0);
        issue(id0, y0, w0, sm);
        if (nbatch > 1) ld(1, nid, ny, nw);
    }
    for (int64_t bt = 0; bt < nbatch; ++bt) {
        float *cur = sm + (bt & 1) * C::STAGE;
        if (bt + 1 < nbatch) {
            issue(nid, ny, nw, sm + ((bt + 1) & 1) * C::STAGE);
            if (bt + 2 < nbatch) ld(bt + 2, nid, ny, nw);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        const float *ys = cur + BT * C::ROWS;
        if (lane < BT)   // the copies have landed; column D in split-halves order
            cur[lane * C::ROWS + ((D & 4) ? 4 * NB8 : 0) + 4 * (D >> 3) + (D & 3)] = ys[lane];
        __syncwarp();
        for (int kb = 0; kb < BT; ++kb) {
            const float *xr = cur + kb * C::ROWS;
            const float w = HAS_W ? ys[BT + kb] : 1.f;
            // every slot runs (an unused slot repeats tile 0): no branches
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const float4 a0 = *reinterpret_cast<const float4 *>(xr + 4 * tI[s]);
                const float4 a1 = *reinterpret_cast<const float4 *>(xr + 4 * (NB8 + tI[s]));
                const float4 b0 = *reinterpret_cast<const float4 *>(xr + 4 * tJ[s]);
                const float4 b1 = *reinterpret_cast<const float4 *>(xr + 4 * (NB8 + tJ[s]));
                float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                if (HAS_W) {
#pragma unroll
                    for (int m = 0; m < 8; ++m) a[m] *= w;
                }
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    ffma2(acc[s][m][0], a[m], b0.x, b0.y);
                    ffma2(acc[s][m][1], a[m], b0.z, b0.w);
                    ffma2(acc[s][m][2], a[m], b1.x, b1.y);
                    ffma2(acc[s][m][3], a[m], b1.z, b1.w);
                }
            }
        }
        __syncwarp();   // this stage is refilled two batches later
    }

    // ---- hot rows: chunk partials, summed in chunk order by the last chunk ----
    if (it.nch > 1) {
        float *slot0 = p.partials + (size_t)p.slot_off[it.j] * C::PSTRIDE;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (!tok[s]) continue;
            float *dst = slot0 + (size_t)it.c * C::PSTRIDE + (lane + 32 * s) * 72;
#pragma unroll
            for (int m = 0; m < 8; ++m)
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    *reinterpret_cast<float2 *>(dst + m * 8 + 2 * k) = acc[s][m][k];
        }
        __threadfence();
        __syncwarp();
        int prev = 0;
        if (lane == 0) prev = atomicAdd(p.counters + it.j, 1);
        prev = __shfl_sync(FULL, prev, 0);
        if (prev != it.nch - 1) return;
        __threadfence();
        if (lane == 0) p.counters[it.j] = 0;
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int m = 0; m < 8; ++m)
#pragma unroll
                for (int k = 0; k < 4; ++k) acc[s][m][k] = make_float2(0.f, 0.f);
        for (int c = 0; c < it.nch; ++c) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (!tok[s]) continue;
                const float *src = slot0 + (size_t)c * C::PSTRIDE + (lane + 32 * s) * 72;
#pragma unroll
                for (int m = 0; m < 8; ++m)
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const float2 v = __ldcg(reinterpret_cast<const float2 *>(src + m * 8 + 2 * k));
                        acc[s][m][k].x += v.x;
                        acc[s][m][k].y += v.y;
                    }
            }
        }
    }

    const int r = it.r;
    const float Sr = p.tax_S ? p.tax_S[r] : 0.f;
    if (it.n == 0 && Sr == 0.f) {
        if (p.lam_c > 0.f || p.lam_n > 0.f) {
            for (int i = lane; i < p.ld; i += 32) put_out(p, r, i, 0.f);
        } else if (lane == 0) {
            report_fail(p.fail, r);
        }
        return;
    }
    const float diag = p.lam_c + p.lam_n * (float)it.n + p.tau * Sr;

    // ---- solve ----------------------------------------------------------------
    float *PT = sm;                 // [8][LDK] published panel column, transposed
    float *Ls = PT + 8 * LDK;       // [64] L_JJ, row-major
    float *invd = Ls + 64;          // [LDK] 1 / L_ii
    float *bv = invd + LDK;         // [LDK] b -> y -> x
    int *flag = reinterpret_cast<int *>(bv + LDK);
    __syncwarp();                   // stages are dead (all cp.async drained)
    {   // row D of the augmented Gram is b^T: publish it to bv, then clear it
        const int ID = D >> 3, mD = D & 7;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (!tok[s] || tI[s] != ID) continue;
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                if (m != mD) continue;
#pragma unroll
                for (int n = 0; n < 8; ++n) {
                    const int col = 8 * tJ[s] + n;
                    if (col < D) bv[col] = tel(acc[s], m, n);
                    tel(acc[s], m, n) = 0.f;
                }
            }
        }
    }
    __syncwarp();
    if (dslot >= 0) {
        // diagonal tile: + (lam_c + lam_n n + tau S) on the diagonal, identity
        // on the padding rows; its b block (+ tau T)
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (s != dslot) continue;
            const int I = tI[s];
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int i = 8 * I + m;
                float &d = tel(acc[s], m, m);
                d = i < D ? d + diag_at(p, i, diag, (float)it.n) : 1.f;
                bv[i] = i < D ? tax_rhs(p, r, i, bv[i]) : 0.f;
            }
        }
    }
    if (lane == 0) *flag = 0;
    __syncwarp();

    for (int J = 0; J < NB8; ++J) {
        // (1) diagonal lane: factor L_JJ, publish it, forward-solve y_J
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (s != dslot || tI[s] != J) continue;
            float2 (&t)[8][4] = acc[s];
            bool ok = true;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const float d = tel(t, c, c);
                ok = ok && d > 0.f && d < INFINITY;
                const float inv = rsqrtf(d), l = d * inv;   // MUFU.RSQ: ~2 ulp
                tel(t, c, c) = l;
                invd[8 * J + c] = inv;
#pragma unroll
                for (int rr = c + 1; rr < 8; ++rr) tel(t, rr, c) *= inv;
#pragma unroll
                for (int c2 = c + 1; c2 < 8; ++c2)
#pragma unroll
                    for (int rr = c2; rr < 8; ++rr)
                        tel(t, rr, c2) = fmaf(-tel(t, rr, c), tel(t, c2, c), tel(t, rr, c2));
            }
#pragma unroll
            for (int m = 0; m < 8; ++m) {   // row m of L_JJ: two 16-byte stores
                float4 *d4 = reinterpret_cast<float4 *>(Ls + 8 * m);
                d4[0] = make_float4(tel(t, m, 0), 1 <= m ? tel(t, m, 1) : 0.f,
                                    2 <= m ? tel(t, m, 2) : 0.f, 3 <= m ? tel(t, m, 3) : 0.f);
                d4[1] = make_float4(4 <= m ? tel(t, m, 4) : 0.f, 5 <= m ? tel(t, m, 5) : 0.f,
                                    6 <= m ? tel(t, m, 6) : 0.f, 7 <= m ? tel(t, m, 7) : 0.f);
            }
            float yv[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                float v = bv[8 * J + c];
#pragma unroll
                for (int c2 = 0; c2 < c; ++c2) v = fmaf(-tel(t, c, c2), yv[c2], v);
                yv[c] = v * invd[8 * J + c];
                bv[8 * J + c] = yv[c];
            }
            if (!ok) *flag = 1;
        }
        __syncwarp();
        if (*flag) {
            if (lane == 0) report_fail(p.fail, r);
            return;
        }
        // (2) panel: owners publish A_IJ transposed (PT[c][i]); all lanes solve
        // rows i of the panel against L_JJ in place and update b_i; owners
        // reload the solved tile (kept for the back substitution)
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (!tok[s] || tJ[s] != J || tI[s] == J) continue;
            float2 (&t)[8][4] = acc[s];
            const int I = tI[s];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                float4 *dst = reinterpret_cast<float4 *>(PT + c * LDK + 8 * I);
                dst[0] = make_float4(tel(t, 0, c), tel(t, 1, c), tel(t, 2, c), tel(t, 3, c));
                dst[1] = make_float4(tel(t, 4, c), tel(t, 5, c), tel(t, 6, c), tel(t, 7, c));
            }
        }
        __syncwarp();
        {
            float yv[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) yv[c] = bv[8 * J + c];
            for (int i = 8 * (J + 1) + lane; i < LDK; i += 32) {
                float x[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) x[c] = PT[c * LDK + i];
                float bi = bv[i];
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float4 l0 = *reinterpret_cast<const float4 *>(Ls + 8 * c);
                    const float4 l1 = *reinterpret_cast<const float4 *>(Ls + 8 * c + 4);
                    const float lr[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
                    float v = x[c];
#pragma unroll
                    for (int c2 = 0; c2 < c; ++c2) v = fmaf(-x[c2], lr[c2], v);
                    x[c] = v * invd[8 * J + c];
                    PT[c * LDK + i] = x[c];
                    bi = fmaf(-x[c], yv[c], bi);
                }
                bv[i] = bi;
            }
        }
        __syncwarp();
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (!tok[s] || tJ[s] != J || tI[s] == J) continue;
            float2 (&t)[8][4] = acc[s];
            const int I = tI[s];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const float4 v0 = *reinterpret_cast<const float4 *>(PT + c * LDK + 8 * I);
                const float4 v1 = *reinterpret_cast<const float4 *>(PT + c * LDK + 8 * I + 4);
                tel(t, 0, c) = v0.x; tel(t, 1, c) = v0.y; tel(t, 2, c) = v0.z; tel(t, 3, c) = v0.w;
                tel(t, 4, c) = v1.x; tel(t, 5, c) = v1.y; tel(t, 6, c) = v1.z; tel(t, 7, c) = v1.w;
            }
        }
        // (3) trailing tiles (I, K), J < K <= I:  A_IK -= L_IJ L_KJ^T
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (!tok[s] || tJ[s] <= J) continue;
            const int I = tI[s], K = tJ[s];
#pragma unroll 2
            for (int c = 0; c < 8; ++c) {
                const float4 a0 = *reinterpret_cast<const float4 *>(PT + c * LDK + 8 * I);
                const float4 a1 = *reinterpret_cast<const float4 *>(PT + c * LDK + 8 * I + 4);
                const float4 b0 = *reinterpret_cast<const float4 *>(PT + c * LDK + 8 * K);
                const float4 b1 = *reinterpret_cast<const float4 *>(PT + c * LDK + 8 * K + 4);
                const float a[8] = {-a0.x, -a0.y, -a0.z, -a0.w, -a1.x, -a1.y, -a1.z, -a1.w};
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    ffma2(acc[s][m][0], a[m], b0.x, b0.y);
                    ffma2(acc[s][m][1], a[m], b0.z, b0.w);
                    ffma2(acc[s][m][2], a[m], b1.x, b1.y);
                    ffma2(acc[s][m][3], a[m], b1.z, b1.w);
                }
            }
        }
        // the next step's diagonal lane writes Ls / PT only after the barrier
        // that follows its factorisation, so one __syncwarp per phase suffices
    }

    // back substitution, block rows bottom-up: x_J = L_JJ^-T b_J, then every
    // tile (J, K < J) pushes L_JK^T x_J into b_K (one writer per K)
    for (int J = NB8 - 1; J >= 0; --J) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (s != dslot || tI[s] != J) continue;
            float2 (&t)[8][4] = acc[s];
            float xv[8];
#pragma unroll
            for (int c = 7; c >= 0; --c) {
                float v = bv[8 * J + c];
#pragma unroll
                for (int c2 = c + 1; c2 < 8; ++c2) v = fmaf(-tel(t, c2, c), xv[c2], v);
                xv[c] = v * invd[8 * J + c];
                bv[8 * J + c] = xv[c];
            }
        }
        __syncwarp();
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (!tok[s] || tI[s] != J || tJ[s] == J) continue;
            float2 (&t)[8][4] = acc[s];
            const int K = tJ[s];
            float xv[8];
#pragma unroll
            for (int m = 0; m < 8; ++m) xv[m] = bv[8 * J + m];
#pragma unroll
            for (int n = 0; n < 8; ++n) {
                float v = bv[8 * K + n];
#pragma unroll
                for (int m = 0; m < 8; ++m) v = fmaf(-tel(t, m, n), xv[m], v);
                bv[8 * K + n] = v;
            }
        }
        __syncwarp();
    }
    for (int i = lane; i < p.ld; i += 32) put_out(p, r, i, i < D ? bv[i] : 0.f);
}

// persistent: every warp pulls work items from an atomic counter (no CTA
// waits on its slowest warp); the item order is the plan's
template <int NB8, bool HAS_W>
__global__ void __launch_bounds__(128) k_als_tile_warp(AlsParams p) {
    using C = TileWarpCfg<NB8>;
    extern __shared__ float4 smem4[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float *sm = reinterpret_cast<float *>(smem4) + warp * C::WARP_FLOATS;
    int *ctr = p.counters + p.n_list + 1;
    for (;;) {
        int64_t item = 0;
        if (lane == 0) item = atomicAdd(ctr, 1);
        item = __shfl_sync(FULL, item, 0);
        if (item >= p.total_items) break;
        tile_warp_item<NB8, HAS_W>(p, item, sm, lane);
        __syncwarp();   // the next item's gathers reuse the solve scratch
    }
}

// ---------------------------------------------------------------------------
// pair path, D <= 20 (the hot kernel of configs 0-2)
//
// Row-parallel: a warp takes 16 tasks (rows, or CHUNK-long chunks of hot
// rows) of similar length -- the plan sorts tasks by length, longest first,
// and warps pull groups of 16 from an atomic counter (persistent grid, LPT
// order).  A lane PAIR owns one task and walks its ratings one per step, so
// no cross-lane reduction is ever needed.  The pair splits the lower
// triangle of [A | b] by a cyclic block symmetry: NBK (odd) 4-wide blocks,
// lane h holds register block p = memory block (p + h) mod NBK; the static
// FMA list covers block pairs {p, p + d} for even p and d = 0..(NBK-1)/2
// plus the rhs blocks y * x_p for even p, so lane 0 and lane 1 together
// cover every entry (NBK = 5: 138 FMA per lane per rating for the 230
// useful ones, one instruction stream, no divergence).
//
// Partner rows (+ rating, + weight) are gathered into a 4-stage shared
// memory ring with 16-byte cp.async, NS-1 steps ahead of the FMAs.  After a
// light task, the pair writes its packed Gram to shared memory and lane 0
// solves it (thread-level Cholesky, reference row-oriented order,
// _kernels.py:187-213); a hot-row chunk instead writes its packed partial
// Gram to the workspace and k_als_heavy sums the chunks in chunk order and
// solves.

template <int NBK>
struct PairGeom {
    static_assert(NBK % 2 == 1, "odd block count");
    static constexpr int LDK = 4 * NBK;
    static constexpr int HALF = (NBK + 1) / 2;
    static constexpr int NACC = HALF * 10 + ((NBK - 1) / 2) * HALF * 16 + HALF * 4;
    static constexpr int RHS0 = LDK * (LDK + 1) / 2;
    static constexpr int GRAM = RHS0 + LDK;        // packed lower + rhs
    static constexpr int PSTR = GRAM + 1;          // partial slot: + sum w y^2
    static constexpr int GSTRIDE = GRAM | 1;       // odd stride: conflict-free per-lane rows
    // Schur-bias variant: packed system + u (LDK) + d; partial + u + d
    static constexpr int UOFF = GRAM, DOFF = GRAM + LDK;
    static constexpr int GSTRIDE_S = (GRAM + LDK + 1) | 1;
    static constexpr int PSTR_S = GRAM + 1 + LDK + 1;
    static constexpr int PU = GRAM + 1, PD = GRAM + 1 + LDK;   // u, d in a partial slot
};

// smallest 16-byte unit count >= u that is 2 or 6 mod 8: the 4 pairs of a
// quarter-warp then start on disjoint bank groups (units 0,2,4,6 or 0,6,4,2)
// and the two lanes of a pair (adjacent blocks) fill the odd ones
__host__ __device__ constexpr int slot_units(int u) {
    return (u % 8 == 2 || u % 8 == 6) ? u : slot_units(u + 1);
}

template <int NBK, int R_, bool YSUB_ = false>
struct PairCfg : PairGeom<NBK> {
    using G = PairGeom<NBK>;
    static constexpr int LDK = G::LDK;
    static constexpr int R = R_;                   // ratings per pipeline stage per pair
    // pair slot of one stage: R partner rows | R ratings | R weights; with
    // YSUB the partner rows carry one more 16-byte block (the y subtrahend)
    static constexpr int RROW = LDK + (YSUB_ ? 4 : 0);
    static constexpr int YOFF = R * RROW;
    static constexpr int WOFF = YOFF + R;
    static constexpr int SLOT = 4 * slot_units((WOFF + R + 3) / 4);   // floats
    static constexpr int PAIRS = 16;
    static constexpr int STAGE_BYTES = PAIRS * SLOT * 4;
    static constexpr int NS = R == 2 ? 7 : 4;      // pipeline stages (lead = (NS-1)*R ratings)
    static constexpr int RING_BYTES = NS * STAGE_BYTES;
    static constexpr int SOLVE_BYTES = PAIRS * G::GSTRIDE_S * 4;
    // the gather ring and the solve buffer are never live at the same time
    static constexpr int RING_AREA =
        ((RING_BYTES > SOLVE_BYTES ? RING_BYTES : SOLVE_BYTES) + 127) / 128 * 128;
    static constexpr int NR = R == 2 ? 8 : 4;      // id ring entries (>= NS - 1 ahead)
    static constexpr int IDSTR = NR * R + 4;       // ints per pair (+4: pairs on distinct banks)
    static constexpr int WARP_BYTES = RING_AREA + PAIRS * IDSTR * 4;
    static constexpr int WARPS = 4;
    static constexpr int MIN_CTAS = 2;             // 8 warps / SM (register bound: 138 accumulators)
    static constexpr int PF = 64;                  // L2 prefetch distance (ratings)
    static_assert(NR >= NS - 1 && (R == 2 || R == 4), "pair ring geometry");
};

__device__ __forceinline__ constexpr int pidx(int i, int j) { return i * (i + 1) / 2 + j; }

// Packed Cholesky + both substitutions by ONE thread, unrolled to LDK with
// row i held in registers (one shared-memory load per FMA).  g: packed
// lower triangle (pidx) and rhs at RHS0 (overwritten with the solution).
template <int LDK>
__device__ __forceinline__ bool thread_solve(float *g, int D, float diag_add, int bias_dim = -1,
                                             float bias_add = 0.f) {
    constexpr int RHS0 = LDK * (LDK + 1) / 2;
    float inv[LDK];
    float y[LDK];   // forward substitution fused into the row loop (row i of L is in r[])
    bool ok = true;
#pragma unroll
    for (int i = 0; i < LDK; ++i) {
        if (i < D) {
            float r[LDK];
#pragma unroll
            for (int j = 0; j <= i; ++j) r[j] = g[pidx(i, j)];
#pragma unroll
            for (int j = 0; j < i; ++j) {
                float t = r[j];
#pragma unroll
                for (int k = 0; k < j; ++k) t = fmaf(-r[k], g[pidx(j, k)], t);
                r[j] = t * inv[j];
                g[pidx(i, j)] = r[j];
            }
            float d = r[i] + (i == bias_dim ? bias_add : diag_add);
#pragma unroll
            for (int k = 0; k < i; ++k) d = fmaf(-r[k], r[k], d);
            ok = ok && (d > 0.f) && isfinite(d);
            // MUFU.RSQ (~2 ulp) instead of IEEE sqrt + divide: the pivot chain
            // of the one-lane solve is ~20 % shorter; well inside the 1e-4 budget
            const float ri = rsqrtf(d);
            g[pidx(i, i)] = d * ri;
            inv[i] = ri;
            float t = g[RHS0 + i];
#pragma unroll
            for (int k = 0; k < i; ++k) t = fmaf(-r[k], y[k], t);
            y[i] = t * ri;
        }
    }
    if (!ok) return false;
#pragma unroll
    for (int i = LDK - 1; i >= 0; --i) {
        if (i < D) {
            float t = y[i];
#pragma unroll
            for (int k = i + 1; k < LDK; ++k)
                if (k < D) t = fmaf(-g[pidx(k, i)], y[k], t);
            y[i] = t * inv[i];
            g[RHS0 + i] = y[i];
        }
    }
    return true;
}


// regularise + solve one packed system (one thread) and write the row.
// Regularise + solve one packed system (one thread), write the row, and
// return the row's objective terms: with x = (A_d + lam I)^{-1} b,
//   sum_k w_k (y_k - x_k^T x)^2 = sum w y^2 - b^T x - lam |x|^2   (sse)
//   (lam_c + lam_n n) |x|^2                                        (reg)
// (yy = sum w y^2 accumulated with the Gram; exact for tau = 0).
template <int LDK, bool SCHUR = false>
__device__ void finish_row(const AlsParams &p, float *g, int r, int64_t n, float yy,
                           double &sse, double &reg, bool emitted = false) {
    constexpr int RHS0 = LDK * (LDK + 1) / 2;
    constexpr int UOFF = RHS0 + LDK, DOFF = UOFF + LDK;
    const int D = p.D;
    sse = reg = 0.0;
    if (SCHUR && !emitted) {   // (the pair kernel emits and corrects warp-wide)
        if (p.emit) {   // [A | c | u | d | n] for the artist step (before any correction)
            float *e = p.emit + (size_t)r * EMIT_STRIDE;
            for (int i = 0; i < RHS0 + LDK; ++i) e[i] = g[i];
            for (int i = 0; i < LDK; ++i) e[RHS0 + LDK + i] = g[UOFF + i];
            e[RHS0 + 2 * LDK] = g[DOFF];
            e[RHS0 + 2 * LDK + 1] = (float)n;
        }
        if (p.corr_idx && p.corr_idx[r] >= 0) {   // the row's artist terms, from its Gram
            const float *v = p.corr_tab + (size_t)p.corr_idx[r] * p.ld;
            const float ba = v[D];
            float ud = 0.f;
            for (int i = 0; i < D; ++i) {
                float t = fmaf(g[UOFF + i], ba, 0.f);
                for (int k = 0; k < D; ++k) t = fmaf(g[i >= k ? pidx(i, k) : pidx(k, i)], v[k], t);
                g[RHS0 + i] -= t;
                ud = fmaf(g[UOFF + i], v[i], ud);
            }
            g[DOFF] -= fmaf((float)n, ba, ud);
        }
    }
    const float S = p.tax_S ? p.tax_S[r] : 0.f;
    if (n == 0 && S == 0.f) {
        if (p.lam_c > 0.f || p.lam_n > 0.f) {
            for (int i = 0; i < p.ld; ++i) put_out(p, r, i, 0.f);
        } else {
            report_fail(p.fail, r);
        }
        return;
    }
    const float lam_row = p.lam_c + p.lam_n * (float)n;
    const float diag = lam_row + p.tau * S;
    if (p.tax_T)
        for (int i = 0; i < D; ++i) g[RHS0 + i] = tax_rhs(p, r, i, g[RHS0 + i]);
    float sb = 1.f, db = 0.f;
    if constexpr (SCHUR) {   // eliminate the bias: A -= u u^T / s, c -= u d / s
        sb = (float)n + (n > 0 ? fmaf(p.bias_lam_n, (float)n, p.bias_lam_c) : 1.f);
        db = g[DOFF];
        const float is = 1.f / sb;
        for (int i = 0; i < D; ++i) {
            const float ui = g[UOFF + i] * is;
            for (int j = 0; j <= i; ++j) g[pidx(i, j)] = fmaf(-ui, g[UOFF + j], g[pidx(i, j)]);
            g[RHS0 + i] = fmaf(-ui, db, g[RHS0 + i]);
        }
    }
    float b[LDK];
#pragma unroll
    for (int i = 0; i < LDK; ++i) b[i] = i < D ? g[RHS0 + i] : 0.f;
    if (!thread_solve<LDK>(g, D, diag, p.bias_dim, diag_at(p, p.bias_dim, diag, (float)n))) {
        report_fail(p.fail, r);
        return;
    }
    float bias = 0.f;
    if constexpr (SCHUR) {   // b = (d - u.f) / s
        float uf = 0.f;
        for (int i = 0; i < D; ++i) uf = fmaf(g[UOFF + i], g[RHS0 + i], uf);
        bias = (db - uf) / sb;
    }
    float bx = 0.f, xx = 0.f;
#pragma unroll
    for (int i = 0; i < LDK; ++i) {
        if (i < D) {
            const float x = g[RHS0 + i];
            bx = fmaf(b[i], x, bx);
            xx = fmaf(x, x, xx);
        }
    }
    sse = (double)yy - (double)bx - (double)diag * (double)xx;
    reg = (double)lam_row * (double)xx;
    for (int i = 0; i < p.ld; ++i)
        put_out(p, r, i, i < D ? g[RHS0 + i] : (SCHUR && i == D) ? bias : 0.f);
}

__global__ void k_obj_sum(const double *part, int64_t n, double *out) {
    __shared__ double sh[2][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double a = 0.0, b = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        a += part[2 * i];
        b += part[2 * i + 1];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_down_sync(FULL, a, o);
        b += __shfl_down_sync(FULL, b, o);
    }
    if (lane == 0) {
        sh[0][warp] = a;
        sh[1][warp] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            s0 += sh[0][w];
            s1 += sh[1][w];
        }
        out[0] = s0;
        out[1] = s1;
    }
}



// Per-lane accumulators of the pair path, FFMA2-shaped: for each of HALF
// diagonal blocks the lower 4x4 triangle (m=0: 1 scalar; m=1: a pair; m=2: a
// pair + a scalar; m=3: two pairs), for each of NOFF off-diagonal blocks
// 4 rows x 2 pairs, for each of HALF rhs blocks 2 pairs.
template <int NBK, bool SCHUR = false>
struct PairAcc {
    static constexpr int HALF = (NBK + 1) / 2;
    static constexpr int NOFF = ((NBK - 1) / 2) * HALF;
    float dsc[HALF][2];
    float2 dpr[HALF][4];
    float2 off[NOFF > 0 ? NOFF : 1][4][2];
    float2 rhs[HALF][2];
    float yy;   // sum w y^2 (fused objective)
    float2 ux[HALF][2];   // Schur: sum x of the lane's register blocks
    float dd;             // Schur: sum y
    __device__ __forceinline__ void zero() {
        yy = 0.f;
        if constexpr (SCHUR) {
            dd = 0.f;
#pragma unroll
            for (int i = 0; i < HALF; ++i) ux[i][0] = ux[i][1] = make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < HALF; ++i) {
            dsc[i][0] = dsc[i][1] = 0.f;
#pragma unroll
            for (int k = 0; k < 4; ++k) dpr[i][k] = make_float2(0.f, 0.f);
            rhs[i][0] = rhs[i][1] = make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < (NOFF > 0 ? NOFF : 1); ++i)
#pragma unroll
            for (int m = 0; m < 4; ++m) off[i][m][0] = off[i][m][1] = make_float2(0.f, 0.f);
    }
    // one rating: register blocks xr (unscaled) / xa (weight-scaled), target y
    __device__ __forceinline__ void add(const float4 (&xa)[NBK], const float4 (&xr)[NBK], float y,
                                        float wy) {
        yy = fmaf(wy, y, yy);
        if constexpr (SCHUR) {
            dd += wy;
#pragma unroll
            for (int i = 0; i < HALF; ++i) {
                ffma2(ux[i][0], 1.f, xa[2 * i].x, xa[2 * i].y);
                ffma2(ux[i][1], 1.f, xa[2 * i].z, xa[2 * i].w);
            }
        }
#pragma unroll
        for (int i = 0; i < HALF; ++i) {
            const int b = 2 * i;
            const float a[4] = {xa[b].x, xa[b].y, xa[b].z, xa[b].w};
            const float4 u = xr[b];
            dsc[i][0] = fmaf(a[0], u.x, dsc[i][0]);
            ffma2(dpr[i][0], a[1], u.x, u.y);
            ffma2(dpr[i][1], a[2], u.x, u.y);
            dsc[i][1] = fmaf(a[2], u.z, dsc[i][1]);
            ffma2(dpr[i][2], a[3], u.x, u.y);
            ffma2(dpr[i][3], a[3], u.z, u.w);
            ffma2(rhs[i][0], y, a[0], a[1]);
            ffma2(rhs[i][1], y, a[2], a[3]);
        }
        int o = 0;
#pragma unroll
        for (int d = 1; d <= (NBK - 1) / 2; ++d) {
#pragma unroll
            for (int i = 0; i < HALF; ++i, ++o) {
                const int b = 2 * i;
                const float a[4] = {xa[b].x, xa[b].y, xa[b].z, xa[b].w};
                const float4 u = xr[(b + d) % NBK];
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    ffma2(off[o][m][0], a[m], u.x, u.y);
                    ffma2(off[o][m][1], a[m], u.z, u.w);
                }
            }
        }
    }
    // write into the packed [A | b] (pidx layout) of lane h's memory blocks
    __device__ __forceinline__ void scatter(float *g, int h, int rhs0) const {
#pragma unroll
        for (int i = 0; i < HALF; ++i) {
            const int A = (2 * i + h) % NBK, r = 4 * A;
            g[pidx(r, r)] = dsc[i][0];
            g[pidx(r + 1, r)] = dpr[i][0].x;
            g[pidx(r + 1, r + 1)] = dpr[i][0].y;
            g[pidx(r + 2, r)] = dpr[i][1].x;
            g[pidx(r + 2, r + 1)] = dpr[i][1].y;
            g[pidx(r + 2, r + 2)] = dsc[i][1];
            g[pidx(r + 3, r)] = dpr[i][2].x;
            g[pidx(r + 3, r + 1)] = dpr[i][2].y;
            g[pidx(r + 3, r + 2)] = dpr[i][3].x;
            g[pidx(r + 3, r + 3)] = dpr[i][3].y;
            g[rhs0 + r] = rhs[i][0].x;
            g[rhs0 + r + 1] = rhs[i][0].y;
            g[rhs0 + r + 2] = rhs[i][1].x;
            g[rhs0 + r + 3] = rhs[i][1].y;
            if constexpr (SCHUR) {   // block 0 is held by both lanes: same sums
                constexpr int UO = PairGeom<NBK>::UOFF;
                g[UO + r] = ux[i][0].x;
                g[UO + r + 1] = ux[i][0].y;
                g[UO + r + 2] = ux[i][1].x;
                g[UO + r + 3] = ux[i][1].y;
            }
        }
        if constexpr (SCHUR)
            if (h == 0) g[PairGeom<NBK>::DOFF] = dd;
        int o = 0;
#pragma unroll
        for (int d = 1; d <= (NBK - 1) / 2; ++d) {
#pragma unroll
            for (int i = 0; i < HALF; ++i, ++o) {
                const int A = (2 * i + h) % NBK, B = (2 * i + d + h) % NBK;
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const float v[4] = {off[o][m][0].x, off[o][m][0].y, off[o][m][1].x,
                                        off[o][m][1].y};
#pragma unroll
                    for (int nn = 0; nn < 4; ++nn) {
                        const int r_ = 4 * A + m, c_ = 4 * B + nn;
                        g[r_ >= c_ ? pidx(r_, c_) : pidx(c_, r_)] = v[nn];
                    }
                }
            }
        }
    }
};

// Each lane pair gathers its own partner rows with cp.async (16 B blocks
// split between the two lanes, zero-fill past the task end) and the ratings
// with 4 B cp.async, R ratings per pipeline stage; every lane's copies are
// tracked by the stage's mbarrier (cp.async.mbarrier.arrive.noinc, 32
// arrivals), so a stage is waited on individually, NS-2 stages after its
// issue.  Partner ids travel the same way: issuing stage s also cp.asyncs
// the ids of stage s+NS-1 into a small per-pair ring in shared memory, and
// they are read (after stage s's barrier has been waited on) when stage
// s+NS-1 is issued -- no register ever waits on an in-flight load.
// L2 policy: the once-read idx/val/weight streams are loaded evict_first,
// so they do not push the fixed factor rows (50-80 MB at config 1) out of L2.
template <int NBK, int R, bool HAS_W, bool FULLBLK, bool SCHUR = false, bool YSUB = false>
__global__ void __launch_bounds__(PairCfg<NBK, R, YSUB>::WARPS * 32, PairCfg<NBK, R, YSUB>::MIN_CTAS)
k_als_pair(AlsParams p, PairPlan q) {
    using C = PairCfg<NBK, R, YSUB>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    __shared__ __align__(8) unsigned long long bars[C::WARPS][C::NS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pair = lane >> 1, h = lane & 1;
    unsigned char *wbase = smem_raw + warp * C::WARP_BYTES;
    const unsigned wbase_s = static_cast<unsigned>(__cvta_generic_to_shared(wbase));
    const unsigned bar0 = static_cast<unsigned>(__cvta_generic_to_shared(&bars[warp][0]));
    float *my_g = reinterpret_cast<float *>(wbase) +
                  pair * (SCHUR ? C::GSTRIDE_S : C::GSTRIDE);   // aliases the ring
    const unsigned my_slot_s = wbase_s + pair * C::SLOT * 4;
    const float *my_slot = reinterpret_cast<const float *>(wbase) + pair * C::SLOT;
    // ids ring: [PAIRS][IDSTR] int32 after the gather ring / solve area
    const int *ring_ids = reinterpret_cast<const int *>(wbase + C::RING_AREA) + pair * C::IDSTR;
    const unsigned ring_ids_s = wbase_s + C::RING_AREA + pair * C::IDSTR * 4;
    const int nb_real = FULLBLK ? NBK : (p.D + 3) / 4;
    const int ysub_blk = YSUB ? (p.D + 1) >> 2 : -1;   // the block holding the y subtrahend
    int boff[NBK];   // float offset of register block b inside a row
#pragma unroll
    for (int b = 0; b < NBK; ++b) boff[b] = 4 * ((b + h) % NBK);
    uint64_t pol_stream;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < C::NS; ++s) mbar_init(bar0 + 8 * s, 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int64_t n_groups = (q.n_tasks + C::PAIRS - 1) / C::PAIRS;
    unsigned gst = 0;   // stages issued by this warp so far (slot = gst % NS)

    for (;;) {
        int64_t grp = 0;
        if (lane == 0) grp = atomicAdd(q.group_counter, 1);
        grp = __shfl_sync(FULL, grp, 0);
        if (grp >= n_groups) break;
        const int64_t task = grp * C::PAIRS + pair;
        int row = 0, slot = -1, n = 0;
        int64_t k0 = 0;
        if (task < q.n_tasks) {
            row = q.task_row[task];
            k0 = q.task_k0[task];
            n = q.task_n[task];
            slot = q.task_slot[task];
        }
        int nmax = n;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) nmax = max(nmax, __shfl_xor_sync(FULL, nmax, o));
        const int nst = (nmax + R - 1) / R;   // stages of this group
        const int32_t *idxp = p.idx + k0;
        const float *valp = p.val + k0;
        const float *wtsp = HAS_W ? p.wts + k0 : nullptr;
        const int k0lo = (int)k0 & 31;
        // stream bases as opaque 64-bit values: one IMAD.WIDE per copy address
        // (the compiler otherwise rebuilds base + 4 (k0 + k) from k0 for every copy)
        unsigned long long valb = reinterpret_cast<unsigned long long>(valp);
        unsigned long long idxb = reinterpret_cast<unsigned long long>(idxp);
        unsigned long long wtsb = reinterpret_cast<unsigned long long>(wtsp);
        asm volatile("" : "+l"(valb), "+l"(idxb));
        if (HAS_W) asm volatile("" : "+l"(wtsb));
        if (n > 0)
            for (int o = 0; o < min(n, C::PF); o += 32)
                prefetch_l2(h ? (const void *)(valp + o) : (const void *)(idxp + o));
        __syncwarp();   // the previous group's solve is done with the (aliased) ring

        PairAcc<NBK, SCHUR> acc;
        acc.zero();

        const unsigned gbase = gst;
        // gathers of stage s (ratings R*s .. R*s+R-1, partner ids in ids[]);
        // also brings the ids of stage s+NS-1 into the ring
        // (addresses: one IMAD.WIDE per copy off 64-bit bases kept in registers;
        // padded ratings keep a valid id and copy 0 bytes -- the issue block is
        // ~1/3 of the warp's instructions and all dependent integer chains)
        const char *fixed_h = reinterpret_cast<const char *>(p.fixed + 4 * h);
        const unsigned ldb = (unsigned)p.ld * 4u;
        auto issue = [&](int s, const int (&ids)[R]) {
            const unsigned gs = gbase + (unsigned)s;
            const unsigned slot = gs % C::NS;
            unsigned ss = my_slot_s + slot * C::STAGE_BYTES;
            asm volatile("" : "+r"(ss));
            const int nv = n - R * s;   // ratings of this stage that exist
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const bool ok = r < nv;
                const char *src = fixed_h + (size_t)(unsigned)ids[r] * ldb;
                const unsigned rs = ss + r * C::RROW * 4 + 16 * h;
                // lanes h = 0, 1 copy adjacent 16-byte blocks in one instruction
                // (one 32-byte sector when the row is sector-aligned)
#pragma unroll
                for (int b2 = 0; b2 < (NBK + (YSUB ? 1 : 0) + 1) / 2; ++b2) {
                    const int b = 2 * b2 + h;
                    if (2 * b2 + 1 < NBK + (YSUB ? 1 : 0) || h == 0)
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n"
                                     ::"r"(rs + 32 * b2), "l"(src + 32 * b2),
                                     "r"((ok && (FULLBLK || b < nb_real || b == ysub_blk)) ? 16 : 0));
                }
            }
            // lane h brings the ratings (and weights) of rows h, h+2, ... and
            // the partner ids of the same rows of stage s + NS - 1
            const unsigned ids_dst = ring_ids_s + 4 * (R * ((gs + C::NS - 1) % C::NR));
#pragma unroll
            for (int r2 = 0; r2 < R / 2; ++r2) {
                const int r = 2 * r2 + h;
                const bool okv = r < nv;
                const unsigned k = okv ? (unsigned)(R * s + r) : 0u;
                asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2, %3;\n"
                             ::"r"(ss + 4 * (C::YOFF + r)), "l"(valb + 4ull * k),
                             "r"(okv ? 4 : 0), "l"(pol_stream));
                if (HAS_W)
                    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2, %3;\n"
                                 ::"r"(ss + 4 * (C::WOFF + r)), "l"(wtsb + 4ull * k),
                                 "r"(okv ? 4 : 0), "l"(pol_stream));
                const bool oku = r + R * (C::NS - 1) < nv;
                const unsigned ku = oku ? (unsigned)(R * (s + C::NS - 1) + r) : 0u;
                asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2, %3;\n"
                             ::"r"(ids_dst + 4 * r), "l"(idxb + 4ull * ku), "r"(oku ? 4 : 0),
                             "l"(pol_stream));
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar0 + 8 * slot)
                         : "memory");
            const int pf = R * s + C::PF;
            if (pf < n && ((k0lo + pf) & 31) < R)
                prefetch_l2(reinterpret_cast<const void *>((h ? valb : idxb) + 4ull * (unsigned)pf));
        };
        auto consume = [&](int t) {
            const unsigned gs = gbase + (unsigned)t;
            mbar_wait(bar0 + 8 * (gs % C::NS), (gs / C::NS) & 1);
            const float *sl = my_slot + (gs % C::NS) * (C::STAGE_BYTES / 4);
            float ys[R];
            if constexpr (R == 4) {
                const float4 v = *reinterpret_cast<const float4 *>(sl + C::YOFF);
                ys[0] = v.x; ys[1] = v.y; ys[2] = v.z; ys[3] = v.w;
            } else {
                const float2 v = *reinterpret_cast<const float2 *>(sl + C::YOFF);
                ys[0] = v.x; ys[1] = v.y;
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const float *rw = sl + r * C::RROW;
                float4 xr[NBK];
#pragma unroll
                for (int b = 0; b < NBK; ++b) xr[b] = *reinterpret_cast<const float4 *>(rw + boff[b]);
                float y = ys[r] - p.y_shift;
                if constexpr (YSUB) y -= rw[p.D + 1];   // [x | 1 | subtrahend] partner rows
                // padding past the task end: zero rows, and zero targets (the Schur
                // bias sums d = sum y, so a shifted pad value would leak into it)
                if constexpr (SCHUR) y = R * t + r < n ? y : 0.f;
                float4 xa[NBK];
#pragma unroll
                for (int b = 0; b < NBK; ++b) xa[b] = xr[b];
                float wy = y;
                if (HAS_W) {
                    const float w = sl[C::WOFF + r];
                    wy = w * y;
#pragma unroll
                    for (int b = 0; b < NBK; ++b) {
                        xa[b].x *= w; xa[b].y *= w; xa[b].z *= w; xa[b].w *= w;
                    }
                }
                acc.add(xa, xr, y, wy);
            }
            __syncwarp();   // all lanes done with this stage before it is refilled
        };

        // prologue: stages 0 .. NS-2 with ids loaded directly
        for (int s = 0; s < C::NS - 1 && s < nst; ++s) {
            int ids[R];
#pragma unroll
            for (int r = 0; r < R; ++r) ids[r] = R * s + r < n ? idxp[R * s + r] : 0;
            issue(s, ids);
        }
        for (int t = 0; t < nst; ++t) {
            consume(t);   // waits stage t: the ids of stage t+NS-1 have landed too
            const int s = t + C::NS - 1;
            if (s < nst) {
                const int *rid = ring_ids + R * ((gbase + s) % C::NR);
                int ids[R];
                if constexpr (R == 4) {
                    const int4 v = *reinterpret_cast<const int4 *>(rid);
                    ids[0] = v.x; ids[1] = v.y; ids[2] = v.z; ids[3] = v.w;
                } else {
                    const int2 v = *reinterpret_cast<const int2 *>(rid);
                    ids[0] = v.x; ids[1] = v.y;
                }
                // (an id past the task end was zero-filled: row 0, copied with size 0)
                issue(s, ids);
            }
        }
        gst = gbase + (unsigned)nst;

        // scatter the lane's accumulators into the pair's packed [A | b]
        acc.scatter(my_g, h, C::RHS0);
        __syncwarp();
        if constexpr (SCHUR) {
            const bool whole = task < q.n_tasks && slot < 0;
            if (p.emit) {
                // [A | c | u | d | n] of every whole row of the group for the artist
                // step (before any correction): the packed system, u and d are
                // contiguous in a pair's buffer, so the warp copies them row by
                // row with coalesced stores
                constexpr int NE = C::RHS0 + 2 * C::LDK + 1;
                static_assert(NE + 1 <= EMIT_STRIDE, "emit row");
#pragma unroll 1
                for (int pp = 0; pp < C::PAIRS; ++pp) {
                    const bool wp = __shfl_sync(FULL, whole, 2 * pp);
                    if (!wp) continue;
                    const int rp = __shfl_sync(FULL, row, 2 * pp);
                    const int np = __shfl_sync(FULL, n, 2 * pp);
                    const float *gp = reinterpret_cast<const float *>(wbase) + pp * C::GSTRIDE_S;
                    float *e = p.emit + (size_t)rp * EMIT_STRIDE;
                    for (int i = lane; i <= NE; i += 32) e[i] = i < NE ? gp[i] : (float)np;
                }
            }
            if (whole && p.corr_idx && p.corr_idx[row] >= 0) {
                // the row's artist terms from its own Gram, c -= A q_a + u b_a,
                // d -= u.q_a + n b_a; lane h takes the rows i = h mod 2
                const float *v = p.corr_tab + (size_t)p.corr_idx[row] * p.ld;
                const int D = p.D;
                const float ba = v[D];
                float t[(C::LDK + 1) / 2], ud = 0.f;
#pragma unroll
                for (int ii = 0; ii < (C::LDK + 1) / 2; ++ii) {
                    const int i = 2 * ii + h;
                    t[ii] = 0.f;
                    if (i < D) {
                        float a = my_g[C::UOFF + i] * ba;
                        for (int k = 0; k < D; ++k)
                            a = fmaf(my_g[i >= k ? pidx(i, k) : pidx(k, i)], v[k], a);
                        t[ii] = a;
                        ud = fmaf(my_g[C::UOFF + i], v[i], ud);
                    }
                }
                ud += __shfl_xor_sync(0x3u << (2 * pair), ud, 1);
                __syncwarp(0x3u << (2 * pair));
#pragma unroll
                for (int ii = 0; ii < (C::LDK + 1) / 2; ++ii)
                    if (2 * ii + h < D) my_g[C::RHS0 + 2 * ii + h] -= t[ii];
                if (h == 0) my_g[C::DOFF] -= fmaf((float)n, ba, ud);
            }
            __syncwarp();
        }
        double o_sse = 0.0, o_reg = 0.0;
        if (task < q.n_tasks) {
            if (slot >= 0) {
                float *dst = p.partials + (size_t)slot * (SCHUR ? C::PSTR_S : C::PSTR);
                for (int i = h; i < C::GRAM; i += 2) dst[i] = my_g[i];
                if (h == 0) dst[C::GRAM] = acc.yy;
                if constexpr (SCHUR) {
                    for (int i = h; i <= C::LDK; i += 2) dst[C::PU + i] = my_g[C::UOFF + i];
                }
            } else if (h == 0) {
                finish_row<C::LDK, SCHUR>(p, my_g, row, n, acc.yy, o_sse, o_reg, true);
            }
        }
        if (p.obj_partial) {   // fixed-order butterfly: deterministic per group
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                o_sse += __shfl_xor_sync(FULL, o_sse, o);
                o_reg += __shfl_xor_sync(FULL, o_reg, o);
            }
            if (lane == 0) {
                p.obj_partial[2 * grp] = o_sse;
                p.obj_partial[2 * grp + 1] = o_reg;
            }
        }
        __syncwarp();
    }
}

// Hot rows: a CTA takes 8 hot rows; all 8 warps sum each row's chunk
// partials (chunks split over the warps, combined in a fixed order), then
// warp w solves row w cooperatively (lane i owns row i of A, right-looking
// Cholesky with shuffles).
template <int NBK, bool SCHUR = false>
__global__ void __launch_bounds__(256) k_als_heavy(AlsParams p, PairPlan q) {
    using C = PairGeom<NBK>;
    constexpr int LDK = C::LDK;
    constexpr int HW = 8;                            // warps (and hot rows) per CTA
    constexpr int PS = SCHUR ? C::PSTR_S : C::PSTR;  // floats per partial slot
    constexpr int NE = (PS + 31) / 32;               // partial elements per lane
    __shared__ float part[HW][PS];
    __shared__ float Gs[HW][(SCHUR ? C::PSTR_S : C::GSTRIDE) + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // phase 1, row by row: warp w sums chunks s0+w, s0+w+HW, ... (incl.
    // sum w y^2 at GRAM), the HW warp sums are then added in warp order --
    // a fixed order, so the result is deterministic
    for (int k = 0; k < HW; ++k) {
        const int64_t hk = (int64_t)blockIdx.x * HW + k;
        if (hk >= q.n_heavy) break;
        const int jk = q.sorted_j[hk];
        const int c0 = q.hoff[jk], c1 = q.hoff[jk + 1];
        float a[NE];
#pragma unroll
        for (int e = 0; e < NE; ++e) a[e] = 0.f;
        for (int c = c0 + warp; c < c1; c += HW) {
            const float *src = p.partials + (size_t)c * PS;
            float v[NE];
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                const int i = lane + 32 * e;
                v[e] = i < PS ? __ldcg(src + i) : 0.f;
            }
#pragma unroll
            for (int e = 0; e < NE; ++e) a[e] += v[e];
        }
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            const int i = lane + 32 * e;
            if (i < PS) part[warp][i] = a[e];
        }
        __syncthreads();
        for (int i = threadIdx.x; i < PS; i += 32 * HW) {
            float t = 0.f;
#pragma unroll
            for (int w = 0; w < HW; ++w) t += part[w][i];
            Gs[k][i] = t;
        }
        __syncthreads();
    }
    // phase 2: warp w solves hot row HW * block + w
    const int64_t hr = (int64_t)blockIdx.x * HW + warp;
    if (hr >= q.n_heavy) return;
    const int j = q.sorted_j[hr];
    const int r = p.row_list ? p.row_list[j] : p.row_lo + j;
    float *G = Gs[warp];
    const int D = p.D;
    const int64_t n = p.ptr[r + 1] - p.ptr[r];
    if constexpr (SCHUR) {
        if (p.emit) {   // [A | c | u | d | n] for the artist step (before any correction)
            float *e = p.emit + (size_t)r * EMIT_STRIDE;
            for (int i = lane; i < C::RHS0 + LDK; i += 32) e[i] = G[i];
            if (lane < LDK) e[C::RHS0 + LDK + lane] = G[C::PU + lane];
            if (lane == 0) {
                e[C::RHS0 + 2 * LDK] = G[C::PD];
                e[C::RHS0 + 2 * LDK + 1] = (float)n;
            }
        }
        if (p.corr_idx && p.corr_idx[r] >= 0) {   // the row's artist terms, from its Gram
            const float *v = p.corr_tab + (size_t)p.corr_idx[r] * p.ld;
            const float ba = v[D];
            float t = 0.f, ud = 0.f;
            if (lane < D) {
                t = G[C::PU + lane] * ba;
                for (int k = 0; k < D; ++k)
                    t = fmaf(G[lane >= k ? pidx(lane, k) : pidx(k, lane)], v[k], t);
                ud = G[C::PU + lane] * v[lane];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ud += __shfl_xor_sync(FULL, ud, o);
            __syncwarp();
            if (lane < D) G[C::RHS0 + lane] -= t;
            if (lane == 0) G[C::PD] -= fmaf((float)n, ba, ud);
            __syncwarp();
        }
    }
    const float S = p.tax_S ? p.tax_S[r] : 0.f;
    const float lam_row = p.lam_c + p.lam_n * (float)n;
    const float diag = lam_row + p.tau * S;
    float a[LDK];
#pragma unroll
    for (int c = 0; c < LDK; ++c) a[c] = (lane < D && c <= lane) ? G[pidx(lane, c)] : 0.f;
    float b = lane < D ? G[C::RHS0 + lane] : 0.f;
    if (lane < D) b = tax_rhs(p, r, lane, b);
    float sb = 1.f, db = 0.f, ul = 0.f;
    if constexpr (SCHUR) {   // eliminate the bias: A -= u u^T / s, c -= u d / s
        sb = (float)n + (n > 0 ? fmaf(p.bias_lam_n, (float)n, p.bias_lam_c) : 1.f);
        db = G[C::PD];
        ul = lane < D ? G[C::PU + lane] : 0.f;
        const float us = ul / sb;
#pragma unroll
        for (int c = 0; c < LDK; ++c)
            if (lane < D && c <= lane) a[c] = fmaf(-us, G[C::PU + c], a[c]);
        b = fmaf(-us, db, b);
    }
    const float b0 = b, yy = G[C::GRAM];
#pragma unroll
    for (int c = 0; c < LDK; ++c)
        if (c == lane) a[c] += diag_at(p, lane, diag, (float)n);
    bool bad = false;
#pragma unroll
    for (int j2 = 0; j2 < LDK; ++j2) {
        if (j2 < D) {
            const float piv = __shfl_sync(FULL, a[j2], j2);
            bad |= !(piv > 0.f) || !isfinite(piv);
            const float inv = rsqrtf(piv), l = piv * inv;   // MUFU.RSQ, as thread_solve
            if (lane == j2) a[j2] = l;
            else if (lane > j2) a[j2] *= inv;
#pragma unroll
            for (int k2 = j2 + 1; k2 < LDK; ++k2) {
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
#pragma unroll
    for (int j2 = 0; j2 < LDK; ++j2) {
        if (j2 < D) {
            if (lane == j2) b = b / a[j2];
            const float yj = __shfl_sync(FULL, b, j2);
            if (lane > j2) b = fmaf(-a[j2], yj, b);
        }
    }
    __syncwarp();
    if (lane < D) {
#pragma unroll
        for (int c = 0; c < LDK; ++c)
            if (c <= lane) G[pidx(lane, c)] = a[c];
    }
    __syncwarp();
    for (int j2 = D - 1; j2 >= 0; --j2) {
        if (lane == j2) b = b / G[pidx(j2, j2)];
        const float xj = __shfl_sync(FULL, b, j2);
        if (lane < j2) b = fmaf(-G[pidx(j2, lane)], xj, b);
    }
    float bias = 0.f;
    if constexpr (SCHUR) {   // b = (d - u.f) / s
        float uf = lane < D ? ul * b : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) uf += __shfl_xor_sync(FULL, uf, o);
        bias = (db - uf) / sb;
    }
    if (lane < p.ld) put_out(p, r, lane, lane < D ? b : (SCHUR && lane == D) ? bias : 0.f);
    if (p.obj_partial) {
        float bx = lane < D ? b0 * b : 0.f, xx = lane < D ? b * b : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            bx += __shfl_xor_sync(FULL, bx, o);
            xx += __shfl_xor_sync(FULL, xx, o);
        }
        if (lane == 0) {
            p.obj_partial[2 * (p.obj_groups + hr)] = (double)yy - (double)bx - (double)diag * xx;
            p.obj_partial[2 * (p.obj_groups + hr) + 1] = (double)lam_row * xx;
        }
    }
}

// --- MFITR artist step from the item layers' emitted systems.  An artist's
// block [q_a | b_a] has x = [p_u | 1] over the ratings of its items, so its
// Gram is the sum of its items' Grams and its rhs the sum of the items'
// base rhs minus G_i [q_i | b_i] (mfitr.py:203-216 with q_i, b_i fixed):
// one pass over I emitted systems instead of one over every rating.  Warp per
// artist, items in CSR order (fixed order); the summed system lands in a
// Schur partial slot (PSTR_S) that k_als_heavy<_, true> then solves.
template <int NBK>
__global__ void k_mfitr_artist_reduce(const int64_t *art_ptr, const int32_t *art_items,
                                      int32_t n_art, const float *emit, const float *Qa, int ld,
                                      int D, float *slots) {
    using C = PairGeom<NBK>;
    constexpr int LDK = C::LDK, RHS0 = C::RHS0;
    constexpr int NA = (RHS0 + 31) / 32;   // packed A entries per lane
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < n_art; a += warps) {
        float accA[NA], accC = 0.f, accU = 0.f, accD = 0.f;
#pragma unroll
        for (int t = 0; t < NA; ++t) accA[t] = 0.f;
        for (int64_t k = art_ptr[a]; k < art_ptr[a + 1]; ++k) {
            const int i = art_items[k];
            const float *e = emit + (size_t)i * EMIT_STRIDE;
            const float *v = Qa + (size_t)i * ld;          // [q_i | b_i]
#pragma unroll
            for (int t = 0; t < NA; ++t) {
                const int idx = lane + 32 * t;
                if (idx < RHS0) accA[t] += __ldg(e + idx);
            }
            const float bi = __ldg(v + D);
            float corr = 0.f, ud = 0.f;
            if (lane < D) {
                corr = __ldg(e + RHS0 + LDK + lane) * bi;
                for (int c = 0; c < D; ++c)
                    corr = fmaf(__ldg(e + (lane >= c ? pidx(lane, c) : pidx(c, lane))), __ldg(v + c),
                                corr);
                accC += __ldg(e + RHS0 + lane) - corr;
                accU += __ldg(e + RHS0 + LDK + lane);
                ud = __ldg(e + RHS0 + LDK + lane) * __ldg(v + lane);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ud += __shfl_xor_sync(FULL, ud, o);
            if (lane == 0)
                accD += __ldg(e + RHS0 + 2 * LDK) - fmaf(__ldg(e + RHS0 + 2 * LDK + 1), bi, ud);
        }
        float *dst = slots + (size_t)a * C::PSTR_S;
#pragma unroll
        for (int t = 0; t < NA; ++t) {
            const int idx = lane + 32 * t;
            if (idx < RHS0) dst[idx] = accA[t];
        }
        if (lane < LDK) {
            dst[RHS0 + lane] = lane < D ? accC : 0.f;
            dst[C::PU + lane] = lane < D ? accU : 0.f;
        }
        if (lane == 0) {
            dst[C::GRAM] = 0.f;
            dst[C::PD] = accD;
        }
    }
}

__global__ void k_iota(int32_t *a, int32_t *b, int32_t n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) {
        if (i < n) a[i] = i;
        b[i] = i;
    }
}

// --- plan kernels for the pair path
__global__ void k_pair_keys(const int64_t *ptr, const int32_t *row_list, int32_t n_list,
                            int32_t row_lo, int32_t chunk, int32_t *keys, int32_t *jcols,
                            float *dvals, int32_t *hch) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= n_list; j += gridDim.x * blockDim.x) {
        if (j == n_list) {
            hch[j] = 0;
            continue;
        }
        const int r = row_list ? row_list[j] : row_lo + j;
        const int64_t n = ptr[r + 1] - ptr[r];
        keys[j] = n > chunk ? 0 : (int32_t)(chunk + 1 - n);
        jcols[j] = j;
        dvals[j] = 0.f;
        hch[j] = n > chunk ? (int32_t)((n + chunk - 1) / chunk) : 0;
    }
}

__global__ void k_pair_fill(const int64_t *ptr, const int32_t *row_list, int32_t n_list,
                            int32_t row_lo, int32_t chunk, const int32_t *sorted_j,
                            const int64_t *kptr, const int32_t *hoff, int32_t *task_row,
                            int64_t *task_k0, int32_t *task_n, int32_t *task_slot) {
    const int64_t nh = kptr[1];               // rows with key 0 = hot rows
    const int64_t H = hoff[n_list];           // hot chunks (tasks 0..H-1)
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_list; q += gridDim.x * blockDim.x) {
        const int j = sorted_j[q];
        const int r = row_list ? row_list[j] : row_lo + j;
        const int64_t a = ptr[r], n = ptr[r + 1] - a;
        if (q < nh) {
            const int s0 = hoff[j];
            const int nch = hoff[j + 1] - s0;
            for (int c = 0; c < nch; ++c) {
                const int t = s0 + c;
                task_row[t] = r;
                task_k0[t] = a + (int64_t)c * chunk;
                task_n[t] = (int32_t)min((int64_t)chunk, n - (int64_t)c * chunk);
                task_slot[t] = t;
            }
        } else {
            const int64_t t = H + (q - nh);
            task_row[t] = r;
            task_k0[t] = a;
            task_n[t] = (int32_t)n;
            task_slot[t] = -1;
        }
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

template <int NB8, bool W>
int launch_cta(const AlsParams &p, cudaStream_t s) {
    using C = WideCfg<NB8>;
    const size_t smem = sizeof(float) * C::SMEM_FLOATS;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_als_cta<NB8, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attr = true;
    }
    if (p.total_items > 0) k_als_cta<NB8, W><<<(unsigned)p.total_items, CTA_THREADS, smem, s>>>(p);
    return check_launch("mcf_als_half_step(wide)");
}

template <int NB8, bool W>
int launch_tile_warp(const AlsParams &p, cudaStream_t s) {
    using C = TileWarpCfg<NB8>;
    const size_t smem = sizeof(float) * C::WARP_FLOATS * C::WARPS;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_als_tile_warp<NB8, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attr = true;
    }
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_als_tile_warp<NB8, W>, C::WARPS * 32,
                                                  smem);
    const int64_t grid = std::min<int64_t>(ceil_div(p.total_items, C::WARPS),
                                           (int64_t)sms * std::max(per_sm, 1));
    if (grid > 0) k_als_tile_warp<NB8, W><<<(unsigned)grid, C::WARPS * 32, smem, s>>>(p);
    return check_launch("mcf_als_half_step(tile-warp)");
}

int nb8_for(int D) {
    const int nb = (D + 7) / 8;
    return nb <= 4 ? 4 : nb <= 6 ? 6 : nb <= 7 ? 7 : nb <= 8 ? 8 : nb <= 10 ? 10 : nb <= 13 ? 13 : 16;
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
    switch (nb8_for(p.D + 1)) {   // + 1: the augmented rating column
        case 4: return launch_tile_warp<4, W>(p, s);
        case 6: return launch_tile_warp<6, W>(p, s);
        case 7: return launch_tile_warp<7, W>(p, s);
        case 8: return launch_tile_warp<8, W>(p, s);
        case 10: return launch_tile_warp<10, W>(p, s);
        case 13: return launch_tile_warp<13, W>(p, s);
        default: return launch_cta<16, W>(p, s);
    }
}

size_t pstride_of(int D) {
    const int nb = (D + 3) / 4;
    if (nb <= 7) return (size_t)(nb * (nb + 1) / 2) * 20;   // warp path, 4x4 tiles
    const int n8 = nb8_for(D + 1);
    return (size_t)(n8 * (n8 + 1) / 2) * 72;                // wide path, 8x8 tiles
}

struct PlanLayout {
    // warp / CTA paths (D > 20)
    int32_t *items, *slots, *item_row;
    void *scan_tmp;
    size_t scan_bytes;
    // pair path (D <= 20)
    int32_t *keys, *jcols, *sorted_j, *hch;
    float *dvals, *dvals_out;
    int64_t *kptr;
    void *csr_ws;
    size_t csr_bytes;
    int32_t *task_row, *task_n, *task_slot;
    int64_t *task_k0;
};

PlanLayout carve_plan(void *buf, size_t cap, int32_t n_list, int64_t nnz, int32_t chunk,
                      size_t *need) {
    Carve c(buf, cap);
    PlanLayout L;
    const size_t nl = (size_t)n_list;
    L.items = c.take<int32_t>(nl + 1);
    L.slots = c.take<int32_t>(nl + 1);
    L.hch = c.take<int32_t>(nl + 1);
    L.scan_bytes = scan_exclusive<int32_t>(nullptr, nullptr, (int64_t)n_list + 1, nullptr, 0,
                                           nullptr, nullptr);
    L.scan_tmp = c.take<char>(L.scan_bytes + 256);
    L.keys = c.take<int32_t>(nl);
    L.jcols = c.take<int32_t>(nl);
    L.sorted_j = c.take<int32_t>(nl);
    L.dvals = c.take<float>(nl);
    L.dvals_out = c.take<float>(nl);
    L.kptr = c.take<int64_t>((size_t)chunk + 3);
    L.csr_bytes = mcf_csr_workspace_bytes(n_list, chunk + 2);
    L.csr_ws = c.take<char>(L.csr_bytes);
    const int64_t max_items = (int64_t)n_list + ceil_div(nnz, chunk) + 1;
    L.task_row = c.take<int32_t>((size_t)max_items);
    L.task_n = c.take<int32_t>((size_t)max_items);
    L.task_slot = c.take<int32_t>((size_t)max_items);
    L.task_k0 = c.take<int64_t>((size_t)max_items);
    L.item_row = c.take<int32_t>((size_t)max_items);
    *need = c.used;
    return L;
}

bool use_pair(int D) { return D <= 20; }

template <int NBK, int R, bool W, bool FB, bool SC = false, bool YS = false>
int launch_pair(const AlsParams &p, const PairPlan &q, cudaStream_t s) {
    using C = PairCfg<NBK, R, YS>;
    const size_t smem = (size_t)C::WARP_BYTES * C::WARPS;

    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_als_pair<NBK, R, W, FB, SC, YS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attr = true;
    }
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_als_pair<NBK, R, W, FB, SC, YS>, C::WARPS * 32,
                                                  smem);
    const int64_t groups = ceil_div(q.n_tasks, C::PAIRS);
    const int64_t want = ceil_div(groups, C::WARPS);
    const int64_t grid = std::min<int64_t>(want, (int64_t)sms * std::max(per_sm, 1));
    if (grid > 0) k_als_pair<NBK, R, W, FB, SC, YS><<<(unsigned)grid, C::WARPS * 32, smem, s>>>(p, q);
    if (q.n_heavy > 0)
        k_als_heavy<NBK, SC><<<(unsigned)ceil_div(q.n_heavy, 8), 256, 0, s>>>(p, q);
    if (p.obj_partial) k_obj_sum<<<1, 256, 0, s>>>(p.obj_partial, p.obj_groups + q.n_heavy, q.obj_out);
    return check_launch("mcf_als_half_step(pair)");
}

template <bool W>
int dispatch_pair(const AlsParams &p, const PairPlan &q, cudaStream_t s) {
    const int nb = (p.D + 3) / 4;
    if (p.schur && p.ysub) {   // ... with [x | 1 | subtrahend] partner rows
        if (nb <= 1) return launch_pair<1, 4, false, false, true, true>(p, q, s);
        if (nb <= 3) return launch_pair<3, 4, false, false, true, true>(p, q, s);
        return launch_pair<5, 4, false, false, true, true>(p, q, s);
    }
    if (p.schur) {   // [f | b] rows with the bias eliminated in the epilogue (no weights)
        if (nb <= 1) return launch_pair<1, 4, false, false, true>(p, q, s);
        if (nb <= 3) return launch_pair<3, 4, false, false, true>(p, q, s);
        return launch_pair<5, 4, false, false, true>(p, q, s);
    }
    if (nb <= 1) return launch_pair<1, 4, W, false>(p, q, s);
    if (nb <= 3) return launch_pair<3, 4, W, false>(p, q, s);
    if (nb == 5) return launch_pair<5, 4, W, true>(p, q, s);
    return launch_pair<5, 4, W, false>(p, q, s);
}

size_t pair_gram(int D) {   // partial slot floats: packed [A | b] + sum w y^2
    const int nb = (D + 3) / 4;
    const int nbk = nb <= 1 ? 1 : nb <= 3 ? 3 : 5;
    const int ldk = 4 * nbk;
    return (size_t)(ldk * (ldk + 1) / 2 + ldk + 1);
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
    // pair path: tasks sorted by length (hot-row chunks first), LPT order
    k_pair_keys<<<grid, 256, 0, s>>>(ptr, row_list, n_list, row_lo, chunk, L.keys, L.jcols,
                                     L.dvals, L.hch);
    scan_exclusive<int32_t>(L.hch, L.hch, (int64_t)n_list + 1, L.scan_tmp, L.scan_bytes, s, &err);
    int rc;
    if (n_list > 0) {
        if ((rc = mcf_csr_build(L.keys, L.jcols, L.dvals, n_list, chunk + 2, L.kptr, L.sorted_j,
                                L.dvals_out, nullptr, L.csr_ws, L.csr_bytes, stream)))
            return rc;
        k_pair_fill<<<grid, 256, 0, s>>>(ptr, row_list, n_list, row_lo, chunk, L.sorted_j, L.kptr,
                                         L.hch, L.task_row, L.task_k0, L.task_n, L.task_slot);
    } else {
        if ((rc = cuda_status(cudaMemsetAsync(L.kptr, 0, sizeof(int64_t) * 2, s), "memset")))
            return rc;
    }
    int32_t tot[2];
    int64_t nh = 0;
    int32_t H = 0;
    if ((rc = cuda_status(cudaMemcpyAsync(&tot[0], L.items + n_list, sizeof(int32_t),
                                          cudaMemcpyDeviceToHost, s), "memcpy")))
        return rc;
    if ((rc = cuda_status(cudaMemcpyAsync(&tot[1], L.slots + n_list, sizeof(int32_t),
                                          cudaMemcpyDeviceToHost, s), "memcpy")))
        return rc;
    if ((rc = cuda_status(cudaMemcpyAsync(&nh, L.kptr + 1, sizeof(int64_t),
                                          cudaMemcpyDeviceToHost, s), "memcpy")))
        return rc;
    if ((rc = cuda_status(cudaMemcpyAsync(&H, L.hch + n_list, sizeof(int32_t),
                                          cudaMemcpyDeviceToHost, s), "memcpy")))
        return rc;
    if ((rc = cuda_status(cudaStreamSynchronize(s), "sync"))) return rc;
    if (n_list == 0) nh = 0;
    totals[0] = tot[0];               // warp/CTA path work items
    totals[1] = tot[1];               // warp/CTA path partial slots
    totals[2] = H + (n_list - nh);    // pair path tasks
    totals[3] = H;                    // pair path partial slots (hot-row chunks)
    totals[4] = nh;                   // hot rows
    totals[5] = nnz;                  // plan geometry
    return check_launch("mcf_als_plan");
}

extern "C" size_t mcf_als_workspace_bytes_fixed(int32_t n_list, int64_t slots, int32_t D,
                                                int64_t n_fixed, int64_t nnz) {
    if (D < 1 || n_list < 0 || slots < 0 || n_fixed < 0 || nnz < 0) return 0;
    size_t per = use_pair(D) ? pair_gram(D) : pstride_of(D);
    if (D >= 2 && D - 1 <= 20) {   // a bias-last system may run as D - 1 + Schur (+ u, d)
        const int nb = (D - 1 + 3) / 4;
        const int ldk = 4 * (nb <= 1 ? 1 : nb <= 3 ? 3 : 5);
        per = std::max(per, pair_gram(D - 1) + (size_t)ldk + 1);
    }
    const size_t obj = sizeof(double) * 2 * ((size_t)n_list + (size_t)slots + 64);
    size_t part = sizeof(float) * (size_t)slots * per;
    if ((D >= tc_min_d() || tc_hybrid_min_n(D, false) > 0) && D <= 128 && n_fixed > 0)
        part = std::max(part, tc_workspace_bytes(D, slots, n_fixed, nnz));
    return align_up(sizeof(int32_t) * ((size_t)n_list + 64), 256) + align_up(obj, 256) + part;
}

// without the fixed-table size the tensor-core path has no room for its
// split tables: the CUDA-core kernels run (same results to the tolerance)
extern "C" size_t mcf_als_workspace_bytes(int32_t n_list, int64_t slots, int32_t D) {
    return mcf_als_workspace_bytes_fixed(n_list, slots, D, 0, 0);
}

// MFITR item-layer extras for the next half_step_impl call (set by
// mcf_als_half_step_mfitr_items only)
static thread_local float *g_emit = nullptr;
static thread_local const float *g_corr_tab = nullptr;
static thread_local const int32_t *g_corr_idx = nullptr;
static thread_local int g_ysub = 0;

static int half_step_impl(const int64_t *ptr, const int32_t *idx, const float *val,
                          const float *wts, const float *fixed, int64_t n_fixed, float *out,
                          int32_t D, float lam_c, float lam_n, float y_shift, const float *tax_S,
                          const float *tax_T, float tau, const int32_t *row_list, int32_t n_list,
                          int32_t row_lo, int32_t chunk, const void *plan,
                          const int64_t *plan_info, int64_t *fail_row, double *obj_out, void *ws,
                          size_t ws_bytes, void *stream, int32_t bias_dim, float bias_lam_c,
                          float bias_lam_n, float *const *peer_out = nullptr,
                          int32_t n_peers = 0, float *mc_out = nullptr) {
    if (D < 1 || D > 128) {
        set_error("mcf_als_half_step: D must be in [1, 128]");
        return MCF_E_UNSUPPORTED;
    }
    if (!ptr || !fixed || !out || !plan || !plan_info || !fail_row || n_list < 0 ||
        chunk < BATCH || chunk % BATCH) {
        set_error("mcf_als_half_step: invalid arguments");
        return MCF_E_ARG;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int rc;
    if ((rc = cuda_status(cudaMemsetAsync(fail_row, 0xff, sizeof(int64_t), s), "memset")))
        return rc;
    const int64_t total_items = plan_info[0];
    if (n_list == 0) return MCF_OK;
    size_t need_plan = 0;
    PlanLayout L = carve_plan(const_cast<void *>(plan), SIZE_MAX, n_list, plan_info[5], chunk,
                              &need_plan);
    AlsParams p{};
    p.ptr = ptr; p.idx = idx; p.val = val; p.wts = wts; p.fixed = fixed; p.n_fixed = n_fixed;
    p.out = out;
    p.D = D; p.ld = mcf_factor_ld(D);
    p.lam_c = lam_c; p.lam_n = lam_n; p.y_shift = y_shift; p.tau = tau;
    p.tax_S = tax_S; p.tax_T = tax_T;
    p.row_list = row_list; p.n_list = n_list; p.row_lo = row_lo; p.chunk = chunk;
    p.item_off = L.items; p.slot_off = L.slots;
    // item_row sits after items/slots; its offset does not depend on nnz
    p.item_row = L.item_row;
    p.total_items = total_items;
    p.fail = reinterpret_cast<unsigned long long *>(fail_row);
    p.bias_dim = bias_dim;
    // a bias in the last coordinate of a D <= 21 system, unweighted: the pair
    // kernel solves the D - 1 factor coordinates and eliminates the bias
    // (Schur complement) instead of the 4x4-tile warp kernel on D + 1
    if (bias_dim >= 1 && bias_dim == D - 1 && D - 1 <= 20 && !wts && !obj_out &&
        !getenv("MCF_NO_SCHUR")) {
        p.D = D - 1;
        p.schur = 1;
        p.bias_dim = -1;
    }
    p.peer_out = peer_out;
    p.n_peers = peer_out ? n_peers : 0;
    p.emit = g_emit;
    p.corr_tab = g_corr_tab;
    p.corr_idx = g_corr_idx;
    p.ysub = g_ysub;
    if ((p.emit || p.corr_idx || p.ysub) && !p.schur) {
        set_error("mcf_als_half_step_mfitr_items: the row systems did not take the Schur pair path");
        return MCF_E_UNSUPPORTED;
    }
    p.mc_out = mc_out;
    if (n_peers < 0 || (n_peers > 0 && !peer_out)) {
        set_error("mcf_als_half_step: peer_out must hold n_peers >= 0 device pointers");
        return MCF_E_ARG;
    }
    p.bias_lam_c = bias_lam_c;
    p.bias_lam_n = bias_lam_n;
    if (bias_dim >= D || (bias_dim >= 0 && obj_out)) {
        set_error("mcf_als_half_step: bias_dim must be < D, and excludes the fused objective");
        return MCF_E_ARG;
    }
    // workspace: counters [n_list] + partial slots
    if (obj_out && !use_pair(D)) {
        set_error("mcf_als_half_step: obj_out (fused objective) is implemented for D <= 20");
        return MCF_E_UNSUPPORTED;
    }
    Carve c(ws, ws_bytes);
    p.counters = c.take<int32_t>((size_t)n_list + 64);
    double *objp = c.take<double>(2 * ((size_t)n_list + (size_t)std::max<int64_t>(plan_info[3], plan_info[1]) + 64));
    p.obj_partial = obj_out ? objp : nullptr;
    p.partials = c.take<float>(0);
    const size_t fixed_part = c.used;
    if (!ws || ws_bytes < fixed_part) {
        set_error("mcf_als_half_step: workspace too small");
        return MCF_E_WORKSPACE;
    }
    p.partials = reinterpret_cast<float *>(static_cast<char *>(ws) + fixed_part);
    // the tensor-core path (64 <= D <= 128, no weights) when the workspace holds
    // its split tables (mcf_als_workspace_bytes_fixed), else the CUDA-core kernels
    const bool use_tc = tc_path(p.D, wts != nullptr) && !p.schur &&
                        ws_bytes >= fixed_part + tc_workspace_bytes(p.D, plan_info[3], n_fixed, plan_info[5]);
    {   // the partial-Gram slots of the hot-row chunks must fit too
        size_t per;
        if (p.schur) {
            const int nb = (p.D + 3) / 4;
            per = pair_gram(p.D) + (size_t)(4 * (nb <= 1 ? 1 : nb <= 3 ? 3 : 5)) + 1;
        } else {
            per = use_pair(p.D) ? pair_gram(p.D) : pstride_of(p.D);
        }
        const size_t slots = (size_t)std::max<int64_t>(plan_info[3], plan_info[1]);
        const size_t need = sizeof(float) * slots * per;
        if (!use_tc && ws_bytes < fixed_part + need) {
            set_error("mcf_als_half_step: workspace too small for the partial slots");
            return MCF_E_WORKSPACE;
        }
    }
    if ((rc = cuda_status(cudaMemsetAsync(p.counters, 0, sizeof(int32_t) * ((size_t)n_list + 64), s),
                          "memset")))
        return rc;
    if (use_pair(p.D)) {
        PairPlan q;
        q.task_row = L.task_row;
        q.task_k0 = L.task_k0;
        q.task_n = L.task_n;
        q.task_slot = L.task_slot;
        q.n_tasks = plan_info[2];
        q.sorted_j = L.sorted_j;
        q.hoff = L.hch;
        q.n_heavy = plan_info[4];
        q.group_counter = p.counters + n_list;
        q.obj_out = obj_out;
        p.obj_groups = ceil_div(q.n_tasks, 16);
        if (q.n_tasks == 0) {
            if (obj_out) return cuda_status(cudaMemsetAsync(obj_out, 0, 2 * sizeof(double), s), "memset");
            return MCF_OK;
        }
        return wts ? dispatch_pair<true>(p, q, s) : dispatch_pair<false>(p, q, s);
    }
    if (use_tc) {   // tensor-core wide path
        PairPlan q{};
        q.task_row = L.task_row;
        q.task_k0 = L.task_k0;
        q.task_n = L.task_n;
        q.task_slot = L.task_slot;
        q.n_tasks = plan_info[2];
        q.sorted_j = L.sorted_j;
        q.hoff = L.hch;
        q.n_heavy = plan_info[4];
        q.group_counter = p.counters + n_list;
        if (q.n_tasks == 0) return MCF_OK;
        const int cut = als_dual_cut(p, wts != nullptr);
        if ((rc = launch_als_tc(p, q, p.partials, ws_bytes - fixed_part, plan_info[3], plan_info[5], cut, s)))
            return rc;
        return launch_als_dual(p, q, plan_info[3], p.counters + n_list + 3, cut, s);
    }
    if (total_items == 0) return MCF_OK;
    // hybrid (49 <= D < 64, workspace with the split tables): long rows on the
    // tensor-core kernel, the rest on the CUDA-core kernels
    // (a row longer than the plan's chunk is a hot row: its chunks are tensor-core tasks)
    const int hyb = (!p.schur && p.D > 28) ? std::min(tc_hybrid_min_n(p.D, wts != nullptr), chunk + 1) : 0;
    if (hyb > 0 && ws_bytes >= fixed_part + tc_workspace_bytes(p.D, plan_info[3], n_fixed, plan_info[5]) &&
        plan_info[2] > 0) {
        PairPlan q{};
        q.task_row = L.task_row;
        q.task_k0 = L.task_k0;
        q.task_n = L.task_n;
        q.task_slot = L.task_slot;
        q.n_tasks = plan_info[2];
        q.sorted_j = L.sorted_j;
        q.hoff = L.hch;
        q.n_heavy = plan_info[4];
        q.group_counter = p.counters + n_list;
        if ((rc = launch_als_tc(p, q, p.partials, ws_bytes - fixed_part, plan_info[3], plan_info[5],
                                hyb - 1, s)))
            return rc;
        p.skip_min_n = hyb;
    }
    return wts ? dispatch<true>(p, s) : dispatch<false>(p, s);
}

extern "C" int mcf_als_half_step(const int64_t *ptr, const int32_t *idx, const float *val,
                                 const float *wts, const float *fixed, int64_t n_fixed, float *out,
                                 int32_t D,
                                 float lam_c, float lam_n, float y_shift, const float *tax_S,
                                 const float *tax_T, float tau, const int32_t *row_list,
                                 int32_t n_list, int32_t row_lo, int32_t chunk, const void *plan,
                                 const int64_t *plan_info, int64_t *fail_row, double *obj_out,
                                 void *ws, size_t ws_bytes, void *stream) {
    return half_step_impl(ptr, idx, val, wts, fixed, n_fixed, out, D, lam_c, lam_n, y_shift, tax_S,
                          tax_T, tau, row_list, n_list, row_lo, chunk, plan, plan_info, fail_row,
                          obj_out, ws, ws_bytes, stream, -1, 0.f, 0.f);
}

extern "C" int mcf_als_half_step_bias(const int64_t *ptr, const int32_t *idx, const float *val,
                                      const float *wts, const float *fixed, int64_t n_fixed,
                                      float *out, int32_t D, float lam_c, float lam_n,
                                      float y_shift, const float *tax_S, const float *tax_T,
                                      float tau, const int32_t *row_list, int32_t n_list,
                                      int32_t row_lo, int32_t chunk, const void *plan,
                                      const int64_t *plan_info, int64_t *fail_row, void *ws,
                                      size_t ws_bytes, int32_t bias_dim, float bias_lam_c,
                                      float bias_lam_n, void *stream) {
    if (bias_dim < 0) {
        set_error("mcf_als_half_step_bias: bias_dim must be >= 0");
        return MCF_E_ARG;
    }
    return half_step_impl(ptr, idx, val, wts, fixed, n_fixed, out, D, lam_c, lam_n, y_shift, tax_S,
                          tax_T, tau, row_list, n_list, row_lo, chunk, plan, plan_info, fail_row,
                          nullptr, ws, ws_bytes, stream, bias_dim, bias_lam_c, bias_lam_n);
}

extern "C" int mcf_als_half_step_peers(const int64_t *ptr, const int32_t *idx, const float *val,
                                       const float *wts, const float *fixed, int64_t n_fixed,
                                       float *out, int32_t D, float lam_c, float lam_n,
                                       float y_shift, const float *tax_S, const float *tax_T,
                                       float tau, const int32_t *row_list, int32_t n_list,
                                       int32_t row_lo, int32_t chunk, const void *plan,
                                       const int64_t *plan_info, int64_t *fail_row,
                                       double *obj_out, void *ws, size_t ws_bytes,
                                       float *const *peer_out, int32_t n_peers, void *stream) {
    return half_step_impl(ptr, idx, val, wts, fixed, n_fixed, out, D, lam_c, lam_n, y_shift, tax_S,
                          tax_T, tau, row_list, n_list, row_lo, chunk, plan, plan_info, fail_row,
                          obj_out, ws, ws_bytes, stream, -1, 0.f, 0.f, peer_out, n_peers);
}

extern "C" int mcf_als_half_step_multicast(const int64_t *ptr, const int32_t *idx,
                                           const float *val, const float *wts, const float *fixed,
                                           int64_t n_fixed, float *out, int32_t D, float lam_c,
                                           float lam_n, float y_shift, const float *tax_S,
                                           const float *tax_T, float tau, const int32_t *row_list,
                                           int32_t n_list, int32_t row_lo, int32_t chunk,
                                           const void *plan, const int64_t *plan_info,
                                           int64_t *fail_row, double *obj_out, void *ws,
                                           size_t ws_bytes, float *mc_out, void *stream) {
    if (!mc_out) {
        set_error("mcf_als_half_step_multicast: mc_out (multicast address) is required");
        return MCF_E_ARG;
    }
    return half_step_impl(ptr, idx, val, wts, fixed, n_fixed, out, D, lam_c, lam_n, y_shift, tax_S,
                          tax_T, tau, row_list, n_list, row_lo, chunk, plan, plan_info, fail_row,
                          obj_out, ws, ws_bytes, stream, -1, 0.f, 0.f, nullptr, 0, mc_out);
}

// MFITR block on the Schur pair path (bias last, D - 1 <= 20, no weights):
// optional emission of the row systems + artist correction (item layers),
// optional y subtrahend in column D of the partner rows (ysub).
extern "C" int mcf_als_half_step_mfitr(const int64_t *ptr, const int32_t *idx, const float *val,
                                       const float *fixed, int64_t n_fixed, float *out, int32_t D,
                                       float lam_n, float y_shift, const float *tax_S,
                                       const float *tax_T, float tau, const int32_t *row_list,
                                       int32_t n_list, int32_t chunk, const void *plan,
                                       const int64_t *plan_info, int64_t *fail_row, void *ws,
                                       size_t ws_bytes, float bias_lam_n, float *emit,
                                       const float *corr_tab, const int32_t *corr_idx,
                                       int32_t ysub, void *stream) {
    if (D < 2 || D - 1 > 20 || (corr_idx && !corr_tab) || getenv("MCF_NO_SCHUR")) {
        set_error("mcf_als_half_step_mfitr: needs the Schur pair path (D <= 21)");
        return MCF_E_UNSUPPORTED;
    }
    g_emit = emit;
    g_corr_tab = corr_tab;
    g_corr_idx = corr_idx;
    g_ysub = ysub ? 1 : 0;
    const int rc = half_step_impl(ptr, idx, val, nullptr, fixed, n_fixed, out, D, 0.f, lam_n,
                                  y_shift, tax_S, tax_T, tau, row_list, n_list, 0, chunk, plan,
                                  plan_info, fail_row, nullptr, ws, ws_bytes, stream, D - 1, 0.f,
                                  bias_lam_n);
    g_emit = nullptr;
    g_corr_tab = nullptr;
    g_corr_idx = nullptr;
    g_ysub = 0;
    return rc;
}

extern "C" size_t mcf_mfitr_artist_workspace_bytes(int32_t n_artists) {
    if (n_artists < 0) return 0;
    using C = PairGeom<5>;
    return align_up(sizeof(float) * (size_t)n_artists * C::PSTR_S, 256) +
           2 * align_up(sizeof(int32_t) * ((size_t)n_artists + 1), 256) + 256;
}

extern "C" int mcf_mfitr_artist_step(const int64_t *art_ptr, const int32_t *art_items,
                                     const int32_t *artist_row, int32_t n_artists,
                                     const int64_t *cnt_ptr, const float *emit, const float *Qa,
                                     float *Aa, int32_t D, float lam_n, float bias_lam_n,
                                     int64_t *fail_row, void *ws, size_t ws_bytes,
                                     void *stream) {
    if (!art_ptr || !art_items || !artist_row || n_artists < 0 || !cnt_ptr || !emit || !Qa ||
        !Aa || D < 2 || D - 1 > 20 || !fail_row) {
        set_error("mcf_mfitr_artist_step: invalid arguments (D + 1 <= 21 bias systems)");
        return MCF_E_ARG;
    }
    if (ws_bytes < mcf_mfitr_artist_workspace_bytes(n_artists)) {
        set_error("mcf_mfitr_artist_step: workspace too small");
        return MCF_E_WORKSPACE;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int rc;
    if ((rc = cuda_status(cudaMemsetAsync(fail_row, 0xff, sizeof(int64_t), s), "memset"))) return rc;
    if (n_artists == 0) return MCF_OK;
    const int Df = D - 1;   // factor coordinates; the bias is column Df
    const int nb = (Df + 3) / 4, nbk = nb <= 1 ? 1 : nb <= 3 ? 3 : 5;   // as dispatch_pair
    Carve c(ws, ws_bytes);
    float *slots = c.take<float>((size_t)n_artists * PairGeom<5>::PSTR_S);
    int32_t *sorted = c.take<int32_t>((size_t)n_artists + 1);
    int32_t *hoff = c.take<int32_t>((size_t)n_artists + 1);
    const int ld = mcf_factor_ld(D);
    const unsigned rgrid = 148 * 8, hgrid = (unsigned)ceil_div(n_artists, 8);
    if (nbk == 1)
        k_mfitr_artist_reduce<1><<<rgrid, 256, 0, s>>>(art_ptr, art_items, n_artists, emit, Qa, ld, Df, slots);
    else if (nbk == 3)
        k_mfitr_artist_reduce<3><<<rgrid, 256, 0, s>>>(art_ptr, art_items, n_artists, emit, Qa, ld, Df, slots);
    else
        k_mfitr_artist_reduce<5><<<rgrid, 256, 0, s>>>(art_ptr, art_items, n_artists, emit, Qa, ld, Df, slots);
    k_iota<<<(unsigned)ceil_div((int64_t)n_artists + 1, 256), 256, 0, s>>>(sorted, hoff, n_artists);
    AlsParams p{};
    p.ptr = cnt_ptr;
    p.out = Aa;
    p.D = Df;
    p.ld = ld;
    p.lam_n = lam_n;
    p.row_list = artist_row;
    p.n_list = n_artists;
    p.partials = slots;
    p.fail = reinterpret_cast<unsigned long long *>(fail_row);
    p.bias_dim = -1;
    p.bias_lam_n = bias_lam_n;
    p.schur = 1;
    PairPlan q{};
    q.sorted_j = sorted;
    q.hoff = hoff;
    q.n_heavy = n_artists;
    if (nbk == 1) k_als_heavy<1, true><<<hgrid, 256, 0, s>>>(p, q);
    else if (nbk == 3) k_als_heavy<3, true><<<hgrid, 256, 0, s>>>(p, q);
    else k_als_heavy<5, true><<<hgrid, 256, 0, s>>>(p, q);
    return check_launch("mcf_mfitr_artist_step");
}
