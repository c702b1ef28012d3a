// ALS half-step, wide path on the 5th-generation tensor cores (sm_100a):
// Gram, Cholesky and both substitutions of every row system in one
// persistent kernel, the system never leaving the SM.
//
// Replaces _kernels.als_solve_rows (reference _kernels.py:151-215) for
// 64 <= D <= 128 without per-observation weights; same plan, same
// arithmetic contract as als.cu:
//     A_r = sum_k x_k x_k^T + (lam_c + lam_n n_r + tau S_r) I,
//     b_r = sum_k (y_k - y_shift) x_k + tau T_r,   out_r = A_r^{-1} b_r.
//
// Team = 4 warps (128 threads = the 128 TMEM lanes, thread m = row m of the
// system); 4 teams per CTA, each owning DP + 16 TMEM columns (Gram | rhs),
// DP = round_up(D, 16).  Per half-step the fixed table is split once into
// fp16 tables s x = h + l (k_tc_split, 22 significant bits, s a power of two)
// and the layout's ratings into (y_h, y_l) pairs.
// * Gram (rows with n > 64 or n >= D): 16 ratings per stage in a 5-slot smem
//   ring; the team copies the partner rows' split chunks with 16-byte
//   cp.async straight into SWIZZLE_128B MN-major tiles (and the ratings with
//   4-byte cp.async into an N = 16 tile); the stage's full mbarrier counts
//   the copies' completions, thread 0 issues C += H H^T + H L^T + L H^T and
//   rhs += (H + L) [y_h y_l] (tcgen05.mma kind::f16, M 128, fp32 in TMEM)
//   and commits them to the slot's empty barrier.
// * Dual form (n <= 64 < D, no taxonomy / bias term): (X X^T + lam I)
//   alpha = y from K-major tiles of the n gathered rows, x = X^T alpha from
//   the fp32 rows (prefetched into the dead tiles during the Cholesky).
// * Cholesky: right-looking, 16-column blocks, unscaled.  Per block the
//   diagonal block is factorised by 16 lanes of one warp (the reference's
//   > 0 and finite pivot test) with the forward substitution fused, the
//   panel solved by every row thread (L packed in smem), split into fp16
//   h / l K-major tiles, and the trailing update issued as three negated
//   MMAs on the trailing columns.  Back substitution by one warp.
// * Rows with n < D: one step of iterative refinement from the ratings
//   (the rank-deficient Gram's fp32 rounding exceeds 1e-4 otherwise).
// * Hot rows (more than `chunk` ratings): every chunk dumps its C | rhs to a
//   workspace slot; the last chunk to finish sums the slots in chunk order
//   (deterministic) into TMEM (tcgen05.st) and solves.
//
// Scaling: s and s_y are powers of two chosen per call (k_tc_prep) so that
// every scaled diagonal entry stays below 2^30: all panel values then fit
// fp16 (|L_ij| <= sqrt(A_ii) < 2^15) and the result is exact rescaling.

#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "als_params.cuh"
#include "../../include/mcf.h"

#ifndef TC_DIAG_SMEM
#define TC_DIAG_SMEM 1   // diagonal-block broadcasts: 1 smem (measured faster), 0 shuffles
#endif

namespace mcf {
namespace {

__host__ __device__ constexpr int tc_pow2_cols(int c) {
    return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512;
}

template <int NBLK>
struct TcCfg {
    static constexpr int DP = 16 * NBLK;           // padded dimension (features = rows of L)
    static constexpr int NA = (DP + 63) / 64;      // 64-feature SWIZZLE_128B atoms per operand row
    static constexpr int TW = 64 * NA;             // split-table row width (fp16)
    static constexpr int HT = 2 * NA * 1024;       // H (or L) tile: 2 k-groups x NA atoms x 1 KB
    static constexpr int YT = 512;                 // rating tile: 16 ratings x 16 cols (y_h, y_l)
    static constexpr int STAGE = 2 * HT + 1024;    // H | L | Y (1 KB-aligned)
    static constexpr int NST = 5;                  // Gram stage ring (3 gathers + 2 MMA stages in flight)
    static constexpr int MMA_DEPTH = 2;
    static constexpr int KGP = (DP / 8) * 128;     // panel tile k-chunk stride (K-major, no swizzle)
    static constexpr int PT = 2 * KGP;             // panel tile: DP rows x 16 k
    static constexpr int COLS = DP + 16;           // TMEM columns per team: Gram | rhs
    static constexpr int LS_BYTES = DP * (DP + 1) / 2 * 4;
    // dual form (rows with n <= DUAL_MAX < D ratings): the gathered rows as
    // K-major tiles (8-row core matrices, 16-byte feature chunks DLBO apart),
    // after the (at most 64 x 64) packed L
    static constexpr int DUAL_MAX = 64;
    static constexpr int DLBO = DUAL_MAX / 8 * 128;
    static constexpr int DTILE = DP / 8 * DLBO;
    static constexpr int OFF_DX = 9216;
    // the stage ring (Gram) and the packed L (Cholesky .. back substitution)
    // are never live together: one region
    static constexpr int RING0 = NST * STAGE > LS_BYTES ? NST * STAGE : LS_BYTES;
    static constexpr int RING = RING0 > OFF_DX + 2 * DTILE ? RING0 : OFF_DX + 2 * DTILE;
    static constexpr int OFF_L = 0;
    static constexpr int OFF_PH = (RING + 1023) / 1024 * 1024;
    static constexpr int OFF_PL = OFF_PH + PT;
    static constexpr int OFF_LJJ = OFF_PL + PT;    // L_JJ, column-major 16 x 16
    static constexpr int OFF_RD = OFF_LJJ + 1024;  // 1 / L_ii [DP]
    static constexpr int OFF_Z = OFF_RD + DP * 4;  // z = L^{-1} b [DP]
    static constexpr int OFF_X = OFF_Z + DP * 4;   // x [128]
    static constexpr int TEAM_BYTES = (OFF_X + 512 + 1023) / 1024 * 1024;
    static constexpr int SLACK = 2048 + 1024;      // operand over-read past the last team + base alignment
    static constexpr int TEAMS = (4 * TEAM_BYTES + SLACK <= 227 * 1024 && 4 * COLS <= 512) ? 4 : 3;
    static constexpr int SMEM = TEAMS * TEAM_BYTES + SLACK;
    static constexpr int TMEM_COLS = tc_pow2_cols(TEAMS * COLS);
    static_assert(SMEM <= 227 * 1024 && TEAMS * COLS <= 512, "tensor-core path resources");
};

struct TcWs {
    unsigned *scal;      // [0] max|x| bits, [1] max|y| bits, [2] max n, [3] max tau*S bits
    int32_t *hot_count;  // [slots] chunks finished per hot row (at its first slot)
    float *partials;     // [slots][DP * (DP + 16)]
    int64_t n_slots;
    unsigned long long *prof;   // phase cycle counters (MCF_TC_PROF) or null
    int team_limit;             // teams per CTA that take work (MCF_TC_TEAMS, experiments)
    int dual_cut;               // light tasks with n <= dual_cut are left to k_als_dual (0: none)
    __half *th, *tl;            // split fixed table: s*x = h + l, [n_fixed][TW] fp16
    uint32_t *ysp;              // split ratings s_y (y - y_shift) = h + l, (h | l << 16) [nnz]
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void team_bar(int team) {
    asm volatile("bar.sync %0, 128;" ::"r"(team + 1) : "memory");
}
// shared-memory matrix descriptor, no swizzle (version 1, sm_100)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}
// kind::f16 instruction descriptor: fp16 A/B, fp32 accumulator, M = 128
__device__ __forceinline__ uint32_t idesc(int N, bool mn_major, bool neg_a) {
    return (1u << 4) | (neg_a ? 1u << 13 : 0u) | (mn_major ? (1u << 15) | (1u << 16) : 0u) |
           ((uint32_t)(N >> 3) << 17) | (8u << 24);
}
__device__ __forceinline__ void umma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t id,
                                     uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
// all threads of a warp wait for an mbarrier phase: lane 0 polls (no
// suspend), the warp follows
__device__ __forceinline__ void warp_mbar_wait(uint32_t bar, uint32_t parity) {
    if ((threadIdx.x & 31) == 0) mbar_wait(bar, parity);   // try_wait: suspends in hardware
    __syncwarp();
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void proxy_fence() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16};" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15]))
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// fp32 -> (h, l) fp16 pairs: v = h + l with h = rn(v), l = rn(v - h)
__device__ __forceinline__ void split2(float a, float b, uint32_t &h, uint32_t &l2) {
    const __half2 hh = __floats2half2_rn(a, b);
    const float2 hf = __half22float2(hh);
    const __half2 ll = __floats2half2_rn(a - hf.x, b - hf.y);
    h = *reinterpret_cast<const uint32_t *>(&hh);
    l2 = *reinterpret_cast<const uint32_t *>(&ll);
}

// power of two s with s^2 * den <= 2^30 (1 when den == 0)
__device__ __forceinline__ float tc_scale(float den) {
    if (!(den > 0.f) || !isfinite(den)) return 1.f;
    const float e = floorf(0.5f * log2f(1073741824.f / den));
    return exp2f(fminf(fmaxf(e, -100.f), 40.f));
}

// maxima for the scales, over the planned rows' ratings and the fixed table;
// zeroes the hot-row chunk counters
__global__ void k_tc_prep(AlsParams p, PairPlan q, TcWs w) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int nthr = gridDim.x * blockDim.x;
    for (int64_t i = tid; i < w.n_slots; i += nthr) w.hot_count[i] = 0;
    float mx = 0.f, my = 0.f, ms = 0.f;
    unsigned mn = 0;
    // (the padding columns D..ld-1 are zero by the table contract: they cannot raise the maximum)
    const int64_t nf4 = p.n_fixed * (int64_t)(p.ld >> 2);
    for (int64_t i = tid; i < nf4; i += nthr) {
        const float4 v = __ldg(reinterpret_cast<const float4 *>(p.fixed) + i);
        mx = fmaxf(fmaxf(mx, fmaxf(fabsf(v.x), fabsf(v.y))), fmaxf(fabsf(v.z), fabsf(v.w)));
    }
    const int warp = tid >> 5, lane = threadIdx.x & 31, nwarps = nthr >> 5;
    if (!p.row_list) {
        // a contiguous row range: its ratings are one contiguous span (coalesced pass)
        const int64_t a = p.ptr[p.row_lo], b = p.ptr[p.row_lo + p.n_list];
        // four independent loads in flight per thread
        float m1 = 0.f, m2 = 0.f, m3 = 0.f;
        int64_t i = a + tid;
        for (; i + 3 * (int64_t)nthr < b; i += 4 * (int64_t)nthr) {
            const float v0 = __ldg(p.val + i), v1 = __ldg(p.val + i + nthr);
            const float v2 = __ldg(p.val + i + 2 * (int64_t)nthr), v3 = __ldg(p.val + i + 3 * (int64_t)nthr);
            my = fmaxf(my, fabsf(v0 - p.y_shift));
            m1 = fmaxf(m1, fabsf(v1 - p.y_shift));
            m2 = fmaxf(m2, fabsf(v2 - p.y_shift));
            m3 = fmaxf(m3, fabsf(v3 - p.y_shift));
        }
        for (; i < b; i += nthr) my = fmaxf(my, fabsf(__ldg(p.val + i) - p.y_shift));
        my = fmaxf(fmaxf(my, m1), fmaxf(m2, m3));
        for (int64_t j = tid; j < p.n_list; j += nthr) {
            const int64_t r = p.row_lo + j;
            mn = max(mn, (unsigned)(p.ptr[r + 1] - p.ptr[r]));
            if (p.tax_S) ms = fmaxf(ms, p.tau * fabsf(p.tax_S[r]));
        }
    }
    // a row list: a warp per task, lanes over its ratings
    for (int64_t t = p.row_list ? warp : q.n_tasks; t < q.n_tasks; t += nwarps) {
        const int r = q.task_row[t];
        const int64_t k0 = q.task_k0[t];
        const int n = q.task_n[t];
        for (int k = lane; k < n; k += 32) my = fmaxf(my, fabsf(__ldg(p.val + k0 + k) - p.y_shift));
        if (lane == 0) {
            mn = max(mn, (unsigned)(p.ptr[r + 1] - p.ptr[r]));
            if (p.tax_S) ms = fmaxf(ms, p.tau * fabsf(p.tax_S[r]));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
        my = fmaxf(my, __shfl_xor_sync(FULL, my, o));
        ms = fmaxf(ms, __shfl_xor_sync(FULL, ms, o));
        mn = max(mn, __shfl_xor_sync(FULL, mn, o));
    }
    if (lane == 0) {
        atomicMax(&w.scal[0], __float_as_uint(mx));
        atomicMax(&w.scal[1], __float_as_uint(my));
        atomicMax(&w.scal[2], mn);
        atomicMax(&w.scal[3], __float_as_uint(ms));
    }
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void ffma2(float &x, float &y, float a, float bx, float by) {
    unsigned long long A, B, C;
    asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a));
    asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(bx), "f"(by));
    asm("mov.b64 %0, {%1, %2};" : "=l"(C) : "f"(x), "f"(y));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C) : "l"(A), "l"(B));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(C));
}
__device__ __forceinline__ void lds16(const float *p, float (&v)[16]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float4 t = reinterpret_cast<const float4 *>(p)[q];
        v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
    }
}

// the per-call scales (powers of two, see the header comment)
__device__ __forceinline__ void tc_scales(const AlsParams &p, const TcWs &w, float &s, float &sy) {
    const float xmax = __uint_as_float(w.scal[0]), ymax = __uint_as_float(w.scal[1]);
    const float nmax = (float)w.scal[2], smax = __uint_as_float(w.scal[3]);
    const float regmax = p.lam_c + p.lam_n * nmax + smax + 1.f +
                         (p.bias_dim >= 0 ? p.bias_lam_c + p.bias_lam_n * nmax : 0.f);
    s = tc_scale(nmax * xmax * xmax + regmax);
    sy = ymax > 0.f ? exp2f(floorf(log2f(16384.f / ymax))) : 1.f;
}

// fixed table -> fp16 split tables (s*x = h + l), zero beyond D: the TMA
// gathers of the Gram read these rows
__global__ void k_tc_split(AlsParams p, PairPlan q, TcWs w, int TW) {
    float s, sy;
    tc_scales(p, w, s, sy);
    // a thread per 4 features: one 16-byte load (ld and D's padding are multiples of 4
    // floats; the padding columns D..ld-1 are zero), two 8-byte stores; TW is 64 or 128
    const int sh = TW == 128 ? 5 : 4;   // log2(TW / 4)
    const int64_t n = p.n_fixed << sh;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e >> sh;
        const int f = 4 * (int)(e & ((1 << sh) - 1));
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (f < p.ld) v = __ldg(reinterpret_cast<const float4 *>(p.fixed + r * p.ld + f));
        uint2 h, l;
        split2(f < p.D ? v.x * s : 0.f, f + 1 < p.D ? v.y * s : 0.f, h.x, l.x);
        split2(f + 2 < p.D ? v.z * s : 0.f, f + 3 < p.D ? v.w * s : 0.f, h.y, l.y);
        reinterpret_cast<uint2 *>(w.th)[e] = h;
        reinterpret_cast<uint2 *>(w.tl)[e] = l;
    }
    // the planned ratings at their CSR positions: the Gram's rating tiles are
    // 4-byte copies of these.  A contiguous row range is one coalesced span ...
    if (!p.row_list) {
        const int64_t a = p.ptr[p.row_lo], b = p.ptr[p.row_lo + p.n_list];
        const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
        int64_t i = a + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        for (; i + 3 * nthr < b; i += 4 * nthr) {   // four independent loads in flight per thread
            float v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = __ldg(p.val + i + k * nthr);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint32_t h, l;
                split2((v[k] - p.y_shift) * sy, 0.f, h, l);
                w.ysp[i + k * nthr] = (h & 0xffffu) | (l << 16);
            }
        }
        for (; i < b; i += nthr) {
            uint32_t h, l;
            split2((__ldg(p.val + i) - p.y_shift) * sy, 0.f, h, l);
            w.ysp[i] = (h & 0xffffu) | (l << 16);
        }
        return;
    }
    // ... a row list takes a warp per task
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < q.n_tasks; t += nw) {
        const int64_t k0 = q.task_k0[t];
        const int nt = q.task_n[t];
        for (int i = lane; i < nt; i += 32) {
            uint32_t h, l;
            split2((__ldg(p.val + k0 + i) - p.y_shift) * sy, 0.f, h, l);
            w.ysp[k0 + i] = (h & 0xffffu) | (l << 16);
        }
    }
}

__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return sdesc(addr, lbo, sbo) | (2ull << 61);
}

// Triangular solve with the packed lower factor L (smem, row r at r(r+1)/2)
// by one warp, lane l holding rows l, l + 32, l + 64, l + 96 of the
// right-hand side zr.  8 unknowns per step: their right-hand sides are
// shuffled to every lane, each lane solves the 8 x 8 diagonal block
// redundantly (rdiag = 1 / L_ii), then updates its own rows.
//   UPPER: L^T x = z, x -> out[128];   else L z = r, z -> zr (in place).
template <int DP, bool UPPER>
__device__ __forceinline__ void warp_trsv(float (&zr)[4], const float *Ls, const float *rdiag,
                                          int lane, float *out, int dim = DP) {
    float xr[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
    const int qs = UPPER ? 3 - qq : qq;
    if (32 * qs >= DP) continue;
#pragma unroll
    for (int gq = 0; gq < 4; ++gq) {
        const int l0 = 8 * (UPPER ? 3 - gq : gq), i0 = 32 * qs + l0;
        if (i0 >= DP || i0 >= dim) continue;
        // all loads of the group first (their latency overlaps the shuffles)
        float lb[8][8], lu[4][8], rd[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int k2 = 0; k2 < 8; ++k2)
                if (k2 < k) lb[k][k2] = Ls[(i0 + k) * (i0 + k + 1) / 2 + i0 + k2];   // L[i0+k][i0+k2]
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float4 v = reinterpret_cast<const float4 *>(rdiag + i0)[h];
            rd[4 * h] = v.x; rd[4 * h + 1] = v.y; rd[4 * h + 2] = v.z; rd[4 * h + 3] = v.w;
        }
#pragma unroll
        for (int q5 = 0; q5 < 4; ++q5) {
            if (UPPER ? (q5 <= qs) : (q5 >= qs && 32 * q5 < DP)) {
                const int mq = lane + 32 * q5, ma = min(mq, DP - 1);
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    lu[q5][k] = UPPER ? Ls[(i0 + k) * (i0 + k + 1) / 2 + mq]   // L[i0+k][mq]
                                      : Ls[ma * (ma + 1) / 2 + i0 + k];        // L[mq][i0+k]
            }
        }
        float zs[8], x8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) zs[k] = __shfl_sync(FULL, zr[qs], l0 + k);
        // right-looking inside the block: each solved unknown updates the rest
        // at once (dependency chain of 8 multiply + fma pairs)
        if (UPPER) {
#pragma unroll
            for (int k = 7; k >= 0; --k) {
                x8[k] = zs[k] * rd[k];
#pragma unroll
                for (int k2 = 0; k2 < k; ++k2) zs[k2] = fmaf(-lb[k][k2], x8[k], zs[k2]);
            }
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                x8[k] = zs[k] * rd[k];
#pragma unroll
                for (int k2 = k + 1; k2 < 8; ++k2) zs[k2] = fmaf(-lb[k2][k], x8[k], zs[k2]);
            }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) xr[qs] = lane == l0 + k ? x8[k] : xr[qs];
#pragma unroll
        for (int q5 = 0; q5 < 4; ++q5) {
            if (UPPER ? (q5 <= qs) : (q5 >= qs && 32 * q5 < DP)) {
                const int mq = lane + 32 * q5;
                float za = 0.f, zb = 0.f;   // two short chains
#pragma unroll
                for (int k = 0; k < 8; k += 2) {
                    za = fmaf(lu[q5][k], x8[k], za);
                    zb = fmaf(lu[q5][k + 1], x8[k + 1], zb);
                }
                zr[q5] = (UPPER ? mq < i0 : mq > i0 + 7) ? zr[q5] - (za + zb) : zr[q5];
            }
        }
    }
    }
    if (UPPER) {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) out[lane + 32 * q4] = xr[q4];
    } else {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) zr[q4] = xr[q4];
    }
}

// the refinement's two solves, out of line (keeps the kernel's registers)
template <int DP>
__device__ __noinline__ float4 trsv_fwd(float4 z, const float *Ls, const float *rdiag, int lane,
                                        int dim) {
    float zr[4] = {z.x, z.y, z.z, z.w};
    warp_trsv<DP, false>(zr, Ls, rdiag, lane, nullptr, dim);
    return make_float4(zr[0], zr[1], zr[2], zr[3]);
}
template <int DP>
__device__ __noinline__ void trsv_back(float4 z, const float *Ls, const float *rdiag, int lane,
                                       float *out, int dim) {
    float zr[4] = {z.x, z.y, z.z, z.w};
    warp_trsv<DP, true>(zr, Ls, rdiag, lane, out, dim);
}

template <int NBLK>
__global__ void __launch_bounds__(512, 1)
    k_als_tc(AlsParams p, PairPlan q, TcWs w) {
    using C = TcCfg<NBLK>;
    constexpr int DP = C::DP, NST = C::NST;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    __shared__ uint32_t tmem_base_sh;
    __shared__ __align__(8) unsigned long long bars[4][2 * C::NST + 1];   // full | empty | chol
    struct TaskSh {   // a team's next task, fetched ahead by thread PF
        int64_t task, k0, nrow;
        int row, n, slot;
        float S;
    };
    __shared__ TaskSh tsh[4];
    __shared__ int team_flag[4];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int team = warp >> 2, wq = warp & 3, m = threadIdx.x & 127;
    // the team's single-warp work (MMA issue, triangular solves) runs on warp
    // `lead`: warp id mod 4 selects the SM sub-partition, so the four teams'
    // serial phases land on four different schedulers
    const int lead = team & 3;
    // SWIZZLE_128B atoms need 1 KB alignment
    unsigned char *smem = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    unsigned char *tb = smem + team * C::TEAM_BYTES;
    const uint32_t tbs = smem_u32(tb);
    float *Ljj = reinterpret_cast<float *>(tb + C::OFF_LJJ);
    float *rdiag = reinterpret_cast<float *>(tb + C::OFF_RD);
    float *zbuf = reinterpret_cast<float *>(tb + C::OFF_Z);
    float *xbuf = reinterpret_cast<float *>(tb + C::OFF_X);
    float *Ls = reinterpret_cast<float *>(tb + C::OFF_L);
    const uint32_t fbar0 = smem_u32(&bars[team][0]);        // stage landed (TMA + rating tile)
    const uint32_t ebar0 = fbar0 + 8 * NST;                 // stage consumed (MMA commit)
    const uint32_t cbar = fbar0 + 16 * NST;                 // Cholesky trailing update

    for (int e = threadIdx.x; e < (C::SMEM - 1024) / 16; e += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[e] = make_uint4(0u, 0u, 0u, 0u);
    if (m == 0) {
        // full: the 96 cp.async completion arrivals of the team's three copying warps
        for (int st = 0; st < NST; ++st) mbar_init(fbar0 + 8 * st, 96);
        for (int st = NST; st <= 2 * NST; ++st) mbar_init(fbar0 + 8 * st, 1);   // empty, chol: commits
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&tmem_base_sh)),
                     "r"(C::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    proxy_fence();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh + (uint32_t)(team * C::COLS);
    const uint32_t tl = tmem + ((uint32_t)(32 * wq) << 16);   // this warp's lane quadrant

    const int D = p.D;
    float s, sy;
    tc_scales(p, w, s, sy);
    const float s2 = s * s, ssy = s * sy, out_scale = s / sy;

    const uint32_t id_gram = idesc(DP, true, false);
    const uint32_t id_rhs = idesc(16, true, false);
    unsigned gst = 0;                          // Gram stages issued by this team
    unsigned cph = 0;                          // Cholesky barrier phase
    // phase cycle counters (tools/tc_phases*.py): compiled in only with
    // MCF_TC_PROFILE (tools/variant.sh); the product build carries none
#ifdef MCF_TC_PROFILE
    long long tcp_t = clock64();
    unsigned long long tcp_acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long tcp_fl[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#define TCP(k)                                                       \
    do {                                                             \
        if (w.prof && m == 0) {                                      \
            const long long t1_ = clock64();                         \
            tcp_acc[k] += (unsigned long long)(t1_ - tcp_t);         \
            tcp_t = t1_;                                             \
        }                                                            \
    } while (0)
#define TCP_FLUSH(cls)                                                        \
    do {                                                                      \
        if (w.prof && m == 0) {                                               \
            for (int k_ = 0; k_ < 10; ++k_) {                                 \
                atomicAdd(w.prof + 16 + 16 * (cls) + k_, tcp_acc[k_] - tcp_fl[k_]); \
                tcp_fl[k_] = tcp_acc[k_];                                     \
            }                                                                 \
            atomicAdd(w.prof + 16 + 16 * (cls) + 10, 1ull);                   \
        }                                                                     \
    } while (0)
#else
#define TCP(k) \
    do {       \
    } while (0)
#define TCP_FLUSH(cls) \
    do {               \
    } while (0)
#endif

    // The next task is fetched during the current one by thread PF (warp 3,
    // idle during warp 0's back substitution): the counter atomic right
    // after the Gram, the plan and row-pointer loads at the back
    // substitution; published to tsh for the next iteration.
    const int PF = 32 * ((lead + 2) & 3);   // a thread of a warp that idles during the lead warp's solves
    int64_t pf_task = 0;
    bool pf_started = false;
    auto pf_start = [&]() {
        if (m == PF && !pf_started) {
            pf_task = atomicAdd(q.group_counter, 1);
            pf_started = true;
        }
    };
    auto pf_finish = [&]() {
        if (m == PF) {
            if (!pf_started) pf_task = atomicAdd(q.group_counter, 1);
            pf_started = false;
            TaskSh t;
            t.task = pf_task;
            t.row = 0, t.k0 = 0, t.n = 0, t.slot = -1, t.nrow = 0, t.S = 0.f;
            if (pf_task < q.n_tasks) {
                t.row = q.task_row[pf_task];
                t.k0 = q.task_k0[pf_task];
                t.n = q.task_n[pf_task];
                t.slot = q.task_slot[pf_task];
                t.nrow = p.ptr[t.row + 1] - p.ptr[t.row];
                t.S = p.tax_S ? p.tax_S[t.row] : 0.f;
            }
            tsh[team] = t;
        }
    };
    if (team < w.team_limit) pf_finish();
    for (;;) {
        if (team >= w.team_limit) break;
        team_bar(team);
        const TaskSh cur = tsh[team];
        if (cur.task >= q.n_tasks) break;
        // the list is sorted by length: every later task is within the cut too
        if (w.dual_cut > 0 && cur.slot < 0 && cur.n <= w.dual_cut) break;
        const int row = cur.row;
        const int64_t k0 = cur.k0;
        const int n = cur.n;
        const int slot = cur.slot;
        const int64_t nrow = cur.nrow;
        const float Srow = cur.S;
        if (nrow == 0 && Srow == 0.f) {   // empty row: 0 with a regulariser, else singular
            if (p.lam_c > 0.f || p.lam_n > 0.f) {
                if (m < p.ld) put_out(p, row, m, 0.f);
            } else if (m == 0) {
                report_fail(p.fail, row);
            }
            team_bar(team);   // every thread has read tsh
            pf_finish();
            continue;
        }
        TCP(0);
        // dual form for short rows: (X X^T + lam I) alpha = y, x = X^T alpha
        // (push-through identity) -- an n x n system instead of D x D
        const bool dual = slot < 0 && nrow > 0 && nrow <= C::DUAL_MAX && nrow < D && !p.tax_T &&
                          p.bias_dim < 0 && Srow == 0.f;
        const int dim = dual ? (int)((nrow + 15) & ~15) : DP;
        const int nblk = dim / 16;
        if (!dual) {

        // ---------------- Gram: C = H H^T + H L^T + L H^T, rhs = (H + L) [y_h y_l].
        // An NST-stage smem ring of 16-rating stages (split rows of the fixed
        // table + the rating tile), filled by the whole team (below); thread 0
        // issues the MMAs of the oldest landed stage and commits them to the
        // stage's empty barrier.
        const int nst = (n + 15) >> 4;
        if (nst == 0) {   // taxonomy-only row: zero accumulator
            float zr[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) zr[i] = 0.f;
#pragma unroll
            for (int c = 0; c <= NBLK; ++c) tmem_st16(tl + 16 * c, zr);
            tmem_wait_st();
        }
        if (nst > 0) {
            // cp.async pipeline over the split tables, warp-specialised.  The
            // team's lead warp only issues MMAs: it waits for a stage's full
            // barrier, issues C += H H^T + H L^T + L H^T and rhs += (H + L) [y_h y_l]
            // and commits them to the slot's empty barrier -- never waiting for an
            // MMA to finish.  The three other warps copy: warp rank c takes
            // ratings c, c + 3, ... of a stage, a lane per 16-byte chunk (lanes 0-15
            // the h row, 16-31 the l row), straight into the SWIZZLE_128B MN-major
            // tiles (chunk index XOR row-in-atom), rank 0 also the rating tile;
            // they run up to NST stages ahead, gated only by the empty barrier
            // of the slot they refill.  Completion is tracked by the stage's full
            // barrier (cp.async.mbarrier.arrive, 96 arrivals).
            const int tab = lane >> 4, cc = lane & 15, at = cc >> 3, c8 = cc & 7;
            // chunks past DP only feed Gram rows / columns >= DP (never read): not copied
            const bool chunk_ok = cc < DP / 8;
            const __half *tsrc = (tab ? w.tl : w.th) + 8 * cc;
            const int crank = (wq - lead - 1) & 3;   // 0..2 for the copying warps
            unsigned sb = gst % NST, sq = gst / NST;   // slot / generation of the warp's next stage
            if (wq == lead) {
                for (int st = 0; st < nst; ++st) {
                    if (lane == 0) {
                        mbar_wait(fbar0 + 8 * sb, sq & 1);   // every copy + the rating tile landed
                        tc_fence_after();
                        const uint32_t ha = tbs + sb * C::STAGE;
                        const uint64_t dh = sdesc_sw128(ha, 1024, C::NA * 1024);
                        const uint64_t dl = sdesc_sw128(ha + C::HT, 1024, C::NA * 1024);
                        const uint64_t dy = sdesc(ha + 2 * C::HT, 256, 128);
                        const uint32_t acc = st > 0 ? 1u : 0u;
                        umma(tmem, dh, dh, id_gram, acc);
                        umma(tmem, dh, dl, id_gram, 1u);
                        umma(tmem, dl, dh, id_gram, 1u);
                        umma(tmem + DP, dh, dy, id_rhs, acc);
                        umma(tmem + DP, dl, dy, id_rhs, 1u);
                        umma_commit(ebar0 + 8 * sb);
                    }
                    if (++sb == NST) {
                        sb = 0;
                        ++sq;
                    }
                }
                __syncwarp();
            } else {
                uint32_t doff[6];   // smem offsets of this thread's chunks in a stage
#pragma unroll
                for (int j = 0; j < 6; ++j) {
                    const int kk = crank + 3 * j, r = kk & 7;
                    doff[j] = tab * C::HT + ((kk >> 3) & 1) * (C::NA * 1024) + at * 1024 + r * 128 + ((c8 ^ r) << 4);
                }
                // Partner ids: one coalesced load per warp per 2 stages (lane l holds
                // rating 32 blk + l), two blocks ahead of its use; a stage's ids are
                // shuffled out of the block
                auto load_idblk = [&](int blk) { return __ldg(p.idx + k0 + min(32 * blk + lane, n - 1)); };
                int ida = load_idblk(0), idb = load_idblk(1), idc = load_idblk(2);
                const uint32_t *ysrc = w.ysp + k0;
                const uint32_t ydst = 2 * C::HT + (lane >> 3) * 256 + (lane & 7) * 16;
                for (int t = 0; t < nst; ++t) {
                    if ((t & 1) == 0 && t > 0) {
                        ida = idb;
                        idb = idc;
                        idc = load_idblk((t >> 1) + 2);
                    }
                    if (sq > 0) warp_mbar_wait(ebar0 + 8 * sb, (sq - 1) & 1);   // the slot's MMAs are done
                    const uint32_t sts = tbs + sb * C::STAGE;
                    const int l0 = 16 * (t & 1) + crank, rem = n - 16 * t - crank;
#pragma unroll
                    for (int j = 0; j < 6; ++j) {
                        const int id = __shfl_sync(FULL, ida, (l0 + 3 * j) & 31);
                        if (chunk_ok && crank + 3 * j < 16)
                            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sts + doff[j]),
                                         "l"(tsrc + (size_t)id * C::TW), "r"(3 * j < rem ? 16 : 0));
                    }
                    if (crank == 0 && lane < 16)
                        // rating tile: (k = lane, n = 0 / 1) = (y_h, y_l); columns 2..15 are never read
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sts + ydst),
                                     "l"(ysrc + min(16 * t + lane, n - 1)), "r"(16 * t + lane < n ? 4 : 0));
                    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(fbar0 + 8 * sb)
                                 : "memory");
                    if (++sb == NST) {
                        sb = 0;
                        ++sq;
                    }
                }
            }
            // last MMAs done (the stage before (sb, sq))
            warp_mbar_wait(ebar0 + 8 * (sb == 0 ? NST - 1 : sb - 1), (sb == 0 ? sq - 1 : sq) & 1);
        }
        gst += (unsigned)nst;
        tc_fence_before();
        team_bar(team);
        tc_fence_after();
        } else {
            // ---------------- dual Gram K = X X^T (n x n): the n gathered split
            // rows as K-major tiles (ratings = M/N, features = K), 3 MMAs per 16
            // features
            int *ids = reinterpret_cast<int *>(xbuf);
            if (m < dim) ids[m] = m < n ? __ldg(p.idx + k0 + m) : -1;
            team_bar(team);
            const uint32_t dx = tbs + C::OFF_DX;
            const int items = 2 * (DP / 8) * dim;
            for (int e = m; e < items; e += 128) {
                const int r = e % dim, rest = e / dim, c = rest % (DP / 8), t2 = rest / (DP / 8);
                const int id = ids[r];
                const bool ok = id >= 0;
                const __half *src = (t2 ? w.tl : w.th) + (size_t)(ok ? id : 0) * C::TW + 8 * c;
                const uint32_t dst = dx + t2 * C::DTILE + c * C::DLBO + (r >> 3) * 128 + (r & 7) * 16;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                             "r"(ok ? 16 : 0));
            }
            asm volatile("cp.async.commit_group;\n" ::: "memory");
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            proxy_fence();
            tc_fence_before();
            team_bar(team);
            if (m == 32 * lead) {
                tc_fence_after();
                const uint32_t idd = idesc(dim, false, false);
                for (int kk = 0; kk < DP / 16; ++kk) {
                    const uint64_t dh = sdesc(dx + 2 * kk * C::DLBO, C::DLBO, 128);
                    const uint64_t dl = sdesc(dx + C::DTILE + 2 * kk * C::DLBO, C::DLBO, 128);
                    umma(tmem, dh, dh, idd, kk > 0 ? 1u : 0u);
                    umma(tmem, dh, dl, idd, 1u);
                    umma(tmem, dl, dh, idd, 1u);
                }
                umma_commit(cbar);
            }
            warp_mbar_wait(cbar, cph);
            cph ^= 1u;
            tc_fence_after();
            // the n fp32 rows (x = X^T alpha and the refinement) into the tile
            // region, free once the MMAs above completed; they land during the
            // Cholesky (n * ld floats <= DUAL_MAX * DP = the two tiles)
            const int ld4 = p.ld >> 2;
            for (int e = m; e < n * ld4; e += 128) {
                const int r = e / ld4, c = e - r * ld4;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dx + (uint32_t)e * 16),
                             "l"(p.fixed + (size_t)ids[r] * p.ld + 4 * c));
            }
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        }
        TCP(1);
        pf_start();

        // ---------------- hot-row chunk: dump C | rhs, the last chunk sums them
        if (slot >= 0) {
            float *dst = w.partials + (size_t)slot * DP * C::COLS + (size_t)m * C::COLS;
#pragma unroll 1
            for (int c = 0; c <= NBLK; ++c) {
                float v[16];
                tmem_ld16(tl + 16 * c, v);
                tmem_wait_ld();
                if (m < DP) {
#pragma unroll
                    for (int j = 0; j < 16; j += 4)
                        __stcg(reinterpret_cast<float4 *>(dst + 16 * c + j),
                               make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
                }
            }
            __threadfence();
            tc_fence_before();
            team_bar(team);
            const int chunk_i = (int)((k0 - p.ptr[row]) / p.chunk);
            const int s0 = slot - chunk_i;
            const int nch = (int)((nrow + p.chunk - 1) / p.chunk);
            if (m == 0) team_flag[team] = atomicAdd(w.hot_count + s0, 1) == nch - 1;
            team_bar(team);
            if (!team_flag[team]) {
                TCP(2);
                TCP_FLUSH(3);
                pf_finish();
                continue;
            }
            __threadfence();
#pragma unroll 1
            for (int c = 0; c <= NBLK; ++c) {
                float acc[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[j] = 0.f;
                if (m < DP) {
                    for (int sl = s0; sl < s0 + nch; ++sl) {
                        const float4 *src = reinterpret_cast<const float4 *>(
                            w.partials + (size_t)sl * DP * C::COLS + (size_t)m * C::COLS + 16 * c);
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float4 v = __ldcg(src + j);
                            acc[4 * j] += v.x;
                            acc[4 * j + 1] += v.y;
                            acc[4 * j + 2] += v.z;
                            acc[4 * j + 3] += v.w;
                        }
                    }
                }
                tmem_st16(tl + 16 * c, acc);
            }
            tmem_wait_st();
            tc_fence_before();
            team_bar(team);
            tc_fence_after();
        }
        TCP(2);

        // ---------------- blocked Cholesky, forward substitution fused.  Padding
        // coordinates (>= D) have zero Gram rows and a unit regulariser: pivot
        // s^2, L = s I there, z = x = 0 -- every block runs the same code.
        float rg = s2;   // this row's regulariser (scaled)
        float r;         // rhs b_m, reduced by the finished blocks (forward subst.)
        if (dual) {      // (s^2 (X X^T + lam I)) alpha' = s_y y
            rg = m < n ? (p.lam_c + p.lam_n * (float)nrow) * s2 : s2;
            r = m < n ? (__ldg(p.val + k0 + m) - p.y_shift) * sy : 0.f;
        } else {
            const float diag = p.lam_c + p.lam_n * (float)nrow + p.tau * Srow;
            if (m < D) rg = diag_at(p, m, diag, (float)nrow) * s2;
            uint32_t rb[2];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                         : "=r"(rb[0]), "=r"(rb[1])
                         : "r"(tl + DP));
            tmem_wait_ld();
            r = __uint_as_float(rb[0]) + __uint_as_float(rb[1]);
            if (m < D && p.tax_T && m != p.bias_dim)
                r = fmaf(ssy * p.tau, p.tax_T[(size_t)row * p.ld + m], r);
        }
        if (m < DP) zbuf[m] = rg;   // read by the diagonal warp of m's block
        bool failed = false;
#pragma unroll 1
        for (int J = 0; J < nblk; ++J) {
            const int c0 = 16 * J;
            const int dw = c0 >> 5, lo = c0 & 31, ime = lane - lo;
            const bool inblk = wq == dw && ime >= 0 && ime < 16;
            float a[16];
            if (32 * wq + 31 >= c0) tmem_ld16(tl + c0, a);
            if (wq == dw) {
#ifdef MCF_TC_PROFILE
                const long long dg0 = clock64();
#endif
                tmem_wait_ld();
#ifdef MCF_TC_PROFILE
                const long long dg1 = clock64();
#endif
                // the block rows' regularisers (written to zbuf by these lanes
                // before the loop; their z values replace them below)
                __syncwarp();
                float rgv[16];
                lds16(zbuf + c0, rgv);
                float fr = inblk ? r : 0.f;
                const int iml = inblk ? ime : -1;   // lanes outside the block keep their rows
                // right-looking on the unscaled Schur complement: a_mj -= a_mi a_ij / p_i
                // (the regulariser only enters the pivots; rows at or above the
                // pivot get t = 0, their entries right of it are never read)
                float ri[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    float lj[16], pv, rv;
#if TC_DIAG_SMEM
                    float *bb = Ljj + 32 * (i & 1);   // broadcast scratch (Ljj is written below)
                    if (inblk) {
                        bb[ime] = a[i];
                        bb[16 + ime] = fr;
                    }
                    __syncwarp();
                    lds16(bb, lj);
                    pv = lj[i] + rgv[i];
                    rv = bb[16 + i];
#else
                    pv = __shfl_sync(FULL, a[i], lo + i) + rgv[i];
#pragma unroll
                    for (int j = i + 1; j < 16; ++j) lj[j] = __shfl_sync(FULL, a[i], lo + j);
                    rv = __shfl_sync(FULL, fr, lo + i);
#endif
                    const float t = iml > i ? a[i] * rcp_approx(pv) : 0.f;
                    ri[i] = rsqrtf(pv);   // off the pivot chain
                    int j = i + 1;
                    if (j & 1 && j < 16) {
                        a[j] = fmaf(-t, lj[j], a[j]);
                        ++j;
                    }
#pragma unroll
                    for (; j < 16; j += 2) ffma2(a[j], a[j + 1], -t, lj[j], lj[j + 1]);
                    fr = fmaf(-t, rv, fr);
                }
                // the reference's pivot test (> 0 and finite) <=> 1 / sqrt(p) in (0, inf)
                if (lane == 0) {
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4)
                        reinterpret_cast<float4 *>(rdiag + c0)[q4] =
                            make_float4(ri[4 * q4], ri[4 * q4 + 1], ri[4 * q4 + 2], ri[4 * q4 + 3]);
                }
                __syncwarp();
                const float myri = inblk ? rdiag[c0 + ime] : 1.f;
                const bool bad = __any_sync(FULL, !(myri > 0.f && myri < INFINITY));
                if (inblk) {   // L row = a_mi / sqrt(p_i) (i < m; the diagonal is never read); z_m = r / sqrt(p_m)
#pragma unroll
                    for (int i = 0; i < 16; ++i) a[i] *= ri[i];
                    const int mr = c0 + ime;
#pragma unroll
                    for (int j = 0; j < 16; ++j) Ljj[j * 16 + ime] = a[j];   // column-major
                    float *Lr = Ls + mr * (mr + 1) / 2 + c0;
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (j <= ime) Lr[j] = a[j];
                    zbuf[mr] = fr * myri;
                }
                if (lane == 0) team_flag[team] = bad;
#ifdef MCF_TC_PROFILE
                if (w.prof && lane == 0) {   // diagonal warp: TMEM load wait, factorisation
                    const long long dg2 = clock64();
                    atomicAdd(w.prof + 11, (unsigned long long)(dg1 - dg0));
                    atomicAdd(w.prof + 12, (unsigned long long)(dg2 - dg1));
                    atomicAdd(w.prof + 13, 1ull);
                }
#endif
            }
            tmem_wait_ld();
            team_bar(team);
            TCP(3);
            if (team_flag[team]) {
                failed = true;
                break;
            }
            if (m >= c0 + 16 && m < dim) {   // panel rows: x L_JJ^T = a (right-looking), r -= x.z_J
                float rd[16], zj[16];
                lds16(rdiag + c0, rd);
                lds16(zbuf + c0, zj);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    float lc[16];   // column i of L_JJ
#pragma unroll
                    for (int q4 = (i + 1) / 4; q4 < 4; ++q4) {
                        const float4 v = reinterpret_cast<const float4 *>(Ljj + 16 * i)[q4];
                        lc[4 * q4] = v.x; lc[4 * q4 + 1] = v.y; lc[4 * q4 + 2] = v.z; lc[4 * q4 + 3] = v.w;
                    }
                    const float xi = a[i] * rd[i];
                    a[i] = xi;
                    int j = i + 1;
                    if (j & 1 && j < 16) {
                        a[j] = fmaf(-xi, lc[j], a[j]);
                        ++j;
                    }
#pragma unroll
                    for (; j < 16; j += 2) ffma2(a[j], a[j + 1], -xi, lc[j], lc[j + 1]);
                }
                float r0 = 0.f, r1 = 0.f;
#pragma unroll
                for (int i = 0; i < 16; i += 2) {
                    r0 = fmaf(a[i], zj[i], r0);
                    r1 = fmaf(a[i + 1], zj[i + 1], r1);
                }
                r -= r0 + r1;
                float *Lr = Ls + m * (m + 1) / 2 + c0;
#pragma unroll
                for (int j = 0; j < 16; ++j) Lr[j] = a[j];
            }
            TCP(4);
            if (c0 + 16 < dim) {   // panel tiles, K-major: rows >= c0 + 16 carry L, others 0
                const bool pr = m >= c0 + 16 && m < dim;
                uint4 h0, l0, h1, l1;
                split2(pr ? a[0] : 0.f, pr ? a[1] : 0.f, h0.x, l0.x);
                split2(pr ? a[2] : 0.f, pr ? a[3] : 0.f, h0.y, l0.y);
                split2(pr ? a[4] : 0.f, pr ? a[5] : 0.f, h0.z, l0.z);
                split2(pr ? a[6] : 0.f, pr ? a[7] : 0.f, h0.w, l0.w);
                split2(pr ? a[8] : 0.f, pr ? a[9] : 0.f, h1.x, l1.x);
                split2(pr ? a[10] : 0.f, pr ? a[11] : 0.f, h1.y, l1.y);
                split2(pr ? a[12] : 0.f, pr ? a[13] : 0.f, h1.z, l1.z);
                split2(pr ? a[14] : 0.f, pr ? a[15] : 0.f, h1.w, l1.w);
                if (m < DP) {
                    const int off = (m >> 3) * 128 + (m & 7) * 16;
                    *reinterpret_cast<uint4 *>(tb + C::OFF_PH + off) = h0;
                    *reinterpret_cast<uint4 *>(tb + C::OFF_PH + C::KGP + off) = h1;
                    *reinterpret_cast<uint4 *>(tb + C::OFF_PL + off) = l0;
                    *reinterpret_cast<uint4 *>(tb + C::OFF_PL + C::KGP + off) = l1;
                }
                TCP(9);
                tc_fence_before();
                proxy_fence();
                team_bar(team);
                // trailing update C -= P_h P_h^T + P_h P_l^T + P_l P_h^T
                if (m == 32 * lead) {
                    tc_fence_after();
                    const int N = dim - c0 - 16;
                    const uint32_t id = idesc(N, false, true);
                    const uint32_t boff = (uint32_t)((c0 + 16) >> 3) * 128;
                    const uint64_t da = sdesc(tbs + C::OFF_PH, C::KGP, 128);
                    const uint64_t dl = sdesc(tbs + C::OFF_PL, C::KGP, 128);
                    umma(tmem + c0 + 16, da, sdesc(tbs + C::OFF_PH + boff, C::KGP, 128), id, 1u);
                    umma(tmem + c0 + 16, da, sdesc(tbs + C::OFF_PL + boff, C::KGP, 128), id, 1u);
                    umma(tmem + c0 + 16, dl, sdesc(tbs + C::OFF_PH + boff, C::KGP, 128), id, 1u);
                    umma_commit(cbar);
                }
                warp_mbar_wait(cbar, cph);
                cph ^= 1u;
                tc_fence_after();
                TCP(7);
            }
        }
        tc_fence_before();   // TMEM is free for the next task from here on
        if (failed) {
            if (m == 0) report_fail(p.fail, row);
            team_bar(team);
            pf_finish();
            continue;
        }
        TCP(5);

        // ---------------- back substitution L^T x = z by warp 0 (L from smem), 8
        // unknowns per step; x -> xbuf (meanwhile thread PF fetches the next task)
        team_bar(team);
        pf_finish();
        if (wq == lead) {
            float zr[4];
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
                const int mq = lane + 32 * q4;
                zr[q4] = mq < dim ? zbuf[mq] : 0.f;
            }
            warp_trsv<DP, true>(zr, Ls, rdiag, lane, xbuf, dim);
        }
        team_bar(team);
        TCP(6);
        float xo = (m < DP ? xbuf[m] : 0.f) * out_scale;
        if (dual) {   // x = out_scale s X^T alpha' from the prefetched fp32 rows
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            team_bar(team);
            const float *rows = reinterpret_cast<const float *>(tb + C::OFF_DX);
            const int ld = p.ld;
            float acc = 0.f;
            if (m < D) {
                float acc1 = 0.f;
                int rr = 0;
                for (; rr + 1 < n; rr += 2) {
                    acc = fmaf(xbuf[rr], rows[rr * ld + m], acc);
                    acc1 = fmaf(xbuf[rr + 1], rows[(rr + 1) * ld + m], acc1);
                }
                if (rr < n) acc = fmaf(xbuf[rr], rows[rr * ld + m], acc);
                acc += acc1;
            }
            xo = acc * (s * out_scale);
            // one refinement step in the dual space: rho_r = y_r - x_r.x - lam alpha_r,
            // alpha += (X X^T + lam I)^{-1} rho, x += X^T (that correction)
            const float alpha_m = m < n ? xbuf[m] * (s2 / sy) : 0.f;
            team_bar(team);   // xbuf (alpha') is rewritten below
            if (m < DP) zbuf[m] = m < D ? xo : 0.f;   // x
            float *rho = reinterpret_cast<float *>(tb + C::OFF_PH);
            const float lam2 = p.lam_c + p.lam_n * (float)nrow;
            team_bar(team);
            if (m < dim) {
                float rh = 0.f;
                if (m < n) {
                    const float4 *xr4 = reinterpret_cast<const float4 *>(rows + m * ld);
                    float d0 = 0.f, d1 = 0.f;
                    for (int c4 = 0; c4 < ld / 4; ++c4) {
                        const float4 u = xr4[c4];
                        const float4 xv = *reinterpret_cast<const float4 *>(zbuf + 4 * c4);
                        d0 = fmaf(u.x, xv.x, d0); d1 = fmaf(u.y, xv.y, d1);
                        d0 = fmaf(u.z, xv.z, d0); d1 = fmaf(u.w, xv.w, d1);
                    }
                    rh = (__ldg(p.val + k0 + m) - p.y_shift) - (d0 + d1) - lam2 * alpha_m;
                }
                rho[m] = rh;
            }
            team_bar(team);
            if (wq == lead) {
                float zr[4];
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    const int mq = lane + 32 * q4;
                    zr[q4] = mq < dim ? rho[mq] : 0.f;
                }
                const float4 w4 = trsv_fwd<DP>(make_float4(zr[0], zr[1], zr[2], zr[3]), Ls, rdiag,
                                               lane, dim);
                trsv_back<DP>(w4, Ls, rdiag, lane, xbuf, dim);
            }
            team_bar(team);
            if (m < D) {   // x += X^T (s^2 w)
                float acc2 = 0.f, acc3 = 0.f;
                int rr = 0;
                for (; rr + 1 < n; rr += 2) {
                    acc2 = fmaf(xbuf[rr], rows[rr * ld + m], acc2);
                    acc3 = fmaf(xbuf[rr + 1], rows[(rr + 1) * ld + m], acc3);
                }
                if (rr < n) acc2 = fmaf(xbuf[rr], rows[rr * ld + m], acc2);
                xo = fmaf(s2, acc2 + acc3, xo);
            }
        }
        // ---------------- one step of iterative refinement for short rows
        // (n < D): fp32 rounding of the Gram times cond(A) (up to ~1e4 at
        // D = 100: the partner factors share a dominant mean direction, the
        // rank-deficient Gram leaves D - n eigenvalues at lam n) exceeds the
        // 1e-4 budget there; r = b - A x0 is formed from the ratings
        // (e_k = y_k - x_k.x0, r = sum x_k e_k + tau T - reg x0) and
        // x1 = x0 + A^{-1} r reuses the factorisation.
        if (!dual && slot < 0 && nrow < D && nrow > 0) {
            xbuf[m] = m < D ? xo : 0.f;   // x0, original units (own element)
            team_bar(team);
            // residuals e_k, a thread per rating (n < D <= 128)
            if (m < n) {
                const int id = __ldg(p.idx + k0 + m);
                const float4 *xr4 = reinterpret_cast<const float4 *>(p.fixed + (size_t)id * p.ld);
                float d0 = 0.f, d1 = 0.f;
                const int nc4 = p.ld >> 2;
                for (int c = 0; c < nc4; c += 8) {   // 8 independent 16-byte loads in flight
                    float4 u[8];
#pragma unroll
                    for (int q4 = 0; q4 < 8; ++q4) u[q4] = __ldg(xr4 + min(c + q4, nc4 - 1));
#pragma unroll
                    for (int q4 = 0; q4 < 8; ++q4) {
                        if (c + q4 < nc4) {
                            const float4 xv = *reinterpret_cast<const float4 *>(xbuf + 4 * (c + q4));
                            d0 = fmaf(u[q4].x, xv.x, d0); d1 = fmaf(u[q4].y, xv.y, d1);
                            d0 = fmaf(u[q4].z, xv.z, d0); d1 = fmaf(u[q4].w, xv.w, d1);
                        }
                    }
                }
                zbuf[m] = (__ldg(p.val + k0 + m) - p.y_shift) - (d0 + d1);
                reinterpret_cast<int *>(tb + C::OFF_PH)[m] = id;
            }
            team_bar(team);
            // r_f = sum_k x_k[f] e_k, a thread per feature
            float rf = 0.f;
            if (m < D) {
                const int *ids = reinterpret_cast<const int *>(tb + C::OFF_PH);
                float r1 = 0.f;
                for (int k = 0; k < n; k += 8) {   // 8 independent (coalesced) row loads in flight
                    float v[8];
#pragma unroll
                    for (int q8 = 0; q8 < 8; ++q8)
                        v[q8] = __ldg(p.fixed + (size_t)ids[min(k + q8, n - 1)] * p.ld + m);
#pragma unroll
                    for (int q8 = 0; q8 < 8; q8 += 2) {
                        if (k + q8 < n) rf = fmaf(v[q8], zbuf[k + q8], rf);
                        if (k + q8 + 1 < n) r1 = fmaf(v[q8 + 1], zbuf[k + q8 + 1], r1);
                    }
                }
                rf += r1;
            }
            team_bar(team);
            if (m < D) {
                rf = fmaf(-rg / s2, xo, rf);
                if (p.tax_T && m != p.bias_dim) rf = fmaf(p.tau, p.tax_T[(size_t)row * p.ld + m], rf);
            }
            if (m < DP) zbuf[m] = m < D ? rf : 0.f;
            team_bar(team);
            if (wq == lead) {
                float zr[4];
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    const int mq = lane + 32 * q4;
                    zr[q4] = mq < DP ? zbuf[mq] : 0.f;
                }
                const float4 w4 = trsv_fwd<DP>(make_float4(zr[0], zr[1], zr[2], zr[3]), Ls, rdiag,
                                               lane, DP);
                trsv_back<DP>(w4, Ls, rdiag, lane, xbuf, DP);
            }
            team_bar(team);
            if (m < D) xo = fmaf(s2, xbuf[m], xo);
        }
        if (m == 0) team_flag[team] = 0;
        team_bar(team);
        if (m < D && !isfinite(xo)) team_flag[team] = 1;
        team_bar(team);
        if (team_flag[team]) {
            if (m == 0) report_fail(p.fail, row);
        } else if (m < p.ld) {
            put_out(p, row, m, m < D ? xo : 0.f);
        }
        TCP(8);
        TCP_FLUSH(dual ? 0 : slot >= 0 ? 3 : nrow < D ? 1 : 2);
    }
#undef TCP_FLUSH
#undef TCP
#ifdef MCF_TC_PROFILE
    if (w.prof && m == 0)
        for (int k = 0; k < 10; ++k) atomicAdd(w.prof + k, tcp_acc[k]);
#endif
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_sh),
                     "r"(C::TMEM_COLS));
    }
}

template <int NBLK>
int launch_tc(const AlsParams &p, const PairPlan &q, const TcWs &w, cudaStream_t s) {
    using C = TcCfg<NBLK>;
    int rc;
    k_tc_split<<<148 * 8, 256, 0, s>>>(p, q, w, C::TW);
    if ((rc = check_launch("mcf_als_half_step(tensor-core split)"))) return rc;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_als_tc<NBLK>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        attr = true;
    }
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_als_tc<NBLK>, C::TEAMS * 128, C::SMEM);
    per_sm = std::max(1, std::min(per_sm, 512 / C::TMEM_COLS));
    const int64_t want = ceil_div(q.n_tasks, C::TEAMS);
    const int64_t grid = std::min<int64_t>(want, (int64_t)sms * per_sm);
    if (grid > 0) k_als_tc<NBLK><<<(unsigned)grid, C::TEAMS * 128, C::SMEM, s>>>(p, q, w);
    return check_launch("mcf_als_half_step(tensor core)");
}

}  // namespace

static unsigned long long *g_tc_prof = nullptr;

// lowest D routed to the tensor-core path (MCF_TC_MIN_D: experiments; the
// kernel handles any 49 <= D <= 128 -- DP = 64 is its smallest geometry)
int tc_min_d() {
    static const int v = [] {
        const char *e = getenv("MCF_TC_MIN_D");
        const int d = e ? atoi(e) : 64;
        return d < 49 ? 49 : d;
    }();
    return v;
}

// Hybrid experiment for 49 <= D < tc_min_d(): rows with at least
// MCF_TC_HYBRID_MIN_N ratings (and every hot-row chunk) take the tensor-core
// kernel, the others the CUDA-core tile-warp kernel.  Off by default (0):
// measured at config 4 (D = 50) 267 ms against 254 ms for the tile-warp kernel
// alone -- at DP = 64 the tensor-core Gram is bound by its per-stage cost,
// not by the gather bandwidth (profiles/r2_tc_path_notes.txt).
int tc_hybrid_min_n(int D, bool weighted) {
    const char *e = getenv("MCF_TC_HYBRID_MIN_N");
    const int v = e ? atoi(e) : 0;
    if (weighted || D < 49 || D >= tc_min_d() || getenv("MCF_NO_TC")) return 0;
    return v > 0 ? std::max(v, 2) : 0;
}

bool tc_path(int D, bool weighted) {
    return !weighted && D >= tc_min_d() && D <= 128 && !getenv("MCF_NO_TC");
}

size_t tc_slot_floats(int D) {
    const int dp = (D + 15) / 16 * 16;
    return (size_t)dp * (dp + 16);
}

static size_t tc_table_width(int D) { return (size_t)((D + 15) / 16 * 16 + 63) / 64 * 64; }

size_t tc_workspace_bytes(int D, int64_t slots, int64_t n_fixed, int64_t nnz) {
    return 256 + align_up(sizeof(int32_t) * (size_t)(slots + 1), 256) +
           align_up(sizeof(float) * (size_t)slots * tc_slot_floats(D), 256) +
           2 * align_up(2 * (size_t)n_fixed * tc_table_width(D) + 256, 256) +
           align_up(sizeof(uint32_t) * (size_t)(nnz + 64), 256);
}

int launch_als_tc(const AlsParams &p, const PairPlan &q, void *ws, size_t ws_bytes, int64_t slots,
                  int64_t nnz, int dual_cut, cudaStream_t s) {
    if (ws_bytes < tc_workspace_bytes(p.D, slots, p.n_fixed, nnz)) {
        set_error("mcf_als_half_step: workspace too small for the tensor-core path");
        return MCF_E_WORKSPACE;
    }
    Carve c(ws, ws_bytes);
    TcWs w;
    w.scal = c.take<unsigned>(4);
    w.hot_count = c.take<int32_t>((size_t)slots + 1);
    w.partials = c.take<float>((size_t)slots * tc_slot_floats(p.D));
    w.th = c.take<__half>((size_t)p.n_fixed * tc_table_width(p.D) + 128);
    w.tl = c.take<__half>((size_t)p.n_fixed * tc_table_width(p.D) + 128);
    w.ysp = c.take<uint32_t>((size_t)nnz + 64);
    w.n_slots = slots;
    w.prof = nullptr;
    w.team_limit = getenv("MCF_TC_TEAMS") ? atoi(getenv("MCF_TC_TEAMS")) : 4;
    w.dual_cut = dual_cut;
    if (getenv("MCF_TC_PROF")) {
        static unsigned long long *buf = nullptr;
        if (!buf) cudaMalloc(&buf, 80 * sizeof(unsigned long long));
        cudaMemset(buf, 0, 80 * sizeof(unsigned long long));
        w.prof = buf;
        g_tc_prof = buf;
    }
    int rc;
    if ((rc = cuda_status(cudaMemsetAsync(w.scal, 0, 4 * sizeof(unsigned), s), "memset"))) return rc;
    k_tc_prep<<<148 * 8, 256, 0, s>>>(p, q, w);
    if ((rc = check_launch("mcf_als_half_step(tensor-core prep)"))) return rc;
    switch ((p.D + 15) / 16) {
        case 4: return launch_tc<4>(p, q, w, s);
        case 5: return launch_tc<5>(p, q, w, s);
        case 6: return launch_tc<6>(p, q, w, s);
        case 7: return launch_tc<7>(p, q, w, s);
        case 8: return launch_tc<8>(p, q, w, s);
        default:
            set_error("mcf_als_half_step: tensor-core path needs 64 <= D <= 128");
            return MCF_E_UNSUPPORTED;
    }
}

}  // namespace mcf

// phase cycle counters of the tensor-core path (MCF_TC_PROF=1): per team,
// summed over CTAs; read and reset
extern "C" int mcf_tc_prof_read(unsigned long long *out10) {
    if (!mcf::g_tc_prof) return -1;
    cudaDeviceSynchronize();
    cudaMemcpy(out10, mcf::g_tc_prof, 14 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaMemset(mcf::g_tc_prof, 0, 80 * sizeof(unsigned long long));
    return 0;
}

// all 80 counters: [0..9] phases, [11..13] diagonal warp (TMEM-load wait,
// factorisation cycles, blocks), then per task class 16 each (10 phases,
// [10] = tasks): 0 dual rows, 1 primal rows with n < D (refined), 2 primal
// rows, 3 hot chunks
extern "C" int mcf_tc_prof_read_classes(unsigned long long *out80) {
    if (!mcf::g_tc_prof) return -1;
    cudaDeviceSynchronize();
    cudaMemcpy(out80, mcf::g_tc_prof, 80 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaMemset(mcf::g_tc_prof, 0, 80 * sizeof(unsigned long long));
    return 0;
}
