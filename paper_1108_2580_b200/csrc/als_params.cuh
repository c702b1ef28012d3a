// ALS half-step parameters and device helpers shared by the kernels of
// als.cu (pair / warp / tile-warp / CTA paths) and als_tc.cu (tensor-core
// wide path).
#pragma once
#include "common.cuh"

namespace mcf {

constexpr int BATCH = 32;

struct AlsParams {
    const int64_t *ptr;
    const int32_t *idx;
    const float *val;
    const float *wts;
    const float *fixed;
    int64_t n_fixed;   // rows of `fixed` (TMA bounds)
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
    double *obj_partial;       // [(groups + hot rows) * 2] or null (fused objective)
    int64_t obj_groups;        // pair-path groups (hot rows follow them)
    // optional bias coordinate (MFITR full blocks): its own regulariser
    // bias_lam_c + bias_lam_n * n, no taxonomy terms; -1 = none
    int bias_dim;
    float bias_lam_c, bias_lam_n;
    // fused all-gather (multi-GPU): every solved row is also stored into
    // n_peers peer replicas (NVLink peer pointers, same row offsets as out)
    float *const *peer_out;
    int n_peers;
    // fused all-gather through NVLS multicast: the multicast address of the
    // replicated table (offset to this shard); one multimem store reaches
    // every GPU's replica, this one's included (replaces out + peer_out)
    float *mc_out;
    // Schur bias (pair path): the rows are [f | b] with f in columns 0..D-1
    // and b in column D; the kernel accumulates u = sum x, d = sum y beside
    // the Gram and eliminates b exactly: (A - u u^T/s) f = c - u d/s,
    // b = (d - u.f)/s, s = n + bias regulariser
    int schur;
    // MFITR item layers (Schur pair path): every row's [A | c | u | d | n]
    // (before any correction) is stored to emit[r * EMIT_STRIDE] for the
    // artist step, and the row's artist terms are removed from its rhs:
    // c -= A q_a + u b_a, d -= u.q_a + n b_a with [q_a | b_a] =
    // corr_tab[corr_idx[r]] (corr_idx[r] < 0: none)
    float *emit;
    const float *corr_tab;
    const int32_t *corr_idx;
    // pair Schur path: partner rows [x | 1 | t], the rating's target is
    // y - y_shift - t (the per-rating MFITR bias terms folded into the gather)
    int ysub;
    // hybrid wide path (49 <= D < 64): rows with at least skip_min_n ratings are
    // solved by the tensor-core kernel, the CUDA-core kernels skip them (0: none)
    int skip_min_n;
};
constexpr int EMIT_STRIDE = 256;

// one element of row r of the solved shard: local table + every peer replica
__device__ __forceinline__ void put_out(const AlsParams &p, int r, int i, float v) {
    const size_t off = (size_t)r * p.ld + i;
    if (p.mc_out) {
        asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p.mc_out + off), "f"(v)
                     : "memory");
        return;
    }
    p.out[off] = v;
    for (int k = 0; k < p.n_peers; ++k) p.peer_out[k][off] = v;
}

// diagonal regulariser of coordinate i of row system with n ratings.  A
// bias of a row without ratings (an item only the taxonomy touches) has a
// zero Gram row and zero right-hand side: pivot 1 -> bias 0 (any value
// minimises the loss then; 0 is the reference's initial value).
__device__ __forceinline__ float diag_at(const AlsParams &p, int i, float diag, float n) {
    return i == p.bias_dim ? (n > 0.f ? fmaf(p.bias_lam_n, n, p.bias_lam_c) : 1.f) : diag;
}
// taxonomy T term of coordinate i (none on the bias coordinate)
__device__ __forceinline__ float tax_rhs(const AlsParams &p, int r, int i, float b) {
    return (p.tax_T && i != p.bias_dim) ? fmaf(p.tau, p.tax_T[(size_t)r * p.ld + i], b) : b;
}

__device__ __forceinline__ void prefetch_l2(const void *a) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
}

__device__ __forceinline__ void report_fail(unsigned long long *fail, int r) {
    atomicMin(fail, static_cast<unsigned long long>(r));
}

struct PairPlan {
    const int32_t *task_row;
    const int64_t *task_k0;
    const int32_t *task_n;
    const int32_t *task_slot;
    int64_t n_tasks;
    const int32_t *sorted_j;   // heavy list indices first
    const int32_t *hoff;       // [n_list + 1] first chunk slot of list entry j
    int64_t n_heavy;
    int32_t *group_counter;
    double *obj_out;           // [2] = (sum sse, sum reg) or null
};

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
// try_wait with a suspend-time hint: the thread sleeps in hardware until the
// phase completes (or ~10 ms pass) instead of returning every few hundred
// cycles -- a polling loop of bare try_waits issued ~60 times per wait and
// took issue slots from the other warps of its SM sub-partition
__device__ __forceinline__ bool mbar_try(unsigned bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(bar), "r"(parity), "r"(10000000u)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    while (!mbar_try(bar, parity)) {
    }
}

// tensor-core wide path (als_tc.cu): 21 <= D <= 127, no per-observation weights
bool tc_path(int D, bool weighted);
int tc_min_d();
// 49 <= D < tc_min_d(): rows this long go to the tensor-core kernel (0: hybrid off)
int tc_hybrid_min_n(int D, bool weighted);
size_t tc_workspace_bytes(int D, int64_t slots, int64_t n_fixed, int64_t nnz);
int launch_als_tc(const AlsParams &p, const PairPlan &q, void *ws, size_t ws_bytes, int64_t slots,
                  int64_t nnz, int dual_cut, cudaStream_t s);

// short rows of the wide path on CUDA cores in the dual form (als_dual.cu):
// light tasks with at most als_dual_cut() ratings (0: call not eligible) are
// left by the tensor-core kernel and taken from the end of the task list
int als_dual_cut(const AlsParams &p, bool weighted);
int launch_als_dual(const AlsParams &p, const PairPlan &q, int64_t first_light, int *counters, int cut,
                    cudaStream_t s);

}  // namespace mcf
