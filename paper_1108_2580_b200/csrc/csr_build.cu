// Rating layout: stable CSR / CSC build from COO records (sm_100a).
//
// Replaces factor._side_csr (reference factor.py:493-509): the reference
// rebuilds the layout with a serial stable argsort every half-step; here it
// is built once, on device, and stays resident.  In-row order must equal
// record order (argsort kind="stable"), bit for bit.
//
//   1. range check of the keys (reported after the build, one sync)
//   2. stable LSD radix sort of (key, record index) with 7/8-bit digits:
//      per pass  (a) per-tile digit histograms, (b) one device-wide exclusive
//      scan over the digit-major [bins][tiles] table, (c) stable scatter.
//      Stability inside a tile: each warp owns a contiguous 256-record
//      sub-tile read slot by slot (record = slot*32 + lane), ranks equal
//      digits with __match_any_sync, and keeps a warp-private running
//      histogram; warps are then offset in order.  Record order is therefore
//      (tile, warp, slot, lane) = ascending record index.
//   3. ptr from the row boundaries of the sorted keys (no atomics: Zipf-hot
//      rows would serialise a histogram), gather idx[k] = cols[perm[k]],
//      val[k] = vals[perm[k]].
#include "common.cuh"
#include "../../include/mcf.h"

namespace mcf {
namespace {

constexpr int RS_WARPS = 8;
constexpr int RS_SLOTS = 8;
constexpr int RS_THREADS = RS_WARPS * 32;
constexpr int RS_TILE = RS_THREADS * RS_SLOTS;  // 2048 records
constexpr int RS_MAX_BINS = 256;

__global__ void k_check(const int32_t *keys, int64_t nnz, int32_t n_rows, int *bad) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t key = keys[k];
        if (key < 0 || key >= n_rows) atomicExch(bad, 1);
    }
}

// ptr from the sorted keys: ptr[r] = first position whose key >= r (no
// atomics -- the Zipf-hot rows would serialise a histogram).
__global__ void k_bounds(const uint32_t *sk, int64_t nnz, int32_t n_rows, int64_t *ptr) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= nnz;
         k += (int64_t)gridDim.x * blockDim.x) {
        // clamped: out-of-range keys are reported by k_check, never written past ptr
        const int64_t lo = k == 0 ? -1 : min((int64_t)sk[k - 1], (int64_t)n_rows);
        const int64_t hi = k == nnz ? (int64_t)n_rows : min((int64_t)sk[k], (int64_t)n_rows);
        for (int64_t r = lo + 1; r <= hi; ++r) ptr[r] = k;
    }
}

__global__ void k_bounds_single(int64_t nnz, int32_t n_rows, int64_t *ptr) {
    for (int32_t r = threadIdx.x; r <= n_rows; r += blockDim.x) ptr[r] = r == 0 ? 0 : nnz;
}

// Ranks of the tile's records by digit; returns per-slot local ranks (within
// the warp's running histogram) and leaves per-warp digit counts in hist.
__device__ __forceinline__ void warp_rank(const uint32_t *dig, int *rank, int *hist_w) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int s = 0; s < RS_SLOTS; ++s) {
        const uint32_t d = dig[s];
        const unsigned peers = __match_any_sync(FULL, d);
        const int leader = __ffs(peers) - 1;
        int base = 0;
        if (d < RS_MAX_BINS) base = hist_w[d];
        __syncwarp();
        if (d < RS_MAX_BINS && lane == leader) hist_w[d] = base + __popc(peers);
        __syncwarp();
        rank[s] = base + __popc(peers & lt);
    }
}

__device__ __forceinline__ uint32_t load_key(const int32_t *keys_in, const uint32_t *keys_u,
                                             int64_t r, int64_t nnz) {
    if (r >= nnz) return 0xffffffffu;
    return keys_u ? keys_u[r] : static_cast<uint32_t>(keys_in[r]);
}

__global__ void __launch_bounds__(RS_THREADS) k_tile_hist(const int32_t *keys_in,
                                                          const uint32_t *keys_u, int64_t nnz,
                                                          int shift, int bins, int64_t n_tiles,
                                                          int32_t *tile_hist) {
    __shared__ int hist[RS_WARPS][RS_MAX_BINS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < RS_WARPS * RS_MAX_BINS; i += RS_THREADS) (&hist[0][0])[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE + warp * (32 * RS_SLOTS);
    uint32_t dig[RS_SLOTS];
    int rank[RS_SLOTS];
#pragma unroll
    for (int s = 0; s < RS_SLOTS; ++s) {
        const uint32_t key = load_key(keys_in, keys_u, base + s * 32 + lane, nnz);
        dig[s] = key == 0xffffffffu ? RS_MAX_BINS : (key >> shift) & (bins - 1);
    }
    warp_rank(dig, rank, hist[warp]);
    __syncthreads();
    for (int d = threadIdx.x; d < bins; d += RS_THREADS) {
        int t = 0;
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) t += hist[w][d];
        tile_hist[(int64_t)d * n_tiles + blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(RS_THREADS) k_scatter(
    const int32_t *keys_in, const uint32_t *keys_u, const int32_t *vals_in, int64_t nnz,
    int shift, int bins, int64_t n_tiles, const int32_t *tile_off, uint32_t *keys_out,
    int32_t *vals_out) {
    __shared__ int hist[RS_WARPS][RS_MAX_BINS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < RS_WARPS * RS_MAX_BINS; i += RS_THREADS) (&hist[0][0])[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE + warp * (32 * RS_SLOTS);
    uint32_t key[RS_SLOTS], dig[RS_SLOTS];
    int32_t val[RS_SLOTS];
    int rank[RS_SLOTS];
#pragma unroll
    for (int s = 0; s < RS_SLOTS; ++s) {
        const int64_t r = base + s * 32 + lane;
        key[s] = load_key(keys_in, keys_u, r, nnz);
        val[s] = r < nnz ? (vals_in ? vals_in[r] : static_cast<int32_t>(r)) : 0;
        dig[s] = key[s] == 0xffffffffu ? RS_MAX_BINS : (key[s] >> shift) & (bins - 1);
    }
    warp_rank(dig, rank, hist[warp]);
    __syncthreads();
    // exclusive prefix over warps per digit, seeded with the tile's global offset
    for (int d = threadIdx.x; d < bins; d += RS_THREADS) {
        int run = tile_off[(int64_t)d * n_tiles + blockIdx.x];
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) {
            const int t = hist[w][d];
            hist[w][d] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < RS_SLOTS; ++s) {
        if (dig[s] >= RS_MAX_BINS) continue;
        const int dst = hist[warp][dig[s]] + rank[s];
        keys_out[dst] = key[s];
        vals_out[dst] = val[s];
    }
}

__global__ void k_gather(const int32_t *perm, const int32_t *cols, const float *vals, int64_t nnz,
                         int32_t *idx_out, float *val_out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = perm[k];
        idx_out[k] = cols[p];
        val_out[k] = vals[p];
    }
}

__global__ void k_iota(int32_t *perm, int64_t nnz) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
         k += (int64_t)gridDim.x * blockDim.x)
        perm[k] = static_cast<int32_t>(k);
}

int key_bits(int32_t n_rows) {
    int b = 0;
    while (b < 31 && (int64_t(1) << b) < n_rows) ++b;
    return b;
}

struct CsrWs {
    int *bad;
    uint32_t *keys[2];
    int32_t *vals[2];
    int32_t *tile_hist;
    void *scan_tmp;
    size_t scan_bytes;
};

CsrWs carve_csr(void *ws, size_t cap, int64_t nnz, int32_t n_rows, size_t *need) {
    Carve c(ws, cap);
    CsrWs w;
    w.bad = c.take<int>(1);
    for (int i = 0; i < 2; ++i) {
        w.keys[i] = c.take<uint32_t>((size_t)nnz);
        w.vals[i] = c.take<int32_t>((size_t)nnz);
    }
    const int64_t n_tiles = ceil_div(nnz, RS_TILE);
    w.tile_hist = c.take<int32_t>((size_t)(n_tiles * RS_MAX_BINS));
    size_t sb1 = scan_exclusive<int32_t>(nullptr, nullptr, n_tiles * RS_MAX_BINS, nullptr, 0,
                                         nullptr, nullptr);
    size_t sb2 = scan_exclusive<int64_t>(nullptr, nullptr, (int64_t)n_rows + 1, nullptr, 0,
                                         nullptr, nullptr);
    w.scan_bytes = sb1 > sb2 ? sb1 : sb2;
    w.scan_tmp = c.take<char>(w.scan_bytes + 256);
    *need = c.used;
    return w;
}

}  // namespace
}  // namespace mcf

using namespace mcf;

extern "C" size_t mcf_csr_workspace_bytes(int64_t nnz, int32_t n_rows) {
    size_t need = 0;
    carve_csr(nullptr, 0, nnz, n_rows, &need);
    return need;
}

extern "C" int mcf_csr_build(const int32_t *keys, const int32_t *cols, const float *vals,
                             int64_t nnz, int32_t n_rows, int64_t *ptr_out, int32_t *idx_out,
                             float *val_out, int32_t *perm_out, void *ws, size_t ws_bytes,
                             void *stream) {
    if (nnz < 0 || n_rows < 0 || nnz >= (int64_t(1) << 31) || !ptr_out ||
        (nnz > 0 && (!keys || !cols || !vals || !idx_out || !val_out))) {
        set_error("mcf_csr_build: invalid arguments");
        return MCF_E_ARG;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    size_t need = 0;
    CsrWs w = carve_csr(ws, ws_bytes, nnz, n_rows, &need);
    if (!ws || ws_bytes < need) {
        set_error("mcf_csr_build: workspace too small");
        return MCF_E_WORKSPACE;
    }
    int rc;
    if ((rc = cuda_status(cudaMemsetAsync(w.bad, 0, sizeof(int), s), "memset"))) return rc;
    const int gs = 148 * 8;
    int err = 0;
    if (nnz > 0) k_check<<<gs, 256, 0, s>>>(keys, nnz, n_rows, w.bad);
    if (nnz == 0) {
        k_bounds_single<<<1, 256, 0, s>>>(0, n_rows, ptr_out);
        return check_launch("mcf_csr_build");
    }

    const int bits = key_bits(n_rows);
    const int64_t n_tiles = ceil_div(nnz, RS_TILE);
    int32_t *perm = w.vals[0];
    if (bits == 0) {
        k_iota<<<gs, 256, 0, s>>>(perm, nnz);
        k_bounds_single<<<1, 256, 0, s>>>(nnz, n_rows, ptr_out);
    } else {
        const int passes = (bits + 7) / 8;
        const int dbits = (bits + passes - 1) / passes;
        const int bins = 1 << dbits;
        int cur = 0;
        for (int p = 0; p < passes; ++p) {
            const int shift = p * dbits;
            const int32_t *kin = p == 0 ? keys : nullptr;
            const uint32_t *ku = p == 0 ? nullptr : w.keys[cur];
            const int32_t *vin = p == 0 ? nullptr : w.vals[cur];
            k_tile_hist<<<(unsigned)n_tiles, RS_THREADS, 0, s>>>(kin, ku, nnz, shift, bins,
                                                                 n_tiles, w.tile_hist);
            scan_exclusive<int32_t>(w.tile_hist, w.tile_hist, n_tiles * bins, w.scan_tmp,
                                    w.scan_bytes, s, &err);
            k_scatter<<<(unsigned)n_tiles, RS_THREADS, 0, s>>>(kin, ku, vin, nnz, shift, bins,
                                                               n_tiles, w.tile_hist,
                                                               w.keys[cur ^ 1], w.vals[cur ^ 1]);
            cur ^= 1;
        }
        perm = w.vals[cur];
        k_bounds<<<gs, 256, 0, s>>>(w.keys[cur], nnz, n_rows, ptr_out);
    }
    k_gather<<<gs, 256, 0, s>>>(perm, cols, vals, nnz, idx_out, val_out);
    if (perm_out)
        if ((rc = cuda_status(cudaMemcpyAsync(perm_out, perm, sizeof(int32_t) * nnz,
                                              cudaMemcpyDeviceToDevice, s),
                              "memcpy")))
            return rc;
    if ((rc = check_launch("mcf_csr_build"))) return rc;
    int bad = 0;
    if ((rc = cuda_status(cudaMemcpyAsync(&bad, w.bad, sizeof(int), cudaMemcpyDeviceToHost, s),
                          "memcpy")))
        return rc;
    if ((rc = cuda_status(cudaStreamSynchronize(s), "sync"))) return rc;
    if (bad) {
        set_error("mcf_csr_build: key outside [0, n_rows)");
        return MCF_E_RANGE;
    }
    return MCF_OK;
}
