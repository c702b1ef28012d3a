// Rating layout: stable CSR / CSC build from COO records (sm_100a).
//
// Replaces factor._side_csr (reference factor.py:493-509): the reference
// rebuilds the layout with a serial stable argsort every half-step; here it
// is built once, on device, and stays resident.  In-row order must equal
// record order (argsort kind="stable"), bit for bit.
//
// Stable LSD radix sort of whole records (key, partner, value[, record
// index]) with 7/8-bit digits; no gather pass afterwards (a random gather
// of partner/value by permutation fetched a 128 B line per 4 B element).
// Per pass:
//   (a) k_tile_hist: per-tile digit counts (shared-memory atomics, 16 B
//       loads); pass 0 also range-checks the keys (reported after the build);
//   (b) one device-wide exclusive scan over the digit-major [bins][tiles]
//       table -> each tile's global offset per digit;
//   (c) k_scatter: each warp ranks its contiguous 512-record sub-tile slot
//       by slot with a ballot multi-split (record = slot*32 + lane, so the
//       rank order is ascending record index), the tile is reordered by
//       digit in shared memory, and written out as contiguous per-digit
//       runs (coalesced).  The last pass writes partner/value straight into
//       the CSR arrays.
// Then ptr from the row boundaries of the sorted keys (no atomics: Zipf-hot
// rows would serialise a histogram).
#include "common.cuh"
#include "../../include/mcf.h"

namespace mcf {
namespace {

constexpr int RS_WARPS = 8;
constexpr int RS_SLOTS = 16;
constexpr int RS_THREADS = RS_WARPS * 32;
constexpr int RS_SUB = RS_SLOTS * 32;           // records per warp sub-tile
constexpr int RS_TILE = RS_THREADS * RS_SLOTS;  // 4096 records
constexpr int RS_MAX_BITS = 8;
constexpr int RS_MAX_BINS = 1 << RS_MAX_BITS;

// ptr from the sorted keys: ptr[r] = first position whose key >= r (no
// atomics -- the Zipf-hot rows would serialise a histogram).
__global__ void k_bounds(const uint32_t *sk, int64_t nnz, int32_t n_rows, int64_t *ptr) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= nnz;
         k += (int64_t)gridDim.x * blockDim.x) {
        // clamped: out-of-range keys are reported by the range check, never written past ptr
        const int64_t lo = k == 0 ? -1 : min((int64_t)sk[k - 1], (int64_t)n_rows);
        const int64_t hi = k == nnz ? (int64_t)n_rows : min((int64_t)sk[k], (int64_t)n_rows);
        for (int64_t r = lo + 1; r <= hi; ++r) ptr[r] = k;
    }
}

__global__ void k_bounds_single(int64_t nnz, int32_t n_rows, int64_t *ptr) {
    for (int32_t r = threadIdx.x; r <= n_rows; r += blockDim.x) ptr[r] = r == 0 ? 0 : nnz;
}

__global__ void k_check(const int32_t *keys, int64_t nnz, int32_t n_rows, int *bad) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t key = keys[k];
        if (key < 0 || key >= n_rows) atomicExch(bad, 1);
    }
}

__global__ void __launch_bounds__(RS_THREADS) k_tile_hist(const uint32_t *keys, int64_t nnz,
                                                          int shift, int bins, int64_t n_tiles,
                                                          int32_t *tile_hist, uint32_t n_rows,
                                                          int *bad) {
    __shared__ int hist[RS_WARPS][RS_MAX_BINS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < RS_WARPS * RS_MAX_BINS; i += RS_THREADS) (&hist[0][0])[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    const uint32_t mask = bins - 1;
    bool oob = false;
    if (base + RS_TILE <= nnz && (reinterpret_cast<uintptr_t>(keys) & 15) == 0) {
        const uint4 *k4 = reinterpret_cast<const uint4 *>(keys + base);
#pragma unroll
        for (int j = 0; j < RS_TILE / 4 / RS_THREADS; ++j) {
            const uint4 v = __ldcs(k4 + j * RS_THREADS + threadIdx.x);
            atomicAdd(&hist[warp][(v.x >> shift) & mask], 1);
            atomicAdd(&hist[warp][(v.y >> shift) & mask], 1);
            atomicAdd(&hist[warp][(v.z >> shift) & mask], 1);
            atomicAdd(&hist[warp][(v.w >> shift) & mask], 1);
            if (bad) oob |= (v.x >= n_rows) | (v.y >= n_rows) | (v.z >= n_rows) | (v.w >= n_rows);
        }
    } else {
        for (int j = threadIdx.x; j < RS_TILE; j += RS_THREADS) {
            if (base + j >= nnz) break;
            const uint32_t v = keys[base + j];
            atomicAdd(&hist[warp][(v >> shift) & mask], 1);
            if (bad) oob |= v >= n_rows;
        }
    }
    if (oob) atomicExch(bad, 1);
    __syncthreads();
    for (int d = threadIdx.x; d < bins; d += RS_THREADS) {
        int t = 0;
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) t += hist[w][d];
        tile_hist[(int64_t)d * n_tiles + blockIdx.x] = t;
    }
}

struct ScatterIO {
    const uint32_t *keys_in;
    const int32_t *cols_in;
    const float *vals_in;
    const int32_t *perm_in;   // nullptr on pass 0 (record index = position)
    uint32_t *keys_out;       // nullptr: not needed
    int32_t *cols_out;
    float *vals_out;
    int32_t *perm_out;        // nullptr: not carried
};

// Shared memory: the tile reordered by digit (keys, cols, vals[, perm]).
template <bool PERM>
__global__ void __launch_bounds__(RS_THREADS, 2) k_scatter(ScatterIO io, int64_t nnz, int shift,
                                                          int dbits, int64_t n_tiles,
                                                          const int32_t *tile_off) {
    extern __shared__ uint32_t rs_smem[];
    uint32_t *skey = rs_smem;
    int32_t *scol = reinterpret_cast<int32_t *>(skey + RS_TILE);
    float *sval = reinterpret_cast<float *>(scol + RS_TILE);
    int32_t *sperm = reinterpret_cast<int32_t *>(sval + RS_TILE);
    __shared__ int hist[RS_WARPS][RS_MAX_BINS + 1];
    __shared__ int gbase[RS_MAX_BINS];
    __shared__ int wsum[RS_WARPS];
    const int bins = 1 << dbits;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    for (int i = threadIdx.x; i < RS_WARPS * (RS_MAX_BINS + 1); i += RS_THREADS)
        (&hist[0][0])[i] = 0;
    const int64_t tile0 = (int64_t)blockIdx.x * RS_TILE;
    const int64_t base = tile0 + warp * RS_SUB;
    uint32_t key[RS_SLOTS];
    int32_t col[RS_SLOTS], pm[RS_SLOTS];
    float val[RS_SLOTS];
#pragma unroll
    for (int s = 0; s < RS_SLOTS; ++s) {
        const int64_t r = base + s * 32 + lane;
        const bool ok = r < nnz;
        key[s] = ok ? __ldcs(io.keys_in + r) : 0u;
        col[s] = ok ? __ldcs(io.cols_in + r) : 0;
        val[s] = ok ? __ldcs(io.vals_in + r) : 0.f;
        if (PERM) pm[s] = ok ? (io.perm_in ? __ldcs(io.perm_in + r) : (int32_t)r) : 0;
    }
    __syncthreads();
    // ballot multi-split: peers = lanes of this slot with the same digit
    int rank[RS_SLOTS];
    int *hw = hist[warp];
#pragma unroll
    for (int s = 0; s < RS_SLOTS; ++s) {
        const bool ok = base + s * 32 + lane < nnz;
        const uint32_t d = ok ? (key[s] >> shift) & (bins - 1) : (uint32_t)bins;
        unsigned peers = __ballot_sync(FULL, ok);
        if (!ok) peers = ~peers;
        for (int b = 0; b < dbits; ++b) {
            const unsigned bal = __ballot_sync(FULL, (d >> b) & 1u);
            peers &= ((d >> b) & 1u) ? bal : ~bal;
        }
        const int cnt = hw[d];
        __syncwarp();
        if ((peers & lt) == 0) hw[d] = cnt + __popc(peers);
        __syncwarp();
        rank[s] = cnt + __popc(peers & lt);
    }
    __syncthreads();
    // per digit: warp offsets inside the tile's digit run, tile digit starts
    int tot = 0;
    const int d = threadIdx.x;   // bins <= RS_THREADS
    if (d < bins) {
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) {
            const int t = hist[w][d];
            hist[w][d] = tot;
            tot += t;
        }
    }
    // block exclusive scan of tot over digits
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int wpre = 0;
    for (int w = 0; w < warp; ++w) wpre += wsum[w];
    const int start = wpre + incl - tot;
    if (d < bins) {
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) hist[w][d] += start;
        gbase[d] = tile_off[(int64_t)d * n_tiles + blockIdx.x] - start;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < RS_SLOTS; ++s) {
        if (base + s * 32 + lane >= nnz) continue;
        const uint32_t dg = (key[s] >> shift) & (bins - 1);
        const int lp = hw[dg] + rank[s];
        skey[lp] = key[s];
        scol[lp] = col[s];
        sval[lp] = val[s];
        if (PERM) sperm[lp] = pm[s];
    }
    __syncthreads();
    const int valid = nnz - tile0 < RS_TILE ? (int)(nnz - tile0) : RS_TILE;
    for (int i = threadIdx.x; i < valid; i += RS_THREADS) {
        const uint32_t k = skey[i];
        const int64_t g = (int64_t)gbase[(k >> shift) & (bins - 1)] + i;
        if (io.keys_out) __stcs(io.keys_out + g, k);
        __stcs(io.cols_out + g, scol[i]);
        __stcs(io.vals_out + g, sval[i]);
        if (PERM) __stcs(io.perm_out + g, sperm[i]);
    }
}

__global__ void k_copy_rows(const int32_t *cols, const float *vals, int64_t nnz, int32_t *idx_out,
                            float *val_out, int32_t *perm) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
         k += (int64_t)gridDim.x * blockDim.x) {
        idx_out[k] = cols[k];
        val_out[k] = vals[k];
        if (perm) perm[k] = static_cast<int32_t>(k);
    }
}

int key_bits(int32_t n_rows) {
    int b = 0;
    while (b < 31 && (int64_t(1) << b) < n_rows) ++b;
    return b;
}

struct CsrWs {
    int *bad;
    uint32_t *keys[2];
    int32_t *cols[2];
    float *vals[2];
    int32_t *perm[2];
    int32_t *tile_hist;
    void *scan_tmp;
    size_t scan_bytes;
};

CsrWs carve_csr(void *ws, size_t cap, int64_t nnz, int32_t n_rows, bool with_perm, size_t *need) {
    Carve c(ws, cap);
    CsrWs w;
    w.bad = c.take<int>(1);
    for (int i = 0; i < 2; ++i) {
        w.keys[i] = c.take<uint32_t>((size_t)nnz);
        w.cols[i] = c.take<int32_t>((size_t)nnz);
        w.vals[i] = c.take<float>((size_t)nnz);
        w.perm[i] = with_perm ? c.take<int32_t>((size_t)nnz) : nullptr;
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

size_t scatter_smem(bool perm) { return (size_t)RS_TILE * (perm ? 16 : 12); }

}  // namespace
}  // namespace mcf

using namespace mcf;

// The workspace always has room for the record-index payload, so the size
// does not depend on whether the caller asks for perm_out.
extern "C" size_t mcf_csr_workspace_bytes(int64_t nnz, int32_t n_rows) {
    size_t need = 0;
    carve_csr(nullptr, 0, nnz, n_rows, true, &need);
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
    const bool with_perm = perm_out != nullptr;
    CsrWs w = carve_csr(ws, ws_bytes, nnz, n_rows, with_perm, &need);
    if (!ws || ws_bytes < mcf_csr_workspace_bytes(nnz, n_rows)) {
        set_error("mcf_csr_build: workspace too small");
        return MCF_E_WORKSPACE;
    }
    int rc;
    if ((rc = cuda_status(cudaMemsetAsync(w.bad, 0, sizeof(int), s), "memset"))) return rc;
    const int gs = 148 * 8;
    int err = 0;
    if (nnz == 0) {
        k_bounds_single<<<1, 256, 0, s>>>(0, n_rows, ptr_out);
        return check_launch("mcf_csr_build");
    }

    const int bits = key_bits(n_rows);
    const int64_t n_tiles = ceil_div(nnz, RS_TILE);
    if (bits == 0) {   // one row: record order is the row order
        k_check<<<gs, 256, 0, s>>>(keys, nnz, n_rows, w.bad);
        k_copy_rows<<<gs, 256, 0, s>>>(cols, vals, nnz, idx_out, val_out, perm_out);
        k_bounds_single<<<1, 256, 0, s>>>(nnz, n_rows, ptr_out);
    } else {
        const int passes = (bits + RS_MAX_BITS - 1) / RS_MAX_BITS;
        const int dbits = (bits + passes - 1) / passes;
        const int bins = 1 << dbits;
        const size_t smem = scatter_smem(with_perm);
        static bool attr_set[2] = {false, false};
        if (!attr_set[with_perm]) {
            cudaError_t e = with_perm
                ? cudaFuncSetAttribute(k_scatter<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                : cudaFuncSetAttribute(k_scatter<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if ((rc = cuda_status(e, "cudaFuncSetAttribute"))) return rc;
            attr_set[with_perm] = true;
        }
        const uint32_t *kin = reinterpret_cast<const uint32_t *>(keys);
        const int32_t *cin = cols, *pin = nullptr;
        const float *vin = vals;
        for (int p = 0; p < passes; ++p) {
            const int shift = p * dbits;
            const bool last = p == passes - 1;
            const int o = p & 1;
            k_tile_hist<<<(unsigned)n_tiles, RS_THREADS, 0, s>>>(
                kin, nnz, shift, bins, n_tiles, w.tile_hist, (uint32_t)n_rows, p == 0 ? w.bad : nullptr);
            scan_exclusive<int32_t>(w.tile_hist, w.tile_hist, n_tiles * bins, w.scan_tmp,
                                    w.scan_bytes, s, &err);
            ScatterIO io{kin, cin, vin, pin, w.keys[o], last ? idx_out : w.cols[o],
                         last ? val_out : w.vals[o], last ? perm_out : w.perm[o]};
            if (with_perm)
                k_scatter<true><<<(unsigned)n_tiles, RS_THREADS, smem, s>>>(io, nnz, shift, dbits,
                                                                           n_tiles, w.tile_hist);
            else
                k_scatter<false><<<(unsigned)n_tiles, RS_THREADS, smem, s>>>(io, nnz, shift, dbits,
                                                                            n_tiles, w.tile_hist);
            kin = w.keys[o];
            cin = w.cols[o];
            vin = w.vals[o];
            pin = w.perm[o];
        }
        k_bounds<<<gs, 256, 0, s>>>(kin, nnz, n_rows, ptr_out);
    }
    if (err) {
        set_error("mcf_csr_build: scan workspace too small");
        return MCF_E_WORKSPACE;
    }
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
