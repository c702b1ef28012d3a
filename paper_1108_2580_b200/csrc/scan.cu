// Device-wide exclusive prefix sum (reduce -> recursive scan of block sums ->
// block scan + offset).  Integer only, so results are exact and the order of
// operations never matters.
#include "common.cuh"

namespace mcf {
namespace {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <typename T>
__device__ T block_exclusive(T v, T *warp_tot, T *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T t = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T w = lane < SCAN_THREADS / 32 ? warp_tot[lane] : T(0);
        T wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T t = __shfl_up_sync(FULL, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < SCAN_THREADS / 32) warp_tot[lane] = wi - w;
        if (lane == SCAN_THREADS / 32 - 1) *total = wi;
    }
    __syncthreads();
    return inc - v + warp_tot[warp];
}

template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS) k_reduce(const T *in, int64_t n, T *sums) {
    __shared__ T wt[SCAN_THREADS / 32];
    __shared__ T tot;
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    T s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i)
        if (base + i < n) s += in[base + i];
    block_exclusive<T>(s, wt, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS) k_down(const T *in, T *out, int64_t n,
                                                       const T *offs) {
    __shared__ T wt[SCAN_THREADS / 32];
    __shared__ T tot;
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    T v[SCAN_ITEMS];
    T s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        v[i] = base + i < n ? in[base + i] : T(0);
        s += v[i];
    }
    T run = block_exclusive<T>(s, wt, &tot) + (offs ? offs[blockIdx.x] : T(0));
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
}

}  // namespace

template <typename T>
size_t scan_exclusive(const T *in, T *out, int64_t n, void *temp, size_t temp_bytes,
                      cudaStream_t s, int *err) {
    const int64_t nb = ceil_div(n, SCAN_TILE);
    size_t need = nb > 1 ? align_up(nb * sizeof(T), 256) : 0;
    if (nb > 1) need += scan_exclusive<T>(nullptr, nullptr, nb, nullptr, 0, s, nullptr);
    if (temp == nullptr && err == nullptr) return need;
    if (n <= 0) return need;
    if (temp_bytes < need) {
        *err = -2;
        return need;
    }
    if (nb == 1) {
        k_down<T><<<1, SCAN_THREADS, 0, s>>>(in, out, n, nullptr);
        return need;
    }
    T *sums = static_cast<T *>(temp);
    char *rest = static_cast<char *>(temp) + align_up(nb * sizeof(T), 256);
    k_reduce<T><<<(unsigned)nb, SCAN_THREADS, 0, s>>>(in, n, sums);
    scan_exclusive<T>(sums, sums, nb, rest, temp_bytes - align_up(nb * sizeof(T), 256), s, err);
    k_down<T><<<(unsigned)nb, SCAN_THREADS, 0, s>>>(in, out, n, sums);
    return need;
}

template size_t scan_exclusive<int32_t>(const int32_t *, int32_t *, int64_t, void *, size_t,
                                        cudaStream_t, int *);
template size_t scan_exclusive<int64_t>(const int64_t *, int64_t *, int64_t, void *, size_t,
                                        cudaStream_t, int *);

}  // namespace mcf
