// Shared device helpers for libmcf (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace mcf {

constexpr unsigned FULL = 0xffffffffu;

// thread-local last error (mcf_last_error)
void set_error(const std::string &msg);
int cuda_status(cudaError_t e, const char *where);
int check_launch(const char *where);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Bump allocator over a caller workspace.
struct Carve {
    char *base;
    size_t used = 0, cap;
    Carve(void *p, size_t c) : base(static_cast<char *>(p)), cap(c) {}
    template <typename T>
    T *take(size_t n) {
        used = align_up(used, 256);
        T *p = reinterpret_cast<T *>(base ? base + used : nullptr);
        used += n * sizeof(T);
        return p;
    }
    bool ok() const { return used <= cap; }
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int src_bytes) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Device-wide exclusive scan (3 phases, recursive on block sums).
// in/out may alias.  Returns bytes of temp needed when temp == nullptr.
template <typename T>
size_t scan_exclusive(const T *in, T *out, int64_t n, void *temp, size_t temp_bytes,
                      cudaStream_t s, int *err);

}  // namespace mcf
