// Probe of the tcgen05 kind::f16 mechanics the tensor-core wide path needs
// (sm_100a), checked against the CPU:
//   mode 0  Gram C = X^T X, X (K ratings x F features, fp16) MN-major, no swizzle,
//           desc LBO = k-group stride, SBO = 16-byte-chunk stride (CuTe reading)
//   mode 1  same layout, LBO/SBO swapped in the descriptor
//   mode 2  Gram, MN-major SWIZZLE_128B (64-feature atoms, k-groups outer)
//   mode 3  panel update C = -P P^T[:, r0:], P (128 rows x 16 k) K-major no
//           swizzle, B starting at row r0, accumulator column offset r0,
//           a_negate, accumulating onto a first MMA (C = X^T X first)
// M = 128, N = 112 (mode 3: N = 112 - r0), K = 16 per instruction.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint64_t layout = 0) {
    return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46) | (layout << 61);
}
__device__ __forceinline__ uint32_t idesc_f16(int M, int N, bool a_mn, bool b_mn, bool neg_a) {
    return (1u << 4) | (neg_a ? 1u << 13 : 0u) | (a_mn ? 1u << 15 : 0u) | (b_mn ? 1u << 16 : 0u) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(id), "r"(acc));
}

constexpr int M = 128, F = 112, K = 32, NMAX = 112, R0 = 32;

__global__ void k_probe(const float *X, const float *Pm, float *C, int *status, int mode) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) unsigned long long bar;
    __shared__ uint32_t tbase;
    __half *xs = reinterpret_cast<__half *>(smem);            // Gram operand tile (K x 128 features)
    __half *ps = reinterpret_cast<__half *>(smem + 65536);    // panel tile (128 rows x 16 k)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int e = tid; e < (65536 + 8192) / 2; e += blockDim.x) reinterpret_cast<__half *>(smem)[e] = __float2half(0.f);
    __syncthreads();
    constexpr int CHUNKS = 128 / 8;        // 16-byte chunks along MN (128 features)
    constexpr int LBO_K = CHUNKS * 128;    // interleave: k-group stride
    for (int e = tid; e < K * F; e += blockDim.x) {
        const int k = e / F, f = e % F;
        size_t off;
        if (mode == 2) {                   // SW128: k-groups outer, 2 atoms of 64 features each
            const int a = f >> 6, ch = (f >> 3) & 7, r = k & 7;
            off = (size_t)(k >> 3) * 2048 + a * 1024 + r * 128 + ((ch ^ r) << 4) + (f & 7) * 2;
        } else {
            off = (size_t)(k >> 3) * LBO_K + (f >> 3) * 128 + (k & 7) * 16 + (f & 7) * 2;
        }
        *reinterpret_cast<__half *>(smem + off) = __float2half(X[e]);
    }
    // panel: rows m (0..127) x k (0..15), K-major interleave: 8-row groups SBO = 128, k-chunks LBO = 16*128
    for (int e = tid; e < 128 * 16; e += blockDim.x) {
        const int m = e / 16, k = e % 16;
        const size_t off = (size_t)(m >> 3) * 128 + (m & 7) * 16 + (k >> 3) * (16 * 128) + (k & 7) * 2;
        *reinterpret_cast<__half *>(reinterpret_cast<unsigned char *>(ps) + off) = __float2half(Pm[e]);
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t taddr = tbase;
    if (tid == 0) {
        for (int kg = 0; kg < K / 16; ++kg) {   // 16 k per instruction = 2 k-groups of 8
            uint64_t d;
            if (mode == 0) d = sdesc(smem_u32(xs) + kg * 2 * LBO_K, LBO_K, 128);
            else if (mode == 1) d = sdesc(smem_u32(xs) + kg * 2 * LBO_K, 128, LBO_K);
            else if (mode == 2) d = sdesc(smem_u32(xs) + kg * 2 * 2048, 1024, 2048, 2);
            else d = sdesc(smem_u32(xs) + kg * 2 * LBO_K, LBO_K, 128);
            mma(taddr, d, d, idesc_f16(M, NMAX, true, true, false), kg > 0);
        }
        if (mode == 3) {
            const uint64_t da = sdesc(smem_u32(ps), 16 * 128, 128);
            const uint64_t db = sdesc(smem_u32(ps) + (R0 / 8) * 128, 16 * 128, 128);
            mma(taddr + R0, da, db, idesc_f16(M, NMAX - R0, false, false, true), 1);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(smem_u32(&bar)) : "memory");
    }
    {
        uint32_t done = 0;
        for (long it = 0; it < (1l << 26) && !done; ++it)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
        if (!done && lane == 0) atomicExch(status, 1);
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp & 3;
    const int row = 32 * q + lane;
    for (int j = 0; j < NMAX / 8; ++j) {
        uint32_t r[8];
        const uint32_t ta = taddr + ((uint32_t)(32 * q) << 16) + 8 * j;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                       "=r"(r[6]), "=r"(r[7])
                     : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 8; ++i) C[row * NMAX + 8 * j + i] = __uint_as_float(r[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(taddr));
}

int run(int mode) {
    std::vector<float> X(K * F), P(128 * 16), C(M * NMAX, -1.f);
    srand(7 + mode);
    for (auto &x : X) x = (float)((rand() % 17) - 8) / 4.f;
    for (auto &x : P) x = (float)((rand() % 9) - 4) / 2.f;
    float *dX, *dP, *dC;
    int *dS, st = 0;
    cudaMalloc(&dX, X.size() * 4);
    cudaMalloc(&dP, P.size() * 4);
    cudaMalloc(&dC, C.size() * 4);
    cudaMalloc(&dS, 4);
    cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dP, P.data(), P.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dS, 0, 4);
    const int smem = 65536 + 8192 + 1024;
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemset(dC, 0xff, C.size() * 4);
    k_probe<<<1, 128, smem>>>(dX, dP, dC, dS, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&st, dS, 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    int bad = 0;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < NMAX; ++j) {
            double ref = 0;
            if (i < F)
                for (int k = 0; k < K; ++k) ref += (double)X[k * F + i] * X[k * F + j];
            if (mode == 3 && j >= R0)
                for (int k = 0; k < 16; ++k) ref -= (double)P[i * 16 + k] * P[j * 16 + k];
            const double d = fabs(ref - C[i * NMAX + j]);
            if (d > maxerr) maxerr = d;
            if (d > 1e-3 && bad++ < 4) printf("  mismatch (%d,%d): got %g want %g\n", i, j, C[i * NMAX + j], ref);
        }
    printf("mode %d: cuda=%s timeout=%d max|err|=%g bad=%d\n", mode, cudaGetErrorString(e), st, maxerr, bad);
    cudaFree(dX); cudaFree(dP); cudaFree(dC); cudaFree(dS);
    return bad == 0 && st == 0 && e == cudaSuccess ? 0 : 1;
}

int main() {
    int rc = 0;
    for (int mode : {0, 1, 2, 3}) rc |= run(mode) << mode;
    printf("result mask %d (0 = all pass)\n", rc);
    return 0;
}
