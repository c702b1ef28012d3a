// Probe: TMA tile::gather4 of rows of an fp16 table (SWIZZLE_128B tensor map,
// box {64, 1}) lands in the MN-major SWIZZLE_128B canonical layout that
// tcgen05.mma kind::f16 reads: K = 16 gathered rows (ratings) x 128 features
// (2 atoms of 64), Gram C = X^T X with both operands from that tile.
// Checked against the CPU.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
#include <cudaTypedefs.h>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint64_t layout) {
    return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46) | (layout << 61);
}

constexpr int F = 112, FT = 128, K = 32, N = 112, NROWS = 1000;

__global__ void k_probe(const __grid_constant__ CUtensorMap map, const int *rows, float *C, int *status) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) unsigned long long bar_tma, bar_mma;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_tma)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_mma)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // tile: k-group g (8 rows) x atom a (64 features): 1 KB at g*2048 + a*1024
    if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar_tma)),
                     "r"(K * FT * 2) : "memory");
        for (int q = 0; q < K / 4; ++q)          // 4 rows per gather4
            for (int a = 0; a < 2; ++a) {
                const uint32_t dst = smem_u32(smem) + (q >> 1) * 2048 + a * 1024 + (q & 1) * 512;
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
                    "l"(&map), "r"(64 * a), "r"(rows[4 * q]), "r"(rows[4 * q + 1]), "r"(rows[4 * q + 2]),
                    "r"(rows[4 * q + 3]), "r"(smem_u32(&bar_tma))
                    : "memory");
            }
    }
    {
        uint32_t done = 0;
        for (long it = 0; it < (1l << 26) && !done; ++it)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"(smem_u32(&bar_tma)) : "memory");
        if (!done && lane == 0) atomicExch(status, 1);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t taddr = tbase;
    if (tid == 0) {
        const uint32_t id = (1u << 4) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
        for (int kk = 0; kk < K / 16; ++kk) {
            const uint64_t d = sdesc(smem_u32(smem) + kk * 2 * 2048, 1024, 2048, 2);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(taddr),
                         "l"(d), "l"(d), "r"(id), "r"((uint32_t)(kk > 0)));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(smem_u32(&bar_mma)) : "memory");
    }
    {
        uint32_t done = 0;
        for (long it = 0; it < (1l << 26) && !done; ++it)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"(smem_u32(&bar_mma)) : "memory");
        if (!done && lane == 0) atomicExch(status, 2);
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = 32 * (warp & 3) + lane;
    for (int j = 0; j < N / 8; ++j) {
        uint32_t r[8];
        const uint32_t ta = taddr + ((uint32_t)(32 * (warp & 3)) << 16) + 8 * j;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                       "=r"(r[6]), "=r"(r[7])
                     : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 8; ++i) C[row * N + 8 * j + i] = __uint_as_float(r[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(taddr));
}

int main() {
    std::vector<__half> T((size_t)NROWS * FT);
    std::vector<float> Tf((size_t)NROWS * FT);
    srand(3);
    for (int r = 0; r < NROWS; ++r)
        for (int f = 0; f < FT; ++f) {
            const float v = f < F ? (float)((rand() % 17) - 8) / 4.f : 0.f;
            T[(size_t)r * FT + f] = __float2half(v);
            Tf[(size_t)r * FT + f] = v;
        }
    int rows[K];
    for (int k = 0; k < K; ++k) rows[k] = (k * 37 + 11) % NROWS;
    __half *dT;
    int *dR, *dS, st = 0;
    float *dC;
    cudaMalloc(&dT, T.size() * 2);
    cudaMalloc(&dR, sizeof(rows));
    cudaMalloc(&dC, 128 * N * 4);
    cudaMalloc(&dS, 4);
    cudaMemcpy(dT, T.data(), T.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dR, rows, sizeof(rows), cudaMemcpyHostToDevice);
    cudaMemset(dS, 0, 4);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
    CUtensorMap map;
    cuuint64_t dims[2] = {FT, NROWS}, strides[1] = {FT * 2};
    cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
    CUresult cr = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn)(
        &map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, dT, dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)cr);
    int *hrows = rows;
    // rows are passed by value through device memory copy in kernel args: use host array via __constant? simpler: kernel reads dR
    (void)hrows;
    const int smem = K * FT * 2 + 2048;
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_probe<<<1, 128, smem>>>(map, dR, dC, dS);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> C(128 * N);
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&st, dS, 4, cudaMemcpyDeviceToHost);
    double mx = 0;
    int bad = 0;
    for (int i = 0; i < F; ++i)
        for (int j = 0; j < N; ++j) {
            double ref = 0;
            for (int k = 0; k < K; ++k) ref += (double)Tf[(size_t)rows[k] * FT + i] * Tf[(size_t)rows[k] * FT + j];
            const double d = fabs(ref - C[i * N + j]);
            mx = d > mx ? d : mx;
            if (d > 1e-3 && bad++ < 4) printf("  (%d,%d) got %g want %g\n", i, j, C[i * N + j], ref);
        }
    printf("gather4 + SW128 MN-major Gram: cuda=%s status=%d max|err|=%g bad=%d -> %s\n",
           cudaGetErrorString(e), st, mx, bad, (bad == 0 && st == 0 && e == cudaSuccess) ? "PASS" : "FAIL");
    return 0;
}
