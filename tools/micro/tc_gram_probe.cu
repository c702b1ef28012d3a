// Probe of the tcgen05 mechanics the wide-path Gram needs (sm_100a):
// X (K ratings x F features, fp32 values exact in tf32) staged in shared
// memory in the MN-major no-swizzle canonical layout (core matrix = 8 K rows
// x 16 B, MN chunks SBO = 128 B apart, 8-K groups LBO apart); C = X^T X by
// tcgen05.mma kind::tf32 with BOTH operands MN-major from the same tile;
// accumulator read back with tcgen05.ld 32x32b.  Checks M = 128 (N = 112)
// and M = 64 (N = 56) against the CPU.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint64_t layout = 0) {
    return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46) | (layout << 61);   // version 1
}
template <int M, int N>
__device__ __forceinline__ uint32_t idesc_tf32_mn() {
    return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

template <int M, int N, int F, int K>
__global__ void k_probe(const float *X, float *C, int *status, int mode) {
    constexpr int CH = F / 4;            // 16-byte chunks per rating row
    constexpr int KG = K / 8;
    constexpr int LBO = CH * 128;
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ uint32_t tbase;
    float *xs = reinterpret_cast<float *>(smem);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // stage: element (k, f) -> (k/8)*LBO + (f/4)*128 + (k%8)*16 + (f%4)*4 bytes
    for (int e = tid; e < 8192 + 1024; e += blockDim.x) xs[e] = 0.f;   // data + over-read slack
    __syncthreads();
    // K-major: element (f, k) -> (f/8)*SBOK + (f%8)*16 + (k/4)*128*... see below
    constexpr int KCH = K / 4;                     // 16-byte chunks along K
    constexpr int KTILE = 16384;                   // byte offset of the K-major copy (modes 4, 5)
    for (int e = tid; e < K * F; e += blockDim.x) {
        const int k = e / F, f = e % F;
        if (mode >= 4) {   // both layouts: MN tile at xs, K tile at xs + KTILE
            xs[((k >> 3) * LBO + (f >> 2) * 128 + (k & 7) * 16) / 4 + (f & 3)] = X[e];
            xs[KTILE / 4 + ((k >> 2) * (F / 8) * 128 + (f >> 3) * 128 + (f & 7) * 16) / 4 + (k & 3)] = X[e];
        } else if (mode == 3) {   // SW128 MN-major: atom 8 k-rows x 128 B (32 f), 16-B chunk ^= row
            const int n = f >> 5, c = (f & 31) >> 2, r = k & 7;
            xs[((k >> 3) * 4096 + n * 1024 + r * 128 + ((c ^ r) << 4)) / 4 + (f & 3)] = X[e];
        } else if (mode < 2)
            xs[((k >> 3) * LBO + (f >> 2) * 128 + (k & 7) * 16) / 4 + (f & 3)] = X[e];
        else   // core matrix = 8 f-rows x 16 B (4 k); f-groups SBO = 128 B apart; k chunks LBO = (F/8)*128 apart
            xs[((k >> 2) * (F / 8) * 128 + (f >> 3) * 128 + (f & 7) * 16) / 4 + (k & 3)] = X[e];
    }
    (void)KCH;
    // zero the over-read slack (A reads M/4 chunks per k-group)

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
        uint32_t id = (mode < 2 || mode == 3) ? idesc_tf32_mn<M, N>() : (idesc_tf32_mn<M, N>() & ~((1u << 15) | (1u << 16)));
        if (mode == 4) id |= 1u << 15;   // A MN-major
        if (mode == 5) id |= 1u << 16;   // B MN-major
        for (int kg = 0; kg < KG; ++kg) {
            uint64_t da, db;
            if (mode == 0) {
                const uint32_t a = smem_u32(xs) + kg * LBO;
                da = db = sdesc(a, LBO, 128);
            } else if (mode == 1) {
                const uint32_t a = smem_u32(xs) + kg * LBO;
                da = db = sdesc(a, 128, LBO);
            } else if (mode == 4 || mode == 5) {
                const uint64_t dmn = sdesc(smem_u32(xs) + kg * LBO, LBO, 128);
                const uint64_t dk = sdesc(smem_u32(xs) + KTILE + kg * 2 * (F / 8) * 128, (F / 8) * 128, 128);
                da = mode == 4 ? dmn : dk;
                db = mode == 4 ? dk : dmn;
            } else if (mode == 3) {
                const uint32_t a = smem_u32(xs) + kg * 4096;
                da = db = sdesc(a, 1024, 4096, 2);
            } else {
                const uint32_t a = smem_u32(xs) + kg * 2 * (F / 8) * 128;   // 8 k = 2 chunks
                da = db = sdesc(a, (F / 8) * 128, 128);
            }
            const uint32_t acc = kg > 0;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                ::"r"(taddr), "l"(da), "l"(db), "r"(id), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(smem_u32(&bar)) : "memory");
    }
    // wait (bounded)
    {
        uint32_t done = 0;
        for (long it = 0; it < (1l << 26) && !done; ++it)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
        if (!done && lane == 0) atomicExch(status, 1);
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // read back: warp w reads TMEM lanes 32(w%4)..; row mapping depends on M
    const int q = warp & 3;
    const int row = M == 128 ? 32 * q + lane : (lane < 16 ? 16 * q + lane : -1);
    for (int j = 0; j < N / 8; ++j) {
        uint32_t r[8];
        const uint32_t ta = taddr + ((uint32_t)(32 * q) << 16) + 8 * j;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                       "=r"(r[6]), "=r"(r[7])
                     : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row >= 0)
            for (int i = 0; i < 8; ++i) C[row * N + 8 * j + i] = __uint_as_float(r[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(taddr));
}

template <int M, int N, int F, int K>
int run(int mode) {
    std::vector<float> X(K * F), C(M * N, -1.f);
    srand(7);
    for (auto &x : X) x = (float)((rand() % 17) - 8) / 4.f;   // exact in tf32
    float *dX, *dC;
    int *dS, st = 0;
    cudaMalloc(&dX, X.size() * 4);
    cudaMalloc(&dC, C.size() * 4);
    cudaMalloc(&dS, 4);
    cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dS, 0, 4);
    const int smem = 16384 + 16384 + 8192;
    cudaFuncSetAttribute(k_probe<M, N, F, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemset(dC, 0xff, C.size() * 4);
    k_probe<M, N, F, K><<<1, 128, smem>>>(dX, dC, dS, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&st, dS, 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    int bad = 0;
    const int rows = M == 128 ? F : (F < 64 ? F : 64);
    for (int i = 0; i < rows && i < M; ++i)
        for (int j = 0; j < N && j < F; ++j) {
            double ref = 0;
            for (int k = 0; k < K; ++k) ref += (double)X[k * F + i] * X[k * F + j];
            const double d = fabs(ref - C[i * N + j]);
            if (d > maxerr) maxerr = d;
            if (d > 1e-3 && bad++ < 5) printf("  mismatch (%d,%d): got %g want %g\n", i, j, C[i * N + j], ref);
        }
    printf("mode %d: M=%d N=%d F=%d K=%d: cuda=%s timeout=%d max|err|=%g bad=%d\n", mode, M, N, F, K,
           cudaGetErrorString(e), st, maxerr, bad);
    return bad == 0 && st == 0 && e == cudaSuccess ? 0 : 1;
}

int main() {
    int rc = 0;
    for (int mode : {0, 2, 4, 5}) {
        rc |= run<128, 112, 112, 32>(mode);
    }
    printf(rc ? "FAIL\n" : "PASS\n");
    return rc;
}
