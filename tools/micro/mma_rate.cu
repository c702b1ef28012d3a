// Throughput probe: legacy warp-level mma.sync m16n8k8 tf32 and FFMA2 on
// sm_100a (independent accumulator chains, no memory traffic).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_mma(float *out, int iters) {
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    float c[8][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_mma_bf16(float *out, int iters) {
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    float c[8][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float *out, int iters) {
    float2 c[16];
    for (int j = 0; j < 16; ++j) c[j] = make_float2(threadIdx.x * j, j);
    const float a = threadIdx.x * 1e-3f;
    const float bx = 0.999f, by = 1.001f;
    unsigned long long A, B;
    asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a));
    asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(bx), "f"(by));
    unsigned long long C[16];
    for (int j = 0; j < 16; ++j) asm("mov.b64 %0, {%1, %2};" : "=l"(C[j]) : "f"(c[j].x), "f"(c[j].y));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C[j]) : "l"(A), "l"(B));
    }
    float s = 0;
    for (int j = 0; j < 16; ++j) {
        float x, y;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(C[j]));
        s += x + y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float *out;
    cudaMalloc(&out, 148 * 16 * 1024 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int warps : {4, 8, 16, 32}) {
        const int blocks = 148 * 2, threads = warps * 16;  // 2 CTAs per SM
        k_mma<<<blocks, threads>>>(out, 16);
        cudaEventRecord(e0);
        k_mma<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 16 * 8 * 8 * 8.0 * iters * (blocks * threads / 32);
        printf("mma.sync tf32 m16n8k8: %2d warps/SM: %.1f TFLOP/s\n", warps, flops / ms / 1e9);
        k_mma_bf16<<<blocks, threads>>>(out, 16);
        cudaEventRecord(e0);
        k_mma_bf16<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flops = 2.0 * 16 * 8 * 16 * 8.0 * iters * (blocks * threads / 32);
        printf("mma.sync bf16 m16n8k16: %2d warps/SM: %.1f TFLOP/s\n", warps, flops / ms / 1e9);
        k_ffma2<<<blocks, threads>>>(out, 16);
        cudaEventRecord(e0);
        k_ffma2<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flops = 2.0 * 2 * 16.0 * iters * blocks * threads;
        printf("ffma2: %2d warps/SM: %.1f TFLOP/s\n", warps, flops / ms / 1e9);
    }
    return 0;
}
