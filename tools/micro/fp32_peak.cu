// FP32 CUDA-core peak on this GPU: FFMA2 (paired FP32 FMA, the instruction the
// Gram kernels issue) over independent register chains, one persistent CTA
// set covering every SM.  Prints one JSON line {"fp32_tflops": ..}.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_peak fp32_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void ffma2(float2 &d, float a, float bx, float by) {
    asm volatile("fma.rn.f32x2 %0, %1, %2, %0;"
                 : "+l"(*reinterpret_cast<unsigned long long *>(&d))
                 : "l"(((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint(a)),
                   "l"(((unsigned long long)__float_as_uint(by) << 32) | __float_as_uint(bx)));
}

template <int CH>
__global__ void k_peak(float *out, int iters, float a) {
    float2 acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
    const float bx = 0.999f, by = 1.001f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) ffma2(acc[c], a, bx, by);
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c].x + acc[c].y;
    if (s == 1234.5f) out[threadIdx.x] = s;   // keep the chains live
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    cudaMalloc(&out, 4096);
    constexpr int CH = 16;
    const int threads = 512, blocks = sms * 4, iters = 1 << 16;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_peak<CH><<<blocks, threads>>>(out, 1024, 1.0001f);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        k_peak<CH><<<blocks, threads>>>(out, iters, 1.0001f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * 2.0 * CH * (double)iters * threads * blocks;   // 2 FMA per FFMA2
    printf("{\"fp32_tflops\": %.2f, \"how\": \"FFMA2 chains, %d SMs x %d CTAs x %d threads, best of 5\"}\n",
           flops / (best * 1e-3) / 1e12, sms, 4, threads);
    return cudaGetLastError() != cudaSuccess;
}
