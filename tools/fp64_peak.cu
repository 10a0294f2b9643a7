// fp64_peak.cu -- FP64 pipe microbenchmark (hard part 3: the
// competing bound of the force sweep).  Measures DFMA, IEEE sqrt and IEEE div
// throughput on the whole GPU with CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;

__global__ void dfma_kernel(double *out, int iters, double a, double b)
{
    double v[kChains];
#pragma unroll
    for (int k = 0; k < kChains; ++k) v[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < kChains; ++k) v[k] = fma(v[k], a, b);
    double s = 0;
#pragma unroll
    for (int k = 0; k < kChains; ++k) s += v[k];
    if (s == 12345.678) out[0] = s;
}

__global__ void dsqrt_kernel(double *out, int iters)
{
    double v[kChains];
#pragma unroll
    for (int k = 0; k < kChains; ++k) v[k] = 1.5 + threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < kChains; ++k) v[k] = sqrt(v[k]) + 1.25;
    double s = 0;
#pragma unroll
    for (int k = 0; k < kChains; ++k) s += v[k];
    if (s == 12345.678) out[0] = s;
}

__global__ void ddiv_kernel(double *out, int iters)
{
    double v[kChains];
#pragma unroll
    for (int k = 0; k < kChains; ++k) v[k] = 1.5 + threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < kChains; ++k) v[k] = 3.0 / v[k] + 1.25;
    double s = 0;
#pragma unroll
    for (int k = 0; k < kChains; ++k) s += v[k];
    if (s == 12345.678) out[0] = s;
}

__global__ void ffma_kernel(float *out, int iters, float a, float b)
{
    float v[kChains];
#pragma unroll
    for (int k = 0; k < kChains; ++k) v[k] = threadIdx.x * 1e-3f + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < kChains; ++k) v[k] = fmaf(v[k], a, b);
    float s = 0;
#pragma unroll
    for (int k = 0; k < kChains; ++k) s += v[k];
    if (s == 12345.678f) out[0] = s;
}

template <typename F>
static float time_it(F launch)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
}

int main()
{
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
    double *d;
    cudaMalloc(&d, 64);
    const double nthr = (double)blocks * threads * kChains * iters;
    float ms = time_it([&] { dfma_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7); });
    printf("{\"dfma_tflops\": %.2f, ", 2.0 * nthr / (ms * 1e-3) / 1e12);
    ms = time_it([&] { dsqrt_kernel<<<blocks, threads>>>(d, iters / 8); });
    printf("\"dsqrt_gops\": %.1f, ", nthr / 8 / (ms * 1e-3) / 1e9);
    ms = time_it([&] { ddiv_kernel<<<blocks, threads>>>(d, iters / 8); });
    printf("\"ddiv_gops\": %.1f, ", nthr / 8 / (ms * 1e-3) / 1e9);
    ms = time_it([&] { ffma_kernel<<<blocks, threads>>>((float *)d, iters, 0.999999f, 1e-7f); });
    printf("\"ffma_tflops\": %.2f, \"sms\": %d}\n", 2.0 * nthr / (ms * 1e-3) / 1e12,
           p.multiProcessorCount);
    return 0;
}
