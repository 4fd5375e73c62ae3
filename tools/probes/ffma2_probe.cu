// Probe: FP32 FMA throughput of FFMA (scalar) vs FFMA2 (fma.rn.f32x2, sm_100a
// packed pairs, one operand a broadcast scalar) on all SMs.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}

template <int N>
__global__ void ffma(float* out, float a, float b, int iters) {
    float acc[N];
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < N; ++i) acc[i] = fmaf(acc[i], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < N; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int N>  // N pairs
__global__ void ffma2(float* out, float a, float b, int iters) {
    unsigned long long acc[N];
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = pk(threadIdx.x * 1e-3f + i, i + 0.5f);
    const unsigned long long bb = pk(b, b);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < N; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(pk(a, a)), "l"(bb));
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        float lo, hi;
        asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[i]));
        s += lo + hi;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 4, threads = 256, iters = 20000;
    float* out;
    cudaMalloc(&out, blocks * threads * 4);
    cudaEvent_t s, e;
    cudaEventCreate(&s);
    cudaEventCreate(&e);
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        ffma<16><<<blocks, threads>>>(out, 0.999f, 0.001f, iters);
        cudaEventRecord(s);
        ffma<16><<<blocks, threads>>>(out, 0.999f, 0.001f, iters);
        cudaEventRecord(e);
        cudaEventSynchronize(e);
        cudaEventElapsedTime(&ms, s, e);
        const double fl = 2.0 * 16 * iters * double(blocks) * threads;
        printf("FFMA  : %.1f TFLOP/s\n", fl / ms / 1e9);
        ffma2<8><<<blocks, threads>>>(out, 0.999f, 0.001f, iters);
        cudaEventRecord(s);
        ffma2<8><<<blocks, threads>>>(out, 0.999f, 0.001f, iters);
        cudaEventRecord(e);
        cudaEventSynchronize(e);
        cudaEventElapsedTime(&ms, s, e);
        printf("FFMA2 : %.1f TFLOP/s (same FMA count)\n", fl / ms / 1e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
