// Probe: what HBM3e streams at for the read:write mixes of this library's
// kernels -- the roofline each HBM-bound path is judged against.
//   read-only  (dW: read gy, x)                  sum of 2 arrays
//   1:1 copy   (fwd / dX: read x, write y)       y = x
//   2:1 triad  (fused backward: read gy, x, write dx)   z = x + y
// Each with 256-bit (v8.f32) global accesses, one 32-byte sector per thread per
// access, a grid-stride loop over 4 GiB arrays (>> L2), CUDA-event timed.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld8(const float* p, float (&v)[8]) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
}
__device__ __forceinline__ void st8(float* p, const float (&v)[8]) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]),
                 "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}

template <int MODE>  // 0 read-only, 1 copy, 2 triad
__global__ void __launch_bounds__(256) stream(const float* __restrict__ x, const float* __restrict__ y,
                                              float* __restrict__ z, size_t n8, float* sink) {
    float acc = 0.f;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n8; i += size_t(gridDim.x) * blockDim.x) {
        float a[8], b[8];
        ld8(x + 8 * i, a);
        if (MODE != 1) ld8(y + 8 * i, b);
        if (MODE == 0) {
#pragma unroll
            for (int k = 0; k < 8; ++k) acc += a[k] + b[k];
        } else if (MODE == 1) {
            st8(z + 8 * i, a);
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] += b[k];
            st8(z + 8 * i, a);
        }
    }
    if (MODE == 0 && acc == 12345.f) *sink = acc;
}

int main() {
    const size_t n = size_t(1) << 30;  // 4 GiB per array
    float *x, *y, *z, *sink;
    cudaMalloc(&x, n * 4); cudaMalloc(&y, n * 4); cudaMalloc(&z, n * 4); cudaMalloc(&sink, 4);
    cudaMemset(x, 0, n * 4); cudaMemset(y, 0, n * 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    const char* names[3] = {"read-only 2 arrays", "copy 1:1", "triad 2:1"};
    const double bytes[3] = {8.0 * n, 8.0 * n, 12.0 * n};
    for (int mode = 0; mode < 3; ++mode)
        for (int g : {sms * 4, sms * 8, sms * 16}) {
            auto k = mode == 0 ? stream<0> : mode == 1 ? stream<1> : stream<2>;
            float best = 1e30f;
            for (int rep = 0; rep < 6; ++rep) {
                cudaEventRecord(s);
                k<<<g, 256>>>(x, y, z, n / 8, sink);
                cudaEventRecord(e);
                cudaEventSynchronize(e);
                float ms; cudaEventElapsedTime(&ms, s, e);
                if (rep >= 1 && ms < best) best = ms;
            }
            printf("%-20s grid %5d  %8.3f ms  %7.1f GB/s\n", names[mode], g, best, bytes[mode] / best * 1e-6);
        }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
