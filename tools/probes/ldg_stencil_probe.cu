// Probe: is a TMA-free stencil (128-bit LDG of the window straight into
// registers, 256-bit STG of 8 outputs) closer to the copy rate than the
// TMA load -> shared -> TMA store kernels at config 3's shape?
//   y[t] = sum_{j<7} x[t+j-3] * k[j], rows of L = 8192, 131072 rows (4 GiB).
// Variants: A = one thread per 8 outputs, window via 4 x LDG.128 (overlapping
// reads hit L1); B = the same with .L1::no_allocate / .cs streaming hints.
// Prints ms and GB/s (8 B per element) next to a plain float4 copy kernel.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ld4_nc(const float* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
template <bool CS = false>
__device__ __forceinline__ void st8(float* p, const float (&d)[8]) {
    if (CS)
        asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(d[0]), "f"(d[1]),
                     "f"(d[2]), "f"(d[3]), "f"(d[4]), "f"(d[5]), "f"(d[6]), "f"(d[7])
                     : "memory");
    else
        asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(d[0]), "f"(d[1]),
                     "f"(d[2]), "f"(d[3]), "f"(d[4]), "f"(d[5]), "f"(d[6]), "f"(d[7])
                     : "memory");
}

template <bool NC, bool CS = false>
__global__ void __launch_bounds__(256) stencil7(const float* __restrict__ x, const float* __restrict__ k,
                                                float* __restrict__ y, int64_t rows, int L) {
    const int64_t n8 = rows * (L / 8);
    float w[7];
    for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n8; i += int64_t(gridDim.x) * 256) {
        const int64_t row = i / (L / 8);
        const int t = static_cast<int>(i - row * (L / 8)) * 8;
        const int h = static_cast<int>(row % 512);
#pragma unroll
        for (int j = 0; j < 7; ++j) w[j] = __ldg(k + h * 7 + j);
        const float* xr = x + row * L;
        float v[16];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int s = t - 4 + 4 * c;
            float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
            if (s >= 0 && s < L) q = NC ? ld4_nc(xr + s) : ld4(xr + s);
            v[4 * c] = q.x;
            v[4 * c + 1] = q.y;
            v[4 * c + 2] = q.z;
            v[4 * c + 3] = q.w;
        }
        float d[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            float a = 0.f;
#pragma unroll
            for (int j = 0; j < 7; ++j) a = __fmaf_rn(v[r + j + 1], w[j], a);  // x[t+r+j-3] = v[r+j+1]
            d[r] = a;
        }
        st8<CS>(y + row * L + t, d);
    }
}

__global__ void copy4(const float4* __restrict__ a, float4* __restrict__ b, int64_t n4) {
    for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n4; i += int64_t(gridDim.x) * 256) b[i] = a[i];
}

int main() {
    const int64_t rows = 131072;
    const int L = 8192;
    const int64_t n = rows * L;
    float *x, *y, *k;
    cudaMalloc(&x, n * 4);
    cudaMalloc(&y, n * 4);
    cudaMalloc(&k, 512 * 7 * 4);
    cudaMemset(x, 0, n * 4);
    cudaMemset(k, 0, 512 * 7 * 4);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](const char* name, auto fn) {
        float best = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
            cudaEventRecord(a);
            fn();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep && ms < best) best = ms;
        }
        printf("%-28s %.4f ms  %.0f GB/s  (%s)\n", name, best, 8.0 * n / (best * 1e6),
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int per : {2, 3, 4, 5, 6, 8, 12, 16, 32}) {
        char nm[64];
        snprintf(nm, sizeof nm, "ldg stencil7 grid=%dx148", per);
        timeit(nm, [&] { stencil7<false><<<per * nsm, 256>>>(x, k, y, rows, L); });
        snprintf(nm, sizeof nm, "ldg st.cs stencil7 grid=%dx148", per);
        timeit(nm, [&] { stencil7<false, true><<<per * nsm, 256>>>(x, k, y, rows, L); });
    }
    {
        const int64_t nb = rows * (L / 8);
        timeit("ldg stencil7 grid=all", [&] { stencil7<false><<<(nb + 255) / 256, 256>>>(x, k, y, rows, L); });
    }
    timeit("copy float4 grid=8x148", [&] { copy4<<<8 * nsm, 256>>>((const float4*)x, (float4*)y, n / 4); });
    timeit("cudaMemcpy d2d", [&] { cudaMemcpyAsync(y, x, n * 4, cudaMemcpyDeviceToDevice); });
    return 0;
}
