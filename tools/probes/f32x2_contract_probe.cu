// Probe: does ptxas keep mul.rn.f32x2 followed by add.rn.f32x2 as two
// roundings (FMUL2 + FADD2), as PTX's .rn promises, or contract the pair into
// one FFMA2?  The SASS of this file (cuobjdump -sass) shows a single FFMA2 for
// variant A even with --fmad=false; this run counts the bit differences
// against scalar __fadd_rn(acc, __fmul_rn(x, w)) on random data.  Variant B
// adds the product through fma.rn.f32x2(p, one, acc) with `one` a runtime
// kernel argument: ptxas cannot fold the multiply into that (FMUL2 + FFMA2 in
// the SASS), and p * 1 + acc rounds once, like the scalar add.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk(unsigned long long v, float& lo, float& hi) {
    asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}

__global__ void k(const float* x, const float* w, const float* acc, float* ref, float* a_out, float* b_out, int n,
                  float one) {
    const int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (i + 1 >= n) return;
    ref[i] = __fadd_rn(acc[i], __fmul_rn(x[i], w[i]));
    ref[i + 1] = __fadd_rn(acc[i + 1], __fmul_rn(x[i + 1], w[i + 1]));
    const unsigned long long X = pk(x[i], x[i + 1]), W = pk(w[i], w[i + 1]), A = pk(acc[i], acc[i + 1]);
    unsigned long long p, s;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"(X), "l"(W));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s) : "l"(A), "l"(p));
    upk(s, a_out[i], a_out[i + 1]);
    const unsigned long long ONE = pk(one, one);
    unsigned long long q, t = A;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(q) : "l"(X), "l"(W));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(t) : "l"(q), "l"(ONE));
    upk(t, b_out[i], b_out[i + 1]);
}

int main() {
    const int n = 1 << 22;
    float *hx = new float[n], *hw = new float[n], *ha = new float[n];
    uint64_t s = 0x9E3779B97F4A7C15ull;
    auto rnd = [&]() {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        return static_cast<float>(static_cast<int64_t>(s >> 11) - (int64_t(1) << 52)) * (1.0f / 4503599627370496.0f);
    };
    for (int i = 0; i < n; ++i) { hx[i] = rnd(); hw[i] = rnd(); ha[i] = rnd(); }
    float *x, *w, *a, *r, *o1, *o2;
    cudaMalloc(&x, n * 4); cudaMalloc(&w, n * 4); cudaMalloc(&a, n * 4);
    cudaMalloc(&r, n * 4); cudaMalloc(&o1, n * 4); cudaMalloc(&o2, n * 4);
    cudaMemcpy(x, hx, n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(w, hw, n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(a, ha, n * 4, cudaMemcpyHostToDevice);
    k<<<n / 2 / 256, 256>>>(x, w, a, r, o1, o2, n, 1.0f);
    uint32_t *hr = new uint32_t[n], *h1 = new uint32_t[n], *h2 = new uint32_t[n];
    cudaMemcpy(hr, r, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h1, o1, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2, o2, n * 4, cudaMemcpyDeviceToHost);
    size_t d1 = 0, d2 = 0;
    for (int i = 0; i < n; ++i) { d1 += hr[i] != h1[i]; d2 += hr[i] != h2[i]; }
    printf("A mul.rn.f32x2 + add.rn.f32x2 vs scalar two-rounding: %zu of %d differ\n", d1, n);
    printf("B mul.rn.f32x2 + fma.rn.f32x2(p, one, acc):          %zu of %d differ (%s)\n", d2, n,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
