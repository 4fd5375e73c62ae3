// Probe: can one TMA load produce the 36-per-32 padded shared layout directly?
// 4-D view {4 floats, 8 quads, L/32 rows, R tensor rows} of a [R, L] fp32
// tensor with box {4, 9, n, 1}: quad 8 of every 32-float row lies outside
// dim 1 (extent 8) and must come back zero-filled.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void probe(const __grid_constant__ CUtensorMap map, float* out, int n, int r0, int row) {
    __shared__ __align__(128) float buf[9 * 4 * 16];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)),
                     "r"(n * 144));
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
                (unsigned)__cvta_generic_to_shared(buf)),
            "l"(&map), "r"(0), "r"(0), "r"(r0), "r"(row), "r"((unsigned)__cvta_generic_to_shared(&bar))
            : "memory");
        asm volatile(
            "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
                (unsigned)__cvta_generic_to_shared(&bar)));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n * 36; i += blockDim.x) out[i] = buf[i];
}

int main() {
    const int R = 3, L = 128, n = 6;
    float* h = new float[R * L];
    for (int i = 0; i < R * L; ++i) h[i] = 1.f + i;
    float *d, *o;
    cudaMalloc(&d, R * L * 4);
    cudaMalloc(&o, n * 36 * 4);
    cudaMemcpy(d, h, R * L * 4, cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap map;
    const cuuint64_t dims[4] = {4, 8, (cuuint64_t)L / 32, (cuuint64_t)R};
    const cuuint64_t strides[3] = {16, 128, (cuuint64_t)L * 4};
    const cuuint32_t box[4] = {4, 9, (cuuint32_t)n, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = ((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)r);
    if (r != CUDA_SUCCESS) return 1;
    // rows -1 .. 4 of tensor row 1: row -1 and row 4 are outside (zero)
    probe<<<1, 128>>>(map, o, n, -1, 1);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    float out[n * 36];
    cudaMemcpy(out, o, sizeof(out), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int rr = 0; rr < n; ++rr)
        for (int c = 0; c < 36; ++c) {
            const int lr = rr - 1;  // logical 32-row
            float want = 0.f;
            if (c < 32 && lr >= 0 && lr < L / 32) want = h[1 * L + lr * 32 + c];
            if (out[rr * 36 + c] != want) {
                if (bad < 10) printf("mismatch row %d col %d: got %g want %g\n", rr, c, out[rr * 36 + c], want);
                ++bad;
            }
        }
    printf("padded TMA probe: %s (%d mismatches)\n", bad ? "FAIL" : "OK", bad);
    return bad != 0;
}
