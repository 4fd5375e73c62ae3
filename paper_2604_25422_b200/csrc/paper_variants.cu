// paper_variants.cu -- the paper's four CUDA kernel designs, as real sm_100a
// kernels, for the controlled B200 ablation.
//
// The reference ships these only as prose and as an
// analytical mirror (src/exec_model.cpp:80-135, constants
// include/kernelscope/exec_model.hpp:29-36).  Each kernel below follows that
// launch geometry and thread->element mapping exactly:
//
//   variant    fwd / dX mapping                                    dW
//   naive      grid (ceil(L/512), H, B) x 512, one output/thread    one thread per (h,j), sequential
//              (exec_model.cpp:93-95, :107-112)                     over B*L (:82-86)
//   coalesced  TTILE=32 x HTILE=8 tile, grid (ceil(L/32),           B*L split into 64 chunks per
//              ceil(H/8), B) x 256 (:96-98, :114-120)               channel, warp-shuffle partials,
//                                                                   second stage (:87-90)
//   shared     TPB=256 outputs per block with a TPB+K-1 halo tile   same two-stage split, chunk
//              in shared memory, s = b*H+h flattened (:99-100)      staged in shared memory
//   warp       one warp per (b,h), lanes t = lane + 32*i, the row   same two-stage split, warp then
//              and taps in shared memory (:101-102, :130-135)       block reduction
//
// fwd / dX accumulate taps in ascending j from +0 like the reference, so all
// four variants are bit-identical to conv::forward / backward_input; naive dW
// is bit-identical to the Sequential scheme.  The shared variant's grid puts
// the flattened s = b*H+h on the x axis (B*H exceeds CUDA's 65535 limit for
// grid.y at the paper's shape).
#include <algorithm>

#include "ks_common.cuh"

namespace ks {

namespace {

constexpr int kNaiveThreads = 512;
constexpr int kTTile = 32, kHTile = 8, kCoalThreads = 256;
constexpr int kTpb = 256;
constexpr int kChunks = 64;  // kBwdkChunkCount

// One output of the stencil over global memory, taps in [j_lo, j_hi) ascending
// (src/conv_core.cpp:35-40 / 64-69).
template <bool FUSED>
__device__ __forceinline__ float stencil_point(const float* __restrict__ rin, const float* __restrict__ kr, int L,
                                               int K, int off, int reverse, int t) {
    const int j_lo = max(0, off - t);
    const int j_hi = min(K, L + off - t);
    float acc = 0.f;
    for (int j = j_lo; j < j_hi; ++j) acc = muladd<FUSED>(acc, rin[t + j - off], kr[reverse ? K - 1 - j : j]);
    return acc;
}

template <bool FUSED>
__global__ void __launch_bounds__(kNaiveThreads)
naive_stencil(const float* __restrict__ in, const float* __restrict__ k, float* __restrict__ out, int H, int L,
              int K, int off, int reverse) {
    const int b = blockIdx.z, h = blockIdx.y;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= L) return;
    const int64_t row = static_cast<int64_t>(b) * H + h;
    out[row * L + t] = stencil_point<FUSED>(in + row * L, k + static_cast<int64_t>(h) * K, L, K, off, reverse, t);
}

template <bool FUSED>
__global__ void __launch_bounds__(kCoalThreads)
coalesced_stencil(const float* __restrict__ in, const float* __restrict__ k, float* __restrict__ out, int H, int L,
                  int K, int off, int reverse) {
    const int t = blockIdx.x * kTTile + threadIdx.x % kTTile;
    const int h = blockIdx.y * kHTile + threadIdx.x / kTTile;
    const int b = blockIdx.z;
    if (t >= L || h >= H) return;
    const int64_t row = static_cast<int64_t>(b) * H + h;
    out[row * L + t] = stencil_point<FUSED>(in + row * L, k + static_cast<int64_t>(h) * K, L, K, off, reverse, t);
}

template <bool FUSED>
__global__ void __launch_bounds__(kTpb)
shared_stencil(const float* __restrict__ in, const float* __restrict__ k, float* __restrict__ out, int H, int L,
               int K, int off, int reverse, int tiles) {
    extern __shared__ float sm[];
    float* tile = sm;              // TPB + K - 1 input values (zero halo)
    float* sk = sm + kTpb + K - 1;  // K taps
    const int64_t s = blockIdx.x / tiles;  // flattened b*H + h
    const int t0 = static_cast<int>(blockIdx.x - s * tiles) * kTpb;
    const int h = static_cast<int>(s % H);
    const float* rin = in + s * L;
    for (int i = threadIdx.x; i < kTpb + K - 1; i += kTpb) {
        const int q = t0 + i - off;
        tile[i] = (q >= 0 && q < L) ? rin[q] : 0.f;
    }
    for (int j = threadIdx.x; j < K; j += kTpb) sk[j] = k[static_cast<int64_t>(h) * K + (reverse ? K - 1 - j : j)];
    __syncthreads();
    const int t = t0 + threadIdx.x;
    if (t >= L) return;
    float acc = 0.f;
    // taps in ascending j; the zero halo entries are exact no-ops (+-0)
    for (int j = 0; j < K; ++j) acc = muladd<FUSED>(acc, tile[threadIdx.x + j], sk[j]);
    out[s * L + t] = acc;
}

template <bool FUSED>
__global__ void __launch_bounds__(32)
warp_stencil(const float* __restrict__ in, const float* __restrict__ k, float* __restrict__ out, int H, int L,
             int K, int off, int reverse) {
    extern __shared__ float sm[];
    float* sx = sm;      // the whole row
    float* sk = sm + L;  // taps
    const int b = blockIdx.x, h = blockIdx.y, lane = threadIdx.x;
    const int64_t row = static_cast<int64_t>(b) * H + h;
    for (int i = lane; i < L; i += 32) sx[i] = in[row * L + i];
    for (int j = lane; j < K; j += 32) sk[j] = k[static_cast<int64_t>(h) * K + (reverse ? K - 1 - j : j)];
    __syncwarp();
    for (int t = lane; t < L; t += 32) {
        const int j_lo = max(0, off - t);
        const int j_hi = min(K, L + off - t);
        float acc = 0.f;
        for (int j = j_lo; j < j_hi; ++j) acc = muladd<FUSED>(acc, sx[t + j - off], sk[j]);
        out[row * L + t] = acc;
    }
}

// naive dW: one thread per (h,j), sequential over the flat B*L domain
// (= reduce_sequential, src/conv_core.cpp:98-111).
template <bool FUSED>
__global__ void __launch_bounds__(kNaiveThreads)
naive_dw(const float* __restrict__ gy, const float* __restrict__ x, float* __restrict__ dk, int B, int H, int L,
         int K) {
    const int h = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= K) return;
    const int d = j - K / 2;
    const int t_lo = max(0, -d), t_hi = min(L, L - d);
    float acc = 0.f;
    for (int b = 0; b < B; ++b) {
        const int64_t row = (static_cast<int64_t>(b) * H + h) * L;
        for (int t = t_lo; t < t_hi; ++t) acc = muladd<FUSED>(acc, gy[row + t], x[row + t + d]);
    }
    dk[static_cast<int64_t>(h) * K + j] = acc;
}

// Two-stage dW of the coalesced / shared / warp variants: block (chunk c, h)
// reduces its 1/64 of the flat B*L domain for every tap: per-thread strided
// partials, warp shuffle, block pass, partial[c][h][j].  STAGE_SMEM stages the
// chunk (gy and the x window) in shared memory first (shared / warp variants).
template <bool STAGE_SMEM, bool FUSED>
__global__ void __launch_bounds__(256)
twostage_dw(const float* __restrict__ gy, const float* __restrict__ x, float* __restrict__ part, int B, int H,
            int L, int K, int64_t span) {
    extern __shared__ float sm[];
    __shared__ float red[8];
    const int c = blockIdx.x, h = blockIdx.y;
    const int64_t n = static_cast<int64_t>(B) * L;
    const int64_t f0 = c * span, f1 = std::min<int64_t>(f0 + span, n);
    const int p = K / 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // staged slice: flat [f0, f1) of gy, and for x the same positions; the
    // taps reach t+d inside the same row, read from global when out of the slice
    if (STAGE_SMEM) {
        for (int64_t f = f0 + tid; f < f1; f += 256) {
            const int64_t b = f / L, t = f - b * L;
            const int64_t off = (b * H + h) * L + t;
            sm[f - f0] = gy[off];
            sm[span + (f - f0)] = x[off];
        }
        __syncthreads();
    }
    for (int j = 0; j < K; ++j) {
        const int d = j - p;
        float acc = 0.f;
        for (int64_t f = f0 + tid; f < f1; f += 256) {
            const int64_t b = f / L, t = f - b * L;
            if (t + d < 0 || t + d >= L) continue;
            const int64_t off = (b * H + h) * L + t;
            float g, xv;
            if (STAGE_SMEM) {
                g = sm[f - f0];
                const int64_t fx = f + d;
                xv = (fx >= f0 && fx < f1) ? sm[span + (fx - f0)] : x[off + d];
            } else {
                g = gy[off];
                xv = x[off + d];
            }
            acc = muladd<FUSED>(acc, g, xv);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) red[warp] = acc;
        __syncthreads();
        if (tid == 0) {
            float s = 0.f;
            for (int w = 0; w < 8; ++w) s += red[w];
            part[(static_cast<int64_t>(c) * H + h) * K + j] = s;
        }
        __syncthreads();
    }
}

__global__ void sum_chunks(const float* __restrict__ part, float* __restrict__ dk, int64_t HK) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= HK) return;
    float s = 0.f;
    for (int c = 0; c < kChunks; ++c) s += part[c * HK + i];
    dk[i] = s;
}

template <bool FUSED>
ks_status run(int variant, int path, const float* a, const float* b, float* out, int64_t B, int64_t H, int64_t L,
              int64_t K, void* ws, cudaStream_t st) {
    const int Bi = static_cast<int>(B), Hi = static_cast<int>(H), Li = static_cast<int>(L), Ki = static_cast<int>(K);
    if (path == 0 || path == 1) {
        const int off = path == 0 ? Ki / 2 : Ki - 1 - Ki / 2;
        const int rev = path == 1;
        switch (variant) {
            case 0: {
                const dim3 grid((Li + kNaiveThreads - 1) / kNaiveThreads, Hi, Bi);
                launch_kernel(naive_stencil<FUSED>, grid, kNaiveThreads, 0, st, a, b, out, Hi, Li, Ki, off, rev);
                break;
            }
            case 1: {
                const dim3 grid((Li + kTTile - 1) / kTTile, (Hi + kHTile - 1) / kHTile, Bi);
                launch_kernel(coalesced_stencil<FUSED>, grid, kCoalThreads, 0, st, a, b, out, Hi, Li, Ki, off, rev);
                break;
            }
            case 2: {
                const int tiles = (Li + kTpb - 1) / kTpb;
                const size_t smem = sizeof(float) * (kTpb + 2 * Ki - 1);
                cudaFuncSetAttribute(shared_stencil<FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(std::min<size_t>(smem, 227 * 1024)));
                launch_kernel(shared_stencil<FUSED>, static_cast<unsigned>(B * H * tiles), kTpb, smem, st, a, b, out, Hi, Li,
                                                                                               Ki, off, rev, tiles);
                break;
            }
            default: {
                const size_t smem = sizeof(float) * (L + K);
                cudaFuncSetAttribute(warp_stencil<FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(std::min<size_t>(smem, 227 * 1024)));
                launch_kernel(warp_stencil<FUSED>, dim3(Bi, Hi), 32, smem, st, a, b, out, Hi, Li, Ki, off, rev);
                break;
            }
        }
        return check_launch();
    }
    // dW: a = gy, b = x
    if (variant == 0) {
        const dim3 grid((Ki + kNaiveThreads - 1) / kNaiveThreads, Hi);
        launch_kernel(naive_dw<FUSED>, grid, kNaiveThreads, 0, st, a, b, out, Bi, Hi, Li, Ki);
        return check_launch();
    }
    const int64_t n = B * L;
    const int64_t span = (n + kChunks - 1) / kChunks;
    float* part = static_cast<float*>(ws);
    const dim3 grid(kChunks, Hi);
    if (variant == 1) {
        launch_kernel(twostage_dw<false, FUSED>, grid, 256, 0, st, a, b, part, Bi, Hi, Li, Ki, span);
    } else {
        const size_t smem = sizeof(float) * 2 * span;
        cudaFuncSetAttribute(twostage_dw<true, FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(std::min<size_t>(smem, 227 * 1024)));
        launch_kernel(twostage_dw<true, FUSED>, grid, 256, smem, st, a, b, part, Bi, Hi, Li, Ki, span);
    }
    ks_status s = check_launch();
    if (s != KS_OK) return s;
    const int64_t HK = H * K;
    launch_kernel(sum_chunks, static_cast<unsigned>((HK + 255) / 256), 256, 0, st, part, out, HK);
    return check_launch();
}

}  // namespace

size_t variant_workspace_bytes(int variant, int path, int64_t H, int64_t K) {
    return (path == 2 && variant != 0) ? size_t(kChunks) * H * K * sizeof(float) : 0;
}

// Shape limits of the literal paper mappings (grid.y/z <= 65535, a whole row
// or a 1/64 chunk in shared memory).  Returns false when a variant cannot run.
bool variant_supported(int variant, int path, int64_t B, int64_t H, int64_t L, int64_t K) {
    if (B * H * L >= (int64_t(1) << 40) || L >= (int64_t(1) << 30) || K >= (int64_t(1) << 30)) return false;
    if (path != 2) {
        if (variant == 0) return H <= 65535 && B <= 65535;
        if (variant == 1) return (H + kHTile - 1) / kHTile <= 65535 && B <= 65535;
        if (variant == 2) return sizeof(float) * (kTpb + 2 * K - 1) <= 227 * 1024;
        return B <= 2147483647 && H <= 65535 && sizeof(float) * (L + K) <= 227 * 1024;
    }
    if (variant == 0) return H <= 65535;
    if (variant == 1) return H <= 65535;
    const int64_t span = (B * L + kChunks - 1) / kChunks;
    return H <= 65535 && sizeof(float) * 2 * span <= 227 * 1024;
}

ks_status variant_f32(int variant, int path, const float* a, const float* b, float* out, int64_t B, int64_t H,
                      int64_t L, int64_t K, int mode, void* ws, cudaStream_t st) {
    return mode == KS_MULADD_FUSED ? run<true>(variant, path, a, b, out, B, H, L, K, ws, st)
                                   : run<false>(variant, path, a, b, out, B, H, L, K, ws, st);
}

}  // namespace ks
