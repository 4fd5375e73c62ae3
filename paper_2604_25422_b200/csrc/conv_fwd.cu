// conv_fwd.cu -- forward y and input-gradient dX kernels (sm_100a).
//
// Both paths are one stencil:  out[b,h,t] = sum_{j=0}^{K-1} in[b,h,t+j-off] * w[h,j]
//   forward         : in = x,  w[j] = k[h,j],      off = p = K/2
//                     (reference src/conv_core.cpp:21-46)
//   backward_input  : in = gy, w[j] = k[h,K-1-j],  off = q = K-1-p
//                     (reference src/conv_core.cpp:48-75)
// Every output accumulates its taps in ascending j from +0 with the selected
// MulAddMode, so results are bit-identical to the reference: taps that fall
// outside the row read an explicit zero from the halo, and acc + (+-0) == acc
// for every acc the chain can hold (acc starts at +0 and round-to-nearest never
// produces -0 from a +0 start).
//
// Tile kernel: one CTA = one (b,h) row segment of T = 256*R outputs.  The CTA
// stages the input window [t0-off, t0+T+K-1-off) once in shared memory
// (128-bit read-only loads, zero halo at the row ends, padded layout that keeps
// the register-tile float4 reads conflict-free) and the channel's K taps; each
// thread then keeps R consecutive outputs in registers and slides a register
// window over the taps in blocks of JB, so every shared-memory word feeds
// R*JB/(R+JB) FMAs.  Stores are 128-bit streaming stores.
#include <algorithm>
#include <cstdlib>

#include "ks_common.cuh"

namespace ks {

constexpr int kTileThreads = 256;
constexpr int kJB = 8;  // taps per register block

template <int R>
struct TileGeom {
    static constexpr int T = kTileThreads * R;  // outputs per CTA
};

// Number of float4 registers a thread reads per tap block for shift S.
template <int R, int S>
constexpr int nv4() { return (S + R + kJB - 1 + 3) / 4; }

// Logical window length (floats) staged per CTA, for padded tap count Kp.
template <int R, int S>
__host__ __device__ constexpr int window_len(int Kp) {
    return (kTileThreads - 1) * R + (Kp - kJB) + 4 * nv4<R, S>();
}

__host__ __device__ inline int round_up(int a, int b) { return (a + b - 1) / b * b; }

template <int R, int S, bool FUSED>
__global__ void __launch_bounds__(kTileThreads)
conv_tile_f32(const float* __restrict__ in, const float* __restrict__ k, float* __restrict__ out,
              int H, int L, int K, int off, int reverse, int tiles_per_row) {
    extern __shared__ float4 smem4[];
    constexpr int T = TileGeom<R>::T;
    constexpr int NV = nv4<R, S>();
    const int Kp = round_up(K, kJB);
    const int WL = window_len<R, S>(Kp);
    float* win = reinterpret_cast<float*>(smem4);
    float* wk = win + round_up(padded_len(WL), 4);

    const int64_t row = blockIdx.x / tiles_per_row;
    const int tile = blockIdx.x - static_cast<int>(row * tiles_per_row);
    const int h = static_cast<int>(row % H);
    const int t0 = tile * T;
    const int a0 = t0 - off - S;  // global position of logical window index 0 (4-aligned)
    const float* rin = in + row * static_cast<int64_t>(L);
    const int tid = threadIdx.x;

    // ---- stage the channel taps (zero padded to a multiple of JB) ----
    for (int j = tid; j < Kp; j += kTileThreads) {
        float v = 0.f;
        if (j < K) v = k[static_cast<int64_t>(h) * K + (reverse ? K - 1 - j : j)];
        wk[j] = v;
    }
    // ---- stage the input window with a zero halo ----
    // (128-bit global accesses need 16-byte aligned rows: L % 4 == 0 and
    // 16-byte aligned base pointers -- callers may pass any float views)
    const bool vec_ok = (L & 3) == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0;
    const bool vec_out = (L & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    for (int c = tid; c < WL / 4; c += kTileThreads) {
        const int g = a0 + 4 * c;
        float4 v;
        if (vec_ok && g >= 0 && g + 3 < L) {
            v = ld_nc_v4(rin + g);
        } else {
            v.x = (g + 0 >= 0 && g + 0 < L) ? rin[g + 0] : 0.f;
            v.y = (g + 1 >= 0 && g + 1 < L) ? rin[g + 1] : 0.f;
            v.z = (g + 2 >= 0 && g + 2 < L) ? rin[g + 2] : 0.f;
            v.w = (g + 3 >= 0 && g + 3 < L) ? rin[g + 3] : 0.f;
        }
        *reinterpret_cast<float4*>(win + pad_idx(4 * c)) = v;
    }
    __syncthreads();

    const int base = tid * R;
    if (t0 + base >= L) return;  // whole register tile past the row end

    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.f;

    auto block = [&](int j0, int nj) {
        float v[4 * NV];
#pragma unroll
        for (int c = 0; c < NV; ++c) {
            const float4 q = *reinterpret_cast<const float4*>(win + pad_idx(base + j0 + 4 * c));
            v[4 * c + 0] = q.x;
            v[4 * c + 1] = q.y;
            v[4 * c + 2] = q.z;
            v[4 * c + 3] = q.w;
        }
        float w[kJB];
#pragma unroll
        for (int c = 0; c < kJB / 4; ++c) {
            const float4 q = *reinterpret_cast<const float4*>(wk + j0 + 4 * c);
            w[4 * c + 0] = q.x;
            w[4 * c + 1] = q.y;
            w[4 * c + 2] = q.z;
            w[4 * c + 3] = q.w;
        }
#pragma unroll
        for (int jj = 0; jj < kJB; ++jj) {
            if (jj < nj) {
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r] = muladd<FUSED>(acc[r], v[S + r + jj], w[jj]);
            }
        }
    };

    const int Kfull = K - K % kJB;
    for (int j0 = 0; j0 < Kfull; j0 += kJB) block(j0, kJB);
    if (Kfull < K) block(Kfull, K - Kfull);

    float* rout = out + row * static_cast<int64_t>(L) + t0 + base;
    if (vec_out && t0 + base + R <= L) {
#pragma unroll
        for (int r = 0; r < R; r += 4)
            st_cs_v4(rout + r, make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]));
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (t0 + base + r < L) rout[r] = acc[r];
    }
}

// Direct kernel: one thread per output, taps over exactly the reference's
// in-range window [j_lo, j_hi) (src/conv_core.cpp:35-36, 64-65).  Used for
// fp64 and as the fp32 fallback when the staged window would not fit in
// shared memory.
template <typename T, bool FUSED>
__global__ void __launch_bounds__(256)
conv_direct(const T* __restrict__ in, const T* __restrict__ k, T* __restrict__ out, int64_t H,
            int64_t L, int64_t K, int64_t off, int reverse, int64_t total) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t row = i / L;
        const int64_t t = i - row * L;
        const int64_t h = row % H;
        const T* rin = in + row * L;
        const T* kr = k + h * K;
        const int64_t j_lo = t < off ? off - t : 0;
        const int64_t j_hi = (L + off - t) < K ? (L + off - t) : K;
        T acc = T(0);
        for (int64_t j = j_lo; j < j_hi; ++j)
            acc = muladd<FUSED>(acc, rin[t + j - off], kr[reverse ? K - 1 - j : j]);
        out[i] = acc;
    }
}

// ---------------------------------------------------------------------------
// host-side launchers

template <int R, int S, bool FUSED>
static size_t tile_smem_bytes(int K) {
    const int Kp = round_up(K, kJB);
    return sizeof(float) * (round_up(padded_len(window_len<R, S>(Kp)), 4) + Kp);
}

template <int R, int S, bool FUSED>
static ks_status launch_tile(const float* in, const float* k, float* out, int64_t B, int64_t H,
                             int64_t L, int64_t K, int64_t off, int reverse, cudaStream_t st) {
    const size_t smem = tile_smem_bytes<R, S, FUSED>(static_cast<int>(K));
    // per device and thread-safe (a function-local flag would opt in only the
    // first device a process uses)
    prepare_kernel(reinterpret_cast<const void*>(conv_tile_f32<R, S, FUSED>), kTileThreads, static_cast<int>(smem));
    const int tiles = static_cast<int>((L + TileGeom<R>::T - 1) / TileGeom<R>::T);
    const int64_t blocks = B * H * tiles;
    launch_kernel(conv_tile_f32<R, S, FUSED>, static_cast<unsigned>(blocks), kTileThreads, smem, st, 
        in, k, out, static_cast<int>(H), static_cast<int>(L), static_cast<int>(K),
        static_cast<int>(off), reverse, tiles);
    return check_launch();
}

template <int R, bool FUSED>
static ks_status launch_tile_s(int s, const float* in, const float* k, float* out, int64_t B,
                               int64_t H, int64_t L, int64_t K, int64_t off, int reverse,
                               cudaStream_t st) {
    switch (s) {
        case 0: return launch_tile<R, 0, FUSED>(in, k, out, B, H, L, K, off, reverse, st);
        case 1: return launch_tile<R, 1, FUSED>(in, k, out, B, H, L, K, off, reverse, st);
        case 2: return launch_tile<R, 2, FUSED>(in, k, out, B, H, L, K, off, reverse, st);
        default: return launch_tile<R, 3, FUSED>(in, k, out, B, H, L, K, off, reverse, st);
    }
}

template <typename T>
static ks_status launch_direct(const T* in, const T* k, T* out, int64_t B, int64_t H, int64_t L,
                               int64_t K, int64_t off, int reverse, int mode, cudaStream_t st) {
    const int64_t total = B * H * L;
    const int64_t want = (total + 255) / 256;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(want, int64_t(num_sms()) * 32));
    if (mode == KS_MULADD_FUSED)
        launch_kernel(conv_direct<T, true>, blocks, 256, 0, st, in, k, out, H, L, K, off, reverse, total);
    else
        launch_kernel(conv_direct<T, false>, blocks, 256, 0, st, in, k, out, H, L, K, off, reverse, total);
    return check_launch();
}

ks_status stencil_ldg_f32(const float*, const float*, float*, int64_t, int64_t, int64_t, int64_t, int64_t, int, int,
                          cudaStream_t, bool*);
ks_status stencil_tma_f32(const float*, const float*, float*, int64_t, int64_t, int64_t, int64_t, int64_t,
                          int, int, cudaStream_t, bool*);
ks_status stencil_rows_f32(const float*, const float*, float*, int64_t, int64_t, int64_t, int64_t, int64_t,
                           int, int, cudaStream_t, bool*);


// Entry used by the C ABI for both fp32 paths (shapes already validated).
ks_status conv_stencil_f32(const float* in, const float* k, float* out, int64_t B, int64_t H,
                           int64_t L, int64_t K, int64_t off, int reverse, int mode,
                           cudaStream_t st) {
    if (L < 1024) {  // short rows: whole rows per CTA (rows_short.cu)
        bool handled = false;
        const ks_status s = stencil_rows_f32(in, k, out, B, H, L, K, off, reverse, mode, st, &handled);
        if (handled) return s;
    }
    if (!tma_disabled() && K <= 32 && L >= 256) {  // short kernels: register windows, 256-bit stores
        bool handled = false;
        const ks_status s = stencil_ldg_f32(in, k, out, B, H, L, K, off, reverse, mode, st, &handled);
        if (handled) return s;
    }
    if (!tma_disabled()) {
        bool handled = false;
        const ks_status s = stencil_tma_f32(in, k, out, B, H, L, K, off, reverse, mode, st, &handled);
        if (handled) return s;
    }
    // Register tile of 16 outputs for long rows, 4 for short ones so small-L
    // problems still spread over many CTAs.
    const bool small = L <= 1024;
    const int s = static_cast<int>((4 - off % 4) % 4);
    const size_t smem = small ? tile_smem_bytes<4, 3, false>(static_cast<int>(K))
                              : tile_smem_bytes<16, 3, false>(static_cast<int>(K));
    const bool fits = K <= (1 << 20) && smem <= 200 * 1024 && L < (1ll << 30);
    if (!fits) return launch_direct<float>(in, k, out, B, H, L, K, off, reverse, mode, st);
    if (small) {
        if (mode == KS_MULADD_FUSED)
            return launch_tile_s<4, true>(s, in, k, out, B, H, L, K, off, reverse, st);
        return launch_tile_s<4, false>(s, in, k, out, B, H, L, K, off, reverse, st);
    }
    if (mode == KS_MULADD_FUSED)
        return launch_tile_s<16, true>(s, in, k, out, B, H, L, K, off, reverse, st);
    return launch_tile_s<16, false>(s, in, k, out, B, H, L, K, off, reverse, st);
}

ks_status conv_stencil_f64(const double* in, const double* k, double* out, int64_t B,
                           int64_t H, int64_t L, int64_t K, int64_t off, int reverse, int mode,
                           cudaStream_t st) {
    return launch_direct<double>(in, k, out, B, H, L, K, off, reverse, mode, st);
}

}  // namespace ks
