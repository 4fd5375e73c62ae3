// rows_short.cu -- forward / dX and dW for short rows (sm_100a), e.g. the
// paper's S4ConvD training shape (B,H,L,K) = (16384,128,48,48)
// (fixtures/table2.csv).
//
// The long-row kernels tile the sequence axis; with L = 48 a tile would be
// mostly empty.  Here a CTA takes a chunk of whole rows instead:
//
// stencil_rows (fwd / dX, reference src/conv_core.cpp:21-75): 64 consecutive
//   (b,h) rows -- one contiguous block of memory -- are staged in shared memory
//   with their zero halos, row stride LS = 4 (mod 32) floats, together with
//   each row's taps (stride KS = 4 (mod 32)).  Lanes take consecutive rows, so
//   every 128-bit shared load of a warp is bank-conflict-free, and each thread
//   keeps R = 16 consecutive outputs of its row in registers and slides a
//   register window over the taps in ascending j from +0 (bit-identical to the
//   reference in both MulAddModes).
//
// dw_rows (dW, HIERARCHICAL order, src/conv_core.cpp:148-181): CTA =
//   (channel h, batch group); per iteration 32 rows b*H+h of gy and x (strided
//   in global memory) are staged the same way; thread (tap group, row, t phase)
//   accumulates 8 taps x 8 t FMAs per register block; then a fixed shuffle tree
//   over the rows, a fixed pass over t phases, one partial per CTA, and the
//   shared fixed-order cross-block pass (dw_sum_groups).  No atomics.
#include <algorithm>

#include "ks_common.cuh"

namespace ks {

template <typename T>
__global__ void dw_sum_groups(const T* __restrict__ part, T* __restrict__ dk, int64_t HK, int G);

namespace {

constexpr int kNT = 256;
constexpr int kJB = 8;

__host__ __device__ inline int round_up_i(int a, int b) { return (a + b - 1) / b * b; }
// smallest s >= n with s % 32 == 4 (128-bit loads by lanes s floats apart are conflict-free)
__host__ __device__ inline int stride4(int n) { return round_up_i(n - 4, 32) + 4; }

struct RowsGeom {
    int NRC;  // rows per chunk (multiple of 32)
    int LS;   // padded row stride (floats)
    int KS;   // padded tap-row stride (floats)
    int PL;   // left pad = round_up(off, 4)
    int segs; // R-wide output segments per row
};

template <int R, int S, bool FUSED>
__global__ void __launch_bounds__(kNT)
stencil_rows(const float* __restrict__ in, const float* __restrict__ k, float* __restrict__ out, int64_t nrows,
             int H, int L, int K, int reverse, RowsGeom g) {
    constexpr int NV = (S + R + kJB - 1 + 3) / 4;
    extern __shared__ __align__(16) float sm[];
    float* xs = sm;                    // [NRC][LS]
    float* tk = sm + g.NRC * g.LS;     // [NRC][KS]
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * g.NRC;
    const int64_t left = nrows - r0;
    const int nr = left < g.NRC ? static_cast<int>(left) : g.NRC;
    const int tid = threadIdx.x;

    // stage: zero everything, then the rows (contiguous in global memory) and taps
    for (int i = tid; i < g.NRC * g.LS / 4; i += kNT) reinterpret_cast<float4*>(xs)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    const float* src = in + r0 * L;
    const int n4 = nr * L / 4;  // L % 4 == 0
    for (int q = tid; q < n4; q += kNT) {
        const int f = 4 * q;
        const int i = f / L, t = f - i * L;
        *reinterpret_cast<float4*>(xs + i * g.LS + g.PL + t) = ld_nc_v4(src + f);
    }
    for (int q = tid; q < nr * K; q += kNT) {
        const int i = q / K, j = q - i * K;
        const int h = static_cast<int>((r0 + i) % H);
        tk[i * g.KS + j] = k[static_cast<int64_t>(h) * K + (reverse ? K - 1 - j : j)];
    }
    __syncthreads();

    const int Kfull = K - K % kJB;
    for (int q = tid; q < g.NRC * g.segs; q += kNT) {
        const int i = q % g.NRC, seg = q / g.NRC;
        const int ts = seg * R;
        if (i >= nr) continue;
        const float* xr = xs + i * g.LS + ts;  // + S + r + j  <->  x[ts + r + j - off]
        const float* kr = tk + i * g.KS;
        float acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0.f;
        auto block = [&](int j0, int nj) {
            float v[4 * NV];
#pragma unroll
            for (int c = 0; c < NV; ++c) {
                const float4 a = *reinterpret_cast<const float4*>(xr + j0 + 4 * c);
                v[4 * c + 0] = a.x;
                v[4 * c + 1] = a.y;
                v[4 * c + 2] = a.z;
                v[4 * c + 3] = a.w;
            }
            float w[kJB];
#pragma unroll
            for (int c = 0; c < kJB / 4; ++c) {
                const float4 a = *reinterpret_cast<const float4*>(kr + j0 + 4 * c);
                w[4 * c + 0] = a.x;
                w[4 * c + 1] = a.y;
                w[4 * c + 2] = a.z;
                w[4 * c + 3] = a.w;
            }
#pragma unroll
            for (int jj = 0; jj < kJB; ++jj)
                if (jj < nj) {
#pragma unroll
                    for (int r = 0; r < R; ++r) acc[r] = muladd<FUSED>(acc[r], v[S + r + jj], w[jj]);
                }
        };
        for (int j0 = 0; j0 < Kfull; j0 += kJB) block(j0, kJB);
        if (Kfull < K) block(Kfull, K - Kfull);
        float* o = out + (r0 + i) * L + ts;
        if (ts + R <= L) {
#pragma unroll
            for (int r = 0; r < R; r += 4) st_cs_v4(o + r, make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]));
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (ts + r < L) o[r] = acc[r];
        }
    }
}

// dW over short rows.  NJ tap groups of 8 taps, TP = 8/NJ t-phases, 32 rows
// per iteration: thread = (tap group, t phase, row lane).
template <int NJ, int S, bool FUSED>
__global__ void __launch_bounds__(kNT)
dw_rows(const float* __restrict__ gy, const float* __restrict__ x, float* __restrict__ part, int B, int H, int L,
        int K, int G, int NJT, int LS) {
    constexpr int TP = 8 / NJ;
    constexpr int NVX = (S + 8 + kJB - 1 + 3) / 4;
    constexpr int NR = 32;
    extern __shared__ __align__(16) float sm[];
    float* gs = sm;            // [32][LS], gy at [PLg + t] with PLg = 0
    float* xsm = sm + NR * LS; // [32][LS], x at [PLx + t]
    __shared__ float red[kNT / 32][kJB];

    int bid = blockIdx.x;
    const int jt = bid % NJT;
    bid /= NJT;
    const int h = bid % H;
    const int grp = bid / H;
    const int b_begin = static_cast<int>(static_cast<int64_t>(B) * grp / G);
    const int b_end = static_cast<int>(static_cast<int64_t>(B) * (grp + 1) / G);
    const int JT = NJ * kJB;
    const int j0 = jt * JT;
    const int p = K / 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int jg = warp / TP;  // tap group
    const int tp = warp % TP;  // t phase
    // x window of tap group jg: x[t + j0 + jg*8 + jj - p]; stored x[t] at xsm[PLx + t]
    const int dmin = j0 - p;                         // smallest tap offset in the tile
    const int PLx = round_up_i(max(0, -dmin), 4);    // left zero pad
    const int xoff = PLx + j0 + jg * kJB - p - S;    // index of x[t - ...] for t = 0 minus S, 4-aligned
    const int nblk = (L + 7) / 8;

    float acc[kJB];
#pragma unroll
    for (int i = 0; i < kJB; ++i) acc[i] = 0.f;

    for (int b0 = b_begin; b0 < b_end; b0 += NR) {
        const int nr = min(NR, b_end - b0);
        __syncthreads();
        for (int i = tid; i < 2 * NR * LS / 4; i += kNT) reinterpret_cast<float4*>(sm)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        __syncthreads();
        for (int q = tid; q < nr * (L / 4); q += kNT) {
            const int i = q / (L / 4), t = 4 * (q - i * (L / 4));
            const int64_t off = (static_cast<int64_t>(b0 + i) * H + h) * L + t;
            *reinterpret_cast<float4*>(gs + i * LS + t) = ld_nc_v4(gy + off);
            *reinterpret_cast<float4*>(xsm + i * LS + PLx + t) = ld_nc_v4(x + off);
        }
        __syncthreads();
        if (lane < nr) {
            const float* gr = gs + lane * LS;
            const float* xr = xsm + lane * LS + xoff;
            for (int blk = tp; blk < nblk; blk += TP) {
                const int t = blk * 8;
                float gv[8];
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const float4 a = *reinterpret_cast<const float4*>(gr + t + 4 * c);
                    gv[4 * c + 0] = a.x;
                    gv[4 * c + 1] = a.y;
                    gv[4 * c + 2] = a.z;
                    gv[4 * c + 3] = a.w;
                }
                float xv[4 * NVX];
#pragma unroll
                for (int c = 0; c < NVX; ++c) {
                    const float4 a = *reinterpret_cast<const float4*>(xr + t + 4 * c);
                    xv[4 * c + 0] = a.x;
                    xv[4 * c + 1] = a.y;
                    xv[4 * c + 2] = a.z;
                    xv[4 * c + 3] = a.w;
                }
#pragma unroll
                for (int tt = 0; tt < 8; ++tt)
#pragma unroll
                    for (int jj = 0; jj < kJB; ++jj) acc[jj] = muladd<FUSED>(acc[jj], gv[tt], xv[S + tt + jj]);
            }
        }
    }
    // fixed-order reduction: rows (lanes) by a shuffle tree, then t phases
#pragma unroll
    for (int jj = 0; jj < kJB; ++jj) {
        float v = acc[jj];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc[jj] = v;
    }
    if (lane == 0) {
#pragma unroll
        for (int jj = 0; jj < kJB; ++jj) red[warp][jj] = acc[jj];
    }
    __syncthreads();
    if (tid < JT) {
        const int gj = tid / kJB, jj = tid % kJB;
        float s = 0.f;
        for (int w = 0; w < TP; ++w) s += red[gj * TP + w][jj];
        const int j = j0 + tid;
        if (j < K) part[(static_cast<int64_t>(grp) * H + h) * K + j] = s;
    }
}

}  // namespace

// fwd / dX for short rows; *handled = false outside the envelope.
ks_status stencil_rows_f32(const float* in, const float* k, float* out, int64_t B, int64_t H, int64_t L, int64_t K,
                           int64_t off, int reverse, int mode, cudaStream_t st, bool* handled) {
    *handled = false;
    if (L % 4 != 0 || L > 1024 || K > 1024 || B * H >= (int64_t(1) << 40)) return KS_OK;
    if ((reinterpret_cast<uintptr_t>(in) & 15) || (reinterpret_cast<uintptr_t>(out) & 15)) return KS_OK;
    constexpr int R = 16;
    RowsGeom g;
    g.PL = round_up_i(static_cast<int>(off), 4);
    g.LS = stride4(g.PL + static_cast<int>(L + K) + R + 16);
    g.KS = stride4(round_up_i(static_cast<int>(K), kJB) + 4);
    g.segs = static_cast<int>((L + R - 1) / R);
    g.NRC = 64;
    while (g.NRC > 32 && (g.NRC * (g.LS + g.KS)) * 4 > 100 * 1024) g.NRC -= 32;
    const int smem = g.NRC * (g.LS + g.KS) * 4;
    if (smem > 200 * 1024) return KS_OK;
    const int64_t nrows = B * H;
    const int64_t chunks = (nrows + g.NRC - 1) / g.NRC;
    if (chunks >= (int64_t(1) << 31)) return KS_OK;
    const int s = g.PL - static_cast<int>(off);  // 0..3
    const bool fused = mode == KS_MULADD_FUSED;
    *handled = true;
#define KS_SR_CASE(SV)                                                                                       \
    case SV: {                                                                                               \
        auto kern = fused ? stencil_rows<R, SV, true> : stencil_rows<R, SV, false>;                          \
        prepare_kernel(reinterpret_cast<const void*>(kern), kNT, smem);                                      \
        kern<<<static_cast<unsigned>(chunks), kNT, smem, st>>>(in, k, out, nrows, static_cast<int>(H),       \
                                                                static_cast<int>(L), static_cast<int>(K),    \
                                                                reverse, g);                                 \
        break;                                                                                               \
    }
    switch (s) {
        KS_SR_CASE(0)
        KS_SR_CASE(1)
        KS_SR_CASE(2)
        default:
        KS_SR_CASE(3)
    }
#undef KS_SR_CASE
    return check_launch();
}

// dW stage 1 for short rows into part[G,H,K] (G = the caller's row groups).
ks_status dw_rows_stage1(const float* gy, const float* x, float* part, int64_t B, int64_t H, int64_t L, int64_t K,
                         int G, int mode, cudaStream_t st, bool* handled) {
    *handled = false;
    if (L % 4 != 0 || L > 1024 || B * H >= (int64_t(1) << 31)) return KS_OK;
    if ((reinterpret_cast<uintptr_t>(gy) & 15) || (reinterpret_cast<uintptr_t>(x) & 15)) return KS_OK;
    int nj = 1;
    while (nj < 8 && nj * kJB < K) nj *= 2;
    const int njt = static_cast<int>((K + nj * kJB - 1) / (nj * kJB));
    const int JT = nj * kJB;
    const int p = static_cast<int>(K / 2);
    // x rows are stored at [PLx, PLx + L) with PLx <= p + 3; a thread's window
    // reads reach index PLx + j0 + JT - p + L + 20 <= L + K + JT + 24 (PLx <= p + 3)
    const int LS = stride4(static_cast<int>(L + K) + JT + 32);
    const int smem = 2 * 32 * LS * 4;
    if (smem > 200 * 1024) return KS_OK;
    if (int64_t(G) * H * njt >= (int64_t(1) << 31)) return KS_OK;
    const int s = (4 - p % 4) % 4;
    const bool fused = mode == KS_MULADD_FUSED;
    const unsigned blocks = static_cast<unsigned>(int64_t(G) * H * njt);
    *handled = true;
#define KS_DR_CASE(NJV, SV)                                                                                    \
    if (nj == NJV && s == SV) {                                                                                \
        auto kern = fused ? dw_rows<NJV, SV, true> : dw_rows<NJV, SV, false>;                                  \
        prepare_kernel(reinterpret_cast<const void*>(kern), kNT, smem);                                        \
        kern<<<blocks, kNT, smem, st>>>(gy, x, part, static_cast<int>(B), static_cast<int>(H),                 \
                                        static_cast<int>(L), static_cast<int>(K), G, njt, LS);                 \
        return check_launch();                                                                                 \
    }
    KS_DR_CASE(1, 0) KS_DR_CASE(1, 1) KS_DR_CASE(1, 2) KS_DR_CASE(1, 3)
    KS_DR_CASE(2, 0) KS_DR_CASE(2, 1) KS_DR_CASE(2, 2) KS_DR_CASE(2, 3)
    KS_DR_CASE(4, 0) KS_DR_CASE(4, 1) KS_DR_CASE(4, 2) KS_DR_CASE(4, 3)
    KS_DR_CASE(8, 0) KS_DR_CASE(8, 1) KS_DR_CASE(8, 2) KS_DR_CASE(8, 3)
#undef KS_DR_CASE
    *handled = false;
    return KS_OK;
}

}  // namespace ks
