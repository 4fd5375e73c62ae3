// ATTIC (not built): measured 3x slower than bwd_short at config 3 (5.41 vs 1.88 ms,
// tools/gpu_runs/gpu_run80.sh) -- lanes 128 B apart (the dw_tma block mapping dk must keep)
// make every 128-bit load touch 32 lines; kept as the record of the experiment.
// bwd_ldg.cu -- the fused backward (dX + HIERARCHICAL dW stage 1) for short
// kernels from register windows, without a staging ring (the stencil_ldg.cu
// design applied to bwd_short.cuh's MODE 1).
//
//   dx[b,h,t] = sum_j gy[b,h,t+j-q] * k[h,K-1-j]        (reference src/conv_core.cpp:48-75)
//   dk[h,j]   = sum_b sum_t gy[b,h,t] * x[b,h,t+j-p]    (src/conv_core.cpp:148-181)
//
// Same decomposition and association order as dw_tma / bwd_short (CTA = (row
// group, channel), work items = (row, 2048-wide tile) in flat order, thread
// (warp w, lane l) owns the 8-wide block at tl = 32 l + 8 (w & 3) + 1024 (w >> 2),
// ascending-t chains per tap, the same xor-shuffle / warp tree), so dk is
// bit-identical to the dW-only call and dx to the stencils.  What changes is
// the data path: each thread loads its gy window (which also holds the 8 gy
// values of its dW block) and its x window with 128-bit loads straight into
// registers -- the overlap with neighbouring blocks is served by L1 -- and
// writes its 8 dx outputs with one 256-bit store.  No shared-memory ring, no
// per-item CTA barrier: warps run their items independently.
#include <algorithm>
#include <cstdlib>

#include "ks_common.cuh"

namespace ks {

namespace {

__device__ __forceinline__ void st_v8(float* p, const float (&d)[8]) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(d[0]), "f"(d[1]), "f"(d[2]),
                 "f"(d[3]), "f"(d[4]), "f"(d[5]), "f"(d[6]), "f"(d[7])
                 : "memory");
}

template <int NQ>
__device__ __forceinline__ void load_window(const float* row, int a0, int L, float (&v)[4 * NQ]) {
#pragma unroll
    for (int c = 0; c < NQ; ++c) {
        const int s = a0 + 4 * c;
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);  // quads are wholly in or out of the row (L % 8 == 0)
        if (s >= 0 && s < L) q = *reinterpret_cast<const float4*>(row + s);
        v[4 * c + 0] = q.x;
        v[4 * c + 1] = q.y;
        v[4 * c + 2] = q.z;
        v[4 * c + 3] = q.w;
    }
}

template <int KT, bool FUSED>
__global__ void __launch_bounds__(256)
bwd_ldg(const float* __restrict__ gy, const float* __restrict__ x, const float* __restrict__ k,
        float* __restrict__ dx, float* __restrict__ part, int B, int H, int L, int G) {
    constexpr int p = KT / 2, q = KT - 1 - p;
    constexpr int S = (4 - p % 4) % 4;                    // x window shift: (-p) mod 4
    constexpr int S2 = (4 - q % 4) % 4;                   // gy window shift: (-q) mod 4
    constexpr int QS = q + S2;                            // gy[t] sits at window index QS (multiple of 4)
    constexpr int NVX = (S + 8 + KT - 1 + 3) / 4;
    constexpr int NV2 = (S2 + 8 + KT - 1 + 3) / 4;
    static_assert(QS % 4 == 0 && QS + 8 <= 4 * NV2, "gy block inside the dX window");
    __shared__ float red[8][KT];

    const int h = blockIdx.x % H;
    const int grp = blockIdx.x / H;
    const int b_begin = static_cast<int>(static_cast<int64_t>(B) * grp / G);
    const int b_end = static_cast<int>(static_cast<int64_t>(B) * (grp + 1) / G);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tl = 32 * lane + 8 * (warp & 3) + 1024 * (warp >> 2);

    float w[KT];  // dX taps, reversed (the reference's k[h, K-1-j], src/conv_core.cpp:68)
#pragma unroll
    for (int jj = 0; jj < KT; ++jj) w[jj] = __ldg(k + static_cast<int64_t>(h) * KT + KT - 1 - jj);
    float acc[KT];
#pragma unroll
    for (int jj = 0; jj < KT; ++jj) acc[jj] = 0.f;

    for (int b = b_begin; b < b_end; ++b) {
        const int64_t roff = (static_cast<int64_t>(b) * H + h) * L;
        const float* gyr = gy + roff;
        const float* xr = x + roff;
        for (int t0 = 0; t0 < L; t0 += 2048) {
            const int t = t0 + tl;
            if (t >= L) continue;
            float v2[4 * NV2], xv[4 * NVX];
            load_window<NV2>(gyr, t - QS, L, v2);  // gy[t - QS + i]
            load_window<NVX>(xr, t - p - S, L, xv);  // x[t - p - S + i]
            // dx[t+r] = sum_j gy[t+r+j-q] * w[j], j ascending from +0
            float d[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) d[r] = 0.f;
#pragma unroll
            for (int jj = 0; jj < KT; ++jj)
#pragma unroll
                for (int r = 0; r < 8; ++r) d[r] = muladd<FUSED>(d[r], v2[S2 + r + jj], w[jj]);
            st_v8(dx + roff + t, d);
            // dW: acc[jj] += gy[t+tt] * x[t+tt+jj-p]
#pragma unroll
            for (int tt = 0; tt < 8; ++tt)
#pragma unroll
                for (int jj = 0; jj < KT; ++jj) acc[jj] = muladd<FUSED>(acc[jj], v2[QS + tt], xv[S + tt + jj]);
        }
    }

    // fixed xor-shuffle tree per warp, then the 8 warps in ascending order (as dw_tma / bwd_short)
#pragma unroll
    for (int jj = 0; jj < KT; ++jj) {
        float v = acc[jj];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc[jj] = v;
    }
    if (lane == 0) {
#pragma unroll
        for (int jj = 0; jj < KT; ++jj) red[warp][jj] = acc[jj];
    }
    __syncthreads();
    if (tid < KT) {
        float s = 0.f;
#pragma unroll
        for (int ww = 0; ww < 8; ++ww) s += red[ww][tid];
        part[(static_cast<int64_t>(grp) * H + h) * KT + tid] = s;
    }
}

template <int KT>
ks_status launch_k(bool fused, const float* gy, const float* x, const float* k, float* dx, float* part, int64_t B,
                   int64_t H, int64_t L, int G, cudaStream_t st) {
    const unsigned blocks = static_cast<unsigned>(int64_t(G) * H);
    const int b = static_cast<int>(B), h = static_cast<int>(H), l = static_cast<int>(L);
    if (fused) bwd_ldg<KT, true><<<blocks, 256, 0, st>>>(gy, x, k, dx, part, b, h, l, G);
    else bwd_ldg<KT, false><<<blocks, 256, 0, st>>>(gy, x, k, dx, part, b, h, l, G);
    return check_launch();
}

}  // namespace

// K <= 8 (KS_BLDG=2: K <= 16; 0: never), L % 8 == 0, 16-byte gy / x and
// 32-byte dx bases; *handled = false otherwise (the caller uses bwd_short).
ks_status bwd_ldg_stage1(const float* gy, const float* x, const float* k, float* dx, float* part, int64_t B,
                         int64_t H, int64_t L, int64_t K, int G, int mode, cudaStream_t st, bool* handled) {
    *handled = false;
    const char* e = getenv("KS_BLDG");
    const int knob = e && *e ? atoi(e) : 1;
    if (knob == 0 || K < 1 || K > (knob >= 2 ? 16 : 8) || L % 8 != 0 || L >= (int64_t(1) << 30)) return KS_OK;
    if (B * H >= (int64_t(1) << 31) || int64_t(G) * H >= (int64_t(1) << 31)) return KS_OK;
    if ((reinterpret_cast<uintptr_t>(gy) & 15) || (reinterpret_cast<uintptr_t>(x) & 15) ||
        (reinterpret_cast<uintptr_t>(dx) & 31))
        return KS_OK;
    *handled = true;
    const bool f = mode == KS_MULADD_FUSED;
    switch (K) {
#define KS_BLDG_CASE(KV) \
    case KV: return launch_k<KV>(f, gy, x, k, dx, part, B, H, L, G, st);
        KS_BLDG_CASE(1) KS_BLDG_CASE(2) KS_BLDG_CASE(3) KS_BLDG_CASE(4) KS_BLDG_CASE(5) KS_BLDG_CASE(6)
        KS_BLDG_CASE(7) KS_BLDG_CASE(8) KS_BLDG_CASE(9) KS_BLDG_CASE(10) KS_BLDG_CASE(11) KS_BLDG_CASE(12)
        KS_BLDG_CASE(13) KS_BLDG_CASE(14) KS_BLDG_CASE(15) KS_BLDG_CASE(16)
#undef KS_BLDG_CASE
        default: return KS_ERR_CUDA;
    }
}

}  // namespace ks
