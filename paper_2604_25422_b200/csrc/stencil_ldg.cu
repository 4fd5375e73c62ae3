// stencil_ldg.cu -- forward / dX for short kernels (K <= 16) without a staging
// ring: every thread owns 8 consecutive outputs, reads its window with 128-bit
// loads straight into registers (the overlapping halo of neighbouring threads
// is served by L1, the same on-chip SRAM the TMA kernels stage through) and
// writes the 8 outputs with ONE 256-bit store -- a whole 32-byte sector.
//
//   out[b,h,t] = sum_{j<K} in[b,h,t+j-off] * w[h,j]     (reference src/conv_core.cpp:21-75)
//
// Why: at config 3's shape a probe (tools/probes/ldg_stencil_probe.cu) ran
// this shape of kernel at 6.63 TB/s -- cudaMemcpy's rate -- against 6.1-6.2
// for the TMA load -> shared -> TMA store kernels (stencil_tma, bwd_short),
// whose 1:1 read/write stream tops out near 95% of the copy rate.  One thread
// per 8 outputs and a full (non-persistent) grid of (row, 2048-output tile)
// CTAs: the probe's persistent grids were 2-40% slower.
//
// Bits: each output is the reference's ascending-j chain from +0; quads wholly
// outside the row are zero (the reference's zero padding), and a zero tap
// contribution never changes a chain that starts at +0 -- bit-identical to
// the reference and to the other stencils.  K, the offset and the sub-quad
// window shift are template constants (the fused backward's dX uses the same
// arithmetic).
#include <algorithm>
#include <cstdlib>

#include "ks_common.cuh"

namespace ks {

__global__ void prep_taps(const float*, float*, int64_t, int64_t, int64_t, int, int);

namespace {

__device__ __forceinline__ void st_v8(float* p, const float (&d)[8]) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(d[0]), "f"(d[1]), "f"(d[2]),
                 "f"(d[3]), "f"(d[4]), "f"(d[5]), "f"(d[6]), "f"(d[7])
                 : "memory");
}

// REV = 0: forward (off = p = K/2); REV = 1: dX (off = q = K-1-p).  kp: the
// prepared taps [H, 16] (reversed for dX, zero past K).
// V8: L % 8 == 0 and a 32-byte aligned output -- one 256-bit store per
// thread; otherwise (L % 8 == 4) two 128-bit stores, the second dropped for
// the last half-block of a row.
// MRW: rows shorter than 1024, several whole rows per CTA (a template switch:
// the runtime branch cost the single-row Separate kernel 8% at K = 7).
template <int KT, bool FUSED, bool REV, bool V8, bool MRW>
__global__ void __launch_bounds__(256)
stencil_ldg(const float* __restrict__ in, const float4* __restrict__ kp, float* __restrict__ out, int tpr, int H,
            int L, int rows, int rpc, int tprow) {
    pdl_wait();  // launched with PDL after prep_taps: kp must be complete
    constexpr int OFF = REV ? KT - 1 - KT / 2 : KT / 2;
    constexpr int S = (4 - OFF % 4) % 4;              // window starts S floats into its first quad
    constexpr int NV = (S + 8 + KT - 1 + 3) / 4;      // quads per window
    // CTA = (row, 2048-output tile): the row, channel and tile are CTA-uniform
    // (uniform datapath), the thread's 8 outputs start at 8 * threadIdx.x.
    // Rows shorter than 1024 (rpc > 1): a CTA takes rpc whole rows, tprow =
    // ceil(L / 8) threads each, instead of leaving most of its threads idle.
    int row, t;
    if constexpr (MRW) {
        const int r = static_cast<int>(threadIdx.x) / tprow;
        row = static_cast<int>(blockIdx.x) * rpc + r;
        t = 8 * (static_cast<int>(threadIdx.x) - r * tprow);
        if (r >= rpc || row >= rows) return;
    } else {
        row = static_cast<int>(blockIdx.x) / tpr;
        t = (static_cast<int>(blockIdx.x) - row * tpr) * 2048 + 8 * static_cast<int>(threadIdx.x);
    }
    if (t >= L) return;
    const int h = row % H;
    constexpr int KPS = KT <= 16 ? 16 : 32;  // prepared taps per channel
    float w[KPS];
#pragma unroll
    for (int c = 0; c < (KT + 3) / 4; ++c) {
        const float4 q = __ldg(kp + h * (KPS / 4) + c);
        w[4 * c + 0] = q.x;
        w[4 * c + 1] = q.y;
        w[4 * c + 2] = q.z;
        w[4 * c + 3] = q.w;
    }
    const float* xr = in + static_cast<int64_t>(row) * L;
    const int a0 = t - OFF - S;                       // 4-aligned: t % 8 == 0, (OFF + S) % 4 == 0
    float v[4 * NV];
#pragma unroll
    for (int c = 0; c < NV; ++c) {
        const int s = a0 + 4 * c;
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);   // quads are wholly in or out of the row (L % 4 == 0)
        if (s >= 0 && s < L) q = *reinterpret_cast<const float4*>(xr + s);
        v[4 * c + 0] = q.x;
        v[4 * c + 1] = q.y;
        v[4 * c + 2] = q.z;
        v[4 * c + 3] = q.w;
    }
    float d[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) d[r] = 0.f;
#pragma unroll
    for (int jj = 0; jj < KT; ++jj)
#pragma unroll
        for (int r = 0; r < 8; ++r) d[r] = muladd<FUSED>(d[r], v[S + r + jj], w[jj]);
    float* o = out + static_cast<int64_t>(row) * L + t;
    if constexpr (V8) {
        st_v8(o, d);
    } else {
        *reinterpret_cast<float4*>(o) = make_float4(d[0], d[1], d[2], d[3]);
        if (t + 8 <= L) *reinterpret_cast<float4*>(o + 4) = make_float4(d[4], d[5], d[6], d[7]);
    }
}

template <int KT, bool REV>
ks_status launch_k(bool fused, const float* in, const float4* kp, float* out, int64_t rows, int64_t H, int64_t L,
                   cudaStream_t st) {
    const int tpr = static_cast<int>((L + 2047) / 2048);
    const int tprow = static_cast<int>((L + 7) / 8);
    const int rpc = L < 1024 ? 256 / tprow : 1;
    const unsigned grid = static_cast<unsigned>(rpc > 1 ? (rows + rpc - 1) / rpc : rows * tpr);
    const int h = static_cast<int>(H), l = static_cast<int>(L), nr = static_cast<int>(rows);
    const bool v8 = L % 8 == 0 && (reinterpret_cast<uintptr_t>(out) & 31) == 0;
#define KS_LDG_LAUNCH(F, V, M) \
    launch_kernel_pdl(stencil_ldg<KT, F, REV, V, M>, grid, 256, 0, st, in, kp, out, tpr, h, l, nr, rpc, tprow)
    if (rpc > 1) {
        if (v8) { if (fused) KS_LDG_LAUNCH(true, true, true); else KS_LDG_LAUNCH(false, true, true); }
        else { if (fused) KS_LDG_LAUNCH(true, false, true); else KS_LDG_LAUNCH(false, false, true); }
    } else {
        if (v8) { if (fused) KS_LDG_LAUNCH(true, true, false); else KS_LDG_LAUNCH(false, true, false); }
        else { if (fused) KS_LDG_LAUNCH(true, false, false); else KS_LDG_LAUNCH(false, false, false); }
    }
#undef KS_LDG_LAUNCH
    return check_launch();
}

template <bool REV>
ks_status launch_any(int64_t K, bool fused, const float* in, const float4* kp, float* out, int64_t rows, int64_t H,
                     int64_t L, cudaStream_t st) {
    switch (K) {
#define KS_LDG_CASE(KV) \
    case KV: return launch_k<KV, REV>(fused, in, kp, out, rows, H, L, st);
        KS_LDG_CASE(1) KS_LDG_CASE(2) KS_LDG_CASE(3) KS_LDG_CASE(4) KS_LDG_CASE(5) KS_LDG_CASE(6)
        KS_LDG_CASE(7) KS_LDG_CASE(8) KS_LDG_CASE(9) KS_LDG_CASE(10) KS_LDG_CASE(11) KS_LDG_CASE(12)
        KS_LDG_CASE(13) KS_LDG_CASE(14) KS_LDG_CASE(15) KS_LDG_CASE(16) KS_LDG_CASE(17) KS_LDG_CASE(18)
        KS_LDG_CASE(19) KS_LDG_CASE(20) KS_LDG_CASE(21) KS_LDG_CASE(22) KS_LDG_CASE(23) KS_LDG_CASE(24)
        KS_LDG_CASE(25) KS_LDG_CASE(26) KS_LDG_CASE(27) KS_LDG_CASE(28) KS_LDG_CASE(29) KS_LDG_CASE(30)
        KS_LDG_CASE(31) KS_LDG_CASE(32)
#undef KS_LDG_CASE
        default: return KS_ERR_CUDA;
    }
}

}  // namespace

// *handled = false when the shape / alignment is outside this kernel's
// envelope (L % 4 == 0, 16-byte aligned bases; 256-bit stores where L % 8 == 0
// and the output is 32-byte aligned) or the knob
// says otherwise.  Default on rows of 2048 or more: K <= 10 (round-2 ABAB
// sweep over K = 9..16 at (256,512,8192,K), tools/sweep_options.py,
// gpurun_out/s5: K = 9 fwd 1.45 -> 1.25 ms Fused, 1.50 -> 1.32 Separate;
// K = 10 Fused 1.46 -> 1.36, Separate even; K >= 11 the TMA kernels win,
// Separate mode by up to 25% at K = 16).  Measured on the B200 (bench.py, ABAB):
// config 3 (K = 7) fwd 1.40 -> 1.22 ms and dX 1.42 -> 1.22 ms (7.0 TB/s),
// but config 5a (K = 16, (512,1024,16384)) fwd 11.5 -> 13.3 and dX 11.2 ->
// 14.1 ms under the power cap (at (256,512,8192,16) it was 4% faster), so the
// K-specialised TMA kernels keep 8 < K <= 16.  KS_LDG=0 / 1 / 2: never /
// default / every K <= 16.
ks_status stencil_ldg_f32(const float* in, const float* k, float* out, int64_t B, int64_t H, int64_t L, int64_t K,
                          int64_t off, int reverse, int mode, cudaStream_t st, bool* handled) {
    *handled = false;
    const int knob = static_cast<int>(opt(kOptLdg));
    if (knob == 0 || L < 256) return KS_OK;
    // default (knob 1): K <= 10 on long rows; below L = 2048 -- where the TMA
    // kernels' 2048-wide items run partly past the row end -- K <= 12, and
    // K <= 16 in Fused mode from L = 1024 (round-2 ABAB over L = 256..1984,
    // gpurun_out/s18: K <= 12 -7..-36%, K = 16 Fused at L = 1984 -31%,
    // K = 16 Separate or L = 256 slower)
    const bool fused_mode = mode == KS_MULADD_FUSED;
    // rows the TMA views cannot take (L % 32 != 0) have no better kernel up to K = 16
    // rows shorter than 1024 (whole rows per CTA): K <= 32 in both modes
    // (gpurun_out/s25: L = 256 / 512, K = 14..32, -30..-50% against the TMA
    // kernels; from L = 1024 on, K = 24 / 32 lose by 0-15%)
    const int64_t kmax = knob >= 2 ? 32 : L < 1024 ? 32 : L % 32 != 0 ? 16 : L >= 2048 ? 10
                                                     : fused_mode ? 16 : 12;
    if (K > kmax) return KS_OK;
    if (K < 1 || K > 32 || L % 4 != 0 || L >= (int64_t(1) << 30) || off != (reverse ? K - 1 - K / 2 : K / 2))
        return KS_OK;
    if ((reinterpret_cast<uintptr_t>(in) & 15) != 0 || (reinterpret_cast<uintptr_t>(out) & 15) != 0) return KS_OK;
    const int64_t rows = B * H;
    if (rows * ((L + 2047) / 2048) >= (int64_t(1) << 31)) return KS_OK;
    float* kp = nullptr;
    const int64_t kps = K <= 16 ? 16 : 32;  // the kernel's KPS
    ks_status rc = cuda_status(scratch_alloc(reinterpret_cast<void**>(&kp), sizeof(float) * H * kps, st));
    if (rc != KS_OK) return rc;
    *handled = true;
    launch_kernel(prep_taps, static_cast<unsigned>(std::min<int64_t>((H * kps + 255) / 256, 4096)), 256, 0, st, k, kp, H, K, kps,
                                                                                                   reverse, 0);
    rc = check_launch();
    if (rc == KS_OK) {
        const bool fused = mode == KS_MULADD_FUSED;
        const float4* kp4 = reinterpret_cast<const float4*>(kp);
        rc = reverse ? launch_any<true>(K, fused, in, kp4, out, rows, H, L, st)
                     : launch_any<false>(K, fused, in, kp4, out, rows, H, L, st);
    }
    scratch_free(kp, st);
    return rc;
}

}  // namespace ks
