// bwd_short_impl.cuh -- host launchers of bwd_short (bwd_short.cuh) for one
// kernel family; included by bwd_short_dw.cu / bwd_short_dx.cu /
// bwd_short_st.cu so the specialisations compile in parallel.
#pragma once

#include <algorithm>
#include <cstdlib>

#include "bwd_short.cuh"

namespace ks {

__global__ void prep_taps(const float*, float*, int64_t, int64_t, int64_t, int, int);

namespace bwds {

template <int KT, bool FUSED, int MODE>
ks_status launch_k(const CUtensorMap& im, const CUtensorMap& xm, const CUtensorMap& om, const float* k, float* part,
                   int64_t B, int64_t H, int64_t L, int G, float* out, cudaStream_t st, int rpi = 0) {
    auto kern = bwd_short<KT, FUSED, MODE>;
    constexpr int smem = Geo<KT, MODE>::Smem;
    const int per_sm = prepare_kernel(reinterpret_cast<const void*>(kern), kThreads, smem);
    // stencils: a persistent grid in Separate mode (issue-bound: two FP
    // instructions per tap), one CTA per row in Fused mode, where an item is
    // short and the hardware scheduler's rebalancing of many CTAs pays
    // (round-2 ABAB, gpurun_out/s8: (64,1024,16384,16) fwd 1.50 -> 1.27 ms,
    // config 5a fwd 11.8 -> 10.9 ms; Separate 1-9% slower with it)
    // (rows of at least two items: with one 2048-wide item per row a per-row
    // CTA has nothing to prefetch -- (1024,64,2048,K) lost 38-55%, s28)
    const int64_t rows_opt = opt(kOptStsRows);
    const bool per_row = rows_opt == 1 || (rows_opt < 0 && FUSED && L >= 2 * kTT);
    const int64_t blocks = (MODE & 7) <= kFUSED ? int64_t(G) * H
                           : per_row ? B * H : std::min<int64_t>(B * H, int64_t(num_sms()) * per_sm);
    launch_kernel_pdl(kern, static_cast<unsigned>(blocks), kThreads, smem, st, im, xm, om, k, part, static_cast<int>(B),
                                                                static_cast<int>(H), static_cast<int>(L), G, out, rpi);
    return check_launch();
}

template <int KT, int MODE>
ks_status launch_m(bool fused, const CUtensorMap& im, const CUtensorMap& xm, const CUtensorMap& om, const float* k,
                   float* part, int64_t B, int64_t H, int64_t L, int G, float* out, cudaStream_t st, int rpi = 0) {
    // dW only: HIERARCHICAL accumulates with FMA in either MulAddMode (conv_dw.cu)
    if constexpr ((MODE & 7) == kDW) return launch_k<KT, true, MODE>(im, xm, om, k, part, B, H, L, G, out, st, rpi);
    else
        return fused ? launch_k<KT, true, MODE>(im, xm, om, k, part, B, H, L, G, out, st)
                     : launch_k<KT, false, MODE>(im, xm, om, k, part, B, H, L, G, out, st);
}

template <int MODE>
ks_status launch_any_k(int64_t K, bool f, const CUtensorMap& im, const CUtensorMap& xm, const CUtensorMap& om,
                       const float* k, float* part, int64_t B, int64_t H, int64_t L, int G, float* out,
                       cudaStream_t st, int rpi = 0) {
    switch (K) {
#define KS_BWDS_CASE(KV) \
    case KV: return launch_m<KV, MODE>(f, im, xm, om, k, part, B, H, L, G, out, st, rpi);
        KS_BWDS_CASE(1) KS_BWDS_CASE(2) KS_BWDS_CASE(3) KS_BWDS_CASE(4) KS_BWDS_CASE(5) KS_BWDS_CASE(6)
        KS_BWDS_CASE(7) KS_BWDS_CASE(8) KS_BWDS_CASE(9) KS_BWDS_CASE(10) KS_BWDS_CASE(11) KS_BWDS_CASE(12)
        KS_BWDS_CASE(13) KS_BWDS_CASE(14) KS_BWDS_CASE(15) KS_BWDS_CASE(16)
#undef KS_BWDS_CASE
        default: return KS_ERR_CUDA;
    }
}

// The stencils (MODE kFWD / kDXS) and dW (kDW) also take 16 < K <= 32 (the
// fused backward stays at K <= 16).
template <int MODE>
ks_status launch_any_k32(int64_t K, bool f, const CUtensorMap& im, const CUtensorMap& xm, const CUtensorMap& om,
                         const float* k, float* part, int64_t B, int64_t H, int64_t L, int G, float* out,
                         cudaStream_t st, int rpi = 0) {
    if (K <= 16) return launch_any_k<MODE>(K, f, im, xm, om, k, part, B, H, L, G, out, st, rpi);
    switch (K) {
#define KS_BWDS_CASE(KV) \
    case KV: return launch_m<KV, MODE>(f, im, xm, om, k, part, B, H, L, G, out, st, rpi);
        KS_BWDS_CASE(17) KS_BWDS_CASE(18) KS_BWDS_CASE(19) KS_BWDS_CASE(20) KS_BWDS_CASE(21) KS_BWDS_CASE(22)
        KS_BWDS_CASE(23) KS_BWDS_CASE(24) KS_BWDS_CASE(25) KS_BWDS_CASE(26) KS_BWDS_CASE(27) KS_BWDS_CASE(28)
        KS_BWDS_CASE(29) KS_BWDS_CASE(30) KS_BWDS_CASE(31) KS_BWDS_CASE(32)
#undef KS_BWDS_CASE
        default: return KS_ERR_CUDA;
    }
}

// Stencil outputs straight from registers (one 256-bit store = one 32-byte
// sector per thread and block) instead of a TMA store of the staged tile.
// An A/B knob, off by default: on the B200 (tools/time_paths.py, bench.py)
// direct stores won at (256,512,8192,K >= 11) (K = 16: fwd 1.49 -> 1.38 ms)
// but lost at K <= 9 (K = 7: 1.45 -> 1.49 ms), in the fused backward (K = 16:
// 1.89 -> 2.22 ms) and at config 5a's full size (fwd 11.1 -> 13.4 ms in the
// bench, ABAB).  KS_DST=1 turns them on (both paths give the same bits).
inline bool direct_store(const float* out) {
    return opt(kOptDst) > 0 && (reinterpret_cast<uintptr_t>(out) & 31) == 0;
}

inline bool shape_ok(int64_t B, int64_t H, int64_t L, int64_t K) {
    return K >= 1 && K <= 32 && L % 32 == 0 && B * H < (int64_t(1) << 31) && L < (int64_t(1) << 30);
}

// dW (DX = false) or the fused backward (DX = true).  *handled = false: shape
// or alignment outside the envelope (the caller falls back to dw_tma).
template <bool DX>
ks_status launch_bwd_short(const float* gy, const float* x, const float* k, float* dx, float* part, int64_t B,
                           int64_t H, int64_t L, int64_t K, int G, int mode, cudaStream_t st, bool* handled) {
    *handled = false;
    if (!shape_ok(B, H, L, K) || (DX && K > 16) || int64_t(G) * H >= (int64_t(1) << 31)) return KS_OK;
    CUtensorMap gm, xm, dm;
    if constexpr (!DX) {
        // rows shorter than a 2048-wide item: items of RPI whole rows of the
        // CTA's channel ({32, L/32, H, B} view, one box per tensor per item)
        if (L < kTT && opt(kOptDwMrow) != 0) {
            const int npr = static_cast<int>(L / 32);
            const int rpi = std::min(kMaxRPI, 64 / npr);
            if (!encode_padded_view(&gm, gy, B * H, L, H, npr, 1, rpi)) return KS_OK;
            if (!encode_padded_view(&xm, x, B * H, L, H, npr + 2, 1, rpi)) return KS_OK;
            *handled = true;
            return launch_any_k32<kDW | kMRow>(K, true, gm, xm, gm, k, part, B, H, L, G, nullptr, st, rpi);
        }
    }
    if (!encode_row_view_padded(&gm, gy, B * H, L, DX ? 66 : 64)) return KS_OK;
    if (!encode_row_view_padded(&xm, x, B * H, L, kXP)) return KS_OK;
    if constexpr (DX) {
        if (!encode_row_view(&dm, dx, B * H, L, 32, kTT / 32, 128)) return KS_OK;
    } else {
        dm = gm;  // unused
    }
    *handled = true;
    const bool f = mode == KS_MULADD_FUSED;
    if constexpr (!DX) return launch_any_k32<kDW>(K, f, gm, xm, dm, k, part, B, H, L, G, nullptr, st);
    else return direct_store(dx) ? launch_any_k<kFUSED | kDirect>(K, f, gm, xm, dm, k, part, B, H, L, G, dx, st)
                            : launch_any_k<kFUSED>(K, f, gm, xm, dm, k, part, B, H, L, G, dx, st);
}

}  // namespace bwds
}  // namespace ks
