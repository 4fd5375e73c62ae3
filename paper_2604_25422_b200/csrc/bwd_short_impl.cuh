// bwd_short_impl.cuh -- host launcher of bwd_short (bwd_short.cuh) for one of
// the two kernel families; instantiated by bwd_short_dw.cu / bwd_short_dx.cu so
// the 2 x 16 x 2 specialisations compile in parallel.
#pragma once

#include "bwd_short.cuh"

namespace ks {

namespace bwds {

template <int KT, bool FUSED, bool DX>
ks_status launch_k(const CUtensorMap& gm, const CUtensorMap& xm, const CUtensorMap& dm, const float* k, float* part,
                   int64_t B, int64_t H, int64_t L, int G, cudaStream_t st) {
    auto kern = bwd_short<KT, FUSED, DX>;
    constexpr int smem = Geo<KT, DX>::Smem;
    prepare_kernel(reinterpret_cast<const void*>(kern), kThreads, smem);
    const unsigned blocks = static_cast<unsigned>(int64_t(G) * H);
    kern<<<blocks, kThreads, smem, st>>>(gm, xm, dm, k, part, static_cast<int>(B), static_cast<int>(H),
                                         static_cast<int>(L), G);
    return check_launch();
}

template <int KT, bool DX>
ks_status launch_m(bool fused, const CUtensorMap& gm, const CUtensorMap& xm, const CUtensorMap& dm, const float* k,
                   float* part, int64_t B, int64_t H, int64_t L, int G, cudaStream_t st) {
    return fused ? launch_k<KT, true, DX>(gm, xm, dm, k, part, B, H, L, G, st)
                 : launch_k<KT, false, DX>(gm, xm, dm, k, part, B, H, L, G, st);
}

template <bool DX>
ks_status launch_bwd_short(const float* gy, const float* x, const float* k, float* dx, float* part, int64_t B,
                           int64_t H, int64_t L, int64_t K, int G, int mode, cudaStream_t st, bool* handled) {
    *handled = false;
    if (K < 1 || K > 16 || L % 32 != 0 || B * H >= (int64_t(1) << 31) || L >= (int64_t(1) << 30) ||
        int64_t(G) * H >= (int64_t(1) << 31))
        return KS_OK;
    CUtensorMap gm, xm, dm;
    if (!encode_row_view_padded(&gm, gy, B * H, L, Geo<1, DX>::GYP)) return KS_OK;
    if (!encode_row_view_padded(&xm, x, B * H, L, kXP)) return KS_OK;
    if constexpr (DX) {
        if (!encode_row_view(&dm, dx, B * H, L, 32, kTT / 32, 128)) return KS_OK;
    } else {
        dm = gm;  // unused
    }
    *handled = true;
    const bool f = mode == KS_MULADD_FUSED;
    switch (K) {
#define KS_BWDS_CASE(KV) \
    case KV: return launch_m<KV, DX>(f, gm, xm, dm, k, part, B, H, L, G, st);
        KS_BWDS_CASE(1) KS_BWDS_CASE(2) KS_BWDS_CASE(3) KS_BWDS_CASE(4) KS_BWDS_CASE(5) KS_BWDS_CASE(6)
        KS_BWDS_CASE(7) KS_BWDS_CASE(8) KS_BWDS_CASE(9) KS_BWDS_CASE(10) KS_BWDS_CASE(11) KS_BWDS_CASE(12)
        KS_BWDS_CASE(13) KS_BWDS_CASE(14) KS_BWDS_CASE(15) KS_BWDS_CASE(16)
#undef KS_BWDS_CASE
        default: return KS_ERR_CUDA;
    }
}

}  // namespace bwds
}  // namespace ks
