// bwd_short_st.cu -- forward / dX stencils for K <= 16, specialised on K;
// kernel and design in bwd_short.cuh.
#include "bwd_short_impl.cuh"

namespace ks {
namespace bwds {

// Forward (reverse = 0, off = p) or dX (reverse = 1, off = q) stencil.
static ks_status launch_stencil_short(const float* in, const float* k, float* out, int64_t B, int64_t H, int64_t L,
                                      int64_t K, int64_t off, int reverse, int mode, cudaStream_t st,
                                      bool* handled) {
    *handled = false;
    // stencils: 1 <= K <= 32 (the shape envelope of dW / the fused backward is K <= 16)
    if (!shape_ok(B, H, L, K) || off != (reverse ? K - 1 - K / 2 : K / 2))
        return KS_OK;
    CUtensorMap im, om;
    if (!encode_row_view_padded(&im, in, B * H, L, 66)) return KS_OK;
    if (!encode_row_view(&om, out, B * H, L, 32, kTT / 32, 128)) return KS_OK;
    const int64_t nw = K <= 16 ? 16 : 32;  // Geo::NW
    float* kp = nullptr;
    ks_status rc = cuda_status(scratch_alloc(reinterpret_cast<void**>(&kp), sizeof(float) * H * nw, st));
    if (rc != KS_OK) return rc;
    *handled = true;
    launch_kernel(prep_taps, static_cast<unsigned>(std::min<int64_t>((H * nw + 255) / 256, 4096)), 256, 0, st, k, kp, H, K,
                  nw, reverse, 0);
    rc = check_launch();
    if (rc == KS_OK) {
        const bool f = mode == KS_MULADD_FUSED;
        if (direct_store(out))
            rc = reverse ? launch_any_k32<kDXS | kDirect>(K, f, im, im, om, kp, nullptr, B, H, L, 1, out, st)
                         : launch_any_k32<kFWD | kDirect>(K, f, im, im, om, kp, nullptr, B, H, L, 1, out, st);
        else
            rc = reverse ? launch_any_k32<kDXS>(K, f, im, im, om, kp, nullptr, B, H, L, 1, out, st)
                         : launch_any_k32<kFWD>(K, f, im, im, om, kp, nullptr, B, H, L, 1, out, st);
    }
    scratch_free(kp, st);
    return rc;
}

}  // namespace bwds

ks_status stencil_short_f32(const float* in, const float* k, float* out, int64_t B, int64_t H, int64_t L, int64_t K,
                            int64_t off, int reverse, int mode, cudaStream_t st, bool* handled) {
    return bwds::launch_stencil_short(in, k, out, B, H, L, K, off, reverse, mode, st, handled);
}

}  // namespace ks
