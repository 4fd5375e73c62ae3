// bwd_short_st.cu -- forward / dX stencils for K <= 16, specialised on K;
// kernel and design in bwd_short.cuh.
#include "bwd_short_impl.cuh"

namespace ks {

ks_status stencil_short_f32(const float* in, const float* k, float* out, int64_t B, int64_t H, int64_t L, int64_t K,
                            int64_t off, int reverse, int mode, cudaStream_t st, bool* handled) {
    return bwds::launch_stencil_short(in, k, out, B, H, L, K, off, reverse, mode, st, handled);
}

}  // namespace ks
