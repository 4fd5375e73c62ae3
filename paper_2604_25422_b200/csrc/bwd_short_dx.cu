// bwd_short_dx.cu -- the fused backward (dX + HIERARCHICAL dW stage 1) for
// K <= 16, specialised on K; kernel and design in bwd_short.cuh.
#include "bwd_short_impl.cuh"

namespace ks {

ks_status bwd_short_fused_stage1(const float* gy, const float* x, const float* k, float* dx, float* part, int64_t B,
                                 int64_t H, int64_t L, int64_t K, int G, int mode, cudaStream_t st, bool* handled) {
    return bwds::launch_bwd_short<true>(gy, x, k, dx, part, B, H, L, K, G, mode, st, handled);
}

}  // namespace ks
