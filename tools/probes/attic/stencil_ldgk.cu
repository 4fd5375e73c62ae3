// ATTIC (not built): measured ~2x slower than stencil_pad on every compute-bound config
// (tools/gpu_runs/gpu_run85.sh: config 4 fwd 8.60 vs 4.56 ms) -- lanes own 16 outputs, so each
// 128-bit window load spreads a warp over 2 KB and L1 (not the FMA pipe) becomes the limiter.
// stencil_ldgk.cu -- forward / dX for long kernels (K > 16) from register
// windows with the taps in uniform registers (no staging ring).
//
//   out[b,h,t] = sum_{j<K} in[b,h,t+j-off] * w[h,j]     (reference src/conv_core.cpp:21-75)
//
// A thread owns R = 16 consecutive outputs of one row; the CTA (256 threads)
// covers 4096 outputs of that row.  Taps are walked in blocks of 16: per
// block the thread loads its 32-float input window with eight 128-bit loads
// (neighbouring threads' windows overlap; L1 / L2 serve the overlap) and the
// block's 16 taps -- the same for every thread of the CTA, so the compiler
// can keep them in uniform registers -- and issues 256 FFMAs in anti-diagonal
// order (the window value stays in the operand-reuse cache), so an FFMA reads
// one operand, the accumulator, from the register file: no even/odd bank
// conflicts, the limiter of the shared-memory kernels.
//
// The taps are prepared with Z = (-off) mod 4 leading zeros (prep_taps), so
// every window starts on a float4; a zero tap adds x*0 = +-0 to a chain that
// starts at +0, which never changes it, and input quads outside the row are
// zero -- the reference's padding.  Each output is the reference's
// ascending-j chain from +0: bit-identical to the reference and to the other
// stencils.  Tap blocks that read only zero padding for a whole warp (its
// 512-output span) are skipped, as in stencil_pad.
#include <algorithm>
#include <cstdlib>

#include "ks_common.cuh"

namespace ks {

__global__ void prep_taps(const float*, float*, int64_t, int64_t, int64_t, int, int);

namespace {

constexpr int kR = 16;      // outputs per thread
constexpr int kJB = 16;     // taps per block
constexpr int kNT = 256;    // threads per CTA
constexpr int kNQ = (kR + kJB - 1 + 3) / 4;  // 8 window quads per block

__device__ __forceinline__ void st_v8(float* p, float a0, float a1, float a2, float a3, float a4, float a5, float a6,
                                      float a7) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(a0), "f"(a1), "f"(a2), "f"(a3),
                 "f"(a4), "f"(a5), "f"(a6), "f"(a7)
                 : "memory");
}

template <bool FUSED>
__global__ void __launch_bounds__(kNT)
stencil_ldgk(const float* __restrict__ in, const float* __restrict__ kp, float* __restrict__ out, int tpr, int H,
             int L, int Kp, int offz, int nblk_total) {
    const int row = static_cast<int>(blockIdx.x) / tpr;
    const int t0 = (static_cast<int>(blockIdx.x) - row * tpr) * (kNT * kR);
    const int t = t0 + kR * static_cast<int>(threadIdx.x);
    const int h = row % H;
    const float* xr = in + static_cast<int64_t>(row) * L;
    const float* wr = kp + static_cast<int64_t>(h) * Kp;
    // the warp's outputs [tw, tw + 512): keep tap blocks whose window
    // [tw + 16 jb - offz, tw + 511 + 16 jb - offz + 15] reaches [0, L)
    // (broadcast from lane 0 so the compiler can prove the block range -- and
    // with it the tap addresses -- warp-uniform)
    const int tw = __shfl_sync(0xffffffffu, t0 + kR * (static_cast<int>(threadIdx.x) & ~31), 0);
    const int jb_lo = max(0, (offz - 15 - (tw + 32 * kR - 1) + 15 + 16 * 4096) / 16 - 4096);
    const int jb_hi = min(nblk_total, (L + offz - tw + 15) / 16);
    float acc[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) acc[r] = 0.f;
    for (int jb = jb_lo; jb < jb_hi; ++jb) {
        const int a0 = t + kJB * jb - offz;  // 4-aligned
        float v[4 * kNQ];
#pragma unroll
        for (int c = 0; c < kNQ; ++c) {
            const int s = a0 + 4 * c;
            float4 q = make_float4(0.f, 0.f, 0.f, 0.f);  // quads wholly in or out of the row (L % 4 == 0)
            if (s >= 0 && s < L) q = __ldg(reinterpret_cast<const float4*>(xr + s));
            v[4 * c + 0] = q.x;
            v[4 * c + 1] = q.y;
            v[4 * c + 2] = q.z;
            v[4 * c + 3] = q.w;
        }
        float w[kJB];
#pragma unroll
        for (int c = 0; c < kJB / 4; ++c) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(wr + kJB * jb) + c);
            w[4 * c + 0] = q.x;
            w[4 * c + 1] = q.y;
            w[4 * c + 2] = q.z;
            w[4 * c + 3] = q.w;
        }
        // anti-diagonal: m = r + jj; acc[r] still sees jj ascending
#pragma unroll
        for (int m = 0; m < kR + kJB - 1; ++m)
#pragma unroll
            for (int r = 0; r < kR; ++r) {
                const int jj = m - r;
                if (jj >= 0 && jj < kJB) acc[r] = muladd<FUSED>(acc[r], v[m], w[jj]);
            }
    }
    if (t < L) {
        float* o = out + static_cast<int64_t>(row) * L + t;
        st_v8(o, acc[0], acc[1], acc[2], acc[3], acc[4], acc[5], acc[6], acc[7]);
        st_v8(o + 8, acc[8], acc[9], acc[10], acc[11], acc[12], acc[13], acc[14], acc[15]);
    }
}

}  // namespace

// Opt-in (KS_LDGK=1) while being measured: K > 16, L % 16 == 0, 16-byte input
// and 32-byte output bases.  *handled = false otherwise.
ks_status stencil_ldgk_f32(const float* in, const float* k, float* out, int64_t B, int64_t H, int64_t L, int64_t K,
                           int64_t off, int reverse, int mode, cudaStream_t st, bool* handled) {
    *handled = false;
    const char* e = getenv("KS_LDGK");
    if (!(e && *e == '1')) return KS_OK;
    if (K <= 16 || K > 8192 || L % 16 != 0 || L >= (int64_t(1) << 30)) return KS_OK;
    if ((reinterpret_cast<uintptr_t>(in) & 15) != 0 || (reinterpret_cast<uintptr_t>(out) & 31) != 0) return KS_OK;
    const int tpr = static_cast<int>((L + kNT * kR - 1) / (kNT * kR));
    if (B * H * tpr >= (int64_t(1) << 31)) return KS_OK;
    const int Z = static_cast<int>((4 - off % 4) % 4);
    const int64_t Kp = (K + Z + kJB - 1) / kJB * kJB;
    float* kp = nullptr;
    ks_status rc = cuda_status(scratch_alloc(reinterpret_cast<void**>(&kp), sizeof(float) * H * Kp, st));
    if (rc != KS_OK) return rc;
    *handled = true;
    prep_taps<<<static_cast<unsigned>(std::min<int64_t>((H * Kp + 255) / 256, 4096)), 256, 0, st>>>(k, kp, H, K, Kp,
                                                                                                   reverse, Z);
    rc = check_launch();
    if (rc == KS_OK) {
        const unsigned grid = static_cast<unsigned>(B * H * tpr);
        const int offz = static_cast<int>(off) + Z;
        const int nb = static_cast<int>(Kp / kJB);
        if (mode == KS_MULADD_FUSED)
            stencil_ldgk<true><<<grid, kNT, 0, st>>>(in, kp, out, tpr, static_cast<int>(H), static_cast<int>(L),
                                                     static_cast<int>(Kp), offz, nb);
        else
            stencil_ldgk<false><<<grid, kNT, 0, st>>>(in, kp, out, tpr, static_cast<int>(H), static_cast<int>(L),
                                                      static_cast<int>(Kp), offz, nb);
        rc = check_launch();
    }
    scratch_free(kp, st);
    return rc;
}

}  // namespace ks
