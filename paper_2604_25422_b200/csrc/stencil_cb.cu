// stencil_cb.cu -- compute-bound forward / dX (long K), sm_100a.
//
//   out[b,h,t] = sum_{j=0}^{K-1} in[b,h,t+j-off] * w[h,j]   (reference src/conv_core.cpp:21-75)
//
// At K >= 64 the stencil is FP32-FMA-bound (arithmetic intensity ~K/4 FLOP/B
// against a ~11 FLOP/B ridge), so the kernel is built to keep the FMA pipe
// issuing:
//   * TMA brings the input window and the channel's taps into a staging stage
//     (zero fill outside the row = the reference's zero padding);
//   * the CTA re-lays the window out once per tile into a padded buffer
//     (4 floats of padding per 32, shifted so output 0's first tap sits at
//     index 0) and copies the taps, then releases the stage so the next tile's
//     TMA load overlaps this tile's math;
//   * each thread owns R = 32 consecutive outputs (padded rows 144 B apart:
//     conflict-free 128-bit reads) and walks the taps in 32-tap iterations of
//     two 16-tap register windows whose shared-memory offsets are compile-time
//     immediates -- 512 FMAs per 12 window loads + 4 tap loads, no address math
//     in the inner loop;
//   * taps accumulate in ascending j from +0 (fmaf or mul+add), so results are
//     bit-identical to the reference; tail taps past K are predicated off.
#include <algorithm>
#include <cstdlib>

#include "ks_common.cuh"
#include "ks_tma.cuh"

namespace ks {

__global__ void prep_taps(const float*, float*, int64_t, int64_t, int64_t, int, int);

namespace {

constexpr int kR = 32;    // outputs per thread
constexpr int kJS = 16;   // taps per register window
constexpr int kIn = 32;   // floats per TMA row piece
constexpr int kNV = (kR + kJS - 1 + 3) / 4;  // float4 loads per window (12)

struct CbGeom {
    int T;            // outputs per tile (NT*R)
    int HH;           // halo rows (32 floats) on each side
    int NB, nbox;     // input boxes per stage
    int D0;           // 32*HH - off: staging index of output 0's first tap
    int Kp;           // taps padded to a multiple of 32
    int WL;           // logical window length re-laid out (multiple of 32)
    int win_bytes;    // staged window bytes
    int stage_bytes;  // staging stage (window + taps), 1024-aligned
    int pw_floats;    // padded window floats
};

__device__ __forceinline__ int padi(int i) { return i + ((i >> 5) << 2); }

// One thread's R = 32 outputs of a tile: acc[r] = sum_j pw[padi(pbase' + r + j)] * wk[j]
// in ascending j from +0, over the padded window `pw` (thread's first tap at
// padded index pbase) and the channel's taps `wk` (Kp floats, zero past K).
template <bool FUSED>
__device__ __forceinline__ void cb_tile(const float* pw, const float* wk, int pbase, int K, float (&acc)[kR]) {
#pragma unroll
    for (int r = 0; r < kR; ++r) acc[r] = 0.f;
    // one 16-tap register window (compile-time sub-offsets), taps w16[0 .. 16),
    // `nj` of them live; `base` = padded address of a 32-aligned logical index;
    // the window starts `sub` (0 or 16, a literal) floats later
    auto window = [&](const float* base, const int sub, const float* w16, int nj) {
        float v[4 * kNV];
#pragma unroll
        for (int c = 0; c < kNV; ++c) {
            const float4 q = *reinterpret_cast<const float4*>(base + sub + 4 * c + (((sub + 4 * c) >> 5) << 2));
            v[4 * c + 0] = q.x;
            v[4 * c + 1] = q.y;
            v[4 * c + 2] = q.z;
            v[4 * c + 3] = q.w;
        }
        float w[kJS];
#pragma unroll
        for (int c = 0; c < kJS / 4; ++c) {
            const float4 q = *reinterpret_cast<const float4*>(w16 + 4 * c);
            w[4 * c + 0] = q.x;
            w[4 * c + 1] = q.y;
            w[4 * c + 2] = q.z;
            w[4 * c + 3] = q.w;
        }
#pragma unroll
        for (int jj = 0; jj < kJS; ++jj)
            if (jj < nj) {
#pragma unroll
                for (int r = 0; r < kR; ++r) acc[r] = muladd<FUSED>(acc[r], v[r + jj], w[jj]);
            }
    };
    // 32 taps per iteration: windows at logical base + j0 and + j0 + 16.
    // logical base + j0 is a multiple of 32, so its padded address is
    // pbase + j0*36/32 and the +16 window starts 16 floats further.
    const int Kfull = K & ~31;
    for (int j0 = 0; j0 < Kfull; j0 += 32) {
        const float* b0 = pw + pbase + (j0 >> 5) * 36;
        window(b0, 0, wk + j0, kJS);
        window(b0, 16, wk + j0 + 16, kJS);
    }
    if (Kfull < K) {
        const float* b0 = pw + pbase + (Kfull >> 5) * 36;
        const int rem = K - Kfull;
        window(b0, 0, wk + Kfull, rem < kJS ? rem : kJS);
        if (rem > kJS) window(b0, 16, wk + Kfull + 16, rem - kJS);
    }
}

template <int NT, bool FUSED>
__global__ void __launch_bounds__(NT)
stencil_cb(const __grid_constant__ CUtensorMap in_map, const float* __restrict__ kp, float* __restrict__ out, int H,
           int L, int K, int tiles_per_row, int ntiles, CbGeom g) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = align_smem<1024>(smem_raw);
    const float* stage = reinterpret_cast<const float*>(smem);
    float* pw = reinterpret_cast<float*>(smem + g.stage_bytes);  // padded window
    float* wk = pw + g.pw_floats;                                // taps (Kp floats)
    uint64_t* full = reinterpret_cast<uint64_t*>(wk + g.Kp);
    const int tid = threadIdx.x;

    if (tid == 0) {
        prefetch_tmap(&in_map);
        mbar_init(full, 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint32_t tx_bytes = static_cast<uint32_t>(g.win_bytes + g.Kp * 4);
    auto issue = [&](int tile) {
        const int row = tile / tiles_per_row;
        const int t0 = (tile - row * tiles_per_row) * g.T;
        unsigned char* sb = smem;
        mbar_arrive_expect_tx(full, tx_bytes);
        const int r0 = t0 / kIn - g.HH;
        tma_load_3d(sb, &in_map, 0, r0, row, full);
        if (g.nbox > 1) tma_load_3d(sb + g.NB * 128, &in_map, 0, r0 + g.NB, row, full);
        bulk_load(sb + g.win_bytes, kp + static_cast<int64_t>(row % H) * g.Kp, static_cast<uint32_t>(g.Kp) * 4u, full);
    };
    if (tid == 0 && static_cast<int>(blockIdx.x) < ntiles) issue(blockIdx.x);

    const int win_floats = g.win_bytes / 4;
    const float* sk = stage + win_floats;
    const int pbase = tid * (kR + 4);  // padi(tid * 32)
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        mbar_wait(full, static_cast<uint32_t>(it & 1));
        // re-layout: pw[padi(i)] = staging[i + D0] (0 past the staged window)
        for (int i = tid; i < g.WL; i += NT) {
            const int s = i + g.D0;
            pw[padi(i)] = s < win_floats ? stage[s] : 0.f;
        }
        for (int j = tid; j < g.Kp; j += NT) wk[j] = sk[j];
        __syncthreads();  // staging consumed, padded window ready
        const int nt = tile + gridDim.x;
        if (tid == 0 && nt < ntiles) issue(nt);  // next load overlaps this tile's math

        const int row = tile / tiles_per_row;
        const int t0 = (tile - row * tiles_per_row) * g.T;
        if (t0 + tid * kR < L) {  // L % 32 == 0: a register tile is wholly in or out
            float acc[kR];
            cb_tile<FUSED>(pw, wk, pbase, K, acc);
            float* o = out + static_cast<int64_t>(row) * L + t0 + tid * kR;
#pragma unroll
            for (int r = 0; r < kR; r += 4) st_cs_v4(o + r, make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]));
        }
        __syncthreads();  // padded window and taps free for the next tile
    }
}

template <int NT, bool FUSED>
ks_status launch(const CUtensorMap& im, const float* kp, float* out, int64_t B, int64_t H, int64_t L, int64_t K,
                 const CbGeom& g, cudaStream_t st) {
    auto kern = stencil_cb<NT, FUSED>;
    const int smem = g.stage_bytes + (g.pw_floats + g.Kp) * 4 + 64 + 1024;
    const int per_sm = prepare_kernel(reinterpret_cast<const void*>(kern), NT, smem);
    const int tiles_per_row = static_cast<int>((L + g.T - 1) / g.T);
    const int ntiles = static_cast<int>(B * H * tiles_per_row);
    const int grid = std::min(ntiles, num_sms() * per_sm);
    kern<<<grid, NT, smem, st>>>(im, kp, out, static_cast<int>(H), static_cast<int>(L), static_cast<int>(K),
                                 tiles_per_row, ntiles, g);
    return check_launch();
}

}  // namespace

// Compute-bound fwd/dX (K > 32, L >= 2048, L % 32 == 0).  *handled = false
// when the shape is outside this kernel's envelope.
ks_status stencil_cb_f32(const float* in, const float* k, float* out, int64_t B, int64_t H, int64_t L, int64_t K,
                         int64_t off, int reverse, int mode, cudaStream_t st, bool* handled) {
    *handled = false;
    if (L % kIn != 0 || L < 2048 || L >= (int64_t(1) << 30) || K > 8192 || K <= 32) return KS_OK;
    if ((reinterpret_cast<uintptr_t>(out) & 15) != 0) return KS_OK;
    const int NT = L >= 8192 ? 256 : L >= 4096 ? 128 : 64;
    CbGeom g;
    g.T = NT * kR;
    const int64_t need = std::max<int64_t>(off, K - 1 - off);
    g.HH = static_cast<int>((need + kIn - 1) / kIn);
    if (g.HH == 0) g.HH = 1;
    const int W = g.T / kIn + 2 * g.HH;
    if (W <= 256) {
        g.nbox = 1;
        g.NB = W;
    } else if (W <= 512) {
        g.nbox = 2;
        g.NB = W / 2;
    } else {
        return KS_OK;
    }
    const int64_t ntiles = B * H * ((L + g.T - 1) / g.T);
    if (ntiles >= (int64_t(1) << 31)) return KS_OK;
    g.D0 = kIn * g.HH - static_cast<int>(off);
    g.Kp = static_cast<int>((K + 31) / 32 * 32);
    g.WL = g.T + g.Kp + 32;  // every padded index a thread can read
    g.win_bytes = g.nbox * g.NB * 128;
    g.stage_bytes = (g.win_bytes + g.Kp * 4 + 1023) / 1024 * 1024;
    g.pw_floats = (g.WL / 32) * 36;
    const int smem = g.stage_bytes + (g.pw_floats + g.Kp) * 4 + 64 + 1024;
    if (smem > 220 * 1024) return KS_OK;
    CUtensorMap im;
    if (!encode_row_view(&im, in, B * H, L, kIn, g.NB, 0)) return KS_OK;

    float* kp = nullptr;
    ks_status rc = cuda_status(scratch_alloc(reinterpret_cast<void**>(&kp), sizeof(float) * H * g.Kp, st));
    if (rc != KS_OK) return rc;
    prep_taps<<<static_cast<unsigned>(std::min<int64_t>((H * g.Kp + 255) / 256, 4096)), 256, 0, st>>>(
        k, kp, H, K, g.Kp, reverse, 0);
    rc = check_launch();
    if (rc == KS_OK) {
        const bool fused = mode == KS_MULADD_FUSED;
        if (NT == 256) rc = fused ? launch<256, true>(im, kp, out, B, H, L, K, g, st)
                                  : launch<256, false>(im, kp, out, B, H, L, K, g, st);
        else if (NT == 128) rc = fused ? launch<128, true>(im, kp, out, B, H, L, K, g, st)
                                       : launch<128, false>(im, kp, out, B, H, L, K, g, st);
        else rc = fused ? launch<64, true>(im, kp, out, B, H, L, K, g, st)
                        : launch<64, false>(im, kp, out, B, H, L, K, g, st);
    }
    scratch_free(kp, st);
    *handled = true;
    return rc;
}

}  // namespace ks
