// bwd_short.cuh -- short-kernel (K <= 16) weight gradient and fused backward,
// fully specialised on K (sm_100a).  Included by bwd_short_dw.cu (dW only) and
// bwd_short_dx.cu (dX + dW in one pass).
//
//   dk[h,j] = sum_b sum_t gy[b,h,t] * x[b,h,t+j-p]    (reference src/conv_core.cpp:148-181)
//   dx[b,h,t] = sum_j gy[b,h,t+j-q] * k[h,K-1-j]       (reference src/conv_core.cpp:48-75)
//
// Same decomposition and association order as dw_tma (dw_tma.cu) -- CTA =
// (row group, channel), 256 threads, work items = (row, 2048-wide t tile) in
// flat order, thread (warp w, lane l) owns the 8-wide t block at
// tl = 32 l + 8 (w & 3) + 1024 (w >> 2), ascending-t FMA chains per tap, the
// same xor-shuffle / warp tree -- so dk is bit-identical to the dW-only call
// and dx to the stencil.  What changes is the instruction stream around the
// FMAs, which ncu showed was half of the issued instructions at K = 16
// (the fused backward at config 5a was issue-bound at 82% of slots):
//
// * K, p, q and every window offset are template constants: no tap-count
//   branches, no runtime sub-quad offsets.
// * gy and x land through the padded row view (encode_row_view_padded: box
//   {36, n} over 32-float pieces, 128-byte global rows): every 32-float piece
//   is a 36-float shared row, so a thread's quads sit at
//   (piece * 144 + compile-time) bytes and every LDS.128 is [base + imm] --
//   conflict-free (lanes 144 B apart) with no swizzle arithmetic.  The column
//   8 (w & 3) is made compile-time by one warp-uniform switch at entry.
// * The fused kernel takes the 8 gy values of the dW block from the dX
//   window it already holds (the dX window of a block covers gy[t, t+8)).
// * Stage / phase / (row, tile) are carried incrementally: no integer
//   divisions in the item loop.
#pragma once

#include "ks_common.cuh"
#include "ks_tma.cuh"

namespace ks {
namespace bwds {

constexpr int kThreads = 256;
constexpr int kTT = 2048;                // t per work item
constexpr int kPitch = 144;              // bytes per padded 32-float piece
constexpr int kXP = 66;                  // x window pieces (2048 + taps + register overrun)
constexpr int kXRegion = (kXP * kPitch + 127) / 128 * 128;  // 9600
constexpr int kOutBytes = kTT * 4;       // one dX tile, 128B-swizzled rows

template <int KT, bool DX>
struct Geo {
    static constexpr int p = KT / 2;
    static constexpr int q = KT - 1 - p;                  // dX offset (src/conv_core.cpp:56)
    static constexpr int D = (32 - p % 32) % 32;          // x window origin t0 - p - D on a piece
    static constexpr int A = D & ~3;
    static constexpr int S = D & 3;                       // (-p) mod 4
    static constexpr int XR0 = (p + D) / 32;              // x window first piece = t0/32 - XR0
    static constexpr int S2 = (4 - q % 4) % 4;            // (-q) mod 4
    static constexpr int QS = q + S2;                     // multiple of 4
    static constexpr int NVX = (S + 8 + KT - 1 + 3) / 4;  // x quads per block
    static constexpr int NV2 = (S2 + 8 + KT - 1 + 3) / 4; // dX window quads per block
    static constexpr int GYP = DX ? 66 : 64;              // gy pieces (DX: one halo piece each side)
    static constexpr int GYRegion = (GYP * kPitch + 127) / 128 * 128;
    static constexpr int Stage = GYRegion + kXRegion;
    static constexpr int NS = KT <= 8 ? 4 : 3;            // as dw_tma: 4 stages when the FMAs are light
    static constexpr uint32_t TX = static_cast<uint32_t>((GYP + kXP) * kPitch);
    static constexpr int Smem = (DX ? 2 * kOutBytes : 0) + NS * Stage + 64 + 1024;
    static_assert(QS % 4 == 0 && QS + 8 <= 4 * NV2, "gy block inside the dX window");
    static_assert(A + 2040 + 4 * NVX <= kXP * 32, "x window inside the staged pieces");
};

// byte offset of the quad at logical index e (>= 0, 4-aligned) from a piece base
__host__ __device__ constexpr int pofs(int e) { return (e >> 5) * kPitch + (e & 31) * 4; }

template <int KT, bool FUSED, bool DX, int C0>
__device__ __forceinline__ void run(const CUtensorMap* gy_map, const CUtensorMap* x_map, const CUtensorMap* dx_map,
                                    const float* __restrict__ k, float* __restrict__ part, unsigned char* smem,
                                    uint64_t* full, float (*red)[KT], int H, int L, int h, int grp, int b_begin,
                                    int b_end) {
    using Gm = Geo<KT, DX>;
    constexpr int NS = Gm::NS;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int ntt = (L + kTT - 1) / kTT;
    const int nunits = (b_end - b_begin) * ntt;
    unsigned char* stages = smem + (DX ? 2 * kOutBytes : 0);

    // producer state (thread 0): next item to load
    int ib = b_begin, it0 = 0;
    auto issue = [&](int stage) {
        uint64_t* bar = &full[stage];
        mbar_arrive_expect_tx(bar, Gm::TX);
        const int row = ib * H + h;
        tma_load_3d(stages + stage * Gm::Stage, gy_map, 0, it0 / 32 - (DX ? 1 : 0), row, bar);
        tma_load_3d(stages + stage * Gm::Stage + Gm::GYRegion, x_map, 0, it0 / 32 - Gm::XR0, row, bar);
        it0 += kTT;
        if (it0 >= L) {
            it0 = 0;
            ++ib;
        }
    };
    if (tid == 0)
        for (int s = 0; s < NS && s < nunits; ++s) issue(s);

    float wr[DX ? KT : 1];
    if constexpr (DX) {
#pragma unroll
        for (int jj = 0; jj < KT; ++jj) wr[jj] = k[static_cast<int64_t>(h) * KT + KT - 1 - jj];
    }
    float acc[KT];
#pragma unroll
    for (int i = 0; i < KT; ++i) acc[i] = 0.f;

    const int R = lane + 32 * (warp >> 2);  // piece of this thread's block within the tile
    const unsigned char* tb = stages + R * kPitch;
    // dX tile: 128B-swizzled rows of 32 floats, this thread's 8 outputs at row R, quads C0/4, C0/4+1
    const uint32_t o0 = static_cast<uint32_t>(R * 128 + (((C0 / 4) ^ (R & 7)) << 4));
    const uint32_t o1 = static_cast<uint32_t>(R * 128 + (((C0 / 4 + 1) ^ (R & 7)) << 4));

    int stage = 0, t0 = 0, b = b_begin;
    uint32_t phase = 0;
    for (int u = 0; u < nunits; ++u) {
        mbar_wait(&full[stage], phase);
        const unsigned char* gys = tb + stage * Gm::Stage;
        const unsigned char* xs = gys + Gm::GYRegion;
        unsigned char* ob = smem + (u & 1) * kOutBytes;
        if (t0 + 32 * R < L) {
            float gv[8];
            if constexpr (DX) {
                // dx[t0+tl+r] = sum_j gy[t0+tl+r+j-q] * k[K-1-j], j ascending from +0;
                // window quad c = gy logical (t0-32 origin) 32 + tl - QS + 4c
                float v2[4 * Gm::NV2];
#pragma unroll
                for (int c = 0; c < Gm::NV2; ++c) {
                    const float4 qv = lds4(gys + pofs(32 + C0 - Gm::QS + 4 * c));
                    v2[4 * c + 0] = qv.x;
                    v2[4 * c + 1] = qv.y;
                    v2[4 * c + 2] = qv.z;
                    v2[4 * c + 3] = qv.w;
                }
                float d[8];
#pragma unroll
                for (int r = 0; r < 8; ++r) d[r] = 0.f;
#pragma unroll
                for (int jj = 0; jj < KT; ++jj)
#pragma unroll
                    for (int r = 0; r < 8; ++r) d[r] = muladd<FUSED>(d[r], v2[Gm::S2 + r + jj], wr[jj]);
                *reinterpret_cast<float4*>(ob + o0) = make_float4(d[0], d[1], d[2], d[3]);
                *reinterpret_cast<float4*>(ob + o1) = make_float4(d[4], d[5], d[6], d[7]);
#pragma unroll
                for (int tt = 0; tt < 8; ++tt) gv[tt] = v2[Gm::QS + tt];
            } else {
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const float4 qv = lds4(gys + pofs(C0 + 4 * c));
                    gv[4 * c + 0] = qv.x;
                    gv[4 * c + 1] = qv.y;
                    gv[4 * c + 2] = qv.z;
                    gv[4 * c + 3] = qv.w;
                }
            }
            // dW: x logical (origin t0 - p - D) A + tl + 4c; acc[jj] += gy[t] * x[t + jj - p]
            float xv[4 * Gm::NVX];
#pragma unroll
            for (int c = 0; c < Gm::NVX; ++c) {
                const float4 qv = lds4(xs + pofs(Gm::A + C0 + 4 * c));
                xv[4 * c + 0] = qv.x;
                xv[4 * c + 1] = qv.y;
                xv[4 * c + 2] = qv.z;
                xv[4 * c + 3] = qv.w;
            }
#pragma unroll
            for (int tt = 0; tt < 8; ++tt)
#pragma unroll
                for (int jj = 0; jj < KT; ++jj) acc[jj] = muladd<FUSED>(acc[jj], gv[tt], xv[Gm::S + tt + jj]);
        }
        if constexpr (DX) {
            fence_proxy_async_smem();           // dX tile visible to the TMA store
            if (tid == 0) bulk_wait_read_all();  // store u-1 has read buffer (u+1)&1
        }
        __syncthreads();
        if (tid == 0) {
            if constexpr (DX) {
                tma_store_3d(dx_map, ob, 0, t0 / 32, b * H + h);  // columns past L are clipped
                bulk_commit();
            }
            if (u + NS < nunits) issue(stage);
        }
        if (++stage == NS) {
            stage = 0;
            phase ^= 1u;
        }
        t0 += kTT;
        if (t0 >= L) {
            t0 = 0;
            ++b;
        }
    }
    if (DX && tid == 0) bulk_wait_all();

    // fixed xor-shuffle tree per warp, then the 8 warps in ascending order (as dw_tma)
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
        for (int w = 0; w < kThreads / 32; ++w) s += red[w][tid];
        part[(static_cast<int64_t>(grp) * H + h) * KT + tid] = s;
    }
}

template <int KT, bool FUSED, bool DX>
__global__ void __launch_bounds__(kThreads, 3)  // 3 CTAs per SM: <= 80 registers
bwd_short(const __grid_constant__ CUtensorMap gy_map, const __grid_constant__ CUtensorMap x_map,
          const __grid_constant__ CUtensorMap dx_map, const float* __restrict__ k, float* __restrict__ part, int B,
          int H, int L, int G) {
    using Gm = Geo<KT, DX>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = align_smem<1024>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (DX ? 2 * kOutBytes : 0) + Gm::NS * Gm::Stage);
    __shared__ float red[kThreads / 32][KT];

    const int h = blockIdx.x % H;
    const int grp = blockIdx.x / H;
    const int b_begin = static_cast<int>(static_cast<int64_t>(B) * grp / G);
    const int b_end = static_cast<int>(static_cast<int64_t>(B) * (grp + 1) / G);
    if (threadIdx.x == 0) {
        prefetch_tmap(&gy_map);
        prefetch_tmap(&x_map);
        if (DX) prefetch_tmap(&dx_map);
        for (int s = 0; s < Gm::NS; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    switch ((threadIdx.x >> 5) & 3) {  // warp-uniform: the block's column 8 (w & 3) becomes a constant
        case 0: run<KT, FUSED, DX, 0>(&gy_map, &x_map, &dx_map, k, part, smem, full, red, H, L, h, grp, b_begin, b_end); break;
        case 1: run<KT, FUSED, DX, 8>(&gy_map, &x_map, &dx_map, k, part, smem, full, red, H, L, h, grp, b_begin, b_end); break;
        case 2: run<KT, FUSED, DX, 16>(&gy_map, &x_map, &dx_map, k, part, smem, full, red, H, L, h, grp, b_begin, b_end); break;
        default: run<KT, FUSED, DX, 24>(&gy_map, &x_map, &dx_map, k, part, smem, full, red, H, L, h, grp, b_begin, b_end); break;
    }
}

// Host launcher for one K: maps, smem opt-in, launch.
template <bool DX>
ks_status launch_bwd_short(const float* gy, const float* x, const float* k, float* dx, float* part, int64_t B,
                           int64_t H, int64_t L, int64_t K, int G, int mode, cudaStream_t st);

}  // namespace bwds
}  // namespace ks
