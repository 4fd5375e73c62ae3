// bwd_short.cuh -- the short-kernel (K <= 16) paths, fully specialised on K
// (sm_100a): HIERARCHICAL dW stage 1, the fused backward (dX + dW in one pass),
// and the forward / dX stencils.  Instantiated by bwd_short_{dw,dx,st}.cu.
//
//   y[b,h,t]  = sum_j x[b,h,t+j-p] * k[h,j]             (reference src/conv_core.cpp:21-46)
//   dx[b,h,t] = sum_j gy[b,h,t+j-q] * k[h,K-1-j]        (src/conv_core.cpp:48-75)
//   dk[h,j]   = sum_b sum_t gy[b,h,t] * x[b,h,t+j-p]    (src/conv_core.cpp:148-181)
//
// Work items are (row, 2048-wide t tile); 256 threads, thread (warp w, lane l)
// owns the 8-wide t block at tl = 32 l + 8 (w & 3) + 1024 (w >> 2).  For dW
// this is dw_tma's decomposition (dw_tma.cu): CTA = (row group, channel),
// items in flat order, ascending-t FMA chains per tap, the same xor-shuffle /
// warp tree -- so dk is bit-identical to dw_tma's.  Every output of the
// stencils is the reference's ascending-j chain from +0 (zero-filled halo taps
// add +-0, which never changes a chain that starts at +0), so y and dx are
// bit-identical to the reference.  What this file changes is the instruction
// stream around the FMAs (half of all issued instructions at K = 16 in
// dw_tma, where the fused backward at config 5a was issue-bound at 82%):
//
// * K, p, q and every window offset are template constants: no tap-count
//   branches, no runtime sub-quad offsets.
// * Tiles land through the padded row view (encode_row_view_padded: box
//   {36, n} over 32-float pieces, 128-byte global rows): every piece is a
//   36-float shared row, so a thread's quads sit at (piece * 144 +
//   compile-time) bytes and every LDS.128 is [base + imm] -- conflict-free
//   (lanes 144 B apart) with no swizzle arithmetic.  The column 8 (w & 3) is
//   made compile-time by a warp-uniform switch around each item's math.
// * The fused kernel takes the 8 gy values of the dW block from the dX
//   window it already holds (the dX window of a block covers gy[t, t+8)).
// * Stage / phase / (row, tile) are carried incrementally: no integer
//   divisions in the item loop.
#pragma once

#include "ks_common.cuh"
#include "ks_tma.cuh"

// experiment knobs (compile-time; the defaults are the measured choice)
#ifndef KS_ST_NS
#define KS_ST_NS 4      // stencil stages
#endif
#ifndef KS_ST_MINB
#define KS_ST_MINB 4    // stencil CTAs per SM (launch bounds)
#endif
#ifndef KS_EVICT_FIRST
#define KS_EVICT_FIRST 0  // 1: TMA loads / stores carry an L2 evict_first policy
#endif
#ifndef KS_DW_NS_SHORT
#define KS_DW_NS_SHORT 4  // dW / fused backward stages, K <= 8
#endif
#ifndef KS_DW_NS_LONG
#define KS_DW_NS_LONG 3   // dW / fused backward stages, 8 < K <= 16
#endif
#ifndef KS_FUSED_NS_SHORT
#define KS_FUSED_NS_SHORT KS_DW_NS_SHORT  // fused backward stages, K <= 8
#endif

namespace ks {
namespace bwds {

// MODE: what a kernel instance computes
constexpr int kDW = 0;      // HIERARCHICAL dW stage 1 (part[G,H,K])
constexpr int kFUSED = 1;   // dX + dW stage 1 from one pass over gy and x
constexpr int kFWD = 2;     // forward stencil: out = x (*) k, offset p
constexpr int kDXS = 3;     // dX stencil: out = gy (*) reversed k, offset q
constexpr int kDirect = 8;  // | kDirect: stencil outputs go straight to HBM (one 256-bit store per 8 outputs)
constexpr int kMRow = 16;   // | kMRow (dW, L < 2048): an item is RPI whole rows of the CTA's channel, not one
                            //   2048-wide tile of one row (the tile would be mostly past the row end)
constexpr int kMaxRPI = 8;  // rows per multi-row item (L >= 256)

constexpr int kThreads = 256;
constexpr int kTT = 2048;                // t per work item
constexpr int kPitch = 144;              // bytes per padded 32-float piece
constexpr int kXP = 66;                  // window pieces (2048 + halo / taps + register overrun)
constexpr int kXRegion = (kXP * kPitch + 127) / 128 * 128;  // 9600
constexpr int kOutBytes = kTT * 4;       // one output tile, 128B-swizzled rows

template <int KT, int MODE>
struct Geo {
    static constexpr int BASE = MODE & 7;             // kDW / kFUSED / kFWD / kDXS
    static constexpr bool DST = (MODE & kDirect) != 0;  // stencil output stored straight from registers
    static constexpr bool MR = (MODE & kMRow) != 0;     // multi-row dW items
    static constexpr bool HAS_DW = BASE <= kFUSED;  // x window + dW accumulators
    static constexpr bool HAS_ST = BASE >= kFUSED;  // a stencil output tile per item
    static constexpr int p = KT / 2;
    static constexpr int q = KT - 1 - p;                  // dX offset (src/conv_core.cpp:56)
    static constexpr int D = (32 - p % 32) % 32;          // x window origin t0 - p - D on a piece
    static constexpr int A = D & ~3;
    static constexpr int S = D & 3;                       // (-p) mod 4
    static constexpr int XR0 = (p + D) / 32;              // x window first piece = t0/32 - XR0
    static constexpr int OFF = BASE == kFWD ? p : q;      // stencil offset
    static constexpr int S2 = (4 - OFF % 4) % 4;          // (-OFF) mod 4
    static constexpr int QS = OFF + S2;                   // multiple of 4
    static constexpr int NVX = (S + 8 + KT - 1 + 3) / 4;  // x quads per block
    static constexpr int NV2 = (S2 + 8 + KT - 1 + 3) / 4; // stencil window quads per block
    static constexpr int GYP = BASE == kDW ? 64 : 66;     // stencil input: one halo piece each side
    static constexpr int GYRegion = (GYP * kPitch + 127) / 128 * 128;
    static constexpr int NW = KT <= 16 ? 16 : 32;             // stencil taps per prepared row (kp stride)
    static constexpr int TapBytes = BASE >= kFWD ? 4 * 32 : 0;  // stencils: the row's NW taps ride in the stage
    // multi-row items: each row's x window carries its own two halo pieces
    static constexpr int XRegion = MR ? ((64 + 2 * kMaxRPI) * kPitch + 127) / 128 * 128 : kXRegion;
    static constexpr int Stage = GYRegion + (HAS_DW ? XRegion : 0) + TapBytes;
    static constexpr int NS = BASE >= kFWD ? KS_ST_NS
                              : MR ? 3
                              : KT <= 8 ? (BASE == kFUSED ? KS_FUSED_NS_SHORT : KS_DW_NS_SHORT)
                                        : KS_DW_NS_LONG;  // dW as dw_tma: 4 stages when FMAs are light
    static constexpr int MinBlocks = BASE >= kFWD ? KS_ST_MINB : KT > 16 ? 2 : 3;  // dW with 32 accumulators: 2
    static constexpr uint32_t TX =
        static_cast<uint32_t>(GYP * kPitch + (HAS_DW ? kXP * kPitch : 0) + (BASE >= kFWD ? 4 * NW : 0));
    static constexpr bool HAS_OBUF = HAS_ST && !DST;  // output tiles leave by TMA store from shared memory
    static constexpr int Smem = (HAS_OBUF ? 2 * kOutBytes : 0) + NS * Stage + 64 + 1024;
    static_assert(QS % 4 == 0 && QS + 8 <= 4 * NV2, "gy block inside the dX window");
    static_assert(A + 2040 + 4 * NVX <= kXP * 32, "x window inside the staged pieces");
    static_assert(!HAS_ST || 32 + 2040 - QS + 4 * NV2 <= GYP * 32, "stencil window inside the staged pieces");
};

// byte offset of the quad at logical index e (>= 0, 4-aligned) from a piece base
__host__ __device__ constexpr int pofs(int e) { return (e >> 5) * kPitch + (e & 31) * 4; }

// 256-bit global store (STG.E.256 on sm_100): 8 floats = one whole 32-byte sector
__device__ __forceinline__ void st_v8(float* p, const float (&d)[8]) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(d[0]), "f"(d[1]), "f"(d[2]),
                 "f"(d[3]), "f"(d[4]), "f"(d[5]), "f"(d[6]), "f"(d[7])
                 : "memory");
}

struct Args {
    int H, L;
    float* out;              // kDirect: the stencil output tensor
    int row0, rstep, nrows;  // this CTA's rows: row0 + i * rstep, i < nrows (row = b * H + h)
    int h;                   // dW modes: the CTA's channel
    int grp;                 // dW modes: the CTA's row group
    int npr, rpi;            // multi-row dW: pieces per row (L / 32), rows per item
    uint32_t tx;             // multi-row dW: bytes per item (both boxes)
};

// One work item's math for the thread whose block starts at column C0 of its
// piece (C0 = 8 (w & 3), a template constant so every shared access is
// [base + imm]); the caller switches on the warp-uniform column around this
// call only, so all warps meet the same barrier instructions.
template <int KT, bool FUSED, int MODE, int C0>
__device__ __forceinline__ void item(const unsigned char* gys, int xshift, unsigned char* ob, uint32_t o0, uint32_t o1,
                                     float* gout,
                                     const float (&w)[Geo<KT, MODE>::HAS_ST ? Geo<KT, MODE>::NW : 1],
                                     float (&acc)[Geo<KT, MODE>::HAS_DW ? KT : 1]) {
    using Gm = Geo<KT, MODE>;
    float gv[8];
    if constexpr (Gm::HAS_ST) {
        // out[t0+tl+r] = sum_j in[t0+tl+r+j-OFF] * w[j], j ascending from +0;
        // window quad c = input logical (t0-32 origin) 32 + tl - QS + 4c
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
            for (int r = 0; r < 8; ++r) d[r] = muladd<FUSED>(d[r], v2[Gm::S2 + r + jj], w[jj]);
        if constexpr (Gm::DST) {
            st_v8(gout, d);  // the block's 8 outputs = one whole 32-byte sector
        } else {
            *reinterpret_cast<float4*>(ob + o0) = make_float4(d[0], d[1], d[2], d[3]);
            *reinterpret_cast<float4*>(ob + o1) = make_float4(d[4], d[5], d[6], d[7]);
        }
        if constexpr (Gm::BASE == kFUSED) {
#pragma unroll
            for (int tt = 0; tt < 8; ++tt) gv[tt] = v2[Gm::QS + tt];
        }
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
    if constexpr (Gm::HAS_DW) {
        // dW: x logical (origin t0 - p - D) A + tl + 4c; acc[jj] += gy[t] * x[t + jj - p]
        const unsigned char* xs = gys + Gm::GYRegion + (Gm::MR ? xshift : 0);
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
            for (int jj = 0; jj < KT; ++jj) acc[jj] = muladd<true>(acc[jj], gv[tt], xv[Gm::S + tt + jj]);
    }
}

template <int KT, bool FUSED, int MODE>
__device__ __forceinline__ void run(const CUtensorMap* in_map, const CUtensorMap* x_map, const CUtensorMap* out_map,
                                    const float* __restrict__ k, float* __restrict__ part, unsigned char* smem,
                                    uint64_t* full, const Args a) {
    using Gm = Geo<KT, MODE>;
    constexpr int NS = Gm::NS;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int ntt = (a.L + kTT - 1) / kTT;
    const int nunits = Gm::MR ? (a.nrows + a.rpi - 1) / a.rpi : a.nrows * ntt;
    unsigned char* stages = smem + (Gm::HAS_OBUF ? 2 * kOutBytes : 0);

    // producer state (thread 0): next item to load
    int irow = a.row0, it0 = 0;
    auto issue = [&](int stage) {
        uint64_t* bar = &full[stage];
        unsigned char* sb = stages + stage * Gm::Stage;
        if constexpr (Gm::MR) {
            // RPI rows b .. b + RPI - 1 of channel h from the {32, L/32, H, B}
            // padded view: gy as NPR pieces per row, x as NPR + 2 pieces from
            // piece -XR0 (each row's own zero-filled halo)
            mbar_arrive_expect_tx(bar, a.tx);
            const int b = irow / a.H;
            tma_load_pad(sb, in_map, 0, a.h, b, bar);
            tma_load_pad(sb + Gm::GYRegion, x_map, -Gm::XR0, a.h, b, bar);
            irow += a.rpi * a.rstep;
            return;
        }
        mbar_arrive_expect_tx(bar, Gm::TX);
#if KS_EVICT_FIRST
        const uint64_t pol = policy_evict_first();
        tma_load_3d_hint(sb, in_map, 0, it0 / 32 - (Gm::BASE == kDW ? 0 : 1), irow, bar, pol);
        if constexpr (Gm::HAS_DW) tma_load_3d_hint(sb + Gm::GYRegion, x_map, 0, it0 / 32 - Gm::XR0, irow, bar, pol);
#else
        tma_load_3d(sb, in_map, 0, it0 / 32 - (Gm::BASE == kDW ? 0 : 1), irow, bar);
        if constexpr (Gm::HAS_DW) tma_load_3d(sb + Gm::GYRegion, x_map, 0, it0 / 32 - Gm::XR0, irow, bar);
#endif
        if constexpr (Gm::BASE >= kFWD)
            bulk_load(sb + Gm::GYRegion, k + static_cast<int64_t>(irow % a.H) * Gm::NW, 4 * Gm::NW, bar);
        it0 += kTT;
        if (it0 >= a.L) {
            it0 = 0;
            irow += a.rstep;
        }
    };
    if (tid == 0)
        for (int s = 0; s < NS && s < nunits; ++s) issue(s);

    // stencil taps: the fused backward holds the CTA's reversed row in
    // registers; the stencils read the row's prepared taps (prep_taps:
    // reversed for dX, zero past K) from each stage
    float w[Gm::HAS_ST ? Gm::NW : 1];
    if constexpr (Gm::BASE == kFUSED) {
#pragma unroll
        for (int jj = 0; jj < KT; ++jj) w[jj] = k[static_cast<int64_t>(a.h) * KT + KT - 1 - jj];
    }
    float acc[Gm::HAS_DW ? KT : 1];
#pragma unroll
    for (int i = 0; i < (Gm::HAS_DW ? KT : 1); ++i) acc[i] = 0.f;

    const int R = lane + 32 * (warp >> 2);  // piece of this thread's block within the tile
    const unsigned char* tb = stages + R * kPitch;
    // multi-row items: piece R is piece q of row ri of the item (gy rows packed,
    // x rows NPR + 2 pieces apart)
    const int ri = Gm::MR ? R / a.npr : 0;
    const int xshift = Gm::MR ? 2 * ri * kPitch : 0;
    const int cw = warp & 3;                // the block's column is 8 cw
    // output tile: 128B-swizzled rows of 32 floats, this thread's 8 outputs at row R, quads 2 cw, 2 cw + 1
    const uint32_t o0 = static_cast<uint32_t>(R * 128 + (((2 * cw) ^ (R & 7)) << 4));
    const uint32_t o1 = static_cast<uint32_t>(R * 128 + (((2 * cw + 1) ^ (R & 7)) << 4));

    int stage = 0, t0 = 0, row = a.row0;
    uint32_t phase = 0;
    for (int u = 0; u < nunits; ++u) {
        mbar_wait(&full[stage], phase);
        const unsigned char* gys = tb + stage * Gm::Stage;
        unsigned char* ob = smem + (u & 1) * kOutBytes;
        if constexpr (Gm::BASE >= kFWD) {
            const float* tp = reinterpret_cast<const float*>(stages + stage * Gm::Stage + Gm::GYRegion);
#pragma unroll
            for (int c = 0; c < (KT + 3) / 4; ++c) {
                const float4 qv = *reinterpret_cast<const float4*>(tp + 4 * c);
                w[4 * c + 0] = qv.x;
                w[4 * c + 1] = qv.y;
                w[4 * c + 2] = qv.z;
                w[4 * c + 3] = qv.w;
            }
        }
        const bool live = Gm::MR ? ri < min(a.rpi, a.nrows - u * a.rpi) : t0 + 32 * R < a.L;
        if (live) {
            float* gout = Gm::DST ? a.out + static_cast<int64_t>(row) * a.L + t0 + 32 * R + 8 * cw : nullptr;
            switch (cw) {
                case 0: item<KT, FUSED, MODE, 0>(gys, xshift, ob, o0, o1, gout, w, acc); break;
                case 1: item<KT, FUSED, MODE, 8>(gys, xshift, ob, o0, o1, gout, w, acc); break;
                case 2: item<KT, FUSED, MODE, 16>(gys, xshift, ob, o0, o1, gout, w, acc); break;
                default: item<KT, FUSED, MODE, 24>(gys, xshift, ob, o0, o1, gout, w, acc); break;
            }
        }
        if constexpr (Gm::HAS_OBUF) {
            fence_proxy_async_smem();           // output tile visible to the TMA store
            if (tid == 0) bulk_wait_read_all();  // store u-1 has read buffer (u+1)&1
        }
        __syncthreads();
        if (tid == 0) {
            if constexpr (Gm::HAS_OBUF) {
#if KS_EVICT_FIRST
                tma_store_3d_hint(out_map, ob, 0, t0 / 32, row, policy_evict_first());
#else
                tma_store_3d(out_map, ob, 0, t0 / 32, row);  // columns past L are clipped
#endif
                bulk_commit();
            }
            if (u + NS < nunits) issue(stage);
        }
        if (++stage == NS) {
            stage = 0;
            phase ^= 1u;
        }
        t0 += kTT;
        if (t0 >= a.L) {
            t0 = 0;
            row += a.rstep;
        }
    }
    if (Gm::HAS_OBUF && tid == 0) bulk_wait_all();

    if constexpr (Gm::HAS_DW) {
        // the 8 warp partials go to stage memory (every loaded stage has been
        // consumed by now): no static shared array, which would round the
        // CTA's static shared memory up to 1 KiB and cost the dW kernel its
        // third CTA per SM
        float (*red)[KT] = reinterpret_cast<float (*)[KT]>(stages);
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
            for (int jj = 0; jj < KT; ++jj) red[warp][jj] = acc[jj];  // (stage memory: every item is consumed)
        }
        __syncthreads();
        if (tid < KT) {
            float s = 0.f;
#pragma unroll
            for (int ww = 0; ww < kThreads / 32; ++ww) s += red[ww][tid];
            part[(static_cast<int64_t>(a.grp) * a.H + a.h) * KT + tid] = s;
        }
    }
}

// dW modes: grid = G x H CTAs, CTA = (row group, channel).  Stencils: a
// persistent grid, CTA c takes rows c, c + gridDim.x, ...
template <int KT, bool FUSED, int MODE>
__global__ void __launch_bounds__(kThreads, Geo<KT, MODE>::MinBlocks)  // 3 CTAs/SM (<= 80 regs), stencils 4
bwd_short(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap x_map,
          const __grid_constant__ CUtensorMap out_map, const float* __restrict__ k, float* __restrict__ part, int B,
          int H, int L, int G, float* __restrict__ out, int rpi) {
    pdl_wait();  // launched with PDL (the stencils follow prep_taps): predecessor complete first
    using Gm = Geo<KT, MODE>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = align_smem<1024>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (Gm::HAS_OBUF ? 2 * kOutBytes : 0) + Gm::NS * Gm::Stage);

    Args a;
    a.H = H;
    a.L = L;
    a.out = out;
    a.npr = L / 32;
    a.rpi = rpi;
    a.tx = static_cast<uint32_t>(rpi * (2 * a.npr + 2) * kPitch);
    if constexpr (Gm::HAS_DW) {
        a.h = blockIdx.x % H;
        a.grp = blockIdx.x / H;
        const int b_begin = static_cast<int>(static_cast<int64_t>(B) * a.grp / G);
        const int b_end = static_cast<int>(static_cast<int64_t>(B) * (a.grp + 1) / G);
        a.row0 = b_begin * H + a.h;
        a.rstep = H;
        a.nrows = b_end - b_begin;
    } else {
        const int rows = B * H;
        a.h = a.grp = 0;
        a.row0 = blockIdx.x;
        a.rstep = gridDim.x;
        a.nrows = static_cast<int>(blockIdx.x) < rows
                      ? (rows - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                      : 0;
    }
    if (threadIdx.x == 0) {
        prefetch_tmap(&in_map);
        if (Gm::HAS_DW) prefetch_tmap(&x_map);
        if (Gm::HAS_OBUF) prefetch_tmap(&out_map);
        for (int s = 0; s < Gm::NS; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    run<KT, FUSED, MODE>(&in_map, &x_map, &out_map, k, part, smem, full, a);
}

}  // namespace bwds
}  // namespace ks
