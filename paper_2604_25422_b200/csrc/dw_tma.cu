// dw_tma.cu -- TMA-pipelined weight gradient, HIERARCHICAL order (sm_100a),
// rows with L % 32 == 0.
//
//   dk[h,j] = sum_b sum_t gy[b,h,t] * x[b,h,t+j-p]     (reference src/conv_core.cpp:148-181)
//
// CTA = (row group g, channel h, tap tile of JT = NJ*JR taps); 256 threads =
// NJ tap groups x NTS t-slices.  Work items are (row b, 2048-wide t tile) in
// flat order; each of NS stages holds the gy tile and the x window
// [t0+j0-p-D, ...) (TMA, zero outside the row), completing on an mbarrier.
// Thread (tap group, t-slice) reads TB gy values and TB+JR-1 x values per
// register block with 128-bit conflict-free loads (lanes 128 B apart under
// SWIZZLE_128B) and accumulates JR taps x TB t FMAs into JR registers -- the
// in-register partial sums over L.  Then a fixed xor-shuffle tree per warp, a
// fixed pass over the warps of each tap group, one partial per CTA into
// part[g,h,j]; dw_sum_groups (conv_dw.cu) adds the G partials in ascending g.
// No atomics anywhere: the result is a deterministic function of the shape.
//
// (JR, TB) = (8, 8) for K <= 8 (memory-bound, e.g. BASELINE config 3),
// (16, 8) for 8 < K <= 16 (config 5a) and (16, 16) for longer K, where 256 FMAs per 13 shared loads keep the FMA pipe
// fed (compute-bound, configs 2 / 4 / 5b / 5c).
#include <algorithm>
#include <cstdlib>

#include "ks_common.cuh"
#include "ks_tma.cuh"

namespace ks {

namespace {

constexpr int kThreads = 256;
constexpr int kDwTT = 2048;              // t per work item
constexpr int kDwIn = 32;                // floats per TMA row piece (128 B)
constexpr int kDwMain = kDwTT / kDwIn;   // x window main-box rows

struct DwGeomT {
    int XR;           // x window rows (32 floats): kDwMain main + XT tail
    int XT;           // tail rows
    int gy_bytes;     // gy region in a stage (1024-aligned: 64 rows, or 72 when BWD stages a halo)
    int gy_box;       // gy rows loaded per item (64, or 66 = tile + one halo row each side)
    int stage_bytes;
};

// Register block `q` (0 <= q < TT/TB) -> first t of the block; consecutive
// lanes get blocks 128 B apart.
template <int TB>
__device__ __forceinline__ int block_t(int q) {
    if constexpr (TB == 8) return ((q & 31) * 4 + ((q >> 5) & 3) + (q >> 7) * 128) * TB;
    else return ((q & 31) * 2 + ((q >> 5) & 1) + (q >> 6) * 64) * TB;
}

// BWD = the fused backward: the same dW work (identical decomposition and
// accumulation order, so dk is bit-identical to the dW-only kernel) plus dX
// from the gy tile already in shared memory.  The gy box then carries one
// 32-float halo row on each side (gy logical index 0 = t0 - 32); every thread
// computes the 8 dX outputs of its own dW t-block (taps reversed, held in
// registers, window sub-quad offset S2 = (-q) mod 4), writes them to a
// swizzled output buffer, and thread 0 stores each 2048-wide tile with one
// TMA tensor store (double-buffered).  gy and x are read from HBM once for
// both gradients: 12 B per element instead of 16 (dX 8 + dW 8).
//
// MR (dW only, L = 256 / 512 / 1024): a work item is RPI = 2048 / L whole rows
// of the CTA's channel instead of one 2048-wide tile of one row (most of which
// would lie past the row end): the 4-D view {32, L/32, H, B} (encode_chan_view)
// brings RPI rows per box -- gy rows packed, so block t-offset tl addresses row
// tl >> lsh exactly as in one long row, and each row's x window with its own
// XT tail pieces (zero outside the row), so a row's x index moves by XT pieces
// per row.  Same per-block math and reduction tree.
template <int JR, int TB, int NJ, int S, bool FUSED, bool BWD, int S2, bool MR>
__global__ void __launch_bounds__(kThreads)
dw_tma(const __grid_constant__ CUtensorMap gy_map, const __grid_constant__ CUtensorMap x_map,
       const __grid_constant__ CUtensorMap x_tail_map, const __grid_constant__ CUtensorMap dx_map,
       const float* __restrict__ k, float* __restrict__ part, int B, int H, int L, int K, int p, int G, int NJT,
       DwGeomT g, int NS, int lsh, int rpi) {
    constexpr int NTS = kThreads / NJ;
    constexpr int JT = NJ * JR;
    constexpr int SPT = kDwTT / (NTS * TB);
    constexpr int NVX = (S + TB + JR - 1 + 3) / 4;
    constexpr int NV2 = (S2 + TB + JR - 1 + 3) / 4;  // dX window quads (K <= JR)
    constexpr int GOFS = BWD ? kDwIn : 0;            // gy logical index of t0
    static_assert(!BWD || (NJ == 1 && TB == 8), "the fused backward needs one tap group of 8-wide blocks");
    static_assert(!(BWD && MR), "multi-row items are for dW only");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = align_smem<1024>(smem_raw);
    unsigned char* outb = smem + NS * g.stage_bytes;  // BWD: 2 x 8 KB dX tiles
    uint64_t* full = reinterpret_cast<uint64_t*>(outb + (BWD ? 2 * kDwTT * 4 : 0));
    __shared__ float red[kThreads / 32][JR];

    int bid = blockIdx.x;
    const int jt = bid % NJT;
    bid /= NJT;
    const int h = bid % H;
    const int grp = bid / H;
    const int b_begin = static_cast<int>(static_cast<int64_t>(B) * grp / G);
    const int b_end = static_cast<int>(static_cast<int64_t>(B) * (grp + 1) / G);
    const int j0 = jt * JT;
    const int tid = threadIdx.x;
    const int jg = tid / NTS;
    const int ts = tid - jg * NTS;
    const int ntt = (L + kDwTT - 1) / kDwTT;
    const int nrows = b_end - b_begin;
    const int nunits = MR ? (nrows + rpi - 1) / rpi : nrows * ntt;
    // the x window of a work item at t0 starts at position t0 + j0 - p - D
    const int xoff = j0 - p;
    const int D = ((xoff % kDwIn) + kDwIn) % kDwIn;
    const int xr_rel = (xoff - D) / kDwIn;  // exact division
    const int A = D & ~3;                   // D & 3 == S

    if (tid == 0) {
        prefetch_tmap(&gy_map);
        prefetch_tmap(&x_map);
        prefetch_tmap(&x_tail_map);
        if (BWD) prefetch_tmap(&dx_map);
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint32_t tx_bytes = static_cast<uint32_t>(g.gy_box * kDwIn * 4 + g.XR * kDwIn * 4);
    auto issue = [&](int stage, int u) {
        if constexpr (MR) {  // rows b .. b + rpi - 1 of channel h: gy packed, x windows with their tails
            const int b = b_begin + u * rpi;
            unsigned char* sb = smem + stage * g.stage_bytes;
            mbar_arrive_expect_tx(&full[stage], tx_bytes);
            tma_load_pad(sb, &gy_map, 0, h, b, &full[stage]);
            tma_load_pad(sb + g.gy_bytes, &x_map, xr_rel, h, b, &full[stage]);
            return;
        }
        const int b = b_begin + u / ntt;
        const int t0 = (u % ntt) * kDwTT;
        const int row = b * H + h;
        unsigned char* sb = smem + stage * g.stage_bytes;
        mbar_arrive_expect_tx(&full[stage], tx_bytes);
        tma_load_3d(sb, &gy_map, 0, t0 / kDwIn - (BWD ? 1 : 0), row, &full[stage]);
        const int xr = t0 / kDwIn + xr_rel;
        tma_load_3d(sb + g.gy_bytes, &x_map, 0, xr, row, &full[stage]);
        tma_load_3d(sb + g.gy_bytes + kDwMain * kDwIn * 4, &x_tail_map, 0, xr + kDwMain, row, &full[stage]);
    };
    if (tid == 0)
        for (int s = 0; s < NS && s < nunits; ++s) issue(s, s);

    // dX taps, reversed (the reference's k[h, K-1-j], src/conv_core.cpp:68), zero past K
    float wr[BWD ? JR : 1];
    int a2 = 0;
    if constexpr (BWD) {
#pragma unroll
        for (int jj = 0; jj < JR; ++jj) wr[jj] = jj < K ? k[static_cast<int64_t>(h) * K + K - 1 - jj] : 0.f;
        const int q = K - 1 - p;    // dX offset (src/conv_core.cpp:56)
        a2 = GOFS - q - S2;         // 4-aligned gy index of a block's first dX tap, minus tl
    }

    float acc[JR];
#pragma unroll
    for (int i = 0; i < JR; ++i) acc[i] = 0.f;

    for (int u = 0; u < nunits; ++u) {
        const int stage = u % NS;
        mbar_wait(&full[stage], static_cast<uint32_t>((u / NS) & 1));
        const unsigned char* gys = smem + stage * g.stage_bytes;
        const unsigned char* xs = gys + g.gy_bytes;
        unsigned char* ob = outb + (u & 1) * kDwTT * 4;
        const int t0 = MR ? 0 : (u % ntt) * kDwTT;
        const int tlim = MR ? min(rpi, nrows - u * rpi) << lsh : L - t0;  // live blocks: tl < tlim
#pragma unroll 2
        for (int s = 0; s < SPT; ++s) {
            const int tl = block_t<TB>(s * NTS + ts);
            if (tl < tlim) {
                float gv[TB];
#pragma unroll
                for (int c = 0; c < TB / 4; ++c) {
                    const float4 q =
                        lds4(gys + swz<128>(static_cast<uint32_t>(GOFS + tl + 4 * c)));
                    gv[4 * c + 0] = q.x;
                    gv[4 * c + 1] = q.y;
                    gv[4 * c + 2] = q.z;
                    gv[4 * c + 3] = q.w;
                }
                float xv[4 * NVX];
                const uint32_t xi = static_cast<uint32_t>(A + tl + jg * JR + (MR ? (tl >> lsh) * g.XT * kDwIn : 0));
#pragma unroll
                for (int c = 0; c < NVX; ++c) {
                    const float4 q = lds4(xs + swz<128>(xi + 4 * c));
                    xv[4 * c + 0] = q.x;
                    xv[4 * c + 1] = q.y;
                    xv[4 * c + 2] = q.z;
                    xv[4 * c + 3] = q.w;
                }
#pragma unroll
                for (int tt = 0; tt < TB; ++tt)
#pragma unroll
                    for (int jj = 0; jj < JR; ++jj) acc[jj] = muladd<true>(acc[jj], gv[tt], xv[S + tt + jj]);
                if constexpr (BWD) {
                    // dx[t0+tl+r] = sum_j gy[t0+tl+r+j-q] * k[K-1-j], j ascending from +0
                    float v2[4 * NV2];
                    const uint32_t gi = static_cast<uint32_t>(a2 + tl);
#pragma unroll
                    for (int c = 0; c < NV2; ++c) {
                        const float4 q = lds4(gys + swz<128>(gi + 4 * c));
                        v2[4 * c + 0] = q.x;
                        v2[4 * c + 1] = q.y;
                        v2[4 * c + 2] = q.z;
                        v2[4 * c + 3] = q.w;
                    }
                    float d[TB];
#pragma unroll
                    for (int r = 0; r < TB; ++r) d[r] = 0.f;
#pragma unroll
                    for (int jj = 0; jj < JR; ++jj)
                        if (jj < K) {
#pragma unroll
                            for (int r = 0; r < TB; ++r) d[r] = muladd<FUSED>(d[r], v2[S2 + r + jj], wr[jj]);
                        }
#pragma unroll
                    for (int r = 0; r < TB; r += 4)
                        *reinterpret_cast<float4*>(ob + swz<128>(static_cast<uint32_t>(tl + r))) =
                            make_float4(d[r], d[r + 1], d[r + 2], d[r + 3]);
                }
            }
        }
        if constexpr (BWD) {
            fence_proxy_async_smem();           // dX tile visible to the TMA store
            if (tid == 0) bulk_wait_read_all();  // store u-1 has read buffer (u+1)&1
        }
        __syncthreads();
        if (tid == 0) {
            if constexpr (BWD) {
                const int b = b_begin + u / ntt;
                tma_store_3d(&dx_map, ob, 0, t0 / kDwIn, b * H + h);  // columns past L are clipped
                bulk_commit();
            }
            if (u + NS < nunits) issue(stage, u + NS);
        }
    }
    if (BWD && tid == 0) bulk_wait_all();

#pragma unroll
    for (int jj = 0; jj < JR; ++jj) {
        float v = acc[jj];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc[jj] = v;
    }
    const int warp = tid >> 5, lane = tid & 31;
    if (lane == 0) {
#pragma unroll
        for (int jj = 0; jj < JR; ++jj) red[warp][jj] = acc[jj];
    }
    __syncthreads();
    constexpr int WPG = NTS / 32;  // warps per tap group
    if (tid < JT) {
        const int gj = tid / JR, jj = tid % JR;
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < WPG; ++w) s += red[gj * WPG + w][jj];
        const int j = j0 + tid;
        if (j < K) part[(static_cast<int64_t>(grp) * H + h) * K + j] = s;
    }
}

struct Maps {
    CUtensorMap gm, xm, xt, dxm;
};

template <int JR, int TB, int NJ, bool FUSED, bool BWD>
ks_status launch(int s, int s2, const Maps& mp, const float* k, float* part, int64_t B, int64_t H, int64_t L,
                 int64_t K, int G, int NJT, const DwGeomT& g, int NS, cudaStream_t st, int lsh = -1, int rpi = 0) {
    const int smem = NS * g.stage_bytes + (BWD ? 2 * kDwTT * 4 : 0) + 64 + 1024;
    const unsigned blocks = static_cast<unsigned>(int64_t(G) * H * NJT);
    const int p = static_cast<int>(K / 2);
#define KS_DW_CASE_M(SV, S2V, MRV)                                                                             \
    if (s == SV && s2 == S2V) {                                                                                \
        auto kern = dw_tma<JR, TB, NJ, SV, FUSED, BWD, S2V, MRV>;                                              \
        prepare_kernel(reinterpret_cast<const void*>(kern), kThreads, smem);                                 \
        launch_kernel(kern, blocks, kThreads, smem, st, mp.gm, mp.xm, mp.xt, mp.dxm, k, part, static_cast<int>(B),        \
                                             static_cast<int>(H), static_cast<int>(L), static_cast<int>(K), p, \
                                             G, NJT, g, NS, lsh, rpi);                                         \
        return check_launch();                                                                                 \
    }
#define KS_DW_CASE(SV, S2V) KS_DW_CASE_M(SV, S2V, false)
    if constexpr (!BWD) {
        if (rpi > 0) {
            KS_DW_CASE_M(0, 0, true) KS_DW_CASE_M(1, 0, true) KS_DW_CASE_M(2, 0, true) KS_DW_CASE_M(3, 0, true)
            return KS_ERR_CUDA;
        }
    }
    if constexpr (BWD) {
        // S2 = (-q) mod 4 with q = K-1-p: S2 = S for odd K, S + 1 (mod 4) for even K
        KS_DW_CASE(0, 0) KS_DW_CASE(0, 1) KS_DW_CASE(1, 1) KS_DW_CASE(1, 2)
        KS_DW_CASE(2, 2) KS_DW_CASE(2, 3) KS_DW_CASE(3, 3) KS_DW_CASE(3, 0)
    } else {
        KS_DW_CASE(0, 0) KS_DW_CASE(1, 0) KS_DW_CASE(2, 0) KS_DW_CASE(3, 0)
    }
#undef KS_DW_CASE
#undef KS_DW_CASE_M
    return KS_ERR_CUDA;
}

template <int JR, int TB, int NJ, bool BWD>
ks_status launch_m(int s, int s2, bool fused, const Maps& mp, const float* k, float* part, int64_t B, int64_t H,
                   int64_t L, int64_t K, int G, int NJT, const DwGeomT& g, int NS, cudaStream_t st, int lsh = -1,
                   int rpi = 0) {
    return fused ? launch<JR, TB, NJ, true, BWD>(s, s2, mp, k, part, B, H, L, K, G, NJT, g, NS, st, lsh, rpi)
                 : launch<JR, TB, NJ, false, BWD>(s, s2, mp, k, part, B, H, L, K, G, NJT, g, NS, st, lsh, rpi);
}

// Shared by the dW-only and the fused backward entry points.
ks_status run_dw_tma(const float* gy, const float* x, const float* k, float* dx, float* part, int64_t B, int64_t H,
                     int64_t L, int64_t K, int G, int mode, bool bwd, cudaStream_t st, bool* handled) {
    *handled = false;
    if (L % kDwIn != 0 || B * H >= (int64_t(1) << 31) || L >= (int64_t(1) << 30) || K >= (int64_t(1) << 30))
        return KS_OK;
    // (8,8) with 1-2 tap groups up to K = 16; (16,16) with >= 2 tap groups beyond
    // (a t-slice must cover a whole 16-wide block of the 2048-wide work item)
    // 8 < K <= 16: one tap group of 16 taps over 8-wide t blocks (16 x 8 FMAs
    // per 2 gy + 6-7 x loads, half the shared traffic of two 8-tap groups)
    const bool j16 = K > 8 && K <= 16 && opt(kOptDwtmaJ16) != 0;  // option 0: two 8-tap groups
    const int JR = K <= 16 && !j16 ? 8 : 16;
    int nj = JR == 8 || j16 ? 1 : 2;
    while (nj < 8 && nj * JR < K) nj *= 2;
    if (bwd && !(nj == 1 && (JR == 8 || j16))) return KS_OK;  // fused backward: one tap group, TB = 8
    const int njt = static_cast<int>((K + nj * JR - 1) / (nj * JR));
    if (int64_t(G) * H * njt >= (int64_t(1) << 31)) return KS_OK;
    DwGeomT g;
    g.gy_box = kDwMain + (bwd ? 2 : 0);
    g.gy_bytes = (g.gy_box * kDwIn * 4 + 1023) / 1024 * 1024;
    g.XT = (nj * JR + 40 + kDwIn - 1) / kDwIn;  // covers D + JT + the register-window overrun
    g.XR = kDwMain + g.XT;
    Maps mp;
    // rows of 256 / 512 / 1024: items of 2048 / L whole rows (see the kernel)
    int lsh = -1, rpi = 0;
    if (!bwd && L < kDwTT && L >= 256 && (L & (L - 1)) == 0 && opt(kOptDwMrow) != 0) {
        const int npr = static_cast<int>(L / kDwIn);
        rpi = static_cast<int>(kDwTT / L);
        lsh = 0;
        while ((int64_t(1) << lsh) < L) ++lsh;
        g.XR = rpi * (npr + g.XT);
        if (!encode_chan_view(&mp.gm, gy, B * H, L, H, npr, rpi)) return KS_OK;
        if (!encode_chan_view(&mp.xm, x, B * H, L, H, npr + g.XT, rpi)) return KS_OK;
        mp.xt = mp.xm;   // unused
        mp.dxm = mp.gm;  // unused
    } else {
        if (!encode_row_view(&mp.gm, gy, B * H, L, kDwIn, g.gy_box, 128)) return KS_OK;
        if (!encode_row_view(&mp.xm, x, B * H, L, kDwIn, kDwMain, 128)) return KS_OK;
        if (!encode_row_view(&mp.xt, x, B * H, L, kDwIn, g.XT, 128)) return KS_OK;
        if (bwd) {
            if (!encode_row_view(&mp.dxm, dx, B * H, L, kDwIn, kDwMain, 128)) return KS_OK;
        } else {
            mp.dxm = mp.gm;  // unused
        }
    }
    g.stage_bytes = (g.gy_bytes + g.XR * kDwIn * 4 + 1023) / 1024 * 1024;
    // 4 stages for the lightest blocks (K <= 8: bandwidth wants bytes in flight);
    // 3 for K > 8, where a fourth CTA per SM hides more FMA latency
    // (config 5a dW 10.7 -> 10.1 ms, fused backward 22.4 -> 20.4 ms)
    int NS = std::max(2, std::min(K > 8 ? 3 : 4, (72 * 1024) / g.stage_bytes));
    if (opt(kOptDwtmaNs) > 0) NS = static_cast<int>(opt(kOptDwtmaNs));  // tuning option
    const int p = static_cast<int>(K / 2);
    const int s = (4 - p % 4) % 4;
    const int q = static_cast<int>(K) - 1 - p;
    const int s2 = bwd ? (4 - q % 4) % 4 : 0;
    const bool fused = mode == KS_MULADD_FUSED;
    *handled = true;
    if (bwd)
        return j16 ? launch_m<16, 8, 1, true>(s, s2, fused, mp, k, part, B, H, L, K, G, njt, g, NS, st)
                   : launch_m<8, 8, 1, true>(s, s2, fused, mp, k, part, B, H, L, K, G, njt, g, NS, st);
    // dW only: HIERARCHICAL accumulates with FMA in either MulAddMode (conv_dw.cu)
    if (j16) return launch<16, 8, 1, true, false>(s, 0, mp, k, part, B, H, L, K, G, njt, g, NS, st, lsh, rpi);
    if (JR == 8)
        return nj == 1 ? launch<8, 8, 1, true, false>(s, 0, mp, k, part, B, H, L, K, G, njt, g, NS, st, lsh, rpi)
                       : launch<8, 8, 2, true, false>(s, 0, mp, k, part, B, H, L, K, G, njt, g, NS, st, lsh, rpi);
    switch (nj) {
        case 2: return launch<16, 16, 2, true, false>(s, 0, mp, k, part, B, H, L, K, G, njt, g, NS, st, lsh, rpi);
        case 4: return launch<16, 16, 4, true, false>(s, 0, mp, k, part, B, H, L, K, G, njt, g, NS, st, lsh, rpi);
        default: return launch<16, 16, 8, true, false>(s, 0, mp, k, part, B, H, L, K, G, njt, g, NS, st, lsh, rpi);
    }
}

}  // namespace

ks_status bwd_short_dw_stage1(const float*, const float*, float*, int64_t, int64_t, int64_t, int64_t, int, int,
                              cudaStream_t, bool*);
ks_status bwd_short_fused_stage1(const float*, const float*, const float*, float*, float*, int64_t, int64_t,
                                 int64_t, int64_t, int, int, cudaStream_t, bool*);

// K <= 16: the K-specialised kernels of bwd_short.cuh (same bits, fewer
// instructions) unless an A/B knob asks for this file's generic kernel.
// dW up to K = 32 (round 2, gpurun_out/s30: K = 17..32 -11..-40% against this
// file's kernel, e.g. (256,512,8192,24) 2.21 -> 1.32 ms); the fused backward
// checks K <= 16 itself.
static bool use_bwd_short(int64_t K) {
    if (opt(kOptBwds) == 0 || K > 32) return false;
    return opt(kOptDwtmaNs) == 0 && opt(kOptDwtmaJ16) != 0;
}

// Stage 1 of HIERARCHICAL dW through TMA into part[G,H,K] (G = the caller's row
// groups; stage 2 is shared with the generic path).  *handled = false means
// the shape is not supported here and the caller falls back.
ks_status dw_tma_stage1(const float* gy, const float* x, float* part, int64_t B, int64_t H, int64_t L, int64_t K,
                        int G, int mode, cudaStream_t st, bool* handled) {
    if (use_bwd_short(K)) {
        const ks_status s = bwd_short_dw_stage1(gy, x, part, B, H, L, K, G, mode, st, handled);
        if (*handled) return s;
    }
    return run_dw_tma(gy, x, nullptr, nullptr, part, B, H, L, K, G, mode, false, st, handled);
}

// Fused backward (dX + stage 1 of HIERARCHICAL dW) for K <= 16, L % 32 == 0:
// dx is written in full, part[G,H,K] exactly as dw_tma_stage1 would write it.
ks_status bwd_tma_stage1(const float* gy, const float* x, const float* k, float* dx, float* part, int64_t B,
                         int64_t H, int64_t L, int64_t K, int G, int mode, cudaStream_t st, bool* handled) {
    if (K > 16 || (reinterpret_cast<uintptr_t>(dx) & 15) != 0) {
        *handled = false;
        return KS_OK;
    }
    if (use_bwd_short(K)) {
        const ks_status s = bwd_short_fused_stage1(gy, x, k, dx, part, B, H, L, K, G, mode, st, handled);
        if (*handled) return s;
    }
    return run_dw_tma(gy, x, k, dx, part, B, H, L, K, G, mode, true, st, handled);
}

}  // namespace ks
