// stencil_pad.cu -- compute-bound forward / dX (K > 32), sm_100a, fed straight
// from TMA in the padded layout.
//
//   out[b,h,t] = sum_{j=0}^{K-1} in[b,h,t+j-off] * w[h,j]   (reference src/conv_core.cpp:21-75)
//
// The FMA inner loop wants each thread's 32-output register tile to read its
// input window with 128-bit loads at compile-time offsets, bank-conflict free:
// rows of 32 floats at a 36-float (144 B) pitch.  TMA writes that layout
// itself: the tensor is viewed as {32 floats, L/32 pieces, H, B} and loaded
// with box {36, n, RPT, 1} -- floats 32..35 of every piece lie outside dim 0
// and are zero-filled, so every 32-float piece lands as a 36-float row.  No re-layout
// pass, no producer warp: the CTA computes straight from the stage ring.
//
// The window must start on a 32-float piece: the taps are given `lead` =
// (-off) mod 32 leading zeros (prep_taps), so the window origin t0 - off - lead
// is a multiple of 32.  A leading zero tap adds x*0 = +-0 to an accumulator
// that starts at +0, which leaves every partial sum unchanged (round to
// nearest never yields -0 from a +0 start) -- the same argument that makes the
// zero-filled halo exact -- so results stay bit-identical to the reference.
//
// Zero-halo tap blocks are skipped per LANE: a tap block whose x positions
// all fall outside the row only multiplies TMA's zero fill.  A warp covers
// 1024 consecutive outputs, so where K is comparable to L (config 2, K = L)
// its lanes' valid block ranges are shifted by one block per lane; skipping
// per warp still computes the union (~31 blocks of ~96 per lane: 25% of the
// FFMAs on zeros), skipping per lane computes each lane's own range (the
// loop diverges by at most a block).  Warps whose lanes agree (every warp
// away from the row ends) keep warp-uniform bounds, so their taps stay
// provably uniform.  Taps are staged at the window's 36-float pitch per
// 32-tap block, so lanes reading different blocks are 144 B apart
// (conflict-free), as the window reads are.
//
// Tiles: RPT consecutive channels of one batch entry x (TPR*32)-output pieces
// of their rows; NT = 128 threads (one warp per SM sub-partition), thread
// (r, lt) owns outputs [t0 + 32 lt, +32) of channel h0 + r.  NS-stage TMA ring
// (one mbarrier per stage), one CTA barrier per tile before its stage is
// refilled.
#include <algorithm>
#include <cstdlib>

#include "ks_common.cuh"
#include "ks_tma.cuh"

// Two code-shape choices whose effect depends on how ptxas schedules each
// instantiation (measured on the B200 with tools/time_paths.py, ABAB):
//  * warp-uniform row index (lane-0 broadcast): the taps move to uniform
//    registers, so an FFMA reads two RF operands instead of three -- dX at
//    K = 128 / 256 (S = 1, producer lane) 4.5% faster, forward (S = 0) 1-1.5%
//    slower;
//  * anti-diagonal FFMA order in full windows: forward at K = 4096 (S = 0,
//    barrier refill) 1% faster, dX there 1-2% slower.
// Defaults follow those measurements; -DKS_SHFL_RSUB / -DKS_ANTIDIAG = 0 / 1
// force either everywhere (tools/build_variant.sh).
template <int S, bool PROD>
constexpr bool use_shfl() {
#ifdef KS_SHFL_RSUB
    return KS_SHFL_RSUB;
#else
    return PROD && S == 1;
#endif
}
template <int S, bool PROD>
constexpr bool use_antidiag() {
#ifdef KS_ANTIDIAG
    return KS_ANTIDIAG;
#else
    return !PROD && S == 0;
#endif
}

namespace ks {

__global__ void prep_taps(const float*, float*, int64_t, int64_t, int64_t, int, int);

// kp[h] = `lead` zeros, then k[h, j] (forward) or k[h, K-1-j] (dX), zero
// padded -- laid out at a 36-float pitch per 32-tap block (the window's
// padded layout), Kpp = Kp / 32 * 36 floats per row.
__global__ void prep_taps_pad36(const float* __restrict__ k, float* __restrict__ kp, int64_t H, int64_t K,
                                int64_t Kpp, int reverse, int lead) {
    pdl_trigger();  // the stencil that reads kp may launch now (it waits for this grid)
    const int64_t n = H * Kpp;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t h = i / Kpp, q = i - h * Kpp, blk = q / 36, c = q - blk * 36;
        const int64_t j = blk * 32 + c - lead;
        kp[i] = c < 32 && j >= 0 && j < K ? k[h * K + (reverse ? K - 1 - j : j)] : 0.f;
    }
}

namespace {

constexpr int kNT = 128;                     // FMA threads per CTA (one warp per SM sub-partition)
constexpr int kR = 32;                       // outputs per thread
constexpr int kJS = 16;                      // taps per register window

struct PadGeom {
    int RPT, TPR;      // channels per tile, threads per channel row (TPR*32 outputs)
    int NR;            // padded 36-float rows per channel window (T/32 + Kp/32 [+1])
    int NB, nbox;      // rows per TMA box, boxes per channel window (RPT == 1 when nbox > 1)
    int Kp;            // taps (with lead zeros) padded to a multiple of 32
    int Kpp;           // staged tap row: Kp, or Kp / 32 * 36 with `mirror` (36-float pitch per 32-tap block)
    int Ke;            // taps incl. lead zeros (the live ones)
    int base_row;      // (off + lead) / 32: window origin = t0/32 - base_row
    int off, zlead;    // stencil offset, leading zero taps (tap block jb covers j = 32 jb - zlead ...)
    int skip;          // drop zero-halo tap blocks (option pad_skip=0: compute them)
    int mirror;        // balance each warp's lanes: pair outputs mirrored about the row centre
    int win_floats;    // RPT * nbox * NB * 36
    int stage_bytes;   // window + RPT tap rows, 1024-aligned
};

// One thread's 32 outputs: acc[r] = sum_{j<Ke} win[S + r + j] * wk[j] in
// ascending j from +0, where win is the thread's window starting at the padded
// address pw + pbase (a 32-aligned logical index) and S = 0..3 the sub-quad
// offset of its first tap.  Each 16-tap register window takes
// ceil((S + 47) / 4) 128-bit loads (12 for S <= 1, 13 otherwise).
template <int S, bool FUSED, bool ANTID, int TP>  // TP: staged tap pitch per 32-tap block (32 or 36)
__device__ __forceinline__ void tile32(const float* pw, const float* wk, int pbase, int Ke, int jb_lo, int jb_hi,
                                       float (&acc)[kR]) {
    constexpr int NV = (S + kR + kJS - 1 + 3) / 4;
#pragma unroll
    for (int r = 0; r < kR; ++r) acc[r] = 0.f;
    auto window = [&](const float* base, const int sub, const float* w16, int nj) {  // w16: 16 taps
        float v[4 * NV];
#pragma unroll
        for (int c = 0; c < NV; ++c) {
            const float4 q = lds4(base + sub + 4 * c + (((sub + 4 * c) >> 5) << 2));
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
        if (ANTID && nj == kJS) {
            // anti-diagonal order: the FFMAs sharing window value v[S + m] run
            // back to back, so it stays in the operand-reuse cache, the tap
            // comes from a uniform register, and only the accumulator is read
            // from the register file.  Each acc[r] still sees its taps in
            // ascending jj = m - r (bit-identical chains).
#pragma unroll
            for (int m = 0; m < kR + kJS - 1; ++m)
#pragma unroll
                for (int r = 0; r < kR; ++r) {
                    const int jj = m - r;
                    if (jj >= 0 && jj < kJS) acc[r] = muladd<FUSED>(acc[r], v[S + m], w[jj]);
                }
        } else {
#pragma unroll
            for (int jj = 0; jj < kJS; ++jj)
                if (jj < nj) {
#pragma unroll
                    for (int r = 0; r < kR; ++r) acc[r] = muladd<FUSED>(acc[r], v[S + r + jj], w[jj]);
                }
        }
    };
    // 32-tap blocks [jb_lo, jb_hi) only: the caller drops blocks whose every
    // tap lands in the zero halo for the whole warp (x*0 never changes a chain
    // that starts at +0, and the reference skips those taps anyway)
    const int Kfull = Ke & ~31;
    const int jend = min(Kfull, jb_hi * 32);
    for (int j0 = jb_lo * 32; j0 < jend; j0 += 32) {
        const float* b0 = pw + pbase + (j0 >> 5) * 36;
        const float* w0 = TP == 32 ? wk + j0 : wk + (j0 >> 5) * TP;
        window(b0, 0, w0, kJS);
        window(b0, 16, w0 + 16, kJS);
    }
    if (Kfull < Ke && (Kfull >> 5) >= jb_lo && (Kfull >> 5) < jb_hi) {
        const float* b0 = pw + pbase + (Kfull >> 5) * 36;
        const float* w0 = TP == 32 ? wk + Kfull : wk + (Kfull >> 5) * TP;
        const int rem = Ke - Kfull;
        window(b0, 0, w0, rem < kJS ? rem : kJS);
        if (rem > kJS) window(b0, 16, w0 + 16, rem - kJS);
    }
}

// The warp-uniform variant of tile32 (every lane of the warp in the same
// channel row with the same tap-block bounds): the tap addresses are provably
// warp-uniform, so ptxas keeps each 16-tap window's taps in uniform registers
// (LDS + R2UR) and, in anti-diagonal order, the shared window value sits in
// the operand-reuse cache -- each FFMA reads only its accumulator from the
// register file (no even/odd bank conflicts, tools/sass_banks.py ~1.03 per
// FFMA against ~1.45 for tile32).  No tail special case: the staged taps are
// zero-padded to Kp, a block's second window is skipped when all its taps
// are padding, and a partially padded window multiplies in exact zeros (the
// leading-zero argument above; trailing taps stay within the documented
// non-finite contract).  Each register tile keeps the reference's ascending-j
// chain from +0.
template <int S, bool FUSED>
__device__ __forceinline__ void tile32u(const float* pw, const float* wk, int pbase, int Ke, int jend, int jb_lo,
                                        float (&acc)[kR]) {
    constexpr int NV = (S + kR + kJS - 1 + 3) / 4;
#pragma unroll
    for (int r = 0; r < kR; ++r) acc[r] = 0.f;
    const uint32_t wbase = opaque_u32(smem_u32(pw + pbase));  // this thread's window, in a register
    auto window = [&](const uint32_t base, const int sub, const float* w16) {
        float v[4 * NV];
#pragma unroll
        for (int c = 0; c < NV; ++c) {
            const float4 q = lds4_u32(base + 4u * (sub + 4 * c + (((sub + 4 * c) >> 5) << 2)));
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
        for (int m = 0; m < kR + kJS - 1; ++m)
#pragma unroll
            for (int r = 0; r < kR; ++r) {
                const int jj = m - r;
                if (jj >= 0 && jj < kJS) acc[r] = muladd<FUSED>(acc[r], v[S + m], w[jj]);
            }
    };
    for (int j0 = jb_lo * 32; j0 < jend; j0 += 32) {
        const uint32_t b0 = wbase + static_cast<uint32_t>(j0 >> 5) * 144u;
        window(b0, 0, wk + j0);
        if (j0 + kJS < Ke) window(b0, 16, wk + j0 + 16);
    }
}

// PROD: one extra warp whose lane 0 keeps the ring NS tiles ahead, and every
// consumer thread releases a stage as soon as it is done with it (moderate K,
// where tiles are short); !PROD: thread 0 refills a stage after a CTA barrier
// (long K, K >= 1024, where one stage suffices and the barrier is rare).
// LANEB: per-lane zero-halo bounds with the mirrored, rotating lane rings
// (g.mirror: K comparable to L); otherwise the round-1 per-warp bounds over
// the warp's 1024 consecutive outputs, warp-uniform by construction.
template <int S, bool FUSED, bool PROD, bool LANEB>
__global__ void __launch_bounds__(kNT + (PROD ? 32 : 0))
stencil_pad(const __grid_constant__ CUtensorMap in_map, const float* __restrict__ kp, float* __restrict__ out,
            int H, int L, int tiles_per_row, int ntiles, PadGeom g, int NS) {
    pdl_wait();  // launched with PDL after prep_taps: kp must be complete
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = align_smem<1024>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * g.stage_bytes);
    uint64_t* empty = full + NS;
    const int tid = threadIdx.x;
    const int T = g.TPR * kR;
    const int ngroups = H / g.RPT;  // channel groups per batch entry
    const uint32_t tx_bytes = static_cast<uint32_t>(g.win_floats * 4 + g.RPT * g.Kpp * 4);
    auto issue = [&](int stage, int tile) {
        const int rg = tile / tiles_per_row;
        const int t0 = (tile - rg * tiles_per_row) * T;
        const int b = rg / ngroups, h0 = (rg - b * ngroups) * g.RPT;
        unsigned char* sb = smem + stage * g.stage_bytes;
        mbar_arrive_expect_tx(&full[stage], tx_bytes);
        const int r0 = t0 / 32 - g.base_row;
        tma_load_pad(sb, &in_map, r0, h0, b, &full[stage]);
        if (g.nbox > 1) tma_load_pad(sb + g.NB * 144, &in_map, r0 + g.NB, h0, b, &full[stage]);
        bulk_load(sb + g.win_floats * 4, kp + static_cast<int64_t>(h0) * g.Kpp,
                  static_cast<uint32_t>(g.RPT * g.Kpp) * 4u, &full[stage]);
    };

    if (tid == 0) {
        prefetch_tmap(&in_map);
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kNT);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if constexpr (PROD) {
        if (tid >= kNT) {  // producer warp: lane 0 issues the loads, NS tiles ahead
            if (tid != kNT) return;
            int it = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
                const int stage = it % NS;
                // (parked: a spinning producer measured the same, and refilling
                // from the last consumer warp to finish a stage 1-4% slower)
                if (it >= NS) mbar_wait_sleep(&empty[stage], static_cast<uint32_t>((it / NS - 1) & 1));
                issue(stage, tile);
            }
            return;
        }
    } else {
        if (tid == 0)
            for (int s = 0; s < NS; ++s) {
                const int t = blockIdx.x + s * gridDim.x;
                if (t < ntiles) issue(s, t);
            }
    }

    // a warp lies within one channel row (TPR = 128 / RPT >= 32 since L >= 1024
    // keeps RPT <= 4); where use_shfl() says so, rsub is broadcast from lane 0
    // so the compiler can prove the tap addresses warp-uniform and keep the
    // taps in uniform registers
    const int rsub = (use_shfl<S, PROD>() || !LANEB) ? __shfl_sync(0xffffffffu, tid / g.TPR, 0) : tid / g.TPR;
    // lt: this thread's 32-output register tile within the channel row.  With
    // `mirror` (a tile spans the whole row and K is comparable to L, where an
    // output's valid tap count is ~ K - |t - L/2|), lane pairs take tiles
    // mirrored about the row's centre and each warp a ring of them, so a
    // warp's lanes have similar counts and the per-lane block bounds below
    // leave little divergence; the rings rotate over the warps with the CTA
    // and the tile, so the heavy centre ring does not always land on the same
    // SM sub-partition (warp w of every CTA shares one).  Lanes stay
    // conflict-free (lt mod 8 distinct per quarter-warp).
    const int q = tid - rsub * g.TPR;
    const int nwr = g.TPR / 32;
    const int win_rows = g.nbox * g.NB;
    const uint32_t full_u = opaque_u32(smem_u32(full)), empty_u = full_u + 8u * NS;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int stage = it % NS;
        const int ring = LANEB ? ((q >> 5) + static_cast<int>(blockIdx.x) + it) % nwr : 0;
        const int lt = !LANEB ? q
                              : ((q & 1) ? g.TPR / 2 + 16 * ring + ((q & 31) >> 1)
                                         : g.TPR / 2 - 1 - 16 * ring - ((q & 31) >> 1));
        mbar_wait_u32(full_u + 8u * stage, static_cast<uint32_t>((it / NS) & 1));
        const float* sw = reinterpret_cast<const float*>(smem + stage * g.stage_bytes);
        const int rg = tile / tiles_per_row;
        const int t0 = (tile - rg * tiles_per_row) * T;
        const bool live = t0 + lt * kR < L;  // L % 32 == 0: a register tile is wholly in or out
        float acc[kR];
        const float* pw_r = sw + rsub * win_rows * 36;
        const float* wk_r = sw + g.win_floats + rsub * g.Kpp;
        if constexpr (LANEB) {
            // this lane's outputs t in [ts, ts + 32): tap block jb reads x at
            // t + 32 jb - zlead - off + [0, 32); keep the blocks that reach [0, L)
            const int ts = t0 + lt * kR;
            const int jb_lo = g.skip ? max(0, (g.off + g.zlead - 31 - (ts + kR - 1) + 31 + 32 * 64) / 32 - 64) : 0;
            const int jb_hi = g.skip ? (L + g.off + g.zlead - ts + 31) / 32 : g.Kp / 32;
            if (live) tile32<S, FUSED, false, 36>(pw_r, wk_r, lt * 36, g.Ke, jb_lo, jb_hi, acc);
        } else {
            // the warp's outputs t in [tw, tw + 1024): tap block jb reads x at
            // t + 32 jb - zlead - off + [0, 32); keep the blocks that reach [0, L)
            const int tw = t0 + (lt & ~31) * kR;
            // (broadcast from lane 0: equal on every lane, and provably uniform
            // to ptxas, which then keeps the taps in uniform registers)
            const int jb_lo = __shfl_sync(0xffffffffu,
                                          g.skip ? max(0, (g.off + g.zlead - 31 - (tw + 32 * kR - 1) + 31 + 32 * 64) / 32 - 64) : 0, 0);
            const int jb_hi = __shfl_sync(0xffffffffu, g.skip ? (L + g.off + g.zlead - tw + 31) / 32 : g.Kp / 32, 0);
            // lanes past the row end compute on the stage's zero fill (their
            // outputs are not stored): no divergent branch around the FFMAs
            tile32u<S, FUSED>(pw_r, wk_r, lt * 36, g.Ke, min(g.Kp, 32 * jb_hi), jb_lo, acc);
        }
        if constexpr (PROD) {
            mbar_arrive_u32(empty_u + 8u * stage);  // this thread is done with the stage
        } else {
            __syncthreads();  // stage consumed by every thread
            if (tid == 0) {
                const int nt = tile + NS * gridDim.x;
                if (nt < ntiles) issue(stage, nt);
            }
        }
        if (live) {
            float* o = out + static_cast<int64_t>(rg * g.RPT + rsub) * L + t0 + lt * kR;
#pragma unroll
            for (int r = 0; r < kR; r += 4) st_cs_v4(o + r, make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]));
        }
    }
}

// ---------------------------------------------------------------------------
// Batch-lane stencil (K comparable to L, e.g. config 2's K = L): the lanes of
// a warp are 32 batch rows of ONE channel at the SAME 32 outputs, so every
// lane has the same taps (uniform registers), the same valid tap blocks (no
// zero-halo waste beyond the 32-tap block granularity, no lane divergence)
// and warps need no per-tile barrier.  CTA = (channel h, 32 batch rows,
// 4 x 32 outputs); warp c owns outputs [t0 + 32 c, +32) of the 32 rows.
// The input streams through a ring of one-piece slots: slot = 32 rows x one
// padded 32-float piece (box {36, 1, 1, 32} of the padded view, rows 144 B
// apart -- conflict-free 128-bit lane reads), loaded in ascending piece order
// by one producer lane; tap block jb of warp c reads pieces Q = ts/32 -
// base_row + jb, Q + 1 (and Q + 2 when S >= 2), so consecutive blocks reuse a
// piece and each warp releases a piece once it is past it (per-thread arrives
// on the slot's empty barrier).  Taps: the CTA's prepared row (prep_taps,
// `lead` zeros) bulk-loaded once.  Bits: each output's chain is tile32u's
// (ascending j from +0, zero taps / zero fill exact for finite inputs).
constexpr int kBlNW = 4;                  // consumer warps = output columns of 32
constexpr int kBlSlots = 8;               // ring slots (pieces; 12 slots, or taps read from L1 to make room, measured 1-2% slower)
constexpr int kBlSlotBytes = 32 * 144;    // 32 rows x one padded piece

struct BlGeom {
    int Kp, Ke, base_row, off, zlead, skip;
    int ncol, ngrp;  // output tiles of 128 per row, groups of 32 batch rows
};

__device__ __forceinline__ void bl_bounds(const BlGeom& g, int L, int ts, int& lo, int& hi) {
    if (ts >= L) {
        lo = 0;
        hi = 0;
        return;
    }
    lo = g.skip ? max(0, (g.off + g.zlead - 31 - (ts + kR - 1) + 31 + 32 * 64) / 32 - 64) : 0;
    hi = min(g.Kp / 32, g.skip ? (L + g.off + g.zlead - ts + 31) / 32 : g.Kp / 32);
}

template <int S, bool FUSED>
__global__ void __launch_bounds__(kNT + 32)
stencil_bl(const __grid_constant__ CUtensorMap in_map, const float* __restrict__ kp, float* __restrict__ out, int B,
           int H, int L, BlGeom g) {
    pdl_wait();  // launched with PDL after prep_taps: kp must be complete
    constexpr int NV = (S + kR + kJS - 1 + 3) / 4;
    constexpr int XP = S >= 2 ? 2 : 1;  // pieces past Q a block reads
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = align_smem<1024>(smem_raw);
    unsigned char* slots = smem;
    float* taps = reinterpret_cast<float*>(smem + kBlSlots * kBlSlotBytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kBlSlots * kBlSlotBytes + g.Kp * 4);
    uint64_t* empty = full + kBlSlots;
    uint64_t* tapbar = empty + kBlSlots;

    const int bid = static_cast<int>(blockIdx.x);
    const int col = bid % g.ncol, rest = bid / g.ncol;
    const int grp = rest % g.ngrp, h = rest / g.ngrp;
    const int t0 = col * kBlNW * kR, b0 = grp * 32;
    // the CTA's piece range: the union of its warps' blocks (all uniform)
    int pfirst = 1 << 30, plast = -(1 << 30);
#pragma unroll
    for (int c = 0; c < kBlNW; ++c) {
        int lo, hi;
        bl_bounds(g, L, t0 + c * kR, lo, hi);
        if (lo < hi) {
            const int q0 = (t0 + c * kR) / 32 - g.base_row;
            pfirst = min(pfirst, q0 + lo);
            plast = max(plast, q0 + hi - 1 + XP);
        }
    }
    const int npieces = plast >= pfirst ? plast - pfirst + 1 : 0;
    const int tid = threadIdx.x;
    if (tid == 0) {
        prefetch_tmap(&in_map);
        for (int s = 0; s < kBlSlots; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kNT);
        }
        mbar_init(tapbar, 1);
        fence_mbar_init();
    }
    __syncthreads();

    if (tid >= kNT) {  // producer warp: lane 0 streams the pieces
        if (tid == kNT) {
            mbar_arrive_expect_tx(tapbar, static_cast<uint32_t>(g.Kp) * 4u);
            bulk_load(taps, kp + static_cast<int64_t>(h) * g.Kp, static_cast<uint32_t>(g.Kp) * 4u, tapbar);
            int slot = 0;
            uint32_t phase = 0;
            for (int i = 0; i < npieces; ++i) {
                if (i >= kBlSlots) mbar_wait_sleep(&empty[slot], phase ^ 1u);
                mbar_arrive_expect_tx(&full[slot], kBlSlotBytes);
                tma_load_pad(slots + slot * kBlSlotBytes, &in_map, pfirst + i, h, b0, &full[slot]);
                if (++slot == kBlSlots) {
                    slot = 0;
                    phase ^= 1u;
                }
            }
        }
        return;
    }

    const int warp = tid >> 5, lane = tid & 31;
    const int ts = t0 + warp * kR;
    int jb_lo, jb_hi;
    bl_bounds(g, L, ts, jb_lo, jb_hi);
    jb_lo = __shfl_sync(0xffffffffu, jb_lo, 0);  // provably uniform to ptxas
    jb_hi = __shfl_sync(0xffffffffu, jb_hi, 0);
    const int q0 = __shfl_sync(0xffffffffu, ts / 32 - g.base_row, 0);
    const uint32_t lrow = opaque_u32(smem_u32(slots) + static_cast<uint32_t>(lane) * 144u);
    mbar_wait(tapbar, 0);

    float acc[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) acc[r] = 0.f;
    // one 16-tap window: quads at logical sub + 4c of the block's pieces
    auto window = [&](const uint32_t (&pb)[3], const int sub, const float* w16) {
        float v[4 * NV];
#pragma unroll
        for (int c = 0; c < NV; ++c) {
            const int e = sub + 4 * c;
            const float4 q = lds4_u32(pb[e >> 5] + 4u * (e & 31));
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
        for (int m = 0; m < kR + kJS - 1; ++m)
#pragma unroll
            for (int r = 0; r < kR; ++r) {
                const int jj = m - r;
                if (jj >= 0 && jj < kJS) acc[r] = muladd<FUSED>(acc[r], v[S + m], w[jj]);
            }
    };
    int slot = 0;
    uint32_t phase = 0;
    const uint32_t full_u = opaque_u32(smem_u32(full)), empty_u = full_u + 8u * kBlSlots;
    for (int i = 0; i < npieces; ++i) {
        mbar_wait_u32(full_u + 8u * slot, phase);
        const int jb = pfirst + i - q0;  // the block whose first piece is this one
        if (jb >= jb_lo && jb < jb_hi) {
            uint32_t pb[3];
            pb[0] = lrow + static_cast<uint32_t>(slot * kBlSlotBytes);
#pragma unroll
            for (int x = 1; x <= XP; ++x) {
                const int sx = slot + x >= kBlSlots ? slot + x - kBlSlots : slot + x;
                const uint32_t px = slot + x >= kBlSlots ? phase ^ 1u : phase;
                mbar_wait_u32(full_u + 8u * sx, px);
                pb[x] = lrow + static_cast<uint32_t>(sx * kBlSlotBytes);
            }
            if (XP == 1) pb[2] = pb[1];
            const int j0 = jb * 32;
            window(pb, 0, taps + j0);
            if (j0 + kJS < g.Ke) window(pb, 16, taps + j0 + 16);
        }
        mbar_arrive_u32(empty_u + 8u * slot);  // this thread is past the piece
        if (++slot == kBlSlots) {
            slot = 0;
            phase ^= 1u;
        }
    }
    if (ts < L && b0 + lane < B) {
        float* o = out + (static_cast<int64_t>(b0 + lane) * H + h) * L + ts;
#pragma unroll
        for (int r = 0; r < kR; r += 4) st_cs_v4(o + r, make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]));
    }
}

int bl_smem(const BlGeom& g) { return kBlSlots * kBlSlotBytes + g.Kp * 4 + 256 + 1024; }

template <int S, bool FUSED>
ks_status launch_bl(const CUtensorMap& im, const float* kp, float* out, int64_t B, int64_t H, int64_t L,
                    const BlGeom& g, cudaStream_t st) {
    auto kern = stencil_bl<S, FUSED>;
    const int smem = bl_smem(g);
    prepare_kernel(reinterpret_cast<const void*>(kern), kNT + 32, smem);
    launch_kernel_pdl(kern, static_cast<unsigned>(int64_t(g.ncol) * g.ngrp * H), kNT + 32, smem, st, im, kp, out,
                  static_cast<int>(B), static_cast<int>(H), static_cast<int>(L), g);
    return check_launch();
}

int pad_smem(const PadGeom& g, int NS) { return NS * g.stage_bytes + 128 + 1024; }

template <int S, bool FUSED, bool PROD>
ks_status launch(const CUtensorMap& im, const float* kp, float* out, int64_t B, int64_t H, int64_t L,
                 const PadGeom& g, int NS, cudaStream_t st) {
    auto kern = g.mirror ? stencil_pad<S, FUSED, PROD, true> : stencil_pad<S, FUSED, PROD, false>;
    constexpr int threads = kNT + (PROD ? 32 : 0);
    const int smem = pad_smem(g, NS);
    const int per_sm = prepare_kernel(reinterpret_cast<const void*>(kern), threads, smem);
    const int T = g.TPR * kR;
    const int tiles_per_row = static_cast<int>((L + T - 1) / T);
    const int ntiles = static_cast<int>(B * H / g.RPT * tiles_per_row);
    const int grid = std::min(ntiles, num_sms() * per_sm);
    launch_kernel_pdl(kern, grid, threads, smem, st, im, kp, out, static_cast<int>(H), static_cast<int>(L), tiles_per_row, ntiles,
                                      g, NS);
    return check_launch();
}

template <bool PROD>
ks_status launch_s(int s, bool fused, const CUtensorMap& im, const float* kp, float* out, int64_t B, int64_t H,
                   int64_t L, const PadGeom& g, int NS, cudaStream_t st) {
    switch (s) {
        case 0: return fused ? launch<0, true, PROD>(im, kp, out, B, H, L, g, NS, st)
                             : launch<0, false, PROD>(im, kp, out, B, H, L, g, NS, st);
        case 1: return fused ? launch<1, true, PROD>(im, kp, out, B, H, L, g, NS, st)
                             : launch<1, false, PROD>(im, kp, out, B, H, L, g, NS, st);
        case 2: return fused ? launch<2, true, PROD>(im, kp, out, B, H, L, g, NS, st)
                             : launch<2, false, PROD>(im, kp, out, B, H, L, g, NS, st);
        default: return fused ? launch<3, true, PROD>(im, kp, out, B, H, L, g, NS, st)
                              : launch<3, false, PROD>(im, kp, out, B, H, L, g, NS, st);
    }
}


}  // namespace

// Compute-bound fwd/dX from the padded TMA view (K > 32, L >= 1024,
// L % 32 == 0).  *handled = false when the shape is outside the envelope.
ks_status stencil_pad_f32(const float* in, const float* k, float* out, int64_t B, int64_t H, int64_t L, int64_t K,
                          int64_t off, int reverse, int mode, cudaStream_t st, bool* handled) {
    *handled = false;
    if (L % 32 != 0 || L < 1024 || L >= (int64_t(1) << 30) || K > 8192 || K <= 32) return KS_OK;
    if ((reinterpret_cast<uintptr_t>(out) & 15) != 0) return KS_OK;
    constexpr int NT = kNT;
    PadGeom g{};
    // window origin t0 - off - lead on a 32-float piece; the first tap sits
    // `lead` floats in: `lead & ~3` leading zero taps plus a sub-quad offset S
    const int lead = static_cast<int>((32 - off % 32) % 32);
    const int S = lead & 3, zlead = lead - S;
    g.Ke = static_cast<int>(K) + zlead;
    g.Kp = (g.Ke + 31) / 32 * 32;
    g.Kpp = g.Kp;  // the mirrored path (set below) stages taps at the window's pitch
    g.base_row = static_cast<int>((off + lead) / 32);
    g.off = static_cast<int>(off);
    g.zlead = zlead;
    g.skip = opt(kOptPadSkip) != 0;
    // batch-lane kernel: K comparable to L (the per-lane tap ranges of the
    // row-tile kernel diverge there), at least one full warp of batch rows
    const int64_t bl_opt = opt(kOptStencilBl);
    if (bl_opt != 0 && B >= 32 && (bl_opt > 0 || 4 * K >= L) && B * H < (int64_t(1) << 31)) {
        BlGeom bg{};
        bg.Kp = g.Kp;
        bg.Ke = g.Ke;
        bg.base_row = g.base_row;
        bg.off = g.off;
        bg.zlead = g.zlead;
        bg.skip = g.skip;
        bg.ncol = static_cast<int>((L + kBlNW * kR - 1) / (kBlNW * kR));
        bg.ngrp = static_cast<int>((B + 31) / 32);
        CUtensorMap bm;
        if (bl_smem(bg) <= 200 * 1024 && int64_t(bg.ncol) * bg.ngrp * H < (int64_t(1) << 31) &&
            encode_padded_view(&bm, in, B * H, L, H, 1, 1, 32)) {
            float* kpb = nullptr;
            ks_status rc = cuda_status(scratch_alloc(reinterpret_cast<void**>(&kpb), sizeof(float) * H * g.Kp, st));
            if (rc != KS_OK) return rc;
            launch_kernel(prep_taps, static_cast<unsigned>(std::min<int64_t>((H * g.Kp + 255) / 256, 4096)), 256, 0,
                          st, k, kpb, H, K, int64_t(g.Kp), reverse, zlead);
            rc = check_launch();
            if (rc == KS_OK) {
                const bool fused = mode == KS_MULADD_FUSED;
                switch (S) {
                    case 0: rc = fused ? launch_bl<0, true>(bm, kpb, out, B, H, L, bg, st) : launch_bl<0, false>(bm, kpb, out, B, H, L, bg, st); break;
                    case 1: rc = fused ? launch_bl<1, true>(bm, kpb, out, B, H, L, bg, st) : launch_bl<1, false>(bm, kpb, out, B, H, L, bg, st); break;
                    case 2: rc = fused ? launch_bl<2, true>(bm, kpb, out, B, H, L, bg, st) : launch_bl<2, false>(bm, kpb, out, B, H, L, bg, st); break;
                    default: rc = fused ? launch_bl<3, true>(bm, kpb, out, B, H, L, bg, st) : launch_bl<3, false>(bm, kpb, out, B, H, L, bg, st); break;
                }
            }
            scratch_free(kpb, st);
            *handled = true;
            return rc;
        }
    }
    // Separate mode below K = 1024: the R = 32 register-tile kernel of
    // stencil_tma.cu is faster (two FP instructions per tap; round-2 ABAB,
    // gpurun_out/s10: config 4 fwd 9.50 -> 8.95 ms, dX 9.13 -> 8.93, 5b shard
    // fwd 10.01 -> 9.57), Fused mode and K >= 1024 keep this kernel (Fused
    // config 4 fwd 4.35 vs 5.80 ms).  Option stencil_pad = 2 forces it.
    if ((mode != KS_MULADD_FUSED && K < 1024) || K < 48) {
        // (and in Fused mode below K = 48, where a padded tile's 64 computed
        // taps outweigh the register tiles: K = 40 fwd 0.346 -> 0.318 ms,
        // gpurun_out/s27; from K = 48 on this kernel is ahead)
        if (opt(kOptStencilPad) < 2) return KS_OK;
    }
    g.mirror = 0;  // set below, once the tile width is known
    g.RPT = 1;
    while (g.RPT < 4 && static_cast<int64_t>(NT * kR / (2 * g.RPT)) >= L && H % (2 * g.RPT) == 0) g.RPT *= 2;
    g.TPR = NT / g.RPT;
    const int T = g.TPR * kR;
    g.mirror = g.skip && T >= L && 4 * K >= L && g.TPR % 64 == 0;
    if (g.mirror) g.Kpp = g.Kp / 32 * 36;
    g.NR = T / 32 + g.Kp / 32 + (S >= 2 ? 1 : 0);  // S >= 2: 13-quad windows read 4 floats further
    if (g.NR <= 256) {
        g.nbox = 1;
        g.NB = g.NR;
    } else if (g.RPT == 1 && g.NR <= 512) {
        g.nbox = 2;  // second box 128-byte aligned: NB a multiple of 8 (8 rows = 1152 B)
        g.NB = ((g.NR + 1) / 2 + 7) / 8 * 8;
    } else {
        return KS_OK;
    }
    g.win_floats = g.RPT * g.nbox * g.NB * 36;
    g.stage_bytes = (g.win_floats * 4 + g.RPT * g.Kpp * 4 + 1023) / 1024 * 1024;
    if (B * H / g.RPT * ((L + T - 1) / T) >= (int64_t(1) << 31)) return KS_OK;
    // stages: one in flight beyond the one being computed (a tile computes
    // ~10x longer than its load takes to land; two stages leave room for a
    // fourth CTA per SM, measured 1-1.5% faster than three at K = 128 / 256);
    // long K (>= 1024) computes ~100x longer than it loads: one stage
    int NS = K >= 1024 ? 1 : 2;
    while (NS > 1 && pad_smem(g, NS) > 110 * 1024) --NS;
    if (opt(kOptPadNs) > 0) NS = static_cast<int>(std::min<int64_t>(4, opt(kOptPadNs)));
    if (pad_smem(g, NS) > 220 * 1024) return KS_OK;
    CUtensorMap im;
    if (!encode_padded_view(&im, in, B * H, L, H, g.NB, g.RPT, 1)) return KS_OK;

    float* kp = nullptr;
    ks_status rc = cuda_status(scratch_alloc(reinterpret_cast<void**>(&kp), sizeof(float) * H * g.Kpp, st));
    if (rc != KS_OK) return rc;
    if (g.mirror)
        launch_kernel(prep_taps_pad36, static_cast<unsigned>(std::min<int64_t>((H * g.Kpp + 255) / 256, 4096)), 256,
                      0, st, k, kp, H, K, g.Kpp, reverse, zlead);
    else
        launch_kernel(prep_taps, static_cast<unsigned>(std::min<int64_t>((H * g.Kp + 255) / 256, 4096)), 256, 0, st,
                      k, kp, H, K, g.Kp, reverse, zlead);
    rc = check_launch();
    if (rc == KS_OK) {
        const bool fused = mode == KS_MULADD_FUSED;
        // long K: one stage, refilled after a CTA barrier; moderate K: producer lane
        const bool prod = opt(kOptPadProd) < 0 ? K < 1024 : opt(kOptPadProd) != 0;
        rc = prod ? launch_s<true>(S, fused, im, kp, out, B, H, L, g, NS, st)
                  : launch_s<false>(S, fused, im, kp, out, B, H, L, g, NS, st);
    }
    scratch_free(kp, st);
    *handled = true;
    return rc;
}

}  // namespace ks
