// dw_pad.cu -- compute-bound weight gradient (K >= 128), HIERARCHICAL order,
// sm_100a, fed straight from TMA in the padded layout (see stencil_pad.cu).
//
//   dk[h,j] = sum_b sum_t gy[b,h,t] * x[b,h,t+j-p]     (reference src/conv_core.cpp:148-181)
//
// CTA = (row group g, channel h, tile of JT = 32*NJG taps), 256 threads = NJG
// tap groups x NTS t-slices.  A thread owns 32 taps (registers) and walks its
// t-slice in 32-t chunks of two 16-t register windows: 16 gy values (4 loads)
// and 47 x values (12 loads) feed 512 FMAs at compile-time shared offsets.
// Work item = (row b, TT-wide t tile): TMA brings gy[t0, t0+TT) and the x
// window as 36-float padded rows (box {36, n, 1, 1} of the padded view, the
// 4 floats past each 32-float piece out of bounds and zero-filled), so the CTA computes straight from an NS-stage ring with no
// re-layout; one producer lane keeps the ring NS items ahead (full / empty
// mbarriers; every consumer thread arrives on a stage's empty barrier once it
// is done with it).  The x window must start on a 32-float piece, so tap
// tiles start at j0 = base + jt*JT with base = (p mod 32) - 32 (or 0), making t0 + j0 - p
// a multiple of 32; taps outside [0, K) are computed on zero-weight and not
// written.  Accumulators stay in registers across all the CTA's work items;
// then the NTS partials of each tap are added in fixed t-slice order, one
// partial per CTA goes to part[g,h,j], and dw_sum_groups adds the G partials
// in ascending g.  No atomics: deterministic for a fixed shape.
#include <algorithm>
#include <cstdlib>

#include "ks_common.cuh"
#include "ks_tma.cuh"

#ifndef KS_DWPAD_ANTIDIAG
#define KS_DWPAD_ANTIDIAG 1  // anti-diagonal FFMA order with the uniform-gy mapping (-3.9% at K = 1024 / 4096)
#endif
#ifndef KS_DWPAD_LANEJG
#define KS_DWPAD_LANEJG 1  // A/B (tools/build_variant.sh): lanes = tap groups at NJG = 32
#endif

namespace ks {

namespace {

constexpr int kNT = 256;
constexpr int kJR = 32;                         // taps per thread
constexpr int kTW = 16;                         // t per register window
constexpr int kNVX = (kJR + kTW - 1 + 3) / 4;  // 12 float4

struct DwPadGeom {
    int TT;            // t per work item (multiple of 32)
    int JT, NJT;       // taps per CTA, tap tiles
    int base;          // first tap of tile 0 (<= 0)
    int gy_rows;       // TT/32
    int gy_alloc;      // gy rows rounded up to a multiple of 8 (128-byte aligned x box)
    int NBX, nbx;      // x rows per box, x boxes (window = (TT + JT)/32 rows)
    int stage_bytes;   // 1024-aligned
    int skip;          // skip chunks that read only zero halo (KS_PAD_SKIP=0: compute them)
};

template <int NJG, bool FUSED>
__global__ void __launch_bounds__(kNT + 32, 2)
dw_pad(const __grid_constant__ CUtensorMap gy_map, const __grid_constant__ CUtensorMap x_map,
       float* __restrict__ part, int B, int H, int L, int K, int G, DwPadGeom g, int NS) {
    constexpr int NTS = kNT / NJG;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = align_smem<1024>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * g.stage_bytes);

    int bid = blockIdx.x;
    const int jt = bid % g.NJT;
    bid /= g.NJT;
    const int h = bid % H;
    const int grp = bid / H;
    const int b_begin = static_cast<int>(static_cast<int64_t>(B) * grp / G);
    const int b_end = static_cast<int>(static_cast<int64_t>(B) * (grp + 1) / G);
    const int j0 = g.base + jt * g.JT;
    const int p = K / 2;
    const int tid = threadIdx.x;
    // NJG = 32 (K >= 1024): lanes are the 32 tap groups and a warp is one
    // t-slice, so the gy values of a chunk are warp-uniform (uniform registers,
    // the FFMA then reads two RF operands; bits unchanged: the same (tap
    // group, t-slice) work and reduction order, only the thread numbering
    // moves).  Otherwise a warp spans several t-slices of NJG groups.
    constexpr bool LANE_JG = NJG == 32 && KS_DWPAD_LANEJG;
    const int jg = LANE_JG ? (tid & 31) : tid / NTS;
    const int ts = LANE_JG ? __shfl_sync(0xffffffffu, tid >> 5, 0) : tid - jg * NTS;
    const int ntt = (L + g.TT - 1) / g.TT;
    const int nunits = (b_end - b_begin) * ntt;
    const int xrow_rel = (j0 - p) / 32;  // exact: j0 - p is a multiple of 32

    uint64_t* empty = full + NS;
    if (tid == 0) {
        prefetch_tmap(&gy_map);
        prefetch_tmap(&x_map);
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kNT);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (tid >= kNT) {  // producer warp: one lane issues the loads, NS items ahead
        if (tid == kNT) {
            const uint32_t tx_bytes = static_cast<uint32_t>((g.gy_rows + g.nbx * g.NBX) * 144);
            // stage / phase / (row, tile) carried incrementally: no integer
            // divisions by the runtime NS and tile count per item
            int stage = 0, b = b_begin, r0 = 0;
            uint32_t phase = 0;
            for (int u = 0; u < nunits; ++u) {
                if (u >= NS) mbar_wait_sleep(&empty[stage], phase ^ 1u);
                unsigned char* sb = smem + stage * g.stage_bytes;
                mbar_arrive_expect_tx(&full[stage], tx_bytes);
                tma_load_pad(sb, &gy_map, r0, h, b, &full[stage]);
                unsigned char* xb = sb + g.gy_alloc * 144;
                tma_load_pad(xb, &x_map, r0 + xrow_rel, h, b, &full[stage]);
                if (g.nbx > 1) tma_load_pad(xb + g.NBX * 144, &x_map, r0 + xrow_rel + g.NBX, h, b, &full[stage]);
                r0 += g.TT / 32;
                if (r0 * 32 >= L) {
                    r0 = 0;
                    ++b;
                }
                if (++stage == NS) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
        return;
    }

    float acc[kJR];
#pragma unroll
    for (int i = 0; i < kJR; ++i) acc[i] = 0.f;

    const int nchunks = g.TT / 32;
    // this warp's lanes: tap groups [jgw, jgw + JGW) x t-slices [ts_lo, ts_lo + TSW)
    constexpr int JGW = LANE_JG ? 32 : NTS >= 32 ? 1 : 32 / NTS;
    constexpr int TSW = LANE_JG ? 1 : NTS >= 32 ? 32 : NTS;
    const int jgw = LANE_JG ? 0 : (tid & ~31) / NTS;
    const int ts_lo = LANE_JG ? ts : NTS >= 32 ? (tid & ~31) % NTS : 0;
    const int xw_lo = j0 + 32 * jgw - p + 32 * ts_lo;                         // + t0 of the chunk row
    const int xw_hi = j0 + 32 * (jgw + JGW) - 1 - p + 32 * (ts_lo + TSW) - 1;  // (chunk base i * NTS)
    int stage = 0, tu = 0;
    uint32_t phase = 0;
    // barrier addresses in registers (not re-derived from SR_CgaCtaId per item)
    const uint32_t full_u = opaque_u32(smem_u32(full)), empty_u = full_u + 8u * NS;
    for (int u = 0; u < nunits; ++u) {
        mbar_wait_u32(full_u + 8u * stage, phase);
        const float* pg = reinterpret_cast<const float*>(smem + stage * g.stage_bytes);
        const float* px = pg + g.gy_alloc * 36;
        for (int c = ts; c < nchunks; c += NTS) {
            // skip the chunk when, for the whole warp, every x it would read is
            // zero halo: gy * 0 never changes a sum that starts at +0 (and the
            // reference's WeightTerm skips those terms).  x positions are
            // t + j - p over the warp's chunks and taps.
            const int cb = tu + 32 * (c - ts);
            const int xlo = cb + xw_lo, xhi = cb + xw_hi;
            if (g.skip && (xhi < 0 || xlo >= L)) continue;
            const float* gb = pg + c * 36;         // padded row c of the gy tile
            const float* xb = px + (c + jg) * 36;  // padded row c + jg of the x window
            auto window = [&](const int sub) {
                float gv[kTW];
#pragma unroll
                for (int q = 0; q < kTW / 4; ++q) {
                    const float4 a = lds4(gb + sub + 4 * q + (((sub + 4 * q) >> 5) << 2));
                    gv[4 * q + 0] = a.x;
                    gv[4 * q + 1] = a.y;
                    gv[4 * q + 2] = a.z;
                    gv[4 * q + 3] = a.w;
                }
                float xv[4 * kNVX];
#pragma unroll
                for (int q = 0; q < kNVX; ++q) {
                    const float4 a = lds4(xb + sub + 4 * q + (((sub + 4 * q) >> 5) << 2));
                    xv[4 * q + 0] = a.x;
                    xv[4 * q + 1] = a.y;
                    xv[4 * q + 2] = a.z;
                    xv[4 * q + 3] = a.w;
                }
                if constexpr (LANE_JG && KS_DWPAD_ANTIDIAG) {
                    // gy is uniform here: order by x value (m = tt + jj) so it
                    // stays in the operand-reuse cache; acc[jj] still sees tt ascending
#pragma unroll
                    for (int m = 0; m < kTW + kJR - 1; ++m)
#pragma unroll
                        for (int tt = 0; tt < kTW; ++tt) {
                            const int jj = m - tt;
                            if (jj >= 0 && jj < kJR) acc[jj] = muladd<true>(acc[jj], gv[tt], xv[m]);
                        }
                } else {
#pragma unroll
                    for (int tt = 0; tt < kTW; ++tt)
#pragma unroll
                        for (int jj = 0; jj < kJR; ++jj) acc[jj] = muladd<true>(acc[jj], gv[tt], xv[tt + jj]);
                }
            };
            window(0);
            window(16);
        }
        mbar_arrive_u32(empty_u + 8u * stage);  // this thread is done with the stage
        if (++stage == NS) {
            stage = 0;
            phase ^= 1u;
        }
        tu += g.TT;
        if (tu >= L) tu = 0;
    }

    // fixed-order reduction over the NTS t-slices of each tap group; the stage
    // ring is idle once every consumer warp is past its last item (every
    // issued load has been consumed); consumers sync on named barrier 1
    asm volatile("bar.sync 1, %0;" ::"n"(kNT) : "memory");
    float* red = reinterpret_cast<float*>(smem);  // [kNT][kJR + 1]
#pragma unroll
    for (int jj = 0; jj < kJR; ++jj) red[tid * (kJR + 1) + jj] = acc[jj];
    asm volatile("bar.sync 1, %0;" ::"n"(kNT) : "memory");
    for (int o = tid; o < g.JT; o += kNT) {
        const int gj = o / kJR, jj = o % kJR;
        float s = 0.f;
        for (int q = 0; q < NTS; ++q) s += red[(LANE_JG ? q * 32 + gj : gj * NTS + q) * (kJR + 1) + jj];
        const int j = j0 + o;
        if (j >= 0 && j < K) part[(static_cast<int64_t>(grp) * H + h) * K + j] = s;
    }
}

int dwpad_smem(const DwPadGeom& g, int NS) {
    return std::max(NS * g.stage_bytes, kNT * (kJR + 1) * 4) + 128 + 1024;
}

template <int NJG, bool FUSED>
ks_status launch(const CUtensorMap& gm, const CUtensorMap& xm, float* part, int64_t B, int64_t H, int64_t L,
                 int64_t K, int G, const DwPadGeom& g, int NS, cudaStream_t st) {
    auto kern = dw_pad<NJG, FUSED>;
    const int smem = dwpad_smem(g, NS);
    prepare_kernel(reinterpret_cast<const void*>(kern), kNT + 32, smem);
    launch_kernel(kern, static_cast<unsigned>(int64_t(G) * H * g.NJT), kNT + 32, smem, st, 
        gm, xm, part, static_cast<int>(B), static_cast<int>(H), static_cast<int>(L), static_cast<int>(K), G, g, NS);
    return check_launch();
}

}  // namespace

// Tap groups of 32 per CTA for K (the tile starts `base` <= 0 taps early so
// the x window sits on a 32-float piece).
static int dwpad_njg(int64_t K) {
    const int p = static_cast<int>(K / 2);
    const int64_t KK = K - (p % 32 ? p % 32 - 32 : 0);
    int njg = 1;
    while (njg < 32 && njg * kJR < KK) njg *= 2;
    return njg;
}

// Envelope of the compute-bound dW kernel: K >= dwpad_min_k (48 by default:
// round-2 ABAB against dw_tma, gpurun_out/s21 -- K = 48 / 64 / 100 at
// L >= 4096: -21 / -14 / -29%; K = 24 / 32: +29-40%, so they stay on dw_tma),
// L >= 2048, L % 32 == 0, and a row at least one work item long for the
// tap-group count (2048 / 4096 / 8192 t at 4+ / 2 / 1 groups).
bool dw_pad_applies(int64_t B, int64_t H, int64_t L, int64_t K) {
    if (!(K >= std::max<int64_t>(17, opt(kOptDwpadMinK)) && K <= 8192 && L >= 2048 && L % 32 == 0 &&
          L < (int64_t(1) << 30) && B * H < (int64_t(1) << 31)))
        return false;
    return L >= 32 * (kNT / dwpad_njg(K));
}

// Row groups G of dw_pad's partial buffer: enough CTAs to fill the GPU a few
// times over (G * H * tap tiles ~ 2048).
int dw_pad_groups(int64_t B, int64_t H, int64_t K) {
    int njg = 4;
    while (njg < 32 && njg * kJR < K) njg *= 2;
    const int64_t njt = (K + njg * kJR - 1) / (njg * kJR);
    const int64_t G = (2048 + H * njt - 1) / (H * njt);
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(G, B)));
}

// Compute-bound dW stage 1 from the padded TMA view (K >= 128, L >= 2048,
// L % 32 == 0), into part[G,H,K].  *handled = false outside the envelope.
ks_status dw_pad_stage1(const float* gy, const float* x, float* part, int64_t B, int64_t H, int64_t L, int64_t K,
                        int G, int mode, cudaStream_t st, bool* handled) {
    *handled = false;
    if (!dw_pad_applies(B, H, L, K)) return KS_OK;
    DwPadGeom g{};
    const int p = static_cast<int>(K / 2);
    g.base = p % 32 ? p % 32 - 32 : 0;
    const int64_t KK = K - g.base;  // taps to cover, from base
    const int njg = dwpad_njg(K);
    const int nts = kNT / njg;
    g.JT = njg * kJR;
    g.NJT = static_cast<int>((KK + g.JT - 1) / g.JT);
    if (int64_t(G) * H * g.NJT >= (int64_t(1) << 31)) return KS_OK;
    // t per work item: >= 2 chunks of 32 per thread, capped by the row and by
    // one TMA box (256 rows)
    int64_t TT = std::min<int64_t>(std::max(64 * nts, 4096), L);
    TT = std::max<int64_t>(TT, 32 * nts);
    TT = std::min<int64_t>(TT, 8192);
    g.TT = static_cast<int>(TT);
    g.gy_rows = g.TT / 32;
    g.gy_alloc = (g.gy_rows + 7) / 8 * 8;
    const int xr = (g.TT + g.JT) / 32;
    if (xr <= 256) {
        g.nbx = 1;
        g.NBX = xr;
    } else if (xr <= 512) {
        g.nbx = 2;
        g.NBX = ((xr + 1) / 2 + 7) / 8 * 8;
    } else {
        return KS_OK;
    }
    g.stage_bytes = ((g.gy_alloc + g.nbx * g.NBX) * 144 + 1023) / 1024 * 1024;
    g.skip = opt(kOptPadSkip) != 0;
    int NS = 3;
    while (NS > 2 && dwpad_smem(g, NS) > 110 * 1024) --NS;
    if (opt(kOptDwpadNs) > 0) NS = static_cast<int>(opt(kOptDwpadNs));  // tuning option
    if (dwpad_smem(g, NS) > 220 * 1024) return KS_OK;
    CUtensorMap gm, xm;
    if (!encode_padded_view(&gm, gy, B * H, L, H, g.gy_rows, 1, 1)) return KS_OK;
    if (!encode_padded_view(&xm, x, B * H, L, H, g.NBX, 1, 1)) return KS_OK;
    (void)mode;  // HIERARCHICAL accumulates with FMA in either MulAddMode (conv_dw.cu)
    *handled = true;
    switch (njg) {
        case 1: return launch<1, true>(gm, xm, part, B, H, L, K, G, g, NS, st);
        case 2: return launch<2, true>(gm, xm, part, B, H, L, K, G, g, NS, st);
        case 4: return launch<4, true>(gm, xm, part, B, H, L, K, G, g, NS, st);
        case 8: return launch<8, true>(gm, xm, part, B, H, L, K, G, g, NS, st);
        case 16: return launch<16, true>(gm, xm, part, B, H, L, K, G, g, NS, st);
        default: return launch<32, true>(gm, xm, part, B, H, L, K, G, g, NS, st);
    }
}

}  // namespace ks
