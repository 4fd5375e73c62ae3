// dw_cb.cu -- compute-bound weight gradient (long K), HIERARCHICAL order, sm_100a.
//
//   dk[h,j] = sum_b sum_t gy[b,h,t] * x[b,h,t+j-p]     (reference src/conv_core.cpp:148-181)
//
// The dual of stencil_cb.cu: there the taps are the short axis and the outputs
// the long one; here the outputs (taps j) sit in registers and the reduction
// runs over t.  CTA = (row group, channel h, tile of JT = 32*NJG taps), 256
// threads = NJG tap groups x NTS t-slices.  Per work item (row, TT-wide t
// tile) TMA stages gy and the x window; the CTA re-lays both out into padded
// buffers (36-float pitch per 32) and releases the stage so the next load
// overlaps the math.  A thread owns 32 taps and walks its t-slice in 32-t
// chunks of two 16-t register windows: 16 gy values (4 loads) and 47 x values
// (12 loads) feed 512 FMAs, all with compile-time shared-memory offsets.
// Accumulators stay in registers across all the CTA's rows; at the end the NTS
// partials of each tap are added in fixed t-slice order, one partial per CTA
// goes to part[g,h,j], and dw_sum_groups adds the G partials in ascending g.
// No atomics: deterministic for a fixed shape.
#include <algorithm>
#include <cstdlib>

#include "ks_common.cuh"
#include "ks_tma.cuh"

namespace ks {

namespace {

constexpr int kNT = 256;
constexpr int kIn = 32;
constexpr int kJR = 32;   // taps per thread
constexpr int kTW = 16;   // t per register window
constexpr int kNVX = (kJR + kTW - 1 + 3) / 4;  // 12 float4

struct DwCbGeom {
    int TT;           // t per work item
    int JT;           // taps per CTA
    int XW;           // x window floats staged (multiple of 32)
    int gy_bytes, x_bytes, stage_bytes;
    int pg_floats, px_floats;
};

__device__ __forceinline__ int padi(int i) { return i + ((i >> 5) << 2); }

template <int NJG, bool FUSED>
__global__ void __launch_bounds__(kNT)
dw_cb(const __grid_constant__ CUtensorMap gy_map, const __grid_constant__ CUtensorMap x_map,
      float* __restrict__ part, int B, int H, int L, int K, int G, int NJT, DwCbGeom g) {
    constexpr int NTS = kNT / NJG;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = align_smem<1024>(smem_raw);
    const float* sgy = reinterpret_cast<const float*>(smem);
    const float* sx = reinterpret_cast<const float*>(smem + g.gy_bytes);
    float* pg = reinterpret_cast<float*>(smem + g.stage_bytes);
    float* px = pg + g.pg_floats;
    uint64_t* full = reinterpret_cast<uint64_t*>(px + g.px_floats);

    int bid = blockIdx.x;
    const int jt = bid % NJT;
    bid /= NJT;
    const int h = bid % H;
    const int grp = bid / H;
    const int b_begin = static_cast<int>(static_cast<int64_t>(B) * grp / G);
    const int b_end = static_cast<int>(static_cast<int64_t>(B) * (grp + 1) / G);
    const int j0 = jt * g.JT;
    const int p = K / 2;
    const int tid = threadIdx.x;
    const int jg = tid / NTS, ts = tid - jg * NTS;
    const int ntt = (L + g.TT - 1) / g.TT;
    const int nunits = (b_end - b_begin) * ntt;
    const int xoff = j0 - p;
    const int D = ((xoff % kIn) + kIn) % kIn;
    const int xr_rel = (xoff - D) / kIn;

    if (tid == 0) {
        prefetch_tmap(&gy_map);
        prefetch_tmap(&x_map);
        mbar_init(full, 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint32_t tx_bytes = static_cast<uint32_t>(g.gy_bytes + g.x_bytes);
    auto issue = [&](int u) {
        const int b = b_begin + u / ntt;
        const int t0 = (u % ntt) * g.TT;
        const int row = b * H + h;
        mbar_arrive_expect_tx(full, tx_bytes);
        tma_load_3d(smem, &gy_map, 0, t0 / kIn, row, full);
        const int xr = t0 / kIn + xr_rel;
        const int xrows = g.XW / kIn;
        const int half = xrows > 256 ? xrows / 2 : xrows;
        tma_load_3d(smem + g.gy_bytes, &x_map, 0, xr, row, full);
        if (half != xrows) tma_load_3d(smem + g.gy_bytes + half * 128, &x_map, 0, xr + half, row, full);
    };
    if (tid == 0 && nunits > 0) issue(0);

    float acc[kJR];
#pragma unroll
    for (int i = 0; i < kJR; ++i) acc[i] = 0.f;

    const int nchunks = g.TT / 32;
    for (int u = 0; u < nunits; ++u) {
        mbar_wait(full, static_cast<uint32_t>(u & 1));
        // re-layout: pg[padi(t)] = gy tile, px[padi(i)] = x window shifted by D
        for (int i = tid; i < g.TT; i += kNT) pg[padi(i)] = sgy[i];
        for (int i = tid; i < g.XW - 32; i += kNT) px[padi(i)] = sx[i + D];
        __syncthreads();
        if (tid == 0 && u + 1 < nunits) issue(u + 1);  // next load overlaps this item's math

        for (int c = ts; c < nchunks; c += NTS) {
            const float* gb = pg + c * 36;              // padi(32c)
            const float* xb = px + (c + jg) * 36;       // padi(32c + 32jg)
            auto window = [&](const int sub) {
                float gv[kTW];
#pragma unroll
                for (int q = 0; q < kTW / 4; ++q) {
                    const float4 a = *reinterpret_cast<const float4*>(gb + sub + 4 * q + (((sub + 4 * q) >> 5) << 2));
                    gv[4 * q + 0] = a.x;
                    gv[4 * q + 1] = a.y;
                    gv[4 * q + 2] = a.z;
                    gv[4 * q + 3] = a.w;
                }
                float xv[4 * kNVX];
#pragma unroll
                for (int q = 0; q < kNVX; ++q) {
                    const float4 a = *reinterpret_cast<const float4*>(xb + sub + 4 * q + (((sub + 4 * q) >> 5) << 2));
                    xv[4 * q + 0] = a.x;
                    xv[4 * q + 1] = a.y;
                    xv[4 * q + 2] = a.z;
                    xv[4 * q + 3] = a.w;
                }
#pragma unroll
                for (int tt = 0; tt < kTW; ++tt)
#pragma unroll
                    for (int jj = 0; jj < kJR; ++jj) acc[jj] = muladd<FUSED>(acc[jj], gv[tt], xv[tt + jj]);
            };
            window(0);
            window(16);
        }
        __syncthreads();  // padded buffers free for the next item
    }

    // fixed-order reduction over the NTS t-slices of each tap group
    float* red = px;  // [kNT][kJR + 1], reused
#pragma unroll
    for (int jj = 0; jj < kJR; ++jj) red[tid * (kJR + 1) + jj] = acc[jj];
    __syncthreads();
    for (int o = tid; o < g.JT; o += kNT) {
        const int gj = o / kJR, jj = o % kJR;
        float s = 0.f;
        for (int q = 0; q < NTS; ++q) s += red[(gj * NTS + q) * (kJR + 1) + jj];
        const int j = j0 + o;
        if (j < K) part[(static_cast<int64_t>(grp) * H + h) * K + j] = s;
    }
}

template <int NJG, bool FUSED>
ks_status launch(const CUtensorMap& gm, const CUtensorMap& xm, float* part, int64_t B, int64_t H, int64_t L,
                 int64_t K, int G, int NJT, const DwCbGeom& g, cudaStream_t st) {
    auto kern = dw_cb<NJG, FUSED>;
    const int smem = g.stage_bytes + (g.pg_floats + g.px_floats) * 4 + 64 + 1024;
    prepare_kernel(reinterpret_cast<const void*>(kern), kNT, smem);
    kern<<<static_cast<unsigned>(int64_t(G) * H * NJT), kNT, smem, st>>>(
        gm, xm, part, static_cast<int>(B), static_cast<int>(H), static_cast<int>(L), static_cast<int>(K), G, NJT, g);
    return check_launch();
}

}  // namespace

// Envelope of the compute-bound dW kernel (K >= 128, L >= 2048, L % 32 == 0).
bool dw_cb_applies(int64_t B, int64_t H, int64_t L, int64_t K) {
    return K >= 128 && K < (int64_t(1) << 30) && L >= 2048 && L % kIn == 0 && L < (int64_t(1) << 30) &&
           B * H < (int64_t(1) << 31);
}

// Row groups for dw_cb: enough CTAs to fill the GPU a few times over.
int dw_cb_groups(int64_t B, int64_t H, int64_t K) {
    int njg = 4;
    while (njg < 32 && njg * kJR < K) njg *= 2;
    const int64_t njt = (K + njg * kJR - 1) / (njg * kJR);
    int64_t G = (2048 + H * njt - 1) / (H * njt);
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(G, B)));
}

ks_status dw_pad_stage1(const float* gy, const float* x, float* part, int64_t B, int64_t H, int64_t L, int64_t K,
                        int G, int mode, cudaStream_t st, bool* handled);

ks_status dw_cb_stage1(const float* gy, const float* x, float* part, int64_t B, int64_t H, int64_t L, int64_t K,
                       int G, int mode, cudaStream_t st, bool* handled) {
    *handled = false;
    {  // padded TMA view (dw_pad.cu); KS_CB_IMPL=1 selects the kernels below (A/B knob)
        const char* e = getenv("KS_CB_IMPL");
        if (!(e && atoi(e) == 1)) {
            const ks_status s = dw_pad_stage1(gy, x, part, B, H, L, K, G, mode, st, handled);
            if (*handled) return s;
        }
    }
    if (!dw_cb_applies(B, H, L, K)) return KS_OK;
    int njg = 4;
    while (njg < 32 && njg * kJR < K) njg *= 2;
    const int nts = kNT / njg;
    DwCbGeom g;
    g.JT = njg * kJR;
    // t per work item: >= 2 chunks of 32 per thread (amortises the re-layout),
    // capped by the row
    g.TT = std::min<int64_t>(std::max(64 * nts, 4096), (L + 31) / 32 * 32);
    g.TT = std::max(g.TT, 32 * nts);
    const int njt = static_cast<int>((K + g.JT - 1) / g.JT);
    if (int64_t(G) * H * njt >= (int64_t(1) << 31)) return KS_OK;
    g.XW = (g.TT + g.JT + 32 + 31) / 32 * 32 + 32;  // window + the D shift + read overrun
    if (g.XW / kIn > 512 || g.TT / kIn > 256) return KS_OK;
    g.gy_bytes = g.TT * 4;
    g.x_bytes = g.XW * 4;
    g.stage_bytes = (g.gy_bytes + g.x_bytes + 1023) / 1024 * 1024;
    g.pg_floats = (g.TT / 32) * 36;
    g.px_floats = std::max((g.XW / 32) * 36, kNT * (kJR + 1));
    const int xrows = g.XW / kIn;
    if (xrows > 256 && (xrows & 1)) return KS_OK;
    CUtensorMap gm, xm;
    if (!encode_row_view(&gm, gy, B * H, L, kIn, g.TT / kIn, 0)) return KS_OK;
    if (!encode_row_view(&xm, x, B * H, L, kIn, xrows > 256 ? xrows / 2 : xrows, 0)) return KS_OK;
    const bool fused = mode == KS_MULADD_FUSED;
    *handled = true;
    switch (njg) {
        case 4: return fused ? launch<4, true>(gm, xm, part, B, H, L, K, G, njt, g, st)
                             : launch<4, false>(gm, xm, part, B, H, L, K, G, njt, g, st);
        case 8: return fused ? launch<8, true>(gm, xm, part, B, H, L, K, G, njt, g, st)
                             : launch<8, false>(gm, xm, part, B, H, L, K, G, njt, g, st);
        case 16: return fused ? launch<16, true>(gm, xm, part, B, H, L, K, G, njt, g, st)
                              : launch<16, false>(gm, xm, part, B, H, L, K, G, njt, g, st);
        default: return fused ? launch<32, true>(gm, xm, part, B, H, L, K, G, njt, g, st)
                              : launch<32, false>(gm, xm, part, B, H, L, K, G, njt, g, st);
    }
}

}  // namespace ks
