// conv_tma.cu -- TMA-pipelined sm_100a kernels for rows with L % 32 == 0.
//
// Stencil (forward y / input-gradient dX, reference src/conv_core.cpp:21-75):
//   persistent CTAs walk (row, 4096-output tile) work items; one thread keeps
//   NS-1 tiles in flight with cp.async.bulk.tensor loads of the input window
//   (TMA zero-fills the halo outside the row) plus a 1-D bulk copy of the
//   channel's taps, all completing on one mbarrier per stage.  Every thread
//   then keeps R consecutive outputs in registers and slides a register window
//   over the taps in ascending j (bit-identical to the reference), reading the
//   128B-swizzled window with conflict-free 128-bit shared loads, and writes
//   its outputs with 128-bit streaming stores.
//
// dW (reference src/conv_core.cpp:148-181), HIERARCHICAL order:
//   CTA = (row group, channel h, 8*NJ-tap tile).  Work items are
//   (row b, 2048-wide t tile); each stage holds the gy tile and the x window
//   [t0+j0-p, ...) loaded by TMA.  Thread (tap group, t-slice) accumulates
//   8 taps x 8 t per register block with FMAs, then a fixed shuffle tree, a
//   fixed pass over warps and a per-CTA partial; the cross-block pass is
//   dw_sum_groups in conv_dw.cu.  No atomics, fixed order -> deterministic.
#include <algorithm>

#include "ks_common.cuh"
#include "ks_tma.cuh"

namespace ks {

// ---------------------------------------------------------------------------
// tensor-map encoding (driver entry point fetched through the runtime)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

bool encode_row_view(CUtensorMap* map, const float* base, int64_t rows, int64_t L, int box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || (L % 32) != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
    if (rows > (int64_t(1) << 31) || L / 32 > (int64_t(1) << 31) || box_rows < 1 || box_rows > 256) return false;
    const cuuint64_t dims[3] = {32, static_cast<cuuint64_t>(L / 32), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[2] = {128, static_cast<cuuint64_t>(L) * 4};
    const cuuint32_t box[3] = {32, static_cast<cuuint32_t>(box_rows), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// ---------------------------------------------------------------------------
// taps: kp[h, 0:Kp) = k[h, j] (forward) or k[h, K-1-j] (dX), zero padded

__global__ void prep_taps(const float* __restrict__ k, float* __restrict__ kp, int64_t H, int64_t K, int64_t Kp,
                          int reverse) {
    const int64_t n = H * Kp;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t h = i / Kp, j = i - h * Kp;
        kp[i] = j < K ? k[h * K + (reverse ? K - 1 - j : j)] : 0.f;
    }
}

// ---------------------------------------------------------------------------
// stencil

constexpr int kThreads = 256;
constexpr int kJB = 8;

struct StencilGeom {
    int T;         // outputs per tile
    int HL, HR;    // halo rows (32 floats) before / after the tile
    int NRB;       // window rows per stage (loaded)
    int A;         // (32*HL - off) & ~3: float offset of output 0's first tap, 4-aligned
    int Kp;        // taps padded to a multiple of 8 (and of 32 floats in smem)
    int win_bytes; // NRB*128 rounded
    int stage_bytes;
};

template <int R, int S, bool FUSED>
__global__ void __launch_bounds__(kThreads)
stencil_tma(const __grid_constant__ CUtensorMap in_map, const float* __restrict__ kp, float* __restrict__ out,
            int H, int L, int K, int tiles_per_row, int64_t ntiles, StencilGeom g, int NS) {
    constexpr int NV = (S + R + kJB - 1 + 3) / 4;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-align the dynamic buffer (the runtime only guarantees 16 B)
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * g.stage_bytes);
    const int tid = threadIdx.x;

    if (tid == 0) {
        prefetch_tmap(&in_map);
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint32_t tx_bytes = static_cast<uint32_t>(g.NRB) * 128u + static_cast<uint32_t>(g.Kp) * 4u;
    auto issue = [&](int stage, int64_t tile) {
        const int64_t row = tile / tiles_per_row;
        const int t0 = static_cast<int>(tile - row * tiles_per_row) * g.T;
        unsigned char* sb = smem + stage * g.stage_bytes;
        mbar_arrive_expect_tx(&full[stage], tx_bytes);
        tma_load_3d(sb, &in_map, 0, t0 / 32 - g.HL, static_cast<int>(row), &full[stage]);
        const int h = static_cast<int>(row % H);
        bulk_load(sb + g.win_bytes, kp + static_cast<int64_t>(h) * g.Kp, static_cast<uint32_t>(g.Kp) * 4u,
                  &full[stage]);
    };

    int64_t tile = blockIdx.x;
    if (tid == 0)
        for (int s = 0; s < NS; ++s) {
            const int64_t t = tile + static_cast<int64_t>(s) * gridDim.x;
            if (t < ntiles) issue(s, t);
        }

    const int base = tid * R;
    const int Kfull = K - K % kJB;
    for (int it = 0; tile < ntiles; tile += gridDim.x, ++it) {
        const int stage = it % NS;
        mbar_wait(&full[stage], static_cast<uint32_t>((it / NS) & 1));
        const char* win = reinterpret_cast<const char*>(smem + stage * g.stage_bytes);
        const float* wk = reinterpret_cast<const float*>(win + g.win_bytes);
        const int64_t row = tile / tiles_per_row;
        const int t0 = static_cast<int>(tile - row * tiles_per_row) * g.T;

        if (t0 + base < L) {
            float acc[R];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = 0.f;
            auto block = [&](int j0, int nj) {
                float v[4 * NV];
                const uint32_t i0 = static_cast<uint32_t>(base + g.A + j0);
#pragma unroll
                for (int c = 0; c < NV; ++c) {
                    const float4 q = lds128(win, swz128(i0 + 4 * c));
                    v[4 * c + 0] = q.x;
                    v[4 * c + 1] = q.y;
                    v[4 * c + 2] = q.z;
                    v[4 * c + 3] = q.w;
                }
                float w[kJB];
#pragma unroll
                for (int c = 0; c < kJB / 4; ++c) {
                    const float4 q = *reinterpret_cast<const float4*>(wk + j0 + 4 * c);
                    w[4 * c + 0] = q.x;
                    w[4 * c + 1] = q.y;
                    w[4 * c + 2] = q.z;
                    w[4 * c + 3] = q.w;
                }
#pragma unroll
                for (int jj = 0; jj < kJB; ++jj)
                    if (jj < nj) {
#pragma unroll
                        for (int r = 0; r < R; ++r) acc[r] = muladd<FUSED>(acc[r], v[S + r + jj], w[jj]);
                    }
            };
            for (int j0 = 0; j0 < Kfull; j0 += kJB) block(j0, kJB);
            if (Kfull < K) block(Kfull, K - Kfull);
            float* o = out + row * static_cast<int64_t>(L) + t0 + base;
#pragma unroll
            for (int r = 0; r < R; r += 4) st_cs_v4(o + r, make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]));
        }
        __syncthreads();  // every thread is done with this stage
        if (tid == 0) {
            const int64_t nt = tile + static_cast<int64_t>(NS) * gridDim.x;
            if (nt < ntiles) issue(stage, nt);
        }
    }
}

template <int R, int S, bool FUSED>
static ks_status launch_stencil_tma(const CUtensorMap& map, const float* kp, float* out, int64_t B, int64_t H,
                                    int64_t L, int64_t K, const StencilGeom& g, int NS, cudaStream_t st) {
    auto kern = stencil_tma<R, S, FUSED>;
    const size_t smem = size_t(NS) * g.stage_bytes + 64 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
    if (per_sm < 1) per_sm = 1;
    const int tiles_per_row = static_cast<int>((L + g.T - 1) / g.T);
    const int64_t ntiles = B * H * tiles_per_row;
    const int64_t grid = std::min<int64_t>(ntiles, int64_t(num_sms()) * per_sm);
    kern<<<static_cast<unsigned>(grid), kThreads, smem, st>>>(map, kp, out, static_cast<int>(H), static_cast<int>(L),
                                                                static_cast<int>(K), tiles_per_row, ntiles, g, NS);
    return check_launch();
}

template <int R, bool FUSED>
static ks_status dispatch_s(int s, const CUtensorMap& map, const float* kp, float* out, int64_t B, int64_t H,
                            int64_t L, int64_t K, const StencilGeom& g, int NS, cudaStream_t st) {
    switch (s) {
        case 0: return launch_stencil_tma<R, 0, FUSED>(map, kp, out, B, H, L, K, g, NS, st);
        case 1: return launch_stencil_tma<R, 1, FUSED>(map, kp, out, B, H, L, K, g, NS, st);
        case 2: return launch_stencil_tma<R, 2, FUSED>(map, kp, out, B, H, L, K, g, NS, st);
        default: return launch_stencil_tma<R, 3, FUSED>(map, kp, out, B, H, L, K, g, NS, st);
    }
}

// Returns KS_ERR_BAD_MODE (as "not handled") when this path does not apply, so
// the caller falls back to the generic tile kernel.
ks_status stencil_tma_f32(const float* in, const float* k, float* out, int64_t B, int64_t H, int64_t L, int64_t K,
                          int64_t off, int reverse, int mode, cudaStream_t st, bool* handled) {
    *handled = false;
    if (L % 32 != 0 || B * H >= (int64_t(1) << 31) || L >= (int64_t(1) << 30) || K > 8192) return KS_OK;
    if ((reinterpret_cast<uintptr_t>(out) & 15) != 0) return KS_OK;
    const int R = L <= 1024 ? 4 : 16;
    StencilGeom g;
    g.T = kThreads * R;
    g.HL = static_cast<int>((off + 31) / 32);
    g.HR = static_cast<int>((K - 1 - off + 31) / 32);
    // +1 row when it fits: the last register window may read past the halo (padded
    // taps only, never accumulated); without it those reads land in the tap area.
    g.NRB = std::min(256, g.T / 32 + g.HL + g.HR + 1);
    if (g.T / 32 + g.HL + g.HR > 256) return KS_OK;
    g.A = (32 * g.HL - static_cast<int>(off)) & ~3;
    g.Kp = static_cast<int>((K + 31) / 32 * 32);
    g.win_bytes = g.NRB * 128;
    g.stage_bytes = (g.win_bytes + g.Kp * 4 + 1023) / 1024 * 1024;
    CUtensorMap map;
    if (!encode_row_view(&map, in, B * H, L, g.NRB)) return KS_OK;
    const int s = static_cast<int>((4 - off % 4) % 4);
    int NS = static_cast<int>(std::max<int64_t>(2, std::min<int64_t>(4, (96 * 1024) / g.stage_bytes)));

    float* kp = nullptr;
    ks_status rc = cuda_status(cudaMallocAsync(&kp, sizeof(float) * H * g.Kp, st));
    if (rc != KS_OK) return rc;
    prep_taps<<<static_cast<unsigned>(std::min<int64_t>((H * g.Kp + 255) / 256, 4096)), 256, 0, st>>>(
        k, kp, H, K, g.Kp, reverse);
    rc = check_launch();
    if (rc == KS_OK) {
        const bool fused = mode == KS_MULADD_FUSED;
        if (R == 4)
            rc = fused ? dispatch_s<4, true>(s, map, kp, out, B, H, L, K, g, NS, st)
                       : dispatch_s<4, false>(s, map, kp, out, B, H, L, K, g, NS, st);
        else
            rc = fused ? dispatch_s<16, true>(s, map, kp, out, B, H, L, K, g, NS, st)
                       : dispatch_s<16, false>(s, map, kp, out, B, H, L, K, g, NS, st);
    }
    cudaFreeAsync(kp, st);
    *handled = true;
    return rc;
}

// ---------------------------------------------------------------------------
// dW, HIERARCHICAL

constexpr int kDwTT = 2048;  // t per work item
constexpr int kJR = 8;
constexpr int kTB = 8;

struct DwGeomT {
    int NRX;         // x window rows per stage
    int gy_bytes;    // kDwTT*4
    int stage_bytes;
};

template <int NJ, int S, bool FUSED>
__global__ void __launch_bounds__(kThreads)
dw_tma(const __grid_constant__ CUtensorMap gy_map, const __grid_constant__ CUtensorMap x_map,
       float* __restrict__ part, int B, int H, int L, int K, int p, int G, int NJT, DwGeomT g, int NS) {
    constexpr int NTS = kThreads / NJ;
    constexpr int JT = NJ * kJR;
    constexpr int SPT = kDwTT / (NTS * kTB);
    constexpr int NVX = (S + kTB + kJR - 1 + 3) / 4;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * g.stage_bytes);
    __shared__ float red[kThreads / 32][kJR];

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
    const int nunits = (b_end - b_begin) * ntt;
    // x window of work item t0 starts at row floor((t0+j0-p)/32); D = its float offset
    const int xoff = j0 - p;                      // t0 is a multiple of 32
    const int xr_rel = (xoff >= 0) ? xoff / 32 : -((-xoff + 31) / 32);
    const int D = xoff - 32 * xr_rel;             // in [0, 32)
    const int A = D & ~3;

    if (tid == 0) {
        prefetch_tmap(&gy_map);
        prefetch_tmap(&x_map);
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint32_t tx_bytes = static_cast<uint32_t>(g.gy_bytes) + static_cast<uint32_t>(g.NRX) * 128u;
    auto issue = [&](int stage, int u) {
        const int b = b_begin + u / ntt;
        const int t0 = (u % ntt) * kDwTT;
        const int row = b * H + h;
        unsigned char* sb = smem + stage * g.stage_bytes;
        mbar_arrive_expect_tx(&full[stage], tx_bytes);
        tma_load_3d(sb, &gy_map, 0, t0 / 32, row, &full[stage]);
        tma_load_3d(sb + g.gy_bytes, &x_map, 0, t0 / 32 + xr_rel, row, &full[stage]);
    };
    if (tid == 0)
        for (int s = 0; s < NS && s < nunits; ++s) issue(s, s);

    float acc[kJR];
#pragma unroll
    for (int i = 0; i < kJR; ++i) acc[i] = 0.f;

    for (int u = 0; u < nunits; ++u) {
        const int stage = u % NS;
        mbar_wait(&full[stage], static_cast<uint32_t>((u / NS) & 1));
        const char* gys = reinterpret_cast<const char*>(smem + stage * g.stage_bytes);
        const char* xs = gys + g.gy_bytes;
        const int t0 = (u % ntt) * kDwTT;
#pragma unroll 2
        for (int s = 0; s < SPT; ++s) {
            const int tl = (s * NTS + ts) * kTB;
            if (t0 + tl < L) {
                float gv[kTB];
#pragma unroll
                for (int c = 0; c < kTB / 4; ++c) {
                    const float4 q = lds128(gys, swz128(static_cast<uint32_t>(tl + 4 * c)));
                    gv[4 * c + 0] = q.x;
                    gv[4 * c + 1] = q.y;
                    gv[4 * c + 2] = q.z;
                    gv[4 * c + 3] = q.w;
                }
                float xv[4 * NVX];
                const uint32_t xi = static_cast<uint32_t>(A + tl + jg * kJR);
#pragma unroll
                for (int c = 0; c < NVX; ++c) {
                    const float4 q = lds128(xs, swz128(xi + 4 * c));
                    xv[4 * c + 0] = q.x;
                    xv[4 * c + 1] = q.y;
                    xv[4 * c + 2] = q.z;
                    xv[4 * c + 3] = q.w;
                }
#pragma unroll
                for (int tt = 0; tt < kTB; ++tt)
#pragma unroll
                    for (int jj = 0; jj < kJR; ++jj) acc[jj] = muladd<FUSED>(acc[jj], gv[tt], xv[S + tt + jj]);
            }
        }
        __syncthreads();
        if (tid == 0 && u + NS < nunits) issue(stage, u + NS);
    }

#pragma unroll
    for (int jj = 0; jj < kJR; ++jj) {
        float v = acc[jj];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc[jj] = v;
    }
    const int warp = tid >> 5, lane = tid & 31;
    if (lane == 0) {
#pragma unroll
        for (int jj = 0; jj < kJR; ++jj) red[warp][jj] = acc[jj];
    }
    __syncthreads();
    constexpr int WPG = NTS / 32;
    if (tid < JT) {
        const int gj = tid / kJR, jj = tid % kJR;
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < WPG; ++w) s += red[gj * WPG + w][jj];
        const int j = j0 + tid;
        if (j < K) part[(static_cast<int64_t>(grp) * H + h) * K + j] = s;
    }
}

template <int NJ, bool FUSED>
static ks_status launch_dw_tma_s(int s, const CUtensorMap& gm, const CUtensorMap& xm, float* part, int64_t B,
                                 int64_t H, int64_t L, int64_t K, int G, int NJT, const DwGeomT& g, int NS,
                                 cudaStream_t st) {
    const size_t smem = size_t(NS) * g.stage_bytes + 64 + 1024;
    const unsigned blocks = static_cast<unsigned>(int64_t(G) * H * NJT);
    const int p = static_cast<int>(K / 2);
#define KS_DW_CASE(SV)                                                                                        \
    case SV: {                                                                                                \
        auto kern = dw_tma<NJ, SV, FUSED>;                                                                    \
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));      \
        kern<<<blocks, kThreads, smem, st>>>(gm, xm, part, static_cast<int>(B), static_cast<int>(H),          \
                                             static_cast<int>(L), static_cast<int>(K), p, G, NJT, g, NS);     \
        break;                                                                                                \
    }
    switch (s) {
        KS_DW_CASE(0)
        KS_DW_CASE(1)
        KS_DW_CASE(2)
        default:
        KS_DW_CASE(3)
    }
#undef KS_DW_CASE
    return check_launch();
}

// Stage 1 of HIERARCHICAL dW through TMA; same work split (nj, njt, G) as the
// generic kernel so the partial buffer and stage 2 are shared.
ks_status dw_tma_stage1(const float* gy, const float* x, float* part, int64_t B, int64_t H, int64_t L, int64_t K,
                        int nj, int njt, int G, int mode, cudaStream_t st, bool* handled) {
    *handled = false;
    if (L % 32 != 0 || B * H >= (int64_t(1) << 31) || L >= (int64_t(1) << 30)) return KS_OK;
    const int JT = nj * kJR;
    DwGeomT g;
    g.gy_bytes = kDwTT * 4;
    g.NRX = (31 + kDwTT + JT + 8 + 31) / 32;
    g.stage_bytes = (g.gy_bytes + g.NRX * 128 + 1023) / 1024 * 1024;
    CUtensorMap gm, xm;
    if (!encode_row_view(&gm, gy, B * H, L, kDwTT / 32)) return KS_OK;
    if (!encode_row_view(&xm, x, B * H, L, g.NRX)) return KS_OK;
    const int NS = static_cast<int>(std::max(2, std::min(4, (72 * 1024) / g.stage_bytes)));
    const int p = static_cast<int>(K / 2);
    const int s = (4 - p % 4) % 4;
    const bool fused = mode == KS_MULADD_FUSED;
    *handled = true;
    switch (nj) {
        case 1: return fused ? launch_dw_tma_s<1, true>(s, gm, xm, part, B, H, L, K, G, njt, g, NS, st)
                             : launch_dw_tma_s<1, false>(s, gm, xm, part, B, H, L, K, G, njt, g, NS, st);
        case 2: return fused ? launch_dw_tma_s<2, true>(s, gm, xm, part, B, H, L, K, G, njt, g, NS, st)
                             : launch_dw_tma_s<2, false>(s, gm, xm, part, B, H, L, K, G, njt, g, NS, st);
        case 4: return fused ? launch_dw_tma_s<4, true>(s, gm, xm, part, B, H, L, K, G, njt, g, NS, st)
                             : launch_dw_tma_s<4, false>(s, gm, xm, part, B, H, L, K, G, njt, g, NS, st);
        default: return fused ? launch_dw_tma_s<8, true>(s, gm, xm, part, B, H, L, K, G, njt, g, NS, st)
                              : launch_dw_tma_s<8, false>(s, gm, xm, part, B, H, L, K, G, njt, g, NS, st);
    }
}

}  // namespace ks
