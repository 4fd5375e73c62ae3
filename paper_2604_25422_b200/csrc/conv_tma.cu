// conv_tma.cu -- TMA-pipelined sm_100a kernels for rows with L % 16 == 0.
//
// Stencil (forward y / input-gradient dX, reference src/conv_core.cpp:21-75):
//   persistent CTAs walk (row, T-output tile) work items.  Thread 0 keeps NS-1
//   tiles in flight: per stage a cp.async.bulk.tensor load of the input window
//   (TMA zero-fills the halo outside the row) and a 1-D bulk copy of the
//   channel's taps, all completing on the stage's mbarrier.  Each thread keeps
//   R consecutive outputs in registers and slides a register window over the
//   taps in ascending j (bit-identical to the reference), reading the swizzled
//   window with conflict-free 128-bit shared loads.  Outputs go registers ->
//   swizzled shared buffer -> one TMA tensor store per tile (double-buffered,
//   bulk-group tracked), so global writes are full-line and asynchronous.
//
// dW (reference src/conv_core.cpp:148-181), HIERARCHICAL order:
//   CTA = (row group, channel h, 8*NJ-tap tile).  Work items are
//   (row b, 2048-wide t tile); each stage holds the gy tile and the x window
//   [t0+j0-p-D, ...) loaded by TMA.  Thread (tap group, t-slice) accumulates
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
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<EncodeTiledFn>(p);
        return static_cast<EncodeTiledFn>(nullptr);
    }();
    return fn;
}

bool encode_row_view(CUtensorMap* map, const float* base, int64_t rows, int64_t L, int inner, int box_rows,
                     int sw) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || L % inner != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
    if (rows >= (int64_t(1) << 31) || L / inner >= (int64_t(1) << 31) || box_rows < 1 || box_rows > 256)
        return false;
    if (sw && inner * 4 > sw) return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(L / inner),
                                static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(inner) * 4, static_cast<cuuint64_t>(L) * 4};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(inner), static_cast<cuuint32_t>(box_rows), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUtensorMapSwizzle swz = sw == 32    ? CU_TENSOR_MAP_SWIZZLE_32B
                                   : sw == 64  ? CU_TENSOR_MAP_SWIZZLE_64B
                                   : sw == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                               : CU_TENSOR_MAP_SWIZZLE_NONE;
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
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
constexpr int kIn = 32;  // floats per TMA row piece (128 B)

struct StencilGeom {
    int T;            // outputs per tile (256*R)
    int HH;           // halo rows (32 floats) on each side
    int MR;           // main rows = T/32
    int NB;           // rows per input box (window = nbox*NB rows)
    int nbox;         // 1 or 2 input boxes per stage
    int A;            // (32*HH - off) & ~3
    int Kp;           // taps padded to a multiple of 32
    int win_bytes;    // nbox*NB*128
    int stage_bytes;  // window + taps, 1024-aligned
    int out_bytes;    // T*4, 1024-aligned
};

// First output of thread `tid`'s R-output register tile.  For R = 16 the 256
// chunks of a tile are dealt so that the lanes of a warp own every other
// chunk: their 128-bit window / output accesses are 128 B apart, which the
// SWIZZLE_128B layout serves without bank conflicts for any window offset.
template <int R>
__device__ __forceinline__ int tile_base(int tid) {
    if constexpr (R == 16) {
        const int lane = tid & 31, w = tid >> 5;
        return (lane * 2 + (w & 1) + (w >> 1) * 64) * R;
    } else {
        return tid * R;  // R = 4: lanes 16 B apart, contiguous, unswizzled
    }
}

template <int R, int S, bool FUSED>
__global__ void __launch_bounds__(kThreads)
stencil_tma(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap out_map,
            const float* __restrict__ kp, int H, int L, int K, int tiles_per_row, int ntiles, StencilGeom g,
            int NS) {
    constexpr int SW = R == 16 ? 128 : 0;  // lanes read 128 B (R=16) / 16 B (R=4) apart
    constexpr int NV = (S + R + kJB - 1 + 3) / 4;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = align_smem<1024>(smem_raw);
    unsigned char* outb = smem + NS * g.stage_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(outb + 2 * g.out_bytes);
    const int tid = threadIdx.x;

    if (tid == 0) {
        prefetch_tmap(&in_map);
        prefetch_tmap(&out_map);
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint32_t tx_bytes = static_cast<uint32_t>(g.win_bytes + g.Kp * 4);
    auto issue = [&](int stage, int tile) {
        const int row = tile / tiles_per_row;
        const int t0 = (tile - row * tiles_per_row) * g.T;
        unsigned char* sb = smem + stage * g.stage_bytes;
        mbar_arrive_expect_tx(&full[stage], tx_bytes);
        const int r0 = t0 / kIn - g.HH;
        tma_load_3d(sb, &in_map, 0, r0, row, &full[stage]);
        if (g.nbox > 1) tma_load_3d(sb + g.NB * 128, &in_map, 0, r0 + g.NB, row, &full[stage]);
        bulk_load(sb + g.win_bytes, kp + static_cast<int64_t>(row % H) * g.Kp, static_cast<uint32_t>(g.Kp) * 4u,
                  &full[stage]);
    };

    if (tid == 0)
        for (int s = 0; s < NS; ++s) {
            const int t = blockIdx.x + s * gridDim.x;
            if (t < ntiles) issue(s, t);
        }

    const int base = tile_base<R>(tid);
    const int Kfull = K - K % kJB;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int stage = it % NS;
        mbar_wait(&full[stage], static_cast<uint32_t>((it / NS) & 1));
        const unsigned char* win = smem + stage * g.stage_bytes;
        const float* wk = reinterpret_cast<const float*>(win + g.win_bytes);
        const int row = tile / tiles_per_row;
        const int t0 = (tile - row * tiles_per_row) * g.T;

        float acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0.f;
        if (t0 + base < L) {
            auto block = [&](int j0, int nj) {
                float v[4 * NV];
                const uint32_t i0 = static_cast<uint32_t>(base + g.A + j0);
#pragma unroll
                for (int c = 0; c < NV; ++c) {
                    const float4 q = *reinterpret_cast<const float4*>(win + swz<SW>(i0 + 4 * c));
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
        }
        // registers -> swizzled output buffer (its previous TMA store finished
        // reading before the last barrier, see below)
        unsigned char* ob = outb + (it & 1) * g.out_bytes;
#pragma unroll
        for (int r = 0; r < R; r += 4)
            *reinterpret_cast<float4*>(ob + swz<SW>(static_cast<uint32_t>(base + r))) =
                make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]);
        fence_proxy_async_smem();
        if (tid == 0) bulk_wait_read_all();  // store it-1 done reading: buffer (it+1)&1 is free next tile
        __syncthreads();                     // window of `stage` consumed, outputs of this tile written
        if (tid == 0) {
            tma_store_3d(&out_map, ob, 0, t0 / kIn, row);  // OOB columns past L are clipped
            bulk_commit();
            const int nt = tile + NS * gridDim.x;
            if (nt < ntiles) issue(stage, nt);
        }
    }
    if (tid == 0) bulk_wait_all();
}

static int stencil_smem_bytes(const StencilGeom& g, int NS) { return NS * g.stage_bytes + 2 * g.out_bytes + 64 + 1024; }

template <int R, int S, bool FUSED>
static ks_status launch_stencil_tma(const CUtensorMap& im, const CUtensorMap& om, const float* kp, int64_t B,
                                    int64_t H, int64_t L, int64_t K, const StencilGeom& g, int NS, cudaStream_t st) {
    auto kern = stencil_tma<R, S, FUSED>;
    const int smem = stencil_smem_bytes(g, NS);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
    if (per_sm < 1) per_sm = 1;
    const int tiles_per_row = static_cast<int>((L + g.T - 1) / g.T);
    const int ntiles = static_cast<int>(B * H * tiles_per_row);
    const int grid = std::min(ntiles, num_sms() * per_sm);
    kern<<<grid, kThreads, smem, st>>>(im, om, kp, static_cast<int>(H), static_cast<int>(L), static_cast<int>(K),
                                       tiles_per_row, ntiles, g, NS);
    return check_launch();
}

template <int R, bool FUSED>
static ks_status dispatch_s(int s, const CUtensorMap& im, const CUtensorMap& om, const float* kp, int64_t B,
                            int64_t H, int64_t L, int64_t K, const StencilGeom& g, int NS, cudaStream_t st) {
    switch (s) {
        case 0: return launch_stencil_tma<R, 0, FUSED>(im, om, kp, B, H, L, K, g, NS, st);
        case 1: return launch_stencil_tma<R, 1, FUSED>(im, om, kp, B, H, L, K, g, NS, st);
        case 2: return launch_stencil_tma<R, 2, FUSED>(im, om, kp, B, H, L, K, g, NS, st);
        default: return launch_stencil_tma<R, 3, FUSED>(im, om, kp, B, H, L, K, g, NS, st);
    }
}

// Sets *handled = false (and does nothing) when this path does not apply; the
// caller then uses the generic kernels of conv_fwd.cu.
ks_status stencil_tma_f32(const float* in, const float* k, float* out, int64_t B, int64_t H, int64_t L, int64_t K,
                          int64_t off, int reverse, int mode, cudaStream_t st, bool* handled) {
    *handled = false;
    if (L % kIn != 0 || L >= (int64_t(1) << 30) || K > 8192) return KS_OK;
    const int R = L <= 1024 ? 4 : 16;
    StencilGeom g;
    g.T = kThreads * R;
    g.MR = g.T / kIn;
    const int64_t need = std::max<int64_t>(off, K - 1 - off);
    g.HH = static_cast<int>((need + kIn - 1) / kIn);
    if (g.HH == 0) g.HH = 1;  // the last register window may read one row past the tile
    const int W = g.MR + 2 * g.HH;  // even (MR is even)
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
    g.A = (kIn * g.HH - static_cast<int>(off)) & ~3;
    g.Kp = static_cast<int>((K + 31) / 32 * 32);
    g.win_bytes = g.nbox * g.NB * 128;
    g.stage_bytes = (g.win_bytes + g.Kp * 4 + 1023) / 1024 * 1024;
    g.out_bytes = (g.T * 4 + 1023) / 1024 * 1024;
    const int sw = R == 16 ? 128 : 0;
    CUtensorMap im, om;
    if (!encode_row_view(&im, in, B * H, L, kIn, g.NB, sw)) return KS_OK;
    if (!encode_row_view(&om, out, B * H, L, kIn, g.MR, sw)) return KS_OK;
    const int s = static_cast<int>((4 - off % 4) % 4);
    int NS = 4;
    while (NS > 2 && stencil_smem_bytes(g, NS) > 110 * 1024) --NS;
    if (stencil_smem_bytes(g, NS) > 220 * 1024) return KS_OK;

    float* kp = nullptr;
    ks_status rc = cuda_status(cudaMallocAsync(&kp, sizeof(float) * H * g.Kp, st));
    if (rc != KS_OK) return rc;
    prep_taps<<<static_cast<unsigned>(std::min<int64_t>((H * g.Kp + 255) / 256, 4096)), 256, 0, st>>>(
        k, kp, H, K, g.Kp, reverse);
    rc = check_launch();
    if (rc == KS_OK) {
        const bool fused = mode == KS_MULADD_FUSED;
        if (R == 4)
            rc = fused ? dispatch_s<4, true>(s, im, om, kp, B, H, L, K, g, NS, st)
                       : dispatch_s<4, false>(s, im, om, kp, B, H, L, K, g, NS, st);
        else
            rc = fused ? dispatch_s<16, true>(s, im, om, kp, B, H, L, K, g, NS, st)
                       : dispatch_s<16, false>(s, im, om, kp, B, H, L, K, g, NS, st);
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
constexpr int kDwIn = 32;    // floats per TMA row piece (128 B, SWIZZLE_128B)
constexpr int kDwMain = kDwTT / kDwIn;  // x window main-box rows

struct DwGeomT {
    int XR;           // x window rows (32 floats): kDwMain main + XT tail
    int XT;           // tail rows
    int gy_bytes;     // kDwTT*4
    int stage_bytes;
};

template <int NJ, int S, bool FUSED>
__global__ void __launch_bounds__(kThreads)
dw_tma(const __grid_constant__ CUtensorMap gy_map, const __grid_constant__ CUtensorMap x_map,
       const __grid_constant__ CUtensorMap x_tail_map, float* __restrict__ part, int B, int H, int L, int K, int p,
       int G, int NJT, DwGeomT g, int NS) {
    constexpr int NTS = kThreads / NJ;
    constexpr int JT = NJ * kJR;
    constexpr int SPT = kDwTT / (NTS * kTB);
    constexpr int NVX = (S + kTB + kJR - 1 + 3) / 4;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = align_smem<1024>(smem_raw);
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
    // the x window of a work item at t0 starts at position t0 + j0 - p - D
    const int xoff = j0 - p;
    const int D = ((xoff % kDwIn) + kDwIn) % kDwIn;
    const int xr_rel = (xoff - D) / kDwIn;  // exact division
    const int A = D & ~3;

    if (tid == 0) {
        prefetch_tmap(&gy_map);
        prefetch_tmap(&x_map);
        prefetch_tmap(&x_tail_map);
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint32_t tx_bytes = static_cast<uint32_t>(g.gy_bytes + g.XR * kDwIn * 4);
    auto issue = [&](int stage, int u) {
        const int b = b_begin + u / ntt;
        const int t0 = (u % ntt) * kDwTT;
        const int row = b * H + h;
        unsigned char* sb = smem + stage * g.stage_bytes;
        mbar_arrive_expect_tx(&full[stage], tx_bytes);
        tma_load_3d(sb, &gy_map, 0, t0 / kDwIn, row, &full[stage]);
        const int xr = t0 / kDwIn + xr_rel;
        tma_load_3d(sb + g.gy_bytes, &x_map, 0, xr, row, &full[stage]);
        tma_load_3d(sb + g.gy_bytes + kDwMain * kDwIn * 4, &x_tail_map, 0, xr + kDwMain, row, &full[stage]);
    };
    if (tid == 0)
        for (int s = 0; s < NS && s < nunits; ++s) issue(s, s);

    float acc[kJR];
#pragma unroll
    for (int i = 0; i < kJR; ++i) acc[i] = 0.f;

    for (int u = 0; u < nunits; ++u) {
        const int stage = u % NS;
        mbar_wait(&full[stage], static_cast<uint32_t>((u / NS) & 1));
        const unsigned char* gys = smem + stage * g.stage_bytes;
        const unsigned char* xs = gys + g.gy_bytes;
        const int t0 = (u % ntt) * kDwTT;
#pragma unroll 2
        for (int s = 0; s < SPT; ++s) {
            // 8-wide t block of this (s, t-slice): consecutive lanes take blocks
            // 4 apart (128 B), conflict-free under SWIZZLE_128B
            const int q = s * NTS + ts;
            const int tl = ((q & 31) * 4 + ((q >> 5) & 3) + (q >> 7) * 128) * kTB;
            if (t0 + tl < L) {
                float gv[kTB];
#pragma unroll
                for (int c = 0; c < kTB / 4; ++c) {
                    const float4 q =
                        *reinterpret_cast<const float4*>(gys + swz<128>(static_cast<uint32_t>(tl + 4 * c)));
                    gv[4 * c + 0] = q.x;
                    gv[4 * c + 1] = q.y;
                    gv[4 * c + 2] = q.z;
                    gv[4 * c + 3] = q.w;
                }
                float xv[4 * NVX];
                const uint32_t xi = static_cast<uint32_t>(A + tl + jg * kJR);
#pragma unroll
                for (int c = 0; c < NVX; ++c) {
                    const float4 q = *reinterpret_cast<const float4*>(xs + swz<128>(xi + 4 * c));
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
static ks_status launch_dw_tma_s(int s, const CUtensorMap& gm, const CUtensorMap& xm, const CUtensorMap& xt,
                                 float* part, int64_t B, int64_t H, int64_t L, int64_t K, int G, int NJT,
                                 const DwGeomT& g, int NS, cudaStream_t st) {
    const int smem = NS * g.stage_bytes + 64 + 1024;
    const unsigned blocks = static_cast<unsigned>(int64_t(G) * H * NJT);
    const int p = static_cast<int>(K / 2);
#define KS_DW_CASE(SV)                                                                                         \
    case SV: {                                                                                                 \
        auto kern = dw_tma<NJ, SV, FUSED>;                                                                     \
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);                         \
        kern<<<blocks, kThreads, smem, st>>>(gm, xm, xt, part, static_cast<int>(B), static_cast<int>(H),       \
                                             static_cast<int>(L), static_cast<int>(K), p, G, NJT, g, NS);      \
        break;                                                                                                 \
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
    if (L % kDwIn != 0 || B * H >= (int64_t(1) << 31) || L >= (int64_t(1) << 30) || K >= (int64_t(1) << 30))
        return KS_OK;
    DwGeomT g;
    g.gy_bytes = kDwTT * 4;
    g.XT = (nj * kJR + 40 + kDwIn - 1) / kDwIn;  // covers D + JT + register-window overrun

    g.XR = kDwMain + g.XT;
    g.stage_bytes = (g.gy_bytes + g.XR * kDwIn * 4 + 1023) / 1024 * 1024;
    CUtensorMap gm, xm, xt;
    if (!encode_row_view(&gm, gy, B * H, L, kDwIn, kDwTT / kDwIn, 128)) return KS_OK;
    if (!encode_row_view(&xm, x, B * H, L, kDwIn, kDwMain, 128)) return KS_OK;
    if (!encode_row_view(&xt, x, B * H, L, kDwIn, g.XT, 128)) return KS_OK;
    const int NS = std::max(2, std::min(4, (72 * 1024) / g.stage_bytes));
    const int p = static_cast<int>(K / 2);
    const int s = (4 - p % 4) % 4;
    const bool fused = mode == KS_MULADD_FUSED;
    *handled = true;
    switch (nj) {
        case 1: return fused ? launch_dw_tma_s<1, true>(s, gm, xm, xt, part, B, H, L, K, G, njt, g, NS, st)
                             : launch_dw_tma_s<1, false>(s, gm, xm, xt, part, B, H, L, K, G, njt, g, NS, st);
        case 2: return fused ? launch_dw_tma_s<2, true>(s, gm, xm, xt, part, B, H, L, K, G, njt, g, NS, st)
                             : launch_dw_tma_s<2, false>(s, gm, xm, xt, part, B, H, L, K, G, njt, g, NS, st);
        case 4: return fused ? launch_dw_tma_s<4, true>(s, gm, xm, xt, part, B, H, L, K, G, njt, g, NS, st)
                             : launch_dw_tma_s<4, false>(s, gm, xm, xt, part, B, H, L, K, G, njt, g, NS, st);
        default: return fused ? launch_dw_tma_s<8, true>(s, gm, xm, xt, part, B, H, L, K, G, njt, g, NS, st)
                              : launch_dw_tma_s<8, false>(s, gm, xm, xt, part, B, H, L, K, G, njt, g, NS, st);
    }
}

}  // namespace ks
