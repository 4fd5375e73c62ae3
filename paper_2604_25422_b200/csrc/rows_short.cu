// rows_short.cu -- forward / dX and dW for short rows (sm_100a), e.g. the
// paper's S4ConvD training shape (B,H,L,K) = (16384,128,48,48)
// (fixtures/table2.csv).
//
// The long-row kernels tile the sequence axis; with L = 48 a tile would be
// mostly empty.  Here one TMA box fetches a whole chunk of rows *with their
// halos*: the tensor map views the data as rows of L floats and the box is
// {BOX (>= L+K-1), rows} starting at column -off, so TMA zero-fills the columns
// outside [0, L) -- the reference's zero padding (src/conv_core.cpp:35-36) --
// and lays the rows out in shared memory at a pitch of BOX floats, chosen
// = 4 (mod 32) so lanes on consecutive rows read conflict-free.
//
// stencil_rows (fwd / dX, src/conv_core.cpp:21-75): persistent CTAs walk
//   chunks of NRC consecutive (b,h) rows through an NS-stage mbarrier ring
//   (one 2-D box per stage); every channel's taps are staged once per CTA.  A
//   thread keeps R = 16 consecutive outputs of its row in registers and slides
//   a register window over the taps in ascending j from +0 (bit-identical to
//   the reference); the block has NRC * ceil(L/16) threads (<= 256).
//
// dw_rows (dW, HIERARCHICAL order, src/conv_core.cpp:148-181): CTA =
//   (channel h, batch group, tap tile), 32*NJG*TP threads.  A 3-D view
//   {L, H, B} fetches 32 rows b*H+h of gy and the matching x windows (shifted
//   by the tap tile) per stage; thread (tap group, t phase, row lane)
//   accumulates 8 taps x 8 t FMAs per register block; then a fixed shuffle
//   tree over rows, a fixed pass over t phases, one partial per CTA, and the
//   shared fixed-order cross-block pass (dw_sum_groups).  No atomics.
#include <algorithm>

#include "ks_common.cuh"
#include "ks_tma.cuh"

namespace ks {

typedef CUresult (*EncodeTiledFnR)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

namespace {

constexpr int kJB = 8;
constexpr int kR = 16;

__host__ __device__ inline int round_up_i(int a, int b) { return (a + b - 1) / b * b; }
// smallest s >= n with s % 32 == 4 (128-bit loads by lanes s floats apart are conflict-free)
__host__ __device__ inline int stride4(int n) { return round_up_i(n - 4, 32) + 4; }

EncodeTiledFnR encode_fn_r() {
    static EncodeTiledFnR fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<EncodeTiledFnR>(p);
        return static_cast<EncodeTiledFnR>(nullptr);
    }();
    return fn;
}

// Rank-2 {L, rows} or rank-3 {L, H, B} fp32 view, unswizzled, zero OOB fill.
bool encode_rows(CUtensorMap* map, const float* base, int rank, const cuuint64_t* dims, const cuuint32_t* box) {
    EncodeTiledFnR fn = encode_fn_r();
    if (!fn || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
    cuuint64_t strides[2];
    strides[0] = dims[0] * 4;
    strides[1] = dims[0] * dims[1] * 4;
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

struct RowsGeom {
    int NRC;    // rows per chunk (box rows)
    int BOX;    // padded row pitch = box columns
    int KS;     // padded tap-row stride
    int segs;   // R-wide output segments per row
    int stage;  // floats per stage
    int NS;     // stages
};

template <int S, bool FUSED>
__global__ void __launch_bounds__(256)
stencil_rows(const __grid_constant__ CUtensorMap in_map, const float* __restrict__ k, float* __restrict__ out,
             int64_t nrows, int H, int L, int K, int off, int reverse, int nchunks, RowsGeom g) {
    constexpr int NV = (S + kR + kJB - 1 + 3) / 4;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* sm = reinterpret_cast<float*>(align_smem<128>(smem_raw));  // TMA boxes need 128-B alignment
    float* ring = sm;                      // [NS][NRC][BOX]
    float* tk = sm + g.NS * g.stage;       // [H][KS]
    uint64_t* full = reinterpret_cast<uint64_t*>(tk + H * g.KS);
    const int tid = threadIdx.x, nt = blockDim.x;

    if (tid == 0) {
        prefetch_tmap(&in_map);
        for (int s = 0; s < g.NS; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int stage, int c) {
        mbar_arrive_expect_tx(&full[stage], static_cast<uint32_t>(g.stage) * 4u);
        // innermost box coordinates must be 16-byte aligned: start S floats early
        tma_load_2d(ring + stage * g.stage, &in_map, -off - S, c * g.NRC, &full[stage]);
    };
    if (tid == 0)
        for (int s = 0; s < g.NS; ++s)
            if (static_cast<int>(blockIdx.x) + s * static_cast<int>(gridDim.x) < nchunks)
                issue(s, blockIdx.x + s * gridDim.x);
    // every channel's taps, once per CTA (reversed for dX)
    for (int q = tid; q < H * K; q += nt) {
        const int h = q / K, j = q - h * K;
        tk[h * g.KS + j] = k[static_cast<int64_t>(h) * K + (reverse ? K - 1 - j : j)];
    }
    __syncthreads();

    const int Kfull = K - K % kJB;
    int it = 0;
    for (int c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        const int stage = it % g.NS;
        mbar_wait(&full[stage], static_cast<uint32_t>((it / g.NS) & 1));
        const int64_t r0 = static_cast<int64_t>(c) * g.NRC;
        const int h0 = static_cast<int>(r0 % H);
        for (int q = tid; q < g.NRC * g.segs; q += nt) {
            const int i = q % g.NRC, seg = q / g.NRC;
            const int ts = seg * kR;
            if (r0 + i >= nrows) continue;
            // box column S + t + j  <->  x[t + j - off]
            const float* xr = ring + stage * g.stage + i * g.BOX + ts;
            const float* kr = tk + ((h0 + i) % H) * g.KS;
            float acc[kR];
#pragma unroll
            for (int r = 0; r < kR; ++r) acc[r] = 0.f;
            auto block = [&](int j0, int nj) {
                float v[4 * NV];
#pragma unroll
                for (int u = 0; u < NV; ++u) {
                    const float4 a = lds4(xr + j0 + 4 * u);
                    v[4 * u + 0] = a.x;
                    v[4 * u + 1] = a.y;
                    v[4 * u + 2] = a.z;
                    v[4 * u + 3] = a.w;
                }
                float w[kJB];
#pragma unroll
                for (int u = 0; u < kJB / 4; ++u) {
                    const float4 a = *reinterpret_cast<const float4*>(kr + j0 + 4 * u);
                    w[4 * u + 0] = a.x;
                    w[4 * u + 1] = a.y;
                    w[4 * u + 2] = a.z;
                    w[4 * u + 3] = a.w;
                }
#pragma unroll
                for (int jj = 0; jj < kJB; ++jj)
                    if (jj < nj) {
#pragma unroll
                        for (int r = 0; r < kR; ++r) acc[r] = muladd<FUSED>(acc[r], v[S + r + jj], w[jj]);
                    }
            };
            for (int j0 = 0; j0 < Kfull; j0 += kJB) block(j0, kJB);
            if (Kfull < K) block(Kfull, K - Kfull);
            float* o = out + (r0 + i) * L + ts;
            if (ts + kR <= L) {
#pragma unroll
                for (int r = 0; r < kR; r += 4) st_cs_v4(o + r, make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]));
            } else {
#pragma unroll
                for (int r = 0; r < kR; ++r)
                    if (ts + r < L) o[r] = acc[r];
            }
        }
        __syncthreads();  // stage consumed
        const int nc = c + g.NS * static_cast<int>(gridDim.x);
        if (tid == 0 && nc < nchunks) issue(stage, nc);
    }
}

// dW over short rows: block = NJG tap groups x TP t phases x 32 row lanes.
template <int S, bool FUSED>
__global__ void __launch_bounds__(256)
dw_rows(const __grid_constant__ CUtensorMap gy_map, const __grid_constant__ CUtensorMap x_map,
        float* __restrict__ part, int B, int H, int L, int K, int G, int NJT, int NJG, int TP, int BOXG, int BOXX) {
    constexpr int NVX = (S + 8 + kJB - 1 + 3) / 4;
    constexpr int NR = 32;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* sm = reinterpret_cast<float*>(align_smem<128>(smem_raw));
    const int stage_f = NR * (BOXG + BOXX);
    float* ring = sm;  // [2][ gy 32 x BOXG | x 32 x BOXX ]
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + 2 * stage_f);
    __shared__ float red[8][kJB];

    int bid = blockIdx.x;
    const int jt = bid % NJT;
    bid /= NJT;
    const int h = bid % H;
    const int grp = bid / H;
    const int b_begin = static_cast<int>(static_cast<int64_t>(B) * grp / G);
    const int b_end = static_cast<int>(static_cast<int64_t>(B) * (grp + 1) / G);
    const int JT = NJG * kJB;
    const int j0 = jt * JT;
    const int p = K / 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int jg = warp / TP, tp = warp % TP;
    const int nblk = (L + 7) / 8;
    const int nchunk = (b_end - b_begin + NR - 1) / NR;

    if (tid == 0) {
        prefetch_tmap(&gy_map);
        prefetch_tmap(&x_map);
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    // box column c of the x box <-> x[c + j0 - p - S] (16-byte aligned start);
    // rows past b_end are never read
    auto issue = [&](int stage, int c) {
        float* sb = ring + stage * stage_f;
        mbar_arrive_expect_tx(&full[stage], static_cast<uint32_t>(stage_f) * 4u);
        tma_load_3d(sb, &gy_map, 0, h, b_begin + c * NR, &full[stage]);
        tma_load_3d(sb + NR * BOXG, &x_map, j0 - p - S, h, b_begin + c * NR, &full[stage]);
    };
    if (tid == 0) {
        if (nchunk > 0) issue(0, 0);
        if (nchunk > 1) issue(1, 1);
    }

    float acc[kJB];
#pragma unroll
    for (int q = 0; q < kJB; ++q) acc[q] = 0.f;
    for (int c = 0; c < nchunk; ++c) {
        const int stage = c & 1;
        mbar_wait(&full[stage], static_cast<uint32_t>((c >> 1) & 1));
        const int nr = min(NR, b_end - (b_begin + c * NR));
        if (lane < nr) {
            const float* gr = ring + stage * stage_f + lane * BOXG;
            const float* xr = ring + stage * stage_f + NR * BOXG + lane * BOXX + jg * kJB;
            for (int blk = tp; blk < nblk; blk += TP) {
                const int t = blk * 8;
                float gv[8];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const float4 a = lds4(gr + t + 4 * q);
                    gv[4 * q + 0] = a.x;
                    gv[4 * q + 1] = a.y;
                    gv[4 * q + 2] = a.z;
                    gv[4 * q + 3] = a.w;
                }
                float xv[4 * NVX];
#pragma unroll
                for (int q = 0; q < NVX; ++q) {
                    const float4 a = lds4(xr + t + 4 * q);
                    xv[4 * q + 0] = a.x;
                    xv[4 * q + 1] = a.y;
                    xv[4 * q + 2] = a.z;
                    xv[4 * q + 3] = a.w;
                }
#pragma unroll
                for (int tt = 0; tt < 8; ++tt)
#pragma unroll
                    for (int jj = 0; jj < kJB; ++jj) acc[jj] = muladd<true>(acc[jj], gv[tt], xv[S + tt + jj]);
            }
        }
        __syncthreads();  // stage consumed
        if (tid == 0 && c + 2 < nchunk) issue(stage, c + 2);
    }
    // fixed-order reduction: rows (lanes) by a shuffle tree, then t phases
#pragma unroll
    for (int jj = 0; jj < kJB; ++jj) {
        float v = acc[jj];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc[jj] = v;
    }
    if (lane == 0) {
#pragma unroll
        for (int jj = 0; jj < kJB; ++jj) red[warp][jj] = acc[jj];
    }
    __syncthreads();
    if (tid < JT) {
        const int gj = tid / kJB, jj = tid % kJB;
        float s = 0.f;
        for (int w = 0; w < TP; ++w) s += red[gj * TP + w][jj];
        const int j = j0 + tid;
        if (j < K) part[(static_cast<int64_t>(grp) * H + h) * K + j] = s;
    }
}

}  // namespace

// fwd / dX for short rows; *handled = false outside the envelope.
ks_status stencil_rows_f32(const float* in, const float* k, float* out, int64_t B, int64_t H, int64_t L, int64_t K,
                           int64_t off, int reverse, int mode, cudaStream_t st, bool* handled) {
    *handled = false;
    if (L % 4 != 0 || B * H >= (int64_t(1) << 31)) return KS_OK;
    if ((reinterpret_cast<uintptr_t>(in) & 15) || (reinterpret_cast<uintptr_t>(out) & 15)) return KS_OK;
    RowsGeom g;
    // box columns cover every tap of every output; register windows may read a
    // few floats past a row, which land in the next row / the tap area and only
    // feed predicated-off taps
    const int sh = static_cast<int>((4 - off % 4) % 4);
    g.BOX = stride4(static_cast<int>(L + K) - 1 + sh);
    if (g.BOX > 256) return KS_OK;
    g.KS = stride4(round_up_i(static_cast<int>(K), kJB) + 4);
    g.segs = static_cast<int>((L + kR - 1) / kR);
    g.NRC = std::max(32, (256 / g.segs) / 32 * 32);
    g.NRC = std::min(g.NRC, 256);
    g.stage = g.NRC * g.BOX;
    const int64_t tap_floats = H * g.KS;
    g.NS = 3;
    auto smem_of = [&](int ns) { return (int64_t(ns) * g.stage + tap_floats) * 4 + 64 + 128; };
    while (g.NS > 2 && smem_of(g.NS) > 110 * 1024) --g.NS;
    const int64_t smem = smem_of(g.NS);
    if (smem > 200 * 1024) return KS_OK;
    const int64_t nrows = B * H;
    const int64_t nchunks = (nrows + g.NRC - 1) / g.NRC;
    CUtensorMap im;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(L), static_cast<cuuint64_t>(nrows)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(g.BOX), static_cast<cuuint32_t>(g.NRC)};
    if (!encode_rows(&im, in, 2, dims, box)) return KS_OK;
    const int threads = std::min(256, g.NRC * g.segs);
    const bool fused = mode == KS_MULADD_FUSED;
    auto kern = fused ? stencil_rows<0, true> : stencil_rows<0, false>;
    switch (sh) {
        case 1: kern = fused ? stencil_rows<1, true> : stencil_rows<1, false>; break;
        case 2: kern = fused ? stencil_rows<2, true> : stencil_rows<2, false>; break;
        case 3: kern = fused ? stencil_rows<3, true> : stencil_rows<3, false>; break;
        default: break;
    }
    const int per_sm = prepare_kernel(reinterpret_cast<const void*>(kern), threads, static_cast<int>(smem));
    const int64_t grid = std::min<int64_t>(nchunks, int64_t(num_sms()) * per_sm);
    *handled = true;
    launch_kernel(kern, static_cast<unsigned>(grid), threads, smem, st, im, k, out, nrows, static_cast<int>(H),
                                                             static_cast<int>(L), static_cast<int>(K),
                                                             static_cast<int>(off), reverse,
                                                             static_cast<int>(nchunks), g);
    return check_launch();
}

// dW stage 1 for short rows into part[G,H,K] (G = the caller's row groups).
ks_status dw_rows_stage1(const float* gy, const float* x, float* part, int64_t B, int64_t H, int64_t L, int64_t K,
                         int G, int mode, cudaStream_t st, bool* handled) {
    *handled = false;
    if (L % 4 != 0 || B * H >= (int64_t(1) << 31)) return KS_OK;
    const int ngroups8 = static_cast<int>((K + kJB - 1) / kJB);
    const int NJG = std::min(8, ngroups8);  // tap groups per CTA
    const int TP = std::max(1, 8 / NJG);    // t phases
    const int njt = (ngroups8 + NJG - 1) / NJG;
    const int JT = NJG * kJB;
    // gy reads reach t + 7 <= L + 3; x reads reach t + jg*8 + 4*NVX - 1 <= L + JT + 8
    const int BOXG = stride4(static_cast<int>(L) + 4);
    const int BOXX = stride4(static_cast<int>(L) + JT + 16);
    if (BOXG > 256 || BOXX > 256) return KS_OK;
    const int smem = 2 * 32 * (BOXG + BOXX) * 4 + 64 + 128;
    if (smem > 200 * 1024) return KS_OK;
    if (int64_t(G) * H * njt >= (int64_t(1) << 31)) return KS_OK;
    CUtensorMap gm, xm;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(L), static_cast<cuuint64_t>(H), static_cast<cuuint64_t>(B)};
    const cuuint32_t boxg[3] = {static_cast<cuuint32_t>(BOXG), 1, 32};
    const cuuint32_t boxx[3] = {static_cast<cuuint32_t>(BOXX), 1, 32};
    if (!encode_rows(&gm, gy, 3, dims, boxg) || !encode_rows(&xm, x, 3, dims, boxx)) return KS_OK;
    (void)mode;  // HIERARCHICAL accumulates with FMA in either MulAddMode (conv_dw.cu)
    const unsigned blocks = static_cast<unsigned>(int64_t(G) * H * njt);
    const int threads = 32 * NJG * TP;
    const int p4 = static_cast<int>((4 - (K / 2) % 4) % 4);  // (j0 - p) mod 4 with j0 % 8 == 0
    auto kern = dw_rows<0, true>;
    switch (p4) {
        case 1: kern = dw_rows<1, true>; break;
        case 2: kern = dw_rows<2, true>; break;
        case 3: kern = dw_rows<3, true>; break;
        default: break;
    }
    prepare_kernel(reinterpret_cast<const void*>(kern), threads, smem);
    *handled = true;
    launch_kernel(kern, blocks, threads, smem, st, gm, xm, part, static_cast<int>(B), static_cast<int>(H), static_cast<int>(L),
                                        static_cast<int>(K), G, njt, NJG, TP, BOXG, BOXX);
    return check_launch();
}

}  // namespace ks
