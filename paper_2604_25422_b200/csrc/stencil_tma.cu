// stencil_tma.cu -- TMA-pipelined forward y / input-gradient dX (sm_100a),
// rows with L % 32 == 0.
//
//   out[b,h,t] = sum_{j=0}^{K-1} in[b,h,t+j-off] * w[h,j]
//   forward: in = x, w = k[h], off = p = K/2      (reference src/conv_core.cpp:21-46)
//   dX:      in = gy, w = reversed k[h], off = q  (reference src/conv_core.cpp:48-75)
//
// Persistent CTAs of NT threads walk (row, T = NT*R output) tiles.  Thread 0
// keeps NS-1 tiles in flight: per stage a cp.async.bulk.tensor load of the
// window [t0 - 32*HH, t0 + T + 32*HH) (TMA zero-fills what lies outside the
// row = the reference's zero padding) and a 1-D bulk copy of the channel's
// taps, both completing on the stage's mbarrier.  Each thread keeps R
// consecutive outputs in registers and slides a register window over the taps
// in blocks of 8, ascending in j from +0 -- bit-identical to the reference in
// both MulAddModes.  Window reads are 128-bit and bank-conflict-free: lanes
// read 128 B apart under SWIZZLE_128B (R = 16 deals chunks so, R = 32 is so
// naturally) or 16 B apart unswizzled (R = 4).
//
// Two output paths: memory-bound shapes (short K) stage outputs in a swizzled
// shared buffer and write each tile with one TMA tensor store (double
// buffered), compute-bound shapes (long K, R = 32) store 128-bit streaming
// writes straight from registers and spend the shared memory on occupancy.
#include <algorithm>
#include <cstdlib>

#include "ks_common.cuh"
#include "ks_tma.cuh"

namespace ks {

__global__ void prep_taps(const float*, float*, int64_t, int64_t, int64_t, int, int);
ks_status stencil_pad_f32(const float* in, const float* k, float* out, int64_t B, int64_t H, int64_t L, int64_t K,
                          int64_t off, int reverse, int mode, cudaStream_t st, bool* handled);

namespace {

constexpr int kJB = 8;   // taps per register block
constexpr int kIn = 32;  // floats per TMA row piece (128 B)

struct StencilGeom {
    int T;            // outputs per tile (NT*R)
    int HH;           // halo rows (32 floats) on each side
    int MR;           // main rows = T/32
    int NB;           // rows per input box (window = nbox*NB rows)
    int nbox;         // 1 or 2 input boxes per stage
    int A;            // (32*HH - off) & ~3: logical window index of output 0's first tap, 4-aligned
    int Kp;           // taps padded to a multiple of 32
    int win_bytes;    // nbox*NB*128
    int stage_bytes;  // window + taps, 1024-aligned
    int out_bytes;    // T*4, 1024-aligned (TMA_OUT only)
};

// First output of a thread's R-output register tile within the tile.
template <int R>
__device__ __forceinline__ int tile_base(int tid) {
    if constexpr (R == 16) {
        // lanes own every other 16-output chunk -> 128 B apart
        const int lane = tid & 31, w = tid >> 5;
        return (lane * 2 + (w & 1) + (w >> 1) * 64) * R;
    } else {
        return tid * R;  // R = 32: 128 B apart; R = 4: 16 B apart, contiguous
    }
}

template <int R, int NT, int S, bool FUSED, bool TMA_OUT>
__global__ void __launch_bounds__(NT)
stencil_tma(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap out_map,
            const float* __restrict__ kp, float* __restrict__ out, int H, int L, int K, int tiles_per_row,
            int ntiles, StencilGeom g, int NS) {
    pdl_wait();  // launched with PDL after prep_taps: kp must be complete
    constexpr int SW = R == 4 ? 0 : 128;
    constexpr int NV = (S + R + kJB - 1 + 3) / 4;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = align_smem<1024>(smem_raw);
    unsigned char* outb = smem + NS * g.stage_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(outb + (TMA_OUT ? 2 * g.out_bytes : 0));
    const int tid = threadIdx.x;

    if (tid == 0) {
        prefetch_tmap(&in_map);
        if (TMA_OUT) prefetch_tmap(&out_map);
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
        const bool live = t0 + base < L;  // L % 32 == 0: a register tile is wholly in or out

        float acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0.f;
        if (live) {
            auto block = [&](int j0, int nj) {
                float v[4 * NV];
                const uint32_t i0 = static_cast<uint32_t>(base + g.A + j0);
#pragma unroll
                for (int c = 0; c < NV; ++c) {
                    const float4 q = lds4(win + swz<SW>(i0 + 4 * c));
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
        if constexpr (TMA_OUT) {
            // registers -> swizzled output buffer; its previous TMA store finished
            // reading before the last barrier (thread 0's wait below)
            unsigned char* ob = outb + (it & 1) * g.out_bytes;
#pragma unroll
            for (int r = 0; r < R; r += 4)
                *reinterpret_cast<float4*>(ob + swz<SW>(static_cast<uint32_t>(base + r))) =
                    make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]);
            fence_proxy_async_smem();
            if (tid == 0) bulk_wait_read_all();  // store it-1 has read buffer (it+1)&1
            __syncthreads();                     // stage consumed, tile outputs staged
            if (tid == 0) {
                tma_store_3d(&out_map, ob, 0, t0 / kIn, row);  // columns past L are clipped
                bulk_commit();
                const int nt = tile + NS * gridDim.x;
                if (nt < ntiles) issue(stage, nt);
            }
        } else {
            if (live) {
                float* o = out + static_cast<int64_t>(row) * L + t0 + base;
#pragma unroll
                for (int r = 0; r < R; r += 4)
                    st_cs_v4(o + r, make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]));
            }
            __syncthreads();  // stage consumed
            if (tid == 0) {
                const int nt = tile + NS * gridDim.x;
                if (nt < ntiles) issue(stage, nt);
            }
        }
    }
    if (TMA_OUT && tid == 0) bulk_wait_all();
}

int stencil_smem_bytes(const StencilGeom& g, int NS, bool tma_out) {
    return NS * g.stage_bytes + (tma_out ? 2 * g.out_bytes : 0) + 64 + 1024;
}

template <int R, int NT, int S, bool FUSED>
ks_status launch(const CUtensorMap& im, const CUtensorMap& om, const float* kp, float* out, int64_t B, int64_t H,
                 int64_t L, int64_t K, const StencilGeom& g, int NS, cudaStream_t st) {
    constexpr bool TMA_OUT = R != 32;
    auto kern = stencil_tma<R, NT, S, FUSED, TMA_OUT>;
    const int smem = stencil_smem_bytes(g, NS, TMA_OUT);
    const int per_sm = prepare_kernel(reinterpret_cast<const void*>(kern), NT, smem);
    const int tiles_per_row = static_cast<int>((L + g.T - 1) / g.T);
    const int ntiles = static_cast<int>(B * H * tiles_per_row);
    const int grid = std::min(ntiles, num_sms() * per_sm);
    launch_kernel_pdl(kern, grid, NT, smem, st, im, om, kp, out, static_cast<int>(H), static_cast<int>(L), static_cast<int>(K),
                                 tiles_per_row, ntiles, g, NS);
    return check_launch();
}

template <int R, int NT>
ks_status launch_s(int s, bool fused, const CUtensorMap& im, const CUtensorMap& om, const float* kp, float* out,
                   int64_t B, int64_t H, int64_t L, int64_t K, const StencilGeom& g, int NS, cudaStream_t st) {
#define KS_ST_CASE(SV)                                                                                 \
    case SV:                                                                                           \
        return fused ? launch<R, NT, SV, true>(im, om, kp, out, B, H, L, K, g, NS, st)                 \
                     : launch<R, NT, SV, false>(im, om, kp, out, B, H, L, K, g, NS, st);
    switch (s) {
        KS_ST_CASE(0)
        KS_ST_CASE(1)
        KS_ST_CASE(2)
        default:
        KS_ST_CASE(3)
    }
#undef KS_ST_CASE
}

}  // namespace

// Register-tile shape for (L, K): R = 32 for compute-bound long K, R = 16 for
// memory-bound short K, R = 4 for short rows; NT chosen so a tile (NT*R
// outputs) does not exceed the row.
static void pick_tile(int64_t L, int64_t K, int* R, int* NT) {
    if (K > 32 && L >= 2048) {
        *R = 32;
        *NT = L >= 8192 ? 256 : L >= 4096 ? 128 : 64;
    } else if (L >= 1024) {
        // K > 8 does twice the FMAs per byte: 128-thread CTAs (more of them
        // per SM) hide it better (config 5a fwd 12.3 -> 11.4 ms)
        *R = 16;
        *NT = L >= 4096 && K <= 8 ? 256 : L >= 2048 ? 128 : 64;
    } else {
        // short rows the row kernels cannot take (L + K too long for one box):
        // the smallest tile that still covers a row, so a tile is not mostly
        // past the row end ((4096,128,256,32): T = 1024 left 3/4 of every
        // tile empty)
        *R = 4;
        *NT = L > 512 ? 256 : L > 256 ? 128 : L > 128 ? 64 : 32;
    }
}

ks_status stencil_short_f32(const float*, const float*, float*, int64_t, int64_t, int64_t, int64_t, int64_t, int,
                            int, cudaStream_t, bool*);

// Sets *handled = false (and does nothing) when this path does not apply; the
// caller then uses the generic kernels of conv_fwd.cu.
ks_status stencil_tma_f32(const float* in, const float* k, float* out, int64_t B, int64_t H, int64_t L, int64_t K,
                          int64_t off, int reverse, int mode, cudaStream_t st, bool* handled) {
    *handled = false;
    if (L % kIn != 0 || L >= (int64_t(1) << 30) || K > 8192) return KS_OK;
    if ((reinterpret_cast<uintptr_t>(out) & 15) != 0) return KS_OK;
    if (opt(kOptStencilPad)) {  // compute-bound long-K kernels from the padded TMA view (stencil_pad.cu)
        const ks_status s = stencil_pad_f32(in, k, out, B, H, L, K, off, reverse, mode, st, handled);
        if (*handled) return s;
    }
    // K-specialised stencil (bwd_short.cuh): K <= 16, and 16 < K <= 28 in
    // Separate mode / K <= 32 in Fused mode on rows of 4096 or more (round-2
    // ABAB against these register tiles, gpurun_out/s28: Separate K = 17..28
    // -8..-14%, K = 32 +10%; Fused L >= 8192 K = 20..32 -8..-15%)
    const int64_t sts = opt(kOptSts);
    const int64_t kmax_sts = sts >= 2 ? 32 : sts == 0 ? 0 : mode == KS_MULADD_FUSED ? (L >= 4096 ? 32 : 16) : 28;
    if (K <= kmax_sts && L >= 1024) {
        const ks_status s = stencil_short_f32(in, k, out, B, H, L, K, off, reverse, mode, st, handled);
        if (*handled) return s;
    }
    int R, NT;
    pick_tile(L, K, &R, &NT);
    if (opt(kOptStencilR) == 32 && L >= 2048) {  // tuning option: R = 32 register tiles at short K
        R = 32;
        NT = L >= 8192 ? 256 : L >= 4096 ? 128 : 64;
    }
    if (R == 16 && opt(kOptStencilNt) > 0) {  // tuning option (bench sweeps)
        const int nt = static_cast<int>(opt(kOptStencilNt));
        if ((nt == 64 || nt == 128 || nt == 256) && nt * R <= L) NT = nt;
    }
    const bool tma_out = R != 32;
    StencilGeom g;
    g.T = NT * R;
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
    const int sw = R == 4 ? 0 : 128;
    CUtensorMap im, om;
    if (!encode_row_view(&im, in, B * H, L, kIn, g.NB, sw)) return KS_OK;
    if (tma_out && !encode_row_view(&om, out, B * H, L, kIn, g.MR, sw)) return KS_OK;
    if (!tma_out) om = im;  // unused
    const int s = static_cast<int>((4 - off % 4) % 4);
    // memory-bound tiles: 3 stages x 2 CTAs/SM measured best on config 3 (a
    // sweep of NT in {128,256} x NS in {2,3,4,6,8} spans 5.9-6.3 TB/s); 2
    // stages of 128-thread tiles for K > 8 (config 5a)
    int NS = K > 8 ? 2 : 3;
    while (NS > 2 && stencil_smem_bytes(g, NS, tma_out) > 110 * 1024) --NS;
    if (R == 32) {
        // compute-bound: spend shared memory on resident warps rather than deep
        // prefetch.  With K >= 1024 a tile's FMAs (R*K per thread) outlast its
        // load by ~100x and one stage suffices; shorter K keeps one tile in flight.
        NS = K >= 1024 ? 1 : 2;
    }
    if (opt(kOptStencilNs) > 0) NS = static_cast<int>(opt(kOptStencilNs));  // tuning option
    if (stencil_smem_bytes(g, NS, tma_out) > 220 * 1024) return KS_OK;

    float* kp = nullptr;
    ks_status rc = cuda_status(scratch_alloc(reinterpret_cast<void**>(&kp), sizeof(float) * H * g.Kp, st));
    if (rc != KS_OK) return rc;
    launch_kernel(prep_taps, static_cast<unsigned>(std::min<int64_t>((H * g.Kp + 255) / 256, 4096)), 256, 0, st, 
        k, kp, H, K, g.Kp, reverse, 0);
    rc = check_launch();
    if (rc == KS_OK) {
        const bool fused = mode == KS_MULADD_FUSED;
        if (R == 4 && NT == 256) rc = launch_s<4, 256>(s, fused, im, om, kp, out, B, H, L, K, g, NS, st);
        else if (R == 4 && NT == 128) rc = launch_s<4, 128>(s, fused, im, om, kp, out, B, H, L, K, g, NS, st);
        else if (R == 4 && NT == 64) rc = launch_s<4, 64>(s, fused, im, om, kp, out, B, H, L, K, g, NS, st);
        else if (R == 4) rc = launch_s<4, 32>(s, fused, im, om, kp, out, B, H, L, K, g, NS, st);
        else if (R == 16 && NT == 256) rc = launch_s<16, 256>(s, fused, im, om, kp, out, B, H, L, K, g, NS, st);
        else if (R == 16 && NT == 128) rc = launch_s<16, 128>(s, fused, im, om, kp, out, B, H, L, K, g, NS, st);
        else if (R == 16) rc = launch_s<16, 64>(s, fused, im, om, kp, out, B, H, L, K, g, NS, st);
        else if (NT == 256) rc = launch_s<32, 256>(s, fused, im, om, kp, out, B, H, L, K, g, NS, st);
        else if (NT == 128) rc = launch_s<32, 128>(s, fused, im, om, kp, out, B, H, L, K, g, NS, st);
        else rc = launch_s<32, 64>(s, fused, im, om, kp, out, B, H, L, K, g, NS, st);
    }
    scratch_free(kp, st);
    *handled = true;
    return rc;
}

}  // namespace ks
