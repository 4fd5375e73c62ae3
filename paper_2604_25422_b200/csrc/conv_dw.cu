// conv_dw.cu -- weight-gradient dW kernels (sm_100a).
//
//   dk[h,j] = sum_b sum_t gy[b,h,t] * x[b,h,t+j-p]      (src/conv_core.cpp:148-181)
//
// The association order of that B*L-deep sum is the whole story of dW:
//
//  * HIERARCHICAL (fast path): in-register FMA partials over t for an 8-tap
//    register block, a fixed warp-shuffle tree, a fixed shared-memory pass over
//    warps, per-CTA partials [G,H,K] in global scratch, then a fixed-order
//    cross-block pass.  Deterministic, no atomics; parity by tolerance.  Its
//    association order is this library's own, so the reference's MulAddMode
//    does not define its bits: it always accumulates with fused multiply-add
//    (one rounding per term -- closer to the exact sum than two, and half
//    the instructions of Separate, which at K = 16 is the difference between
//    an HBM-bound and an issue-bound kernel).  dk is the same in both modes.
//  * PAIRWISE: the reference's midpoint tree over the flat index
//    (src/conv_core.cpp:113-118), evaluated bit-exactly: the top 8 tree levels
//    in shared memory, each depth-8 subtree by one thread.
//  * CHUNKED / SEQUENTIAL: per-chunk sequential chains then `total += partial`
//    in chunk order (src/conv_core.cpp:98-146), bit-exactly.
#include <algorithm>

#include "ks_common.cuh"

namespace ks {

// ---------------------------------------------------------------------------
// HIERARCHICAL
//
// CTA = (row group g, channel h, tap tile jt).  256 threads = NJ tap groups of
// JR=8 taps x NTS = 256/NJ t-slices.  Per (row, 2048-wide t tile) the CTA stages
// gy[t0, t0+TT) and x[t0+j0-p-S, ...) in padded shared memory; thread (jg,ts)
// walks 8-wide t blocks interleaved across the t-slices (lane stride 8 floats,
// conflict-free float4 reads) and does 8x8 FMAs per block from registers.
constexpr int kDwThreads = 256;
constexpr int kDwTT = 2048;  // t per staged tile
constexpr int kJR = 8;       // taps per thread
constexpr int kTB = 8;       // t per register block

template <int NJ, int S>
struct DwGeom {
    static constexpr int NTS = kDwThreads / NJ;
    static constexpr int JT = NJ * kJR;
    static constexpr int SPT = kDwTT / (NTS * kTB);  // register blocks per tile per thread
    static constexpr int NVX = (S + kTB + kJR - 1 + 3) / 4;
    static constexpr int XL = kDwTT + JT + 8;  // staged x window (logical floats, %4 == 0)
    static constexpr int MAXR = 8;             // rows per item on rows shorter than the tile
    static constexpr int GY_FLOATS = padded_len(kDwTT);
    static constexpr int X_FLOATS = padded_len(XL + (MAXR - 1) * (JT + 8));
};

template <int NJ, int S, bool FUSED, bool MR>
__global__ void __launch_bounds__(kDwThreads)
dw_hier_stage1(const float* __restrict__ gy, const float* __restrict__ x,
               float* __restrict__ part, int B, int H, int L, int K, int p, int G, int NJT) {
    using Geo = DwGeom<NJ, S>;
    __shared__ __align__(16) float gys[Geo::GY_FLOATS];
    __shared__ __align__(16) float xs[Geo::X_FLOATS];
    __shared__ float red[kDwThreads / 32][kJR];

    int bid = blockIdx.x;
    const int jt = bid % NJT;
    bid /= NJT;
    const int h = bid % H;
    const int g = bid / H;
    const int b_begin = static_cast<int>(static_cast<int64_t>(B) * g / G);
    const int b_end = static_cast<int>(static_cast<int64_t>(B) * (g + 1) / G);
    const int j0 = jt * Geo::JT;
    const int tid = threadIdx.x;
    const int jg = tid / Geo::NTS;
    const int ts = tid - jg * Geo::NTS;
    // 128-bit loads need 16-byte aligned rows (L % 4 == 0, aligned bases)
    const bool vec_ok = (L & 3) == 0 && ((reinterpret_cast<uintptr_t>(gy) | reinterpret_cast<uintptr_t>(x)) & 15) == 0;

    float acc[kJR];
#pragma unroll
    for (int i = 0; i < kJR; ++i) acc[i] = 0.f;

    // rows shorter than the 2048-wide tile: an item is R whole rows, row r at
    // tile offset r * Lp (Lp = L rounded up to a t block; gy zero in between)
    // with its own x window (XW = Lp + JT + 8 floats, its own zero halo), so
    // a block's x index moves by XW - Lp per row
    const int Lp = (L + kTB - 1) / kTB * kTB;
    const int R = MR ? min(Geo::MAXR, kDwTT / Lp) : 1;  // MR: the host picks it for L <= 512
    const int XW = Lp + Geo::JT + 8;
    for (int b = b_begin; b < b_end; b += R) {
        const int nr = min(R, b_end - b);
        for (int t0 = 0; t0 < L; t0 += kDwTT) {
            // stage gy tile
            for (int c = tid; c < kDwTT / 4; c += kDwThreads) {
                int q = t0 + 4 * c, r = 0;
                if (MR) {
                    r = (4 * c) / Lp;
                    q = 4 * c - r * Lp;
                }
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (r < nr) {
                    const float* rg = gy + (static_cast<int64_t>(b + r) * H + h) * L;
                    if (vec_ok && q + 3 < L) {
                        v = ld_nc_v4(rg + q);
                    } else {
                        v.x = q + 0 < L ? rg[q + 0] : 0.f;
                        v.y = q + 1 < L ? rg[q + 1] : 0.f;
                        v.z = q + 2 < L ? rg[q + 2] : 0.f;
                        v.w = q + 3 < L ? rg[q + 3] : 0.f;
                    }
                }
                *reinterpret_cast<float4*>(gys + pad_idx(4 * c)) = v;
            }
            // stage x window(s), logical index i <-> x position a0 + i (of row r's window)
            const int a0 = t0 + j0 - p - S;
            const int nxw = MR ? nr * XW : Geo::XL;
            for (int c = tid; c < nxw / 4; c += kDwThreads) {
                int q = a0 + 4 * c, r = 0;
                if (MR) {
                    r = (4 * c) / XW;
                    q = a0 + 4 * c - r * XW;
                }
                const float* rx = x + (static_cast<int64_t>(b + r) * H + h) * L;
                float4 v;
                if (vec_ok && q >= 0 && q + 3 < L) {
                    v = ld_nc_v4(rx + q);
                } else {
                    v.x = (q + 0 >= 0 && q + 0 < L) ? rx[q + 0] : 0.f;
                    v.y = (q + 1 >= 0 && q + 1 < L) ? rx[q + 1] : 0.f;
                    v.z = (q + 2 >= 0 && q + 2 < L) ? rx[q + 2] : 0.f;
                    v.w = (q + 3 >= 0 && q + 3 < L) ? rx[q + 3] : 0.f;
                }
                *reinterpret_cast<float4*>(xs + pad_idx(4 * c)) = v;
            }
            __syncthreads();
#pragma unroll 2
            for (int s = 0; s < Geo::SPT; ++s) {
                int tl = (s * Geo::NTS + ts) * kTB;
                bool live = t0 + tl < L;
                int xsh = 0;
                if (MR) {
                    const int r = tl / Lp;
                    live = r < nr && tl - r * Lp < L;
                    xsh = r * (XW - Lp);
                }
                if (live) {
                    float gv[kTB];
#pragma unroll
                    for (int c = 0; c < kTB / 4; ++c) {
                        const float4 q = *reinterpret_cast<const float4*>(gys + pad_idx(tl + 4 * c));
                        gv[4 * c + 0] = q.x;
                        gv[4 * c + 1] = q.y;
                        gv[4 * c + 2] = q.z;
                        gv[4 * c + 3] = q.w;
                    }
                    float xv[4 * Geo::NVX];
#pragma unroll
                    for (int c = 0; c < Geo::NVX; ++c) {
                        const float4 q = *reinterpret_cast<const float4*>(
                            xs + pad_idx(tl + xsh + jg * kJR + 4 * c));
                        xv[4 * c + 0] = q.x;
                        xv[4 * c + 1] = q.y;
                        xv[4 * c + 2] = q.z;
                        xv[4 * c + 3] = q.w;
                    }
#pragma unroll
                    for (int tt = 0; tt < kTB; ++tt)
#pragma unroll
                        for (int jj = 0; jj < kJR; ++jj)
                            acc[jj] = muladd<true>(acc[jj], gv[tt], xv[S + tt + jj]);
                }
            }
            __syncthreads();
        }
    }

    // fixed-order reduction over the t-slices of each tap group
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
    constexpr int WPG = Geo::NTS / 32;  // warps per tap group
    if (tid < Geo::JT) {
        const int gj = tid / kJR, jj = tid % kJR;
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < WPG; ++w) s += red[gj * WPG + w][jj];
        const int j = j0 + tid;
        if (j < K) part[(static_cast<int64_t>(g) * H + h) * K + j] = s;
    }
}

// dk[h,j] = fixed-order sum over the G row-group partials.
template <typename T>
__global__ void dw_sum_groups(const T* __restrict__ part, T* __restrict__ dk, int64_t HK, int G) {
    pdl_wait();  // launched with PDL after stage 1
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= HK) return;
    // ascending g, plain adds; the loads of a block of 8 groups are issued
    // before its adds (independent), so the chain waits on memory once per
    // 8 groups, not once per group (config 1: G = 16, 5.2 -> ~1.5 us)
    T s = part[i];
    int g = 1;
    for (; g + 8 <= G; g += 8) {
        T v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = part[static_cast<int64_t>(g + u) * HK + i];
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; g < G; ++g) s += part[static_cast<int64_t>(g) * HK + i];
    dk[i] = s;
}

// ---------------------------------------------------------------------------
// PAIRWISE (exact)

template <typename T>
__device__ __forceinline__ T dw_leaf(const T* __restrict__ gy, const T* __restrict__ x,
                                     int64_t H, int64_t h, int64_t d, int64_t L, int64_t flat) {
    // WeightTerm::operator() (src/conv_core.cpp:88-95): plain product or +0.
    const int64_t b = flat / L;
    const int64_t t = flat - b * L;
    const int64_t xi = t + d;
    if (xi < 0 || xi >= L) return T(0);
    const int64_t row = (b * H + h) * L;
    if constexpr (sizeof(T) == 4) return __fmul_rn(gy[row + t], x[row + xi]);
    else return __dmul_rn(gy[row + t], x[row + xi]);
}

// Midpoint-split recursion of reduce_pairwise, restated iteratively with an
// explicit stack so deep subtrees need no device call stack.
template <typename T>
__device__ T dw_pairwise_subtree(const T* __restrict__ gy, const T* __restrict__ x, int64_t H,
                                 int64_t h, int64_t d, int64_t L, int64_t lo, int64_t hi) {
    // Post-order walk: each frame is [lo,hi) with a flag telling whether its
    // left child's value has been pushed.
    int64_t st_lo[48], st_hi[48];
    T vals[48];
    int st_state[48];
    int sp = 0, vp = 0;
    st_lo[0] = lo;
    st_hi[0] = hi;
    st_state[0] = 0;
    sp = 1;
    while (sp > 0) {
        const int top = sp - 1;
        const int64_t a = st_lo[top], c = st_hi[top];
        if (c - a == 1) {
            vals[vp++] = dw_leaf<T>(gy, x, H, h, d, L, a);
            --sp;
            continue;
        }
        const int64_t mid = a + (c - a) / 2;
        if (st_state[top] == 0) {
            st_state[top] = 1;
            st_lo[sp] = a;
            st_hi[sp] = mid;
            st_state[sp] = 0;
            ++sp;
        } else if (st_state[top] == 1) {
            st_state[top] = 2;
            st_lo[sp] = mid;
            st_hi[sp] = c;
            st_state[sp] = 0;
            ++sp;
        } else {
            const T right = vals[--vp];
            const T left = vals[--vp];
            vals[vp++] = left + right;
            --sp;
        }
    }
    return vals[0];
}

// One CTA per (h,j).  Depth-D nodes (D <= 8) each computed by one thread; all
// nodes above depth D are internal (size >= 2), so the top is a perfect binary
// tree combined in shared memory with children (2i, 2i+1).
template <typename T>
__global__ void __launch_bounds__(256)
dw_pairwise_exact(const T* __restrict__ gy, const T* __restrict__ x, T* __restrict__ dk,
                  int64_t B, int64_t H, int64_t L, int64_t K, int D) {
    __shared__ T buf[2][256];
    const int64_t hj = blockIdx.x;
    const int64_t h = hj / K, j = hj - h * K;
    const int64_t d = j - K / 2;
    const int64_t n = B * L;
    const int nn = 1 << D;
    const int i = threadIdx.x;
    if (i < nn) {
        int64_t lo = 0, hi = n;
        for (int lev = D - 1; lev >= 0; --lev) {
            const int64_t mid = lo + (hi - lo) / 2;
            if ((i >> lev) & 1) lo = mid;
            else hi = mid;
        }
        buf[0][i] = dw_pairwise_subtree<T>(gy, x, H, h, d, L, lo, hi);
    }
    __syncthreads();
    int src = 0;
    for (int w = nn >> 1; w >= 1; w >>= 1) {
        if (i < w) buf[src ^ 1][i] = buf[src][2 * i] + buf[src][2 * i + 1];
        __syncthreads();
        src ^= 1;
    }
    if (i == 0) dk[hj] = buf[src][0];
}

// ---------------------------------------------------------------------------
// CHUNKED / SEQUENTIAL (exact)

// Sequential chain over the valid flat indices of [f_lo, f_hi) for tap offset d
// (the inner loops of reduce_sequential / reduce_chunked).
template <typename T, bool FUSED>
__device__ T dw_chain(const T* __restrict__ gy, const T* __restrict__ x, int64_t H, int64_t h,
                      int64_t d, int64_t L, int64_t f_lo, int64_t f_hi) {
    const int64_t t_lo = d < 0 ? -d : 0;
    const int64_t t_hi = d > 0 ? L - d : L;
    T acc = T(0);
    int64_t b = f_lo / L;
    for (int64_t f = b * L; f < f_hi; f += L, ++b) {
        const int64_t row = (b * H + h) * L;
        int64_t ta = f_lo > f ? f_lo - f : 0;
        int64_t tb = f_hi - f < L ? f_hi - f : L;
        if (ta < t_lo) ta = t_lo;
        if (tb > t_hi) tb = t_hi;
        for (int64_t t = ta; t < tb; ++t) acc = muladd<FUSED>(acc, gy[row + t], x[row + t + d]);
    }
    return acc;
}

// part[c,h,j] = chain over chunk c.  Threads of a warp take consecutive taps of
// one (h, chunk), so gy reads broadcast and x reads coalesce.
template <typename T, bool FUSED>
__global__ void __launch_bounds__(256)
dw_chunk_partials(const T* __restrict__ gy, const T* __restrict__ x, T* __restrict__ part,
                  int64_t B, int64_t H, int64_t L, int64_t K, int64_t chunk, int64_t nchunks) {
    const int64_t total = nchunks * H * K;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = i % K;
        const int64_t ch = i / K;  // c*H + h
        const int64_t h = ch % H;
        const int64_t c = ch / H;
        const int64_t f_lo = c * chunk;
        const int64_t f_hi = std::min<int64_t>(f_lo + chunk, B * L);
        part[i] = dw_chain<T, FUSED>(gy, x, H, h, j - K / 2, L, f_lo, f_hi);
    }
}

// dk = ((0 + part[0]) + part[1]) + ... in chunk order (reduce_chunked's
// `total += partial`, :135-145).  With one chunk (SEQUENTIAL or chunk >= B*L)
// the chain is returned as is (reduce_sequential).
template <typename T>
__global__ void dw_chunk_total(const T* __restrict__ part, T* __restrict__ dk, int64_t HK,
                               int64_t nchunks) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= HK) return;
    if (nchunks == 1) {
        dk[i] = part[i];
        return;
    }
    T total = T(0);
    for (int64_t c = 0; c < nchunks; ++c) total = total + part[c * HK + i];
    dk[i] = total;
}

// Workspace-free variant for huge chunk counts: one thread per (h,j) walks its
// chunks in order.
template <typename T, bool FUSED>
__global__ void dw_chunked_fused(const T* __restrict__ gy, const T* __restrict__ x,
                                 T* __restrict__ dk, int64_t B, int64_t H, int64_t L, int64_t K,
                                 int64_t chunk, int64_t nchunks) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= H * K) return;
    const int64_t h = i / K, j = i - h * K;
    T total = T(0);
    for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t f_lo = c * chunk;
        const int64_t f_hi = std::min<int64_t>(f_lo + chunk, B * L);
        total = total + dw_chain<T, FUSED>(gy, x, H, h, j - K / 2, L, f_lo, f_hi);
    }
    dk[i] = total;
}

// ---------------------------------------------------------------------------
// host side

namespace {

struct HierPlan {
    int nj;   // tap groups per CTA (1,2,4,8)
    int njt;  // tap tiles
    int g;    // row groups
};

// CTA target: dw_ctas (8192 by default) -- but never so many that a CTA holds
// less than ~2^18 multiply-adds: small problems (config 1: 67 M MACs) are
// latency-bound per CTA, and fewer, fuller CTAs amortise the per-CTA tile
// loads and reduction trees (config 1 dW 12.3 -> 10.0 us at 256 CTAs instead
// of 1024; `tools/sweep_options.py`, gpurun_out/s5).  Large shapes are
// unaffected (the paper's shape wants its 8192).
HierPlan hier_plan(int64_t B, int64_t H, int64_t L, int64_t K) {
    HierPlan pl;
    const int64_t groups8 = (K + kJR - 1) / kJR;
    pl.nj = 1;
    while (pl.nj < 8 && pl.nj < groups8) pl.nj *= 2;
    pl.njt = static_cast<int>((K + pl.nj * kJR - 1) / (pl.nj * kJR));
    const double macs = static_cast<double>(B) * H * L * K;
    const int64_t target = std::min<int64_t>(opt(kOptDwCtas), std::max<int64_t>(256, static_cast<int64_t>(macs / 262144.0)));
    int64_t g = (target + H * pl.njt - 1) / (H * pl.njt);
    g = std::max<int64_t>(1, std::min<int64_t>(g, B));
    pl.g = static_cast<int>(g);
    return pl;
}

constexpr size_t kChunkWsCap = size_t(512) << 20;

int64_t chunk_count(int64_t B, int64_t L, int scheme, int64_t chunk) {
    const int64_t n = B * L;
    if (scheme == KS_DW_SEQUENTIAL || chunk >= n) return 1;
    return (n + chunk - 1) / chunk;
}

template <int NJ, bool FUSED>
ks_status launch_hier_s(int s, const float* gy, const float* x, float* part, int64_t B,
                        int64_t H, int64_t L, int64_t K, const HierPlan& pl, cudaStream_t st) {
    const unsigned blocks = static_cast<unsigned>(int64_t(pl.g) * H * pl.njt);
    const int p = static_cast<int>(K / 2);
    // rows of at most 512: items of several whole rows (-35..-69% at L = 250 / 500;
    // at L = 1000 two rows per item measured 4% slower, gpurun_out/ab_head_generic)
    const bool mr = L <= 512;
#define KS_HIER_CASE(SV)                                                                  \
    case SV:                                                                              \
        if (mr)                                                                           \
            launch_kernel(dw_hier_stage1<NJ, SV, FUSED, true>, blocks, kDwThreads, 0, st,  \
                gy, x, part, static_cast<int>(B), static_cast<int>(H), static_cast<int>(L), \
                static_cast<int>(K), p, pl.g, pl.njt);                                    \
        else                                                                              \
            launch_kernel(dw_hier_stage1<NJ, SV, FUSED, false>, blocks, kDwThreads, 0, st, \
                gy, x, part, static_cast<int>(B), static_cast<int>(H), static_cast<int>(L), \
                static_cast<int>(K), p, pl.g, pl.njt);                                    \
        break;
    switch (s) {
        KS_HIER_CASE(0)
        KS_HIER_CASE(1)
        KS_HIER_CASE(2)
        default:
        KS_HIER_CASE(3)
    }
#undef KS_HIER_CASE
    return check_launch();
}

template <bool FUSED>
ks_status launch_hier(const float* gy, const float* x, float* part, int64_t B, int64_t H,
                      int64_t L, int64_t K, const HierPlan& pl, cudaStream_t st) {
    const int p = static_cast<int>(K / 2);
    const int s = (4 - p % 4) % 4;
    switch (pl.nj) {
        case 1: return launch_hier_s<1, FUSED>(s, gy, x, part, B, H, L, K, pl, st);
        case 2: return launch_hier_s<2, FUSED>(s, gy, x, part, B, H, L, K, pl, st);
        case 4: return launch_hier_s<4, FUSED>(s, gy, x, part, B, H, L, K, pl, st);
        default: return launch_hier_s<8, FUSED>(s, gy, x, part, B, H, L, K, pl, st);
    }
}

}  // namespace

size_t dw_pairwise_tma_workspace(int64_t B, int64_t H, int64_t L, int64_t K);
ks_status dw_pairwise_tma_f32(const float* gy, const float* x, float* dk, int64_t B, int64_t H, int64_t L,
                              int64_t K, void* ws, cudaStream_t st, bool* handled);
bool dw_pad_applies(int64_t B, int64_t H, int64_t L, int64_t K);
int dw_pad_groups(int64_t B, int64_t H, int64_t K);
ks_status dw_pad_stage1(const float* gy, const float* x, float* part, int64_t B, int64_t H, int64_t L, int64_t K,
                       int G, int mode, cudaStream_t st, bool* handled);

// Row groups G of the HIERARCHICAL partial buffer part[G,H,K] for this shape.
static int hier_groups(int64_t B, int64_t H, int64_t L, int64_t K) {
    if (!tma_disabled() && dw_pad_applies(B, H, L, K)) return dw_pad_groups(B, H, K);
    return hier_plan(B, H, L, K).g;
}

size_t dw_workspace_bytes(int64_t B, int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk,
                          int elem) {
    if (scheme == KS_DW_HIERARCHICAL) {
        if (elem != 4) return 0;  // fp64 HIERARCHICAL runs the exact pairwise kernel
        const int g = std::max(hier_groups(B, H, L, K), hier_plan(B, H, L, K).g);
        return size_t(g) * H * K * sizeof(float);
    }
    if (scheme == KS_DW_PAIRWISE) return elem == 4 ? dw_pairwise_tma_workspace(B, H, L, K) : 0;
    const int64_t nc = chunk_count(B, L, scheme, chunk);
    const size_t bytes = size_t(nc) * H * K * elem;
    return bytes <= kChunkWsCap ? bytes : 0;
}

template <typename T>
static ks_status dw_exact(const T* gy, const T* x, T* dk, int64_t B, int64_t H, int64_t L,
                          int64_t K, int scheme, int64_t chunk, int mode, void* ws,
                          cudaStream_t st) {
    const int64_t HK = H * K;
    if (scheme == KS_DW_PAIRWISE || scheme == KS_DW_HIERARCHICAL) {
        const int64_t n = B * L;
        int D = 0;
        while (D < 8 && (int64_t(2) << D) <= n) ++D;
        launch_kernel(dw_pairwise_exact<T>, static_cast<unsigned>(HK), 256, 0, st, gy, x, dk, B, H, L, K, D);
        return check_launch();
    }
    const int64_t nc = chunk_count(B, L, scheme, chunk);
    const size_t need = size_t(nc) * HK * sizeof(T);
    if (need <= kChunkWsCap) {
        T* part = static_cast<T*>(ws);
        const int64_t total = nc * HK;
        const unsigned blocks =
            static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, int64_t(num_sms()) * 64));
        if (mode == KS_MULADD_FUSED)
            launch_kernel(dw_chunk_partials<T, true>, blocks, 256, 0, st, gy, x, part, B, H, L, K,
                                                               nc == 1 ? B * L : chunk, nc);
        else
            launch_kernel(dw_chunk_partials<T, false>, blocks, 256, 0, st, gy, x, part, B, H, L, K,
                                                                nc == 1 ? B * L : chunk, nc);
        ks_status s = check_launch();
        if (s != KS_OK) return s;
        launch_kernel(dw_chunk_total<T>, static_cast<unsigned>((HK + 255) / 256), 256, 0, st, part, dk, HK, nc);
        return check_launch();
    }
    const unsigned blocks = static_cast<unsigned>((HK + 127) / 128);
    if (mode == KS_MULADD_FUSED)
        launch_kernel(dw_chunked_fused<T, true>, blocks, 128, 0, st, gy, x, dk, B, H, L, K, chunk, nc);
    else
        launch_kernel(dw_chunked_fused<T, false>, blocks, 128, 0, st, gy, x, dk, B, H, L, K, chunk, nc);
    return check_launch();
}

// Sharded CHUNKED(c) support (dist.cu): the partials of `nchunks` chunks of
// this rank's rows (flat index from the rank's first row), and the total over
// the gathered partials of every rank in rank order = global chunk order.
ks_status dw_chunk_partials_f32(const float* gy, const float* x, float* part, int64_t B, int64_t H, int64_t L,
                                int64_t K, int64_t chunk, int64_t nchunks, int mode, cudaStream_t st) {
    const int64_t total = nchunks * H * K;
    if (total == 0) return KS_OK;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, int64_t(num_sms()) * 64));
    if (mode == KS_MULADD_FUSED)
        launch_kernel(dw_chunk_partials<float, true>, blocks, 256, 0, st, gy, x, part, B, H, L, K, chunk, nchunks);
    else
        launch_kernel(dw_chunk_partials<float, false>, blocks, 256, 0, st, gy, x, part, B, H, L, K, chunk, nchunks);
    return check_launch();
}

struct RankChunks {
    int n[64];  // chunks held by each rank
};

// dk[i] = ((0 + p[0]) + p[1]) + ... over every rank's chunks in rank order --
// dw_chunk_total's order on the global chunk list (one chunk in all: copied).
__global__ void dw_chunk_total_ranks(const float* __restrict__ gather, float* __restrict__ dk, int64_t HK,
                                     int world, int ncmax, RankChunks rc) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= HK) return;
    int ntot = 0;
    for (int r = 0; r < world; ++r) ntot += rc.n[r];
    float total = 0.f;
    bool first = true;
    for (int r = 0; r < world; ++r)
        for (int c = 0; c < rc.n[r]; ++c) {
            const float v = gather[(static_cast<int64_t>(r) * ncmax + c) * HK + i];
            total = (ntot == 1 && first) ? v : total + v;
            first = false;
        }
    dk[i] = total;
}

ks_status dw_chunk_total_ranks_f32(const float* gather, float* dk, int64_t HK, int world, int ncmax,
                                   const int* counts, cudaStream_t st) {
    RankChunks rc{};
    for (int r = 0; r < world && r < 64; ++r) rc.n[r] = counts[r];
    launch_kernel(dw_chunk_total_ranks, static_cast<unsigned>((HK + 255) / 256), 256, 0, st, gather, dk, HK, world,
                  ncmax, rc);
    return check_launch();
}

ks_status dw_tma_stage1(const float*, const float*, float*, int64_t, int64_t, int64_t, int64_t, int, int,
                        cudaStream_t, bool*);

ks_status dw_rows_stage1(const float*, const float*, float*, int64_t, int64_t, int64_t, int64_t, int, int,
                         cudaStream_t, bool*);
ks_status dw_stage1_only(const float*, const float*, float*, int64_t, int64_t, int64_t, int64_t, int, int, int*,
                         cudaStream_t);

ks_status dw_f32(const float* gy, const float* x, float* dk, int64_t B, int64_t H, int64_t L,
                 int64_t K, int scheme, int64_t chunk, int mode, void* ws, cudaStream_t st) {
    if (scheme == KS_DW_PAIRWISE && !tma_disabled()) {
        bool handled = false;
        const ks_status s = dw_pairwise_tma_f32(gy, x, dk, B, H, L, K, ws, st, &handled);
        if (handled) return s;
    }
    if (scheme != KS_DW_HIERARCHICAL)
        return dw_exact<float>(gy, x, dk, B, H, L, K, scheme, chunk, mode, ws, st);
    if (L > (1ll << 30) || K > (1ll << 30) || B > (1ll << 30))
        return dw_exact<float>(gy, x, dk, B, H, L, K, KS_DW_PAIRWISE, 0, mode, ws, st);
    float* part = static_cast<float*>(ws);
    int G = 0;
    ks_status s = dw_stage1_only(gy, x, part, B, H, L, K, mode, 0, &G, st);
    if (s != KS_OK) return s;
    const int64_t HK = H * K;
    launch_kernel_pdl(dw_sum_groups<float>, static_cast<unsigned>((HK + 255) / 256), 256, 0, st, part, dk, HK, G);
    return check_launch();
}

// Row groups the HIERARCHICAL plan gives this shape (the G of part[G,H,K]).
int dw_plan_groups(int64_t B, int64_t H, int64_t L, int64_t K) { return hier_groups(B, H, L, K); }

// HIERARCHICAL stage 1 only: per-CTA partials part[G,H,K] (G returned), for
// the fused cross-GPU combine of peer.cu and for dw_f32 above.  G_req > 0
// overrides the plan's row-group count (peer.cu: this rank's share of the
// global plan's groups); the kernel tier is chosen exactly as without it.
//
// The TMA tiers need 16-byte aligned bases; a caller's offset view that is
// not (L % 4 == 0 but the base is off by 4, 8 or 12 bytes) is first copied
// into aligned stream-ordered scratch, so the kernel -- and with it the
// association order, i.e. the bits of dk -- never depends on where the
// caller's tensors sit in memory.  (L % 4 != 0 cannot be encoded as a TMA
// view at any alignment: those shapes always take the generic kernel.)
ks_status dw_stage1_only(const float* gy, const float* x, float* part, int64_t B, int64_t H, int64_t L, int64_t K,
                         int mode, int G_req, int* G, cudaStream_t st) {
    if ((((reinterpret_cast<uintptr_t>(gy) | reinterpret_cast<uintptr_t>(x)) & 15) != 0) && L % 4 == 0 &&
        !tma_disabled()) {
        const size_t n = size_t(B) * size_t(H) * size_t(L);
        float* a = nullptr;
        ks_status s = cuda_status(scratch_alloc(reinterpret_cast<void**>(&a), 2 * n * sizeof(float), st));
        if (s != KS_OK) return s;
        if (!planning()) {
            s = cuda_status(cudaMemcpyAsync(a, gy, n * sizeof(float), cudaMemcpyDeviceToDevice, st));
            if (s == KS_OK) s = cuda_status(cudaMemcpyAsync(a + n, x, n * sizeof(float), cudaMemcpyDeviceToDevice, st));
        }
        if (s == KS_OK) s = dw_stage1_only(a, a + n, part, B, H, L, K, mode, G_req, G, st);
        scratch_free(a, st);
        return s;
    }
    HierPlan pl = hier_plan(B, H, L, K);
    bool handled = false;
    ks_status s = KS_OK;
    if (!tma_disabled() && dw_pad_applies(B, H, L, K)) {  // compute-bound long K (dw_pad.cu)
        pl.g = G_req > 0 ? G_req : dw_pad_groups(B, H, K);
        s = dw_pad_stage1(gy, x, part, B, H, L, K, pl.g, mode, st, &handled);
        if (!handled) pl = hier_plan(B, H, L, K);
    }
    if (G_req > 0) pl.g = G_req;
    if (!handled && L < 2048) s = dw_rows_stage1(gy, x, part, B, H, L, K, pl.g, mode, st, &handled);  // short rows
    if (!handled && !tma_disabled()) s = dw_tma_stage1(gy, x, part, B, H, L, K, pl.g, mode, st, &handled);
    if (!handled)
        s = launch_hier<true>(gy, x, part, B, H, L, K, pl, st);
    *G = pl.g;
    return s;
}

ks_status bwd_tma_stage1(const float*, const float*, const float*, float*, float*, int64_t, int64_t, int64_t,
                         int64_t, int, int, cudaStream_t, bool*);

// Fused backward (dx + HIERARCHICAL dk) where dw_f32 would run the TMA dW
// kernel with one tap group (L % 32 == 0, L >= 2048, K <= 16): same row
// groups G, same decomposition, so dk's bits equal dw_f32's and dx's equal
// the stencil's.  *fused = false: the caller runs dX and dW in turn.
ks_status bwd_fused_f32(const float* gy, const float* x, const float* k, float* dx, float* dk, int64_t B,
                        int64_t H, int64_t L, int64_t K, int mode, void* ws, cudaStream_t st, bool* fused) {
    *fused = false;
    if (tma_disabled() || L < 2048 || L % 32 != 0 || K > 16 || dw_pad_applies(B, H, L, K)) return KS_OK;
    // unaligned bases: the split path (dw_f32 stages them into aligned scratch)
    if (((reinterpret_cast<uintptr_t>(gy) | reinterpret_cast<uintptr_t>(x)) & 15) != 0) return KS_OK;
    if (L > (1ll << 30) || B > (1ll << 30)) return KS_OK;
    const HierPlan pl = hier_plan(B, H, L, K);
    float* part = static_cast<float*>(ws);
    const ks_status s = bwd_tma_stage1(gy, x, k, dx, part, B, H, L, K, pl.g, mode, st, fused);
    if (s != KS_OK || !*fused) return s;
    const int64_t HK = H * K;
    launch_kernel_pdl(dw_sum_groups<float>, static_cast<unsigned>((HK + 255) / 256), 256, 0, st, part, dk, HK, pl.g);
    return check_launch();
}

ks_status dw_f64(const double* gy, const double* x, double* dk, int64_t B, int64_t H, int64_t L,
                 int64_t K, int scheme, int64_t chunk, int mode, void* ws, cudaStream_t st) {
    return dw_exact<double>(gy, x, dk, B, H, L, K, scheme, chunk, mode, ws, st);
}

}  // namespace ks
