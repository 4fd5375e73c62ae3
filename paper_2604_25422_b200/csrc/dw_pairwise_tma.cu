// dw_pairwise_tma.cu -- weight gradient in the reference's PAIRWISE order,
// bit-exact, at HBM speed (sm_100a).
//
// reduce_pairwise (reference src/conv_core.cpp:113-118) sums the B*L leaves
// leaf(f) = gy[b,h,t] * x[b,h,t+d]  (f = b*L+t; +0 when t+d leaves the row,
// WeightTerm::operator(), :88-95) with a midpoint-split binary tree.  When B
// and L are powers of two that tree is the perfect binary tree over f, whose
// nodes are aligned power-of-two blocks; every row, every 2048-wide tile and
// every aligned group of rows is a node.  So it can be evaluated bottom-up in
// any decomposition that respects node boundaries, and this kernel does:
//
//   level   0..2   8 leaves of a lane, in registers          ((l0+l1)+(l2+l3))+...
//   level   3..    NJ blocks of a lane, in registers (unrolled tree)
//   next 5 levels  the 32 lanes of a warp: reduce-scatter butterfly over the
//                  8 taps (4+2+1 shuffles), then two full exchanges
//   next levels    the WG warps covering one 2048-leaf tile, in shared memory
//   next levels    the work items of the CTA (rows x tiles, flat order), in
//                  shared memory, at the end
//   top levels     the G row groups: dw_sum_groups_tree (a perfect tree over g)
//
// Every addition is (left subtree) + (right subtree) of the reference tree
// (IEEE addition is commutative, so which lane performs it does not matter);
// leaves are plain products (__fmul_rn), +0 for out-of-row taps.  The result is
// bit-identical to conv::backward_weight(..., AccumulationScheme::pairwise()).
// Inputs arrive through the same TMA/mbarrier stage ring as dw_tma.cu.
#include <algorithm>

#include "ks_common.cuh"
#include "ks_tma.cuh"

namespace ks {

namespace {

constexpr int kThreads = 256;
constexpr int kTT = 2048;              // leaves (t) per work item = one tree node
constexpr int kIn = 32;                // floats per TMA row piece (128 B)
constexpr int kMain = kTT / kIn;       // rows of the gy box / x main box
constexpr int kJR = 8;                 // taps per tap group
constexpr int kLevels = 20;            // log2 of the max work items per CTA
constexpr int kMaxUnits = 1 << kLevels;

struct PwGeom {
    int XT;           // x tail rows
    int gy_bytes;
    int stage_bytes;
};

// Tree over the 8 leaves of one 8-wide block for 8 taps: out[j] = node sum.
// g: gy[t..t+7]; xv: x window with xv[S + tt + jj] = x[t + tt + j0 + jj - p].
template <int S, bool MASK>
__device__ __forceinline__ void block_tree(const float* gv, const float* xv, float* out, int t, int jbase, int L) {
#pragma unroll
    for (int jj = 0; jj < kJR; ++jj) {
        float l[8];
#pragma unroll
        for (int tt = 0; tt < 8; ++tt) {
            float v = __fmul_rn(gv[tt], xv[S + tt + jj]);
            if constexpr (MASK) {
                const int xi = t + tt + jbase + jj;  // t + d
                v = (xi >= 0 && xi < L) ? v : 0.f;
            }
            l[tt] = v;
        }
        const float a = __fadd_rn(l[0], l[1]), b = __fadd_rn(l[2], l[3]);
        const float c = __fadd_rn(l[4], l[5]), d = __fadd_rn(l[6], l[7]);
        out[jj] = __fadd_rn(__fadd_rn(a, b), __fadd_rn(c, d));
    }
}

// Perfect tree over NB consecutive 8-leaf blocks starting at block `b0` of the
// lane's segment (unrolled; left + right at every level).
template <int NB, int S, bool MASK>
__device__ __forceinline__ void seg_tree(const unsigned char* gys, const unsigned char* xs, uint32_t seg_t, int b0,
                                         int A, int jgbase, int t0, int jbase, int L, float* out) {
    if constexpr (NB == 1) {
        constexpr int NVX = (S + 8 + kJR - 1 + 3) / 4;
        const uint32_t tl = seg_t + 8 * b0;
        float gv[8];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const float4 q = lds4(gys + swz<128>(tl + 4 * c));
            gv[4 * c + 0] = q.x;
            gv[4 * c + 1] = q.y;
            gv[4 * c + 2] = q.z;
            gv[4 * c + 3] = q.w;
        }
        float xv[4 * NVX];
        const uint32_t xi = static_cast<uint32_t>(A) + tl + static_cast<uint32_t>(jgbase);
#pragma unroll
        for (int c = 0; c < NVX; ++c) {
            const float4 q = lds4(xs + swz<128>(xi + 4 * c));
            xv[4 * c + 0] = q.x;
            xv[4 * c + 1] = q.y;
            xv[4 * c + 2] = q.z;
            xv[4 * c + 3] = q.w;
        }
        block_tree<S, MASK>(gv, xv, out, t0 + static_cast<int>(tl), jbase, L);
    } else {
        float left[kJR], right[kJR];
        seg_tree<NB / 2, S, MASK>(gys, xs, seg_t, b0, A, jgbase, t0, jbase, L, left);
        seg_tree<NB / 2, S, MASK>(gys, xs, seg_t, b0 + NB / 2, A, jgbase, t0, jbase, L, right);
#pragma unroll
        for (int jj = 0; jj < kJR; ++jj) out[jj] = __fadd_rn(left[jj], right[jj]);
    }
}

// NJ tap groups of 8 taps; WG = 8/NJ warps per group cover one 2048-leaf item;
// each lane owns NB = NJ consecutive 8-leaf blocks.
template <int NJ, int S>
__global__ void __launch_bounds__(kThreads)
dw_pairwise_tma(const __grid_constant__ CUtensorMap gy_map, const __grid_constant__ CUtensorMap x_map,
                const __grid_constant__ CUtensorMap x_tail_map, float* __restrict__ part, int B, int H, int L,
                int K, int p, int G, int NJT, PwGeom g, int NS) {
    constexpr int WG = 8 / NJ;
    constexpr int NB = NJ;  // blocks per lane: 32*WG lanes * 8*NB leaves = 2048
    constexpr int JT = NJ * kJR;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = align_smem<1024>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * g.stage_bytes);
    __shared__ float warp_node[2][8][kJR];  // [unit parity][warp][tap]
    __shared__ float pending[kLevels][JT];  // left siblings awaiting their right (binary counter)

    int bid = blockIdx.x;
    const int jt = bid % NJT;
    bid /= NJT;
    const int h = bid % H;
    const int grp = bid / H;
    const int rows = B / G;  // power of two
    const int b_begin = grp * rows;
    const int j0 = jt * JT;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int jg = warp / WG;        // tap group
    const int wg = warp - jg * WG;   // warp within the group
    const int ntt = L / kTT;         // power of two
    const int nunits = rows * ntt;
    const int xoff = j0 - p;
    const int D = ((xoff % kIn) + kIn) % kIn;
    const int xr_rel = (xoff - D) / kIn;
    const int A = D & ~3;
    const int jbase = j0 + jg * kJR - p;  // d of this lane's tap 0
    const uint32_t seg_t = static_cast<uint32_t>((wg * 32 + lane) * 8 * NB);

    if (tid == 0) {
        prefetch_tmap(&gy_map);
        prefetch_tmap(&x_map);
        prefetch_tmap(&x_tail_map);
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint32_t tx_bytes = static_cast<uint32_t>(g.gy_bytes + (kMain + g.XT) * kIn * 4);
    auto issue = [&](int stage, int u) {
        const int b = b_begin + u / ntt;
        const int t0 = (u % ntt) * kTT;
        const int row = b * H + h;
        unsigned char* sb = smem + stage * g.stage_bytes;
        mbar_arrive_expect_tx(&full[stage], tx_bytes);
        tma_load_3d(sb, &gy_map, 0, t0 / kIn, row, &full[stage]);
        const int xr = t0 / kIn + xr_rel;
        tma_load_3d(sb + g.gy_bytes, &x_map, 0, xr, row, &full[stage]);
        tma_load_3d(sb + g.gy_bytes + kMain * kIn * 4, &x_tail_map, 0, xr + kMain, row, &full[stage]);
    };
    if (tid == 0)
        for (int s = 0; s < NS && s < nunits; ++s) issue(s, s);

    // Finishes the tile node of work item u from the per-warp nodes (levels
    // above the warp), then folds it into the tree over work items: items
    // complete in flat order, so a binary counter pairs every node with its
    // left sibling exactly when the reference tree does.  One thread per tap.
    float root = 0.f;
    auto finish_unit = [&](int u) {
        if (tid < JT) {
            const int gj = tid / kJR, jj = tid % kJR;
            float v[WG];
#pragma unroll
            for (int w = 0; w < WG; ++w) v[w] = warp_node[u & 1][gj * WG + w][jj];
#pragma unroll
            for (int width = WG; width > 1; width >>= 1)
#pragma unroll
                for (int i = 0; i < width / 2; ++i) v[i] = __fadd_rn(v[2 * i], v[2 * i + 1]);
            float n = v[0];
            int level = 0;
            while ((u >> level) & 1) {
                n = __fadd_rn(pending[level][tid], n);
                ++level;
            }
            if (u == nunits - 1) root = n;  // nunits is a power of two: the last fold is the root
            else pending[level][tid] = n;
        }
    };

    for (int u = 0; u < nunits; ++u) {
        const int stage = u % NS;
        mbar_wait(&full[stage], static_cast<uint32_t>((u / NS) & 1));
        const unsigned char* gys = smem + stage * g.stage_bytes;
        const unsigned char* xs = gys + g.gy_bytes;
        const int t0 = (u % ntt) * kTT;
        float node[kJR];
        // every x tap of this lane's leaves inside the row -> no leaf masking
        // (only the lanes at a row's two ends take the masked path)
        const int lt = t0 + static_cast<int>(seg_t);
        const bool interior = lt + jbase >= 0 && lt + 8 * NB - 1 + jbase + kJR - 1 < L;
        if (interior)
            seg_tree<NB, S, false>(gys, xs, seg_t, 0, A, jg * kJR, t0, jbase, L, node);
        else
            seg_tree<NB, S, true>(gys, xs, seg_t, 0, A, jg * kJR, t0, jbase, L, node);

        // 5 lane levels.  Reduce-scatter over the 8 taps: after xor 1, 2, 4 the
        // lane keeps tap (lane & 7) summed over its 8-lane group.
        {
            float a[4];
            const bool hi1 = lane & 1;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float send = hi1 ? node[i] : node[i + 4];
                const float keep = hi1 ? node[i + 4] : node[i];
                a[i] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 1));
            }
            // a[i] = tap (hi1 ? i+4 : i)
            float b2[2];
            const bool hi2 = lane & 2;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const float send = hi2 ? a[i] : a[i + 2];
                const float keep = hi2 ? a[i + 2] : a[i];
                b2[i] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 2));
            }
            // b2[i] = tap (hi1?4:0) + (hi2?2:0) + i
            const bool hi4 = lane & 4;
            const float send = hi4 ? b2[0] : b2[1];
            const float keep = hi4 ? b2[1] : b2[0];
            float c = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 4));
            // c = tap (hi1?4:0) + (hi2?2:0) + (hi4?1:0), over lanes (lane & ~7)..+7
            c = __fadd_rn(c, __shfl_xor_sync(0xffffffffu, c, 8));
            c = __fadd_rn(c, __shfl_xor_sync(0xffffffffu, c, 16));
            if (lane < 8) {
                const int tap = ((lane & 1) ? 4 : 0) + ((lane & 2) ? 2 : 0) + ((lane & 4) ? 1 : 0);
                warp_node[u & 1][warp][tap] = c;
            }
        }
        __syncthreads();  // stage consumed; warp nodes of item u visible
        if (tid == 0 && u + NS < nunits) issue(stage, u + NS);
        finish_unit(u);   // reads parity u&1, next writer of it is item u+2 (after the next barrier)
    }
    if (tid < JT) {
        const int j = j0 + tid;
        if (j < K) part[(static_cast<int64_t>(grp) * H + h) * K + j] = root;
    }
}

// dk = perfect tree over the G (power of two) row-group partials, in order.
__global__ void dw_sum_groups_tree(const float* __restrict__ part, float* __restrict__ dk, int64_t HK, int G) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= HK) return;
    float v[64];
    for (int g = 0; g < G; ++g) v[g] = part[static_cast<int64_t>(g) * HK + i];
    for (int width = G; width > 1; width >>= 1)
        for (int n = 0; n < width / 2; ++n) v[n] = __fadd_rn(v[2 * n], v[2 * n + 1]);
    dk[i] = v[0];
}

template <int NJ>
ks_status launch(int s, const CUtensorMap& gm, const CUtensorMap& xm, const CUtensorMap& xt, float* part, int64_t B,
                 int64_t H, int64_t L, int64_t K, int G, int NJT, const PwGeom& g, int NS, cudaStream_t st) {
    const int smem = NS * g.stage_bytes + 64 + 1024;
    const unsigned blocks = static_cast<unsigned>(int64_t(G) * H * NJT);
    const int p = static_cast<int>(K / 2);
#define KS_PW_CASE(SV)                                                                                        \
    case SV: {                                                                                                \
        auto kern = dw_pairwise_tma<NJ, SV>;                                                                  \
        prepare_kernel(reinterpret_cast<const void*>(kern), kThreads, smem);                                \
        launch_kernel(kern, blocks, kThreads, smem, st, gm, xm, xt, part, static_cast<int>(B), static_cast<int>(H),      \
                                             static_cast<int>(L), static_cast<int>(K), p, G, NJT, g, NS);     \
        break;                                                                                                \
    }
    switch (s) {
        KS_PW_CASE(0)
        KS_PW_CASE(1)
        KS_PW_CASE(2)
        default:
        KS_PW_CASE(3)
    }
#undef KS_PW_CASE
    return check_launch();
}

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

struct PwPlan {
    bool ok = false;
    int nj = 1, njt = 1, G = 1;
};

PwPlan pw_plan(int64_t B, int64_t H, int64_t L, int64_t K) {
    PwPlan pl;
    if (!is_pow2(B) || !is_pow2(L) || L < kTT || L >= (int64_t(1) << 30) || B * H >= (int64_t(1) << 31)) return pl;
    while (pl.nj < 8 && pl.nj * kJR < K) pl.nj *= 2;
    pl.njt = static_cast<int>((K + pl.nj * kJR - 1) / (pl.nj * kJR));
    // row groups: power of two dividing B, <= 64 (stage-2 tree), enough CTAs,
    // and at most kMaxUnits work items per CTA
    int64_t G = 1;
    while (G < B && G < 64 && G * H * pl.njt < 8192) G *= 2;
    while (G < B && G < 64 && (B / G) * (L / kTT) > kMaxUnits) G *= 2;
    if ((B / G) * (L / kTT) > kMaxUnits) return pl;
    if (G * H * pl.njt >= (int64_t(1) << 31)) return pl;
    pl.G = static_cast<int>(G);
    pl.ok = true;
    return pl;
}

}  // namespace

size_t dw_pairwise_tma_workspace(int64_t B, int64_t H, int64_t L, int64_t K) {
    const PwPlan pl = pw_plan(B, H, L, K);
    return pl.ok ? size_t(pl.G) * H * K * sizeof(float) : 0;
}

// PAIRWISE dW through TMA; *handled = false when the shape is not a
// power-of-two B x L (>= 2048) problem or TMA is unavailable.
ks_status dw_pairwise_tma_f32(const float* gy, const float* x, float* dk, int64_t B, int64_t H, int64_t L, int64_t K,
                              void* ws, cudaStream_t st, bool* handled) {
    *handled = false;
    const PwPlan pl = pw_plan(B, H, L, K);
    if (!pl.ok || !ws) return KS_OK;
    PwGeom g;
    g.gy_bytes = kTT * 4;
    g.XT = (pl.nj * kJR + 40 + kIn - 1) / kIn;
    g.stage_bytes = (g.gy_bytes + (kMain + g.XT) * kIn * 4 + 1023) / 1024 * 1024;
    CUtensorMap gm, xm, xt;
    if (!encode_row_view(&gm, gy, B * H, L, kIn, kMain, 128)) return KS_OK;
    if (!encode_row_view(&xm, x, B * H, L, kIn, kMain, 128)) return KS_OK;
    if (!encode_row_view(&xt, x, B * H, L, kIn, g.XT, 128)) return KS_OK;
    const int NS = std::max(2, std::min(4, (64 * 1024) / g.stage_bytes));
    const int p = static_cast<int>(K / 2);
    const int s = (4 - p % 4) % 4;
    float* part = static_cast<float*>(ws);
    *handled = true;
    ks_status rc;
    switch (pl.nj) {
        case 1: rc = launch<1>(s, gm, xm, xt, part, B, H, L, K, pl.G, pl.njt, g, NS, st); break;
        case 2: rc = launch<2>(s, gm, xm, xt, part, B, H, L, K, pl.G, pl.njt, g, NS, st); break;
        case 4: rc = launch<4>(s, gm, xm, xt, part, B, H, L, K, pl.G, pl.njt, g, NS, st); break;
        default: rc = launch<8>(s, gm, xm, xt, part, B, H, L, K, pl.G, pl.njt, g, NS, st); break;
    }
    if (rc != KS_OK) return rc;
    const int64_t HK = H * K;
    launch_kernel(dw_sum_groups_tree, static_cast<unsigned>((HK + 255) / 256), 256, 0, st, part, dk, HK, pl.G);
    return check_launch();
}

}  // namespace ks
