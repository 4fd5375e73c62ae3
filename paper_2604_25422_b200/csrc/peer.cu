// peer.cu -- dW with the cross-GPU combine fused into the reduction kernel,
// over peer memory (one process per GPU: NVLink/NVSwitch; or several
// processes on one GPU, where the same IPC mappings are local).
//
// The dW path is a compute step (stage 1: per-CTA partials [G,H,K]) followed
// by a collective (the sum over ranks).  Instead of stage 2 + ncclAllReduce,
// every rank exposes its partial buffer to the others through CUDA IPC, and
// ONE kernel per rank
//   1. publishes this call's (G, H, K) in a header next to its partials and
//      signals "my partials are ready" by storing the call's epoch into a flag
//      slot of every peer (system-scope release),
//   2. waits until every peer's flag in its own buffer has reached the epoch
//      (system-scope acquire),
//   3. reads each rank's header -- so uneven shards, whose group counts
//      differ, combine correctly -- and then its partials straight from peer
//      memory, adding them in fixed (rank, group) order into dk.
// Every rank therefore computes the identical dk (bitwise), and the result
// does not depend on any collective algorithm.  With the global plan
// (B_total, see ks_dwconv1d.h) rank r's groups are the global groups
// r*G/N .. (r+1)*G/N - 1, so the (rank, group) order is the 1-GPU group order
// and dk equals the 1-GPU HIERARCHICAL result bit for bit.
//
// The handle exchange (cudaIpcGetMemHandle -> all-gather -> cudaIpcOpenMemHandle)
// uses the communicator's all-gather once, at setup.
#include <algorithm>
#include <cstring>
#include <vector>

#include "ks_common.cuh"
#include "ks_dist.cuh"

namespace ks {

ks_status dw_stage1_only(const float*, const float*, float*, int64_t, int64_t, int64_t, int64_t, int, int, int*,
                         cudaStream_t);
size_t dw_workspace_bytes(int64_t, int64_t, int64_t, int64_t, int, int64_t, int);
int dw_plan_groups(int64_t B, int64_t H, int64_t L, int64_t K);

constexpr int kMaxRanks = 16;

// Per-parity header a rank publishes with its partials.
struct PeerHdr {
    int64_t G, H, K, epoch;
};

struct PeerPtrs {
    float* part[kMaxRanks];          // every rank's partial buffer (two halves, by epoch parity)
    unsigned int* flags[kMaxRanks];  // every rank's flag array [kMaxRanks]
    PeerHdr* hdr[kMaxRanks];         // every rank's headers [2]
    int64_t half_floats[kMaxRanks];  // every rank's half-buffer size
};

// One kernel: publish, signal, wait, combine.  Partials are double-buffered by
// epoch parity: a rank can only reach epoch e+2 after every peer signalled
// e+1, which each peer does after finishing its epoch-e reads.  A peer that
// never arrives (a crashed rank) releases the wait after ~10 s; then, as for
// a peer whose (H, K) differ, dk becomes NaN and the host-mapped flag is set
// (the next call returns KS_ERR_TIMEOUT) instead of the device hanging.
__global__ void __launch_bounds__(256)
peer_combine(PeerPtrs pp, float* __restrict__ dk, int world, int rank, int64_t G, int64_t H, int64_t K,
             unsigned int epoch, int* failed) {
    __shared__ int64_t gs[kMaxRanks];
    __shared__ int bad;
    const int par = static_cast<int>(epoch & 1u);
    if (threadIdx.x == 0) {
        PeerHdr* mine = pp.hdr[rank] + par;
        mine->G = G;
        mine->H = H;
        mine->K = K;
        mine->epoch = epoch;
        __threadfence_system();  // this rank's partials (previous kernel) and header before the flag
        for (int r = 0; r < world; ++r) {
            unsigned int* f = pp.flags[r] + rank;
            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
        }
        int b = 0;
        for (int r = 0; r < world; ++r) {
            const unsigned int* f = pp.flags[rank] + r;
            unsigned int v;
            long long spins = 0;
            do {
                asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                if (static_cast<int>(v - epoch) >= 0) break;
                __nanosleep(100);
            } while (++spins < 100000000ll);
            if (static_cast<int>(v - epoch) < 0) {
                b = 1;
                gs[r] = 0;
                continue;
            }
            const PeerHdr* hp = pp.hdr[r] + par;
            const int64_t g = *reinterpret_cast<const volatile int64_t*>(&hp->G);
            const int64_t h = *reinterpret_cast<const volatile int64_t*>(&hp->H);
            const int64_t k = *reinterpret_cast<const volatile int64_t*>(&hp->K);
            if (h != H || k != K || g < 1 || g * H * K > pp.half_floats[r]) {
                b = 1;
                gs[r] = 0;
            } else {
                gs[r] = g;
            }
        }
        bad = b;
        if (b) *reinterpret_cast<volatile int*>(failed) = 1;
    }
    __syncthreads();
    const int64_t HK = H * K;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < HK;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (bad) {
            dk[i] = __int_as_float(0x7fc00000);
            continue;
        }
        // the order of dw_sum_groups (conv_dw.cu): s = first partial, then += in (rank, group) order
        float s = 0.f;
        bool first = true;
        for (int r = 0; r < world; ++r) {
            const float* p = pp.part[r] + par * pp.half_floats[r];
            for (int64_t g = 0; g < gs[r]; ++g) {
                const float v = p[g * HK + i];
                s = first ? v : s + v;
                first = false;
            }
        }
        dk[i] = s;
    }
}

}  // namespace ks

using namespace ks;

struct ks_peer {
    ks_comm* comm = nullptr;
    size_t half = 0;            // bytes of one partial buffer (two, by epoch parity)
    size_t bytes = 0;           // 2 * half
    void* local = nullptr;      // local allocation: [partials x2 | flags | headers x2]
    int* failed_host = nullptr; // mapped pinned host flag: a combine timed out / mismatched
    int* failed_dev = nullptr;
    PeerPtrs ptrs{};
    std::vector<void*> opened;  // peer mappings to close
    unsigned int epoch = 0;
};

namespace {

constexpr size_t kFlagBytes = kMaxRanks * sizeof(unsigned int);

struct Exchange {  // what every rank publishes once, at setup
    cudaIpcMemHandle_t handle;
    int64_t half_bytes;
};

void release(ks_peer* p) {
    for (void* q : p->opened) cudaIpcCloseMemHandle(q);
    if (p->local) cudaFree(p->local);
    if (p->failed_host) cudaFreeHost(p->failed_host);
    delete p;
}

}  // namespace

extern "C" {

ks_status ks_peer_create(ks_comm* comm, size_t partial_bytes, ks_peer** out) {
    if (!comm || !out) return KS_ERR_NULL;
    if (comm->world > kMaxRanks) return KS_ERR_SHARD;
    ks_peer* p = new ks_peer;
    p->comm = comm;
    p->half = (partial_bytes + 255) / 256 * 256;
    p->bytes = 2 * p->half;
    const size_t total = p->bytes + kFlagBytes + 2 * sizeof(PeerHdr) + 256;
    ks_status s = cuda_status(cudaMalloc(&p->local, total));
    if (s == KS_OK) s = cuda_status(cudaMemset(p->local, 0, total));
    if (s == KS_OK) s = cuda_status(cudaHostAlloc(reinterpret_cast<void**>(&p->failed_host), sizeof(int), cudaHostAllocMapped));
    if (s == KS_OK) {
        *p->failed_host = 0;
        s = cuda_status(cudaHostGetDevicePointer(reinterpret_cast<void**>(&p->failed_dev), p->failed_host, 0));
    }
    if (s != KS_OK) {
        release(p);
        return s;
    }
    const int world = comm->world, rank = comm->rank;
    Exchange mine{};
    mine.half_bytes = static_cast<int64_t>(p->half);
    if (world > 1) s = cuda_status(cudaIpcGetMemHandle(&mine.handle, p->local));
    std::vector<Exchange> all(world);
    if (s == KS_OK) s = comm_allgather_host(comm, &mine, all.data(), sizeof(Exchange));
    for (int r = 0; r < world && s == KS_OK; ++r) {
        void* base = p->local;
        if (r != rank) {
            s = cuda_status(cudaIpcOpenMemHandle(&base, all[r].handle, cudaIpcMemLazyEnablePeerAccess));
            if (s == KS_OK) p->opened.push_back(base);
        }
        const size_t half_r = static_cast<size_t>(all[r].half_bytes);
        p->ptrs.part[r] = static_cast<float*>(base);
        p->ptrs.flags[r] = reinterpret_cast<unsigned int*>(static_cast<char*>(base) + 2 * half_r);
        p->ptrs.hdr[r] = reinterpret_cast<PeerHdr*>(static_cast<char*>(base) + 2 * half_r + kFlagBytes);
        p->ptrs.half_floats[r] = static_cast<int64_t>(half_r / sizeof(float));
    }
    if (s != KS_OK) {
        release(p);
        return s;
    }
    *out = p;
    return KS_OK;
}

ks_status ks_peer_destroy(ks_peer* p) {
    if (!p) return KS_OK;
    const ks_status s = cuda_status(cudaDeviceSynchronize());  // no combine may still read our buffer
    release(p);
    return s;
}

ks_status ks_dwconv1d_dw_f32_peer(const float* gy, const float* x, float* dk, int64_t B, int64_t H, int64_t L,
                                  int64_t K, int64_t B_total, int mode, ks_peer* p, void* stream) {
    if (!gy || !x || !dk || !p) return KS_ERR_NULL;
    if (B < 1) return KS_ERR_DIM_B;
    if (H < 1) return KS_ERR_DIM_H;
    if (L < 1) return KS_ERR_DIM_L;
    if (K < 1) return KS_ERR_DIM_K;
    if (B_total < 0) return KS_ERR_SHARD;
    if (mode != KS_MULADD_SEPARATE && mode != KS_MULADD_FUSED) return KS_ERR_BAD_MODE;
    if (*reinterpret_cast<volatile int*>(p->failed_host)) {
        set_last_error("a previous peer combine timed out or met a mismatched rank");
        return KS_ERR_TIMEOUT;
    }
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int world = p->comm->world, rank = p->comm->rank;
    // the global plan when the shards fall on its row-group boundaries
    int G_req = 0;
    if (B_total > 0 && B_total * H < (int64_t(1) << 31)) {
        const int Gt = dw_plan_groups(B_total, H, L, K);
        int64_t b0 = 0, nb = 0;
        if (Gt % world == 0 && B_total % Gt == 0 && ks_shard_rows(B_total, world, rank, &b0, &nb) == KS_OK &&
            nb == B && dw_plan_groups(B_total, H, L, K) == Gt)
            G_req = Gt / world;
    }
    const size_t need = G_req > 0 ? size_t(G_req) * H * K * sizeof(float)
                                  : dw_workspace_bytes(B, H, L, K, KS_DW_HIERARCHICAL, 0, 4);
    if (need > p->half) return KS_ERR_WORKSPACE;
    const unsigned int epoch = ++p->epoch;
    float* part = reinterpret_cast<float*>(static_cast<char*>(p->local) + (epoch & 1u) * p->half);
    int G = 0;
    ks_status s = dw_stage1_only(gy, x, part, B, H, L, K, mode, G_req, &G, st);
    if (s != KS_OK) return s;
    const int64_t HK = H * K;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((HK + 255) / 256, int64_t(num_sms()) * 4));
    launch_kernel(peer_combine, blocks, 256, 0, st, p->ptrs, dk, world, rank, G, H, K, epoch, p->failed_dev);
    return check_launch();
}

// 1 if a peer_combine ever gave up waiting for a peer or met a mismatched one
// (mapped host memory: no device synchronisation).
ks_status ks_peer_timed_out(ks_peer* p, int* flag) {
    if (!p || !flag) return KS_ERR_NULL;
    *flag = *reinterpret_cast<volatile int*>(p->failed_host);
    return KS_OK;
}

}  // extern "C"
