// peer.cu -- dW with the cross-GPU combine fused into the reduction kernel,
// over NVLink peer memory (one process per GPU).
//
// The dW path is a compute step (stage 1: per-CTA partials [G,H,K]) followed
// by a collective (the sum over ranks).  Instead of stage 2 + ncclAllReduce,
// every rank exposes its partial buffer to the others through CUDA IPC
// (mapped over NVLink/NVSwitch), and ONE kernel per rank
//   1. signals "my partials are ready" by storing the call's epoch into a flag
//      slot of every peer (system-scope release),
//   2. waits until every peer's flag in its own buffer has reached the epoch
//      (system-scope acquire),
//   3. reads the partials of all ranks straight from peer memory and adds them
//      in fixed (rank, group) order into dk.
// Every rank therefore computes the identical dk (bitwise), and the result
// does not depend on any collective algorithm choice.  The handle exchange
// (cudaIpcGetMemHandle -> all-gather -> cudaIpcOpenMemHandle) uses the NCCL
// communicator once, at setup.
#include <nccl.h>

#include <cstring>
#include <vector>

#include "ks_common.cuh"
#include "ks_dist.cuh"

namespace ks {

ks_status dw_f32(const float*, const float*, float*, int64_t, int64_t, int64_t, int64_t, int, int64_t, int, void*,
                 cudaStream_t);
ks_status dw_stage1_only(const float*, const float*, float*, int64_t, int64_t, int64_t, int64_t, int, void*, int*,
                         cudaStream_t);
size_t dw_workspace_bytes(int64_t, int64_t, int64_t, int64_t, int, int64_t, int);
void set_last_error(const char*);

constexpr int kMaxRanks = 16;

struct PeerPtrs {
    float* part[kMaxRanks];              // every rank's partial buffer
    unsigned int* flags[kMaxRanks];      // every rank's flag array [kMaxRanks]
};

// One kernel: signal, wait, combine.  Partials are double-buffered by epoch
// parity: a rank can only reach epoch e+2 after every peer signalled e+1,
// which each peer does after finishing its epoch-e reads.  A peer that never
// arrives (a crashed rank) releases the wait after ~10 s with *timed_out set
// instead of hanging the device.
__global__ void __launch_bounds__(256)
peer_combine(PeerPtrs pp, float* __restrict__ dk, int world, int rank, int G, int64_t HK, size_t half_floats,
             unsigned int epoch, int* timed_out) {
    if (threadIdx.x == 0) {
        __threadfence_system();  // this rank's partials (previous kernel) before the flag
        for (int r = 0; r < world; ++r) {
            unsigned int* f = pp.flags[r] + rank;
            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
        }
        for (int r = 0; r < world; ++r) {
            const unsigned int* f = pp.flags[rank] + r;
            unsigned int v;
            long long spins = 0;
            do {
                asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                if (static_cast<int>(v - epoch) >= 0) break;
                __nanosleep(100);
            } while (++spins < 100000000ll);
            if (static_cast<int>(v - epoch) < 0) *timed_out = 1;
        }
    }
    __syncthreads();
    const size_t off = (epoch & 1u) * half_floats;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < HK;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float s = 0.f;
        for (int r = 0; r < world; ++r) {
            const float* p = pp.part[r] + off;
            for (int g = 0; g < G; ++g) s += p[static_cast<int64_t>(g) * HK + i];
        }
        dk[i] = s;
    }
}

}  // namespace ks

using namespace ks;

struct ks_peer {
    ks_comm* comm = nullptr;
    size_t half = 0;           // bytes of one partial buffer (two, by epoch parity)
    size_t bytes = 0;          // 2 * half
    void* local = nullptr;     // local allocation: [partials x2 | flags | timeout flag]
    PeerPtrs ptrs{};
    std::vector<void*> opened; // peer mappings to close
    unsigned int epoch = 0;
};

extern "C" {

ks_status ks_peer_create(ks_comm* comm, size_t partial_bytes, ks_peer** out) {
    if (!comm || !out) return KS_ERR_NULL;
    if (comm->world > kMaxRanks) return KS_ERR_SHARD;
    ks_peer* p = new ks_peer;
    p->comm = comm;
    p->half = (partial_bytes + 255) / 256 * 256;
    p->bytes = 2 * p->half;
    const size_t total = p->bytes + kMaxRanks * sizeof(unsigned int) + 256;
    ks_status s = cuda_status(cudaMalloc(&p->local, total));
    if (s == KS_OK) s = cuda_status(cudaMemset(p->local, 0, total));
    if (s != KS_OK) {
        delete p;
        return s;
    }
    const int world = comm->world, rank = comm->rank;
    if (world == 1) {
        p->ptrs.part[0] = static_cast<float*>(p->local);
        p->ptrs.flags[0] = reinterpret_cast<unsigned int*>(static_cast<char*>(p->local) + p->bytes);
        *out = p;
        return KS_OK;
    }
    // exchange IPC handles with one all-gather over the NCCL communicator
    cudaIpcMemHandle_t mine;
    s = cuda_status(cudaIpcGetMemHandle(&mine, p->local));
    void* dbuf = nullptr;
    if (s == KS_OK) s = cuda_status(cudaMalloc(&dbuf, sizeof(cudaIpcMemHandle_t) * world));
    if (s == KS_OK)
        s = cuda_status(cudaMemcpy(static_cast<char*>(dbuf) + rank * sizeof(mine), &mine, sizeof(mine),
                                   cudaMemcpyHostToDevice));
    if (s == KS_OK) {
        const ncclResult_t r = ncclAllGather(static_cast<char*>(dbuf) + rank * sizeof(mine), dbuf, sizeof(mine),
                                             ncclUint8, comm->nccl, nullptr);
        if (r != ncclSuccess) {
            set_last_error(ncclGetErrorString(r));
            s = KS_ERR_NCCL;
        }
    }
    std::vector<cudaIpcMemHandle_t> all(world);
    if (s == KS_OK) s = cuda_status(cudaStreamSynchronize(nullptr));
    if (s == KS_OK) s = cuda_status(cudaMemcpy(all.data(), dbuf, sizeof(mine) * world, cudaMemcpyDeviceToHost));
    if (dbuf) cudaFree(dbuf);
    for (int r = 0; r < world && s == KS_OK; ++r) {
        void* base = p->local;
        if (r != rank) {
            s = cuda_status(cudaIpcOpenMemHandle(&base, all[r], cudaIpcMemLazyEnablePeerAccess));
            if (s == KS_OK) p->opened.push_back(base);
        }
        p->ptrs.part[r] = static_cast<float*>(base);
        p->ptrs.flags[r] = reinterpret_cast<unsigned int*>(static_cast<char*>(base) + p->bytes);
    }
    if (s != KS_OK) {
        for (void* q : p->opened) cudaIpcCloseMemHandle(q);
        cudaFree(p->local);
        delete p;
        return s;
    }
    *out = p;
    return KS_OK;
}

ks_status ks_peer_destroy(ks_peer* p) {
    if (!p) return KS_OK;
    for (void* q : p->opened) cudaIpcCloseMemHandle(q);
    ks_status s = cuda_status(cudaFree(p->local));
    delete p;
    return s;
}

ks_status ks_dwconv1d_dw_f32_peer(const float* gy, const float* x, float* dk, int64_t B, int64_t H, int64_t L,
                                  int64_t K, int mode, ks_peer* p, void* stream) {
    if (!gy || !x || !dk || !p) return KS_ERR_NULL;
    if (B < 1) return KS_ERR_DIM_B;
    if (H < 1) return KS_ERR_DIM_H;
    if (L < 1) return KS_ERR_DIM_L;
    if (K < 1) return KS_ERR_DIM_K;
    if (mode != KS_MULADD_SEPARATE && mode != KS_MULADD_FUSED) return KS_ERR_BAD_MODE;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t need = dw_workspace_bytes(B, H, L, K, KS_DW_HIERARCHICAL, 0, 4);
    if (need > p->half) return KS_ERR_WORKSPACE;
    const unsigned int epoch = ++p->epoch;
    float* part = reinterpret_cast<float*>(static_cast<char*>(p->local) + (epoch & 1u) * p->half);
    int G = 0;
    ks_status s = dw_stage1_only(gy, x, part, B, H, L, K, mode, nullptr, &G, st);
    if (s != KS_OK) return s;
    const int64_t HK = H * K;
    int* timed_out = reinterpret_cast<int*>(static_cast<char*>(p->local) + p->bytes + kMaxRanks * sizeof(unsigned));
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((HK + 255) / 256, int64_t(num_sms()) * 4));
    peer_combine<<<blocks, 256, 0, st>>>(p->ptrs, dk, p->comm->world, p->comm->rank, G, HK, p->half / 4, epoch,
                                         timed_out);
    return check_launch();
}

// 1 if a peer_combine ever gave up waiting for a peer (synchronous read).
ks_status ks_peer_timed_out(ks_peer* p, int* flag) {
    if (!p || !flag) return KS_ERR_NULL;
    const int* d = reinterpret_cast<const int*>(static_cast<const char*>(p->local) + p->bytes +
                                                kMaxRanks * sizeof(unsigned));
    return cuda_status(cudaMemcpy(flag, d, sizeof(int), cudaMemcpyDeviceToHost));
}

}  // extern "C"
