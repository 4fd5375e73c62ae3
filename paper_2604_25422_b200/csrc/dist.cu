// dist.cu -- batch sharding and the dW combine across GPUs (one process per
// GPU).  The reference is single-process CPU code with no collectives; batch
// sharding is the natural partition of this operator (rows (b,.,.) are
// independent for y and dX, and dW is a sum over b), so the only exchange is
// one reduction of the H*K weight gradient.
//
//  * ks_dwconv1d_dw_allreduce_f32: one ncclAllReduce(sum) over NVLink/NVSwitch.
//  * ks_dwconv1d_dw_allgather_sum_f32: ncclAllGather of the rank partials, then
//    a fixed pairwise tree in rank order on every rank, so the result does not
//    depend on NCCL's algorithm/protocol choice and is bitwise identical on all
//    ranks for a given world size.
//  * ks_comm_init_host: the same combines over a caller-supplied host
//    all-gather (MPI, torch.distributed gloo, ...): the bytes cross the host,
//    the sums stay on the device.  Ranks may share a GPU, which NCCL refuses,
//    so this is also how the multi-rank paths are exercised on one B200.
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "ks_common.cuh"
#include "ks_dist.cuh"

namespace ks {

static ks_status nccl_status(ncclResult_t r) {
    if (r == ncclSuccess) return KS_OK;
    set_last_error(ncclGetErrorString(r));
    return KS_ERR_NCCL;
}

// out[i] = pairwise tree over the `world` rank slices of gather[world][n], in
// rank order (midpoint split, like the reference's reduce_pairwise).
__global__ void rank_tree_sum(const float* __restrict__ gather, float* __restrict__ out,
                              int64_t n, int world) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    float v[64];
    int w = world < 64 ? world : 64;
    for (int r = 0; r < w; ++r) v[r] = gather[static_cast<int64_t>(r) * n + i];
    // midpoint-split recursion, evaluated with an explicit stack
    struct Frame { int lo, hi, state; };
    Frame st[16];
    float vals[16];
    int sp = 0, vp = 0;
    st[sp++] = {0, w, 0};
    while (sp) {
        Frame& f = st[sp - 1];
        if (f.hi - f.lo == 1) {
            vals[vp++] = v[f.lo];
            --sp;
            continue;
        }
        const int mid = f.lo + (f.hi - f.lo) / 2;
        if (f.state == 0) {
            f.state = 1;
            st[sp++] = {f.lo, mid, 0};
        } else if (f.state == 1) {
            f.state = 2;
            st[sp++] = {mid, f.hi, 0};
        } else {
            const float r = vals[--vp];
            const float l = vals[--vp];
            vals[vp++] = l + r;
            --sp;
        }
    }
    out[i] = vals[0];
}

ks_status comm_allgather_host(ks_comm* c, const void* send, void* recv, size_t bytes) {
    if (c->world == 1) {
        memcpy(recv, send, bytes);
        return KS_OK;
    }
    if (c->host_allgather) {
        if (c->host_allgather(send, recv, bytes, c->host_ctx) != 0) {
            set_last_error("host all-gather callback failed");
            return KS_ERR_NCCL;
        }
        return KS_OK;
    }
    // NCCL moves device memory: stage through a small device buffer
    void* d = nullptr;
    ks_status s = cuda_status(cudaMalloc(&d, bytes * c->world));
    if (s == KS_OK)
        s = cuda_status(cudaMemcpy(static_cast<char*>(d) + c->rank * bytes, send, bytes, cudaMemcpyHostToDevice));
    if (s == KS_OK)
        s = nccl_status(ncclAllGather(static_cast<char*>(d) + c->rank * bytes, d, bytes, ncclUint8, c->nccl, nullptr));
    if (s == KS_OK) s = cuda_status(cudaStreamSynchronize(nullptr));
    if (s == KS_OK) s = cuda_status(cudaMemcpy(recv, d, bytes * c->world, cudaMemcpyDeviceToHost));
    if (d) cudaFree(d);
    return s;
}

// Host-communicator all-gather of a device array dk[n] into the device array
// gather[world, n]: D2H after the stream's prior work, the caller's exchange,
// H2D back on the stream.
static ks_status host_gather_device(ks_comm* c, const float* dk, float* gather, size_t n, cudaStream_t st) {
    std::vector<float> mine(n), all(n * c->world);
    ks_status s = cuda_status(cudaMemcpyAsync(mine.data(), dk, n * sizeof(float), cudaMemcpyDeviceToHost, st));
    if (s == KS_OK) s = cuda_status(cudaStreamSynchronize(st));
    if (s == KS_OK) s = comm_allgather_host(c, mine.data(), all.data(), n * sizeof(float));
    if (s == KS_OK)
        s = cuda_status(cudaMemcpyAsync(gather, all.data(), all.size() * sizeof(float), cudaMemcpyHostToDevice, st));
    if (s == KS_OK) s = cuda_status(cudaStreamSynchronize(st));  // `all` is pageable and goes out of scope
    return s;
}

ks_status dw_chunk_partials_f32(const float*, const float*, float*, int64_t, int64_t, int64_t, int64_t, int64_t,
                                int64_t, int, cudaStream_t);
ks_status dw_chunk_total_ranks_f32(const float*, float*, int64_t, int, int, const int*, cudaStream_t);

}  // namespace ks

using namespace ks;

extern "C" {

ks_status ks_dwconv1d_dw_chunked_sharded_f32(const float* gy, const float* x, float* dk, int64_t B_local,
                                             int64_t b0, int64_t B_total, int64_t H, int64_t L, int64_t K,
                                             int64_t chunk, int mode, ks_comm* comm, void* stream) {
    if (!dk || !comm || (B_local > 0 && (!gy || !x))) return KS_ERR_NULL;
    if (B_total < 1 || B_local < 0 || b0 < 0 || b0 + B_local > B_total) return KS_ERR_DIM_B;
    if (H < 1) return KS_ERR_DIM_H;
    if (L < 1) return KS_ERR_DIM_L;
    if (K < 1) return KS_ERR_DIM_K;
    if (chunk < 1) return KS_ERR_BAD_CHUNK;
    if (mode != KS_MULADD_SEPARATE && mode != KS_MULADD_FUSED) return KS_ERR_BAD_MODE;
    if (comm->world > 64) return KS_ERR_SHARD;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int world = comm->world;
    // every rank's rows: they must tile [0, B_total) in rank order, and no
    // chunk may straddle two ranks (each chunk's chain is computed whole)
    // every rank's rows, and the shape / chunk / mode every rank must agree on
    // (a disagreement would make the gathers mismatch)
    constexpr int kRec = 8;
    int64_t mine[kRec] = {b0, B_local, B_total, H, L, K, chunk, mode};
    std::vector<int64_t> rec(kRec * static_cast<size_t>(world));
    ks_status s = comm_allgather_host(comm, mine, rec.data(), sizeof(mine));
    if (s != KS_OK) return s;
    std::vector<int64_t> all(2 * static_cast<size_t>(world));
    for (int r = 0; r < world; ++r) {
        for (int f = 2; f < kRec; ++f)
            if (rec[kRec * r + f] != mine[f]) {
                set_last_error("sharded CHUNKED dW: ranks disagree on (B_total, H, L, K, chunk, mode)");
                return KS_ERR_SHARD;
            }
        all[2 * r] = rec[kRec * r];
        all[2 * r + 1] = rec[kRec * r + 1];
    }
    const int64_t n_flat = B_total * L;
    const int64_t c_eff = std::min(chunk, n_flat);  // chunk >= B*L: one chunk (SEQUENTIAL)
    std::vector<int> counts(world);
    int64_t next = 0, ncmax = 0;
    for (int r = 0; r < world; ++r) {
        const int64_t rb0 = all[2 * r], rnb = all[2 * r + 1];
        if (rb0 != next) {
            set_last_error("sharded CHUNKED dW: ranks' rows must tile [0, B) in rank order");
            return KS_ERR_SHARD;
        }
        const int64_t f0 = rb0 * L, f1 = (rb0 + rnb) * L;
        if (rnb > 0 && (f0 % c_eff != 0 || (f1 % c_eff != 0 && f1 != n_flat))) {
            set_last_error("sharded CHUNKED dW: a chunk straddles two ranks (shard rows * L must be multiples of chunk)");
            return KS_ERR_SHARD;
        }
        const int64_t nc = rnb > 0 ? (f1 - f0 + c_eff - 1) / c_eff : 0;
        if (nc >= (int64_t(1) << 30)) return KS_ERR_SHARD;
        counts[r] = static_cast<int>(nc);
        ncmax = std::max(ncmax, nc);
        next = rb0 + rnb;
    }
    if (next != B_total) {
        set_last_error("sharded CHUNKED dW: ranks' rows must cover [0, B)");
        return KS_ERR_SHARD;
    }
    const int64_t HK = H * K;
    const size_t n = static_cast<size_t>(std::max<int64_t>(1, ncmax) * HK);
    if (double(n) * world * sizeof(float) > double(size_t(4) << 30)) {  // the gathered partials of every rank
        set_last_error("sharded CHUNKED dW: more than 4 GiB of chunk partials to gather (use a larger chunk)");
        return KS_ERR_SHARD;
    }
    float *part = nullptr, *gather = nullptr;
    s = cuda_status(cudaMallocAsync(reinterpret_cast<void**>(&part), n * sizeof(float), st));
    if (s == KS_OK) s = cuda_status(cudaMallocAsync(reinterpret_cast<void**>(&gather), n * world * sizeof(float), st));
    if (s == KS_OK) s = cuda_status(cudaMemsetAsync(part, 0, n * sizeof(float), st));
    if (s == KS_OK)
        s = dw_chunk_partials_f32(gy, x, part, B_local, H, L, K, c_eff, counts[comm->rank], mode, st);
    if (s == KS_OK)
        s = comm->host_allgather || world == 1
                ? (world == 1 ? cuda_status(cudaMemcpyAsync(gather, part, n * sizeof(float), cudaMemcpyDeviceToDevice, st))
                              : host_gather_device(comm, part, gather, n, st))
                : nccl_status(ncclAllGather(part, gather, n, ncclFloat, comm->nccl, st));
    if (s == KS_OK)
        s = dw_chunk_total_ranks_f32(gather, dk, HK, world, static_cast<int>(std::max<int64_t>(1, ncmax)),
                                     counts.data(), st);
    if (gather) cudaFreeAsync(gather, st);
    if (part) cudaFreeAsync(part, st);
    return s;
}


ks_status ks_shard_rows(int64_t B, int world, int rank, int64_t* b0, int64_t* nb) {
    if (!b0 || !nb) return KS_ERR_NULL;
    if (B < 1) return KS_ERR_DIM_B;
    if (world < 1 || rank < 0 || rank >= world || world > B) return KS_ERR_SHARD;
    const int64_t lo = B * rank / world;
    const int64_t hi = B * (rank + 1) / world;
    *b0 = lo;
    *nb = hi - lo;
    return KS_OK;
}

ks_status ks_comm_unique_id(void* id128) {
    if (!id128) return KS_ERR_NULL;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    return nccl_status(ncclGetUniqueId(static_cast<ncclUniqueId*>(id128)));
}

ks_status ks_comm_init(ks_comm** comm, const void* id128, int world, int rank) {
    if (!comm || !id128) return KS_ERR_NULL;
    if (world < 1 || rank < 0 || rank >= world) return KS_ERR_SHARD;
    ks_comm* c = new ks_comm;
    c->world = world;
    c->rank = rank;
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    const ks_status s = nccl_status(ncclCommInitRank(&c->nccl, world, id, rank));
    if (s != KS_OK) {
        delete c;
        return s;
    }
    *comm = c;
    return KS_OK;
}

ks_status ks_comm_init_host(ks_comm** comm, int world, int rank, ks_allgather_fn allgather, void* ctx) {
    if (!comm || !allgather) return KS_ERR_NULL;
    if (world < 1 || rank < 0 || rank >= world) return KS_ERR_SHARD;
    ks_comm* c = new ks_comm;
    c->world = world;
    c->rank = rank;
    c->host_allgather = allgather;
    c->host_ctx = ctx;
    *comm = c;
    return KS_OK;
}

ks_status ks_rank_tree_sum_f32(const float* gather, float* out, int64_t n, int world, void* stream) {
    if (!gather || !out) return KS_ERR_NULL;
    if (world < 1 || world > 64) return KS_ERR_SHARD;
    if (n < 0) return KS_ERR_DIM_H;
    if (n == 0) return KS_OK;
    launch_kernel(rank_tree_sum, static_cast<unsigned>((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream), 
        gather, out, n, world);
    return check_launch();
}

ks_status ks_comm_allgather_host(ks_comm* comm, const void* send, void* recv, size_t bytes) {
    if (!comm || (bytes && (!send || !recv))) return KS_ERR_NULL;
    if (bytes == 0) return KS_OK;
    return comm_allgather_host(comm, send, recv, bytes);
}

ks_status ks_comm_destroy(ks_comm* comm) {
    if (!comm) return KS_OK;
    ks_status s = KS_OK;
    if (comm->nccl) s = nccl_status(ncclCommDestroy(comm->nccl));  // host communicators own nothing
    delete comm;
    return s;
}

ks_status ks_dwconv1d_dw_allreduce_f32(float* dk, int64_t H, int64_t K, ks_comm* comm,
                                       void* stream) {
    if (!dk || !comm) return KS_ERR_NULL;
    if (H < 1) return KS_ERR_DIM_H;
    if (K < 1) return KS_ERR_DIM_K;
    if (comm->host_allgather) {  // deterministic: gather every rank's dk, fixed tree on the device
        if (comm->world == 1) return KS_OK;
        float* gather = nullptr;
        const size_t n = static_cast<size_t>(H * K);
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        ks_status s = cuda_status(cudaMallocAsync(reinterpret_cast<void**>(&gather), n * comm->world * sizeof(float), st));
        if (s == KS_OK) s = ks_dwconv1d_dw_allgather_sum_f32(dk, gather, H, K, comm, stream);
        if (gather) cudaFreeAsync(gather, st);
        return s;
    }
    // (a 1-rank communicator still goes through NCCL: same code path at every N)
    return nccl_status(ncclAllReduce(dk, dk, static_cast<size_t>(H * K), ncclFloat, ncclSum,
                                     comm->nccl, static_cast<cudaStream_t>(stream)));
}

ks_status ks_dwconv1d_dw_allgather_sum_f32(float* dk, float* gather, int64_t H, int64_t K,
                                           ks_comm* comm, void* stream) {
    if (!dk || !gather || !comm) return KS_ERR_NULL;
    if (H < 1) return KS_ERR_DIM_H;
    if (K < 1) return KS_ERR_DIM_K;
    if (comm->world > 64) return KS_ERR_SHARD;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t n = static_cast<size_t>(H * K);
    ks_status s = comm->host_allgather ? host_gather_device(comm, dk, gather, n, st)
                                       : nccl_status(ncclAllGather(dk, gather, n, ncclFloat, comm->nccl, st));
    if (s != KS_OK) return s;
    return ks_rank_tree_sum_f32(gather, dk, static_cast<int64_t>(n), comm->world, stream);
}

}  // extern "C"
