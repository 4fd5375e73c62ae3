// ks_dist.cuh -- the communicator behind the opaque ks_comm of ks_dwconv1d.h
// (shared by dist.cu and peer.cu): an NCCL communicator, or a caller-supplied
// host all-gather (ks_comm_init_host) that only ever moves bytes.
#pragma once

#include <nccl.h>

#include "ks_dwconv1d.h"

struct ks_comm {
    ncclComm_t nccl = nullptr;
    ks_allgather_fn host_allgather = nullptr;  // set for a host communicator
    void* host_ctx = nullptr;
    int world = 1;
    int rank = 0;
};

namespace ks {
// All-gather of `bytes` HOST bytes per rank into recv[world * bytes] (rank
// order) over either transport; synchronous.
ks_status comm_allgather_host(ks_comm* c, const void* send, void* recv, size_t bytes);
}  // namespace ks
