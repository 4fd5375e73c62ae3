// ks_dist.cuh -- the communicator behind the opaque ks_comm of ks_dwconv1d.h
// (shared by dist.cu and peer.cu).
#pragma once

#include <nccl.h>

struct ks_comm {
    ncclComm_t nccl = nullptr;
    int world = 1;
    int rank = 0;
};
