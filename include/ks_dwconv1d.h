/*
 * ks_dwconv1d.h -- C ABI of the B200-native S4ConvD depthwise conv1d operator.
 *
 * This is the drop-in boundary for the reference's hot path, the three
 * operator entry points of kernelscope::conv
 * (/root/reference/proj/include/kernelscope/conv_core.hpp:49-69):
 *
 *   reference (C++, host value types)             C ABI here (device pointers)
 *   conv::forward(x,k,shape,mode)        :49-52   ks_dwconv1d_fwd_f32 / _f64
 *   conv::backward_input(gy,k,shape,mode):56-59   ks_dwconv1d_dx_f32  / _f64
 *   conv::backward_weight(gy,x,shape,
 *                         scheme,mode)   :64-69   ks_dwconv1d_dw_f32  / _f64
 *
 * plus host-buffer twins (*_host) that take plain host pointers, which is the
 * shape of the reference's value-type API, and the batch-sharded multi-GPU
 * combine for dW.  The C++ drop-in (include/kernelscope/conv_core.hpp, same
 * names and signatures as the reference) is a thin layer over these calls.
 *
 * Conventions
 *  - Layout: x, y, gy, dx are row-major [B,H,L] (element (b,h,t) at
 *    (b*H+h)*L+t, reference tensor.hpp:15-32); k and dk are row-major [H,K]
 *    (tensor.hpp:45-69).  Padding p = K/2 (shape.hpp:16); dX uses q = K-1-p
 *    (src/conv_core.cpp:56).
 *  - Device entry points take device pointers, are asynchronous on `stream`
 *    (a cudaStream_t passed as void*, NULL = legacy default stream) and never
 *    synchronise.  No exceptions cross the boundary; every call returns a
 *    ks_status.
 *  - Determinism: for fixed (shape, mode, scheme) and default tuning options
 *    (ks_set_option) results are bitwise reproducible run to run, whatever the
 *    alignment of the caller's pointers and whichever thread calls; there are
 *    no floating-point atomics anywhere.
 *  - Rounding: y and dX accumulate taps in ascending j from +0, exactly like
 *    the reference loops (src/conv_core.cpp:37-40, 66-69), so they are
 *    bit-identical to the reference in both MulAddModes for finite inputs.
 *    (The kernels multiply the zero padding where the reference skips a tap:
 *    with an Inf or NaN among the inputs, outputs within K of it may be NaN
 *    where the reference's are not; every other output keeps its bits.)  dW schemes
 *    SEQUENTIAL / PAIRWISE / CHUNKED reproduce the reference association order
 *    bit-for-bit (src/conv_core.cpp:98-146); HIERARCHICAL is this library's
 *    fast deterministic order (parity within a stated tolerance).
 */
#ifndef KS_DWCONV1D_H
#define KS_DWCONV1D_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KS_DWCONV1D_ABI_VERSION 2

typedef enum ks_status {
    KS_OK = 0,
    KS_ERR_DIM_B = 1,      /* B < 1                         (shape.hpp:27)          */
    KS_ERR_DIM_H = 2,      /* H < 1                         (shape.hpp:28)          */
    KS_ERR_DIM_L = 3,      /* L < 1                         (shape.hpp:29)          */
    KS_ERR_DIM_K = 4,      /* K < 1                         (shape.hpp:30)          */
    KS_ERR_BAD_CHUNK = 5,  /* chunked scheme, chunk < 1     (src/conv_core.cpp:154) */
    KS_ERR_BAD_MODE = 6,   /* mode not a ks_muladd                                  */
    KS_ERR_BAD_SCHEME = 7, /* scheme not a ks_dw_scheme                             */
    KS_ERR_NULL = 8,       /* a required pointer is NULL                             */
    KS_ERR_WORKSPACE = 9,  /* ws_bytes smaller than ks_dwconv1d_dw_workspace_bytes   */
    KS_ERR_NO_DEVICE = 10, /* no CUDA device / driver                                */
    KS_ERR_CUDA = 11,      /* CUDA runtime error (ks_last_error_string for text)     */
    KS_ERR_NCCL = 12,      /* NCCL error                                             */
    KS_ERR_SHARD = 13,     /* bad rank / world size / shard geometry                 */
    KS_ERR_BAD_OPTION = 14,/* unknown tuning option name or value out of range       */
    KS_ERR_TIMEOUT = 15    /* a peer combine gave up waiting for a rank (dk is NaN)  */
} ks_status;

/* MulAddMode (conv_core.hpp:45): SEPARATE = acc + a*b with two roundings (the
 * reference default), FUSED = fma(a,b,acc). */
typedef enum ks_muladd { KS_MULADD_SEPARATE = 0, KS_MULADD_FUSED = 1 } ks_muladd;

/* dW association order.  The first three are the reference's SumScheme
 * (conv_core.hpp:14-18) and are reproduced bit-for-bit; HIERARCHICAL is the
 * fast path (in-register FMA partials over t, shared-memory tree, fixed-order
 * cross-block pass; no atomics). */
typedef enum ks_dw_scheme {
    KS_DW_SEQUENTIAL = 0,
    KS_DW_PAIRWISE = 1,
    KS_DW_CHUNKED = 2,
    KS_DW_HIERARCHICAL = 3
} ks_dw_scheme;

const char* ks_status_string(ks_status s);
/* Text of the last CUDA/NCCL error seen by this thread ("" if none). */
const char* ks_last_error_string(void);
int ks_abi_version(void);

/* ---- device-pointer entry points (asynchronous on `stream`) -------------- */

ks_status ks_dwconv1d_fwd_f32(const float* x, const float* k, float* y, int64_t B, int64_t H,
                              int64_t L, int64_t K, int mode, void* stream);
ks_status ks_dwconv1d_fwd_f64(const double* x, const double* k, double* y, int64_t B,
                              int64_t H, int64_t L, int64_t K, int mode, void* stream);

ks_status ks_dwconv1d_dx_f32(const float* gy, const float* k, float* dx, int64_t B, int64_t H,
                             int64_t L, int64_t K, int mode, void* stream);
ks_status ks_dwconv1d_dx_f64(const double* gy, const double* k, double* dx, int64_t B,
                             int64_t H, int64_t L, int64_t K, int mode, void* stream);

/* Scratch bytes ks_dwconv1d_dw_* needs for this shape/scheme (may be 0). */
ks_status ks_dwconv1d_dw_workspace_bytes(int64_t B, int64_t H, int64_t L, int64_t K,
                                         int scheme, int64_t chunk, int elem_bytes,
                                         size_t* bytes);
/* ws may be NULL (then the library takes stream-ordered scratch itself);
 * otherwise ws_bytes must be >= ks_dwconv1d_dw_workspace_bytes(...).
 * `chunk` is only read for KS_DW_CHUNKED (chunk >= B*L degenerates to
 * SEQUENTIAL, src/conv_core.cpp:172-174); `mode` is ignored by PAIRWISE, whose
 * leaves are plain products (src/conv_core.cpp:88-95), and by HIERARCHICAL,
 * whose order is this library's own and which always accumulates with fused
 * multiply-add (the same dk in both modes). */
ks_status ks_dwconv1d_dw_f32(const float* gy, const float* x, float* dk, int64_t B, int64_t H,
                             int64_t L, int64_t K, int scheme, int64_t chunk, int mode,
                             void* ws, size_t ws_bytes, void* stream);
ks_status ks_dwconv1d_dw_f64(const double* gy, const double* x, double* dk, int64_t B,
                             int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk,
                             int mode, void* ws, size_t ws_bytes, void* stream);

/* The layer's whole backward in one call: dx = backward_input(gy, k) and
 * dk = backward_weight(gy, x, HIERARCHICAL) -- the pair
 * conv::backward_input (conv_core.hpp:56-59) + conv::backward_weight
 * (:64-69) a training step makes back to back.  Where the fused kernel
 * applies (K <= 16, L % 32 == 0, L >= 2048) gy and x are read from HBM once
 * for both gradients (12 instead of 16 bytes moved per element); elsewhere
 * the two kernels run in turn.  dx is bit-identical to ks_dwconv1d_dx_f32
 * and dk to ks_dwconv1d_dw_f32(..., KS_DW_HIERARCHICAL, ...) in every case.
 * ws / ws_bytes as for ks_dwconv1d_dw_f32 with KS_DW_HIERARCHICAL. */
ks_status ks_dwconv1d_bwd_f32(const float* gy, const float* x, const float* k, float* dx, float* dk,
                              int64_t B, int64_t H, int64_t L, int64_t K, int mode, void* ws,
                              size_t ws_bytes, void* stream);

/* On-device splitmix64 generator, bit-identical to the reference's
 * SplitMix64::next_pm1 (include/kernelscope/rng.hpp:12-28): out[i] = draw
 * (first+1+i) of the stream seeded with `seed`.  validate() draws x, then k,
 * then gy (src/conv_core.cpp:241-247), so x = fill(seed,0), k =
 * fill(seed,B*H*L), gy = fill(seed,B*H*L+H*K). */
ks_status ks_fill_pm1_f32(uint64_t seed, uint64_t first, float* out, int64_t n, void* stream);

/* Number of kernels this library has launched in this process (every
 * launch site counts; a CUDA-graph replay of captured calls does not call
 * the library and is not counted). */
ks_status ks_launch_count(uint64_t* count);

/* Tuning options: tier switches and pipeline depths, process-wide, atomic.
 * The defaults are the measured choices; the library never
 * reads the environment.  Options that pick a kernel tier can change the bits
 * of HIERARCHICAL dW (every tier keeps y / dX bit-identical to the
 * reference); the determinism promise above is for the defaults.  Names:
 * disable_tma, ldg, sts, bwds, dst, dwtma_j16, dwtma_ns, pad_skip, pad_ns,
 * pad_prod, dwpad_ns, stencil_pad, stencil_r, stencil_nt, stencil_ns,
 * host_block_mb, stencil_bl, dw_ctas, dw_mrow, dwpad_min_k, sts_rows, pdl.  KS_OPTION_DEFAULT restores an option's default. */
#define KS_OPTION_DEFAULT INT64_MIN
ks_status ks_set_option(const char* name, int64_t value);
ks_status ks_get_option(const char* name, int64_t* value);

/* The launch plan of one entry point for a shape -- this library's
 * counterpart of the reference's launch_geometry / shared_mem_footprint
 * (proj/include/kernelscope/exec_model.hpp:14-127), produced by the real
 * dispatch code run without launching: every kernel the call would launch, in
 * order, with its grid, block and dynamic shared memory.  path: 0 forward,
 * 1 dX, 2 dW (scheme, chunk as ks_dwconv1d_dw_f32), 3 the layer backward
 * (ks_dwconv1d_bwd_f32).  Operands are taken as 16-byte aligned.  *n = the
 * number of launches (records beyond `cap` are not written).  Needs a
 * device (occupancy and tensor-map queries); no device memory is touched. */
typedef struct ks_launch_rec {
    char kernel[256]; /* demangled kernel signature */
    uint32_t grid[3], block[3];
    uint64_t smem_bytes;  /* dynamic shared memory */
    int32_t regs;         /* registers per thread (cudaFuncGetAttributes) */
    int32_t static_smem;  /* static shared memory per CTA (cudaFuncGetAttributes) */
    int32_t ctas_per_sm;  /* resident CTAs per SM at this block / smem (occupancy API) */
} ks_launch_rec;
ks_status ks_dwconv1d_plan(int path, int64_t B, int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk,
                           int mode, ks_launch_rec* recs, int cap, int* n);

/* Measured FP32 FMA throughput of the current device (TFLOP/s, 2 FLOP per
 * FMA): the compute roof for the long-K (FP32-bound) shapes.  Synchronous. */
ks_status ks_probe_fp32_tflops(double* tflops);

/* ---- host-buffer entry points (synchronous; the value-type API shape) ---- */
/* Inputs/outputs are host pointers (pinned or pageable).  The call streams
 * row blocks host->device, runs the kernels and streams results back with
 * copy/compute overlap on the current device, then returns. */
ks_status ks_dwconv1d_fwd_f32_host(const float* x, const float* k, float* y, int64_t B,
                                   int64_t H, int64_t L, int64_t K, int mode);
ks_status ks_dwconv1d_dx_f32_host(const float* gy, const float* k, float* dx, int64_t B,
                                  int64_t H, int64_t L, int64_t K, int mode);
ks_status ks_dwconv1d_dw_f32_host(const float* gy, const float* x, float* dk, int64_t B,
                                  int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk,
                                  int mode);
ks_status ks_dwconv1d_fwd_f64_host(const double* x, const double* k, double* y, int64_t B,
                                   int64_t H, int64_t L, int64_t K, int mode);
ks_status ks_dwconv1d_dx_f64_host(const double* gy, const double* k, double* dx, int64_t B,
                                  int64_t H, int64_t L, int64_t K, int mode);
ks_status ks_dwconv1d_dw_f64_host(const double* gy, const double* x, double* dk, int64_t B,
                                  int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk,
                                  int mode);

/* One fwd + bwd step of the layer on host buffers (no reference counterpart:
 * the three calls above fused so x and gy cross PCIe once).  y = forward(x),
 * dx = backward_input(gy), dk = backward_weight(gy, x); bits equal the three
 * separate calls. */
ks_status ks_dwconv1d_step_f32_host(const float* x, const float* k, const float* gy, float* y, float* dx,
                                    float* dk, int64_t B, int64_t H, int64_t L, int64_t K, int scheme,
                                    int64_t chunk, int mode);

/* ---- the paper's four kernel designs (ablation) -------- */
/* Real sm_100a kernels with the launch geometry and thread mapping of the
 * reference's analytical model (src/exec_model.cpp:80-135): variant 0 naive,
 * 1 coalesced (TTILE=32, HTILE=8), 2 shared (TPB=256 halo tile), 3 warp-tiled;
 * path 0 forward (a=x, b=k), 1 dX (a=gy, b=k), 2 dW (a=gy, b=x; out=[H,K]).
 * fwd/dX are bit-identical to the reference; naive dW = SEQUENTIAL.  Returns
 * KS_ERR_SHARD when the literal mapping cannot launch this shape (grid
 * limits, a row or chunk that does not fit shared memory), KS_ERR_BAD_SCHEME
 * for an unknown variant or path. */
typedef enum ks_variant {
    KS_VARIANT_NAIVE = 0,
    KS_VARIANT_COALESCED = 1,
    KS_VARIANT_SHARED = 2,
    KS_VARIANT_WARP = 3
} ks_variant;
ks_status ks_dwconv1d_variant_workspace_bytes(int variant, int path, int64_t H, int64_t K, size_t* bytes);
ks_status ks_dwconv1d_variant_f32(int variant, int path, const float* a, const float* b, float* out,
                                  int64_t B, int64_t H, int64_t L, int64_t K, int mode, void* ws,
                                  size_t ws_bytes, void* stream);

/* ---- batch sharding across GPUs (one process per GPU) --------------------- */
/* Contiguous batch slice of rank `rank` out of `world`: rows [*b0, *b0+*nb).
 * Slices differ by at most one row; pure host arithmetic (no device). */
ks_status ks_shard_rows(int64_t B, int world, int rank, int64_t* b0, int64_t* nb);

typedef struct ks_comm ks_comm;
/* 128-byte NCCL unique id, created on rank 0 and broadcast by the caller. */
ks_status ks_comm_unique_id(void* id128);
ks_status ks_comm_init(ks_comm** comm, const void* id128, int world, int rank);
/* A communicator whose transport is the caller's: `allgather(send, recv,
 * bytes, ctx)` must gather `bytes` host bytes from every rank into
 * recv[world * bytes] in rank order and return 0 on success (e.g. an MPI or
 * torch.distributed gloo all-gather).  Only bytes cross it -- every sum stays
 * on the device -- so ranks may even share one GPU.  The dW combines below
 * then run synchronously on the host side of `stream`. */
typedef int (*ks_allgather_fn)(const void* send, void* recv, size_t bytes, void* ctx);
ks_status ks_comm_init_host(ks_comm** comm, int world, int rank, ks_allgather_fn allgather, void* ctx);
ks_status ks_comm_destroy(ks_comm* comm);
/* Host-bytes all-gather over the communicator's transport (NCCL through a
 * device bounce buffer, or the caller's callback): `bytes` from every rank
 * into recv[world * bytes] in rank order.  Synchronous.  (What ks_peer_create
 * uses to exchange IPC handles; exposed for setup-time agreement.) */
ks_status ks_comm_allgather_host(ks_comm* comm, const void* send, void* recv, size_t bytes);
/* In-place sum of the rank-local dk[H,K] over all ranks: one ncclAllReduce on
 * `stream` (NCCL communicator); a host communicator gathers the dk of every
 * rank and sums them with ks_rank_tree_sum_f32. */
ks_status ks_dwconv1d_dw_allreduce_f32(float* dk, int64_t H, int64_t K, ks_comm* comm,
                                       void* stream);
/* Deterministic combine that does not depend on the collective's algorithm:
 * all-gathers the per-rank dk[H,K] into gather[world,H,K] (device scratch)
 * and sums it with ks_rank_tree_sum_f32, so every rank ends with the same
 * bits for a given world size. */
ks_status ks_dwconv1d_dw_allgather_sum_f32(float* dk, float* gather, int64_t H, int64_t K,
                                           ks_comm* comm, void* stream);
/* Sharded CHUNKED(chunk) dW, bitwise the single-device
 * ks_dwconv1d_dw_f32(KS_DW_CHUNKED, chunk) of the whole batch -- the
 * reference's reduce_chunked (src/conv_core.cpp:122-146) with its chunks
 * spread over the ranks, so the bits do not depend on the number of GPUs
 * (SURVEY 8(e)'s G-invariant option).  Rank r holds global rows
 * [b0, b0 + B_local) of B_total; the ranks' rows must tile [0, B_total) in
 * rank order with every rank boundary (row * L) a multiple of `chunk`, and
 * all ranks must pass the same (B_total, H, L, K, chunk, mode); else
 * KS_ERR_SHARD on every rank.  Each rank computes the partials of its own chunks, they are
 * all-gathered (rank order = global chunk order) and every rank adds them in
 * chunk order.  dk[H,K] is written on every rank.  Synchronous on a host
 * communicator; on an NCCL communicator the gather runs on `stream`. */
ks_status ks_dwconv1d_dw_chunked_sharded_f32(const float* gy, const float* x, float* dk, int64_t B_local,
                                             int64_t b0, int64_t B_total, int64_t H, int64_t L, int64_t K,
                                             int64_t chunk, int mode, ks_comm* comm, void* stream);
/* out[i] = the midpoint-split pairwise tree over gather[r * n + i], r = 0 ..
 * world-1 (the reference's reduce_pairwise shape, src/conv_core.cpp:113-118,
 * over ranks); 1 <= world <= 64. */
ks_status ks_rank_tree_sum_f32(const float* gather, float* out, int64_t n, int world, void* stream);

/* ---- dW with the cross-GPU combine fused into the reduction (NVLink) ----- */
/* The dW step of a batch-sharded training step is a compute step followed by
 * a collective.  ks_peer exposes each rank's partial buffer to every peer via
 * CUDA IPC (mapped over NVLink/NVSwitch, or the same GPU; handles exchanged
 * once through the communicator's all-gather); ks_dwconv1d_dw_f32_peer then
 * runs the HIERARCHICAL stage 1 into it and ONE kernel that signals the peers,
 * waits for them (system-scope release/acquire flags) and sums every rank's
 * partials straight from peer memory in fixed (rank, group) order -- identical
 * bits on every rank, no collective on the data path.  Each rank publishes its
 * group count and shape with its partials, so uneven shards combine
 * correctly; ranks whose (H, K) differ make the call fail.
 *
 * B is this rank's batch rows.  B_total > 0 names the global batch: when this
 * rank holds rows ks_shard_rows(B_total, world, rank) and the global plan's
 * row groups fall on shard boundaries (its group count G is a multiple of
 * world and divides B_total), every rank computes exactly its shard's global
 * groups, and dk is bitwise equal to the 1-GPU
 * ks_dwconv1d_dw_f32(HIERARCHICAL) over the whole batch.  Otherwise (or
 * B_total = 0) each rank plans its own groups: rank-consistent bits for a
 * given world size.  Collective: every rank must call it, in the same order.
 * partial_bytes >= ks_dwconv1d_dw_workspace_bytes(B, H, L, K, HIERARCHICAL)
 * for the largest local B (and for B_total when the global plan is used). */
typedef struct ks_peer ks_peer;
ks_status ks_peer_create(ks_comm* comm, size_t partial_bytes, ks_peer** peer);
ks_status ks_peer_destroy(ks_peer* peer);
ks_status ks_dwconv1d_dw_f32_peer(const float* gy, const float* x, float* dk, int64_t B, int64_t H,
                                  int64_t L, int64_t K, int64_t B_total, int mode, ks_peer* peer,
                                  void* stream);
/* 1 when a combine gave up waiting (~10 s) for a peer that never arrived or
 * found a peer with a different (H, K); that combine wrote NaN into dk and
 * every later ks_dwconv1d_dw_f32_peer call returns KS_ERR_TIMEOUT.  Reads
 * mapped host memory: no device synchronisation. */
ks_status ks_peer_timed_out(ks_peer* peer, int* flag);

#ifdef __cplusplus
}
#endif
#endif /* KS_DWCONV1D_H */
