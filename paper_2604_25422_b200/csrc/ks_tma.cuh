// ks_tma.cuh -- raw-PTX helpers for TMA (cp.async.bulk.tensor) + mbarrier
// pipelines on sm_100a, and the host-side tensor-map encoder.
//
// Row views: a [rows, L] fp32 tensor (L % IN == 0) is described to TMA as the
// 3-D tensor {IN, L/IN, rows} (innermost first), so one box {IN, n, 1} is n
// consecutive IN-float pieces of one row.  Out-of-bounds coordinates (a halo
// before t=0 or past t=L) are zero-filled by the TMA unit on loads and
// clipped on stores -- exactly the reference's zero padding
// (src/conv_core.cpp:35-36) with no halo code in the kernels.
//
// Shared-memory swizzles (TMA SWIZZLE_32B / 64B / 128B): 16-byte chunk bits
// [4:4+w) of the byte address are XORed with bits [7:7+w), w = 1 / 2 / 3.  The
// right mode depends on the lane stride of the consumer's 128-bit reads:
// 32 B apart -> SWIZZLE_32B, 64 B apart -> SWIZZLE_64B, 16 B -> none; each is
// conflict-free for every starting offset (checked exhaustively).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ks {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 128-bit shared load the compiler cannot narrow.  When only some lanes of a
// window's last float4 are used, nvcc otherwise splits it into LDS.64 / LDS,
// whose 8- / 4-byte accesses at a 128-byte (or 144-byte) lane stride
// conflict 2- / 4-way where the full 16-byte access is conflict-free.
// volatile: keeps the load after the stage's mbarrier wait.
__device__ __forceinline__ float4 lds4(const void* p) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
    return v;
}

// 128-bit shared load from a 32-bit shared-window address.
__device__ __forceinline__ float4 lds4_u32(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}

// A per-thread value ptxas must keep in a register: without it ptxas may
// rematerialise a thread's shared-window address inside the FMA loop from
// SR_TID.X (an S2R + IMAD chain per window whose latency stalls the warp).
__device__ __forceinline__ uint32_t opaque_u32(uint32_t v) {
    asm volatile("mov.b32 %0, %0;" : "+r"(v));
    return v;
}

// Pointer into the dynamic shared buffer rounded up to `align` bytes, derived
// from the __shared__ array itself so the compiler keeps the shared address
// space (LDS/STS rather than generic LD/ST).
template <uint32_t ALIGN>
__device__ __forceinline__ unsigned char* align_smem(unsigned char* raw) {
    const uint32_t pad = (ALIGN - (smem_u32(raw) & (ALIGN - 1))) & (ALIGN - 1);
    return raw + pad;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Generic-proxy shared writes -> visible to the async proxy (TMA store).
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// Plain arrive (release at CTA scope): consumer warps hand a stage back to
// the producer lane of the padded-view kernels (stencil_pad.cu, dw_pad.cu).
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "KS_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra KS_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// The same on a 32-bit shared address held in a register (hot loops: keeps
// ptxas from re-deriving the barrier's shared-window address per iteration).
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "KS_WAITU_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra KS_WAITU_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_u32(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Parked wait for a producer lane: try_wait with a suspend-time hint blocks
// the thread in hardware until the phase completes (or ~1 ms passes), so the
// producer takes no issue slots from the FMA warps it feeds.  (The previous
// try_wait + __nanosleep(128) loop spun: at config 5b its SYNCS / BRA /
// NANOSLEEP were 25% of all instructions issued by stencil_pad.)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
            : "memory");
    } while (!done);
}

// 3-D tiled TMA load of one box into shared memory, completing on `bar`.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// L2 eviction-priority policy (createpolicy) for streamed-once data, and the
// 3-D TMA load / store carrying it (.L2::cache_hint).
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_store_3d_hint(const CUtensorMap* map, const void* src, int c0, int c1, int c2,
                                                  uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src)), "l"(pol)
        : "memory");
}

// Tiled TMA load of the padded view (encode_padded_view, 4-D {32, L/32, H, B}):
// piece c2 of channel c3 of batch entry c4.
__device__ __forceinline__ void tma_load_pad(void* dst, const CUtensorMap* map, int c2, int c3, int c4,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
        : "memory");
}

// 3-D tiled TMA store of one box from shared memory (bulk-group tracked).
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
        : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// All committed bulk stores have finished READING shared memory.
__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// All committed bulk stores are complete (writes performed).
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// 1-D bulk copy global -> shared (16-byte aligned, size % 16 == 0).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Swizzled byte offset of the float4 at logical float index i (i % 4 == 0)
// in a buffer aligned to at least 1024 B.  SW = 0 (none), 32, 64, 128.
template <int SW>
__device__ __forceinline__ uint32_t swz(uint32_t i) {
    const uint32_t b = i << 2;
    if constexpr (SW == 0) return b;
    else if constexpr (SW == 32) return b ^ ((b >> 3) & 0x10u);
    else if constexpr (SW == 64) return b ^ ((b >> 3) & 0x30u);
    else return b ^ ((b >> 3) & 0x70u);
}

// Host: encode the {IN, L/IN, rows} view of a [rows, L] fp32 tensor with box
// {IN, box_rows, 1} and swizzle SW (0/32/64/128; IN*4 must be <= SW when SW>0).
// Returns false when the driver entry point is unavailable or the tensor
// violates TMA's constraints (the caller then uses the generic kernels).
bool encode_row_view(CUtensorMap* map, const float* base, int64_t rows, int64_t L, int inner, int box_rows,
                     int sw);

// Host: the padded view {32, L/32, H, rows/H} of a [rows, L] fp32 tensor
// (rows = batch x H channels) with box {36, n, chan_box, depth}: every
// 32-float piece lands as a 36-float shared row (conflict-free 128-bit reads
// 144 B apart, no re-layout pass).
bool encode_chan_view(CUtensorMap* map, const float* base, int64_t rows, int64_t L, int64_t H, int n, int depth);
bool encode_padded_view(CUtensorMap* map, const float* base, int64_t rows, int64_t L, int64_t H, int n,
                        int chan_box, int depth);

// Host: the {32, L/32, rows} view with box {36, n, 1}: the same 36-float padded
// shared rows from 128-byte global rows (streams at near copy bandwidth).
bool encode_row_view_padded(CUtensorMap* map, const float* base, int64_t rows, int64_t L, int n);

}  // namespace ks
