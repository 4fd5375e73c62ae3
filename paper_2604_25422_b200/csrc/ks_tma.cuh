// ks_tma.cuh -- raw-PTX helpers for TMA (cp.async.bulk.tensor) + mbarrier
// pipelines on sm_100a, and the host-side tensor-map encoder.
//
// Row views: a [rows, L] fp32 tensor (L % 32 == 0) is described to TMA as the
// 3-D tensor {32, L/32, rows} (innermost first) with SWIZZLE_128B, so one box
// {32, n, 1} is n consecutive 128-byte pieces of one row.  Out-of-bounds
// coordinates (a halo before t=0 or past t=L) are zero-filled by the TMA unit,
// which is exactly the zero padding of the reference's window
// (src/conv_core.cpp:35-36).  In shared memory the 16-byte chunk c of 128-byte
// row r lands at chunk c ^ (r & 7) of that row (1024-byte aligned buffer).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ks {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
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

// 3-D tiled TMA load of one box into shared memory, completing on `bar`.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

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

// Byte offset of the float4 at logical float index i (i % 4 == 0) inside a
// SWIZZLE_128B box that starts at a 1024-byte aligned address.
__device__ __forceinline__ uint32_t swz128(uint32_t i) {
    const uint32_t row = i >> 5;
    const uint32_t chunk = (i >> 2) & 7u;
    return (row << 7) | ((chunk ^ (row & 7u)) << 4);
}

__device__ __forceinline__ float4 lds128(const char* base, uint32_t byte_off) {
    return *reinterpret_cast<const float4*>(base + byte_off);
}

// Host: encode the {32, L/32, rows} SWIZZLE_128B row view of a [rows, L] fp32
// tensor with a box of {32, box_rows, 1}.  Returns false when the driver entry
// point is unavailable or the tensor violates TMA's constraints.
bool encode_row_view(CUtensorMap* map, const float* base, int64_t rows, int64_t L, int box_rows);

}  // namespace ks
