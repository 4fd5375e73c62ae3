// ks_common.cuh -- shared device helpers for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "ks_dwconv1d.h"

namespace ks {

// Multiply-add in the reference's two rounding modes (src/conv_core.cpp:14-19).
// The intrinsics are never contracted by nvcc, so Separate really rounds twice.
template <bool FUSED>
__device__ __forceinline__ float muladd(float acc, float a, float b) {
    if constexpr (FUSED) return __fmaf_rn(a, b, acc);
    else return __fadd_rn(acc, __fmul_rn(a, b));
}
template <bool FUSED>
__device__ __forceinline__ double muladd(double acc, double a, double b) {
    if constexpr (FUSED) return __fma_rn(a, b, acc);
    else return __dadd_rn(acc, __dmul_rn(a, b));
}

// Shared-memory window layout: 4 floats of padding after every 32, so float4
// reads by lanes 32 B or 64 B apart (the register-tile strides used below)
// hit 8 distinct 16-byte bank groups per quarter-warp phase.  A float4 at a
// 4-aligned logical index never straddles a pad.
__device__ __forceinline__ int pad_idx(int i) { return i + ((i >> 5) << 2); }
__host__ __device__ constexpr int padded_len(int n) { return n + ((n + 31) >> 5) * 4 + 4; }

__device__ __forceinline__ float4 ld_nc_v4(const float* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st_cs_v4(float* p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}

inline int num_sms() {
    static const int n = [] {  // thread-safe static init
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 148;
    }();
    return n;
}

// Stream-ordered scratch from a library-owned memory pool (one per device,
// release threshold = unlimited): freed blocks stay cached across stream
// synchronisations, so a call after a sync does not re-map memory, and the
// process-wide default pool is left untouched.
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t st);
void scratch_free(void* p, cudaStream_t st);

// Opts `func` in to `smem` bytes of dynamic shared memory on the current device
// and returns its resident CTAs per SM, caching both per (device, kernel,
// smem, threads) so the per-call host cost is a table lookup.
int prepare_kernel(const void* func, int threads, int smem);

// Records a CUDA error for ks_last_error_string and maps it to a status.
ks_status cuda_status(cudaError_t e);
// Called after every kernel launch of the library: maps a launch error to a
// status.
ks_status check_launch();

// Every kernel launch of the library goes through launch_kernel(): it records the
// launch (kernel, grid, block, dynamic shared memory) when the calling thread
// is planning (ks_dwconv1d_plan: the dispatch runs, nothing launches) and
// counts it otherwise (ks_launch_count).  Returns whether to launch.
bool note_launch(const void* fn, dim3 grid, dim3 block, size_t smem);

template <typename... KArgs, typename... Args>
inline void launch_kernel(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    if (note_launch(reinterpret_cast<const void*>(kern), grid, block, smem))
        kern<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
}
// Programmatic dependent launch (sm_90+): a kernel launched through
// launch_kernel_pdl may start while its stream predecessor is still running;
// it must call pdl_wait() before touching global memory (the wait returns once
// the predecessor has completed and its writes are visible; without PDL it is
// a no-op).  prep_taps triggers its dependents as it starts.  Option `pdl`.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
int64_t opt_pdl();
template <typename... KArgs, typename... Args>
inline void launch_kernel_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    if (!note_launch(reinterpret_cast<const void*>(kern), grid, block, smem)) return;
    // auto (-1): only small grids, where the launch gap is a visible share of
    // the kernel (config 1 step -3..-5%; the large configs measured within noise)
    const int64_t o = opt_pdl();
    const bool use = o > 0 || (o < 0 && int64_t(grid.x) * grid.y * grid.z <= 1024);
    if (!use) {
        kern<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
// True while the calling thread is planning: no device work may be issued
// (kernels are recorded by launch_kernel(); copies must be skipped by the caller).
bool planning();
void set_last_error(const char* what);

// Tuning options (options.cu; ks_set_option).  Order = the table in options.cu.
enum Opt {
    kOptDisableTma = 0,
    kOptLdg,
    kOptSts,
    kOptBwds,
    kOptDst,
    kOptDwtmaJ16,
    kOptDwtmaNs,
    kOptPadSkip,
    kOptPadNs,
    kOptPadProd,
    kOptDwpadNs,
    kOptStencilPad,
    kOptStencilR,
    kOptStencilNt,
    kOptStencilNs,
    kOptHostBlockMb,
    kOptStencilBl,
    kOptDwCtas,
    kOptDwMrow,
    kOptDwpadMinK,
    kOptStsRows,
    kOptPdl,
    kOptCount
};
int64_t opt(Opt o);
inline bool tma_disabled() { return opt(kOptDisableTma) != 0; }

}  // namespace ks
