// capi.cu -- the extern "C" device-pointer entry points of include/ks_dwconv1d.h:
// argument validation in the reference's order (ConvShape ctor checks B,H,L,K,
// shape.hpp:27-31; chunk_size >= 1, src/conv_core.cpp:154-156), launch
// selection, scratch management and the on-device splitmix64 generator.
#include <cxxabi.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "ks_common.cuh"

namespace ks {

ks_status conv_stencil_f32(const float*, const float*, float*, int64_t, int64_t, int64_t, int64_t,
                           int64_t, int, int, cudaStream_t);
ks_status conv_stencil_f64(const double*, const double*, double*, int64_t, int64_t, int64_t,
                           int64_t, int64_t, int, int, cudaStream_t);
size_t dw_workspace_bytes(int64_t, int64_t, int64_t, int64_t, int, int64_t, int);
ks_status dw_f32(const float*, const float*, float*, int64_t, int64_t, int64_t, int64_t, int,
                 int64_t, int, void*, cudaStream_t);
ks_status dw_f64(const double*, const double*, double*, int64_t, int64_t, int64_t, int64_t, int,
                 int64_t, int, void*, cudaStream_t);
ks_status bwd_fused_f32(const float* gy, const float* x, const float* k, float* dx, float* dk, int64_t B,
                        int64_t H, int64_t L, int64_t K, int mode, void* ws, cudaStream_t st, bool* fused);

size_t variant_workspace_bytes(int variant, int path, int64_t H, int64_t K);
bool variant_supported(int variant, int path, int64_t B, int64_t H, int64_t L, int64_t K);
ks_status variant_f32(int variant, int path, const float* a, const float* b, float* out, int64_t B, int64_t H,
                      int64_t L, int64_t K, int mode, void* ws, cudaStream_t st);

static thread_local std::string g_last_error;

void set_last_error(const char* what) { g_last_error = what ? what : ""; }

ks_status cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return KS_OK;
    g_last_error = cudaGetErrorString(e);
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return KS_ERR_NO_DEVICE;
    return KS_ERR_CUDA;
}

static std::atomic<uint64_t> g_launches{0};

ks_status check_launch() { return cuda_status(cudaGetLastError()); }

// ---- launch accounting and planning ---------------------------------------
struct PlanRec {
    const void* fn;
    dim3 grid, block;
    size_t smem;
};
static thread_local std::vector<PlanRec>* g_plan = nullptr;

bool planning() { return g_plan != nullptr; }

bool note_launch(const void* fn, dim3 grid, dim3 block, size_t smem) {
    if (g_plan) {
        g_plan->push_back({fn, grid, block, smem});
        return false;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return true;
}

// One library-owned pool per device, created once under a lock (concurrent
// first calls from several host threads must not race on it).
static cudaMemPool_t scratch_pool() {
    constexpr int kMaxDev = 64;
    static cudaMemPool_t pools[kMaxDev] = {};
    static std::once_flag made[kMaxDev];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDev) return nullptr;
    std::call_once(made[dev], [dev] {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if (cudaMemPoolCreate(&pools[dev], &props) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
        } else {
            pools[dev] = nullptr;
            cudaGetLastError();
        }
    });
    return pools[dev];
}

// While planning, scratch is a placeholder address (aligned, never touched).
static char* const kPlanScratch = reinterpret_cast<char*>(uintptr_t(0x7e0000000000ull));

cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t st) {
    if (planning()) {
        *p = kPlanScratch;
        return cudaSuccess;
    }
    cudaMemPool_t pool = scratch_pool();
    return pool ? cudaMallocFromPoolAsync(p, bytes, pool, st) : cudaMallocAsync(p, bytes, st);
}

void scratch_free(void* p, cudaStream_t st) {
    if (!planning()) cudaFreeAsync(p, st);
}

int prepare_kernel(const void* func, int threads, int smem) {
    // The dynamic-smem opt-in is per (kernel, device) and only ever raised, so a
    // later smaller request never lowers the limit under a larger cached one.
    struct Limit {
        const void* func;
        int dev, smem;
    };
    struct Occ {
        const void* func;
        int dev, threads, smem, per_sm;
    };
    static std::mutex mu;
    static std::vector<Limit> limits;
    static std::vector<Occ> occ;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    Limit* lim = nullptr;
    for (Limit& l : limits)
        if (l.func == func && l.dev == dev) lim = &l;
    if (!lim) {
        limits.push_back({func, dev, 0});
        lim = &limits.back();
        // ask for the largest shared-memory carveout: the driver otherwise may
        // pick a smaller one and hold a kernel below the CTAs/SM its shared
        // memory allows (bwd_short dW at config 3: 2 CTAs/SM where 3 fit)
        cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    }
    if (smem > lim->smem) {
        cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        lim->smem = smem;
    }
    for (const Occ& o : occ)
        if (o.func == func && o.dev == dev && o.threads == threads && o.smem == smem) return o.per_sm;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, func, threads, smem);
    if (per_sm < 1) per_sm = 1;
    if (occ.size() > 4096) occ.clear();
    occ.push_back({func, dev, threads, smem, per_sm});
    return per_sm;
}

static ks_status check_shape(int64_t B, int64_t H, int64_t L, int64_t K) {
    if (B < 1) return KS_ERR_DIM_B;
    if (H < 1) return KS_ERR_DIM_H;
    if (L < 1) return KS_ERR_DIM_L;
    if (K < 1) return KS_ERR_DIM_K;
    return KS_OK;
}

static ks_status check_mode(int mode) {
    return (mode == KS_MULADD_SEPARATE || mode == KS_MULADD_FUSED) ? KS_OK : KS_ERR_BAD_MODE;
}

static ks_status check_dw(int scheme, int64_t chunk) {
    if (scheme < KS_DW_SEQUENTIAL || scheme > KS_DW_HIERARCHICAL) return KS_ERR_BAD_SCHEME;
    if (scheme == KS_DW_CHUNKED && chunk < 1) return KS_ERR_BAD_CHUNK;
    return KS_OK;
}

// Fails loudly when there is no usable device: this library has no CPU path.
static ks_status check_device() {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        g_last_error = e != cudaSuccess ? cudaGetErrorString(e) : "no CUDA device";
        return KS_ERR_NO_DEVICE;
    }
    return KS_OK;
}

#define KS_TRY(expr)                        \
    do {                                    \
        const ks_status _s = (expr);        \
        if (_s != KS_OK) return _s;         \
    } while (0)

// splitmix64 draw n (1-based) of SplitMix64(seed) mapped like next_pm1()
// (include/kernelscope/rng.hpp:17-28).  The 2u-1 step is done in double with
// explicit round-to-nearest intrinsics, then rounded to float once.
__global__ void fill_pm1_kernel(uint64_t seed, uint64_t first, float* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint64_t z = seed + (first + 1 + static_cast<uint64_t>(i)) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z = z ^ (z >> 31);
        const double unit = __dmul_rn(static_cast<double>(z >> 11), 0x1.0p-53);
        out[i] = __double2float_rn(__dadd_rn(__dmul_rn(2.0, unit), -1.0));
    }
}

// FP32 FMA throughput probe (the compute roof of the long-K configs): 8
// independent FMA chains per thread, enough CTAs for every SM.
__global__ void __launch_bounds__(256) fp32_peak_probe(float* out, int iters, float b, float c) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = __fmaf_rn(a[i], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 12345.f) out[0] = s;  // keeps the chains alive
}

// Scratch for dW: caller-provided, or stream-ordered from the device pool.
struct Scratch {
    void* ptr = nullptr;
    bool owned = false;
    cudaStream_t st = nullptr;
    ks_status take(void* ws, size_t ws_bytes, size_t need, cudaStream_t s) {
        st = s;
        if (need == 0) return KS_OK;
        if (ws) {
            if (ws_bytes < need) return KS_ERR_WORKSPACE;
            ptr = ws;
            return KS_OK;
        }
        owned = true;
        return cuda_status(scratch_alloc(&ptr, need, s));
    }
    ~Scratch() {
        if (owned && ptr) scratch_free(ptr, st);
    }
};

}  // namespace ks

using namespace ks;

extern "C" {

const char* ks_status_string(ks_status s) {
    switch (s) {
        case KS_OK: return "ok";
        case KS_ERR_DIM_B: return "axis B must be >= 1";
        case KS_ERR_DIM_H: return "axis H must be >= 1";
        case KS_ERR_DIM_L: return "axis L must be >= 1";
        case KS_ERR_DIM_K: return "axis K must be >= 1";
        case KS_ERR_BAD_CHUNK: return "chunk_size must be >= 1";
        case KS_ERR_BAD_MODE: return "unknown MulAddMode";
        case KS_ERR_BAD_SCHEME: return "unknown accumulation scheme";
        case KS_ERR_NULL: return "null pointer argument";
        case KS_ERR_WORKSPACE: return "workspace too small";
        case KS_ERR_NO_DEVICE: return "no CUDA device";
        case KS_ERR_CUDA: return "CUDA error";
        case KS_ERR_NCCL: return "NCCL error";
        case KS_ERR_SHARD: return "bad shard geometry";
        case KS_ERR_BAD_OPTION: return "unknown option or value out of range";
        case KS_ERR_TIMEOUT: return "peer combine timed out or met a mismatched rank";
    }
    return "unknown status";
}

const char* ks_last_error_string(void) { return g_last_error.c_str(); }

ks_status ks_launch_count(uint64_t* count) {
    if (!count) return KS_ERR_NULL;
    *count = g_launches.load(std::memory_order_relaxed);
    return KS_OK;
}
int ks_abi_version(void) { return KS_DWCONV1D_ABI_VERSION; }

ks_status ks_dwconv1d_fwd_f32(const float* x, const float* k, float* y, int64_t B, int64_t H,
                              int64_t L, int64_t K, int mode, void* stream) {
    KS_TRY(check_shape(B, H, L, K));
    KS_TRY(check_mode(mode));
    if (!x || !k || !y) return KS_ERR_NULL;
    KS_TRY(check_device());
    return conv_stencil_f32(x, k, y, B, H, L, K, K / 2, 0, mode, static_cast<cudaStream_t>(stream));
}

ks_status ks_dwconv1d_fwd_f64(const double* x, const double* k, double* y, int64_t B, int64_t H,
                              int64_t L, int64_t K, int mode, void* stream) {
    KS_TRY(check_shape(B, H, L, K));
    KS_TRY(check_mode(mode));
    if (!x || !k || !y) return KS_ERR_NULL;
    KS_TRY(check_device());
    return conv_stencil_f64(x, k, y, B, H, L, K, K / 2, 0, mode, static_cast<cudaStream_t>(stream));
}

ks_status ks_dwconv1d_dx_f32(const float* gy, const float* k, float* dx, int64_t B, int64_t H,
                             int64_t L, int64_t K, int mode, void* stream) {
    KS_TRY(check_shape(B, H, L, K));
    KS_TRY(check_mode(mode));
    if (!gy || !k || !dx) return KS_ERR_NULL;
    KS_TRY(check_device());
    return conv_stencil_f32(gy, k, dx, B, H, L, K, K - 1 - K / 2, 1, mode,
                            static_cast<cudaStream_t>(stream));
}

ks_status ks_dwconv1d_dx_f64(const double* gy, const double* k, double* dx, int64_t B, int64_t H,
                             int64_t L, int64_t K, int mode, void* stream) {
    KS_TRY(check_shape(B, H, L, K));
    KS_TRY(check_mode(mode));
    if (!gy || !k || !dx) return KS_ERR_NULL;
    KS_TRY(check_device());
    return conv_stencil_f64(gy, k, dx, B, H, L, K, K - 1 - K / 2, 1, mode,
                            static_cast<cudaStream_t>(stream));
}

ks_status ks_dwconv1d_dw_workspace_bytes(int64_t B, int64_t H, int64_t L, int64_t K, int scheme,
                                         int64_t chunk, int elem_bytes, size_t* bytes) {
    KS_TRY(check_shape(B, H, L, K));
    KS_TRY(check_dw(scheme, chunk));
    if (!bytes) return KS_ERR_NULL;
    if (elem_bytes != 4 && elem_bytes != 8) return KS_ERR_BAD_MODE;
    *bytes = dw_workspace_bytes(B, H, L, K, scheme, chunk, elem_bytes);
    return KS_OK;
}

ks_status ks_dwconv1d_dw_f32(const float* gy, const float* x, float* dk, int64_t B, int64_t H,
                             int64_t L, int64_t K, int scheme, int64_t chunk, int mode, void* ws,
                             size_t ws_bytes, void* stream) {
    KS_TRY(check_shape(B, H, L, K));
    KS_TRY(check_dw(scheme, chunk));
    KS_TRY(check_mode(mode));
    if (!gy || !x || !dk) return KS_ERR_NULL;
    KS_TRY(check_device());
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch s;
    KS_TRY(s.take(ws, ws_bytes, dw_workspace_bytes(B, H, L, K, scheme, chunk, 4), st));
    return dw_f32(gy, x, dk, B, H, L, K, scheme, chunk, mode, s.ptr, st);
}

ks_status ks_dwconv1d_bwd_f32(const float* gy, const float* x, const float* k, float* dx, float* dk, int64_t B,
                              int64_t H, int64_t L, int64_t K, int mode, void* ws, size_t ws_bytes, void* stream) {
    KS_TRY(check_shape(B, H, L, K));
    KS_TRY(check_mode(mode));
    if (!gy || !x || !k || !dx || !dk) return KS_ERR_NULL;
    KS_TRY(check_device());
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch s;
    KS_TRY(s.take(ws, ws_bytes, dw_workspace_bytes(B, H, L, K, KS_DW_HIERARCHICAL, 0, 4), st));
    bool fused = false;
    KS_TRY(bwd_fused_f32(gy, x, k, dx, dk, B, H, L, K, mode, s.ptr, st, &fused));
    if (fused) return KS_OK;
    KS_TRY(ks_dwconv1d_dx_f32(gy, k, dx, B, H, L, K, mode, stream));
    return dw_f32(gy, x, dk, B, H, L, K, KS_DW_HIERARCHICAL, 0, mode, s.ptr, st);
}

ks_status ks_dwconv1d_dw_f64(const double* gy, const double* x, double* dk, int64_t B, int64_t H,
                             int64_t L, int64_t K, int scheme, int64_t chunk, int mode, void* ws,
                             size_t ws_bytes, void* stream) {
    KS_TRY(check_shape(B, H, L, K));
    KS_TRY(check_dw(scheme, chunk));
    KS_TRY(check_mode(mode));
    if (!gy || !x || !dk) return KS_ERR_NULL;
    KS_TRY(check_device());
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch s;
    KS_TRY(s.take(ws, ws_bytes, dw_workspace_bytes(B, H, L, K, scheme, chunk, 8), st));
    return dw_f64(gy, x, dk, B, H, L, K, scheme, chunk, mode, s.ptr, st);
}

ks_status ks_dwconv1d_variant_workspace_bytes(int variant, int path, int64_t H, int64_t K, size_t* bytes) {
    if (!bytes) return KS_ERR_NULL;
    if (variant < 0 || variant > 3 || path < 0 || path > 2) return KS_ERR_BAD_SCHEME;
    if (H < 1) return KS_ERR_DIM_H;
    if (K < 1) return KS_ERR_DIM_K;
    *bytes = variant_workspace_bytes(variant, path, H, K);
    return KS_OK;
}

ks_status ks_dwconv1d_variant_f32(int variant, int path, const float* a, const float* b, float* out, int64_t B,
                                  int64_t H, int64_t L, int64_t K, int mode, void* ws, size_t ws_bytes,
                                  void* stream) {
    KS_TRY(check_shape(B, H, L, K));
    KS_TRY(check_mode(mode));
    if (variant < 0 || variant > 3 || path < 0 || path > 2) return KS_ERR_BAD_SCHEME;
    if (!a || !b || !out) return KS_ERR_NULL;
    if (!variant_supported(variant, path, B, H, L, K)) return KS_ERR_SHARD;
    KS_TRY(check_device());
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch s;
    KS_TRY(s.take(ws, ws_bytes, variant_workspace_bytes(variant, path, H, K), st));
    return variant_f32(variant, path, a, b, out, B, H, L, K, mode, s.ptr, st);
}

ks_status ks_probe_fp32_tflops(double* tflops) {
    if (!tflops) return KS_ERR_NULL;
    KS_TRY(check_device());
    float* out = nullptr;
    KS_TRY(cuda_status(cudaMalloc(&out, sizeof(float))));
    const int blocks = num_sms() * 8, iters = 4096;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch_kernel(fp32_peak_probe, blocks, 256, 0, nullptr, out, 64, 0.999f, 1e-4f);  // warm-up (clocks up)
    cudaEventRecord(a);
    launch_kernel(fp32_peak_probe, blocks, 256, 0, nullptr, out, iters, 0.999f, 1e-4f);
    cudaEventRecord(b);
    ks_status s = cuda_status(cudaEventSynchronize(b));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    if (s != KS_OK) return s;
    const double fma = double(blocks) * 256 * iters * 16 * 8;
    *tflops = 2.0 * fma / (ms * 1e-3) / 1e12;
    return KS_OK;
}

ks_status ks_dwconv1d_plan(int path, int64_t B, int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk,
                           int mode, ks_launch_rec* recs, int cap, int* n) {
    if (!n || (cap > 0 && !recs)) return KS_ERR_NULL;
    if (path < 0 || path > 3) return KS_ERR_BAD_SCHEME;
    KS_TRY(check_shape(B, H, L, K));
    KS_TRY(check_mode(mode));
    if (path == 2) KS_TRY(check_dw(scheme, chunk));
    KS_TRY(check_device());
    KS_TRY(cuda_status(cudaFree(nullptr)));  // a current context: tensor-map encoding needs one
    // placeholder operands: 1 KiB aligned, never dereferenced (nothing launches)
    auto fake = [](int i) { return reinterpret_cast<float*>(uintptr_t(0x7f0000000000ull) + (uintptr_t(i) << 36)); };
    float *a = fake(0), *b = fake(1), *c = fake(2), *d = fake(3), *e = fake(4);
    std::vector<PlanRec> recs_v;
    g_plan = &recs_v;
    ks_status s = KS_OK;
    const cudaStream_t st = nullptr;
    switch (path) {
        case 0: s = conv_stencil_f32(a, b, c, B, H, L, K, K / 2, 0, mode, st); break;
        case 1: s = conv_stencil_f32(a, b, c, B, H, L, K, K - 1 - K / 2, 1, mode, st); break;
        case 2: s = dw_f32(a, b, c, B, H, L, K, scheme, chunk, mode, d, st); break;
        default: {
            bool fused = false;
            s = bwd_fused_f32(a, b, c, d, e, B, H, L, K, mode, fake(5), st, &fused);
            if (s == KS_OK && !fused) s = conv_stencil_f32(a, c, d, B, H, L, K, K - 1 - K / 2, 1, mode, st);
            if (s == KS_OK && !fused) s = dw_f32(a, b, e, B, H, L, K, KS_DW_HIERARCHICAL, 0, mode, fake(5), st);
        }
    }
    g_plan = nullptr;
    if (s != KS_OK) return s;
    *n = static_cast<int>(recs_v.size());
    for (int i = 0; i < *n && i < cap; ++i) {
        ks_launch_rec& r = recs[i];
        memset(&r, 0, sizeof(r));
        const char* mangled = nullptr;
        if (cudaFuncGetName(&mangled, recs_v[i].fn) != cudaSuccess || !mangled) {
            cudaGetLastError();
            mangled = "?";
        }
        int dst = 0;
        char* dem = abi::__cxa_demangle(mangled, nullptr, nullptr, &dst);
        strncpy(r.kernel, dst == 0 && dem ? dem : mangled, sizeof(r.kernel) - 1);
        free(dem);
        r.grid[0] = recs_v[i].grid.x, r.grid[1] = recs_v[i].grid.y, r.grid[2] = recs_v[i].grid.z;
        r.block[0] = recs_v[i].block.x, r.block[1] = recs_v[i].block.y, r.block[2] = recs_v[i].block.z;
        r.smem_bytes = recs_v[i].smem;
        cudaFuncAttributes fa{};
        if (cudaFuncGetAttributes(&fa, recs_v[i].fn) == cudaSuccess) {
            r.regs = fa.numRegs;
            r.static_smem = static_cast<int32_t>(fa.sharedSizeBytes);
        }
        int occ = 0;
        const int threads = static_cast<int>(r.block[0] * r.block[1] * r.block[2]);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, recs_v[i].fn, threads, recs_v[i].smem) == cudaSuccess)
            r.ctas_per_sm = occ;
        cudaGetLastError();
    }
    return KS_OK;
}

ks_status ks_fill_pm1_f32(uint64_t seed, uint64_t first, float* out, int64_t n, void* stream) {
    if (n < 0) return KS_ERR_DIM_L;
    if (n == 0) return KS_OK;
    if (!out) return KS_ERR_NULL;
    KS_TRY(check_device());
    const int64_t want = (n + 255) / 256;
    const unsigned blocks = static_cast<unsigned>(want < int64_t(num_sms()) * 64 ? want : int64_t(num_sms()) * 64);
    launch_kernel(fill_pm1_kernel, blocks, 256, 0, static_cast<cudaStream_t>(stream), seed, first, out, n);
    return check_launch();
}

}  // extern "C"
