// host_api.cu -- host-buffer entry points (the value-type API shape of the
// reference, include/kernelscope/conv_core.hpp:49-69, where inputs and outputs
// live in host memory).
//
// fwd / dX: rows are independent, so the call streams blocks of whole batch
// entries (nb*H rows) through a 3-slot ring of device buffers on three CUDA
// streams: H2D of block i+1, the stencil kernel on block i and D2H of block i-1
// overlap (separate copy engines for each direction).  Bits are identical to
// the device-pointer call because every output row is computed the same way.
//
// dW: every output depends on all rows and the exact schemes fix a global
// association order, so the inputs are uploaded (two streams, one per tensor)
// and the device entry point runs once; only dk[H,K] comes back.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "ks_common.cuh"

namespace ks {

namespace {

// target bytes per streamed block (tuning knob KS_HOST_BLOCK_MB)
size_t block_bytes() {
    return size_t(opt(kOptHostBlockMb)) << 20;
}
constexpr int kSlots = 3;

// Device buffers come from the library's own stream-ordered pool (capi.cu),
// never the process-wide default pool, whose settings belong to the caller.
template <typename T>
cudaError_t scratch_alloc_t(T** p, size_t bytes, cudaStream_t st) {
    return scratch_alloc(reinterpret_cast<void**>(p), bytes, st);
}

template <typename T>
using StencilFn = ks_status (*)(const T*, const T*, T*, int64_t, int64_t, int64_t, int64_t, int,
                                void*);

template <typename T>
ks_status stencil_host(StencilFn<T> fn, const T* in, const T* k, T* out, int64_t B, int64_t H,
                       int64_t L, int64_t K, int mode) {
    if (!in || !k || !out) return KS_ERR_NULL;
    const size_t entry = sizeof(T) * size_t(H) * size_t(L);  // one batch entry
    const int64_t nb = std::max<int64_t>(1, std::min<int64_t>(B, int64_t(block_bytes() / std::max<size_t>(entry, 1))));
    const int64_t nblocks = (B + nb - 1) / nb;
    const int slots = static_cast<int>(std::min<int64_t>(kSlots, nblocks));

    cudaStream_t st[kSlots] = {};
    T* din[kSlots] = {};
    T* dout[kSlots] = {};
    T* dk = nullptr;
    ks_status rc = KS_OK;
    for (int s = 0; s < slots && rc == KS_OK; ++s)
        rc = cuda_status(cudaStreamCreateWithFlags(&st[s], cudaStreamNonBlocking));
    if (rc == KS_OK) rc = cuda_status(scratch_alloc_t(&dk, sizeof(T) * H * K, st[0]));
    if (rc == KS_OK)
        rc = cuda_status(cudaMemcpyAsync(dk, k, sizeof(T) * H * K, cudaMemcpyHostToDevice, st[0]));
    cudaEvent_t k_ready = nullptr;
    if (rc == KS_OK) rc = cuda_status(cudaEventCreateWithFlags(&k_ready, cudaEventDisableTiming));
    if (rc == KS_OK) rc = cuda_status(cudaEventRecord(k_ready, st[0]));
    for (int s = 0; s < slots && rc == KS_OK; ++s) {
        if (s) rc = cuda_status(cudaStreamWaitEvent(st[s], k_ready, 0));
        if (rc == KS_OK) rc = cuda_status(scratch_alloc_t(&din[s], entry * nb, st[s]));
        if (rc == KS_OK) rc = cuda_status(scratch_alloc_t(&dout[s], entry * nb, st[s]));
    }
    for (int64_t i = 0; i < nblocks && rc == KS_OK; ++i) {
        const int s = static_cast<int>(i % slots);
        const int64_t b0 = i * nb;
        const int64_t bn = std::min<int64_t>(nb, B - b0);
        const size_t off = size_t(b0) * H * L;
        rc = cuda_status(cudaMemcpyAsync(din[s], in + off, entry * bn, cudaMemcpyHostToDevice, st[s]));
        if (rc == KS_OK) rc = fn(din[s], dk, dout[s], bn, H, L, K, mode, st[s]);
        if (rc == KS_OK)
            rc = cuda_status(cudaMemcpyAsync(out + off, dout[s], entry * bn, cudaMemcpyDeviceToHost, st[s]));
    }
    for (int s = 0; s < slots; ++s) {
        if (!st[s]) continue;
        if (din[s]) scratch_free(din[s], st[s]);
        if (dout[s]) scratch_free(dout[s], st[s]);
    }
    if (dk && st[0]) {
        for (int s = 1; s < slots; ++s) {
            cudaEvent_t e;
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess) {
                cudaEventRecord(e, st[s]);
                cudaStreamWaitEvent(st[0], e, 0);
                cudaEventDestroy(e);
            }
        }
        scratch_free(dk, st[0]);
    }
    for (int s = 0; s < slots; ++s) {
        if (!st[s]) continue;
        const ks_status e = cuda_status(cudaStreamSynchronize(st[s]));
        if (rc == KS_OK) rc = e;
        cudaStreamDestroy(st[s]);
    }
    if (k_ready) cudaEventDestroy(k_ready);
    return rc;
}

template <typename T>
using DwFn = ks_status (*)(const T*, const T*, T*, int64_t, int64_t, int64_t, int64_t, int,
                           int64_t, int, void*, size_t, void*);

template <typename T>
ks_status dw_host(DwFn<T> fn, const T* gy, const T* x, T* dk, int64_t B, int64_t H, int64_t L,
                  int64_t K, int scheme, int64_t chunk, int mode) {
    if (!gy || !x || !dk) return KS_ERR_NULL;
    const size_t tbytes = sizeof(T) * size_t(B) * size_t(H) * size_t(L);
    cudaStream_t s0 = nullptr, s1 = nullptr;
    T *dgy = nullptr, *dx = nullptr, *ddk = nullptr;
    cudaEvent_t x_ready = nullptr;
    ks_status rc = cuda_status(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    if (rc == KS_OK) rc = cuda_status(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    if (rc == KS_OK) rc = cuda_status(cudaEventCreateWithFlags(&x_ready, cudaEventDisableTiming));
    if (rc == KS_OK) rc = cuda_status(scratch_alloc_t(&dgy, tbytes, s0));
    if (rc == KS_OK) rc = cuda_status(scratch_alloc_t(&dx, tbytes, s1));
    if (rc == KS_OK) rc = cuda_status(scratch_alloc_t(&ddk, sizeof(T) * H * K, s0));
    if (rc == KS_OK) rc = cuda_status(cudaMemcpyAsync(dgy, gy, tbytes, cudaMemcpyHostToDevice, s0));
    if (rc == KS_OK) rc = cuda_status(cudaMemcpyAsync(dx, x, tbytes, cudaMemcpyHostToDevice, s1));
    if (rc == KS_OK) rc = cuda_status(cudaEventRecord(x_ready, s1));
    if (rc == KS_OK) rc = cuda_status(cudaStreamWaitEvent(s0, x_ready, 0));
    if (rc == KS_OK) rc = fn(dgy, dx, ddk, B, H, L, K, scheme, chunk, mode, nullptr, 0, s0);
    if (rc == KS_OK)
        rc = cuda_status(cudaMemcpyAsync(dk, ddk, sizeof(T) * H * K, cudaMemcpyDeviceToHost, s0));
    if (s1 && x_ready && rc != KS_OK) {
        cudaEventRecord(x_ready, s1);
        cudaStreamWaitEvent(s0, x_ready, 0);
    }
    if (s0) {
        if (dgy) scratch_free(dgy, s0);
        if (dx) scratch_free(dx, s0);
        if (ddk) scratch_free(ddk, s0);
        const ks_status e = cuda_status(cudaStreamSynchronize(s0));
        if (rc == KS_OK) rc = e;
        cudaStreamDestroy(s0);
    }
    if (s1) {
        cudaStreamSynchronize(s1);
        cudaStreamDestroy(s1);
    }
    if (x_ready) cudaEventDestroy(x_ready);
    return rc;
}

// One training step of the layer on host buffers: y = fwd(x), dx = dX(gy),
// dk = dW(gy, x).  x and gy are uploaded once (block by block, three streams)
// into full device copies; forward and dX run per block as soon as that block
// has landed and their results stream back while later blocks upload; dW runs
// once on the full device copies after the last upload, so its bits equal the
// device-pointer call for every scheme.
ks_status step_host(const float* x, const float* k, const float* gy, float* y, float* dxo, float* dk, int64_t B,
                    int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk, int mode) {
    if (!x || !k || !gy || !y || !dxo || !dk) return KS_ERR_NULL;
    const size_t entry = sizeof(float) * size_t(H) * size_t(L);
    const size_t tbytes = entry * size_t(B);
    const int64_t nb = std::max<int64_t>(1, std::min<int64_t>(B, int64_t(block_bytes() / std::max<size_t>(entry, 1))));
    const int64_t nblocks = (B + nb - 1) / nb;
    const int slots = static_cast<int>(std::min<int64_t>(kSlots, nblocks));
    cudaStream_t st[kSlots] = {};
    float *dxin = nullptr, *dgy = nullptr, *dkk = nullptr, *ddk = nullptr;
    float* dy[kSlots] = {};
    float* ddx[kSlots] = {};
    cudaEvent_t ev[kSlots] = {};
    cudaEvent_t up[kSlots] = {};  // per stream: its latest block upload has landed
    cudaStream_t sdw = nullptr;   // dW (and dk's download) overlap the trailing downloads
    ks_status rc = KS_OK;
    for (int s = 0; s < slots && rc == KS_OK; ++s) {
        rc = cuda_status(cudaStreamCreateWithFlags(&st[s], cudaStreamNonBlocking));
        if (rc == KS_OK) rc = cuda_status(cudaEventCreateWithFlags(&ev[s], cudaEventDisableTiming));
        if (rc == KS_OK) rc = cuda_status(cudaEventCreateWithFlags(&up[s], cudaEventDisableTiming));
    }
    if (rc == KS_OK) rc = cuda_status(cudaStreamCreateWithFlags(&sdw, cudaStreamNonBlocking));
    if (rc == KS_OK) rc = cuda_status(scratch_alloc_t(&dxin, tbytes, st[0]));
    if (rc == KS_OK) rc = cuda_status(scratch_alloc_t(&dgy, tbytes, st[0]));
    if (rc == KS_OK) rc = cuda_status(scratch_alloc_t(&dkk, sizeof(float) * H * K, st[0]));
    if (rc == KS_OK) rc = cuda_status(scratch_alloc_t(&ddk, sizeof(float) * H * K, st[0]));
    for (int s = 0; s < slots && rc == KS_OK; ++s) {
        rc = cuda_status(scratch_alloc_t(&dy[s], entry * nb, st[0]));
        if (rc == KS_OK) rc = cuda_status(scratch_alloc_t(&ddx[s], entry * nb, st[0]));
    }
    if (rc == KS_OK) rc = cuda_status(cudaMemcpyAsync(dkk, k, sizeof(float) * H * K, cudaMemcpyHostToDevice, st[0]));
    if (rc == KS_OK) rc = cuda_status(cudaEventRecord(ev[0], st[0]));
    for (int s = 1; s < slots && rc == KS_OK; ++s) rc = cuda_status(cudaStreamWaitEvent(st[s], ev[0], 0));
    for (int64_t i = 0; i < nblocks && rc == KS_OK; ++i) {
        const int s = static_cast<int>(i % slots);
        const int64_t b0 = i * nb, bn = std::min<int64_t>(nb, B - b0);
        const size_t off = size_t(b0) * H * L, bytes = entry * bn;
        rc = cuda_status(cudaMemcpyAsync(dxin + off, x + off, bytes, cudaMemcpyHostToDevice, st[s]));
        if (rc == KS_OK) rc = cuda_status(cudaMemcpyAsync(dgy + off, gy + off, bytes, cudaMemcpyHostToDevice, st[s]));
        if (rc == KS_OK) rc = cuda_status(cudaEventRecord(up[s], st[s]));
        if (rc == KS_OK) rc = ks_dwconv1d_fwd_f32(dxin + off, dkk, dy[s], bn, H, L, K, mode, st[s]);
        if (rc == KS_OK) rc = ks_dwconv1d_dx_f32(dgy + off, dkk, ddx[s], bn, H, L, K, mode, st[s]);
        if (rc == KS_OK) rc = cuda_status(cudaMemcpyAsync(y + off, dy[s], bytes, cudaMemcpyDeviceToHost, st[s]));
        if (rc == KS_OK) rc = cuda_status(cudaMemcpyAsync(dxo + off, ddx[s], bytes, cudaMemcpyDeviceToHost, st[s]));
    }
    // dW once every upload has landed (not after the downloads): its own
    // stream waits on each slot stream's last upload, so dW and dk's copy
    // overlap the trailing y / dx downloads
    for (int s = 0; s < slots && rc == KS_OK; ++s) rc = cuda_status(cudaStreamWaitEvent(sdw, up[s], 0));
    if (rc == KS_OK) rc = ks_dwconv1d_dw_f32(dgy, dxin, ddk, B, H, L, K, scheme, chunk, mode, nullptr, 0, sdw);
    if (rc == KS_OK) rc = cuda_status(cudaMemcpyAsync(dk, ddk, sizeof(float) * H * K, cudaMemcpyDeviceToHost, sdw));
    if (sdw) {
        const ks_status e = cuda_status(cudaStreamSynchronize(sdw));
        if (rc == KS_OK) rc = e;
    }
    for (int s = 0; s < slots; ++s)
        if (st[s]) cudaStreamSynchronize(st[s]);
    if (st[0]) {
        if (dxin) scratch_free(dxin, st[0]);
        if (dgy) scratch_free(dgy, st[0]);
        if (dkk) scratch_free(dkk, st[0]);
        if (ddk) scratch_free(ddk, st[0]);
        for (int s = 0; s < slots; ++s) {
            if (dy[s]) scratch_free(dy[s], st[0]);
            if (ddx[s]) scratch_free(ddx[s], st[0]);
        }
        const ks_status e = cuda_status(cudaStreamSynchronize(st[0]));
        if (rc == KS_OK) rc = e;
    }
    for (int s = 0; s < slots; ++s) {
        if (st[s]) cudaStreamDestroy(st[s]);
        if (ev[s]) cudaEventDestroy(ev[s]);
        if (up[s]) cudaEventDestroy(up[s]);
    }
    if (sdw) cudaStreamDestroy(sdw);
    return rc;
}

}  // namespace
}  // namespace ks

using namespace ks;

extern "C" {

ks_status ks_dwconv1d_fwd_f32_host(const float* x, const float* k, float* y, int64_t B, int64_t H,
                                   int64_t L, int64_t K, int mode) {
    if (B < 1) return KS_ERR_DIM_B;
    if (H < 1) return KS_ERR_DIM_H;
    if (L < 1) return KS_ERR_DIM_L;
    if (K < 1) return KS_ERR_DIM_K;
    return stencil_host<float>(ks_dwconv1d_fwd_f32, x, k, y, B, H, L, K, mode);
}
ks_status ks_dwconv1d_dx_f32_host(const float* gy, const float* k, float* dx, int64_t B,
                                  int64_t H, int64_t L, int64_t K, int mode) {
    if (B < 1) return KS_ERR_DIM_B;
    if (H < 1) return KS_ERR_DIM_H;
    if (L < 1) return KS_ERR_DIM_L;
    if (K < 1) return KS_ERR_DIM_K;
    return stencil_host<float>(ks_dwconv1d_dx_f32, gy, k, dx, B, H, L, K, mode);
}
ks_status ks_dwconv1d_fwd_f64_host(const double* x, const double* k, double* y, int64_t B,
                                   int64_t H, int64_t L, int64_t K, int mode) {
    if (B < 1) return KS_ERR_DIM_B;
    if (H < 1) return KS_ERR_DIM_H;
    if (L < 1) return KS_ERR_DIM_L;
    if (K < 1) return KS_ERR_DIM_K;
    return stencil_host<double>(ks_dwconv1d_fwd_f64, x, k, y, B, H, L, K, mode);
}
ks_status ks_dwconv1d_dx_f64_host(const double* gy, const double* k, double* dx, int64_t B,
                                  int64_t H, int64_t L, int64_t K, int mode) {
    if (B < 1) return KS_ERR_DIM_B;
    if (H < 1) return KS_ERR_DIM_H;
    if (L < 1) return KS_ERR_DIM_L;
    if (K < 1) return KS_ERR_DIM_K;
    return stencil_host<double>(ks_dwconv1d_dx_f64, gy, k, dx, B, H, L, K, mode);
}
ks_status ks_dwconv1d_dw_f32_host(const float* gy, const float* x, float* dk, int64_t B,
                                  int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk,
                                  int mode) {
    if (B < 1) return KS_ERR_DIM_B;
    if (H < 1) return KS_ERR_DIM_H;
    if (L < 1) return KS_ERR_DIM_L;
    if (K < 1) return KS_ERR_DIM_K;
    if (scheme < KS_DW_SEQUENTIAL || scheme > KS_DW_HIERARCHICAL) return KS_ERR_BAD_SCHEME;
    if (scheme == KS_DW_CHUNKED && chunk < 1) return KS_ERR_BAD_CHUNK;
    return dw_host<float>(ks_dwconv1d_dw_f32, gy, x, dk, B, H, L, K, scheme, chunk, mode);
}
ks_status ks_dwconv1d_dw_f64_host(const double* gy, const double* x, double* dk, int64_t B,
                                  int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk,
                                  int mode) {
    if (B < 1) return KS_ERR_DIM_B;
    if (H < 1) return KS_ERR_DIM_H;
    if (L < 1) return KS_ERR_DIM_L;
    if (K < 1) return KS_ERR_DIM_K;
    if (scheme < KS_DW_SEQUENTIAL || scheme > KS_DW_HIERARCHICAL) return KS_ERR_BAD_SCHEME;
    if (scheme == KS_DW_CHUNKED && chunk < 1) return KS_ERR_BAD_CHUNK;
    return dw_host<double>(ks_dwconv1d_dw_f64, gy, x, dk, B, H, L, K, scheme, chunk, mode);
}

ks_status ks_dwconv1d_step_f32_host(const float* x, const float* k, const float* gy, float* y, float* dx,
                                    float* dk, int64_t B, int64_t H, int64_t L, int64_t K, int scheme, int64_t chunk,
                                    int mode) {
    if (B < 1) return KS_ERR_DIM_B;
    if (H < 1) return KS_ERR_DIM_H;
    if (L < 1) return KS_ERR_DIM_L;
    if (K < 1) return KS_ERR_DIM_K;
    if (mode != KS_MULADD_SEPARATE && mode != KS_MULADD_FUSED) return KS_ERR_BAD_MODE;
    if (scheme < KS_DW_SEQUENTIAL || scheme > KS_DW_HIERARCHICAL) return KS_ERR_BAD_SCHEME;
    if (scheme == KS_DW_CHUNKED && chunk < 1) return KS_ERR_BAD_CHUNK;
    return step_host(x, k, gy, y, dx, dk, B, H, L, K, scheme, chunk, mode);
}

}  // extern "C"
