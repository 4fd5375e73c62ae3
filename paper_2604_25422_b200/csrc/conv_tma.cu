// conv_tma.cu -- host-side TMA tensor-map encoding shared by the TMA kernels
// (stencil_tma.cu: forward / dX; dw_tma.cu: dW), and the tap-staging kernel.
#include <algorithm>

#include "ks_common.cuh"
#include "ks_tma.cuh"

namespace ks {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// cuTensorMapEncodeTiled through the runtime's driver entry-point query, so
// the library does not link libcuda directly.
static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<EncodeTiledFn>(p);
        return static_cast<EncodeTiledFn>(nullptr);
    }();
    return fn;
}

bool encode_row_view(CUtensorMap* map, const float* base, int64_t rows, int64_t L, int inner, int box_rows,
                     int sw) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || L % inner != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
    if (rows >= (int64_t(1) << 31) || L / inner >= (int64_t(1) << 31) || box_rows < 1 || box_rows > 256)
        return false;
    if (sw && inner * 4 > sw) return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(L / inner),
                                static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(inner) * 4, static_cast<cuuint64_t>(L) * 4};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(inner), static_cast<cuuint32_t>(box_rows), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUtensorMapSwizzle swz = sw == 32    ? CU_TENSOR_MAP_SWIZZLE_32B
                                   : sw == 64  ? CU_TENSOR_MAP_SWIZZLE_64B
                                   : sw == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                               : CU_TENSOR_MAP_SWIZZLE_NONE;
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Channel view, 128B-swizzled: the [rows, L] tensor (rows = batch x H
// channels) as {32, L/32, H, rows/H} with box {32, n, 1, depth} -- `depth`
// batch entries of one channel, each n 128-byte pieces (dw_tma's multi-row
// items; the swizzle pattern follows the shared address, so the rows read
// as one long swizzled window).
bool encode_chan_view(CUtensorMap* map, const float* base, int64_t rows, int64_t L, int64_t H, int n, int depth) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || L % 32 != 0 || H < 1 || rows % H != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
    if (n < 1 || n > 256 || depth < 1 || depth > 256) return false;
    if (L / 32 >= (int64_t(1) << 31) || H >= (int64_t(1) << 31) || rows / H >= (int64_t(1) << 31)) return false;
    const cuuint64_t dims[4] = {32, static_cast<cuuint64_t>(L / 32), static_cast<cuuint64_t>(H),
                                static_cast<cuuint64_t>(rows / H)};
    const cuuint64_t strides[3] = {128, static_cast<cuuint64_t>(L) * 4, static_cast<cuuint64_t>(L * H) * 4};
    const cuuint32_t box[4] = {32, static_cast<cuuint32_t>(n), 1, static_cast<cuuint32_t>(depth)};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Padded view: the [rows, L] tensor (rows = batch x H channels) as the 4-D
// tensor {32, L/32, H, rows/H} (floats, 32-float pieces, channels, batch
// entries) with box {36, n, chan_box, depth}.  The box's inner extent runs 4
// floats past the 32-float inner dimension, so TMA fetches each 128-byte
// piece and lands it as a 144-byte shared row (the excess quad is out of
// bounds): the bank-conflict-free padded layout with no re-layout pass.
// `depth` > 1 stacks the same channel of consecutive batch entries (the dW
// kernel); chan_box > 1 stacks channels (the stencil).  This replaced a 5-D
// view {4, 8, L/32, H, B} with box {4, 9, n, ...} that produced the same
// shared layout from 16-byte rows and streamed at only 4.05 TB/s
// (tools/probes/tma_box_probe.cu: 7.07 TB/s for the 128-byte-row box).
bool encode_padded_view(CUtensorMap* map, const float* base, int64_t rows, int64_t L, int64_t H, int n,
                        int chan_box, int depth) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || L % 32 != 0 || H < 1 || rows % H != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
    if (n < 1 || n > 256 || chan_box < 1 || chan_box > 256 || depth < 1 || depth > 256) return false;
    if (L / 32 >= (int64_t(1) << 31) || H >= (int64_t(1) << 31) || rows / H >= (int64_t(1) << 31)) return false;
    const cuuint64_t dims[4] = {32, static_cast<cuuint64_t>(L / 32), static_cast<cuuint64_t>(H),
                                static_cast<cuuint64_t>(rows / H)};
    const cuuint64_t strides[3] = {128, static_cast<cuuint64_t>(L) * 4, static_cast<cuuint64_t>(L * H) * 4};
    const cuuint32_t box[4] = {36, static_cast<cuuint32_t>(n), static_cast<cuuint32_t>(chan_box),
                               static_cast<cuuint32_t>(depth)};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Padded row view: the [rows, L] tensor as {32, L/32, rows} with box
// {36, n, 1} -- the box's inner extent runs 4 floats past the inner dimension,
// so every 128-byte global piece lands as a 144-byte shared row (the excess
// quad is out of bounds and never fetched) -- encode_padded_view's layout for
// a plain [rows, L] row index (7.07 TB/s streamed on the B200, 7.25 for the
// 128B-swizzled 32-float box, tools/probes/tma_box_probe.cu).
bool encode_row_view_padded(CUtensorMap* map, const float* base, int64_t rows, int64_t L, int n) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || L % 32 != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
    if (rows >= (int64_t(1) << 31) || L / 32 >= (int64_t(1) << 31) || n < 1 || n > 256) return false;
    const cuuint64_t dims[3] = {32, static_cast<cuuint64_t>(L / 32), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[2] = {128, static_cast<cuuint64_t>(L) * 4};
    const cuuint32_t box[3] = {36, static_cast<cuuint32_t>(n), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// kp[h, 0:Kp) = `lead` zeros, then k[h, j] (forward) or k[h, K-1-j] (dX, the
// reference's k[h, K-1-j] of src/conv_core.cpp:68), zero padded to Kp.
__global__ void prep_taps(const float* __restrict__ k, float* __restrict__ kp, int64_t H, int64_t K, int64_t Kp,
                          int reverse, int lead) {
    pdl_trigger();  // the stencil that reads kp may launch now (it waits for this grid)
    const int64_t n = H * Kp;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t h = i / Kp, j = i - h * Kp - lead;
        kp[i] = j >= 0 && j < K ? k[h * K + (reverse ? K - 1 - j : j)] : 0.f;
    }
}

}  // namespace ks
