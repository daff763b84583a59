// fvr_preprocess.cu -- input-frame preparation on the device (§8f rank 2):
// flame threshold + blanking (preprocess.py:59-66), the union bounding box
// of the masks (preprocess.py:69-93), and the summed-area tables the hull
// carving reads (volume.py:319-324).  All integer / comparison work, so the
// results are bit-identical to numpy's.
#include "fvr_internal.cuh"

namespace fvr {

// bits = max_c data > threshold (numpy compares the f32 image with the
// threshold converted to f32: a Python float is a "weak" scalar); blanked =
// where(bits, data, 0); bbox4 = (min col, min row, max col, max row) of the
// set pixels over all views, via integer atomics.
__global__ void threshold_kernel(const float* __restrict__ img, int64_t n_pix, int channels, float thr,
                                 int width, int height, uint8_t* __restrict__ bits, float* __restrict__ blanked,
                                 int* __restrict__ bbox4) {
    int u_min = INT_MAX, v_min = INT_MAX, u_max = -1, v_max = -1;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pix;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float* p = img + i * channels;
        float m = p[0];
        for (int c = 1; c < channels; ++c) m = fmaxf(m, p[c]);
        const bool on = m > thr;
        bits[i] = on ? 1 : 0;
        if (blanked)
            for (int c = 0; c < channels; ++c) blanked[i * channels + c] = on ? p[c] : 0.f;
        if (on) {
            const int64_t pix = i % ((int64_t)width * height);
            const int u = (int)(pix % width), v = (int)(pix / width);
            u_min = min(u_min, u);
            u_max = max(u_max, u);
            v_min = min(v_min, v);
            v_max = max(v_max, v);
        }
    }
    // warp-aggregate, then one atomic per warp
    for (int off = 16; off > 0; off >>= 1) {
        u_min = min(u_min, __shfl_xor_sync(0xffffffffu, u_min, off));
        v_min = min(v_min, __shfl_xor_sync(0xffffffffu, v_min, off));
        u_max = max(u_max, __shfl_xor_sync(0xffffffffu, u_max, off));
        v_max = max(v_max, __shfl_xor_sync(0xffffffffu, v_max, off));
    }
    if ((threadIdx.x & 31) == 0 && u_max >= 0) {
        atomicMin(bbox4 + 0, u_min);
        atomicMin(bbox4 + 1, v_min);
        atomicMax(bbox4 + 2, u_max);
        atomicMax(bbox4 + 3, v_max);
    }
}

// Row-wise then column-wise inclusive prefix sums of one view's mask into the
// (h+1, w+1) i64 summed-area table (row 0 and column 0 are zero).
__global__ void sat_rows_kernel(const uint8_t* __restrict__ bits, int width, int height,
                                long long* __restrict__ sat) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v <= height; v += gridDim.x * blockDim.x) {
        long long* row = sat + (int64_t)v * (width + 1);
        row[0] = 0;
        long long acc = 0;
        for (int u = 0; u < width; ++u) {
            if (v > 0) acc += bits[(int64_t)(v - 1) * width + u];
            row[u + 1] = acc;
        }
    }
}

__global__ void sat_cols_kernel(int width, int height, long long* __restrict__ sat) {
    for (int u = blockIdx.x * blockDim.x + threadIdx.x; u <= width; u += gridDim.x * blockDim.x) {
        long long acc = 0;
        for (int v = 0; v <= height; ++v) {
            long long* cell = sat + (int64_t)v * (width + 1) + u;
            acc += *cell;
            *cell = acc;
        }
    }
}

}  // namespace fvr

using namespace fvr;

extern "C" int fvr_threshold_mask(const float* images, int32_t n_views, int32_t width, int32_t height,
                                  int32_t channels, double threshold, uint8_t* bits, float* blanked,
                                  int32_t* bbox4, void* stream) {
    FVR_TRY_BEGIN
    if (n_views < 1 || width < 1 || height < 1 || channels < 1)
        return set_error(FVR_ERR_INVALID, "empty image stack");
    const int64_t n_pix = (int64_t)n_views * width * height;
    int64_t blocks = (n_pix + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    threshold_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        images, n_pix, channels, (float)threshold, width, height, bits, blanked, bbox4);
    return check_launch("threshold_mask");
    FVR_TRY_END
}

extern "C" int fvr_mask_sat(const uint8_t* bits, int32_t width, int32_t height, int64_t* sat, void* stream) {
    FVR_TRY_BEGIN
    if (width < 1 || height < 1) return set_error(FVR_ERR_INVALID, "empty mask");
    cudaStream_t st = (cudaStream_t)stream;
    sat_rows_kernel<<<(unsigned)((height + 1 + 127) / 128), 128, 0, st>>>(bits, width, height,
                                                                         reinterpret_cast<long long*>(sat));
    sat_cols_kernel<<<(unsigned)((width + 1 + 127) / 128), 128, 0, st>>>(width, height,
                                                                        reinterpret_cast<long long*>(sat));
    count_launch(1);
    return check_launch("mask_sat");
    FVR_TRY_END
}
