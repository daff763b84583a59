// fvr_host.cu -- native host-side staging of a reconstruct_channel call's
// inputs (multithreaded, OpenMP).  One pass over the caller's host arrays
// writes everything the device loop needs into one page-locked buffer, which
// then crosses to the device in a single asynchronous copy:
//
//   inside   u8 (nx, ny, nz): tags == 2^V - 1 (HullTags.inside_voxels,
//            volume.py:142-145), computed here instead of by a numpy pass;
//   src      f32 (V, h, w): the bbox crop of every view's single-channel
//            image (reconstruct.py:299-301 src_blocks);
//   masks    u8 (V, h, w): the bbox crop of every flame mask
//            (reconstruct.py:144-149 _flame_ray_pixels);
//   counts   i64 (V): flame pixels per view in the bbox (so the device
//            compaction of the flame rays needs no synchronisation).
#include <omp.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "fvr_internal.cuh"

using namespace fvr;

extern "C" int fvr_stage_inputs_host(const uint32_t* tags, int64_t n_vox, uint32_t full_mask, int32_t n_views,
                                     const float* const* images, const int64_t* image_row_stride,
                                     int64_t image_col_stride, const uint8_t* const* masks,
                                     const int64_t* mask_row_stride, int32_t u0, int32_t v0, int32_t w, int32_t h,
                                     uint8_t* inside_out, float* src_out, uint8_t* masks_out, int64_t* counts_out) {
    FVR_TRY_BEGIN
    if (n_vox < 0 || n_views < 0 || w < 1 || h < 1) return set_error(FVR_ERR_INVALID, "bad sizes");
    if (tags && inside_out) {
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n_vox; ++i) inside_out[i] = tags[i] == full_mask;
    }
    const int64_t pix = (int64_t)w * h;
#pragma omp parallel for schedule(static) collapse(2)
    for (int v = 0; v < n_views; ++v)
        for (int r = 0; r < h; ++r) {
            if (images && src_out) {
                const float* row = images[v] + (int64_t)(v0 + r) * image_row_stride[v] + (int64_t)u0 * image_col_stride;
                float* dst = src_out + v * pix + (int64_t)r * w;
                if (image_col_stride == 1)
                    std::memcpy(dst, row, sizeof(float) * (size_t)w);
                else
                    for (int c = 0; c < w; ++c) dst[c] = row[(int64_t)c * image_col_stride];
            }
            if (masks && masks_out) {
                const uint8_t* row = masks[v] + (int64_t)(v0 + r) * mask_row_stride[v] + u0;
                uint8_t* dst = masks_out + v * pix + (int64_t)r * w;
                for (int c = 0; c < w; ++c) dst[c] = row[c] != 0;
            }
        }
    if (masks && counts_out) {
        for (int v = 0; v < n_views; ++v) {
            int64_t n = 0;
            const uint8_t* m = masks_out + v * pix;
#pragma omp parallel for reduction(+ : n) schedule(static)
            for (int64_t i = 0; i < pix; ++i) n += m[i];
            counts_out[v] = n;
        }
    }
    return FVR_OK;
    FVR_TRY_END
}

// n host buffers concatenated into dst (a page-locked staging buffer) by all
// host threads: big buffers are split into 1 MiB pieces so every thread has
// work (one 12 MB frame per thread would leave most of them idle).
extern "C" int fvr_copy_host_parallel(const void* const* srcs, const int64_t* nbytes, int32_t n, void* dst) {
    FVR_TRY_BEGIN
    if (n < 0) return set_error(FVR_ERR_INVALID, "bad buffer count");
    constexpr int64_t kPiece = 1 << 20;
    std::vector<int64_t> first(n + 1, 0), off(n + 1, 0);
    for (int i = 0; i < n; ++i) {
        if (nbytes[i] < 0) return set_error(FVR_ERR_INVALID, "negative size");
        first[i + 1] = first[i] + (nbytes[i] + kPiece - 1) / kPiece;
        off[i + 1] = off[i] + nbytes[i];
    }
    const int64_t pieces = first[n];
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t q = 0; q < pieces; ++q) {
        int i = 0;
        while (first[i + 1] <= q) ++i;
        const int64_t s = (q - first[i]) * kPiece, len = std::min(kPiece, nbytes[i] - s);
        std::memcpy(static_cast<char*>(dst) + off[i] + s, static_cast<const char*>(srcs[i]) + s, (size_t)len);
    }
    return FVR_OK;
    FVR_TRY_END
}
