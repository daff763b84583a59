// fvr_loop.cu -- per-iteration bookkeeping of the device-resident loop:
// per-view RMSE, mean over views, trace append and the convergence rule of
// reconstruct_channel (reconstruct.py:311-323), plus the optional
// vol_rmse reduction (reconstruct.py:133-141, 314-315).
//
// All sums are fixed-order (per-block partials written by the producing
// kernels, reduced here sequentially), so the trace is bit-reproducible.
#include "fvr_internal.cuh"

namespace fvr {

__global__ void __launch_bounds__(256) volume_sq_kernel(const float* __restrict__ values,
                                                        const float* __restrict__ truth,
                                                        const int32_t* __restrict__ kp, int64_t n,
                                                        double* __restrict__ partials,
                                                        const fvr_loop_state_t* __restrict__ state) {
    if (state && state->done) return;
    __shared__ double red[8];
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = kp[i];
        const double d = (double)values[j] - (double)truth[j];
        s += d * d;
    }
    const double t = block_sum<256>(s, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

__global__ void finalize_kernel(const double* __restrict__ sq, int n_views, int bpv,
                                double pixels, const double* __restrict__ vol, int n_vol,
                                double n_kp, double eps, double* __restrict__ trace,
                                double* __restrict__ trace_vol, fvr_loop_state_t* __restrict__ st) {
    __shared__ double view_rmse[33];
    finalize_block(sq, n_views, bpv, pixels, vol, n_vol, n_kp, eps, trace, trace_vol, st, view_rmse);
}

}  // namespace fvr

using namespace fvr;

extern "C" int fvr_loop_volume_sq(const float* values, const float* truth, const int32_t* kp_index,
                                  int64_t n_kp, double* partials, int32_t* n_blocks,
                                  const fvr_loop_state_t* state, void* stream) {
    FVR_TRY_BEGIN
    int64_t b = (n_kp + 255) / 256;
    if (b > 1024) b = 1024;
    if (b < 1) b = 1;
    if (n_blocks) *n_blocks = (int32_t)b;
    if (!values) return FVR_OK;  // size query
    volume_sq_kernel<<<(unsigned)b, 256, 0, (cudaStream_t)stream>>>(values, truth, kp_index, n_kp,
                                                                      partials, state);
    return check_launch("loop_volume_sq");
    FVR_TRY_END
}

extern "C" int fvr_loop_finalize(const double* sq_partials, int32_t n_views, int32_t blocks_per_view,
                                 int64_t pixels_per_view, const double* vol_partials,
                                 int32_t n_vol_blocks, int64_t n_kp, double converge_eps,
                                 double* trace_rmse, double* trace_vol, fvr_loop_state_t* state,
                                 void* stream) {
    FVR_TRY_BEGIN
    if (n_views < 1 || n_views > 32) return set_error(FVR_ERR_INVALID, "n_views must be in 1..32");
    if (pixels_per_view < 1) return set_error(FVR_ERR_INVALID, "empty bounding box");
    finalize_kernel<<<1, 32 * n_views, 0, (cudaStream_t)stream>>>(
        sq_partials, n_views, blocks_per_view, (double)pixels_per_view, vol_partials, n_vol_blocks,
        (double)n_kp, converge_eps, trace_rmse, trace_vol, state);
    return check_launch("loop_finalize");
    FVR_TRY_END
}
