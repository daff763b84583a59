// fvr_internal.cuh -- host-side plumbing shared by the C-ABI translation
// units: error reporting (fvr_last_error), argument checks, launch counting,
// and the render constants block passed by value to the kernels.
#pragma once

#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "fvr_common.cuh"

namespace fvr {

struct RenderConsts {
    double tau, one_minus_tau, sigma_a, sigma_s, phase_g, half_gather;
    double scat_scale;  // sigma_s*4π/S, times 1/4π when g == 0 (ph folded in)
    double bg[4];
    int n_scat;
};

inline RenderConsts make_render_consts(const fvr_render_params_t& p, const double* bg, int nch) {
    RenderConsts rc;
    rc.tau = p.tau;
    rc.one_minus_tau = 1.0 - p.tau;
    rc.sigma_a = p.sigma_a;
    rc.sigma_s = p.sigma_s;
    rc.phase_g = p.phase_g;
    rc.half_gather = 0.5 * p.gather_dist;
    rc.n_scat = p.n_scat > 0 ? p.n_scat : 1;
    const double four_pi = 4.0 * kPi;
    const double ph0 = 1.0 / four_pi;  // phase_hg at g = 0 (radiometry.py:78-92)
    rc.scat_scale = p.sigma_s * four_pi / (double)rc.n_scat;
    if (p.phase_g == 0.0) rc.scat_scale *= ph0;
    for (int c = 0; c < 4; ++c) rc.bg[c] = (bg && c < nch) ? bg[c] : 0.0;
    return rc;
}

int set_error(int code, const std::string& msg);
int check_launch(const char* what);

// Programmatic dependent launch (sm_90+): the loop's per-iteration kernels
// (render plan -> weigh -> gather -> next render) are launched with
// programmatic stream serialisation.  Each calls pdl_trigger() once running,
// so the next one is scheduled onto SMs as this one's last CTAs retire, and
// pdl_wait() before it touches anything its predecessor wrote: the launch
// latency and the grid ramp-up hide under the predecessor's tail.  A kernel
// launched this way must call pdl_wait() before dependent reads (it is a
// no-op for a normal launch).  FVR_PDL=0 launches them normally.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

bool pdl_enabled();

// L2 prefetch of a line a kernel will read right after pdl_wait(): issued
// while the predecessor finishes (the plans are never written by it).
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// Stream-ordered scratch (cudaMallocAsync) comes from the device's default
// pool; the pool keeps up to 256 MB across synchronisations (the default
// threshold, 0, hands every block back to the driver at each sync, so every
// call would pay a fresh allocation).
inline void keep_default_pool() {
    static bool done[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = 256ull << 20;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[dev] = true;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
void count_launch(int n = 1);

inline int check_grid(const fvr_grid_t& g) {
    if (g.nx < 1 || g.ny < 1 || g.nz < 1) return set_error(FVR_ERR_INVALID, "voxel counts must be >= 1");
    if (!(g.edge > 0.0)) return set_error(FVR_ERR_INVALID, "voxel edge must be positive");
    const double kp = (double)(g.nx + 1) * (g.ny + 1) * (g.nz + 1);
    if (kp * 4.0 > 2147483647.0) return set_error(FVR_ERR_INVALID, "lattice too large for 32-bit indexing");
    return FVR_OK;
}

// Write max(v, 0) of key point idx into every float4 slot of the packed
// layout that holds it; p points at the channel's first float (layout + 4c).
__device__ __forceinline__ void layout_store(float* __restrict__ p, int nch, int kind, int sy, int ny1,
                                             int64_t idx, float v) {
    const float c = fmaxf(v, 0.f);
    const int z = (int)(idx % sy);
    if (kind == 2) {  // Z4 (fvr_stencil.cuh); else YZQ
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (z >= k) p[4 * (idx - k) * nch + k] = c;
    } else {
        const int y = (int)((idx / sy) % ny1);
        p[4 * idx * nch] = c;
        if (z >= 1) p[4 * (idx - 1) * nch + 1] = c;
        if (y >= 1) p[4 * (idx - sy) * nch + 2] = c;
        if (y >= 1 && z >= 1) p[4 * (idx - sy - 1) * nch + 3] = c;
    }
}

// Per-pixel (and per-sample) channel pitch of the residual / rho buffers of
// a loop with NCH channels: 1, or 4 (padded) for the batched RGB loop.
template <int NCH>
constexpr int kResPitch = NCH == 1 ? 1 : 4;

// The convergence bookkeeping of one channel (reconstruct.py:311-323), run by
// one block: per-view RMSE from the kernels' squared-residual partials (warp
// per view: lane-strided sums, then a fixed shuffle tree), mean over views,
#ifndef FVR_FINALIZE_UNROLL
#define FVR_FINALIZE_UNROLL 16  // (config 2 render + finalize 0.0892 -> 0.0887 ms; full unroll: 0.0985)
#endif
constexpr int kFinalizeUnroll = FVR_FINALIZE_UNROLL;
// Per-view squared-residual sums in fixed point: each unit's f64 partial is
// rounded to an integer multiple of 2^-kSqFixBits and the per-view sums are
// integer sums -- order-free, so a fused finalize fed by per-unit atomics, a
// separate finalize over the partials and any view sharding agree to the bit.
// While every partial stays below sq_fix_limit(bpv) no per-view sum can
// overflow; beyond that the f64 sums of the partials (in unit order) are used
// by every path alike.
constexpr int kSqFixBits = 24;
__device__ __forceinline__ long long sq_fix(double s) { return __double2ll_rn(ldexp(s, kSqFixBits)); }
__device__ __forceinline__ double sq_fix_limit(int bpv) { return ldexp(1.0, 62 - kSqFixBits) / (double)bpv; }

// trace append, optional vol_rmse and the rule.  Fixed order: bit-identical
// wherever it runs.  s_view: >= n_views doubles of shared memory (plus one int
// slot after them).  acc (may be NULL): n_views fixed-point sums accumulated by
// the partials' producers, acc[n_views] = their overflow flag; they are reset
// here for the next iteration.  Without acc the sums come from the partials.
__device__ __forceinline__ void finalize_block(const double* sq, int n_views, int bpv, double pixels,
                                               const double* vol, int n_vol, double n_kp, double eps,
                                               double* trace, double* trace_vol, fvr_loop_state_t* st,
                                               double* s_view, long long* acc = nullptr) {
    if (st->done) return;  // uniform: every thread reads the same state
    const int lane = threadIdx.x & 31;
    int* s_ovf = reinterpret_cast<int*>(s_view + n_views);
    bool ovf;
    if (acc) {
        ovf = __ldcg(acc + n_views) != 0;
    } else {  // any partial beyond the fixed-point range?
        if (threadIdx.x == 0) *s_ovf = 0;
        __syncthreads();
        const double lim = sq_fix_limit(bpv);
        bool big = false;
        for (int64_t b = threadIdx.x; b < (int64_t)n_views * bpv; b += blockDim.x) big |= !(__ldcg(sq + b) < lim);
        if (__any_sync(0xffffffffu, big) && lane == 0) *s_ovf = 1;
        __syncthreads();
        ovf = *s_ovf != 0;
    }
    if (!ovf && acc) {
        if (threadIdx.x < n_views) {
            s_view[threadIdx.x] = sqrt(ldexp((double)__ldcg(acc + threadIdx.x), -kSqFixBits) / pixels);
            acc[threadIdx.x] = 0;
        }
    } else {
        for (int v = threadIdx.x >> 5; v < n_views; v += blockDim.x >> 5) {
            if (!ovf) {  // the fixed-point sums from the partials
                long long s = 0;
#pragma unroll kFinalizeUnroll
                for (int b = lane; b < bpv; b += 32) s += sq_fix(__ldcg(sq + (int64_t)v * bpv + b));
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
                if (lane == 0) s_view[v] = sqrt(ldexp((double)s, -kSqFixBits) / pixels);
            } else {
                double s = 0.0;
                // FVR_FINALIZE_UNROLL loads in flight per lane (the sum keeps its order)
#pragma unroll kFinalizeUnroll
                for (int b = lane; b < bpv; b += 32) s += __ldcg(sq + (int64_t)v * bpv + b);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
                if (lane == 0) s_view[v] = sqrt(s / pixels);
            }
        }
        if (acc && threadIdx.x < n_views) acc[threadIdx.x] = 0;
    }
    if (acc && threadIdx.x == 0) acc[n_views] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = 0.0;
        for (int i = 0; i < n_views; ++i) acc += s_view[i];
        const double rmse = acc / (double)n_views;
        const int it = st->it;
        trace[it] = rmse;
        if (vol && trace_vol) {
            double s = 0.0;
            for (int b = 0; b < n_vol; ++b) s += __ldcg(vol + b);
            trace_vol[it] = sqrt(s / n_kp);
        }
        const bool conv = rmse < eps || (it > 0 && fabs(rmse - st->prev_rmse) < eps);
        st->prev_rmse = rmse;
        st->it = it + 1;
        if (conv) {
            st->converged = 1;
            st->done = 1;
        }
    }
    __syncthreads();
}

}  // namespace fvr

namespace fvr {
// Every C-ABI entry point is an NVTX range named after it (NVTX v3 is
// header-only: without an attached tool a range costs a pointer check).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace fvr

#define FVR_TRY_BEGIN \
    try {             \
        ::fvr::NvtxRange fvr_nvtx_range_(__func__);
#define FVR_TRY_END                                                   \
    }                                                                 \
    catch (const std::exception& e) {                                 \
        return ::fvr::set_error(FVR_ERR_CUDA, e.what());              \
    }                                                                 \
    catch (...) {                                                     \
        return ::fvr::set_error(FVR_ERR_CUDA, "unknown C++ exception"); \
    }
