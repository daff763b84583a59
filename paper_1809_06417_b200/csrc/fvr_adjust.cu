// fvr_adjust.cu -- K-adjust (residual back-projection) and K-update (clamped
// merge).  Replaces _kernels.count_hull_samples / adjust_rays_chunked
// (_kernels.py:189-306) and the merge of adjust_pass (reconstruct.py:221-226).
//
// Ray-driven scatter: one thread per flame ray marches the same samples as
// the renderer; the cell of every sample is the exact fp64 IEEE quotient
// floor((p - lo)/edge) (the deposit is discontinuous in it), and each in-hull
// sample adds base*exp(-alpha_d*|p - corner|) to its 8 corner key points.
// Deposits are accumulated as signed 32.32 fixed point with 64-bit integer
// atomics (RED.E.ADD.64): integer addition is associative, so the corrected
// lattice is bit-identical run to run and across any view sharding.
#include "fvr_internal.cuh"

namespace fvr {

struct AdjustConsts {
    double tau_keep;  // 1 - tau
    double alpha_l;
    float alpha_d;
    float g_sigma;
    uint64_t seed;
};

template <bool USE_G, bool PHILOX>
__device__ __forceinline__ void march_adjust(const double o[3], const double d[3], const Geom& g,
                                             double residual, const uint8_t* __restrict__ inside,
                                             const AdjustConsts& ac, const double* __restrict__ gv,
                                             int64_t g_off, uint32_t iteration, uint32_t ray_id,
                                             unsigned long long* __restrict__ accum) {
    double te, tx;
    if (!slab_span(o, d, g, te, tx)) return;
    const int n = sample_count(te, tx, g.edge);
    double trans = 1.0;  // (1 - tau)^(k-1), repeated multiplication as in the reference
    int64_t gi = g_off;
    for (int k = 1; k <= n; ++k) {
        double p[3];
        sample_pos(o, d, te, g.edge, k, p);
        const int ix = clampi(exact_cell(p[0], g.lo[0], g.edge, g.inv_edge), g.nx - 1);
        const int iy = clampi(exact_cell(p[1], g.lo[1], g.edge, g.inv_edge), g.ny - 1);
        const int iz = clampi(exact_cell(p[2], g.lo[2], g.edge, g.inv_edge), g.nz - 1);
        if (__ldg(inside + ((int64_t)ix * g.ny + iy) * g.nz + iz)) {
            double gw = 1.0;
            if (USE_G) gw = gv[gi];
            if (PHILOX) gw = (double)gauss_weight(ac.seed, iteration, ray_id, (uint32_t)k, ac.g_sigma);
            ++gi;
            const float base = (float)(ac.alpha_l * residual * trans * gw);
            if (base != 0.f) {
                // corner offsets p - (lo + (i + c)*edge), fp64 then fp32 (continuous)
                float ex[2], ey[2], ez[2];
                ex[0] = (float)(p[0] - (g.lo[0] + (double)ix * g.edge));
                ex[1] = (float)(p[0] - (g.lo[0] + (double)(ix + 1) * g.edge));
                ey[0] = (float)(p[1] - (g.lo[1] + (double)iy * g.edge));
                ey[1] = (float)(p[1] - (g.lo[1] + (double)(iy + 1) * g.edge));
                ez[0] = (float)(p[2] - (g.lo[2] + (double)iz * g.edge));
                ez[1] = (float)(p[2] - (g.lo[2] + (double)(iz + 1) * g.edge));
                unsigned long long* b = accum + ix * g.sx + iy * g.sy + iz;
#pragma unroll
                for (int cx = 0; cx < 2; ++cx)
#pragma unroll
                    for (int cy = 0; cy < 2; ++cy)
#pragma unroll
                        for (int cz = 0; cz < 2; ++cz) {
                            const float dist = sqrtf(fmaf(ex[cx], ex[cx], fmaf(ey[cy], ey[cy], ez[cz] * ez[cz])));
                            const float dep = base * expf(-ac.alpha_d * dist);
                            atomicAdd(b + cx * g.sx + cy * g.sy + cz,
                                      (unsigned long long)to_fix(dep));
                        }
            }
        }
        trans *= ac.tau_keep;
    }
}

template <bool USE_G>
__global__ void __launch_bounds__(128) adjust_rays_kernel(
    double ox, double oy, double oz, const double* __restrict__ dirs, int64_t n_rays,
    const double* __restrict__ residuals, const double* __restrict__ g_values,
    const int64_t* __restrict__ g_offsets, const uint8_t* __restrict__ inside, Geom g,
    AdjustConsts ac, unsigned long long* __restrict__ accum) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rays) return;
    const double o[3] = {ox, oy, oz};
    const double d[3] = {dirs[3 * r], dirs[3 * r + 1], dirs[3 * r + 2]};
    march_adjust<USE_G, false>(o, d, g, residuals[r], inside, ac, g_values,
                               USE_G ? g_offsets[r] : 0, 0, 0, accum);
}

__global__ void __launch_bounds__(128) count_hull_kernel(double ox, double oy, double oz,
                                                         const double* __restrict__ dirs,
                                                         int64_t n_rays,
                                                         const uint8_t* __restrict__ inside,
                                                         Geom g, int64_t* __restrict__ counts) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rays) return;
    const double o[3] = {ox, oy, oz};
    const double d[3] = {dirs[3 * r], dirs[3 * r + 1], dirs[3 * r + 2]};
    int64_t n_in = 0;
    double te, tx;
    if (slab_span(o, d, g, te, tx)) {
        const int n = sample_count(te, tx, g.edge);
        for (int k = 1; k <= n; ++k) {
            double p[3];
            sample_pos(o, d, te, g.edge, k, p);
            const int ix = clampi(exact_cell(p[0], g.lo[0], g.edge, g.inv_edge), g.nx - 1);
            const int iy = clampi(exact_cell(p[1], g.lo[1], g.edge, g.inv_edge), g.ny - 1);
            const int iz = clampi(exact_cell(p[2], g.lo[2], g.edge, g.inv_edge), g.nz - 1);
            n_in += __ldg(inside + ((int64_t)ix * g.ny + iy) * g.nz + iz) ? 1 : 0;
        }
    }
    counts[r] = n_in;
}

// Loop adjust: flame rays of all views, rays generated from the cameras.
template <bool PHILOX>
__global__ void __launch_bounds__(128) loop_adjust_kernel(
    const fvr_camera_t* __restrict__ cams, const int32_t* __restrict__ ray_list, int64_t n_rays,
    int u0, int v0, int w, int h, const float* __restrict__ residual, int res_pitch,
    const uint8_t* __restrict__ inside, Geom g, AdjustConsts ac, int64_t ray_id_base,
    unsigned long long* __restrict__ accum, const fvr_loop_state_t* __restrict__ state) {
    if (state && state->done) return;
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rays) return;
    const int32_t e = ray_list[r];
    const int view = (int)((uint32_t)e >> 24), pix = e & 0xFFFFFF;
    const int row = pix / w, col = pix - row * w;
    const float res = residual[((int64_t)view * w * h + pix) * res_pitch];
    if (res == 0.f && !PHILOX) return;  // every deposit would be exactly zero
    const fvr_camera_t& cam = cams[view];
    double d[3];
    pixel_dir(cam, (double)(u0 + col) + 0.5, (double)(v0 + row) + 0.5, d);
    const uint32_t it = state ? (uint32_t)state->it : 0u;
    march_adjust<false, PHILOX>(cam.center, d, g, (double)res, inside, ac, nullptr, 0, it,
                                (uint32_t)(ray_id_base + r), accum);
}

// v = f32(max(f64(v) + acc*2^-32, -1)); acc = 0  (reconstruct.py:221-226).
// When the renderer's packed copy of max(v, 0) exists (fvr_stencil.cuh), the
// new value is written into every float4 slot that holds it.
struct LayoutRef {
    float* p;   // channel's first float of the float4 layout (layout + 4c), or nullptr
    int kind;   // 1 = YZQ, 2 = Z4
    int nch;    // interleaved channels
    int sy;     // nz + 1
    int ny1;    // ny + 1
};

__device__ __forceinline__ void apply_one(float* __restrict__ values,
                                          long long* __restrict__ accum, int64_t idx,
                                          const LayoutRef& L) {
    const long long a = accum[idx];
    if (a != 0) {
        const double nv = (double)values[idx] + (double)a * kFixInv;
        const float f = (float)(nv > -1.0 ? nv : -1.0);
        values[idx] = f;
        accum[idx] = 0;
        if (L.p) layout_store(L.p, L.nch, L.kind, L.sy, L.ny1, idx, f);
    }
}

__global__ void apply_correction_kernel(float* __restrict__ values, long long* __restrict__ accum,
                                        const int32_t* __restrict__ kp, int64_t n, LayoutRef L,
                                        const fvr_loop_state_t* __restrict__ state) {
    if (state && state->done) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        apply_one(values, accum, kp ? (int64_t)kp[i] : i, L);
}

__global__ void pack_kernel(const long long* __restrict__ accum, const int32_t* __restrict__ kp,
                            int64_t n, long long* __restrict__ packed) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        packed[i] = accum[kp[i]];
}

__global__ void unpack_kernel(const long long* __restrict__ packed, const int32_t* __restrict__ kp,
                              int64_t n, long long* __restrict__ accum) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        accum[kp[i]] = packed[i];
}

// Fixed-point lattice -> f64 added into a host-visible partial (host adjust variant).
__global__ void fix_to_f64_kernel(const long long* __restrict__ accum, int64_t n,
                                  double* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (double)accum[i] * kFixInv;
}

inline unsigned grid_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    if (b > 148 * 32) b = 148 * 32;
    return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace fvr

using namespace fvr;

extern "C" int fvr_count_hull_samples(const double origin[3], const double* dirs, int64_t n_rays,
                                      const uint8_t* inside_vox, fvr_grid_t grid, int64_t* counts,
                                      void* stream) {
    FVR_TRY_BEGIN
    if (int rc = check_grid(grid)) return rc;
    if (n_rays == 0) return FVR_OK;
    const Geom g = make_geom(grid);
    count_hull_kernel<<<(unsigned)((n_rays + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        origin[0], origin[1], origin[2], dirs, n_rays, inside_vox, g, counts);
    return check_launch("count_hull_samples");
    FVR_TRY_END
}

extern "C" int fvr_adjust_rays(const double origin[3], const double* dirs, int64_t n_rays,
                               const double* residuals, const double* g_values,
                               const int64_t* g_offsets, int32_t use_g, const uint8_t* inside_vox,
                               fvr_grid_t grid, double tau, double alpha_l, double alpha_d,
                               int64_t* accum, void* stream) {
    FVR_TRY_BEGIN
    if (int rc = check_grid(grid)) return rc;
    if (n_rays == 0) return FVR_OK;
    if (use_g && (!g_values || !g_offsets)) return set_error(FVR_ERR_INVALID, "use_g needs g_values and g_offsets");
    const Geom g = make_geom(grid);
    AdjustConsts ac{1.0 - tau, alpha_l, (float)alpha_d, 0.f, 0};
    const unsigned blocks = (unsigned)((n_rays + 127) / 128);
    cudaStream_t st = (cudaStream_t)stream;
    auto* acc = reinterpret_cast<unsigned long long*>(accum);
    if (use_g)
        adjust_rays_kernel<true><<<blocks, 128, 0, st>>>(origin[0], origin[1], origin[2], dirs, n_rays,
                                                         residuals, g_values, g_offsets, inside_vox, g,
                                                         ac, acc);
    else
        adjust_rays_kernel<false><<<blocks, 128, 0, st>>>(origin[0], origin[1], origin[2], dirs, n_rays,
                                                          residuals, g_values, g_offsets, inside_vox, g,
                                                          ac, acc);
    return check_launch("adjust_rays");
    FVR_TRY_END
}

extern "C" int fvr_apply_correction(float* values, int64_t* accum, const int32_t* kp_index,
                                    int64_t n, void* stream) {
    FVR_TRY_BEGIN
    if (n == 0) return FVR_OK;
    apply_correction_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
        values, reinterpret_cast<long long*>(accum), kp_index, n, LayoutRef{nullptr, 0, 1, 1, 1}, nullptr);
    return check_launch("apply_correction");
    FVR_TRY_END
}

extern "C" int fvr_loop_adjust(const fvr_camera_t* cams, const int32_t* ray_list, int64_t n_rays,
                               int32_t u0, int32_t v0, int32_t bbox_w, int32_t bbox_h,
                               const float* residual, int32_t res_pitch, const uint8_t* inside_vox,
                               fvr_grid_t grid, double tau, double alpha_l, double alpha_d, int32_t stochastic,
                               double g_sigma, uint64_t seed, int64_t ray_id_base, int64_t* accum,
                               const fvr_loop_state_t* state, void* stream) {
    FVR_TRY_BEGIN
    if (int rc = check_grid(grid)) return rc;
    if ((int64_t)bbox_w * bbox_h > 0xFFFFFF) return set_error(FVR_ERR_INVALID, "bounding box exceeds 2^24 pixels");
    if (n_rays == 0) return FVR_OK;
    const Geom g = make_geom(grid);
    AdjustConsts ac{1.0 - tau, alpha_l, (float)alpha_d, (float)g_sigma, seed};
    const unsigned blocks = (unsigned)((n_rays + 127) / 128);
    cudaStream_t st = (cudaStream_t)stream;
    auto* acc = reinterpret_cast<unsigned long long*>(accum);
    if (stochastic)
        loop_adjust_kernel<true><<<blocks, 128, 0, st>>>(cams, ray_list, n_rays, u0, v0, bbox_w, bbox_h,
                                                         residual, res_pitch > 0 ? res_pitch : 1, inside_vox, g,
                                                         ac, ray_id_base, acc, state);
    else
        loop_adjust_kernel<false><<<blocks, 128, 0, st>>>(cams, ray_list, n_rays, u0, v0, bbox_w, bbox_h,
                                                          residual, res_pitch > 0 ? res_pitch : 1, inside_vox, g,
                                                         ac, ray_id_base, acc, state);
    return check_launch("loop_adjust");
    FVR_TRY_END
}

extern "C" int fvr_loop_update(float* values, int64_t* accum, const int32_t* kp_index, int64_t n_kp,
                               float* layout, int32_t layout_kind, int32_t layout_nch, fvr_grid_t grid,
                               const fvr_loop_state_t* state, void* stream) {
    FVR_TRY_BEGIN
    if (n_kp == 0) return FVR_OK;
    if (layout && layout_kind != 1 && layout_kind != 2) return set_error(FVR_ERR_INVALID, "unknown layout kind");
    const LayoutRef L{layout, layout_kind, layout_nch > 0 ? layout_nch : 1, grid.nz + 1, grid.ny + 1};
    apply_correction_kernel<<<grid_for(n_kp, 256), 256, 0, (cudaStream_t)stream>>>(
        values, reinterpret_cast<long long*>(accum), kp_index, n_kp, L, state);
    return check_launch("loop_update");
    FVR_TRY_END
}

extern "C" int fvr_pack_correction(const int64_t* accum, const int32_t* kp_index, int64_t n_kp,
                                   int64_t* packed, void* stream) {
    FVR_TRY_BEGIN
    if (n_kp == 0) return FVR_OK;
    pack_kernel<<<grid_for(n_kp, 256), 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const long long*>(accum), kp_index, n_kp, reinterpret_cast<long long*>(packed));
    return check_launch("pack_correction");
    FVR_TRY_END
}

extern "C" int fvr_unpack_correction(const int64_t* packed, const int32_t* kp_index, int64_t n_kp,
                                     int64_t* accum, void* stream) {
    FVR_TRY_BEGIN
    if (n_kp == 0) return FVR_OK;
    unpack_kernel<<<grid_for(n_kp, 256), 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const long long*>(packed), kp_index, n_kp, reinterpret_cast<long long*>(accum));
    return check_launch("unpack_correction");
    FVR_TRY_END
}

namespace fvr {
int fix_to_f64(const int64_t* accum, int64_t n, double* out, cudaStream_t st) {
    fix_to_f64_kernel<<<grid_for(n, 256), 256, 0, st>>>(reinterpret_cast<const long long*>(accum), n, out);
    return check_launch("fix_to_f64");
}
}  // namespace fvr
