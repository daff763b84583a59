// fvr_render.cu -- K-render: ray generation, slab clip, front-to-back
// under-blending of emission (+ single in-scatter) through the key-point
// lattice.  Replaces _kernels.render_rays (_kernels.py:101-186) and the
// per-view render of the reconstruction loop (reconstruct.py:308-311).
//
// Work decomposition: one thread per ray; rays of a 16x8 pixel tile share a
// CTA so that at equal depth the 128 rays gather from a compact patch of the
// L2/L1-resident lattice.  Blending state (transparency, radiance) is fp64 as
// in the reference; each trilinear read is fp32.  Position and sample count
// use the exact fp64 helpers of fvr_common.cuh.
#include "fvr_internal.cuh"

namespace fvr {

template <int NCH, bool SCAT, bool G0>
__device__ __forceinline__ void march_render(const double o[3], const double d[3], const Geom& g,
                                             const float* __restrict__ values, int plane,
                                             const RenderConsts& rc,
                                             const double* __restrict__ scat, double out[NCH]) {
    double l[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) l[c] = 0.0;
    double t_dst = 1.0;
    double te, tx;
    if (slab_span(o, d, g, te, tx)) {
        const int n = sample_count(te, tx, g.edge);
        for (int k = 1; k <= n; ++k) {
            double p[3];
            sample_pos(o, d, te, g.edge, k, p);
            const double qx = (p[0] - g.lo[0]) * g.inv_edge;
            const double qy = (p[1] - g.lo[1]) * g.inv_edge;
            const double qz = (p[2] - g.lo[2]) * g.inv_edge;
            int ix, iy, iz;
            float fx, fy, fz;
            cell_frac(qx, g.nx, ix, fx);
            cell_frac(qy, g.ny, iy, fy);
            cell_frac(qz, g.nz, iz, fz);
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                const float* vc = values + c * plane;
                double l_src = rc.sigma_a * (double)tri_read(vc, g, ix, iy, iz, fx, fy, fz);
                if (SCAT) {
                    float acc = 0.f;
                    for (int s = 0; s < rc.n_scat; ++s) {
                        const double s0 = __ldg(scat + 3 * s);
                        const double s1 = __ldg(scat + 3 * s + 1);
                        const double s2 = __ldg(scat + 3 * s + 2);
                        // in-box test on the exact gather point (_kernels.py:154-161)
                        const double sx = __dadd_rn(p[0], __dmul_rn(rc.half_gather, s0));
                        const double sy = __dadd_rn(p[1], __dmul_rn(rc.half_gather, s1));
                        const double sz = __dadd_rn(p[2], __dmul_rn(rc.half_gather, s2));
                        if (g.lo[0] <= sx && sx <= g.hi[0] && g.lo[1] <= sy && sy <= g.hi[1] &&
                            g.lo[2] <= sz && sz <= g.hi[2]) {
                            const float e = tri_at(vc, g, (sx - g.lo[0]) * g.inv_edge,
                                                   (sy - g.lo[1]) * g.inv_edge,
                                                   (sz - g.lo[2]) * g.inv_edge);
                            if (G0) {
                                acc += e;
                            } else {
                                const float mu = (float)(d[0] * s0 + d[1] * s1 + d[2] * s2);
                                const float gg = (float)rc.phase_g;
                                const float den = 1.f + gg * gg + 2.f * gg * mu;
                                const float ph = (1.f - gg * gg) /
                                                 (4.f * (float)kPi * den * sqrtf(den));
                                acc = fmaf(e, ph, acc);
                            }
                        }
                    }
                    // l_src += sigma_s * acc * 4π / S (ph = 1/4π folded in when g = 0)
                    l_src += (double)acc * rc.scat_scale;
                }
                l[c] += t_dst * (rc.tau * l_src);
            }
            t_dst *= rc.one_minus_tau;
        }
    }
#pragma unroll
    for (int c = 0; c < NCH; ++c) out[c] = l[c] + t_dst * rc.bg[c];
}

// ---- _kernels.render_rays drop-in -----------------------------------------

template <int NCH, bool SCAT, bool G0>
__global__ void __launch_bounds__(128) render_rays_kernel(double ox, double oy, double oz,
                                                          const double* __restrict__ dirs,
                                                          int64_t n_rays,
                                                          const float* __restrict__ values,
                                                          int plane, Geom g, RenderConsts rc,
                                                          const double* __restrict__ scat,
                                                          double* __restrict__ out) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rays) return;
    const double o[3] = {ox, oy, oz};
    const double d[3] = {dirs[3 * r], dirs[3 * r + 1], dirs[3 * r + 2]};
    double res[NCH];
    march_render<NCH, SCAT, G0>(o, d, g, values, plane, rc, scat, res);
#pragma unroll
    for (int c = 0; c < NCH; ++c) out[r * NCH + c] = res[c];
}

// ---- render_pixels / render_view: rays built on the device ----------------

template <int NCH, bool SCAT, bool G0>
__global__ void __launch_bounds__(128) render_pixels_kernel(fvr_camera_t cam,
                                                            const double* __restrict__ us,
                                                            const double* __restrict__ vs,
                                                            int64_t n,
                                                            const float* __restrict__ values,
                                                            int plane, Geom g, RenderConsts rc,
                                                            const double* __restrict__ scat,
                                                            double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double u, v;
    if (us) {
        u = us[i];
        v = vs[i];
    } else {  // full frame, row-major, centres at +0.5 (render.py:228-232)
        u = (double)(i % cam.width) + 0.5;
        v = (double)(i / cam.width) + 0.5;
    }
    double d[3];
    pixel_dir(cam, u, v, d);
    double res[NCH];
    march_render<NCH, SCAT, G0>(cam.center, d, g, values, plane, rc, scat, res);
#pragma unroll
    for (int c = 0; c < NCH; ++c) out[i * NCH + c] = res[c];
}

// ---- loop render: every bbox pixel of every view + residual + RMSE partials

constexpr int kTileW = 16, kTileH = 8, kTileThreads = kTileW * kTileH;

template <bool SCAT>
__global__ void __launch_bounds__(kTileThreads) loop_render_kernel(
    const fvr_camera_t* __restrict__ cams, int u0, int v0, int w, int h, int tiles_x,
    const float* __restrict__ src, const float* __restrict__ values, Geom g, RenderConsts rc,
    const double* __restrict__ scat, float* __restrict__ residual,
    double* __restrict__ sq_partials, const fvr_loop_state_t* __restrict__ state) {
    if (state && state->done) return;
    __shared__ double red[kTileThreads / 32];
    const int view = blockIdx.y;
    const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
    const int col = tx * kTileW + (threadIdx.x % kTileW);
    const int row = ty * kTileH + (threadIdx.x / kTileW);
    double sq = 0.0;
    if (col < w && row < h) {
        const fvr_camera_t& cam = cams[view];
        double d[3];
        pixel_dir(cam, (double)(u0 + col) + 0.5, (double)(v0 + row) + 0.5, d);
        double rec[1];
        march_render<1, SCAT, true>(cam.center, d, g, values, 0, rc, scat, rec);
        const int64_t pix = ((int64_t)view * h + row) * w + col;
        const double r = (double)src[pix] - rec[0];
        residual[pix] = (float)r;
        sq = r * r;
    }
    const double total = block_sum<kTileThreads>(sq, red);
    if (threadIdx.x == 0) sq_partials[(int64_t)view * gridDim.x + blockIdx.x] = total;
}

}  // namespace fvr

using namespace fvr;

namespace {

template <int NCH>
void launch_render_rays(const double origin[3], const double* dirs, int64_t n_rays,
                        const float* values, int plane, const Geom& g, const RenderConsts& rc,
                        bool scat, bool g0, const double* scat_dirs, double* out,
                        cudaStream_t st) {
    const dim3 grid((unsigned)((n_rays + 127) / 128)), block(128);
    if (!scat)
        render_rays_kernel<NCH, false, true><<<grid, block, 0, st>>>(
            origin[0], origin[1], origin[2], dirs, n_rays, values, plane, g, rc, scat_dirs, out);
    else if (g0)
        render_rays_kernel<NCH, true, true><<<grid, block, 0, st>>>(
            origin[0], origin[1], origin[2], dirs, n_rays, values, plane, g, rc, scat_dirs, out);
    else
        render_rays_kernel<NCH, true, false><<<grid, block, 0, st>>>(
            origin[0], origin[1], origin[2], dirs, n_rays, values, plane, g, rc, scat_dirs, out);
}

template <int NCH>
void launch_render_pixels(const fvr_camera_t& cam, const double* us, const double* vs, int64_t n,
                          const float* values, int plane, const Geom& g, const RenderConsts& rc,
                          bool scat, bool g0, const double* scat_dirs, double* out,
                          cudaStream_t st) {
    const dim3 grid((unsigned)((n + 127) / 128)), block(128);
    if (!scat)
        render_pixels_kernel<NCH, false, true>
            <<<grid, block, 0, st>>>(cam, us, vs, n, values, plane, g, rc, scat_dirs, out);
    else if (g0)
        render_pixels_kernel<NCH, true, true>
            <<<grid, block, 0, st>>>(cam, us, vs, n, values, plane, g, rc, scat_dirs, out);
    else
        render_pixels_kernel<NCH, true, false>
            <<<grid, block, 0, st>>>(cam, us, vs, n, values, plane, g, rc, scat_dirs, out);
}

}  // namespace

extern "C" int fvr_render_rays(const double origin[3], const double* dirs, int64_t n_rays,
                               const float* values, int32_t n_channels, fvr_grid_t grid,
                               fvr_render_params_t params, const double* background,
                               const double* scat_dirs, double* out, void* stream) {
    FVR_TRY_BEGIN
    if (n_channels < 1 || n_channels > 4) return set_error(FVR_ERR_INVALID, "n_channels must be 1..4");
    if (int rc = check_grid(grid)) return rc;
    if (n_rays == 0) return FVR_OK;
    const bool scat = params.scattering && params.sigma_s > 0.0;
    if (scat && (params.n_scat < 1 || !scat_dirs))
        return set_error(FVR_ERR_INVALID, "scattering needs n_scat >= 1 directions");
    const Geom g = make_geom(grid);
    const RenderConsts rc = make_render_consts(params, background, n_channels);
    const int plane = (grid.nx + 1) * (grid.ny + 1) * (grid.nz + 1);
    const bool g0 = params.phase_g == 0.0;
    cudaStream_t st = (cudaStream_t)stream;
    switch (n_channels) {
        case 1: launch_render_rays<1>(origin, dirs, n_rays, values, plane, g, rc, scat, g0, scat_dirs, out, st); break;
        case 2: launch_render_rays<2>(origin, dirs, n_rays, values, plane, g, rc, scat, g0, scat_dirs, out, st); break;
        case 3: launch_render_rays<3>(origin, dirs, n_rays, values, plane, g, rc, scat, g0, scat_dirs, out, st); break;
        default: launch_render_rays<4>(origin, dirs, n_rays, values, plane, g, rc, scat, g0, scat_dirs, out, st); break;
    }
    return check_launch("render_rays");
    FVR_TRY_END
}

extern "C" int fvr_render_pixels(const fvr_camera_t* camera, const double* us, const double* vs,
                                 int64_t n, const float* values, int32_t n_channels,
                                 fvr_grid_t grid, fvr_render_params_t params,
                                 const double* background, const double* scat_dirs, double* out,
                                 void* stream) {
    FVR_TRY_BEGIN
    if (!camera) return set_error(FVR_ERR_INVALID, "camera is NULL");
    if (n_channels < 1 || n_channels > 4) return set_error(FVR_ERR_INVALID, "n_channels must be 1..4");
    if (int rc = check_grid(grid)) return rc;
    if ((us == nullptr) != (vs == nullptr)) return set_error(FVR_ERR_INVALID, "us and vs must both be given");
    if (!us) n = (int64_t)camera->width * camera->height;
    if (n == 0) return FVR_OK;
    const bool scat = params.scattering && params.sigma_s > 0.0;
    if (scat && (params.n_scat < 1 || !scat_dirs))
        return set_error(FVR_ERR_INVALID, "scattering needs n_scat >= 1 directions");
    const Geom g = make_geom(grid);
    const RenderConsts rc = make_render_consts(params, background, n_channels);
    const int plane = (grid.nx + 1) * (grid.ny + 1) * (grid.nz + 1);
    const bool g0 = params.phase_g == 0.0;
    cudaStream_t st = (cudaStream_t)stream;
    switch (n_channels) {
        case 1: launch_render_pixels<1>(*camera, us, vs, n, values, plane, g, rc, scat, g0, scat_dirs, out, st); break;
        case 2: launch_render_pixels<2>(*camera, us, vs, n, values, plane, g, rc, scat, g0, scat_dirs, out, st); break;
        case 3: launch_render_pixels<3>(*camera, us, vs, n, values, plane, g, rc, scat, g0, scat_dirs, out, st); break;
        default: launch_render_pixels<4>(*camera, us, vs, n, values, plane, g, rc, scat, g0, scat_dirs, out, st); break;
    }
    return check_launch("render_pixels");
    FVR_TRY_END
}

extern "C" int fvr_loop_blocks_per_view(int32_t bbox_w, int32_t bbox_h) {
    return ((bbox_w + kTileW - 1) / kTileW) * ((bbox_h + kTileH - 1) / kTileH);
}

extern "C" int fvr_loop_render(const fvr_camera_t* cams, int32_t n_views, int32_t u0, int32_t v0,
                               int32_t bbox_w, int32_t bbox_h, const float* src,
                               const float* values, fvr_grid_t grid, fvr_render_params_t params,
                               double background, const double* scat_dirs, float* residual,
                               double* sq_partials, const fvr_loop_state_t* state, void* stream) {
    FVR_TRY_BEGIN
    if (n_views < 1 || n_views > 65535) return set_error(FVR_ERR_INVALID, "bad view count");
    if (bbox_w < 1 || bbox_h < 1) return set_error(FVR_ERR_INVALID, "empty bounding box");
    if (int rc = check_grid(grid)) return rc;
    const bool scat = params.scattering && params.sigma_s > 0.0;
    if (scat && (params.n_scat < 1 || !scat_dirs))
        return set_error(FVR_ERR_INVALID, "scattering needs n_scat >= 1 directions");
    if (scat && params.phase_g != 0.0)
        return set_error(FVR_ERR_INVALID, "the reconstruction loop renders with g = 0 (render.py:196)");
    const Geom g = make_geom(grid);
    const RenderConsts rc = make_render_consts(params, &background, 1);
    const int tiles_x = (bbox_w + kTileW - 1) / kTileW;
    const int tiles = fvr_loop_blocks_per_view(bbox_w, bbox_h);
    const dim3 gridd((unsigned)tiles, (unsigned)n_views), block(kTileThreads);
    cudaStream_t st = (cudaStream_t)stream;
    if (scat)
        loop_render_kernel<true><<<gridd, block, 0, st>>>(cams, u0, v0, bbox_w, bbox_h, tiles_x, src,
                                                          values, g, rc, scat_dirs, residual,
                                                          sq_partials, state);
    else
        loop_render_kernel<false><<<gridd, block, 0, st>>>(cams, u0, v0, bbox_w, bbox_h, tiles_x, src,
                                                           values, g, rc, scat_dirs, residual,
                                                           sq_partials, state);
    return check_launch("loop_render");
    FVR_TRY_END
}
