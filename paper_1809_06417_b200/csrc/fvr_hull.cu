// fvr_hull.cu -- K-hull: visual-hull carving, one view per launch
// (volume.py:272-328; the paper's Alg. 1).
//
// One thread per voxel projects the voxel's 8 key points into the view,
// takes the pixel-space bounding box of the footprint and asks the view's
// summed-area table whether any flame pixel lies in it; on a hit it ORs the
// view's bit into the voxel tag.  The projection reproduces numpy's
// kp @ R.T + t (OpenBLAS FMA chain, then the translation add) and
// u = fx*X/z + cx in IEEE fp64, so tags equal the reference bit for bit.
#include "fvr_internal.cuh"

namespace fvr {

__device__ __forceinline__ void project_kp(const fvr_camera_t& cam, const double* __restrict__ t,
                                           double x, double y, double z, double& u, double& v,
                                           bool& ok) {
    double c[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        double s = __dmul_rn(x, cam.rotation[3 * j]);
        s = __fma_rn(y, cam.rotation[3 * j + 1], s);
        s = __fma_rn(z, cam.rotation[3 * j + 2], s);
        c[j] = __dadd_rn(s, t[j]);
    }
    ok = c[2] > 0.0;
    const double zs = ok ? c[2] : 1.0;
    u = __dadd_rn(__ddiv_rn(__dmul_rn(cam.fx, c[0]), zs), cam.cx);
    v = __dadd_rn(__ddiv_rn(__dmul_rn(cam.fy, c[1]), zs), cam.cy);
}

__device__ __forceinline__ int64_t clamp_pix(double f, int hi) {
    // numpy: float -> int64 then clip(0, hi); out-of-range floats only occur
    // for footprints that are off-image or unseen, where the result is unused.
    if (!(f > 0.0)) return 0;
    if (f > (double)hi) return hi;
    return (int64_t)f;
}

__global__ void hull_view_kernel(fvr_camera_t cam, double tx, double ty, double tz, Geom g,
                                 const long long* __restrict__ sat, uint32_t bit,
                                 uint32_t* __restrict__ tags) {
    const int64_t n_vox = (int64_t)g.nx * g.ny * g.nz;
    const double t[3] = {tx, ty, tz};
    for (int64_t vi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; vi < n_vox;
         vi += (int64_t)gridDim.x * blockDim.x) {
        const int iz = (int)(vi % g.nz);
        const int iy = (int)((vi / g.nz) % g.ny);
        const int ix = (int)(vi / ((int64_t)g.nz * g.ny));
        double umin = 1e308, umax = -1e308, vmin = 1e308, vmax = -1e308;
        bool all_ok = true;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int kx = ix + (c >> 2), ky = iy + ((c >> 1) & 1), kz = iz + (c & 1);
            // key_point_positions: origin + edge * index (volume.py:96-102)
            const double x = __dadd_rn(g.lo[0], __dmul_rn(g.edge, (double)kx));
            const double y = __dadd_rn(g.lo[1], __dmul_rn(g.edge, (double)ky));
            const double z = __dadd_rn(g.lo[2], __dmul_rn(g.edge, (double)kz));
            double u, v;
            bool ok;
            project_kp(cam, t, x, y, z, u, v, ok);
            all_ok = all_ok && ok;
            umin = fmin(umin, u);
            umax = fmax(umax, u);
            vmin = fmin(vmin, v);
            vmax = fmax(vmax, v);
        }
        if (!all_ok) continue;
        const int w = cam.width, h = cam.height;
        if (umax <= 0.0 || umin >= (double)w || vmax <= 0.0 || vmin >= (double)h) continue;
        const int64_t iu0 = clamp_pix(floor(umin), w - 1);
        const int64_t iu1 = clamp_pix(ceil(umax) - 1.0, w - 1);
        const int64_t iv0 = clamp_pix(floor(vmin), h - 1);
        const int64_t iv1 = clamp_pix(ceil(vmax) - 1.0, h - 1);
        const int64_t W = w + 1;
        const long long s = sat[(iv1 + 1) * W + iu1 + 1] - sat[iv0 * W + iu1 + 1] -
                            sat[(iv1 + 1) * W + iu0] + sat[iv0 * W + iu0];
        if (s > 0) tags[vi] |= bit;
    }
}

// Key points adjacent to >= 1 inside voxel (volume.py:139-165,
// key_point_mask with core_erosion = 0) and, optionally, the loop's initial
// lattice: 0 at those key points, the outside-hull sentinel elsewhere
// (reconstruct.py _init_grid).  One thread per key point reads its <= 8
// neighbouring voxels.
__global__ void hull_keypoints_kernel(const uint8_t* __restrict__ inside, int nx, int ny, int nz,
                                      uint8_t* __restrict__ kp_mask, float* __restrict__ values) {
    const int64_t n_kp = (int64_t)(nx + 1) * (ny + 1) * (nz + 1);
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_kp;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int iz = (int)(k % (nz + 1));
        const int iy = (int)((k / (nz + 1)) % (ny + 1));
        const int ix = (int)(k / ((int64_t)(ny + 1) * (nz + 1)));
        bool hit = false;
        for (int x = max(ix - 1, 0); x <= min(ix, nx - 1) && !hit; ++x)
            for (int y = max(iy - 1, 0); y <= min(iy, ny - 1) && !hit; ++y)
                for (int z = max(iz - 1, 0); z <= min(iz, nz - 1); ++z)
                    if (inside[((int64_t)x * ny + y) * nz + z]) {
                        hit = true;
                        break;
                    }
        kp_mask[k] = hit ? 1 : 0;
        if (values) values[k] = hit ? 0.f : -1.f;
    }
}

}  // namespace fvr

using namespace fvr;

extern "C" int fvr_visual_hull_view(const fvr_camera_t* camera, const double translation[3],
                                    fvr_grid_t grid, const int64_t* sat, int32_t view_bit,
                                    uint32_t* tags, void* stream) {
    FVR_TRY_BEGIN
    if (!camera || !translation) return set_error(FVR_ERR_INVALID, "camera is NULL");
    if (view_bit < 0 || view_bit > 31) return set_error(FVR_ERR_INVALID, "at most 32 views supported");
    if (int rc = check_grid(grid)) return rc;
    const Geom g = make_geom(grid);
    const int64_t n_vox = (int64_t)grid.nx * grid.ny * grid.nz;
    int64_t blocks = (n_vox + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    hull_view_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        *camera, translation[0], translation[1], translation[2], g,
        reinterpret_cast<const long long*>(sat), 1u << view_bit, tags);
    return check_launch("visual_hull_view");
    FVR_TRY_END
}

extern "C" int fvr_hull_keypoints(const uint8_t* inside, fvr_grid_t grid, uint8_t* kp_mask, float* values,
                                  void* stream) {
    FVR_TRY_BEGIN
    if (int rc = check_grid(grid)) return rc;
    if (!inside || !kp_mask) return set_error(FVR_ERR_INVALID, "inside / kp_mask is NULL");
    const int64_t n_kp = (int64_t)(grid.nx + 1) * (grid.ny + 1) * (grid.nz + 1);
    int64_t blocks = (n_kp + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    hull_keypoints_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(inside, grid.nx, grid.ny, grid.nz,
                                                                           kp_mask, values);
    return check_launch("hull_keypoints");
    FVR_TRY_END
}
