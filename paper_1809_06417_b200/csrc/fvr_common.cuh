// fvr_common.cuh -- device helpers shared by the sm_100a kernels.
//
// Exactness rules (SURVEY.md §7.1, §8a "Exact arithmetic the GPU must
// reproduce"): every quantity that feeds a floor or a comparison -- the slab
// clip, the sample count, the per-sample cell index of the back-projection,
// the in-box test of the scattering gather -- is evaluated in IEEE fp64 in
// the reference's expression order with explicit __d*_rn intrinsics, so nvcc
// cannot contract it into FMAs.  Everything continuous in those quantities
// (trilinear weights, blending, deposits) runs in fp32/fp64 with FMA.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fvr_b200.h"

// Device-side bounds checks of the debug build (make debug ->
// libfvr_b200_debug.so, -DFVR_BOUNDS_CHECK; compute-sanitizer is not
// available on the GPU pool): a failed check prints its site and traps, so
// the launch fails loudly; the release build compiles them away.
#ifdef FVR_BOUNDS_CHECK
#include <cstdio>
#define FVR_DCHECK(cond, what)                                                                          \
    do {                                                                                                \
        if (!(cond)) {                                                                                  \
            printf("fvr bounds check failed: %s (%s:%d, block %d thread %d)\n", what, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                                  \
            __trap();                                                                                   \
        }                                                                                               \
    } while (0)
#else
#define FVR_DCHECK(cond, what) \
    do {                       \
    } while (0)
#endif

namespace fvr {

constexpr double kMarchCountEps = 1e-9;      // _kernels.py:25
constexpr double kPi = 3.141592653589793;    // np.pi
constexpr double kFixScale = 4294967296.0;   // 2^32: 32.32 fixed-point deposits
constexpr double kFixInv = 1.0 / 4294967296.0;

struct Geom {
    int nx, ny, nz;
    int sx, sy;  // key-point strides: x -> (ny+1)(nz+1), y -> (nz+1)
    double lo[3], hi[3];
    double edge, inv_edge;
};

// hi = lo + n*edge exactly as _kernels.py:127-129.
inline Geom make_geom(const fvr_grid_t& g) {
    Geom r;
    r.nx = g.nx;
    r.ny = g.ny;
    r.nz = g.nz;
    r.sy = g.nz + 1;
    r.sx = (g.ny + 1) * (g.nz + 1);
    const int n[3] = {g.nx, g.ny, g.nz};
    for (int a = 0; a < 3; ++a) {
        r.lo[a] = g.origin[a];
        volatile double prod = (double)n[a] * g.edge;  // keep the host compiler from fusing
        r.hi[a] = g.origin[a] + prod;
    }
    r.edge = g.edge;
    r.inv_edge = 1.0 / g.edge;
    return r;
}

struct Cam {
    double fx, fy, cx, cy;
    double R[9];
    double c[3];
    int w, h;
};

// pixel_rays (geometry.py:125-137) for one pixel centre (u, v):
//   d = [(u-cx)/fx, (v-cy)/fy, 1] @ R ; d /= |d|
// numpy's d @ R runs through OpenBLAS dgemm, whose K=3 inner product is the
// FMA chain RN(R2j + RN(y*R1j + RN(x*R0j))) (verified bit-for-bit against
// numpy 2.3 / OpenBLAS 0.3.30 in tests/golden); the norm is ((d0²+d1²)+d2²).
__device__ __forceinline__ void pixel_dir(const fvr_camera_t& cam, double u, double v,
                                          double d[3]) {
    const double x = __ddiv_rn(__dsub_rn(u, cam.cx), cam.fx);
    const double y = __ddiv_rn(__dsub_rn(v, cam.cy), cam.fy);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        double t = __dmul_rn(x, cam.rotation[j]);
        t = __fma_rn(y, cam.rotation[3 + j], t);
        d[j] = __dadd_rn(cam.rotation[6 + j], t);
    }
    const double s = __dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])),
                               __dmul_rn(d[2], d[2]));
    const double nrm = __dsqrt_rn(s);
#pragma unroll
    for (int j = 0; j < 3; ++j) d[j] = __ddiv_rn(d[j], nrm);
}

// Slab clip, _kernels.py:36-63.
__device__ __forceinline__ bool slab_span(const double o[3], const double d[3], const Geom& g,
                                          double& t_in, double& t_out) {
    double tmin = -1.0e300, tmax = 1.0e300;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (d[a] == 0.0) {
            if (o[a] < g.lo[a] || o[a] > g.hi[a]) return false;
        } else {
            double t0 = __ddiv_rn(__dsub_rn(g.lo[a], o[a]), d[a]);
            double t1 = __ddiv_rn(__dsub_rn(g.hi[a], o[a]), d[a]);
            if (t0 > t1) {
                const double s = t0;
                t0 = t1;
                t1 = s;
            }
            if (t0 > tmin) tmin = t0;
            if (t1 < tmax) tmax = t1;
        }
    }
    const double te = tmin > 0.0 ? tmin : 0.0;
    if (tmax <= te) return false;
    t_in = te;
    t_out = tmax;
    return true;
}

// n = int(floor((t_exit - t_entry)/edge + 1e-9)), _kernels.py:140.
__device__ __forceinline__ int sample_count(double te, double tx, double edge) {
    return (int)floor(__dadd_rn(__ddiv_rn(__dsub_rn(tx, te), edge), kMarchCountEps));
}

// Sample position t = t_entry + (k - 0.5)*edge; p = o + t*d, _kernels.py:142-145.
__device__ __forceinline__ void sample_pos(const double o[3], const double d[3], double te,
                                           double edge, int k, double p[3]) {
    const double t = __dadd_rn(te, __dmul_rn(__dsub_rn((double)k, 0.5), edge));
#pragma unroll
    for (int a = 0; a < 3; ++a) p[a] = __dadd_rn(o[a], __dmul_rn(t, d[a]));
}

__device__ __forceinline__ int clampi(int v, int hi) { return v < 0 ? 0 : (v > hi ? hi : v); }

// floor((p - lo)/edge) with the IEEE quotient: a multiply by 1/edge is within
// ~2 ulp of the correctly rounded quotient, so its floor can only differ when
// the quotient sits within 1e-9 of an integer; only then is the division done.
__device__ __forceinline__ int exact_cell(double p, double lo, double edge, double inv_edge) {
    const double num = __dsub_rn(p, lo);
    double q = __dmul_rn(num, inv_edge);
    double fl = floor(q);
    const double fr = q - fl;
    if (fr < 1e-9 || fr > 1.0 - 1e-9) {
        q = __ddiv_rn(num, edge);
        fl = floor(q);
    }
    return (int)fl;
}

// Cell + fp32 fractions of a lattice coordinate q for the clamped trilinear
// read (_kernels.py:69-86).  Trilinear interpolation is continuous in q, so q
// need not be the exact IEEE quotient here.
__device__ __forceinline__ void cell_frac(double q, int n, int& i, float& f) {
    int fl = (int)floor(q);
    i = clampi(fl, n - 1);
    f = (float)(q - (double)i);
}

// 8-corner read, negative corners clamped to zero, fp32 weights.
__device__ __forceinline__ float tri_read(const float* __restrict__ v, const Geom& g, int ix, int iy,
                                          int iz, float fx, float fy, float fz) {
    const float* b = v + ix * g.sx + iy * g.sy + iz;
    const float c000 = fmaxf(__ldg(b), 0.f);
    const float c001 = fmaxf(__ldg(b + 1), 0.f);
    const float c010 = fmaxf(__ldg(b + g.sy), 0.f);
    const float c011 = fmaxf(__ldg(b + g.sy + 1), 0.f);
    const float c100 = fmaxf(__ldg(b + g.sx), 0.f);
    const float c101 = fmaxf(__ldg(b + g.sx + 1), 0.f);
    const float c110 = fmaxf(__ldg(b + g.sx + g.sy), 0.f);
    const float c111 = fmaxf(__ldg(b + g.sx + g.sy + 1), 0.f);
    const float c00 = fmaf(fz, c001 - c000, c000);
    const float c01 = fmaf(fz, c011 - c010, c010);
    const float c10 = fmaf(fz, c101 - c100, c100);
    const float c11 = fmaf(fz, c111 - c110, c110);
    const float c0 = fmaf(fy, c01 - c00, c00);
    const float c1 = fmaf(fy, c11 - c10, c10);
    return fmaf(fx, c1 - c0, c0);
}

__device__ __forceinline__ float tri_at(const float* __restrict__ v, const Geom& g, double qx,
                                        double qy, double qz) {
    int ix, iy, iz;
    float fx, fy, fz;
    cell_frac(qx, g.nx, ix, fx);
    cell_frac(qy, g.ny, iy, fy);
    cell_frac(qz, g.nz, iz, fz);
    return tri_read(v, g, ix, iy, iz, fx, fy, fz);
}

// Philox4x32-10 counter-based generator (stochastic G(s)).
__device__ __forceinline__ uint4 philox(uint4 ctr, uint2 key) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, ctr.x), lo0 = 0xD2511F53u * ctr.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, ctr.z), lo1 = 0xCD9E8D57u * ctr.z;
        ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
        key.x += 0x9E3779B9u;
        key.y += 0xBB67AE85u;
    }
    return ctr;
}

// G = clip(N(1, sigma), 0, 2) for (seed, iteration, ray, march index k).
// One Philox4x32-10 block keyed (k >> 2, ray, iteration) feeds the four
// samples of a group: words (x, y) and (z, w) are two Box-Muller pairs, and
// each pair yields both R cos(2 pi u2) and R sin(2 pi u2), so consecutive
// samples of a ray share one Philox evaluation and one log/sqrt/sincos per
// pair (the weigh pass reuses them, gauss_weight evaluates one sample).
__device__ __forceinline__ uint4 gauss_block(uint64_t seed, uint32_t iteration, uint32_t ray, uint32_t group) {
    return philox(make_uint4(group, ray, iteration, 0x46565242u), make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}
// the Box-Muller pair (z_cos, z_sin) of words (a, b)
__device__ __forceinline__ float2 gauss_pair(uint32_t a, uint32_t b) {
    const float u1 = ((a >> 8) + 1) * (1.0f / 16777216.0f);  // (0, 1]
    const float u2 = (b >> 8) * (1.0f / 16777216.0f);
    const float r = sqrtf(-2.0f * __logf(u1));
    float s, c;
    sincospif(2.0f * u2, &s, &c);
    return make_float2(r * c, r * s);
}
__device__ __forceinline__ float gauss_clip(float z, float sigma) {
    return fminf(fmaxf(fmaf(sigma, z, 1.0f), 0.0f), 2.0f);
}
__device__ __forceinline__ float gauss_weight(uint64_t seed, uint32_t iteration, uint32_t ray,
                                              uint32_t k, float sigma) {
    const uint4 r = gauss_block(seed, iteration, ray, k >> 2);
    const float2 z = (k & 2) ? gauss_pair(r.z, r.w) : gauss_pair(r.x, r.y);
    return gauss_clip((k & 1) ? z.y : z.x, sigma);
}

__device__ __forceinline__ long long to_fix(float x) {
    return __double2ll_rn((double)x * kFixScale);
}

// Deterministic block reduction of one double per thread (fixed tree order).
template <int kThreads>
__device__ __forceinline__ double block_sum(double v, double* smem) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) smem[warp] = v;
    __syncthreads();
    double total = 0.0;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) total += smem[w];
    }
    return total;
}

}  // namespace fvr
