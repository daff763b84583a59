// fvr_stencil.cuh -- the fast sample evaluators of K-render.
//
// Two packed copies of the clamped lattice c = max(v, 0) (the renderer never
// reads a negative value, _kernels.py:95-96) serve the two render modes:
//
//  * YZQ  (emission + extinction): float4 at key point j holds the 2x2 (y,z)
//    face (c[j], c[j+1], c[j+sy], c[j+sy+1]); a trilinear read is two 16-byte
//    loads (x and x+1).
//  * Z4   (single scattering): float4 at key point j holds the z-run
//    (c[j], c[j+1], c[j+2], c[j+3]); the 3x3x3 neighbourhood of the nearest
//    key point m -- which contains every corner of the emission read and of
//    all gathers p +- edge/2 * s -- is nine 16-byte loads.
//
// With x = q + c_s - m in [-1, 1] per axis, the trilinear read at the gather
// point is sum_j h(j_x; x_x) h(j_y; x_y) h(j_z; x_z) v_j with the hat
// weights h(0) = 1 - |x|, h(sign x) = |x|: the same value the reference's
// floor/clamp cell read produces (trilinear interpolation is continuous), so
// the gathers need no per-direction division or cell index.  Samples within
// half a voxel of the box faces evaluate the reference's exact fp64 in-box
// test per direction (_kernels.py:154-161) and mask the gathers.
#pragma once

#include "fvr_internal.cuh"

namespace fvr {

constexpr int kLayoutNone = 0, kLayoutYZQ = 1, kLayoutZ4 = 2;
constexpr int kScatDirs = 32;

// 0.5 * s (f32) of fibonacci_sphere(32) and s itself (f64) for the exact test.
__constant__ float c_half_dir[3][kScatDirs];
__constant__ double c_dir[3][kScatDirs];  // (single TU: fvr_render.cu)

// ---- emission-only: two 16-byte loads per sample --------------------------
__device__ __forceinline__ float tri_yzq(const float4* __restrict__ Q, const Geom& g, int ix, int iy,
                                         int iz, float fx, float fy, float fz) {
    const int j = ix * g.sx + iy * g.sy + iz;
    const float4 a = __ldg(Q + j);         // x = ix
    const float4 b = __ldg(Q + j + g.sx);  // x = ix + 1
    const float a0 = fmaf(fz, a.y - a.x, a.x), a1 = fmaf(fz, a.w - a.z, a.z);
    const float b0 = fmaf(fz, b.y - b.x, b.x), b1 = fmaf(fz, b.w - b.z, b.z);
    const float a01 = fmaf(fy, a1 - a0, a0), b01 = fmaf(fy, b1 - b0, b0);
    return fmaf(fx, b01 - a01, a01);
}

// ---- 3x3x3 stencil ----------------------------------------------------------
struct Stencil {
    // line data along x for each (jy, jz): mid value and the differences to
    // the x-1 and x+1 neighbours
    float mid[9], dlo[9], dhi[9];
};

__device__ __forceinline__ void stencil_from(const float v[27], Stencil& s) {
#pragma unroll
    for (int l = 0; l < 9; ++l) {
        s.mid[l] = v[9 + l];
        s.dlo[l] = v[l] - v[9 + l];
        s.dhi[l] = v[18 + l] - v[9 + l];
    }
}

// v[(jx*3 + jy)*3 + jz] = c at m + (jx-1, jy-1, jz-1); interior: 9 float4 loads
__device__ __forceinline__ void load_stencil_z4(const float4* __restrict__ Z4, const Geom& g, int mx,
                                                int my, int mz, float v[27]) {
    const int base = (mx - 1) * g.sx + (my - 1) * g.sy + (mz - 1);
#pragma unroll
    for (int jx = 0; jx < 3; ++jx)
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) {
            const float4 r = __ldg(Z4 + base + jx * g.sx + jy * g.sy);
            v[(jx * 3 + jy) * 3 + 0] = r.x;
            v[(jx * 3 + jy) * 3 + 1] = r.y;
            v[(jx * 3 + jy) * 3 + 2] = r.z;
        }
}

// boundary: scalar loads at clamped coordinates (only zero-weight or masked
// gathers ever touch a clamped duplicate)
__device__ __forceinline__ void load_stencil_clamped(const float* __restrict__ vals, const Geom& g,
                                                     int mx, int my, int mz, float v[27]) {
#pragma unroll
    for (int jx = 0; jx < 3; ++jx) {
        const int x = min(max(mx + jx - 1, 0), g.nx);
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) {
            const int y = min(max(my + jy - 1, 0), g.ny);
#pragma unroll
            for (int jz = 0; jz < 3; ++jz) {
                const int z = min(max(mz + jz - 1, 0), g.nz);
                v[(jx * 3 + jy) * 3 + jz] = fmaxf(__ldg(vals + x * g.sx + y * g.sy + z), 0.f);
            }
        }
    }
}

// trilinear read at offset (x, y, z) in [-1, 1]^3 from the stencil centre
__device__ __forceinline__ float stencil_tri(const Stencil& s, float x, float y, float z) {
    const float ax = fabsf(x), ay = fabsf(y), az = fabsf(z);
    const bool px = x >= 0.f, py = y >= 0.f, pz = z >= 0.f;
    float r[9];
#pragma unroll
    for (int l = 0; l < 9; ++l) r[l] = fmaf(ax, px ? s.dhi[l] : s.dlo[l], s.mid[l]);
    // r[jy*3 + jz]; y stage
    float R[3];
#pragma unroll
    for (int jz = 0; jz < 3; ++jz) {
        const float side = py ? r[6 + jz] : r[jz];
        R[jz] = fmaf(ay, side - r[3 + jz], r[3 + jz]);
    }
    const float side = pz ? R[2] : R[0];
    return fmaf(az, side - R[1], R[1]);
}

// sum over the 32 Fibonacci gathers; bit s of mask keeps direction s
template <bool MASKED>
__device__ __forceinline__ float stencil_scatter(const Stencil& s, float dx, float dy, float dz,
                                                 uint32_t mask) {
    float acc = 0.f;
#pragma unroll
    for (int d = 0; d < kScatDirs; ++d) {
        const float t = stencil_tri(s, dx + c_half_dir[0][d], dy + c_half_dir[1][d], dz + c_half_dir[2][d]);
        if (MASKED) {
            if (mask & (1u << d)) acc += t;
        } else {
            acc += t;
        }
    }
    return acc;
}

// exact per-direction in-box mask of the reference for a sample at p
__device__ __forceinline__ uint32_t inbox_mask(const double p[3], const Geom& g, double half_gather) {
    uint32_t m = 0;
#pragma unroll 4
    for (int d = 0; d < kScatDirs; ++d) {
        bool in = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double sa = __dadd_rn(p[a], __dmul_rn(half_gather, c_dir[a][d]));
            in = in && (g.lo[a] <= sa) && (sa <= g.hi[a]);
        }
        m |= in ? (1u << d) : 0u;
    }
    return m;
}

}  // namespace fvr
