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
// Channels are interleaved: key point j of channel c is float4 element
// j * nch + c (Q points at channel c's first element), so the channels of a
// batched loop read the same cache lines.
__device__ __forceinline__ float tri_yzq(const float4* __restrict__ Q, int nch, const Geom& g, int ix, int iy,
                                         int iz, float fx, float fy, float fz) {
    const int j = ix * g.sx + iy * g.sy + iz;
    const float4 a = __ldg(Q + j * nch);           // x = ix
    const float4 b = __ldg(Q + (j + g.sx) * nch);  // x = ix + 1
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
__device__ __forceinline__ void load_stencil_z4(const float4* __restrict__ Z4, int nch, const Geom& g, int mx,
                                                int my, int mz, float v[27]) {
    const int base = (mx - 1) * g.sx + (my - 1) * g.sy + (mz - 1);
#pragma unroll
    for (int jx = 0; jx < 3; ++jx)
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) {
            const float4 r = __ldg(Z4 + (base + jx * g.sx + jy * g.sy) * nch);
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

// ---- moment evaluation of the 32-direction gather (interior samples) -------
//
// In the basis (1, x/2, |x|/2) per axis the trilinear read at offset x from
// the stencil centre is  sum_k V[k] prod_a u_{k_a}(x_a)  with the separable
// stencil transform  V = (v0, v+ - v-, v+ + v- - 2 v0)^{(x) 3}.  Summed over
// the gathers x_s = delta + c_s (c_s = s/2), the direction sum becomes
//
//   S = sum_k V[k] M[k],   M[k] = sum_{E subset P(k)} delta'^{P(k) \ E} Q_{A(k)}[E]
//
// where P(k) are the axes with k_a != 1, A(k) the axes with k_a = |x|,
// delta' = delta/2, and Q_A[E] = sum_s sigma_s^A prod_{a in E} c_{s,a}/2 with
// sigma_{s,a} = sign(delta_a + c_{s,a}).  Q_A depends on delta only through
// the split index i_a = #{s : c_{s,a} < -delta_a} of each axis in A, so it
// is tabulated once per direction set: Q1 (3 x 33 x 8), Q2 (3 x 33^2 x 8),
// Q3 (33^3 x 8).  Exact in real arithmetic (checked against the brute-force
// sum to 1e-15 in fp64); ~400 instructions per sample instead of ~1400.
#ifndef FVR_Q3_TABLE
#define FVR_Q3_TABLE 0
#endif
#ifndef FVR_OMEGA
#define FVR_OMEGA 1
#endif
#ifndef FVR_MOMENT_PACKED
#define FVR_MOMENT_PACKED 1
#endif
constexpr int kSplits = kScatDirs + 1;
__constant__ float c_thr[3][kScatDirs];  // sorted c_{s,a} = s_a / 2 per axis
__constant__ uint32_t c_nmask[3][kScatDirs + 1];  // directions of the first i per axis (c_{s,a} < -delta_a)
__constant__ float c_q0[8];              // Q_{empty}[E]
__device__ float4 g_q1[3 * kSplits * 2];
__device__ float4 g_q2[3 * kSplits * kSplits * 2];
__device__ float4 g_q3[kSplits * kSplits * kSplits * 2];

// #{thr < key} over 32 sorted thresholds in shared memory
__device__ __forceinline__ int split_index(const float* __restrict__ thr, float key) {
    int i = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1)
        if (thr[i + step - 1] < key) i += step;
    if (i == 31 && thr[31] < key) i = 32;
    return i;
}

// The same count; the first two levels compare against the constant-bank copy
// (no shared-memory round trip on the critical path), the last three read
// the shared copy.
__device__ __forceinline__ int split_index_c(int axis, const float* __restrict__ thr, float key) {
    // sorted: #{t7, t15, t23 < key} * 8 is the first two levels of the search
    int i = ((c_thr[axis][7] < key) + (c_thr[axis][15] < key) + (c_thr[axis][23] < key)) * 8;
#pragma unroll
    for (int step = 4; step >= 1; step >>= 1)
        if (thr[i + step - 1] < key) i += step;
    if (i == 31 && c_thr[axis][31] < key) i = 32;
    return i;
}

__device__ __forceinline__ void load_q8(const float4* __restrict__ t, int row, float q[8]) {
    const float4 a = t[2 * row], b = t[2 * row + 1];
    q[0] = a.x; q[1] = a.y; q[2] = a.z; q[3] = a.w;
    q[4] = b.x; q[5] = b.y; q[6] = b.z; q[7] = b.w;
}

// (emission, direction sum) at the stencil centre offset delta; v as in
// load_stencil_z4, thr the shared-memory copy of c_thr, q1/q2 the Q1/Q2
// tables (shared memory in the persistent loop kernel, else global).  The
// all-|x| moment M[|x|,|y|,|z|] = 1/8 sum_s |x_s y_s z_s| is summed directly:
// its table (Q3, 1.15 MB) would cost a random 32-byte L2 gather per sample,
// the L1/TEX bottleneck measured by ncu (profiles/r1b_*).
__device__ __forceinline__ void moment_eval(const float v[27], float dx, float dy, float dz,
                                            const float* __restrict__ thr, const float4* q1,
                                            const float4* q2, float& emit, float& scat) {
    // separable transform of the stencil: V[kx][ky][kz]
    float V[27];
    {
        float t1[27];
        // along z (innermost)
#pragma unroll
        for (int l = 0; l < 9; ++l) {
            const float m = v[3 * l], c = v[3 * l + 1], p = v[3 * l + 2];
            t1[3 * l] = c;
            t1[3 * l + 1] = p - m;
            t1[3 * l + 2] = fmaf(-2.f, c, p + m);
        }
        float t2[27];
        // along y
#pragma unroll
        for (int jx = 0; jx < 3; ++jx)
#pragma unroll
            for (int kz = 0; kz < 3; ++kz) {
                const float m = t1[(jx * 3 + 0) * 3 + kz], c = t1[(jx * 3 + 1) * 3 + kz],
                            p = t1[(jx * 3 + 2) * 3 + kz];
                t2[(jx * 3 + 0) * 3 + kz] = c;
                t2[(jx * 3 + 1) * 3 + kz] = p - m;
                t2[(jx * 3 + 2) * 3 + kz] = fmaf(-2.f, c, p + m);
            }
        // along x
#pragma unroll
        for (int l = 0; l < 9; ++l) {
            const float m = t2[l], c = t2[9 + l], p = t2[18 + l];
            V[l] = c;
            V[9 + l] = p - m;
            V[18 + l] = fmaf(-2.f, c, p + m);
        }
    }
    const float hx = 0.5f * dx, hy = 0.5f * dy, hz = 0.5f * dz;
    // emission: basis values (1, x/2, |x|/2) at delta
    {
        const float ux[3] = {1.f, hx, fabsf(hx)}, uy[3] = {1.f, hy, fabsf(hy)}, uz[3] = {1.f, hz, fabsf(hz)};
        float e = 0.f;
#pragma unroll
        for (int kx = 0; kx < 3; ++kx)
#pragma unroll
            for (int ky = 0; ky < 3; ++ky) {
                const float uxy = ux[kx] * uy[ky];
#pragma unroll
                for (int kz = 0; kz < 3; ++kz) e = fmaf(V[(kx * 3 + ky) * 3 + kz], uxy * uz[kz], e);
            }
        emit = e;
    }
    // split indices and the sign-dependent moment tables
    const int ix = split_index(thr, -dx), iy = split_index(thr + kScatDirs, -dy),
              iz = split_index(thr + 2 * kScatDirs, -dz);
    float Q[8][8];  // Q[A mask: x=4,y=2,z=1][E mask]
#pragma unroll
    for (int e = 0; e < 8; ++e) Q[0][e] = c_q0[e];
    load_q8(q1, 0 * kSplits + ix, Q[4]);
    load_q8(q1, 1 * kSplits + iy, Q[2]);
    load_q8(q1, 2 * kSplits + iz, Q[1]);
    load_q8(q2, (0 * kSplits + ix) * kSplits + iy, Q[6]);
    load_q8(q2, (1 * kSplits + ix) * kSplits + iz, Q[5]);
    load_q8(q2, (2 * kSplits + iy) * kSplits + iz, Q[3]);
    // delta' monomials D[m] = prod_{a in m} delta'_a
    float D[8];
    D[0] = 1.f; D[4] = hx; D[2] = hy; D[1] = hz;
    D[6] = hx * hy; D[5] = hx * hz; D[3] = hy * hz; D[7] = D[6] * hz;
    float m222 = 0.f;
#if FVR_Q3_TABLE
    {
        float q3[8];
        load_q8(g_q3, (ix * kSplits + iy) * kSplits + iz, q3);
#pragma unroll
        for (int E = 0; E < 8; ++E) m222 = fmaf(D[7 ^ E], q3[E], m222);
    }
#else
#pragma unroll
    for (int d = 0; d < kScatDirs; ++d) {
        const float p = (dx + c_half_dir[0][d]) * (dy + c_half_dir[1][d]) * (dz + c_half_dir[2][d]);
        m222 += fabsf(p);
    }
    m222 *= 0.125f;
#endif
    float s = 0.f;
#pragma unroll
    for (int kx = 0; kx < 3; ++kx)
#pragma unroll
        for (int ky = 0; ky < 3; ++ky)
#pragma unroll
            for (int kz = 0; kz < 3; ++kz) {
                const int P = ((kx != 0) << 2) | ((ky != 0) << 1) | (kz != 0);
                const int A = ((kx == 2) << 2) | ((ky == 2) << 1) | (kz == 2);
                float M = 0.f;
                if (A == 7) {
                    M = m222;
                } else {
#pragma unroll
                    for (int E = 0; E < 8; ++E)
                        if ((E & ~P) == 0) M = fmaf(D[P ^ E], Q[A][E], M);
                }
                s = fmaf(V[(kx * 3 + ky) * 3 + kz], M, s);
            }
    scat = s;
}

// ---- packed (f32x2) moment evaluation -------------------------------------
//
// The same sums as moment_eval, arranged for Blackwell's paired FP32 ops
// (FADD2 / FMUL2 / FFMA2: one issue slot for two lanes of math):
//  * the stencil arrives as nine float4 z-runs r = (v[z-1], v[z], v[z+1], w)
//    whose register pairs (x, y) and (z, w) carry the x- and y-stages of the
//    separable transform two z-slots at a time (w is ignored);
//  * each sign table Q_A[E] (E bits x=4 y=2 z=1) is four float2 pairs (E, E|z),
//    and M_A[P] = sum_{E subset P} delta'^{P\E} Q_A[E] is its per-axis zeta
//    transform: 4 scalar FFMA (z, inside the pairs) + 2 FFMA2 (y) + 2 FFMA2 (x)
//    instead of one FFMA per (P, E) pair;
//  * the all-|x| moment pairs direction s with s + 16 against a broadcast delta.
// Rounding differs from moment_eval only in summation order.
__constant__ float2 c_half_dir2[3][kScatDirs / 2];  // (c_half_dir[a][s], c_half_dir[a][s + 16])

__device__ __forceinline__ float2 bcast2(float a) { return make_float2(a, a); }

// sx, sy: lattice strides -- compile-time constants for the specialised
// cubic lattices, so the nine loads are one pointer plus immediate offsets
__device__ __forceinline__ void load_stencil_z4_raw(const float4* __restrict__ Z4, int nch, int sx, int sy, int mx,
                                                    int my, int mz, float4 r[9]) {
    const float4* p = Z4 + (mx * sx + my * sy + (mz - 1)) * nch;
#pragma unroll
    for (int jx = 0; jx < 3; ++jx)
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) r[jx * 3 + jy] = __ldg(p + ((jx - 1) * sx + (jy - 1) * sy) * nch);
}


__device__ __forceinline__ void zeta8(float2 q[4], float hx, float hy, float hz) {
#pragma unroll
    for (int i = 0; i < 4; ++i) q[i].y = fmaf(hz, q[i].x, q[i].y);
    q[1] = __ffma2_rn(bcast2(hy), q[0], q[1]);
    q[3] = __ffma2_rn(bcast2(hy), q[2], q[3]);
    q[2] = __ffma2_rn(bcast2(hx), q[0], q[2]);
    q[3] = __ffma2_rn(bcast2(hx), q[1], q[3]);
}

__device__ __forceinline__ void load_q8x2(const float4* __restrict__ t, int row, float2 q[4]) {
    const float4 a = t[2 * row], b = t[2 * row + 1];
    q[0] = make_float2(a.x, a.y);
    q[1] = make_float2(a.z, a.w);
    q[2] = make_float2(b.x, b.y);
    q[3] = make_float2(b.z, b.w);
}

__device__ __forceinline__ float pick8(const float2 q[4], int P) { return (P & 1) ? q[P >> 1].y : q[P >> 1].x; }

// s += sum over the stencil moments k with A(k) = A of V[k] * M_A[P(k)]
template <int A>
__device__ __forceinline__ float dot_moments(const float V[27], const float2 q[4], float s) {
#pragma unroll
    for (int kx = 0; kx < 3; ++kx)
#pragma unroll
        for (int ky = 0; ky < 3; ++ky)
#pragma unroll
            for (int kz = 0; kz < 3; ++kz) {
                const int Ak = ((kx == 2) << 2) | ((ky == 2) << 1) | (kz == 2);
                const int Pk = ((kx != 0) << 2) | ((ky != 0) << 1) | (kz != 0);
                if (Ak == A) s = fmaf(V[(kx * 3 + ky) * 3 + kz], pick8(q, Pk), s);
            }
    return s;
}

__device__ __forceinline__ void moment_eval2(const float4 r[9], float dx, float dy, float dz,
                                             const float* __restrict__ thr, const float4* q1, const float4* q2,
                                             float& emit, float& scat) {
    float V[27];
    {
        // x- then y-stage on (z-1, z) and (z+1, w) pairs
        float2 a[9], b[9];
#pragma unroll
        for (int l = 0; l < 9; ++l) {
            a[l] = make_float2(r[l].x, r[l].y);
            b[l] = make_float2(r[l].z, r[l].w);
        }
        float2 ta[9], tb[9];
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) {  // along x: l = jx*3 + jy
            const float2 am = a[jy], ac = a[3 + jy], ap = a[6 + jy];
            const float2 bm = b[jy], bc = b[3 + jy], bp = b[6 + jy];
            ta[jy] = ac;
            ta[3 + jy] = __fadd2_rn(ap, make_float2(-am.x, -am.y));
            ta[6 + jy] = __ffma2_rn(bcast2(-2.f), ac, __fadd2_rn(ap, am));
            tb[jy] = bc;
            tb[3 + jy] = __fadd2_rn(bp, make_float2(-bm.x, -bm.y));
            tb[6 + jy] = __ffma2_rn(bcast2(-2.f), bc, __fadd2_rn(bp, bm));
        }
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {  // along y
            const float2 am = ta[kx * 3], ac = ta[kx * 3 + 1], ap = ta[kx * 3 + 2];
            const float2 bm = tb[kx * 3], bc = tb[kx * 3 + 1], bp = tb[kx * 3 + 2];
            a[kx * 3] = ac;
            a[kx * 3 + 1] = __fadd2_rn(ap, make_float2(-am.x, -am.y));
            a[kx * 3 + 2] = __ffma2_rn(bcast2(-2.f), ac, __fadd2_rn(ap, am));
            b[kx * 3] = bc;
            b[kx * 3 + 1] = __fadd2_rn(bp, make_float2(-bm.x, -bm.y));
            b[kx * 3 + 2] = __ffma2_rn(bcast2(-2.f), bc, __fadd2_rn(bp, bm));
        }
#pragma unroll
        for (int l = 0; l < 9; ++l) {  // along z, inside the pairs
            const float m = a[l].x, c = a[l].y, p = b[l].x;
            V[3 * l] = c;
            V[3 * l + 1] = p - m;
            V[3 * l + 2] = fmaf(-2.f, c, p + m);
        }
    }
    const float hx = 0.5f * dx, hy = 0.5f * dy, hz = 0.5f * dz;
    {
        const float ahx = fabsf(hx), ahy = fabsf(hy), ahz = fabsf(hz);
        float ey[3];
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
            float t[3];
#pragma unroll
            for (int ky = 0; ky < 3; ++ky) {
                const int l = kx * 3 + ky;
                t[ky] = fmaf(ahz, V[3 * l + 2], fmaf(hz, V[3 * l + 1], V[3 * l]));
            }
            ey[kx] = fmaf(ahy, t[2], fmaf(hy, t[1], t[0]));
        }
        emit = fmaf(ahx, ey[2], fmaf(hx, ey[1], ey[0]));
    }
    const int ix = split_index_c(0, thr, -dx), iy = split_index_c(1, thr + kScatDirs, -dy),
              iz = split_index_c(2, thr + 2 * kScatDirs, -dz);
#if FVR_Q3_TABLE
    // all-|x| moment from its table: issued first, consumed last
    const float4 q3a = __ldg(g_q3 + 2 * ((ix * kSplits + iy) * kSplits + iz));
    const float4 q3b = __ldg(g_q3 + 2 * ((ix * kSplits + iy) * kSplits + iz) + 1);
#endif
    float s = 0.f;
    {
        float2 q[4] = {make_float2(c_q0[0], c_q0[1]), make_float2(c_q0[2], c_q0[3]),
                       make_float2(c_q0[4], c_q0[5]), make_float2(c_q0[6], c_q0[7])};
        zeta8(q, hx, hy, hz);
        s = dot_moments<0>(V, q, s);
    }
    {
        float2 q[4];
        load_q8x2(q1, 0 * kSplits + ix, q);
        zeta8(q, hx, hy, hz);
        s = dot_moments<4>(V, q, s);
        load_q8x2(q1, 1 * kSplits + iy, q);
        zeta8(q, hx, hy, hz);
        s = dot_moments<2>(V, q, s);
        load_q8x2(q1, 2 * kSplits + iz, q);
        zeta8(q, hx, hy, hz);
        s = dot_moments<1>(V, q, s);
        load_q8x2(q2, (0 * kSplits + ix) * kSplits + iy, q);
        zeta8(q, hx, hy, hz);
        s = dot_moments<6>(V, q, s);
        load_q8x2(q2, (1 * kSplits + ix) * kSplits + iz, q);
        zeta8(q, hx, hy, hz);
        s = dot_moments<5>(V, q, s);
        load_q8x2(q2, (2 * kSplits + iy) * kSplits + iz, q);
        zeta8(q, hx, hy, hz);
        s = dot_moments<3>(V, q, s);
    }
#if FVR_Q3_TABLE
    {
        float2 q[4] = {make_float2(q3a.x, q3a.y), make_float2(q3a.z, q3a.w), make_float2(q3b.x, q3b.y),
                       make_float2(q3b.z, q3b.w)};
        zeta8(q, hx, hy, hz);
        s = fmaf(V[26], q[3].y, s);
    }
#else
    {
        // |x y| * |z| accumulated by FFMA2 with |.| operand modifiers; two
        // accumulators halve the dependent chain
        float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        const float2 DX = bcast2(dx), DY = bcast2(dy), DZ = bcast2(dz);
#pragma unroll
        for (int d = 0; d < kScatDirs / 2; ++d) {
            const float2 x = __fadd2_rn(DX, c_half_dir2[0][d]);
            const float2 y = __fadd2_rn(DY, c_half_dir2[1][d]);
            const float2 z = __fadd2_rn(DZ, c_half_dir2[2][d]);
            float2 xy = __fmul2_rn(x, y);
            xy.x = fabsf(xy.x);
            xy.y = fabsf(xy.y);
            acc[d & 1] = __ffma2_rn(xy, make_float2(fabsf(z.x), fabsf(z.y)), acc[d & 1]);
        }
        const float2 a2 = __fadd2_rn(acc[0], acc[1]);
        s = fmaf(V[26], 0.125f * (a2.x + a2.y), s);
    }
#endif
    scat = s;
}

// ---- stencil weights: the evaluation as one dot product per channel --------
//
// Both sums are linear in the stencil: e = sum_j v_j hat_j(delta) (the
// trilinear hat weights) and the direction sum S = sum_k V[k] M[k] =
// sum_j v_j W_j with W = (T^T)^{(x)3} M, T the per-axis basis transform of
// moment_eval.  So  sigma_a e + kappa S = kappa * sum_j v_j Omega_j  with
// Omega = W + (sigma_a / kappa) hat, computed once per sample and shared by
// every channel; a channel then costs its nine stencil loads and one
// 27-term dot (9 FFMA2 on the (z-1, z) register pairs + 9 FFMA).
// om01[l] = (Omega[l][z-1], Omega[l][z]), om2[l] = Omega[l][z+1], l = jx*3 + jy.
__device__ __forceinline__ void moment_omega(float dx, float dy, float dz, const float* __restrict__ thr,
                                             const float4* q1, const float4* q2, float ek, float2 om01[9],
                                             float om2[9]) {
    const float hx = 0.5f * dx, hy = 0.5f * dy, hz = 0.5f * dz;
    const int ix = split_index_c(0, thr, -dx), iy = split_index_c(1, thr + kScatDirs, -dy),
              iz = split_index_c(2, thr + 2 * kScatDirs, -dz);
    // moments per (kx, ky): M01 = (M[k,0], M[k,1]) = q_A[P >> 1], M2 = M[k,2] = q_{A|z}[P >> 1].y
    float2 M01[9];
    float M2[9];
    auto put = [&](int A, const float2 q[4]) {
#pragma unroll
        for (int kx = 0; kx < 3; ++kx)
#pragma unroll
            for (int ky = 0; ky < 3; ++ky) {
                const int Axy = ((kx == 2) << 2) | ((ky == 2) << 1);
                const int pi = ((kx != 0) << 1) | (ky != 0);
                if (Axy == A) M01[kx * 3 + ky] = q[pi];
                if ((Axy | 1) == A) M2[kx * 3 + ky] = q[pi].y;
            }
    };
    {
        float2 q[4] = {make_float2(c_q0[0], c_q0[1]), make_float2(c_q0[2], c_q0[3]),
                       make_float2(c_q0[4], c_q0[5]), make_float2(c_q0[6], c_q0[7])};
        zeta8(q, hx, hy, hz);
        put(0, q);
    }
    {
        float2 q[4];
        load_q8x2(q1, 0 * kSplits + ix, q);
        zeta8(q, hx, hy, hz);
        put(4, q);
        load_q8x2(q1, 1 * kSplits + iy, q);
        zeta8(q, hx, hy, hz);
        put(2, q);
        load_q8x2(q1, 2 * kSplits + iz, q);
        zeta8(q, hx, hy, hz);
        put(1, q);
        load_q8x2(q2, (0 * kSplits + ix) * kSplits + iy, q);
        zeta8(q, hx, hy, hz);
        put(6, q);
        load_q8x2(q2, (1 * kSplits + ix) * kSplits + iz, q);
        zeta8(q, hx, hy, hz);
        put(5, q);
        load_q8x2(q2, (2 * kSplits + iy) * kSplits + iz, q);
        zeta8(q, hx, hy, hz);
        put(3, q);
    }
    {
        // all-|x| moment, directions s and s + 16 paired
        float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        const float2 DX = bcast2(dx), DY = bcast2(dy), DZ = bcast2(dz);
#pragma unroll
        for (int d = 0; d < kScatDirs / 2; ++d) {
            const float2 x = __fadd2_rn(DX, c_half_dir2[0][d]);
            const float2 y = __fadd2_rn(DY, c_half_dir2[1][d]);
            const float2 z = __fadd2_rn(DZ, c_half_dir2[2][d]);
            float2 xy = __fmul2_rn(x, y);
            xy.x = fabsf(xy.x);
            xy.y = fabsf(xy.y);
            acc[d & 1] = __ffma2_rn(xy, make_float2(fabsf(z.x), fabsf(z.y)), acc[d & 1]);
        }
        const float2 a2 = __fadd2_rn(acc[0], acc[1]);
        M2[8] = 0.125f * (a2.x + a2.y);
    }
    // T^T along z (inside the lines): (M0, M1, M2) -> (M2 - M1, M0 - 2 M2, M1 + M2)
    float2 W01[9];
    float W2[9];
#pragma unroll
    for (int l = 0; l < 9; ++l) {
        const float m0 = M01[l].x, m1 = M01[l].y, m2 = M2[l];
        W01[l] = make_float2(m2 - m1, fmaf(-2.f, m2, m0));
        W2[l] = m1 + m2;
    }
    // along y (l = kx*3 + ky), then along x, on the z-pairs
#pragma unroll
    for (int kx = 0; kx < 3; ++kx) {
        const float2 a0 = W01[kx * 3], a1 = W01[kx * 3 + 1], a2 = W01[kx * 3 + 2];
        const float b0 = W2[kx * 3], b1 = W2[kx * 3 + 1], b2 = W2[kx * 3 + 2];
        W01[kx * 3] = __fadd2_rn(a2, make_float2(-a1.x, -a1.y));
        W01[kx * 3 + 1] = __ffma2_rn(bcast2(-2.f), a2, a0);
        W01[kx * 3 + 2] = __fadd2_rn(a1, a2);
        W2[kx * 3] = b2 - b1;
        W2[kx * 3 + 1] = fmaf(-2.f, b2, b0);
        W2[kx * 3 + 2] = b1 + b2;
    }
#pragma unroll
    for (int jy = 0; jy < 3; ++jy) {
        const float2 a0 = W01[jy], a1 = W01[3 + jy], a2 = W01[6 + jy];
        const float b0 = W2[jy], b1 = W2[3 + jy], b2 = W2[6 + jy];
        W01[jy] = __fadd2_rn(a2, make_float2(-a1.x, -a1.y));
        W01[3 + jy] = __ffma2_rn(bcast2(-2.f), a2, a0);
        W01[6 + jy] = __fadd2_rn(a1, a2);
        W2[jy] = b2 - b1;
        W2[3 + jy] = fmaf(-2.f, b2, b0);
        W2[6 + jy] = b1 + b2;
    }
    // hat weights (max(-x,0), 1 - |x|, max(x,0)) per axis; sigma_a/kappa folded into x
    const float hatx[3] = {ek * fmaxf(-dx, 0.f), ek * (1.f - fabsf(dx)), ek * fmaxf(dx, 0.f)};
    const float haty[3] = {fmaxf(-dy, 0.f), 1.f - fabsf(dy), fmaxf(dy, 0.f)};
    const float2 hz01 = make_float2(fmaxf(-dz, 0.f), 1.f - fabsf(dz));
    const float hz2 = fmaxf(dz, 0.f);
#pragma unroll
    for (int jx = 0; jx < 3; ++jx)
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) {
            const int l = jx * 3 + jy;
            const float hxy = hatx[jx] * haty[jy];
            om01[l] = __ffma2_rn(bcast2(hxy), hz01, W01[l]);
            om2[l] = fmaf(hxy, hz2, W2[l]);
        }
}

// sum_j v_j Omega_j for one channel's stencil (r as in load_stencil_z4_raw)
__device__ __forceinline__ float omega_dot(const float4 r[9], const float2 om01[9], const float om2[9]) {
    float2 a[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    float b = 0.f;
#pragma unroll
    for (int l = 0; l < 9; ++l) {
        a[l & 1] = __ffma2_rn(make_float2(r[l].x, r[l].y), om01[l], a[l & 1]);
        b = fmaf(r[l].z, om2[l], b);
    }
    const float2 s = __fadd2_rn(a[0], a[1]);
    return s.x + s.y + b;
}

}  // namespace fvr
