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
#include <algorithm>
#include <type_traits>
#include <vector>

#include "fvr_stencil.cuh"

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

// Fast evaluator over a packed layout (fvr_stencil.cuh).  Per sample the
// lattice coordinate is q = qb + k*d in fp64 (continuous quantities only);
// the sample count, and for samples within half a voxel of a box face the
// exact gather points, follow the reference arithmetic.
template <int NCH, bool SCAT, int NS = 0>
__device__ __forceinline__ void march_render_fast(const double o[3], const double d[3], const Geom& g,
                                                  const float* __restrict__ values, int plane,
                                                  const float4* __restrict__ layout,
                                                  const uint8_t* __restrict__ occ,
                                                  const RenderConsts& rc, const float* __restrict__ thr,
                                                  const float4* q1, const float4* q2, double out[NCH]) {
    // NS > 0: cubic lattice of NS key points per axis, strides known at compile time
    const int SY = NS ? NS : g.sy, SX = NS ? NS * NS : g.sx;
    double l[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) l[c] = 0.0;
    double t_dst = 1.0;
    double te, tx;
    if (slab_span(o, d, g, te, tx)) {
        const int n = sample_count(te, tx, g.edge);
        const double t0 = te - 0.5 * g.edge;
        double qb[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) qb[a] = ((o[a] - g.lo[a]) + t0 * d[a]) * g.inv_edge;
        const double nmax[3] = {(double)g.nx, (double)g.ny, (double)g.nz};
        int k = 1;
        // occupancy probe of sample kk, issued one sample ahead of its use so
        // the load overlaps the evaluation of the current sample
        auto probe = [&](int kk) -> int {
            if (!occ || kk > n) return 0;
            int mm[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const double qa = fma((double)kk, d[a], qb[a]);
                const int na = a == 0 ? g.nx : (a == 1 ? g.ny : g.nz);
                if (SCAT) {
                    mm[a] = min(max((int)rint(qa), 0), na);
                } else {
                    int ca;
                    float fa;
                    cell_frac(qa, na, ca, fa);
                    mm[a] = ca;
                }
            }
            return (int)__ldg(occ + (unsigned)(mm[0] * SX + mm[1] * SY + mm[2]));
        };
        int D_next = probe(1);
        while (k <= n) {
            double q[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) q[a] = fma((double)k, d[a], qb[a]);
            int m[3];
            float dl[3];
            bool interior = true;
            if (!SCAT) {
                // cell of the trilinear read (the 2x2x2 corners are within distance 1 of it)
                cell_frac(q[0], g.nx, m[0], dl[0]);
                cell_frac(q[1], g.ny, m[1], dl[1]);
                cell_frac(q[2], g.nz, m[2], dl[2]);
            } else {
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    interior = interior && q[a] >= 0.5 + 1e-7 && q[a] <= nmax[a] - 0.5 - 1e-7;
                    const double r = rint(q[a]);
                    m[a] = min(max((int)r, 0), a == 0 ? g.nx : (a == 1 ? g.ny : g.nz));
                    dl[a] = (float)(q[a] - (double)m[a]);
                }
            }
            // Empty-space skipping.  dist[j] is a lower bound on the Chebyshev
            // distance from key point j to the nearest key point that may be
            // non-zero.  dist <= 1: the sample's neighbourhood may be live.
            // Otherwise samples k .. k+s-1 read only zeros and add exactly 0,
            // s = max(1, dist-2) (sample k+j stays within j+1 of m, its
            // neighbourhood within j+2).  The skip is the minimum over the
            // warp so the lanes stay aligned on k; the transparency still
            // advances by repeated multiplication, as in the reference.
            const int D = D_next;
            const unsigned act = __activemask();
            if (__any_sync(act, D <= 1)) {
                D_next = probe(k + 1);
                if (D <= 1) {
                    // Several channels: the interior scattering samples compute the
                    // stencil weights Omega once and every channel is one dot
                    // (moment_omega); one channel: the transform-then-moments form
                    // (moment_eval2) is ~7% faster (no spills).
                    constexpr bool kOmega = FVR_OMEGA && SCAT && NCH > 1;
                    float2 om01[kOmega ? 9 : 1];
                    float om2[kOmega ? 9 : 1];
                    if (kOmega && interior)
                        moment_omega(dl[0], dl[1], dl[2], thr, q1, q2, (float)(rc.sigma_a / rc.scat_scale), om01, om2);
#pragma unroll 1
                    for (int c = 0; c < NCH; ++c) {
                        float e = 0.f, acc = 0.f;
                        if (!SCAT) {
                            e = tri_yzq(layout + c, NCH, g, m[0], m[1], m[2], dl[0], dl[1], dl[2]);
                        } else if (kOmega && interior) {
                            float4 r[9];
                            load_stencil_z4_raw(layout + c, NCH, SX, SY, m[0], m[1], m[2], r);
                            // a sum of non-negative terms in exact arithmetic; the expanded
                            // form can round a vanishing sum below zero
                            acc = fmaxf(omega_dot(r, om01, om2), 0.f);
                            l[c] += t_dst * (rc.tau * ((double)acc * rc.scat_scale));
                            continue;
                        } else if (interior) {
#if FVR_MOMENT_PACKED
                            float4 r[9];
                            load_stencil_z4_raw(layout + c, NCH, SX, SY, m[0], m[1], m[2], r);
                            moment_eval2(r, dl[0], dl[1], dl[2], thr, q1, q2, e, acc);
#else
                            float v[27];
                            load_stencil_z4(layout + c, NCH, g, m[0], m[1], m[2], v);
                            moment_eval(v, dl[0], dl[1], dl[2], thr, q1, q2, e, acc);
#endif
                            // sums of non-negative terms in exact arithmetic; the
                            // expanded form can round a vanishing sum below zero
                            e = fmaxf(e, 0.f);
                            acc = fmaxf(acc, 0.f);
                        } else {
                            // within half a voxel of a box face: the reference's exact
                            // per-direction in-box test masks the gathers
                            float v[27];
                            load_stencil_clamped(values + (int64_t)c * plane, g, m[0], m[1], m[2], v);
                            bool any = false;
#pragma unroll
                            for (int j = 0; j < 27; ++j) any = any || v[j] != 0.f;
                            if (any) {
                                double p[3];
                                sample_pos(o, d, te, g.edge, k, p);
                                const uint32_t mask = inbox_mask(p, g, rc.half_gather);
                                Stencil st;
                                stencil_from(v, st);
                                e = stencil_tri(st, dl[0], dl[1], dl[2]);
                                acc = stencil_scatter<true>(st, dl[0], dl[1], dl[2], mask);
                            }
                        }
                        const double l_src = SCAT ? rc.sigma_a * (double)e + (double)acc * rc.scat_scale
                                                  : rc.sigma_a * (double)e;
                        l[c] += t_dst * (rc.tau * l_src);
                    }
                }
                t_dst *= rc.one_minus_tau;
                ++k;
            } else {
                int s = D - 2 > 1 ? D - 2 : 1;
                s = (int)__reduce_min_sync(act, (unsigned)s);
                s = min(s, n - k + 1);
                for (int j = 0; j < s; ++j) t_dst *= rc.one_minus_tau;
                k += s;
                D_next = probe(k);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < NCH; ++c) out[c] = l[c] + t_dst * rc.bg[c];
}

// Empty-space distance map.  M[j] = 1 when key point j may be non-zero: it
// is positive in some channel, or flagged by `force` (the hull key points of
// the loop, whose values change).  dist[j] = min(L-inf distance from j to the
// nearest M = 1 key point, kDistCap + 1), computed separably (z, y, x passes):
// f_z = 1-D distance along z; g = min_dy max(|dy|, f_z); D = min_dx max(|dx|, g).
// Windows are limited to +-kDistCap, which keeps every value a lower bound on
// the true distance -- what the skip in march_render_fast needs.
constexpr int kDistCap = 30;

__global__ void dist_seed_kernel(const float* __restrict__ values, int64_t n_kp, int nch,
                                 const uint8_t* __restrict__ force, uint8_t* __restrict__ out) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_kp;
         j += (int64_t)gridDim.x * blockDim.x) {
        bool m = force && force[j];
        for (int c = 0; c < nch && !m; ++c) m = values[c * n_kp + j] > 0.f;
        out[j] = m ? 0 : (uint8_t)(kDistCap + 1);
    }
}

// one separable pass along an axis with stride `st` and extent `len`
__global__ void dist_pass_kernel(const uint8_t* __restrict__ in, int64_t n_kp, int st, int len, int period,
                                 uint8_t* __restrict__ out) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_kp;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int pos = (int)((j / st) % period);
        int best = in[j];
        for (int dd = 1; dd <= kDistCap && dd < best; ++dd) {
            if (pos - dd >= 0) best = min(best, max(dd, (int)in[j - (int64_t)dd * st]));
            if (pos + dd < len) best = min(best, max(dd, (int)in[j + (int64_t)dd * st]));
        }
        out[j] = (uint8_t)best;
    }
}

// The same pass with W whole lines staged in shared memory (one CTA per W
// lines): the up-to-2 * kDistCap window reads hit shared memory instead of
// L1/L2 (config 2: 65 -> ~15 us per pass).  AXIS 0 = z (contiguous lines),
// 1 = y, 2 = x; lines of the y and x passes are grouped by consecutive base
// address (adjacent z), so the tile loads are coalesced either way.
template <int AXIS>
__global__ void __launch_bounds__(256) dist_lines_kernel(const uint8_t* __restrict__ in, int nx1, int ny1, int nz1,
                                                         uint8_t* __restrict__ out) {
    constexpr int W = AXIS == 0 ? 8 : 32;  // lines per CTA
    extern __shared__ uint8_t s_line[];     // [W][len] (AXIS 0) or [len][W]
    const int64_t sx = (int64_t)ny1 * nz1;
    const int len = AXIS == 0 ? nz1 : AXIS == 1 ? ny1 : nx1;
    const int64_t st = AXIS == 0 ? 1 : AXIS == 1 ? nz1 : sx;
    const int64_t n_lines = AXIS == 0 ? (int64_t)nx1 * ny1 : AXIS == 1 ? (int64_t)nx1 * nz1 : sx;
    const int64_t l0 = (int64_t)blockIdx.x * W;
    auto base = [&](int64_t l) -> int64_t {
        return AXIS == 0 ? l * nz1 : AXIS == 1 ? (l / nz1) * sx + l % nz1 : l;
    };
    auto slot = [&](int w, int p) { return AXIS == 0 ? w * len + p : p * W + w; };
    const int n = len * W;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int w = AXIS == 0 ? i / len : i % W, p = AXIS == 0 ? i % len : i / W;
        const int64_t l = l0 + w;
        s_line[slot(w, p)] = l < n_lines ? in[base(l) + p * st] : (uint8_t)0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int w = AXIS == 0 ? i / len : i % W, p = AXIS == 0 ? i % len : i / W;
        const int64_t l = l0 + w;
        if (l >= n_lines) continue;
        int best = s_line[slot(w, p)];
        for (int dd = 1; dd <= kDistCap && dd < best; ++dd) {
            if (p - dd >= 0) best = min(best, max(dd, (int)s_line[slot(w, p - dd)]));
            if (p + dd < len) best = min(best, max(dd, (int)s_line[slot(w, p + dd)]));
        }
        out[base(l) + p * st] = (uint8_t)best;
    }
}

// Packed layouts of max(v, 0): see fvr_stencil.cuh.
__global__ void pack_layout_kernel(const float* __restrict__ values, int64_t n_kp, int nch, int kind,
                                   int sy, float4* __restrict__ out) {
    const int64_t total = n_kp * nch;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i / n_kp, j = i - c * n_kp;
        const float* v = values + c * n_kp;
        auto at = [&](int64_t k) { return k < n_kp ? fmaxf(v[k], 0.f) : 0.f; };
        float4 r;
        if (kind == kLayoutZ4)
            r = make_float4(at(j), at(j + 1), at(j + 2), at(j + 3));
        else
            r = make_float4(at(j), at(j + 1), at(j + sy), at(j + sy + 1));
        out[j * nch + c] = r;  // channels interleaved per key point
    }
}

// ---- mode dispatch ------------------------------------------------------------
// MODE: 0 general emission, 1 general scattering g = 0, 2 general scattering
// g != 0, 3 fast emission (YZQ layout), 4 fast scattering (Z4 layout).
enum { kModePlain = 0, kModeScatG0 = 1, kModeScatG = 2, kModeFastPlain = 3, kModeFastScat = 4 };

template <int NCH, int MODE>
__device__ __forceinline__ void march_dispatch(const double o[3], const double d[3], const Geom& g,
                                               const float* __restrict__ values, int plane,
                                               const float4* __restrict__ layout,
                                               const uint8_t* __restrict__ occ,
                                               const RenderConsts& rc, const double* __restrict__ scat,
                                               const float* __restrict__ thr, double out[NCH]) {
    if (MODE == kModePlain) march_render<NCH, false, true>(o, d, g, values, plane, rc, scat, out);
    if (MODE == kModeScatG0) march_render<NCH, true, true>(o, d, g, values, plane, rc, scat, out);
    if (MODE == kModeScatG) march_render<NCH, true, false>(o, d, g, values, plane, rc, scat, out);
    if (MODE == kModeFastPlain) march_render_fast<NCH, false>(o, d, g, values, plane, layout, occ, rc, thr, g_q1, g_q2, out);
    if (MODE == kModeFastScat) march_render_fast<NCH, true>(o, d, g, values, plane, layout, occ, rc, thr, g_q1, g_q2, out);
}

// Shared-memory copy of the sorted gather offsets (moment split search).
__device__ __forceinline__ void load_thresholds(float* s_thr) {
    for (int i = threadIdx.x; i < 3 * kScatDirs; i += blockDim.x) s_thr[i] = (&c_thr[0][0])[i];
    __syncthreads();
}

// ---- _kernels.render_rays drop-in -----------------------------------------

template <int NCH, int MODE>
__global__ void __launch_bounds__(128) render_rays_kernel(double ox, double oy, double oz,
                                                          const double* __restrict__ dirs,
                                                          int64_t n_rays,
                                                          const float* __restrict__ values,
                                                          int plane, const float4* __restrict__ layout,
                                                          const uint8_t* __restrict__ occ, Geom g, RenderConsts rc,
                                                          const double* __restrict__ scat,
                                                          double* __restrict__ out) {
    __shared__ float s_thr[3 * kScatDirs];
    if (MODE == kModeFastScat) load_thresholds(s_thr);
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rays) return;
    const double o[3] = {ox, oy, oz};
    const double d[3] = {dirs[3 * r], dirs[3 * r + 1], dirs[3 * r + 2]};
    double res[NCH];
    march_dispatch<NCH, MODE>(o, d, g, values, plane, layout, occ, rc, scat, s_thr, res);
#pragma unroll
    for (int c = 0; c < NCH; ++c) out[r * NCH + c] = res[c];
}

// ---- render_pixels / render_view: rays built on the device ----------------

template <int NCH, int MODE>
__global__ void __launch_bounds__(128) render_pixels_kernel(fvr_camera_t cam,
                                                            const double* __restrict__ us,
                                                            const double* __restrict__ vs,
                                                            int64_t n,
                                                            const float* __restrict__ values,
                                                            int plane, const float4* __restrict__ layout,
                                                            const uint8_t* __restrict__ occ, Geom g, RenderConsts rc,
                                                            const double* __restrict__ scat,
                                                            double* __restrict__ out) {
    __shared__ float s_thr[3 * kScatDirs];
    if (MODE == kModeFastScat) load_thresholds(s_thr);
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
    march_dispatch<NCH, MODE>(cam.center, d, g, values, plane, layout, occ, rc, scat, s_thr, res);
#pragma unroll
    for (int c = 0; c < NCH; ++c) out[i * NCH + c] = res[c];
}

// ---- render_views: every pixel of several same-size views, one launch ------

template <int NCH, int MODE>
__global__ void __launch_bounds__(128) render_views_kernel(const fvr_camera_t* __restrict__ cams, int width,
                                                           int height, const float* __restrict__ values,
                                                           int plane, const float4* __restrict__ layout,
                                                           const uint8_t* __restrict__ occ, Geom g,
                                                           RenderConsts rc, const double* __restrict__ scat,
                                                           float* __restrict__ out) {
    __shared__ float s_thr[3 * kScatDirs];
    if (MODE == kModeFastScat) load_thresholds(s_thr);
    const int view = blockIdx.y;
    // 8x4 pixel patches per warp for ray coherence
    const int lane = threadIdx.x & 31;
    const int unit = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int units_x = (width + 7) / 8;
    const int col = (unit % units_x) * 8 + (lane & 7), row = (unit / units_x) * 4 + (lane >> 3);
    if (col >= width || row >= height) return;
    const fvr_camera_t& cam = cams[view];
    double d[3];
    pixel_dir(cam, (double)col + 0.5, (double)row + 0.5, d);
    double res[NCH];
    march_dispatch<NCH, MODE>(cam.center, d, g, values, plane, layout, occ, rc, scat, s_thr, res);
    float* o = out + (((int64_t)view * height + row) * width + col) * NCH;
#pragma unroll
    for (int c = 0; c < NCH; ++c) o[c] = (float)res[c];
}

// ---- loop render: every bbox pixel of every view + residual + RMSE partials

// Work unit = one warp = an 8x4 patch of bbox pixels of one view.  Each warp
// reduces its 32 squared residuals itself (fixed shuffle tree) and writes one
// f64 partial per unit, so no CTA-wide barrier ever makes a warp wait for the
// longest ray of its neighbours.
constexpr int kUnitW = 8, kUnitH = 4, kBlockThreads = 256, kWarpsPerBlock = kBlockThreads / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// NCH channels share the rays: src is (NCH, V, h, w), residual (V, h, w,
// pitch) with the channels interleaved (pitch 1 for one channel, 4 for
// three: one 16-byte load serves a pixel's channels in the gather), values
// NCH lattice planes, sq_partials[c * sq_stride + unit].
template <int MODE, int NS = 0, int NCH = 1>
__device__ __forceinline__ void render_unit(int unit, int units_x, int units_per_view,
                                            const fvr_camera_t* __restrict__ cams, int n_views, int u0, int v0,
                                            int w, int h, const float* __restrict__ src,
                                            const float* __restrict__ values, int plane,
                                            const float4* __restrict__ layout, const uint8_t* __restrict__ occ,
                                            const Geom& g, const RenderConsts& rc,
                                            const double* __restrict__ scat, const float* thr, const float4* q1,
                                            const float4* q2, float* __restrict__ residual,
                                            double* __restrict__ sq_partials, int64_t sq_stride) {
    const int lane = threadIdx.x & 31;
    const int view = unit / units_per_view, u = unit - view * units_per_view;
    const int ux = u % units_x, uy = u / units_x;
    const int col = ux * kUnitW + (lane % kUnitW);
    const int row = uy * kUnitH + (lane / kUnitW);
    const int64_t cstride = (int64_t)n_views * h * w;
    double sq[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) sq[c] = 0.0;
    if (col < w && row < h) {
        const fvr_camera_t& cam = cams[view];
        double d[3];
        pixel_dir(cam, (double)(u0 + col) + 0.5, (double)(v0 + row) + 0.5, d);
        double rec[NCH];
        if (MODE == kModeFastScat)
            march_render_fast<NCH, true, NS>(cam.center, d, g, values, plane, layout, occ, rc, thr, q1, q2, rec);
        else
            march_dispatch<NCH, MODE>(cam.center, d, g, values, plane, layout, occ, rc, scat, thr, rec);
        const int64_t pix = ((int64_t)view * h + row) * w + col;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const double r = (double)src[c * cstride + pix] - rec[c];
            residual[pix * kResPitch<NCH> + c] = (float)r;  // channels interleaved per pixel
            sq[c] = r * r;
        }
    }
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const double tot = warp_sum(sq[c]);
        if (lane == 0) sq_partials[c * sq_stride + unit] = tot;
    }
}

template <int NCH>
__device__ __forceinline__ bool all_done(const fvr_loop_state_t* __restrict__ state) {
    if (!state) return false;
    bool d = true;
#pragma unroll
    for (int c = 0; c < NCH; ++c) d = d && state[c].done;
    return d;
}

template <int MODE, int NCH>
__global__ void __launch_bounds__(kBlockThreads) loop_render_kernel(
    const fvr_camera_t* __restrict__ cams, int n_views, int u0, int v0, int w, int h, int units_x,
    int units_per_view, int n_units, const float* __restrict__ src, const float* __restrict__ values, int plane,
    const float4* __restrict__ layout, const uint8_t* __restrict__ occ, Geom g, RenderConsts rc,
    const double* __restrict__ scat, float* __restrict__ residual, double* __restrict__ sq_partials,
    int64_t sq_stride, const fvr_loop_state_t* __restrict__ state) {
    if (all_done<NCH>(state)) return;
    __shared__ float s_thr[3 * kScatDirs];
    if (MODE == kModeFastScat) load_thresholds(s_thr);
    const int unit = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (unit >= n_units) return;
    render_unit<MODE == kModeFastScat ? kModeScatG0 : MODE, 0, NCH>(
        unit, units_x, units_per_view, cams, n_views, u0, v0, w, h, src, values, plane, layout, occ, g, rc, scat,
        s_thr, g_q1, g_q2, residual, sq_partials, sq_stride);
}

// Persistent variant for the single-scattering fast path: two CTAs per SM,
// each stages the Q1/Q2 moment tables (107 KB) and the split thresholds in
// shared memory once; every warp then walks the unit list on its own.
constexpr int kQ1Vec = 3 * kSplits * 2, kQ2Vec = 3 * kSplits * kSplits * 2;
constexpr size_t kScatSmem = sizeof(float4) * (kQ1Vec + kQ2Vec) + sizeof(float) * 3 * kScatDirs;

// One 512-thread CTA per SM: the tables are staged once per SM (105 KB), which
// leaves the rest of the 256 KB L1/shared array to cache the stencil loads.
#ifndef FVR_SCAT_THREADS
#define FVR_SCAT_THREADS 512
#endif
constexpr int kScatThreads = FVR_SCAT_THREADS, kScatWarps = kScatThreads / 32,
              kScatCtasPerSm = kScatThreads >= 512 ? 1 : 512 / kScatThreads;

template <int NS, int NCH>
__global__ void __launch_bounds__(kScatThreads, kScatCtasPerSm) loop_render_scat_kernel(
    const fvr_camera_t* __restrict__ cams, int n_views, int u0, int v0, int w, int h, int units_x,
    int units_per_view, int n_units, const float* __restrict__ src, const float* __restrict__ values, int plane,
    const float4* __restrict__ layout, const uint8_t* __restrict__ occ, Geom g, RenderConsts rc,
    float* __restrict__ residual, double* __restrict__ sq_partials, int64_t sq_stride,
    fvr_loop_state_t* __restrict__ state) {
    if (all_done<NCH>(state)) return;
    extern __shared__ float4 smem[];
    float4* s_q1 = smem;
    float4* s_q2 = smem + kQ1Vec;
    float* s_thr = reinterpret_cast<float*>(smem + kQ1Vec + kQ2Vec);
    for (int i = threadIdx.x; i < kQ1Vec; i += blockDim.x) s_q1[i] = g_q1[i];
    for (int i = threadIdx.x; i < kQ2Vec; i += blockDim.x) s_q2[i] = g_q2[i];
    for (int i = threadIdx.x; i < 3 * kScatDirs; i += blockDim.x) s_thr[i] = (&c_thr[0][0])[i];
    __syncthreads();
    const int stride = gridDim.x * kScatWarps;
    if (!state) {
        for (int unit = blockIdx.x * kScatWarps + (threadIdx.x >> 5); unit < n_units; unit += stride)
            render_unit<kModeFastScat, NS, NCH>(unit, units_x, units_per_view, cams, n_views, u0, v0, w, h, src,
                                                values, plane, layout, occ, g, rc, nullptr, s_thr, s_q1, s_q2,
                                                residual, sq_partials, sq_stride);
        return;
    }
    // Work queue: a unit's cost ranges over two orders of magnitude (rays
    // through the flame core vs. the bbox margin), so a static round-robin
    // leaves most SMs idle behind the slowest warps.  Each warp takes the next
    // unit from a global counter (channel 0's state); the last warp to find the
    // queue empty resets it for the next iteration (every warp retires once).
    const int lane = threadIdx.x & 31;
    int* next = &state->work_next;
    for (;;) {
        int unit = 0;
        if (lane == 0) unit = atomicAdd(next, 1);
        unit = __shfl_sync(0xffffffffu, unit, 0);
        if (unit >= n_units) break;
        render_unit<kModeFastScat, NS, NCH>(unit, units_x, units_per_view, cams, n_views, u0, v0, w, h, src,
                                            values, plane, layout, occ, g, rc, nullptr, s_thr, s_q1, s_q2,
                                            residual, sq_partials, sq_stride);
    }
    if (lane == 0) {
        __threadfence();
        if (atomicAdd(&state->work_retired, 1) == stride - 1) {
            atomicExch(next, 0);
            atomicExch(&state->work_retired, 0);
        }
    }
}

}  // namespace fvr

#include "fvr_rplan.cuh"

using namespace fvr;

namespace {

bool g_dirs_ready = false;
double g_dirs_host[3 * kScatDirs];

int pick_mode(const fvr_render_params_t& p, const float4* layout, bool& scat) {
    scat = p.scattering && p.sigma_s > 0.0;
    if (!scat) return layout ? kModeFastPlain : kModePlain;
    const bool g0 = p.phase_g == 0.0;
    const bool stencil_ok = g0 && p.n_scat == kScatDirs && layout && g_dirs_ready;
    return stencil_ok ? kModeFastScat : (g0 ? kModeScatG0 : kModeScatG);
}

// the stencil path also needs gather_dist == edge (all gathers within the 3^3 block)
int effective_mode(const fvr_render_params_t& p, const fvr_grid_t& grid, const float4* layout, bool& scat) {
    int mode = pick_mode(p, layout, scat);
    if (mode == kModeFastScat && p.gather_dist != grid.edge) mode = kModeScatG0;
    return mode;
}

int layout_kind(int mode) {
    return mode == kModeFastScat ? kLayoutZ4 : (mode == kModeFastPlain ? kLayoutYZQ : kLayoutNone);
}

int pack(const float* values, int nch, const fvr_grid_t& grid, int kind, float4* out, cudaStream_t st) {
    const int64_t n_kp = (int64_t)(grid.nx + 1) * (grid.ny + 1) * (grid.nz + 1);
    int64_t blocks = (n_kp * nch + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    pack_layout_kernel<<<(unsigned)blocks, 256, 0, st>>>(values, n_kp, nch, kind, grid.nz + 1, out);
    return check_launch("pack_layout");
}

int occupancy(const float* values, int nch, const uint8_t* force, const fvr_grid_t& grid, uint8_t* occ,
              cudaStream_t st) {
    const int64_t n_kp = (int64_t)(grid.nx + 1) * (grid.ny + 1) * (grid.nz + 1);
    // ping-pong scratch, grown on demand and kept for the process
    static uint8_t* scratch = nullptr;
    static int64_t scratch_size = 0;
    if (scratch_size < n_kp) {
        if (scratch) cudaFree(scratch);
        scratch = nullptr;
        scratch_size = 0;
        if (cudaMalloc(&scratch, (size_t)n_kp) != cudaSuccess) return set_error(FVR_ERR_CUDA, "cudaMalloc failed");
        scratch_size = n_kp;
    }
    auto blocks = [](int64_t n) { int64_t b = (n + 255) / 256; return (unsigned)(b > 148 * 32 ? 148 * 32 : b); };
    const int sy = grid.nz + 1, sx = (grid.ny + 1) * (grid.nz + 1);
    dist_seed_kernel<<<blocks(n_kp), 256, 0, st>>>(values, n_kp, nch, force, scratch);
    const int nx1 = grid.nx + 1, ny1 = grid.ny + 1, nz1 = grid.nz + 1;
    if (std::max(nx1, std::max(ny1, nz1)) <= 1536) {  // whole lines fit shared memory: staged passes
        const int64_t lz = (int64_t)nx1 * ny1, ly = (int64_t)nx1 * nz1, lx = (int64_t)ny1 * nz1;
        dist_lines_kernel<0><<<(unsigned)((lz + 7) / 8), 256, 8 * nz1, st>>>(scratch, nx1, ny1, nz1, occ);
        dist_lines_kernel<1><<<(unsigned)((ly + 31) / 32), 256, 32 * ny1, st>>>(occ, nx1, ny1, nz1, scratch);
        dist_lines_kernel<2><<<(unsigned)((lx + 31) / 32), 256, 32 * nx1, st>>>(scratch, nx1, ny1, nz1, occ);
    } else {
        dist_pass_kernel<<<blocks(n_kp), 256, 0, st>>>(scratch, n_kp, 1, grid.nz + 1, grid.nz + 1, occ);
        dist_pass_kernel<<<blocks(n_kp), 256, 0, st>>>(occ, n_kp, sy, grid.ny + 1, grid.ny + 1, scratch);
        dist_pass_kernel<<<blocks(n_kp), 256, 0, st>>>(scratch, n_kp, sx, grid.nx + 1, grid.nx + 1, occ);
    }
    count_launch(3);
    return check_launch("occupancy_distance");
}

template <int NCH, int MODE>
void launch_rays(const double origin[3], const double* dirs, int64_t n_rays, const float* values,
                 int plane, const float4* layout, const uint8_t* occ, const Geom& g, const RenderConsts& rc,
                 const double* scat_dirs, double* out, cudaStream_t st) {
    render_rays_kernel<NCH, MODE><<<(unsigned)((n_rays + 127) / 128), 128, 0, st>>>(
        origin[0], origin[1], origin[2], dirs, n_rays, values, plane, layout, occ, g, rc, scat_dirs, out);
}

template <int NCH>
void launch_rays_mode(int mode, const double origin[3], const double* dirs, int64_t n_rays,
                      const float* values, int plane, const float4* layout, const uint8_t* occ, const Geom& g,
                      const RenderConsts& rc, const double* scat_dirs, double* out, cudaStream_t st) {
    switch (mode) {
        case kModePlain: launch_rays<NCH, kModePlain>(origin, dirs, n_rays, values, plane, layout, occ, g, rc, scat_dirs, out, st); break;
        case kModeScatG0: launch_rays<NCH, kModeScatG0>(origin, dirs, n_rays, values, plane, layout, occ, g, rc, scat_dirs, out, st); break;
        case kModeScatG: launch_rays<NCH, kModeScatG>(origin, dirs, n_rays, values, plane, layout, occ, g, rc, scat_dirs, out, st); break;
        case kModeFastPlain: launch_rays<NCH, kModeFastPlain>(origin, dirs, n_rays, values, plane, layout, occ, g, rc, scat_dirs, out, st); break;
        default: launch_rays<NCH, kModeFastScat>(origin, dirs, n_rays, values, plane, layout, occ, g, rc, scat_dirs, out, st); break;
    }
}

template <int NCH, int MODE>
void launch_pix(const fvr_camera_t& cam, const double* us, const double* vs, int64_t n,
                const float* values, int plane, const float4* layout, const uint8_t* occ, const Geom& g,
                const RenderConsts& rc, const double* scat_dirs, double* out, cudaStream_t st) {
    render_pixels_kernel<NCH, MODE><<<(unsigned)((n + 127) / 128), 128, 0, st>>>(
        cam, us, vs, n, values, plane, layout, occ, g, rc, scat_dirs, out);
}

template <int NCH>
void launch_pix_mode(int mode, const fvr_camera_t& cam, const double* us, const double* vs, int64_t n,
                     const float* values, int plane, const float4* layout, const uint8_t* occ, const Geom& g,
                     const RenderConsts& rc, const double* scat_dirs, double* out, cudaStream_t st) {
    switch (mode) {
        case kModePlain: launch_pix<NCH, kModePlain>(cam, us, vs, n, values, plane, layout, occ, g, rc, scat_dirs, out, st); break;
        case kModeScatG0: launch_pix<NCH, kModeScatG0>(cam, us, vs, n, values, plane, layout, occ, g, rc, scat_dirs, out, st); break;
        case kModeScatG: launch_pix<NCH, kModeScatG>(cam, us, vs, n, values, plane, layout, occ, g, rc, scat_dirs, out, st); break;
        case kModeFastPlain: launch_pix<NCH, kModeFastPlain>(cam, us, vs, n, values, plane, layout, occ, g, rc, scat_dirs, out, st); break;
        default: launch_pix<NCH, kModeFastScat>(cam, us, vs, n, values, plane, layout, occ, g, rc, scat_dirs, out, st); break;
    }
}

template <int NCH, int MODE>
void launch_views(const fvr_camera_t* cams, int n_views, int width, int height, const float* values, int plane,
                  const float4* layout, const uint8_t* occ, const Geom& g, const RenderConsts& rc,
                  const double* scat_dirs, float* out, cudaStream_t st) {
    const int units = ((width + 7) / 8) * ((height + 3) / 4);
    const dim3 grid((unsigned)((units + 3) / 4), (unsigned)n_views);
    render_views_kernel<NCH, MODE><<<grid, 128, 0, st>>>(cams, width, height, values, plane, layout, occ, g, rc,
                                                         scat_dirs, out);
}

template <int NCH>
void launch_views_mode(int mode, const fvr_camera_t* cams, int n_views, int width, int height,
                       const float* values, int plane, const float4* layout, const uint8_t* occ, const Geom& g,
                       const RenderConsts& rc, const double* scat_dirs, float* out, cudaStream_t st) {
    switch (mode) {
        case kModePlain: launch_views<NCH, kModePlain>(cams, n_views, width, height, values, plane, layout, occ, g, rc, scat_dirs, out, st); break;
        case kModeScatG0: launch_views<NCH, kModeScatG0>(cams, n_views, width, height, values, plane, layout, occ, g, rc, scat_dirs, out, st); break;
        case kModeScatG: launch_views<NCH, kModeScatG>(cams, n_views, width, height, values, plane, layout, occ, g, rc, scat_dirs, out, st); break;
        case kModeFastPlain: launch_views<NCH, kModeFastPlain>(cams, n_views, width, height, values, plane, layout, occ, g, rc, scat_dirs, out, st); break;
        default: launch_views<NCH, kModeFastScat>(cams, n_views, width, height, values, plane, layout, occ, g, rc, scat_dirs, out, st); break;
    }
}

int check_common(int32_t n_channels, const fvr_grid_t& grid, const fvr_render_params_t& params,
                 const double* scat_dirs) {
    if (n_channels < 1 || n_channels > 4) return set_error(FVR_ERR_INVALID, "n_channels must be 1..4");
    if (int rc = check_grid(grid)) return rc;
    const bool scat = params.scattering && params.sigma_s > 0.0;
    if (scat && (params.n_scat < 1 || !scat_dirs))
        return set_error(FVR_ERR_INVALID, "scattering needs n_scat >= 1 directions");
    return FVR_OK;
}

}  // namespace

namespace fvr {
bool scatter_dirs_match(const double* host_dirs, int n) {
    if (!g_dirs_ready || n != kScatDirs || !host_dirs) return false;
    for (int i = 0; i < 3 * kScatDirs; ++i)
        if (host_dirs[i] != g_dirs_host[i]) return false;
    return true;
}
}  // namespace fvr

namespace {
// Moment tables of fvr_stencil.cuh for one direction set (fp64, stored f32).
int build_moment_tables(const double* dirs) {
    constexpr int S = kScatDirs, K = kSplits;
    double c[3][S], ch[3][S];
    int rank[3][S];
    float thr[3][S];
    for (int a = 0; a < 3; ++a) {
        int ord[S];
        for (int s = 0; s < S; ++s) {
            c[a][s] = 0.5 * dirs[3 * s + a];
            ch[a][s] = 0.5 * c[a][s];
            ord[s] = s;
        }
        std::stable_sort(ord, ord + S, [&](int i, int j) { return (float)c[a][i] < (float)c[a][j]; });
        for (int r = 0; r < S; ++r) {
            rank[a][ord[r]] = r;
            thr[a][r] = (float)c[a][ord[r]];
        }
    }
    // prod_{a in E} c_{s,a}/2, E mask x=4 y=2 z=1
    double cE[8][S];
    for (int e = 0; e < 8; ++e)
        for (int s = 0; s < S; ++s)
            cE[e][s] = ((e & 4) ? ch[0][s] : 1.0) * ((e & 2) ? ch[1][s] : 1.0) * ((e & 1) ? ch[2][s] : 1.0);
    auto sig = [&](int a, int i, int s) { return rank[a][s] < i ? -1.0 : 1.0; };
    std::vector<float> q1(3 * K * 8), q2(3 * K * K * 8), q3((size_t)K * K * K * 8);
    float q0[8];
    for (int e = 0; e < 8; ++e) {
        double acc = 0.0;
        for (int s = 0; s < S; ++s) acc += cE[e][s];
        q0[e] = (float)acc;
    }
    for (int a = 0; a < 3; ++a)
        for (int i = 0; i < K; ++i)
            for (int e = 0; e < 8; ++e) {
                double acc = 0.0;
                for (int s = 0; s < S; ++s) acc += sig(a, i, s) * cE[e][s];
                q1[(a * K + i) * 8 + e] = (float)acc;
            }
    const int pa[3] = {0, 0, 1}, pb[3] = {1, 2, 2};
    for (int p = 0; p < 3; ++p)
        for (int i = 0; i < K; ++i)
            for (int j = 0; j < K; ++j)
                for (int e = 0; e < 8; ++e) {
                    double acc = 0.0;
                    for (int s = 0; s < S; ++s) acc += sig(pa[p], i, s) * sig(pb[p], j, s) * cE[e][s];
                    q2[((p * K + i) * K + j) * 8 + e] = (float)acc;
                }
    for (int i = 0; i < K; ++i)
        for (int j = 0; j < K; ++j)
            for (int l = 0; l < K; ++l) {
                double sg[S];
                for (int s = 0; s < S; ++s) sg[s] = sig(0, i, s) * sig(1, j, s) * sig(2, l, s);
                for (int e = 0; e < 8; ++e) {
                    double acc = 0.0;
                    for (int s = 0; s < S; ++s) acc += sg[s] * cE[e][s];
                    q3[(((size_t)i * K + j) * K + l) * 8 + e] = (float)acc;
                }
            }
    uint32_t nmask[3][K];
    for (int a = 0; a < 3; ++a)
        for (int i = 0; i < K; ++i) {
            uint32_t m = 0;
            for (int sdir = 0; sdir < S; ++sdir)
                if (rank[a][sdir] < i) m |= 1u << sdir;
            nmask[a][i] = m;
        }
    if (cudaMemcpyToSymbol(c_nmask, nmask, sizeof(nmask)) != cudaSuccess) return set_error(FVR_ERR_CUDA, "upload");
    if (cudaMemcpyToSymbol(c_thr, thr, sizeof(thr)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_q0, q0, sizeof(q0)) != cudaSuccess ||
        cudaMemcpyToSymbol(g_q1, q1.data(), q1.size() * sizeof(float)) != cudaSuccess ||
        cudaMemcpyToSymbol(g_q2, q2.data(), q2.size() * sizeof(float)) != cudaSuccess ||
        cudaMemcpyToSymbol(g_q3, q3.data(), q3.size() * sizeof(float)) != cudaSuccess)
        return set_error(FVR_ERR_CUDA, "moment table upload failed");
    return FVR_OK;
}
}  // namespace

extern "C" int fvr_set_scatter_dirs(const double* dirs_host, int32_t n) {
    FVR_TRY_BEGIN
    if (n != kScatDirs) return set_error(FVR_ERR_INVALID, "the stencil path is compiled for 32 directions");
    double d[3][kScatDirs];
    float h[3][kScatDirs];
    for (int s = 0; s < n; ++s)
        for (int a = 0; a < 3; ++a) {
            d[a][s] = dirs_host[3 * s + a];
            h[a][s] = (float)(0.5 * dirs_host[3 * s + a]);
        }
    float2 h2[3][kScatDirs / 2];
    for (int a = 0; a < 3; ++a)
        for (int s = 0; s < kScatDirs / 2; ++s) h2[a][s] = make_float2(h[a][s], h[a][s + kScatDirs / 2]);
    if (cudaMemcpyToSymbol(c_dir, d, sizeof(d)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_half_dir, h, sizeof(h)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_half_dir2, h2, sizeof(h2)) != cudaSuccess)
        return set_error(FVR_ERR_CUDA, "cudaMemcpyToSymbol failed");
    if (int e = build_moment_tables(dirs_host)) return e;
    for (int i = 0; i < 3 * kScatDirs; ++i) g_dirs_host[i] = dirs_host[i];
    g_dirs_ready = true;
    return FVR_OK;
    FVR_TRY_END
}

extern "C" int fvr_pack_layout(const float* values, int32_t n_channels, fvr_grid_t grid, int32_t kind,
                               float* layout, void* stream) {
    FVR_TRY_BEGIN
    if (int rc = check_grid(grid)) return rc;
    if (kind != kLayoutYZQ && kind != kLayoutZ4) return set_error(FVR_ERR_INVALID, "unknown layout kind");
    return pack(values, n_channels, grid, kind, reinterpret_cast<float4*>(layout), (cudaStream_t)stream);
    FVR_TRY_END
}

extern "C" int fvr_occupancy(const float* values, int32_t n_channels, const uint8_t* force_mask,
                             fvr_grid_t grid, uint8_t* occ, void* stream) {
    FVR_TRY_BEGIN
    if (int rc = check_grid(grid)) return rc;
    return occupancy(values, n_channels, force_mask, grid, occ, (cudaStream_t)stream);
    FVR_TRY_END
}

extern "C" int fvr_render_layout_kind(fvr_render_params_t params, fvr_grid_t grid) {
    bool scat;
    const float4* dummy = reinterpret_cast<const float4*>(16);
    return layout_kind(effective_mode(params, grid, dummy, scat));
}

extern "C" int fvr_render_rays(const double origin[3], const double* dirs, int64_t n_rays,
                               const float* values, int32_t n_channels, fvr_grid_t grid,
                               fvr_render_params_t params, const double* background,
                               const double* scat_dirs, float* layout, uint8_t* occ, double* out,
                               void* stream) {
    FVR_TRY_BEGIN
    if (int rc = check_common(n_channels, grid, params, scat_dirs)) return rc;
    if (n_rays == 0) return FVR_OK;
    bool scat;
    const float4* lay = reinterpret_cast<const float4*>(layout);
    const int mode = effective_mode(params, grid, lay, scat);
    const Geom g = make_geom(grid);
    const RenderConsts rc = make_render_consts(params, background, n_channels);
    const int plane = (grid.nx + 1) * (grid.ny + 1) * (grid.nz + 1);
    cudaStream_t st = (cudaStream_t)stream;
    if (layout_kind(mode) != kLayoutNone)
        if (int e = pack(values, n_channels, grid, layout_kind(mode), reinterpret_cast<float4*>(layout), st)) return e;
    if (layout_kind(mode) == kLayoutNone) occ = nullptr;  // the general path never skips
    if (occ)
        if (int e = occupancy(values, n_channels, nullptr, grid, occ, st)) return e;
    switch (n_channels) {
        case 1: launch_rays_mode<1>(mode, origin, dirs, n_rays, values, plane, lay, occ, g, rc, scat_dirs, out, st); break;
        case 2: launch_rays_mode<2>(mode, origin, dirs, n_rays, values, plane, lay, occ, g, rc, scat_dirs, out, st); break;
        case 3: launch_rays_mode<3>(mode, origin, dirs, n_rays, values, plane, lay, occ, g, rc, scat_dirs, out, st); break;
        default: launch_rays_mode<4>(mode, origin, dirs, n_rays, values, plane, lay, occ, g, rc, scat_dirs, out, st); break;
    }
    return check_launch("render_rays");
    FVR_TRY_END
}

extern "C" int fvr_render_pixels(const fvr_camera_t* camera, const double* us, const double* vs,
                                 int64_t n, const float* values, int32_t n_channels,
                                 fvr_grid_t grid, fvr_render_params_t params,
                                 const double* background, const double* scat_dirs, float* layout,
                                 uint8_t* occ, double* out, void* stream) {
    FVR_TRY_BEGIN
    if (!camera) return set_error(FVR_ERR_INVALID, "camera is NULL");
    if (int rc = check_common(n_channels, grid, params, scat_dirs)) return rc;
    if ((us == nullptr) != (vs == nullptr)) return set_error(FVR_ERR_INVALID, "us and vs must both be given");
    if (!us) n = (int64_t)camera->width * camera->height;
    if (n == 0) return FVR_OK;
    bool scat;
    const float4* lay = reinterpret_cast<const float4*>(layout);
    const int mode = effective_mode(params, grid, lay, scat);
    const Geom g = make_geom(grid);
    const RenderConsts rc = make_render_consts(params, background, n_channels);
    const int plane = (grid.nx + 1) * (grid.ny + 1) * (grid.nz + 1);
    cudaStream_t st = (cudaStream_t)stream;
    if (layout_kind(mode) != kLayoutNone)
        if (int e = pack(values, n_channels, grid, layout_kind(mode), reinterpret_cast<float4*>(layout), st)) return e;
    if (layout_kind(mode) == kLayoutNone) occ = nullptr;  // the general path never skips
    if (occ)
        if (int e = occupancy(values, n_channels, nullptr, grid, occ, st)) return e;
    switch (n_channels) {
        case 1: launch_pix_mode<1>(mode, *camera, us, vs, n, values, plane, lay, occ, g, rc, scat_dirs, out, st); break;
        case 2: launch_pix_mode<2>(mode, *camera, us, vs, n, values, plane, lay, occ, g, rc, scat_dirs, out, st); break;
        case 3: launch_pix_mode<3>(mode, *camera, us, vs, n, values, plane, lay, occ, g, rc, scat_dirs, out, st); break;
        default: launch_pix_mode<4>(mode, *camera, us, vs, n, values, plane, lay, occ, g, rc, scat_dirs, out, st); break;
    }
    return check_launch("render_pixels");
    FVR_TRY_END
}

extern "C" int fvr_render_views(const fvr_camera_t* cams, int32_t n_views, int32_t width, int32_t height,
                                const float* values, int32_t n_channels, fvr_grid_t grid,
                                fvr_render_params_t params, const double* background,
                                const double* scat_dirs, const float* layout, const uint8_t* occ, float* out,
                                void* stream) {
    FVR_TRY_BEGIN
    if (!cams || n_views < 1 || n_views > 65535) return set_error(FVR_ERR_INVALID, "bad camera array");
    if (width < 1 || height < 1) return set_error(FVR_ERR_INVALID, "empty frame");
    if (int rc = check_common(n_channels, grid, params, scat_dirs)) return rc;
    bool scat;
    const float4* lay = reinterpret_cast<const float4*>(layout);
    const int mode = effective_mode(params, grid, lay, scat);
    if (layout_kind(mode) == kLayoutNone) occ = nullptr;
    const Geom g = make_geom(grid);
    const RenderConsts rc = make_render_consts(params, background, n_channels);
    const int plane = (grid.nx + 1) * (grid.ny + 1) * (grid.nz + 1);
    cudaStream_t st = (cudaStream_t)stream;
    switch (n_channels) {
        case 1: launch_views_mode<1>(mode, cams, n_views, width, height, values, plane, lay, occ, g, rc, scat_dirs, out, st); break;
        case 2: launch_views_mode<2>(mode, cams, n_views, width, height, values, plane, lay, occ, g, rc, scat_dirs, out, st); break;
        case 3: launch_views_mode<3>(mode, cams, n_views, width, height, values, plane, lay, occ, g, rc, scat_dirs, out, st); break;
        default: launch_views_mode<4>(mode, cams, n_views, width, height, values, plane, lay, occ, g, rc, scat_dirs, out, st); break;
    }
    return check_launch("render_views");
    FVR_TRY_END
}

extern "C" int fvr_loop_blocks_per_view(int32_t bbox_w, int32_t bbox_h) {
    return ((bbox_w + kUnitW - 1) / kUnitW) * ((bbox_h + kUnitH - 1) / kUnitH);
}

namespace {
template <int NS, int NCH>
int launch_scat(int blocks, cudaStream_t st, const fvr_camera_t* cams, int n_views, int u0, int v0, int w, int h,
                int units_x, int upv, int n_units, const float* src, const float* values, int plane,
                const float4* lay, const uint8_t* occ, const Geom& g, const RenderConsts& rc, float* residual,
                double* sq_partials, int64_t sq_stride, fvr_loop_state_t* state) {
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(loop_render_scat_kernel<NS, NCH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kScatSmem) != cudaSuccess)
            return set_error(FVR_ERR_CUDA, "cannot reserve shared memory for the moment tables");
        // smallest carveout that holds the tables: the remainder is L1
        int carve = kScatCtasPerSm == 1 ? 50 : 100;
        if (const char* e = getenv("FVR_SCAT_CARVEOUT")) carve = atoi(e);
        if (carve >= 0)
            cudaFuncSetAttribute(loop_render_scat_kernel<NS, NCH>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 carve);
        attr_set = true;
    }
    loop_render_scat_kernel<NS, NCH><<<blocks, kScatThreads, kScatSmem, st>>>(
        cams, n_views, u0, v0, w, h, units_x, upv, n_units, src, values, plane, lay, occ, g, rc, residual,
        sq_partials, sq_stride, state);
    return FVR_OK;
}
}  // namespace

extern "C" int fvr_loop_render(const fvr_camera_t* cams, int32_t n_views, int32_t u0, int32_t v0,
                               int32_t bbox_w, int32_t bbox_h, const float* src,
                               const float* values, const float* layout, const uint8_t* occ,
                               fvr_grid_t grid, fvr_render_params_t params, const double* background,
                               int32_t n_channels, const double* scat_dirs, float* residual,
                               double* sq_partials, int64_t sq_stride, fvr_loop_state_t* state, void* stream) {
    FVR_TRY_BEGIN
    if (n_views < 1 || n_views > 65535) return set_error(FVR_ERR_INVALID, "bad view count");
    if (bbox_w < 1 || bbox_h < 1) return set_error(FVR_ERR_INVALID, "empty bounding box");
    if (n_channels != 1 && n_channels != 3) return set_error(FVR_ERR_INVALID, "the loop renders 1 or 3 channels");
    if (!background) return set_error(FVR_ERR_INVALID, "background is NULL");
    if (int rc = check_common(n_channels, grid, params, scat_dirs)) return rc;
    bool scat;
    const float4* lay = reinterpret_cast<const float4*>(layout);
    const int mode = effective_mode(params, grid, lay, scat);
    if (mode == kModeScatG) return set_error(FVR_ERR_INVALID, "the reconstruction loop renders with g = 0 (render.py:196)");
    const Geom g = make_geom(grid);
    const RenderConsts rc = make_render_consts(params, background, n_channels);
    const int plane = (grid.nx + 1) * (grid.ny + 1) * (grid.nz + 1);
    const int units_x = (bbox_w + kUnitW - 1) / kUnitW;
    const int upv = fvr_loop_blocks_per_view(bbox_w, bbox_h);
    const int n_units = upv * n_views;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned blocks = (unsigned)((n_units + kWarpsPerBlock - 1) / kWarpsPerBlock);
#define FVR_LOOP_RENDER(M, C)                                                                                  \
    loop_render_kernel<M, C><<<blocks, kBlockThreads, 0, st>>>(cams, n_views, u0, v0, bbox_w, bbox_h, units_x, \
                                                               upv, n_units, src, values, plane, lay, occ, g, rc,  \
                                                               scat_dirs, residual, sq_partials, sq_stride, state)
    if (mode != kModeFastScat) {
        if (n_channels == 1) {
            switch (mode) {
                case kModePlain: FVR_LOOP_RENDER(kModePlain, 1); break;
                case kModeScatG0: FVR_LOOP_RENDER(kModeScatG0, 1); break;
                default: FVR_LOOP_RENDER(kModeFastPlain, 1); break;
            }
        } else {
            switch (mode) {
                case kModePlain: FVR_LOOP_RENDER(kModePlain, 3); break;
                case kModeScatG0: FVR_LOOP_RENDER(kModeScatG0, 3); break;
                default: FVR_LOOP_RENDER(kModeFastPlain, 3); break;
            }
        }
    } else {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int want = (n_units + kScatWarps - 1) / kScatWarps;
        const int pblocks = want < kScatCtasPerSm * sms ? want : kScatCtasPerSm * sms;
        const int e = n_channels == 1
                          ? launch_scat<0, 1>(pblocks, st, cams, n_views, u0, v0, bbox_w, bbox_h, units_x, upv,
                                              n_units, src, values, plane, lay, occ, g, rc, residual, sq_partials,
                                              sq_stride, state)
                          : launch_scat<0, 3>(pblocks, st, cams, n_views, u0, v0, bbox_w, bbox_h, units_x, upv,
                                              n_units, src, values, plane, lay, occ, g, rc, residual, sq_partials,
                                              sq_stride, state);
        if (e) return e;
    }
#undef FVR_LOOP_RENDER
    return check_launch("loop_render");
    FVR_TRY_END
}

// ---- K-render as a fixed operator (fvr_rplan.cuh) -----------------------------

namespace {
// dyn27 masks of `dynamic`: recomputed by every count pass (`fresh`), reused
// by the fill pass that follows it for the same array; grown on demand and
// kept for the process
uint32_t* dyn27_scratch(const fvr_grid_t& grid, const uint8_t* dynamic, cudaStream_t st, bool fresh) {
    static uint32_t* buf = nullptr;
    static int64_t cap = 0;
    static const uint8_t* last = nullptr;
    static fvr_grid_t last_grid{};
    const int64_t n = (int64_t)(grid.nx + 1) * (grid.ny + 1) * (grid.nz + 1);
    if (cap < n) {
        if (buf) cudaFree(buf);
        buf = nullptr;
        cap = 0;
        last = nullptr;
        if (cudaMalloc(&buf, (size_t)n * 4) != cudaSuccess) return nullptr;
        cap = n;
    }
    if (fresh || last != dynamic || last_grid.nx != grid.nx || last_grid.ny != grid.ny || last_grid.nz != grid.nz) {
        int64_t blocks = (n + 255) / 256;
        if (blocks > 148 * 16) blocks = 148 * 16;
        rplan_dyn27_kernel<<<(unsigned)blocks, 256, 0, st>>>(dynamic, make_geom(grid), buf);
        count_launch(1);
        last = dynamic;
        last_grid = grid;
    }
    return buf;
}
// pos27 masks of the current values (rplan_pos27_kernel), recomputed per fill
uint32_t* pos27_scratch(const fvr_grid_t& grid, const uint8_t* dynamic, const float* values, int nch,
                        cudaStream_t st) {
    static uint32_t* buf = nullptr;
    static int64_t cap = 0;
    const int64_t n = (int64_t)(grid.nx + 1) * (grid.ny + 1) * (grid.nz + 1);
    if (cap < n) {
        if (buf) cudaFree(buf);
        buf = nullptr;
        cap = 0;
        if (cudaMalloc(&buf, (size_t)n * 4) != cudaSuccess) return nullptr;
        cap = n;
    }
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    rplan_pos27_kernel<<<(unsigned)blocks, 256, 0, st>>>(dynamic, values, nch, n, make_geom(grid), buf);
    count_launch(1);
    return buf;
}
// the plan covers the two fast modes (g = 0, gather = edge, 32 loaded directions)
int rplan_mode(const fvr_render_params_t& params, const fvr_grid_t& grid, bool& scat) {
    const float4* dummy = reinterpret_cast<const float4*>(&params);  // any non-null layout: mode query only
    const int mode = effective_mode(params, grid, dummy, scat);
    if (mode == kModeFastScat) return 1;
    if (mode == kModeFastPlain) return 0;
    return -1;
}
}  // namespace

extern "C" int fvr_rplan_chunk_entries(void) { return kRpB; }

extern "C" int fvr_rplan_count(const fvr_camera_t* cams, int32_t n_views, int32_t u0, int32_t v0, int32_t bbox_w,
                               int32_t bbox_h, fvr_grid_t grid, fvr_render_params_t params,
                               const uint8_t* occ, const uint8_t* dynamic, int32_t* unit_len, int32_t* row_len,
                               void* stream) {
    FVR_TRY_BEGIN
    if (n_views < 1 || bbox_w < 1 || bbox_h < 1) return set_error(FVR_ERR_INVALID, "empty render plan");
    if (!dynamic || !unit_len) return set_error(FVR_ERR_INVALID, "dynamic / unit_len is NULL");
    if (int rc = check_grid(grid)) return rc;
    bool scat;
    const int m = rplan_mode(params, grid, scat);
    if (m < 0) return set_error(FVR_ERR_INVALID, "render plan needs g = 0, gather = edge and 32 directions");
    const Geom g = make_geom(grid);
    const double bg = 0.0;
    const RenderConsts rc = make_render_consts(params, &bg, 1);
    const int units_x = (bbox_w + kUnitW - 1) / kUnitW, upv = fvr_loop_blocks_per_view(bbox_w, bbox_h);
    const int n_units = upv * n_views;
    const unsigned blocks = (unsigned)(((int64_t)n_units * 32 + 127) / 128);
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t* d27 = dyn27_scratch(grid, dynamic, st, true);
    if (!d27) return set_error(FVR_ERR_CUDA, "cannot allocate the render-plan scratch");
    if (m)
        rplan_count_kernel<true><<<blocks, 128, 0, st>>>(cams, u0, v0, bbox_w, bbox_h, units_x, upv, n_units, g, rc,
                                                          occ, dynamic, d27, unit_len, row_len);
    else
        rplan_count_kernel<false><<<blocks, 128, 0, st>>>(cams, u0, v0, bbox_w, bbox_h, units_x, upv, n_units, g, rc,
                                                           occ, dynamic, d27, unit_len, row_len);
    return check_launch("rplan_count");
    FVR_TRY_END
}

extern "C" int fvr_rplan_pos27(fvr_grid_t grid, const uint8_t* dynamic, const float* values, int32_t n_channels,
                               uint32_t* pos27, void* stream) {
    FVR_TRY_BEGIN
    if (int rc = check_grid(grid)) return rc;
    if (!dynamic || !values || !pos27) return set_error(FVR_ERR_INVALID, "dynamic / values / pos27 are NULL");
    const int64_t n = (int64_t)(grid.nx + 1) * (grid.ny + 1) * (grid.nz + 1);
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    rplan_pos27_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(dynamic, values, n_channels, n,
                                                                          make_geom(grid), pos27);
    return check_launch("rplan_pos27");
    FVR_TRY_END
}

// Unit order of the render plan: key = (length class, descending) << 40 |
// spatial rank (2x4-unit tiles, row-major, then the units inside a tile), so
// one sort visits the units longest class first and neighbouring units
// together inside a class.
__global__ void rplan_unit_keys_kernel(const int32_t* __restrict__ unit_len, int n_units, int upv, int units_x,
                                       int buckets, const int32_t* __restrict__ max_len,
                                       uint64_t* __restrict__ keys) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_units) return;
    const int q = max(1, (*max_len + buckets - 1) / buckets);  // class width: buckets classes up to the longest
    const int units_y = upv / units_x;
    const int txn = (units_x + 1) / 2, tyn = (units_y + 3) / 4;
    const int view = i / upv, u = i - view * upv;
    const int64_t tile = ((int64_t)view * tyn + (u / units_x) / 4) * txn + (u % units_x) / 2;
    const uint64_t spatial = (uint64_t)(tile * 8 + ((u / units_x) % 4) * 2 + (u % units_x) % 2);
    const uint64_t cls = (uint64_t)(unit_len[i] / q);
    keys[i] = ((0xFFFFFull - cls) << 40) | spatial;
}

extern "C" int fvr_rplan_unit_keys(const int32_t* unit_len, int32_t n_views, int32_t bbox_w, int32_t bbox_h,
                                   int32_t buckets, const int32_t* max_len, int64_t* keys, void* stream) {
    FVR_TRY_BEGIN
    if (buckets < 1) return set_error(FVR_ERR_INVALID, "buckets must be positive");
    if (!max_len) return set_error(FVR_ERR_INVALID, "max_len is NULL");
    const int units_x = (bbox_w + kUnitW - 1) / kUnitW, upv = fvr_loop_blocks_per_view(bbox_w, bbox_h);
    const int n_units = upv * n_views;
    if (n_units == 0) return FVR_OK;
    rplan_unit_keys_kernel<<<(n_units + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
        unit_len, n_units, upv, units_x, buckets, max_len, reinterpret_cast<uint64_t*>(keys));
    return check_launch("rplan_unit_keys");
    FVR_TRY_END
}

extern "C" int fvr_rplan_fill(const fvr_camera_t* cams, int32_t n_views, int32_t u0, int32_t v0, int32_t bbox_w,
                              int32_t bbox_h, fvr_grid_t grid, fvr_render_params_t params, const uint8_t* occ,
                              const uint8_t* dynamic, const float* values, int32_t n_channels,
                              const int64_t* unit_off, const int32_t* unit_order, const int32_t* row_src,
                              const int32_t* kp_map, uint32_t* entries_a, uint32_t* entries_b, double* base,
                              double* t_fin, const uint32_t* pos27, int32_t wide, void* stream) {
    FVR_TRY_BEGIN
    if (n_views < 1 || bbox_w < 1 || bbox_h < 1) return set_error(FVR_ERR_INVALID, "empty render plan");
    if (n_channels < 1 || n_channels > 4) return set_error(FVR_ERR_INVALID, "n_channels must be 1..4");
    if (int rc = check_grid(grid)) return rc;
    bool scat;
    const int m = rplan_mode(params, grid, scat);
    if (m < 0) return set_error(FVR_ERR_INVALID, "render plan needs g = 0, gather = edge and 32 directions");
    const Geom g = make_geom(grid);
    const double bg = 0.0;
    const RenderConsts rc = make_render_consts(params, &bg, 1);
    const int units_x = (bbox_w + kUnitW - 1) / kUnitW, upv = fvr_loop_blocks_per_view(bbox_w, bbox_h);
    const int n_units = upv * n_views;
    const int64_t plane = (int64_t)(grid.nx + 1) * (grid.ny + 1) * (grid.nz + 1);
    const unsigned blocks = (unsigned)(((int64_t)n_units * 32 + 127) / 128);
    cudaStream_t st = (cudaStream_t)stream;
    const auto* uo = reinterpret_cast<const long long*>(unit_off);
    if (!kp_map || !entries_a || !entries_b) return set_error(FVR_ERR_INVALID, "kp_map / entries are NULL");
    uint32_t* d27 = dyn27_scratch(grid, dynamic, st, false);
    if (!d27) return set_error(FVR_ERR_CUDA, "cannot allocate the render-plan scratch");
    // values == NULL: every key point outside `dynamic` is <= 0 (the loop's
    // own initial lattice), so nothing static folds into base
    const uint32_t* p27 = pos27 || !values ? pos27 : pos27_scratch(grid, dynamic, values, n_channels, st);
    if (values && !p27) return set_error(FVR_ERR_CUDA, "cannot allocate the render-plan scratch");
#define FVR_RPLAN_FILL(S, W)                                                                                   \
    rplan_fill_kernel<S, W><<<blocks, 128, 0, st>>>(cams, u0, v0, bbox_w, bbox_h, units_x, upv, n_units, g, rc, occ, \
                                                     dynamic, d27, values, n_channels, plane, uo, unit_order, row_src, \
                                                     kp_map, entries_a, entries_b, p27, base, t_fin)
    if (m && wide) FVR_RPLAN_FILL(true, true);
    else if (m) FVR_RPLAN_FILL(true, false);
    else if (wide) FVR_RPLAN_FILL(false, true);
    else FVR_RPLAN_FILL(false, false);
#undef FVR_RPLAN_FILL
    return check_launch("rplan_fill");
    FVR_TRY_END
}

extern "C" int fvr_rplan_pack(const float* values, int32_t n_channels, fvr_grid_t grid, const int32_t* kp_index,
                              int64_t n_kp, float* kp_values, const fvr_loop_state_t* state, void* stream) {
    FVR_TRY_BEGIN
    if (n_channels != 1 && n_channels != 3) return set_error(FVR_ERR_INVALID, "1 or 3 channels");
    if (n_kp <= 0) return FVR_OK;
    const int64_t plane = (int64_t)(grid.nx + 1) * (grid.ny + 1) * (grid.nz + 1);
    int64_t b = (n_kp + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    cudaStream_t st = (cudaStream_t)stream;
    if (n_channels == 1)
        rplan_pack_kernel<1><<<(unsigned)b, 256, 0, st>>>(values, plane, kp_index, n_kp, kp_values, state);
    else
        rplan_pack_kernel<3><<<(unsigned)b, 256, 0, st>>>(values, plane, kp_index, n_kp, kp_values, state);
    return check_launch("rplan_pack");
    FVR_TRY_END
}

extern "C" int fvr_rplan_render(const int32_t* unit_len, const int64_t* unit_off, const uint32_t* entries_a,
                                const uint32_t* entries_b, const double* base, const double* t_fin,
                                const int32_t* unit_order, const int32_t* row_src, int32_t n_views, int32_t bbox_w,
                                int32_t bbox_h, const float* src, const float* kp_values, int32_t n_channels,
                                const double* background, float* residual, double* sq_partials, int64_t sq_stride,
                                fvr_loop_state_t* state, const fvr_loop_finalize_t* finalize, int32_t wide,
                                void* stream) {
    FVR_TRY_BEGIN
    if (n_channels != 1 && n_channels != 3) return set_error(FVR_ERR_INVALID, "the loop renders 1 or 3 channels");
    if (!background) return set_error(FVR_ERR_INVALID, "background is NULL");
    RplanFinalize fin{};
    if (finalize) {
        if (!state) return set_error(FVR_ERR_INVALID, "a fused finalize needs the loop state");
        if (finalize->n_views < 1 || finalize->n_views > 32)
            return set_error(FVR_ERR_INVALID, "n_views must be in 1..32");
        if (finalize->pixels_per_view < 1) return set_error(FVR_ERR_INVALID, "empty bounding box");
        if (!finalize->trace_rmse) return set_error(FVR_ERR_INVALID, "trace_rmse is NULL");
        fin.on = true;
        fin.n_views = finalize->n_views;
        fin.bpv = finalize->blocks_per_view;
        fin.n_vol = finalize->n_vol_blocks;
        fin.pixels = (double)finalize->pixels_per_view;
        fin.n_kp = (double)finalize->n_kp;
        fin.eps = finalize->converge_eps;
        fin.vol = finalize->vol_partials;
        fin.trace = finalize->trace_rmse;
        fin.trace_vol = finalize->trace_vol;
        fin.trace_stride = finalize->trace_stride;
        fin.acc = reinterpret_cast<long long*>(finalize->sq_accum);
        if (finalize->l2_discard && finalize->l2_discard_bytes >= 128) {
            if (reinterpret_cast<uintptr_t>(finalize->l2_discard) % 128)
                return set_error(FVR_ERR_INVALID, "l2_discard must be 128-byte aligned");
            fin.discard = static_cast<char*>(finalize->l2_discard);
            fin.discard_lines = finalize->l2_discard_bytes / 128;
        }
    }
    if (!kp_values || !entries_a || !entries_b) return set_error(FVR_ERR_INVALID, "kp_values / entries are NULL");
    fvr_render_params_t p{};
    p.tau = 0.0;
    RenderConsts rc = make_render_consts(p, background, n_channels);
    const int units_x = (bbox_w + kUnitW - 1) / kUnitW, upv = fvr_loop_blocks_per_view(bbox_w, bbox_h);
    const int n_units = upv * n_views;
    int64_t blocks = ((int64_t)n_units * 32 + FVR_RPLAN_THREADS - 1) / FVR_RPLAN_THREADS;
#ifdef FVR_RPLAN_GRID_CAP
    if (blocks > FVR_RPLAN_GRID_CAP) blocks = FVR_RPLAN_GRID_CAP;
#endif
    if (blocks > 148 * 64) blocks = 148 * 64;
    cudaStream_t st = (cudaStream_t)stream;
    const auto* uo = reinterpret_cast<const long long*>(unit_off);
    cudaError_t e;
#define FVR_RPLAN_RENDER(C, W)                                                                                       \
    e = launch_pdl(rplan_render_kernel<C, W>, (unsigned)blocks, FVR_RPLAN_THREADS, st, unit_len, uo, entries_a, entries_b, base,    \
                   t_fin, unit_order, row_src, n_units, units_x, upv, n_views, bbox_w, bbox_h, src, kp_values, rc,    \
                   residual, sq_partials, sq_stride, state, fin)
    if (n_channels == 1 && !wide) FVR_RPLAN_RENDER(1, false);
    else if (n_channels == 1) FVR_RPLAN_RENDER(1, true);
    else if (!wide) FVR_RPLAN_RENDER(3, false);
    else FVR_RPLAN_RENDER(3, true);
#undef FVR_RPLAN_RENDER
    if (e != cudaSuccess) return set_error(FVR_ERR_CUDA, std::string("rplan_render: ") + cudaGetErrorString(e));
    return check_launch("rplan_render");
    FVR_TRY_END
}
