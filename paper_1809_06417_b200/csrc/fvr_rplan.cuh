// fvr_rplan.cuh -- K-render as a fixed sparse operator (included by
// fvr_render.cu, which owns the direction constants).
//
// The loop's forward model is linear in c = max(v, 0): every sample of a
// pixel's ray adds t_k tau (sigma_a c(p) + kappa sum_d c(p + h s_d)), the
// transparency t_k = (1-tau)^(k-1) and the in-box masks depend only on the
// geometry, and the trilinear reads are linear in the 27 key points around
// the sample.  So one iteration's render is rec = B c + base + t_n bg with a
// matrix B that never changes during a reconstruction.  The render plan stores
// B in SELL-32 form: rows are the bbox pixels in K-render's 8x4 warp units
// (a 16x16-pixel tile's rows dealt to its units by length), entry t of lane i
// in 16-byte chunks per lane (coalesced, 6 bytes: see RplanOut), columns are
// the key points that can change (hull key points, numbered by the loop's
// key-point list); key points that cannot change fold into `base`.  Consecutive samples of a ray share most of their 27
// stencil key points, so the weights are merged along the ray in a 3x3x3
// window that shifts with the nearest key point (~10 entries per live sample
// instead of 27).
//
// Weights are summed directly (hat weights of the sample and of its 32 gather
// points, fp32), so B's entries are sums of non-negative terms; K-render's
// moment evaluation reaches the same values up to float rounding.
#pragma once

namespace fvr {

__device__ __forceinline__ void hat3(float x, float h[3]) {
    h[0] = fmaxf(-x, 0.f);
    h[1] = 1.f - fabsf(x);
    h[2] = fmaxf(x, 0.f);
}

// w[(jx*3 + jy)*3 + jz]: coefficient of the key point at offset (jx-1, jy-1,
// jz-1) from the sample's nearest key point in sigma_a e + kappa S.
template <bool SCAT>
__device__ __forceinline__ void sample_weights(float dx, float dy, float dz, float sig_a, float kappa,
                                               uint32_t mask, float w[27]) {
    float hx[3], hy[3], hz[3];
    hat3(dx, hx);
    hat3(dy, hy);
    hat3(dz, hz);
#pragma unroll
    for (int jx = 0; jx < 3; ++jx)
#pragma unroll
        for (int jy = 0; jy < 3; ++jy)
#pragma unroll
            for (int jz = 0; jz < 3; ++jz) w[(jx * 3 + jy) * 3 + jz] = sig_a * (hx[jx] * hy[jy] * hz[jz]);
    if (SCAT) {
        float s[27];
#pragma unroll
        for (int j = 0; j < 27; ++j) s[j] = 0.f;
#pragma unroll 2
        for (int d = 0; d < kScatDirs; ++d) {
            if (!((mask >> d) & 1u)) continue;
            hat3(dx + c_half_dir[0][d], hx);
            hat3(dy + c_half_dir[1][d], hy);
            hat3(dz + c_half_dir[2][d], hz);
#pragma unroll
            for (int jx = 0; jx < 3; ++jx)
#pragma unroll
                for (int jy = 0; jy < 3; ++jy) {
                    const float hxy = hx[jx] * hy[jy];
#pragma unroll
                    for (int jz = 0; jz < 3; ++jz) s[(jx * 3 + jy) * 3 + jz] = fmaf(hxy, hz[jz], s[(jx * 3 + jy) * 3 + jz]);
                }
        }
#pragma unroll
        for (int j = 0; j < 27; ++j) w[j] = fmaf(kappa, s[j], w[j]);
    }
}

// Slots whose weight can be non-zero: the trilinear corners of the sample
// (emission) and, with scattering, every slot some gather point reaches.  A
// gather point x_s = delta + s/2 gives slot offset -1 weight iff x_s < 0 and
// +1 iff x_s > 0 per axis; the directions with x_s < 0 on axis a are the
// first split_index ones in that axis' sorted order (nm[a][i]), so slot
// (jx, jy, jz) is reached iff the three per-axis direction sets intersect.
// Depends on the geometry only: the count pass needs no weights.
__device__ __forceinline__ uint32_t support_mask(bool scat, const float dl[3], const float* __restrict__ thr,
                                                 const uint32_t* __restrict__ nm) {
    uint32_t ax[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) ax[a] = 2u | (dl[a] > 0.f ? 4u : 0u) | (dl[a] < 0.f ? 1u : 0u);  // slot bits 0..2
    uint32_t m = 0;
#pragma unroll
    for (int j = 0; j < 27; ++j)
        if (((ax[0] >> (j / 9)) & (ax[1] >> ((j / 3) % 3)) & (ax[2] >> (j % 3))) & 1u) m |= 1u << j;
    if (scat) {
        uint32_t S[3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const uint32_t neg = nm[a * (kScatDirs + 1) + split_index(thr + a * kScatDirs, -dl[a])];
            S[a][0] = neg;
            S[a][1] = 0xffffffffu;
            S[a][2] = ~neg;  // x_s >= 0 (a zero coordinate only adds a zero-weight entry)
        }
#pragma unroll
        for (int jx = 0; jx < 3; ++jx)
#pragma unroll
            for (int jy = 0; jy < 3; ++jy) {
                const uint32_t sxy = S[0][jx] & S[1][jy];
#pragma unroll
                for (int jz = 0; jz < 3; ++jz)
                    if (sxy & S[2][jz]) m |= 1u << ((jx * 3 + jy) * 3 + jz);
            }
    }
    return m;
}

// Render-plan entries, 6 bytes each: word a = hull key-point index (24 bits,
// the row of the loop's key-point list) | the weight's exponent << 24, and a
// 16-bit word with the weight's top 16 mantissa bits (weights are >= 0;
// relative rounding error <= 2^-17).  Row r = unit * 32 + lane: with
// A = kRpA a words and 2A 16-bit words per chunk, its entries t..t+A-1 are
// one chunk of a words at u32 ((unit_off + t)/A * 32 + lane) * A + t % A and
// its entries t..t+2A-1 one chunk of 16-bit words at u16 ((unit_off +
// t)/(2A) * 32 + lane) * 2A + t % 2A (unit_off and unit lengths multiples of
// 2A): K-render loads a batch with coalesced 32-byte loads.
constexpr uint32_t kRplanIdxMask = 0xFFFFFFu;

__device__ __forceinline__ float rplan_weight(uint32_t a, uint32_t half16) {
    return __uint_as_float(((a >> 24) << 23) | (half16 << 7));
}

// Move the bits of a 3x3x3 stencil mask (bit jx*9 + jy*3 + jz) to the window
// slots ((r0 + jx) % 3) * 9 + ((r1 + jy) % 3) * 3 + (r2 + jz) % 3: a cyclic
// shift along each axis.
__device__ __forceinline__ uint32_t rotate_axis(uint32_t m, int r, uint32_t a0, int sh) {
    const uint32_t a1 = a0 << sh, a2 = a0 << (2 * sh);
    if (r == 1) return ((m & (a0 | a1)) << sh) | ((m & a2) >> (2 * sh));
    if (r == 2) return ((m & a0) << (2 * sh)) | ((m & (a1 | a2)) >> sh);
    return m;
}
__device__ __forceinline__ uint32_t rotate27(uint32_t m, int r0, int r1, int r2) {
    m = rotate_axis(m, r2, 0x1249249u, 1);                              // jz
    m = rotate_axis(m, r1, 0x7u | (0x7u << 9) | (0x7u << 18), 3);       // jy
    return rotate_axis(m, r0, 0x1FFu, 9);                               // jx
}

// Bytes per lane chunk of the plan layout: 32 (sm_100 LDG.256, units padded
// to 16 entries) or 16 (LDG.128, units padded to 8).  Config 2 K-render:
// 0.1012 / 0.1035 ms; one u32 load per entry was 0.118 ms.  The engine pads
// units to kRpB entries (fvr_rplan_chunk_entries).
#ifndef FVR_RPLAN_CHUNK
#define FVR_RPLAN_CHUNK 32
#endif
constexpr int kRpA = FVR_RPLAN_CHUNK / 4;  // a words per chunk
constexpr int kRpB = FVR_RPLAN_CHUNK / 2;  // 16-bit weight words per chunk

// 256-bit store of one lane chunk (sm_100 st.global.v8.b32)
__device__ __forceinline__ void store_zero_chunk(uint32_t* p) {
#if FVR_RPLAN_CHUNK == 32
    asm volatile("st.global.v8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"l"(p), "r"(0u) : "memory");
#else
    *reinterpret_cast<uint4*>(p) = make_uint4(0u, 0u, 0u, 0u);
#endif
}

// The fill's output for one row: entry t goes to its lane chunk (a word and
// 16-bit weight word) -- staged in registers and stored 32 bytes at a time
// (FVR_RPLAN_FILL_BUF); staging whole chunks in shared memory cost more
// instructions than the scattered stores (1.83 vs 1.62 ms at config 2).
// finish() pads the row with (0, 0.0) entries up to the unit's length --
// whole chunks with 32-byte stores -- so the plan buffers need no clearing.
// 6-byte fill output staged per lane chunk in registers (one 32-byte store
// per full chunk): config 2 render fill 1.42 -> 1.22 ms at 4 CTAs per SM
// (128 registers; 1.30 ms at 5 CTAs with spills)
#ifndef FVR_RPLAN_FILL_BUF
#define FVR_RPLAN_FILL_BUF 1
#endif
__device__ __forceinline__ void store_chunk(uint32_t* p, const uint32_t (&v)[8]) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

template <bool WIDE>
struct RplanOut {
    uint32_t* a;         // this row's first a word
    void* b;             // this row's first weight word (u16; u32 when WIDE)
#if FVR_RPLAN_FILL_BUF
    // (6-byte entries) the current lane chunks in registers, written as one
    // 32-byte store each when full: a warp's scattered 4- and 2-byte stores
    // touched 32 sectors per instruction
    uint32_t ab[8], bb[8];
    __device__ __forceinline__ void shift_in(uint32_t aw, uint32_t h) {
#pragma unroll
        for (int i = 0; i < 7; ++i) ab[i] = ab[i + 1];
        ab[7] = aw;
#pragma unroll
        for (int i = 0; i < 7; ++i) bb[i] = __funnelshift_r(bb[i], bb[i + 1], 16);
        bb[7] = (bb[7] >> 16) | (h << 16);
    }
#endif
    __device__ __forceinline__ void put(int t, int col, float w) {
#if FVR_RPLAN_FILL_BUF
        if (!WIDE) {
            FVR_DCHECK(col >= 0 && col < (1 << 24), "render plan: column not a hull key point");
            const uint32_t bits = (__float_as_uint(w) + 0x40u) >> 7;  // round to 16 mantissa bits
            shift_in((uint32_t)col | ((bits >> 16) << 24), bits & 0xFFFFu);
            if ((t & (kRpA - 1)) == kRpA - 1) store_chunk(a + (int64_t)(t / kRpA) * (32 * kRpA), ab);
            if ((t & (kRpB - 1)) == kRpB - 1)
                store_chunk(static_cast<uint32_t*>(b) + (int64_t)(t / kRpB) * (32 * kRpA), bb);
            return;
        }
#endif
        if (WIDE) {  // 8-byte entries: u32 column, f32 weight (hulls of >= 2^24 key points)
            a[(int64_t)(t / kRpA) * (32 * kRpA) + (t % kRpA)] = (uint32_t)col;
            static_cast<uint32_t*>(b)[(int64_t)(t / kRpA) * (32 * kRpA) + (t % kRpA)] = __float_as_uint(w);
            return;
        }
        FVR_DCHECK(col >= 0 && col < (1 << 24), "render plan: column not a hull key point");
        const uint32_t bits = (__float_as_uint(w) + 0x40u) >> 7;  // round to 16 mantissa bits
        a[(int64_t)(t / kRpA) * (32 * kRpA) + (t % kRpA)] = (uint32_t)col | ((bits >> 16) << 24);
        static_cast<uint16_t*>(b)[(int64_t)(t / kRpB) * (32 * kRpB) + (t % kRpB)] = (uint16_t)(bits & 0xFFFFu);
    }
    // entries count..len-1 are padding (len: the unit's length, a multiple of kRpB)
    __device__ __forceinline__ void finish(int count, int len) {
        FVR_DCHECK(count <= len, "render plan: row longer than its unit (count pass disagrees with fill)");
        constexpr int kB = WIDE ? kRpA : kRpB;  // weight words per chunk
        const int ca = (count + kRpA - 1) / kRpA * kRpA, cb = (count + kB - 1) / kB * kB;
#if FVR_RPLAN_FILL_BUF
        if (!WIDE) {  // pad the partial chunks in registers with (0, 0.0) and store them
            for (int t = count; t < cb; ++t) {
                shift_in(0u, 0u);
                if ((t & (kRpA - 1)) == kRpA - 1) store_chunk(a + (int64_t)(t / kRpA) * (32 * kRpA), ab);
                if ((t & (kRpB - 1)) == kRpB - 1)
                    store_chunk(static_cast<uint32_t*>(b) + (int64_t)(t / kRpB) * (32 * kRpA), bb);
            }
            for (int c = cb / kRpA; c < len / kRpA; ++c) store_zero_chunk(a + (int64_t)c * (32 * kRpA));
            for (int c = cb / kRpB; c < len / kRpB; ++c)
                store_zero_chunk(static_cast<uint32_t*>(b) + (int64_t)c * (32 * kRpA));
            return;
        }
#endif
        for (int t = count; t < ca; ++t) a[(int64_t)(t / kRpA) * (32 * kRpA) + (t % kRpA)] = 0u;
        for (int t = count; t < cb; ++t) {
            if (WIDE)
                static_cast<uint32_t*>(b)[(int64_t)(t / kRpA) * (32 * kRpA) + (t % kRpA)] = 0u;
            else
                static_cast<uint16_t*>(b)[(int64_t)(t / kRpB) * (32 * kRpB) + (t % kRpB)] = 0;
        }
        for (int c = ca / kRpA; c < len / kRpA; ++c) store_zero_chunk(a + (int64_t)c * (32 * kRpA));
        uint32_t* bw = static_cast<uint32_t*>(b);  // a weight chunk is kRpA u32 too
        for (int c = cb / kB; c < len / kB; ++c) store_zero_chunk(bw + (int64_t)c * (32 * kRpA));
    }
};


// Walk one pixel's ray exactly as K-render samples it and produce its row of
// B.  Which entries a row holds depends only on the geometry (a window slot
// holds an entry once a sample whose support covers it placed a `dynamic`
// key point there), so FILL = false counts them without evaluating any
// weight.  Key points not in `dynamic` (the loop's hull key points)
// contribute max(v, 0) * weight to base[c] (values: nch lattice planes).
// Interior scattering samples take their 27 weights from the moment form
// (moment_omega), face samples from the direct masked sum.
//
// The merge window holds the 3x3x3 key points around the last sample's
// nearest key point in toroidal slots (x mod 3, y mod 3, z mod 3) kept in
// shared memory (acc[slot * stride]): moving the window by one key point
// only retires the plane of slots it leaves, nothing is shifted.  dyn27[m]
// is the 27-bit mask of dynamic key points around m (one load per sample).
// Returns the entry count; t_fin receives the transparency after the last
// sample.
template <bool SCAT, bool FILL, bool WIDE = false>
__device__ int rplan_row(const double o[3], const double d[3], const Geom& g, const RenderConsts& rc,
                         const uint8_t* __restrict__ occ, const uint8_t* __restrict__ dynamic,
                         const uint32_t* __restrict__ dyn27, const float* __restrict__ values, int nch,
                         int64_t plane, const float* __restrict__ thr, const uint32_t* __restrict__ nm,
                         float* __restrict__ acc, float* __restrict__ wsm, int stride, RplanOut<WIDE>& out,
                         double* base, double& t_fin, const uint8_t* __restrict__ slot_tab = nullptr,
                         const int* __restrict__ kp_map = nullptr, int* __restrict__ skp = nullptr,
                         const uint32_t* __restrict__ pos27 = nullptr, const int* __restrict__ off27 = nullptr) {
    constexpr uint32_t kPX[3] = {0x1FFu, 0x1FFu << 9, 0x1FFu << 18};
    constexpr uint32_t kPY[3] = {0x7u | (0x7u << 9) | (0x7u << 18), (0x7u << 3) | (0x7u << 12) | (0x7u << 21),
                                 (0x7u << 6) | (0x7u << 15) | (0x7u << 24)};
    constexpr uint32_t kPZ[3] = {0x1249249u, 0x1249249u << 1, 0x1249249u << 2};
    int count = 0;
    double t_dst = 1.0;
    uint32_t live = 0;      // window slots holding an entry
    int wm[3] = {0, 0, 0};  // window centre
    bool have = false;
    const float sig_a = (float)rc.sigma_a, kappa = (float)rc.scat_scale;
    auto put = [&](int col, float wt) {  // col: the hull key point's column
        if (FILL) out.put(count, col, wt);
        ++count;
    };
    auto retire = [&](uint32_t slots) {
        if (!FILL) {  // count pass: one entry per retired slot
            count += __popc(slots);
            live &= ~slots;
            return;
        }
        // each slot's column was looked up when its key point entered the window
#pragma unroll 1
        for (uint32_t b = slots; b; b &= b - 1) {
            const int sl = __ffs(b) - 1;
            const float wt = acc[sl * stride];
            acc[sl * stride] = 0.f;
            put(skp[sl * stride], wt);
        }
        live &= ~slots;
    };
    double te, tx;
    if (slab_span(o, d, g, te, tx)) {
        const int n = sample_count(te, tx, g.edge);
        const double t0 = te - 0.5 * g.edge;
        double qb[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) qb[a] = ((o[a] - g.lo[a]) + t0 * d[a]) * g.inv_edge;
        const double nmax[3] = {(double)g.nx, (double)g.ny, (double)g.nz};
#pragma unroll 1
        for (int k = 1; k <= n; ++k, t_dst *= rc.one_minus_tau) {
            double q[3];
            int m[3];
            float dl[3];
            bool interior = true;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                q[a] = fma((double)k, d[a], qb[a]);
                interior = interior && q[a] >= 0.5 + 1e-7 && q[a] <= nmax[a] - 0.5 - 1e-7;
                m[a] = min(max((int)rint(q[a]), 0), a == 0 ? g.nx : (a == 1 ? g.ny : g.nz));
                dl[a] = (float)(q[a] - (double)m[a]);
            }
            const int mlin = m[0] * g.sx + m[1] * g.sy + m[2];
            if (occ) {
                // empty space: occ = D >= 2 bounds the L-inf distance from m to
                // any key point that may be non-zero, so samples k .. k+D-3 read
                // none (sample k+j stays within j+1 of m); skip them all, the
                // transparency advancing by repeated multiplication
                const int D = __ldg(occ + mlin);
                if (D > 1) {
                    const int extra = min(max(D - 3, 0), n - k);
                    for (int j = 0; j < extra; ++j) t_dst *= rc.one_minus_tau;
                    k += extra;
                    continue;
                }
            }
            const uint32_t sup = support_mask(SCAT, dl, thr, nm);
            const float scale = (float)(t_dst * rc.tau);
            if (!interior) {
                // within half a voxel of a box face: clamped stencil, entries unmerged
                if (have) retire(live);
                have = false;
                if (FILL) {
                    uint32_t inbox = 0xffffffffu;
                    if (SCAT) {
                        double p[3];
                        sample_pos(o, d, te, g.edge, k, p);
                        inbox = inbox_mask(p, g, rc.half_gather);
                    }
                    float w[27];
                    sample_weights<SCAT>(dl[0], dl[1], dl[2], sig_a, kappa, inbox, w);
#pragma unroll
                    for (int j = 0; j < 27; ++j) wsm[j * stride] = w[j] * scale;
                }
#pragma unroll 1
                for (uint32_t b = sup; b; b &= b - 1) {
                    const int j = __ffs(b) - 1, jx = j / 9, jy = (j / 3) % 3, jz = j % 3;
                    const int x = min(max(m[0] + jx - 1, 0), g.nx), y = min(max(m[1] + jy - 1, 0), g.ny),
                              z = min(max(m[2] + jz - 1, 0), g.nz);
                    const int kp = x * g.sx + y * g.sy + z;
                    const float wt = FILL ? wsm[j * stride] : 0.f;
                    if (__ldg(dynamic + kp)) {
                        put(FILL ? __ldg(kp_map + kp) : 0, wt);
                    } else if (FILL && values) {  // values == NULL: no static key point is positive
                        for (int c = 0; c < nch; ++c) base[c] += (double)wt * fmaxf(__ldg(values + c * plane + kp), 0.f);
                    }
                }
                continue;
            }
            const uint32_t dyn = __ldg(dyn27 + mlin);
            // move the window to m: retire the planes it leaves
            const int dx = m[0] - wm[0], dy = m[1] - wm[1], dz = m[2] - wm[2];
            if (have && abs(dx) <= 1 && abs(dy) <= 1 && abs(dz) <= 1) {
                uint32_t gone = 0;
                if (dx) gone |= kPX[(wm[0] - dx + 3) % 3];
                if (dy) gone |= kPY[(wm[1] - dy + 3) % 3];
                if (dz) gone |= kPZ[(wm[2] - dz + 3) % 3];
                if (gone & live) retire(gone & live);
            } else if (have) {
                retire(live);
            }
            wm[0] = m[0];
            wm[1] = m[1];
            wm[2] = m[2];
            have = true;
            // toroidal slot of offset (jx, jy, jz): ((m + j - 1) mod 3) per axis
            const int r0 = (m[0] + 2) % 3, r1 = (m[1] + 2) % 3, r2 = (m[2] + 2) % 3;
            float w[27];  // the sample's stencil weights (fill only; kept in registers for the merge)
            if (FILL) {
                if (SCAT) {
                    float2 om01[9];
                    float om2[9];
                    moment_omega(dl[0], dl[1], dl[2], thr, g_q1, g_q2, sig_a / kappa, om01, om2);
#pragma unroll
                    for (int l = 0; l < 9; ++l) {
                        w[3 * l] = kappa * om01[l].x;
                        w[3 * l + 1] = kappa * om01[l].y;
                        w[3 * l + 2] = kappa * om2[l];
                    }
                } else {
                    sample_weights<false>(dl[0], dl[1], dl[2], sig_a, kappa, 0xffffffffu, w);
                }
#pragma unroll
                for (int j = 0; j < 27; ++j) w[j] = __fmul_rn(w[j], scale);
                if (values) {  // the static base term reads them by stencil offset
#pragma unroll
                    for (int j = 0; j < 27; ++j) wsm[j * stride] = w[j];
                }
            }
            // the stencil's dynamic key points, moved to window slots at once
            // (count pass: that is all; config 2: 0.83 -> 0.36 ms)
            if (FILL) {
                // key points entering the window: look their columns up now,
                // four loads in flight at a time, so a retire reads shared
                // memory only (a lookup per retired entry stalled the fill)
                const uint32_t in_win = rotate27(live, (3 - r0) % 3, (3 - r1) % 3, (3 - r2) % 3);
                uint32_t fresh = sup & dyn & ~in_win;
                const uint8_t* tab = slot_tab + (r0 * 9 + r1 * 3 + r2) * 27;
                while (fresh) {
                    int j4[4], c4[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        j4[i] = fresh ? __ffs(fresh) - 1 : -1;
                        fresh &= fresh - 1;
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i) c4[i] = j4[i] < 0 ? 0 : __ldg(kp_map + mlin + off27[j4[i]]);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (j4[i] >= 0) skp[tab[j4[i]] * stride] = c4[i];
                }
            }
            live |= rotate27(sup & dyn, r0, r1, r2);
            if (FILL) {
                // merge into the window: unrolled over the 27 stencil offsets
                // (weights in registers, slot = per-axis residues), predicated
                // on the dynamic support -- no shared-memory weight round trip
                const uint32_t md = sup & dyn;
                const int SX[3] = {(r0 % 3) * 9, ((r0 + 1) % 3) * 9, ((r0 + 2) % 3) * 9};
                const int SY[3] = {(r1 % 3) * 3, ((r1 + 1) % 3) * 3, ((r1 + 2) % 3) * 3};
                const int SZ[3] = {r2 % 3, (r2 + 1) % 3, (r2 + 2) % 3};
#pragma unroll
                for (int j = 0; j < 27; ++j)
                    if ((md >> j) & 1u) acc[(SX[j / 9] + SY[(j / 3) % 3] + SZ[j % 3]) * stride] += w[j];
#pragma unroll 1
                // static key points with a positive value (pos27; none for the
                // reference's initial grid) fold into base
                for (uint32_t b = values ? sup & (pos27 ? __ldg(pos27 + mlin) : ~dyn) : 0u; b; b &= b - 1) {
                    const int j = __ffs(b) - 1;
                    const float wt = wsm[j * stride];
                    if (wt == 0.f) continue;
                    const int kp = mlin + (j / 9 - 1) * g.sx + ((j / 3) % 3 - 1) * g.sy + (j % 3 - 1);
                    for (int c = 0; c < nch; ++c) base[c] += (double)wt * fmaxf(__ldg(values + c * plane + kp), 0.f);
                }
            }
        }
        if (have) retire(live);
    }
    t_fin = t_dst;
    return count;
}

// dyn27[m] = bit (jx*9 + jy*3 + jz) set when key point m + (jx-1, jy-1, jz-1)
// is dynamic (interior key points; the border ones are never a window centre)
__global__ void rplan_dyn27_kernel(const uint8_t* __restrict__ dynamic, Geom g, uint32_t* __restrict__ dyn27) {
    const int64_t n = (int64_t)(g.nx + 1) * (g.ny + 1) * (g.nz + 1);
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const int z = (int)(k % (g.nz + 1)), y = (int)((k / (g.nz + 1)) % (g.ny + 1)), x = (int)(k / g.sx);
        uint32_t m = 0;
        if (x >= 1 && x < g.nx && y >= 1 && y < g.ny && z >= 1 && z < g.nz)
            for (int j = 0; j < 27; ++j)
                if (dynamic[k + (j / 9 - 1) * g.sx + ((j / 3) % 3 - 1) * g.sy + (j % 3 - 1)]) m |= 1u << j;
        dyn27[k] = m;
    }
}

// pos27[k]: the stencil key points around interior key point k that are
// static (not in `dynamic`) and positive in some channel -- the only static
// ones that add to a row's base (max(v, 0) = 0 for the rest).
__global__ void rplan_pos27_kernel(const uint8_t* __restrict__ dynamic, const float* __restrict__ values, int nch,
                                   int64_t plane, Geom g, uint32_t* __restrict__ pos27) {
    const int64_t n = (int64_t)(g.nx + 1) * (g.ny + 1) * (g.nz + 1);
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const int z = (int)(k % (g.nz + 1)), y = (int)((k / (g.nz + 1)) % (g.ny + 1)), x = (int)(k / g.sx);
        uint32_t m = 0;
        if (x >= 1 && x < g.nx && y >= 1 && y < g.ny && z >= 1 && z < g.nz)
            for (int j = 0; j < 27; ++j) {
                const int64_t q = k + (j / 9 - 1) * g.sx + ((j / 3) % 3 - 1) * g.sy + (j % 3 - 1);
                if (dynamic[q]) continue;
                bool pos = false;
                for (int c = 0; c < nch; ++c) pos = pos || values[c * plane + q] > 0.f;
                if (pos) m |= 1u << j;
            }
        pos27[k] = m;
    }
}

__device__ __forceinline__ void load_split_tables(float* s_thr, uint32_t* s_nm) {
    for (int i = threadIdx.x; i < 3 * kScatDirs; i += blockDim.x) s_thr[i] = (&c_thr[0][0])[i];
    for (int i = threadIdx.x; i < 3 * (kScatDirs + 1); i += blockDim.x) s_nm[i] = (&c_nmask[0][0])[i];
    __syncthreads();
}

// Pixel of natural row r = unit * 32 + lane (unit = 8x4 pixel tile, lanes
// row-major); false when the unit overhangs the bbox there.
__device__ __forceinline__ bool rplan_pixel(int64_t r, int units_x, int units_per_view, int w, int h, int& view,
                                            int& col, int& row) {
    const int unit = (int)(r >> 5), lane = (int)(r & 31);
    view = unit / units_per_view;
    const int u = unit - view * units_per_view;
    col = (u % units_x) * kUnitW + (lane % kUnitW);
    row = (u / units_x) * kUnitH + (lane / kUnitW);
    return col < w && row < h;
}

// Count pass: one warp per 8x4 unit, unit_len[unit] = longest row of the
// unit and, when row_len is given, row_len[r] = the length of natural row r.
template <bool SCAT>
__global__ void __launch_bounds__(128) rplan_count_kernel(
    const fvr_camera_t* __restrict__ cams, int u0, int v0, int w, int h, int units_x, int units_per_view,
    int n_units, Geom g, RenderConsts rc, const uint8_t* __restrict__ occ, const uint8_t* __restrict__ dynamic,
    const uint32_t* __restrict__ dyn27, int* __restrict__ unit_len, int* __restrict__ row_len) {
    __shared__ float s_thr[3 * kScatDirs];
    __shared__ uint32_t s_nm[3 * (kScatDirs + 1)];
    load_split_tables(s_thr, s_nm);
    const int unit = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (unit >= n_units) return;
    const int lane = threadIdx.x & 31;
    const int view = unit / units_per_view, u = unit - view * units_per_view;
    const int col = (u % units_x) * kUnitW + (lane % kUnitW), row = (u / units_x) * kUnitH + (lane / kUnitW);
    int cnt = 0;
    if (col < w && row < h) {
        const fvr_camera_t& cam = cams[view];
        double d[3], base[1] = {0.0}, t_fin;
        pixel_dir(cam, (double)(u0 + col) + 0.5, (double)(v0 + row) + 0.5, d);
        RplanOut<false> none{};
        cnt = rplan_row<SCAT, false>(cam.center, d, g, rc, occ, dynamic, dyn27, nullptr, 0, 0, s_thr, s_nm, nullptr,
                                     nullptr, 0, none, base, t_fin);
    }
    if (row_len) row_len[(int64_t)unit * 32 + lane] = cnt;
    cnt = (int)__reduce_max_sync(0xffffffffu, (unsigned)cnt);
    if (lane == 0) unit_len[unit] = cnt;
}

// Fill pass: rows in SELL-32 order; base[c * rows + r] and t_fin[r] per row
// r = unit * 32 + lane (entries beyond a row's length stay (0, 0.0)).
// Unbuffered stores: 5 CTAs per SM (96 registers, no spills): config 2 fill
// 1.44 ms, against 2.10 at the compiler's 122 registers (4 CTAs) and 1.48 at
// 6 (spills).  Register-staged chunks (FVR_RPLAN_FILL_BUF): 4 CTAs, 1.22 ms.
#ifndef FVR_RPLAN_FILL_MINB
#define FVR_RPLAN_FILL_MINB (FVR_RPLAN_FILL_BUF ? 4 : 5)
#endif
#ifndef FVR_RPLAN_FILL_WIDE_MINB
#define FVR_RPLAN_FILL_WIDE_MINB 5
#endif
template <bool SCAT, bool WIDE>
__global__ void __launch_bounds__(128, WIDE ? FVR_RPLAN_FILL_WIDE_MINB : FVR_RPLAN_FILL_MINB) rplan_fill_kernel(
    const fvr_camera_t* __restrict__ cams, int u0, int v0, int w, int h, int units_x, int units_per_view,
    int n_units, Geom g, RenderConsts rc, const uint8_t* __restrict__ occ, const uint8_t* __restrict__ dynamic,
    const uint32_t* __restrict__ dyn27, const float* __restrict__ values, int nch, int64_t plane,
    const long long* __restrict__ unit_off, const int* __restrict__ unit_order, const int* __restrict__ row_src,
    const int* __restrict__ kp_map, uint32_t* __restrict__ ent_a, uint32_t* __restrict__ ent_b,
    const uint32_t* __restrict__ pos27, double* __restrict__ base_out, double* __restrict__ t_fin_out) {
    __shared__ float s_acc[27 * 128], s_w[27 * 128];
    __shared__ int s_kp[27 * 128];  // column of the key point in each window slot
    for (int i = threadIdx.x; i < 27 * 128; i += blockDim.x) s_acc[i] = 0.f;
    __shared__ uint8_t s_slot[27 * 27];  // (residues r0 r1 r2, stencil offset j) -> window slot
    for (int i = threadIdx.x; i < 27 * 27; i += blockDim.x) {
        const int rr = i / 27, j = i % 27;
        s_slot[i] = (uint8_t)(((rr / 9 + j / 9) % 3) * 9 + (((rr / 3) % 3 + (j / 3) % 3) % 3) * 3 + (rr % 3 + j % 3) % 3);
    }
    __shared__ int s_off27[27];  // lattice offset of stencil slot j from the centre key point
    if (threadIdx.x < 27)
        s_off27[threadIdx.x] = (threadIdx.x / 9 - 1) * g.sx + ((threadIdx.x / 3) % 3 - 1) * g.sy + (threadIdx.x % 3 - 1);
    __shared__ float s_thr[3 * kScatDirs];
    __shared__ uint32_t s_nm[3 * (kScatDirs + 1)];
    load_split_tables(s_thr, s_nm);  // (its barrier also publishes s_off27)
    const int slot = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (slot >= n_units) return;
    const int unit = unit_order ? __ldg(unit_order + slot) : slot;  // longest first: a short tail
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)unit * 32 + lane, rows = (int64_t)n_units * 32;
    int view, col, row;
    const bool in = rplan_pixel(row_src ? __ldg(row_src + r) : r, units_x, units_per_view, w, h, view, col, row);
    double base[4] = {0.0, 0.0, 0.0, 0.0}, t_fin = 0.0;
    const long long uoff = unit_off[unit];
    RplanOut<WIDE> out;
    out.a = ent_a + ((uoff / kRpA) * 32 + lane) * kRpA;
    if (WIDE)
        out.b = ent_b + ((uoff / kRpA) * 32 + lane) * kRpA;
    else
        out.b = reinterpret_cast<uint16_t*>(ent_b) + ((uoff / kRpB) * 32 + lane) * kRpB;
    int count = 0;
    if (in) {
        const fvr_camera_t& cam = cams[view];
        double d[3];
        pixel_dir(cam, (double)(u0 + col) + 0.5, (double)(v0 + row) + 0.5, d);
        count = rplan_row<SCAT, true, WIDE>(cam.center, d, g, rc, occ, dynamic, dyn27, values, nch, plane, s_thr, s_nm,
                                      s_acc + threadIdx.x, s_w + threadIdx.x, 128, out, base, t_fin, s_slot, kp_map,
                                      s_kp + threadIdx.x, pos27, s_off27);
    }
    out.finish(count, (int)(unit_off[unit + 1] - uoff));
    for (int c = 0; c < nch; ++c) base_out[c * rows + r] = base[c];
    t_fin_out[r] = t_fin;
}

// K-render through the plan: one warp per unit, lane = pixel; rec = B c +
// base + t_fin bg, then the same residual / squared-residual epilogue as the
// marching kernel.  Products in fp32, summed in fp64 a batch at a time.
// Entries per lane in flight per batch x CTAs per SM (config 2, 16-byte
// chunks): 16x3 / 24x3 / 32x3 / 16x4: 0.1059 / 0.1061 / 0.105 / 0.112 ms
// (one u32 load per entry before: 16x3 / 24x3 / 32x3 / 32x2 / 24x4 / 16x4 /
// 48x2 / 64x3: 0.1245 / 0.1245 / 0.128 / 0.1248 / 0.128 / 0.1306 / 0.1307 /
// 0.1295 ms); ptxas keeps a batch's loads ahead of their uses only with the
// registers to hold them.
#ifndef FVR_RPLAN_BATCH
#define FVR_RPLAN_BATCH 32
#endif
#ifndef FVR_RPLAN_MINB
#define FVR_RPLAN_MINB 3
#endif
// The one-channel 6-byte render software-pipelined in batches of
// FVR_RPLAN_PIPE entries (0: the batch loop above): config 2 K-render 0.0911
// -> 0.0903 ms at 16 entries and 3 CTAs (80 registers); 16 at 4 / 5 CTAs and
// 32 at 2 CTAs lose (0.0912 / 0.1034 / 0.0976 ms;
// profiles/r2_ab_render_pipelined.log)
#ifndef FVR_RPLAN_PIPE
#define FVR_RPLAN_PIPE 16
#endif

// fvr_loop_finalize_t on the device (on = false: no fused finalize).
struct RplanFinalize {
    bool on;
    int n_views, bpv, n_vol;
    double pixels, n_kp, eps;
    long long* acc;  // (NCH, n_views + 1) fixed-point sums + overflow flag, or NULL
    char* discard;   // a dead buffer whose dirty L2 lines are dropped (rho), or NULL
    int64_t discard_lines;
    const double* vol;
    double* trace;
    double* trace_vol;
    int64_t trace_stride;
};

struct RpChunk {
    uint32_t w[kRpA];
};
__device__ __forceinline__ RpChunk rplan_stream(const uint32_t* p) {
    RpChunk c;
#if FVR_RPLAN_CHUNK == 32
    asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(c.w[0]), "=r"(c.w[1]), "=r"(c.w[2]), "=r"(c.w[3]), "=r"(c.w[4]), "=r"(c.w[5]), "=r"(c.w[6]),
          "=r"(c.w[7])
        : "l"(p));
#else
    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(p));
    c.w[0] = v.x;
    c.w[1] = v.y;
    c.w[2] = v.z;
    c.w[3] = v.w;
#endif
    return c;
}

// One unit (8x4 pixels, lane = pixel) of K-render through the plan.
template <int NCH, bool WIDE>
__device__ __forceinline__ void rplan_render_unit(
    int unit, int lane, const int* __restrict__ unit_len, const long long* __restrict__ unit_off,
    const uint32_t* __restrict__ ent_a, const uint32_t* __restrict__ ent_b, const double* __restrict__ base,
    const double* __restrict__ t_fin, const int* __restrict__ row_src, int64_t rows, int units_x,
    int units_per_view, int n_views, int w, int h, const float* __restrict__ src, const float* __restrict__ kpv,
    const RenderConsts& rc, float* __restrict__ residual, double* __restrict__ sq_partials, int64_t sq_stride,
    long long* __restrict__ sq_acc = nullptr, int bpv = 0) {
    // kpv: max(v, 0) per hull key point (NCH = 1: f32; NCH = 3: float4)
    const int len = unit_len[unit];  // a multiple of 8
    const long long off = unit_off[unit];  // a multiple of 8
    double acc[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[c] = 0.0;
    auto term = [&](uint32_t av, uint32_t bw, float* part) {  // bw: 16-bit weight word (u32 weight when WIDE)
        const float wgt = WIDE ? __uint_as_float(bw) : rplan_weight(av, bw);
        const uint32_t k = WIDE ? av : (av & kRplanIdxMask);
        if (NCH == 1) {
            part[0] = fmaf(wgt, __ldg(kpv + k), part[0]);
        } else {
            const float4 cv = __ldg(reinterpret_cast<const float4*>(kpv) + k);
            const float cc[3] = {cv.x, cv.y, cv.z};
#pragma unroll
            for (int c = 0; c < NCH; ++c) part[c] = fmaf(wgt, cc[c], part[c]);
        }
    };
    int t = 0;
    // three channels: a float4 operand per entry, so half the batch (no spills)
    constexpr int B = NCH > 1 ? 16 : FVR_RPLAN_BATCH;
    static_assert(B % kRpB == 0, "batches of whole chunks");
    const uint32_t* va = ent_a + ((off / kRpA) * 32 + lane) * kRpA;
    constexpr int kB = WIDE ? kRpA : kRpB;  // weight entries per (kRpA-word) chunk
    const uint32_t* vb = ent_b + ((off / kB) * 32 + lane) * kRpA;  // a weight chunk is kRpA u32 too
    auto batch = [&](auto nb, int t0) {  // nb = entries (a multiple of kRpB) from t0
        constexpr int N = decltype(nb)::value;
        RpChunk av[N / kRpA], bv[N / kB];
#pragma unroll
        for (int i = 0; i < N / kRpA; ++i) av[i] = rplan_stream(va + (int64_t)(t0 / kRpA + i) * (32 * kRpA));
#pragma unroll
        for (int i = 0; i < N / kB; ++i) bv[i] = rplan_stream(vb + (int64_t)(t0 / kB + i) * (32 * kRpA));
        float part[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) part[c] = 0.f;
#pragma unroll
        for (int i = 0; i < N; ++i) {
            if (WIDE) {
                term(av[i / kRpA].w[i % kRpA], bv[i / kRpA].w[i % kRpA], part);
            } else {
                const uint32_t hw = bv[i / kRpB].w[(i % kRpB) >> 1];
                term(av[i / kRpA].w[i % kRpA], (i & 1) ? (hw >> 16) : (hw & 0xFFFFu), part);
            }
        }
#pragma unroll
        for (int c = 0; c < NCH; ++c) acc[c] += (double)part[c];
    };
#if FVR_RPLAN_PIPE
    if constexpr (!WIDE && NCH == 1) {
        // software-pipelined: the next batch's chunks are loaded before this
        // batch's operand reads
        constexpr int D = FVR_RPLAN_PIPE;  // a multiple of kRpB
        static_assert(D % kRpB == 0, "batches of whole chunks");
        RpChunk ca[D / kRpA], cb[D / kRpB], na[D / kRpA], nb[D / kRpB];
        RpChunk zc;
#pragma unroll
        for (int i = 0; i < kRpA; ++i) zc.w[i] = 0u;
#pragma unroll
        for (int i = 0; i < D / kRpA; ++i) ca[i] = i * kRpA < len ? rplan_stream(va + (int64_t)i * (32 * kRpA)) : zc;
#pragma unroll
        for (int i = 0; i < D / kRpB; ++i) cb[i] = i * kRpB < len ? rplan_stream(vb + (int64_t)i * (32 * kRpA)) : zc;
        for (; t < len; t += D) {
            const int tn = t + D;
#pragma unroll
            for (int i = 0; i < D / kRpA; ++i)
                na[i] = tn + i * kRpA < len ? rplan_stream(va + (int64_t)(tn / kRpA + i) * (32 * kRpA)) : zc;
#pragma unroll
            for (int i = 0; i < D / kRpB; ++i)
                nb[i] = tn + i * kRpB < len ? rplan_stream(vb + (int64_t)(tn / kRpB + i) * (32 * kRpA)) : zc;
            float part[1] = {0.f};
#pragma unroll
            for (int i = 0; i < D; ++i) {
                const uint32_t hw = cb[i / kRpB].w[(i % kRpB) >> 1];
                term(ca[i / kRpA].w[i % kRpA], (i & 1) ? (hw >> 16) : (hw & 0xFFFFu), part);
            }
            acc[0] += (double)part[0];
#pragma unroll
            for (int i = 0; i < D / kRpA; ++i) ca[i] = na[i];
#pragma unroll
            for (int i = 0; i < D / kRpB; ++i) cb[i] = nb[i];
        }
    } else
#endif
    {
        for (; t + B <= len; t += B) batch(std::integral_constant<int, B>{}, t);
        for (; t < len; t += kRpB) batch(std::integral_constant<int, kRpB>{}, t);
    }
    const int64_t r = (int64_t)unit * 32 + lane;
    int view, col, row;
    const bool in = rplan_pixel(row_src ? __ldg(row_src + r) : r, units_x, units_per_view, w, h, view, col, row);
    const int64_t cstride = (int64_t)n_views * h * w;
    double sq[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) sq[c] = 0.0;
    if (in) {
        const int64_t pix = ((int64_t)view * h + row) * w + col;
        // (base NULL: no static term; t_fin NULL: a zero background -- both
        // add exactly +0.0, so skipping their 16 B per row changes no bit)
        const double tf = t_fin ? t_fin[r] : 0.0;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const double rec = acc[c] + (base ? base[c * rows + r] : 0.0) + tf * rc.bg[c];
            const double res = (double)src[c * cstride + pix] - rec;
            residual[pix * kResPitch<NCH> + c] = (float)res;
            sq[c] = res * res;
        }
    }
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const double tot = warp_sum(sq[c]);
        if (lane == 0) {
            sq_partials[c * sq_stride + unit] = tot;
            if (sq_acc) {  // the fused finalize's per-view fixed-point sum (see finalize_block)
                long long* a = sq_acc + c * (n_views + 1);
                atomicAdd(reinterpret_cast<unsigned long long*>(a + unit / units_per_view),
                          (unsigned long long)sq_fix(tot));
                if (!(tot < sq_fix_limit(bpv))) atomicExch(reinterpret_cast<unsigned long long*>(a + n_views), 1ull);
            }
        }
    }
}

template <int NCH, bool WIDE>
// CTA size (MINB counts are per 256 threads): 256 is the measured best
// (128 / 512: 0.0918 / 0.1018 ms against 0.0894; r2_ab_render_cta_size.log)
#ifndef FVR_RPLAN_THREADS
#define FVR_RPLAN_THREADS 256
#endif
__global__ void __launch_bounds__(FVR_RPLAN_THREADS, (NCH == 1 ? FVR_RPLAN_MINB : 2) * 256 / FVR_RPLAN_THREADS)
rplan_render_kernel(
    const int* __restrict__ unit_len, const long long* __restrict__ unit_off, const uint32_t* __restrict__ ent_a,
    const uint32_t* __restrict__ ent_b, const double* __restrict__ base, const double* __restrict__ t_fin,
    const int* __restrict__ unit_order, const int* __restrict__ row_src, int n_units, int units_x,
    int units_per_view, int n_views, int w, int h, const float* __restrict__ src, const float* __restrict__ kpv,
    RenderConsts rc, float* __restrict__ residual, double* __restrict__ sq_partials, int64_t sq_stride,
    fvr_loop_state_t* __restrict__ state, RplanFinalize fin) {
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    {  // the first unit's first chunks into L2 while the previous gather finishes
        const int u0 = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
        if (u0 < n_units) {
            const int unit = unit_order ? __ldg(unit_order + u0) : u0;
            const long long off = __ldg(unit_off + unit);
            const int len = __ldg(unit_len + unit);
            constexpr int kB = WIDE ? kRpA : kRpB;
            for (int i = 0; i < 4 && i * kRpA < len; ++i)
                prefetch_l2(ent_a + ((off / kRpA + i) * 32 + lane) * kRpA);
            for (int i = 0; i < 2 && i * kB < len; ++i) prefetch_l2(ent_b + ((off / kB + i) * 32 + lane) * kRpA);
        }
    }
    pdl_wait();  // the previous gather's operand update and state
    if (all_done<NCH>(state)) return;
    if (fin.discard) {  // (after the wait: the previous gather has read it)
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < fin.discard_lines;
             i += (int64_t)gridDim.x * blockDim.x)
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(fin.discard + i * 128) : "memory");
    }
    const int64_t rows = (int64_t)n_units * 32;
    // units longest first (unit_order): the block scheduler then hands the
    // short bbox-margin units to SMs as they free up, with no long unit left
    // for the tail (config 2: 0.157 -> 0.139 ms)
    for (int unit = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); unit < n_units;
         unit += (int)(((int64_t)gridDim.x * blockDim.x) >> 5)) {
#if FVR_RPLAN_NEXT_PREFETCH
        {  // (persistent grids) the warp's next unit's first chunks into L2
            const int nu = unit + (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
            if (nu < n_units) {
                const int un = unit_order ? __ldg(unit_order + nu) : nu;
                const long long off = __ldg(unit_off + un);
                const int len = __ldg(unit_len + un);
                constexpr int kB = WIDE ? kRpA : kRpB;
                for (int i = 0; i < 4 && i * kRpA < len; ++i)
                    prefetch_l2(ent_a + ((off / kRpA + i) * 32 + lane) * kRpA);
                for (int i = 0; i < 2 && i * kB < len; ++i) prefetch_l2(ent_b + ((off / kB + i) * 32 + lane) * kRpA);
            }
        }
#endif
        rplan_render_unit<NCH, WIDE>(unit_order ? __ldg(unit_order + unit) : unit, lane, unit_len, unit_off, ent_a, ent_b,
                               base, t_fin, row_src, rows, units_x, units_per_view, n_views, w, h, src, kpv, rc,
                               residual, sq_partials, sq_stride, fin.on ? fin.acc : nullptr, fin.bpv);
    }
    if (!fin.on) return;
    // the last block to finish runs the loop's finalize (fvr_loop.cu)
    __shared__ int s_last;
    __shared__ double s_view[33];  // (n_views + an overflow slot)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&state->work_retired, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int c = 0; c < NCH; ++c)
        finalize_block(sq_partials + c * sq_stride, fin.n_views, fin.bpv, fin.pixels,
                       fin.vol ? fin.vol + c * fin.n_vol : nullptr, fin.n_vol, fin.n_kp, fin.eps,
                       fin.trace + c * fin.trace_stride, fin.trace_vol ? fin.trace_vol + c * fin.trace_stride : nullptr,
                       state + c, s_view, fin.acc ? fin.acc + c * (fin.n_views + 1) : nullptr);
    if (threadIdx.x == 0) state->work_retired = 0;
}

// kpv[i] = max(v, 0) at hull key point kp[i] of every channel (NCH = 1: f32,
// NCH = 3: float4): the render plan's operand, kept current by the gather.
template <int NCH>
__global__ void rplan_pack_kernel(const float* __restrict__ values, int64_t plane, const int32_t* __restrict__ kp,
                                  int64_t n_kp, float* __restrict__ kpv, const fvr_loop_state_t* __restrict__ state) {
    if (state && all_done<NCH>(state)) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_kp; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = kp[i];
        if (NCH == 1)
            kpv[i] = fmaxf(values[k], 0.f);
        else
            reinterpret_cast<float4*>(kpv)[i] = make_float4(fmaxf(values[k], 0.f), fmaxf(values[plane + k], 0.f),
                                                            fmaxf(values[2 * plane + k], 0.f), 0.f);
    }
}

}  // namespace fvr
