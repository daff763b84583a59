// fvr_plan.cu -- K-adjust as a voxel-driven gather (deterministic mode).
//
// In deterministic mode (G = 1) every in-hull sample of every flame ray adds
// res[ray] * W to its 8 corner key points with W = alpha_l * (1-tau)^(k-1) *
// exp(-alpha_d' |p - corner|) (_kernels.py:290-306).  Rays, samples, cells
// and W depend only on the cameras, the grid and the hull -- not on the
// iteration -- so the back-projection of one iteration is the sparse
// product delta = A . res with a fixed A.  The plan (built once per
// reconstruct_channel call) stores A in CSR by hull key point: each entry is
// (index of the residual pixel, W).  Per iteration one warp per key point
// gathers its row, sums res * W in 32.32 fixed point (order-independent, so
// the result is bit-reproducible and identical under view sharding) and
// applies the clamped update -- no atomics, and ~8 bytes of streamed HBM
// traffic per (ray, corner) pair instead of an L2 read-modify-write.
//
// ncu on the ray-driven scatter (fvr_adjust.cu, kept for stochastic mode and
// the operator layer): 504 us per iteration at config 2, L2 56% busy with
// 62 M RED.ADD.64, IPC 1.25 (profiles/r1a_*).
#include "fvr_internal.cuh"

namespace fvr {

// Visit every in-hull sample of a ray: f(k, q[3], cell[3], trans).  Cells use
// q = qb + k*d (fp64) and fall back to the reference's exact expression
// (sample_pos + exact_cell) only when a coordinate is within 1e-9 of an
// integer; q_est differs from the exact quotient by < 1e-12 lattice units.
template <class F>
__device__ __forceinline__ void visit_inhull(const double o[3], const double d[3], const Geom& g,
                                             const uint8_t* __restrict__ inside, double tau_keep,
                                             F&& f) {
    double te, tx;
    if (!slab_span(o, d, g, te, tx)) return;
    const int n = sample_count(te, tx, g.edge);
    if (n < 1) return;
    const double t0 = te - 0.5 * g.edge;
    double qb[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) qb[a] = ((o[a] - g.lo[a]) + t0 * d[a]) * g.inv_edge;
    const int nn[3] = {g.nx, g.ny, g.nz};
    auto cell_of = [&](int k, double q[3], int c[3]) {
        bool safe = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            q[a] = fma((double)k, d[a], qb[a]);
            const double fl = floor(q[a]);
            const double fr = q[a] - fl;
            safe = safe && fr > 1e-9 && fr < 1.0 - 1e-9;
            c[a] = (int)fl;
        }
        if (!safe) {
            double p[3];
            sample_pos(o, d, te, g.edge, k, p);
#pragma unroll
            for (int a = 0; a < 3; ++a) c[a] = exact_cell(p[a], g.lo[a], g.edge, g.inv_edge);
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) c[a] = clampi(c[a], nn[a] - 1);
        return __ldg(inside + ((int64_t)c[0] * g.ny + c[1]) * g.nz + c[2]);
    };
    // the next sample's hull probe is issued before this sample's work, so
    // its latency overlaps the caller's (dependent) plan writes
    double q[3];
    int c[3];
    uint8_t in = cell_of(1, q, c);
    double trans = 1.0;
    for (int k = 1; k <= n; ++k) {
        double qn[3];
        int cn[3];
        uint8_t in_n = 0;
        if (k < n) in_n = cell_of(k + 1, qn, cn);
        if (in) f(k, q, c, trans);
        trans *= tau_keep;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            q[a] = qn[a];
            c[a] = cn[a];
        }
        in = in_n;
    }
}

struct PlanRay {
    double d[3];
    const double* o;
    int res_index;
};

__device__ __forceinline__ bool plan_ray(const fvr_camera_t* __restrict__ cams,
                                         const int32_t* __restrict__ ray_list, int64_t r, int u0,
                                         int v0, int w, int h, PlanRay& pr) {
    const int32_t e = ray_list[r];
    const int view = (int)((uint32_t)e >> 24), pix = e & 0xFFFFFF;
    const int row = pix / w, col = pix - row * w;
    const fvr_camera_t& cam = cams[view];
    pixel_dir(cam, (double)(u0 + col) + 0.5, (double)(v0 + row) + 0.5, pr.d);
    pr.o = cam.center;
    pr.res_index = view * w * h + pix;
    return true;
}

// The (key point, W) entries of one ray, with runs merged: consecutive
// in-hull samples whose cells share corners would emit the same key point
// again; a straight ray meets the 2x2x2 cell block around a key point in one
// contiguous run, so carrying the previous sample's 8 corners and summing
// matches removes most duplicates (about 2-3x fewer plan entries).  Count and
// fill run the identical merge, so their entry counts agree.
//
// A corner's plan row (kp_map) is looked up when its run starts and carried
// with it, so when the run ends one sample later the emit can go straight to
// the row's cursor atomic: the lookup's latency overlaps a whole sample
// instead of sitting on the fill's dependent chain.
// emit(kp[8], row[8], w[8], mask): the corners (bits of mask) whose run ended.
template <bool WEIGHTS, class Emit>
__device__ __forceinline__ void ray_entries(const PlanRay& pr, const Geom& g, const uint8_t* __restrict__ inside,
                                            double tau_keep, double alpha_l, float alpha_d,
                                            const int32_t* __restrict__ kp_map, Emit&& emit) {
    int pk[8], prow[8];
    float pw[8];
    bool have = false;
    const float edge = (float)g.edge;
    visit_inhull(pr.o, pr.d, g, inside, tau_keep, [&](int, const double* q, const int* c, double trans) {
        int nk[8], nrow[8];
        float nw[8];
        const int base_kp = c[0] * g.sx + c[1] * g.sy + c[2];
#pragma unroll
        for (int k8 = 0; k8 < 8; ++k8) nk[k8] = base_kp + (k8 >> 2) * g.sx + ((k8 >> 1) & 1) * g.sy + (k8 & 1);
        // which corners continue a run of the previous sample (their row and
        // weight so far come along), and which of the previous runs end
        uint32_t carried = 0, cont = 0;
#pragma unroll
        for (int n = 0; n < 8; ++n) {
            nrow[n] = 0;
            nw[n] = 0.f;
#pragma unroll
            for (int p = 0; p < 8; ++p)
                if (have && pk[p] == nk[n]) {
                    nrow[n] = prow[p];
                    if (WEIGHTS) nw[n] = pw[p];
                    carried |= 1u << p;
                    cont |= 1u << n;
                }
        }
#pragma unroll
        for (int n = 0; n < 8; ++n)
            if (!((cont >> n) & 1u)) nrow[n] = __ldg(kp_map + nk[n]);  // a run starts: its row
        if (WEIGHTS) {
            float e[3][2];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const float f = (float)(q[a] - (double)c[a]);
                e[a][0] = f * edge;
                e[a][1] = (f - 1.0f) * edge;
            }
            const float base = (float)(alpha_l * trans);
#pragma unroll
            for (int k8 = 0; k8 < 8; ++k8) {
                const int cx = k8 >> 2, cy = (k8 >> 1) & 1, cz = k8 & 1;
                const float dist = sqrtf(fmaf(e[0][cx], e[0][cx], fmaf(e[1][cy], e[1][cy], e[2][cz] * e[2][cz])));
                nw[k8] += base * expf(-alpha_d * dist);
            }
        }
        if (have) emit(pk, prow, pw, ~carried & 0xFFu);  // the corners whose run ended
#pragma unroll
        for (int k8 = 0; k8 < 8; ++k8) {
            pk[k8] = nk[k8];
            prow[k8] = nrow[k8];
            pw[k8] = nw[k8];
        }
        have = true;
    });
    if (have) emit(pk, prow, pw, 0xFFu);
}

__global__ void __launch_bounds__(128) plan_count_kernel(
    const fvr_camera_t* __restrict__ cams, const int32_t* __restrict__ ray_list, int64_t n_rays,
    int u0, int v0, int w, int h, const uint8_t* __restrict__ inside, Geom g,
    const int32_t* __restrict__ kp_map, int32_t* __restrict__ counts) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rays) return;
    PlanRay pr;
    plan_ray(cams, ray_list, r, u0, v0, w, h, pr);
    ray_entries<false>(pr, g, inside, 1.0, 0.0, 0.f, kp_map, [&](const int*, const int* row, const float*,
                                                                    uint32_t mask) {
#pragma unroll
        for (int p = 0; p < 8; ++p)
            if ((mask >> p) & 1u) atomicAdd(counts + row[p], 1);
    });
}

// int2 sample-plan entries per lane chunk: 2 (16-byte loads) or 4 (sm_100
// 32-byte loads; the engine pads sample-plan slices to 4 entries).  Config
// 2 sample-plan gather: 0.157 / 0.1525 ms.
#ifndef FVR_SPLAN_CHUNK
#define FVR_SPLAN_CHUNK 32
#endif
constexpr int kSE = FVR_SPLAN_CHUNK / 8;

// Plans are stored SELL-32: rows (hull key points) sorted by length within
// windows and cut into slices of 32; the row at sorted position p is lane
// p % 32 of slice p / 32, whose entries start at entry slice_off[p / 32] of
// every lane.  A lane's consecutive entries are packed into 16-byte chunks
// (store6 / put8_batch), so a warp streams a slice with fully coalesced
// LDG.128s, one lane per row (padding entries are (0, 0.0)).
struct SellMap {
    // per row: (entry offset of its slice) << 5 | its lane -- the SELL
    // position folded into one word, so a corner's entry address needs the
    // row lookup and then the cursor atomic and this word in parallel
    const long long* row_info;
    unsigned long long* cursor;      // per row, entries written so far
    // 6-byte entries in 16-byte chunks per lane (slice offsets and lengths
    // multiples of 8): entry e = off + t of lane l has its a word at u32
    // (e / 4 * 32 + l) * 4 + e % 4 and its 16-bit weight word at u16
    // (e / 8 * 32 + l) * 8 + e % 8, so the gather loads LDG.128s
    __device__ __forceinline__ static void store6(long long e, int l, uint32_t idx, float w, uint32_t* a,
                                                  uint16_t* b) {
        const uint32_t bits = (__float_as_uint(w) + 0x40u) >> 7;  // round to 16 mantissa bits (w >= 0)
        a[((e >> 2) * 32 + l) * 4 + (e & 3)] = idx | ((bits >> 16) << 24);
        b[((e >> 3) * 32 + l) * 8 + (e & 7)] = (uint16_t)(bits & 0xFFFFu);
    }
    // the 8 corner entries of one sample, int2 (sample id, W), batched as below
    __device__ __forceinline__ void put8_batch(const int* kp, const float* w, const int32_t* __restrict__ kp_map,
                                               int sid, int2* entries) const {
        int row[8];
        long long t[8], ri[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) row[i] = __ldg(kp_map + kp[i]);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            FVR_DCHECK(row[i] >= 0, "sample plan: corner is not a hull key point");
            t[i] = (long long)atomicAdd(cursor + row[i], 1ull);
            ri[i] = __ldg(row_info + row[i]);
        }
        // entry e = off + t of lane l at int2 (e / S * 32 + l) * S + e % S with
        // S = kSE: a lane's S consecutive entries are one chunk (slice offsets
        // and lengths multiples of S)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const long long e = (ri[i] >> 5) + t[i];
            entries[((e / kSE) * 32 + (ri[i] & 31)) * kSE + (e % kSE)] = make_int2(sid, __float_as_int(w[i]));
        }
    }
    // int2 (residual index, f32 W) entries of up to 8 corner runs (mask): the
    // wide deterministic plan, for residual indices of >= 2^24 (V * P)
    __device__ __forceinline__ void put_wide_batch(const int* row, const float* w, uint32_t mask, uint32_t idx,
                                                   int2* entries) const {
        long long t[8], ri[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if ((mask >> i) & 1u) {
                FVR_DCHECK(row[i] >= 0, "adjust plan: corner is not a hull key point");
                t[i] = (long long)atomicAdd(cursor + row[i], 1ull);
                ri[i] = __ldg(row_info + row[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if ((mask >> i) & 1u) {
                const long long e = (ri[i] >> 5) + t[i];
                entries[((e / kSE) * 32 + (ri[i] & 31)) * kSE + (e % kSE)] = make_int2((int)idx, __float_as_int(w[i]));
            }
        }
    }
    // up to 8 entries of one sample's corners (mask): each dependent step
    // (row lookup, then cursor atomic + row word) is issued for all of them
    // before any result is used, so their latencies overlap
    __device__ __forceinline__ void put6_batch(const int* row, const float* w, uint32_t mask, uint32_t idx,
                                               uint32_t* a, uint16_t* b) const {
        long long t[8], ri[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if ((mask >> i) & 1u) {
                FVR_DCHECK(row[i] >= 0, "adjust plan: corner is not a hull key point");
                t[i] = (long long)atomicAdd(cursor + row[i], 1ull);
                ri[i] = __ldg(row_info + row[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if ((mask >> i) & 1u) {
                FVR_DCHECK(idx < (1u << 24), "adjust plan: residual index beyond 24 bits");
                store6((ri[i] >> 5) + t[i], (int)(ri[i] & 31), idx, w[i], a, b);
            }
        }
    }
};

#ifndef FVR_PLAN_FILL_MINB
#define FVR_PLAN_FILL_MINB 3
#endif
template <bool WIDE>
__global__ void __launch_bounds__(128, FVR_PLAN_FILL_MINB) plan_fill_kernel(
    const fvr_camera_t* __restrict__ cams, const int32_t* __restrict__ ray_list, int64_t n_rays,
    int u0, int v0, int w, int h, const uint8_t* __restrict__ inside, Geom g, double tau_keep,
    double alpha_l, float alpha_d, const int32_t* __restrict__ kp_map, SellMap sm, uint32_t* __restrict__ ent_a,
    uint16_t* __restrict__ ent_b) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rays) return;
    PlanRay pr;
    plan_ray(cams, ray_list, r, u0, v0, w, h, pr);
    ray_entries<true>(pr, g, inside, tau_keep, alpha_l, alpha_d, kp_map,
                      [&](const int*, const int* row, const float* pw, uint32_t mask) {
        if (!WIDE)
            sm.put6_batch(row, pw, mask, (uint32_t)pr.res_index, ent_a, ent_b);
        else  // wide plan: int2 entries in ent_a
            sm.put_wide_batch(row, pw, mask, (uint32_t)pr.res_index, reinterpret_cast<int2*>(ent_a));
    });
}

// ---- stochastic mode: the sample plan ---------------------------------------
//
// With random G (reconstruct.py:193-201) each in-hull sample carries its own
// weight, so runs cannot be merged and the operator changes every iteration
// -- but only through the per-sample factor G.  The sample plan stores A
// unmerged, one entry (sample id, W) per (sample, corner); per iteration a
// flat kernel writes rho[sid] = res[ray] * G(seed, it, ray, k) with the same
// Philox key as the ray-driven scatter (fvr_adjust.cu), and the gather above
// runs over the plan with rho in place of the residual.
// Sample ids are laid out in blocks of 4 slots, one block per (ray, k >> 2)
// group with in-hull samples: sample (ray, k) has id 4 * block + (k & 3).  The
// 4 draws of a block come from one Philox block (gauss_block), so the weigh
// pass is one uniform thread per block (no divergence between lanes whose
// samples start a new group at different places); empty slots are never
// referenced by the plan.  ray_slots[r] = 4 * (groups of ray r).
__global__ void __launch_bounds__(128) splan_count_kernel(
    const fvr_camera_t* __restrict__ cams, const int32_t* __restrict__ ray_list, int64_t n_rays,
    int u0, int v0, int w, int h, const uint8_t* __restrict__ inside, Geom g,
    const int32_t* __restrict__ kp_map, int32_t* __restrict__ counts, int32_t* __restrict__ ray_slots) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rays) return;
    PlanRay pr;
    plan_ray(cams, ray_list, r, u0, v0, w, h, pr);
    int groups = 0, prev = -1;
    visit_inhull(pr.o, pr.d, g, inside, 1.0, [&](int k, const double*, const int* c, double) {
        const int base_kp = c[0] * g.sx + c[1] * g.sy + c[2];
#pragma unroll
        for (int k8 = 0; k8 < 8; ++k8)
            atomicAdd(counts + kp_map[base_kp + (k8 >> 2) * g.sx + ((k8 >> 1) & 1) * g.sy + (k8 & 1)], 1);
        if ((k >> 2) != prev) {
            prev = k >> 2;
            ++groups;
        }
    });
    ray_slots[r] = 4 * groups;
}

// E6: 6-byte entries (sample id < 2^24 | weight exponent, 16 mantissa bits;
// SellMap::store6 layout, read by the gather's 6-byte path); else int2.
// blk_keys (may be NULL): per block, (Morton code of the cell of its first
// sample) << 32 | block -- sorted, they renumber the blocks spatially
// (fvr_sample_plan_reorder).
__device__ __forceinline__ uint32_t spread10(uint32_t v) {
    v &= 0x3FFu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    return (v | (v << 2)) & 0x09249249u;
}

template <bool E6>
__global__ void __launch_bounds__(128) splan_fill_kernel(
    const fvr_camera_t* __restrict__ cams, const int32_t* __restrict__ ray_list, int64_t n_rays,
    int u0, int v0, int w, int h, const uint8_t* __restrict__ inside, Geom g, double tau_keep,
    double alpha_l, float alpha_d, const int32_t* __restrict__ kp_map, const long long* __restrict__ ray_sid0,
    SellMap sm, int2* __restrict__ entries, uint16_t* __restrict__ ent_b, int2* __restrict__ meta,
    unsigned long long* __restrict__ blk_keys) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rays) return;
    PlanRay pr;
    plan_ray(cams, ray_list, r, u0, v0, w, h, pr);
    long long blk = ray_sid0[r] / 4 - 1;  // block of the current group
    int prev = -1, mask = 0;
    const float edge = (float)g.edge;
    visit_inhull(pr.o, pr.d, g, inside, tau_keep, [&](int k, const double* q, const int* c, double trans) {
        if ((k >> 2) != prev) {
            if (prev >= 0) meta[blk] = make_int2((int)r, (prev << 4) | mask);
            prev = k >> 2;
            mask = 0;
            ++blk;
            if (blk_keys)
                blk_keys[blk] = ((unsigned long long)((spread10(c[0]) << 2) | (spread10(c[1]) << 1) | spread10(c[2]))
                                 << 32) | (unsigned long long)blk;
        }
        mask |= 1 << (k & 3);
        const long long sid = blk * 4 + (k & 3);
        float e[3][2];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float f = (float)(q[a] - (double)c[a]);
            e[a][0] = f * edge;
            e[a][1] = (f - 1.0f) * edge;
        }
        const float base = (float)(alpha_l * trans);
        const int base_kp = c[0] * g.sx + c[1] * g.sy + c[2];
        int kp[8];
        float wgt[8];
#pragma unroll
        for (int k8 = 0; k8 < 8; ++k8) {
            const int cx = k8 >> 2, cy = (k8 >> 1) & 1, cz = k8 & 1;
            const float dist = sqrtf(fmaf(e[0][cx], e[0][cx], fmaf(e[1][cy], e[1][cy], e[2][cz] * e[2][cz])));
            wgt[k8] = base * expf(-alpha_d * dist);
            kp[k8] = base_kp + cx * g.sx + cy * g.sy + cz;
        }
        if (E6) {
            int row[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) row[i] = __ldg(kp_map + kp[i]);
            sm.put6_batch(row, wgt, 0xFFu, (uint32_t)sid, reinterpret_cast<uint32_t*>(entries), ent_b);
        } else {
            sm.put8_batch(kp, wgt, kp_map, (int)sid, entries);
        }
    });
    if (prev >= 0) meta[blk] = make_int2((int)r, (prev << 4) | mask);
}

template <int NCH>
__global__ void __launch_bounds__(256) weighted_residual_kernel(
    const int2* __restrict__ bmeta, int64_t n_blocks, const int32_t* __restrict__ ray_list, int w, int h,
    const float* __restrict__ residual, uint64_t seed, float g_sigma, int64_t ray_id_base,
    float* __restrict__ rho, const fvr_loop_state_t* __restrict__ state, int it_back) {
    pdl_trigger();
    if ((int64_t)blockIdx.x * blockDim.x + threadIdx.x < n_blocks)  // its first meta word into L2
        prefetch_l2(bmeta + (int64_t)blockIdx.x * blockDim.x + threadIdx.x);
    pdl_wait();  // the render's residual and state
    // the live channels share the iteration count (a converged one stops
    // counting); it_back = 1 when this iteration's finalize already ran
    uint32_t it = 0;
    bool any = !state;
    if (state) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            any = any || !state[c].done;
            it = max(it, (uint32_t)state[c].it);
        }
    }
    if (!any) return;
    it -= (uint32_t)it_back;
    // one thread per 4-slot block (ray, group k >> 2): one Philox block and two
    // Box-Muller pairs give the group's four G values (gauss_weight's values,
    // bit for bit); every lane does the same work
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < n_blocks;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int2 m = __ldcs(bmeta + b);
        const int32_t e = __ldg(ray_list + m.x);
        const int64_t pix = (int64_t)((uint32_t)e >> 24) * w * h + (e & 0xFFFFFF);
        const uint4 blk = gauss_block(seed, it, (uint32_t)(ray_id_base + m.x), (uint32_t)(m.y >> 4));
        const float2 z01 = gauss_pair(blk.x, blk.y), z23 = gauss_pair(blk.z, blk.w);
        float gw[4] = {gauss_clip(z01.x, g_sigma), gauss_clip(z01.y, g_sigma), gauss_clip(z23.x, g_sigma),
                       gauss_clip(z23.y, g_sigma)};
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (!((m.y >> i) & 1)) gw[i] = 0.f;  // empty slot (never referenced by the plan)
        if (NCH == 1) {
            const float r = __ldg(residual + pix);
            __stcs(reinterpret_cast<float4*>(rho) + b, make_float4(r * gw[0], r * gw[1], r * gw[2], r * gw[3]));
        } else {
            const float4 r = __ldg(reinterpret_cast<const float4*>(residual) + pix);
            float4* d = reinterpret_cast<float4*>(rho) + 4 * b;
#pragma unroll
            for (int i = 0; i < 4; ++i) __stcs(d + i, make_float4(r.x * gw[i], r.y * gw[i], r.z * gw[i], 0.f));
        }
    }
}

// NCH channels share the plan (A depends only on geometry and hull): each
// entry is read once and multiplies NCH residuals (interleaved per pixel /
// sample: one 16-byte load for three channels); values / layout are NCH
// lattice planes, packed (NCH, n_rows), state NCH loop states (a converged
// channel is left untouched).  One warp per SELL slice, one lane per row,
// delta = sum_e res[idx_e] * W_e in 32.32 fixed point (order-independent).
#ifndef FVR_GATHER_BATCH
#define FVR_GATHER_BATCH 32
#endif
// The merged plan's gather (6-byte entries) is software-pipelined in batches
// of FVR_GATHER_PIPE entries at 5 CTAs per SM (46 registers): config 2
// K-adjust 0.0527 ms unpipelined (batch 32, 4 CTAs) -> 0.0500 / 0.0514 /
// 0.0489 ms pipelined at 16 / 24 / 8 (8: 5 CTAs).  The sample plan's gather
// (rho reads instead of residuals) keeps the unpipelined loop: pipelined it
// took 0.100 / 0.107 ms against 0.0985 (profiles/r2_ab_gather_pipelined.log).
#ifndef FVR_GATHER_PIPE
#define FVR_GATHER_PIPE 8
#endif
// the int2 sample plan: batch 32 / 24 / 16 = 0.190 (spills) / 0.157 / 0.169 ms
// at config 2 with entry pairs per load; with 32-byte chunks 24 / 16 = 0.1525 /
// 0.1565 ms
#ifndef FVR_SPLAN_BATCH
#define FVR_SPLAN_BATCH 24
#endif
// CTAs per SM: 6-byte entries leave room for 4 (config 2, deterministic,
// batch x CTAs 32x3 / 32x4 / 32x5 / 24x5 / 16x4 / 64x2: 0.0763 / 0.0718 /
// 0.0718 / 0.0714 / 0.0766 / 0.0845 ms); the int2 sample plan keeps 3.
#ifndef FVR_GATHER_E6_MINB
#define FVR_GATHER_E6_MINB 4
#endif
#ifndef FVR_GATHER_PIPE_MINB
#define FVR_GATHER_PIPE_MINB 5
#endif
// (three channels, unpipelined: FVR_GATHER3_MINB CTAs, batch FVR_GATHER3_BATCH)
#ifndef FVR_GATHER3_E6_MINB
#define FVR_GATHER3_E6_MINB 3
#endif
#define FVR_GATHER3_MINB(E6) ((E6) ? FVR_GATHER3_E6_MINB : 2)
#ifndef FVR_GATHER3_BATCH
#define FVR_GATHER3_BATCH 16
#endif
#define FVR_GATHER_MINB(E6, PIPE, NCH)                                                         \
    ((PIPE) ? ((NCH) == 1 ? FVR_GATHER_PIPE_MINB : 4)                                          \
            : (NCH) > 1 ? FVR_GATHER3_MINB(E6) : (E6) ? FVR_GATHER_E6_MINB : 3)
template <bool PACKED, int NCH, bool E6, bool PIPE>
// CTA size: 128 threads (4 slices) at the same warps per SM as 256-thread
// CTAs (the MINB counts above are per 256 threads): config 2 K-adjust 0.0490
// -> 0.0485 ms (512: 0.0563; profiles/r2_ab_gather_cta_size.log)
#ifndef FVR_GATHER_THREADS
#define FVR_GATHER_THREADS 128
#endif
__global__ void __launch_bounds__(FVR_GATHER_THREADS, FVR_GATHER_MINB(E6, PIPE, NCH) * 256 / FVR_GATHER_THREADS)
gather_kernel(
    const int32_t* __restrict__ slice_len, const long long* __restrict__ slice_off,
    const int32_t* __restrict__ row_of_pos, const int2* __restrict__ entries, const uint32_t* __restrict__ ent_b,
    int64_t n_rows,
    const float* __restrict__ residual, const int32_t* __restrict__ kp_index,
    float* __restrict__ values, int64_t plane, float* __restrict__ layout, int layout_kind, int sy, int ny1,
    float* __restrict__ kpv, long long* __restrict__ packed, const fvr_loop_state_t* __restrict__ state) {
    pdl_trigger();
    {  // the first slice's first chunks into L2 while the predecessor finishes
        const int64_t sl0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        if (sl0 < ((n_rows + 31) >> 5)) {
            const long long off = __ldg(slice_off + sl0);
            const int len = __ldg(slice_len + sl0);
            const int ln = threadIdx.x & 31;
            if (E6) {
                for (int i = 0; i < 8 && 4 * i < len; ++i)
                    prefetch_l2(reinterpret_cast<const uint4*>(entries) + ((off >> 2) + i) * 32 + ln);
                for (int i = 0; i < 4 && 8 * i < len; ++i)
                    prefetch_l2(reinterpret_cast<const uint4*>(ent_b) + ((off >> 3) + i) * 32 + ln);
            } else {
                for (int i = 0; i < 6 && kSE * i < len; ++i)
                    prefetch_l2(entries + ((off / kSE + i) * 32 + ln) * kSE);
            }
        }
    }
    pdl_wait();  // the render's residual / the weigh's rho, and the state
    bool live[NCH];
    bool any = false;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        live[c] = !(state && state[c].done);
        any = any || live[c];
    }
    if (!any) return;
    const int lane = threadIdx.x & 31;
    const int64_t n_slices = (n_rows + 31) >> 5;
    // three channels: a float4 residual per entry, so half the batch (no spills)
    constexpr int B = NCH > 1 ? (PIPE ? 16 : FVR_GATHER3_BATCH) : E6 ? FVR_GATHER_BATCH : FVR_SPLAN_BATCH;
    for (int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; sl < n_slices;
         sl += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int len = slice_len[sl];
        const long long off = slice_off[sl];
        // the row's update operands, loaded now so their latency hides under
        // the row's entries (the end-of-slice update stalled on them)
        const int64_t pos0 = sl * 32 + lane;
        const int64_t row0 = pos0 < n_rows ? (int64_t)__ldg(row_of_pos + pos0) : 0;
        const int64_t idx0 = (!PACKED && pos0 < n_rows) ? (int64_t)__ldg(kp_index + row0) : 0;
        float v0[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) v0[c] = (!PACKED && pos0 < n_rows) ? values[c * plane + idx0] : 0.f;
        const int2* e = entries + ((off / kSE) * 32 + lane) * kSE;  // chunks of kSE entries
        // E6: 6-byte entries (fvr_adjust_plan_fill, SellMap::store6): 16-byte
        // chunks of a words in `entries`, of 16-bit weight words in ent_b
        const uint4* ea = reinterpret_cast<const uint4*>(entries) + (off >> 2) * 32 + lane;
        const uint4* eb = reinterpret_cast<const uint4*>(ent_b) + (off >> 3) * 32 + lane;
        long long acc[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) acc[c] = 0;
        if constexpr (E6 && PIPE) {
            // software-pipelined: the next batch's chunks are loaded before
            // this batch's residual reads, so the plan stream keeps flowing
            // while the warp waits on L1/L2
            constexpr int D = FVR_GATHER_PIPE > 0 ? FVR_GATHER_PIPE : 8;  // entries per batch (a multiple of 8)
            static_assert(D % 8 == 0, "batches of whole 16-byte chunks");
            const uint4 z = make_uint4(0u, 0u, 0u, 0u);
            uint4 ca[D / 4], cb[D / 8], na[D / 4], nb[D / 8];
#pragma unroll
            for (int i = 0; i < D / 4; ++i) ca[i] = 4 * i < len ? __ldcs(ea + (int64_t)i * 32) : z;
#pragma unroll
            for (int i = 0; i < D / 8; ++i) cb[i] = 8 * i < len ? __ldcs(eb + (int64_t)i * 32) : z;
            for (int t = 0; t < len; t += D) {
                const int tn = t + D;
#pragma unroll
                for (int i = 0; i < D / 4; ++i) na[i] = tn + 4 * i < len ? __ldcs(ea + (int64_t)(tn / 4 + i) * 32) : z;
#pragma unroll
                for (int i = 0; i < D / 8; ++i) nb[i] = tn + 8 * i < len ? __ldcs(eb + (int64_t)(tn / 8 + i) * 32) : z;
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    const uint4& q = ca[i / 4];
                    const uint32_t a = (i & 3) == 0 ? q.x : (i & 3) == 1 ? q.y : (i & 3) == 2 ? q.z : q.w;
                    const uint4& h = cb[i / 8];
                    const uint32_t hw = ((i & 7) >> 1) == 0 ? h.x : ((i & 7) >> 1) == 1 ? h.y : ((i & 7) >> 1) == 2 ? h.z : h.w;
                    const uint32_t half = (i & 1) ? (hw >> 16) : (hw & 0xFFFFu);
                    const int idx = (int)(a & 0xFFFFFFu);
                    const float wgt = __uint_as_float(((a >> 24) << 23) | (half << 7));
                    if (NCH == 1) {
                        acc[0] += __float2ll_rn(__ldg(residual + idx) * wgt * 4294967296.0f);
                    } else {
                        const float4 r = __ldg(reinterpret_cast<const float4*>(residual) + idx);
                        const float rr[3] = {r.x, r.y, r.z};
#pragma unroll
                        for (int c = 0; c < NCH; ++c) acc[c] += __float2ll_rn(rr[c] * wgt * 4294967296.0f);
                    }
                }
#pragma unroll
                for (int i = 0; i < D / 4; ++i) ca[i] = na[i];
#pragma unroll
                for (int i = 0; i < D / 8; ++i) cb[i] = nb[i];
            }
        } else
        for (int t = 0; t < len; t += B) {
            int2 en[B];
            if (E6) {
                static_assert(B % 8 == 0, "batches of whole 16-byte chunks");
                uint4 av[B / 4], bv[B / 8];
                const uint4 z = make_uint4(0u, 0u, 0u, 0u);
#if FVR_PLAN_EVICT_FIRST
                uint64_t pol;
                asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
                auto ldp = [&](const uint4* ptr) {
                    uint4 r;
                    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(ptr), "l"(pol));
                    return r;
                };
#pragma unroll
                for (int i = 0; i < B / 4; ++i) av[i] = t + 4 * i < len ? ldp(ea + (int64_t)(t / 4 + i) * 32) : z;
#pragma unroll
                for (int i = 0; i < B / 8; ++i) bv[i] = t + 8 * i < len ? ldp(eb + (int64_t)(t / 8 + i) * 32) : z;
#else
#pragma unroll
                for (int i = 0; i < B / 4; ++i) av[i] = t + 4 * i < len ? __ldcs(ea + (int64_t)(t / 4 + i) * 32) : z;
#pragma unroll
                for (int i = 0; i < B / 8; ++i) bv[i] = t + 8 * i < len ? __ldcs(eb + (int64_t)(t / 8 + i) * 32) : z;
#endif
#pragma unroll
                for (int i = 0; i < B; ++i) {
                    const uint4& q = av[i / 4];
                    const uint32_t a = (i & 3) == 0 ? q.x : (i & 3) == 1 ? q.y : (i & 3) == 2 ? q.z : q.w;
                    const uint4& h = bv[i / 8];
                    const uint32_t hw = ((i & 7) >> 1) == 0 ? h.x : ((i & 7) >> 1) == 1 ? h.y : ((i & 7) >> 1) == 2 ? h.z : h.w;
                    const uint32_t half = (i & 1) ? (hw >> 16) : (hw & 0xFFFFu);
                    en[i] = make_int2((int)(a & 0xFFFFFFu), (int)(((a >> 24) << 23) | (half << 7)));
                }
            } else {
                static_assert(E6 || B % kSE == 0, "batches of whole chunks");
#pragma unroll
                for (int i = 0; i < B / kSE; ++i) {
                    const int2* q = e + (int64_t)(t / kSE + i) * (32 * kSE);
#if FVR_SPLAN_CHUNK == 32
                    uint32_t w[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
                    if (t + kSE * i < len)
                        asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                            : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
                              "=r"(w[7])
                            : "l"(q));
#pragma unroll
                    for (int j = 0; j < 4; ++j) en[4 * i + j] = make_int2((int)w[2 * j], (int)w[2 * j + 1]);
#else
                    const int4 v = t + 2 * i < len ? __ldcs(reinterpret_cast<const int4*>(q)) : make_int4(0, 0, 0, 0);
                    en[2 * i] = make_int2(v.x, v.y);
                    en[2 * i + 1] = make_int2(v.z, v.w);
#endif
                }
            }
#pragma unroll
            for (int i = 0; i < B; ++i) {
                const float wgt = __int_as_float(en[i].y);
                if (NCH == 1) {
#if FVR_RHO_EVICT_LAST
                    float rv;
                    uint64_t pol;
                    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
                    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(rv) : "l"(residual + en[i].x), "l"(pol));
                    acc[0] += __float2ll_rn(rv * wgt * 4294967296.0f);
#else
                    acc[0] += __float2ll_rn(__ldg(residual + en[i].x) * wgt * 4294967296.0f);
#endif
                } else {
                    const float4 r = __ldg(reinterpret_cast<const float4*>(residual) + en[i].x);
                    const float rr[3] = {r.x, r.y, r.z};
#pragma unroll
                    for (int c = 0; c < NCH; ++c) acc[c] += __float2ll_rn(rr[c] * wgt * 4294967296.0f);
                }
            }
        }
        if (pos0 >= n_rows) continue;
        const int64_t row = row0;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            if (PACKED) {
                packed[c * n_rows + row] = acc[c];
            } else if (live[c] && acc[c] != 0) {
                const int64_t idx = idx0;
                float* vals = values + c * plane;
                const double nv = (double)v0[c] + (double)acc[c] * kFixInv;
                const float f = (float)(nv > -1.0 ? nv : -1.0);
                vals[idx] = f;
                if (layout) layout_store(layout + 4 * c, NCH, layout_kind, sy, ny1, idx, f);
                if (kpv) kpv[row * (NCH == 1 ? 1 : 4) + c] = fmaxf(f, 0.f);  // the render plan's operand
            }
        }
    }
}

// Apply a packed (all-reduced) correction: one thread per hull key point.
__global__ void update_packed_kernel(const long long* __restrict__ packed, int64_t n_rows,
                                     const int32_t* __restrict__ kp_index, float* __restrict__ values,
                                     float* __restrict__ layout, int layout_kind, int layout_nch, int sy, int ny1,
                                     float* __restrict__ kpv, int kpv_pitch,
                                     const fvr_loop_state_t* __restrict__ state) {
    if (state && state->done) return;
    for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n_rows;
         row += (int64_t)gridDim.x * blockDim.x) {
        const long long acc = packed[row];
        if (acc == 0) continue;
        const int64_t idx = kp_index[row];
        const double nv = (double)values[idx] + (double)acc * kFixInv;
        const float f = (float)(nv > -1.0 ? nv : -1.0);
        values[idx] = f;
        if (layout) layout_store(layout, layout_nch, layout_kind, sy, ny1, idx, f);
        if (kpv) kpv[row * kpv_pitch] = fmaxf(f, 0.f);
    }
}

}  // namespace fvr

using namespace fvr;

extern "C" int fvr_adjust_plan_count(const fvr_camera_t* cams, const int32_t* ray_list, int64_t n_rays,
                                     int32_t u0, int32_t v0, int32_t bbox_w, int32_t bbox_h,
                                     const uint8_t* inside_vox, fvr_grid_t grid, const int32_t* kp_map,
                                     int32_t* row_counts, void* stream) {
    FVR_TRY_BEGIN
    if (int rc = check_grid(grid)) return rc;
    if (n_rays == 0) return FVR_OK;
    const Geom g = make_geom(grid);
    plan_count_kernel<<<(unsigned)((n_rays + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        cams, ray_list, n_rays, u0, v0, bbox_w, bbox_h, inside_vox, g, kp_map, row_counts);
    return check_launch("adjust_plan_count");
    FVR_TRY_END
}

extern "C" int fvr_adjust_plan_fill(const fvr_camera_t* cams, const int32_t* ray_list, int64_t n_rays,
                                    int32_t u0, int32_t v0, int32_t bbox_w, int32_t bbox_h,
                                    const uint8_t* inside_vox, fvr_grid_t grid, double tau,
                                    double alpha_l, double alpha_d, const int32_t* kp_map,
                                    const int64_t* row_info, int64_t* cursor,
                                    uint32_t* entries_a, uint32_t* entries_b, void* stream) {
    FVR_TRY_BEGIN
    if (int rc = check_grid(grid)) return rc;
    if (n_rays == 0) return FVR_OK;
    const Geom g = make_geom(grid);
    const SellMap sm{reinterpret_cast<const long long*>(row_info), reinterpret_cast<unsigned long long*>(cursor)};
    const unsigned blocks = (unsigned)((n_rays + 127) / 128);
    if (entries_b)  // 6-byte entries (the wide path is a separate instance: its registers slowed this one 0.92 -> 1.54 ms)
        plan_fill_kernel<false><<<blocks, 128, 0, (cudaStream_t)stream>>>(
            cams, ray_list, n_rays, u0, v0, bbox_w, bbox_h, inside_vox, g, 1.0 - tau, alpha_l, (float)alpha_d, kp_map,
            sm, entries_a, reinterpret_cast<uint16_t*>(entries_b));
    else
        plan_fill_kernel<true><<<blocks, 128, 0, (cudaStream_t)stream>>>(
            cams, ray_list, n_rays, u0, v0, bbox_w, bbox_h, inside_vox, g, 1.0 - tau, alpha_l, (float)alpha_d, kp_map,
            sm, entries_a, nullptr);
    return check_launch("adjust_plan_fill");
    FVR_TRY_END
}

extern "C" int fvr_loop_gather(const int32_t* slice_len, const int64_t* slice_off, const int32_t* row_of_pos,
                               const int32_t* entries, const uint32_t* entries_b, int64_t n_kp, const float* residual, int32_t n_channels,
                               const int32_t* kp_index, float* values, float* layout, int32_t layout_kind,
                               fvr_grid_t grid, float* kp_values, int64_t* packed, const fvr_loop_state_t* state,
                               int32_t sample_plan, void* stream) {
    FVR_TRY_BEGIN
    if (n_kp == 0) return FVR_OK;
    if (n_channels != 1 && n_channels != 3) return set_error(FVR_ERR_INVALID, "the loop gathers 1 or 3 channels");
    const int64_t n_slices = (n_kp + 31) / 32;
    int64_t blocks = (n_slices * 32 + FVR_GATHER_THREADS - 1) / FVR_GATHER_THREADS;
    // (a grid-stride loop beyond 148 x 24 CTAs of 256 threads: the same warps for any CTA size)
#ifdef FVR_GATHER_CAP
    const int64_t cap = FVR_GATHER_CAP;
#else
    const int64_t cap = 148 * 24 * 256 / FVR_GATHER_THREADS;
#endif
    if (blocks > cap) blocks = cap;
    const int sy = grid.nz + 1, ny1 = grid.ny + 1;
    const int64_t plane = (int64_t)(grid.nx + 1) * (grid.ny + 1) * (grid.nz + 1);
    cudaStream_t st = (cudaStream_t)stream;
    const auto* so = reinterpret_cast<const long long*>(slice_off);
    const auto* en = reinterpret_cast<const int2*>(entries);
    long long* pk = reinterpret_cast<long long*>(packed);
    cudaError_t e = cudaSuccess;
#define FVR_GATHER(P, C, E, Q)                                                                                \
    e = launch_pdl(gather_kernel<P, C, E, Q>, (unsigned)blocks, FVR_GATHER_THREADS, st, slice_len, so, row_of_pos, en, entries_b,  \
                   n_kp, residual, kp_index, values, plane, layout, layout_kind, sy, ny1, kp_values, pk, state)
#define FVR_GATHER_E(P, C)                                 \
    if (entries_b && !sample_plan && FVR_GATHER_PIPE > 0) FVR_GATHER(P, C, true, true); \
    else if (entries_b) FVR_GATHER(P, C, true, false);           \
    else FVR_GATHER(P, C, false, false)
    if (packed) {
        if (n_channels == 1) { FVR_GATHER_E(true, 1); } else { FVR_GATHER_E(true, 3); }
    } else {
        if (n_channels == 1) { FVR_GATHER_E(false, 1); } else { FVR_GATHER_E(false, 3); }
    }
#undef FVR_GATHER_E
#undef FVR_GATHER
    if (e != cudaSuccess) return set_error(FVR_ERR_CUDA, std::string("loop_gather: ") + cudaGetErrorString(e));
    return check_launch("loop_gather");
    FVR_TRY_END
}

extern "C" int fvr_loop_update_packed(const int64_t* packed, int64_t n_kp, const int32_t* kp_index,
                                      float* values, float* layout, int32_t layout_kind, int32_t layout_nch,
                                      fvr_grid_t grid, float* kp_values, int32_t kp_values_pitch,
                                      const fvr_loop_state_t* state, void* stream) {
    FVR_TRY_BEGIN
    if (n_kp == 0) return FVR_OK;
    int64_t blocks = (n_kp + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    update_packed_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const long long*>(packed), n_kp, kp_index, values, layout, layout_kind, layout_nch,
        grid.nz + 1, grid.ny + 1, kp_values, kp_values_pitch, state);
    return check_launch("loop_update_packed");
    FVR_TRY_END
}

extern "C" int fvr_sample_plan_count(const fvr_camera_t* cams, const int32_t* ray_list, int64_t n_rays,
                                     int32_t u0, int32_t v0, int32_t bbox_w, int32_t bbox_h,
                                     const uint8_t* inside_vox, fvr_grid_t grid, const int32_t* kp_map,
                                     int32_t* row_counts, int32_t* ray_samples, void* stream) {
    FVR_TRY_BEGIN
    if (int rc = check_grid(grid)) return rc;
    if (n_rays == 0) return FVR_OK;
    const Geom g = make_geom(grid);
    splan_count_kernel<<<(unsigned)((n_rays + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        cams, ray_list, n_rays, u0, v0, bbox_w, bbox_h, inside_vox, g, kp_map, row_counts, ray_samples);
    return check_launch("sample_plan_count");
    FVR_TRY_END
}

extern "C" int fvr_sample_plan_fill(const fvr_camera_t* cams, const int32_t* ray_list, int64_t n_rays,
                                    int32_t u0, int32_t v0, int32_t bbox_w, int32_t bbox_h,
                                    const uint8_t* inside_vox, fvr_grid_t grid, double tau, double alpha_l,
                                    double alpha_d, const int32_t* kp_map, const int64_t* ray_sid0,
                                    const int64_t* row_info, int64_t* cursor,
                                    int32_t* entries, uint32_t* entries_b, int32_t* sample_meta,
                                    int64_t* block_keys, void* stream) {
    FVR_TRY_BEGIN
    if (int rc = check_grid(grid)) return rc;
    if (n_rays == 0) return FVR_OK;
    const Geom g = make_geom(grid);
    const SellMap sm{reinterpret_cast<const long long*>(row_info), reinterpret_cast<unsigned long long*>(cursor)};
    const unsigned blocks = (unsigned)((n_rays + 127) / 128);
    if (entries_b)
        splan_fill_kernel<true><<<blocks, 128, 0, (cudaStream_t)stream>>>(
            cams, ray_list, n_rays, u0, v0, bbox_w, bbox_h, inside_vox, g, 1.0 - tau, alpha_l, (float)alpha_d, kp_map,
            reinterpret_cast<const long long*>(ray_sid0), sm, reinterpret_cast<int2*>(entries),
            reinterpret_cast<uint16_t*>(entries_b), reinterpret_cast<int2*>(sample_meta),
            reinterpret_cast<unsigned long long*>(block_keys));
    else
        splan_fill_kernel<false><<<blocks, 128, 0, (cudaStream_t)stream>>>(
            cams, ray_list, n_rays, u0, v0, bbox_w, bbox_h, inside_vox, g, 1.0 - tau, alpha_l, (float)alpha_d, kp_map,
            reinterpret_cast<const long long*>(ray_sid0), sm, reinterpret_cast<int2*>(entries), nullptr,
            reinterpret_cast<int2*>(sample_meta), reinterpret_cast<unsigned long long*>(block_keys));
    return check_launch("sample_plan_fill");
    FVR_TRY_END
}

// Renumber the sample plan's blocks: sid -> new_of_nat[sid >> 2] * 4 + (sid & 3)
// in every stored entry (6-byte: the low 24 bits of the a word; int2: .x),
// and meta_out[new] = meta_in[nat].
template <bool E6>
__global__ void splan_renumber_kernel(uint32_t* __restrict__ words, int64_t n_entries,
                                      const int32_t* __restrict__ new_of_nat) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_entries;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (E6) {
            const uint32_t a = words[i];
            const uint32_t sid = a & 0xFFFFFFu;
            words[i] = (a & 0xFF000000u) | (uint32_t)(__ldg(new_of_nat + (sid >> 2)) * 4 + (sid & 3));
        } else {
            const uint32_t sid = words[2 * i];
            words[2 * i] = (uint32_t)(__ldg(new_of_nat + (sid >> 2)) * 4 + (sid & 3));
        }
    }
}
__global__ void splan_permute_meta_kernel(const int2* __restrict__ meta_in, int64_t n_blocks,
                                          const int32_t* __restrict__ new_of_nat, int2* __restrict__ meta_out) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < n_blocks; b += (int64_t)gridDim.x * blockDim.x)
        meta_out[__ldg(new_of_nat + b)] = meta_in[b];
}

extern "C" int fvr_sample_plan_reorder(int32_t* entries, int64_t n_slots, int32_t e6, const int32_t* new_of_nat,
                                       int64_t n_blocks, const int32_t* meta_in, int32_t* meta_out, void* stream) {
    FVR_TRY_BEGIN
    if (!entries || !new_of_nat || !meta_in || !meta_out) return set_error(FVR_ERR_INVALID, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    int64_t b = (n_slots + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    if (n_slots > 0) {
        if (e6)
            splan_renumber_kernel<true><<<(unsigned)b, 256, 0, st>>>(reinterpret_cast<uint32_t*>(entries), n_slots,
                                                                      new_of_nat);
        else
            splan_renumber_kernel<false><<<(unsigned)b, 256, 0, st>>>(reinterpret_cast<uint32_t*>(entries), n_slots,
                                                                       new_of_nat);
        count_launch(1);
    }
    int64_t bb = (n_blocks + 255) / 256;
    if (bb > 148 * 16) bb = 148 * 16;
    if (n_blocks > 0)
        splan_permute_meta_kernel<<<(unsigned)bb, 256, 0, st>>>(reinterpret_cast<const int2*>(meta_in), n_blocks,
                                                                new_of_nat, reinterpret_cast<int2*>(meta_out));
    return check_launch("sample_plan_reorder");
    FVR_TRY_END
}

__global__ void stochastic_g_kernel(uint64_t seed, uint32_t iteration, const uint32_t* __restrict__ ray,
                                    const uint32_t* __restrict__ k, int64_t n, float sigma, float* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = gauss_weight(seed, iteration, ray[i], k[i], sigma);
}

extern "C" int fvr_stochastic_g(uint64_t seed, uint32_t iteration, const uint32_t* ray, const uint32_t* k,
                                int64_t n, double g_sigma, float* out, void* stream) {
    FVR_TRY_BEGIN
    if (n <= 0) return FVR_OK;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    stochastic_g_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(seed, iteration, ray, k, n,
                                                                            (float)g_sigma, out);
    return check_launch("stochastic_g");
    FVR_TRY_END
}

extern "C" int fvr_loop_weighted_residual(const int32_t* sample_meta, int64_t n_samples, const int32_t* ray_list,
                                          int32_t bbox_w, int32_t bbox_h, const float* residual,
                                          int32_t n_channels, uint64_t seed, double g_sigma, int64_t ray_id_base,
                                          float* rho, const fvr_loop_state_t* state, int32_t state_advanced,
                                          void* stream) {
    FVR_TRY_BEGIN
    if (n_samples == 0) return FVR_OK;
    if (n_channels != 1 && n_channels != 3) return set_error(FVR_ERR_INVALID, "1 or 3 channels");
    if (n_samples % 4) return set_error(FVR_ERR_INVALID, "sample slots come in blocks of 4");
    const int64_t n_blocks = n_samples / 4;
    int64_t blocks = (n_blocks + 255) / 256;  // one thread per 4-slot block
    if (blocks > 148 * 16) blocks = 148 * 16;
    const auto* meta = reinterpret_cast<const int2*>(sample_meta);
    cudaError_t e;
    if (n_channels == 1)
        e = launch_pdl(weighted_residual_kernel<1>, (unsigned)blocks, 256, (cudaStream_t)stream,
            meta, n_blocks, ray_list, bbox_w, bbox_h, residual, seed, (float)g_sigma, ray_id_base, rho, state,
            state_advanced ? 1 : 0);
    else
        e = launch_pdl(weighted_residual_kernel<3>, (unsigned)blocks, 256, (cudaStream_t)stream,
            meta, n_blocks, ray_list, bbox_w, bbox_h, residual, seed, (float)g_sigma, ray_id_base, rho, state,
            state_advanced ? 1 : 0);
    if (e != cudaSuccess) return set_error(FVR_ERR_CUDA, std::string("loop_weighted_residual: ") + cudaGetErrorString(e));
    return check_launch("loop_weighted_residual");
    FVR_TRY_END
}
