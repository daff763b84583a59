/*
 * fvr_b200.h -- C ABI of libfvr_b200.so, the sm_100a implementation of the
 * iterative RTE flame-volume reconstruction loop (arXiv 1809.06417).
 *
 * Every entry point takes plain pointers and sizes (no torch types), is
 * asynchronous on the caller's cudaStream_t (passed as void*), and returns
 * an int status: FVR_OK, or an FVR_ERR_* code with a message available from
 * fvr_last_error() (thread-local).  Device pointers are owned by the caller
 * (the reference's ownership rule, _kernels.py: callers allocate every
 * output and kernels write in place).  The *_host variants take host
 * pointers and do their own staging; they are synchronous.
 *
 * Reference interfaces each group replaces (paths relative to
 * /root/reference/pkg/src/fvr/):
 *   fvr_render_rays[_host]       _kernels.py:101-186  render_rays
 *   fvr_count_hull_samples[_host]_kernels.py:189-224  count_hull_samples
 *   fvr_adjust_rays[_host]       _kernels.py:227-306  adjust_rays_chunked
 *   fvr_apply_correction         reconstruct.py:221-226 (fixed-order merge + clamp)
 *   fvr_render_pixels            render.py:183-217 render_pixels (rays built on device
 *                                from geometry.py:125-137 pixel_rays)
 *   fvr_loop_*                   reconstruct.py:304-334 (one iteration of the loop of
 *                                reconstruct_channel: render, RMSE, convergence rule,
 *                                residual, adjust_pass)
 *   fvr_ctmap_build              radiometry.py:173-203 build_color_temp_map
 *   fvr_temp_lookup              radiometry.py:206-219 temp_from_green +
 *                                reconstruct.py:444-455 green_to_temp
 *   fvr_temp_rgb                 reconstruct.py:389-401 rgb_grids_from_temperature (+ the
 *                                fused green -> T -> RGB snapshot path)
 *   fvr_visual_hull              volume.py:272-328 compute_visual_hull
 *   fvr_comm_* / fvr_allreduce_sum  reconstruct.py:181-226 (the per-view loop and fixed-order
 *                                merge, sharded over GPUs)
 */
#ifndef FVR_B200_H
#define FVR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FVR_ABI_VERSION 1

#define FVR_OK 0
#define FVR_ERR_INVALID 1    /* maps to ValueError */
#define FVR_ERR_CUDA 2       /* maps to RuntimeError */
#define FVR_ERR_EMPTY_HULL 3 /* maps to EmptyHullError */
#define FVR_ERR_NO_FLAME 4   /* maps to NoFlameError */

/* Voxel lattice geometry: nx*ny*nz cubic voxels of side `edge`, key points
 * (nx+1)(ny+1)(nz+1) stored C-order (z fastest), volume.py:62-120. */
typedef struct fvr_grid {
    int32_t nx, ny, nz, reserved;
    double origin[3];
    double edge;
} fvr_grid_t;

/* Pinhole camera, geometry.py:24-60.  rotation is world->camera, row-major;
 * center is the optical center -R^T t as computed by the host. */
typedef struct fvr_camera {
    double fx, fy, cx, cy;
    double rotation[9];
    double center[3];
    int32_t width, height;
} fvr_camera_t;

/* RenderConfig (render.py:29-48) plus the kernel-level extras of
 * render_rays (_kernels.py:101-116). */
typedef struct fvr_render_params {
    double tau;
    double sigma_a;
    double sigma_s;
    double phase_g;
    double gather_dist;
    int32_t scattering; /* bool */
    int32_t n_scat;     /* rows of scat_dirs */
} fvr_render_params_t;

/* Device-resident loop state (one per reconstruct_channel call). */
typedef struct fvr_loop_state {
    int32_t it;        /* iterations whose RMSE has been recorded */
    int32_t done;      /* convergence rule fired: later launches are no-ops */
    int32_t converged; /* trace.converged */
    int32_t reserved;
    double prev_rmse;
    int32_t work_next;    /* K-render work queue: next unit to hand out */
    int32_t work_retired; /* warps that found the queue empty (the last one resets both) */
} fvr_loop_state_t;

/* fvr_loop_finalize's arguments for a kernel that runs it in its last block
 * (fvr_rplan_render): per channel c, the RMSE partials are sq_partials + c *
 * sq_stride (n_views x blocks_per_view), the volume partials vol_partials +
 * c * n_vol_blocks (NULL: none), the traces trace_rmse / trace_vol + c *
 * trace_stride.  sq_accum (may be NULL; zeroed once by the caller): per
 * channel n_views + 1 int64 -- the per-view squared-residual sums in fixed
 * point (2^-24) that the render's units accumulate, then an overflow flag;
 * the finalize reads and re-zeroes them.  Per-view sums are integer sums of
 * the per-unit partials rounded to 2^-24 in every finalize (fused, separate,
 * sharded), so all agree to the bit; a partial beyond 2^38 / blocks_per_view
 * switches every path to the f64 sums of the partials.  l2_discard: the
 * stochastic mode's rho, consumed by the previous gather and rewritten by the
 * next weigh pass -- discard.global.L2 over it (128-byte lines) keeps its
 * ~33 MB of dirty lines from being written back while the render streams. */
typedef struct fvr_loop_finalize {
    int32_t n_views;
    int32_t blocks_per_view;
    int64_t pixels_per_view;
    const double* vol_partials;
    int32_t n_vol_blocks;
    int32_t reserved;
    int64_t n_kp;
    double converge_eps;
    double* trace_rmse;
    double* trace_vol;
    int64_t trace_stride;
    int64_t* sq_accum;
    void* l2_discard;           /* (may be NULL) a buffer that is dead once this render starts: its */
    int64_t l2_discard_bytes;   /* dirty L2 lines are dropped instead of written back (see below) */
} fvr_loop_finalize_t;

const char* fvr_last_error(void);
int fvr_abi_version(void);
/* Number of kernels this library has launched since load (for bench.py's
 * gpu_launches claim). */
int64_t fvr_launch_count(void);

/* ---- operator layer: drop-ins for fvr._kernels ------------------------- */

/* render_rays: dirs (n_rays,3) f64, values (n_channels, lattice) f32,
 * scat_dirs (n_scat,3) f64 (device), background host (n_channels) f64,
 * out (n_rays, n_channels) f64. n_channels <= 4.  layout (optional, device,
 * n_channels * lattice * 4 f32) is scratch for the packed copy the fast
 * evaluators read (see fvr_render_layout_kind); NULL selects the general
 * per-sample path.  occ (optional, device, lattice u8) is scratch for the
 * empty-space occupancy map (fvr_occupancy) the fast paths skip with. */
int fvr_render_rays(const double origin[3], const double* dirs, int64_t n_rays,
                    const float* values, int32_t n_channels, fvr_grid_t grid,
                    fvr_render_params_t params, const double* background,
                    const double* scat_dirs, float* layout, uint8_t* occ, double* out, void* stream);
int fvr_render_rays_host(const double origin[3], const double* dirs, int64_t n_rays,
                         const float* values, int32_t n_channels, fvr_grid_t grid,
                         fvr_render_params_t params, const double* background,
                         const double* scat_dirs, double* out);

/* count_hull_samples: inside_vox (nx,ny,nz) u8, counts (n_rays) i64. */
int fvr_count_hull_samples(const double origin[3], const double* dirs, int64_t n_rays,
                           const uint8_t* inside_vox, fvr_grid_t grid, int64_t* counts,
                           void* stream);
int fvr_count_hull_samples_host(const double origin[3], const double* dirs, int64_t n_rays,
                                const uint8_t* inside_vox, fvr_grid_t grid, int64_t* counts);

/* adjust_rays_chunked: deposits into a signed 32.32 fixed-point lattice
 * accum (lattice) i64 instead of f64 chunk partials; integer sums are
 * order-independent, so the result is bit-reproducible. */
int fvr_adjust_rays(const double origin[3], const double* dirs, int64_t n_rays,
                    const double* residuals, const double* g_values, const int64_t* g_offsets,
                    int32_t use_g, const uint8_t* inside_vox, fvr_grid_t grid, double tau,
                    double alpha_l, double alpha_d, int64_t* accum, void* stream);
/* Host variant: same contract as the reference (partials (n_chunks,lattice)
 * f64 accumulated in place; the device sum lands in chunk 0). */
int fvr_adjust_rays_host(const double origin[3], const double* dirs, int64_t n_rays,
                         const double* residuals, const double* g_values,
                         const int64_t* g_offsets, int32_t use_g, const uint8_t* inside_vox,
                         fvr_grid_t grid, double tau, double alpha_l, double alpha_d,
                         double* partials, int32_t n_chunks);

/* v = f32(max(f64(v) + accum * 2^-32, -1)); accum = 0 -- over the listed
 * key points (kp_index, n_kp) or, when kp_index is NULL, over all n. */
int fvr_apply_correction(float* values, int64_t* accum, const int32_t* kp_index, int64_t n,
                         void* stream);

/* ---- forward render of pixel centres (render_pixels / render_view) ----- */

/* us, vs (n) f64 device; out (n, n_channels) f64 device.  When us == NULL
 * the full frame is rendered with pixel centres u+0.5, v+0.5 (render_view). */
int fvr_render_pixels(const fvr_camera_t* camera, const double* us, const double* vs,
                      int64_t n, const float* values, int32_t n_channels, fvr_grid_t grid,
                      fvr_render_params_t params, const double* background,
                      const double* scat_dirs, float* layout, uint8_t* occ, double* out, void* stream);

/* Every pixel centre of n_views same-size cameras (cams: device array) in one
 * launch; out (n_views, height, width, n_channels) f32.  layout / occ must
 * have been prepared with fvr_pack_layout / fvr_occupancy (or be NULL). */
int fvr_render_views(const fvr_camera_t* cams, int32_t n_views, int32_t width, int32_t height,
                     const float* values, int32_t n_channels, fvr_grid_t grid,
                     fvr_render_params_t params, const double* background, const double* scat_dirs,
                     const float* layout, const uint8_t* occ, float* out, void* stream);

/* Packed copies of max(v, 0) read by the fast render paths: kind 1 (YZQ,
 * emission only) or 2 (Z4, single scattering); 0 = none applies.  The Z4
 * path needs the 32 Fibonacci directions loaded once per process with
 * fvr_set_scatter_dirs (radiometry.py:222-230, gather = edge, g = 0). */
int fvr_set_scatter_dirs(const double* dirs_host, int32_t n);
int fvr_render_layout_kind(fvr_render_params_t params, fvr_grid_t grid);
/* layout: float4 per (key point, channel), channels interleaved (element
 * j * n_channels + c), so the channels of one key point share cache lines. */
int fvr_pack_layout(const float* values, int32_t n_channels, fvr_grid_t grid, int32_t kind,
                    float* layout, void* stream);
/* occ[j] = 1 when a key point within Chebyshev distance 1 of j is positive in
 * some channel or set in force_mask (lattice u8, may be NULL).  Samples whose
 * neighbourhood is unoccupied contribute exactly 0 and are skipped. */
int fvr_occupancy(const float* values, int32_t n_channels, const uint8_t* force_mask,
                  fvr_grid_t grid, uint8_t* occ, void* stream);

/* ---- one iteration of the reconstruction loop (device resident) ------- */

/* Launch configuration the loop render uses; blocks_per_view sizes the
 * sq_partials buffer (n_views * blocks_per_view f64). */
int fvr_loop_blocks_per_view(int32_t bbox_w, int32_t bbox_h);

/* Render every bbox pixel of every view, residual = src - rec (f32), and
 * per-block squared-residual sums (f64). cams is a device array.
 * n_channels (1, or 3 for the batched RGB loop, reconstruct.py:370-385)
 * channels share the rays: src is (n_channels, V, h, w), residual (V, h, w,
 * pitch) with the channels interleaved (pitch 1, or 4 for 3 channels), values
 * and layout hold n_channels lattice planes, background[c] per channel,
 * sq_partials[c * sq_stride + unit], and state points at n_channels loop
 * states (the launch is a no-op once every channel is done). */
int fvr_loop_render(const fvr_camera_t* cams, int32_t n_views, int32_t u0, int32_t v0,
                    int32_t bbox_w, int32_t bbox_h, const float* src, const float* values,
                    const float* layout, const uint8_t* occ, fvr_grid_t grid, fvr_render_params_t params,
                    const double* background, int32_t n_channels, const double* scat_dirs, float* residual,
                    double* sq_partials, int64_t sq_stride, fvr_loop_state_t* state, void* stream);

/* K-render as a fixed operator (the render plan, csrc/fvr_rplan.cuh).  The
 * loop's forward model is linear in max(v, 0) with geometry-only weights, so
 * rec = B c + base + t_fin * bg.  B is stored SELL-32 by K-render's 8x4
 * pixel units: unit_len[unit] (count pass) = longest row of the unit
 * (the caller rounds it up to even); unit_off = exclusive scan of unit_len.
 * Entry t of row (unit, lane) is 6 bytes: entries_a[(unit_off[unit] + t) *
 * 32 + lane] = column | weight exponent << 24, and the weight's top 16
 * mantissa bits in half t % 2 of entries_b[((unit_off[unit] + t) / 2) * 32 +
 * lane] (weights >= 0, relative rounding <= 2^-17).  Columns are the
 * key points flagged in `dynamic` (the loop's hull key points), numbered by
 * kp_map (lattice -> index in the loop's key-point list); the others fold
 * into base (n_channels x rows f64, rows = n_units * 32) from `values`.
 * Needs the fast render modes (g = 0, gather = edge, 32 directions loaded);
 * occ is the distance map (may be NULL).
 * fvr_rplan_render replaces fvr_loop_render with identical outputs (to the
 * weight rounding); its operand kp_values holds max(v, 0) per hull key point
 * (f32, or float4 for 3 channels): fvr_rplan_pack fills it, and
 * fvr_loop_gather / fvr_loop_update_packed keep it current.  Fill and
 * render visit the units in the
 * order unit_order (a permutation of the units, longest first; NULL =
 * natural order).  Row r = unit * 32 + lane renders the pixel of natural row
 * row_src[r] (NULL = r; natural row q is lane q % 32 of the 8x4 pixel unit
 * q / 32): the caller sorts the rows of a few neighbouring units by length
 * (row_len from the count pass) so a unit's rows need less padding.  With
 * `finalize` (single-rank loops) the last block to finish runs
 * fvr_loop_finalize on state (one launch less per iteration; the block
 * counter is state[0].work_retired).
 * fvr_rplan_fill with values == NULL asserts that no key point outside
 * `dynamic` is positive (base then holds zeros); fvr_rplan_render may then
 * take base == NULL, and t_fin == NULL when every background is 0 (each adds
 * exactly +0.0, so the outputs are the same bits without streaming them).
 * wide != 0 (fill and render must agree): 8-byte entries, u32 column in
 * entries_a and f32 weight in entries_b at the same layout as entries_a
 * (entries_b holds unit_off-total u32) -- for hulls of >= 2^24 key points,
 * whose columns do not fit the 24-bit field. */
/* Entries per lane chunk of the render-plan layout: unit_len and unit_off
 * must be multiples of it (the caller pads unit_len from the count pass). */
int fvr_rplan_chunk_entries(void);
int fvr_rplan_count(const fvr_camera_t* cams, int32_t n_views, int32_t u0, int32_t v0, int32_t bbox_w,
                    int32_t bbox_h, fvr_grid_t grid, fvr_render_params_t params, const uint8_t* occ,
                    const uint8_t* dynamic, int32_t* unit_len, int32_t* row_len, void* stream);
int fvr_rplan_fill(const fvr_camera_t* cams, int32_t n_views, int32_t u0, int32_t v0, int32_t bbox_w,
                   int32_t bbox_h, fvr_grid_t grid, fvr_render_params_t params, const uint8_t* occ,
                   const uint8_t* dynamic, const float* values, int32_t n_channels, const int64_t* unit_off,
                   const int32_t* unit_order, const int32_t* row_src, const int32_t* kp_map,
                   uint32_t* entries_a, uint32_t* entries_b, double* base, double* t_fin, const uint32_t* pos27, int32_t wide, void* stream);
/* pos27[k] (lattice, u32): the stencil key points around interior key point k
 * that are static (not in dynamic) and positive in some channel -- the only
 * static ones a row's base needs.  fvr_rplan_fill computes it itself when its
 * pos27 argument is NULL; computing it early (right after the count pass)
 * keeps it off the fill's critical path. */
int fvr_rplan_pos27(fvr_grid_t grid, const uint8_t* dynamic, const float* values, int32_t n_channels,
                    uint32_t* pos27, void* stream);
/* Sort keys of the render plan's unit order (units longest class first, in
 * `buckets` classes up to the longest unit, *max_len on the device; 2x4-unit
 * tiles inside a class): ascending keys = visiting order. */
int fvr_rplan_unit_keys(const int32_t* unit_len, int32_t n_views, int32_t bbox_w, int32_t bbox_h, int32_t buckets,
                        const int32_t* max_len, int64_t* keys, void* stream);
int fvr_rplan_render(const int32_t* unit_len, const int64_t* unit_off, const uint32_t* entries_a,
                     const uint32_t* entries_b, const double* base, const double* t_fin,
                     const int32_t* unit_order, const int32_t* row_src, int32_t n_views, int32_t bbox_w,
                     int32_t bbox_h, const float* src, const float* kp_values, int32_t n_channels,
                     const double* background, float* residual, double* sq_partials, int64_t sq_stride,
                     fvr_loop_state_t* state, const fvr_loop_finalize_t* finalize, int32_t wide, void* stream);
int fvr_rplan_pack(const float* values, int32_t n_channels, fvr_grid_t grid, const int32_t* kp_index,
                   int64_t n_kp, float* kp_values, const fvr_loop_state_t* state, void* stream);

/* Back-project the residual of every listed flame ray (ray_list entries are
 * view << 24 | (row_in_bbox * bbox_w + col_in_bbox); the top byte is read
 * unsigned, so a view index never decodes negative). stochastic != 0 draws
 * G ~ clip(N(1, g_sigma), 0, 2) from a counter-based Philox stream keyed by
 * seed and (iteration, ray_id_base + ray, sample), so a view-sharded run
 * draws the same weights as a single-GPU run. */
int fvr_loop_adjust(const fvr_camera_t* cams, const int32_t* ray_list, int64_t n_rays,
                    int32_t u0, int32_t v0, int32_t bbox_w, int32_t bbox_h,
                    const float* residual, int32_t res_pitch, const uint8_t* inside_vox, fvr_grid_t grid,
                    double tau, double alpha_l, double alpha_d, int32_t stochastic,
                    double g_sigma, uint64_t seed, int64_t ray_id_base, int64_t* accum,
                    const fvr_loop_state_t* state, void* stream);

/* Sum (values - truth)^2 over the listed key points into per-block f64
 * partials (vol_rmse of the trace). Returns the block count via *n_blocks. */
int fvr_loop_volume_sq(const float* values, const float* truth, const int32_t* kp_index,
                       int64_t n_kp, double* partials, int32_t* n_blocks,
                       const fvr_loop_state_t* state, void* stream);

/* Per-iteration bookkeeping (1 block): per-view RMSE from sq_partials,
 * mean over views, trace append, convergence rule (reconstruct.py:311-323).
 * vol_partials may be NULL. */
int fvr_loop_finalize(const double* sq_partials, int32_t n_views, int32_t blocks_per_view,
                      int64_t pixels_per_view, const double* vol_partials,
                      int32_t n_vol_blocks, int64_t n_kp, double converge_eps,
                      double* trace_rmse, double* trace_vol, fvr_loop_state_t* state,
                      void* stream);

/* Clamped update over hull key points unless the state says done; keeps the
 * renderer's packed layout (may be NULL) in sync. */
int fvr_loop_update(float* values, int64_t* accum, const int32_t* kp_index, int64_t n_kp,
                    float* layout, int32_t layout_kind, int32_t layout_nch, fvr_grid_t grid,
                    const fvr_loop_state_t* state, void* stream);

/* ---- deterministic back-projection as a voxel-driven gather ------------
 * (reconstruct.py:152-227 with G = 1).  The operator A (delta = A . res) is
 * fixed for a reconstruction: build its CSR by hull key point once, then
 * apply it every iteration.  kp_map (lattice) maps a key point to its row
 * (hull key points) or -1; row_counts (n_kp) i32 zeroed by the caller;
 * cursor (n_kp) i64 = row offsets (exclusive scan of the counts); entries
 * (2*nnz) i32 = (residual index, f32 bits of W) pairs. */
int fvr_adjust_plan_count(const fvr_camera_t* cams, const int32_t* ray_list, int64_t n_rays,
                          int32_t u0, int32_t v0, int32_t bbox_w, int32_t bbox_h,
                          const uint8_t* inside_vox, fvr_grid_t grid, const int32_t* kp_map,
                          int32_t* row_counts, void* stream);
int fvr_adjust_plan_fill(const fvr_camera_t* cams, const int32_t* ray_list, int64_t n_rays,
                         int32_t u0, int32_t v0, int32_t bbox_w, int32_t bbox_h,
                         const uint8_t* inside_vox, fvr_grid_t grid, double tau, double alpha_l,
                         double alpha_d, const int32_t* kp_map, const int64_t* row_info, int64_t* cursor,
                         uint32_t* entries_a, uint32_t* entries_b, void* stream);
/* Stochastic mode (random G, reconstruct.py:193-201): the sample plan.
 * Count: per-row entry counts (8 per in-hull sample) and per-ray in-hull
 * sample slots.  Sample ids come in blocks of 4 slots, one block per (ray,
 * k >> 2) group holding in-hull samples; sample (ray, k) has id 4 * block +
 * (k & 3), so ray_samples[r] = 4 * (groups of ray r).  Fill (ray_sid0 =
 * exclusive scan of ray_samples): entries (sample id, W) unmerged -- 6-byte
 * (the deterministic plan's layout, sample id < 2^24) when entries_b is
 * given, int2 otherwise --
 * sample_meta[block] = (ray index, group << 4 | mask of used slots).
 * Per iteration fvr_loop_weighted_residual (n_samples = total slots) writes
 * rho[sid] = residual[ray] * G(seed, iteration, ray_id_base + ray, k) -- one
 * Philox block per 4-slot block, the stream of
 * fvr_loop_adjust -- and fvr_loop_gather runs over the sample plan with rho
 * in place of the residual.  state_advanced = 1 when the iteration's finalize
 * has already run (fused into fvr_rplan_render): the key is then it - 1. */
int fvr_sample_plan_count(const fvr_camera_t* cams, const int32_t* ray_list, int64_t n_rays,
                          int32_t u0, int32_t v0, int32_t bbox_w, int32_t bbox_h,
                          const uint8_t* inside_vox, fvr_grid_t grid, const int32_t* kp_map,
                          int32_t* row_counts, int32_t* ray_samples, void* stream);
int fvr_sample_plan_fill(const fvr_camera_t* cams, const int32_t* ray_list, int64_t n_rays,
                         int32_t u0, int32_t v0, int32_t bbox_w, int32_t bbox_h,
                         const uint8_t* inside_vox, fvr_grid_t grid, double tau, double alpha_l,
                         double alpha_d, const int32_t* kp_map, const int64_t* ray_sid0,
                         const int64_t* row_info, int64_t* cursor, int32_t* entries, uint32_t* entries_b,
                         int32_t* sample_meta, int64_t* block_keys, void* stream);
/* Spatial renumbering of the sample plan's blocks (block_keys from the fill,
 * sorted: new_of_nat[natural block] = rank), so the sample ids one SELL slice
 * of neighbouring key points reads sit close together (the gather's rho reads
 * hit cache lines): entries (n_slots stored entries, 6-byte layout when e6)
 * have their sample ids rewritten in place, meta_out[new] = meta_in[natural]. */
int fvr_sample_plan_reorder(int32_t* entries, int64_t n_slots, int32_t e6, const int32_t* new_of_nat,
                            int64_t n_blocks, const int32_t* meta_in, int32_t* meta_out, void* stream);
/* The same from the fill's block_keys directly (csrc/fvr_layout.cu): a
 * stable radix sort of their 30-bit Morton part gives new_of_nat, then
 * fvr_sample_plan_reorder. */
int fvr_sample_plan_spatial(int32_t* entries, int64_t n_slots, int32_t e6, const int64_t* block_keys,
                            int64_t n_blocks, const int32_t* meta_in, int32_t* meta_out, void* stream);
/* Sort every row of a 6-byte SELL plan (fvr_adjust_plan_fill /
 * fvr_sample_plan_fill layout) by column in place; rows of slices longer than
 * 1024 entries keep their order.  The gather's sums are order-independent
 * (32.32 fixed point), so only the memory access pattern changes. */
int fvr_plan_sort_rows(const int32_t* slice_len, const int64_t* slice_off, int64_t n_slices, int32_t* entries,
                       uint32_t* entries_b, void* stream);
/* Zero the padding of a filled 6-byte SELL plan: lane-row pos of slice s holds
 * cursor[row_of_pos[pos]] entries (the fill's final per-row cursors); positions
 * from there to slice_len[s] are cleared, so the entry buffers need no
 * clearing before the fill. */
int fvr_sell_pad_zero(const int64_t* cursor, const int32_t* row_of_pos, int64_t n_rows, const int32_t* slice_len,
                      const int64_t* slice_off, int64_t n_slices, int32_t* entries, uint32_t* entries_b,
                      void* stream);
/* The stochastic mode's G = clip(N(1, g_sigma), 0, 2) for (seed, iteration,
 * ray, march index k) -- the counter-based replacement of the reference's
 * rng.normal draw (reconstruct.py:191-204); the weigh pass and the ray-driven
 * scatter evaluate exactly these values.  ray, k, out: n device elements. */
int fvr_stochastic_g(uint64_t seed, uint32_t iteration, const uint32_t* ray, const uint32_t* k, int64_t n,
                     double g_sigma, float* out, void* stream);
int fvr_loop_weighted_residual(const int32_t* sample_meta, int64_t n_samples, const int32_t* ray_list,
                               int32_t bbox_w, int32_t bbox_h, const float* residual, int32_t n_channels,
                               uint64_t seed, double g_sigma, int64_t ray_id_base, float* rho,
                               const fvr_loop_state_t* state, int32_t state_advanced, void* stream);
/* Plans are SELL-32 (fvr_plan.cu): rows (hull key points) sorted by length,
 * row_pos[row] = sorted position, row_of_pos its inverse, slices of 32
 * positions with slice_len (longest row) and slice_off (exclusive scan, in
 * units of 32 entries); entry t of position p at slice_off[p/32]*32 + 32t +
 * p%32; cursor (n_rows i64, zeroed) counts the entries written per row.
 * The fills take row_info[row] = slice_off[p/32] << 5 | p%32 (p = row_pos[row])
 * (i64): the row's SELL position in one word.  fvr_adjust_plan_fill with
 * entries_b == NULL writes the wide format: int2 (residual index, f32 W) in
 * entries_a, chunks of 4 (slices padded to 4) -- for V * P >= 2^24, where
 * the residual index outgrows the 24-bit field; fvr_loop_gather reads it as
 * the int2 path (entries_b == NULL).
 * The deterministic plan (fvr_adjust_plan_fill) has 6-byte entries: a word
 * (u32, at that index) = residual index (< 2^24) | weight exponent << 24, and
 * the weight's top 16 mantissa bits in half t % 2 of entries_b[(slice_off +
 * t) / 2 * 32 + p % 32] (slice_off and slice_len even); fvr_loop_gather reads
 * them when entries_b is given, int2 (index, f32 weight) entries otherwise
 * (the stochastic sample plan).
 * Per iteration: row sums in 32.32 fixed point; with packed == NULL the
 * clamped update is applied in place (and the packed layout refreshed),
 * otherwise the sums go to packed (n_channels, n_kp) for the multi-GPU
 * all-reduce.  n_channels (1 or 3) share the plan: the residual (or rho)
 * holds a pixel's (sample's) channels interleaved with pitch 1 or 4, values /
 * layout hold n_channels lattice planes and state n_channels loop states
 * (converged channels are skipped).  kp_values (may be NULL): the render
 * plan's operand (fvr_rplan_pack), updated with every written value.
 * sample_plan = 1 when the plan is the stochastic sample plan (residual =
 * rho): it selects the loop schedule tuned for each (the merged plan's
 * gather is software-pipelined); results do not depend on it. */
int fvr_loop_gather(const int32_t* slice_len, const int64_t* slice_off, const int32_t* row_of_pos,
                    const int32_t* entries, const uint32_t* entries_b, int64_t n_kp, const float* residual, int32_t n_channels,
                    const int32_t* kp_index, float* values, float* layout, int32_t layout_kind,
                    fvr_grid_t grid, float* kp_values, int64_t* packed, const fvr_loop_state_t* state,
                    int32_t sample_plan, void* stream);
int fvr_loop_update_packed(const int64_t* packed, int64_t n_kp, const int32_t* kp_index,
                           float* values, float* layout, int32_t layout_kind, int32_t layout_nch,
                           fvr_grid_t grid, float* kp_values, int32_t kp_values_pitch,
                           const fvr_loop_state_t* state, void* stream);

/* Multi-GPU helpers: gather accum at kp_index into a compact buffer and
 * scatter it back (the NCCL allreduce runs between them). */
int fvr_pack_correction(const int64_t* accum, const int32_t* kp_index, int64_t n_kp,
                        int64_t* packed, void* stream);
int fvr_unpack_correction(const int64_t* packed, const int32_t* kp_index, int64_t n_kp,
                          int64_t* accum, void* stream);

/* ---- loop setup: host staging (once per reconstruct_channel) ------------- */

/* One multithreaded host pass over the caller's arrays into page-locked
 * staging (all outputs are host pointers; NULL skips a part): inside_out
 * (n_vox u8) = tags == full_mask (HullTags.inside_voxels, volume.py:142-145);
 * src_out (V, h, w) f32 and masks_out (V, h, w) u8 = the bbox crops
 * [v0:v0+h, u0:u0+w] of each view's image (row / column strides in
 * elements) and flame mask (row stride in bytes, bool bytes);
 * counts_out[v] = flame pixels of view v in the bbox (needs masks_out). */
int fvr_stage_inputs_host(const uint32_t* tags, int64_t n_vox, uint32_t full_mask, int32_t n_views,
                          const float* const* images, const int64_t* image_row_stride, int64_t image_col_stride,
                          const uint8_t* const* masks, const int64_t* mask_row_stride, int32_t u0, int32_t v0,
                          int32_t w, int32_t h, uint8_t* inside_out, float* src_out, uint8_t* masks_out,
                          int64_t* counts_out);

/* ---- loop setup: index preparation (once per reconstruct_channel) -------- */

/* Morton (x, y, z) key of each of the n lattice indices kp_index (C order):
 * the hull key points are numbered in this order (plan rows and columns). */
int fvr_morton_keys(const int32_t* kp_index, int64_t n, fvr_grid_t grid, int64_t* keys, void* stream);
/* SELL row order of the adjust plans: positions in windows of `window` (a
 * power of two <= 1024), rows longest first inside a window (ties in row
 * order); row_of_pos[pos] = row. */
int fvr_sell_window_order(const int32_t* counts, int64_t n, int32_t window, int32_t* row_of_pos, void* stream);
/* Render-plan row order: each tile of tile_units_x x tile_units_y units
 * (8x4-pixel warp units of one view) deals its rows, longest first, to its
 * slots in natural order: row_src[slot] = natural row; unit_len[unit] = the
 * unit's longest row rounded up to `align` entries.  row_len from
 * fvr_rplan_count. */
int fvr_rplan_tile_rows(const int32_t* row_len, int32_t n_views, int32_t bbox_w, int32_t bbox_h,
                        int32_t tile_units_x, int32_t tile_units_y, int32_t align, int32_t* row_src,
                        int32_t* unit_len, void* stream);

/* The setup's layout steps as one call each (csrc/fvr_layout.cu; CUB scans
 * and radix sorts on `stream`, scratch from the device's default pool). */
/* kp_index sorted by Morton key into out (n < 2^31; out != kp_index). */
int fvr_morton_order(const int32_t* kp_index, int64_t n, fvr_grid_t grid, int32_t* out, void* stream);
/* map[lattice index] = position in kp_index, -1 elsewhere (n_vox entries). */
int fvr_kp_map(const int32_t* kp_index, int64_t n_kp, int64_t n_vox, int32_t* map, void* stream);
/* The adjust plan's SELL layout after its count pass: row_of_pos
 * (fvr_sell_window_order), slice_len[s] = the slice's longest row rounded up
 * to `pad` entries, slice_off (n_slices + 1, exclusive scan of slice_len),
 * row_info[row] = slice_off[pos >> 5] << 5 | (pos & 31); totals[0] = entries
 * per lane over all slices, totals[1] = sum of counts, totals[2] = sum of
 * ray_samples (0 when ray_samples is NULL) and, when ray_sid0 is given, its
 * exclusive scan (n_rays int64: the sample plan's first sample id per ray).
 * n_slices = ceil(n_rows / 32). */
int fvr_sell_layout(const int32_t* counts, int64_t n_rows, int32_t window, int32_t pad,
                    const int32_t* ray_samples, int64_t n_rays, int64_t* ray_sid0, int32_t* row_of_pos,
                    int32_t* slice_len, int64_t* slice_off, int64_t* row_info, int64_t* totals, void* stream);
/* The render plan's layout after its count pass: fvr_rplan_tile_rows
 * (row_src, unit_len), unit_off (n_units + 1, exclusive scan of unit_len),
 * unit_order (the fvr_rplan_unit_keys order: longest class first, 2x4-unit
 * tiles inside a class); totals[0] = unit_off[n_units], totals[1] = the
 * longest unit. */
int fvr_rplan_layout(const int32_t* row_len, int32_t n_views, int32_t bbox_w, int32_t bbox_h, int32_t tile_units_x,
                     int32_t tile_units_y, int32_t align, int32_t buckets, int32_t* row_src, int32_t* unit_len,
                     int64_t* unit_off, int32_t* unit_order, int64_t* totals, void* stream);
/* Nonzero bytes of v (n of them): *count (device) = how many; the select
 * writes their indices in order (*n_sel = the number found) into out, which
 * must hold them all: capacity >= the count (fvr_count_nonzero_u8's) -- the
 * hull key-point list from fvr_hull_keypoints' mask. */
int fvr_count_nonzero_u8(const uint8_t* v, int64_t n, int64_t* count, void* stream);
int fvr_select_nonzero_u8(const uint8_t* v, int64_t n, int64_t capacity, int32_t* out, int64_t* n_sel,
                          void* stream);
/* Host-side concatenation of n buffers into dst (page-locked staging for one
 * H2D copy), all host threads (OpenMP). */
int fvr_copy_host_parallel(const void* const* srcs, const int64_t* nbytes, int32_t n, void* dst);
/* Flame rays of the bbox crops (u8, n_views x bbox_h x bbox_w, row-major):
 * rays[i] = view << 24 | (row * bbox_w + col) of the i-th nonzero pixel in
 * that order (reconstruct.py:144-149); capacity must be >= their number
 * (the host's flame count); *n_rays (device) = the number found. */
int fvr_flame_rays(const uint8_t* crops, int32_t n_views, int32_t bbox_w, int32_t bbox_h, int64_t capacity,
                   int32_t* rays, int64_t* n_rays, void* stream);

/* ---- the per-iteration collective ------------------
 * Replaces the per-view loop + fixed-order merge of adjust_pass
 * (reconstruct.py:181-226; the reference itself has no distribution,
 * SPEC.md:622): every rank back-projects its views into the packed i64
 * correction and one all-reduce(sum) over NVLink makes the ranks' lattices
 * identical (integer sums: exact, partition-independent).  The communicator
 * is an ncclComm_t owned by the caller, resolved from the libnccl.so.2 the
 * process already mapped (or FVR_NCCL_LIB); the 128-byte unique id travels
 * through the caller's rendezvous. */
#define FVR_COMM_ID_BYTES 128
#define FVR_DT_INT64 0
#define FVR_DT_FLOAT32 1
#define FVR_DT_FLOAT64 2
typedef void* fvr_comm_t;
int fvr_comm_available(void); /* 1 when NCCL could be resolved */
int fvr_comm_nccl_version(int32_t* version);
int fvr_comm_unique_id(uint8_t* id_out /* FVR_COMM_ID_BYTES */);
int fvr_comm_init(int32_t rank, int32_t world, const uint8_t* unique_id, int32_t device, fvr_comm_t* comm_out);
/* in place, asynchronous on `stream`; dtype FVR_DT_* */
int fvr_allreduce_sum(fvr_comm_t comm, void* buf, int64_t count, int32_t dtype, void* stream);
int fvr_comm_destroy(fvr_comm_t comm);

/* ---- temperature (stage 5) --------------------------------------------- */

/* Planck x CIE-1931 -> linear sRGB, clip, /max*255 (fp64).  temps (n) and
 * entries (n,3) are device outputs; temperatures t_min + step*i. */
int fvr_ctmap_build(double t_min, double step, int32_t n, int32_t append_t_max, double t_max,
                    double* temps, double* entries, void* stream);

/* green -> temperature through the map's green column (np.interp on the
 * clipped value); optional idx_out (bracket index j), clamp_counts[2]
 * (below, above).  kp_index NULL means every element of values (n). */
int fvr_temp_lookup(const float* values, const int32_t* kp_index, int64_t n,
                    const double* green, const double* temps, int32_t n_lut, float* temp_out,
                    int32_t* idx_out, int64_t* clamp_counts, void* stream);

/* T -> RGB through the map (rgb_grids_from_temperature, reconstruct.py:389-401):
 * at the n key points kp_index (NULL: every element), rgb_out plane c (plane
 * elements apart) = f32(np.interp(clip(T, temps[0], temps[n_lut-1]), temps,
 * entries[:, c])) in fp64 from the f32 temperature, entries (n_lut, 3) f64.
 * green == NULL: values holds the temperatures.  green != NULL: values holds
 * the green lattice, the temperature is looked up first (as fvr_temp_lookup,
 * written to temp_out, clamp counts in clamp_counts) -- the fused snapshot
 * path of reconstruct_temperature.  Other lattice points are not written. */
int fvr_temp_rgb(const float* values, const int32_t* kp_index, int64_t n, const double* green,
                 const double* temps, const double* entries, int32_t n_lut, float* temp_out, float* rgb_out,
                 int64_t plane, int64_t* clamp_counts, void* stream);

/* Same lookup on f64 inputs (temp_from_green on arrays). */
int fvr_temp_from_green(const double* g, int64_t n, const double* green, const double* temps,
                        int32_t n_lut, double* temp_out, uint8_t* clamped_out, void* stream);

/* ---- input preparation (preprocess.py:59-93, §8f rank 2) ---------------- */

/* images (n_views, height, width, channels) f32 device.  bits (n_views,
 * height, width) u8 = max over channels > threshold (compared in f32, as
 * numpy does); blanked (same shape as images, may be NULL) = where(bits,
 * images, 0); bbox4 (u0, v0, u1, v1) i32 device, initialised by the caller to
 * (INT_MAX, INT_MAX, -1, -1), receives the tight union box of the set pixels
 * (u1 < 0: no flame pixel). */
int fvr_threshold_mask(const float* images, int32_t n_views, int32_t width, int32_t height,
                       int32_t channels, double threshold, uint8_t* bits, float* blanked,
                       int32_t* bbox4, void* stream);
/* (height+1, width+1) i64 summed-area table of one view's mask (device). */
int fvr_mask_sat(const uint8_t* bits, int32_t width, int32_t height, int64_t* sat, void* stream);

/* ---- visual hull (volume.py:272-328) ----------------------------------- */

/* OR bit `view_bit` into tags (nx,ny,nz) u32 for every voxel whose projected
 * footprint in the camera overlaps a flame pixel.  translation is the
 * camera's t (x_cam = R x + t); sat is the (h+1,w+1) i64 summed-area table
 * of the view's mask (device). */
int fvr_visual_hull_view(const fvr_camera_t* camera, const double translation[3],
                         fvr_grid_t grid, const int64_t* sat, int32_t view_bit, uint32_t* tags,
                         void* stream);

/* Key points adjacent to >= 1 inside voxel (volume.py:139-165 key_point_mask,
 * core_erosion = 0): inside (nx, ny, nz) u8 -> kp_mask (nx+1, ny+1, nz+1) u8.
 * When values is non-NULL it also receives the loop's initial lattice
 * (0 at those key points, the outside-hull sentinel -1 elsewhere;
 * reconstruct.py _init_grid). */
int fvr_hull_keypoints(const uint8_t* inside, fvr_grid_t grid, uint8_t* kp_mask, float* values, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FVR_B200_H */
