// fvr_setup.cu -- index preparation of the loop setup (once per
// reconstruct_channel call), as single kernels instead of chains of generic
// tensor ops: the Morton keys of the hull key points, the SELL row order of
// the adjust plans (rows sorted by length within windows of neighbouring
// rows) and the render plan's row order (each 16x16-pixel tile's rows sorted
// by length and dealt to its units).  At config 2 the generic versions were
// ~60 small launches and three radix sorts, ~1.3 ms of the call.
#include "fvr_internal.cuh"

namespace fvr {

__device__ __forceinline__ uint64_t spread3(uint32_t v) {  // 21 bits -> every third bit
    uint64_t x = v & 0x1FFFFFu;
    x = (x | (x << 32)) & 0x1F00000000FFFFull;
    x = (x | (x << 16)) & 0x1F0000FF0000FFull;
    x = (x | (x << 8)) & 0x100F00F00F00F00Full;
    x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
    x = (x | (x << 2)) & 0x1249249249249249ull;
    return x;
}

// Morton (x, y, z) key of each lattice index (C order, z fastest).
__global__ void morton_keys_kernel(const int32_t* __restrict__ kp, int64_t n, int sy, int sx, int ny1,
                                   int64_t* __restrict__ keys) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = kp[i];
        const uint32_t x = (uint32_t)(k / sx), y = (uint32_t)((k / sy) % ny1), z = (uint32_t)(k % sy);
        keys[i] = (int64_t)((spread3(x) << 2) | (spread3(y) << 1) | spread3(z));
    }
}

// Bitonic sort of (key, value) pairs held in shared memory, n a power of two
// (= blockDim.x); ascending by key.
__device__ void block_bitonic(uint64_t* key, int n) {
    for (int size = 2; size <= n; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            __syncthreads();
            const int i = threadIdx.x, j = i ^ stride;
            if (j > i) {
                const bool up = (i & size) == 0;
                const uint64_t a = key[i], b = key[j];
                if ((a > b) == up) {
                    key[i] = b;
                    key[j] = a;
                }
            }
        }
    }
    __syncthreads();
}

// SELL row order: positions are cut into windows of `window` (a power of two
// <= 1024); inside a window rows go longest first, ties in row order.
// row_of_pos[pos] = row.
__global__ void window_sort_kernel(const int32_t* __restrict__ counts, int64_t n, int32_t* __restrict__ row_of_pos) {
    extern __shared__ uint64_t s_key[];
    const int64_t base = (int64_t)blockIdx.x * blockDim.x;
    const int64_t r = base + threadIdx.x;
    // key: (~count) in the high half (longest first), row in the low half;
    // rows past the end sort last
    s_key[threadIdx.x] = r < n ? ((uint64_t)(0xFFFFFFFFu - (uint32_t)counts[r]) << 32) | (uint32_t)(r - base)
                               : ~0ull;
    block_bitonic(s_key, blockDim.x);
    if (r < n) row_of_pos[r] = (int32_t)(base + (int64_t)(s_key[threadIdx.x] & 0xFFFFFFFFu));
}

// Render-plan rows: natural row r = unit * 32 + lane.  A tile is tx x ty
// units of one view (16x16 pixels for 2x4); its slots are its units' rows in
// natural order, and slot k receives the tile's k-th longest row (ties in
// natural order).  row_src[slot] = natural row; unit_len[unit] = the longest
// row dealt to the unit, rounded up to `align` entries.  One block (256 =
// 32 * tx * ty threads) per tile.
__global__ void tile_rows_kernel(const int32_t* __restrict__ row_len, int units_x, int units_y, int upv, int tx,
                                 int ty, int tiles_x, int tiles_y, int align, int32_t* __restrict__ row_src,
                                 int32_t* __restrict__ unit_len) {
    extern __shared__ uint64_t s_key[];
    const int tile = blockIdx.x;
    const int per_view = tiles_x * tiles_y;
    const int view = tile / per_view, t = tile % per_view;
    const int tile_x = t % tiles_x, tile_y = t / tiles_x;
    // slot s of the tile -> (unit, lane): units in ascending order (row-major
    // over the tile's unit grid, clipped at the bbox), 32 lanes each
    const int s = threadIdx.x;
    const int ui = s >> 5, lane = s & 31;
    // count the tile's valid units to find the ui-th
    const int cols = min(tx, units_x - tile_x * tx), rows = min(ty, units_y - tile_y * ty);
    const int n_units = cols * rows;
    int unit = -1;
    if (ui < n_units) unit = view * upv + (tile_y * ty + ui / cols) * units_x + tile_x * tx + ui % cols;
    const int64_t nat = unit >= 0 ? (int64_t)unit * 32 + lane : -1;
    const uint32_t len = unit >= 0 ? (uint32_t)row_len[nat] : 0u;
    // key: longest first, then natural order (slot index orders natural rows)
    s_key[s] = unit >= 0 ? ((uint64_t)(0xFFFFFFFFu - len) << 32) | (uint32_t)s : ~0ull;
    block_bitonic(s_key, blockDim.x);
    __shared__ int s_len[1024];
    if (unit >= 0) {
        const int src_slot = (int)(s_key[s] & 0xFFFFFFFFu);  // slot s gets the s-th longest row
        const int su = src_slot >> 5, sl = src_slot & 31;
        const int src_unit = view * upv + (tile_y * ty + su / cols) * units_x + tile_x * tx + su % cols;
        row_src[nat] = src_unit * 32 + sl;
        s_len[s] = (int)(0xFFFFFFFFu - (uint32_t)(s_key[s] >> 32));
    }
    __syncthreads();
    if (unit >= 0 && lane == 0) {
        int m = 0;
        for (int l = 0; l < 32; ++l) m = max(m, s_len[s + l]);
        unit_len[unit] = (m + align - 1) / align * align;
    }
}

}  // namespace fvr

using namespace fvr;

extern "C" int fvr_morton_keys(const int32_t* kp_index, int64_t n, fvr_grid_t grid, int64_t* keys, void* stream) {
    FVR_TRY_BEGIN
    if (int rc = check_grid(grid)) return rc;
    if (grid.nx >= (1 << 21) || grid.ny >= (1 << 21) || grid.nz >= (1 << 21))
        return set_error(FVR_ERR_INVALID, "Morton keys take at most 2^21 key points per axis");
    if (n == 0) return FVR_OK;
    int64_t b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    morton_keys_kernel<<<(unsigned)b, 256, 0, (cudaStream_t)stream>>>(kp_index, n, grid.nz + 1,
                                                                      (grid.ny + 1) * (grid.nz + 1), grid.ny + 1, keys);
    return check_launch("morton_keys");
    FVR_TRY_END
}

extern "C" int fvr_sell_window_order(const int32_t* counts, int64_t n, int32_t window, int32_t* row_of_pos,
                                     void* stream) {
    FVR_TRY_BEGIN
    if (window < 2 || window > 1024 || (window & (window - 1)))
        return set_error(FVR_ERR_INVALID, "window must be a power of two in 2..1024");
    if (n == 0) return FVR_OK;
    const int64_t blocks = (n + window - 1) / window;
    window_sort_kernel<<<(unsigned)blocks, window, window * sizeof(uint64_t), (cudaStream_t)stream>>>(counts, n,
                                                                                                  row_of_pos);
    return check_launch("sell_window_order");
    FVR_TRY_END
}

extern "C" int fvr_rplan_tile_rows(const int32_t* row_len, int32_t n_views, int32_t bbox_w, int32_t bbox_h,
                                   int32_t tile_units_x, int32_t tile_units_y, int32_t align, int32_t* row_src,
                                   int32_t* unit_len, void* stream) {
    FVR_TRY_BEGIN
    const int threads = 32 * tile_units_x * tile_units_y;
    if (tile_units_x < 1 || tile_units_y < 1 || threads > 1024 || (threads & (threads - 1)))
        return set_error(FVR_ERR_INVALID, "a tile holds 1..32 units, a power of two");
    if (align < 1) return set_error(FVR_ERR_INVALID, "align must be positive");
    constexpr int kUnitWidth = 8;  // K-render's warp unit: 8x4 pixels (fvr_render.cu kUnitW)
    const int units_x = (bbox_w + kUnitWidth - 1) / kUnitWidth, upv = fvr_loop_blocks_per_view(bbox_w, bbox_h);
    const int units_y = upv / units_x;
    const int tiles_x = (units_x + tile_units_x - 1) / tile_units_x;
    const int tiles_y = (units_y + tile_units_y - 1) / tile_units_y;
    const int64_t tiles = (int64_t)n_views * tiles_x * tiles_y;
    if (tiles == 0) return FVR_OK;
    tile_rows_kernel<<<(unsigned)tiles, threads, threads * sizeof(uint64_t), (cudaStream_t)stream>>>(
        row_len, units_x, units_y, upv, tile_units_x, tile_units_y, tiles_x, tiles_y, align, row_src, unit_len);
    return check_launch("rplan_tile_rows");
    FVR_TRY_END
}
