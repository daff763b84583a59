// fvr_layout.cu -- the loop setup's layout steps as single C calls: what
// lies between a plan's count pass and its fill (SELL layout, scans, unit
// order), the Morton order of the hull key points, the key-point map and the
// flame-ray list.  Each was a chain of 5-25 generic tensor ops whose host
// enqueue cost (~10-20 us per op) dominated the per-call setup once the
// kernels themselves had been made cheap; here each is a few launches plus
// CUB scans / radix sorts on the caller's stream, with stream-ordered
// scratch from the device's default memory pool.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include "fvr_internal.cuh"

namespace fvr {

namespace {

struct Scratch {
    cudaStream_t st;
    void* p[6] = {};
    int n = 0;
    explicit Scratch(cudaStream_t s) : st(s) { keep_default_pool(); }
    template <typename T>
    T* get(size_t count) {
        void* q = nullptr;
        if (cudaMallocAsync(&q, count * sizeof(T) + 16, st) != cudaSuccess) throw std::bad_alloc();
        p[n++] = q;
        return static_cast<T*>(q);
    }
    ~Scratch() {
        for (int i = 0; i < n; ++i) cudaFreeAsync(p[i], st);
    }
};

unsigned grid_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    if (b > 148 * 32) b = 148 * 32;
    return (unsigned)(b < 1 ? 1 : b);
}

int bits_for(uint64_t v) {  // bits needed to hold values 0..v
    int b = 0;
    while (b < 64 && (v >> b)) ++b;
    return b < 1 ? 1 : b;
}

}  // namespace

__device__ __forceinline__ uint64_t spread3_21(uint32_t v) {  // 21 bits -> every third bit
    uint64_t x = v & 0x1FFFFFu;
    x = (x | (x << 32)) & 0x1F00000000FFFFull;
    x = (x | (x << 16)) & 0x1F0000FF0000FFull;
    x = (x | (x << 8)) & 0x100F00F00F00F00Full;
    x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
    x = (x | (x << 2)) & 0x1249249249249249ull;
    return x;
}

__global__ void morton_pairs_kernel(const int32_t* __restrict__ kp, int64_t n, int sy, int sx, int ny1,
                                    uint64_t* __restrict__ keys) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = kp[i];
        const uint32_t x = (uint32_t)(k / sx), y = (uint32_t)((k / sy) % ny1), z = (uint32_t)(k % sy);
        keys[i] = (spread3_21(x) << 2) | (spread3_21(y) << 1) | spread3_21(z);
    }
}

__global__ void kp_map_kernel(const int32_t* __restrict__ kp, int64_t n, int32_t* __restrict__ map) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        map[kp[i]] = (int32_t)i;
}

// per SELL slice (one warp): its padded length into slice_len and, as int64,
// into off[s + 1] (scanned in place afterwards); the rows' count sum into
// totals[1]
__global__ void sell_slices_kernel(const int32_t* __restrict__ counts, const int32_t* __restrict__ row_of_pos,
                                   int64_t n, int64_t n_slices, int pad, int32_t* __restrict__ slice_len,
                                   int64_t* __restrict__ off, unsigned long long* __restrict__ totals) {
    const int lane = threadIdx.x & 31;
    unsigned long long sum = 0;
    for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < n_slices;
         s += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t p = s * 32 + lane;
        const int c = p < n ? counts[row_of_pos[p]] : 0;
        sum += (unsigned)c;
        int m = (int)__reduce_max_sync(0xffffffffu, (unsigned)c);
        m = (m + pad - 1) / pad * pad;
        if (lane == 0) {
            slice_len[s] = m;
            off[s + 1] = m;
        }
    }
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0 && sum) atomicAdd(totals + 1, sum);
}

// row_info[row] = slice_off[pos >> 5] << 5 | (pos & 31); totals[0] = the
// slices' entry total
__global__ void sell_row_info_kernel(const int32_t* __restrict__ row_of_pos, int64_t n, int64_t n_slices,
                                     const int64_t* __restrict__ off, int64_t* __restrict__ row_info,
                                     int64_t* __restrict__ totals) {
    const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i0 == 0) totals[0] = off[n_slices];
    for (int64_t p = i0; p < n; p += (int64_t)gridDim.x * blockDim.x)
        row_info[row_of_pos[p]] = (off[p >> 5] << 5) | (p & 31);
}

// sid0[r + 1] = ray_samples[r] (int64, scanned in place afterwards); sid0[0] = 0
__global__ void shift_to_i64_kernel(const int32_t* __restrict__ v, int64_t n, int64_t* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i + 1] = v[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = 0;
}

// the sample plan's block keys ((Morton code << 32) | block) split into a
// 32-bit key and the block index for a stable pair sort
__global__ void split_keys_kernel(const unsigned long long* __restrict__ keys, int64_t n, uint32_t* __restrict__ k,
                                  uint32_t* __restrict__ v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long x = keys[i];
        k[i] = (uint32_t)(x >> 32);
        v[i] = (uint32_t)x;
    }
}

__global__ void inverse_perm_kernel(const uint32_t* __restrict__ sorted_blk, int64_t n, int32_t* __restrict__ inv) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        inv[sorted_blk[i]] = (int32_t)i;
}

__global__ void count_u8_kernel(const uint8_t* __restrict__ v, int64_t n, unsigned long long* __restrict__ out) {
    unsigned long long s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s += v[i] != 0;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

__global__ void sum_kernel(const int32_t* __restrict__ v, int64_t n, unsigned long long* __restrict__ out) {
    unsigned long long s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s += (unsigned)v[i];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// unit lengths as int64 into off[u + 1] and their maximum into totals[1]
__global__ void unit_len_kernel(const int32_t* __restrict__ unit_len, int64_t n, int64_t* __restrict__ off,
                                unsigned long long* __restrict__ totals) {
    unsigned m = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned l = (unsigned)unit_len[i];
        off[i + 1] = l;
        m = max(m, l);
    }
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0 && m) atomicMax(totals + 1, (unsigned long long)m);
}

// The render plan's unit visiting order (engine._rplan_unit_order): longest
// first in `buckets` length classes, inside a class by 2x4-unit tiles.  The
// key packs (buckets - class) above the unit's tiled position (sb bits).
__global__ void unit_order_keys_kernel(const int32_t* __restrict__ unit_len, int n_units, int upv, int units_x,
                                       int buckets, int sb, const unsigned long long* __restrict__ totals,
                                       uint64_t* __restrict__ keys, int32_t* __restrict__ vals) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_units) return;
    const int mx = (int)totals[1];
    const int q = max(1, (mx + buckets - 1) / buckets);
    const int units_y = upv / units_x;
    const int txn = (units_x + 1) / 2, tyn = (units_y + 3) / 4;
    const int view = i / upv, u = i - view * upv;
    const int64_t tile = ((int64_t)view * tyn + (u / units_x) / 4) * txn + (u % units_x) / 2;
    const uint64_t spatial = (uint64_t)(tile * 8 + ((u / units_x) % 4) * 2 + (u % units_x) % 2);
    const uint64_t cls = (uint64_t)min(unit_len[i] / q, buckets);
    keys[i] = ((uint64_t)(buckets - cls) << sb) | spatial;
    vals[i] = i;
}

__global__ void flame_ray_kernel(int32_t* __restrict__ rays, const int64_t* __restrict__ n_sel, int64_t cap,
                                 int pix) {
    const int64_t n = min(*n_sel, cap);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t k = rays[i];
        rays[i] = ((k / pix) << 24) | (k % pix);
    }
}

// Rows of a 6-byte SELL plan sorted by column (the a-word's low 24 bits), one
// warp per row: the row is read out of its lane's 16-byte chunks into shared
// memory as (column << 32 | exponent << 16 | mantissa half), bitonic-sorted,
// and written back.  The gather's fixed-point sums do not depend on entry
// order, so this only changes which rho lines a warp's lanes touch together.
constexpr int kRowSortMax = 1024;
constexpr int kRowSortWarps = 4;
__global__ void __launch_bounds__(32 * kRowSortWarps)
plan_sort_rows_kernel(const int32_t* __restrict__ slice_len, const long long* __restrict__ slice_off,
                      int64_t n_slices, uint32_t* __restrict__ ea, uint16_t* __restrict__ eb) {
    __shared__ unsigned long long buf[kRowSortWarps][kRowSortMax];
    const int lane = threadIdx.x & 31;
    unsigned long long* s = buf[threadIdx.x >> 5];
    const int64_t stride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_slices * 32; r += stride) {
        const int64_t sl = r >> 5;
        const int ln = (int)(r & 31);
        const int len = slice_len[sl];
        if (len <= 1 || len > kRowSortMax) continue;
        const long long off = slice_off[sl];
        int n = 32;
        while (n < len) n <<= 1;
        for (int p = lane; p < n; p += 32) {
            unsigned long long v = ~0ull;
            if (p < len) {
                const uint32_t a = ea[(((off >> 2) + (p >> 2)) * 32 + ln) * 4 + (p & 3)];
                const uint16_t b = eb[(((off >> 3) + (p >> 3)) * 32 + ln) * 8 + (p & 7)];
                v = ((unsigned long long)(a & 0xFFFFFFu) << 32) | ((unsigned long long)(a >> 24) << 16) | b;
            }
            s[p] = v;
        }
        __syncwarp();
        for (int k = 2; k <= n; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = lane; i < n; i += 32) {
                    const int ixj = i ^ j;
                    if (ixj > i) {
                        const unsigned long long x = s[i], y = s[ixj];
                        if ((x > y) == ((i & k) == 0)) {
                            s[i] = y;
                            s[ixj] = x;
                        }
                    }
                }
                __syncwarp();
            }
        for (int p = lane; p < len; p += 32) {
            const unsigned long long v = s[p];
            ea[(((off >> 2) + (p >> 2)) * 32 + ln) * 4 + (p & 3)] =
                (uint32_t)(v >> 32) | ((uint32_t)((v >> 16) & 0xFFu) << 24);
            eb[(((off >> 3) + (p >> 3)) * 32 + ln) * 8 + (p & 7)] = (uint16_t)(v & 0xFFFFu);
        }
        __syncwarp();
    }
}

// The padding of a 6-byte SELL plan zeroed after its fill: lane-row `pos`
// holds cursor[row] entries (the fill's final cursors), positions up to the
// slice length are padding the gather reads with weight 0.
__global__ void sell_pad_zero_kernel(const long long* __restrict__ cursor, const int32_t* __restrict__ row_of_pos,
                                     int64_t n_rows, const int32_t* __restrict__ slice_len,
                                     const long long* __restrict__ slice_off, int64_t n_pos, uint32_t* __restrict__ ea,
                                     uint16_t* __restrict__ eb) {
    for (int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < n_pos;
         pos += (int64_t)gridDim.x * blockDim.x) {
        const int64_t sl = pos >> 5;
        const int ln = (int)(pos & 31);
        const int len = slice_len[sl];
        const long long off = slice_off[sl];
        const int c = pos < n_rows ? (int)cursor[row_of_pos[pos]] : 0;
        for (int p = c; p < len; ++p) {
            ea[(((off >> 2) + (p >> 2)) * 32 + ln) * 4 + (p & 3)] = 0u;
            eb[(((off >> 3) + (p >> 3)) * 32 + ln) * 8 + (p & 7)] = 0;
        }
    }
}

}  // namespace fvr

using namespace fvr;

extern "C" int fvr_sell_pad_zero(const int64_t* cursor, const int32_t* row_of_pos, int64_t n_rows,
                                 const int32_t* slice_len, const int64_t* slice_off, int64_t n_slices,
                                 int32_t* entries, uint32_t* entries_b, void* stream) {
    FVR_TRY_BEGIN
    if (n_slices <= 0) return FVR_OK;
    if (!entries_b) return set_error(FVR_ERR_INVALID, "pad zero: 6-byte plans only");
    const int64_t n_pos = n_slices * 32;
    int64_t blocks = (n_pos + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    sell_pad_zero_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const long long*>(cursor), row_of_pos, n_rows, slice_len,
        reinterpret_cast<const long long*>(slice_off), n_pos, reinterpret_cast<uint32_t*>(entries),
        reinterpret_cast<uint16_t*>(entries_b));
    return check_launch("sell_pad_zero");
    FVR_TRY_END
}

extern "C" int fvr_plan_sort_rows(const int32_t* slice_len, const int64_t* slice_off, int64_t n_slices,
                                  int32_t* entries, uint32_t* entries_b, void* stream) {
    FVR_TRY_BEGIN
    if (n_slices <= 0) return FVR_OK;
    if (!entries_b) return set_error(FVR_ERR_INVALID, "row sort: 6-byte plans only");
    const int64_t warps = n_slices * 32;
    int64_t blocks = (warps + kRowSortWarps - 1) / kRowSortWarps;
    if (blocks > 148 * 16) blocks = 148 * 16;
    plan_sort_rows_kernel<<<(unsigned)blocks, 32 * kRowSortWarps, 0, (cudaStream_t)stream>>>(
        slice_len, reinterpret_cast<const long long*>(slice_off), n_slices, reinterpret_cast<uint32_t*>(entries),
        reinterpret_cast<uint16_t*>(entries_b));
    return check_launch("plan_sort_rows");
    FVR_TRY_END
}

extern "C" int fvr_morton_order(const int32_t* kp_index, int64_t n, fvr_grid_t grid, int32_t* out, void* stream) {
    FVR_TRY_BEGIN
    if (int rc = check_grid(grid)) return rc;
    if (grid.nx >= (1 << 21) || grid.ny >= (1 << 21) || grid.nz >= (1 << 21))
        return set_error(FVR_ERR_INVALID, "Morton keys take at most 2^21 key points per axis");
    if (n <= 0) return FVR_OK;
    if (n >= (1ll << 31)) return set_error(FVR_ERR_INVALID, "at most 2^31 - 1 key points");
    cudaStream_t st = (cudaStream_t)stream;
    Scratch sc(st);
    uint64_t* keys = sc.get<uint64_t>(n);
    uint64_t* keys2 = sc.get<uint64_t>(n);
    morton_pairs_kernel<<<grid_for(n, 256), 256, 0, st>>>(kp_index, n, grid.nz + 1, (grid.ny + 1) * (grid.nz + 1),
                                                          grid.ny + 1, keys);
    const int axis_bits = bits_for((uint64_t)std::max(grid.nx, std::max(grid.ny, grid.nz)));
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, keys2, kp_index, out, (int)n, 0, 3 * axis_bits, st);
    void* t = sc.get<uint8_t>(tmp);
    cub::DeviceRadixSort::SortPairs(t, tmp, keys, keys2, kp_index, out, (int)n, 0, 3 * axis_bits, st);
    return check_launch("morton_order");
    FVR_TRY_END
}

extern "C" int fvr_kp_map(const int32_t* kp_index, int64_t n_kp, int64_t n_vox, int32_t* map, void* stream) {
    FVR_TRY_BEGIN
    if (n_vox <= 0) return FVR_OK;
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(map, 0xFF, sizeof(int32_t) * (size_t)n_vox, st);
    if (n_kp > 0) kp_map_kernel<<<grid_for(n_kp, 256), 256, 0, st>>>(kp_index, n_kp, map);
    return check_launch("kp_map");
    FVR_TRY_END
}

extern "C" int fvr_sell_layout(const int32_t* counts, int64_t n_rows, int32_t window, int32_t pad,
                               const int32_t* ray_samples, int64_t n_rays, int64_t* ray_sid0, int32_t* row_of_pos,
                               int32_t* slice_len, int64_t* slice_off, int64_t* row_info, int64_t* totals,
                               void* stream) {
    FVR_TRY_BEGIN
    if (pad < 1) return set_error(FVR_ERR_INVALID, "pad must be positive");
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(totals, 0, 3 * sizeof(int64_t), st);
    cudaMemsetAsync(slice_off, 0, sizeof(int64_t), st);
    auto* tot = reinterpret_cast<unsigned long long*>(totals);
    if (ray_samples && n_rays > 0) {
        sum_kernel<<<grid_for(n_rays, 256), 256, 0, st>>>(ray_samples, n_rays, tot + 2);
        if (ray_sid0) {  // exclusive scan of the rays' sample slots
            shift_to_i64_kernel<<<grid_for(n_rays - 1, 256), 256, 0, st>>>(ray_samples, n_rays - 1, ray_sid0);
            if (n_rays > 1) {
                Scratch sc(st);
                size_t tmp = 0;
                cub::DeviceScan::InclusiveSum(nullptr, tmp, ray_sid0 + 1, ray_sid0 + 1, (int)(n_rays - 1), st);
                void* t = sc.get<uint8_t>(tmp);
                cub::DeviceScan::InclusiveSum(t, tmp, ray_sid0 + 1, ray_sid0 + 1, (int)(n_rays - 1), st);
            }
        }
    }
    if (n_rows <= 0) return check_launch("sell_layout");
    if (int rc = fvr_sell_window_order(counts, n_rows, window, row_of_pos, stream)) return rc;
    const int64_t n_slices = (n_rows + 31) / 32;
    sell_slices_kernel<<<grid_for(n_slices * 32, 256), 256, 0, st>>>(counts, row_of_pos, n_rows, n_slices, pad,
                                                                      slice_len, slice_off, tot);
    Scratch sc(st);
    size_t tmp = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp, slice_off + 1, slice_off + 1, (int)n_slices, st);
    void* t = sc.get<uint8_t>(tmp);
    cub::DeviceScan::InclusiveSum(t, tmp, slice_off + 1, slice_off + 1, (int)n_slices, st);
    sell_row_info_kernel<<<grid_for(n_rows, 256), 256, 0, st>>>(row_of_pos, n_rows, n_slices, slice_off, row_info,
                                                                 totals);
    return check_launch("sell_layout");
    FVR_TRY_END
}

extern "C" int fvr_rplan_layout(const int32_t* row_len, int32_t n_views, int32_t bbox_w, int32_t bbox_h,
                                int32_t tile_units_x, int32_t tile_units_y, int32_t align, int32_t buckets,
                                int32_t* row_src, int32_t* unit_len, int64_t* unit_off, int32_t* unit_order,
                                int64_t* totals, void* stream) {
    FVR_TRY_BEGIN
    if (buckets < 1 || buckets > (1 << 20)) return set_error(FVR_ERR_INVALID, "buckets must be in 1..2^20");
    cudaStream_t st = (cudaStream_t)stream;
    constexpr int kUnitWidth = 8;
    const int units_x = (bbox_w + kUnitWidth - 1) / kUnitWidth, upv = fvr_loop_blocks_per_view(bbox_w, bbox_h);
    const int64_t n_units = (int64_t)upv * n_views;
    cudaMemsetAsync(totals, 0, 2 * sizeof(int64_t), st);
    cudaMemsetAsync(unit_off, 0, sizeof(int64_t), st);
    if (n_units <= 0) return check_launch("rplan_layout");
    if (int rc = fvr_rplan_tile_rows(row_len, n_views, bbox_w, bbox_h, tile_units_x, tile_units_y, align, row_src,
                                     unit_len, stream))
        return rc;
    auto* tot = reinterpret_cast<unsigned long long*>(totals);
    unit_len_kernel<<<grid_for(n_units, 256), 256, 0, st>>>(unit_len, n_units, unit_off, tot);
    Scratch sc(st);
    size_t tmp_scan = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp_scan, unit_off + 1, unit_off + 1, (int)n_units, st);
    // the unit order: radix sort of (class, tiled position) keys
    const int units_y = upv / units_x;
    const int64_t tiles = (int64_t)n_views * ((units_y + 3) / 4) * ((units_x + 1) / 2);
    const int sb = bits_for((uint64_t)(tiles * 8));
    const int end_bit = sb + bits_for((uint64_t)buckets);
    uint64_t* keys = sc.get<uint64_t>(n_units);
    uint64_t* keys2 = sc.get<uint64_t>(n_units);
    int32_t* vals = sc.get<int32_t>(n_units);
    size_t tmp_sort = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, keys, keys2, vals, unit_order, (int)n_units, 0, end_bit, st);
    void* t = sc.get<uint8_t>(std::max(tmp_scan, tmp_sort));
    cub::DeviceScan::InclusiveSum(t, tmp_scan, unit_off + 1, unit_off + 1, (int)n_units, st);
    cudaMemcpyAsync(totals, unit_off + n_units, sizeof(int64_t), cudaMemcpyDeviceToDevice, st);
    unit_order_keys_kernel<<<(unsigned)((n_units + 255) / 256), 256, 0, st>>>(unit_len, (int)n_units, upv, units_x,
                                                                             buckets, sb, tot, keys, vals);
    cub::DeviceRadixSort::SortPairs(t, tmp_sort, keys, keys2, vals, unit_order, (int)n_units, 0, end_bit, st);
    return check_launch("rplan_layout");
    FVR_TRY_END
}

extern "C" int fvr_count_nonzero_u8(const uint8_t* v, int64_t n, int64_t* count, void* stream) {
    FVR_TRY_BEGIN
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(count, 0, sizeof(int64_t), st);
    if (n > 0) count_u8_kernel<<<grid_for(n, 256), 256, 0, st>>>(v, n, reinterpret_cast<unsigned long long*>(count));
    return check_launch("count_nonzero_u8");
    FVR_TRY_END
}

extern "C" int fvr_select_nonzero_u8(const uint8_t* v, int64_t n, int64_t capacity, int32_t* out, int64_t* n_sel,
                                     void* stream) {
    FVR_TRY_BEGIN
    if (n >= (1ll << 31)) return set_error(FVR_ERR_INVALID, "at most 2^31 - 1 elements");
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(n_sel, 0, sizeof(int64_t), st);
    if (n <= 0 || capacity <= 0) return check_launch("select_nonzero_u8");
    Scratch sc(st);
    cub::CountingInputIterator<int32_t> idx(0);
    size_t tmp = 0;
    cub::DeviceSelect::Flagged(nullptr, tmp, idx, v, out, n_sel, (int)n, st);
    void* t = sc.get<uint8_t>(tmp);
    cub::DeviceSelect::Flagged(t, tmp, idx, v, out, n_sel, (int)n, st);
    return check_launch("select_nonzero_u8");
    FVR_TRY_END
}

extern "C" int fvr_sample_plan_spatial(int32_t* entries, int64_t n_slots, int32_t e6, const int64_t* block_keys,
                                       int64_t n_blocks, const int32_t* meta_in, int32_t* meta_out, void* stream) {
    FVR_TRY_BEGIN
    if (n_blocks <= 0) return FVR_OK;
    if (n_blocks >= (1ll << 31)) return set_error(FVR_ERR_INVALID, "at most 2^31 - 1 sample blocks");
    cudaStream_t st = (cudaStream_t)stream;
    Scratch sc(st);
    uint32_t* k = sc.get<uint32_t>(n_blocks);
    uint32_t* k2 = sc.get<uint32_t>(n_blocks);
    uint32_t* v = sc.get<uint32_t>(n_blocks);
    uint32_t* v2 = sc.get<uint32_t>(n_blocks);
    int32_t* inv = sc.get<int32_t>(n_blocks);
    split_keys_kernel<<<grid_for(n_blocks, 256), 256, 0, st>>>(
        reinterpret_cast<const unsigned long long*>(block_keys), n_blocks, k, v);
    // the Morton part holds 30 bits; the radix sort is stable, so ties keep
    // block order (= sorting the full (Morton << 32 | block) keys)
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, k, k2, v, v2, (int)n_blocks, 0, 30, st);
    void* t = sc.get<uint8_t>(tmp);
    cub::DeviceRadixSort::SortPairs(t, tmp, k, k2, v, v2, (int)n_blocks, 0, 30, st);
    inverse_perm_kernel<<<grid_for(n_blocks, 256), 256, 0, st>>>(v2, n_blocks, inv);
    if (int rc = fvr_sample_plan_reorder(entries, n_slots, e6, inv, n_blocks, meta_in, meta_out, stream)) return rc;
    return check_launch("sample_plan_spatial");
    FVR_TRY_END
}

extern "C" int fvr_flame_rays(const uint8_t* crops, int32_t n_views, int32_t bbox_w, int32_t bbox_h,
                              int64_t capacity, int32_t* rays, int64_t* n_rays, void* stream) {
    FVR_TRY_BEGIN
    const int64_t pix = (int64_t)bbox_w * bbox_h, n = pix * n_views;
    if (n_views < 0 || bbox_w < 1 || bbox_h < 1) return set_error(FVR_ERR_INVALID, "bad crop sizes");
    if (n_views > 127 || pix >= (1 << 24))
        return set_error(FVR_ERR_INVALID, "flame rays pack view << 24 | pixel: at most 127 views of < 2^24 pixels");
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(n_rays, 0, sizeof(int64_t), st);
    if (n == 0 || capacity <= 0) return check_launch("flame_rays");
    Scratch sc(st);
    // (the selection writes exactly the flagged count, which the caller's
    // capacity covers: no full-size scratch)
    cub::CountingInputIterator<int32_t> idx(0);
    size_t tmp = 0;
    cub::DeviceSelect::Flagged(nullptr, tmp, idx, crops, rays, n_rays, (int)n, st);
    void* t = sc.get<uint8_t>(tmp);
    cub::DeviceSelect::Flagged(t, tmp, idx, crops, rays, n_rays, (int)n, st);
    flame_ray_kernel<<<grid_for(capacity, 256), 256, 0, st>>>(rays, n_rays, capacity, (int)pix);
    return check_launch("flame_rays");
    FVR_TRY_END
}
