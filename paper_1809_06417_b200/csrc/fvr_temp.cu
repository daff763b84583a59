// fvr_temp.cu -- stage 5: the black-body colour/temperature map and the
// green -> temperature inversion at hull key points.
//
// K-ctmap (radiometry.py:173-203): Planck radiance at the 81 CIE-1931 nodes
// per tabulated temperature, trapezoid integration against x̄ȳz̄, linear sRGB
// via XYZ_TO_SRGB, negatives clipped, global scale so the table peak is
// exactly 255.  The reference evaluates this with numpy; the kernel follows
// numpy's arithmetic: lam**5 and expm1 are evaluated in double-double and
// rounded once (glibc's pow/expm1 are correctly rounded on these inputs in
// all cases we checked), np.trapezoid's add.reduce uses numpy's 8-accumulator
// pairwise order, and the (n,3)@(3,3) product uses OpenBLAS's FMA chain.
//
// K-temp (radiometry.py:206-219, reconstruct.py:444-455): np.interp on the
// clipped green with numpy's bracket rule (largest j with green[j] <= g,
// exact node hits and the right end return the node temperature).
#include "fvr_internal.cuh"

namespace fvr {

// CIE 1931 2-degree observer, 380..780 nm in 5 nm steps (81 nodes): x̄, ȳ, z̄.
__constant__ double kCieX[81] = {
    0.001368, 0.002236, 0.004243, 0.007650, 0.014310, 0.023190, 0.043510, 0.077630, 0.134380,
    0.214770, 0.283900, 0.328500, 0.348280, 0.348060, 0.336200, 0.318700, 0.290800, 0.251100,
    0.195360, 0.142100, 0.095640, 0.057950, 0.032010, 0.014700, 0.004900, 0.002400, 0.009300,
    0.029100, 0.063270, 0.109600, 0.165500, 0.225750, 0.290400, 0.359700, 0.433450, 0.512050,
    0.594500, 0.678400, 0.762100, 0.842500, 0.916300, 0.978600, 1.026300, 1.056700, 1.062200,
    1.045600, 1.002600, 0.938400, 0.854450, 0.751400, 0.642400, 0.541900, 0.447900, 0.360800,
    0.283500, 0.218700, 0.164900, 0.121200, 0.087400, 0.063600, 0.046770, 0.032900, 0.022700,
    0.015840, 0.011359, 0.008111, 0.005790, 0.004109, 0.002899, 0.002049, 0.001440, 0.001000,
    0.000690, 0.000476, 0.000332, 0.000235, 0.000166, 0.000117, 0.000083, 0.000059, 0.000042};
__constant__ double kCieY[81] = {
    0.000039, 0.000064, 0.000120, 0.000217, 0.000396, 0.000640, 0.001210, 0.002180, 0.004000,
    0.007300, 0.011600, 0.016840, 0.023000, 0.029800, 0.038000, 0.048000, 0.060000, 0.073900,
    0.090980, 0.112600, 0.139020, 0.169300, 0.208020, 0.258600, 0.323000, 0.407300, 0.503000,
    0.608200, 0.710000, 0.793200, 0.862000, 0.914850, 0.954000, 0.980300, 0.994950, 1.000000,
    0.995000, 0.978600, 0.952000, 0.915400, 0.870000, 0.816300, 0.757000, 0.694900, 0.631000,
    0.566800, 0.503000, 0.441200, 0.381000, 0.321000, 0.265000, 0.217000, 0.175000, 0.138200,
    0.107000, 0.081600, 0.061000, 0.044580, 0.032000, 0.023200, 0.017000, 0.011920, 0.008210,
    0.005723, 0.004102, 0.002929, 0.002091, 0.001484, 0.001047, 0.000740, 0.000520, 0.000361,
    0.000249, 0.000172, 0.000120, 0.000085, 0.000060, 0.000042, 0.000030, 0.000021, 0.000015};
__constant__ double kCieZ[81] = {
    0.006450, 0.010550, 0.020050, 0.036210, 0.067850, 0.110200, 0.207400, 0.371300, 0.645600,
    1.039050, 1.385600, 1.622960, 1.747060, 1.782600, 1.772110, 1.744100, 1.669200, 1.528100,
    1.287640, 1.041900, 0.812950, 0.616200, 0.465180, 0.353300, 0.272000, 0.212300, 0.158200,
    0.111700, 0.078250, 0.057250, 0.042160, 0.029840, 0.020300, 0.013400, 0.008750, 0.005750,
    0.003900, 0.002750, 0.002100, 0.001800, 0.001650, 0.001400, 0.001100, 0.001000, 0.000800,
    0.000600, 0.000340, 0.000240, 0.000190, 0.000100, 0.000050, 0.000030, 0.000020, 0.000010,
    0.000000, 0.000000, 0.000000, 0.000000, 0.000000, 0.000000, 0.000000, 0.000000, 0.000000,
    0.000000, 0.000000, 0.000000, 0.000000, 0.000000, 0.000000, 0.000000, 0.000000, 0.000000,
    0.000000, 0.000000, 0.000000, 0.000000, 0.000000, 0.000000, 0.000000, 0.000000, 0.000000};

// linear sRGB (D65) from CIE XYZ (radiometry.py:39-45), row-major.
__constant__ double kXyzToSrgb[9] = {3.2404542, -1.5371385, -0.4985314, -0.9692660, 1.8760108,
                                     0.0415560, 0.0556434,  -0.2040259, 1.0572252};

constexpr double kPlanckH = 6.62607015e-34;
constexpr double kLightC = 299792458.0;
constexpr double kBoltzmann = 1.380649e-23;

// ---- double-double helpers ---------------------------------------------
struct dd {
    double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return {s, e};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
    const double p = __dmul_rn(a, b);
    return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    dd t = two_sum(a.lo, b.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = quick_two_sum(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo = __fma_rn(a.hi, b.lo, p.lo);
    p.lo = __fma_rn(a.lo, b.hi, p.lo);
    return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
    dd p = two_prod(a.hi, b);
    p.lo = __fma_rn(a.lo, b, p.lo);
    return quick_two_sum(p.hi, p.lo);
}

__device__ __forceinline__ dd dd_div_d(dd a, double b) {
    const double q1 = __ddiv_rn(a.hi, b);
    const dd p = two_prod(q1, b);
    dd s = two_sum(a.hi, -p.hi);
    s.lo = __dadd_rn(__dsub_rn(s.lo, p.lo), a.lo);
    const double q2 = __ddiv_rn(__dadd_rn(s.hi, s.lo), b);
    return quick_two_sum(q1, q2);
}

// x**5 correctly rounded (numpy lam**5 -> libm pow).
__device__ double pow5_cr(double x) {
    const dd x2 = two_prod(x, x);
    const dd x4 = dd_mul(x2, x2);
    const dd x5 = dd_mul_d(x4, x);
    return __dadd_rn(x5.hi, x5.lo);
}

// expm1(x) correctly rounded for moderate positive x (the Planck exponent
// hc/(lam k T) lies in [~4.6, ~38] for 1000-2300 K over 380-780 nm).
__device__ double expm1_cr(double x) {
    const dd ln2 = {6.931471805599452862e-01, 2.319046813846299558e-17};
    const double k = rint(x / 0.6931471805599453);
    dd r = dd_add({x, 0.0}, dd_mul_d(ln2, -k));  // x - k ln2, |r| <= ~0.35
    // exp(r) = (exp(r/2^8))^(2^8), Taylor to degree 14 at |r/256| < 1.4e-3
    r.hi = ldexp(r.hi, -8);
    r.lo = ldexp(r.lo, -8);
    dd term = {1.0, 0.0}, sum = {1.0, 0.0};
    for (int i = 1; i <= 14; ++i) {
        term = dd_div_d(dd_mul(term, r), (double)i);
        sum = dd_add(sum, term);
    }
    for (int i = 0; i < 8; ++i) sum = dd_mul(sum, sum);
    sum.hi = ldexp(sum.hi, (int)k);
    sum.lo = ldexp(sum.lo, (int)k);
    const dd m1 = dd_add(sum, {-1.0, 0.0});
    return __dadd_rn(m1.hi, m1.lo);
}

// numpy pairwise_sum for 8 <= n <= 128 (8 accumulators, then a tree).
__device__ double np_pairwise(const double* a, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
        return r;
    }
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
}

// The table in three launches (it was one 1024-thread block, 3.4 ms):
// (1) one thread per (temperature, wavelength) node evaluates the Planck
// radiance once (the three channels share it); (2) one thread per
// temperature integrates the three channels (numpy's trapezoid terms and
// pairwise sum) and maps XYZ to clipped linear sRGB; (3) one block finds the
// peak and scales to 255.  Same operations per element as before, so the
// same bits.
__device__ __forceinline__ double ctmap_temperature(int row, double t_min, double step, int n, int append_max,
                                                    double t_max) {
    return (append_max && row == n - 1) ? t_max : __dadd_rn(t_min, __dmul_rn(step, (double)row));
}

__global__ void planck_nodes_kernel(double t_min, double step, int n, int append_max, double t_max,
                                    double* __restrict__ temps, double* __restrict__ radiance) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * 81) return;
    const int row = i / 81, j = i % 81;
    const double T = ctmap_temperature(row, t_min, step, n, append_max, t_max);
    if (j == 0) temps[row] = T;
    const double lam = __dmul_rn(380.0 + 5.0 * j, 1e-9);
    const double x = __ddiv_rn(kPlanckH * kLightC, __dmul_rn(__dmul_rn(lam, kBoltzmann), T));
    const double amp = __ddiv_rn(2.0 * kPlanckH * (kLightC * kLightC), pow5_cr(lam));
    radiance[i] = x > 700.0 ? __dmul_rn(amp, exp(-fmin(x, 1e6))) : __ddiv_rn(amp, expm1_cr(x));
}

__global__ void ctmap_rows_kernel(int n, const double* __restrict__ radiance, double* __restrict__ entries) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    const double* L = radiance + (int64_t)row * 81;
    double terms[80];
    double xyz[3];
    for (int c = 0; c < 3; ++c) {
        const double* cmf = c == 0 ? kCieX : (c == 1 ? kCieY : kCieZ);
        double y_prev = 0.0, lam_prev = 0.0;
        for (int j = 0; j < 81; ++j) {
            const double lam = __dmul_rn(380.0 + 5.0 * j, 1e-9);
            const double y = __dmul_rn(L[j], cmf[j]);
            if (j > 0) {
                const double dl = __dsub_rn(lam, lam_prev);
                terms[j - 1] = __ddiv_rn(__dmul_rn(dl, __dadd_rn(y, y_prev)), 2.0);
            }
            y_prev = y;
            lam_prev = lam;
        }
        xyz[c] = np_pairwise(terms, 80);
    }
    for (int j = 0; j < 3; ++j) {
        double t = __dmul_rn(xyz[0], kXyzToSrgb[3 * j]);
        t = __fma_rn(xyz[1], kXyzToSrgb[3 * j + 1], t);
        t = __fma_rn(xyz[2], kXyzToSrgb[3 * j + 2], t);
        entries[3 * row + j] = t > 0.0 ? t : 0.0;  // np.maximum(rgb, 0)
    }
}

// the peak (max is order independent), then entries / peak * 255
__global__ void __launch_bounds__(1024) ctmap_normalize_kernel(int n, double* __restrict__ entries) {
    __shared__ double red[32];
    double local_max = 0.0;
    for (int i = threadIdx.x; i < 3 * n; i += blockDim.x) local_max = fmax(local_max, entries[i]);
    for (int off = 16; off > 0; off >>= 1)
        local_max = fmax(local_max, __shfl_xor_sync(0xffffffffu, local_max, off));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = local_max;
    __syncthreads();
    if (threadIdx.x < 32) {
        double m = threadIdx.x < (blockDim.x + 31) / 32 ? red[threadIdx.x] : 0.0;
        for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
        if (threadIdx.x == 0) red[0] = m;
    }
    __syncthreads();
    const double peak = red[0];
    for (int i = threadIdx.x; i < 3 * n; i += blockDim.x) entries[i] = __dmul_rn(__ddiv_rn(entries[i], peak), 255.0);
}

// np.interp(clip(g, lo, hi), green, temps) -- see the file comment.
__device__ __forceinline__ double interp_green(double g, const double* __restrict__ green,
                                               const double* __restrict__ temps, int n,
                                               int& j_out) {
    const double lo = green[0], hi = green[n - 1];
    const double x = g < lo ? lo : (g > hi ? hi : g);
    // largest j with green[j] <= x
    int a = 0, b = n - 1;
    while (a < b) {
        const int m = (a + b + 1) >> 1;
        if (green[m] <= x) a = m;
        else b = m - 1;
    }
    const int j = a;
    j_out = j;
    if (j == n - 1 || green[j] == x) return temps[j];
    const double slope = __ddiv_rn(__dsub_rn(temps[j + 1], temps[j]), __dsub_rn(green[j + 1], green[j]));
    return __dadd_rn(__dmul_rn(slope, __dsub_rn(x, green[j])), temps[j]);
}

__global__ void temp_lookup_kernel(const float* __restrict__ values, const int32_t* __restrict__ kp,
                                   int64_t n, const double* __restrict__ green,
                                   const double* __restrict__ temps, int n_lut,
                                   float* __restrict__ out, int32_t* __restrict__ idx_out,
                                   unsigned long long* __restrict__ clamps) {
    unsigned long long lowc = 0, highc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t src = kp ? (int64_t)kp[i] : i;
        const double gval = (double)values[src];
        lowc += gval < green[0];
        highc += gval > green[n_lut - 1];
        int j;
        const double T = interp_green(gval, green, temps, n_lut, j);
        out[src] = (float)T;
        if (idx_out) idx_out[i] = j;
    }
    if (clamps) {
        for (int off = 16; off > 0; off >>= 1) {
            lowc += __shfl_xor_sync(0xffffffffu, lowc, off);
            highc += __shfl_xor_sync(0xffffffffu, highc, off);
        }
        if ((threadIdx.x & 31) == 0) {
            if (lowc) atomicAdd(clamps, lowc);
            if (highc) atomicAdd(clamps + 1, highc);
        }
    }
}

// np.interp(x, xp, fp) for x already inside [xp[0], xp[n-1]] and a known
// bracket j (largest j with xp[j] <= x): numpy's slope form, no contraction.
__device__ __forceinline__ double interp_at(double x, const double* __restrict__ xp, const double* __restrict__ fp,
                                            int fstride, int n, int j) {
    if (j == n - 1 || xp[j] == x) return fp[j * fstride];
    const double slope = __ddiv_rn(__dsub_rn(fp[(j + 1) * fstride], fp[j * fstride]), __dsub_rn(xp[j + 1], xp[j]));
    return __dadd_rn(__dmul_rn(slope, __dsub_rn(x, xp[j])), fp[j * fstride]);
}

__device__ __forceinline__ int bracket(const double* __restrict__ xp, int n, double x) {
    int a = 0, b = n - 1;
    while (a < b) {
        const int m = (a + b + 1) >> 1;
        if (xp[m] <= x) a = m;
        else b = m - 1;
    }
    return a;
}

// rgb_grids_from_temperature (reconstruct.py:389-401): at every hull key
// point, rgb_c = np.interp(clip(T, t_min, t_max), temps, entries[:, c]) in
// fp64 from the f32 temperature, stored f32 in plane c of rgb (the caller
// keeps the outside-hull sentinel elsewhere).  With `green` non-NULL the
// temperature itself is first derived from the green lattice (K-temp,
// radiometry.py:206-219) and written to temp_out: the fused snapshot path of
// reconstruct_temperature.
__global__ void temp_rgb_kernel(const float* __restrict__ values, const int32_t* __restrict__ kp, int64_t n,
                                const double* __restrict__ green, const double* __restrict__ temps,
                                const double* __restrict__ entries, int n_lut, float* __restrict__ temp_out,
                                float* __restrict__ rgb, int64_t plane, unsigned long long* __restrict__ clamps) {
    unsigned long long lowc = 0, highc = 0;
    const double t_lo = temps[0], t_hi = temps[n_lut - 1];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t src = kp ? (int64_t)kp[i] : i;
        float T;
        if (green) {
            const double gval = (double)values[src];
            lowc += gval < green[0];
            highc += gval > green[n_lut - 1];
            int j;
            T = (float)interp_green(gval, green, temps, n_lut, j);
            temp_out[src] = T;
        } else {
            T = values[src];
        }
        double x = (double)T;
        x = x < t_lo ? t_lo : (x > t_hi ? t_hi : x);
        const int j = bracket(temps, n_lut, x);
#pragma unroll
        for (int c = 0; c < 3; ++c) rgb[c * plane + src] = (float)interp_at(x, temps, entries + c, 3, n_lut, j);
    }
    if (clamps && green) {
        for (int off = 16; off > 0; off >>= 1) {
            lowc += __shfl_xor_sync(0xffffffffu, lowc, off);
            highc += __shfl_xor_sync(0xffffffffu, highc, off);
        }
        if ((threadIdx.x & 31) == 0) {
            if (lowc) atomicAdd(clamps, lowc);
            if (highc) atomicAdd(clamps + 1, highc);
        }
    }
}

__global__ void temp_from_green_kernel(const double* __restrict__ g, int64_t n,
                                       const double* __restrict__ green,
                                       const double* __restrict__ temps, int n_lut,
                                       double* __restrict__ out, uint8_t* __restrict__ clamped) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double x = g[i];
        int j;
        out[i] = interp_green(x, green, temps, n_lut, j);
        if (clamped) clamped[i] = (x < green[0]) || (x > green[n_lut - 1]);
    }
}

}  // namespace fvr

using namespace fvr;

extern "C" int fvr_ctmap_build(double t_min, double step, int32_t n, int32_t append_t_max,
                               double t_max, double* temps, double* entries, void* stream) {
    FVR_TRY_BEGIN
    if (n < 1) return set_error(FVR_ERR_INVALID, "empty temperature table");
    cudaStream_t st = (cudaStream_t)stream;
    const int rows = n + (append_t_max ? 1 : 0);
    double* radiance = nullptr;
    keep_default_pool();
    if (cudaMallocAsync(&radiance, sizeof(double) * (size_t)rows * 81, st) != cudaSuccess)
        return set_error(FVR_ERR_CUDA, "ctmap_build: cannot allocate the radiance scratch");
    planck_nodes_kernel<<<(rows * 81 + 127) / 128, 128, 0, st>>>(t_min, step, rows, append_t_max, t_max, temps,
                                                                 radiance);
    ctmap_rows_kernel<<<(rows + 63) / 64, 64, 0, st>>>(rows, radiance, entries);
    ctmap_normalize_kernel<<<1, 1024, 0, st>>>(rows, entries);
    count_launch(2);
    cudaFreeAsync(radiance, st);
    return check_launch("ctmap_build");
    FVR_TRY_END
}

extern "C" int fvr_temp_lookup(const float* values, const int32_t* kp_index, int64_t n,
                               const double* green, const double* temps, int32_t n_lut,
                               float* temp_out, int32_t* idx_out, int64_t* clamp_counts,
                               void* stream) {
    FVR_TRY_BEGIN
    if (n_lut < 2) return set_error(FVR_ERR_INVALID, "need at least two table rows");
    if (n == 0) return FVR_OK;
    int64_t b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    temp_lookup_kernel<<<(unsigned)b, 256, 0, (cudaStream_t)stream>>>(
        values, kp_index, n, green, temps, n_lut, temp_out, idx_out,
        reinterpret_cast<unsigned long long*>(clamp_counts));
    return check_launch("temp_lookup");
    FVR_TRY_END
}

extern "C" int fvr_temp_from_green(const double* g, int64_t n, const double* green,
                                   const double* temps, int32_t n_lut, double* temp_out,
                                   uint8_t* clamped_out, void* stream) {
    FVR_TRY_BEGIN
    if (n_lut < 2) return set_error(FVR_ERR_INVALID, "need at least two table rows");
    if (n == 0) return FVR_OK;
    int64_t b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    temp_from_green_kernel<<<(unsigned)b, 256, 0, (cudaStream_t)stream>>>(g, n, green, temps, n_lut,
                                                                          temp_out, clamped_out);
    return check_launch("temp_from_green");
    FVR_TRY_END
}

extern "C" int fvr_temp_rgb(const float* values, const int32_t* kp_index, int64_t n, const double* green,
                            const double* temps, const double* entries, int32_t n_lut, float* temp_out, float* rgb_out,
                            int64_t plane, int64_t* clamp_counts, void* stream) {
    FVR_TRY_BEGIN
    if (n_lut < 2) return set_error(FVR_ERR_INVALID, "need at least two table rows");
    if (!rgb_out || !temps || !entries) return set_error(FVR_ERR_INVALID, "temps / entries / rgb_out are NULL");
    if (green && !temp_out) return set_error(FVR_ERR_INVALID, "temp_out is NULL");
    if (n == 0) return FVR_OK;
    int64_t b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    temp_rgb_kernel<<<(unsigned)b, 256, 0, (cudaStream_t)stream>>>(
        values, kp_index, n, green, temps, entries, n_lut, temp_out, rgb_out, plane,
        reinterpret_cast<unsigned long long*>(clamp_counts));
    return check_launch("temp_rgb");
    FVR_TRY_END
}
