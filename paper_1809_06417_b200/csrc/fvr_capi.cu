// fvr_capi.cu -- error state, launch accounting and the synchronous *_host
// variants of the operator layer (drop-in targets for a ctypes/cffi shim of
// fvr._kernels).
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "fvr_internal.cuh"

namespace fvr {

namespace {
thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};
}  // namespace

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FVR_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

int check_launch(const char* what) {
    count_launch(1);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return set_error(FVR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return FVR_OK;
}

int fix_to_f64(const int64_t* accum, int64_t n, double* out, cudaStream_t st);
bool scatter_dirs_match(const double* host_dirs, int n);

// RAII device buffer for the host variants.
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t bytes) {
        if (bytes && cudaMalloc(&p, bytes) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

inline void h2d(void* dst, const void* src, size_t bytes) {
    if (bytes && cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
        throw std::runtime_error("cudaMemcpy H2D failed");
}
inline void d2h(void* dst, const void* src, size_t bytes) {
    if (bytes && cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
        throw std::runtime_error("cudaMemcpy D2H failed");
}
inline int sync_check(const char* what) {
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return set_error(FVR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return FVR_OK;
}

inline size_t lattice_size(const fvr_grid_t& g) {
    return (size_t)(g.nx + 1) * (g.ny + 1) * (g.nz + 1);
}

}  // namespace fvr

using namespace fvr;

extern "C" const char* fvr_last_error(void) { return g_last_error.c_str(); }
extern "C" int fvr_abi_version(void) { return FVR_ABI_VERSION; }
extern "C" int64_t fvr_launch_count(void) { return g_launches.load(); }

extern "C" int fvr_render_rays_host(const double origin[3], const double* dirs, int64_t n_rays,
                                    const float* values, int32_t n_channels, fvr_grid_t grid,
                                    fvr_render_params_t params, const double* background,
                                    const double* scat_dirs, double* out) {
    FVR_TRY_BEGIN
    if (int rc = check_grid(grid)) return rc;
    if (n_rays <= 0) return FVR_OK;
    const size_t lat = lattice_size(grid) * (size_t)n_channels;
    const int n_scat = params.n_scat > 0 ? params.n_scat : 0;
    DevBuf d_dirs(sizeof(double) * 3 * n_rays), d_vals(sizeof(float) * lat),
        d_scat(sizeof(double) * 3 * (n_scat ? n_scat : 1)), d_out(sizeof(double) * n_rays * n_channels),
        d_layout(sizeof(float) * 4 * lat), d_occ(lattice_size(grid));
    h2d(d_dirs.p, dirs, sizeof(double) * 3 * n_rays);
    h2d(d_vals.p, values, sizeof(float) * lat);
    if (n_scat && scat_dirs) h2d(d_scat.p, scat_dirs, sizeof(double) * 3 * n_scat);
    // the stencil path may only see the directions loaded by fvr_set_scatter_dirs
    const bool scat = params.scattering && params.sigma_s > 0.0;
    const bool same_dirs = !scat || scatter_dirs_match(scat_dirs, n_scat);
    int rc = fvr_render_rays(origin, d_dirs.as<double>(), n_rays, d_vals.as<float>(), n_channels, grid,
                             params, background, d_scat.as<double>(),
                             same_dirs ? d_layout.as<float>() : nullptr, same_dirs ? d_occ.as<uint8_t>() : nullptr,
                             d_out.as<double>(), nullptr);
    if (rc) return rc;
    if ((rc = sync_check("render_rays_host"))) return rc;
    d2h(out, d_out.p, sizeof(double) * n_rays * n_channels);
    return FVR_OK;
    FVR_TRY_END
}

extern "C" int fvr_count_hull_samples_host(const double origin[3], const double* dirs,
                                           int64_t n_rays, const uint8_t* inside_vox,
                                           fvr_grid_t grid, int64_t* counts) {
    FVR_TRY_BEGIN
    if (int rc = check_grid(grid)) return rc;
    if (n_rays <= 0) return FVR_OK;
    const size_t nvox = (size_t)grid.nx * grid.ny * grid.nz;
    DevBuf d_dirs(sizeof(double) * 3 * n_rays), d_in(nvox), d_cnt(sizeof(int64_t) * n_rays);
    h2d(d_dirs.p, dirs, sizeof(double) * 3 * n_rays);
    h2d(d_in.p, inside_vox, nvox);
    int rc = fvr_count_hull_samples(origin, d_dirs.as<double>(), n_rays, d_in.as<uint8_t>(), grid,
                                    d_cnt.as<int64_t>(), nullptr);
    if (rc) return rc;
    if ((rc = sync_check("count_hull_samples_host"))) return rc;
    d2h(counts, d_cnt.p, sizeof(int64_t) * n_rays);
    return FVR_OK;
    FVR_TRY_END
}

extern "C" int fvr_adjust_rays_host(const double origin[3], const double* dirs, int64_t n_rays,
                                    const double* residuals, const double* g_values,
                                    const int64_t* g_offsets, int32_t use_g,
                                    const uint8_t* inside_vox, fvr_grid_t grid, double tau,
                                    double alpha_l, double alpha_d, double* partials,
                                    int32_t n_chunks) {
    FVR_TRY_BEGIN
    if (int rc = check_grid(grid)) return rc;
    if (n_chunks < 1) return set_error(FVR_ERR_INVALID, "n_chunks must be >= 1");
    if (n_rays <= 0) return FVR_OK;
    const size_t nvox = (size_t)grid.nx * grid.ny * grid.nz;
    const size_t lat = lattice_size(grid);
    int64_t n_g = 0;
    if (use_g) {
        // g_values holds one entry per in-hull sample: the last offset plus
        // that ray's count bounds it; the caller passes the exact array, so
        // size it from the offsets' maximum conservatively via a count pass.
        std::vector<int64_t> counts(n_rays);
        int rc = fvr_count_hull_samples_host(origin, dirs, n_rays, inside_vox, grid, counts.data());
        if (rc) return rc;
        n_g = g_offsets[n_rays - 1] + counts[n_rays - 1];
        if (n_g < 1) n_g = 1;
    }
    DevBuf d_dirs(sizeof(double) * 3 * n_rays), d_res(sizeof(double) * n_rays), d_in(nvox),
        d_acc(sizeof(int64_t) * lat), d_f64(sizeof(double) * lat),
        d_gv(sizeof(double) * (n_g ? n_g : 1)), d_go(sizeof(int64_t) * (use_g ? n_rays : 1));
    h2d(d_dirs.p, dirs, sizeof(double) * 3 * n_rays);
    h2d(d_res.p, residuals, sizeof(double) * n_rays);
    h2d(d_in.p, inside_vox, nvox);
    if (use_g) {
        h2d(d_gv.p, g_values, sizeof(double) * n_g);
        h2d(d_go.p, g_offsets, sizeof(int64_t) * n_rays);
    }
    if (cudaMemset(d_acc.p, 0, sizeof(int64_t) * lat) != cudaSuccess) throw std::runtime_error("cudaMemset failed");
    int rc = fvr_adjust_rays(origin, d_dirs.as<double>(), n_rays, d_res.as<double>(), d_gv.as<double>(),
                             d_go.as<int64_t>(), use_g, d_in.as<uint8_t>(), grid, tau, alpha_l, alpha_d,
                             d_acc.as<int64_t>(), nullptr);
    if (rc) return rc;
    if ((rc = fix_to_f64(d_acc.as<int64_t>(), (int64_t)lat, d_f64.as<double>(), nullptr))) return rc;
    if ((rc = sync_check("adjust_rays_host"))) return rc;
    std::vector<double> tmp(lat);
    d2h(tmp.data(), d_f64.p, sizeof(double) * lat);
    for (size_t i = 0; i < lat; ++i) partials[i] += tmp[i];  // chunk 0
    return FVR_OK;
    FVR_TRY_END
}
