// Radar products on the GPU: range profiles and
// small-angle ISAR images from the estimator's frequency x azimuth sweeps.
//
// Restates proj/src/signal_processing.cpp:
//   uniform_step           :11-19    (host validation, same messages)
//   window_coefficients    :21-28    (Hann 0.5 - 0.5 cos(2 pi k / (n-1)))
//   padded_idft            :31-46    out[m] = (1/M) sum_k in[k] e^{+-j 2 pi k m / M}
//   center_shift           :49-53    rotate by M - M/2
//   range_profile          :66-89
//   isar                   :91-162   down-range IDFT per angle, conjugate
//                                    cross-range IDFT per range bin, dB with floor
// The reference evaluates e^{j 2 pi k m / M} by a running product (z *= w);
// here each term's phase is reduced exactly in integers ((k m) mod M) and
// evaluated with sincospi, so the two agree to ~1e-13 relative.
//
// One thread per output bin: the IDFTs are O(rows x M x N) with N, M <= a few
// thousand, trivially parallel and L1-resident (the input row is shared by
// all threads of a block).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "mcsbr_gpu.h"

namespace {

constexpr double kC = 299792458.0;
constexpr double kPi = 3.14159265358979323846;

thread_local std::string g_sig_err;

int sig_err(const std::string& m) {
    g_sig_err = m;
    return MCSBR_EINVAL;
}

// in: rows x n complex (row stride n), out: rows x m complex, centre-shifted:
// out[(j + (m - m/2)) % m ... ] -- we write bin `j` of the rotated axis, i.e.
// the unshifted index (j + m - m/2) % m ... computed directly.
__global__ void idft_rows(const double2* __restrict__ in, uint32_t rows, uint32_t n, uint32_t m,
                          bool conjugate, double2* __restrict__ out) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;  // output bin (after the shift)
    if (j >= m) return;
    // center_shift rotates left by (m - m/2): shifted[j] = raw[(j + m - m/2) % m]
    const uint32_t mm = (j + (m - m / 2)) % m;
    for (uint32_t row = blockIdx.y; row < rows; row += gridDim.y) {  // rows beyond the 65535 grid limit
        const double2* x = in + static_cast<size_t>(row) * n;
        double re = 0.0, im = 0.0;
        for (uint32_t k = 0; k < n; ++k) {
            const double2 v = x[k];
            if (v.x == 0.0 && v.y == 0.0) continue;
            const uint64_t km = (static_cast<uint64_t>(k) * mm) % m;
            double s, c;
            sincospi(2.0 * static_cast<double>(km) / static_cast<double>(m), &s, &c);
            if (conjugate) s = -s;
            re += v.x * c - v.y * s;
            im += v.x * s + v.y * c;
        }
        const double scale = 1.0 / static_cast<double>(m);
        out[static_cast<size_t>(row) * m + j] = make_double2(re * scale, im * scale);
    }
}

// transpose a (rows x cols) complex matrix
__global__ void transpose_c(const double2* __restrict__ in, uint32_t rows, uint32_t cols,
                            double2* __restrict__ out) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    for (uint32_t r = blockIdx.y; r < rows; r += gridDim.y)
        out[static_cast<size_t>(c) * rows + r] = in[static_cast<size_t>(r) * cols + c];
}

__global__ void magnitude(const double2* __restrict__ in, size_t n, double* __restrict__ mag) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    mag[i] = hypot(in[i].x, in[i].y);
}

// uniform_step (signal_processing.cpp:11-19)
int uniform_step(const double* g, uint32_t n, const char* what, double* step) {
    if (n < 2) return sig_err(std::string(what) + ": need at least 2 samples");
    const double s = g[1] - g[0];
    for (uint32_t i = 1; i < n; ++i)
        if (std::abs(g[i] - g[i - 1] - s) > 1e-6 * std::abs(s))
            return sig_err(std::string(what) + ": grid is not uniform");
    *step = s;
    return MCSBR_OK;
}

std::vector<double> window_coefficients(int window, uint32_t n) {
    std::vector<double> w(n, 1.0);
    if (window == MCSBR_WINDOW_HANN && n > 1)
        for (uint32_t k = 0; k < n; ++k) w[k] = 0.5 - 0.5 * std::cos(2.0 * kPi * k / (n - 1));
    return w;
}

double to_db(double mag) { return 20.0 * std::log10(std::max(mag, 1e-300)); }

std::vector<double> centered_axis(size_t m, double bin) {
    std::vector<double> a(m);
    for (size_t i = 0; i < m; ++i) a[i] = (static_cast<double>(i) - static_cast<double>(m / 2)) * bin;
    return a;
}

struct Dev {
    std::vector<void*> ptrs;
    ~Dev() {
        for (void* p : ptrs) cudaFree(p);
    }
    template <class T>
    T* alloc(size_t n) {
        void* p = nullptr;
        if (cudaMalloc(&p, sizeof(T) * (n ? n : 1)) != cudaSuccess) return nullptr;
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
};

int cuda_fail(const char* what) {
    g_sig_err = std::string(what) + ": " + cudaGetErrorString(cudaGetLastError());
    return MCSBR_ECUDA;
}

}  // namespace

// declared in mcsbr_gpu.h; the error text is shared with mcsbr_gpu_last_error
// through capi.cu's setter
extern "C" void mcsbr_gpu_internal_set_error(const char* msg);

static int finish(int rc) {
    if (rc != MCSBR_OK) mcsbr_gpu_internal_set_error(g_sig_err.c_str());
    return rc;
}

extern "C" {

int mcsbr_gpu_range_profile(const double* values, const double* freqs, uint32_t nf, int window,
                            int zero_pad, double* range_m, double* mag_db, double* bin_spacing) {
    if (zero_pad < 1) return finish(sig_err("range_profile: zero_pad must be >= 1"));
    if (!values || !freqs || !range_m || !mag_db) return finish(sig_err("range_profile: null argument"));
    double df = 0.0;
    int rc = uniform_step(freqs, nf, "range_profile", &df);
    if (rc) return finish(rc);
    const uint32_t m = nf * static_cast<uint32_t>(zero_pad);
    const std::vector<double> w = window_coefficients(window, nf);
    std::vector<double> data(2ull * nf);
    for (uint32_t k = 0; k < nf; ++k) {  // sweep.values[channel][k] * w[k]
        data[2 * k] = values[2 * k] * w[k];
        data[2 * k + 1] = values[2 * k + 1] * w[k];
    }
    Dev d;
    double2* din = d.alloc<double2>(nf);
    double2* dout = d.alloc<double2>(m);
    double* dmag = d.alloc<double>(m);
    if (!din || !dout || !dmag) return finish(cuda_fail("range_profile alloc"));
    if (cudaMemcpy(din, data.data(), sizeof(double2) * nf, cudaMemcpyHostToDevice) != cudaSuccess)
        return finish(cuda_fail("range_profile upload"));
    idft_rows<<<dim3((m + 127) / 128, 1), 128>>>(din, 1, nf, m, false, dout);
    magnitude<<<(m + 255) / 256, 256>>>(dout, m, dmag);
    if (cudaGetLastError() != cudaSuccess) return finish(cuda_fail("range_profile launch"));
    std::vector<double> mag(m);
    if (cudaMemcpy(mag.data(), dmag, sizeof(double) * m, cudaMemcpyDeviceToHost) != cudaSuccess)
        return finish(cuda_fail("range_profile"));
    const double bin = kC / (2.0 * df * static_cast<double>(m));
    const std::vector<double> axis = centered_axis(m, bin);
    for (uint32_t i = 0; i < m; ++i) {
        range_m[i] = axis[i];
        mag_db[i] = to_db(mag[i]);
    }
    if (bin_spacing) *bin_spacing = bin;
    return MCSBR_OK;
}

int mcsbr_gpu_isar(const double* values, const double* freqs, uint32_t nf, const double* angles_deg,
                   uint32_t na, int window, int zero_pad, double floor_db, double* down_range_m,
                   double* cross_range_m, double* mag_db, double* peak_db) {
    if (zero_pad < 1) return finish(sig_err("isar: zero_pad must be >= 1"));
    if (na == 0 || !values || !angles_deg) return finish(sig_err("isar: one sweep per angle required"));
    double dtheta_deg = 0.0, df = 0.0;
    int rc = uniform_step(angles_deg, na, "isar angles", &dtheta_deg);
    if (rc) return finish(rc);
    if (std::abs(angles_deg[na - 1] - angles_deg[0]) > 30.0)
        return finish(sig_err("isar: aperture exceeds the small-angle limit (30 degrees)"));
    rc = uniform_step(freqs, nf, "isar frequencies", &df);
    if (rc) return finish(rc);
    const uint32_t mr = nf * static_cast<uint32_t>(zero_pad);
    const uint32_t mc = na * static_cast<uint32_t>(zero_pad);
    const std::vector<double> wf = window_coefficients(window, nf);
    const std::vector<double> wa = window_coefficients(window, na);
    std::vector<double> data(2ull * na * nf);
    for (uint32_t a = 0; a < na; ++a)
        for (uint32_t k = 0; k < nf; ++k) {  // values * wf[k] * wa[a] (:122-124)
            const size_t i = static_cast<size_t>(a) * nf + k;
            data[2 * i] = values[2 * i] * wf[k] * wa[a];
            data[2 * i + 1] = values[2 * i + 1] * wf[k] * wa[a];
        }
    Dev d;
    double2* din = d.alloc<double2>(static_cast<size_t>(na) * nf);
    double2* cols = d.alloc<double2>(static_cast<size_t>(na) * mr);   // [a][r]
    double2* rows = d.alloc<double2>(static_cast<size_t>(mr) * na);   // [r][a]
    double2* img = d.alloc<double2>(static_cast<size_t>(mr) * mc);    // [r][c]
    double* dmag = d.alloc<double>(static_cast<size_t>(mr) * mc);
    if (!din || !cols || !rows || !img || !dmag) return finish(cuda_fail("isar alloc"));
    if (cudaMemcpy(din, data.data(), sizeof(double2) * na * nf, cudaMemcpyHostToDevice) != cudaSuccess)
        return finish(cuda_fail("isar upload"));
    auto gy = [](uint32_t rows_) { return std::min<uint32_t>(rows_, 65535u); };  // kernels stride over rows
    idft_rows<<<dim3((mr + 127) / 128, gy(na)), 128>>>(din, na, nf, mr, false, cols);     // down-range
    transpose_c<<<dim3((mr + 127) / 128, gy(na)), 128>>>(cols, na, mr, rows);
    idft_rows<<<dim3((mc + 127) / 128, gy(mr)), 128>>>(rows, mr, na, mc, true, img);      // cross-range
    const size_t npx = static_cast<size_t>(mr) * mc;
    magnitude<<<static_cast<unsigned>((npx + 255) / 256), 256>>>(img, npx, dmag);
    if (cudaGetLastError() != cudaSuccess) return finish(cuda_fail("isar launch"));
    std::vector<double> mag(npx);
    if (cudaMemcpy(mag.data(), dmag, sizeof(double) * npx, cudaMemcpyDeviceToHost) != cudaSuccess)
        return finish(cuda_fail("isar"));
    double peak = 0.0;
    for (double m : mag) peak = std::max(peak, m);
    const double pk_db = to_db(peak);
    const double fl = pk_db + floor_db;
    for (size_t i = 0; i < npx; ++i) mag_db[i] = std::max(to_db(mag[i]), fl);
    const double f_center = 0.5 * (freqs[0] + freqs[nf - 1]);
    const double dtheta = dtheta_deg * kPi / 180.0;
    const double range_bin = kC / (2.0 * df * static_cast<double>(mr));
    const double cross_bin = kC / (2.0 * f_center * dtheta * static_cast<double>(mc));
    const std::vector<double> ra = centered_axis(mr, range_bin), ca = centered_axis(mc, cross_bin);
    for (uint32_t i = 0; i < mr; ++i) down_range_m[i] = ra[i];
    for (uint32_t i = 0; i < mc; ++i) cross_range_m[i] = ca[i];
    if (peak_db) *peak_db = pk_db;
    return MCSBR_OK;
}

}  // extern "C"
