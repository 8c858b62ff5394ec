// Drop-in solver translation unit for the reference's own C++ interface.
//
// A maintainer builds the reference (proj/) with THIS file in place of
// proj/src/solver_mc.cpp and proj/src/solver_det.cpp and links
// libmcsbr_gpu.so: every declaration of proj/include/mcsbr/solver_mc.hpp and
// proj/include/mcsbr/solver_det.hpp is defined here, so the reference's
// runner (run_solver, runner.cpp:67-77), CLI (tools/mcsbr.cpp) and tests run
// unchanged and their estimate() / solve() calls execute on the B200 through
// the C ABI (include/mcsbr_gpu.h).  The artifacts the runner writes
// (sweep.csv, stats.json, manifest.json, ...) are therefore produced by the
// reference's own writers, from results filled exactly as the reference
// fills them (solver names, seeds, stats vector sizes, the 192-byte
// PathState accounting, contribution order).
//
// Only the two solver entry points run on the GPU; the small host helpers
// the header also declares (McConfig::validate, build_strata,
// sample_stratum, choose_branch, roulette_step, DetConfig::validate) are
// restated on the host with the reference's semantics and messages.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <list>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "mcsbr/em_math.hpp"
#include "mcsbr/geometry.hpp"
#include "mcsbr/solver_det.hpp"
#include "mcsbr/solver_mc.hpp"
#include "mcsbr_gpu.h"

namespace mcsbr {

static_assert(sizeof(Triangle) == sizeof(mcsbr_triangle), "Triangle layout (geometry.hpp:23-29)");
static_assert(sizeof(Material) == sizeof(mcsbr_material), "Material layout");
static_assert(sizeof(Contribution) == sizeof(mcsbr_contribution), "Contribution layout (farfield.hpp:45-52)");
static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 layout");

namespace {

constexpr uint64_t kPathStateBytes = sizeof(PathState);  // 192 on LP64

// C-ABI status -> the exception type the reference throws for that failure
[[noreturn]] void raise(int code) {
    const std::string msg = mcsbr_gpu_last_error();
    if (code == MCSBR_EINVAL) throw std::invalid_argument(msg);
    if (code == MCSBR_EDEVICE && msg.find("grazing") != std::string::npos) throw DegenerateGeometryError(msg);
    if (code == MCSBR_EDEVICE) throw DomainError(msg);
    if (code == MCSBR_ESCENE) throw SceneError(msg);
    throw std::runtime_error(msg);
}

void check(int code) {
    if (code != MCSBR_OK) raise(code);
}

int device_index() {
    const char* e = std::getenv("MCSBR_DEVICE");
    return e ? std::atoi(e) : 0;
}

// The GPUs the solvers shard over (estimate's `workers` picks how many):
// MCSBR_DEVICE first, then every other visible device; MCSBR_DEVICES=1 keeps
// one.  run_blocks' worker threads (solver_common.cpp:70-89) become devices.
std::vector<int> device_list() {
    int n = 0;
    mcsbr_gpu_device_count(&n);
    const int first = device_index();
    std::vector<int> d{first};
    const char* lim = std::getenv("MCSBR_DEVICES");
    const int want = lim ? std::max(1, std::atoi(lim)) : n;
    for (int i = 0; i < n && static_cast<int>(d.size()) < want; ++i)
        if (i != first) d.push_back(i);
    return d;
}

// ---- device-resident scenes --------------------------------------------------
// A Scene is immutable after finalize(); the runner re-uses one Scene for a
// whole angle sweep / ISAR, so the uploaded geometry + BVH is cached by
// identity (address, array addresses and sizes) plus a sampled content
// digest that rejects a different scene reusing the same storage.

uint64_t digest(const Scene& s) {
    uint64_t h = 0xcbf29ce484222325ull;
    auto mix = [&h](const void* p, size_t n) {
        const unsigned char* b = static_cast<const unsigned char*>(p);
        for (size_t i = 0; i < n; ++i) {
            h ^= b[i];
            h *= 0x100000001b3ull;
        }
    };
    const size_t nv = s.vertices.size(), nt = s.triangles.size();
    const size_t sv = std::max<size_t>(1, nv / 4096), st = std::max<size_t>(1, nt / 4096);
    for (size_t i = 0; i < nv; i += sv) mix(&s.vertices[i], sizeof(Vec3));
    for (size_t i = 0; i < nt; i += st) mix(&s.triangles[i], sizeof(Triangle));
    if (nv) mix(&s.vertices.back(), sizeof(Vec3));
    if (nt) mix(&s.triangles.back(), sizeof(Triangle));
    mix(s.materials.data(), s.materials.size() * sizeof(Material));
    return h;
}

struct CachedScene {
    const Scene* owner;
    const void* vtx;
    const void* tri;
    size_t nv, nt, nm;
    uint64_t hash;
    mcsbr_scene* dev;
};

std::mutex g_mu;
std::list<CachedScene> g_cache;  // most recent first
constexpr size_t kCacheScenes = 4;

mcsbr_scene* device_scene(const Scene& s) {
    const uint64_t h = digest(s);
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it) {
        if (it->owner == &s && it->vtx == s.vertices.data() && it->tri == s.triangles.data() &&
            it->nv == s.vertices.size() && it->nt == s.triangles.size() && it->nm == s.materials.size() &&
            it->hash == h) {
            g_cache.splice(g_cache.begin(), g_cache, it);
            return g_cache.front().dev;
        }
    }
    std::vector<mcsbr_material> mats(s.materials.size());
    for (size_t i = 0; i < mats.size(); ++i) {
        std::memset(&mats[i], 0, sizeof(mats[i]));
        mats[i].eps_r = s.materials[i].eps_r;
        mats[i].mu_r = s.materials[i].mu_r;
        mats[i].is_pec = s.materials[i].is_pec ? 1 : 0;
    }
    mcsbr_scene* dev = nullptr;
    const std::vector<int> devs = device_list();
    check(mcsbr_gpu_scene_create_multi(reinterpret_cast<const double*>(s.vertices.data()),
                                       static_cast<uint32_t>(s.vertices.size()),
                                       reinterpret_cast<const mcsbr_triangle*>(s.triangles.data()),
                                       static_cast<uint32_t>(s.triangles.size()), mats.data(),
                                       static_cast<uint32_t>(mats.size()), nullptr, devs.data(),
                                       static_cast<int>(devs.size()), &dev));
    g_cache.push_front({&s, s.vertices.data(), s.triangles.data(), s.vertices.size(), s.triangles.size(),
                        s.materials.size(), h, dev});
    while (g_cache.size() > kCacheScenes) {
        mcsbr_gpu_scene_destroy(g_cache.back().dev);
        g_cache.pop_back();
    }
    return dev;
}

mcsbr_excitation to_c(const Excitation& e) {
    mcsbr_excitation x;
    std::memset(&x, 0, sizeof(x));
    auto put = [](double* d, const Vec3& v) {
        d[0] = v.x;
        d[1] = v.y;
        d[2] = v.z;
    };
    put(x.k_inc, e.k_inc);
    put(x.pol_v, e.pol_v);
    put(x.pol_h, e.pol_h);
    put(x.k_scatter, e.k_scatter);
    put(x.rx_v, e.rx_v);
    put(x.rx_h, e.rx_h);
    x.occlusion_enabled = e.occlusion_enabled ? 1 : 0;
    return x;
}

SweepResult to_sweep(const std::vector<double>& freqs, const std::vector<double>& values) {
    SweepResult r;
    r.frequencies = freqs;
    const size_t nf = freqs.size();
    for (int ch = 0; ch < kPolChannelCount; ++ch) {
        r.values[ch].resize(nf);
        for (size_t i = 0; i < nf; ++i)
            r.values[ch][i] = complexd(values[2 * (ch * nf + i)], values[2 * (ch * nf + i) + 1]);
    }
    return r;
}

// RunStats as the reference's blocks + merge leave them (solver_common.cpp:51-68)
RunStats to_stats(const mcsbr_stats& st, bool roulette_vectors) {
    RunStats r;
    r.rays_launched = st.rays_launched;
    r.segments_traced = st.segments_traced;
    r.contributions = st.contributions;
    r.grazing_kills = st.grazing_kills;
    r.cap_kills = st.cap_kills;
    r.rays_per_bounce.assign(st.rays_per_bounce, st.rays_per_bounce + st.n_rounds);
    if (roulette_vectors) {  // both grow to the deepest bounce with a roulette test
        size_t n = 0;
        for (size_t i = 0; i < MCSBR_MAX_BOUNCE_LIMIT; ++i)
            if (st.roulette_candidates[i]) n = i + 1;
        r.roulette_candidates.assign(st.roulette_candidates, st.roulette_candidates + n);
        r.roulette_survivors.assign(st.roulette_survivors, st.roulette_survivors + n);
    }
    r.block_size = st.block_size;
    r.state_bytes_per_ray = kPathStateBytes;
    return r;
}

// run one C-ABI solver call, growing the contribution buffer if needed
template <typename Call>
void run_collect(Call&& call, std::vector<Contribution>* out, uint64_t guess) {
    if (!out) {
        check(call(nullptr, 0, nullptr));
        return;
    }
    std::vector<Contribution> buf(std::max<uint64_t>(guess, 1024));
    uint64_t n = 0;
    check(call(reinterpret_cast<mcsbr_contribution*>(buf.data()), buf.size(), &n));
    if (n > buf.size()) {  // the stream is deterministic: re-run with the exact size
        buf.assign(n, Contribution{});
        check(call(reinterpret_cast<mcsbr_contribution*>(buf.data()), buf.size(), &n));
    }
    buf.resize(n);
    out->insert(out->end(), buf.begin(), buf.end());
}

}  // namespace

// ---- Monte Carlo (solver_mc.hpp) ----------------------------------------------

void McConfig::validate() const {
    mcsbr_mc_config c;
    mcsbr_gpu_default_config(&c);
    c.strata_per_wavelength = strata_per_wavelength;
    c.samples_per_stratum = samples_per_stratum;
    c.roulette_q = roulette.q;
    c.roulette_min_bounce = roulette.min_bounce;
    c.max_bounce = max_bounce;
    c.block_size = block_size;
    // the reference's checks and messages (solver_mc.cpp:10-17), plus the
    // GPU's per-bounce counter limit (max_bounce <= 64)
    check(mcsbr_gpu_validate_config(&c));
}

StrataGrid build_strata(const LaunchRect& rect, double strata_per_wavelength, double reference_wavelength) {
    if (!(reference_wavelength > 0.0))
        throw std::invalid_argument("build_strata: reference wavelength must be > 0");
    const double side = reference_wavelength / strata_per_wavelength;
    StrataGrid g;
    g.rect = rect;
    g.nu = std::max(1, static_cast<int>(std::ceil(2.0 * rect.half_u / side)));
    g.nv = std::max(1, static_cast<int>(std::ceil(2.0 * rect.half_v / side)));
    g.cell_area = rect.area() / (static_cast<double>(g.nu) * g.nv);
    g.pdf_per_cell = 1.0 / g.cell_area;
    return g;
}

StratumSample sample_stratum(const StrataGrid& grid, uint32_t cell, uint32_t sample, uint64_t seed,
                             bool jitter) {
    const uint32_t nu = static_cast<uint32_t>(grid.nu);
    const double ju = jitter ? counter_uniform(seed, cell, sample, 0, RngPurpose::kLaunchU) : 0.5;
    const double jv = jitter ? counter_uniform(seed, cell, sample, 0, RngPurpose::kLaunchV) : 0.5;
    const double su = -1.0 + 2.0 * ((cell % nu) + ju) / grid.nu;
    const double sv = -1.0 + 2.0 * ((cell / nu) + jv) / grid.nv;
    return {grid.rect.point_at(su, sv), grid.pdf_per_cell};
}

BranchChoice choose_branch(const BranchSet& set, BranchStrategy strategy, double p_min, double u) {
    if (set.count == 1) return {0, 1.0};
    double pr = 0.5;
    if (strategy == BranchStrategy::kFresnel)
        pr = std::min(std::max(0.5 * (std::abs(set.coeffs.r_s) + std::abs(set.coeffs.r_p)), p_min), 1.0 - p_min);
    return u < pr ? BranchChoice{0, pr} : BranchChoice{1, 1.0 - pr};
}

bool roulette_step(PathState& state, const RouletteConfig& roulette, double u) {
    if (state.bounce < roulette.min_bounce) return true;
    if (!(u > roulette.q)) {
        state.alive = false;
        return false;
    }
    state.weight /= (1.0 - roulette.q);
    return true;
}

McResult estimate(const Scene& scene, const Excitation& excitation, const std::vector<double>& frequencies,
                  const McConfig& config, int workers, std::vector<Contribution>* contributions_out) {
    const auto t0 = std::chrono::steady_clock::now();
    config.validate();
    if (frequencies.empty()) throw std::invalid_argument("estimate: empty frequency list");
    mcsbr_scene* dev = device_scene(scene);
    const mcsbr_excitation exc = to_c(excitation);
    mcsbr_mc_config c;
    mcsbr_gpu_default_config(&c);
    c.strata_per_wavelength = config.strata_per_wavelength;
    c.samples_per_stratum = config.samples_per_stratum;
    c.branch_strategy = config.branch_strategy == BranchStrategy::kFresnel ? MCSBR_BRANCH_FRESNEL
                                                                           : MCSBR_BRANCH_FIFTY_FIFTY;
    c.roulette_enabled = config.roulette.enabled ? 1 : 0;
    c.roulette_min_bounce = config.roulette.min_bounce;
    c.roulette_q = config.roulette.q;
    c.max_bounce = config.max_bounce;
    c.jitter = config.jitter ? 1 : 0;
    c.seed = config.seed;
    c.reference_wavelength = config.reference_wavelength;
    c.launch_padding = config.launch_padding;
    c.p_min = config.p_min;
    c.block_size = config.block_size;
    c.rng_mode = MCSBR_RNG_REFERENCE;  // the reference's per-ray stream
    // order-independent integer sums: sweeps (and the runner's CSV artifacts)
    // byte-identical across reruns and worker counts, as the reference's
    // fixed-order block merge makes them (solver_mc.cpp:212-216, runner.hpp:2-5)
    c.reduction = MCSBR_REDUCE_EXACT;
    const uint32_t nf = static_cast<uint32_t>(frequencies.size());
    std::vector<double> values(8ull * nf);
    mcsbr_stats st;
    std::vector<Contribution> collected;
    run_collect(
        [&](mcsbr_contribution* buf, uint64_t cap, uint64_t* n) {
            return mcsbr_gpu_estimate(dev, &exc, frequencies.data(), nf, &c, workers, values.data(), &st, buf,
                                      cap, n);
        },
        contributions_out ? &collected : nullptr, 1u << 16);
    if (contributions_out) {
        // the reference's emission order: block by block, and within a block
        // wavefront round (= bounce) by round in entry order (solver_mc.cpp:105-210)
        const uint64_t bs = static_cast<uint64_t>(config.block_size);
        std::stable_sort(collected.begin(), collected.end(), [bs](const Contribution& a, const Contribution& b) {
            const uint64_t ea = a.order_key >> 8, eb = b.order_key >> 8;
            if (ea / bs != eb / bs) return ea / bs < eb / bs;
            if (a.bounce != b.bounce) return a.bounce < b.bounce;
            return ea < eb;
        });
        contributions_out->insert(contributions_out->end(), collected.begin(), collected.end());
    }
    McResult r;
    r.sweep = to_sweep(frequencies, values);
    r.sweep.solver = "mc";
    r.sweep.seed = config.seed;
    r.sweep.rays_launched = st.rays_launched;
    r.stats = to_stats(st, true);
    // largest wavefront block alive at once (solver_mc.cpp:124-127)
    r.stats.peak_live_state_bytes =
        std::min<uint64_t>(st.rays_launched, static_cast<uint64_t>(config.block_size)) * kPathStateBytes;
    r.stats.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return r;
}

// ---- deterministic (solver_det.hpp) ---------------------------------------------

void DetConfig::validate() const {
    mcsbr_det_config c;
    mcsbr_gpu_default_det_config(&c);
    c.rays_per_wavelength = rays_per_wavelength;
    c.max_bounce = max_bounce;
    c.amplitude_cutoff = amplitude_cutoff;
    c.block_size = block_size;
    check(mcsbr_gpu_validate_det_config(&c));
}

DetResult solve(const Scene& scene, const Excitation& excitation, const std::vector<double>& frequencies,
                const DetConfig& config, int workers, std::vector<Contribution>* contributions_out) {
    const auto t0 = std::chrono::steady_clock::now();
    config.validate();
    if (frequencies.empty()) throw std::invalid_argument("solve: empty frequency list");
    mcsbr_scene* dev = device_scene(scene);
    const mcsbr_excitation exc = to_c(excitation);
    mcsbr_det_config c;
    mcsbr_gpu_default_det_config(&c);
    c.rays_per_wavelength = config.rays_per_wavelength;
    c.max_bounce = config.max_bounce;
    c.amplitude_cutoff = config.amplitude_cutoff;
    c.force_stack_accounting = config.force_stack_accounting ? 1 : 0;
    c.launch_padding = config.launch_padding;
    c.reference_wavelength = config.reference_wavelength;
    c.block_size = config.block_size;
    const uint32_t nf = static_cast<uint32_t>(frequencies.size());
    std::vector<double> values(8ull * nf);
    mcsbr_stats st;
    // deterministic keys (cell << 24 | event) sort into the reference's order
    run_collect(
        [&](mcsbr_contribution* buf, uint64_t cap, uint64_t* n) {
            return mcsbr_gpu_solve(dev, &exc, frequencies.data(), nf, &c, workers, values.data(), &st, buf, cap,
                                   n);
        },
        contributions_out, 1u << 16);
    DetResult r;
    r.sweep = to_sweep(frequencies, values);
    r.sweep.solver = "deterministic";
    r.sweep.rays_launched = st.rays_launched;
    r.stats = to_stats(st, false);
    r.stats.peak_live_state_bytes = st.peak_live_state_bytes;
    r.stats.forced_stack_bytes = st.forced_stack_bytes;
    r.stats.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return r;
}

}  // namespace mcsbr
