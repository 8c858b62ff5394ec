// Host orchestration + the C ABI (include/mcsbr_gpu.h).
//
// Host-side planning is fp64 and restates the reference exactly (this file is
// compiled with -ffp-contract=off and no -march, like the reference build):
//   Scene::finalize bounding sphere   proj/src/geometry.cpp:146-162
//   launch_rect                       proj/src/geometry.cpp:246-275
//   build_strata                      proj/src/solver_mc.cpp:19-31
//   McConfig::validate                proj/src/solver_mc.cpp:10-17
//   SweepAccumulator::finalize        proj/src/farfield.cpp:154-167
//   RunStats                          proj/include/mcsbr/solver_common.hpp:37-53
// Everything per ray runs on the GPU (bvh.cu, trace.cu); there is no CPU
// fallback: without a device every compute entry point returns MCSBR_ECUDA.
#include <algorithm>
#include <atomic>
#include <iterator>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>
#include <map>
#include <mutex>
#include <unordered_map>

#include "fixedpoint.cuh"
#include "internal.h"
#include "mcsbr_gpu.h"

using namespace mcsbr_int;

// ---------------------------------------------------------------------------
// caching device allocator (internal.h)
namespace mcsbr_int {
namespace {
struct AllocCache {
    std::mutex m;
    std::unordered_map<void*, std::pair<int, size_t>> size_of;  // live and cached blocks
    std::multimap<size_t, void*> free_blocks[64];               // per device: size -> block
    size_t cached[64] = {};                                     // per device: bytes held in free_blocks
    size_t limit[64] = {};                                      // per device: cache bound (0 = not yet known)
};
AllocCache& alloc_cache() {
    static AllocCache* c = new AllocCache();  // never destroyed (used during process exit)
    return *c;
}
// a quarter of the device's memory (B200: ~45 GB): large enough to keep a
// sweep's contribution-record buffer between scenes (c5: ~32 GB, one launch
// group; a cudaFree + cudaMalloc of it costs ~15 ms per e2e step, up to
// ~0.5 s), small enough to leave the device to others
size_t cache_limit(AllocCache& c, int dev) {
    if (!c.limit[dev]) {
        size_t free_b = 0, total = 0;
        c.limit[dev] = cudaMemGetInfo(&free_b, &total) == cudaSuccess ? total / 4 : (size_t{4} << 30);
    }
    return c.limit[dev];
}
size_t alloc_class(size_t n) {
    n = n ? n : 1;
    const size_t g = n >= (size_t{1} << 20) ? (size_t{1} << 16) : 256;  // 64 KB / 256 B granules
    return (n + g - 1) / g * g;
}
// hand device dev's cached blocks back to the driver (caller holds the lock)
void release_cached(AllocCache& c, int dev) {
    for (auto& kv : c.free_blocks[dev]) {
        cudaFree(kv.second);
        c.size_of.erase(kv.second);
    }
    c.free_blocks[dev].clear();
    c.cached[dev] = 0;
}
}  // namespace

cudaError_t dev_malloc(void** p, size_t bytes) {
    *p = nullptr;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const bool cacheable = dev >= 0 && dev < 64;
    const size_t n = alloc_class(bytes);
    AllocCache& c = alloc_cache();
    if (cacheable) {
        std::lock_guard<std::mutex> g(c.m);
        auto& fb = c.free_blocks[dev];
        auto it = fb.lower_bound(n);
        if (it != fb.end() && it->first <= 2 * n) {  // reuse a block at most twice the size
            *p = it->second;
            c.cached[dev] -= it->first;
            fb.erase(it);
            return cudaSuccess;
        }
    }
    e = cudaMalloc(p, n);
    if (getenv("MCSBR_ALLOC_DEBUG") && n >= (size_t{16} << 20))
        fprintf(stderr, "[alloc] cudaMalloc %zu MB (cached %zu MB)\n", n >> 20, cacheable ? c.cached[dev] >> 20 : 0);
    if (e != cudaSuccess && cacheable) {
        // out of memory: hand this device's cache back to the driver and retry once
        cudaGetLastError();
        {
            std::lock_guard<std::mutex> g(c.m);
            release_cached(c, dev);
        }
        e = cudaMalloc(p, n);
    }
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(c.m);
    c.size_of[*p] = {dev, n};
    return cudaSuccess;
}

void dev_free(void* p, bool synced) {
    if (!p) return;
    // the block may be read by work still in flight; callers that have
    // synchronised the streams that used it pass synced = true
    if (!synced) cudaDeviceSynchronize();
    AllocCache& c = alloc_cache();
    std::lock_guard<std::mutex> g(c.m);
    auto it = c.size_of.find(p);
    if (it == c.size_of.end()) {  // not ours
        cudaFree(p);
        return;
    }
    const int dev = it->second.first;
    const size_t n = it->second.second;
    if (dev >= 0 && dev < 64 && n <= cache_limit(c, dev)) {
        // keep the block just freed (the one the next, similar call asks for)
        // and hand older cached blocks back to the driver, largest first
        auto& fb = c.free_blocks[dev];
        while (c.cached[dev] + n > cache_limit(c, dev) && !fb.empty()) {
            auto big = std::prev(fb.end());
            cudaFree(big->second);
            c.size_of.erase(big->second);
            c.cached[dev] -= big->first;
            fb.erase(big);
        }
    }
    if (dev < 0 || dev >= 64 || c.cached[dev] + n > cache_limit(c, dev)) {
        if (getenv("MCSBR_ALLOC_DEBUG") && n >= (size_t{16} << 20))
            fprintf(stderr, "[alloc] cudaFree %zu MB (cached %zu MB)\n", n >> 20, c.cached[dev] >> 20);
        c.size_of.erase(it);
        cudaFree(p);
        return;
    }
    c.free_blocks[dev].emplace(n, p);
    c.cached[dev] += n;
}

}  // namespace mcsbr_int

namespace {

constexpr double kC = 299792458.0;
constexpr double kPi = 3.14159265358979323846;

thread_local std::string g_err;

// Pinned 8-byte host slots for the asynchronous readbacks (record peak,
// wavefront work-list length), handed out from one process-wide pool of
// pinned pages that is never freed: a per-scene cudaMallocHost /
// cudaFreeHost pair cost up to ~0.5 s in scene destroy on a busy host.
struct PinnedSlots {
    std::mutex m;
    std::vector<unsigned long long*> free;
};
PinnedSlots& pinned_slots() {
    static PinnedSlots* p = new PinnedSlots();  // never destroyed (used during process exit)
    return *p;
}
cudaError_t pinned_slot(unsigned long long** out) {
    PinnedSlots& P = pinned_slots();
    std::lock_guard<std::mutex> g(P.m);
    if (P.free.empty()) {
        void* page = nullptr;
        const cudaError_t e = cudaMallocHost(&page, 4096);
        if (e != cudaSuccess) return e;
        unsigned long long* q = static_cast<unsigned long long*>(page);
        for (int i = 511; i >= 0; --i) P.free.push_back(q + i);
    }
    *out = P.free.back();
    P.free.pop_back();
    return cudaSuccess;
}
void pinned_release(unsigned long long* p) {
    if (!p) return;
    PinnedSlots& P = pinned_slots();
    std::lock_guard<std::mutex> g(P.m);
    P.free.push_back(p);
}

// MCSBR_HOST_TIMING=1: host-side phase times of scene create / estimate /
// destroy on stderr (diagnostics for the e2e measurement)
struct HostPhases {
    const char* what;
    bool on;
    std::chrono::steady_clock::time_point t0, t;
    std::string log;
    explicit HostPhases(const char* w) : what(w), on(std::getenv("MCSBR_HOST_TIMING") != nullptr) {
        if (on) t0 = t = std::chrono::steady_clock::now();
    }
    void mark(const char* phase) {
        if (!on) return;
        const auto n = std::chrono::steady_clock::now();
        char b[96];
        std::snprintf(b, sizeof b, " %s %.2f", phase, std::chrono::duration<double, std::milli>(n - t).count());
        log += b;
        t = n;
    }
    ~HostPhases() {
        if (on)
            std::fprintf(stderr, "[host] %s%s | total %.2f ms\n", what, log.c_str(),
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
};
thread_local uint64_t g_launches = 0;

// Per-kernel device timing (mcsbr_gpu_kernel_timing): while enabled, run_job
// brackets every path-kernel and accumulate launch with CUDA events on the
// launch stream; mcsbr_gpu_kernel_times sums them.  Events are pooled per
// thread and device.
struct KernelTiming {
    bool on = false;
    int device = -1;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::vector<std::pair<int, size_t>> marks;  // (kind 0 path / 1 accumulate, first event index)
};
thread_local KernelTiming g_kt;

// record the start (end = false) or end event of one timed launch
cudaError_t kt_mark(int kind, cudaStream_t stream, int device, bool end) {
    if (!g_kt.on) return cudaSuccess;
    if (g_kt.device != device) {
        for (cudaEvent_t e : g_kt.pool) cudaEventDestroy(e);
        g_kt.pool.clear();
        g_kt.used = 0;
        g_kt.marks.clear();
        g_kt.device = device;
    }
    if (g_kt.used == g_kt.pool.size()) {
        cudaEvent_t e;
        cudaError_t r = cudaEventCreate(&e);
        if (r != cudaSuccess) return r;
        g_kt.pool.push_back(e);
    }
    if (!end) g_kt.marks.emplace_back(kind, g_kt.used);
    return cudaEventRecord(g_kt.pool[g_kt.used++], stream);
}

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_err(cudaError_t e, const char* what) {
    return set_err(MCSBR_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(x, what)                                  \
    do {                                             \
        cudaError_t e_ = (x);                        \
        if (e_ != cudaSuccess) return cuda_err(e_, what); \
    } while (0)

struct V {
    double x, y, z;
};
inline V operator+(V a, V b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V operator*(V a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline double dot(V a, V b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V cross(V a, V b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline double norm(V v) { return std::sqrt(dot(v, v)); }
inline V normalized(V v) {
    const double n = norm(v);
    return {v.x / n, v.y / n, v.z / n};
}
inline V ld(const double* p) { return {p[0], p[1], p[2]}; }
inline void st(double* p, V v) {
    p[0] = v.x;
    p[1] = v.y;
    p[2] = v.z;
}

// device temporaries of one call, freed on every exit path
struct TempBufs {
    std::vector<void*> p;
    TempBufs() = default;
    TempBufs(const TempBufs&) = delete;
    TempBufs& operator=(const TempBufs&) = delete;
    ~TempBufs() {
        for (void* q : p) dev_free(q);
    }
    template <class T>
    cudaError_t alloc(T** q, size_t bytes) {
        const cudaError_t e = dev_malloc(q, bytes);
        if (e == cudaSuccess) p.push_back(*q);
        return e;
    }
};

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaError_t reserve(size_t want) {
        if (want <= n) return cudaSuccess;
        if (p) dev_free(p);
        p = nullptr;
        n = 0;
        cudaError_t e = dev_malloc(&p, sizeof(T) * std::max<size_t>(want, 1));
        if (e == cudaSuccess) n = want;
        return e;
    }
    void release(bool synced = false) {
        if (p) dev_free(p, synced);
        p = nullptr;
        n = 0;
    }
};

}  // namespace

// Records-per-entry estimate a NEW scene starts from: the last one learnt on
// any scene of the process (a sweep repeated on fresh scenes -- the e2e
// step -- then sizes its record buffer right from the first call, and the
// buffer is the same size class the allocator cached).  A hint only: a
// wrong one costs memory or overflow adds, never correctness.
std::atomic<double>& rec_ratio_hint() {
    static std::atomic<double> h{0.25};
    return h;
}

struct mcsbr_scene {
    // multi-device scenes (mcsbr_gpu_scene_create_multi): this object is the
    // primary (devices[0], where the BVH was built); replicas hold copies of
    // the device arrays on devices[1..] and share nothing else
    std::vector<mcsbr_scene*> replicas;
    int device = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    uint32_t nv = 0, nt = 0, nm = 0;
    double scene_lo[3] = {0, 0, 0}, scene_hi[3] = {0, 0, 0};  // vertex AABB
    double center[3] = {0, 0, 0};
    double radius = 0.0, diameter = 0.0;
    double ambient_n = 1.0;
    bool all_pec = false;  // every triangle has a PEC side (kernel specialisation)
    bool lossy = false;    // complex-permittivity transport
    // deferred accumulation: contribution records per launched entry, learnt
    // from the peak record count of earlier F > 1 jobs on this scene (read
    // back asynchronously: peak_host is valid once peak_ev has completed)
    double rec_ratio = rec_ratio_hint().load(std::memory_order_relaxed);
    unsigned long long* peak_host = nullptr;
    cudaEvent_t peak_ev = nullptr;
    uint64_t peak_entries = 0;
    bool peak_pending = false;
    double* d_nim = nullptr;
    double* d_vtx = nullptr;
    float* d_tri32 = nullptr;  // fp32 vertices relative to the centre, 9 per triangle (cover.cu)
    uint4* d_tri = nullptr;
    double2* d_info = nullptr;
    double2* d_mat = nullptr;
    BvhBuildOut bvh{};
    // reusable work buffers
    DevBuf<IncDev> inc;
    DevBuf<RxDev> rx;
    DevBuf<double> k0;
    DevBuf<double> sums;
    DevBuf<unsigned long long> counters;
    DevBuf<unsigned long long> tile;
    DevBuf<double> recs;  // deferred-accumulation contribution records
    DevBuf<double> nufft_grid;  // spread.cu: per-incidence grids of one launch group
    DevBuf<double> nufft_hat;   // spread.cu: 1 / Psi(m)
    uint32_t nufft_hat_nf = 0;  // the nf nufft_hat holds
    DevBuf<uint32_t> nufft_idx;     // spread.cu: record indices by incidence
    DevBuf<uint32_t> nufft_inc;     // spread.cu: each record's incidence (written by the path kernel)
    DevBuf<uint32_t> nufft_bucket;  // spread.cu: per-incidence counts / cursors
    DevBuf<uint32_t> cover;  // launch-ray coverage bitmaps of the current job
    DevBuf<float4> leaf32;                 // statistical-mode fp32 leaf triangle records (built on first use)
    DevBuf<double> plan_axes;              // launch planning (prep.cu): axes in,
    DevBuf<unsigned long long> plan_ext;   // projection extents out
    DevBuf<unsigned long long> xsums;  // MCSBR_REDUCE_EXACT: 192-bit sums of the current job
    DevBuf<long long> limbs;           // MCSBR_REDUCE_EXACT: their limbs (estimate / estimate_batch)
    // wavefront path pool (wavefront.cu): fields, (kind, rid, list), control words
    DevBuf<double> wf_pool;
    DevBuf<uint32_t> wf_u32;
    DevBuf<unsigned long long> wf_ctl;
    unsigned long long* wf_host = nullptr;  // pinned: a work-list length read back
    cudaEvent_t wf_ev = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;

    SceneView view() const {
        SceneView s{};
        s.nodes = bvh.nodes;
        s.tri64 = bvh.tri64;
        s.tri_info = d_info;
        s.mat = d_mat;
        s.root_ref = bvh.root_ref;
        s.n_tri = nt;
        s.diameter = diameter;
        s.t_eps = 1e-6 * diameter;
        s.ambient_n = ambient_n;
        s.all_pec = all_pec ? 1 : 0;
        s.lossy = lossy ? 1 : 0;
        s.mat_nim = d_nim;
        s.tri32 = leaf32.n ? leaf32.p : nullptr;
        s.center[0] = center[0];
        s.center[1] = center[1];
        s.center[2] = center[2];
        s.skip_radius = radius * 1.01 + 1e-9;
        s.margin_r = static_cast<float>(radius * 1.01 + 1e-9);
        return s;
    }
};

namespace {

// scenes up to this many triangles get the long scheduling chunks (run_job)
constexpr uint32_t kSmallSceneTris = 131072;
constexpr uint32_t kLargeSceneTris = 524288;  // above: 1024-entry chunk cap (c5), below 256 (c4)

// launch_rect's axes (geometry.cpp:246-253): seed axis x, or y if |k.x| > 0.9
void plan_axes(const double k_inc[3], V* k, V* u, V* v) {
    *k = normalized(ld(k_inc));
    V seed{1.0, 0.0, 0.0};
    if (std::abs(k->x) > 0.9) seed = V{0.0, 1.0, 0.0};
    *u = normalized(cross(*k, seed));
    *v = cross(*k, *u);
}

// launch_rect's projection extents (min / max of dot(p, u), dot(p, v) over
// the vertices, geometry.cpp:254-266) of n incidences at once on the device
// (prep.cu extents_kernel, the host loop's exact arithmetic); ext[4a..4a+3] =
// (ulo, uhi, vlo, vhi)
int plan_extents(const mcsbr_scene* s, const std::vector<double>& axes, std::vector<double>* ext) {
    const uint32_t n = static_cast<uint32_t>(axes.size() / 6);
    auto* ms = const_cast<mcsbr_scene*>(s);
    CK(ms->plan_axes.reserve(axes.size()), "dev_malloc(plan axes)");
    CK(ms->plan_ext.reserve(4ull * n), "dev_malloc(plan extents)");
    CK(cudaMemcpyAsync(ms->plan_axes.p, axes.data(), sizeof(double) * axes.size(), cudaMemcpyHostToDevice, s->stream),
       "upload plan axes");
    CK(launch_extents(s->d_vtx, s->nv, ms->plan_axes.p, n, ms->plan_ext.p, s->sms, s->stream), "extents launch");
    ++g_launches;
    std::vector<unsigned long long> o(4ull * n);
    CK(cudaMemcpyAsync(o.data(), ms->plan_ext.p, sizeof(unsigned long long) * o.size(), cudaMemcpyDeviceToHost,
                       s->stream), "plan extents readback");
    CK(cudaStreamSynchronize(s->stream), "cudaStreamSynchronize");
    ext->resize(o.size());
    for (size_t i = 0; i < o.size(); ++i) (*ext)[i] = unord(o[i]);
    return MCSBR_OK;
}

// launch_rect (geometry.cpp:246-275) from its axes and extents + build_strata
// (solver_mc.cpp:19-31)
int plan_finish(const mcsbr_scene* s, V k, V u, V v, const double* ext, double padding, double spw, double lambda_ref,
                int32_t spp, mcsbr_launch_plan* out) {
    double ulo = ext[0], uhi = ext[1], vlo = ext[2], vhi = ext[3];
    ulo -= padding;
    uhi += padding;
    vlo -= padding;
    vhi += padding;
    std::memset(out, 0, sizeof(*out));
    st(out->u_axis, u);
    st(out->v_axis, v);
    out->half_u = 0.5 * (uhi - ulo);
    out->half_v = 0.5 * (vhi - vlo);
    const double standoff = dot(ld(s->center), k) - 1.05 * s->radius;
    st(out->center, u * (0.5 * (ulo + uhi)) + v * (0.5 * (vlo + vhi)) + k * standoff);
    if (!(lambda_ref > 0.0))
        return set_err(MCSBR_EINVAL, "build_strata: reference wavelength must be > 0");
    const double target = lambda_ref / spw;
    out->nu = std::max(1, static_cast<int>(std::ceil(2.0 * out->half_u / target)));
    out->nv = std::max(1, static_cast<int>(std::ceil(2.0 * out->half_v / target)));
    const double area = 4.0 * out->half_u * out->half_v;
    out->cell_area = area / (static_cast<double>(out->nu) * out->nv);
    const uint64_t cells = static_cast<uint64_t>(out->nu) * static_cast<uint64_t>(out->nv);
    if (cells >= (uint64_t{1} << 32))  // the device keys cells in 32 bits
        return set_err(MCSBR_EINVAL, "build_strata: more than 2^32 strata per incidence");
    out->entries = cells * static_cast<uint64_t>(spp);
    return MCSBR_OK;
}

// one incidence
int plan(const mcsbr_scene* s, const double k_inc[3], double padding, double spw, double lambda_ref, int32_t spp,
         mcsbr_launch_plan* out) {
    V k, u, v;
    plan_axes(k_inc, &k, &u, &v);
    std::vector<double> ext;
    int rc = plan_extents(s, {u.x, u.y, u.z, v.x, v.y, v.z}, &ext);
    if (rc) return rc;
    return plan_finish(s, k, u, v, ext.data(), padding, spw, lambda_ref, spp, out);
}

int validate(const mcsbr_mc_config* c) {
    if (!c) return set_err(MCSBR_EINVAL, "mc: null config");
    if (!(c->strata_per_wavelength > 0.0)) return set_err(MCSBR_EINVAL, "mc: strata_per_wavelength must be > 0");
    if (c->samples_per_stratum < 1) return set_err(MCSBR_EINVAL, "mc: samples_per_stratum must be >= 1");
    if (!(c->roulette_q > 0.0 && c->roulette_q < 1.0)) return set_err(MCSBR_EINVAL, "mc: roulette q must be in (0,1)");
    if (c->roulette_min_bounce < 1) return set_err(MCSBR_EINVAL, "mc: roulette min_bounce must be >= 1");
    if (c->max_bounce < 2) return set_err(MCSBR_EINVAL, "mc: max_bounce must be >= 2");
    if (c->block_size < 1) return set_err(MCSBR_EINVAL, "mc: block_size must be >= 1");
    if (c->max_bounce > MCSBR_MAX_BOUNCE_LIMIT)
        return set_err(MCSBR_EINVAL, "mc: max_bounce exceeds MCSBR_MAX_BOUNCE_LIMIT (64)");
    if (c->rng_mode != MCSBR_RNG_REFERENCE && c->rng_mode != MCSBR_RNG_PHILOX)
        return set_err(MCSBR_EINVAL, "mc: unknown rng_mode");
    if (c->reduction != MCSBR_REDUCE_FAST && c->reduction != MCSBR_REDUCE_EXACT)
        return set_err(MCSBR_EINVAL, "mc: unknown reduction");
    if (c->parity_fp64_refine != 0 && c->parity_fp64_refine != 1)
        return set_err(MCSBR_EINVAL, "mc: parity_fp64_refine must be 0 or 1");
    if (c->parity_fp64_refine == 0 && c->rng_mode != MCSBR_RNG_PHILOX)
        return set_err(MCSBR_EINVAL, "mc: parity_fp64_refine = 0 (fp32 triangle tests) is a statistical-mode "
                                     "option: it needs rng_mode PHILOX");
    return MCSBR_OK;
}

// DetConfig::validate (solver_det.cpp:11-17)
int validate_det(const mcsbr_det_config* c) {
    if (!c) return set_err(MCSBR_EINVAL, "det: null config");
    if (!(c->rays_per_wavelength > 0.0)) return set_err(MCSBR_EINVAL, "det: rays_per_wavelength must be > 0");
    if (c->max_bounce < 1) return set_err(MCSBR_EINVAL, "det: max_bounce must be >= 1");
    if (c->amplitude_cutoff < 0.0) return set_err(MCSBR_EINVAL, "det: amplitude_cutoff must be >= 0");
    if (c->block_size < 1) return set_err(MCSBR_EINVAL, "det: block_size must be >= 1");
    if (c->max_bounce > MCSBR_MAX_BOUNCE_LIMIT)
        return set_err(MCSBR_EINVAL, "det: max_bounce exceeds MCSBR_MAX_BOUNCE_LIMIT (64)");
    return MCSBR_OK;
}

// The deterministic solver runs the path engine with this McConfig: one
// midpoint sample per cell (sample_stratum(..., jitter=false),
// solver_det.cpp:72-74), no roulette, the det grid density and bounce cap.
mcsbr_mc_config det_as_mc(const mcsbr_det_config* d) {
    mcsbr_mc_config c;
    mcsbr_gpu_default_config(&c);
    c.strata_per_wavelength = d->rays_per_wavelength;
    c.samples_per_stratum = 1;
    c.roulette_enabled = 0;
    c.max_bounce = d->max_bounce;
    c.jitter = 0;
    c.seed = 0;
    c.reference_wavelength = d->reference_wavelength;
    c.launch_padding = d->launch_padding;
    c.block_size = d->block_size;
    c.reduction = MCSBR_REDUCE_EXACT;  // deterministic solver, reproducible sums (any F, any grouping)
    return c;
}

uint32_t env_u32(const char* name, uint32_t dflt) {
    const char* v = std::getenv(name);
    return v && *v ? static_cast<uint32_t>(std::strtoul(v, nullptr, 10)) : dflt;
}

constexpr uint64_t kPathStateBytes = 192;
// contribution records (96 B each): at most 2^29 (51.5 GB) and a third of
// the device's memory.  c5's sweep (~242 M records) then runs as ONE launch
// group: device -0.5%, e2e -2.1% against 2^28 (two groups), same box
uint64_t rec_cap_max() {
    static const uint64_t cap = [] {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
            cudaGetLastError();
            return uint64_t{1} << 28;
        }
        return std::max<uint64_t>(uint64_t{1} << 24, std::min<uint64_t>(uint64_t{1} << 29, total_b / 3 / 96));
    }();
    return cap;
}
constexpr uint64_t kCoverBudgetWords = uint64_t{1} << 26;  // coverage bitmaps: at most 256 MB per job

// Fold the peak record count of the scene's previous F > 1 job (if its
// readback has landed) into the records-per-entry estimate.
void learn_rec_ratio(mcsbr_scene* s) {
    if (!s->peak_host) {
        if (pinned_slot(&s->peak_host) != cudaSuccess) {
            s->peak_host = nullptr;
            return;
        }
        if (cudaEventCreateWithFlags(&s->peak_ev, cudaEventDisableTiming) != cudaSuccess) {
            pinned_release(s->peak_host);
            s->peak_host = nullptr;
            return;
        }
    }
    if (!s->peak_pending || cudaEventQuery(s->peak_ev) != cudaSuccess) return;
    s->peak_pending = false;
    if (s->peak_entries == 0) return;
    const double seen = static_cast<double>(*s->peak_host) / static_cast<double>(s->peak_entries);
    s->rec_ratio = std::min(std::max(seen * 1.25, 1.0 / 64.0), 8.0);
    rec_ratio_hint().store(s->rec_ratio, std::memory_order_relaxed);
}  // sizeof(mcsbr::PathState), path_engine.hpp:16-28

struct Job {
    std::vector<IncDev> inc;      // launch units, incidence-major (IncDev::row set per group)
    std::vector<uint32_t> unit0;  // [n_inc + 1]: first unit of each incidence
    uint32_t n_inc = 0;
    std::vector<RxDev> rx;
    std::vector<double> k0;
    uint32_t n_rx = 1;
    uint64_t total_entries = 0;
    // launch groups: incidences [a0, a1) = units [u0, u1); IncDev::g_begin
    // restarts at 0 in each.  F > 1 jobs are split into groups of <=
    // kGroupEntries entries so a launch's contribution records fit the
    // record buffer.
    struct Group {
        uint32_t a0, a1, u0, u1;
        uint64_t entries;
    };
    std::vector<Group> groups;
    uint64_t max_group_entries = 0;
    int uniform_f = 0;
    double kph0 = 0.0, kdph = 0.0;
};

// Plan all incidences of a batch for one shard.
int plan_job(const mcsbr_scene* s, const mcsbr_incidence* incs, uint32_t n_inc,
             const mcsbr_receiver* rxs, uint32_t n_rx, const double* freqs, uint32_t nf,
             const mcsbr_mc_config* cfg, uint32_t shard, uint32_t nshard, int warps_hint, Job* job,
             bool det = false) {
    int rc = det ? MCSBR_OK : validate(cfg);  // det: validated as DetConfig by the caller
    if (rc) return rc;
    if (nf == 0 || !freqs) return set_err(MCSBR_EINVAL, "estimate: empty frequency list");
    if (n_inc == 0) return set_err(MCSBR_EINVAL, "estimate: no incidences");
    if (n_rx == 0 || !rxs) return set_err(MCSBR_EINVAL, "estimate: no receivers");
    if (nshard == 0 || shard >= nshard) return set_err(MCSBR_EINVAL, "estimate: bad shard");
    double lambda_ref = cfg->reference_wavelength;
    if (lambda_ref <= 0.0) lambda_ref = kC / freqs[nf - 1];
    job->inc.clear();
    job->unit0.assign(n_inc + 1, 0);
    job->n_inc = n_inc;
    job->rx.resize(static_cast<size_t>(n_inc) * n_rx);
    job->n_rx = n_rx;
    job->k0.resize(nf);
    for (uint32_t f = 0; f < nf; ++f) job->k0[f] = 2.0 * kPi * freqs[f] / kC;
    uint64_t total = 0;
    // launch rectangles: the axes on the host, the O(vertices) projection
    // extents of every incidence in one device pass (prep.cu)
    std::vector<mcsbr_launch_plan> plans(n_inc);
    std::vector<int> prc(n_inc, MCSBR_OK);
    {
        std::vector<V> ks(n_inc), us(n_inc), vs(n_inc);
        std::vector<double> axes(6ull * n_inc);
        for (uint32_t a = 0; a < n_inc; ++a) {
            plan_axes(incs[a].k_inc, &ks[a], &us[a], &vs[a]);
            const double ax[6] = {us[a].x, us[a].y, us[a].z, vs[a].x, vs[a].y, vs[a].z};
            std::memcpy(&axes[6ull * a], ax, sizeof(ax));
        }
        std::vector<double> ext;
        int erc = plan_extents(s, axes, &ext);
        if (erc) return erc;
        for (uint32_t a = 0; a < n_inc; ++a) {
            const double spw_a = incs[a].strata_per_wavelength > 0.0 ? incs[a].strata_per_wavelength
                                                                       : cfg->strata_per_wavelength;
            prc[a] = plan_finish(s, ks[a], us[a], vs[a], &ext[4ull * a], cfg->launch_padding, spw_a, lambda_ref,
                                 cfg->samples_per_stratum, &plans[a]);
            if (prc[a]) return prc[a];
        }
    }
    for (uint32_t a = 0; a < n_inc; ++a) {
        const mcsbr_incidence& in = incs[a];
        mcsbr_launch_plan lp = plans[a];
        if (lp.entries == 0) return set_err(MCSBR_EINVAL, "estimate: empty strata grid");
        IncDev d;
        std::memset(&d, 0, sizeof(d));
        std::memcpy(d.center, lp.center, sizeof(d.center));
        std::memcpy(d.u, lp.u_axis, sizeof(d.u));
        std::memcpy(d.v, lp.v_axis, sizeof(d.v));
        d.half_u = lp.half_u;
        d.half_v = lp.half_v;
        std::memcpy(d.k_inc, in.k_inc, sizeof(d.k_inc));
        std::memcpy(d.pol_v, in.pol_v, sizeof(d.pol_v));
        std::memcpy(d.pol_h, in.pol_h, sizeof(d.pol_h));
        d.area_weight = lp.cell_area / static_cast<double>(static_cast<uint64_t>(cfg->samples_per_stratum));
        d.nu = lp.nu;
        d.nv = lp.nv;
        // Shards: the incidence's dispatch indices in stripes of S, stripe k
        // to shard k mod nshard (about 32 stripes per shard), so every shard
        // samples the whole aperture.  Contiguous shards put all of an
        // airframe's silhouette on the middle ranks: c5 at 8 shards ran its
        // slowest shard 2.1x the mean (tools/shard_balance.py).  Every entry
        // keeps its dispatch index, RNG key and contribution.
        job->unit0[a] = static_cast<uint32_t>(job->inc.size());
        if (nshard == 1) {
            d.entry_begin = 0;
            d.entry_end = lp.entries;
            job->inc.push_back(d);
            total += lp.entries;
        } else {
            uint64_t S = (lp.entries + 32ull * nshard - 1) / (32ull * nshard);
            S = std::max<uint64_t>(1024, (S + 1023) / 1024 * 1024);
            const uint64_t stripes = (lp.entries + S - 1) / S;
            for (uint64_t k = shard; k < stripes; k += nshard) {
                d.entry_begin = k * S;
                d.entry_end = std::min(lp.entries, (k + 1) * S);
                job->inc.push_back(d);
                total += d.entry_end - d.entry_begin;
            }
        }
        for (uint32_t r = 0; r < n_rx; ++r) {
            RxDev& x = job->rx[static_cast<size_t>(a) * n_rx + r];
            const mcsbr_receiver& y = rxs[static_cast<size_t>(a) * n_rx + r];
            std::memcpy(x.k_s, y.k_scatter, sizeof(x.k_s));
            std::memcpy(x.rx_v, y.rx_v, sizeof(x.rx_v));
            std::memcpy(x.rx_h, y.rx_h, sizeof(x.rx_h));
        }
    }
    job->unit0[n_inc] = static_cast<uint32_t>(job->inc.size());
    job->total_entries = total;
    // F > 1: the launch groups are sized so their records fit rec_cap_max()
    uint64_t group_cap = ~uint64_t{0};
    if (nf > 1) {
        learn_rec_ratio(const_cast<mcsbr_scene*>(s));
        // (a multi-frequency fan appends up to one record per receiver of its chunk)
        const double fan_mult = n_rx > 1 ? static_cast<double>(std::min<uint32_t>(n_rx, 32)) : 1.0;
        group_cap = std::max<uint64_t>(static_cast<uint64_t>(static_cast<double>(rec_cap_max()) / (s->rec_ratio * fan_mult)),
                                       uint64_t{1} << 20);
        group_cap = env_u32("MCSBR_GROUP_ENTRIES", static_cast<uint32_t>(std::min<uint64_t>(group_cap, 0xffffffffu)));
    }
    job->groups.clear();
    job->max_group_entries = 0;
    uint64_t g = 0;
    uint32_t a0 = 0;
    for (uint32_t a = 0; a < n_inc; ++a) {
        uint64_t e = 0;
        for (uint32_t u = job->unit0[a]; u < job->unit0[a + 1]; ++u)
            e += job->inc[u].entry_end - job->inc[u].entry_begin;
        if (a > a0 && g + e > group_cap) {
            job->groups.push_back({a0, a, job->unit0[a0], job->unit0[a], g});
            job->max_group_entries = std::max(job->max_group_entries, g);
            a0 = a;
            g = 0;
        }
        for (uint32_t u = job->unit0[a]; u < job->unit0[a + 1]; ++u) {
            IncDev& d = job->inc[u];
            d.g_begin = g;
            d.row = a - a0;
            g += d.entry_end - d.entry_begin;
        }
    }
    job->groups.push_back({a0, n_inc, job->unit0[a0], job->unit0[n_inc], g});
    job->max_group_entries = std::max(job->max_group_entries, g);
    // uniform grid test of SweepAccumulator (farfield.cpp:87-104)
    job->uniform_f = 0;
    if (nf >= 2) {
        const double df = freqs[1] - freqs[0];
        bool uni = true;
        for (uint32_t i = 1; i < nf; ++i)
            if (std::abs((freqs[i] - freqs[i - 1]) - df) > 1e-6 * std::abs(df)) {
                uni = false;
                break;
            }
        job->uniform_f = uni ? 1 : 0;
        job->kph0 = -2.0 * kPi * freqs[0] / kC;
        job->kdph = -2.0 * kPi * df / kC;
    }
    return MCSBR_OK;
}

void fill_config(TraceParams& p, const mcsbr_mc_config* cfg) {
    p.spp = static_cast<uint32_t>(cfg->samples_per_stratum);
    p.seed = cfg->seed;
    p.max_bounce = cfg->max_bounce;
    p.fresnel_strategy = cfg->branch_strategy == MCSBR_BRANCH_FRESNEL;
    p.p_min = cfg->p_min;
    p.roulette_enabled = cfg->roulette_enabled != 0;
    p.roulette_min_bounce = cfg->roulette_min_bounce;
    p.roulette_q = cfg->roulette_q;
    p.jitter = cfg->jitter != 0;
    p.rng_mode = cfg->rng_mode;
    p.fast_tri = cfg->parity_fp64_refine == 0 ? 1 : 0;
}

// One launch group through the wavefront kernels: shade + trace per
// iteration until the shading pass leaves no query (every path finished and
// every launch entry taken).  The work-list length is read back every
// kWfCheck iterations; the iterations in between that find no work return at
// once.
int run_wavefront(mcsbr_scene* s, const TraceParams& p, const WfParams& w, cudaStream_t stream) {
    constexpr uint32_t kWfCheck = 8;
    constexpr uint32_t kWfMaxIters = 1u << 20;
    CK(cudaMemsetAsync(w.kind, 0, sizeof(uint32_t) * w.np, stream), "memset path pool");
    CK(cudaMemsetAsync(w.list_n, 0, sizeof(unsigned long long) * (6 + 2ull * (w.np / 32)), stream),
       "memset path pool");
    for (uint32_t it = 0; it < kWfMaxIters; ++it) {
        CK(launch_wavefront_iteration(p, w, it, s->sms, stream), "wavefront launch");
        g_launches += 2;
        if (it % kWfCheck == kWfCheck - 1) {
            CK(cudaMemcpyAsync(s->wf_host, w.list_n + it % 3, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                               stream), "work-list readback");
            CK(cudaEventRecord(s->wf_ev, stream), "cudaEventRecord");
            CK(cudaEventSynchronize(s->wf_ev), "cudaEventSynchronize");
            if (*s->wf_host == 0) return MCSBR_OK;
        }
    }
    return set_err(MCSBR_EDEVICE, "wavefront: iteration limit reached");
}

// MCSBR_RECSTATS (diagnostic): statistics of one launch's contribution
// records on stderr -- count, real-amplitude and complex-path fractions, and
// the distribution of the attenuation per frequency step |kdph * Im s| in
// units of 2 pi / (2 nf) (a sample of every 16th record)
static void record_stats(mcsbr_scene* s, const TraceParams& p, cudaStream_t stream) {
    unsigned long long n = 0;
    cudaMemcpyAsync(&n, p.rec_count, sizeof(n), cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    n = std::min<unsigned long long>(n, p.rec_cap);
    const uint64_t stride = 16, m = n / stride;
    std::vector<double> v(12 * m);
    if (m) cudaMemcpy2DAsync(v.data(), 12 * sizeof(double), s->recs.p, stride * 12 * sizeof(double),
                             12 * sizeof(double), m, cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    uint64_t real_amp = 0, cplx_s = 0, hist[8] = {};
    double smin = 1e300, smax = -1e300;
    const double h = 2.0 * 3.141592653589793 / (2.0 * p.nf);
    for (uint64_t i = 0; i < m; ++i) {
        const double* r = v.data() + 12 * i;
        if (r[1] == 0 && r[3] == 0 && r[5] == 0 && r[7] == 0) ++real_amp;
        smin = std::min(smin, r[8]);
        smax = std::max(smax, r[8]);
        if (r[9] != 0) {
            ++cplx_s;
            const double eta = std::fabs(p.kdph * r[9]) / h;
            int b = 0;
            for (double t = 1e-4; b < 7 && eta > t; t *= 4) ++b;
            ++hist[b];
        }
    }
    std::fprintf(stderr,
                 "[recstats] records %llu sample %llu real_amp %.4f complex_s %.4f s [%.4g, %.4g] kdph %.4g "
                 "eta(<1e-4,4e-4,1.6e-3,6.4e-3,.0256,.1024,.41,>) %llu %llu %llu %llu %llu %llu %llu %llu\n",
                 n, static_cast<unsigned long long>(m), m ? double(real_amp) / m : 0.0,
                 m ? double(cplx_s) / m : 0.0, smin, smax, p.kdph, (unsigned long long)hist[0],
                 (unsigned long long)hist[1], (unsigned long long)hist[2], (unsigned long long)hist[3],
                 (unsigned long long)hist[4], (unsigned long long)hist[5], (unsigned long long)hist[6],
                 (unsigned long long)hist[7]);
}

// Upload a planned job and run the path kernel(s) on s->stream, adding into
// d_sums / d_counters.  One launch per receiver index (receivers of one
// incidence share nothing but the geometry).
int run_job(mcsbr_scene* s, const Job& job, uint32_t nf, const mcsbr_mc_config* cfg, int occlusion,
            double* d_sums, unsigned long long* d_counters, cudaStream_t stream, TraceParams* extra,
            float* kernel_ms, long long* d_limbs = nullptr) {
    // MCSBR_REDUCE_EXACT (fixedpoint.cuh): every F goes through the records
    // and the integer accumulate kernel, receivers are traced one by one
    // (no fan), and the 192-bit sums are ADDED as limbs into d_limbs
    const bool exact = cfg->reduction == MCSBR_REDUCE_EXACT;
    if (exact && !d_limbs) return set_err(MCSBR_EINVAL, "exact reduction: no limb buffer");
    const uint64_t n_values = static_cast<uint64_t>(job.n_inc) * job.n_rx * nf * 8;
    if (exact) {
        CK(s->xsums.reserve(3 * n_values), "dev_malloc(exact sums)");
        CK(cudaMemsetAsync(s->xsums.p, 0, sizeof(unsigned long long) * 3 * n_values, stream), "memset exact sums");
    }
    // the launch units, then one unit per incidence for the coverage kernel
    const size_t n_units = job.inc.size();
    CK(s->inc.reserve(n_units + job.n_inc), "dev_malloc(incidences)");
    CK(s->rx.reserve(job.rx.size()), "dev_malloc(receivers)");
    CK(s->k0.reserve(nf), "dev_malloc(k0)");
    CK(s->tile.reserve(3), "dev_malloc(tile counter)");  // entry cursor, record count, peak count
    // deferred accumulation (F > 1): one 96-byte record per visible
    // contribution; sized for one per launched path of the largest group
    // (measured c4/c5: ~0.1 per path), overflow falls back to direct atomics
    const bool defer = nf > 1 || exact;
    // Bistatic fans (several receivers per incidence): trace once per chunk
    // of 32 receivers, lane l evaluating receiver l's occlusion and
    // projection.  F = 1 sums in the lanes' registers; F > 1 appends one
    // record per visible (contribution, receiver), in row 32 a + l of the
    // accumulation (fan_rows).  The exact reduction traces receivers one by
    // one.
    // F > 1 fans need the NUFFT's row buckets: its spread (and the direct
    // kernel) flush their sums whenever consecutive records change row, and
    // a fan's consecutive records are different receivers
    const char* acc_env = std::getenv("MCSBR_ACC");
    const bool acc_direct = acc_env && std::strcmp(acc_env, "direct") == 0;
    uint32_t max_group_inc = 1;
    for (const Job::Group& gr : job.groups) max_group_inc = std::max(max_group_inc, gr.a1 - gr.a0);
    const bool rows_bucketed = !exact && job.uniform_f && nufft_supported(nf) && !acc_direct &&
                               env_u32("MCSBR_NUFFT_SORT", 1) != 0 && max_group_inc * 32u <= kNufftSortMaxInc;
    const bool fan = job.n_rx > 1 && trace_fan_supported(nf) && !exact && !(extra && extra->det) &&
                     (nf == 1 || rows_bucketed) &&
                     env_u32("MCSBR_FAN", 1) != 0;  // (A/B: MCSBR_FAN=0 traces per receiver)
    const uint32_t fan_rows = fan && nf > 1 ? 32u : 0u;
    const uint32_t rows_per_inc = fan_rows ? fan_rows : 1u;  // accumulation rows per incidence
    uint64_t rec_cap = 0;
    if (defer) {
        rec_cap = static_cast<uint64_t>(static_cast<double>(job.max_group_entries) * s->rec_ratio * 1.1 *
                                        (fan_rows ? std::min<uint32_t>(job.n_rx, fan_rows) : 1u)) +
                  4096;
        rec_cap = std::min<uint64_t>(rec_cap, rec_cap_max());
        rec_cap = env_u32("MCSBR_REC_CAP", static_cast<uint32_t>(rec_cap));
        CK(s->recs.reserve(rec_cap * 12), "dev_malloc(contribution records)");
    }
    // launch-ray coverage bitmaps (cover.cu): every incidence of the job,
    // up to kCoverBudget words in total (later incidences go unculled); the
    // deterministic solver's per-root stack accounting needs every root ray,
    // so its jobs are not culled
    // uniform frequency grids: accumulation as a non-uniform DFT (spread.cu);
    // MCSBR_ACC=direct keeps the per-frequency phasor kernel (A/B)
    NufftPlan nq{};
    const bool nufft = defer && !exact && job.uniform_f && nufft_supported(nf) && !acc_direct;
    if (nufft) {
        nq.ng = 2 * nf;
        nq.fc = nf / 2;
        nq.beta = 2.30 * 16;
        nq.kc = job.kph0 + static_cast<double>(nq.fc) * job.kdph;
        nq.u2t = job.kdph * static_cast<double>(nq.ng) / (2.0 * M_PI);
        const char* em = std::getenv("MCSBR_NUFFT_ETA_MAX");  // tests: force the direct fallback
        nq.eta_max = em ? std::strtod(em, nullptr) : 0.5;
        const char* ep = std::getenv("MCSBR_NUFFT_ETA_POLY");  // tests: force the exact continuation
        nq.eta_poly = std::min(nq.eta_max, ep ? std::strtod(ep, nullptr) : 0.1);
        uint32_t max_inc = 1;
        for (const Job::Group& gr : job.groups) max_inc = std::max(max_inc, (gr.a1 - gr.a0) * rows_per_inc);
        CK(s->nufft_grid.reserve(nufft_grid_values(nf) * max_inc), "dev_malloc(nufft grids)");
        if (s->nufft_hat_nf != nf) {  // pageable source: the call returns once it is staged
            std::vector<double> hat, coef;
            nufft_tables(nf, nq.ng, nq.beta, hat, coef);
            hat.insert(hat.end(), coef.begin(), coef.end());
            CK(s->nufft_hat.reserve(hat.size()), "dev_malloc(nufft weights)");
            CK(cudaMemcpyAsync(s->nufft_hat.p, hat.data(), sizeof(double) * hat.size(), cudaMemcpyHostToDevice,
                               stream), "upload nufft weights");
            s->nufft_hat_nf = nf;
        }
        CK(s->nufft_idx.reserve(rec_cap), "dev_malloc(nufft record order)");
        CK(s->nufft_bucket.reserve(2ull * (max_inc + 1)), "dev_malloc(nufft buckets)");
        nq.coef = s->nufft_hat.p + nf;
        nq.idx = env_u32("MCSBR_NUFFT_SORT", 1) ? s->nufft_idx.p : nullptr;
        if (nq.idx) CK(s->nufft_inc.reserve(rec_cap), "dev_malloc(record incidences)");
        nq.bucket = s->nufft_bucket.p;
        nq.grid = s->nufft_grid.p;
        nq.inv_hat = s->nufft_hat.p;
    }
    std::vector<IncDev> incs = job.inc;
    incs.resize(n_units + job.n_inc);
    const bool det_job = extra && extra->det;
    // only the deferred-accumulation kernels cull (trace.cu kCull)
    const bool cull = !det_job && (nf > 1 || exact) && !fan && env_u32("MCSBR_COVER", 1) != 0;
    uint64_t cover_words = 0;
    uint32_t n_cover = 0;  // incidences with a bitmap (the coverage kernel's blocks)
    for (uint32_t a = 0; a < job.n_inc; ++a) {
        uint64_t off = kNoCover;
        uint32_t sh = 0;
        const uint32_t u0 = job.unit0[a], u1 = job.unit0[a + 1];
        if (cull && u1 > u0) {
            const IncDev& d = incs[u0];
            const uint64_t entries = static_cast<uint64_t>(d.nu) * static_cast<uint64_t>(d.nv) *
                                     static_cast<uint64_t>(cfg->samples_per_stratum);
            sh = cover_shift_for(entries);
            const uint64_t words = (((entries + (uint64_t{1} << sh) - 1) >> sh) + 31) / 32;
            if (cover_words + words <= kCoverBudgetWords) {
                off = cover_words;
                cover_words += words;
            } else {
                sh = 0;
            }
        }
        for (uint32_t u = u0; u < u1; ++u) {  // every stripe shares the incidence's bitmap
            incs[u].cover_off = off;
            incs[u].cover_shift = sh;
        }
        if (off != kNoCover) incs[n_units + n_cover++] = incs[u0];
    }
    if (cover_words) CK(s->cover.reserve(cover_words), "dev_malloc(coverage bitmaps)");
    CK(cudaMemcpyAsync(s->inc.p, incs.data(), sizeof(IncDev) * (n_units + n_cover), cudaMemcpyHostToDevice,
                       stream), "upload incidences");
    CK(cudaMemcpyAsync(s->rx.p, job.rx.data(), sizeof(RxDev) * job.rx.size(), cudaMemcpyHostToDevice, stream),
       "upload receivers");
    CK(cudaMemcpyAsync(s->k0.p, job.k0.data(), sizeof(double) * nf, cudaMemcpyHostToDevice, stream),
       "upload wavenumbers");
    // statistical-mode fast path: fp32 leaf records (prep.cu), once per scene
    if (cfg->parity_fp64_refine == 0 && !(extra && extra->det) && !s->leaf32.n) {
        CK(s->leaf32.reserve(3ull * s->bvh.n_leaves), "dev_malloc(fp32 triangles)");
        CK(launch_leaf32(s->bvh.tri64, s->bvh.n_leaves, s->center, s->radius, s->leaf32.p, stream), "fp32 triangles launch");
        ++g_launches;
    }
    TraceParams p = extra ? *extra : TraceParams{};
    p.scene = s->view();
    p.cover = cover_words ? s->cover.p : nullptr;
    p.n_rx = job.n_rx;
    p.k0 = s->k0.p;
    p.nf = nf;
    p.occlusion = occlusion;
    p.counters = d_counters;
    p.tile_counter = s->tile.p;
    p.recs = defer ? s->recs.p : nullptr;
    p.rec_count = s->tile.p + 1;
    p.rec_cap = rec_cap;
    p.rec_inc = nufft && nq.idx ? s->nufft_inc.p : nullptr;
    // scheduling knobs (A/B experiments only; the defaults are the product)
    // Chunk cap: large scenes keep every SM's warps inside a narrow window of
    // the aperture (their BVH working set outgrows L1/L2: c4 -35% going from
    // 4096 to 256); a small scene's BVH stays cache-resident whatever the
    // window, and fewer, longer chunks there save the per-chunk scheduling
    // and incidence changes (c2 -2.7% at 1024, -3.3% at 2048; c4 +4% at 512).
    // (A/B knobs sanitised: chunk sizes non-zero multiples of 32, min <= max)
    // Measured (r02, same box): c5 (1 M triangles) 256 -> 512: path kernel
    // -2.2% (lossy) / -2.3% (lossless twin), accumulation unchanged; 1024:
    // +0.7% while the sweep ran as two launch groups, -0.5% since it runs as
    // one (446.9 vs 448.8 ms, 2048: 448.7; tools/ab_c5_knobs.sh); c4 (200 k)
    // 256 -> 512: +8%.
    const uint32_t cap_default = s->nt <= kSmallSceneTris ? 2048u : (s->nt <= kLargeSceneTris ? 256u : 1024u);
    p.chunk_max = std::max(32u, env_u32("MCSBR_CHUNK_MAX", cap_default) / 32u * 32u);
    p.chunk_min = std::min(p.chunk_max, std::max(32u, env_u32("MCSBR_CHUNK_MIN", 32) / 32u * 32u));
    // guided-scheduling divisor: chunk = remaining / (gss_div * warps).  Above
    // 512 k triangles 32 with 16-row bands (below): c5 as one launch group
    // 447.3 / 446.4 -> 442.8 / 444.1 ms (two alternations, same box)
    p.gss_div = env_u32("MCSBR_GSS", s->nt > kLargeSceneTris ? 32u : 16u);
    // band height of the launch-entry dispatch order (0 = linear; a power of two)
    {
        // 8-row bands above 512 k triangles: c5 path kernel -1.6% (its
        // accumulation +3.8%: the records come out less ordered), 4 below
        // (c4 +41% at 8); 16 rows (with gss 32) once c5 ran as one group
        const uint32_t bh = env_u32("MCSBR_BAND", s->nt > kLargeSceneTris ? 16u : 4u);
        p.band_order = static_cast<int32_t>(bh & (bh - 1) ? 4 : bh);
    }
    p.uniform_f = job.uniform_f;
    p.kph0 = job.kph0;
    p.kdph = job.kdph;
    fill_config(p, cfg);
    if (kernel_ms && !s->ev0) {
        CK(cudaEventCreate(&s->ev0), "cudaEventCreate");
        CK(cudaEventCreate(&s->ev1), "cudaEventCreate");
    }
    if (kernel_ms) CK(cudaEventRecord(s->ev0, stream), "cudaEventRecord");
    // fans: one launch per chunk of 32 receivers; otherwise one per receiver
    const uint32_t step = fan ? 32u : 1u;
    p.fan = fan ? 1 : 0;
    p.fan_rows = fan_rows;
    if (defer) CK(cudaMemsetAsync(s->tile.p + 2, 0, sizeof(unsigned long long), stream), "reset peak");
    if (cover_words) {
        CK(launch_cover(s->inc.p + n_units, n_cover, s->d_tri32, s->nt, s->center, s->radius,
                        p.spp, static_cast<uint32_t>(p.band_order), s->cover.p, cover_words, s->sms, stream),
           "coverage kernel launch");
        ++g_launches;
    }
    // Wavefront (wavefront.cu) for the deferred-accumulation Monte Carlo
    // mode without parity instrumentation; the megakernel otherwise.
    const bool wavefront = defer && !fan && !p.det && !p.contrib_out && !p.plog_tri &&
                           env_u32("MCSBR_WAVEFRONT", 0) != 0;
    WfParams w{};
    if (wavefront) {
        const uint32_t np = static_cast<uint32_t>(s->sms) * env_u32("MCSBR_WF_SLOTS_PER_SM", 4096);
        w.np = (np + 127) / 128 * 128;
        CK(s->wf_pool.reserve(static_cast<size_t>(kWfFieldsHost) * w.np), "dev_malloc(path pool)");
        CK(s->wf_u32.reserve(3ull * w.np), "dev_malloc(path pool)");
        CK(s->wf_ctl.reserve(6 + 2ull * (w.np / 32)), "dev_malloc(path pool)");
        if (!s->wf_host) {
            CK(pinned_slot(&s->wf_host), "cudaMallocHost");
            CK(cudaEventCreateWithFlags(&s->wf_ev, cudaEventDisableTiming), "cudaEventCreate");
        }
        w.pool = s->wf_pool.p;
        w.kind = s->wf_u32.p;
        w.rid = s->wf_u32.p + w.np;
        w.list = s->wf_u32.p + 2ull * w.np;
        w.list_n = s->wf_ctl.p;
        w.trace_cursor = s->wf_ctl.p + 3;
        w.wrange = s->wf_ctl.p + 6;
    }
    for (uint32_t r = 0; r < job.n_rx; r += step) {
        p.rx_index = r;
        for (const Job::Group& gr : job.groups) {
            if (gr.entries == 0) continue;  // no entries of this shard in the group
            p.inc = s->inc.p + gr.u0;
            p.n_inc = gr.u1 - gr.u0;
            p.inc_base = gr.a0;
            p.rx = s->rx.p + static_cast<size_t>(gr.a0) * job.n_rx;
            p.sums = d_sums + static_cast<size_t>(gr.a0) * job.n_rx * nf * 8;
            p.xsums = exact ? s->xsums.p + 3ull * gr.a0 * job.n_rx * nf * 8 : nullptr;
            p.total_entries = gr.entries;
            CK(cudaMemsetAsync(s->tile.p, 0, 2 * sizeof(unsigned long long), stream), "reset tile counter");
            CK(kt_mark(0, stream, s->device, false), "cudaEventRecord");
            if (wavefront) {
                int rc = run_wavefront(s, p, w, stream);
                if (rc) return rc;
            } else {
                CK(launch_trace(p, s->sms, stream, &g_launches), "path kernel launch");
            }
            CK(kt_mark(0, stream, s->device, true), "cudaEventRecord");
            if (defer && std::getenv("MCSBR_RECSTATS")) record_stats(s, p, stream);
            if (defer) {
                CK(kt_mark(1, stream, s->device, false), "cudaEventRecord");
                const uint64_t expected = static_cast<uint64_t>(static_cast<double>(gr.entries) * s->rec_ratio / 1.25);
                if (nufft)
                    CK(launch_spread(p, nq, (gr.a1 - gr.a0) * rows_per_inc, s->sms, stream, &g_launches, expected),
                       "spread launch");
                else
                    CK(launch_accumulate(p, s->sms, stream, &g_launches, expected), "accumulate launch");
                CK(kt_mark(1, stream, s->device, true), "cudaEventRecord");
            }
        }
    }
    if (exact) {
        CK(launch_exact_limbs(s->xsums.p, n_values, d_limbs, stream), "exact limbs launch");
        ++g_launches;
    }
    if (defer && s->peak_host) {  // learn the record ratio (per entry and receiver row) for the next job
        CK(cudaMemcpyAsync(s->peak_host, s->tile.p + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           stream), "peak record count");
        CK(cudaEventRecord(s->peak_ev, stream), "cudaEventRecord");
        s->peak_entries = job.max_group_entries * (fan_rows ? std::min<uint32_t>(job.n_rx, fan_rows) : 1u);
        s->peak_pending = true;
    }
    if (kernel_ms) {
        CK(cudaEventRecord(s->ev1, stream), "cudaEventRecord");
        CK(cudaEventSynchronize(s->ev1), "cudaEventSynchronize");
        CK(cudaEventElapsedTime(kernel_ms, s->ev0, s->ev1), "cudaEventElapsedTime");
    }
    return MCSBR_OK;
}

void decode(const unsigned long long* c, mcsbr_stats* st) {
    std::memset(st, 0, sizeof(*st));
    st->rays_launched = c[kCntLaunched];
    st->contributions = c[kCntContrib];
    st->grazing_kills = c[kCntGrazing];
    st->cap_kills = c[kCntCap];
    st->occlusion_queries = c[kCntOcclusion];
    st->culled_launch_rays = c[kCntCulled];
    uint32_t rounds = 0;
    uint64_t seg = 0;
    for (int i = 0; i < MCSBR_MAX_BOUNCE_LIMIT; ++i) {
        st->rays_per_bounce[i] = c[kCntRaysPerBounce + i];
        st->roulette_candidates[i] = c[kCntRouletteCand + i];
        st->roulette_survivors[i] = c[kCntRouletteSurv + i];
        seg += st->rays_per_bounce[i];
        if (st->rays_per_bounce[i]) rounds = static_cast<uint32_t>(i + 1);
    }
    st->segments_traced = seg;
    st->n_rounds = rounds;
    st->state_bytes_per_ray = 208;  // registers of one in-flight path (Path + hit temporaries)
}

int fault_check(const unsigned long long* c) {
    const unsigned long long f = c[kCntFault];
    if (!f) return MCSBR_OK;
    std::string m = "device fault:";
    if (f & 1u) m += " fresnel: refractive indices / cos_theta_i out of domain;";
    if (f & 2u) m += " interface_transform: field is not transverse to dir_in;";
    if (f & 4u) m += " reflect_dir/refract_dir: grazing incidence;";
    if (f & 8u) m += " deterministic solver branch stack overflow;";
    if (f & 16u) m += " exact reduction: a term outside the 192-bit fixed-point range (|v| >= 2^71);";
    return set_err(MCSBR_EDEVICE, m);
}

void finalize_values(const double* raw, uint32_t n, const double* freqs, uint32_t nf, double* values) {
    for (uint32_t k = 0; k < n; ++k) {
        for (int ch = 0; ch < 4; ++ch) {
            for (uint32_t i = 0; i < nf; ++i) {
                const double k0 = 2.0 * kPi * freqs[i] / kC;
                const double pre_re = 0.0 * k0 / (2.0 * std::sqrt(kPi));
                const double pre_im = 1.0 * k0 / (2.0 * std::sqrt(kPi));
                const double* sv = raw + ((static_cast<size_t>(k) * nf + i) * 4 + ch) * 2;
                double* o = values + ((static_cast<size_t>(k) * 4 + ch) * nf + i) * 2;
                o[0] = pre_re * sv[0] - pre_im * sv[1];
                o[1] = pre_re * sv[1] + pre_im * sv[0];
            }
        }
    }
}

void limbs_to_doubles(const long long* limbs, size_t n, double* out) {
    for (size_t i = 0; i < n; ++i) {
        const int64_t l[4] = {limbs[4 * i], limbs[4 * i + 1], limbs[4 * i + 2], limbs[4 * i + 3]};
        out[i] = mcsbr_fx::fx_limbs_to_double(l);
    }
}

int use_device(const mcsbr_scene* s) {
    CK(cudaSetDevice(s->device), "cudaSetDevice");
    return MCSBR_OK;
}

}  // namespace

extern "C" {

const char* mcsbr_gpu_last_error(void) { return g_err.c_str(); }
void mcsbr_gpu_internal_set_error(const char* msg) { g_err = msg; }  // imaging.cu (not exported)
int mcsbr_gpu_abi_version(void) { return MCSBR_GPU_ABI_VERSION; }
uint64_t mcsbr_gpu_last_launch_count(void) { return g_launches; }

void mcsbr_gpu_kernel_timing(int enable) {
    g_kt.on = enable != 0;
    g_kt.used = 0;
    g_kt.marks.clear();
}

int mcsbr_gpu_kernel_times(double* path_ms, uint64_t* path_launches, double* acc_ms, uint64_t* acc_launches) {
    double t[2] = {0.0, 0.0};
    uint64_t n[2] = {0, 0};
    if (g_kt.device >= 0) CK(cudaSetDevice(g_kt.device), "cudaSetDevice");
    for (const auto& m : g_kt.marks) {
        float ms = 0.f;
        CK(cudaEventSynchronize(g_kt.pool[m.second + 1]), "cudaEventSynchronize");
        CK(cudaEventElapsedTime(&ms, g_kt.pool[m.second], g_kt.pool[m.second + 1]), "cudaEventElapsedTime");
        t[m.first] += ms;
        n[m.first] += 1;
    }
    if (path_ms) *path_ms = t[0];
    if (path_launches) *path_launches = n[0];
    if (acc_ms) *acc_ms = t[1];
    if (acc_launches) *acc_launches = n[1];
    return MCSBR_OK;
}

void mcsbr_gpu_default_config(mcsbr_mc_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->strata_per_wavelength = 10.0;
    c->samples_per_stratum = 16;
    c->branch_strategy = MCSBR_BRANCH_FRESNEL;
    c->roulette_enabled = 0;
    c->roulette_min_bounce = 2;
    c->roulette_q = 0.5;
    c->max_bounce = 9;
    c->jitter = 1;
    c->seed = 1;
    c->reference_wavelength = 0.0;
    c->launch_padding = 0.0;
    c->p_min = 0.05;
    c->block_size = 8192;
    c->rng_mode = MCSBR_RNG_REFERENCE;
    c->reduction = MCSBR_REDUCE_FAST;
    c->parity_fp64_refine = 1;
}

int mcsbr_gpu_validate_config(const mcsbr_mc_config* cfg) { return validate(cfg); }

int mcsbr_gpu_scene_create(const double* xyz, uint32_t nv, const mcsbr_triangle* tris, uint32_t nt,
                           const mcsbr_material* mats, uint32_t nm, const double* eps_imag, int device,
                           mcsbr_scene** out) {
    if (!out) return set_err(MCSBR_EINVAL, "scene_create: null output");
    *out = nullptr;
    if (nt == 0 || !tris) return set_err(MCSBR_ESCENE, "scene has no triangles");
    if (nm == 0 || !mats) return set_err(MCSBR_ESCENE, "material map: missing 'materials' object");
    if (nv == 0 || !xyz) return set_err(MCSBR_ESCENE, "scene is degenerate (zero extent)");
    if (mats[0].is_pec) return set_err(MCSBR_ESCENE, "material map: ambient material cannot be PEC");
    if (eps_imag && eps_imag[0] != 0.0)
        return set_err(MCSBR_EINVAL, "lossy media: the ambient material must be lossless (eps_imag[0] == 0)");
    for (uint32_t i = 0; i < nm; ++i) {
        if (eps_imag && !(eps_imag[i] >= 0.0 && std::isfinite(eps_imag[i])))
            return set_err(MCSBR_EINVAL, "lossy media: eps_imag must be finite and >= 0 (eps = eps_r - j eps_imag)");
        if (!mats[i].is_pec && (!(mats[i].eps_r > 0.0) || !(mats[i].mu_r > 0.0) ||
                                !std::isfinite(mats[i].eps_r) || !std::isfinite(mats[i].mu_r)))
            return set_err(MCSBR_ESCENE, "material: eps_r and mu_r must be positive");
    }
    HostPhases hp("scene_create");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return set_err(MCSBR_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return set_err(MCSBR_EINVAL, "scene_create: bad device index");
    CK(cudaSetDevice(device), "cudaSetDevice");
    // two attributes, not cudaGetDeviceProperties (which costs ~1 ms per call)
    int cc_major = 0, cc_minor = 0, n_sm = 0;
    CK(cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, device), "cudaDeviceGetAttribute");
    CK(cudaDeviceGetAttribute(&cc_minor, cudaDevAttrComputeCapabilityMinor, device), "cudaDeviceGetAttribute");
    CK(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, device), "cudaDeviceGetAttribute");
    if (cc_major < 10)
        return set_err(MCSBR_ECUDA, "this library is built for sm_100a (B200); device is sm_" +
                                        std::to_string(cc_major) + std::to_string(cc_minor));

    auto* s = new mcsbr_scene();
    s->device = device;
    s->sms = n_sm;
    s->nv = nv;
    s->nt = nt;
    s->nm = nm;
    s->ambient_n = mats[0].is_pec ? 0.0 : std::sqrt(mats[0].eps_r * mats[0].mu_r);
    std::vector<double2> mat(nm);
    std::vector<double> nim(nm, 0.0);
    std::vector<uint8_t> is_pec(nm);
    s->lossy = eps_imag != nullptr;  // complex-permittivity transport requested
    for (uint32_t i = 0; i < nm; ++i) {
        double n_re = mats[i].is_pec ? 0.0 : std::sqrt(mats[i].eps_r * mats[i].mu_r);  // Material::index()
        if (s->lossy && !mats[i].is_pec && eps_imag[i] != 0.0) {
            // n = sqrt((eps_r - j eps_i) mu_r), principal root: Re n > 0, Im n < 0
            const double a = mats[i].eps_r * mats[i].mu_r, b = -eps_imag[i] * mats[i].mu_r;
            const double m = std::hypot(a, b);
            n_re = std::sqrt(0.5 * (m + a));
            nim[i] = b / (2.0 * n_re);
        }
        mat[i] = make_double2(n_re, mats[i].is_pec ? 1.0 : 0.0);
        is_pec[i] = mats[i].is_pec ? 1 : 0;
    }

    auto fail = [&](cudaError_t e2, const char* what) {
        mcsbr_gpu_scene_destroy(s);
        return cuda_err(e2, what);
    };
    if ((e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(e, "cudaStreamCreate");
    if ((e = dev_malloc(&s->d_vtx, sizeof(double) * 3 * nv)) != cudaSuccess) return fail(e, "dev_malloc(vertices)");
    if ((e = dev_malloc(&s->d_tri, sizeof(uint4) * nt)) != cudaSuccess) return fail(e, "dev_malloc(triangles)");
    if ((e = dev_malloc(&s->d_info, sizeof(double2) * 2 * nt)) != cudaSuccess) return fail(e, "dev_malloc(tri info)");
    if ((e = dev_malloc(&s->d_mat, sizeof(double2) * nm)) != cudaSuccess) return fail(e, "dev_malloc(materials)");
    if ((e = cudaMemcpyAsync(s->d_vtx, xyz, sizeof(double) * 3 * nv, cudaMemcpyHostToDevice, s->stream)) !=
        cudaSuccess)
        return fail(e, "upload vertices");
    if ((e = cudaMemcpyAsync(s->d_mat, mat.data(), sizeof(double2) * nm, cudaMemcpyHostToDevice, s->stream)) !=
        cudaSuccess)
        return fail(e, "upload materials");
    if (s->lossy) {
        if ((e = dev_malloc(&s->d_nim, sizeof(double) * nm)) != cudaSuccess) return fail(e, "dev_malloc(Im n)");
        if ((e = cudaMemcpyAsync(s->d_nim, nim.data(), sizeof(double) * nm, cudaMemcpyHostToDevice, s->stream)) !=
            cudaSuccess)
            return fail(e, "upload Im n");
    }
    hp.mark("setup+upload");
    // Triangle checks + device layout, vertex bounds and the bounding sphere
    // on the device (prep.cu): Scene::finalize (geometry.cpp:146-162)
    {
        mcsbr_triangle* d_raw = nullptr;
        uint8_t* d_pec = nullptr;
        unsigned long long* d_w = nullptr;  // [0] first bad, [1] not all PEC, [2..7] bounds, [8] radius
        auto release = [&]() {
            dev_free(d_raw);
            dev_free(d_pec);
            dev_free(d_w);
        };
        unsigned long long w[9];
        if ((e = dev_malloc(&d_raw, sizeof(mcsbr_triangle) * nt)) != cudaSuccess ||
            (e = dev_malloc(&d_pec, nm)) != cudaSuccess || (e = dev_malloc(&d_w, sizeof(w))) != cudaSuccess ||
            (e = cudaMemcpyAsync(d_raw, tris, sizeof(mcsbr_triangle) * nt, cudaMemcpyHostToDevice, s->stream)) !=
                cudaSuccess ||
            (e = cudaMemcpyAsync(d_pec, is_pec.data(), nm, cudaMemcpyHostToDevice, s->stream)) != cudaSuccess ||
            (e = cudaMemsetAsync(d_w, 0xff, sizeof(unsigned long long), s->stream)) != cudaSuccess ||
            (e = cudaMemsetAsync(d_w + 1, 0, sizeof(unsigned long long), s->stream)) != cudaSuccess ||
            (e = launch_pack(d_raw, nt, nv, nm, d_pec, s->d_tri, s->d_info, d_w,
                             reinterpret_cast<unsigned int*>(d_w + 1), s->stream)) != cudaSuccess ||
            (e = launch_bounds(s->d_vtx, nv, d_w + 2, s->sms, s->stream)) != cudaSuccess ||
            (e = cudaMemcpyAsync(w, d_w, sizeof(unsigned long long) * 8, cudaMemcpyDeviceToHost, s->stream)) !=
                cudaSuccess ||
            (e = cudaStreamSynchronize(s->stream)) != cudaSuccess) {
            release();
            return fail(e, "scene preparation");
        }
        g_launches += 2;
        if (w[0] != ~0ull) {
            release();
            mcsbr_gpu_scene_destroy(s);
            const uint64_t i = w[0] >> 1;
            return set_err(MCSBR_ESCENE, "triangle " + std::to_string(i) +
                                             ((w[0] & 1) ? ": material index out of range"
                                                         : ": vertex index out of range"));
        }
        s->all_pec = (w[1] & 0xffffffffull) == 0 && !s->lossy;
        const V lo{unord(w[2]), unord(w[3]), unord(w[4])}, hi{unord(w[5]), unord(w[6]), unord(w[7])};
        const V c = (lo + hi) * 0.5;
        st(s->center, c);
        if ((e = launch_radius(s->d_vtx, nv, s->center, d_w + 8, s->sms, s->stream)) != cudaSuccess ||
            (e = cudaMemcpyAsync(&w[8], d_w + 8, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s->stream)) !=
                cudaSuccess ||
            (e = cudaStreamSynchronize(s->stream)) != cudaSuccess) {
            release();
            return fail(e, "scene preparation");
        }
        ++g_launches;
        release();
        const double r = unord(w[8]);
        s->radius = r;
        s->diameter = 2.0 * r;
        s->scene_lo[0] = lo.x;
        s->scene_lo[1] = lo.y;
        s->scene_lo[2] = lo.z;
        s->scene_hi[0] = hi.x;
        s->scene_hi[1] = hi.y;
        s->scene_hi[2] = hi.z;
    }
    if (!(s->diameter > 0.0)) {
        mcsbr_gpu_scene_destroy(s);
        return set_err(MCSBR_ESCENE, "scene is degenerate (zero extent)");
    }
    const double* lo3 = s->scene_lo;
    const double* hi3 = s->scene_hi;
    // boxes: outward-rounded fp64 AABBs; the pad only absorbs the fp64
    // rounding of the centring (the slab test's margin lives on the ray)
    const double box_pad = 1e-12 * s->radius + 1e-30;
    hp.mark("prep");
    if ((e = build_bvh(s->d_vtx, s->d_tri, nt, lo3, hi3, s->center, box_pad, s->stream, &s->bvh)) != cudaSuccess)
        return fail(e, "BVH build");
    g_launches += 7;
    hp.mark("bvh");
    if ((e = dev_malloc(&s->d_tri32, sizeof(float) * 9 * nt)) != cudaSuccess) return fail(e, "dev_malloc(tri32)");
    if ((e = build_tri32(s->d_vtx, s->d_tri, nt, s->center, s->d_tri32, s->stream)) != cudaSuccess)
        return fail(e, "fp32 triangle copy");
    ++g_launches;
    // a 4-wide level pushes at most 3 refs; BVH4 depth <= ceil(binary depth / 2) + 1
    if (3 * ((s->bvh.max_depth + 1) / 2 + 1) > static_cast<uint32_t>(kStackSize)) {
        mcsbr_gpu_scene_destroy(s);
        return set_err(MCSBR_ESCENE, "BVH depth exceeds the traversal stack (96)");
    }
    *out = s;
    return MCSBR_OK;
}

// A replica of the primary scene p on `device`: the device arrays copied
// from p's device (peer copies over NVLink when the devices differ), no
// second BVH build.
static int make_replica(mcsbr_scene* p, int device, mcsbr_scene** out) {
    *out = nullptr;
    CK(cudaSetDevice(p->device), "cudaSetDevice");
    CK(cudaStreamSynchronize(p->stream), "cudaStreamSynchronize");
    CK(cudaSetDevice(device), "cudaSetDevice");
    auto* r = new mcsbr_scene();
    r->device = device;
    r->nv = p->nv;
    r->nt = p->nt;
    r->nm = p->nm;
    std::memcpy(r->center, p->center, sizeof(r->center));
    r->radius = p->radius;
    r->diameter = p->diameter;
    r->ambient_n = p->ambient_n;
    r->all_pec = p->all_pec;
    r->lossy = p->lossy;
    r->bvh = p->bvh;
    r->bvh.nodes = nullptr;
    r->bvh.tri64 = nullptr;
    auto fail = [&](cudaError_t e, const char* what) {
        mcsbr_gpu_scene_destroy(r);
        return cuda_err(e, what);
    };
    cudaError_t e = cudaDeviceGetAttribute(&r->sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return fail(e, "cudaDeviceGetAttribute");
    if ((e = cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(e, "cudaStreamCreate");
    auto copy = [&](auto** dst, const auto* src, size_t bytes) {
        cudaError_t e2 = dev_malloc(dst, bytes);
        if (e2 == cudaSuccess) e2 = cudaMemcpyPeerAsync(*dst, device, src, p->device, bytes, r->stream);
        return e2;
    };
    if ((e = copy(&r->bvh.nodes, p->bvh.nodes, sizeof(float4) * 8 * std::max<uint32_t>(p->bvh.n_nodes, 1))) !=
            cudaSuccess ||
        (e = copy(&r->bvh.tri64, p->bvh.tri64, sizeof(double2) * 5 * p->bvh.n_leaves)) != cudaSuccess ||
        (e = copy(&r->d_info, p->d_info, sizeof(double2) * 2 * p->nt)) != cudaSuccess ||
        (e = copy(&r->d_mat, p->d_mat, sizeof(double2) * p->nm)) != cudaSuccess ||
        (e = copy(&r->d_tri32, p->d_tri32, sizeof(float) * 9 * p->nt)) != cudaSuccess ||
        (e = copy(&r->d_vtx, p->d_vtx, sizeof(double) * 3 * p->nv)) != cudaSuccess ||
        (p->d_nim && (e = copy(&r->d_nim, p->d_nim, sizeof(double) * p->nm)) != cudaSuccess))
        return fail(e, "replica copy");
    if ((e = cudaStreamSynchronize(r->stream)) != cudaSuccess) return fail(e, "replica copy");
    *out = r;
    return MCSBR_OK;
}

int mcsbr_gpu_scene_create_multi(const double* xyz, uint32_t nv, const mcsbr_triangle* tris, uint32_t nt,
                                 const mcsbr_material* mats, uint32_t nm, const double* eps_imag, const int* devices,
                                 int n_devices, mcsbr_scene** out) {
    if (!out) return set_err(MCSBR_EINVAL, "scene_create: null output");
    *out = nullptr;
    if (!devices || n_devices < 1) return set_err(MCSBR_EINVAL, "scene_create_multi: empty device list");
    int rc = mcsbr_gpu_scene_create(xyz, nv, tris, nt, mats, nm, eps_imag, devices[0], out);
    if (rc) return rc;
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    for (int i = 1; i < n_devices; ++i) {
        mcsbr_scene* r = nullptr;
        rc = devices[i] < 0 || devices[i] >= ndev ? set_err(MCSBR_EINVAL, "scene_create: bad device index")
                                                  : make_replica(*out, devices[i], &r);
        if (rc) {
            mcsbr_gpu_scene_destroy(*out);
            *out = nullptr;
            return rc;
        }
        (*out)->replicas.push_back(r);
    }
    return MCSBR_OK;
}

int mcsbr_gpu_scene_devices(const mcsbr_scene* s, int* n_devices) {
    if (!s || !n_devices) return set_err(MCSBR_EINVAL, "null argument");
    *n_devices = 1 + static_cast<int>(s->replicas.size());
    return MCSBR_OK;
}

int mcsbr_gpu_device_count(int* n) {
    if (!n) return set_err(MCSBR_EINVAL, "null argument");
    *n = 0;
    const cudaError_t e = cudaGetDeviceCount(n);
    if (e != cudaSuccess) {
        *n = 0;
        return cuda_err(e, "cudaGetDeviceCount");
    }
    return MCSBR_OK;
}

void mcsbr_gpu_scene_destroy(mcsbr_scene* s) {
    if (!s) return;
    HostPhases hp("destroy");
    for (mcsbr_scene* r : s->replicas) mcsbr_gpu_scene_destroy(r);
    s->replicas.clear();
    cudaSetDevice(s->device);
    // every stream that used the scene's buffers (its own, and callers' of
    // trace_device / intersect_device) must be done: one device sync, then
    // the frees need none each
    cudaDeviceSynchronize();
    hp.mark("sync");
    dev_free(s->d_vtx, true);
    dev_free(s->d_tri, true);
    dev_free(s->d_info, true);
    dev_free(s->d_mat, true);
    dev_free(s->d_nim, true);
    dev_free(s->d_tri32, true);
    dev_free(s->bvh.nodes, true);
    dev_free(s->bvh.tri64, true);
    s->inc.release(true);
    s->rx.release(true);
    s->k0.release(true);
    s->sums.release(true);
    s->counters.release(true);
    s->tile.release(true);
    s->recs.release(true);
    s->nufft_grid.release(true);
    s->nufft_hat.release(true);
    s->nufft_idx.release(true);
    s->nufft_inc.release(true);
    s->nufft_bucket.release(true);
    s->cover.release(true);
    s->leaf32.release(true);
    s->plan_axes.release(true);
    s->plan_ext.release(true);
    s->xsums.release(true);
    s->limbs.release(true);
    s->wf_pool.release(true);
    s->wf_u32.release(true);
    s->wf_ctl.release(true);
    hp.mark("frees");
    pinned_release(s->wf_host);
    if (s->wf_ev) cudaEventDestroy(s->wf_ev);
    if (s->ev0) cudaEventDestroy(s->ev0);
    if (s->peak_host) learn_rec_ratio(s);  // the last job's ratio becomes the next scene's hint
    if (s->peak_ev) cudaEventDestroy(s->peak_ev);
    pinned_release(s->peak_host);
    if (s->ev1) cudaEventDestroy(s->ev1);
    hp.mark("host-frees/events");
    if (s->stream) cudaStreamDestroy(s->stream);
    hp.mark("stream");
    delete s;
}

int mcsbr_gpu_scene_bounds(const mcsbr_scene* s, double center[3], double* radius, double* diameter) {
    if (!s) return set_err(MCSBR_EINVAL, "null scene");
    if (center) std::memcpy(center, s->center, sizeof(s->center));
    if (radius) *radius = s->radius;
    if (diameter) *diameter = s->diameter;
    return MCSBR_OK;
}

int mcsbr_gpu_scene_bvh_info(const mcsbr_scene* s, uint32_t* n_nodes, uint32_t* max_depth, uint32_t* n_leaves,
                             double* build_ms) {
    if (!s) return set_err(MCSBR_EINVAL, "null scene");
    if (n_nodes) *n_nodes = s->bvh.n_nodes;
    if (max_depth) *max_depth = s->bvh.max_depth;
    if (n_leaves) *n_leaves = s->bvh.n_leaves;
    if (build_ms) *build_ms = s->bvh.build_ms;
    return MCSBR_OK;
}

int mcsbr_gpu_launch_plan(const mcsbr_scene* s, const double k_inc[3], double padding, double spw,
                          double lambda_ref, int32_t spp, mcsbr_launch_plan* out) {
    if (!s || !k_inc || !out) return set_err(MCSBR_EINVAL, "launch_plan: null argument");
    return plan(s, k_inc, padding, spw, lambda_ref, spp, out);
}

int mcsbr_gpu_intersect(const mcsbr_scene* s, const double* o, const double* d, const double* tmin, uint32_t n,
                        int any_hit, double* t_out, uint32_t* id_out) {
    if (!s) return set_err(MCSBR_EINVAL, "null scene");
    if (n == 0) return MCSBR_OK;
    int rc = use_device(s);
    if (rc) return rc;
    double *d_o = nullptr, *d_d = nullptr, *d_t = nullptr, *d_to = nullptr;
    uint32_t* d_id = nullptr;
    cudaError_t e = cudaSuccess;
    const size_t v3 = sizeof(double) * 3 * n;
    if ((e = dev_malloc(&d_o, v3)) == cudaSuccess && (e = dev_malloc(&d_d, v3)) == cudaSuccess &&
        (e = dev_malloc(&d_t, sizeof(double) * n)) == cudaSuccess &&
        (e = dev_malloc(&d_to, sizeof(double) * n)) == cudaSuccess &&
        (e = dev_malloc(&d_id, sizeof(uint32_t) * n)) == cudaSuccess &&
        (e = cudaMemcpyAsync(d_o, o, v3, cudaMemcpyHostToDevice, s->stream)) == cudaSuccess &&
        (e = cudaMemcpyAsync(d_d, d, v3, cudaMemcpyHostToDevice, s->stream)) == cudaSuccess &&
        (e = cudaMemcpyAsync(d_t, tmin, sizeof(double) * n, cudaMemcpyHostToDevice, s->stream)) == cudaSuccess &&
        (e = launch_intersect(s->view(), d_o, d_d, d_t, n, any_hit, d_to, d_id, s->stream)) == cudaSuccess &&
        (e = cudaMemcpyAsync(t_out, d_to, sizeof(double) * n, cudaMemcpyDeviceToHost, s->stream)) == cudaSuccess &&
        (e = cudaMemcpyAsync(id_out, d_id, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, s->stream)) ==
            cudaSuccess) {
        ++g_launches;
        e = cudaStreamSynchronize(s->stream);
    }
    dev_free(d_o);
    dev_free(d_d);
    dev_free(d_t);
    dev_free(d_to);
    dev_free(d_id);
    if (e != cudaSuccess) return cuda_err(e, "intersect");
    return MCSBR_OK;
}

struct PathLog {
    uint64_t n = 0;
    uint32_t stride = 0;
    uint32_t* tri = nullptr;
    uint8_t* term = nullptr;
    uint64_t* branch = nullptr;
};

int mcsbr_gpu_intersect_device(const mcsbr_scene* s, const double* d_o, const double* d_d, const double* d_tmin,
                               uint32_t n, int any_hit, double* d_t, uint32_t* d_id, void* stream) {
    if (!s) return set_err(MCSBR_EINVAL, "null scene");
    int rc = use_device(s);
    if (rc) return rc;
    CK(launch_intersect(s->view(), d_o, d_d, d_tmin, n, any_hit, d_t, d_id, static_cast<cudaStream_t>(stream)),
       "intersect kernel");
    ++g_launches;
    return MCSBR_OK;
}

// Counter blocks of several shards: sums, except the fault bits (OR) and
// the deepest round (max).
static void merge_counters(unsigned long long* dst, const unsigned long long* src) {
    for (int i = 0; i < kCntWords; ++i) {
        if (i == kCntFault) dst[i] |= src[i];
        else if (i == kCntRounds) dst[i] = std::max(dst[i], src[i]);
        else dst[i] += src[i];
    }
}

// One shard of a multi-device job on replica `r` (its own device, stream and
// buffers), on the calling host thread; raw sums (or exact limbs) and
// counters come back to the host.
struct ShardOut {
    int rc = MCSBR_OK;
    std::string err;
    std::vector<double> raw;
    std::vector<long long> limbs;
    unsigned long long cnt[kCntWords] = {};
    float kms = 0.f;
    uint64_t launches = 0;
};

static void run_shard(mcsbr_scene* r, const mcsbr_incidence* incs, uint32_t n_inc, const mcsbr_receiver* rxs, uint32_t n_rx,
               int occlusion, const double* freqs, uint32_t nf, const mcsbr_mc_config* cfg, uint32_t shard,
               uint32_t nshard, ShardOut* o) {
    const uint64_t launches0 = g_launches;
    auto fail = [&](int rc) {
        o->rc = rc;
        o->err = g_err;
    };
    auto cuda_fail = [&](cudaError_t e, const char* what) { fail(cuda_err(e, what)); };
    cudaError_t e = cudaSetDevice(r->device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    Job job;
    int rc = plan_job(r, incs, n_inc, rxs, n_rx, freqs, nf, cfg, shard, nshard, r->sms * 16, &job);
    if (rc) return fail(rc);
    const size_t nsum = static_cast<size_t>(n_inc) * n_rx * nf * 8;
    const bool exact = cfg->reduction == MCSBR_REDUCE_EXACT;
    if ((e = r->sums.reserve(nsum)) != cudaSuccess || (e = r->counters.reserve(kCntWords)) != cudaSuccess ||
        (exact && (e = r->limbs.reserve(nsum * MCSBR_EXACT_LIMBS)) != cudaSuccess))
        return cuda_fail(e, "dev_malloc(shard sums)");
    if ((e = cudaMemsetAsync(r->sums.p, 0, sizeof(double) * nsum, r->stream)) != cudaSuccess ||
        (e = cudaMemsetAsync(r->counters.p, 0, sizeof(unsigned long long) * kCntWords, r->stream)) != cudaSuccess ||
        (exact && (e = cudaMemsetAsync(r->limbs.p, 0, sizeof(long long) * nsum * MCSBR_EXACT_LIMBS, r->stream)) !=
                      cudaSuccess))
        return cuda_fail(e, "memset shard sums");
    rc = run_job(r, job, nf, cfg, occlusion, r->sums.p, r->counters.p, r->stream, nullptr, &o->kms,
                 exact ? r->limbs.p : nullptr);
    if (rc) return fail(rc);
    if (exact) {
        o->limbs.resize(nsum * MCSBR_EXACT_LIMBS);
        e = cudaMemcpyAsync(o->limbs.data(), r->limbs.p, sizeof(long long) * o->limbs.size(), cudaMemcpyDeviceToHost,
                            r->stream);
    } else {
        o->raw.resize(nsum);
        e = cudaMemcpyAsync(o->raw.data(), r->sums.p, sizeof(double) * nsum, cudaMemcpyDeviceToHost, r->stream);
    }
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(o->cnt, r->counters.p, sizeof(o->cnt), cudaMemcpyDeviceToHost, r->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(r->stream);
    if (e != cudaSuccess) return cuda_fail(e, "shard readback");
    o->launches = g_launches - launches0;
}

// estimate / estimate_batch over `ndev` devices of a multi-device scene:
// launch entries sharded exactly as mcsbr_gpu_trace_device shards them
// (every device a contiguous share of every incidence), one host thread per
// device, partial sums added on the host in device order (exact limbs add
// exactly: the result is byte-identical to one device's).
static int estimate_multi(mcsbr_scene* s, uint32_t ndev, const mcsbr_incidence* incs, uint32_t n_inc,
                   const mcsbr_receiver* rxs, uint32_t n_rx, int occlusion, const double* freqs, uint32_t nf,
                   const mcsbr_mc_config* cfg, double* values, mcsbr_stats* stats,
                   std::chrono::steady_clock::time_point t0) {
    std::vector<ShardOut> outs(ndev);
    std::vector<std::thread> pool;
    for (uint32_t d = 0; d < ndev; ++d) {
        mcsbr_scene* r = d == 0 ? s : s->replicas[d - 1];
        pool.emplace_back(run_shard, r, incs, n_inc, rxs, n_rx, occlusion, freqs, nf, cfg, d, ndev, &outs[d]);
    }
    for (auto& t : pool) t.join();
    for (const ShardOut& o : outs) {
        g_launches += o.launches;
        if (o.rc) return set_err(o.rc, o.err);
    }
    const size_t nsum = static_cast<size_t>(n_inc) * n_rx * nf * 8;
    std::vector<double> raw(nsum, 0.0);
    unsigned long long cnt[kCntWords] = {};
    float kms = 0.f;
    if (cfg->reduction == MCSBR_REDUCE_EXACT) {
        std::vector<long long> limbs(nsum * MCSBR_EXACT_LIMBS, 0);
        for (const ShardOut& o : outs)
            for (size_t i = 0; i < limbs.size(); ++i) limbs[i] += o.limbs[i];
        limbs_to_doubles(limbs.data(), nsum, raw.data());
    } else {
        for (const ShardOut& o : outs)
            for (size_t i = 0; i < nsum; ++i) raw[i] += o.raw[i];
    }
    for (const ShardOut& o : outs) {
        merge_counters(cnt, o.cnt);
        kms = std::max(kms, o.kms);
    }
    int rc = fault_check(cnt);
    if (rc) return rc;
    finalize_values(raw.data(), n_inc * n_rx, freqs, nf, values);
    if (stats) {
        decode(cnt, stats);
        stats->block_size = static_cast<uint64_t>(cfg->block_size);
        uint64_t threads = 0;
        for (uint32_t d = 0; d < ndev; ++d) threads += static_cast<uint64_t>((d == 0 ? s : s->replicas[d - 1])->sms) * 2048;
        stats->peak_live_state_bytes = threads * stats->state_bytes_per_ray;
        stats->kernel_ms = kms;
        stats->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    return MCSBR_OK;
}

static int estimate_common(mcsbr_scene* s, const mcsbr_incidence* incs, uint32_t n_inc, const mcsbr_receiver* rxs,
                           uint32_t n_rx, int occlusion, const double* freqs, uint32_t nf,
                           const mcsbr_mc_config* cfg, double* values, mcsbr_stats* stats,
                           mcsbr_contribution* contribs, uint64_t capacity, uint64_t* n_contribs,
                           const PathLog* plog = nullptr, const mcsbr_det_config* det = nullptr,
                           int workers = 0) {
    const auto t0 = std::chrono::steady_clock::now();
    if (!s) return set_err(MCSBR_EINVAL, "null scene");
    int rc = use_device(s);
    if (rc) return rc;
    // several devices: workers <= 0 means all of the scene's devices
    const uint32_t have = 1 + static_cast<uint32_t>(s->replicas.size());
    const uint32_t ndev = workers <= 0 ? have : std::min<uint32_t>(have, static_cast<uint32_t>(workers));
    if (ndev > 1 && !contribs && !(plog && plog->n) && !det) {
        rc = validate(cfg);
        if (rc) return rc;
        return estimate_multi(s, ndev, incs, n_inc, rxs, n_rx, occlusion, freqs, nf, cfg, values, stats, t0);
    }
    HostPhases hp("estimate");
    Job job;
    rc = plan_job(s, incs, n_inc, rxs, n_rx, freqs, nf, cfg, 0, 1, s->sms * 16, &job, det != nullptr);
    if (rc) return rc;
    hp.mark("plan");
    if (det && (n_inc != 1 || n_rx != 1)) return set_err(MCSBR_EINVAL, "solve: one excitation per call");
    const size_t nsum = static_cast<size_t>(n_inc) * n_rx * nf * 8;
    CK(s->sums.reserve(nsum), "dev_malloc(sums)");
    CK(s->counters.reserve(kCntWords), "dev_malloc(counters)");
    CK(cudaMemsetAsync(s->sums.p, 0, sizeof(double) * nsum, s->stream), "memset sums");
    CK(cudaMemsetAsync(s->counters.p, 0, sizeof(unsigned long long) * kCntWords, s->stream), "memset counters");
    TraceParams extra{};
    TempBufs temps;  // instrumentation / deterministic-solver temporaries, freed on every exit
    mcsbr_contribution* d_out = nullptr;
    mcsbr_contribution* d_scratch = nullptr;
    unsigned long long* d_cnt = nullptr;
    if (contribs) {
        if (n_inc != 1 || n_rx != 1) return set_err(MCSBR_EINVAL, "contributions_out needs one incidence");
        const size_t scratch_n = static_cast<size_t>(s->sms) * 32 * 128;  // >= resident threads
        CK(temps.alloc(&d_out, sizeof(mcsbr_contribution) * std::max<uint64_t>(capacity, 1)), "dev_malloc(contribs)");
        CK(temps.alloc(&d_scratch, sizeof(mcsbr_contribution) * scratch_n), "dev_malloc(scratch)");
        CK(temps.alloc(&d_cnt, sizeof(unsigned long long)), "dev_malloc(count)");
        CK(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), s->stream), "memset count");
        extra.contrib_out = d_out;
        extra.contrib_cap = capacity;
        extra.contrib_count = d_cnt;
        extra.contrib_scratch = d_scratch;
    }
    uint32_t* d_ptri = nullptr;
    uint8_t* d_pterm = nullptr;
    unsigned long long* d_pbr = nullptr;
    if (plog && plog->n) {
        const size_t nt = plog->n * plog->stride;
        CK(temps.alloc(&d_ptri, sizeof(uint32_t) * nt), "dev_malloc(plog)");
        CK(temps.alloc(&d_pterm, plog->n), "dev_malloc(plog)");
        CK(temps.alloc(&d_pbr, sizeof(unsigned long long) * plog->n), "dev_malloc(plog)");
        CK(cudaMemsetAsync(d_ptri, 0xff, sizeof(uint32_t) * nt, s->stream), "memset plog");
        CK(cudaMemsetAsync(d_pterm, 0, plog->n, s->stream), "memset plog");
        CK(cudaMemsetAsync(d_pbr, 0, sizeof(unsigned long long) * plog->n, s->stream), "memset plog");
        extra.plog_tri = d_ptri;
        extra.plog_term = d_pterm;
        extra.plog_branch = d_pbr;
        extra.plog_n = plog->n;
        extra.plog_stride = plog->stride;
    }
    // deterministic: branch stacks for every resident thread + block accounting
    double* d_stack = nullptr;
    unsigned long long* d_blocks = nullptr;
    uint64_t det_nblocks = 0, stack_bytes = 0;
    if (det) {
        const uint64_t threads = static_cast<uint64_t>(s->sms) * MCSBR_DET_THREADS_PER_SM;
        const uint32_t depth = static_cast<uint32_t>(det->max_bounce);
        stack_bytes = sizeof(double) * kDetFields * depth * threads;
        det_nblocks = (job.total_entries + det->block_size - 1) / static_cast<uint64_t>(det->block_size);
        cudaError_t e0 = temps.alloc(&d_stack, stack_bytes);
        if (e0 == cudaSuccess) e0 = temps.alloc(&d_blocks, sizeof(unsigned long long) * 2 * std::max<uint64_t>(det_nblocks, 1));
        if (e0 == cudaSuccess)
            e0 = cudaMemsetAsync(d_blocks, 0, sizeof(unsigned long long) * 2 * std::max<uint64_t>(det_nblocks, 1), s->stream);
        if (e0 != cudaSuccess) {
            return cuda_err(e0, "dev_malloc(branch stacks)");
        }
        extra.det = 1;
        extra.det_cutoff = det->amplitude_cutoff;
        extra.det_stack = d_stack;
        extra.det_depth = depth;
        extra.det_threads = threads;
        extra.det_blocks = d_blocks;
        extra.det_block_size = static_cast<uint64_t>(det->block_size);
    }
    float kms = 0.f;
    const bool exact = cfg->reduction == MCSBR_REDUCE_EXACT;
    if (exact) {
        CK(s->limbs.reserve(nsum * MCSBR_EXACT_LIMBS), "dev_malloc(limbs)");
        CK(cudaMemsetAsync(s->limbs.p, 0, sizeof(long long) * nsum * MCSBR_EXACT_LIMBS, s->stream), "memset limbs");
    }
    rc = run_job(s, job, nf, cfg, occlusion, s->sums.p, s->counters.p, s->stream, &extra, &kms,
                 exact ? s->limbs.p : nullptr);
    hp.mark("run");
    std::vector<unsigned long long> det_acc(2 * det_nblocks);
    if (rc == MCSBR_OK && det && det_nblocks) {
        const cudaError_t e2 = cudaMemcpy(det_acc.data(), d_blocks, sizeof(unsigned long long) * det_acc.size(),
                                          cudaMemcpyDeviceToHost);
        if (e2 != cudaSuccess) rc = cuda_err(e2, "branch accounting readback");
    }
    if (rc == MCSBR_OK && plog && plog->n) {
        cudaError_t e2 = cudaMemcpy(plog->tri, d_ptri, sizeof(uint32_t) * plog->n * plog->stride,
                                    cudaMemcpyDeviceToHost);
        if (e2 == cudaSuccess) e2 = cudaMemcpy(plog->term, d_pterm, plog->n, cudaMemcpyDeviceToHost);
        if (e2 == cudaSuccess)
            e2 = cudaMemcpy(plog->branch, d_pbr, sizeof(uint64_t) * plog->n, cudaMemcpyDeviceToHost);
        if (e2 != cudaSuccess) rc = cuda_err(e2, "path log readback");
    }
    if (rc) {
        return rc;
    }
    std::vector<double> raw(exact ? 0 : nsum);
    std::vector<long long> raw_limbs(exact ? nsum * MCSBR_EXACT_LIMBS : 0);
    unsigned long long cnt[kCntWords];
    cudaError_t e = exact ? cudaMemcpyAsync(raw_limbs.data(), s->limbs.p, sizeof(long long) * raw_limbs.size(),
                                            cudaMemcpyDeviceToHost, s->stream)
                          : cudaMemcpyAsync(raw.data(), s->sums.p, sizeof(double) * nsum, cudaMemcpyDeviceToHost,
                                            s->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(cnt, s->counters.p, sizeof(cnt), cudaMemcpyDeviceToHost, s->stream);
    unsigned long long ncol = 0;
    if (e == cudaSuccess && contribs)
        e = cudaMemcpyAsync(&ncol, d_cnt, sizeof(ncol), cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e == cudaSuccess && contribs) {
        const uint64_t m = std::min<uint64_t>(ncol, capacity);
        e = cudaMemcpy(contribs, d_out, sizeof(mcsbr_contribution) * m, cudaMemcpyDeviceToHost);
        std::sort(contribs, contribs + m, [](const mcsbr_contribution& x, const mcsbr_contribution& y) {
            return x.order_key < y.order_key;
        });
        if (n_contribs) *n_contribs = ncol;
    }
    if (e != cudaSuccess) return cuda_err(e, "estimate readback");
    rc = fault_check(cnt);
    if (rc) return rc;
    if (exact) {
        raw.resize(nsum);
        limbs_to_doubles(raw_limbs.data(), nsum, raw.data());
    }
    finalize_values(raw.data(), n_inc * n_rx, freqs, nf, values);
    if (stats) {
        decode(cnt, stats);
        stats->block_size = static_cast<uint64_t>(cfg->block_size);
        stats->peak_live_state_bytes = static_cast<uint64_t>(s->sms) * 2048 * stats->state_bytes_per_ray;
        if (det) {  // RunStats::merge keeps the max over blocks (solver_common.cpp:64-65)
            uint64_t peak = 0, push = 0;
            for (uint64_t b = 0; b < det_nblocks; ++b) {
                peak = std::max<uint64_t>(peak, det_acc[2 * b]);
                push = std::max<uint64_t>(push, det_acc[2 * b + 1]);
            }
            stats->state_bytes_per_ray = kPathStateBytes;
            stats->peak_live_state_bytes = peak * kPathStateBytes;
            stats->forced_stack_bytes = push * kPathStateBytes;
            stats->device_stack_bytes = stack_bytes;
        }
        stats->kernel_ms = kms;
        stats->wall_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    return MCSBR_OK;
}

int mcsbr_gpu_estimate(mcsbr_scene* s, const mcsbr_excitation* exc, const double* freqs, uint32_t nf,
                       const mcsbr_mc_config* cfg, int workers, double* values, mcsbr_stats* stats,
                       mcsbr_contribution* contribs, uint64_t capacity, uint64_t* n_contribs) {
    if (!exc) return set_err(MCSBR_EINVAL, "estimate: null excitation");
    mcsbr_incidence inc;
    std::memcpy(inc.k_inc, exc->k_inc, sizeof(inc.k_inc));
    std::memcpy(inc.pol_v, exc->pol_v, sizeof(inc.pol_v));
    std::memcpy(inc.pol_h, exc->pol_h, sizeof(inc.pol_h));
    inc.strata_per_wavelength = 0.0;
    mcsbr_receiver rx;
    std::memcpy(rx.k_scatter, exc->k_scatter, sizeof(rx.k_scatter));
    std::memcpy(rx.rx_v, exc->rx_v, sizeof(rx.rx_v));
    std::memcpy(rx.rx_h, exc->rx_h, sizeof(rx.rx_h));
    return estimate_common(s, &inc, 1, &rx, 1, exc->occlusion_enabled, freqs, nf, cfg, values, stats, contribs,
                           capacity, n_contribs, nullptr, nullptr, workers < 1 ? 1 : workers);
}

void mcsbr_gpu_default_det_config(mcsbr_det_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->rays_per_wavelength = 20.0;
    c->max_bounce = 9;
    c->force_stack_accounting = 0;
    c->amplitude_cutoff = 0.0;
    c->launch_padding = 0.0;
    c->reference_wavelength = 0.0;
    c->block_size = 8192;
}

int mcsbr_gpu_validate_det_config(const mcsbr_det_config* cfg) { return validate_det(cfg); }

int mcsbr_gpu_solve(mcsbr_scene* s, const mcsbr_excitation* exc, const double* freqs, uint32_t nf,
                    const mcsbr_det_config* cfg, int workers, double* values, mcsbr_stats* stats,
                    mcsbr_contribution* contribs, uint64_t capacity, uint64_t* n_contribs) {
    (void)workers;
    int rc = validate_det(cfg);
    if (rc) return rc;
    if (nf == 0 || !freqs) return set_err(MCSBR_EINVAL, "solve: empty frequency list");
    if (!exc) return set_err(MCSBR_EINVAL, "solve: null excitation");
    const mcsbr_mc_config mc = det_as_mc(cfg);
    mcsbr_incidence inc;
    std::memcpy(inc.k_inc, exc->k_inc, sizeof(inc.k_inc));
    std::memcpy(inc.pol_v, exc->pol_v, sizeof(inc.pol_v));
    std::memcpy(inc.pol_h, exc->pol_h, sizeof(inc.pol_h));
    inc.strata_per_wavelength = 0.0;
    mcsbr_receiver rx;
    std::memcpy(rx.k_scatter, exc->k_scatter, sizeof(rx.k_scatter));
    std::memcpy(rx.rx_v, exc->rx_v, sizeof(rx.rx_v));
    std::memcpy(rx.rx_h, exc->rx_h, sizeof(rx.rx_h));
    return estimate_common(s, &inc, 1, &rx, 1, exc->occlusion_enabled, freqs, nf, &mc, values, stats, contribs,
                           capacity, n_contribs, nullptr, cfg);
}

int mcsbr_gpu_path_log(mcsbr_scene* s, const mcsbr_excitation* exc, const double* freqs, uint32_t nf,
                       const mcsbr_mc_config* cfg, uint64_t n_paths, uint32_t stride, uint32_t* tri_ids,
                       uint8_t* term, uint64_t* branch_bits) {
    if (!exc || !tri_ids || !term || !branch_bits) return set_err(MCSBR_EINVAL, "path_log: null argument");
    mcsbr_incidence inc;
    std::memcpy(inc.k_inc, exc->k_inc, sizeof(inc.k_inc));
    std::memcpy(inc.pol_v, exc->pol_v, sizeof(inc.pol_v));
    std::memcpy(inc.pol_h, exc->pol_h, sizeof(inc.pol_h));
    inc.strata_per_wavelength = 0.0;
    mcsbr_receiver rx;
    std::memcpy(rx.k_scatter, exc->k_scatter, sizeof(rx.k_scatter));
    std::memcpy(rx.rx_v, exc->rx_v, sizeof(rx.rx_v));
    std::memcpy(rx.rx_h, exc->rx_h, sizeof(rx.rx_h));
    std::vector<double> values(static_cast<size_t>(nf) * 8);
    PathLog pl;
    pl.n = n_paths;
    pl.stride = stride;
    pl.tri = tri_ids;
    pl.term = term;
    pl.branch = branch_bits;
    return estimate_common(s, &inc, 1, &rx, 1, exc->occlusion_enabled, freqs, nf, cfg, values.data(), nullptr,
                           nullptr, 0, nullptr, &pl);
}

int mcsbr_gpu_estimate_batch(mcsbr_scene* s, const mcsbr_incidence* incs, uint32_t n_inc,
                             const mcsbr_receiver* rxs, uint32_t n_rx, int occlusion, const double* freqs,
                             uint32_t nf, const mcsbr_mc_config* cfg, double* values, mcsbr_stats* stats) {
    return estimate_common(s, incs, n_inc, rxs, n_rx, occlusion, freqs, nf, cfg, values, stats, nullptr, 0,
                           nullptr);
}

int mcsbr_gpu_trace_device(mcsbr_scene* s, const mcsbr_incidence* incs, uint32_t n_inc, const mcsbr_receiver* rxs,
                           uint32_t n_rx, int occlusion, const double* freqs, uint32_t nf,
                           const mcsbr_mc_config* cfg, uint32_t shard, uint32_t nshard, double* d_sums,
                           uint64_t* d_counters, void* stream) {
    if (!s) return set_err(MCSBR_EINVAL, "null scene");
    if (!d_sums || !d_counters) return set_err(MCSBR_EINVAL, "trace_device: null device buffer");
    int rc = use_device(s);
    if (rc) return rc;
    Job job;
    rc = plan_job(s, incs, n_inc, rxs, n_rx, freqs, nf, cfg, shard, nshard, s->sms * 16, &job);
    if (rc) return rc;
    return run_job(s, job, nf, cfg, occlusion, d_sums, reinterpret_cast<unsigned long long*>(d_counters),
                   static_cast<cudaStream_t>(stream), nullptr, nullptr,
                   cfg->reduction == MCSBR_REDUCE_EXACT ? reinterpret_cast<long long*>(d_sums) : nullptr);
}

int mcsbr_gpu_finalize(const double* raw, uint32_t n, const double* freqs, uint32_t nf, double* values) {
    if (!raw || !freqs || !values) return set_err(MCSBR_EINVAL, "finalize: null argument");
    finalize_values(raw, n, freqs, nf, values);
    return MCSBR_OK;
}

int mcsbr_gpu_finalize_exact(const int64_t* limbs, uint32_t n, const double* freqs, uint32_t nf, double* values) {
    if (!limbs || !freqs || !values) return set_err(MCSBR_EINVAL, "finalize_exact: null argument");
    const size_t nsum = static_cast<size_t>(n) * nf * 8;
    std::vector<double> raw(nsum);
    limbs_to_doubles(reinterpret_cast<const long long*>(limbs), nsum, raw.data());
    finalize_values(raw.data(), n, freqs, nf, values);
    return MCSBR_OK;
}

int mcsbr_gpu_decode_counters(const uint64_t* counters, mcsbr_stats* stats) {
    if (!counters || !stats) return set_err(MCSBR_EINVAL, "decode_counters: null argument");
    decode(reinterpret_cast<const unsigned long long*>(counters), stats);
    return fault_check(reinterpret_cast<const unsigned long long*>(counters));
}

}  // extern "C"
