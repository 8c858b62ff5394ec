// Internal (non-ABI) structures shared by the host orchestration (capi.cu),
// the BVH builder (bvh.cu) and the path kernel (trace.cu).
//
// Device memory layout of a scene (all arrays 16-byte aligned, SoA-by-record):
//   nodes      BVH4, 128 B per node = 8 x float4, child boxes SoA by axis:
//                [0] lo.x of children 0..3   [1] hi.x   [2] lo.y   [3] hi.y
//                [4] lo.z                    [5] hi.z
//                [6] child refs as int bits: ref >= 0 inner node,
//                    ref < 0 leaf: ~ref = (first << 3) | count (count <= MCSBR_LEAF_MAX)
//                [7] (child count, -, -, -)
//              child boxes are fp32 in a frame centred on the scene's
//              bounding sphere, the fp64 triangle boxes rounded outward (no
//              padding): the slab test's rounding margin lives on the ray
//              (trace.cu make_fray), so the fp32 descent can only over-accept.
//   tri64      per leaf-ordered triangle 5 x double2 = 80 B:
//                (a.x, a.y) (a.z, e1.x) (e1.y, e1.z) (e2.x, e2.y) (e2.z, id)
//              e1 = b - a, e2 = c - a in fp64: exactly the values the
//              reference's ray_triangle forms (geometry.cpp:20-39).
//   tri_info   per original triangle id: 2 x double2 (normal.xyz, packed)
//              packed = front | back << 16 | exterior << 32 (as uint64 bits)
//   mat        per material: double2 (index, is_pec)
#pragma once

#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

namespace mcsbr_int {

constexpr int kStackSize = 96;  // >= 3 pushes per 4-wide level
#ifndef MCSBR_LEAF_MAX
#define MCSBR_LEAF_MAX 2  // measured: 2 beats 1, 3, 4 on c1-c5 (fp64 triangle tests cost more than node visits)
#endif
constexpr int kLeafMax = MCSBR_LEAF_MAX;

struct SceneView {
    const float4* nodes;
    const double2* tri64;
    const double2* tri_info;  // 2 per triangle
    const double2* mat;
    int32_t root_ref;
    uint32_t n_tri;
    double diameter;
    double t_eps;      // 1e-6 * diameter (geometry.hpp:78)
    double ambient_n;  // materials[0].index()
    int32_t all_pec;   // every triangle has a PEC side: dielectric code compiled out
    int32_t lossy;     // complex-permittivity transport (eps_imag given at scene creation)
    const double* mat_nim;  // per material Im(n) (lossy scenes), else nullptr
    const float4* tri32;    // leaf-ordered fp32 triangle records (3 float4: a - centre, e1, e2, id) for the
                            // statistical-mode fast path, built on first use; else nullptr
    double center[3];  // bounding-sphere centre: origin of the fp32 box frame
    double skip_radius;  // bounding radius + margin (traversal origin advance)
    float margin_r;      // bounding radius (fp32): scale of the slab-test ray margin
};

// Per incidence (one launch aperture), host-planned in fp64.
struct IncDev {
    double center[3], u[3], v[3];
    double half_u, half_v;
    double k_inc[3], pol_v[3], pol_h[3];
    double area_weight;       // cell_area / spp
    int32_t nu, nv;
    // One launch unit: a range of the incidence's dispatch indices.  A
    // single-shard job has one unit per incidence; a sharded job gives each
    // shard interleaved stripes of every incidence (capi.cu plan_job), each
    // stripe a unit with the incidence's geometry.
    uint64_t entry_begin;     // this unit's dispatch range [begin, end)
    uint64_t entry_end;
    uint64_t g_begin;         // index of entry_begin in the launch's flattened entry space
    uint64_t cover_off;       // launch-ray coverage bitmap (cover.cu): first word, kNoCover = none
    uint32_t cover_shift;     // log2 of the launch entries per coverage bit
    uint32_t row;             // the incidence, relative to the launch's first (sums, receivers, records)
};
constexpr uint64_t kNoCover = ~uint64_t{0};
constexpr uint64_t kCoverMaxBits = uint64_t{1} << 19;  // 64 KB of shared memory per incidence

struct RxDev {
    double k_s[3], rx_v[3], rx_h[3];
};

// counters block (MCSBR_COUNTER_WORDS = 256 uint64)
enum : int {
    kCntLaunched = 0,
    kCntSegments = 1,
    kCntContrib = 2,
    kCntGrazing = 3,
    kCntCap = 4,
    kCntOcclusion = 5,
    kCntFault = 6,  // OR of fault bits (stored via atomicOr)
    kCntRounds = 7, // max bounce index seen (atomicMax)
    kCntRaysPerBounce = 8,
    kCntRouletteCand = 72,
    kCntRouletteSurv = 136,
    kCntCulled = 200,  // launch entries retired by the coverage bitmap (provable bounce-0 misses)
    kCntWords = 256,
};

struct TraceParams {
    SceneView scene;
    const IncDev* inc;      // this launch's units (the incidences of a group of the job)
    uint32_t n_inc;
    uint32_t inc_base;      // job index of the launch's first incidence (RNG keys, path log)
    uint32_t n_rx;          // receivers per incidence
    uint32_t rx_index;      // receiver traced by this launch (fan: the first of up to 32)
    int fan;                // bistatic fan mode (up to 32 receivers per launch)
    uint32_t fan_rows;      // fan with nf > 1 (deferred records): 32, and a record's row is
                            // 32 * incidence + receiver lane (sums_row); else 0
    const RxDev* rx;        // [n_inc * n_rx]
    const double* k0;       // [nf] wavenumbers 2*pi*f/c
    uint32_t nf;
    int occlusion;
    double* sums;           // [n_inc][n_rx][nf][4] complex (re, im)
    const uint32_t* cover;  // launch-ray coverage bitmaps (IncDev::cover_off), or nullptr
    unsigned long long* xsums;  // MCSBR_REDUCE_EXACT: 192-bit fixed-point sums, 3 words per value of `sums`
    // deferred accumulation (F > 1): contribution records of this launch
    double* recs;                      // [rec_cap][12]: amp[4], s (re, im), incidence
    unsigned long long* rec_count;
    uint64_t rec_cap;
    uint32_t* rec_inc;                 // [rec_cap] each record's incidence again, packed (spread.cu buckets), or nullptr
    unsigned long long* counters;
    unsigned long long* tile_counter;  // global cursor over the flattened entry space
    uint64_t total_entries;            // entries of all incidences (this shard)
    uint32_t chunk_max;                // largest chunk a warp takes at once
    uint32_t chunk_min;                // smallest chunk (multiple of 32)
    uint32_t gss_div;                  // chunk = remaining / (gss_div * warps); 0 = always chunk_max
    int32_t band_order;                // dispatch order of launch entries (trace.cu locate)
    // uniform frequency grid (SweepAccumulator::uniform_, farfield.cpp:87-104):
    // phase of frequency i is (kph0 + i * kdph) * s, kph0 = -2 pi f0 / c,
    // kdph = -2 pi df / c, exactly the reference's operation order
    int32_t uniform_f;
    double kph0, kdph;
    // McConfig
    uint32_t spp;
    uint64_t seed;
    int32_t max_bounce;
    int32_t fresnel_strategy;
    double p_min;
    int32_t roulette_enabled;
    int32_t roulette_min_bounce;
    double roulette_q;
    int32_t jitter;
    int32_t rng_mode;
    int32_t fast_tri;       // statistical-mode fp32 triangle tests (parity_fp64_refine = 0)
    // debug / parity instrumentation (all optional)
    void* contrib_out;                       // mcsbr_contribution[contrib_cap]
    unsigned long long* contrib_count;
    uint64_t contrib_cap;
    void* contrib_scratch;                   // one record per resident thread
    uint32_t* plog_tri;                      // [plog_n][plog_stride] (incidence 0 only)
    uint8_t* plog_term;
    unsigned long long* plog_branch;
    uint64_t plog_n;
    uint32_t plog_stride;
    // deterministic solver (solver_det.cpp): every branch explored depth-first
    int det;                                 // 1 = deterministic mode
    double det_cutoff;                       // amplitude_cutoff (0 = off)
    double* det_stack;                       // [kDetFields][det_depth][det_threads]
    uint32_t det_depth;                      // stack entries per thread (max_bounce)
    uint64_t det_threads;                    // threads the stack was sized for
    unsigned long long* det_blocks;          // [n_blocks][2]: sum peak depth, sum pushes
    uint64_t det_block_size;                 // cells per accounting block
};

// Row of the [incidence][receiver] sums that a contribution record's row
// index `a` adds into: an incidence of this launch (receiver rx_index), or,
// in a multi-frequency bistatic fan (fan_rows = 32), receiver rx_index + a % 32
// of incidence a / 32.
#ifdef __CUDACC__
__host__ __device__ __forceinline__ size_t sums_row(const TraceParams& P, uint32_t a) {
    return P.fan_rows ? static_cast<size_t>(a >> 5) * P.n_rx + P.rx_index + (a & 31u)
                      : static_cast<size_t>(a) * P.n_rx + P.rx_index;
}
#endif
constexpr int kDetFields = 24;  // origin 3, dir 3, e0 6, e1 6, phi 2, medium 2, bounce 1 (+1 spare)
// branch stacks are sized for 4 resident 128-thread blocks per SM (the path
// kernel's launch bound); launch_trace caps a det grid at the stack capacity
#define MCSBR_DET_THREADS_PER_SM 512

// capi.cu: caching device allocator.  Scene creation / destruction and the
// BVH build allocate and free dozens of buffers; cudaMalloc / cudaFree cost
// driver round trips (and, on a busy host, occasionally tens of ms), so
// freed blocks are kept per device (bounded) and handed out again.  A free
// synchronises the device first, so a cached block is never still in use.
cudaError_t dev_malloc(void** p, size_t bytes);
void dev_free(void* p, bool synced = false);
template <typename T>
inline cudaError_t dev_malloc(T** p, size_t bytes) {
    return dev_malloc(reinterpret_cast<void**>(p), bytes);
}

// bvh.cu
struct BvhBuildOut {
    float4* nodes;
    double2* tri64;
    uint32_t n_nodes;
    int32_t root_ref;
    uint32_t max_depth;
    uint32_t n_leaves;
    float build_ms;
};
// Builds the BVH on `stream` from device vertices / triangle indices.
// Returns a cudaError_t; fills *out (device arrays owned by the caller).
cudaError_t build_bvh(const double* d_vertices, const uint4* d_tri_idx, uint32_t n_tri,
                      const double scene_lo[3], const double scene_hi[3], const double center[3],
                      double box_pad,
                      cudaStream_t stream, BvhBuildOut* out);

// wavefront.cu: the pool of paths between the shading and traversal kernels
struct WfParams {
    double* pool;                      // [kWfFields][np] doubles (wavefront.cu field map)
    uint32_t np;                       // slots, a multiple of 128
    uint32_t* kind;                    // [np] query kind (0 none / launch / surface / occlusion)
    uint32_t* rid;                     // [np] query result: triangle id or 0xffffffff
    uint32_t* list;                    // [np] work list of the next traversal
    unsigned long long* list_n;        // [3] work-list lengths (rotating per iteration)
    unsigned long long* trace_cursor;  // [3] traversal cursors (rotating per iteration)
    unsigned long long* wrange;        // [np / 32][2] each warp's launch-entry range
};
constexpr int kWfFieldsHost = 41;
cudaError_t launch_wavefront_iteration(const TraceParams& p, const WfParams& w, uint32_t iter, int device_sms,
                                       cudaStream_t stream);

// prep.cu: scene preparation and launch planning on the device
}  // namespace mcsbr_int
struct mcsbr_triangle;
namespace mcsbr_int {
double unord(unsigned long long o);  // inverse of the order-preserving double -> uint64 map
cudaError_t launch_pack(const mcsbr_triangle* d_raw, uint32_t nt, uint32_t nv, uint32_t nm, const uint8_t* d_is_pec,
                        uint4* d_tri, double2* d_info, unsigned long long* d_first_bad, unsigned int* d_not_all_pec,
                        cudaStream_t stream);
cudaError_t launch_bounds(const double* d_vtx, uint32_t nv, unsigned long long* d_out, int device_sms,
                          cudaStream_t stream);
cudaError_t launch_radius(const double* d_vtx, uint32_t nv, const double c[3], unsigned long long* d_out,
                          int device_sms, cudaStream_t stream);
// leaf-ordered fp32 triangle records for the statistical-mode fast path
// sort.cu: stable LSD radix sort of (u64 key, u32 value) pairs over the low
// key_bits bits (8 per pass; *result_in_alt: the sorted pairs are in the
// *_alt buffers), and an exclusive u32 prefix sum; temp of the *_temp_bytes size
size_t radix_sort_temp_bytes(uint32_t n);
cudaError_t radix_sort_pairs(uint64_t* keys, uint64_t* keys_alt, uint32_t* vals, uint32_t* vals_alt, uint32_t n,
                             int key_bits, void* temp, cudaStream_t stream, bool* result_in_alt);
size_t scan_temp_bytes(uint32_t n);
cudaError_t exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint32_t n, void* temp, cudaStream_t stream);
cudaError_t launch_leaf32(const double2* tri64, uint32_t n, const double center[3], double radius, float4* out,
                         cudaStream_t stream);
cudaError_t launch_extents(const double* d_vtx, uint32_t nv, const double* d_axes, uint32_t n_inc,
                           unsigned long long* d_out, int device_sms, cudaStream_t stream);

// cover.cu: launch-ray coverage bitmaps
cudaError_t build_tri32(const double* d_vtx, const uint4* d_tri, uint32_t n, const double center[3], float* out,
                        cudaStream_t stream);
uint32_t cover_shift_for(uint64_t entries);
cudaError_t launch_cover(const IncDev* d_inc, uint32_t n_inc, const float* tri32, uint32_t n_tri,
                         const double center[3], double radius, uint32_t spp, uint32_t band, uint32_t* out,
                         uint64_t out_words, int device_sms, cudaStream_t stream);

// trace.cu
cudaError_t launch_trace(const TraceParams& p, int device_sms, cudaStream_t stream,
                         uint64_t* launches);
// exact sums (3 words per value) -> 48-bit limbs ADDED into limbs (4 per value)
cudaError_t launch_exact_limbs(const unsigned long long* xsums, uint64_t n_values, long long* limbs,
                               cudaStream_t stream);
cudaError_t launch_accumulate(const TraceParams& p, int device_sms, cudaStream_t stream, uint64_t* launches,
                              uint64_t expected_records = 0);
cudaError_t launch_intersect(const SceneView& s, const double* o, const double* d,
                             const double* tmin, uint32_t n, int any_hit, double* t_out,
                             uint32_t* id_out, cudaStream_t stream);
// spread.cu: deferred accumulation on uniform frequency grids as a type-1
// non-uniform DFT (records spread onto a 2F-point grid, then one small DFT
// per incidence)
struct NufftPlan {
    uint32_t ng;             // grid points (2 nf)
    uint32_t fc;             // centre frequency index (nf / 2)
    double beta;             // kernel shape
    double kc;               // kph0 + fc * kdph
    double u2t;              // kdph * ng / (2 pi): grid cells per unit path length
    double eta_poly;         // |Im t| up to which the kernel polynomial is continued (0.1 cells)
    double eta_max;          // |Im t| above which a record is added directly (0.5 cells)
    double* grid;            // [n_inc][8][ng] (group incidences)
    const double* inv_hat;   // [nf] 1 / Psi(f - fc)
    const double* coef;      // [16][kNufftPolyN] psi per window point, monomials in 2 delta - 1
    uint32_t* idx;           // [rec_cap] record indices ordered by incidence (or nullptr)
    uint32_t* bucket;        // [2 (n_inc + 1)] per-incidence counts, then cursors
};
constexpr int kNufftPolyN = 14;
constexpr uint32_t kNufftSortMaxInc = 4096;  // larger groups spread in record order
bool nufft_supported(uint32_t nf);
size_t nufft_grid_values(uint32_t nf);  // doubles per incidence
void nufft_tables(uint32_t nf, uint32_t ng, double beta, std::vector<double>& inv_hat, std::vector<double>& coef);
cudaError_t launch_spread(const TraceParams& p, const NufftPlan& q, uint32_t n_inc, int device_sms,
                          cudaStream_t stream, uint64_t* launches, uint64_t expected_records);
// general-F / receiver mode selection helpers
bool trace_uses_register_accumulator(const TraceParams& p);
bool trace_fan_supported(uint32_t nf);

}  // namespace mcsbr_int
