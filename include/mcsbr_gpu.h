/*
 * mcsbr_gpu.h — C ABI of the B200-native Monte Carlo SBR estimator.
 *
 * Drop-in boundary for the reference's CPU solver entry point
 *     McResult mcsbr::estimate(const Scene&, const Excitation&,
 *                              const std::vector<double>& frequencies,
 *                              const McConfig&, int workers,
 *                              std::vector<Contribution>* contributions_out)
 * declared at reference proj/include/mcsbr/solver_mc.hpp:81-83 and defined at
 * proj/src/solver_mc.cpp:76-229.  The reference has no FFI of its own; every
 * struct below is a plain-old-data mirror of the reference's boundary type,
 * laid out so that the reference's own objects can be passed by pointer
 * (see INTEGRATION.md for the adapter a maintainer adds to run_solver).
 *
 * Conventions (identical to the reference, proj/include/mcsbr/em_math.hpp:6-9):
 * time factor e^{+j w t}, spatial phase e^{-j k0 phi}, lengths in metres,
 * polarisation channels ordered VV, HH, VH, HV (receive letter first,
 * proj/include/mcsbr/farfield.hpp:61-63).  Complex numbers are interleaved
 * (re, im) doubles.
 *
 * Errors: every function returns 0 on success or a negative MCSBR_E* code and
 * leaves a thread-local message readable through mcsbr_gpu_last_error().
 * There is no CPU fallback: without a usable sm_100 device every compute
 * entry point fails with MCSBR_ECUDA.
 */
#ifndef MCSBR_GPU_H_
#define MCSBR_GPU_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MCSBR_API __attribute__((visibility("default")))
#else
#define MCSBR_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define MCSBR_GPU_ABI_VERSION 3

/* ---- status codes ------------------------------------------------------ */
#define MCSBR_OK 0
#define MCSBR_EINVAL (-1)  /* invalid argument; message mirrors the reference's std::invalid_argument text */
#define MCSBR_ENOMEM (-2)  /* device or host allocation failed */
#define MCSBR_ECUDA (-3)   /* CUDA runtime error / no device */
#define MCSBR_ESCENE (-4)  /* scene rejected (reference SceneError) */
#define MCSBR_EDEVICE (-5) /* in-kernel fault: a reference throw site was reached (DomainError) */

/* ---- boundary PODs ------------------------------------------------------ */

/* Mirrors mcsbr::Triangle (proj/include/mcsbr/geometry.hpp:23-29), 48 bytes,
 * byte-compatible with the reference layout on LP64. */
typedef struct mcsbr_triangle {
    uint32_t v0, v1, v2;
    uint32_t _pad0;
    double normal[3];         /* unit, from winding order */
    uint16_t front_material;  /* medium on the side the normal points to */
    uint16_t back_material;
    uint8_t exterior_facing;  /* borders the ambient medium (material 0) */
    uint8_t _pad1[3];
} mcsbr_triangle;

/* Mirrors mcsbr::Material (proj/include/mcsbr/em_math.hpp:99-105), 24 bytes.
 * The lossy-permittivity extension (Im eps) is passed separately to
 * mcsbr_gpu_scene_create so this struct stays layout-compatible. */
typedef struct mcsbr_material {
    double eps_r;
    double mu_r;
    uint8_t is_pec;
    uint8_t _pad[7];
} mcsbr_material;

/* Mirrors mcsbr::Excitation (proj/include/mcsbr/solver_common.hpp:16-22). */
typedef struct mcsbr_excitation {
    double k_inc[3];
    double pol_v[3], pol_h[3];
    double k_scatter[3];
    double rx_v[3], rx_h[3];
    uint8_t occlusion_enabled;
    uint8_t _pad[7];
} mcsbr_excitation;

/* Batched sweeps: one incidence (a launch aperture and its paths) ... */
typedef struct mcsbr_incidence {
    double k_inc[3];
    double pol_v[3], pol_h[3];
    double strata_per_wavelength; /* > 0 overrides the config value for this incidence */
} mcsbr_incidence;

/* ... observed by one or more receivers (bistatic fan, or the monostatic one). */
typedef struct mcsbr_receiver {
    double k_scatter[3];
    double rx_v[3], rx_h[3];
} mcsbr_receiver;

#define MCSBR_BRANCH_FIFTY_FIFTY 0
#define MCSBR_BRANCH_FRESNEL 1

#define MCSBR_RNG_REFERENCE 0 /* parity mode: the reference counter_hash stream (rng.hpp:29-44) */
#define MCSBR_RNG_PHILOX 1    /* statistical mode: Philox4x32-10 keyed by (seed, ray index) */

#define MCSBR_MAX_BOUNCE_LIMIT 64

/* Far-field reduction (mcsbr_mc_config.reduction).  FAST sums contributions
 * with fp64 atomics in whatever order the GPU schedules them (rerun-to-rerun
 * differences in the last bits).  EXACT converts every (contribution,
 * frequency, channel) term to a 192-bit fixed-point integer (LSB 2^-120,
 * range +-2^71) and sums integers, which is associative: the result is
 * byte-identical across reruns, launch groupings and shard / GPU counts,
 * like the reference's fixed-order block merge (solver_mc.cpp:212-216,
 * runner.hpp:2-5).  Raw device sums of EXACT jobs are 4 int64 limbs of 48
 * bits per fp64 value (MCSBR_EXACT_LIMBS), summable across ranks with any
 * integer all-reduce and finalized by mcsbr_gpu_finalize_exact. */
#define MCSBR_REDUCE_FAST 0
#define MCSBR_REDUCE_EXACT 1
#define MCSBR_EXACT_LIMBS 4

/* Mirrors mcsbr::McConfig + RouletteConfig (proj/include/mcsbr/solver_mc.hpp:14-36),
 * plus the GPU-only rng_mode.  mcsbr_gpu_default_config() returns the
 * reference defaults. */
typedef struct mcsbr_mc_config {
    double strata_per_wavelength; /* 10 */
    int32_t samples_per_stratum;  /* 16 */
    int32_t branch_strategy;      /* MCSBR_BRANCH_FRESNEL */
    int32_t roulette_enabled;     /* 0 */
    int32_t roulette_min_bounce;  /* 2 */
    double roulette_q;            /* 0.5 */
    int32_t max_bounce;           /* 9, at most MCSBR_MAX_BOUNCE_LIMIT */
    int32_t jitter;               /* 1 */
    uint64_t seed;                /* 1 */
    double reference_wavelength;  /* 0 = c / max(frequencies) */
    double launch_padding;        /* 0 m */
    double p_min;                 /* 0.05 */
    int32_t block_size;           /* 8192 (validated only; the GPU has no CPU blocks) */
    int32_t rng_mode;             /* MCSBR_RNG_REFERENCE */
    int32_t reduction;            /* MCSBR_REDUCE_FAST */
    int32_t parity_fp64_refine;   /* 1: every triangle test in the reference's fp64 arithmetic (parity);
                                     0: statistical-mode fast path (fp32 triangle tests, PHILOX only) */
} mcsbr_mc_config;

/* Mirrors mcsbr::RunStats (proj/include/mcsbr/solver_common.hpp:37-53). */
typedef struct mcsbr_stats {
    uint64_t rays_launched;
    uint64_t segments_traced;
    uint64_t contributions;   /* contributions accumulated (per receiver) */
    uint64_t grazing_kills;
    uint64_t cap_kills;
    uint64_t occlusion_queries;
    uint64_t peak_live_state_bytes;
    uint64_t state_bytes_per_ray;
    uint64_t block_size;
    uint32_t n_rounds;        /* valid entries of the per-bounce arrays */
    uint32_t _pad;
    uint64_t rays_per_bounce[MCSBR_MAX_BOUNCE_LIMIT];
    uint64_t roulette_candidates[MCSBR_MAX_BOUNCE_LIMIT];
    uint64_t roulette_survivors[MCSBR_MAX_BOUNCE_LIMIT];
    double wall_ms;           /* host wall time of the call */
    double kernel_ms;         /* device time of the path kernel (CUDA events) */
    /* deterministic solver only (solver_det.cpp:119-132): the reference's
     * "all rays of a block in flight" accounting, max over blocks of the sum
     * over rays of peak-depth (resp. every snapshot pushed) x sizeof(PathState)
     * = 192 B; the GPU's actual branch-stack allocation is device_stack_bytes. */
    uint64_t forced_stack_bytes;
    uint64_t device_stack_bytes;
    /* launch rays retired without tracing because no triangle's projection
     * meets their strata group (provable misses; still counted in
     * rays_launched and rays_per_bounce[0] exactly as the reference counts
     * a launch ray that escapes) */
    uint64_t culled_launch_rays;
} mcsbr_stats;

/* Mirrors mcsbr::DetConfig (proj/include/mcsbr/solver_det.hpp:12-22).
 * mcsbr_gpu_default_det_config() returns the reference defaults. */
typedef struct mcsbr_det_config {
    double rays_per_wavelength;     /* 20 */
    int32_t max_bounce;             /* 9, at most MCSBR_MAX_BOUNCE_LIMIT */
    int32_t force_stack_accounting; /* 0 (accepted; both stack figures are always reported) */
    double amplitude_cutoff;        /* 0 = disabled; kill branches with max |E| < cutoff */
    double launch_padding;          /* 0 m */
    double reference_wavelength;    /* 0 = c / max(frequencies) */
    int32_t block_size;             /* 8192 launch cells per accounting block */
    int32_t _pad;
} mcsbr_det_config;

/* Mirrors mcsbr::Contribution (proj/include/mcsbr/farfield.hpp:45-52), 240 bytes. */
typedef struct mcsbr_contribution {
    double a_j[2][3][2]; /* [tx pol][xyz][re,im], eta0 * J with all weights */
    double a_m[2][3][2];
    double phi_total;
    double exit_point[3];
    int32_t bounce;
    int32_t _pad;
    uint64_t order_key;  /* ((cell*spp + sample) << 8) | bounce, solver_mc.cpp:166-168 */
} mcsbr_contribution;

/* Launch aperture (mcsbr::LaunchRect, geometry.hpp:45-53) and strata grid. */
typedef struct mcsbr_launch_plan {
    double center[3];
    double u_axis[3], v_axis[3];
    double half_u, half_v;
    int32_t nu, nv;
    double cell_area;
    uint64_t entries;  /* nu * nv * samples_per_stratum */
} mcsbr_launch_plan;

/* ---- API ---------------------------------------------------------------- */

MCSBR_API const char* mcsbr_gpu_last_error(void);
MCSBR_API int mcsbr_gpu_abi_version(void);
MCSBR_API void mcsbr_gpu_default_config(mcsbr_mc_config* cfg);

/* Mirrors McConfig::validate (proj/src/solver_mc.cpp:10-17). */
MCSBR_API int mcsbr_gpu_validate_config(const mcsbr_mc_config* cfg);

typedef struct mcsbr_scene mcsbr_scene;

/* Upload a finalized scene (the public data of mcsbr::Scene,
 * geometry.hpp:55-60) to `device` and build its BVH on the GPU (binned-SAH
 * top-down build from a Morton order with early split clipping of sliver
 * triangles, collapsed to a 4-wide tree of outward-rounded fp32 boxes; the
 * Karras LBVH is the fallback for trees deeper than the traversal stack).
 * `eps_imag` may be NULL (lossless, the reference
 * model) or hold nm values of Im(eps_r) (e^{+jwt}: eps = eps_r - j eps_imag,
 * the GPU-only lossy extension).  Validates as Scene::finalize does
 * (geometry.cpp:146-162): empty or zero-extent scenes are rejected. */
MCSBR_API int mcsbr_gpu_scene_create(const double* vertices_xyz, uint32_t n_vertices,
                           const mcsbr_triangle* triangles, uint32_t n_triangles,
                           const mcsbr_material* materials, uint32_t n_materials,
                           const double* eps_imag, int device, mcsbr_scene** out);
MCSBR_API void mcsbr_gpu_scene_destroy(mcsbr_scene* scene);

/* A scene on several devices (replaces run_blocks' worker threads,
 * proj/src/solver_common.cpp:70-89, by GPUs): the BVH is built once on
 * devices[0] and its arrays are copied to devices[1..] (peer copies over
 * NVLink).  estimate() with workers = w shards every incidence's launch
 * entries over min(w, n_devices) devices (workers <= 0: all of them),
 * estimate_batch() over all of them; one host thread and stream per device,
 * partial sums added on the host in device order (MCSBR_REDUCE_EXACT: the
 * result is byte-identical to a single device's).  Parity instrumentation
 * (contributions, path logs) and the deterministic solver run on devices[0].
 * A device may be listed more than once (independent streams on one GPU). */
MCSBR_API int mcsbr_gpu_scene_create_multi(const double* vertices_xyz, uint32_t n_vertices,
                                           const mcsbr_triangle* triangles, uint32_t n_triangles,
                                           const mcsbr_material* materials, uint32_t n_materials,
                                           const double* eps_imag, const int* devices, int n_devices,
                                           mcsbr_scene** out);
MCSBR_API int mcsbr_gpu_scene_devices(const mcsbr_scene* scene, int* n_devices);
MCSBR_API int mcsbr_gpu_device_count(int* n_devices);

/* Scene::diameter / bounding_center / bounding_radius (geometry.hpp:77-80). */
MCSBR_API int mcsbr_gpu_scene_bounds(const mcsbr_scene* scene, double center[3], double* radius,
                           double* diameter);
/* BVH shape (for tests and the roofline model): node count, depth, leaves. */
MCSBR_API int mcsbr_gpu_scene_bvh_info(const mcsbr_scene* scene, uint32_t* n_nodes, uint32_t* max_depth,
                             uint32_t* n_leaves, double* build_ms);

/* launch_rect + build_strata on the host in fp64, identical to
 * geometry.cpp:246-275 and solver_mc.cpp:19-31. */
MCSBR_API int mcsbr_gpu_launch_plan(const mcsbr_scene* scene, const double k_inc[3], double padding,
                          double strata_per_wavelength, double reference_wavelength,
                          int32_t samples_per_stratum, mcsbr_launch_plan* out);

/* Batched closest-hit queries (Scene::intersect, geometry.cpp:177-216) with
 * host arrays: origins/dirs are n*3 doubles.  Outputs t (inf on miss) and
 * triangle id (UINT32_MAX on miss).  any_hit=1 answers Scene::occluded-style
 * existence queries (t/id then hold an arbitrary hit). */
MCSBR_API int mcsbr_gpu_intersect(const mcsbr_scene* scene, const double* origins, const double* dirs,
                        const double* t_min, uint32_t n, int any_hit, double* t_out,
                        uint32_t* id_out);

/* Device-pointer variant of mcsbr_gpu_intersect (no copies, no sync), on
 * `stream` (cudaStream_t): d_origins / d_dirs n*3 doubles, d_t_min n doubles,
 * outputs d_t / d_ids. */
MCSBR_API int mcsbr_gpu_intersect_device(const mcsbr_scene* scene, const double* d_origins,
                                         const double* d_dirs, const double* d_t_min, uint32_t n,
                                         int any_hit, double* d_t, uint32_t* d_ids, void* stream);

/* The drop-in: one Excitation, host buffers in and out.  values receives
 * [4][nf] complex (interleaved) sqrt(m^2) values, channel order VV,HH,VH,HV,
 * finalized with j*k0/(2 sqrt(pi)) as SweepAccumulator::finalize does
 * (farfield.cpp:154-167).  `workers`: the number of the scene's devices to
 * shard over (see mcsbr_gpu_scene_create_multi; 1 for a single-device
 * scene).  If contributions != NULL, up to capacity records are written
 * sorted by order_key (the reference emits them in block order, which is the
 * same order for one block) and *n_contributions receives the total count. */
MCSBR_API int mcsbr_gpu_estimate(mcsbr_scene* scene, const mcsbr_excitation* excitation,
                       const double* frequencies, uint32_t n_frequencies,
                       const mcsbr_mc_config* config, int workers, double* values,
                       mcsbr_stats* stats, mcsbr_contribution* contributions,
                       uint64_t capacity, uint64_t* n_contributions);

/* Deterministic SBR (mcsbr::solve, proj/src/solver_det.cpp:30-174): midpoint
 * launch grid, every reflect/transmit branch explored depth-first (reflect
 * first) with per-thread branch stacks in HBM.  Same buffers and semantics as
 * mcsbr_gpu_estimate; contributions carry order_key = cell << 24 | event
 * index, as the reference keys them (solver_det.cpp:104-105). */
MCSBR_API void mcsbr_gpu_default_det_config(mcsbr_det_config* cfg);
/* Mirrors DetConfig::validate (proj/src/solver_det.cpp:11-17). */
MCSBR_API int mcsbr_gpu_validate_det_config(const mcsbr_det_config* cfg);
MCSBR_API int mcsbr_gpu_solve(mcsbr_scene* scene, const mcsbr_excitation* excitation,
                              const double* frequencies, uint32_t n_frequencies,
                              const mcsbr_det_config* config, int workers, double* values,
                              mcsbr_stats* stats, mcsbr_contribution* contributions,
                              uint64_t capacity, uint64_t* n_contributions);

/* Batched sweeps in ONE device launch (per device of a multi-device scene):
 * n_inc incidences, each observed by
 * n_rx receivers (receivers[i*n_rx + r]); occlusion applies to all.  values
 * receives [n_inc][n_rx][4][nf] complex.  Equivalent to n_inc*n_rx calls of
 * mcsbr_gpu_estimate except that each incidence is traced once for all its
 * receivers (valid because the path state does not depend on the receiver). */
MCSBR_API int mcsbr_gpu_estimate_batch(mcsbr_scene* scene, const mcsbr_incidence* incidences,
                             uint32_t n_inc, const mcsbr_receiver* receivers, uint32_t n_rx,
                             int occlusion_enabled, const double* frequencies,
                             uint32_t n_frequencies, const mcsbr_mc_config* config,
                             double* values, mcsbr_stats* stats);

/* Device-resident variant for multi-GPU sharding and benchmarking: traces
 * shard shard_index of shard_count of every incidence's launch entries and
 * ADDS raw
 * (un-finalized) sums into the caller's device buffer d_sums
 * ([n_inc][n_rx][nf][4] complex; for MCSBR_REDUCE_EXACT configs int64 limbs
 * [n_inc][n_rx][nf][8][MCSBR_EXACT_LIMBS]) and counters into d_counters
 * (MCSBR_COUNTER_WORDS uint64), on `stream` (a cudaStream_t, NULL = legacy
 * default).  Asynchronous: no host synchronisation.  The caller all-reduces
 * the buffers (NCCL) and finalizes with mcsbr_gpu_finalize.  A shard is
 * every shard_count-th stripe of the incidence's dispatch indices (stripes
 * of S = max(1024, ceil(entries / (32 shard_count)) rounded up to 1024),
 * stripe k to shard k mod shard_count), so the shards balance whatever the
 * target's silhouette; paths do not depend on the shard count. */
#define MCSBR_COUNTER_WORDS 256
MCSBR_API int mcsbr_gpu_trace_device(mcsbr_scene* scene, const mcsbr_incidence* incidences,
                           uint32_t n_inc, const mcsbr_receiver* receivers, uint32_t n_rx,
                           int occlusion_enabled, const double* frequencies,
                           uint32_t n_frequencies, const mcsbr_mc_config* config,
                           uint32_t shard_index, uint32_t shard_count, double* d_sums,
                           uint64_t* d_counters, void* stream);

/* Apply j*k0/(2 sqrt(pi)) to raw sums [n][nf][4] and transpose to the
 * [n][4][nf] output layout (host arrays). */
MCSBR_API int mcsbr_gpu_finalize(const double* raw_sums, uint32_t n, const double* frequencies,
                       uint32_t n_frequencies, double* values);
/* The same for the raw sums of an MCSBR_REDUCE_EXACT job: limbs
 * [n][nf][8][MCSBR_EXACT_LIMBS] int64 (possibly summed over ranks). */
MCSBR_API int mcsbr_gpu_finalize_exact(const int64_t* limbs, uint32_t n, const double* frequencies,
                                       uint32_t n_frequencies, double* values);

/* Decode a counter block (device layout above, copied to host) into stats. */
MCSBR_API int mcsbr_gpu_decode_counters(const uint64_t* counters, mcsbr_stats* stats);

/* ---- radar products (reference proj/src/signal_processing.cpp) ----
 * Computed on the current CUDA device from host arrays.  Errors mirror the
 * reference's SignalError messages (MCSBR_EINVAL). */
#define MCSBR_WINDOW_NONE 0
#define MCSBR_WINDOW_HANN 1

/* range_profile (signal_processing.cpp:66-89): windowed, zero-padded inverse
 * DFT of one channel's sweep (values: nf complex), centre-shifted; outputs
 * nf*zero_pad range bins (m) and 20 log10 |.|. */
MCSBR_API int mcsbr_gpu_range_profile(const double* values, const double* frequencies,
                                      uint32_t n_frequencies, int window, int zero_pad,
                                      double* range_m, double* mag_db, double* bin_spacing);

/* isar (signal_processing.cpp:91-162): small-angle range-Doppler image from
 * one channel's sweeps over a uniform azimuth grid (values: [na][nf]
 * complex).  Outputs down_range_m[nf*zp], cross_range_m[na*zp],
 * mag_db[(nf*zp) x (na*zp)] row-major (clipped at peak + floor), *peak_db. */
MCSBR_API int mcsbr_gpu_isar(const double* values, const double* frequencies, uint32_t n_frequencies,
                             const double* angles_deg, uint32_t n_angles, int window, int zero_pad,
                             double dynamic_floor_db, double* down_range_m, double* cross_range_m,
                             double* mag_db, double* peak_db);

/* Parity instrumentation: run mcsbr_gpu_estimate and record, for launch
 * entries [0, n_paths) of the incidence, the triangle id of every hit
 * (tri_ids[p*stride + k] for hit k, 0xFFFFFFFF past the end), the
 * termination reason term[p] (0 escaped, 1 grazing, 2 bounce cap,
 * 3 roulette) and the branch bits branch_bits[p] (bit k = transmit chosen
 * after hit k).  Same layout as the oracle's orc_path_log. */
MCSBR_API int mcsbr_gpu_path_log(mcsbr_scene* scene, const mcsbr_excitation* excitation,
                                 const double* frequencies, uint32_t n_frequencies,
                                 const mcsbr_mc_config* config, uint64_t n_paths, uint32_t stride,
                                 uint32_t* tri_ids, uint8_t* term, uint64_t* branch_bits);

/* Number of kernel launches the last compute call on this thread issued
 * (evidence for the benchmark's gpu_launches key). */
MCSBR_API uint64_t mcsbr_gpu_last_launch_count(void);

/* Per-kernel device timing on the calling thread (evidence for the
 * benchmark's roofline): enable = 1 resets the record and starts bracketing
 * every path-kernel and accumulate launch of this thread's compute calls with
 * CUDA events on the launch stream; enable = 0 stops.  mcsbr_gpu_kernel_times
 * waits for the recorded events and returns the summed device milliseconds
 * and launch counts since the last enable. */
MCSBR_API void mcsbr_gpu_kernel_timing(int enable);
MCSBR_API int mcsbr_gpu_kernel_times(double* path_ms, uint64_t* path_launches, double* acc_ms,
                                     uint64_t* acc_launches);

#ifdef __cplusplus
}
#endif

#endif /* MCSBR_GPU_H_ */
