// K2/K3/K4: the persistent Monte Carlo SBR path kernel.
//
// Replaces the body of mcsbr::estimate (proj/src/solver_mc.cpp:105-210) and
// its callees.  One thread owns one path at a time; a warp pulls chunks of
// launch entries from a global cursor (guided self-scheduling) and refills
// lanes as their paths terminate (path regeneration), so the SIMT lanes stay
// busy even though path lengths differ.  Per lane and event:
//
//   closest hit (K2, fp32 conservative BVH4 descent + fp64 Moller-Trumbore in
//   the reference's arithmetic, pathcore.cuh traverse)  -> advance ->
//   branch_outcomes (GO Fresnel / PEC transport) -> MECA currents +
//   contribution -> branch choice and Russian roulette -> occlusion any-hit
//   toward the receiver (K3) -> phasor accumulation (K4).
//
// The wavefront order of the reference (all first hits of a block, then all
// second hits, ...) only changes the ORDER in which contributions are summed;
// every path's arithmetic is independent of it, which is why a depth-first
// per-thread path with a counter-based RNG keyed on (cell, sample, bounce)
// reproduces the reference's per-path events bit for bit.
//
// Accumulation (K4): F = 1 keeps the 4 channel phasor sums of the lane's
// current incidence in its shared-memory slot and reduces them across the
// warp (shuffles) when the warp changes incidence, then one fp64 atomicAdd
// per channel (register mode); bistatic fans give lane l receiver l (fan
// mode).  F > 1 (and every MCSBR_REDUCE_EXACT job) appends each visible
// contribution as a 96-byte record to HBM; accumulate_kernel (or
// accumulate_exact_kernel) turns the records into the [F][4] sums after the
// launch (deferred mode).  Launch entries of deferred-mode kernels are
// culled by the coverage bitmaps of cover.cu.
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <type_traits>

#include "dmath.cuh"
#include "fixedpoint.cuh"
#include "internal.h"
#include "physics.cuh"
#include "rng.cuh"
#include "mcsbr_gpu.h"

using namespace mcsbr_dev;

namespace mcsbr_int {

namespace {
#include "pathcore.cuh"

// ---------------------------------------------------------------------------
// the path kernel

// Accumulation modes:
//   kModeDefer one receiver, F > 1: every visible contribution (4 projected
//              amplitudes, optical path, incidence) is appended to a record
//              buffer in HBM; accumulate_kernel turns the records into the
//              [F][4] phasor sums after the launch (deferred accumulation keeps
//              the path kernel's shared memory -- and so its L1 -- free of
//              per-warp [F][4] arrays).
//   kModeReg   one receiver, F = 1: per-lane register sums, warp-reduced per tile
//   kModeFanRec the same fan with F > 1: lane l appends one record per visible
//              (contribution, receiver l) in row 32 a + l (sums_row), which
//              the accumulation kernels (NUFFT or direct) then sum
//   kModeFan   a bistatic fan of up to 32 receivers per launch (P.rx_index is
//              the first), F = 1: lane l owns receiver rx_index + l; every
//              contribution is broadcast across the warp and each lane runs
//              its receiver's occlusion test and projection (a coherent
//              32-ray bundle from one exit point), so paths are traced once
//              per 32 receivers instead of once per receiver.
enum { kModeDefer = 0, kModeReg = 1, kModeFan = 2, kModeFanRec = 3 };

#ifndef MCSBR_MIN_BLOCKS
#define MCSBR_MIN_BLOCKS 4  // 128 registers: 16 warps/SM (measured best of 1/2/3/4/6)
#endif
// (A/B knob) register budget of the deferred-accumulation and lossy
// instantiations.
#ifndef MCSBR_SMEM_MIN_BLOCKS
#define MCSBR_SMEM_MIN_BLOCKS 4
#endif
// (A/B knob) register budget of the PEC instantiations (all modes)
#ifndef MCSBR_PEC_MIN_BLOCKS
#define MCSBR_PEC_MIN_BLOCKS 5  // against 4: c1 -5%, c4 -3%, c2 -0.1% (96 registers, 5 blocks/SM)
#endif
// (A/B knob) the PEC deferred-accumulation instantiation (F > 1 sweeps)
#ifndef MCSBR_PEC_DEFER_MIN_BLOCKS
#define MCSBR_PEC_DEFER_MIN_BLOCKS 6  // against 5: c4 -2.4% (80 registers)
#endif
template <int kMode, bool kDiel, bool kLossy>
struct MinBlocks {
    static constexpr int value = (!kDiel && !kLossy)    ? (kMode == 0 ? MCSBR_PEC_DEFER_MIN_BLOCKS : MCSBR_PEC_MIN_BLOCKS)
                                 : (kMode == 0 || kLossy) ? MCSBR_SMEM_MIN_BLOCKS
                                                          : MCSBR_MIN_BLOCKS;
};
// kDet: the deterministic solver (solver_det.cpp:30-174) on the same engine:
// midpoint launch (P.jitter = 0, spp = 1), no draws; at a two-branch hit the
// reflect child continues in registers and the transmit child goes on the
// lane's branch stack; a dead lane pops its own stack before it takes a new
// entry, which reproduces the reference's depth-first, reflect-first order.
template <int kMode, bool kDiel, bool kLossy, bool kDet, bool kFast>
__global__ void __launch_bounds__(128, (MinBlocks<kMode, kDiel, kLossy>::value)) path_kernel(TraceParams P) {
    constexpr bool kRegAcc = kMode != kModeDefer;
    constexpr bool kFanM = kMode == kModeFan || kMode == kModeFanRec;  // any bistatic fan
    constexpr bool kFanRec = kMode == kModeFanRec;  // fan with F > 1: deferred records (fan_rows)
    // launch-ray culling by the coverage bitmaps (cover.cu): the deferred-
    // accumulation Monte Carlo kernels (large ISAR scenes); run_job builds
    // bitmaps only for those
    constexpr bool kCull = kMode == kModeDefer && !kDet;
    using NT = typename std::conditional<kLossy, Cx, double>::type;
    using L = Layout<!kDiel && !kLossy, kLossy, kRegAcc>;
    using EF = typename std::conditional<L::pec, V3, CV3>::type;  // field type
    constexpr int kFAcc = L::Acc;               // register-mode phasor sums
    constexpr int kSlotFields = L::Fields;      // doubles per thread
    __shared__ unsigned long long s_cnt[9];  // launched .. rounds (kCntLaunched..kCntRounds), culled
    // per-bounce counters as native 32-bit shared atomics (ATOMS.ADD); the
    // 64-bit shared atomicAdd is a CAS loop on sm_100 and cost ~20% of the
    // kernel.  Per block and bounce they stay far below 2^32.
    __shared__ unsigned int s_bounce[3 * 64];
    __shared__ double s_state[kSlotFields * kSlotThreads];
    __shared__ unsigned long long s_sched[kSlotThreads / 32][4];
    __shared__ double s_rcp[kSlotThreads / 32][2];  // reciprocals of the incidence's nu, nv (init_path)
    for (int i = threadIdx.x; i < 9; i += blockDim.x) s_cnt[i] = 0;
    for (int i = threadIdx.x; i < 3 * 64; i += blockDim.x) s_bounce[i] = 0;
    __syncthreads();
    const Slot sl{s_state + threadIdx.x};

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const SceneView& S = P.scene;
    uint32_t fault = 0;
    uint64_t n_launched = 0, n_contrib = 0, n_graze = 0, n_cap = 0, n_occ = 0;
    uint64_t n_miss0 = 0;  // culled launch entries (launched, escaped at bounce 0)
    int max_round = 0;
    const uint64_t gtid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    mcsbr_contribution* scratch =
        P.contrib_scratch ? static_cast<mcsbr_contribution*>(P.contrib_scratch) + gtid : nullptr;
    // deterministic mode: branch-stack height, event_seq of the root ray, and
    // the reference's stack accounting (peak depth / pushes per root ray,
    // summed per accounting block of det_block_size cells)
    int dsp = 0;
    uint32_t dev = 0, dpeak = 0;
    uint64_t dacc_peak = 0, dacc_push = 0, dblk = ~0ull;

    // Work distribution: a global cursor over the job's flattened entry space
    // (incidence-major).  A warp takes a chunk with one atomicAdd; chunk sizes
    // shrink as the work runs out (guided self-scheduling: remaining / (2 *
    // warps), multiple of 32, in [32, chunk_max]) so the last chunks are small
    // and the warps finish at nearly the same time.  A chunk may span
    // incidences; it is processed as one sub-range per incidence.  The warp's
    // phasor accumulators belong to one incidence and are flushed only when
    // the warp moves to another one (and at the end), not per chunk, and a
    // warp whose sub-range runs dry takes the next chunk without draining its
    // lanes when that chunk continues the same incidence.
    // The warp's scheduling state lives in shared memory (it is touched only
    // when a sub-range runs dry), not in registers the traversal needs:
    // q[0], q[1] = fetched, not yet started global range; q[2] = the cursor
    // value the warp last saw (guides the chunk size; ~0 once exhausted).
    volatile unsigned long long* q = s_sched[warp];
    if (lane == 0) {
        q[0] = 0;
        q[1] = 0;
        q[2] = 0;
    }
    __syncwarp();
    auto fetch = [&]() {
        const unsigned long long seen = q[2];
        if (seen == ~0ull) return;
        const uint64_t n_warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
        const uint64_t rem = P.total_entries > seen ? P.total_entries - seen : 0;
        uint64_t c = P.gss_div ? rem / (P.gss_div * n_warps) : P.chunk_max;
        c = (c + 31) & ~31ull;
        c = c < P.chunk_min ? P.chunk_min : (c > P.chunk_max ? P.chunk_max : c);
        if (lane == 0) {
            const unsigned long long g = atomicAdd(P.tile_counter, static_cast<unsigned long long>(c));
            if (g >= P.total_entries) {
                q[2] = ~0ull;
            } else {
                q[2] = g + c;
                q[0] = g;
                q[1] = min(static_cast<uint64_t>(g + c), P.total_entries);
            }
        }
        __syncwarp();
    };
    // launch unit containing global entry g: last u with g_begin[u] <= g
    auto find_inc = [&](uint64_t g) {
        uint32_t lo = 0, hi = P.n_inc;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (P.inc[mid].g_begin <= g) lo = mid; else hi = mid;
        }
        return lo;
    };
    uint32_t cur_a = 0xffffffffu;  // incidence the accumulators hold (warp-uniform)
    if (kRegAcc) {
#pragma unroll
        for (int k = 0; k < 8; ++k) sl.set(kFAcc + k, 0.0);
    }
    // add the warp's accumulators into incidence cur_a's sums and clear them
    auto flush = [&]() {
        if (kRegAcc && !kFanRec && cur_a != 0xffffffffu)
            flush_sums<kFanM, kFAcc>(P.sums, P.n_rx, P.rx_index, sl.p, cur_a, lane);
    };

    for (;;) {
        // ---- next sub-range (warp-uniform) ----
        if (q[0] >= q[1]) fetch();
        const uint64_t q0 = q[0], q1 = q[1];
        if (q0 >= q1) break;
        const IncDev& I = P.inc[find_inc(q0)];  // the launch unit holding q0
        const uint32_t a = I.row;               // its incidence
        const uint64_t g_end_a = I.g_begin + (I.entry_end - I.entry_begin);
        uint64_t cursor = I.entry_begin + (q0 - I.g_begin);  // warp-uniform
        uint64_t e_end = I.entry_begin + (min(q1, g_end_a) - I.g_begin);
        __syncwarp();
        if (lane == 0) {
            q[0] = min(q1, g_end_a);
            s_rcp[warp][0] = mcsbr_dev::rcp_seed(I.nu);
            s_rcp[warp][1] = mcsbr_dev::rcp_seed(I.nv);
        }
        __syncwarp();
        if (a != cur_a) {
            flush();
            cur_a = a;
        }
        // fan mode: lane l evaluates receiver rx_index + l (if it exists)
        const uint32_t my_rx = P.rx_index + (kFanM ? static_cast<uint32_t>(lane) : 0u);
        const bool has_rx = my_rx < P.n_rx;
        const RxDev& R = P.rx[static_cast<size_t>(a) * P.n_rx + (has_rx ? my_rx : P.rx_index)];

        bool alive = false;  // lane holds a path (possibly only its last occlusion query)
        bool pend = false;   // next query is the chi occlusion test of a contribution
        bool dying = false;  // the path ends once its pending occlusion test is done
        Path<NT, EF> s;
        Cx amp[4];           // contribution: receiver-projected amplitudes (slot while pending)
        NT s_path{};         //               and net optical path
        EF fj0, fm0, fj1, fm1;   // fan mode: the contribution's currents,
        NT fphi{};               // optical path
        V3 fpt = {0.0, 0.0, 0.0};  // and exit point, broadcast to the warp

        // One query per lane per iteration: either the path's next closest
        // hit or the occlusion test of the contribution its last hit made.
        // Lanes in both phases traverse together, so no lane idles while
        // others run occlusion rays, and the traversal loop appears once.
        for (;;) {
            // ---- deterministic: a dead lane resumes its own pending branch ----
            if (kDet && !alive && dsp > 0) {
                det_pop(P, gtid, --dsp, s);
                save_em<L>(sl, s);
                alive = true;
            }
            // ---- regenerate dead lanes from the tile ----
            // Dead lanes take the next launch entries of the warp's sub-range
            // (continuing into the next chunk when it is the same incidence).
            // Entries whose coverage bit is clear provably escape (cover.cu):
            // they are retired here as launched bounce-0 misses, without ray
            // generation or traversal, and whole empty runs of the bitmap are
            // skipped at once; the lanes keep drawing until they hold a path
            // or the incidence's entries are used up.
            unsigned need = __ballot_sync(kFull, !alive);
            if (!kCull) {
                // register-sum / fan kernels (F = 1: small, cache-resident
                // scenes) regenerate in one pass without the bitmap: the
                // culling loop's registers cost them more than it saves
                if (need && cursor >= e_end) {
                    if (q[0] >= q[1]) fetch();
                    const uint64_t n0 = q[0], n1 = q[1];
                    if (n0 < n1 && n0 >= I.g_begin && n0 < g_end_a) {
                        cursor = I.entry_begin + (n0 - I.g_begin);
                        e_end = I.entry_begin + (min(n1, g_end_a) - I.g_begin);
                        __syncwarp();
                        if (lane == 0) q[0] = min(n1, g_end_a);
                        __syncwarp();
                    }
                }
                if (need && cursor < e_end) {
                    const unsigned rank = __popc(need & ((1u << lane) - 1u));
                    const uint64_t mine = cursor + rank;
                    if (!alive && mine < e_end) {
                        init_path(P, I, a + P.inc_base, locate(P, I, mine), s, s_rcp[warp]);
                        save_em<L>(sl, s);
                        alive = true;
                        ++n_launched;
                        if (kDet) {  // a new root ray (solver_det.cpp:72-82)
                            const uint64_t blk = s.cell / P.det_block_size;
                            dacc_peak += dpeak;
                            if (blk != dblk) {
                                det_flush(P, dblk, dacc_peak, dacc_push);
                                dacc_peak = dacc_push = 0;
                                dblk = blk;
                            }
                            dpeak = 1;
                            dacc_push += 1;
                            dev = 0;
                        }
                    }
                    cursor = min(cursor + static_cast<uint64_t>(__popc(need)), e_end);
                }
                need = 0;
            }
            while (need) {
                if (cursor >= e_end) {
                    // sub-range dry: continue with the next chunk if it is the same incidence
                    if (q[0] >= q[1]) fetch();
                    const uint64_t n0 = q[0], n1 = q[1];
                    if (n0 < n1 && n0 >= I.g_begin && n0 < g_end_a) {
                        cursor = I.entry_begin + (n0 - I.g_begin);
                        e_end = I.entry_begin + (min(n1, g_end_a) - I.g_begin);
                        __syncwarp();
                        if (lane == 0) q[0] = min(n1, g_end_a);
                        __syncwarp();
                    } else {
                        break;
                    }
                }
                if (kCull && P.cover && I.cover_off != kNoCover) {
                    const uint64_t c2 = skip_uncovered(P.cover + I.cover_off, I.cover_shift, cursor, e_end);
                    if (lane == 0) n_miss0 += c2 - cursor;  // warp-uniform run, counted once
                    cursor = c2;
                    if (cursor >= e_end) continue;
                }
                const unsigned rank = __popc(need & ((1u << lane) - 1u));
                const uint64_t mine = cursor + rank;
                if (!alive && mine < e_end) {
                    if (kCull && !covered(P, I, mine)) {
                        ++n_miss0;  // provable miss: one launched ray, one bounce-0 segment
                    } else {
                        init_path(P, I, a + P.inc_base, locate(P, I, mine), s, s_rcp[warp]);
                        save_em<L>(sl, s);
                        alive = true;
                        ++n_launched;
                        if (kDet) {  // a new root ray (solver_det.cpp:72-82)
                            const uint64_t blk = s.cell / P.det_block_size;
                            dacc_peak += dpeak;
                            if (blk != dblk) {
                                det_flush(P, dblk, dacc_peak, dacc_push);
                                dacc_peak = dacc_push = 0;
                                dblk = blk;
                            }
                            dpeak = 1;
                            dacc_push += 1;
                            dev = 0;
                        }
                    }
                }
                cursor = min(cursor + static_cast<uint64_t>(__popc(need)), e_end);
                need = __ballot_sync(kFull, !alive);
            }
            if (!__any_sync(kFull, alive)) break;

            double t = 0.0;
            uint32_t id = 0;
            bool hit = false;
            if (alive) {
                if (pend) ++n_occ;
                else if (!kDet) atomicAdd(&s_bounce[min(s.bounce, 63)], 1u);
                // closest hit: solver_mc.cpp:142-144; occlusion: farfield.cpp:63-68 /
                // geometry.cpp:242-244 from the exit point (= origin after advance)
                hit = traverse<kFast>(S, s.origin, pend ? ld3(R.k_s) : s.dir,
                               (pend || s.bounce != 0) ? S.t_eps : 0.0, t, id, fault, pend,
                               !pend && s.bounce == 0);
            }
            bool visible = false;
            bool fan = false;
            if (alive && pend) {
                pend = false;
                visible = !hit;
                if (visible) {  // the queued contribution's amplitudes come back from the slot
#pragma unroll
                    for (int ch = 0; ch < 4; ++ch) amp[ch] = slot_get_amp<L>(sl, ch);
                    s_path = slot_get_nt<NT>(sl, L::SPath, L::SPathIm);
                }
                if (dying) {
                    alive = false;
                    dying = false;
                }
            } else if (alive) {
                bool candidate = false;
                if (!hit) {
                    alive = false;  // escaped
                } else {
                    load_em<L>(sl, s, S.ambient_n);
                    const V3 point = s.origin + s.dir * t;
                    const HitInfo<NT> h = fill_hit<NT>(S, id, s.dir);
                    // advance (path_engine.cpp:17-21); complex in lossy media
                    s.phi = s.phi + s.medium_n * t;
                    s.origin = point;
                    s.bounce += 1;
                    max_round = max(max_round, s.bounce);
                    // the deterministic solver counts segments that hit (solver_det.cpp:88-93)
                    if (kDet) atomicAdd(&s_bounce[min(s.bounce - 1, 63)], 1u);
                    const bool logged = P.plog_tri && a + P.inc_base == 0 && s.entry < P.plog_n;
                    if (logged && static_cast<uint32_t>(s.bounce - 1) < P.plog_stride)
                        P.plog_tri[s.entry * P.plog_stride + (s.bounce - 1)] = id;
                    // branch_outcomes (path_engine.cpp:23-54)
                    const double cos_i = -dot(s.dir, h.normal);
                    if (cos_i < 1e-6) {
                        ++n_graze;
                        alive = false;
                        if (logged) P.plog_term[s.entry] = 1;
                    } else {
                        // kDiel = false: every triangle has a PEC side (checked at
                        // scene creation), so far_side_pec always holds and the
                        // dielectric code (and its registers) is compiled out.
                        const bool pec = kDiel ? h.far_side_pec : true;
                        const NT n1 = s.medium_n;
                        const NT n2 = pec ? n1 : h.n_transmit;
                        const Coeffs co = pec ? coeffs_pec() : fresnel_any(n1, n2, cos_i, fault);
                        // ray geometry from the real parts (exact for the lossless model);
                        // a Monte Carlo PEC hit forms it only after its contribution,
                        // which does not use it (shorter register live ranges)
                        constexpr bool kLateBasis = L::pec && !kDet;
                        Basis b;
                        if constexpr (!kLateBasis) b = sp_basis(s.dir, h.normal, re_of(n1), re_of(n2), !pec, fault);
                        const bool two = !pec && !co.tir;
                        // The deterministic solver needs every branch's fields
                        // at once; the Monte Carlo path forms only what the
                        // contribution and the chosen branch use (fewer live
                        // registers across the shading): identical values, and
                        // the transversality guard raises the same faults.
                        EF er0 = ef_zero<EF>(), er1 = ef_zero<EF>(), et0 = ef_zero<EF>(), et1 = ef_zero<EF>();
                        if constexpr (kDet) {
                            er0 = interface_transform(s.e0, 0, co, b, fault);
                            er1 = interface_transform(s.e1, 0, co, b, fault);
                            if (two) {
                                et0 = interface_transform(s.e0, 1, co, b, fault);
                                et1 = interface_transform(s.e1, 1, co, b, fault);
                            }
                        } else if constexpr (!kLateBasis) {
                            transverse_guard(s.e0, b, fault);
                            transverse_guard(s.e1, b, fault);
                        }
                        // scatter case + chi pre-checks (solver_mc.cpp:150-160)
                        const int sc = pec ? 0 : (h.near_is_ambient ? 1 : 2);
                        const bool dark_exit = sc == 2 && co.tir;
                        candidate = !dark_exit && h.exterior_facing;
                        if (candidate) {
                            // meca_currents (farfield.cpp:11-45) for both pols
                            // The three cases share one copy of the arithmetic
                            // (operands selected per lane, so a warp mixing PEC,
                            // ambient-side and exiting hits runs it once):
                            //   sc 0: j = n x ((d x e) n1) 2,              m = 0
                            //   sc 1: j = n x ((d x e + d_r x e_r) n1),    m = (e + e_r) x n
                            //   sc 2: j = n_o x ((d_t x e_t) n2),          m = e_t x n_o, n_o = -n
                            // each the reference's expression operation for operation.
                            const bool ex = sc == 2;
                            const V3 nrm = ex ? -h.normal : h.normal;
                            V3 dj = s.dir;  // (PEC kernels: sc == 0, and no basis yet)
                            if constexpr (!kLateBasis) {
                                if (ex) dj = b.dir_t;
                            }
                            const NT nj = ex ? h.n_transmit : s.medium_n;
                            // make_contribution (farfield.cpp:70-85)
                            const double cos_n = fabs(dot(s.dir, h.normal));
                            const double scale = s.weight * I.area_weight / (s.prob * cos_n);
                            // one polarisation's currents (e: the incident
                            // field; e_r / e_t for sc 1 / 2), scaled
                            auto currents = [&](const EF& e, int pol, EF& j, EF& m) {
                                EF f = ef_zero<EF>();  // e_r (sc 1) / e_t (sc 2)
                                if (sc != 0) {
                                    if constexpr (kDet) f = ex ? (pol ? et1 : et0) : (pol ? er1 : er0);
                                    else f = branch_field(e, ex ? 1 : 0, co, b);
                                }
                                EF x = cross(dj, ex ? f : e);
                                if (sc == 1) x = x + cross(b.dir_r, f);
                                j = cross(nrm, x * nj);
                                m = ef_zero<EF>();
                                if (sc == 0) j = j * 2.0;
                                else m = cross(ex ? f : e + f, nrm);
                                j = j * scale;
                                m = m * scale;
                            };
                            EF j0, m0, j1, m1;
                            if constexpr (kFanM) {
                                currents(s.e0, 0, j0, m0);
                                currents(s.e1, 1, j1, m1);
                                fj0 = j0;
                                fm0 = m0;
                                fj1 = j1;
                                fm1 = m1;
                                fphi = s.phi;
                                fpt = point;
                            } else {
                                // polarisation by polarisation: half the live
                                // complex vectors of forming all four
                                // currents first (the lossy kernel spilled
                                // them); every value is the same expression
                                currents(s.e0, 0, j0, m0);
                                if constexpr (L::pec) project_pec_pol(R, j0, amp[0], amp[3]);  // m = 0 on PEC hits
                                else project_pol(R, j0, m0, amp[0], amp[3]);
                                if (scratch) {
                                    store_cv(&scratch->a_j[0][0][0], j0);
                                    store_cv(&scratch->a_m[0][0][0], m0);
                                }
                                currents(s.e1, 1, j1, m1);
                                if constexpr (L::pec) project_pec_pol(R, j1, amp[2], amp[1]);
                                else project_pol(R, j1, m1, amp[2], amp[1]);
                                s_path = s.phi - dot(ld3(R.k_s), point);
                            }
                            if (scratch) {
                                if constexpr (kFanM) {
                                    store_cv(&scratch->a_j[0][0][0], j0);
                                    store_cv(&scratch->a_m[0][0][0], m0);
                                }
                                store_cv(&scratch->a_j[1][0][0], j1);
                                store_cv(&scratch->a_m[1][0][0], m1);
                                scratch->phi_total = re_of(s.phi);
                                scratch->exit_point[0] = point.x;
                                scratch->exit_point[1] = point.y;
                                scratch->exit_point[2] = point.z;
                                scratch->bounce = s.bounce;
                                scratch->_pad = 0;
                                scratch->order_key =
                                    kDet ? (static_cast<uint64_t>(s.cell) << 24 | dev)  // solver_det.cpp:104
                                         : ((static_cast<uint64_t>(s.cell) * P.spp + s.sample) << 8) |
                                               static_cast<uint64_t>(s.bounce & 0xff);
                            }
                        }
                        if constexpr (kLateBasis) {
                            b = sp_basis(s.dir, h.normal, re_of(n1), re_of(n2), false, fault);
                            transverse_guard(s.e0, b, fault);
                            transverse_guard(s.e1, b, fault);
                        }
                        if (s.bounce >= P.max_bounce) {  // cap (solver_mc.cpp:176-179)
                            ++n_cap;
                            alive = false;
                            if (logged) P.plog_term[s.entry] = 2;
                        } else if (kDet) {
                            // every surviving branch (solver_det.cpp:127-147)
                            bool keep_r = true, keep_t = two;
                            if (P.det_cutoff > 0.0) {
                                const double nr0 = cvnorm(er0), nr1 = cvnorm(er1);
                                keep_r = !(((nr0 < nr1) ? nr1 : nr0) < P.det_cutoff);
                                if (two) {
                                    const double nt0 = cvnorm(et0), nt1 = cvnorm(et1);
                                    keep_t = !(((nt0 < nt1) ? nt1 : nt0) < P.det_cutoff);
                                }
                            }
                            if (keep_r && keep_t) {
                                if (dsp >= static_cast<int>(P.det_depth)) {
                                    fault |= kFaultStack;
                                } else {
                                    det_push(P, gtid, dsp, s.origin, b.dir_t, et0, et1, s.phi, n2, s.bounce);
                                    ++dsp;
                                }
                            }
                            const uint32_t kept = static_cast<uint32_t>(keep_r) + static_cast<uint32_t>(keep_t);
                            dacc_push += kept;
                            if (keep_r) {
                                s.dir = b.dir_r;
                                s.e0 = er0;
                                s.e1 = er1;
                                s.medium_n = n1;
                            } else if (keep_t) {
                                s.dir = b.dir_t;
                                s.e0 = et0;
                                s.e1 = et1;
                                s.medium_n = n2;
                            } else {
                                alive = false;
                            }
                            // reference stack height after its pushes, + 1 (solver_det.cpp:148)
                            dpeak = max(dpeak, static_cast<uint32_t>(dsp) + (kept ? 1u : 0u) + 1u);
                        } else {
                            // choose_branch (solver_mc.cpp:44-54, :181-190)
                            int pick = 0;
                            double pp = 1.0;
                            if (two) {
                                double p_reflect = 0.5;
                                if (P.fresnel_strategy) {
                                    const double r_bar = co.lossy ? 0.5 * (sqrt(cnorm2(co.r_s)) + sqrt(cnorm2(co.r_p)))
                                                          : 0.5 * (cabs(co.r_s) + cabs(co.r_p));
                                    const double lo_c = (r_bar < P.p_min) ? P.p_min : r_bar;
                                    const double hi_c = 1.0 - P.p_min;
                                    p_reflect = (hi_c < lo_c) ? hi_c : lo_c;
                                }
                                const double u = draw(P, s, static_cast<uint64_t>(s.bounce), kBranch);
                                if (u < p_reflect) {
                                    pp = p_reflect;
                                } else {
                                    pick = 1;
                                    pp = 1.0 - p_reflect;
                                }
                            }
                            if (logged && pick) P.plog_branch[s.entry] |= 1ull << (s.bounce - 1);
                            const EF ne0 = branch_field(s.e0, pick, co, b), ne1 = branch_field(s.e1, pick, co, b);
                            s.e0 = ne0;
                            s.e1 = ne1;
                            if (pick == 0) {
                                s.dir = b.dir_r;
                                s.medium_n = n1;
                            } else {
                                s.dir = b.dir_t;
                                s.medium_n = n2;
                            }
                            s.prob *= pp;
                            // roulette (solver_mc.cpp:56-64, :192-205)
                            if (P.roulette_enabled && s.bounce >= P.roulette_min_bounce) {
                                const int bi = min(s.bounce - 1, 63);
                                atomicAdd(&s_bounce[64 + bi], 1u);
                                const double u = draw(P, s, static_cast<uint64_t>(s.bounce), kRoulette);
                                if (u > P.roulette_q) {
                                    s.weight /= (1.0 - P.roulette_q);
                                    atomicAdd(&s_bounce[128 + bi], 1u);
                                } else {
                                    alive = false;
                                    if (logged) P.plog_term[s.entry] = 3;
                                }
                            }
                        }
                    }
                    save_em<L>(sl, s);
                }
                // ---- chi visibility (farfield.cpp:63-68): queue the occlusion query ----
                if (candidate && kFanM) {
                    fan = true;  // evaluated below by the whole warp
                } else if (candidate) {
                    if (P.occlusion) {
                        pend = true;
#pragma unroll
                        for (int ch = 0; ch < 4; ++ch) slot_set_amp<L>(sl, ch, amp[ch]);
                        slot_set_nt(sl, L::SPath, L::SPathIm, s_path);
                        if (!alive) {
                            alive = true;
                            dying = true;
                        }
                    } else {
                        visible = true;
                    }
                }
            }
            if (visible) {
                ++n_contrib;
                if (kDet) ++dev;
                if (scratch) {
                    const unsigned long long slot = atomicAdd(P.contrib_count, 1ull);
                    if (slot < P.contrib_cap)
                        static_cast<mcsbr_contribution*>(P.contrib_out)[slot] = *scratch;
                }
            }
            // ---- bistatic fan: every contribution against this launch's receivers ----
            if (kFanM) {
                unsigned fm = __ballot_sync(kFull, fan);
                const V3 ks = ld3(R.k_s);
                while (fm) {
                    const int src = __ffs(fm) - 1;
                    fm &= fm - 1;
                    EF c[4] = {fj0, fm0, fj1, fm1};
#pragma unroll
                    for (int k = 0; k < 4; ++k) c[k] = shfl_ef(c[k], src);
                    const NT ph = shfl_nt(fphi, src);
                    const V3 pt = {shfl_d(fpt.x, src), shfl_d(fpt.y, src), shfl_d(fpt.z, src)};
                    if (has_rx) {
                        // project first: only 4 complex amplitudes + s stay live
                        // across this receiver's occlusion traversal
                        Cx am[4];
                        project(R, c[0], c[1], c[2], c[3], am);
                        const NT sp = ph - dot(ks, pt);
                        bool vis = true;
                        if (P.occlusion) {
                            double t2;
                            uint32_t id2;
                            ++n_occ;
                            vis = !traverse<kFast>(S, pt, ks, S.t_eps, t2, id2, fault, true, false);
                        }
                        if (vis) {
                            ++n_contrib;
                            if constexpr (kFanRec) {
                                // multi-frequency fan: one deferred record per
                                // visible (contribution, receiver), row 32 a + lane
                                // (sums_row); one atomic per group of lanes here
                                const unsigned m = __activemask();
                                const int leader = __ffs(m) - 1;
                                unsigned long long base = 0;
                                if (lane == leader)
                                    base = atomicAdd(P.rec_count, static_cast<unsigned long long>(__popc(m)));
                                base = __shfl_sync(m, base, leader);
                                const uint64_t slot = base + __popc(m & ((1u << lane) - 1u));
                                const uint32_t row = a * 32u + static_cast<uint32_t>(lane);
                                if (slot < P.rec_cap) write_record(P, slot, am, sp, row);
                                else fan_record_overflow(P, row, am, sp);
                            } else {
                                acc_add<kFAcc>(sl, am, phasor(P.k0[0], sp));
                            }
                        }
                    }
                }
            } else if (kRegAcc) {
                // ---- phasor accumulation (farfield.cpp:130-146) ----
                if (visible) {
                    if constexpr (L::pec) acc_add_real<kFAcc>(sl, amp, phasor(P.k0[0], s_path));
                    else acc_add<kFAcc>(sl, amp, phasor(P.k0[0], s_path));
                }
            } else {
                // ---- deferred accumulation: append the contribution record ----
                const unsigned vm = __ballot_sync(kFull, visible);
                if (vm) {
                    unsigned long long base = 0;
                    if (lane == 0) base = atomicAdd(P.rec_count, static_cast<unsigned long long>(__popc(vm)));
                    base = __shfl_sync(kFull, base, 0);
                    const uint64_t slot = base + __popc(vm & ((1u << lane) - 1u));
                    const bool stored = visible && slot < P.rec_cap;
                    if (stored) write_record(P, slot, amp, s_path, a);
                    // buffer full (the host sizes it so this is rare): the warp
                    // adds each overflowing contribution straight into the sums,
                    // lanes over frequencies
                    unsigned om = __ballot_sync(kFull, visible && !stored);
                    double* out = P.sums + sums_row(P, a) * P.nf * 8;
                    while (om) {
                        const int src = __ffs(om) - 1;
                        om &= om - 1;
                        Cx am[4];
#pragma unroll
                        for (int ch = 0; ch < 4; ++ch) {
                            am[ch].re = shfl_d(amp[ch].re, src);
                            am[ch].im = shfl_d(amp[ch].im, src);
                        }
                        const NT sp = shfl_nt(s_path, src);
                        for (uint32_t f = lane; f < P.nf; f += 32) {
                            const Cx z = freq_phasor(P, f, sp);
#pragma unroll
                            for (int ch = 0; ch < 4; ++ch) {
                                const Cx v = am[ch] * z;
                                add_value(P, out, f * 8 + 2 * ch, v.re);
                                add_value(P, out, f * 8 + 2 * ch + 1, v.im);
                            }
                        }
                    }
                }
            }
        }

        if (kDet) {  // every root of the sub-range is finished
            dacc_peak += dpeak;
            dpeak = 0;
            det_flush(P, dblk, dacc_peak, dacc_push);
            dacc_peak = dacc_push = 0;
            dblk = ~0ull;
        }
    }
    flush();

    // ---- counters ----
    auto wsum = [](uint64_t v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        return v;
    };
    if (kCull && n_miss0) atomicAdd(&s_bounce[0], static_cast<unsigned int>(n_miss0));
    n_launched = wsum(n_launched + n_miss0);
    n_miss0 = wsum(n_miss0);
    n_contrib = wsum(n_contrib);
    n_graze = wsum(n_graze);
    n_cap = wsum(n_cap);
    n_occ = wsum(n_occ);
    const unsigned fault_w = __reduce_or_sync(kFull, fault);
    const int round_w = __reduce_max_sync(kFull, max_round);
    if (lane == 0) {
        atomicAdd(&s_cnt[kCntLaunched], n_launched);
        atomicAdd(&s_cnt[kCntContrib], n_contrib);
        atomicAdd(&s_cnt[kCntGrazing], n_graze);
        atomicAdd(&s_cnt[kCntCap], n_cap);
        atomicAdd(&s_cnt[kCntOcclusion], n_occ);
        atomicOr(&s_cnt[kCntFault], static_cast<unsigned long long>(fault_w));
        atomicMax(&s_cnt[kCntRounds], static_cast<unsigned long long>(round_w));
        atomicAdd(&s_cnt[8], n_miss0);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 9 + 3 * 64; i += blockDim.x) {
        unsigned long long v;
        int dst;
        if (i < 9) {
            v = s_cnt[i];
            dst = i < 8 ? i : kCntCulled;
        } else {
            const int j = i - 9;
            v = s_bounce[j];
            dst = j < 64 ? kCntRaysPerBounce + j : (j < 128 ? kCntRouletteCand + j - 64 : kCntRouletteSurv + j - 128);
        }
        if (!v) continue;
        if (dst == kCntFault) atomicOr(P.counters + dst, v);
        else if (dst == kCntRounds) atomicMax(P.counters + dst, v);
        else atomicAdd(P.counters + dst, v);
    }
}


// ---------------------------------------------------------------------------
// K4b: deferred phasor accumulation (SweepAccumulator::add, farfield.cpp:130-146)
//
// Each warp owns a contiguous span of contribution records (>= 512, so its
// flushes cost < 1 atomic per record and channel) and keeps the [FPL][4]
// complex sums of its 32 x FPL frequencies in registers: lane l holds
// frequencies f_begin + l + 32 m.  Records are staged 32 at a time through
// shared memory; for each, the staging lane precomputes the phase terms and
// W = e^{-j 32 dk s} (one sincos per record), so an accumulating lane pays one
// sincos per record for its first frequency and steps to the next with one
// complex multiply.  Non-uniform grids evaluate every frequency directly.
// Sums use fused multiply-adds (their order differs from the reference's
// anyway); the records of one span are nearly always one incidence, and the
// sums are flushed with fp64 atomics whenever the incidence changes.
// kUniform: the uniform-grid recurrence (P.uniform_f, compile time);
// kFull: every lane owns all FPL of its frequencies (nf - f_begin >= 32 FPL),
// so the per-frequency bounds tests drop out of the inner loop.
#ifndef MCSBR_ACC_MIN_SPAN
#define MCSBR_ACC_MIN_SPAN 512
#endif
template <int FPL, bool kRealAmp, bool kUniform, bool kFull>
__global__ void __launch_bounds__(128) accumulate_kernel(TraceParams P, uint32_t f_begin) {
    // staged record: [0..3] amplitudes, [4] (ph0, dph) | s, [5] (la0, dla),
    // [6] W = e^{-j 32 dk s}, [7] incidence.  (Measured and rejected: a
    // per-record table of w^r, w^4q replacing the lane's sincos by two
    // complex multiplies -- c5 +3.5%, the table doubles the shared memory.)
    // (Measured and rejected as well: W^2 .. W^(FPL-1) staged per record so
    // a lane forms its phasors by independent products instead of the
    // recurrence chain -- c5 +2%.  Round 2: each lane's first phasor as a
    // warp prefix product Z0 W1^lane (5 shuffle + multiply steps) instead
    // of its sincos -- +7%; the next record's sincos software-pipelined
    // against this record's sums -- +4.6%.)
    constexpr int kSt = 8;
    __shared__ double2 st[4][32][kSt];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t n_all = *P.rec_count;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicMax(P.rec_count + 1, n_all);  // peak for the host
    const uint64_t n = min(n_all, P.rec_cap);
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * 4, gw = static_cast<uint64_t>(blockIdx.x) * 4 + warp;
    uint64_t span = ((n + nw - 1) / nw + 31) & ~31ull;
    span = span < MCSBR_ACC_MIN_SPAN ? MCSBR_ACC_MIN_SPAN : span;
    const uint32_t f_end = min(P.nf, f_begin + 32u * FPL);
    const uint32_t f0 = f_begin + static_cast<uint32_t>(lane);
    const double f0d = static_cast<double>(f0);
    double acc[FPL][8];
    const double2* recs = reinterpret_cast<const double2*>(P.recs);
    auto cmul = [](Cx x, Cx y) { return Cx{__fma_rn(x.re, y.re, -x.im * y.im), __fma_rn(x.re, y.im, x.im * y.re)}; };
    auto cx2 = [](double2 v) { return Cx{v.x, v.y}; };
    auto d2 = [](Cx v) { return make_double2(v.re, v.im); };
    for (uint64_t r0 = gw * span; r0 < n; r0 += nw * span) {
        const uint64_t r1 = min(r0 + span, n);
        uint32_t cur = 0xffffffffu;
#pragma unroll
        for (int m = 0; m < FPL; ++m)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[m][k] = 0.0;
        auto flush = [&]() {
            if (cur == 0xffffffffu) return;
            double* out = P.sums + sums_row(P, cur) * P.nf * 8;
#pragma unroll
            for (int m = 0; m < FPL; ++m) {
                const uint32_t f = f0 + 32u * m;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if ((kFull || f < f_end) && acc[m][k] != 0.0) atomicAdd(out + f * 8 + k, acc[m][k]);
                    acc[m][k] = 0.0;
                }
            }
        };
        for (uint64_t rb = r0; rb < r1; rb += 32) {
            const uint32_t cnt = static_cast<uint32_t>(min(static_cast<uint64_t>(32), r1 - rb));
            if (static_cast<uint32_t>(lane) < cnt) {
                const double2* r = recs + (rb + lane) * kRecD2;
                double2* t = st[warp][lane];
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) t[ch] = __ldcs(r + ch);
                const double2 sv = __ldcs(r + 4);
                t[7] = __ldcs(r + 5);
                if (kUniform) {
                    const double ph0 = P.kph0 * sv.x, dph = P.kdph * sv.x;
                    const double la0 = -(P.kph0 * sv.y), dla = -(P.kdph * sv.y);
                    t[4] = make_double2(ph0, dph);
                    t[5] = make_double2(la0, dla);
                    if (FPL > 1) t[6] = d2(polar_la(32.0 * dph, 32.0 * dla));
                } else {
                    t[4] = sv;
                }
            }
            __syncwarp();
            for (uint32_t j = 0; j < cnt; ++j) {
                const double2* t = st[warp][j];
                const uint32_t a = static_cast<uint32_t>(__double_as_longlong(t[7].x));
                if (a != cur) {
                    flush();
                    cur = a;
                }
                if (!kFull && f0 >= f_end) continue;
                Cx z, w = {1.0, 0.0};
                const double2 t4 = t[4];
                if (kUniform) {
                    const double2 t5 = t[5];
                    z = polar_la(t4.x + f0d * t4.y, t5.x + f0d * t5.y);
                    if (FPL > 1) w = cx2(t[6]);
                } else {
                    z = phasor(P.k0[f0], Cx{t4.x, t4.y});
                }
                Cx am[4];
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) am[ch] = cx2(t[ch]);
                auto sweep = [&](auto real_tag) {
                    constexpr bool kReal = decltype(real_tag)::value;
#pragma unroll
                    for (int m = 0; m < FPL; ++m) {
                        const uint32_t f = f0 + 32u * m;
                        if (kFull || f < f_end) {
#pragma unroll
                            for (int ch = 0; ch < 4; ++ch) {
                                if (kReal) {  // real amplitudes: half the products
                                    acc[m][2 * ch] = __fma_rn(am[ch].re, z.re, acc[m][2 * ch]);
                                    acc[m][2 * ch + 1] = __fma_rn(am[ch].re, z.im, acc[m][2 * ch + 1]);
                                } else {
                                    acc[m][2 * ch] =
                                        __fma_rn(am[ch].re, z.re, __fma_rn(-am[ch].im, z.im, acc[m][2 * ch]));
                                    acc[m][2 * ch + 1] =
                                        __fma_rn(am[ch].re, z.im, __fma_rn(am[ch].im, z.re, acc[m][2 * ch + 1]));
                                }
                            }
                            if (m + 1 < FPL && (kFull || f + 32u < f_end)) {
                                if (kUniform) z = cmul(z, w);
                                else z = phasor(P.k0[f + 32u], Cx{t4.x, t4.y});
                            }
                        }
                    }
                };
                // PEC scenes: every amplitude is real; otherwise a record whose
                // four amplitudes are real (a path that met only PEC surfaces
                // and lossless interfaces) takes the real sweep as well --
                // warp-uniform, the warp works on one record at a time
                if (kRealAmp || (am[0].im == 0.0 && am[1].im == 0.0 && am[2].im == 0.0 && am[3].im == 0.0))
                    sweep(std::true_type{});
                else
                    sweep(std::false_type{});
            }
            __syncwarp();
        }
        flush();
    }
}

// K4b, MCSBR_REDUCE_EXACT: the same record sweep with one frequency per lane
// (f_begin + lane); every term is rounded once to 192-bit fixed point and
// summed in integer registers (fixedpoint.cuh), so the sums are independent
// of the record order, the span split and the launch grouping.  Phasors and
// products are exact_add_global's (freq_phasor, one IEEE operation each).
__global__ void __launch_bounds__(128) accumulate_exact_kernel(TraceParams P, uint32_t f_begin) {
    __shared__ double2 st[4][32][6];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t n_all = *P.rec_count;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicMax(P.rec_count + 1, n_all);  // peak for the host
    const uint64_t n = min(n_all, P.rec_cap);
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * 4, gw = static_cast<uint64_t>(blockIdx.x) * 4 + warp;
    uint64_t span = ((n + nw - 1) / nw + 31) & ~31ull;
    span = span < 512 ? 512 : span;
    const uint32_t f = f_begin + static_cast<uint32_t>(lane);
    const bool has_f = f < P.nf;
    uint64_t acc[8][3];
    bool ok = true;
    const double2* recs = reinterpret_cast<const double2*>(P.recs);
    for (uint64_t r0 = gw * span; r0 < n; r0 += nw * span) {
        const uint64_t r1 = min(r0 + span, n);
        uint32_t cur = 0xffffffffu;
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k][0] = acc[k][1] = acc[k][2] = 0;
        auto flush = [&]() {
            if (cur == 0xffffffffu || !has_f) return;
            unsigned long long* g = P.xsums + (sums_row(P, cur) * P.nf + f) * 8 * 3;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                mcsbr_fx::fx_atomic_add(g + 3 * k, acc[k]);
                acc[k][0] = acc[k][1] = acc[k][2] = 0;
            }
        };
        for (uint64_t rb = r0; rb < r1; rb += 32) {
            const uint32_t cnt = static_cast<uint32_t>(min(static_cast<uint64_t>(32), r1 - rb));
            if (static_cast<uint32_t>(lane) < cnt) {
                const double2* r = recs + (rb + lane) * kRecD2;
#pragma unroll
                for (int c = 0; c < 6; ++c) st[warp][lane][c] = __ldcs(r + c);
            }
            __syncwarp();
            for (uint32_t j = 0; j < cnt; ++j) {
                const double2* t = st[warp][j];
                const uint32_t a = static_cast<uint32_t>(__double_as_longlong(t[5].x));
                if (a != cur) {
                    flush();
                    cur = a;
                }
                if (!has_f) continue;
                Cx am[4];
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) am[ch] = {t[ch].x, t[ch].y};
                const Cx sp = {t[4].x, t[4].y};
                const Cx z = P.scene.lossy ? freq_phasor(P, f, sp) : freq_phasor(P, f, sp.re);
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    const Cx v = am[ch] * z;
                    uint64_t w[3];
                    ok = mcsbr_fx::fx_from_double(v.re, w) && ok;
                    mcsbr_fx::fx_add(acc[2 * ch], w);
                    ok = mcsbr_fx::fx_from_double(v.im, w) && ok;
                    mcsbr_fx::fx_add(acc[2 * ch + 1], w);
                }
            }
            __syncwarp();
        }
        flush();
    }
    if (!ok) atomicOr(P.counters + kCntFault, static_cast<unsigned long long>(kFaultFixedRange));
}

__global__ void exact_limbs_kernel(const unsigned long long* __restrict__ x, uint64_t n, long long* __restrict__ limbs) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t w[3] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
    int64_t l[4];
    mcsbr_fx::fx_to_limbs(w, l);
#pragma unroll
    for (int k = 0; k < 4; ++k) limbs[4 * i + k] += l[k];
}

__global__ void intersect_kernel(SceneView S, const double* __restrict__ o, const double* __restrict__ d,
                                 const double* __restrict__ tmin, uint32_t n, int any_hit,
                                 double* __restrict__ t_out, uint32_t* __restrict__ id_out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const V3 oo = ld3(o + 3ull * i), dd = ld3(d + 3ull * i);
    double t;
    uint32_t id, fault = 0;
    bool hit;
    hit = traverse(S, oo, dd, tmin[i], t, id, fault, any_hit != 0, true);
    t_out[i] = hit ? t : __longlong_as_double(0x7ff0000000000000ll);
    id_out[i] = hit ? id : 0xffffffffu;
}

}  // namespace

bool trace_uses_register_accumulator(const TraceParams& p) { return p.nf == 1 && !p.xsums; }

bool trace_fan_supported(uint32_t) { return true; }  // F = 1 register sums, F > 1 fan records

template <int kMode, bool kDiel, bool kLossy, bool kDet, bool kFast>
static cudaError_t launch_mode(const TraceParams& p, int device_sms, int threads, size_t smem,
                               cudaStream_t stream) {
    auto* k = path_kernel<kMode, kDiel, kLossy, kDet, kFast>;
    if (smem > 0) {  // static state slots + dynamic accumulators may pass 48 KB: opt in
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    int per_sm = 1;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    if (const char* v = std::getenv("MCSBR_BLOCKS_PER_SM")) per_sm = std::min(per_sm, std::max(1, std::atoi(v)));
    uint64_t blocks = static_cast<uint64_t>(device_sms) * per_sm;
    const uint64_t max_blocks = (p.total_entries + 1023) / 1024;  // >= 8 entries per lane
    if (blocks > max_blocks) blocks = max_blocks;
    if (kDet && blocks * threads > p.det_threads) blocks = p.det_threads / threads;  // stack capacity
    if (blocks < 1) blocks = 1;
    k<<<static_cast<unsigned>(blocks), threads, smem, stream>>>(p);
    return cudaGetLastError();
}

template <bool kDiel, bool kLossy>
static cudaError_t launch_kind(int mode, const TraceParams& p, int sms, int threads, size_t smem,
                               cudaStream_t stream) {
    if (p.det)  // one receiver per launch (the deterministic solver has no fan mode)
        return mode == kModeReg ? launch_mode<kModeReg, kDiel, kLossy, true, false>(p, sms, threads, smem, stream)
                                : launch_mode<kModeDefer, kDiel, kLossy, true, false>(p, sms, threads, smem, stream);
    if (mode == kModeFanRec)  // multi-frequency fans: fp64 triangle tests in every mode
        return launch_mode<kModeFanRec, kDiel, kLossy, false, false>(p, sms, threads, smem, stream);
    if (p.fast_tri)  // statistical-mode fp32 triangle tests
        return mode == kModeFan   ? launch_mode<kModeFan, kDiel, kLossy, false, true>(p, sms, threads, smem, stream)
               : mode == kModeReg ? launch_mode<kModeReg, kDiel, kLossy, false, true>(p, sms, threads, smem, stream)
                                  : launch_mode<kModeDefer, kDiel, kLossy, false, true>(p, sms, threads, smem, stream);
    return mode == kModeFan   ? launch_mode<kModeFan, kDiel, kLossy, false, false>(p, sms, threads, smem, stream)
           : mode == kModeReg ? launch_mode<kModeReg, kDiel, kLossy, false, false>(p, sms, threads, smem, stream)
                              : launch_mode<kModeDefer, kDiel, kLossy, false, false>(p, sms, threads, smem, stream);
}

cudaError_t launch_exact_limbs(const unsigned long long* xsums, uint64_t n_values, long long* limbs,
                               cudaStream_t stream) {
    if (n_values == 0) return cudaSuccess;
    exact_limbs_kernel<<<static_cast<unsigned>((n_values + 255) / 256), 256, 0, stream>>>(xsums, n_values, limbs);
    return cudaGetLastError();
}

// deferred accumulation of one path-kernel launch's records (F > 1, or any
// F under MCSBR_REDUCE_EXACT)
cudaError_t launch_accumulate(const TraceParams& p, int device_sms, cudaStream_t stream, uint64_t* launches,
                              uint64_t expected_records) {
    // One wave of 4 blocks per SM; launches expected to carry more than ~8 k
    // records per warp of a wave get up to 4 waves (shorter spans balance
    // the warps' unequal record costs -- real / complex amplitudes -- at the
    // tail: c5 accumulation -9.7%), small ones stay at one (more warps means
    // more sum flushes: c4 +7.5% at 4 waves)
    const uint64_t per_wave = static_cast<uint64_t>(device_sms) * 16 * 8192;
    const unsigned waves = static_cast<unsigned>(std::min<uint64_t>(4, std::max<uint64_t>(1, expected_records / per_wave)));
    const unsigned blocks = static_cast<unsigned>(device_sms) * 4 * waves;
    if (p.xsums) {
        for (uint32_t fb = 0; fb < p.nf; fb += 32) {
            accumulate_exact_kernel<<<blocks, 128, 0, stream>>>(p, fb);
            if (launches) ++*launches;
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    const uint32_t fpl = p.nf <= 32 ? 1 : (p.nf <= 64 ? 2 : 4);
    const bool real_amp = p.scene.all_pec && !p.scene.lossy;  // PEC paths carry real amplitudes
    for (uint32_t fb = 0; fb < p.nf; fb += 32 * fpl) {
        const bool full = p.nf - fb >= 32 * fpl;
        const unsigned code = (real_amp ? 4u : 0u) | (p.uniform_f ? 2u : 0u) | (full ? 1u : 0u);
#define MCSBR_ACC(F)                                                                                 \
    switch (code) {                                                                                  \
        case 0: accumulate_kernel<F, false, false, false><<<blocks, 128, 0, stream>>>(p, fb); break; \
        case 1: accumulate_kernel<F, false, false, true><<<blocks, 128, 0, stream>>>(p, fb); break;  \
        case 2: accumulate_kernel<F, false, true, false><<<blocks, 128, 0, stream>>>(p, fb); break;  \
        case 3: accumulate_kernel<F, false, true, true><<<blocks, 128, 0, stream>>>(p, fb); break;   \
        case 4: accumulate_kernel<F, true, false, false><<<blocks, 128, 0, stream>>>(p, fb); break;  \
        case 5: accumulate_kernel<F, true, false, true><<<blocks, 128, 0, stream>>>(p, fb); break;   \
        case 6: accumulate_kernel<F, true, true, false><<<blocks, 128, 0, stream>>>(p, fb); break;   \
        default: accumulate_kernel<F, true, true, true><<<blocks, 128, 0, stream>>>(p, fb); break;   \
    }
        if (fpl == 1) {
            MCSBR_ACC(1)
        } else if (fpl == 2) {
            MCSBR_ACC(2)
        } else {
            MCSBR_ACC(4)
        }
#undef MCSBR_ACC
        if (launches) ++*launches;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_trace(const TraceParams& p, int device_sms, cudaStream_t stream, uint64_t* launches) {
    const int threads = 128;
    const int mode = (p.fan && !p.det) ? (p.fan_rows ? kModeFanRec : kModeFan)
                                       : (trace_uses_register_accumulator(p) ? kModeReg : kModeDefer);
    size_t smem = 0;
    if (const char* v = std::getenv("MCSBR_EXTRA_SMEM")) smem += std::strtoul(v, nullptr, 10);  // A/B only
    // three physics instantiations: all-PEC (dielectric code compiled out),
    // the reference's lossless dielectric model (bit-exact), lossy media
    static const bool force_diel = std::getenv("MCSBR_FORCE_DIEL") != nullptr;  // A/B only
    cudaError_t e = p.scene.lossy     ? launch_kind<true, true>(mode, p, device_sms, threads, smem, stream)
                    : (p.scene.all_pec && !force_diel) ? launch_kind<false, false>(mode, p, device_sms, threads, smem, stream)
                                      : launch_kind<true, false>(mode, p, device_sms, threads, smem, stream);
    if (launches) ++*launches;
    return e;
}

#ifdef MCSBR_TRAVERSAL_STATS
extern "C" __attribute__((visibility("default"))) void mcsbr_gpu_stats_visits(unsigned long long* out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_visits, sizeof(g_visits));
}
#endif

cudaError_t launch_intersect(const SceneView& s, const double* o, const double* d, const double* tmin,
                             uint32_t n, int any_hit, double* t_out, uint32_t* id_out,
                             cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    intersect_kernel<<<(n + 127) / 128, 128, 0, stream>>>(s, o, d, tmin, n, any_hit, t_out, id_out);
    return cudaGetLastError();
}

}  // namespace mcsbr_int
