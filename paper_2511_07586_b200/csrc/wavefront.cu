// Wavefront Monte Carlo SBR: the path kernel split into a lean traversal
// kernel and a shading kernel over a pool of paths in HBM.
//
// Why (profiles/r02*_c5_*): in the persistent megakernel (trace.cu) every
// lane does one query per iteration and then shades; on the 1M-triangle
// airframe with dielectric skins the dielectric instantiation runs at 128
// registers (16 warps / SM), spills ~1 KB per thread, and its traversal loop
// runs at ~8 of 32 lanes because launch rays (~19 node visits), surface
// rays (~9) and occlusion rays (~8) of different lengths share a warp and
// shading of mixed PEC / dielectric hits diverges.  Here:
//
//   wf_shade   one thread per pool slot: consumes the slot's query result
//              (closest hit -> advance, GO transport, MECA contribution,
//              branch choice, roulette; occlusion -> the contribution's
//              chi), emits contribution records, issues the slot's next
//              query, and regenerates dead slots from the launch entries
//              (coverage-culled, the same chunked cursor and band order as
//              the megakernel).  Active slots are appended to a work list.
//   wf_trace   persistent, 64 registers: warps take work-list batches and
//              every lane traverses its query; a lane whose query finishes
//              takes the next one at once (the traversal loop is one node or
//              leaf per step, refilled per step), so lanes stay busy
//              regardless of query length.
//
// The arithmetic is the megakernel's (pathcore.cuh, physics.cuh), operation
// for operation: hits, contributions and counters are identical; only the
// order of the deferred records differs, which accumulate_kernel sums
// anyway.  Used for the deferred-accumulation (F > 1) Monte Carlo mode
// without parity instrumentation (contribution / path logs keep the
// megakernel).
#include <cstdio>
#include <cstdlib>
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

// pool fields (doubles), SoA: field f of slot k at W.pool[f * W.np + k]
enum : int {
    kFo = 0,       // query origin (3)
    kFd = 3,       // query direction (3)
    kFpd = 6,      // the path's direction while an occlusion query is pending (3)
    kFt = 9,       // query result t
    kFe = 10,      // e0 (6: x.re x.im y.re y.im z.re z.im), e1 (6)
    kFphi = 22,    // phi (re, im)
    kFw = 24,      // weight
    kFprob = 25,   // prob
    kFmed = 26,    // medium_n (re, im)
    kFkey = 28,    // RNG key (u64 bits)
    kFcs = 29,     // cell | sample << 32 (u64 bits)
    kFmeta = 30,   // bounce | dying << 8 | incidence << 32 (u64 bits)
    kFamp = 31,    // pending contribution: 4 projected amplitudes (re, im)
    kFsp = 39,     // and its optical path (re, im)
    kWfFields = 41,
};
enum : uint32_t { kQNone = 0, kQLaunch = 1, kQSurface = 2, kQOcclusion = 3 };

struct Pool {
    double* p;
    uint32_t np;
    __device__ __forceinline__ double& at(int f, uint32_t k) const { return p[static_cast<size_t>(f) * np + k]; }
    __device__ __forceinline__ V3 v3(int f, uint32_t k) const { return {at(f, k), at(f + 1, k), at(f + 2, k)}; }
    __device__ __forceinline__ void set3(int f, uint32_t k, V3 v) const {
        at(f, k) = v.x;
        at(f + 1, k) = v.y;
        at(f + 2, k) = v.z;
    }
    __device__ __forceinline__ uint64_t u64(int f, uint32_t k) const {
        return static_cast<uint64_t>(__double_as_longlong(at(f, k)));
    }
    __device__ __forceinline__ void setu64(int f, uint32_t k, uint64_t v) const {
        at(f, k) = __longlong_as_double(static_cast<long long>(v));
    }
};

__device__ __forceinline__ void store_ef(const Pool& W, int f, uint32_t k, const CV3& e) {
    W.at(f, k) = e.x.re;
    W.at(f + 1, k) = e.x.im;
    W.at(f + 2, k) = e.y.re;
    W.at(f + 3, k) = e.y.im;
    W.at(f + 4, k) = e.z.re;
    W.at(f + 5, k) = e.z.im;
}
__device__ __forceinline__ void store_ef(const Pool& W, int f, uint32_t k, const V3& e) {
    W.at(f, k) = e.x;
    W.at(f + 2, k) = e.y;
    W.at(f + 4, k) = e.z;
}
__device__ __forceinline__ void load_ef(const Pool& W, int f, uint32_t k, CV3& e) {
    e = {{W.at(f, k), W.at(f + 1, k)}, {W.at(f + 2, k), W.at(f + 3, k)}, {W.at(f + 4, k), W.at(f + 5, k)}};
}
__device__ __forceinline__ void load_ef(const Pool& W, int f, uint32_t k, V3& e) {
    e = {W.at(f, k), W.at(f + 2, k), W.at(f + 4, k)};
}
template <typename NT>
__device__ __forceinline__ NT load_nt(const Pool& W, int f, uint32_t k) {
    return make_nt<NT>(W.at(f, k), std::is_same<NT, Cx>::value ? W.at(f + 1, k) : 0.0);
}
__device__ __forceinline__ void store_nt(const Pool& W, int f, uint32_t k, double v) { W.at(f, k) = v; }
__device__ __forceinline__ void store_nt(const Pool& W, int f, uint32_t k, Cx v) {
    W.at(f, k) = v.re;
    W.at(f + 1, k) = v.im;
}

__device__ __forceinline__ uint64_t pack_meta(int bounce, bool dying, uint32_t inc) {
    return static_cast<uint64_t>(bounce & 0xff) | (dying ? 0x100ull : 0ull) | (static_cast<uint64_t>(inc) << 32);
}

// ---------------------------------------------------------------------------
// wf_shade

#ifndef MCSBR_WF_SHADE_BLOCKS
#define MCSBR_WF_SHADE_BLOCKS 4  // 128 registers: 16 warps / SM
#endif
template <bool kDiel, bool kLossy>
__global__ void __launch_bounds__(128, MCSBR_WF_SHADE_BLOCKS) wf_shade(TraceParams P, WfParams Wp, uint32_t iter) {
    constexpr bool kPec = !kDiel && !kLossy;
    using NT = typename std::conditional<kLossy, Cx, double>::type;
    using EF = typename std::conditional<kPec, V3, CV3>::type;
    __shared__ unsigned long long s_cnt[9];
    __shared__ unsigned int s_bounce[3 * 64];
    __shared__ double s_rcp[4][2];
    for (int i = threadIdx.x; i < 9; i += blockDim.x) s_cnt[i] = 0;
    for (int i = threadIdx.x; i < 3 * 64; i += blockDim.x) s_bounce[i] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // the counters of the NEXT iteration (read by nobody now)
        Wp.list_n[(iter + 1) % 3] = 0;
        Wp.trace_cursor[(iter + 1) % 3] = 0;
    }
    __syncthreads();
    const Pool W{Wp.pool, Wp.np};
    const SceneView& S = P.scene;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;  // slot (np is a multiple of 128)
    uint32_t fault = 0;
    uint64_t n_launched = 0, n_contrib = 0, n_graze = 0, n_cap = 0, n_occ = 0, n_miss0 = 0;
    int max_round = 0;

    uint32_t kind = Wp.kind[k];
    bool dead = kind == kQNone;
    bool visible = false;  // a contribution to record now
    Cx amp[4];
    NT s_path{};
    uint32_t rec_inc = 0;
    uint32_t next = kQNone;

    if (kind == kQOcclusion) {
        // ---- chi visibility of the pending contribution (farfield.cpp:63-68) ----
        const uint64_t meta = W.u64(kFmeta, k);
        visible = Wp.rid[k] == 0xffffffffu;
        if (visible) {
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) amp[ch] = {W.at(kFamp + 2 * ch, k), W.at(kFamp + 2 * ch + 1, k)};
            s_path = load_nt<NT>(W, kFsp, k);
            rec_inc = P.inc[static_cast<uint32_t>(meta >> 32)].row;  // the unit's incidence
        }
        if (meta & 0x100ull) {
            dead = true;
        } else {  // the path continues from the exit point (= the occlusion ray's origin)
            W.set3(kFd, k, W.v3(kFpd, k));
            next = kQSurface;
            atomicAdd(&s_bounce[min(static_cast<int>(meta & 0xff), 63)], 1u);
        }
    } else if (kind != kQNone) {
        // ---- closest hit (solver_mc.cpp:142-210) ----
        const uint32_t id = Wp.rid[k];
        if (id == 0xffffffffu) {
            dead = true;  // escaped
        } else {
            const double t = W.at(kFt, k);
            const uint64_t meta = W.u64(kFmeta, k);
            const uint32_t unit = static_cast<uint32_t>(meta >> 32);  // the path's launch unit
            const IncDev& I = P.inc[unit];
            const uint32_t a = I.row;
            const RxDev& R = P.rx[static_cast<size_t>(a) * P.n_rx + P.rx_index];
            Path<NT, EF> s;
            s.origin = W.v3(kFo, k);
            s.dir = W.v3(kFd, k);
            load_ef(W, kFe, k, s.e0);
            load_ef(W, kFe + 6, k, s.e1);
            s.phi = load_nt<NT>(W, kFphi, k);
            s.weight = W.at(kFw, k);
            s.prob = W.at(kFprob, k);
            s.medium_n = load_nt<NT>(W, kFmed, k);
            s.key = W.u64(kFkey, k);
            s.bounce = static_cast<int>(meta & 0xff);
            const V3 point = s.origin + s.dir * t;
            const HitInfo<NT> h = fill_hit<NT>(S, id, s.dir);
            // advance (path_engine.cpp:17-21)
            s.phi = s.phi + s.medium_n * t;
            s.origin = point;
            s.bounce += 1;
            max_round = max(max_round, s.bounce);
            bool alive = true, candidate = false;
            const double cos_i = -dot(s.dir, h.normal);
            if (cos_i < 1e-6) {
                ++n_graze;
                alive = false;
            } else {
                const bool pec = kDiel ? h.far_side_pec : true;
                const NT n1 = s.medium_n;
                const NT n2 = pec ? n1 : h.n_transmit;
                const Coeffs co = pec ? coeffs_pec() : fresnel_any(n1, n2, cos_i, fault);
                Basis b;
                if constexpr (!kPec) b = sp_basis(s.dir, h.normal, re_of(n1), re_of(n2), !pec, fault);
                const bool two = !pec && !co.tir;
                if constexpr (!kPec) {
                    transverse_guard(s.e0, b, fault);
                    transverse_guard(s.e1, b, fault);
                }
                const int sc = pec ? 0 : (h.near_is_ambient ? 1 : 2);
                const bool dark_exit = sc == 2 && co.tir;
                candidate = !dark_exit && h.exterior_facing;
                if (candidate) {
                    // meca_currents (farfield.cpp:11-45), one copy of the three cases
                    const bool ex = sc == 2;
                    EF f0 = ef_zero<EF>(), f1 = ef_zero<EF>();
                    if (sc != 0) {
                        f0 = branch_field(s.e0, ex ? 1 : 0, co, b);
                        f1 = branch_field(s.e1, ex ? 1 : 0, co, b);
                    }
                    const V3 nrm = ex ? -h.normal : h.normal;
                    const V3 dj = ex ? b.dir_t : s.dir;
                    const NT nj = ex ? h.n_transmit : s.medium_n;
                    EF x0 = cross(dj, ex ? f0 : s.e0), x1 = cross(dj, ex ? f1 : s.e1);
                    if (sc == 1) {
                        x0 = x0 + cross(b.dir_r, f0);
                        x1 = x1 + cross(b.dir_r, f1);
                    }
                    EF j0 = cross(nrm, x0 * nj), j1 = cross(nrm, x1 * nj);
                    EF m0 = ef_zero<EF>(), m1 = ef_zero<EF>();
                    if (sc == 0) {
                        j0 = j0 * 2.0;
                        j1 = j1 * 2.0;
                    } else {
                        m0 = cross(ex ? f0 : s.e0 + f0, nrm);
                        m1 = cross(ex ? f1 : s.e1 + f1, nrm);
                    }
                    // make_contribution (farfield.cpp:70-85)
                    const double cos_n = fabs(dot(s.dir, h.normal));
                    const double scale = s.weight * I.area_weight / (s.prob * cos_n);
                    j0 = j0 * scale;
                    m0 = m0 * scale;
                    j1 = j1 * scale;
                    m1 = m1 * scale;
                    if constexpr (kPec) project_pec(R, j0, j1, amp);
                    else project(R, j0, m0, j1, m1, amp);
                    s_path = s.phi - dot(ld3(R.k_s), point);
                    rec_inc = a;
                }
                if constexpr (kPec) {  // PEC hits form the basis after their contribution
                    b = sp_basis(s.dir, h.normal, re_of(n1), re_of(n2), false, fault);
                    transverse_guard(s.e0, b, fault);
                    transverse_guard(s.e1, b, fault);
                }
                if (s.bounce >= P.max_bounce) {  // cap (solver_mc.cpp:176-179)
                    ++n_cap;
                    alive = false;
                } else {
                    // choose_branch (solver_mc.cpp:44-54, :181-190)
                    int pick = 0;
                    double pp = 1.0;
                    if (two) {
                        double p_reflect = 0.5;
                        if (P.fresnel_strategy) {
                            const double r_bar = 0.5 * (cabs(co.r_s) + cabs(co.r_p));
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
                        }
                    }
                }
            }
            // the next query: the chi test of the contribution first, then
            // (if the path lives on) its next closest hit
            if (alive) {
                store_ef(W, kFe, k, s.e0);
                store_ef(W, kFe + 6, k, s.e1);
                store_nt(W, kFphi, k, s.phi);
                W.at(kFw, k) = s.weight;
                W.at(kFprob, k) = s.prob;
                store_nt(W, kFmed, k, s.medium_n);
            }
            if (candidate && P.occlusion) {
                W.set3(kFo, k, point);
                W.set3(kFd, k, ld3(R.k_s));
                if (alive) W.set3(kFpd, k, s.dir);
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    W.at(kFamp + 2 * ch, k) = amp[ch].re;
                    W.at(kFamp + 2 * ch + 1, k) = amp[ch].im;
                }
                store_nt(W, kFsp, k, s_path);
                W.setu64(kFmeta, k, pack_meta(s.bounce, !alive, unit));
                next = kQOcclusion;
                ++n_occ;
            } else {
                visible = candidate;
                if (alive) {
                    W.set3(kFo, k, point);
                    W.set3(kFd, k, s.dir);
                    W.setu64(kFmeta, k, pack_meta(s.bounce, false, unit));
                    next = kQSurface;
                    atomicAdd(&s_bounce[min(s.bounce, 63)], 1u);
                }
            }
            dead = next == kQNone;
        }
    }

    // ---- record the visible contributions (deferred accumulation) ----
    {
        const unsigned vm = __ballot_sync(kFull, visible);
        if (vm) {
            n_contrib += visible ? 1 : 0;
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(P.rec_count, static_cast<unsigned long long>(__popc(vm)));
            base = __shfl_sync(kFull, base, 0);
            const uint64_t slot = base + __popc(vm & ((1u << lane) - 1u));
            const bool stored = visible && slot < P.rec_cap;
            if (stored) {
                double2* r = reinterpret_cast<double2*>(P.recs) + slot * kRecD2;
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) r[ch] = make_double2(amp[ch].re, amp[ch].im);
                r[4] = make_double2(re_of(s_path), im_of(s_path));
                r[5] = make_double2(__longlong_as_double(static_cast<long long>(rec_inc)), 0.0);
                if (P.rec_inc) P.rec_inc[slot] = rec_inc;
            }
            // record buffer full: add the contribution straight into the sums
            unsigned om = __ballot_sync(kFull, visible && !stored);
            while (om) {
                const int src = __ffs(om) - 1;
                om &= om - 1;
                Cx am[4];
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    am[ch].re = __shfl_sync(kFull, amp[ch].re, src);
                    am[ch].im = __shfl_sync(kFull, amp[ch].im, src);
                }
                const NT sp = shfl_nt(s_path, src);
                const uint32_t ia = __shfl_sync(kFull, rec_inc, src);
                double* out = P.sums + (static_cast<size_t>(ia) * P.n_rx + P.rx_index) * P.nf * 8;
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

    // ---- regenerate dead slots from the launch entries ----
    // The warp keeps a range [cur, end) of the group's flattened entry space
    // across launches (Wp.wrange), fetched in guided chunks from the global
    // cursor like the megakernel's; coverage-culled entries are retired as
    // launched bounce-0 misses without generation or traversal.
    unsigned need = __ballot_sync(kFull, dead);
    if (need) {
        const uint64_t gw = k >> 5;
        unsigned long long* wr = Wp.wrange + 2 * gw;
        uint64_t cur = wr[0], end = wr[1];
        const uint64_t n_warps = Wp.np >> 5;
        while (need) {
            if (cur >= end) {
                const unsigned long long seen = *reinterpret_cast<volatile unsigned long long*>(P.tile_counter);
                const uint64_t rem = P.total_entries > seen ? P.total_entries - seen : 0;
                uint64_t c = P.gss_div ? rem / (P.gss_div * n_warps) : P.chunk_max;
                c = (c + 31) & ~31ull;
                c = c < P.chunk_min ? P.chunk_min : (c > P.chunk_max ? P.chunk_max : c);
                unsigned long long g = 0;
                if (lane == 0) g = atomicAdd(P.tile_counter, static_cast<unsigned long long>(c));
                g = __shfl_sync(kFull, g, 0);
                if (g >= P.total_entries) {
                    cur = end = 0;
                    break;  // every entry of the group is taken
                }
                cur = g;
                end = min(static_cast<uint64_t>(g + c), P.total_entries);
            }
            // the incidence containing cur (last a with g_begin[a] <= cur)
            uint32_t lo = 0, hi = P.n_inc;
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (P.inc[mid].g_begin <= cur) lo = mid; else hi = mid;
            }
            const uint32_t u = lo;  // launch unit
            const IncDev& I = P.inc[u];
            const uint32_t a = I.row;
            const uint64_t g_end_a = I.g_begin + (I.entry_end - I.entry_begin);
            const uint64_t sub_end = min(end, g_end_a);
            uint64_t dcur = I.entry_begin + (cur - I.g_begin);
            const uint64_t dend = I.entry_begin + (sub_end - I.g_begin);
            if (P.cover && I.cover_off != kNoCover) {
                const uint64_t d2 = skip_uncovered(P.cover + I.cover_off, I.cover_shift, dcur, dend);
                if (lane == 0) n_miss0 += d2 - dcur;
                dcur = d2;
            }
            if (dcur < dend) {
                if (lane == 0) {
                    s_rcp[warp][0] = mcsbr_dev::rcp_seed(I.nu);
                    s_rcp[warp][1] = mcsbr_dev::rcp_seed(I.nv);
                }
                __syncwarp();
                const unsigned rank = __popc(need & ((1u << lane) - 1u));
                const uint64_t mine = dcur + rank;
                if (dead && mine < dend) {
                    if (!covered(P, I, mine)) {
                        ++n_miss0;
                    } else {
                        Path<NT, EF> s;
                        init_path(P, I, a + P.inc_base, locate(P, I, mine), s, s_rcp[warp]);
                        W.set3(kFo, k, s.origin);
                        W.set3(kFd, k, s.dir);
                        store_ef(W, kFe, k, s.e0);
                        store_ef(W, kFe + 6, k, s.e1);
                        store_nt(W, kFphi, k, s.phi);
                        W.at(kFw, k) = s.weight;
                        W.at(kFprob, k) = s.prob;
                        store_nt(W, kFmed, k, s.medium_n);
                        W.setu64(kFkey, k, s.key);
                        W.setu64(kFcs, k, static_cast<uint64_t>(s.cell) | (static_cast<uint64_t>(s.sample) << 32));
                        W.setu64(kFmeta, k, pack_meta(0, false, u));
                        next = kQLaunch;
                        dead = false;
                        ++n_launched;
                        atomicAdd(&s_bounce[0], 1u);
                    }
                }
                dcur = min(dcur + static_cast<uint64_t>(__popc(need)), dend);
                __syncwarp();
            }
            cur = I.g_begin + (dcur - I.entry_begin);
            need = __ballot_sync(kFull, dead);
        }
        if (lane == 0) {
            wr[0] = cur;
            wr[1] = end;
        }
    }
    Wp.kind[k] = next;

    // ---- the work list of the next trace ----
    {
        const unsigned am = __ballot_sync(kFull, next != kQNone);
        if (am) {
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(Wp.list_n + iter % 3, static_cast<unsigned long long>(__popc(am)));
            base = __shfl_sync(kFull, base, 0);
            if (next != kQNone) Wp.list[base + __popc(am & ((1u << lane) - 1u))] = k;
        }
    }

    // ---- counters (trace.cu path_kernel layout) ----
    auto wsum = [](uint64_t v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        return v;
    };
    if (n_miss0) atomicAdd(&s_bounce[0], static_cast<unsigned int>(n_miss0));
    n_launched = wsum(n_launched + n_miss0);
    n_miss0 = wsum(n_miss0);
    n_contrib = wsum(n_contrib);
    n_graze = wsum(n_graze);
    n_cap = wsum(n_cap);
    n_occ = wsum(n_occ);
    const unsigned fault_w = __reduce_or_sync(kFull, fault);
    const int round_w = __reduce_max_sync(kFull, max_round);
    if (lane == 0) {
        if (n_launched) atomicAdd(&s_cnt[kCntLaunched], n_launched);
        if (n_contrib) atomicAdd(&s_cnt[kCntContrib], n_contrib);
        if (n_graze) atomicAdd(&s_cnt[kCntGrazing], n_graze);
        if (n_cap) atomicAdd(&s_cnt[kCntCap], n_cap);
        if (n_occ) atomicAdd(&s_cnt[kCntOcclusion], n_occ);
        if (fault_w) atomicOr(&s_cnt[kCntFault], static_cast<unsigned long long>(fault_w));
        if (round_w) atomicMax(&s_cnt[kCntRounds], static_cast<unsigned long long>(round_w));
        if (n_miss0) atomicAdd(&s_cnt[8], n_miss0);
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
// wf_trace: traversal of the work list, one node / leaf per step, lanes
// refilled per step (the megakernel's traverse(), pathcore.cuh, restated as a
// resumable state machine; identical box and triangle arithmetic)

#ifndef MCSBR_WF_TRACE_BLOCKS
#define MCSBR_WF_TRACE_BLOCKS 8  // 64 registers: 32 warps / SM
#endif

__global__ void __launch_bounds__(128, MCSBR_WF_TRACE_BLOCKS) wf_trace(SceneView S, WfParams Wp, uint32_t iter) {
    const Pool W{Wp.pool, Wp.np};
    const int lane = threadIdx.x & 31;
    const unsigned long long n = Wp.list_n[iter % 3];
    unsigned long long* cursor = Wp.trace_cursor + iter % 3;
    // the warp's batch of work-list entries [qb, qe)
    unsigned long long qb = 0, qe = 0;
    bool drained = false;  // the work list is used up (warp-uniform)
    bool active = false;
    uint32_t k = 0;
    bool any = false;
    V3 o = {0.0, 0.0, 0.0}, d = {0.0, 0.0, 0.0};
    double t_min = 0.0, best_t = 0.0;
    uint32_t best_id = 0xffffffffu;
    float tmax = 0.f;
    FRay r{};
    int stack[kStackSize];
    int sp = 0, ref = 0;
    for (;;) {
        // ---- refill idle lanes ----
        unsigned idle = __ballot_sync(kFull, !active);
        while (idle && !drained) {
            if (qb >= qe) {
                unsigned long long g = 0;
                if (lane == 0) g = atomicAdd(cursor, 64ull);
                g = __shfl_sync(kFull, g, 0);
                if (g >= n) {
                    drained = true;
                    break;
                }
                qb = g;
                qe = min(g + 64ull, n);
            }
            const unsigned rank = __popc(idle & ((1u << lane) - 1u));
            if (!active && qb + rank < qe) {
                k = Wp.list[qb + rank];
                const uint32_t kind = Wp.kind[k];
                o = W.v3(kFo, k);
                d = W.v3(kFd, k);
                any = kind == kQOcclusion;
                const bool outside = kind == kQLaunch;
                t_min = outside ? 0.0 : S.t_eps;
                r = make_fray(S, o, d, outside, t_min);
                best_t = __longlong_as_double(0x7ff0000000000000ll);
                best_id = 0xffffffffu;
                tmax = __int_as_float(0x7f800000);
                sp = 0;
                ref = S.root_ref;
                active = true;
            }
            qb = min(qb + static_cast<unsigned long long>(__popc(idle)), qe);
            idle = __ballot_sync(kFull, !active);
        }
        if (!__any_sync(kFull, active)) break;
        if (!active) continue;
        // ---- one step ----
        bool done = false;
        if (ref >= 0) {
            const float4* nd = S.nodes + 8ll * ref;
            const uint64_t nb = reinterpret_cast<uint64_t>(nd);
            auto plane = [](uint64_t addr) { return __ldg(reinterpret_cast<const float4*>(addr)); };
            const float4 nx = plane(nb | r.offx), fx = plane((nb | r.offx) ^ 16u);
            const float4 ny = plane(nb | r.offy), fy = plane((nb | r.offy) ^ 16u);
            const float4 nz = plane(nb | r.offz), fz = plane((nb | r.offz) ^ 16u);
            const float4 rf = __ldg(nd + 6);
            const float2 xn[2] = {ffma2(nx.x, nx.y, r.ix, -r.onx), ffma2(nx.z, nx.w, r.ix, -r.onx)};
            const float2 yn[2] = {ffma2(ny.x, ny.y, r.iy, -r.ony), ffma2(ny.z, ny.w, r.iy, -r.ony)};
            const float2 zn[2] = {ffma2(nz.x, nz.y, r.iz, -r.onz), ffma2(nz.z, nz.w, r.iz, -r.onz)};
            const float2 xf[2] = {ffma2(fx.x, fx.y, r.ix, -r.ofx), ffma2(fx.z, fx.w, r.ix, -r.ofx)};
            const float2 yf[2] = {ffma2(fy.x, fy.y, r.iy, -r.ofy), ffma2(fy.z, fy.w, r.iy, -r.ofy)};
            const float2 zf[2] = {ffma2(fz.x, fz.y, r.iz, -r.ofz), ffma2(fz.z, fz.w, r.iz, -r.ofz)};
            uint32_t kk[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int h = j >> 1;
                const float a_n = (j & 1) ? xn[h].y : xn[h].x, b_n = (j & 1) ? yn[h].y : yn[h].x;
                const float c_n = (j & 1) ? zn[h].y : zn[h].x;
                const float a_f = (j & 1) ? xf[h].y : xf[h].x, b_f = (j & 1) ? yf[h].y : yf[h].x;
                const float c_f = (j & 1) ? zf[h].y : zf[h].x;
                const float tn = fmax3(a_n, b_n, fmaxf(c_n, r.tlo));
                const float tf = fmin3(a_f, b_f, fminf(c_f, tmax));
                kk[j] = ((tn <= tf ? __float_as_uint(tn) : 0x7f800000u) & ~3u) | static_cast<uint32_t>(j);
            }
            constexpr uint32_t kMiss = 0x7f800000u;
            const int rc[4] = {__float_as_int(rf.x), __float_as_int(rf.y), __float_as_int(rf.z), __float_as_int(rf.w)};
            auto child = [&](uint32_t key) {
                const uint32_t j = key & 3u;
                return (j & 2u) ? ((j & 1u) ? rc[3] : rc[2]) : ((j & 1u) ? rc[1] : rc[0]);
            };
            const unsigned hm = (kk[0] < kMiss ? 1u : 0u) | (kk[1] < kMiss ? 2u : 0u) | (kk[2] < kMiss ? 4u : 0u) |
                                (kk[3] < kMiss ? 8u : 0u);
            if (hm && (hm & (hm - 1u)) == 0u) {
                ref = child(static_cast<uint32_t>(__ffs(hm) - 1));
            } else if (hm) {
#define MCSBR_KSWAP(a, b)               \
    {                                   \
        const uint32_t lo_ = min(a, b); \
        b = max(a, b);                  \
        a = lo_;                        \
    }
                MCSBR_KSWAP(kk[0], kk[1])
                MCSBR_KSWAP(kk[2], kk[3])
                MCSBR_KSWAP(kk[0], kk[2])
                MCSBR_KSWAP(kk[1], kk[3])
                MCSBR_KSWAP(kk[1], kk[2])
#undef MCSBR_KSWAP
                if (kk[3] < kMiss) stack[sp++] = child(kk[3]);
                if (kk[2] < kMiss) stack[sp++] = child(kk[2]);
                stack[sp++] = child(kk[1]);
                ref = child(kk[0]);
            } else if (sp == 0) {
                done = true;
            } else {
                ref = stack[--sp];
            }
        } else {
            const uint32_t code = static_cast<uint32_t>(~ref);
            const uint32_t first = code >> 3, count = code & 7u;
            for (uint32_t j = 0; j < count; ++j) {
                double t;
                uint32_t id;
                if (tri_test(S.tri64 + 5ull * (first + j), o, d, t_min, t, id)) {
                    if (t < best_t || (t == best_t && id < best_id)) {
                        best_t = t;
                        best_id = id;
                        tmax = __double2float_ru((t - r.t_skip) * (1.0 + 1e-9));
                        if (any) break;
                    }
                }
            }
            if ((any && best_id != 0xffffffffu) || sp == 0) done = true;
            else ref = stack[--sp];
        }
        if (done) {
            W.at(kFt, k) = best_t;
            Wp.rid[k] = best_id;
            active = false;
        }
    }
}

}  // namespace

template <bool kDiel, bool kLossy>
static cudaError_t shade_launch(const TraceParams& p, const WfParams& w, uint32_t iter, cudaStream_t stream) {
    wf_shade<kDiel, kLossy><<<w.np / 128, 128, 0, stream>>>(p, w, iter);
    return cudaGetLastError();
}

cudaError_t launch_wavefront_iteration(const TraceParams& p, const WfParams& w, uint32_t iter, int device_sms,
                                       cudaStream_t stream) {
    cudaError_t e = p.scene.lossy     ? shade_launch<true, true>(p, w, iter, stream)
                    : p.scene.all_pec ? shade_launch<false, false>(p, w, iter, stream)
                                      : shade_launch<true, false>(p, w, iter, stream);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wf_trace, 128, 0);
    if (e != cudaSuccess) return e;
    wf_trace<<<static_cast<unsigned>(device_sms * (per_sm < 1 ? 1 : per_sm)), 128, 0, stream>>>(p.scene, w, iter);
    return cudaGetLastError();
}

}  // namespace mcsbr_int
