// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (compiled from the
// sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libmcsbr_ref.so).  It exposes the reference's public API
// (proj/include/mcsbr/*.hpp) with the same POD structs as the product's C ABI
// (include/mcsbr_gpu.h) so tests can (a) generate golden vectors, (b) pin the
// C restatement in oracle/mcsbr_oracle.c and (c) time the reference CPU solver
// as bench.py's reference arm.  Only tests/, smoke() and bench.py's
// cpu_baseline / --impl reference leg may load it.
#include <cstring>
#include <exception>
#include <map>
#include <string>
#include <vector>

#include "mcsbr/em_math.hpp"
#include "mcsbr/farfield.hpp"
#include "mcsbr/geometry.hpp"
#include "mcsbr/oracles.hpp"
#include "mcsbr/path_engine.hpp"
#include "mcsbr/rng.hpp"
#include "mcsbr/scenes.hpp"
#include "mcsbr/signal_processing.hpp"
#include "mcsbr/solver_common.hpp"
#include "mcsbr/solver_mc.hpp"
#include "mcsbr/solver_det.hpp"
#include "mcsbr/config.hpp"
#include "mcsbr/runner.hpp"
#include "mcsbr_gpu.h"

using namespace mcsbr;

static_assert(sizeof(Triangle) == sizeof(mcsbr_triangle), "Triangle layout");
static_assert(sizeof(Material) == sizeof(mcsbr_material), "Material layout");
static_assert(sizeof(Contribution) == sizeof(mcsbr_contribution), "Contribution layout");

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    return -1;
}
Vec3 v3(const double* p) { return {p[0], p[1], p[2]}; }
void put(double* p, const Vec3& v) {
    p[0] = v.x;
    p[1] = v.y;
    p[2] = v.z;
}
void putc(double* p, const complexd& c) {
    p[0] = c.real();
    p[1] = c.imag();
}
void putcv(double* p, const ComplexVec3& v) {
    putc(p, v.x);
    putc(p + 2, v.y);
    putc(p + 4, v.z);
}
ComplexVec3 getcv(const double* p) {
    return {complexd(p[0], p[1]), complexd(p[2], p[3]), complexd(p[4], p[5])};
}
// coefficient block: r_s, r_p, t_s, t_p, cos_t (complex) + tir flag = 11 doubles
void put_coeffs(double* p, const InterfaceCoefficients& c) {
    putc(p, c.r_s);
    putc(p + 2, c.r_p);
    putc(p + 4, c.t_s);
    putc(p + 6, c.t_p);
    putc(p + 8, c.cos_theta_t);
    p[10] = c.total_internal_reflection ? 1.0 : 0.0;
}
InterfaceCoefficients get_coeffs(const double* p) {
    InterfaceCoefficients c;
    c.r_s = {p[0], p[1]};
    c.r_p = {p[2], p[3]};
    c.t_s = {p[4], p[5]};
    c.t_p = {p[6], p[7]};
    c.cos_theta_t = {p[8], p[9]};
    c.total_internal_reflection = p[10] != 0.0;
    return c;
}
// basis block: s, p_in, p_out_r, p_out_t, dir_r, dir_t = 18 doubles
void put_basis(double* p, const SpBasis& b) {
    put(p, b.s_hat);
    put(p + 3, b.p_hat_in);
    put(p + 6, b.p_hat_out_r);
    put(p + 9, b.p_hat_out_t);
    put(p + 12, b.dir_r);
    put(p + 15, b.dir_t);
}
SpBasis get_basis(const double* p) {
    SpBasis b;
    b.s_hat = v3(p);
    b.p_hat_in = v3(p + 3);
    b.p_hat_out_r = v3(p + 6);
    b.p_hat_out_t = v3(p + 9);
    b.dir_r = v3(p + 12);
    b.dir_t = v3(p + 15);
    return b;
}
// hit block: t, point[3], normal[3], n_incident, n_transmit, far_side_pec,
// exterior_facing, near_is_ambient, triangle_id = 13 doubles
Hit get_hit(const double* p) {
    Hit h;
    h.t = p[0];
    h.point = v3(p + 1);
    h.normal = v3(p + 4);
    h.n_incident = p[7];
    h.n_transmit = p[8];
    h.far_side_pec = p[9] != 0.0;
    h.exterior_facing = p[10] != 0.0;
    h.near_is_ambient = p[11] != 0.0;
    h.triangle_id = static_cast<uint32_t>(p[12]);
    return h;
}
void put_hit(double* p, const Hit& h) {
    p[0] = h.t;
    put(p + 1, h.point);
    put(p + 4, h.normal);
    p[7] = h.n_incident;
    p[8] = h.n_transmit;
    p[9] = h.far_side_pec;
    p[10] = h.exterior_facing;
    p[11] = h.near_is_ambient;
    p[12] = h.triangle_id;
}
McConfig to_mc(const mcsbr_mc_config& c) {
    McConfig m;
    m.strata_per_wavelength = c.strata_per_wavelength;
    m.samples_per_stratum = c.samples_per_stratum;
    m.branch_strategy =
        c.branch_strategy == MCSBR_BRANCH_FRESNEL ? BranchStrategy::kFresnel : BranchStrategy::kFiftyFifty;
    m.roulette.enabled = c.roulette_enabled != 0;
    m.roulette.q = c.roulette_q;
    m.roulette.min_bounce = c.roulette_min_bounce;
    m.max_bounce = c.max_bounce;
    m.seed = c.seed;
    m.reference_wavelength = c.reference_wavelength;
    m.launch_padding = c.launch_padding;
    m.p_min = c.p_min;
    m.jitter = c.jitter != 0;
    m.block_size = c.block_size;
    return m;
}
Excitation to_exc(const mcsbr_excitation& e) {
    Excitation x;
    x.k_inc = v3(e.k_inc);
    x.pol_v = v3(e.pol_v);
    x.pol_h = v3(e.pol_h);
    x.k_scatter = v3(e.k_scatter);
    x.rx_v = v3(e.rx_v);
    x.rx_h = v3(e.rx_h);
    x.occlusion_enabled = e.occlusion_enabled != 0;
    return x;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- rng (rng.hpp:29-44) ---------------------------------------------------
uint64_t ref_counter_hash(uint64_t seed, uint64_t stratum, uint64_t sample, uint64_t bounce,
                          uint64_t purpose) {
    return counter_hash(seed, stratum, sample, bounce, static_cast<RngPurpose>(purpose));
}
double ref_counter_uniform(uint64_t seed, uint64_t stratum, uint64_t sample, uint64_t bounce,
                           uint64_t purpose) {
    return counter_uniform(seed, stratum, sample, bounce, static_cast<RngPurpose>(purpose));
}

// ---- em_math (em_math.cpp) ---------------------------------------------------
int ref_fresnel(double n1, double n2, double cos_i, double* out11) {
    try {
        put_coeffs(out11, fresnel(n1, n2, cos_i));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
int ref_sp_basis(const double* dir, const double* normal, double n1, double n2, double* out18) {
    try {
        put_basis(out18, sp_basis(v3(dir), v3(normal), n1, n2));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
int ref_interface_transform(const double* e6, int branch, const double* coeffs11,
                            const double* basis18, double* out6) {
    try {
        putcv(out6, interface_transform(getcv(e6), branch ? Branch::kTransmit : Branch::kReflect,
                                        get_coeffs(coeffs11), get_basis(basis18)));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- path engine (path_engine.cpp) ------------------------------------------
// state block in: origin[3], dir[3], e0[6], e1[6], phi, prob, weight, medium_n, bounce = 23
// branch set out: count, grazing, coeffs[11], basis[18], then per outcome
// new_dir[3], new_e0[6], new_e1[6], new_n = 16 each  -> 2 + 11 + 18 + 32 = 63 doubles
int ref_branch_outcomes(const double* state23, const double* hit13, double* out63) {
    try {
        PathState s;
        s.origin = v3(state23);
        s.dir = v3(state23 + 3);
        s.e[0] = getcv(state23 + 6);
        s.e[1] = getcv(state23 + 12);
        s.phi = state23[18];
        s.prob = state23[19];
        s.weight = state23[20];
        s.medium_n = state23[21];
        s.bounce = static_cast<int>(state23[22]);
        const BranchSet set = branch_outcomes(s, get_hit(hit13));
        std::memset(out63, 0, 63 * sizeof(double));
        out63[0] = set.count;
        out63[1] = set.grazing;
        if (set.grazing) return 0;
        put_coeffs(out63 + 2, set.coeffs);
        put_basis(out63 + 13, set.basis);
        for (int i = 0; i < set.count; ++i) {
            double* o = out63 + 31 + 16 * i;
            put(o, set.outcomes[i].new_dir);
            putcv(o + 3, set.outcomes[i].new_e[0]);
            putcv(o + 9, set.outcomes[i].new_e[1]);
            o[15] = set.outcomes[i].new_n;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- farfield (farfield.cpp) -------------------------------------------------
// generic meca: out j[6], m[6]
int ref_meca_currents(const double* hit13, const double* e6, const double* dir, int scatter_case,
                      double* out12) {
    try {
        const SurfaceCurrents c = meca_currents(get_hit(hit13), getcv(e6), v3(dir),
                                                static_cast<ScatterCase>(scatter_case));
        putcv(out12, c.j);
        putcv(out12 + 6, c.m);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
int ref_meca_currents_hot(const double* hit13, const double* e6, const double* dir,
                          int scatter_case, const double* coeffs11, const double* basis18,
                          double medium_n, double* out12) {
    try {
        const SurfaceCurrents c =
            meca_currents(get_hit(hit13), getcv(e6), v3(dir), static_cast<ScatterCase>(scatter_case),
                          get_coeffs(coeffs11), get_basis(basis18), medium_n);
        putcv(out12, c.j);
        putcv(out12 + 6, c.m);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Evaluate a contribution list against a sweep grid (evaluate_sweep,
// farfield.cpp:171-176); values out [4][nf] complex.
int ref_evaluate_sweep(const mcsbr_contribution* contribs, uint64_t n, const double* freqs,
                       uint32_t nf, const double* k_s, const double* rx_v, const double* rx_h,
                       double* values) {
    try {
        std::vector<Contribution> list(n);
        std::memcpy(static_cast<void*>(list.data()), contribs, n * sizeof(Contribution));
        SweepGrid grid{std::vector<double>(freqs, freqs + nf), v3(k_s), v3(rx_v), v3(rx_h)};
        const SweepResult r = evaluate_sweep(list, grid);
        for (int ch = 0; ch < kPolChannelCount; ++ch)
            for (uint32_t i = 0; i < nf; ++i) putc(values + 2 * (ch * nf + i), r.values[ch][i]);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- excitation (solver_common.cpp:15-49) ----------------------------------
void ref_monostatic_excitation(double theta, double phi, mcsbr_excitation* out) {
    const Excitation e = monostatic_excitation(theta, phi);
    std::memset(out, 0, sizeof(*out));
    put(out->k_inc, e.k_inc);
    put(out->pol_v, e.pol_v);
    put(out->pol_h, e.pol_h);
    put(out->k_scatter, e.k_scatter);
    put(out->rx_v, e.rx_v);
    put(out->rx_h, e.rx_h);
    out->occlusion_enabled = e.occlusion_enabled;
}
void ref_bistatic_excitation(double theta, double phi, double rx_theta, double rx_phi,
                             mcsbr_excitation* out) {
    const Excitation e = bistatic_excitation(theta, phi, rx_theta, rx_phi);
    std::memset(out, 0, sizeof(*out));
    put(out->k_inc, e.k_inc);
    put(out->pol_v, e.pol_v);
    put(out->pol_h, e.pol_h);
    put(out->k_scatter, e.k_scatter);
    put(out->rx_v, e.rx_v);
    put(out->rx_h, e.rx_h);
    out->occlusion_enabled = e.occlusion_enabled;
}

// ---- scenes (geometry_io.cpp, scenes.cpp) ------------------------------------
void* ref_scene_load(const char* mesh_obj, const char* material_map) {
    try {
        return new Scene(load_scene(mesh_obj, material_map));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}
void* ref_scene_builtin(const char* name, const char** keys, const double* vals, int n) {
    try {
        std::map<std::string, double> params;
        for (int i = 0; i < n; ++i) params[keys[i]] = vals[i];
        return new Scene(make_builtin_scene(name, params));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}
// builtin scene text (OBJ + material JSON) into caller buffers; returns needed sizes
int ref_builtin_text(const char* name, const char** keys, const double* vals, int n, char* obj,
                     uint64_t obj_cap, char* mat, uint64_t mat_cap, uint64_t* obj_len,
                     uint64_t* mat_len) {
    try {
        std::map<std::string, double> params;
        for (int i = 0; i < n; ++i) params[keys[i]] = vals[i];
        const SceneFiles f = builtin_scene(name, params);
        *obj_len = f.mesh_obj.size();
        *mat_len = f.material_map.size();
        if (obj && obj_cap > f.mesh_obj.size()) std::memcpy(obj, f.mesh_obj.c_str(), f.mesh_obj.size() + 1);
        if (mat && mat_cap > f.material_map.size())
            std::memcpy(mat, f.material_map.c_str(), f.material_map.size() + 1);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
void ref_scene_free(void* s) { delete static_cast<Scene*>(s); }
void ref_scene_sizes(const void* sp, uint32_t* nv, uint32_t* nt, uint32_t* nm) {
    const Scene& s = *static_cast<const Scene*>(sp);
    *nv = static_cast<uint32_t>(s.vertices.size());
    *nt = static_cast<uint32_t>(s.triangles.size());
    *nm = static_cast<uint32_t>(s.materials.size());
}
void ref_scene_export(const void* sp, double* xyz, mcsbr_triangle* tris, mcsbr_material* mats,
                      double* bounds5) {
    const Scene& s = *static_cast<const Scene*>(sp);
    for (size_t i = 0; i < s.vertices.size(); ++i) put(xyz + 3 * i, s.vertices[i]);
    for (size_t i = 0; i < s.triangles.size(); ++i) {
        const Triangle& t = s.triangles[i];
        mcsbr_triangle& o = tris[i];
        std::memset(&o, 0, sizeof(o));
        o.v0 = t.v0;
        o.v1 = t.v1;
        o.v2 = t.v2;
        put(o.normal, t.normal);
        o.front_material = t.front_material;
        o.back_material = t.back_material;
        o.exterior_facing = t.exterior_facing;
    }
    for (size_t i = 0; i < s.materials.size(); ++i) {
        std::memset(&mats[i], 0, sizeof(mats[i]));
        mats[i].eps_r = s.materials[i].eps_r;
        mats[i].mu_r = s.materials[i].mu_r;
        mats[i].is_pec = s.materials[i].is_pec;
    }
    put(bounds5, s.bounding_center());
    bounds5[3] = s.bounding_radius();
    bounds5[4] = s.diameter();
}
// Build a reference Scene from POD arrays (public data + finalize()).
void* ref_scene_from_arrays(const double* xyz, uint32_t nv, const mcsbr_triangle* tris,
                            uint32_t nt, const mcsbr_material* mats, uint32_t nm) {
    try {
        auto* s = new Scene();
        s->vertices.resize(nv);
        for (uint32_t i = 0; i < nv; ++i) s->vertices[i] = v3(xyz + 3 * i);
        s->triangles.resize(nt);
        for (uint32_t i = 0; i < nt; ++i) {
            Triangle& t = s->triangles[i];
            t.v0 = tris[i].v0;
            t.v1 = tris[i].v1;
            t.v2 = tris[i].v2;
            t.normal = v3(tris[i].normal);
            t.front_material = tris[i].front_material;
            t.back_material = tris[i].back_material;
            t.exterior_facing = tris[i].exterior_facing != 0;
        }
        s->materials.resize(nm);
        for (uint32_t i = 0; i < nm; ++i) {
            s->materials[i].eps_r = mats[i].eps_r;
            s->materials[i].mu_r = mats[i].mu_r;
            s->materials[i].is_pec = mats[i].is_pec != 0;
            s->material_names.push_back("m" + std::to_string(i));
        }
        s->finalize();
        return s;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

// Batched Scene::intersect / intersect_brute_force / occluded.
// mode 0 = intersect, 1 = brute force, 2 = occluded (t_min ignored).
// hit_out: n x 13 doubles (put_hit) with t = inf, id = 2^32-1 on a miss.
int ref_intersect(const void* sp, const double* o, const double* d, const double* t_min,
                  uint64_t n, int mode, double* hit_out) {
    const Scene& s = *static_cast<const Scene*>(sp);
    for (uint64_t i = 0; i < n; ++i) {
        double* h = hit_out + 13 * i;
        std::memset(h, 0, 13 * sizeof(double));
        if (mode == 2) {
            h[0] = s.occluded(v3(o + 3 * i), v3(d + 3 * i)) ? 1.0 : 0.0;
            continue;
        }
        const auto hit = mode == 1 ? s.intersect_brute_force(v3(o + 3 * i), v3(d + 3 * i), t_min[i])
                                   : s.intersect(v3(o + 3 * i), v3(d + 3 * i), t_min[i]);
        if (!hit) {
            h[0] = std::numeric_limits<double>::infinity();
            h[12] = 4294967295.0;
            continue;
        }
        put_hit(h, *hit);
    }
    return 0;
}

int ref_launch_rect(const void* sp, const double* k_inc, double padding, double* out11) {
    try {
        const LaunchRect r = launch_rect(*static_cast<const Scene*>(sp), v3(k_inc), padding);
        put(out11, r.center);
        put(out11 + 3, r.u_axis);
        put(out11 + 6, r.v_axis);
        out11[9] = r.half_u;
        out11[10] = r.half_v;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_build_strata(const double* rect11, double spw, double lambda_ref, int32_t* nu_nv,
                     double* cell_area) {
    try {
        LaunchRect r;
        r.center = v3(rect11);
        r.u_axis = v3(rect11 + 3);
        r.v_axis = v3(rect11 + 6);
        r.half_u = rect11[9];
        r.half_v = rect11[10];
        const StrataGrid g = build_strata(r, spw, lambda_ref);
        nu_nv[0] = g.nu;
        nu_nv[1] = g.nv;
        *cell_area = g.cell_area;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_sample_stratum(const double* rect11, int32_t nu, int32_t nv, uint32_t cell,
                       uint32_t sample, uint64_t seed, int jitter, double* point3) {
    StrataGrid g;
    g.rect.center = v3(rect11);
    g.rect.u_axis = v3(rect11 + 3);
    g.rect.v_axis = v3(rect11 + 6);
    g.rect.half_u = rect11[9];
    g.rect.half_v = rect11[10];
    g.nu = nu;
    g.nv = nv;
    g.cell_area = g.rect.area() / (static_cast<double>(nu) * nv);
    g.pdf_per_cell = 1.0 / g.cell_area;
    put(point3, sample_stratum(g, cell, sample, seed, jitter != 0).point);
    return 0;
}

// ---- the hot path: estimate (solver_mc.cpp:76-229) ---------------------------
// values: [4][nf] complex; stats: mcsbr_stats (wall_ms = reference wall time).
int ref_estimate(const void* sp, const mcsbr_excitation* exc, const double* freqs, uint32_t nf,
                 const mcsbr_mc_config* cfg, int workers, double* values, mcsbr_stats* st,
                 mcsbr_contribution* contribs, uint64_t capacity, uint64_t* n_contribs) {
    try {
        std::vector<Contribution> collected;
        const McResult r = estimate(*static_cast<const Scene*>(sp), to_exc(*exc),
                                    std::vector<double>(freqs, freqs + nf), to_mc(*cfg), workers,
                                    contribs ? &collected : nullptr);
        for (int ch = 0; ch < kPolChannelCount; ++ch)
            for (uint32_t i = 0; i < nf; ++i) putc(values + 2 * (ch * nf + i), r.sweep.values[ch][i]);
        if (st) {
            std::memset(st, 0, sizeof(*st));
            st->rays_launched = r.stats.rays_launched;
            st->segments_traced = r.stats.segments_traced;
            st->contributions = r.stats.contributions;
            st->grazing_kills = r.stats.grazing_kills;
            st->cap_kills = r.stats.cap_kills;
            st->peak_live_state_bytes = r.stats.peak_live_state_bytes;
            st->state_bytes_per_ray = r.stats.state_bytes_per_ray;
            st->block_size = r.stats.block_size;
            st->n_rounds = static_cast<uint32_t>(r.stats.rays_per_bounce.size());
            for (size_t i = 0; i < r.stats.rays_per_bounce.size() && i < MCSBR_MAX_BOUNCE_LIMIT; ++i)
                st->rays_per_bounce[i] = r.stats.rays_per_bounce[i];
            for (size_t i = 0; i < r.stats.roulette_candidates.size() && i < MCSBR_MAX_BOUNCE_LIMIT; ++i)
                st->roulette_candidates[i] = r.stats.roulette_candidates[i];
            for (size_t i = 0; i < r.stats.roulette_survivors.size() && i < MCSBR_MAX_BOUNCE_LIMIT; ++i)
                st->roulette_survivors[i] = r.stats.roulette_survivors[i];
            st->wall_ms = r.stats.wall_ms;
        }
        if (contribs) {
            const uint64_t m = collected.size() < capacity ? collected.size() : capacity;
            std::memcpy(static_cast<void*>(contribs), collected.data(), m * sizeof(Contribution));
            if (n_contribs) *n_contribs = collected.size();
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- the deterministic solver (solver_det.cpp:30-174) ------------------------
int ref_solve(const void* sp, const mcsbr_excitation* exc, const double* freqs, uint32_t nf,
              const mcsbr_det_config* cfg, int workers, double* values, mcsbr_stats* st,
              mcsbr_contribution* contribs, uint64_t capacity, uint64_t* n_contribs) {
    try {
        DetConfig d;
        d.rays_per_wavelength = cfg->rays_per_wavelength;
        d.max_bounce = cfg->max_bounce;
        d.amplitude_cutoff = cfg->amplitude_cutoff;
        d.force_stack_accounting = cfg->force_stack_accounting != 0;
        d.launch_padding = cfg->launch_padding;
        d.reference_wavelength = cfg->reference_wavelength;
        d.block_size = cfg->block_size;
        std::vector<Contribution> collected;
        const DetResult r = solve(*static_cast<const Scene*>(sp), to_exc(*exc),
                                  std::vector<double>(freqs, freqs + nf), d, workers,
                                  contribs ? &collected : nullptr);
        for (int ch = 0; ch < kPolChannelCount; ++ch)
            for (uint32_t i = 0; i < nf; ++i) putc(values + 2 * (ch * nf + i), r.sweep.values[ch][i]);
        if (st) {
            std::memset(st, 0, sizeof(*st));
            st->rays_launched = r.stats.rays_launched;
            st->segments_traced = r.stats.segments_traced;
            st->contributions = r.stats.contributions;
            st->grazing_kills = r.stats.grazing_kills;
            st->cap_kills = r.stats.cap_kills;
            st->peak_live_state_bytes = r.stats.peak_live_state_bytes;
            st->forced_stack_bytes = r.stats.forced_stack_bytes;
            st->state_bytes_per_ray = r.stats.state_bytes_per_ray;
            st->block_size = r.stats.block_size;
            st->n_rounds = static_cast<uint32_t>(r.stats.rays_per_bounce.size());
            for (size_t i = 0; i < r.stats.rays_per_bounce.size() && i < MCSBR_MAX_BOUNCE_LIMIT; ++i)
                st->rays_per_bounce[i] = r.stats.rays_per_bounce[i];
            st->wall_ms = r.stats.wall_ms;
        }
        if (contribs) {
            const uint64_t m = collected.size() < capacity ? collected.size() : capacity;
            std::memcpy(static_cast<void*>(contribs), collected.data(), m * sizeof(Contribution));
            if (n_contribs) *n_contribs = collected.size();
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- runner artifacts and config (runner.cpp:48-118, config.cpp) -------------
static int put_text(const std::string& t, char* out, uint64_t cap, uint64_t* len) {
    *len = t.size();
    if (out && cap > t.size()) std::memcpy(out, t.c_str(), t.size() + 1);
    return 0;
}

// sweep_csv of a [4][nf] complex value block
int ref_sweep_csv(const double* values, const double* freqs, uint32_t nf, uint64_t seed, const char* solver,
                  const char* config_hash, char* out, uint64_t cap, uint64_t* len) {
    try {
        SweepResult s;
        s.frequencies.assign(freqs, freqs + nf);
        for (int ch = 0; ch < kPolChannelCount; ++ch) {
            s.values[ch].resize(nf);
            for (uint32_t i = 0; i < nf; ++i)
                s.values[ch][i] = complexd(values[2 * (ch * nf + i)], values[2 * (ch * nf + i) + 1]);
        }
        s.seed = seed;
        s.solver = solver;
        return put_text(sweep_csv(s, config_hash), out, cap, len);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_stats_json(const mcsbr_stats* st, const char* solver, char* out, uint64_t cap, uint64_t* len) {
    try {
        RunStats r;
        r.rays_launched = st->rays_launched;
        r.segments_traced = st->segments_traced;
        r.contributions = st->contributions;
        r.grazing_kills = st->grazing_kills;
        r.cap_kills = st->cap_kills;
        r.peak_live_state_bytes = st->peak_live_state_bytes;
        r.forced_stack_bytes = st->forced_stack_bytes;
        r.state_bytes_per_ray = st->state_bytes_per_ray;
        r.block_size = st->block_size;
        r.wall_ms = st->wall_ms;
        r.rays_per_bounce.assign(st->rays_per_bounce, st->rays_per_bounce + st->n_rounds);
        r.roulette_candidates.assign(st->roulette_candidates, st->roulette_candidates + st->n_rounds);
        r.roulette_survivors.assign(st->roulette_survivors, st->roulette_survivors + st->n_rounds);
        return put_text(stats_json(r, solver), out, cap, len);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// parse_config: the config hash, or the ConfigError message (return 1)
int ref_parse_config(const char* json_text, char* out, uint64_t cap, uint64_t* len) {
    try {
        const ExperimentConfig c = parse_config(json_text);
        return put_text(c.config_hash, out, cap, len);
    } catch (const ConfigError& e) {
        put_text(e.what(), out, cap, len);
        return 1;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// run_command end to end on the CPU reference (all artifacts under out_dir)
int ref_run_command(const char* command, const char* json_text, const char* out_dir, int workers,
                    int has_seed, uint64_t seed) {
    try {
        const ExperimentConfig c = parse_config(json_text);
        RunOptions o;
        o.workers = workers;
        o.out_dir = out_dir;
        if (has_seed) o.seed_override = seed;
        return run_command(command, c, o);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- radar products (signal_processing.cpp) -----------------------------------
// values: one channel, nf complex; outputs as mcsbr_gpu_range_profile
int ref_range_profile(const double* values, const double* freqs, uint32_t nf, int window,
                      int zero_pad, double* range_m, double* mag_db, double* bin_spacing) {
    try {
        SweepResult s;
        s.frequencies.assign(freqs, freqs + nf);
        for (int ch = 0; ch < kPolChannelCount; ++ch) s.values[ch].assign(nf, complexd{});
        for (uint32_t k = 0; k < nf; ++k) s.values[kVV][k] = complexd(values[2 * k], values[2 * k + 1]);
        const RangeProfile p =
            range_profile(s, kVV, window == MCSBR_WINDOW_HANN ? Window::kHann : Window::kNone, zero_pad);
        for (size_t i = 0; i < p.range_m.size(); ++i) {
            range_m[i] = p.range_m[i];
            mag_db[i] = p.mag_db[i];
        }
        *bin_spacing = p.bin_spacing;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// values: one channel, [na][nf] complex
int ref_isar(const double* values, const double* freqs, uint32_t nf, const double* angles, uint32_t na,
             int window, int zero_pad, double floor_db, double* down, double* cross, double* mag_db,
             double* peak_db) {
    try {
        std::vector<SweepResult> sweeps(na);
        for (uint32_t a = 0; a < na; ++a) {
            sweeps[a].frequencies.assign(freqs, freqs + nf);
            for (int ch = 0; ch < kPolChannelCount; ++ch) sweeps[a].values[ch].assign(nf, complexd{});
            for (uint32_t k = 0; k < nf; ++k)
                sweeps[a].values[kVV][k] = complexd(values[2 * (a * nf + k)], values[2 * (a * nf + k) + 1]);
        }
        const IsarImage img = isar(sweeps, std::vector<double>(angles, angles + na), kVV,
                                   window == MCSBR_WINDOW_HANN ? Window::kHann : Window::kNone, zero_pad,
                                   floor_db);
        for (size_t i = 0; i < img.down_range_m.size(); ++i) down[i] = img.down_range_m[i];
        for (size_t i = 0; i < img.cross_range_m.size(); ++i) cross[i] = img.cross_range_m[i];
        for (size_t i = 0; i < img.mag_db.size(); ++i) mag_db[i] = img.mag_db[i];
        *peak_db = img.peak_db;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- analytic oracles (oracles.cpp) -------------------------------------------
int ref_slab_reflection(const double* index, const double* thickness, int n_layers,
                        double frequency, int pec_backed, double* out2) {
    try {
        oracles::LayerStack s;
        for (int i = 0; i < n_layers; ++i) s.layers.push_back({index[i], thickness[i]});
        putc(out2, oracles::slab_reflection(s, frequency, pec_backed != 0));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
double ref_plate_rcs(double a, double b, double lambda) { return oracles::plate_rcs(a, b, lambda); }
double ref_sphere_go_rcs(double r) { return oracles::sphere_go_rcs(r); }

}  // extern "C"
