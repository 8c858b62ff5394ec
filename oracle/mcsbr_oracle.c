/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference MC-SBR estimator
 * (see mcsbr_oracle.h).  Compiled with -ffp-contract=off and no -march so
 * every + - * / sqrt is one IEEE double operation in the same order as the
 * reference's C++ (the proj/src C++ sources built without FMA); that is what makes the
 * results bit-identical.  Complex arithmetic restates the C99/libstdc++
 * semantics the reference relies on:
 *   complex*complex  -> (ac - bd, ad + bc)          (GCC inline expansion)
 *   complex*double   -> (re*d, im*d)                (std::complex operator*=)
 *   complex/complex  -> libgcc __divdc3 (Smith's method with scaling), cdiv()
 *   std::abs(complex)-> cabs = hypot(re, im)        (libstdc++ __complex_abs)
 *   std::norm        -> re*re + im*im               (libstdc++ _Norm_helper)
 *   std::polar(1,t)  -> (cos t, sin t)
 * Parity status: PINNED against oracle/_ref (tests/test_oracle_pins.py).
 */
#include "mcsbr_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];
static void set_err(const char* m) { snprintf(g_err, sizeof g_err, "%s", m); }
const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* value types (proj/include/mcsbr/em_math.hpp:26-93)                         */

typedef struct { double x, y, z; } v3;
typedef struct { double re, im; } cx;
typedef struct { cx x, y, z; } cv3;

static const double kC = 299792458.0;                  /* em_math.hpp:20 */
static const double kPI = 3.14159265358979323846;      /* em_math.hpp:21 */

static v3 V(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static v3 vadd(v3 a, v3 b) { return V(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 vsub(v3 a, v3 b) { return V(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 vneg(v3 a) { return V(-a.x, -a.y, -a.z); }
static v3 vmul(v3 a, double s) { return V(a.x * s, a.y * s, a.z * s); }
static v3 vdiv(v3 a, double s) { return V(a.x / s, a.y / s, a.z / s); }
static double vdot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 vcross(v3 a, v3 b) {
    return V(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static double vnorm(v3 v) { return sqrt(vdot(v, v)); }
static v3 vnormalized(v3 v) {
    const double n = vnorm(v);
    return V(v.x / n, v.y / n, v.z / n);
}
static v3 vload(const double* p) { return V(p[0], p[1], p[2]); }
static void vstore(double* p, v3 v) { p[0] = v.x; p[1] = v.y; p[2] = v.z; }
/* std::min / std::max argument order (a, b): min -> (b < a) ? b : a */
static double dmin(double a, double b) { return (b < a) ? b : a; }
static double dmax(double a, double b) { return (a < b) ? b : a; }

static cx C(double re, double im) { cx r = {re, im}; return r; }
static cx cadd(cx a, cx b) { return C(a.re + b.re, a.im + b.im); }
static cx csub(cx a, cx b) { return C(a.re - b.re, a.im - b.im); }
static cx cmul(cx a, cx b) { return C(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re); }
static cx cscale(cx a, double s) { return C(a.re * s, a.im * s); }
static double cabs_(cx a) { return hypot(a.re, a.im); }
static double cnorm2(cx a) { return a.re * a.re + a.im * a.im; }

/* libgcc __divdc3 (Smith's method with the GCC >= 12 range scaling). */
static cx cdiv(cx num, cx den) {
    double a = num.re, b = num.im, c = den.re, d = den.im;
    const double RBIG = DBL_MAX / 2, RMIN = DBL_MIN, RMIN2 = DBL_EPSILON;
    const double RMINSCAL = 1 / DBL_EPSILON, RMAX2 = RBIG * RMIN2;
    double ratio, denom, x, y;
    if (fabs(c) < fabs(d)) {
        if (fabs(d) >= RBIG) { a = a / 2; b = b / 2; c = c / 2; d = d / 2; }
        if (fabs(d) < RMIN2) {
            a = a * RMINSCAL; b = b * RMINSCAL; c = c * RMINSCAL; d = d * RMINSCAL;
        } else if (((fabs(a) < RMIN) && (fabs(b) < RMAX2) && (fabs(d) < RMAX2)) ||
                   ((fabs(b) < RMIN) && (fabs(a) < RMAX2) && (fabs(d) < RMAX2))) {
            a = a * RMINSCAL; b = b * RMINSCAL; c = c * RMINSCAL; d = d * RMINSCAL;
        }
        ratio = c / d;
        denom = (c * ratio) + d;
        if (fabs(ratio) > RMIN) {
            x = ((a * ratio) + b) / denom;
            y = ((b * ratio) - a) / denom;
        } else {
            x = ((c * (a / d)) + b) / denom;
            y = ((c * (b / d)) - a) / denom;
        }
    } else {
        if (fabs(c) >= RBIG) { a = a / 2; b = b / 2; c = c / 2; d = d / 2; }
        if (fabs(c) < RMIN2) {
            a = a * RMINSCAL; b = b * RMINSCAL; c = c * RMINSCAL; d = d * RMINSCAL;
        } else if (((fabs(a) < RMIN) && (fabs(b) < RMAX2) && (fabs(c) < RMAX2)) ||
                   ((fabs(b) < RMIN) && (fabs(a) < RMAX2) && (fabs(c) < RMAX2))) {
            a = a * RMINSCAL; b = b * RMINSCAL; c = c * RMINSCAL; d = d * RMINSCAL;
        }
        ratio = d / c;
        denom = (d * ratio) + c;
        if (fabs(ratio) > RMIN) {
            x = ((b * ratio) + a) / denom;
            y = (b - (a * ratio)) / denom;
        } else {
            x = (a + (d * (b / c))) / denom;
            y = (b - (d * (a / c))) / denom;
        }
    }
    return C(x, y);
}
void orc_cdiv(const double* a2, const double* b2, double* out2) {
    cx r = cdiv(C(a2[0], a2[1]), C(b2[0], b2[1]));
    out2[0] = r.re;
    out2[1] = r.im;
}

static cv3 CV(cx x, cx y, cx z) { cv3 r = {x, y, z}; return r; }
static cv3 cvreal(v3 v) { return CV(C(v.x, 0.0), C(v.y, 0.0), C(v.z, 0.0)); }
static cv3 cvzero(void) { return CV(C(0, 0), C(0, 0), C(0, 0)); }
static cv3 cvadd(cv3 a, cv3 b) { return CV(cadd(a.x, b.x), cadd(a.y, b.y), cadd(a.z, b.z)); }
static cv3 cvmulc(cv3 a, cx s) { return CV(cmul(a.x, s), cmul(a.y, s), cmul(a.z, s)); }
static cv3 cvmuld(cv3 a, double s) { return CV(cscale(a.x, s), cscale(a.y, s), cscale(a.z, s)); }
/* dot(ComplexVec3, Vec3), em_math.hpp:78-80 (no conjugation) */
static cx cvdot(cv3 a, v3 b) {
    return cadd(cadd(cscale(a.x, b.x), cscale(a.y, b.y)), cscale(a.z, b.z));
}
/* cross(Vec3, ComplexVec3), em_math.hpp:83-85 */
static cv3 cross_vc(v3 a, cv3 b) {
    return CV(csub(cscale(b.z, a.y), cscale(b.y, a.z)), csub(cscale(b.x, a.z), cscale(b.z, a.x)),
              csub(cscale(b.y, a.x), cscale(b.x, a.y)));
}
/* cross(ComplexVec3, Vec3), em_math.hpp:86-88 */
static cv3 cross_cv(cv3 a, v3 b) {
    return CV(csub(cscale(a.y, b.z), cscale(a.z, b.y)), csub(cscale(a.z, b.x), cscale(a.x, b.z)),
              csub(cscale(a.x, b.y), cscale(a.y, b.x)));
}
static double cvnorm(cv3 v) { return sqrt(cnorm2(v.x) + cnorm2(v.y) + cnorm2(v.z)); }
static cv3 cvload(const double* p) { return CV(C(p[0], p[1]), C(p[2], p[3]), C(p[4], p[5])); }
static void cvstore(double* p, cv3 v) {
    p[0] = v.x.re; p[1] = v.x.im; p[2] = v.y.re; p[3] = v.y.im; p[4] = v.z.re; p[5] = v.z.im;
}

/* ------------------------------------------------------------------------ */
/* counter RNG (proj/include/mcsbr/rng.hpp:19-44)                            */

static uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
uint64_t orc_counter_hash(uint64_t seed, uint64_t stratum, uint64_t sample, uint64_t bounce,
                          uint64_t purpose) {
    uint64_t h = mix64(seed ^ 0x2545f4914f6cdd1dull);
    h = mix64(h ^ stratum);
    h = mix64(h ^ (sample + 0x632be59bd9b4e019ull));
    h = mix64(h ^ (bounce + 0x9e3779b97f4a7c15ull));
    h = mix64(h ^ purpose);
    return h;
}
double orc_counter_uniform(uint64_t seed, uint64_t stratum, uint64_t sample, uint64_t bounce,
                           uint64_t purpose) {
    return (double)(orc_counter_hash(seed, stratum, sample, bounce, purpose) >> 11) * 0x1.0p-53;
}
enum { kLaunchU = 0x101, kLaunchV = 0x102, kBranch = 0x201, kRoulette = 0x202 };

/* ------------------------------------------------------------------------ */
/* interface physics (proj/src/em_math.cpp)                                   */

typedef struct {
    cx r_s, r_p, t_s, t_p, cos_t;
    int tir;
} coeffs_t;

typedef struct {
    v3 s_hat, p_in, p_out_r, p_out_t, dir_r, dir_t;
} basis_t;

static int g_fault; /* set where the reference throws (DomainError / DegenerateGeometryError) */

static coeffs_t coeffs_pec(void) { /* em_math.hpp:127-133 */
    coeffs_t c;
    memset(&c, 0, sizeof c);
    c.r_s = C(-1.0, 0.0);
    c.r_p = C(1.0, 0.0);
    return c;
}

/* em_math.cpp:5-30 */
static coeffs_t fresnel(double n1, double n2, double cos_i) {
    coeffs_t c;
    memset(&c, 0, sizeof c);
    if (!(isfinite(n1) && isfinite(n2)) || n1 <= 0.0 || n2 <= 0.0) {
        set_err("fresnel: refractive indices must be finite and positive");
        g_fault = 1;
        return c;
    }
    if (!(cos_i > 0.0 && cos_i <= 1.0)) {
        set_err("fresnel: cos_theta_i must lie in (0, 1]");
        g_fault = 1;
        return c;
    }
    const double sin2_i = dmax(0.0, 1.0 - cos_i * cos_i);
    const double s2 = (n1 / n2) * (n1 / n2) * sin2_i;
    cx cos_t;
    if (s2 > 1.0) {
        c.tir = 1;
        cos_t = C(0.0, -sqrt(s2 - 1.0));
    } else {
        cos_t = C(sqrt(1.0 - s2), 0.0);
    }
    c.cos_t = cos_t;
    const cx ci = C(cos_i, 0.0);
    const cx d_s = cadd(cscale(ci, n1), cscale(cos_t, n2));
    const cx d_p = cadd(cscale(ci, n2), cscale(cos_t, n1));
    c.r_s = cdiv(csub(cscale(ci, n1), cscale(cos_t, n2)), d_s);
    c.t_s = cdiv(cscale(ci, 2.0 * n1), d_s);
    c.r_p = cdiv(csub(cscale(ci, n2), cscale(cos_t, n1)), d_p);
    c.t_p = cdiv(cscale(ci, 2.0 * n1), d_p);
    return c;
}

/* em_math.cpp:32-37 */
static v3 reflect_dir(v3 dir, v3 normal) {
    const double dn = vdot(dir, normal);
    if (fabs(dn) < 1e-9) {
        set_err("reflect_dir: grazing incidence");
        g_fault = 1;
    }
    return vsub(dir, vmul(normal, 2.0 * dn));
}

/* em_math.cpp:39-49; returns 0 past the critical angle */
static int refract_dir(v3 dir, v3 normal, double n1, double n2, v3* out) {
    const double dn = vdot(dir, normal);
    if (fabs(dn) < 1e-9) {
        set_err("refract_dir: grazing incidence");
        g_fault = 1;
    }
    const double cos_i = -dn;
    const double eta = n1 / n2;
    const double sin2_t = eta * eta * dmax(0.0, 1.0 - cos_i * cos_i);
    if (sin2_t > 1.0) return 0;
    const double cos_t = sqrt(1.0 - sin2_t);
    *out = vnormalized(vadd(vmul(dir, eta), vmul(normal, eta * cos_i - cos_t)));
    return 1;
}

/* em_math.cpp:51-81 */
static basis_t sp_basis(v3 dir_in, v3 normal, double n1, double n2) {
    basis_t b;
    const v3 c = vcross(dir_in, normal);
    const double cn = vnorm(c);
    if (cn < 1e-6) {
        v3 axis = V(1.0, 0.0, 0.0);
        v3 s = vsub(axis, vmul(dir_in, vdot(axis, dir_in)));
        if (vnorm(s) < 1e-6) {
            axis = V(0.0, 1.0, 0.0);
            s = vsub(axis, vmul(dir_in, vdot(axis, dir_in)));
        }
        b.s_hat = vnormalized(s);
    } else {
        b.s_hat = vdiv(c, cn);
    }
    b.dir_r = reflect_dir(dir_in, normal);
    b.p_in = vcross(dir_in, b.s_hat);
    b.p_out_r = vcross(b.dir_r, b.s_hat);
    v3 t;
    if (refract_dir(dir_in, normal, n1, n2, &t)) {
        b.dir_t = t;
        b.p_out_t = vcross(b.dir_t, b.s_hat);
    } else {
        b.dir_t = dir_in;
        b.p_out_t = b.p_in;
    }
    return b;
}

/* em_math.cpp:83-95; branch 0 = reflect, 1 = transmit */
static cv3 interface_transform(cv3 e, int branch, const coeffs_t* co, const basis_t* b) {
    const v3 dir_in = vcross(b->s_hat, b->p_in);
    if (cabs_(cvdot(e, dir_in)) > 1e-9 * (1.0 + cvnorm(e))) {
        set_err("interface_transform: field is not transverse to dir_in");
        g_fault = 1;
    }
    const cx es = cvdot(e, b->s_hat);
    const cx ep = cvdot(e, b->p_in);
    if (branch == 0)
        return cvadd(cvmulc(cvreal(b->s_hat), cmul(es, co->r_s)),
                     cvmulc(cvreal(b->p_out_r), cmul(ep, co->r_p)));
    return cvadd(cvmulc(cvreal(b->s_hat), cmul(es, co->t_s)),
                 cvmulc(cvreal(b->p_out_t), cmul(ep, co->t_p)));
}

/* ------------------------------------------------------------------------ */
/* path engine (proj/src/path_engine.cpp, proj/include/mcsbr/path_engine.hpp) */

typedef struct {
    v3 origin, dir;
    cv3 e[2];
    double phi, prob, weight, medium_n;
    int bounce;
    uint32_t stratum, sample;
} path_t;

typedef struct {
    double t;
    v3 point, normal;
    uint32_t id;
    double n_incident, n_transmit;
    int far_side_pec, exterior_facing, near_is_ambient;
} hit_t;

typedef struct {
    int count, grazing;
    coeffs_t co;
    basis_t b;
    v3 new_dir[2];
    cv3 new_e[2][2];
    double new_n[2];
} branchset_t;

/* path_engine.cpp:23-54 */
static void branch_outcomes(const path_t* s, const hit_t* h, branchset_t* set) {
    memset(set, 0, sizeof *set);
    const double cos_i = -vdot(s->dir, h->normal);
    if (cos_i < 1e-6) {
        set->grazing = 1;
        return;
    }
    const int pec = h->far_side_pec;
    const double n1 = s->medium_n;
    const double n2 = pec ? n1 : h->n_transmit;
    set->co = pec ? coeffs_pec() : fresnel(n1, n2, cos_i);
    set->b = sp_basis(s->dir, h->normal, n1, n2);
    set->new_dir[0] = set->b.dir_r;
    set->new_e[0][0] = interface_transform(s->e[0], 0, &set->co, &set->b);
    set->new_e[0][1] = interface_transform(s->e[1], 0, &set->co, &set->b);
    set->new_n[0] = n1;
    set->count = 1;
    if (!pec && !set->co.tir) {
        set->new_dir[1] = set->b.dir_t;
        set->new_e[1][0] = interface_transform(s->e[0], 1, &set->co, &set->b);
        set->new_e[1][1] = interface_transform(s->e[1], 1, &set->co, &set->b);
        set->new_n[1] = n2;
        set->count = 2;
    }
}

/* farfield.cpp:11-45 (hot overload); case 0 Pec, 1 Entering, 2 Exiting */
static void meca(const hit_t* h, cv3 e, v3 dir_in, int sc, const coeffs_t* co, const basis_t* b,
                 double medium_n, cv3* j, cv3* m) {
    *j = cvzero();
    *m = cvzero();
    if (sc == 0) {
        const cv3 h_i = cvmuld(cross_vc(dir_in, e), medium_n);
        *j = cvmuld(cross_vc(h->normal, h_i), 2.0);
    } else if (sc == 1) {
        const cv3 e_r = interface_transform(e, 0, co, b);
        const cv3 h_sum = cvmuld(cvadd(cross_vc(dir_in, e), cross_vc(b->dir_r, e_r)), medium_n);
        *j = cross_vc(h->normal, h_sum);
        *m = cross_cv(cvadd(e, e_r), h->normal);
    } else {
        if (co->tir) return;
        const cv3 e_t = interface_transform(e, 1, co, b);
        const v3 n_out = vneg(h->normal);
        const cv3 h_t = cvmuld(cross_vc(b->dir_t, e_t), h->n_transmit);
        *j = cross_vc(n_out, h_t);
        *m = cross_cv(e_t, n_out);
    }
}

/* ------------------------------------------------------------------------ */
/* scene + exact closest-hit (proj/src/geometry.cpp)                          */

typedef struct {
    double lo[3], hi[3];
    uint32_t left, count, right;
} onode_t;

struct orc_scene {
    uint32_t nv, nt, nm;
    v3* vert;
    mcsbr_triangle* tri;
    mcsbr_material* mat;
    double* mat_index; /* Material::index() */
    v3 bcenter;
    double bradius, diameter;
    onode_t* nodes;
    uint32_t n_nodes;
    uint32_t* order;
};

/* geometry.cpp:20-39, Moller-Trumbore in fp64 with the reference's order */
static int ray_triangle(v3 o, v3 d, v3 a, v3 b, v3 c, double t_min, double t_max, double* t_out) {
    const v3 e1 = vsub(b, a);
    const v3 e2 = vsub(c, a);
    const v3 p = vcross(d, e2);
    const double det = vdot(e1, p);
    if (fabs(det) < 1e-14) return 0;
    const double inv_det = 1.0 / det;
    const v3 s = vsub(o, a);
    const double u = vdot(s, p) * inv_det;
    if (u < 0.0 || u > 1.0) return 0;
    const v3 q = vcross(s, e1);
    const double v = vdot(d, q) * inv_det;
    if (v < 0.0 || u + v > 1.0) return 0;
    const double t = vdot(e2, q) * inv_det;
    if (t <= t_min || t >= t_max) return 0;
    *t_out = t;
    return 1;
}

/* Our own BVH (median split on the widest centroid axis, leaves <= 4) with
 * boxes padded by 1e-9 of the scene diameter: the slab test is only a cull,
 * the exact fp64 triangle test decides, so results equal brute force
 * (closest t, ties to the smallest id: geometry.cpp:197). */
static int cmp_axis;
static const v3* cmp_cent;
static int cmp_fn(const void* a, const void* b) {
    const uint32_t ia = *(const uint32_t*)a, ib = *(const uint32_t*)b;
    const double ka = cmp_axis == 0 ? cmp_cent[ia].x : cmp_axis == 1 ? cmp_cent[ia].y : cmp_cent[ia].z;
    const double kb = cmp_axis == 0 ? cmp_cent[ib].x : cmp_axis == 1 ? cmp_cent[ib].y : cmp_cent[ib].z;
    if (ka < kb) return -1;
    if (ka > kb) return 1;
    return (ia < ib) ? -1 : (ia > ib);
}

static void build_bvh(orc_scene* s) {
    const uint32_t n = s->nt;
    s->order = (uint32_t*)malloc(sizeof(uint32_t) * n);
    v3* cent = (v3*)malloc(sizeof(v3) * n);
    double* blo = (double*)malloc(sizeof(double) * 3 * n);
    double* bhi = (double*)malloc(sizeof(double) * 3 * n);
    for (uint32_t i = 0; i < n; ++i) {
        const v3 a = s->vert[s->tri[i].v0], b = s->vert[s->tri[i].v1], c = s->vert[s->tri[i].v2];
        s->order[i] = i;
        cent[i] = vdiv(vadd(vadd(a, b), c), 3.0);
        blo[3 * i + 0] = fmin(a.x, fmin(b.x, c.x));
        blo[3 * i + 1] = fmin(a.y, fmin(b.y, c.y));
        blo[3 * i + 2] = fmin(a.z, fmin(b.z, c.z));
        bhi[3 * i + 0] = fmax(a.x, fmax(b.x, c.x));
        bhi[3 * i + 1] = fmax(a.y, fmax(b.y, c.y));
        bhi[3 * i + 2] = fmax(a.z, fmax(b.z, c.z));
    }
    s->nodes = (onode_t*)calloc(2 * (size_t)n + 1, sizeof(onode_t));
    s->n_nodes = 1;
    const double pad = 1e-9 * s->diameter + 1e-300;
    typedef struct { uint32_t node, begin, end; } task_t;
    task_t* stack = (task_t*)malloc(sizeof(task_t) * (2 * (size_t)n + 2));
    int sp = 0;
    stack[sp++] = (task_t){0, 0, n};
    while (sp > 0) {
        const task_t t = stack[--sp];
        onode_t* nd = &s->nodes[t.node];
        double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
        double clo[3] = {1e300, 1e300, 1e300}, chi[3] = {-1e300, -1e300, -1e300};
        for (uint32_t i = t.begin; i < t.end; ++i) {
            const uint32_t id = s->order[i];
            const double c3[3] = {cent[id].x, cent[id].y, cent[id].z};
            for (int k = 0; k < 3; ++k) {
                lo[k] = fmin(lo[k], blo[3 * id + k]);
                hi[k] = fmax(hi[k], bhi[3 * id + k]);
                clo[k] = fmin(clo[k], c3[k]);
                chi[k] = fmax(chi[k], c3[k]);
            }
        }
        for (int k = 0; k < 3; ++k) {
            nd->lo[k] = lo[k] - pad;
            nd->hi[k] = hi[k] + pad;
        }
        const uint32_t count = t.end - t.begin;
        if (count <= 4) {
            nd->left = t.begin;
            nd->count = count;
            continue;
        }
        int axis = 0;
        if (chi[1] - clo[1] > chi[axis] - clo[axis]) axis = 1;
        if (chi[2] - clo[2] > chi[axis] - clo[axis]) axis = 2;
        cmp_axis = axis;
        cmp_cent = cent;
        qsort(s->order + t.begin, count, sizeof(uint32_t), cmp_fn);
        const uint32_t cut = t.begin + count / 2;
        const uint32_t left = s->n_nodes;
        s->n_nodes += 2;
        nd->left = left;
        nd->right = left + 1;
        nd->count = 0;
        stack[sp++] = (task_t){left, t.begin, cut};
        stack[sp++] = (task_t){left + 1, cut, t.end};
    }
    free(stack);
    free(cent);
    free(blo);
    free(bhi);
}

static int slab(const onode_t* nd, v3 o, v3 inv, double t_max) {
    double t0 = 0.0, t1 = t_max;
    const double oo[3] = {o.x, o.y, o.z}, ii[3] = {inv.x, inv.y, inv.z};
    for (int k = 0; k < 3; ++k) {
        double nr = (nd->lo[k] - oo[k]) * ii[k];
        double fr = (nd->hi[k] - oo[k]) * ii[k];
        if (nr > fr) { const double tmp = nr; nr = fr; fr = tmp; }
        if (isnan(nr)) nr = -INFINITY; /* 0 * inf when the ray lies in a slab plane */
        if (isnan(fr)) fr = INFINITY;
        t0 = fmax(t0, nr);
        t1 = fmin(t1, fr);
        if (t0 > t1) return 0;
    }
    return 1;
}

/* geometry.cpp:164-175 */
static void fill_hit(const orc_scene* s, hit_t* h, v3 dir) {
    const mcsbr_triangle* tri = &s->tri[h->id];
    const v3 nrm = vload(tri->normal);
    const int front = vdot(dir, nrm) < 0.0;
    h->normal = front ? nrm : vneg(nrm);
    const uint16_t near_id = front ? tri->front_material : tri->back_material;
    const uint16_t far_id = front ? tri->back_material : tri->front_material;
    const int near_pec = s->mat[near_id].is_pec != 0, far_pec = s->mat[far_id].is_pec != 0;
    h->n_incident = near_pec ? s->mat_index[0] : s->mat_index[near_id];
    h->far_side_pec = far_pec || near_pec;
    h->n_transmit = far_pec ? 0.0 : s->mat_index[far_id];
    h->exterior_facing = tri->exterior_facing != 0;
    h->near_is_ambient = near_id == 0;
}

static int closest(const orc_scene* s, v3 o, v3 d, double t_min, int any, hit_t* out) {
    const v3 inv = V(1.0 / d.x, 1.0 / d.y, 1.0 / d.z);
    double best_t = INFINITY;
    uint32_t best_id = 0xFFFFFFFFu;
    uint32_t stack[256];
    int sp = 0;
    stack[sp++] = 0;
    while (sp > 0) {
        const onode_t* nd = &s->nodes[stack[--sp]];
        if (!slab(nd, o, inv, best_t == INFINITY ? 1e300 : best_t)) continue;
        if (nd->count > 0) {
            for (uint32_t i = nd->left; i < nd->left + nd->count; ++i) {
                const uint32_t id = s->order[i];
                const mcsbr_triangle* t = &s->tri[id];
                double th;
                if (ray_triangle(o, d, s->vert[t->v0], s->vert[t->v1], s->vert[t->v2], t_min, 1e300,
                                 &th)) {
                    if (th < best_t || (th == best_t && id < best_id)) {
                        best_t = th;
                        best_id = id;
                        if (any) sp = 0;
                    }
                }
            }
        } else {
            stack[sp++] = nd->left;
            stack[sp++] = nd->right;
        }
    }
    if (best_id == 0xFFFFFFFFu) return 0;
    out->t = best_t;
    out->point = vadd(o, vmul(d, best_t));
    out->id = best_id;
    fill_hit(s, out, d);
    return 1;
}

static int brute(const orc_scene* s, v3 o, v3 d, double t_min, hit_t* out) {
    double best_t = INFINITY;
    uint32_t best_id = 0xFFFFFFFFu;
    for (uint32_t id = 0; id < s->nt; ++id) {
        const mcsbr_triangle* t = &s->tri[id];
        double th;
        if (ray_triangle(o, d, s->vert[t->v0], s->vert[t->v1], s->vert[t->v2], t_min, 1e300, &th)) {
            if (th < best_t || (th == best_t && id < best_id)) {
                best_t = th;
                best_id = id;
            }
        }
    }
    if (best_id == 0xFFFFFFFFu) return 0;
    out->t = best_t;
    out->point = vadd(o, vmul(d, best_t));
    out->id = best_id;
    fill_hit(s, out, d);
    return 1;
}

orc_scene* orc_scene_create(const double* xyz, uint32_t nv, const mcsbr_triangle* tris,
                            uint32_t nt, const mcsbr_material* mats, uint32_t nm) {
    if (nt == 0) { /* geometry.cpp:147 */
        set_err("scene has no triangles");
        return NULL;
    }
    orc_scene* s = (orc_scene*)calloc(1, sizeof(orc_scene));
    s->nv = nv;
    s->nt = nt;
    s->nm = nm;
    s->vert = (v3*)malloc(sizeof(v3) * (nv ? nv : 1));
    for (uint32_t i = 0; i < nv; ++i) s->vert[i] = vload(xyz + 3 * i);
    s->tri = (mcsbr_triangle*)malloc(sizeof(mcsbr_triangle) * nt);
    memcpy(s->tri, tris, sizeof(mcsbr_triangle) * nt);
    s->mat = (mcsbr_material*)malloc(sizeof(mcsbr_material) * nm);
    memcpy(s->mat, mats, sizeof(mcsbr_material) * nm);
    s->mat_index = (double*)malloc(sizeof(double) * nm);
    for (uint32_t i = 0; i < nm; ++i) /* em_math.hpp:104 */
        s->mat_index[i] = mats[i].is_pec ? 0.0 : sqrt(mats[i].eps_r * mats[i].mu_r);
    /* Scene::finalize, geometry.cpp:146-162 */
    v3 lo = V(1e300, 1e300, 1e300), hi = V(-1e300, -1e300, -1e300);
    for (uint32_t i = 0; i < nv; ++i) {
        const v3 v = s->vert[i];
        lo = V(dmin(lo.x, v.x), dmin(lo.y, v.y), dmin(lo.z, v.z));
        hi = V(dmax(hi.x, v.x), dmax(hi.y, v.y), dmax(hi.z, v.z));
    }
    s->bcenter = vmul(vadd(lo, hi), 0.5);
    s->bradius = 0.0;
    for (uint32_t i = 0; i < nv; ++i) s->bradius = dmax(s->bradius, vnorm(vsub(s->vert[i], s->bcenter)));
    s->diameter = 2.0 * s->bradius;
    if (!(s->diameter > 0.0)) {
        set_err("scene is degenerate (zero extent)");
        orc_scene_free(s);
        return NULL;
    }
    build_bvh(s);
    return s;
}

void orc_scene_free(orc_scene* s) {
    if (!s) return;
    free(s->vert);
    free(s->tri);
    free(s->mat);
    free(s->mat_index);
    free(s->nodes);
    free(s->order);
    free(s);
}

void orc_scene_bounds(const orc_scene* s, double* b5) {
    vstore(b5, s->bcenter);
    b5[3] = s->bradius;
    b5[4] = s->diameter;
}

static void put_hit(double* h, const hit_t* x) {
    h[0] = x->t;
    vstore(h + 1, x->point);
    vstore(h + 4, x->normal);
    h[7] = x->n_incident;
    h[8] = x->n_transmit;
    h[9] = x->far_side_pec;
    h[10] = x->exterior_facing;
    h[11] = x->near_is_ambient;
    h[12] = x->id;
}
static hit_t get_hit(const double* h) {
    hit_t x;
    x.t = h[0];
    x.point = vload(h + 1);
    x.normal = vload(h + 4);
    x.n_incident = h[7];
    x.n_transmit = h[8];
    x.far_side_pec = h[9] != 0.0;
    x.exterior_facing = h[10] != 0.0;
    x.near_is_ambient = h[11] != 0.0;
    x.id = (uint32_t)h[12];
    return x;
}

int orc_intersect(const orc_scene* s, const double* o, const double* d, const double* t_min,
                  uint64_t n, int mode, double* hit_out) {
    const double eps = 1e-6 * s->diameter; /* geometry.hpp:78 */
    for (uint64_t i = 0; i < n; ++i) {
        double* h = hit_out + 13 * i;
        memset(h, 0, 13 * sizeof(double));
        hit_t x;
        int ok;
        if (mode == 2) { /* geometry.cpp:242-244 */
            h[0] = closest(s, vload(o + 3 * i), vload(d + 3 * i), eps, 1, &x) ? 1.0 : 0.0;
            continue;
        }
        ok = mode == 1 ? brute(s, vload(o + 3 * i), vload(d + 3 * i), t_min[i], &x)
                       : closest(s, vload(o + 3 * i), vload(d + 3 * i), t_min[i], 0, &x);
        if (!ok) {
            h[0] = INFINITY;
            h[12] = 4294967295.0;
            continue;
        }
        put_hit(h, &x);
    }
    return 0;
}

/* geometry.cpp:246-275 */
typedef struct {
    v3 center, u, v;
    double half_u, half_v;
} rect_t;

static rect_t launch_rect(const orc_scene* s, v3 k_inc, double padding) {
    const v3 k = vnormalized(k_inc);
    v3 seed = V(1.0, 0.0, 0.0);
    if (fabs(k.x) > 0.9) seed = V(0.0, 1.0, 0.0);
    const v3 u = vnormalized(vcross(k, seed));
    const v3 v = vcross(k, u);
    double ulo = 1e300, uhi = -1e300, vlo = 1e300, vhi = -1e300;
    for (uint32_t i = 0; i < s->nv; ++i) {
        const double pu = vdot(s->vert[i], u);
        const double pv = vdot(s->vert[i], v);
        ulo = dmin(ulo, pu);
        uhi = dmax(uhi, pu);
        vlo = dmin(vlo, pv);
        vhi = dmax(vhi, pv);
    }
    ulo -= padding;
    uhi += padding;
    vlo -= padding;
    vhi += padding;
    rect_t r;
    r.u = u;
    r.v = v;
    r.half_u = 0.5 * (uhi - ulo);
    r.half_v = 0.5 * (vhi - vlo);
    const double standoff = vdot(s->bcenter, k) - 1.05 * s->bradius;
    r.center = vadd(vadd(vmul(u, 0.5 * (ulo + uhi)), vmul(v, 0.5 * (vlo + vhi))), vmul(k, standoff));
    return r;
}

int orc_launch_rect(const orc_scene* s, const double* k_inc, double padding, double* out11) {
    const rect_t r = launch_rect(s, vload(k_inc), padding);
    vstore(out11, r.center);
    vstore(out11 + 3, r.u);
    vstore(out11 + 6, r.v);
    out11[9] = r.half_u;
    out11[10] = r.half_v;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* flat-block entry points (layouts shared with oracle/ref_shim.cpp)          */

static void put_coeffs(double* p, const coeffs_t* c) {
    p[0] = c->r_s.re; p[1] = c->r_s.im; p[2] = c->r_p.re; p[3] = c->r_p.im;
    p[4] = c->t_s.re; p[5] = c->t_s.im; p[6] = c->t_p.re; p[7] = c->t_p.im;
    p[8] = c->cos_t.re; p[9] = c->cos_t.im; p[10] = c->tir ? 1.0 : 0.0;
}
static coeffs_t get_coeffs(const double* p) {
    coeffs_t c;
    c.r_s = C(p[0], p[1]); c.r_p = C(p[2], p[3]); c.t_s = C(p[4], p[5]);
    c.t_p = C(p[6], p[7]); c.cos_t = C(p[8], p[9]); c.tir = p[10] != 0.0;
    return c;
}
static void put_basis(double* p, const basis_t* b) {
    vstore(p, b->s_hat); vstore(p + 3, b->p_in); vstore(p + 6, b->p_out_r);
    vstore(p + 9, b->p_out_t); vstore(p + 12, b->dir_r); vstore(p + 15, b->dir_t);
}
static basis_t get_basis(const double* p) {
    basis_t b;
    b.s_hat = vload(p); b.p_in = vload(p + 3); b.p_out_r = vload(p + 6);
    b.p_out_t = vload(p + 9); b.dir_r = vload(p + 12); b.dir_t = vload(p + 15);
    return b;
}

int orc_fresnel(double n1, double n2, double cos_i, double* out11) {
    g_fault = 0;
    const coeffs_t c = fresnel(n1, n2, cos_i);
    if (g_fault) return -1;
    put_coeffs(out11, &c);
    return 0;
}
int orc_sp_basis(const double* dir, const double* normal, double n1, double n2, double* out18) {
    g_fault = 0;
    const basis_t b = sp_basis(vload(dir), vload(normal), n1, n2);
    if (g_fault) return -1;
    put_basis(out18, &b);
    return 0;
}
int orc_interface_transform(const double* e6, int branch, const double* coeffs11,
                            const double* basis18, double* out6) {
    g_fault = 0;
    const coeffs_t c = get_coeffs(coeffs11);
    const basis_t b = get_basis(basis18);
    const cv3 r = interface_transform(cvload(e6), branch, &c, &b);
    if (g_fault) return -1;
    cvstore(out6, r);
    return 0;
}
int orc_branch_outcomes(const double* st, const double* hit13, double* out) {
    g_fault = 0;
    path_t s;
    memset(&s, 0, sizeof s);
    s.origin = vload(st);
    s.dir = vload(st + 3);
    s.e[0] = cvload(st + 6);
    s.e[1] = cvload(st + 12);
    s.phi = st[18];
    s.prob = st[19];
    s.weight = st[20];
    s.medium_n = st[21];
    s.bounce = (int)st[22];
    const hit_t h = get_hit(hit13);
    branchset_t set;
    branch_outcomes(&s, &h, &set);
    if (g_fault) return -1;
    memset(out, 0, 63 * sizeof(double));
    out[0] = set.count;
    out[1] = set.grazing;
    if (set.grazing) return 0;
    put_coeffs(out + 2, &set.co);
    put_basis(out + 13, &set.b);
    for (int i = 0; i < set.count; ++i) {
        double* o = out + 31 + 16 * i;
        vstore(o, set.new_dir[i]);
        cvstore(o + 3, set.new_e[i][0]);
        cvstore(o + 9, set.new_e[i][1]);
        o[15] = set.new_n[i];
    }
    return 0;
}
/* farfield.cpp:47-61 (generic overload) */
int orc_meca_currents(const double* hit13, const double* e6, const double* dir, int sc,
                      double* out12) {
    g_fault = 0;
    const hit_t h = get_hit(hit13);
    const v3 d = vload(dir);
    const double cos_i = -vdot(d, h.normal);
    const double n1 = h.n_incident;
    coeffs_t co;
    basis_t b;
    if (sc == 0) {
        co = coeffs_pec();
        b = sp_basis(d, h.normal, n1, n1);
    } else {
        co = fresnel(n1, h.n_transmit, cos_i);
        b = sp_basis(d, h.normal, n1, h.n_transmit);
    }
    cv3 j, m;
    meca(&h, cvload(e6), d, sc, &co, &b, n1, &j, &m);
    if (g_fault) return -1;
    cvstore(out12, j);
    cvstore(out12 + 6, m);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* the estimator (proj/src/solver_mc.cpp:76-229)                              */

typedef struct {
    int nf, uniform;
    double f0, df;
    const double* freqs;
    cx* sums; /* [4][nf] */
    v3 ks, rx_v, rx_h;
} accum_t;

/* farfield.cpp:87-104 */
static void accum_init(accum_t* a, const double* freqs, int nf, v3 ks, v3 rv, v3 rh) {
    a->nf = nf;
    a->freqs = freqs;
    a->ks = ks;
    a->rx_v = rv;
    a->rx_h = rh;
    a->sums = (cx*)calloc(4 * (size_t)nf, sizeof(cx));
    a->uniform = nf >= 2;
    a->f0 = a->df = 0.0;
    if (nf >= 2) {
        a->f0 = freqs[0];
        a->df = freqs[1] - freqs[0];
        for (int i = 1; i < nf; ++i) {
            const double step = freqs[i] - freqs[i - 1];
            if (fabs(step - a->df) > 1e-6 * fabs(a->df)) {
                a->uniform = 0;
                break;
            }
        }
    } else if (nf == 1) {
        a->f0 = freqs[0];
    }
}

/* farfield.cpp:106-146; channels VV=0, HH=1, VH=2, HV=3 */
static void accum_add(accum_t* a, const mcsbr_contribution* c) {
    cx amp[4];
    for (int tx = 0; tx < 2; ++tx) {
        const cv3 aj = cvload(&c->a_j[tx][0][0]);
        const cv3 am = cvload(&c->a_m[tx][0][0]);
        const cv3 f = cvadd(cross_vc(a->ks, cross_vc(a->ks, aj)), cross_vc(a->ks, am));
        const cx av = cvdot(f, a->rx_v);
        const cx ah = cvdot(f, a->rx_h);
        if (tx == 0) {
            amp[0] = av;
            amp[3] = ah;
        } else {
            amp[2] = av;
            amp[1] = ah;
        }
    }
    const double s = c->phi_total - vdot(a->ks, vload(c->exit_point));
    const int n = a->nf;
    if (a->uniform) {
        const double phase0 = -2.0 * kPI * a->f0 / kC * s;
        const double dphase = -2.0 * kPI * a->df / kC * s;
        cx z = C(cos(phase0), sin(phase0));
        const cx w = C(cos(dphase), sin(dphase));
        for (int i = 0; i < n; ++i) {
            for (int ch = 0; ch < 4; ++ch) a->sums[ch * n + i] = cadd(a->sums[ch * n + i], cmul(amp[ch], z));
            z = cmul(z, w);
        }
    } else {
        for (int i = 0; i < n; ++i) {
            const double k0 = 2.0 * kPI * a->freqs[i] / kC;
            const double th = -k0 * s;
            const cx z = C(cos(th), sin(th));
            for (int ch = 0; ch < 4; ++ch) a->sums[ch * n + i] = cadd(a->sums[ch * n + i], cmul(amp[ch], z));
        }
    }
}

typedef struct {
    mcsbr_stats st;
    accum_t acc;
    mcsbr_contribution* col;
    uint64_t ncol, capcol;
} block_t;

static void grow_push(block_t* b, const mcsbr_contribution* c) {
    if (b->ncol == b->capcol) {
        b->capcol = b->capcol ? 2 * b->capcol : 256;
        b->col = (mcsbr_contribution*)realloc(b->col, b->capcol * sizeof(mcsbr_contribution));
    }
    b->col[b->ncol++] = *c;
}

typedef struct { /* per-path event log (orc_path_log) */
    uint64_t first, n;
    uint32_t* tri;
    uint32_t stride;
    uint8_t* term;
    uint64_t* branch;
} plog_t;

static int validate(const mcsbr_mc_config* c) { /* solver_mc.cpp:10-17 */
    if (!(c->strata_per_wavelength > 0.0)) { set_err("mc: strata_per_wavelength must be > 0"); return -1; }
    if (c->samples_per_stratum < 1) { set_err("mc: samples_per_stratum must be >= 1"); return -1; }
    if (!(c->roulette_q > 0.0 && c->roulette_q < 1.0)) { set_err("mc: roulette q must be in (0,1)"); return -1; }
    if (c->roulette_min_bounce < 1) { set_err("mc: roulette min_bounce must be >= 1"); return -1; }
    if (c->max_bounce < 2) { set_err("mc: max_bounce must be >= 2"); return -1; }
    if (c->block_size < 1) { set_err("mc: block_size must be >= 1"); return -1; }
    return 0;
}

static int estimate_impl(const orc_scene* s, const mcsbr_excitation* exc, const double* freqs,
                         uint32_t nf, const mcsbr_mc_config* cfg, double* values, mcsbr_stats* st_out,
                         mcsbr_contribution* contribs, uint64_t capacity, uint64_t* n_contribs,
                         plog_t* plog, uint64_t range_begin, uint64_t range_end, double* raw_out,
                         uint64_t* total_out) {
    g_fault = 0;
    if (validate(cfg)) return -1;
    if (nf == 0) { set_err("estimate: empty frequency list"); return -1; }
    double lambda_ref = cfg->reference_wavelength;
    if (lambda_ref <= 0.0) lambda_ref = kC / freqs[nf - 1];
    const rect_t rect = launch_rect(s, vload(exc->k_inc), cfg->launch_padding);
    /* build_strata, solver_mc.cpp:19-31 */
    if (!(lambda_ref > 0.0)) { set_err("build_strata: reference wavelength must be > 0"); return -1; }
    const double target = lambda_ref / cfg->strata_per_wavelength;
    int nu = (int)ceil(2.0 * rect.half_u / target);
    int nv = (int)ceil(2.0 * rect.half_v / target);
    if (nu < 1) nu = 1;
    if (nv < 1) nv = 1;
    const double cell_area = (4.0 * rect.half_u * rect.half_v) / ((double)nu * nv);
    const uint64_t spp = (uint64_t)cfg->samples_per_stratum;
    const uint64_t total = (uint64_t)(nu * nv) * spp;
    if (total == 0) { set_err("estimate: empty strata grid"); return -1; }

    const v3 ks = vload(exc->k_scatter), rv = vload(exc->rx_v), rh = vload(exc->rx_h);
    const double area_weight = cell_area / (double)spp;
    const double ambient_n = s->mat_index[0];
    const cv3 e0_v = cvreal(vload(exc->pol_v)), e0_h = cvreal(vload(exc->pol_h));
    const double t_eps = 1e-6 * s->diameter;
    const v3 k_inc = vload(exc->k_inc);
    const uint64_t bs = (uint64_t)cfg->block_size;
    const uint64_t nblocks = (total + bs - 1) / bs;

    accum_t total_acc;
    accum_init(&total_acc, freqs, (int)nf, ks, rv, rh);
    mcsbr_stats tot;
    memset(&tot, 0, sizeof tot);
    uint64_t ncontrib_total = 0;
    path_t* live = (path_t*)malloc(sizeof(path_t) * bs);
    path_t* next = (path_t*)malloc(sizeof(path_t) * bs);
    block_t blk;
    memset(&blk, 0, sizeof blk);

    if (total_out) *total_out = total;
    for (uint64_t block = 0; block < nblocks; ++block) {
        uint64_t begin = block * bs;
        uint64_t end = total < begin + bs ? total : begin + bs;
        /* optional entry range (multi-rank sharding checks) */
        if (begin < range_begin) begin = range_begin;
        if (end > range_end) end = range_end;
        if (begin >= end) continue;
        if (plog && (end <= plog->first || begin >= plog->first + plog->n)) continue;
        mcsbr_stats* st = &blk.st;
        memset(st, 0, sizeof *st);
        blk.ncol = 0;
        accum_init(&blk.acc, freqs, (int)nf, ks, rv, rh);
        uint64_t nlive = 0;
        for (uint64_t entry = begin; entry < end; ++entry) {
            const uint32_t cell = (uint32_t)(entry / spp);
            const uint32_t sample = (uint32_t)(entry % spp);
            /* sample_stratum, solver_mc.cpp:33-42 */
            const uint32_t i = cell % (uint32_t)nu, j = cell / (uint32_t)nu;
            const double ju = cfg->jitter ? orc_counter_uniform(cfg->seed, cell, sample, 0, kLaunchU) : 0.5;
            const double jv = cfg->jitter ? orc_counter_uniform(cfg->seed, cell, sample, 0, kLaunchV) : 0.5;
            const double su = -1.0 + 2.0 * ((double)i + ju) / nu;
            const double sv = -1.0 + 2.0 * ((double)j + jv) / nv;
            const v3 p = vadd(vadd(rect.center, vmul(rect.u, su * rect.half_u)), vmul(rect.v, sv * rect.half_v));
            /* init_path, path_engine.cpp:5-15 */
            path_t* ps = &live[nlive++];
            memset(ps, 0, sizeof *ps);
            ps->origin = p;
            ps->dir = k_inc;
            ps->e[0] = e0_v;
            ps->e[1] = e0_h;
            ps->phi = ambient_n * vdot(k_inc, p);
            ps->prob = 1.0;
            ps->weight = 1.0;
            ps->medium_n = ambient_n;
            ps->stratum = cell;
            ps->sample = sample;
        }
        st->rays_launched = nlive;
        int round = 0;
        while (nlive > 0) {
            ++round;
            if (round <= MCSBR_MAX_BOUNCE_LIMIT) st->rays_per_bounce[round - 1] += nlive;
            if ((uint32_t)round > st->n_rounds) st->n_rounds = (uint32_t)round;
            st->segments_traced += nlive;
            uint64_t nnext = 0;
            for (uint64_t li = 0; li < nlive; ++li) {
                path_t state = live[li];
                const uint64_t entry = (uint64_t)state.stratum * spp + state.sample;
                const int logged = plog && entry >= plog->first && entry < plog->first + plog->n;
                const uint64_t lp = logged ? entry - plog->first : 0;
                hit_t hit;
                if (!closest(s, state.origin, state.dir, state.bounce == 0 ? 0.0 : t_eps, 0, &hit)) {
                    if (logged) plog->term[lp] = 0;
                    continue;
                }
                /* advance, path_engine.cpp:17-21 */
                state.phi += state.medium_n * hit.t;
                state.origin = hit.point;
                state.bounce += 1;
                if (logged && (uint32_t)(state.bounce - 1) < plog->stride)
                    plog->tri[lp * plog->stride + (uint32_t)(state.bounce - 1)] = hit.id;
                branchset_t set;
                branch_outcomes(&state, &hit, &set);
                if (g_fault) goto fault;
                if (set.grazing) {
                    ++st->grazing_kills;
                    if (logged) plog->term[lp] = 1;
                    continue;
                }
                const int sc = hit.far_side_pec ? 0 : hit.near_is_ambient ? 1 : 2;
                const int dark_exit = sc == 2 && set.co.tir;
                int visible = 0;
                if (!dark_exit && hit.exterior_facing) { /* chi_visibility, farfield.cpp:63-68 */
                    hit_t occ;
                    visible = !exc->occlusion_enabled ||
                              !closest(s, hit.point, ks, t_eps, 1, &occ);
                }
                if (visible) {
                    cv3 j0, m0, j1, m1;
                    meca(&hit, state.e[0], state.dir, sc, &set.co, &set.b, state.medium_n, &j0, &m0);
                    meca(&hit, state.e[1], state.dir, sc, &set.co, &set.b, state.medium_n, &j1, &m1);
                    if (g_fault) goto fault;
                    /* make_contribution, farfield.cpp:70-85 */
                    const double cos_n = fabs(vdot(state.dir, hit.normal));
                    const double scale = state.weight * area_weight / (state.prob * cos_n);
                    mcsbr_contribution c;
                    memset(&c, 0, sizeof c);
                    cvstore(&c.a_j[0][0][0], cvmuld(j0, scale));
                    cvstore(&c.a_m[0][0][0], cvmuld(m0, scale));
                    cvstore(&c.a_j[1][0][0], cvmuld(j1, scale));
                    cvstore(&c.a_m[1][0][0], cvmuld(m1, scale));
                    c.phi_total = state.phi;
                    vstore(c.exit_point, hit.point);
                    c.bounce = state.bounce;
                    c.order_key = (((uint64_t)state.stratum * spp + state.sample) << 8) |
                                  (uint64_t)(state.bounce & 0xff);
                    accum_add(&blk.acc, &c);
                    if (contribs) grow_push(&blk, &c);
                    ++st->contributions;
                }
                if (state.bounce >= cfg->max_bounce) {
                    ++st->cap_kills;
                    if (logged) plog->term[lp] = 2;
                    continue;
                }
                /* choose_branch, solver_mc.cpp:44-54 */
                const double u_branch =
                    orc_counter_uniform(cfg->seed, state.stratum, state.sample, (uint64_t)state.bounce, kBranch);
                int pick = 0;
                double pprob = 1.0;
                if (set.count != 1) {
                    double p_reflect = 0.5;
                    if (cfg->branch_strategy == MCSBR_BRANCH_FRESNEL) {
                        const double r_bar = 0.5 * (cabs_(set.co.r_s) + cabs_(set.co.r_p));
                        p_reflect = dmin(dmax(r_bar, cfg->p_min), 1.0 - cfg->p_min);
                    }
                    if (u_branch < p_reflect) {
                        pick = 0;
                        pprob = p_reflect;
                    } else {
                        pick = 1;
                        pprob = 1.0 - p_reflect;
                    }
                }
                if (logged && pick) plog->branch[lp] |= 1ull << (state.bounce - 1);
                state.dir = set.new_dir[pick];
                state.e[0] = set.new_e[pick][0];
                state.e[1] = set.new_e[pick][1];
                state.medium_n = set.new_n[pick];
                state.prob *= pprob;
                if (cfg->roulette_enabled && state.bounce >= cfg->roulette_min_bounce) {
                    /* roulette_step, solver_mc.cpp:56-64 */
                    if (state.bounce <= MCSBR_MAX_BOUNCE_LIMIT) ++st->roulette_candidates[state.bounce - 1];
                    const double u_r = orc_counter_uniform(cfg->seed, state.stratum, state.sample,
                                                           (uint64_t)state.bounce, kRoulette);
                    if (!(u_r > cfg->roulette_q)) {
                        if (logged) plog->term[lp] = 3;
                        continue;
                    }
                    state.weight /= (1.0 - cfg->roulette_q);
                    if (state.bounce <= MCSBR_MAX_BOUNCE_LIMIT) ++st->roulette_survivors[state.bounce - 1];
                }
                next[nnext++] = state;
            }
            path_t* tmp = live;
            live = next;
            next = tmp;
            nlive = nnext;
        }
        /* merge in block order, solver_mc.cpp:212-220 */
        for (size_t k = 0; k < 4 * (size_t)nf; ++k) total_acc.sums[k] = cadd(total_acc.sums[k], blk.acc.sums[k]);
        free(blk.acc.sums);
        blk.acc.sums = NULL;
        tot.rays_launched += st->rays_launched;
        tot.segments_traced += st->segments_traced;
        tot.contributions += st->contributions;
        tot.grazing_kills += st->grazing_kills;
        tot.cap_kills += st->cap_kills;
        if (st->n_rounds > tot.n_rounds) tot.n_rounds = st->n_rounds;
        for (int k = 0; k < MCSBR_MAX_BOUNCE_LIMIT; ++k) {
            tot.rays_per_bounce[k] += st->rays_per_bounce[k];
            tot.roulette_candidates[k] += st->roulette_candidates[k];
            tot.roulette_survivors[k] += st->roulette_survivors[k];
        }
        if (contribs) {
            for (uint64_t k = 0; k < blk.ncol && ncontrib_total + k < capacity; ++k)
                contribs[ncontrib_total + k] = blk.col[k];
        }
        ncontrib_total += blk.ncol;
    }
    tot.peak_live_state_bytes = (total < bs ? total : bs) * 192;
    tot.state_bytes_per_ray = 192;
    tot.block_size = bs;
    if (st_out) *st_out = tot;
    if (n_contribs) *n_contribs = ncontrib_total;
    /* raw (un-finalized) sums in the device layout [nf][4] complex */
    if (raw_out) {
        for (uint32_t i = 0; i < nf; ++i)
            for (int ch = 0; ch < 4; ++ch) {
                raw_out[2 * (i * 4 + ch)] = total_acc.sums[ch * nf + i].re;
                raw_out[2 * (i * 4 + ch) + 1] = total_acc.sums[ch * nf + i].im;
            }
    }
    /* finalize, farfield.cpp:154-167 */
    if (values) {
        for (int ch = 0; ch < 4; ++ch) {
            for (uint32_t i = 0; i < nf; ++i) {
                const double k0 = 2.0 * kPI * freqs[i] / kC;
                const cx pre = C(0.0 * k0 / (2.0 * sqrt(kPI)), 1.0 * k0 / (2.0 * sqrt(kPI)));
                const cx v = cmul(pre, total_acc.sums[ch * nf + i]);
                values[2 * (ch * nf + i)] = v.re;
                values[2 * (ch * nf + i) + 1] = v.im;
            }
        }
    }
    free(total_acc.sums);
    free(live);
    free(next);
    free(blk.col);
    return 0;
fault:
    free(total_acc.sums);
    free(blk.acc.sums);
    free(live);
    free(next);
    free(blk.col);
    return -5;
}

int orc_estimate(const orc_scene* s, const mcsbr_excitation* exc, const double* freqs, uint32_t nf,
                 const mcsbr_mc_config* cfg, double* values, mcsbr_stats* st,
                 mcsbr_contribution* contribs, uint64_t capacity, uint64_t* n_contribs) {
    return estimate_impl(s, exc, freqs, nf, cfg, values, st, contribs, capacity, n_contribs, NULL, 0,
                         UINT64_MAX, NULL, NULL);
}

int orc_estimate_range(const orc_scene* s, const mcsbr_excitation* exc, const double* freqs, uint32_t nf,
                       const mcsbr_mc_config* cfg, uint64_t entry_begin, uint64_t entry_end, double* raw_sums,
                       mcsbr_stats* st, uint64_t* total_entries) {
    return estimate_impl(s, exc, freqs, nf, cfg, NULL, st, NULL, 0, NULL, NULL, entry_begin, entry_end,
                         raw_sums, total_entries);
}

int orc_path_log(const orc_scene* s, const mcsbr_excitation* exc, const double* freqs, uint32_t nf,
                 const mcsbr_mc_config* cfg, uint64_t first_entry, uint64_t n_paths, uint32_t* tri_log,
                 uint32_t stride, uint8_t* term, uint64_t* branch_bits) {
    plog_t pl = {first_entry, n_paths, tri_log, stride, term, branch_bits};
    for (uint64_t i = 0; i < n_paths * stride; ++i) tri_log[i] = 0xFFFFFFFFu;
    for (uint64_t i = 0; i < n_paths; ++i) {
        term[i] = 0;
        branch_bits[i] = 0;
    }
    return estimate_impl(s, exc, freqs, nf, cfg, NULL, NULL, NULL, 0, NULL, &pl, 0, UINT64_MAX, NULL, NULL);
}

/* ------------------------------------------------------------------------ */
/* the deterministic solver (proj/src/solver_det.cpp:30-174)                   */

static int validate_det(const mcsbr_det_config* c) { /* solver_det.cpp:11-17 */
    if (!(c->rays_per_wavelength > 0.0)) { set_err("det: rays_per_wavelength must be > 0"); return -1; }
    if (c->max_bounce < 1) { set_err("det: max_bounce must be >= 1"); return -1; }
    if (c->amplitude_cutoff < 0.0) { set_err("det: amplitude_cutoff must be >= 0"); return -1; }
    if (c->block_size < 1) { set_err("det: block_size must be >= 1"); return -1; }
    return 0;
}

int orc_solve(const orc_scene* s, const mcsbr_excitation* exc, const double* freqs, uint32_t nf,
              const mcsbr_det_config* cfg, double* values, mcsbr_stats* st_out,
              mcsbr_contribution* contribs, uint64_t capacity, uint64_t* n_contribs) {
    g_fault = 0;
    if (validate_det(cfg)) return -1;
    if (nf == 0) { set_err("solve: empty frequency list"); return -1; }
    double lambda_ref = cfg->reference_wavelength;
    if (lambda_ref <= 0.0) lambda_ref = kC / freqs[nf - 1];
    const rect_t rect = launch_rect(s, vload(exc->k_inc), cfg->launch_padding);
    /* build_strata, solver_mc.cpp:19-31 */
    if (!(lambda_ref > 0.0)) { set_err("build_strata: reference wavelength must be > 0"); return -1; }
    const double target = lambda_ref / cfg->rays_per_wavelength;
    int nu = (int)ceil(2.0 * rect.half_u / target);
    int nv = (int)ceil(2.0 * rect.half_v / target);
    if (nu < 1) nu = 1;
    if (nv < 1) nv = 1;
    const double cell_area = (4.0 * rect.half_u * rect.half_v) / ((double)nu * nv);
    const uint64_t total = (uint64_t)(nu * nv);

    const v3 ks = vload(exc->k_scatter), rv = vload(exc->rx_v), rh = vload(exc->rx_h);
    const double ambient_n = s->mat_index[0];
    const cv3 e0_v = cvreal(vload(exc->pol_v)), e0_h = cvreal(vload(exc->pol_h));
    const double t_eps = 1e-6 * s->diameter;
    const v3 k_inc = vload(exc->k_inc);
    const double cutoff = cfg->amplitude_cutoff;
    const uint64_t bs = (uint64_t)cfg->block_size;
    const uint64_t nblocks = (total + bs - 1) / bs;

    accum_t total_acc;
    accum_init(&total_acc, freqs, (int)nf, ks, rv, rh);
    mcsbr_stats tot;
    memset(&tot, 0, sizeof tot);
    uint64_t ncontrib_total = 0;
    uint64_t stack_cap = 64;
    path_t* stack = (path_t*)malloc(sizeof(path_t) * stack_cap);
    block_t blk;
    memset(&blk, 0, sizeof blk);

    for (uint64_t block = 0; block < nblocks; ++block) {
        const uint64_t begin = block * bs;
        const uint64_t end = total < begin + bs ? total : begin + bs;
        mcsbr_stats* st = &blk.st;
        memset(st, 0, sizeof *st);
        blk.ncol = 0;
        accum_init(&blk.acc, freqs, (int)nf, ks, rv, rh);
        st->rays_launched = end - begin;
        uint64_t block_peak = 0, block_forced = 0;
        for (uint64_t cell = begin; cell < end; ++cell) {
            /* sample_stratum(jitter = false) + init_path */
            const uint32_t i = (uint32_t)cell % (uint32_t)nu, j = (uint32_t)cell / (uint32_t)nu;
            const double su = -1.0 + 2.0 * ((double)i + 0.5) / nu;
            const double sv = -1.0 + 2.0 * ((double)j + 0.5) / nv;
            const v3 p = vadd(vadd(rect.center, vmul(rect.u, su * rect.half_u)), vmul(rect.v, sv * rect.half_v));
            path_t root;
            memset(&root, 0, sizeof root);
            root.origin = p;
            root.dir = k_inc;
            root.e[0] = e0_v;
            root.e[1] = e0_h;
            root.phi = ambient_n * vdot(k_inc, p);
            root.prob = 1.0;
            root.weight = 1.0;
            root.medium_n = ambient_n;
            root.stratum = (uint32_t)cell;
            uint64_t sp = 0;
            stack[sp++] = root;
            uint64_t ray_peak = 1, ray_pushes = 1;
            uint32_t event_seq = 0;
            while (sp > 0) {
                path_t state = stack[--sp];
                hit_t hit;
                if (!closest(s, state.origin, state.dir, state.bounce == 0 ? 0.0 : t_eps, 0, &hit)) continue;
                ++st->segments_traced;
                state.phi += state.medium_n * hit.t; /* advance */
                state.origin = hit.point;
                state.bounce += 1;
                if (state.bounce <= MCSBR_MAX_BOUNCE_LIMIT) ++st->rays_per_bounce[state.bounce - 1];
                if ((uint32_t)state.bounce > st->n_rounds) st->n_rounds = (uint32_t)state.bounce;
                branchset_t set;
                branch_outcomes(&state, &hit, &set);
                if (g_fault) goto fault;
                if (set.grazing) {
                    ++st->grazing_kills;
                    continue;
                }
                const int sc = hit.far_side_pec ? 0 : hit.near_is_ambient ? 1 : 2;
                const int dark_exit = sc == 2 && set.co.tir;
                int visible = 0;
                if (!dark_exit && hit.exterior_facing) {
                    hit_t occ;
                    visible = !exc->occlusion_enabled || !closest(s, hit.point, ks, t_eps, 1, &occ);
                }
                if (visible) {
                    cv3 j0, m0, j1, m1;
                    meca(&hit, state.e[0], state.dir, sc, &set.co, &set.b, state.medium_n, &j0, &m0);
                    meca(&hit, state.e[1], state.dir, sc, &set.co, &set.b, state.medium_n, &j1, &m1);
                    if (g_fault) goto fault;
                    const double cos_n = fabs(vdot(state.dir, hit.normal));
                    const double scale = state.weight * cell_area / (state.prob * cos_n);
                    mcsbr_contribution c;
                    memset(&c, 0, sizeof c);
                    cvstore(&c.a_j[0][0][0], cvmuld(j0, scale));
                    cvstore(&c.a_m[0][0][0], cvmuld(m0, scale));
                    cvstore(&c.a_j[1][0][0], cvmuld(j1, scale));
                    cvstore(&c.a_m[1][0][0], cvmuld(m1, scale));
                    c.phi_total = state.phi;
                    vstore(c.exit_point, hit.point);
                    c.bounce = state.bounce;
                    c.order_key = ((uint64_t)state.stratum << 24) | (uint64_t)(event_seq++);
                    accum_add(&blk.acc, &c);
                    if (contribs) grow_push(&blk, &c);
                    ++st->contributions;
                }
                if (state.bounce >= cfg->max_bounce) {
                    ++st->cap_kills;
                    continue;
                }
                /* push every surviving branch, transmit first (reflect on top) */
                for (int k = set.count - 1; k >= 0; --k) {
                    if (cutoff > 0.0 && dmax(cvnorm(set.new_e[k][0]), cvnorm(set.new_e[k][1])) < cutoff) continue;
                    if (sp == stack_cap) {
                        stack_cap *= 2;
                        stack = (path_t*)realloc(stack, sizeof(path_t) * stack_cap);
                    }
                    path_t child = state;
                    child.dir = set.new_dir[k];
                    child.e[0] = set.new_e[k][0];
                    child.e[1] = set.new_e[k][1];
                    child.medium_n = set.new_n[k];
                    stack[sp++] = child;
                    ++ray_pushes;
                }
                if (sp + 1 > ray_peak) ray_peak = sp + 1;
            }
            block_peak += ray_peak * 192;
            block_forced += ray_pushes * 192;
        }
        for (size_t k = 0; k < 4 * (size_t)nf; ++k) total_acc.sums[k] = cadd(total_acc.sums[k], blk.acc.sums[k]);
        free(blk.acc.sums);
        blk.acc.sums = NULL;
        tot.rays_launched += st->rays_launched;
        tot.segments_traced += st->segments_traced;
        tot.contributions += st->contributions;
        tot.grazing_kills += st->grazing_kills;
        tot.cap_kills += st->cap_kills;
        if (st->n_rounds > tot.n_rounds) tot.n_rounds = st->n_rounds;
        for (int k = 0; k < MCSBR_MAX_BOUNCE_LIMIT; ++k) tot.rays_per_bounce[k] += st->rays_per_bounce[k];
        if (block_peak > tot.peak_live_state_bytes) tot.peak_live_state_bytes = block_peak;
        if (block_forced > tot.forced_stack_bytes) tot.forced_stack_bytes = block_forced;
        if (contribs) {
            for (uint64_t k = 0; k < blk.ncol && ncontrib_total + k < capacity; ++k)
                contribs[ncontrib_total + k] = blk.col[k];
        }
        ncontrib_total += blk.ncol;
    }
    tot.state_bytes_per_ray = 192;
    tot.block_size = bs;
    if (st_out) *st_out = tot;
    if (n_contribs) *n_contribs = ncontrib_total;
    if (values) { /* finalize, farfield.cpp:154-167 */
        for (int ch = 0; ch < 4; ++ch) {
            for (uint32_t i = 0; i < nf; ++i) {
                const double k0 = 2.0 * kPI * freqs[i] / kC;
                const cx pre = C(0.0 * k0 / (2.0 * sqrt(kPI)), 1.0 * k0 / (2.0 * sqrt(kPI)));
                const cx v = cmul(pre, total_acc.sums[ch * nf + i]);
                values[2 * (ch * nf + i)] = v.re;
                values[2 * (ch * nf + i) + 1] = v.im;
            }
        }
    }
    free(total_acc.sums);
    free(stack);
    free(blk.col);
    return 0;
fault:
    free(total_acc.sums);
    free(blk.acc.sums);
    free(stack);
    free(blk.col);
    return -5;
}
