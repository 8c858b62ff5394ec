// GO field transport at one interface and the MECA surface currents, on the
// device, in the reference's exact fp64 operation order:
//   fresnel            proj/src/em_math.cpp:5-30
//   reflect_dir        proj/src/em_math.cpp:32-37
//   refract_dir        proj/src/em_math.cpp:39-49
//   sp_basis           proj/src/em_math.cpp:51-81
//   interface_transform proj/src/em_math.cpp:83-95
//   branch_outcomes    proj/src/path_engine.cpp:23-54
//   meca_currents      proj/src/farfield.cpp:11-45
// Where the reference throws (DomainError / DegenerateGeometryError) the device
// code raises a fault bit that the host turns into MCSBR_EDEVICE.
#pragma once

#include "dmath.cuh"

namespace mcsbr_dev {

enum : uint32_t {
    kFaultFresnel = 1u,
    kFaultTransverse = 2u,
    kFaultGrazingDir = 4u,
    kFaultStack = 8u,
    kFaultFixedRange = 16u,  // MCSBR_REDUCE_EXACT: a term outside the 192-bit fixed-point range
};

struct Coeffs {
    Cx r_s, r_p, t_s, t_p, cos_t;
    bool tir;
    bool lossy = false;  // an interface with a lossy side (fresnel_c): no reference counterpart
};

struct Basis {
    V3 s_hat, p_in, p_out_r, p_out_t, dir_r, dir_t;
};

__device__ __forceinline__ Coeffs coeffs_pec() {  // em_math.hpp:127-133
    Coeffs c;
    c.r_s = {-1.0, 0.0};
    c.r_p = {1.0, 0.0};
    c.t_s = {0.0, 0.0};
    c.t_p = {0.0, 0.0};
    c.cos_t = {0.0, 0.0};
    c.tir = false;
    return c;
}

// __divdc3 of two complex numbers with zero imaginary parts is
// (num.re / den.re, +-0): ratio = 0, denom = c exactly, x = (a + 0) / c, and
// its range scalings multiply numerator and denominator by the same power of
// two (|c| in [2^-52, 2^1022] skips them anyway).  Real-index Fresnel
// coefficients below the critical angle are exactly that case, so they take
// one IEEE division inline instead of the out-of-line Smith division (which
// was 10% of the lossless dielectric kernel's samples); the sign of a zero
// imaginary part may differ, which no later operation can turn into a
// non-zero difference.  Anything else goes to cdiv.
__device__ __forceinline__ Cx cdiv_r(Cx num, Cx den) {
    if (num.im == 0.0 && den.im == 0.0 && fabs(den.re) >= 2.220446049250313e-16 &&
        fabs(den.re) < 8.98846567431158e307)
        return {num.re / den.re, 0.0};
    return cdiv(num, den);
}

__device__ inline Coeffs fresnel(double n1, double n2, double cos_i, uint32_t& fault) {
    Coeffs c;
    c.tir = false;
    if (!(isfinite(n1) && isfinite(n2)) || n1 <= 0.0 || n2 <= 0.0 || !(cos_i > 0.0 && cos_i <= 1.0)) {
        fault |= kFaultFresnel;
        c.r_s = c.r_p = c.t_s = c.t_p = c.cos_t = {0.0, 0.0};
        return c;
    }
    const double x = 1.0 - cos_i * cos_i;
    const double sin2_i = (0.0 < x) ? x : 0.0;  // std::max(0.0, x)
    const double s2 = (n1 / n2) * (n1 / n2) * sin2_i;
    Cx cos_t;
    if (s2 > 1.0) {
        c.tir = true;
        cos_t = {0.0, -sqrt(s2 - 1.0)};
    } else {
        cos_t = {sqrt(1.0 - s2), 0.0};
    }
    c.cos_t = cos_t;
    const Cx ci = {cos_i, 0.0};
    const Cx den_s = ci * n1 + cos_t * n2;
    const Cx den_p = ci * n2 + cos_t * n1;
    c.r_s = cdiv_r(ci * n1 - cos_t * n2, den_s);
    c.t_s = cdiv_r(ci * (2.0 * n1), den_s);
    c.r_p = cdiv_r(ci * n2 - cos_t * n1, den_p);
    c.t_p = cdiv_r(ci * (2.0 * n1), den_p);
    return c;
}

// ---- lossy-media extension (not in the reference: Material is real there,
// em_math.hpp:99-105).  eps = eps_r - j eps_i, n = sqrt(eps mu) with Im n <= 0.

// principal complex square root; exact sqrt(x) for a non-negative real input
__device__ __forceinline__ Cx csqrt(Cx z) {
    if (z.im == 0.0) return z.re >= 0.0 ? Cx{sqrt(z.re), 0.0} : Cx{0.0, sqrt(-z.re)};
    const double m = hypot(z.re, z.im);
    const double a = sqrt(0.5 * (m + fabs(z.re)));
    const double b = 0.5 * z.im / a;
    return z.re >= 0.0 ? Cx{a, b} : Cx{fabs(b), copysign(a, z.im)};
}

// the principal root on a lossy interface (no reference counterpart): |z|
// as sqrt(re^2 + im^2) instead of hypot, one reciprocal square root instead
// of sqrt + divide (|z| ~ 1e-6 .. 1e6 here, far from over/underflow)
__device__ __forceinline__ Cx csqrt_lossy(Cx z) {
    if (z.im == 0.0) return csqrt(z);
    const double m = sqrt(z.re * z.re + z.im * z.im);
    const double t = 0.5 * (m + fabs(z.re));
    const double r = rsqrt(t);
    const double a = t * r, b = 0.5 * z.im * r;
    return z.re >= 0.0 ? Cx{a, b} : Cx{fabs(b), copysign(a, z.im)};
}

// ---- index-type helpers: the path kernel is written once for NT = double
// (the reference's lossless model, bit-exact) and NT = Cx (lossy extension).
__device__ __forceinline__ double re_of(double x) { return x; }
__device__ __forceinline__ double re_of(Cx x) { return x.re; }
__device__ __forceinline__ double im_of(double) { return 0.0; }
__device__ __forceinline__ double im_of(Cx x) { return x.im; }
__device__ __forceinline__ Cx operator-(Cx a, double b) { return {a.re - b, a.im}; }
template <typename NT>
__device__ __forceinline__ NT make_nt(double re, double im);
template <>
__device__ __forceinline__ double make_nt<double>(double re, double) { return re; }
template <>
__device__ __forceinline__ Cx make_nt<Cx>(double re, double im) { return {re, im}; }

// e^{-j k0 s}: the phase of farfield.cpp:128-145; for a complex optical path
// the imaginary part (<= 0 in lossy media) gives the attenuation e^{k0 Im s}.
__device__ __forceinline__ Cx phasor(double k0, double s) {
    double sn, cs;
    sincos(-k0 * s, &sn, &cs);
    return {cs, sn};
}
// e^{la} (cos ph + j sin ph); la = 0 for the lossless model
__device__ __forceinline__ Cx polar_la(double ph, double la) {
    double sn, cs;
    sincos(ph, &sn, &cs);
    if (la == 0.0) return {cs, sn};
    const double a = exp(la);
    return {cs * a, sn * a};
}
__device__ __forceinline__ Cx phasor(double k0, Cx s) {
    double sn, cs;
    sincos(-k0 * s.re, &sn, &cs);
    const double a = exp(k0 * s.im);
    return {cs * a, sn * a};
}

// Fresnel coefficients for complex indices (fresnel() generalised): the
// transmitted cos_t root is chosen physically (below); `tir` is decided from
// the real parts (the ray geometry uses Re n).  For real n1, n2 this
// reproduces fresnel() operation for operation, incl. the -j branch under TIR.
__device__ inline Coeffs fresnel_c(Cx n1, Cx n2, double cos_i, bool tir, uint32_t& fault) {
    Coeffs c;
    c.tir = tir;
    if (!(n1.re > 0.0) || !(n2.re > 0.0) || !(cos_i > 0.0 && cos_i <= 1.0) || !isfinite(n1.re) ||
        !isfinite(n2.re)) {
        fault |= kFaultFresnel;
        c.r_s = c.r_p = c.t_s = c.t_p = c.cos_t = {0.0, 0.0};
        return c;
    }
    const double x = 1.0 - cos_i * cos_i;
    const double sin2_i = (0.0 < x) ? x : 0.0;
    // An interface with a lossy side has no reference counterpart (the
    // reference is lossless), so its quotients use one reciprocal per
    // denominator (1 / |den|^2 times conj(den): one fp64 division instead of
    // the three of the Smith division, a few ulps from it for |n| ~ 1..1e3);
    // real indices keep cdiv, the reference's __divdc3, bit for bit.
    const bool lossy_if = n1.im != 0.0 || n2.im != 0.0;
    c.lossy = lossy_if;
    auto inv = [](Cx d) {
        const double s = 1.0 / (d.re * d.re + d.im * d.im);
        return Cx{d.re * s, -(d.im * s)};
    };
    const Cx q = lossy_if ? n1 * inv(n2) : cdiv_r(n1, n2);
    const Cx s2 = (q * q) * sin2_i;
    // Root choice for k_z = k0 n2 cos_t: a propagating transmitted wave
    // (|Re k_z| >= |Im k_z|) must carry power away (Re k_z >= 0); an
    // evanescent one must decay away from the interface (Im k_z <= 0).  For
    // real indices this gives the reference's branches exactly: the real
    // root below the critical angle and (0, -sqrt(s2 - 1)) under TIR.
    Cx cos_t = lossy_if ? csqrt_lossy(Cx{1.0 - s2.re, -s2.im}) : csqrt(Cx{1.0 - s2.re, -s2.im});
    const Cx kz = n2 * cos_t;
    const bool flip = fabs(kz.re) >= fabs(kz.im) ? kz.re < 0.0 : kz.im > 0.0;
    if (flip) cos_t = {-cos_t.re, -cos_t.im};
    if (cos_t.re == 0.0) cos_t.re = 0.0;  // no -0 (matches the reference's (0, -x))
    c.cos_t = cos_t;
    const Cx ci = {cos_i, 0.0};
    const Cx den_s = ci * n1 + cos_t * n2;
    const Cx den_p = ci * n2 + cos_t * n1;
    if (lossy_if) {
        const Cx is = inv(den_s), ip = inv(den_p);
        c.r_s = (ci * n1 - cos_t * n2) * is;
        c.t_s = (ci * (n1 * 2.0)) * is;
        c.r_p = (ci * n2 - cos_t * n1) * ip;
        c.t_p = (ci * (n1 * 2.0)) * ip;
    } else {
        c.r_s = cdiv_r(ci * n1 - cos_t * n2, den_s);
        c.t_s = cdiv_r(ci * (n1 * 2.0), den_s);
        c.r_p = cdiv_r(ci * n2 - cos_t * n1, den_p);
        c.t_p = cdiv_r(ci * (n1 * 2.0), den_p);
    }
    return c;
}

// fresnel for either index type; the lossy TIR decision uses the real parts
__device__ __forceinline__ Coeffs fresnel_any(double n1, double n2, double cos_i, uint32_t& fault) {
    return fresnel(n1, n2, cos_i, fault);
}
__device__ __forceinline__ Coeffs fresnel_any(Cx n1, Cx n2, double cos_i, uint32_t& fault) {
    const double x = 1.0 - cos_i * cos_i;
    const double sin2_i = (0.0 < x) ? x : 0.0;
    const double r = n1.re / n2.re;
    return fresnel_c(n1, n2, cos_i, r * r * sin2_i > 1.0, fault);
}

__device__ __forceinline__ V3 reflect_dir(V3 dir, V3 normal, uint32_t& fault) {
    const double dn = dot(dir, normal);
    if (fabs(dn) < 1e-9) fault |= kFaultGrazingDir;
    return dir - normal * (2.0 * dn);
}

__device__ __forceinline__ bool refract_dir(V3 dir, V3 normal, double n1, double n2, V3& out,
                                            uint32_t& fault) {
    const double dn = dot(dir, normal);
    if (fabs(dn) < 1e-9) fault |= kFaultGrazingDir;
    const double cos_i = -dn;
    const double eta = n1 / n2;
    const double x = 1.0 - cos_i * cos_i;
    const double sin2_t = eta * eta * ((0.0 < x) ? x : 0.0);
    if (sin2_t > 1.0) return false;
    const double cos_t = sqrt(1.0 - sin2_t);
    out = normalized(dir * eta + normal * (eta * cos_i - cos_t));
    return true;
}

// need_t = false skips the refracted direction (only used by the transmit
// branch and by exiting currents, neither of which exists on PEC hits).
__device__ inline Basis sp_basis(V3 dir_in, V3 normal, double n1, double n2, bool need_t,
                                 uint32_t& fault) {
    Basis b;
    const V3 c = cross(dir_in, normal);
    const double cn = norm(c);
    if (cn < 1e-6) {
        V3 axis = {1.0, 0.0, 0.0};
        V3 s = axis - dir_in * dot(axis, dir_in);
        if (norm(s) < 1e-6) {
            axis = {0.0, 1.0, 0.0};
            s = axis - dir_in * dot(axis, dir_in);
        }
        b.s_hat = normalized(s);
    } else {
        b.s_hat = c / cn;
    }
    b.dir_r = reflect_dir(dir_in, normal, fault);
    b.p_in = cross(dir_in, b.s_hat);
    b.p_out_r = cross(b.dir_r, b.s_hat);
    V3 t;
    if (need_t && refract_dir(dir_in, normal, n1, n2, t, fault)) {
        b.dir_t = t;
        b.p_out_t = cross(b.dir_t, b.s_hat);
    } else {
        b.dir_t = dir_in;
        b.p_out_t = b.p_in;
    }
    return b;
}

// interface_transform's transversality guard alone (it does not depend on
// the branch, so evaluating it once per field raises exactly the reference's
// faults whichever branches are formed)
__device__ __forceinline__ void transverse_guard(const CV3& e, const Basis& b, uint32_t& fault) {
    const V3 dir_in = cross(b.s_hat, b.p_in);
    // (1 + |e|)^2 >= 1 + |e|^2 (halved for rounding): the square root only when this bound does not clear it
    const double de2 = cnorm2(dot(e, dir_in));
    if (de2 > 0.5e-18 * (1.0 + (cnorm2(e.x) + cnorm2(e.y) + cnorm2(e.z)))) {
        const double lim = 1e-9 * (1.0 + norm(e));
        if (de2 > lim * lim) fault |= kFaultTransverse;
    }
}
__device__ __forceinline__ void transverse_guard(const V3& e, const Basis& b, uint32_t& fault) {
    const V3 dir_in = cross(b.s_hat, b.p_in);
    const double de = dot(e, dir_in);
    if (de * de > 0.5e-18 * (1.0 + dot(e, e))) {
        const double lim = 1e-9 * (1.0 + norm(e));
        if (de * de > lim * lim) fault |= kFaultTransverse;
    }
}
// the transformed field of one branch, without the guard
__device__ __forceinline__ CV3 branch_field(const CV3& e, int branch, const Coeffs& co, const Basis& b) {
    const Cx es = dot(e, b.s_hat);
    const Cx ep = dot(e, b.p_in);
    const bool r = branch == 0;  // operands selected, one copy of the arithmetic
    return vmul(b.s_hat, es * (r ? co.r_s : co.t_s)) + vmul(r ? b.p_out_r : b.p_out_t, ep * (r ? co.r_p : co.t_p));
}
__device__ __forceinline__ V3 branch_field(const V3& e, int branch, const Coeffs& co, const Basis& b) {
    const double es = dot(e, b.s_hat);
    const double ep = dot(e, b.p_in);
    const bool r = branch == 0;
    return b.s_hat * (es * (r ? co.r_s.re : co.t_s.re)) + (r ? b.p_out_r : b.p_out_t) * (ep * (r ? co.r_p.re : co.t_p.re));
}

// branch: 0 = reflect, 1 = transmit
__device__ inline CV3 interface_transform(const CV3& e, int branch, const Coeffs& co,
                                          const Basis& b, uint32_t& fault) {
    // transversality guard (the reference throws DomainError); only the fault
    // flag depends on it
    transverse_guard(e, b, fault);
    return branch_field(e, branch, co, b);
}

// Real-field version for PEC hits (real coefficients r_s = -1, r_p = +1):
// the complex version's real parts, operation for operation (its imaginary
// parts are exactly +-0 there); only the reflected branch exists.
__device__ inline V3 interface_transform(const V3& e, int branch, const Coeffs& co, const Basis& b,
                                         uint32_t& fault) {
    transverse_guard(e, b, fault);
    return branch_field(e, branch, co, b);
}

}  // namespace mcsbr_dev
