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
};

struct Coeffs {
    Cx r_s, r_p, t_s, t_p, cos_t;
    bool tir;
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
    c.r_s = cdiv(ci * n1 - cos_t * n2, den_s);
    c.t_s = cdiv(ci * (2.0 * n1), den_s);
    c.r_p = cdiv(ci * n2 - cos_t * n1, den_p);
    c.t_p = cdiv(ci * (2.0 * n1), den_p);
    return c;
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

// branch: 0 = reflect, 1 = transmit
__device__ inline CV3 interface_transform(const CV3& e, int branch, const Coeffs& co,
                                          const Basis& b, uint32_t& fault) {
    // Transversality guard (the reference throws DomainError).  Only the fault
    // flag depends on it, so it is evaluated on squares: |x|^2 > (1e-9 (1+|e|))^2.
    const V3 dir_in = cross(b.s_hat, b.p_in);
    const double lim = 1e-9 * (1.0 + norm(e));
    if (cnorm2(dot(e, dir_in)) > lim * lim) fault |= kFaultTransverse;
    const Cx es = dot(e, b.s_hat);
    const Cx ep = dot(e, b.p_in);
    if (branch == 0) return cvreal(b.s_hat) * (es * co.r_s) + cvreal(b.p_out_r) * (ep * co.r_p);
    return cvreal(b.s_hat) * (es * co.t_s) + cvreal(b.p_out_t) * (ep * co.t_p);
}

}  // namespace mcsbr_dev
