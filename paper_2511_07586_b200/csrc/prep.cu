// Scene preparation and launch planning on the device (the host-side loops
// they replace cost ~30 ms per sweep on the 1M-triangle airframe, 5% of the
// end-to-end step).  Every result is exactly the host arithmetic's:
//
//   pack_kernel      Scene::finalize's checks (geometry.cpp:146-162 and the
//                    loader's index checks) and the device triangle layout:
//                    vertex indices, normal + packed (front, back, exterior),
//                    the all-PEC flag; the FIRST bad triangle is reported
//                    (atomicMin over index * 2 + kind), as the host loop does.
//   bounds_kernel    the vertex AABB, and radius_kernel the bounding radius
//                    max |v - c| (geometry.cpp:149-158), with norm() in the
//                    reference's operation order (--fmad=false); min / max are
//                    exact, so the result is bit-identical to the host loop.
//   extents_kernel   launch_rect's projection extents (geometry.cpp:254-266):
//                    min / max of dot(p, u) and dot(p, v) over the vertices for
//                    every incidence of a batch, same operation order.
//
// Min / max of doubles use an order-preserving map to uint64 and integer
// atomics (exact for finite values).
#include <cstdint>

#include "internal.h"
#include "mcsbr_gpu.h"

namespace mcsbr_int {

namespace {

__device__ __forceinline__ unsigned long long ord(double x) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ unsigned long long warp_min(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}
__device__ __forceinline__ unsigned long long warp_max(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

__global__ void pack_kernel(const mcsbr_triangle* __restrict__ tris, uint32_t nt, uint32_t nv, uint32_t nm,
                            const uint8_t* __restrict__ is_pec, uint4* __restrict__ tri_idx,
                            double2* __restrict__ info, unsigned long long* __restrict__ first_bad,
                            unsigned int* __restrict__ not_all_pec) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nt) return;
    const mcsbr_triangle t = tris[i];
    if (t.v0 >= nv || t.v1 >= nv || t.v2 >= nv) {
        atomicMin(first_bad, 2ull * i);  // "vertex index out of range" (checked first, as the host did)
        return;
    }
    if (t.front_material >= nm || t.back_material >= nm) {
        atomicMin(first_bad, 2ull * i + 1);  // "material index out of range"
        return;
    }
    tri_idx[i] = make_uint4(t.v0, t.v1, t.v2, 0);
    const unsigned long long packed = static_cast<unsigned long long>(t.front_material) |
                                      (static_cast<unsigned long long>(t.back_material) << 16) |
                                      (static_cast<unsigned long long>(t.exterior_facing ? 1 : 0) << 32);
    info[2ull * i] = make_double2(t.normal[0], t.normal[1]);
    info[2ull * i + 1] = make_double2(t.normal[2], __longlong_as_double(static_cast<long long>(packed)));
    if (!is_pec[t.front_material] && !is_pec[t.back_material]) *not_all_pec = 1u;
}

// out[0..2] = ord(min x, y, z), out[3..5] = ord(max x, y, z)
__global__ void bounds_kernel(const double* __restrict__ v, uint32_t nv, unsigned long long* __restrict__ out) {
    unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const unsigned long long o = ord(v[3ull * i + k]);
            lo[k] = o < lo[k] ? o : lo[k];
            hi[k] = o > hi[k] ? o : hi[k];
        }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        lo[k] = warp_min(lo[k]);
        hi[k] = warp_max(hi[k]);
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            atomicMin(out + k, lo[k]);
            atomicMax(out + 3 + k, hi[k]);
        }
    }
}

// max over vertices of norm(v - c) = sqrt((dx*dx + dy*dy) + dz*dz)
__global__ void radius_kernel(const double* __restrict__ v, uint32_t nv, double cx, double cy, double cz,
                              unsigned long long* __restrict__ out) {
    unsigned long long hi = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x) {
        const double dx = v[3ull * i] - cx, dy = v[3ull * i + 1] - cy, dz = v[3ull * i + 2] - cz;
        const unsigned long long o = ord(sqrt(dx * dx + dy * dy + dz * dz));
        hi = o > hi ? o : hi;
    }
    hi = warp_max(hi);
    if ((threadIdx.x & 31) == 0) atomicMax(out, hi);
}

// axes[a] = (u.xyz, v.xyz); out[a] = ord(min dot(p,u), max dot(p,u), min dot(p,v), max dot(p,v))
__global__ void extents_kernel(const double* __restrict__ v, uint32_t nv, const double* __restrict__ axes,
                               unsigned long long* __restrict__ out) {
    const uint32_t a = blockIdx.y;
    const double ux = axes[6 * a], uy = axes[6 * a + 1], uz = axes[6 * a + 2];
    const double vx = axes[6 * a + 3], vy = axes[6 * a + 4], vz = axes[6 * a + 5];
    unsigned long long ulo = ~0ull, uhi = 0, vlo = ~0ull, vhi = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x) {
        const double px = v[3ull * i], py = v[3ull * i + 1], pz = v[3ull * i + 2];
        const unsigned long long pu = ord(px * ux + py * uy + pz * uz);
        const unsigned long long pv = ord(px * vx + py * vy + pz * vz);
        ulo = pu < ulo ? pu : ulo;
        uhi = pu > uhi ? pu : uhi;
        vlo = pv < vlo ? pv : vlo;
        vhi = pv > vhi ? pv : vhi;
    }
    ulo = warp_min(ulo);
    uhi = warp_max(uhi);
    vlo = warp_min(vlo);
    vhi = warp_max(vhi);
    if ((threadIdx.x & 31) == 0) {
        atomicMin(out + 4 * a, ulo);
        atomicMax(out + 4 * a + 1, uhi);
        atomicMin(out + 4 * a + 2, vlo);
        atomicMax(out + 4 * a + 3, vhi);
    }
}

// tri64 record k = (a.x, a.y) (a.z, e1.x) (e1.y, e1.z) (e2.x, e2.y) (e2.z, id)
__global__ void leaf32_kernel(const double2* __restrict__ t64, uint32_t n, double cx, double cy, double cz,
                              double radius, float4* __restrict__ out) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double2* r = t64 + 5ull * k;
    const double2 r0 = r[0], r1 = r[1], r2 = r[2], r3 = r[3], r4 = r[4];
    const uint32_t id = static_cast<uint32_t>(__double_as_longlong(r4.y));
    // error numerators of pathcore.cuh tri_test32: with every fp32 operand
    // O(R) (|s| <= 2.02 R) and L the longest edge, the rounding of s . p,
    // d . q and e2 . q moves u, v by <= ~8 eps 2R L / |det| and t by <=
    // ~8 eps 2R L^2 / |det|; 8x margin on top (eps = 2^-24)
    const double e1x = r1.y, e1y = r2.x, e1z = r2.y, e2x = r3.x, e2y = r3.y, e2z = r4.x;
    const double l1 = e1x * e1x + e1y * e1y + e1z * e1z, l2 = e2x * e2x + e2y * e2y + e2z * e2z;
    const double l3 = (e2x - e1x) * (e2x - e1x) + (e2y - e1y) * (e2y - e1y) + (e2z - e1z) * (e2z - e1z);
    const double lmax = sqrt(fmax(l1, fmax(l2, l3)));
    const double kb = 64.0 * 0x1p-24 * 2.02 * radius * lmax;
    out[3ull * k] = make_float4(__double2float_rn(r0.x - cx), __double2float_rn(r0.y - cy),
                                __double2float_rn(r1.x - cz), __double2float_rn(e1x));
    out[3ull * k + 1] = make_float4(__double2float_rn(e1y), __double2float_rn(e1z), __double2float_rn(e2x),
                                    __double2float_rn(e2y));
    out[3ull * k + 2] = make_float4(__double2float_rn(e2z), __uint_as_float(id), __double2float_ru(kb),
                                    __double2float_ru(kb * lmax));
}

__global__ void init_minmax_kernel(unsigned long long* out, uint32_t n_pairs) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_pairs) {
        out[2 * i] = ~0ull;
        out[2 * i + 1] = 0ull;
    }
}

}  // namespace

double unord(unsigned long long o) {
    const unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
    double x;
    __builtin_memcpy(&x, &b, sizeof(x));
    return x;
}

cudaError_t launch_pack(const mcsbr_triangle* d_raw, uint32_t nt, uint32_t nv, uint32_t nm, const uint8_t* d_is_pec,
                        uint4* d_tri, double2* d_info, unsigned long long* d_first_bad, unsigned int* d_not_all_pec,
                        cudaStream_t stream) {
    pack_kernel<<<(nt + 255) / 256, 256, 0, stream>>>(d_raw, nt, nv, nm, d_is_pec, d_tri, d_info, d_first_bad,
                                                      d_not_all_pec);
    return cudaGetLastError();
}

cudaError_t launch_bounds(const double* d_vtx, uint32_t nv, unsigned long long* d_out, int device_sms,
                          cudaStream_t stream) {
    unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
    cudaError_t e = cudaMemcpyAsync(d_out, init, sizeof(init), cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return e;
    const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((nv + 255) / 256, 4ull * device_sms));
    bounds_kernel<<<blocks, 256, 0, stream>>>(d_vtx, nv, d_out);
    return cudaGetLastError();
}

cudaError_t launch_radius(const double* d_vtx, uint32_t nv, const double c[3], unsigned long long* d_out,
                          int device_sms, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(d_out, 0, sizeof(unsigned long long), stream);
    if (e != cudaSuccess) return e;
    const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((nv + 255) / 256, 4ull * device_sms));
    radius_kernel<<<blocks, 256, 0, stream>>>(d_vtx, nv, c[0], c[1], c[2], d_out);
    return cudaGetLastError();
}

cudaError_t launch_leaf32(const double2* tri64, uint32_t n, const double center[3], double radius, float4* out,
                         cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    leaf32_kernel<<<(n + 255) / 256, 256, 0, stream>>>(tri64, n, center[0], center[1], center[2], radius, out);
    return cudaGetLastError();
}

cudaError_t launch_extents(const double* d_vtx, uint32_t nv, const double* d_axes, uint32_t n_inc,
                           unsigned long long* d_out, int device_sms, cudaStream_t stream) {
    if (n_inc == 0) return cudaSuccess;
    init_minmax_kernel<<<(2 * n_inc + 255) / 256, 256, 0, stream>>>(d_out, 2 * n_inc);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // enough blocks over all incidences to fill the GPU
    uint64_t bx = (static_cast<uint64_t>(device_sms) * 8 + n_inc - 1) / n_inc;
    bx = std::min<uint64_t>(std::max<uint64_t>(bx, 1), (nv + 255) / 256);
    for (uint32_t a0 = 0; a0 < n_inc; a0 += 65535) {
        const uint32_t na = std::min<uint32_t>(65535u, n_inc - a0);
        extents_kernel<<<dim3(static_cast<unsigned>(bx), na), 256, 0, stream>>>(d_vtx, nv, d_axes + 6ull * a0,
                                                                                 d_out + 4ull * a0);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace mcsbr_int
