// Launch-ray culling: a conservative coverage bitmap of every incidence's
// strata grid.
//
// All launch rays of one incidence are parallel (direction k_inc, origins on
// the launch rectangle of launch_rect, proj/src/geometry.cpp:246-275), so a
// launch ray can only hit a triangle whose orthographic projection onto the
// rectangle's (u, v) plane contains the ray's (u, v) point.  cover_kernel
// projects every triangle onto the plane (fp32, relative to the scene's
// bounding-sphere centre), widens its 2-D bounding box by a margin far above
// every rounding involved (1e-5 R plus one cell on each side: the fp32
// projection errs by < 1e-6 R, the reference's fp64 Moller-Trumbore accepts
// at most ~1e-15 R outside the exact triangle), and sets the bits of the
// dispatch-index groups (2^cover_shift consecutive launch entries in the
// kernel's band order, trace.cu locate) whose cells meet the box.  A launch
// entry whose group bit is clear provably escapes: the path kernel retires it
// (one launched ray, one bounce-0 segment, exactly the reference's RunStats
// for a miss) without generating or tracing it.  Culling changes no hit, no
// contribution and no counter; it removes the ray generation and the BVH
// descent of rays that leave the scene untouched -- 87% of the c5 launch
// rays (nose-on airframe in its bounding aperture).
//
// Blocks (incidence, triangle slice) build the slice's bitmap of the
// incidence in shared memory (<= 64 KB: the group size grows past 32 entries
// only for incidences of more than 2^24 entries) and OR it into the
// incidence's bitmap in HBM.
#include <cstdint>

#include "internal.h"

namespace mcsbr_int {

namespace {

__global__ void tri32_kernel(const double* __restrict__ vtx, const uint4* __restrict__ tri, uint32_t n, double cx,
                             double cy, double cz, float* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint4 t = tri[i];
    const uint32_t v[3] = {t.x, t.y, t.z};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double* p = vtx + 3ull * v[k];
        out[9ull * i + 3 * k + 0] = __double2float_rn(p[0] - cx);
        out[9ull * i + 3 * k + 1] = __double2float_rn(p[1] - cy);
        out[9ull * i + 3 * k + 2] = __double2float_rn(p[2] - cz);
    }
}

__device__ __forceinline__ void set_range(uint32_t* bits, uint64_t g0, uint64_t g1) {
    const uint64_t w0 = g0 >> 5, w1 = g1 >> 5;
    for (uint64_t w = w0; w <= w1; ++w) {
        uint32_t m = 0xffffffffu;
        if (w == w0) m &= 0xffffffffu << (g0 & 31);
        if (w == w1) m &= 0xffffffffu >> (31 - (g1 & 31));
        atomicOr(bits + w, m);
    }
}

__global__ void __launch_bounds__(512) cover_kernel(const IncDev* __restrict__ incs, const float* __restrict__ tri32,
                                                    uint32_t n_tri, double cx, double cy, double cz, uint32_t spp,
                                                    uint32_t band, float margin, uint32_t* __restrict__ out) {
    extern __shared__ uint32_t sbits[];
    const IncDev& I = incs[blockIdx.x];
    if (I.cover_off == kNoCover) return;
    const uint32_t sh = I.cover_shift;
    const uint32_t nu = static_cast<uint32_t>(I.nu), nv = static_cast<uint32_t>(I.nv);
    const uint64_t entries = static_cast<uint64_t>(nu) * nv * spp;
    const uint64_t groups = (entries + (1ull << sh) - 1) >> sh;
    const uint32_t nwords = static_cast<uint32_t>((groups + 31) >> 5);
    for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x) sbits[w] = 0u;
    __syncthreads();
    // cell i spans u in [U0 + 2 hu i / nu, U0 + 2 hu (i + 1) / nu] relative to
    // the scene centre (the rectangle's centre is u (ulo + uhi) / 2 + k standoff)
    const double dcx = I.center[0] - cx, dcy = I.center[1] - cy, dcz = I.center[2] - cz;
    const double U0 = (dcx * I.u[0] + dcy * I.u[1] + dcz * I.u[2]) - I.half_u;
    const double V0 = (dcx * I.v[0] + dcy * I.v[1] + dcz * I.v[2]) - I.half_v;
    const float su = static_cast<float>(static_cast<double>(nu) / (2.0 * I.half_u));
    const float sv = static_cast<float>(static_cast<double>(nv) / (2.0 * I.half_v));
    const float u0 = static_cast<float>(U0), v0 = static_cast<float>(V0);
    const float ux = static_cast<float>(I.u[0]), uy = static_cast<float>(I.u[1]), uz = static_cast<float>(I.u[2]);
    const float vx = static_cast<float>(I.v[0]), vy = static_cast<float>(I.v[1]), vz = static_cast<float>(I.v[2]);
    const uint32_t bh = band ? band : 1u;
    // blockIdx.y of gridDim.y: this block's slice of the triangles
    const uint32_t t0 = static_cast<uint32_t>(static_cast<uint64_t>(n_tri) * blockIdx.y / gridDim.y);
    const uint32_t t1 = static_cast<uint32_t>(static_cast<uint64_t>(n_tri) * (blockIdx.y + 1) / gridDim.y);
    for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
        const float* p = tri32 + 9ull * t;
        float umin = 3e38f, umax = -3e38f, vmin = 3e38f, vmax = -3e38f;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float x = __ldg(p + 3 * k), y = __ldg(p + 3 * k + 1), z = __ldg(p + 3 * k + 2);
            const float pu = __fmaf_rn(x, ux, __fmaf_rn(y, uy, z * uz));
            const float pv = __fmaf_rn(x, vx, __fmaf_rn(y, vy, z * vz));
            umin = fminf(umin, pu);
            umax = fmaxf(umax, pu);
            vmin = fminf(vmin, pv);
            vmax = fmaxf(vmax, pv);
        }
        const float fi0 = (umin - margin - u0) * su, fi1 = (umax + margin - u0) * su;
        const float fj0 = (vmin - margin - v0) * sv, fj1 = (vmax + margin - v0) * sv;
        if (!(fi1 >= -1.0f && fi0 <= static_cast<float>(nu) + 1.0f && fj1 >= -1.0f &&
              fj0 <= static_cast<float>(nv) + 1.0f))
            continue;  // outside the aperture (or NaN)
        const int i0 = max(0, static_cast<int>(floorf(fmaxf(fi0, -2.0f))) - 1);
        const int i1 = min(static_cast<int>(nu) - 1, static_cast<int>(floorf(fminf(fi1, 2.0e9f))) + 1);
        const int j0 = max(0, static_cast<int>(floorf(fmaxf(fj0, -2.0f))) - 1);
        const int j1 = min(static_cast<int>(nv) - 1, static_cast<int>(floorf(fminf(fj1, 2.0e9f))) + 1);
        if (i0 > i1 || j0 > j1) continue;
        // band order (trace.cu locate): band b holds rows [bh b, bh b + h),
        // column-major inside the band, so the rectangle's cells of one band
        // are inside one contiguous dispatch range
        for (uint32_t b = static_cast<uint32_t>(j0) / bh; b <= static_cast<uint32_t>(j1) / bh; ++b) {
            const uint32_t h = min(bh, nv - bh * b);
            const uint64_t base = static_cast<uint64_t>(b) * bh * nu;
            const uint64_t cg0 = base + static_cast<uint64_t>(i0) * h;
            const uint64_t cg1 = base + static_cast<uint64_t>(i1) * h + (h - 1);
            set_range(sbits, (cg0 * spp) >> sh, (cg1 * spp + (spp - 1)) >> sh);
        }
    }
    __syncthreads();
    // merge the slice's bits (the bitmap was zeroed by the host)
    uint32_t* dst = out + I.cover_off;
    for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x)
        if (sbits[w]) atomicOr(dst + w, sbits[w]);
}

}  // namespace

cudaError_t build_tri32(const double* d_vtx, const uint4* d_tri, uint32_t n, const double center[3], float* out,
                        cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    tri32_kernel<<<(n + 255) / 256, 256, 0, stream>>>(d_vtx, d_tri, n, center[0], center[1], center[2], out);
    return cudaGetLastError();
}

uint32_t cover_shift_for(uint64_t entries) {
    uint32_t sh = 5;  // 32 entries per group: one warp's 8 x 4 patch of cells in band order
    while (((entries + (1ull << sh) - 1) >> sh) > kCoverMaxBits) ++sh;
    return sh;
}

cudaError_t launch_cover(const IncDev* d_inc, uint32_t n_inc, const float* tri32, uint32_t n_tri,
                         const double center[3], double radius, uint32_t spp, uint32_t band, uint32_t* out,
                         uint64_t out_words, int device_sms, cudaStream_t stream) {
    if (n_inc == 0) return cudaSuccess;
    cudaError_t z = cudaMemsetAsync(out, 0, sizeof(uint32_t) * out_words, stream);
    if (z != cudaSuccess) return z;
    // enough blocks to fill the GPU: triangle slices per incidence, each slice
    // at least 4096 triangles
    uint32_t slices = static_cast<uint32_t>(device_sms) * 2u / n_inc;
    slices = slices < 1u ? 1u : slices;
    const uint32_t max_slices = (n_tri + 4095u) / 4096u;
    slices = slices > max_slices ? max_slices : slices;
    slices = slices > 65535u ? 65535u : slices;
    const int smem = static_cast<int>(kCoverMaxBits / 8);
    cudaError_t e = cudaFuncSetAttribute(cover_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const float margin = static_cast<float>(1e-5 * radius);
    cover_kernel<<<dim3(n_inc, slices), 512, smem, stream>>>(d_inc, tri32, n_tri, center[0], center[1], center[2], spp,
                                                             band, margin, out);
    return cudaGetLastError();
}

}  // namespace mcsbr_int
