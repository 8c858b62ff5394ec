// K2/K3/K4: the persistent Monte Carlo SBR path kernel.
//
// Replaces the body of mcsbr::estimate (proj/src/solver_mc.cpp:105-210) and
// its callees.  One thread owns one path at a time; a warp pulls tiles of
// launch entries (all from one incidence) from a global atomic tile counter
// and refills lanes as their paths terminate (path regeneration), so the SIMT
// lanes stay busy even though path lengths differ.  Per lane and event:
//
//   closest hit (K2, fp32 conservative BVH2 descent + fp64 Moller-Trumbore in
//   the reference's arithmetic)  -> advance -> branch_outcomes (GO Fresnel /
//   PEC transport) -> MECA currents + contribution -> branch choice and
//   Russian roulette -> occlusion any-hit toward the receiver (K3) -> phasor
//   accumulation (K4).
//
// The wavefront order of the reference (all first hits of a block, then all
// second hits, ...) only changes the ORDER in which contributions are summed;
// every path's arithmetic is independent of it, which is why a depth-first
// per-thread path with a counter-based RNG keyed on (cell, sample, bounce)
// reproduces the reference's per-path events bit for bit.
//
// Accumulation (K4): F = 1 keeps the 4 channel phasor sums of the lane's
// current incidence in registers and reduces them across the warp (shuffles)
// once per tile before one fp64 atomicAdd per channel.  F > 1 stages a
// per-warp [F][4] complex accumulator in shared memory: each visible
// contribution is broadcast across the warp and lane l evaluates frequencies
// l, l+32, ... (fp64 phase, sincos) into its own slots, flushed with atomics
// once per tile.
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <type_traits>

#include "dmath.cuh"
#include "internal.h"
#include "physics.cuh"
#include "rng.cuh"
#include "mcsbr_gpu.h"

using namespace mcsbr_dev;

namespace mcsbr_int {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ V3 ld3(const double* p) { return {p[0], p[1], p[2]}; }

// ---------------------------------------------------------------------------
// K2/K3: traversal

struct FRay {
    float ix, iy, iz;     // 1/dir (fp32, zero components clamped)
    float onx, ony, onz;  // origin * inv + margin: near planes  (t = plane * inv - on)
    float ofx, ofy, ofz;  // origin * inv - margin: far planes
    float tlo;            // lower end of the box interval (0, or t_min rounded down)
    double t_skip;        // parameter of the traversal origin along the fp64 ray
    // byte offsets of the near-plane float4 of each axis inside a 128-byte
    // node (16 * a + 16 iff inv component < 0); the far plane is at ^ 16
    uint32_t offx, offy, offz;
};

// fp32 reciprocal of a direction component: MUFU.RCP plus one Newton step
// (relative error <= 2^-23, inside the 1.8e-7 the ray margin budgets for the
// rounded direction and its reciprocal; __frcp_rn's IEEE path cost ~2.5% of
// the kernel's stall samples); tiny components are clamped so no slab yields
// inf - inf.
__device__ __forceinline__ float safe_inv(double d) {
    const float f = __double2float_rn(d);
    const float a = fabsf(f) < 1e-12f ? copysignf(1e-12f, f) : f;
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    return __fmaf_rn(r, __fmaf_rn(-a, r, 1.0f), r);
}

// The fp32 boxes live in a frame centred on the scene's bounding sphere and
// are the fp64 triangle boxes rounded outward (no padding): they contain
// every triangle exactly.  The slab test's own rounding is covered by a
// margin on the RAY, in t units, widening every slab by m |inv| on both
// sides: m = 1e-6 R for rays that start on a surface (|origin| <= R in the
// box frame; with the fp32 origin off by <= 6e-8 R, 1/d off by a relative
// e <= 1.8e-7 and one rounding of origin * inv and of the fma, the slab
// distance is off by <= (1.2e-7 + 2e + 1.2e-7) R |inv| = 6e-7 R |inv|), and
// m = 1e-5 R for rays that start outside the bounding sphere, which are
// advanced (for the box tests only) to a conservative lower bound of their
// sphere entry so every fp32 coordinate is O(R).  Surface rays also cull by
// t_min: a box the ray leaves (margin included) before t_min holds no
// acceptable hit, which skips the flat-plate subtrees a reflected or
// occlusion ray starts in.  The fp64 triangle test always uses the untouched
// ray, so hits are exactly the reference's.
// `outside`: the origin may lie outside the bounding sphere (launch rays and
// the public intersect API); surface-to-surface and occlusion rays start on a
// triangle, inside the sphere, and skip the advance.
__device__ __forceinline__ FRay make_fray(const SceneView& S, V3 o, V3 d, bool outside, double t_min) {
    FRay r;
    const V3 c = {S.center[0], S.center[1], S.center[2]};
    const V3 oc = o - c;
    r.t_skip = 0.0;
    if (outside) {
        // (b - R' |d|) / |d|^2 = y (b y - R'), y = 1/|d| (rsqrt, ~1 ulp): the
        // advance only has to stay below the sphere entry, and R' = 1.01 R
        // leaves 0.01 R / |d| of slack for the rounding (|b| << 1e13 R)
        const double y = rsqrt(dot(d, d));
        const double b = -dot(oc, d);
        const double skip = y * (b * y - S.skip_radius);
        r.t_skip = skip > 0.0 ? skip : 0.0;
    }
    const V3 ot = oc + d * r.t_skip;
    r.ix = safe_inv(d.x);
    r.iy = safe_inv(d.y);
    r.iz = safe_inv(d.z);
    const float m = S.margin_r * (outside ? 1e-5f : 1e-6f);
    const float ox = __fmul_rn(__double2float_rn(ot.x), r.ix);
    const float oy = __fmul_rn(__double2float_rn(ot.y), r.iy);
    const float oz = __fmul_rn(__double2float_rn(ot.z), r.iz);
    const float ex = __fmul_ru(m, fabsf(r.ix)), ey = __fmul_ru(m, fabsf(r.iy)), ez = __fmul_ru(m, fabsf(r.iz));
    r.onx = __fadd_ru(ox, ex);
    r.ony = __fadd_ru(oy, ey);
    r.onz = __fadd_ru(oz, ez);
    r.ofx = __fadd_rd(ox, -ex);
    r.ofy = __fadd_rd(oy, -ey);
    r.ofz = __fadd_rd(oz, -ez);
    r.tlo = outside ? 0.0f : __double2float_rd(t_min * (1.0 - 1e-6));
    r.offx = r.ix < 0.0f ? 16u : 0u;
    r.offy = r.iy < 0.0f ? 48u : 32u;
    r.offz = r.iz < 0.0f ? 80u : 64u;
    return r;
}

// 3-input fp32 min / max (FMNMX3 on sm_100)
__device__ __forceinline__ float fmin3(float a, float b, float c) {
    float d;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// a * s + c for the pair (a0, a1): one FFMA2 (packed fp32x2, sm_100)
__device__ __forceinline__ float2 ffma2(float a0, float a1, float s, float c) {
    unsigned long long aa, ss, cc, d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(aa) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %1};" : "=l"(ss) : "f"(s));
    asm("mov.b64 %0, {%1, %1};" : "=l"(cc) : "f"(c));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(aa), "l"(ss), "l"(cc));
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(d));
    return r;
}

// Slab test with the near / far planes already chosen by the ray octant
// (the caller loads lo or hi per axis by address): entry = max of the near
// plane distances and tlo, exit = min of the far ones and tmax; returns the
// entry distance or +inf.
__device__ __forceinline__ float slab_nf(const FRay& r, float nx, float fx, float ny, float fy, float nz,
                                         float fz, float tmax) {
    const float tn = fmax3(__fmaf_rn(nx, r.ix, -r.onx), __fmaf_rn(ny, r.iy, -r.ony),
                           fmaxf(__fmaf_rn(nz, r.iz, -r.onz), r.tlo));
    const float tf = fmin3(__fmaf_rn(fx, r.ix, -r.ofx), __fmaf_rn(fy, r.iy, -r.ofy),
                           fminf(__fmaf_rn(fz, r.iz, -r.ofz), tmax));
    return tn <= tf ? tn : __int_as_float(0x7f800000);
}

// Moller-Trumbore in fp64, geometry.cpp:20-39 operation for operation.
// (Measured and rejected: an error-bounded conservative fp32 pre-filter in
// front of this test made the c2 sweep 13% slower; the fp64 pipe is not the
// limiter, dependent latency and register pressure are.)
// (e1 = b - a and e2 = c - a are stored precomputed: same IEEE values).
__device__ __forceinline__ bool tri_test(const double2* __restrict__ rec, V3 o, V3 d, double t_min,
                                         double& t_out, uint32_t& id_out) {
    const double2 r0 = __ldg(rec + 0), r1 = __ldg(rec + 1), r2 = __ldg(rec + 2), r3 = __ldg(rec + 3),
                  r4 = __ldg(rec + 4);
    const V3 a = {r0.x, r0.y, r1.x};
    const V3 e1 = {r1.y, r2.x, r2.y};
    const V3 e2 = {r3.x, r3.y, r4.x};
    const V3 p = cross(d, e2);
    const double det = dot(e1, p);
    if (fabs(det) < 1e-14) return false;
    const V3 s = o - a;
    const double un = dot(s, p);
    const V3 q = cross(s, e1);
    const double vn = dot(d, q);
    // Exact early outs that skip the fp64 divide.  With r = RN(1/det) and
    // u = RN(un * r):  a nonzero un of opposite sign to det gives u < 0 unless
    // the product underflows (|un| <= 1e-290 |det| excluded), and
    // |un| > |det| (1 + 1e-15) with the same sign gives u > 1 (two roundings
    // move the quotient by < 2^-52).  Same for v, and u + v > 1 when
    // un + vn exceeds det by a margin that covers all four roundings.
    // Only triangles the reference would reject are skipped here.
    const double adet = fabs(det);
    const double su = det < 0.0 ? -un : un, sv = det < 0.0 ? -vn : vn;
    if ((su < 0.0 && -su > adet * 1e-290) || su > adet * (1.0 + 1e-15)) return false;
    if ((sv < 0.0 && -sv > adet * 1e-290) || sv > adet * (1.0 + 1e-15)) return false;
    if (su > 0.0 && sv > 0.0 && su + sv > adet * (1.0 + 1e-13)) return false;
    const double inv_det = 1.0 / det;
    const double u = un * inv_det;
    if (u < 0.0 || u > 1.0) return false;
    const double v = vn * inv_det;
    if (v < 0.0 || u + v > 1.0) return false;
    const double t = dot(e2, q) * inv_det;
    if (t <= t_min || t >= 1e300) return false;
    t_out = t;
    id_out = static_cast<uint32_t>(__double_as_longlong(r4.y));
    return true;
}

// Closest hit (kAny = false): Scene::intersect semantics, geometry.cpp:177-216
// (nearest t > t_min, equal-t ties to the smallest triangle id).
// Any hit (kAny = true): Scene::occluded semantics, geometry.cpp:242-244.
// One runtime-flagged routine (not two template copies) so the path kernel
// has a single traversal loop in its instruction stream.
#ifdef MCSBR_TRAVERSAL_STATS
// diagnostic build only (tools/build_variants.py --stats): node visits,
// triangle tests and queries per query kind (0 launch rays, 1 surface
// closest-hit rays, 2 occlusion rays) in g_visits[3 * kind + {0, 1, 2}]
__device__ unsigned long long g_visits[9];
#define MCSBR_STAT(i) (++tstat[i])
#else
#define MCSBR_STAT(i) ((void)0)
#endif

__device__ __forceinline__ bool traverse(const SceneView& S, V3 o, V3 d, double t_min, double& best_t,
                                         uint32_t& best_id, uint32_t& fault, bool kAny, bool outside) {
#ifdef MCSBR_TRAVERSAL_STATS
    uint32_t tstat[2] = {0, 0};
    struct Flush {
        uint32_t* s;
        int kind;
        __device__ ~Flush() {
            atomicAdd(&g_visits[3 * kind], static_cast<unsigned long long>(s[0]));
            atomicAdd(&g_visits[3 * kind + 1], static_cast<unsigned long long>(s[1]));
            atomicAdd(&g_visits[3 * kind + 2], 1ull);
        }
    } flush_{tstat, kAny ? 2 : (outside ? 0 : 1)};
#endif
    const FRay r = make_fray(S, o, d, outside, t_min);
    best_t = __longlong_as_double(0x7ff0000000000000ll);
    best_id = 0xffffffffu;
    float tmax = __int_as_float(0x7f800000);
    int stack[kStackSize];
    int sp = 0;
    int ref = S.root_ref;
    for (;;) {
        if (ref >= 0) {
            // 4-wide node: 128 B, boxes SoA by axis (bvh.cu emit4_kernel)
            MCSBR_STAT(0);
            const float4* nd = S.nodes + 8ll * ref;
            // near planes at (lo | octant bit) per axis, far planes at the other;
            // unused child slots hold empty boxes (lo = +inf, hi = -inf) and
            // always miss, so no child count is needed
            // nodes are 128-byte aligned: plane addresses are node | offset
            // (near) and that ^ 16 (far), two logic ops per axis
            const uint64_t nb = reinterpret_cast<uint64_t>(nd);
            auto plane = [](uint64_t addr) { return __ldg(reinterpret_cast<const float4*>(addr)); };
            const float4 nx = plane(nb | r.offx), fx = plane((nb | r.offx) ^ 16u);
            const float4 ny = plane(nb | r.offy), fy = plane((nb | r.offy) ^ 16u);
            const float4 nz = plane(nb | r.offz), fz = plane((nb | r.offz) ^ 16u);
            const float4 rf = __ldg(nd + 6);
            // plane distances two children at a time (FFMA2): [k].x child k, .y child k + 1
            const float2 xn[2] = {ffma2(nx.x, nx.y, r.ix, -r.onx), ffma2(nx.z, nx.w, r.ix, -r.onx)};
            const float2 yn[2] = {ffma2(ny.x, ny.y, r.iy, -r.ony), ffma2(ny.z, ny.w, r.iy, -r.ony)};
            const float2 zn[2] = {ffma2(nz.x, nz.y, r.iz, -r.onz), ffma2(nz.z, nz.w, r.iz, -r.onz)};
            const float2 xf[2] = {ffma2(fx.x, fx.y, r.ix, -r.ofx), ffma2(fx.z, fx.w, r.ix, -r.ofx)};
            const float2 yf[2] = {ffma2(fy.x, fy.y, r.iy, -r.ofy), ffma2(fy.z, fy.w, r.iy, -r.ofy)};
            const float2 zf[2] = {ffma2(fz.x, fz.y, r.iz, -r.ofz), ffma2(fz.z, fz.w, r.iz, -r.ofz)};
            // sort keys: entry distance (>= 0, so its bits order like the
            // float) with the child slot in the low 2 bits; a miss is >= +inf
            uint32_t k[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int h = j >> 1;
                const float a_n = (j & 1) ? xn[h].y : xn[h].x, b_n = (j & 1) ? yn[h].y : yn[h].x;
                const float c_n = (j & 1) ? zn[h].y : zn[h].x;
                const float a_f = (j & 1) ? xf[h].y : xf[h].x, b_f = (j & 1) ? yf[h].y : yf[h].x;
                const float c_f = (j & 1) ? zf[h].y : zf[h].x;
                const float tn = fmax3(a_n, b_n, fmaxf(c_n, r.tlo));
                const float tf = fmin3(a_f, b_f, fminf(c_f, tmax));
                k[j] = ((tn <= tf ? __float_as_uint(tn) : 0x7f800000u) & ~3u) | static_cast<uint32_t>(j);
            }
            constexpr uint32_t kMiss = 0x7f800000u;
            const int rc[4] = {__float_as_int(rf.x), __float_as_int(rf.y), __float_as_int(rf.z),
                               __float_as_int(rf.w)};
            auto child = [&](uint32_t key) {
                const uint32_t j = key & 3u;
                return (j & 2u) ? ((j & 1u) ? rc[3] : rc[2]) : ((j & 1u) ? rc[1] : rc[0]);
            };
            const unsigned hm = (k[0] < kMiss ? 1u : 0u) | (k[1] < kMiss ? 2u : 0u) | (k[2] < kMiss ? 4u : 0u) |
                                (k[3] < kMiss ? 8u : 0u);
            if (hm && (hm & (hm - 1u)) == 0u) {  // exactly one child entered: no sort, no push
                ref = child(static_cast<uint32_t>(__ffs(hm) - 1));
                continue;
            }
            if (hm) {
                // sorting network (0,1)(2,3)(0,2)(1,3)(1,2) on the keys: integer min / max
#define MCSBR_KSWAP(a, b)               \
    {                                   \
        const uint32_t lo_ = min(a, b); \
        b = max(a, b);                  \
        a = lo_;                        \
    }
                MCSBR_KSWAP(k[0], k[1])
                MCSBR_KSWAP(k[2], k[3])
                MCSBR_KSWAP(k[0], k[2])
                MCSBR_KSWAP(k[1], k[3])
                MCSBR_KSWAP(k[1], k[2])
#undef MCSBR_KSWAP
                // visit the nearest now, push the others far-to-near (the
                // host bounds the tree depth so the stack cannot overflow)
                if (k[3] < kMiss) stack[sp++] = child(k[3]);
                if (k[2] < kMiss) stack[sp++] = child(k[2]);
                stack[sp++] = child(k[1]);  // at least two entered
                ref = child(k[0]);
                continue;
            }
        } else {
            const uint32_t code = static_cast<uint32_t>(~ref);
            const uint32_t first = code >> 3, count = code & 7u;
            for (uint32_t k = 0; k < count; ++k) {
                double t;
                uint32_t id;
                MCSBR_STAT(1);
                if (tri_test(S.tri64 + 5ull * (first + k), o, d, t_min, t, id)) {
                    if (t < best_t || (t == best_t && id < best_id)) {
                        best_t = t;
                        best_id = id;
                        if (kAny) return true;
                        tmax = __double2float_ru((t - r.t_skip) * (1.0 + 1e-9));
                    }
                }
            }
        }
        if (sp == 0) break;
        ref = stack[--sp];
    }
    return best_id != 0xffffffffu;
}

// fill_hit (geometry.cpp:164-175); NT = Cx adds Im(n) from S.mat_nim
template <typename NT>
struct HitInfo {
    V3 normal;
    NT n_incident, n_transmit;
    bool far_side_pec, exterior_facing, near_is_ambient;
};

template <typename NT>
__device__ __forceinline__ HitInfo<NT> fill_hit(const SceneView& S, uint32_t id, V3 dir) {
    const double2 ta = __ldg(S.tri_info + 2ull * id), tb = __ldg(S.tri_info + 2ull * id + 1);
    const uint64_t packed = static_cast<uint64_t>(__double_as_longlong(tb.y));
    const V3 nrm = {ta.x, ta.y, tb.x};
    const bool front = dot(dir, nrm) < 0.0;
    HitInfo<NT> h;
    h.normal = front ? nrm : -nrm;
    const uint32_t fm = static_cast<uint32_t>(packed & 0xffffu);
    const uint32_t bm = static_cast<uint32_t>((packed >> 16) & 0xffffu);
    const uint32_t near_id = front ? fm : bm, far_id = front ? bm : fm;
    const double2 nm = __ldg(S.mat + near_id), fr = __ldg(S.mat + far_id);
    const bool near_pec = nm.y != 0.0, far_pec = fr.y != 0.0;
    const double nim_near = S.mat_nim ? __ldg(S.mat_nim + near_id) : 0.0;
    const double nim_far = S.mat_nim ? __ldg(S.mat_nim + far_id) : 0.0;
    h.n_incident = near_pec ? make_nt<NT>(S.ambient_n, 0.0) : make_nt<NT>(nm.x, nim_near);
    h.far_side_pec = far_pec || near_pec;
    h.n_transmit = far_pec ? make_nt<NT>(0.0, 0.0) : make_nt<NT>(fr.x, nim_far);
    h.exterior_facing = ((packed >> 32) & 1u) != 0;
    h.near_is_ambient = near_id == 0;
    return h;
}

// ---------------------------------------------------------------------------
// per-path state (PathState, proj/include/mcsbr/path_engine.hpp:16-28)

// NT = double: the reference model; NT = Cx: complex optical path / index
// (lossy extension).  EF = CV3: complex transverse fields; EF = V3 on the
// PEC-only instantiation, where every field stays real: the initial
// polarisations are real and the PEC coefficients (-1, +1) are real, so the
// reference's complex arithmetic carries imaginary parts that are exactly
// +-0 and real parts equal to this real arithmetic operation for operation
// (x - (+-0) = x).  Outputs then agree with the reference under IEEE
// equality; only the sign of some exactly-zero imaginary parts can differ.
template <typename NT, typename EF = CV3>
struct Path {
    V3 origin, dir;
    EF e0, e1;
    NT phi;
    double prob, weight;
    NT medium_n;
    int bounce;
    uint32_t cell, sample;
    uint64_t entry;
    uint64_t key;  // counter_prefix(seed, cell, sample) or the Philox ray index
};

// Per-thread shared-memory slot (SoA: field f of thread t at base[f * 128 + t])
// for the state that is NOT needed while a ray is traversed: the two complex
// fields, phi / prob / weight / medium_n, a pending contribution and the
// phasor sums.  Only the ray itself stays in registers across a traversal,
// which removes the register spills (measured: ~15 G local sectors and
// ~55 GB of DRAM write-back per c2 launch when this state lived in
// registers under the 128-register budget).  Accesses go through a volatile
// pointer so the compiler re-reads the slot instead of keeping copies live.
constexpr int kSlotThreads = 128;
// Slot layout per instantiation (field indices in doubles).  kPec: every
// triangle has a PEC side, so a path never branches or leaves the ambient
// medium -- prob stays exactly 1.0 and medium_n the ambient index, and the
// two fields are not stored.  kLossy adds the imaginary parts; kRegAcc the
// register-mode phasor sums.  Every 8 KB of shared memory per block costs
// ~4-7% (measured) through the L1 capacity it takes: the PEC register-mode
// slot (real fields and amplitudes: 21 doubles) keeps a block at ~22 KB, so
// 4 blocks fit the 100 KB shared-memory carve-out and leave ~156 KB of L1.
template <bool kPec, bool kLossy, bool kRegAcc>
struct Layout {
    static constexpr int EW = kPec ? 3 : 6;  // doubles per field vector (real / complex)
    static constexpr int AW = kPec ? 1 : 2;  // doubles per projected amplitude
    static constexpr int E0 = 0, E1 = EW, Phi = 2 * EW, Weight = Phi + 1, Amp = Weight + 1;
    static constexpr int SPath = Amp + 4 * AW;
    static constexpr int Prob = SPath + 1, Medium = SPath + 2;   // !kPec only
    static constexpr int Im0 = kPec ? SPath + 1 : SPath + 3;
    static constexpr int PhiIm = Im0, MediumIm = Im0 + 1, SPathIm = Im0 + 2;  // kLossy only
    static constexpr int Acc = Im0 + (kLossy ? 3 : 0);       // kRegAcc only
    static constexpr int Fields = Acc + (kRegAcc ? 8 : 0);
    static constexpr bool pec = kPec;
};

struct Slot {
    volatile double* p;
    __device__ __forceinline__ double get(int f) const { return p[f * kSlotThreads]; }
    __device__ __forceinline__ void set(int f, double v) const { p[f * kSlotThreads] = v; }
    __device__ __forceinline__ Cx getc(int f) const { return {get(f), get(f + 1)}; }
    __device__ __forceinline__ void setc(int f, Cx v) const {
        set(f, v.re);
        set(f + 1, v.im);
    }
    __device__ __forceinline__ CV3 getv(int f) const { return {getc(f), getc(f + 2), getc(f + 4)}; }
    __device__ __forceinline__ void setv(int f, const CV3& v) const {
        setc(f, v.x);
        setc(f + 2, v.y);
        setc(f + 4, v.z);
    }
};

__device__ __forceinline__ void slot_setv(const Slot& sl, int f, const CV3& v) { sl.setv(f, v); }
__device__ __forceinline__ void slot_setv(const Slot& sl, int f, const V3& v) {
    sl.set(f, v.x);
    sl.set(f + 1, v.y);
    sl.set(f + 2, v.z);
}
__device__ __forceinline__ void slot_getv(const Slot& sl, int f, CV3& v) { v = sl.getv(f); }
__device__ __forceinline__ void slot_getv(const Slot& sl, int f, V3& v) { v = {sl.get(f), sl.get(f + 1), sl.get(f + 2)}; }
// projected amplitude ch of a pending contribution (real on the PEC path)
template <typename L>
__device__ __forceinline__ void slot_set_amp(const Slot& sl, int ch, Cx a) {
    if (L::pec) sl.set(L::Amp + ch, a.re);
    else sl.setc(L::Amp + 2 * ch, a);
}
template <typename L>
__device__ __forceinline__ Cx slot_get_amp(const Slot& sl, int ch) {
    if (L::pec) return {sl.get(L::Amp + ch), 0.0};
    return slot_get_amp<L>(sl, ch);
}

// EF helpers: a real vector as a field, the zero field, field norm
template <typename EF> __device__ __forceinline__ EF ef_real(V3 v);
template <> __device__ __forceinline__ CV3 ef_real<CV3>(V3 v) { return cvreal(v); }
template <> __device__ __forceinline__ V3 ef_real<V3>(V3 v) { return v; }
template <typename EF> __device__ __forceinline__ EF ef_zero();
template <> __device__ __forceinline__ CV3 ef_zero<CV3>() { return cvzero(); }
template <> __device__ __forceinline__ V3 ef_zero<V3>() { return {0.0, 0.0, 0.0}; }

__device__ __forceinline__ void slot_set_nt(const Slot& sl, int f, int fim, double v) {
    (void)fim;
    sl.set(f, v);
}
__device__ __forceinline__ void slot_set_nt(const Slot& sl, int f, int fim, Cx v) {
    sl.set(f, v.re);
    sl.set(fim, v.im);
}
template <typename NT>
__device__ __forceinline__ NT slot_get_nt(const Slot& sl, int f, int fim) {
    return make_nt<NT>(sl.get(f), std::is_same<NT, Cx>::value ? sl.get(fim) : 0.0);
}

template <typename L, typename NT, typename EF>
__device__ __forceinline__ void save_em(const Slot& sl, const Path<NT, EF>& s) {
    slot_setv(sl, L::E0, s.e0);
    slot_setv(sl, L::E1, s.e1);
    slot_set_nt(sl, L::Phi, L::PhiIm, s.phi);
    sl.set(L::Weight, s.weight);
    if (!L::pec) {
        sl.set(L::Prob, s.prob);
        slot_set_nt(sl, L::Medium, L::MediumIm, s.medium_n);
    }
}

template <typename L, typename NT, typename EF>
__device__ __forceinline__ void load_em(const Slot& sl, Path<NT, EF>& s, double ambient_n) {
    slot_getv(sl, L::E0, s.e0);
    slot_getv(sl, L::E1, s.e1);
    s.phi = slot_get_nt<NT>(sl, L::Phi, L::PhiIm);
    s.weight = sl.get(L::Weight);
    if (L::pec) {
        s.prob = 1.0;
        s.medium_n = make_nt<NT>(ambient_n, 0.0);
    } else {
        s.prob = sl.get(L::Prob);
        s.medium_n = slot_get_nt<NT>(sl, L::Medium, L::MediumIm);
    }
}

// real amplitudes (PEC path): am.im is 0, so (am * z) = (am.re z.re, am.re z.im)
// up to the sign of zero
template <int kAcc>
__device__ __forceinline__ void acc_add_real(const Slot& sl, const Cx am[4], Cx z) {
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {
        sl.set(kAcc + 2 * ch, sl.get(kAcc + 2 * ch) + am[ch].re * z.re);
        sl.set(kAcc + 2 * ch + 1, sl.get(kAcc + 2 * ch + 1) + am[ch].re * z.im);
    }
}

template <int kAcc>
__device__ __forceinline__ void acc_add(const Slot& sl, const Cx am[4], Cx z) {
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) sl.setc(kAcc + 2 * ch, sl.getc(kAcc + 2 * ch) + am[ch] * z);
}

template <typename NT, typename EF>
__device__ __forceinline__ double draw(const TraceParams& P, const Path<NT, EF>& s, uint64_t bounce,
                                       uint64_t purpose) {
    if (P.rng_mode == MCSBR_RNG_REFERENCE) return u53(counter_finish(s.key, bounce, purpose));
    return philox_uniform(P.seed, s.key, static_cast<uint32_t>(bounce), static_cast<uint32_t>(purpose));
}

// A launch entry located on the strata grid (solver_mc.cpp:117-125):
// entry = cell * spp + sample, cell = j * nu + i.
struct Entry {
    uint64_t entry;
    uint32_t cell, sample, i, j;
};

// Dispatch order -> launch entry.  Warps take consecutive dispatch indices d.
// Linear order: d is the entry itself.  Band order walks the strata grid in
// bands of 4 rows, column by column, so a warp's 32 lanes get an 8 x 4 patch
// of cells instead of a 32-cell line.  Both are bijections on
// [0, nu*nv*spp): every entry, RNG key and contribution is unchanged; only
// the order lanes take them in is.  32-bit index math (nu*nv < 2^32, like
// the cell index of the reference's keys).
__device__ __forceinline__ Entry locate(const TraceParams& P, const IncDev& I, uint64_t d) {
    uint32_t cg, smp = 0;
    if (P.spp == 1) {
        cg = static_cast<uint32_t>(d);
    } else {
        cg = static_cast<uint32_t>(d / P.spp);
        smp = static_cast<uint32_t>(d - static_cast<uint64_t>(cg) * P.spp);
    }
    const uint32_t nu = static_cast<uint32_t>(I.nu), nv = static_cast<uint32_t>(I.nv);
    Entry e;
    if (P.band_order) {
        const uint32_t bh = static_cast<uint32_t>(P.band_order);  // band height (rows)
        const uint32_t band = cg / (bh * nu);
        const uint32_t r = cg - band * bh * nu;
        const uint32_t h = min(bh, nv - bh * band);
        const uint32_t col = h == bh ? (r >> (31 - __clz(bh))) : r / h;  // bh is a power of two
        e.i = col;
        e.j = bh * band + (r - col * h);
    } else {
        e.j = cg / nu;
        e.i = cg - e.j * nu;
    }
    e.cell = e.j * nu + e.i;
    e.sample = smp;
    e.entry = static_cast<uint64_t>(e.cell) * P.spp + smp;
    return e;
}

// Launch-ray culling (cover.cu): is dispatch index d of incidence I in a
// group whose coverage bit is set?  (No bitmap: every entry is traced.)
__device__ __forceinline__ bool covered(const TraceParams& P, const IncDev& I, uint64_t d) {
    if (!P.cover || I.cover_off == kNoCover) return true;
    const uint64_t g = d >> I.cover_shift;
    return (__ldg(P.cover + I.cover_off + (g >> 5)) >> (g & 31)) & 1u;
}

// First dispatch index >= cursor (and < e_end) in a covered group, reading
// the bitmap a word (32 groups) at a time; warp-uniform.
__device__ __forceinline__ uint64_t skip_uncovered(const uint32_t* bits, uint32_t sh, uint64_t cursor,
                                                   uint64_t e_end) {
    while (cursor < e_end) {
        const uint64_t g = cursor >> sh;
        const uint32_t w = __ldg(bits + (g >> 5)) >> (g & 31);
        if (w) {
            const uint64_t ng = g + static_cast<uint64_t>(__ffs(w) - 1);
            return ng > g ? min(ng << sh, e_end) : cursor;
        }
        cursor = ((g | 31ull) + 1) << sh;
    }
    return e_end;
}

// sample_stratum + init_path (solver_mc.cpp:33-42, :117-125; path_engine.cpp:5-15)
template <typename NT, typename EF>
__device__ __forceinline__ void init_path(const TraceParams& P, const IncDev& I, uint32_t inc_idx,
                                          const Entry& en, Path<NT, EF>& s, const volatile double* rcp) {
    const uint32_t cell = en.cell, sample = en.sample, i = en.i, j = en.j;
    const uint64_t entry = en.entry;
    double ju = 0.5, jv = 0.5;
    if (P.rng_mode == MCSBR_RNG_REFERENCE) {
        s.key = counter_prefix(P.seed, cell, sample);
        if (P.jitter) {
            ju = u53(counter_finish(s.key, 0, kLaunchU));
            jv = u53(counter_finish(s.key, 0, kLaunchV));
        }
    } else {
        s.key = (static_cast<uint64_t>(inc_idx) << 40) | entry;
        if (P.jitter) {
            ju = philox_uniform(P.seed, s.key, 0, kLaunchU);
            jv = philox_uniform(P.seed, s.key, 0, kLaunchV);
        }
    }
    // -1 + 2 (i + ju) / nu, the quotient from the incidence's shared
    // reciprocals rcp[0], rcp[1] (div_by: identical to '/')
    const double pu = 2.0 * (static_cast<double>(i) + ju), pv = 2.0 * (static_cast<double>(j) + jv);
    bool ok = true;
    double qu = mcsbr_dev::div_by(pu, I.nu, rcp[0], ok), qv = mcsbr_dev::div_by(pv, I.nv, rcp[1], ok);
    if (!ok) {
        qu = pu / I.nu;
        qv = pv / I.nv;
    }
    const double su = -1.0 + qu;
    const double sv = -1.0 + qv;
    const V3 c = ld3(I.center), u = ld3(I.u), v = ld3(I.v);
    const V3 p = (c + u * (su * I.half_u)) + v * (sv * I.half_v);
    const V3 k = ld3(I.k_inc);
    s.origin = p;
    s.dir = k;
    s.e0 = ef_real<EF>(ld3(I.pol_v));
    s.e1 = ef_real<EF>(ld3(I.pol_h));
    s.phi = make_nt<NT>(P.scene.ambient_n * dot(k, p), 0.0);  // lossless ambient (validated)
    s.prob = 1.0;
    s.weight = 1.0;
    s.medium_n = make_nt<NT>(P.scene.ambient_n, 0.0);
    s.bounce = 0;
    s.cell = cell;
    s.sample = sample;
    s.entry = entry;
}

// receiver projection of one contribution (SweepAccumulator::add, farfield.cpp:106-128)
__device__ __forceinline__ void project(const RxDev& R, const CV3& aj0, const CV3& am0, const CV3& aj1,
                                        const CV3& am1, Cx amp[4]) {
    const V3 ks = ld3(R.k_s), rv = ld3(R.rx_v), rh = ld3(R.rx_h);
    const CV3 f0 = cross(ks, cross(ks, aj0)) + cross(ks, am0);
    const CV3 f1 = cross(ks, cross(ks, aj1)) + cross(ks, am1);
    amp[0] = dot(f0, rv);  // VV
    amp[3] = dot(f0, rh);  // HV
    amp[2] = dot(f1, rv);  // VH
    amp[1] = dot(f1, rh);  // HH
}

// real fields (PEC path): the same projection in real arithmetic
__device__ __forceinline__ void project(const RxDev& R, const V3& aj0, const V3& am0, const V3& aj1,
                                        const V3& am1, Cx amp[4]) {
    const V3 ks = ld3(R.k_s), rv = ld3(R.rx_v), rh = ld3(R.rx_h);
    const V3 f0 = cross(ks, cross(ks, aj0)) + cross(ks, am0);
    const V3 f1 = cross(ks, cross(ks, aj1)) + cross(ks, am1);
    amp[0] = {dot(f0, rv), 0.0};  // VV
    amp[3] = {dot(f0, rh), 0.0};  // HV
    amp[2] = {dot(f1, rv), 0.0};  // VH
    amp[1] = {dot(f1, rh), 0.0};  // HH
}

// PEC hits have no magnetic current (sc == 0): the k_s x m term of the
// projection is a zero vector and only flips signs of zeros, so it is skipped
__device__ __forceinline__ void project_pec(const RxDev& R, const V3& aj0, const V3& aj1, Cx amp[4]) {
    const V3 ks = ld3(R.k_s), rv = ld3(R.rx_v), rh = ld3(R.rx_h);
    const V3 f0 = cross(ks, cross(ks, aj0));
    const V3 f1 = cross(ks, cross(ks, aj1));
    amp[0] = {dot(f0, rv), 0.0};  // VV
    amp[3] = {dot(f0, rh), 0.0};  // HV
    amp[2] = {dot(f1, rv), 0.0};  // VH
    amp[1] = {dot(f1, rh), 0.0};  // HH
}

__device__ __forceinline__ void store_cv(double* p, const CV3& v) {
    p[0] = v.x.re; p[1] = v.x.im; p[2] = v.y.re; p[3] = v.y.im; p[4] = v.z.re; p[5] = v.z.im;
}
__device__ __forceinline__ void store_cv(double* p, const V3& v) {
    p[0] = v.x; p[1] = 0.0; p[2] = v.y; p[3] = 0.0; p[4] = v.z; p[5] = 0.0;
}

__device__ __forceinline__ double shfl_d(double v, int src) {
    return __shfl_sync(kFull, v, src);
}
__device__ __forceinline__ double shfl_nt(double v, int src) { return shfl_d(v, src); }
__device__ __forceinline__ Cx shfl_nt(Cx v, int src) { return {shfl_d(v.re, src), shfl_d(v.im, src)}; }
__device__ __forceinline__ V3 shfl_ef(const V3& v, int src) { return {shfl_d(v.x, src), shfl_d(v.y, src), shfl_d(v.z, src)}; }
__device__ __forceinline__ CV3 shfl_ef(const CV3& v, int src) {
    return {shfl_nt(v.x, src), shfl_nt(v.y, src), shfl_nt(v.z, src)};
}

// ---------------------------------------------------------------------------
// deterministic mode: per-thread branch stack in HBM, SoA over threads
// (field f, depth d of thread t at det_stack[(f * depth + d) * threads + t]) so
// that lanes pushing together write coalesced.  An entry is the reference's
// child PathState (solver_det.cpp:134-147) minus what is constant per root.

__device__ __forceinline__ double& det_at(const TraceParams& P, uint64_t t, int d, int f) {
    return P.det_stack[(static_cast<size_t>(f) * P.det_depth + d) * P.det_threads + t];
}

__device__ __forceinline__ void ef_store6(double* v, const CV3& e) {
    v[0] = e.x.re; v[1] = e.x.im; v[2] = e.y.re; v[3] = e.y.im; v[4] = e.z.re; v[5] = e.z.im;
}
__device__ __forceinline__ void ef_store6(double* v, const V3& e) {
    v[0] = e.x; v[1] = 0.0; v[2] = e.y; v[3] = 0.0; v[4] = e.z; v[5] = 0.0;
}
__device__ __forceinline__ void ef_load6(const double* v, CV3& e) { e = {{v[0], v[1]}, {v[2], v[3]}, {v[4], v[5]}}; }
__device__ __forceinline__ void ef_load6(const double* v, V3& e) { e = {v[0], v[2], v[4]}; }

template <typename NT, typename EF>
__device__ __forceinline__ void det_push(const TraceParams& P, uint64_t t, int d, V3 o, V3 dir, const EF& e0,
                                         const EF& e1, NT phi, NT n, int bounce) {
    double v[23] = {o.x, o.y, o.z, dir.x, dir.y, dir.z};
    ef_store6(v + 6, e0);
    ef_store6(v + 12, e1);
    v[18] = re_of(phi);
    v[19] = im_of(phi);
    v[20] = re_of(n);
    v[21] = im_of(n);
    v[22] = static_cast<double>(bounce);
#pragma unroll
    for (int f = 0; f < 23; ++f) det_at(P, t, d, f) = v[f];
}

template <typename NT, typename EF>
__device__ __forceinline__ void det_pop(const TraceParams& P, uint64_t t, int d, Path<NT, EF>& s) {
    double v[23];
#pragma unroll
    for (int f = 0; f < 23; ++f) v[f] = det_at(P, t, d, f);
    s.origin = {v[0], v[1], v[2]};
    s.dir = {v[3], v[4], v[5]};
    ef_load6(v + 6, s.e0);
    ef_load6(v + 12, s.e1);
    s.phi = make_nt<NT>(v[18], v[19]);
    s.medium_n = make_nt<NT>(v[20], v[21]);
    s.bounce = static_cast<int>(v[22]);
    s.prob = 1.0;
    s.weight = 1.0;
}

// norm(ComplexVec3) (em_math.hpp:91-93): sqrt(|x|^2 + |y|^2 + |z|^2)
__device__ __forceinline__ double cvnorm(const CV3& v) {
    return sqrt((v.x.re * v.x.re + v.x.im * v.x.im) + (v.y.re * v.y.re + v.y.im * v.y.im) +
                (v.z.re * v.z.re + v.z.im * v.z.im));
}
__device__ __forceinline__ double cvnorm(const V3& v) { return sqrt((v.x * v.x + v.y * v.y) + v.z * v.z); }

// add a lane's stack accounting for one reference block (solver_det.cpp:127-132)
__device__ __forceinline__ void det_flush(const TraceParams& P, uint64_t blk, uint64_t peak, uint64_t push) {
    if (blk == ~0ull || (peak == 0 && push == 0)) return;
    atomicAdd(P.det_blocks + 2 * blk, static_cast<unsigned long long>(peak));
    atomicAdd(P.det_blocks + 2 * blk + 1, static_cast<unsigned long long>(push));
}

// Add a warp's register-mode phasor sums (slot fields kAcc..kAcc+7) into
// incidence a's sums and clear them.  Fan mode: lane l owns receiver
// rx_index + l (nf == 1, no reduction); otherwise the warp reduces its 32
// lanes and lane 0 adds.  Out of line: it runs once per incidence change and
// its warp-collective shuffles would otherwise be inlined at every call site.
template <bool kFan, int kAcc>
__device__ __noinline__ void flush_sums(double* sums, uint32_t n_rx, uint32_t rx_index, volatile double* p,
                                        uint32_t a, int lane) {
    const Slot sl{p};
    if (kFan) {
        const uint32_t rx = rx_index + static_cast<uint32_t>(lane);
        if (rx < n_rx) {
            double* o = sums + (static_cast<size_t>(a) * n_rx + rx) * 8;
            for (int k = 0; k < 8; ++k) {
                const double v = sl.get(kAcc + k);
                if (v != 0.0) atomicAdd(o + k, v);
                sl.set(kAcc + k, 0.0);
            }
        }
        return;
    }
    double* out = sums + (static_cast<size_t>(a) * n_rx + rx_index) * 8;
    for (int k = 0; k < 8; ++k) {
        double v = sl.get(kAcc + k);
        sl.set(kAcc + k, 0.0);
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        if (lane == 0 && v != 0.0) atomicAdd(out + k, v);
    }
}

// e^{-j k_f s} for frequency f: on uniform grids the reference's phase
// (kph0 + f kdph) s (farfield.cpp:131-139), else k0[f] directly (:140-146)
template <typename NT>
__device__ __forceinline__ Cx freq_phasor(const TraceParams& P, uint32_t f, NT s) {
    if (P.uniform_f) {
        const double ph0 = P.kph0 * re_of(s), dph = P.kdph * re_of(s);
        const double la0 = -(P.kph0 * im_of(s)), dla = -(P.kdph * im_of(s));
        return polar_la(ph0 + static_cast<double>(f) * dph, la0 + static_cast<double>(f) * dla);
    }
    return phasor(P.k0[f], s);
}

constexpr int kRecD2 = 6;  // contribution record: 6 double2 = 96 B (amp[4], s, incidence)

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
//   kModeFan   a bistatic fan of up to 32 receivers per launch (P.rx_index is
//              the first), F = 1: lane l owns receiver rx_index + l; every
//              contribution is broadcast across the warp and each lane runs
//              its receiver's occlusion test and projection (a coherent
//              32-ray bundle from one exit point), so paths are traced once
//              per 32 receivers instead of once per receiver.
enum { kModeDefer = 0, kModeReg = 1, kModeFan = 2 };

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
template <int kMode, bool kDiel, bool kLossy, bool kDet>
__global__ void __launch_bounds__(128, (MinBlocks<kMode, kDiel, kLossy>::value)) path_kernel(TraceParams P) {
    constexpr bool kRegAcc = kMode != kModeDefer;
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
    // incidence containing global entry g: last a with g_begin[a] <= g
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
        if (kRegAcc && cur_a != 0xffffffffu)
            flush_sums<kMode == kModeFan, kFAcc>(P.sums, P.n_rx, P.rx_index, sl.p, cur_a, lane);
    };

    for (;;) {
        // ---- next sub-range (warp-uniform) ----
        if (q[0] >= q[1]) fetch();
        const uint64_t q0 = q[0], q1 = q[1];
        if (q0 >= q1) break;
        const uint32_t a = find_inc(q0);
        const IncDev& I = P.inc[a];
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
        const uint32_t my_rx = P.rx_index + (kMode == kModeFan ? static_cast<uint32_t>(lane) : 0u);
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
                if (!kDet && P.cover && I.cover_off != kNoCover) {
                    const uint64_t c2 = skip_uncovered(P.cover + I.cover_off, I.cover_shift, cursor, e_end);
                    if (lane == 0) n_miss0 += c2 - cursor;  // warp-uniform run, counted once
                    cursor = c2;
                    if (cursor >= e_end) continue;
                }
                const unsigned rank = __popc(need & ((1u << lane) - 1u));
                const uint64_t mine = cursor + rank;
                if (!alive && mine < e_end) {
                    if (!kDet && !covered(P, I, mine)) {
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
                hit = traverse(S, s.origin, pend ? ld3(R.k_s) : s.dir,
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
                            EF f0 = ef_zero<EF>(), f1 = ef_zero<EF>();  // e_r (sc 1) / e_t (sc 2)
                            if (sc != 0) {
                                if constexpr (kDet) {
                                    f0 = ex ? et0 : er0;
                                    f1 = ex ? et1 : er1;
                                } else {
                                    f0 = branch_field(s.e0, ex ? 1 : 0, co, b);
                                    f1 = branch_field(s.e1, ex ? 1 : 0, co, b);
                                }
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
                            if (kMode == kModeFan) {
                                fj0 = j0;
                                fm0 = m0;
                                fj1 = j1;
                                fm1 = m1;
                                fphi = s.phi;
                                fpt = point;
                            } else {
                                if constexpr (L::pec) project_pec(R, j0, j1, amp);  // m = 0 on PEC hits
                                else project(R, j0, m0, j1, m1, amp);
                                s_path = s.phi - dot(ld3(R.k_s), point);
                            }
                            if (scratch) {
                                store_cv(&scratch->a_j[0][0][0], j0);
                                store_cv(&scratch->a_m[0][0][0], m0);
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
                if (candidate && kMode == kModeFan) {
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
            if (kMode == kModeFan) {
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
                            vis = !traverse(S, pt, ks, S.t_eps, t2, id2, fault, true, false);
                        }
                        if (vis) {
                            ++n_contrib;
                            acc_add<kFAcc>(sl, am, phasor(P.k0[0], sp));
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
                    if (stored) {
                        double2* r = reinterpret_cast<double2*>(P.recs) + slot * kRecD2;
#pragma unroll
                        for (int ch = 0; ch < 4; ++ch) r[ch] = make_double2(amp[ch].re, amp[ch].im);
                        r[4] = make_double2(re_of(s_path), im_of(s_path));
                        r[5] = make_double2(__longlong_as_double(static_cast<long long>(a)), 0.0);
                    }
                    // buffer full (the host sizes it so this is rare): the warp
                    // adds each overflowing contribution straight into the sums,
                    // lanes over frequencies
                    unsigned om = __ballot_sync(kFull, visible && !stored);
                    double* out = P.sums + (static_cast<size_t>(a) * P.n_rx + P.rx_index) * P.nf * 8;
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
                                atomicAdd(out + f * 8 + 2 * ch, v.re);
                                atomicAdd(out + f * 8 + 2 * ch + 1, v.im);
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
    if (!kDet && n_miss0) atomicAdd(&s_bounce[0], static_cast<unsigned int>(n_miss0));
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
template <int FPL, bool kRealAmp>
__global__ void __launch_bounds__(128) accumulate_kernel(TraceParams P, uint32_t f_begin) {
    // staged record: [0..3] amplitudes, [4] (ph0, dph) | s, [5] (la0, dla),
    // [6] W = e^{-j 32 dk s}, [7] incidence.  (Measured and rejected: a
    // per-record table of w^r, w^4q replacing the lane's sincos by two
    // complex multiplies -- c5 +3.5%, the table doubles the shared memory.)
    constexpr int kSt = 8;
    __shared__ double2 st[4][32][kSt];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t n_all = *P.rec_count;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicMax(P.rec_count + 1, n_all);  // peak for the host
    const uint64_t n = min(n_all, P.rec_cap);
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * 4, gw = static_cast<uint64_t>(blockIdx.x) * 4 + warp;
    uint64_t span = ((n + nw - 1) / nw + 31) & ~31ull;
    span = span < 512 ? 512 : span;
    const uint32_t f_end = min(P.nf, f_begin + 32u * FPL);
    const uint32_t f0 = f_begin + static_cast<uint32_t>(lane);
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
            double* out = P.sums + (static_cast<size_t>(cur) * P.n_rx + P.rx_index) * P.nf * 8;
#pragma unroll
            for (int m = 0; m < FPL; ++m) {
                const uint32_t f = f0 + 32u * m;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (f < f_end && acc[m][k] != 0.0) atomicAdd(out + f * 8 + k, acc[m][k]);
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
                if (P.uniform_f) {
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
                if (f0 >= f_end) continue;
                Cx z, w = {1.0, 0.0};
                const double2 t4 = t[4];
                if (P.uniform_f) {
                    const double2 t5 = t[5];
                    z = polar_la(t4.x + static_cast<double>(f0) * t4.y, t5.x + static_cast<double>(f0) * t5.y);
                    if (FPL > 1) w = cx2(t[6]);
                } else {
                    z = phasor(P.k0[f0], Cx{t4.x, t4.y});
                }
                Cx am[4];
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) am[ch] = cx2(t[ch]);
#pragma unroll
                for (int m = 0; m < FPL; ++m) {
                    const uint32_t f = f0 + 32u * m;
                    if (f < f_end) {
#pragma unroll
                        for (int ch = 0; ch < 4; ++ch) {
                            if (kRealAmp) {  // PEC scenes: the amplitudes are real
                                acc[m][2 * ch] = __fma_rn(am[ch].re, z.re, acc[m][2 * ch]);
                                acc[m][2 * ch + 1] = __fma_rn(am[ch].re, z.im, acc[m][2 * ch + 1]);
                            } else {
                                acc[m][2 * ch] =
                                    __fma_rn(am[ch].re, z.re, __fma_rn(-am[ch].im, z.im, acc[m][2 * ch]));
                                acc[m][2 * ch + 1] =
                                    __fma_rn(am[ch].re, z.im, __fma_rn(am[ch].im, z.re, acc[m][2 * ch + 1]));
                            }
                        }
                        if (m + 1 < FPL && f + 32u < f_end) {
                            if (P.uniform_f) z = cmul(z, w);
                            else z = phasor(P.k0[f + 32u], Cx{t4.x, t4.y});
                        }
                    }
                }
            }
            __syncwarp();
        }
        flush();
    }
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

bool trace_uses_register_accumulator(const TraceParams& p) { return p.nf == 1; }

bool trace_fan_supported(uint32_t nf) { return nf == 1; }

template <int kMode, bool kDiel, bool kLossy, bool kDet>
static cudaError_t launch_mode(const TraceParams& p, int device_sms, int threads, size_t smem,
                               cudaStream_t stream) {
    auto* k = path_kernel<kMode, kDiel, kLossy, kDet>;
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
        return mode == kModeReg ? launch_mode<kModeReg, kDiel, kLossy, true>(p, sms, threads, smem, stream)
                                : launch_mode<kModeDefer, kDiel, kLossy, true>(p, sms, threads, smem, stream);
    return mode == kModeFan   ? launch_mode<kModeFan, kDiel, kLossy, false>(p, sms, threads, smem, stream)
           : mode == kModeReg ? launch_mode<kModeReg, kDiel, kLossy, false>(p, sms, threads, smem, stream)
                              : launch_mode<kModeDefer, kDiel, kLossy, false>(p, sms, threads, smem, stream);
}

// deferred accumulation of one path-kernel launch's records (F > 1)
cudaError_t launch_accumulate(const TraceParams& p, int device_sms, cudaStream_t stream, uint64_t* launches) {
    const unsigned blocks = static_cast<unsigned>(device_sms) * 4;
    const uint32_t fpl = p.nf <= 32 ? 1 : (p.nf <= 64 ? 2 : 4);
    const bool real_amp = p.scene.all_pec && !p.scene.lossy;  // PEC paths carry real amplitudes
    for (uint32_t fb = 0; fb < p.nf; fb += 32 * fpl) {
        if (real_amp) {
            if (fpl == 1) accumulate_kernel<1, true><<<blocks, 128, 0, stream>>>(p, fb);
            else if (fpl == 2) accumulate_kernel<2, true><<<blocks, 128, 0, stream>>>(p, fb);
            else accumulate_kernel<4, true><<<blocks, 128, 0, stream>>>(p, fb);
        } else {
            if (fpl == 1) accumulate_kernel<1, false><<<blocks, 128, 0, stream>>>(p, fb);
            else if (fpl == 2) accumulate_kernel<2, false><<<blocks, 128, 0, stream>>>(p, fb);
            else accumulate_kernel<4, false><<<blocks, 128, 0, stream>>>(p, fb);
        }
        if (launches) ++*launches;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_trace(const TraceParams& p, int device_sms, cudaStream_t stream, uint64_t* launches) {
    const int threads = 128;
    const int mode = (p.fan && !p.det) ? kModeFan : (trace_uses_register_accumulator(p) ? kModeReg : kModeDefer);
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
