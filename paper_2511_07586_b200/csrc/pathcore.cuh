// Device building blocks shared by the persistent path kernel (trace.cu) and
// the wavefront kernels (wavefront.cu): traversal (K2/K3), hit filling, path
// state and its shared-memory slot, launch-entry location and coverage
// culling, init_path, receiver projection, accumulation helpers.
// Included inside `namespace mcsbr_int { namespace { ... } }` by each TU.
#pragma once

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

// Statistical-mode fast path (mcsbr_mc_config.parity_fp64_refine = 0): the
// triangle tests run in fp32 on leaf-ordered fp32 records (vertex a relative
// to the scene centre, e1, e2, id and two error numerators; 48 B instead of
// the fp64 record's 80 B) with the ray's origin advanced into the bounding
// sphere, so every operand is O(R).  The fp32 test only classifies: a hit
// or miss by more than its rounding bound (prep.cu leaf32_kernel: K / |det|
// on u, v, u + v and t) is taken as is; anything within the bound of an edge,
// of t_min, or of a degenerate det is decided by the fp64 test of that
// triangle.  Edge and self-hit decisions are therefore the fp64 test's (no
// cracks between neighbours, no re-hit of the origin triangle); only
// near-ties in t between two clear hits can resolve differently from the
// reference, and the closest hit's t is refined in fp64.  Statistical mode
// only (the host rejects it with the parity RNG stream).
// Measured (r02, Philox stream, path kernel): c4 2.68-2.96 ms fp64 vs
// 3.32-3.76 ms here, c5 (4 azimuths) 17.1-17.3 vs 20.4-20.6 ms; without the
// final fp64 refine 3.52-4.09 / 19.3-19.5 ms.  The fp64 test with its exact
// early outs is not the limiter, so the switch exists
// for the API and is off by default.
constexpr int kTri32Miss = 0, kTri32Hit = 1, kTri32Maybe = 2;
__device__ __forceinline__ int tri_test32(const float4* __restrict__ rec, float ox, float oy, float oz, float dx,
                                          float dy, float dz, float t_min, float& t_out, uint32_t& id_out) {
    const float4 r0 = __ldg(rec), r1 = __ldg(rec + 1), r2 = __ldg(rec + 2);
    const float ax = r0.x, ay = r0.y, az = r0.z, e1x = r0.w, e1y = r1.x, e1z = r1.y, e2x = r1.z, e2y = r1.w,
                e2z = r2.x;
    const float px = dy * e2z - dz * e2y, py = dz * e2x - dx * e2z, pz = dx * e2y - dy * e2x;
    const float det = e1x * px + e1y * py + e1z * pz;
    float inv;  // MUFU.RCP (its ~1 ulp is inside the 8x margin); det = 0 or nan: tol is inf / nan
    asm("rcp.approx.f32 %0, %1;" : "=f"(inv) : "f"(det));
    const float tol = r2.z * fabsf(inv);
    if (!(tol < 0.25f)) return kTri32Maybe;
    const float sx = ox - ax, sy = oy - ay, sz = oz - az;
    const float u = (sx * px + sy * py + sz * pz) * inv;
    if (u < -tol || u > 1.0f + tol) return kTri32Miss;
    const float qx = sy * e1z - sz * e1y, qy = sz * e1x - sx * e1z, qz = sx * e1y - sy * e1x;
    const float v = (dx * qx + dy * qy + dz * qz) * inv;
    if (v < -tol || u + v > 1.0f + 2.0f * tol) return kTri32Miss;
    const float t = (e2x * qx + e2y * qy + e2z * qz) * inv;
    const float ttol = r2.w * fabsf(inv);
    if (t <= t_min - ttol) return kTri32Miss;
    id_out = __float_as_uint(r2.y);
    if (u < tol || v < tol || u + v > 1.0f - 2.0f * tol || t <= t_min + ttol) return kTri32Maybe;
    t_out = t;
    return kTri32Hit;
}

template <bool kFastTri = false>
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
    // fast path: the ray in fp32, relative to the scene centre, from the
    // box tests' advanced origin (t measured from t_skip)
    float of[3] = {0.f, 0.f, 0.f}, df[3] = {0.f, 0.f, 0.f}, tmin32 = 0.f;
    uint32_t best_slot = 0xffffffffu;  // the closest hit if it came from a clear fp32 test
    if constexpr (kFastTri) {
        of[0] = __double2float_rn(o.x - S.center[0] + d.x * r.t_skip);
        of[1] = __double2float_rn(o.y - S.center[1] + d.y * r.t_skip);
        of[2] = __double2float_rn(o.z - S.center[2] + d.z * r.t_skip);
        df[0] = __double2float_rn(d.x);
        df[1] = __double2float_rn(d.y);
        df[2] = __double2float_rn(d.z);
        tmin32 = __double2float_rn(t_min - r.t_skip);
    }
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
                MCSBR_STAT(1);
                if constexpr (kFastTri) {
                    float t32;
                    uint32_t id;
                    const int c = tri_test32(S.tri32 + 3ull * (first + k), of[0], of[1], of[2], df[0], df[1], df[2],
                                             tmin32, t32, id);
                    if (c == kTri32Miss) continue;
                    double t;
                    if (c == kTri32Maybe) {
                        if (!tri_test(S.tri64 + 5ull * (first + k), o, d, t_min, t, id)) continue;
                    } else {
                        t = r.t_skip + static_cast<double>(t32);
                    }
                    if (t < best_t || (t == best_t && id < best_id)) {
                        best_t = t;
                        best_id = id;
                        best_slot = c == kTri32Hit ? first + k : 0xffffffffu;
                        if (kAny) return true;
                        tmax = __double2float_ru((t - r.t_skip) * (1.0 + 1e-5));
                    }
                } else {
                    double t;
                    uint32_t id;
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
        }
        if (sp == 0) break;
        ref = stack[--sp];
    }
    if constexpr (kFastTri) {
        if (best_slot != 0xffffffffu) {  // the winner's t in fp64 (kept from fp32 if fp64 rejects it)
            double t;
            uint32_t id;
            if (tri_test(S.tri64 + 5ull * best_slot, o, d, t_min, t, id)) best_t = t;
        }
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

// one polarisation of project(): (VV, HV) from (j0, m0), (VH, HH) from (j1, m1)
__device__ __forceinline__ void project_pol(const RxDev& R, const CV3& aj, const CV3& am, Cx& a_v, Cx& a_h) {
    const V3 ks = ld3(R.k_s);
    const CV3 f = cross(ks, cross(ks, aj)) + cross(ks, am);
    a_v = dot(f, ld3(R.rx_v));
    a_h = dot(f, ld3(R.rx_h));
}
__device__ __forceinline__ void project_pol(const RxDev& R, const V3& aj, const V3& am, Cx& a_v, Cx& a_h) {
    const V3 ks = ld3(R.k_s);
    const V3 f = cross(ks, cross(ks, aj)) + cross(ks, am);
    a_v = {dot(f, ld3(R.rx_v)), 0.0};
    a_h = {dot(f, ld3(R.rx_h)), 0.0};
}
__device__ __forceinline__ void project_pec_pol(const RxDev& R, const V3& aj, Cx& a_v, Cx& a_h) {
    const V3 ks = ld3(R.k_s);
    const V3 f = cross(ks, cross(ks, aj));
    a_v = {dot(f, ld3(R.rx_v)), 0.0};
    a_h = {dot(f, ld3(R.rx_h)), 0.0};
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

// Append contribution record `slot`: the four projected amplitudes, the net
// optical path and its row (an incidence of the launch, or a fan row, see
// sums_row), plus the row again in the packed array the NUFFT buckets read.
// Streaming stores (evict-first): the records are read once, by the
// accumulation, and should not displace the BVH and the local-memory lines
// from L2 (c5 -0.8% against plain stores).
template <typename NT>
__device__ __forceinline__ void write_record(const TraceParams& P, uint64_t slot, const Cx (&amp)[4], NT s,
                                             uint32_t row) {
    double2* r = reinterpret_cast<double2*>(P.recs) + slot * kRecD2;
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) __stcs(r + ch, make_double2(amp[ch].re, amp[ch].im));
    __stcs(r + 4, make_double2(re_of(s), im_of(s)));
    __stcs(r + 5, make_double2(__longlong_as_double(static_cast<long long>(row)), 0.0));
    if (P.rec_inc) __stcs(P.rec_inc + slot, row);
}

// Record-buffer overflow: one term added straight into the sums -- an fp64
// atomic, or under MCSBR_REDUCE_EXACT the term rounded once to 192-bit fixed
// point (fixedpoint.cuh) and added with carries into P.xsums (the same value
// accumulate_exact_kernel adds for a stored record, so the integer sums stay
// exact).  `out` is this incidence's block of P.sums, k the value's index in it.
__device__ __forceinline__ void add_value(const TraceParams& P, double* out, uint32_t k, double v) {
    if (!P.xsums) {
        atomicAdd(out + k, v);
        return;
    }
    uint64_t w[3];
    if (!mcsbr_fx::fx_from_double(v, w))
        atomicOr(P.counters + kCntFault, static_cast<unsigned long long>(kFaultFixedRange));
    mcsbr_fx::fx_atomic_add(P.xsums + ((out - P.sums) + k) * 3, w);
}

// Fan record that did not fit the buffer (the host sizes it so this is
// rare): the lane adds it straight into its receiver's sums, every
// frequency.
template <typename NT>
__device__ __forceinline__ void fan_record_overflow(const TraceParams& P, uint32_t row, const Cx (&am)[4], NT sp) {
    double* out = P.sums + sums_row(P, row) * P.nf * 8;
    for (uint32_t f = 0; f < P.nf; ++f) {
        const Cx z = freq_phasor(P, f, sp);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
            const Cx v = am[ch] * z;
            add_value(P, out, f * 8 + 2 * ch, v.re);
            add_value(P, out, f * 8 + 2 * ch + 1, v.im);
        }
    }
}

