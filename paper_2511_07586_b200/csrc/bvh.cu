// K1: BVH builder on the GPU (replaces Scene::build_bvh, proj/src/geometry.cpp:68-144,
// a single-threaded fp64 median split).
//
//   1. prim_kernel      per triangle: fp64 AABB padded by box_pad and rounded
//                       outward to fp32; 63-bit Morton code of the centroid.
//   2. radix sort       (morton, id) pairs, stable (sort.cu).
//   3. sah_build_kernel binned-SAH top-down build from the Morton order, one
//                       persistent launch: block tasks for nodes of > 32
//                       triangles, one warp per smaller subtree (default);
//                       fallback / MCSBR_BVH=lbvh:
//      karras_kernel    Karras (HPG 2012) binary radix tree over the sorted codes
//                       (ties broken by sort position), one thread per inner node.
//   4. refit_kernel     bottom-up AABB union with one atomic flag per inner node.
//   5. parity/scan/emit4  collapse to a 4-wide BVH: every inner node at even
//                       depth becomes a 128-B node holding its grandchildren's
//                       boxes (SoA by axis); any subtree holding <= 4
//                       triangles becomes a leaf reference to its contiguous
//                       sorted range (the LBVH ranges are contiguous).
//   6. tri_kernel       leaf-ordered fp64 triangle records (a, e1, e2, id).
//
// Exactness: the tree only culls.  Boxes are conservative (outward rounding
// + padding), the triangle test that decides hits runs in fp64 with the
// reference's arithmetic, so closest hits equal brute force
// (Scene::intersect_brute_force, geometry.cpp:218-240) for ANY tree shape.

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace mcsbr_int {

namespace {

__device__ __forceinline__ uint64_t expand21(uint64_t v) {
    v &= 0x1fffff;
    v = (v | v << 32) & 0x1f00000000ffffull;
    v = (v | v << 16) & 0x1f0000ff0000ffull;
    v = (v | v << 8) & 0x100f00f00f00f00full;
    v = (v | v << 4) & 0x10c30c30c30c30c3ull;
    v = (v | v << 2) & 0x1249249249249249ull;
    return v;
}

struct Box {
    float lo[3], hi[3];
};

// Early split clipping (Ernst & Greiner, RT 2007): a sliver triangle whose
// bounding box is much larger than the triangle itself (the long thin fan
// triangles of a capped cylinder, a wing-tip cap, ...) makes every ray near
// it descend to its leaf.  Such a triangle is referenced by k pieces: its
// box is cut into k equal slabs along the longest axis, and piece j's box is
// the bounding box of the triangle clipped to slab j (fp64, then padded and
// rounded outward like every other box).  The pieces' boxes cover the
// triangle, every piece's leaf record is the WHOLE triangle (same fp64
// record, same id), so closest hits and any-hit answers are unchanged: a
// duplicate test returns the identical (t, id) and never replaces the best
// hit.  Criterion: box surface area > kEscRatio x twice the triangle's area;
// k = ceil(ratio / kEscTarget) <= kEscMaxPieces.  Well-shaped meshes (the
// icospheres, the dihedral plates) have ratios <= ~5 and are not split.
#ifndef MCSBR_ESC_RATIO
#define MCSBR_ESC_RATIO 16.0
#endif
#ifndef MCSBR_ESC_TARGET
#define MCSBR_ESC_TARGET 4.0
#endif
constexpr double kEscRatio = MCSBR_ESC_RATIO;
constexpr double kEscTarget = MCSBR_ESC_TARGET;
constexpr uint32_t kEscMaxPieces = 64;

struct EscInfo {
    uint32_t pieces;
    int axis;
    double lo, hi;  // the triangle's extent along `axis`
};

__device__ __forceinline__ EscInfo esc_info(const double* a, const double* b, const double* c) {
    double lo[3], hi[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        lo[k] = fmin(a[k], fmin(b[k], c[k]));
        hi[k] = fmax(a[k], fmax(b[k], c[k]));
    }
    const double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
    const double sa = 2.0 * (dx * dy + dy * dz + dz * dx);
    const double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
    const double e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
    const double cx = e1[1] * e2[2] - e1[2] * e2[1], cy = e1[2] * e2[0] - e1[0] * e2[2],
                 cz = e1[0] * e2[1] - e1[1] * e2[0];
    const double a2 = sqrt(cx * cx + cy * cy + cz * cz);  // twice the area
    EscInfo r;
    r.axis = dx >= dy && dx >= dz ? 0 : (dy >= dz ? 1 : 2);
    r.lo = lo[r.axis];
    r.hi = hi[r.axis];
    r.pieces = 1;
    if (a2 > 0.0 && sa > kEscRatio * a2)
        r.pieces = static_cast<uint32_t>(fmin(ceil(sa / (kEscTarget * a2)), static_cast<double>(kEscMaxPieces)));
    return r;
}

__global__ void esc_count_kernel(const double* __restrict__ vtx, const uint4* __restrict__ tri, uint32_t n,
                                 uint32_t* __restrict__ extra) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint4 t = tri[i];
    extra[i] = esc_info(vtx + 3ull * t.x, vtx + 3ull * t.y, vtx + 3ull * t.z).pieces - 1;
}

// reference r -> (triangle, piece): piece 0 of triangle t is reference t,
// pieces 1.. follow after the n triangles at the scanned offsets
__global__ void esc_refs_kernel(const uint32_t* __restrict__ extra, const uint32_t* __restrict__ off, uint32_t n,
                                uint32_t* __restrict__ ref_tri, uint32_t* __restrict__ ref_piece) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    ref_tri[i] = i;
    ref_piece[i] = 0;
    for (uint32_t j = 1; j <= extra[i]; ++j) {
        ref_tri[n + off[i] + j - 1] = i;
        ref_piece[n + off[i] + j - 1] = j;
    }
}

// bounding box of the triangle (a, b, c) clipped to lo_s <= p[axis] <= hi_s
// (Sutherland-Hodgman against the two planes)
__device__ void clip_box(const double* a, const double* b, const double* c, int axis, double lo_s, double hi_s,
                         double bl[3], double bh[3]) {
    double P[8][3], Q[8][3];
    int n = 3;
    for (int k = 0; k < 3; ++k) {
        P[0][k] = a[k];
        P[1][k] = b[k];
        P[2][k] = c[k];
    }
    for (int side = 0; side < 2; ++side) {
        const double s = side ? hi_s : lo_s;
        int m = 0;
        for (int i = 0; i < n; ++i) {
            const double* u = P[i];
            const double* v = P[(i + 1) % n];
            const bool ui = side ? u[axis] <= s : u[axis] >= s;
            const bool vi = side ? v[axis] <= s : v[axis] >= s;
            if (ui) {
                for (int k = 0; k < 3; ++k) Q[m][k] = u[k];
                ++m;
            }
            if (ui != vi) {
                const double w = (s - u[axis]) / (v[axis] - u[axis]);
                for (int k = 0; k < 3; ++k) Q[m][k] = u[k] + (v[k] - u[k]) * w;
                Q[m][axis] = s;
                ++m;
            }
        }
        n = m;
        for (int i = 0; i < n; ++i)
            for (int k = 0; k < 3; ++k) P[i][k] = Q[i][k];
    }
    for (int k = 0; k < 3; ++k) {
        bl[k] = 1e300;
        bh[k] = -1e300;
    }
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) {
            bl[k] = fmin(bl[k], P[i][k]);
            bh[k] = fmax(bh[k], P[i][k]);
        }
    if (n == 0) {  // rounding left nothing: the slab of the triangle's box (conservative)
        for (int k = 0; k < 3; ++k) {
            bl[k] = fmin(a[k], fmin(b[k], c[k]));
            bh[k] = fmax(a[k], fmax(b[k], c[k]));
        }
        bl[axis] = lo_s;
        bh[axis] = hi_s;
    }
}

__global__ void prim_kernel(const double* __restrict__ vtx, const uint4* __restrict__ tri,
                            const uint32_t* __restrict__ ref_tri, const uint32_t* __restrict__ ref_piece,
                            uint32_t n,
                            double lox, double loy, double loz, double sx, double sy, double sz,
                            double cx, double cy, double cz, double pad, uint64_t* __restrict__ keys, uint32_t* __restrict__ ids,
                            float4* __restrict__ box_lo, float4* __restrict__ box_hi) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint4 t = tri[ref_tri ? ref_tri[i] : i];
    const double* a = vtx + 3ull * t.x;
    const double* b = vtx + 3ull * t.y;
    const double* c = vtx + 3ull * t.z;
    double mn[3], mx[3], cen[3];
    const EscInfo esc = ref_tri ? esc_info(a, b, c) : EscInfo{1, 0, 0.0, 0.0};
    if (esc.pieces > 1) {
        const uint32_t j = ref_piece[i];
        const double w = esc.hi - esc.lo;
        const double lo_s = j == 0 ? esc.lo : esc.lo + w * (static_cast<double>(j) / esc.pieces);
        const double hi_s = j + 1 == esc.pieces ? esc.hi : esc.lo + w * (static_cast<double>(j + 1) / esc.pieces);
        clip_box(a, b, c, esc.axis, lo_s, hi_s, mn, mx);
#pragma unroll
        for (int k = 0; k < 3; ++k) cen[k] = 0.5 * (mn[k] + mx[k]);
    } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            mn[k] = fmin(a[k], fmin(b[k], c[k]));
            mx[k] = fmax(a[k], fmax(b[k], c[k]));
            cen[k] = (a[k] + b[k] + c[k]) * (1.0 / 3.0);
        }
    }
    float lo[3], hi[3];
    const double ctr[3] = {cx, cy, cz};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        lo[k] = __double2float_rd((mn[k] - ctr[k]) - pad);
        hi[k] = __double2float_ru((mx[k] - ctr[k]) + pad);
    }
    box_lo[i] = make_float4(lo[0], lo[1], lo[2], 0.f);
    box_hi[i] = make_float4(hi[0], hi[1], hi[2], 0.f);
    const double qx = fmin(fmax((cen[0] - lox) * sx, 0.0), 2097151.0);
    const double qy = fmin(fmax((cen[1] - loy) * sy, 0.0), 2097151.0);
    const double qz = fmin(fmax((cen[2] - loz) * sz, 0.0), 2097151.0);
    keys[i] = (expand21(static_cast<uint64_t>(qx)) << 2) | (expand21(static_cast<uint64_t>(qy)) << 1) |
              expand21(static_cast<uint64_t>(qz));
    ids[i] = i;
}

__device__ __forceinline__ int delta(const uint64_t* __restrict__ k, int n, int i, int j) {
    if (j < 0 || j >= n) return -1;
    const uint64_t a = k[i], b = k[j];
    if (a != b) return __clzll(static_cast<long long>(a ^ b));
    return 64 + __clz(static_cast<int>(static_cast<uint32_t>(i) ^ static_cast<uint32_t>(j)));
}

// inner node i in [0, n-2]; child encoding: c >= 0 inner node c, c < 0 leaf ~c
__global__ void karras_kernel(const uint64_t* __restrict__ k, int n, int2* __restrict__ child,
                              int2* __restrict__ range, int* __restrict__ parent_inner,
                              int* __restrict__ parent_leaf) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    const int d = (delta(k, n, i, i + 1) - delta(k, n, i, i - 1)) >= 0 ? 1 : -1;
    const int dmin = delta(k, n, i, i - d);
    int lmax = 2;
    while (delta(k, n, i, i + lmax * d) > dmin) lmax <<= 1;
    int l = 0;
    for (int t = lmax >> 1; t >= 1; t >>= 1)
        if (delta(k, n, i, i + (l + t) * d) > dmin) l += t;
    const int j = i + l * d;
    const int dnode = delta(k, n, i, j);
    int s = 0;
    int t = l;
    do {
        t = (t + 1) >> 1;
        if (delta(k, n, i, i + (s + t) * d) > dnode) s += t;
    } while (t > 1);
    const int gamma = i + s * d + min(d, 0);
    const int first = min(i, j), last = max(i, j);
    const int left = (first == gamma) ? ~gamma : gamma;
    const int right = (last == gamma + 1) ? ~(gamma + 1) : gamma + 1;
    child[i] = make_int2(left, right);
    range[i] = make_int2(first, last);
    if (left >= 0) parent_inner[left] = i; else parent_leaf[~left] = i;
    if (right >= 0) parent_inner[right] = i; else parent_leaf[~right] = i;
}

__device__ __forceinline__ void load_box(int c, const float4* __restrict__ ilo,
                                         const float4* __restrict__ ihi, const float4* __restrict__ llo,
                                         const float4* __restrict__ lhi, float4& lo, float4& hi) {
    if (c >= 0) {
        lo = __ldcg(ilo + c);
        hi = __ldcg(ihi + c);
    } else {
        lo = llo[~c];
        hi = lhi[~c];
    }
}

__global__ void refit_kernel(int n, const int2* __restrict__ child, const int* __restrict__ parent_inner,
                             const int* __restrict__ parent_leaf, const float4* __restrict__ llo,
                             const float4* __restrict__ lhi, float4* ilo, float4* ihi, int* flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int p = parent_leaf[i];
    while (p >= 0) {
        __threadfence();
        if (atomicAdd(flags + p, 1) == 0) return;  // first arrival: sibling not done yet
        __threadfence();
        const int2 c = child[p];
        float4 a0, a1, b0, b1;
        load_box(c.x, ilo, ihi, llo, lhi, a0, a1);
        load_box(c.y, ilo, ihi, llo, lhi, b0, b1);
        __stcg(ilo + p, make_float4(fminf(a0.x, b0.x), fminf(a0.y, b0.y), fminf(a0.z, b0.z), 0.f));
        __stcg(ihi + p, make_float4(fmaxf(a1.x, b1.x), fmaxf(a1.y, b1.y), fmaxf(a1.z, b1.z), 0.f));
        p = parent_inner[p];
    }
}

__global__ void tri_kernel(const double* __restrict__ vtx, const uint4* __restrict__ tri,
                           const uint32_t* __restrict__ order, const uint32_t* __restrict__ ref_tri, uint32_t n,
                           double2* __restrict__ out) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t id = ref_tri ? ref_tri[order[k]] : order[k];
    const uint4 t = tri[id];
    const double* a = vtx + 3ull * t.x;
    const double* b = vtx + 3ull * t.y;
    const double* c = vtx + 3ull * t.z;
    const double e1x = b[0] - a[0], e1y = b[1] - a[1], e1z = b[2] - a[2];
    const double e2x = c[0] - a[0], e2y = c[1] - a[1], e2z = c[2] - a[2];
    double2* o = out + 5ull * k;
    o[0] = make_double2(a[0], a[1]);
    o[1] = make_double2(a[2], e1x);
    o[2] = make_double2(e1y, e1z);
    o[3] = make_double2(e2x, e2y);
    o[4] = make_double2(e2z, __longlong_as_double(static_cast<long long>(id)));
}

// sorted leaf boxes: lo_s[k] = lo[order[k]]
__global__ void iota_kernel(uint32_t* __restrict__ out, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = static_cast<uint32_t>(i);
}

// centroids of the primitives in the given order (the SAH build's cen array)
__global__ void centroid_kernel(const float4* __restrict__ lo, const float4* __restrict__ hi,
                                const uint32_t* __restrict__ order, int n, float4* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t p = order[i];
    const float4 l = lo[p], h = hi[p];
    out[i] = make_float4(0.5f * (l.x + h.x), 0.5f * (l.y + h.y), 0.5f * (l.z + h.z), 0.f);
}

__global__ void gather_boxes(const float4* __restrict__ lo, const float4* __restrict__ hi,
                             const uint32_t* __restrict__ ord, int n, float4* __restrict__ lo_s,
                             float4* __restrict__ hi_s) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    lo_s[k] = lo[ord[k]];
    hi_s[k] = hi[ord[k]];
}

// ---- collapse to a 4-wide BVH --------------------------------------------
// "Effective" inner nodes are those with more than kLeafMax triangles (smaller
// subtrees are referenced as leaves).  Every effective inner node at even
// depth becomes a BVH4 node whose (up to 4) slots are its grandchildren; the
// odd-depth nodes are absorbed.  A ray then needs half the dependent node
// fetches and tests 4 independent boxes per fetch.
__device__ __forceinline__ int range_count(const int2* __restrict__ range, int c) {
    const int2 r = range[c];
    return r.y - r.x + 1;
}

__global__ void parity_kernel(int n, const int2* __restrict__ range, const int* __restrict__ parent_inner,
                              unsigned int* __restrict__ is4) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    unsigned int flag = 0;
    if (range_count(range, i) > kLeafMax) {
        int d = 0;
        for (int p = parent_inner[i]; p >= 0; p = parent_inner[p]) ++d;
        flag = (d & 1) == 0;
    }
    is4[i] = flag;
}

__device__ __forceinline__ void slot_of(int c, const int2* __restrict__ range, const float4* __restrict__ ilo,
                                        const float4* __restrict__ ihi, const float4* __restrict__ llo,
                                        const float4* __restrict__ lhi, const unsigned int* __restrict__ idx4,
                                        int& ref, float4& lo, float4& hi) {
    if (c < 0) {
        ref = ~((~c) << 3 | 1);
        lo = llo[~c];
        hi = lhi[~c];
        return;
    }
    lo = ilo[c];
    hi = ihi[c];
    const int2 r = range[c];
    const int cnt = r.y - r.x + 1;
    ref = cnt <= kLeafMax ? ~(r.x << 3 | cnt) : static_cast<int>(idx4[c]);
}

__global__ void emit4_kernel(int n, const int2* __restrict__ child, const int2* __restrict__ range,
                             const unsigned int* __restrict__ is4, const unsigned int* __restrict__ idx4,
                             const float4* __restrict__ ilo, const float4* __restrict__ ihi,
                             const float4* __restrict__ llo, const float4* __restrict__ lhi,
                             float4* __restrict__ nodes) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1 || !is4[i]) return;
    int cnt = 0;
    int ref[4] = {0, 0, 0, 0};
    float4 lo[4], hi[4];
    const int2 ch = child[i];
    const int kids[2] = {ch.x, ch.y};
    for (int k = 0; k < 2; ++k) {
        const int c = kids[k];
        if (c >= 0 && range_count(range, c) > kLeafMax) {  // absorbed odd-depth node
            const int2 g = child[c];
            slot_of(g.x, range, ilo, ihi, llo, lhi, idx4, ref[cnt], lo[cnt], hi[cnt]);
            ++cnt;
            slot_of(g.y, range, ilo, ihi, llo, lhi, idx4, ref[cnt], lo[cnt], hi[cnt]);
            ++cnt;
        } else {
            slot_of(c, range, ilo, ihi, llo, lhi, idx4, ref[cnt], lo[cnt], hi[cnt]);
            ++cnt;
        }
    }
    for (int k = cnt; k < 4; ++k) {  // unused slots: empty boxes, which every slab test misses
        const float inf = __int_as_float(0x7f800000);
        ref[k] = 0;
        lo[k] = make_float4(inf, inf, inf, 0.f);
        hi[k] = make_float4(-inf, -inf, -inf, 0.f);
    }
    float4* o = nodes + 8ll * idx4[i];
    o[0] = make_float4(lo[0].x, lo[1].x, lo[2].x, lo[3].x);
    o[1] = make_float4(hi[0].x, hi[1].x, hi[2].x, hi[3].x);
    o[2] = make_float4(lo[0].y, lo[1].y, lo[2].y, lo[3].y);
    o[3] = make_float4(hi[0].y, hi[1].y, hi[2].y, hi[3].y);
    o[4] = make_float4(lo[0].z, lo[1].z, lo[2].z, lo[3].z);
    o[5] = make_float4(hi[0].z, hi[1].z, hi[2].z, hi[3].z);
    o[6] = make_float4(__int_as_float(ref[0]), __int_as_float(ref[1]), __int_as_float(ref[2]),
                       __int_as_float(ref[3]));
    o[7] = make_float4(__int_as_float(cnt), 0.f, 0.f, 0.f);
}

// depth of every Karras leaf (number of inner ancestors), for the stack bound
__global__ void depth_kernel(int n, const int* __restrict__ parent_inner, const int* __restrict__ parent_leaf,
                             unsigned int* max_depth) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int d = 0;
    for (int p = parent_leaf[i]; p >= 0; p = parent_inner[p]) ++d;
    atomicMax(max_depth, static_cast<unsigned int>(d));
}


// ---------------------------------------------------------------------------
// Binned-SAH top-down build (default; the Karras LBVH is the fallback).
// A node of more than kWarpBuild primitives is a block task: centroid bounds,
// 16 bins per axis holding counts and primitive boxes (shared atomics on
// order-preserving float encodings), the SAH sweep A_L N_L + A_R N_R over the
// 15 bin boundaries of each axis, then a block-wide partition of the node's
// range into the other index buffer.  Smaller nodes are built to the leaves
// by one warp (warp_subtree).  Nodes split down to single triangles, so the
// output has the exact shape of the Karras tree (n - 1 inner nodes, child /
// range / parent arrays, leaves ~position in the final order) and the refit /
// collapse / emit stages run unchanged; ranges stay contiguous because every
// split partitions its own range.  One persistent launch (sah_build_kernel).

// flip: the range's primitives are in idx (0) or idx2 (1); a block task
// partitions into the other buffer, so no copy-back pass
struct SahTask {
    int first, count, node, flip;
};

#ifndef MCSBR_SAH_BINS
#define MCSBR_SAH_BINS 16
#endif
constexpr int kSahBins = MCSBR_SAH_BINS;
constexpr int kSahThreads = 256;
static uint32_t env_u32_bvh(const char* name, uint32_t dflt) {
    const char* v = std::getenv(name);
    return v ? static_cast<uint32_t>(std::strtoul(v, nullptr, 10)) : dflt;
}
// scenes up to this many references skip the Morton pre-sort before the SAH
// build (all of them: the binned SAH splits do not need the order.  The
// strided split sample of the unsorted references gives c5 a better tree --
// its bench path kernel 436 -> 423 ms -- and c1 / c2 / c4 trees of the same
// quality; the builds save the sort: c5 5.5 -> 5.1 ms, c4 1.85 -> 1.6, c2
// 0.75 -> 0.54, c1 0.85 -> 0.58 ms); the Karras fallback still sorts
#ifndef MCSBR_NO_PRESORT_MAX
#define MCSBR_NO_PRESORT_MAX 0xffffffffu
#endif
constexpr uint32_t kNoPresortMax = MCSBR_NO_PRESORT_MAX;
#ifndef MCSBR_SAH_SAMPLE
#define MCSBR_SAH_SAMPLE 4096
#endif
#ifndef MCSBR_SAH_SAMPLE_X
#define MCSBR_SAH_SAMPLE_X 2
#endif
constexpr int kSahSample = MCSBR_SAH_SAMPLE;  // primitives sampled to choose the split of a large node
constexpr int kSahSampleFrom = MCSBR_SAH_SAMPLE_X * kSahSample;  // ... of more than this many

__device__ __forceinline__ int fenc(float f) {  // int order == float order
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float fdec(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

__device__ __forceinline__ float half_area(float lx, float ly, float lz, float hx, float hy, float hz) {
    const float dx = hx - lx, dy = hy - ly, dz = hz - lz;
    return (dx < 0.f || dy < 0.f || dz < 0.f) ? 0.f : dx * dy + dy * dz + dz * dx;
}

// Subtrees of at most kWarpBuild primitives are built by ONE warp, start to
// finish, instead of one block-wide task per inner node (a small task's block
// time is all barriers and global round trips: ~80% of the build's stall
// samples).  Lane l holds one primitive; per node and axis the members are
// ranked by centroid (ties by lane), the boxes gathered in that order, and
// prefix / suffix bound scans give the exact SAH cost of every object split
// A_L N_L + A_R N_R; the cheapest (axis, position) wins and the members are
// permuted into that order, so each child is again a contiguous lane range.
// Node ids come from the top of the id space (`down` counts down) and are
// marked 2 in `ready`, which tells the persistent loop that no published
// task remains above them.
#ifdef MCSBR_SAH_TIMELINE
// critical-path diagnostics (A/B builds only): (count, start ns, end ns) of the large tasks
__device__ unsigned long long g_sah_tl[256][3];
__device__ unsigned int g_sah_tl_n;
#endif
#ifdef MCSBR_SAH_PROF
// build profile (A/B builds only): per phase, clock cycles summed over tasks
// by each block's thread 0; [0] = waiting for a task, [8] = tasks, [9] = sum of counts
__device__ unsigned long long g_sah_prof[10];
#define SAHP0() long long sahp_t = clock64()
#define SAHP(k)                                                                       \
    do {                                                                              \
        if (threadIdx.x == 0) {                                                       \
            const long long now = clock64();                                          \
            atomicAdd(&g_sah_prof[k], static_cast<unsigned long long>(now - sahp_t)); \
            sahp_t = now;                                                             \
        }                                                                             \
    } while (0)
#else
#define SAHP0() (void)0
#define SAHP(k) (void)0
#endif
constexpr int kWarpBuild = 32;
constexpr int kStkScr = 3 * kWarpBuild;  // per-warp scratch: node stack, then 32 ints of scatter space

__device__ __forceinline__ float wscan_min_up(float v, int lane) {
    for (int o = 1; o < 32; o <<= 1) {
        const float w = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v = fminf(v, w);
    }
    return v;
}
__device__ __forceinline__ float wscan_max_up(float v, int lane) {
    for (int o = 1; o < 32; o <<= 1) {
        const float w = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v = fmaxf(v, w);
    }
    return v;
}
__device__ __forceinline__ float wscan_min_down(float v, int lane) {
    for (int o = 1; o < 32; o <<= 1) {
        const float w = __shfl_down_sync(0xffffffffu, v, o);
        if (lane + o < 32) v = fminf(v, w);
    }
    return v;
}
__device__ __forceinline__ float wscan_max_down(float v, int lane) {
    for (int o = 1; o < 32; o <<= 1) {
        const float w = __shfl_down_sync(0xffffffffu, v, o);
        if (lane + o < 32) v = fmaxf(v, w);
    }
    return v;
}

__device__ __noinline__ void warp_subtree(int first, int count, int root, const float4* __restrict__ blo,
                                          const float4* __restrict__ bhi, const uint32_t* src_buf,
                                          uint32_t* __restrict__ idx, int2* __restrict__ child, int2* __restrict__ range,
                                          int* __restrict__ par_i, int* __restrict__ par_l, int* __restrict__ down,
                                          int* __restrict__ ready, volatile int* stk) {
    constexpr unsigned F = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    uint32_t p = 0;
    float lo[3] = {0.f, 0.f, 0.f}, hi[3] = {0.f, 0.f, 0.f}, c[3] = {0.f, 0.f, 0.f};
    if (lane < count) {
        p = src_buf[first + lane];
        const float4 l = __ldg(blo + p), h = __ldg(bhi + p);
        lo[0] = l.x; lo[1] = l.y; lo[2] = l.z;
        hi[0] = h.x; hi[1] = h.y; hi[2] = h.z;
#pragma unroll
        for (int k = 0; k < 3; ++k) c[k] = 0.5f * (lo[k] + hi[k]);
    }
    int sp = 1;
    if (lane == 0) {
        stk[0] = 0;
        stk[1] = count;
        stk[2] = root;
    }
    __syncwarp();
    while (sp > 0) {
        --sp;
        const int b = stk[3 * sp], cnt = stk[3 * sp + 1], id = stk[3 * sp + 2];
        __syncwarp();
        const bool mem = lane >= b && lane < b + cnt;
        float best = INFINITY;
        int best_k = cnt / 2, best_src = lane;  // (no finite cost: split by position)
#pragma unroll 1
        for (int a = 0; a < 3; ++a) {
            const float ca = a == 0 ? c[0] : (a == 1 ? c[1] : c[2]);
            int rank = 0;
            for (int k = b; k < b + cnt; ++k) {
                const float ck = __shfl_sync(F, ca, k);
                rank += (ck < ca || (ck == ca && k < lane)) ? 1 : 0;
            }
            // member that lands on position `lane` of the sorted order (the
            // ranks are a permutation of the members: scatter, then gather)
            if (mem) stk[kStkScr + b + rank] = lane;
            __syncwarp();
            const int src = mem ? stk[kStkScr + lane] : lane;
            __syncwarp();
            float sl[3], sh[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                sl[k] = __shfl_sync(F, lo[k], src);
                sh[k] = __shfl_sync(F, hi[k], src);
                if (!mem) {
                    sl[k] = INFINITY;
                    sh[k] = -INFINITY;
                }
            }
            float pl[3], ph[3], rl[3], rh[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                pl[k] = wscan_min_up(sl[k], lane);
                ph[k] = wscan_max_up(sh[k], lane);
                rl[k] = __shfl_down_sync(F, wscan_min_down(sl[k], lane), 1);
                rh[k] = __shfl_down_sync(F, wscan_max_down(sh[k], lane), 1);
            }
            float cost = INFINITY;
            if (lane >= b && lane < b + cnt - 1) {  // left = positions b..lane
                const int nl = lane - b + 1;
                cost = half_area(pl[0], pl[1], pl[2], ph[0], ph[1], ph[2]) * nl +
                       half_area(rl[0], rl[1], rl[2], rh[0], rh[1], rh[2]) * (cnt - nl);
            }
            float bc = cost;
            int bk = lane;
            for (int o = 16; o > 0; o >>= 1) {
                const float oc = __shfl_xor_sync(F, bc, o);
                const int ok = __shfl_xor_sync(F, bk, o);
                if (oc < bc || (oc == bc && ok < bk)) {
                    bc = oc;
                    bk = ok;
                }
            }
            if (bc < best) {
                best = bc;
                best_k = bk - b + 1;
                best_src = src;
            }
        }
        // members into the chosen order (non-members keep their lane)
        p = __shfl_sync(F, p, best_src);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            lo[k] = __shfl_sync(F, lo[k], best_src);
            hi[k] = __shfl_sync(F, hi[k], best_src);
            c[k] = __shfl_sync(F, c[k], best_src);
        }
        if (lane == 0) {
            int enc[2];
            for (int sd = 0; sd < 2; ++sd) {
                const int bs = sd ? b + best_k : b, cs = sd ? cnt - best_k : best_k;
                if (cs == 1) {
                    enc[sd] = ~(first + bs);
                    par_l[first + bs] = id;
                } else {
                    const int cid = atomicSub(down, 1) - 1;
                    enc[sd] = cid;
                    par_i[cid] = id;
                    atomicExch(ready + cid, 2);
                    stk[3 * sp] = bs;
                    stk[3 * sp + 1] = cs;
                    stk[3 * sp + 2] = cid;
                    ++sp;
                }
            }
            child[id] = make_int2(enc[0], enc[1]);
            range[id] = make_int2(first + b, first + b + cnt - 1);
        }
        sp = __shfl_sync(F, sp, 0);
        __syncwarp();
    }
    if (lane < count) idx[first + lane] = p;
}

// Cooperative partition of the large nodes (the build's critical path is
// the chain of top-level partitions, one block per node: c5's root of 1.04 M
// references took 1.6 ms, its 838 k child 1.4 ms).  A block that takes a
// node of at least kCoopMin references still chooses the split itself (from
// the sample), then publishes the partition as a job of chunks in a slot of
// `jobs`: blocks that are waiting for their next task grab chunks meanwhile.
// Phase 1 counts each chunk's left references; the owner turns the counts
// into per-chunk prefixes; phase 2 scatters every chunk to its final place.
// The permutation is exactly the single-block partition's (left side in
// order from `first`, right side in order from `end - 1` down), so the tree
// does not change.  The owner works on its own job too, so progress never
// depends on helpers.
constexpr int kCoopSlots = 16;
constexpr int kCoopMaxChunks = 1024;
#ifndef MCSBR_SAH_COOP_MIN
#define MCSBR_SAH_COOP_MIN 16384
#endif
constexpr int kCoopMin = MCSBR_SAH_COOP_MIN;
constexpr int kCoopIdle = 0x3fffffff;  // next1 / next2 of a slot with no open phase

struct CoopJob {
    int first, end, flip, axis, split, nl_pos, chunk, nchunks;
    float cmin, scale;
    int next1, done1, next2, done2, owner, pad;
};

struct CoopArgs {
    CoopJob* jobs;
    int* counts;  // [kCoopSlots][kCoopMaxChunks] left references per chunk, then exclusive prefixes
};

// Block-wide partition of the span [lo, hi) of a node [first, end): a left
// reference goes to first + lb + (its rank among the span's left ones), a
// right one to end - 1 - (rb + its rank among the right ones).  write =
// false only counts.  Returns the span's left count (every thread).
__device__ int partition_span(int lo, int hi, int first, int end, int axis, int split, float cmin, float scale,
                              int nl_pos, const uint32_t* in, uint32_t* out, const float4* cin, float4* cout,
                              int lb, int rb, bool write) {
#ifndef MCSBR_SAH_PU
#define MCSBR_SAH_PU 4
#endif
    constexpr int kPU = MCSBR_SAH_PU;
    __shared__ int s_wl[kPU][kSahThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int left_base = 0, right_base = 0;
    for (int base = lo; base < hi; base += kPU * kSahThreads) {
        uint32_t p[kPU];
        float4 cp[kPU];
        bool valid[kPU], left[kPU];
#pragma unroll
        for (int j = 0; j < kPU; ++j) {
            const int i = base + j * kSahThreads + tid;
            valid[j] = i < hi;
            p[j] = valid[j] && write ? __ldcg(in + i) : 0u;
            cp[j] = valid[j] ? __ldcg(cin + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j < kPU; ++j) {
            const int i = base + j * kSahThreads + tid;
            left[j] = false;
            if (valid[j]) {
                if (axis >= 0) {
                    const float ca = axis == 0 ? cp[j].x : (axis == 1 ? cp[j].y : cp[j].z);
                    const int b = min(kSahBins - 1, max(0, static_cast<int>((ca - cmin) * scale)));
                    left[j] = b < split;
                } else {
                    left[j] = (i - first) < nl_pos;
                }
            }
        }
        unsigned m[kPU], v[kPU];
#pragma unroll
        for (int j = 0; j < kPU; ++j) {
            m[j] = __ballot_sync(0xffffffffu, valid[j] && left[j]);
            v[j] = __ballot_sync(0xffffffffu, valid[j]);
            if (lane == 0) s_wl[j][wid] = __popc(m[j]) | (__popc(v[j]) << 16);
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kPU; ++j) {
            int wl = 0, wv = 0, tl = 0, tv = 0;
            for (int w = 0; w < kSahThreads / 32; ++w) {
                const int x = s_wl[j][w];
                if (w < wid) {
                    wl += x & 0xffff;
                    wv += x >> 16;
                }
                tl += x & 0xffff;
                tv += x >> 16;
            }
            if (write && valid[j]) {
                const unsigned below = (1u << lane) - 1u;
                const int pl = wl + __popc(m[j] & below);
                const int pv = wv + __popc(v[j] & below);
                const int pos = left[j] ? first + lb + left_base + pl : end - 1 - (rb + right_base + (pv - pl));
                out[pos] = p[j];
                cout[pos] = cp[j];
            }
            left_base += tl;
            right_base += tv - tl;
        }
        __syncthreads();
    }
    return left_base;
}

// one chunk of slot `slot`'s open phase (block-wide), then its done count
__device__ void coop_chunk(const CoopArgs& ca, int slot, int phase, int c, uint32_t* idx, uint32_t* idx2,
                           float4* cen, float4* cen2) {
    const volatile CoopJob* J = ca.jobs + slot;
    const int first = J->first, end = J->end, flip = J->flip, chunk = J->chunk;
    const int lo = first + c * chunk, hi = min(end, lo + chunk);
    const uint32_t* in = flip ? idx2 : idx;
    uint32_t* out = flip ? idx : idx2;
    const float4* cin = flip ? cen2 : cen;
    float4* cout = flip ? cen : cen2;
    int* cnt = ca.counts + slot * kCoopMaxChunks;
    if (phase == 1) {
        const int l = partition_span(lo, hi, first, end, J->axis, J->split, J->cmin, J->scale, J->nl_pos, in, out,
                                     cin, cout, 0, 0, false);
        if (threadIdx.x == 0) cnt[c] = l;
    } else {
        const int lb = __ldcg(cnt + c);
        partition_span(lo, hi, first, end, J->axis, J->split, J->cmin, J->scale, J->nl_pos, in, out, cin, cout, lb,
                       (lo - first) - lb, true);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(phase == 1 ? &ca.jobs[slot].done1 : &ca.jobs[slot].done2, 1);
}

// thread 0: grab a chunk of any open cooperative phase
__device__ __forceinline__ bool coop_grab(const CoopArgs& ca, int* slot, int* phase, int* c) {
    for (int s = 0; s < kCoopSlots; ++s) {
        volatile CoopJob* J = ca.jobs + s;
        if (J->owner < 0) continue;
        for (int ph = 1; ph <= 2; ++ph) {
            int* nx = ph == 1 ? &ca.jobs[s].next1 : &ca.jobs[s].next2;
            if (*reinterpret_cast<volatile int*>(nx) < J->nchunks) {
                const int k = atomicAdd(nx, 1);
                __threadfence();
                if (k < J->nchunks) {
                    *slot = s;
                    *phase = ph;
                    *c = k;
                    return true;
                }
            }
        }
    }
    return false;
}

// the owner's side of a cooperative partition; returns the left count
__device__ int coop_partition(const CoopArgs& ca, int node, int first, int end, int flip, int axis, int split,
                              float cmin, float scale, int nl_pos, uint32_t* idx, uint32_t* idx2, float4* cen,
                              float4* cen2) {
    __shared__ int s_slot, s_c, s_total;
    const int count = end - first;
    if (threadIdx.x == 0) {
        int slot = 0;
        while (atomicCAS(&ca.jobs[slot].owner, -1, node) != -1) slot = (slot + 1) % kCoopSlots;
        CoopJob* J = ca.jobs + slot;
        int chunk = (count + kCoopMaxChunks - 1) / kCoopMaxChunks;
        chunk = max(4096, (chunk + 1023) / 1024 * 1024);
        J->first = first;
        J->end = end;
        J->flip = flip;
        J->axis = axis;
        J->split = split;
        J->nl_pos = nl_pos;
        J->chunk = chunk;
        J->nchunks = (count + chunk - 1) / chunk;
        J->cmin = cmin;
        J->scale = scale;
        J->done1 = 0;
        J->done2 = 0;
        J->next2 = kCoopIdle;
        __threadfence();
        atomicExch(&J->next1, 0);  // phase 1 open
        s_slot = slot;
    }
    __syncthreads();
    const int slot = s_slot;
    CoopJob* J = ca.jobs + slot;
    const int nchunks = *reinterpret_cast<volatile int*>(&J->nchunks);
    for (int phase = 1; phase <= 2; ++phase) {
        int* nx = phase == 1 ? &J->next1 : &J->next2;
        int* dn = phase == 1 ? &J->done1 : &J->done2;
        for (;;) {  // work on the own job's chunks
            if (threadIdx.x == 0) s_c = atomicAdd(nx, 1);
            __syncthreads();
            const int c = s_c;
            __syncthreads();
            if (c >= nchunks) break;
            coop_chunk(ca, slot, phase, c, idx, idx2, cen, cen2);
        }
        if (threadIdx.x == 0) {
            while (*reinterpret_cast<volatile int*>(dn) < nchunks) __nanosleep(32);
            __threadfence();
            if (phase == 1) {  // chunk counts -> exclusive prefixes (in place), total
                int* cnt = ca.counts + slot * kCoopMaxChunks;
                int run = 0;
                for (int k = 0; k < nchunks; ++k) {
                    const int v = __ldcg(cnt + k);
                    cnt[k] = run;
                    run += v;
                }
                s_total = run;
                __threadfence();
                atomicExch(&J->next2, 0);  // phase 2 open
            } else {
                atomicExch(&J->next1, kCoopIdle);
                atomicExch(&J->next2, kCoopIdle);
                __threadfence();
                atomicExch(&J->owner, -1);
            }
        }
        __syncthreads();
    }
    return s_total;
}

__device__ __forceinline__ void sah_split(
    const SahTask t, const float4* __restrict__ blo, const float4* __restrict__ bhi,
    uint32_t* __restrict__ idx, uint32_t* __restrict__ idx2, float4* __restrict__ cen, float4* __restrict__ cen2,
    int2* __restrict__ child, int2* __restrict__ range,
    int* __restrict__ par_i, int* __restrict__ par_l, int* __restrict__ node_counter, SahTask* __restrict__ tasks,
    int* __restrict__ ready, int* __restrict__ down, const CoopArgs ca) {
    SAHP0();
    __shared__ int s_cnt[3][kSahBins];
    __shared__ int s_box[3][kSahBins][6];
    __shared__ float s_red[2][3][kSahThreads / 32];
    __shared__ float s_cmin[3], s_scale[3];
    __shared__ float s_cost[3];
    __shared__ int s_split[3], s_nl[3];
    __shared__ float s_ra[3][kSahBins];  // sweep: suffix areas / counts per axis
    __shared__ int s_rc[3][kSahBins];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int end = t.first + t.count;
    const uint32_t* in = t.flip ? idx2 : idx;
    uint32_t* out = t.flip ? idx : idx2;
    // the primitives' centroids travel with their ids (cen pairs with idx,
    // cen2 with idx2): the partition reads them in order instead of
    // gathering two boxes per primitive (the top-level partitions, one block
    // per node, are the build's critical path: c5's root took 3.6 ms)
    const float4* cin = t.flip ? cen2 : cen;
    float4* cout = t.flip ? cen : cen2;
    // large nodes (the top levels, one block each) choose their split from a
    // strided sample of ~16 k primitives; the partition below counts exactly
    const int stride = t.count > kSahSampleFrom ? t.count / kSahSample : 1;
    // 1. centroid bounds
    float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int i = t.first + tid * stride; i < end; i += kSahThreads * stride) {
        const float4 cc = cin[i];
        const float c[3] = {cc.x, cc.y, cc.z};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            mn[a] = fminf(mn[a], c[a]);
            mx[a] = fmaxf(mx[a], c[a]);
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[a] = fminf(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
            mx[a] = fmaxf(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
        }
        if (lane == 0) {
            s_red[0][a][wid] = mn[a];
            s_red[1][a][wid] = mx[a];
        }
    }
    for (int i = tid; i < 3 * kSahBins; i += kSahThreads) {
        const int a = i / kSahBins, b = i % kSahBins;
        s_cnt[a][b] = 0;
        s_box[a][b][0] = s_box[a][b][1] = s_box[a][b][2] = fenc(INFINITY);
        s_box[a][b][3] = s_box[a][b][4] = s_box[a][b][5] = fenc(-INFINITY);
    }
    __syncthreads();
    if (tid < 3) {
        float lo = INFINITY, hi = -INFINITY;
        for (int w = 0; w < kSahThreads / 32; ++w) {
            lo = fminf(lo, s_red[0][tid][w]);
            hi = fmaxf(hi, s_red[1][tid][w]);
        }
        s_cmin[tid] = lo;
        s_scale[tid] = hi > lo ? (kSahBins * (1.0f - 1e-6f)) / (hi - lo) : 0.0f;
    }
    __syncthreads();
    SAHP(1);
    // 2. bins
    for (int i = t.first + tid * stride; i < end; i += kSahThreads * stride) {
        const uint32_t p = in[i];
        const float4 l = __ldg(blo + p), h = __ldg(bhi + p);
        const float4 cc = cin[i];
        const float c[3] = {cc.x, cc.y, cc.z};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (s_scale[a] == 0.0f) continue;
            const int b = min(kSahBins - 1, max(0, static_cast<int>((c[a] - s_cmin[a]) * s_scale[a])));
            atomicAdd(&s_cnt[a][b], 1);
            atomicMin(&s_box[a][b][0], fenc(l.x));
            atomicMin(&s_box[a][b][1], fenc(l.y));
            atomicMin(&s_box[a][b][2], fenc(l.z));
            atomicMax(&s_box[a][b][3], fenc(h.x));
            atomicMax(&s_box[a][b][4], fenc(h.y));
            atomicMax(&s_box[a][b][5], fenc(h.z));
        }
    }
    __syncthreads();
    SAHP(2);
    // 3. SAH sweep per axis
    if (tid < 3) {
        const int a = tid;
        float best = INFINITY;
        int split = -1, nl_best = 0;
        if (s_scale[a] != 0.0f) {
            float* ra = s_ra[a];
            int* rc = s_rc[a];
            float l0 = INFINITY, l1 = INFINITY, l2 = INFINITY, h0 = -INFINITY, h1 = -INFINITY, h2 = -INFINITY;
            int n = 0;
            for (int b = kSahBins - 1; b >= 1; --b) {  // suffix: bins b..15
                n += s_cnt[a][b];
                l0 = fminf(l0, fdec(s_box[a][b][0]));
                l1 = fminf(l1, fdec(s_box[a][b][1]));
                l2 = fminf(l2, fdec(s_box[a][b][2]));
                h0 = fmaxf(h0, fdec(s_box[a][b][3]));
                h1 = fmaxf(h1, fdec(s_box[a][b][4]));
                h2 = fmaxf(h2, fdec(s_box[a][b][5]));
                ra[b] = half_area(l0, l1, l2, h0, h1, h2);
                rc[b] = n;
            }
            l0 = l1 = l2 = INFINITY;
            h0 = h1 = h2 = -INFINITY;
            n = 0;
            for (int b = 0; b < kSahBins - 1; ++b) {  // prefix: bins 0..b | b+1..15
                n += s_cnt[a][b];
                l0 = fminf(l0, fdec(s_box[a][b][0]));
                l1 = fminf(l1, fdec(s_box[a][b][1]));
                l2 = fminf(l2, fdec(s_box[a][b][2]));
                h0 = fmaxf(h0, fdec(s_box[a][b][3]));
                h1 = fmaxf(h1, fdec(s_box[a][b][4]));
                h2 = fmaxf(h2, fdec(s_box[a][b][5]));
                if (n == 0 || rc[b + 1] == 0) continue;
                const float cost = half_area(l0, l1, l2, h0, h1, h2) * n + ra[b + 1] * rc[b + 1];
                if (cost < best) {
                    best = cost;
                    split = b + 1;
                    nl_best = n;
                }
            }
        }
        s_cost[a] = best;
        s_split[a] = split;
        s_nl[a] = nl_best;
    }
    __syncthreads();
    SAHP(3);
    int axis = -1;
    float best = INFINITY;
    for (int a = 0; a < 3; ++a)
        if (s_split[a] >= 0 && s_cost[a] < best) {
            best = s_cost[a];
            axis = a;
        }
    int nl = axis >= 0 ? s_nl[axis] : t.count / 2;  // no usable split: median by position
    const int split = axis >= 0 ? s_split[axis] : 0;
    const float cmin = axis >= 0 ? s_cmin[axis] : 0.0f, scale = axis >= 0 ? s_scale[axis] : 0.0f;
    SAHP(4);
    // 4. partition of [first, end) from `in` into `out`: the left side from
    // `first` up in order, the right side from `end - 1` down, so one pass
    // needs no left count (a sampled split's exact count falls out of it)
    // (kPU sub-chunks of 256 per iteration in partition_span: their loads
    // issued together, one barrier pair per iteration); large nodes
    // cooperatively with the waiting blocks
    int left_base;
    if (t.count >= kCoopMin && ca.jobs)
        left_base = coop_partition(ca, t.node, t.first, end, t.flip, axis, split, cmin, scale, nl, idx, idx2, cen,
                                   cen2);
    else
        left_base = partition_span(t.first, end, t.first, end, axis, split, cmin, scale, nl, in, out, cin, cout, 0, 0,
                                   true);
    nl = left_base;
    if (nl == 0 || nl == t.count) nl = t.count / 2;  // a sampled split that separates nothing: by position
    SAHP(5);
    // 5. children: single primitives are leaves, small ranges are built by
    // warps 0 / 1 of this block right away, the rest are published as tasks
    __shared__ SahTask s_sub[2];
    __shared__ int s_stk[2][kStkScr + 32];
    if (tid == 0) {
        const int starts[2] = {t.first, t.first + nl}, sizes[2] = {nl, t.count - nl};
        int enc[2];
        for (int k = 0; k < 2; ++k) {
            s_sub[k].count = 0;
            if (sizes[k] == 1) {  // a leaf: its primitive goes to the final order (idx)
                enc[k] = ~starts[k];
                par_l[starts[k]] = t.node;
                if (out != idx) idx[starts[k]] = out[starts[k]];
            } else if (sizes[k] <= kWarpBuild) {
                const int id = atomicSub(down, 1) - 1;
                enc[k] = id;
                par_i[id] = t.node;
                atomicExch(ready + id, 2);
                s_sub[k] = SahTask{starts[k], sizes[k], id, 0};
            } else {  // publish the child's task under its inner-node index
                const int id = atomicAdd(node_counter, 1);
                enc[k] = id;
                par_i[id] = t.node;
                tasks[id] = SahTask{starts[k], sizes[k], id, t.flip ^ 1};
                __threadfence();
                atomicExch(ready + id, 1);
            }
        }
        child[t.node] = make_int2(enc[0], enc[1]);
        range[t.node] = make_int2(t.first, end - 1);
    }
    __syncthreads();
    SAHP(6);
    if (wid < 2 && s_sub[wid].count >= 2)
        warp_subtree(s_sub[wid].first, s_sub[wid].count, s_sub[wid].node, blo, bhi, out, idx, child, range, par_i,
                     par_l, down, ready, s_stk[wid]);
    SAHP(7);
}

// Persistent build: every inner node is one task whose index is its node
// id; co-resident blocks take ids 0, 1, 2, ... in order and wait until the
// parent has published the task (a task's parent always has a smaller id and
// is already being processed, so the waits always end).  One launch instead
// of one launch plus a host round trip per tree level.
__global__ void __launch_bounds__(kSahThreads, 4) sah_build_kernel(
    int n_inner, int* __restrict__ head, const float4* __restrict__ blo, const float4* __restrict__ bhi,
    uint32_t* __restrict__ idx, uint32_t* __restrict__ idx2, float4* __restrict__ cen, float4* __restrict__ cen2,
    int2* __restrict__ child, int2* __restrict__ range,
    int* __restrict__ par_i, int* __restrict__ par_l, int* __restrict__ node_counter, SahTask* __restrict__ tasks,
    int* __restrict__ ready, int* __restrict__ down, const CoopArgs ca) {
    __shared__ int s_id;
    __shared__ SahTask s_task;
    __shared__ int s_help[3];  // slot, phase, chunk of a cooperative partition to help with (slot -1: none)
    for (;;) {
        if (threadIdx.x == 0) s_id = atomicAdd(head, 1);
        __syncthreads();
        const int i0 = s_id;
        __syncthreads();
        if (i0 >= n_inner) break;
        // wait for task i0; meanwhile help the open cooperative partitions
        for (;;) {
            if (threadIdx.x == 0) {
#ifdef MCSBR_SAH_PROF
                const long long w0 = clock64();
#endif
                s_help[0] = -1;
                for (;;) {
                    const int r = atomicAdd(ready + i0, 0);
                    if (r != 0) {
                        if (r == 2) {
                            s_id = n_inner;  // a warp-built node: every id from here up is one
                        } else {
                            __threadfence();
                            s_task.first = __ldcg(&tasks[i0].first);
                            s_task.count = __ldcg(&tasks[i0].count);
                            s_task.node = __ldcg(&tasks[i0].node);
                            s_task.flip = __ldcg(&tasks[i0].flip);
                        }
                        break;
                    }
                    if (ca.jobs && coop_grab(ca, &s_help[0], &s_help[1], &s_help[2])) break;
                    __nanosleep(64);
                }
#ifdef MCSBR_SAH_PROF
                atomicAdd(&g_sah_prof[0], static_cast<unsigned long long>(clock64() - w0));
                if (s_help[0] < 0 && s_id < n_inner) {
                    atomicAdd(&g_sah_prof[8], 1ull);
                    atomicAdd(&g_sah_prof[9], static_cast<unsigned long long>(s_task.count));
                }
#endif
            }
            __syncthreads();
            if (s_help[0] < 0) break;
            coop_chunk(ca, s_help[0], s_help[1], s_help[2], idx, idx2, cen, cen2);
            __syncthreads();
        }
        if (s_id >= n_inner) break;
#ifdef MCSBR_SAH_TIMELINE
        unsigned long long tl0 = 0;
        if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl0));
#endif
        sah_split(s_task, blo, bhi, idx, idx2, cen, cen2, child, range, par_i, par_l, node_counter, tasks, ready,
                  down, ca);
        __syncthreads();
#ifdef MCSBR_SAH_TIMELINE
        if (threadIdx.x == 0 && s_task.count >= 16384) {
            unsigned long long tl1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl1));
            const unsigned k = atomicAdd(&g_sah_tl_n, 1u);
            if (k < 256) {
                g_sah_tl[k][0] = static_cast<unsigned long long>(s_task.count);
                g_sah_tl[k][1] = tl0;
                g_sah_tl[k][2] = tl1;
            }
        }
#endif
    }
}

}  // namespace

#define BVH_CHECK(x)                          \
    do {                                      \
        cudaError_t e_ = (x);                 \
        if (e_ != cudaSuccess) {              \
            err = e_;                         \
            goto done;                        \
        }                                     \
    } while (0)

// Early split clipping references (see esc_info): on success *n_refs is the
// number of BVH primitives and, if any triangle is split, *ref_tri /
// *ref_piece map each reference to its triangle and piece (else nullptr:
// reference i is triangle i).
static cudaError_t esc_references(const double* d_vertices, const uint4* d_tri_idx, uint32_t n_tri,
                                  cudaStream_t stream, uint32_t* n_refs, uint32_t** ref_tri, uint32_t** ref_piece) {
    *n_refs = n_tri;
    *ref_tri = *ref_piece = nullptr;
    if (std::getenv("MCSBR_ESC") && std::strcmp(std::getenv("MCSBR_ESC"), "0") == 0) return cudaSuccess;  // A/B
    uint32_t *extra = nullptr, *off = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    uint32_t last[2] = {0, 0};
    cudaError_t e = dev_malloc(&extra, sizeof(uint32_t) * n_tri);
    if (e == cudaSuccess) e = dev_malloc(&off, sizeof(uint32_t) * n_tri);
    if (e == cudaSuccess) {
        esc_count_kernel<<<(n_tri + 255) / 256, 256, 0, stream>>>(d_vertices, d_tri_idx, n_tri, extra);
        e = cudaGetLastError();
    }
    tmp_bytes = scan_temp_bytes(n_tri);
    if (e == cudaSuccess) e = dev_malloc(&tmp, tmp_bytes);
    if (e == cudaSuccess) e = exclusive_scan_u32(extra, off, n_tri, tmp, stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(&last[0], off + (n_tri - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(&last[1], extra + (n_tri - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    const uint64_t total = static_cast<uint64_t>(last[0]) + last[1];
    if (e == cudaSuccess && total > 0 && n_tri + total < (uint64_t{1} << 28)) {
        const uint32_t n = n_tri + static_cast<uint32_t>(total);
        e = dev_malloc(ref_tri, sizeof(uint32_t) * n);
        if (e == cudaSuccess) e = dev_malloc(ref_piece, sizeof(uint32_t) * n);
        if (e == cudaSuccess) {
            esc_refs_kernel<<<(n_tri + 255) / 256, 256, 0, stream>>>(extra, off, n_tri, *ref_tri, *ref_piece);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) {
            *n_refs = n;
        } else {
            dev_free(*ref_tri);
            dev_free(*ref_piece);
            *ref_tri = *ref_piece = nullptr;
        }
    }
    // esc_refs_kernel reads extra / off: wait for it, then free without a device sync
    const bool synced = e == cudaSuccess && cudaStreamSynchronize(stream) == cudaSuccess;
    dev_free(extra, synced);
    dev_free(off, synced);
    dev_free(tmp, synced);
    return e;
}

cudaError_t build_bvh(const double* d_vertices, const uint4* d_tri_idx, uint32_t n_tri,
                      const double scene_lo[3], const double scene_hi[3], const double center[3],
                      double box_pad, cudaStream_t stream, BvhBuildOut* out) {
    uint32_t n_refs = n_tri;
    uint32_t *ref_tri = nullptr, *ref_piece = nullptr;
    {
        const cudaError_t e = esc_references(d_vertices, d_tri_idx, n_tri, stream, &n_refs, &ref_tri, &ref_piece);
        if (e != cudaSuccess) return e;
    }
    cudaError_t err = cudaSuccess;
    const int n = static_cast<int>(n_refs);
    uint64_t *keys = nullptr, *keys_s = nullptr;
    uint32_t *ids = nullptr, *ids_s = nullptr;
    float4 *blo = nullptr, *bhi = nullptr, *blo_s = nullptr, *bhi_s = nullptr;
    float4 *ilo = nullptr, *ihi = nullptr;
    int2 *child = nullptr, *range = nullptr;
    int *par_i = nullptr, *par_l = nullptr, *flags = nullptr;
    unsigned int* dmax = nullptr;
    unsigned int *is4 = nullptr, *idx4 = nullptr;
    uint32_t* sidx = nullptr;         // SAH: the final triangle order
    float4 *cen = nullptr, *cen2 = nullptr;  // SAH: centroids travelling with the ids
    void *coop_jobs = nullptr, *coop_counts = nullptr;  // SAH: cooperative partition slots
    SahTask* tasks = nullptr;
    int* node_counter = nullptr;
    const uint32_t* order = nullptr;  // final leaf order (SAH or Morton)
    void* tmp = nullptr;
    void* scan_tmp = nullptr;
    size_t tmp_bytes = 0, scan_bytes = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    const int B = 256;
    const int G = (n + B - 1) / B;
    const int inner = n > 1 ? n - 1 : 1;
    double s[3];
    // the Morton pre-sort is skipped for small scenes when the SAH build runs (below)
    const char* bvh_env0 = std::getenv("MCSBR_BVH");
    const bool sah_wanted = !(bvh_env0 && std::strcmp(bvh_env0, "lbvh") == 0);
    const bool presort =
        !(sah_wanted && static_cast<uint32_t>(n) <= env_u32_bvh("MCSBR_BVH_PRESORT_MAX", kNoPresortMax));
    out->nodes = nullptr;
    out->tri64 = nullptr;
    for (int k = 0; k < 3; ++k) {
        const double ext = scene_hi[k] - scene_lo[k];
        s[k] = ext > 0.0 ? 2097152.0 / ext : 0.0;
    }
    BVH_CHECK(cudaEventCreate(&e0));
    BVH_CHECK(cudaEventCreate(&e1));
    BVH_CHECK(cudaEventRecord(e0, stream));
    BVH_CHECK(dev_malloc(&keys, sizeof(uint64_t) * n));
    BVH_CHECK(dev_malloc(&keys_s, sizeof(uint64_t) * n));
    BVH_CHECK(dev_malloc(&ids, sizeof(uint32_t) * n));
    BVH_CHECK(dev_malloc(&ids_s, sizeof(uint32_t) * n));
    BVH_CHECK(dev_malloc(&blo, sizeof(float4) * n));
    BVH_CHECK(dev_malloc(&bhi, sizeof(float4) * n));
    BVH_CHECK(dev_malloc(&blo_s, sizeof(float4) * n));
    BVH_CHECK(dev_malloc(&bhi_s, sizeof(float4) * n));
    BVH_CHECK(dev_malloc(&ilo, sizeof(float4) * inner));
    BVH_CHECK(dev_malloc(&ihi, sizeof(float4) * inner));
    BVH_CHECK(dev_malloc(&child, sizeof(int2) * inner));
    BVH_CHECK(dev_malloc(&range, sizeof(int2) * inner));
    BVH_CHECK(dev_malloc(&par_i, sizeof(int) * inner));
    BVH_CHECK(dev_malloc(&par_l, sizeof(int) * n));
    BVH_CHECK(dev_malloc(&flags, sizeof(int) * inner));
    BVH_CHECK(dev_malloc(&dmax, sizeof(unsigned int)));
    BVH_CHECK(dev_malloc(&is4, sizeof(unsigned int) * inner));
    BVH_CHECK(dev_malloc(&idx4, sizeof(unsigned int) * inner));
    BVH_CHECK(dev_malloc(&out->nodes, sizeof(float4) * 8 * inner));
    BVH_CHECK(dev_malloc(&out->tri64, sizeof(double2) * 5 * n));
    BVH_CHECK(cudaMemsetAsync(flags, 0, sizeof(int) * inner, stream));
    BVH_CHECK(cudaMemsetAsync(dmax, 0, sizeof(unsigned int), stream));
    BVH_CHECK(cudaMemsetAsync(par_i, 0xff, sizeof(int) * inner, stream));  // root parent = -1
    BVH_CHECK(cudaMemsetAsync(par_l, 0xff, sizeof(int) * n, stream));

    prim_kernel<<<G, B, 0, stream>>>(d_vertices, d_tri_idx, ref_tri, ref_piece, n_refs, scene_lo[0], scene_lo[1], scene_lo[2],
                                     s[0], s[1], s[2], center[0], center[1], center[2], box_pad, keys,
                                     ids, blo, bhi);
    BVH_CHECK(cudaGetLastError());
    // stable LSD radix sort of the (Morton key, reference) pairs (sort.cu);
    // the sorted pairs end up in keys_s / ids_s.  Skipped when the SAH build
    // runs (kNoPresortMax, MCSBR_BVH_PRESORT_MAX): the binned SAH only needs
    // the references in any order (its splits are spatial); the Karras
    // fallback sorts when it is needed.
    tmp_bytes = radix_sort_temp_bytes(n);
    BVH_CHECK(dev_malloc(&tmp, tmp_bytes));
    if (!presort) {
        BVH_CHECK(cudaMemcpyAsync(ids_s, ids, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, stream));
    } else {
#ifdef MCSBR_BVH_PHASES
        cudaStreamSynchronize(stream);
        const auto ph0 = std::chrono::steady_clock::now();
#endif
        bool in_alt = false;
        BVH_CHECK(radix_sort_pairs(keys, keys_s, ids, ids_s, n, 64, tmp, stream, &in_alt));
#ifdef MCSBR_BVH_PHASES
        cudaStreamSynchronize(stream);
        std::fprintf(stderr, "[bvh] sort %.3f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ph0).count());
#endif
        if (!in_alt) {
            std::swap(keys, keys_s);
            std::swap(ids, ids_s);
        }
    }
    order = ids_s;
    if (n > 1) {
        // binned SAH (from the reference order), unless MCSBR_BVH=lbvh or
        // the tree comes out deeper than the traversal stack allows
        const char* bvh_env = std::getenv("MCSBR_BVH");
        bool sah = !(bvh_env && std::strcmp(bvh_env, "lbvh") == 0);
        if (sah) {
            BVH_CHECK(dev_malloc(&sidx, sizeof(uint32_t) * n));
            BVH_CHECK(dev_malloc(&cen, sizeof(float4) * n));
            BVH_CHECK(dev_malloc(&cen2, sizeof(float4) * n));
            BVH_CHECK(dev_malloc(&tasks, sizeof(SahTask) * inner));
            BVH_CHECK(dev_malloc(&node_counter, sizeof(int) * (inner + 3)));  // counter, head, ready[inner], down
            BVH_CHECK(cudaMemcpyAsync(sidx, ids_s, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, stream));
            BVH_CHECK(cudaMemsetAsync(node_counter, 0, sizeof(int) * (inner + 2), stream));
            BVH_CHECK(cudaMemcpyAsync(node_counter + inner + 2, &inner, sizeof(int), cudaMemcpyHostToDevice, stream));
            {
                const int init[3] = {1, 0, 1};  // next node id, head, ready[0]
                const SahTask root{0, n, 0, 0};
                BVH_CHECK(cudaMemcpyAsync(node_counter, init, sizeof(init), cudaMemcpyHostToDevice, stream));
                BVH_CHECK(cudaMemcpyAsync(tasks, &root, sizeof(SahTask), cudaMemcpyHostToDevice, stream));
                int dev = 0, sms = 148, per_sm = 1;
                BVH_CHECK(cudaGetDevice(&dev));
                BVH_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
                BVH_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sah_build_kernel, kSahThreads, 0));
                const int grid = std::max(1, std::min(inner, sms * std::max(per_sm, 1)));  // co-resident
                centroid_kernel<<<G, B, 0, stream>>>(blo, bhi, sidx, n, cen);
                BVH_CHECK(cudaGetLastError());
                CoopArgs ca{nullptr, nullptr};
                if (n >= kCoopMin) {  // cooperative partitions of the large nodes
                    BVH_CHECK(dev_malloc(&coop_jobs, sizeof(CoopJob) * kCoopSlots));
                    BVH_CHECK(dev_malloc(&coop_counts, sizeof(int) * kCoopSlots * kCoopMaxChunks));
                    CoopJob init[kCoopSlots];
                    std::memset(init, 0, sizeof(init));
                    for (CoopJob& j : init) {
                        j.owner = -1;
                        j.next1 = j.next2 = kCoopIdle;
                    }
                    BVH_CHECK(cudaMemcpyAsync(coop_jobs, init, sizeof(init), cudaMemcpyHostToDevice, stream));
                    ca = CoopArgs{static_cast<CoopJob*>(coop_jobs), static_cast<int*>(coop_counts)};
                }
                sah_build_kernel<<<grid, kSahThreads, 0, stream>>>(inner, node_counter + 1, blo, bhi, sidx, ids,
                                                                   cen, cen2, child, range, par_i, par_l, node_counter,
                                                                   tasks, node_counter + 2, node_counter + inner + 2,
                                                                   ca);
                BVH_CHECK(cudaGetLastError());
            }
            depth_kernel<<<G, B, 0, stream>>>(n, par_i, par_l, dmax);
            BVH_CHECK(cudaGetLastError());
#ifdef MCSBR_SAH_TIMELINE
            {
                unsigned long long tl[256][3];
                unsigned int tn = 0;
                BVH_CHECK(cudaMemcpyFromSymbolAsync(&tn, g_sah_tl_n, sizeof(tn), 0, cudaMemcpyDeviceToHost, stream));
                BVH_CHECK(cudaMemcpyFromSymbolAsync(tl, g_sah_tl, sizeof(tl), 0, cudaMemcpyDeviceToHost, stream));
                BVH_CHECK(cudaStreamSynchronize(stream));
                unsigned long long t0 = ~0ull;
                for (unsigned k = 0; k < std::min(tn, 256u); ++k) t0 = std::min(t0, tl[k][1]);
                for (unsigned k = 0; k < std::min(tn, 256u); ++k)
                    std::fprintf(stderr, "sah task %7llu prims: %8.3f .. %8.3f ms\n", tl[k][0], (tl[k][1] - t0) * 1e-6,
                                 (tl[k][2] - t0) * 1e-6);
                const unsigned z = 0;
                BVH_CHECK(cudaMemcpyToSymbolAsync(g_sah_tl_n, &z, sizeof(z), 0, cudaMemcpyHostToDevice, stream));
            }
#endif
#ifdef MCSBR_SAH_PROF
            {
                unsigned long long pr[10];
                BVH_CHECK(cudaMemcpyFromSymbolAsync(pr, g_sah_prof, sizeof(pr), 0, cudaMemcpyDeviceToHost, stream));
                BVH_CHECK(cudaStreamSynchronize(stream));
                std::fprintf(stderr, "sah prof n=%d tasks=%llu prims=%llu | wait %.3g bounds %.3g bins %.3g sweep %.3g "
                             "select %.3g partition %.3g children %.3g warpbuild %.3g (Mcycles, summed over blocks)\n",
                             n, pr[8], pr[9], pr[0] * 1e-6, pr[1] * 1e-6, pr[2] * 1e-6, pr[3] * 1e-6, pr[4] * 1e-6,
                             pr[5] * 1e-6, pr[6] * 1e-6, pr[7] * 1e-6);
                const unsigned long long z[10] = {};
                BVH_CHECK(cudaMemcpyToSymbolAsync(g_sah_prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, stream));
            }
#endif
            unsigned int md = 0;
            BVH_CHECK(cudaMemcpyAsync(&md, dmax, sizeof(md), cudaMemcpyDeviceToHost, stream));
            BVH_CHECK(cudaStreamSynchronize(stream));
            if (3 * ((md + 1) / 2 + 1) > static_cast<unsigned>(kStackSize) ||
                env_u32_bvh("MCSBR_BVH_FORCE_FALLBACK", 0) != 0) {  // (the knob exercises this path in tests)
                sah = false;  // too deep for the traversal stack: Karras tree instead
                BVH_CHECK(cudaMemsetAsync(dmax, 0, sizeof(unsigned int), stream));
                if (!presort) {  // the Karras tree needs the Morton order
                    // (the SAH build used `ids` as its partition scratch: restore 0..n-1)
                    iota_kernel<<<G, B, 0, stream>>>(ids, n);
                    BVH_CHECK(cudaGetLastError());
                    bool in_alt = false;
                    BVH_CHECK(radix_sort_pairs(keys, keys_s, ids, ids_s, n, 64, tmp, stream, &in_alt));
                    if (!in_alt) {
                        std::swap(keys, keys_s);
                        std::swap(ids, ids_s);
                    }
                    order = ids_s;
                }
                BVH_CHECK(cudaMemsetAsync(par_i, 0xff, sizeof(int) * inner, stream));
                BVH_CHECK(cudaMemsetAsync(par_l, 0xff, sizeof(int) * n, stream));
            } else {
                order = sidx;
            }
        }
        if (!sah) {
            karras_kernel<<<(n - 1 + B - 1) / B, B, 0, stream>>>(keys_s, n, child, range, par_i, par_l);
            BVH_CHECK(cudaGetLastError());
        }
    }
    tri_kernel<<<G, B, 0, stream>>>(d_vertices, d_tri_idx, order, ref_tri, n_refs, out->tri64);
    BVH_CHECK(cudaGetLastError());
    if (n > 1) {
        gather_boxes<<<G, B, 0, stream>>>(blo, bhi, order, n, blo_s, bhi_s);
        BVH_CHECK(cudaGetLastError());
        refit_kernel<<<G, B, 0, stream>>>(n, child, par_i, par_l, blo_s, bhi_s, ilo, ihi, flags);
        BVH_CHECK(cudaGetLastError());
        parity_kernel<<<(n - 1 + B - 1) / B, B, 0, stream>>>(n, range, par_i, is4);
        BVH_CHECK(cudaGetLastError());
        scan_bytes = scan_temp_bytes(n - 1);
        BVH_CHECK(dev_malloc(&scan_tmp, scan_bytes));
        BVH_CHECK(exclusive_scan_u32(is4, idx4, n - 1, scan_tmp, stream));
        emit4_kernel<<<(n - 1 + B - 1) / B, B, 0, stream>>>(n, child, range, is4, idx4, ilo, ihi, blo_s,
                                                            bhi_s, out->nodes);
        BVH_CHECK(cudaGetLastError());
        if (order != sidx) {  // (the SAH path measured its depth already)
            depth_kernel<<<G, B, 0, stream>>>(n, par_i, par_l, dmax);
            BVH_CHECK(cudaGetLastError());
        }
    }
    BVH_CHECK(cudaEventRecord(e1, stream));
    {
        unsigned int md = 0, last[2] = {0, 0};
        BVH_CHECK(cudaMemcpyAsync(&md, dmax, sizeof(md), cudaMemcpyDeviceToHost, stream));
        if (n > 1) {
            BVH_CHECK(cudaMemcpyAsync(&last[0], idx4 + (n - 2), sizeof(unsigned int), cudaMemcpyDeviceToHost,
                                      stream));
            BVH_CHECK(cudaMemcpyAsync(&last[1], is4 + (n - 2), sizeof(unsigned int), cudaMemcpyDeviceToHost,
                                      stream));
        }
        BVH_CHECK(cudaStreamSynchronize(stream));
        out->max_depth = md;
        out->n_nodes = last[0] + last[1];
        out->root_ref = n <= kLeafMax ? ~(0 << 3 | n) : 0;
        out->n_leaves = n_refs;  // leaf references (> n_tri when slivers were split)
        float ms = 0.f;
        BVH_CHECK(cudaEventElapsedTime(&ms, e0, e1));
        out->build_ms = ms;
    }
done:
    // on success the stream was synchronised by the readback above
    const bool synced = err == cudaSuccess;
    dev_free(ref_tri, synced);
    dev_free(ref_piece, synced);
    dev_free(keys, synced);
    dev_free(keys_s, synced);
    dev_free(ids, synced);
    dev_free(ids_s, synced);
    dev_free(blo, synced);
    dev_free(bhi, synced);
    dev_free(blo_s, synced);
    dev_free(bhi_s, synced);
    dev_free(ilo, synced);
    dev_free(ihi, synced);
    dev_free(child, synced);
    dev_free(range, synced);
    dev_free(par_i, synced);
    dev_free(par_l, synced);
    dev_free(flags, synced);
    dev_free(dmax, synced);
    dev_free(is4, synced);
    dev_free(idx4, synced);
    dev_free(tmp, synced);
    dev_free(scan_tmp, synced);
    dev_free(sidx, synced);
    dev_free(cen, synced);
    dev_free(cen2, synced);
    dev_free(coop_jobs, synced);
    dev_free(coop_counts, synced);
    dev_free(tasks, synced);
    dev_free(node_counter, synced);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (err != cudaSuccess) {
        dev_free(out->nodes);
        dev_free(out->tri64);
        out->nodes = nullptr;
        out->tri64 = nullptr;
    }
    return err;
}

}  // namespace mcsbr_int
