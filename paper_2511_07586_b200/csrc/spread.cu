// K4c: deferred phasor accumulation as a type-1 non-uniform DFT
// (SweepAccumulator::add, farfield.cpp:130-146, for uniform frequency grids).
//
// The direct kernel (trace.cu accumulate_kernel) evaluates, per record and
// frequency, z_f = e^{j k_f s} and four complex products: F x 16 FMAs plus
// F/FPL sincos per record (c5: ~3.2 k FP64 lane operations per record).  On
// a uniform grid k_f = kph0 + f kdph, so with f = fc + m (fc = F/2)
//
//     S_f = sum_r a_r e^{j k_f s_r} = sum_r c_r e^{j m u_r},
//     c_r = a_r e^{j kc s_r},  kc = kph0 + fc kdph,  u_r = kdph s_r,
//
// a type-1 NUDFT of the points u_r (mod 2 pi) onto the modes |m| <= F/2.
// Each record is spread onto a periodic grid of NG = 2F points (h = 2 pi/NG)
// with the "exponential of semicircle" kernel
//
//     psi(z) = exp(beta (sqrt(1 - z^2) - 1)),  z = (g - t) / 8,  |z| < 1,
//
// 16 points wide (t = u / h), beta = 2.30 * 16; then
//
//     S_f = (1 / Psi(m)) sum_g G_g e^{j m g h},   Psi(m) = sum_|i|<8 psi(i/8) cos(m i h)
//
// (nufft_finish_kernel).  psi on each of the 16 window points is a degree-13
// polynomial in the record's fractional offset (Chebyshev fit, host), so a
// kernel value is 13 FMAs; two lanes share the points of two records.
// Measured error of one term against e^{j m u}: 2e-13 relative at the worst
// mode (tools/nufft_error.py), below the rounding of the direct phase k_f s
// itself (|k_f s| ~ 1e4 rad: ~1e-12).  Cost per record: one sincos (c_r) and
// ~40 warp instructions, independent of F (the direct kernel: ~3 k lane
// operations per record at F = 128).
//
// Lossy paths (Im s > 0): u_r is complex, t -> t + j eta, and the kernel is
// evaluated at the complex offset: |eta| <= 0.1 cells by the polynomial's
// continuation (4.5e-13), <= 0.5 by the kernel's own analytic continuation
// (csqrt + exp, 2.2e-12), larger ones (strongly attenuated paths; none in c5)
// are added directly, lanes over frequencies, into the sums.
// Records are bucketed by incidence first (bucket_*_kernel) so that a warp's
// span is one incidence.
//
// Layout: each warp owns a private grid [8][NG] doubles in shared memory
// (4 complex channels x NG points; shared-memory fp64 atomics are CAS loops
// on sm_100, so no two warps share one) and flushes it with fp64 atomics into
// the per-incidence grid in HBM whenever its record span changes incidence.
// Lane (i, hh) = (lane & 15, lane >> 4) owns window point i and channels
// 2hh, 2hh+1: 16 points x 2 halves = the whole warp, no idle lanes.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "dmath.cuh"
#include "internal.h"
#include "physics.cuh"

namespace mcsbr_int {
namespace {

using namespace mcsbr_dev;

constexpr int kRecWords = 12;  // contribution record: amp[4], s (re, im), incidence (pathcore.cuh kRecD2)
constexpr int kSt = 6;         // staged record: c[4], (t, eta), incidence
constexpr int kPolyN = kNufftPolyN;
#ifndef MCSBR_SPREAD_POLY
#define MCSBR_SPREAD_POLY estrin  // A/B: -DMCSBR_SPREAD_POLY=horner
#endif

__device__ __forceinline__ Cx csqrt_pos(Cx q) {  // principal root, Re q > 0 (no cancellation)
    const double r = sqrt(__fma_rn(q.re, q.re, q.im * q.im));
    const double sr = sqrt(0.5 * (r + q.re));
    return {sr, q.im / (2.0 * sr)};
}

// The same polynomial by Estrin's scheme: 16 operations in a dependency
// chain 4 deep instead of Horner's 13 (the spread kernel's top stall is
// the fixed-latency 'wait' on DFMA chains); the value differs from Horner's
// by rounding only (~1e-16 relative, the kernel fit itself is 2e-13)
__device__ __forceinline__ double estrin(const double (&cf)[kPolyN], double x) {
    static_assert(kPolyN == 14, "estrin() is written for degree 13");
    const double x2 = x * x, x4 = x2 * x2, x8 = x4 * x4;
    const double p0 = __fma_rn(cf[1], x, cf[0]), p1 = __fma_rn(cf[3], x, cf[2]);
    const double p2 = __fma_rn(cf[5], x, cf[4]), p3 = __fma_rn(cf[7], x, cf[6]);
    const double p4 = __fma_rn(cf[9], x, cf[8]), p5 = __fma_rn(cf[11], x, cf[10]);
    const double p6 = __fma_rn(cf[13], x, cf[12]);
    const double q0 = __fma_rn(p1, x2, p0), q1 = __fma_rn(p3, x2, p2), q2 = __fma_rn(p5, x2, p4);
    const double r0 = __fma_rn(q1, x4, q0), r1 = __fma_rn(p6, x4, q2);
    return __fma_rn(r1, x8, r0);
}

__device__ __forceinline__ double horner(const double (&cf)[kPolyN], double x) {
    double w = cf[kPolyN - 1];
#pragma unroll
    for (int k = kPolyN - 2; k >= 0; --k) w = __fma_rn(w, x, cf[k]);
    return w;
}

// the same polynomial at x + j y (its analytic continuation, for a complex
// offset; accurate to ~4e-13 for |y| <= 0.2, tools/nufft_error.py)
__device__ __forceinline__ Cx horner_c(const double (&cf)[kPolyN], double x, double y) {
    double wr = cf[kPolyN - 1], wi = 0.0;
#pragma unroll
    for (int k = kPolyN - 2; k >= 0; --k) {
        const double nr = __fma_rn(wr, x, __fma_rn(-wi, y, cf[k]));
        wi = __fma_rn(wr, y, wi * x);
        wr = nr;
    }
    return {wr, wi};
}

// grid[row][g] += w * c for this lane's two channels (rows: re, im, re, im);
// all loads first (the rows cannot alias, the compiler cannot know)
__device__ __forceinline__ void add_real(double* Gh, uint32_t ng, int g, double w, double2 c0, double2 c1) {
    double v0 = Gh[g], v1 = Gh[ng + g], v2 = Gh[2 * ng + g], v3 = Gh[3 * ng + g];
    Gh[g] = __fma_rn(w, c0.x, v0);
    Gh[ng + g] = __fma_rn(w, c0.y, v1);
    Gh[2 * ng + g] = __fma_rn(w, c1.x, v2);
    Gh[3 * ng + g] = __fma_rn(w, c1.y, v3);
}

__device__ __forceinline__ void add_cx(double* Gh, uint32_t ng, int g, Cx w, double2 c0, double2 c1) {
    double v0 = Gh[g], v1 = Gh[ng + g], v2 = Gh[2 * ng + g], v3 = Gh[3 * ng + g];
    Gh[g] = __fma_rn(w.re, c0.x, __fma_rn(-w.im, c0.y, v0));
    Gh[ng + g] = __fma_rn(w.re, c0.y, __fma_rn(w.im, c0.x, v1));
    Gh[2 * ng + g] = __fma_rn(w.re, c1.x, __fma_rn(-w.im, c1.y, v2));
    Gh[3 * ng + g] = __fma_rn(w.re, c1.y, __fma_rn(w.im, c1.x, v3));
}

__global__ void __launch_bounds__(64) spread_kernel(TraceParams P, NufftPlan Q) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t ng = Q.ng;
    double* G = smem + static_cast<size_t>(warp) * (8 * ng + 32 * 2 * kSt);
    double2* st = reinterpret_cast<double2*>(G + 8 * ng);
    const int pi = lane & 15, hh = lane >> 4;
    double* Gh = G + 4 * hh * ng;  // this lane's rows: channel 2hh (re, im), 2hh + 1 (re, im)
    double cf[kPolyN];             // psi on this lane's window point, a polynomial in 2 delta - 1
#pragma unroll
    for (int k = 0; k < kPolyN; ++k) cf[k] = Q.coef[pi * kPolyN + k];
    for (uint32_t i = lane; i < 8 * ng; i += 32) G[i] = 0.0;
    const uint64_t n_all = *P.rec_count;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicMax(P.rec_count + 1, n_all);  // peak for the host
    const uint64_t n = min(n_all, P.rec_cap);
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * 2, gw = static_cast<uint64_t>(blockIdx.x) * 2 + warp;
    uint64_t span = ((n + nw - 1) / nw + 31) & ~31ull;
    span = span < 512 ? 512 : span;
    const double2* recs = reinterpret_cast<const double2*>(P.recs);
    const double dng = static_cast<double>(ng), beta = Q.beta;
    __syncwarp();
    for (uint64_t r0 = gw * span; r0 < n; r0 += nw * span) {
        const uint64_t r1 = min(r0 + span, n);
        uint32_t cur = 0xffffffffu;
        auto flush = [&]() {
            __syncwarp();
            if (cur == 0xffffffffu) return;
            double* out = Q.grid + static_cast<size_t>(cur) * 8 * ng;
            for (uint32_t i = lane; i < 8 * ng; i += 32) {
                const double v = G[i];
                if (v != 0.0) {
                    atomicAdd(out + i, v);
                    G[i] = 0.0;
                }
            }
            __syncwarp();
        };
        // software pipeline: the next batch's record (and the index after
        // it) are loaded into registers while this batch is spread
        auto rec_index = [&](uint64_t r) -> uint64_t { return Q.idx ? Q.idx[r] : r; };
        double2 raw[6];
        auto load_raw = [&](uint64_t ri) {
            const double2* r = recs + ri * (kRecWords / 2);
#pragma unroll
            for (int k = 0; k < 6; ++k) raw[k] = __ldcs(r + k);
        };
        uint64_t ri_next = 0;
        if (r0 + lane < r1) load_raw(rec_index(r0 + lane));
        if (r0 + 32 + lane < r1) ri_next = rec_index(r0 + 32 + lane);
        for (uint64_t rb = r0; rb < r1; rb += 32) {
            const uint32_t cnt = static_cast<uint32_t>(min(static_cast<uint64_t>(32), r1 - rb));
            if (static_cast<uint32_t>(lane) < cnt) {
                const double2 sv = raw[4];
                const Cx e = polar_la(Q.kc * sv.x, -(Q.kc * sv.y));  // e^{j kc s}
                double2* t = st + lane * kSt;
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    const Cx c = Cx{raw[ch].x, raw[ch].y} * e;
                    t[ch] = make_double2(c.re, c.im);
                }
                double u = sv.x * Q.u2t;
                u = __fma_rn(-dng, floor(u / dng), u);  // [0, NG)
                if (u >= dng) u -= dng;
                t[4] = make_double2(u, sv.y * Q.u2t);
                t[5] = raw[5];
            }
            __syncwarp();
            if (rb + 32 + lane < r1) load_raw(ri_next);
            if (rb + 64 + lane < r1) ri_next = rec_index(rb + 64 + lane);
            for (uint32_t j = 0; j < cnt;) {
                const double2* t = st + j * kSt;
                const double2 te = t[4];
                const uint32_t a = static_cast<uint32_t>(__double_as_longlong(t[5].x));
                if (a != cur) {
                    flush();
                    cur = a;
                }
                const double g0 = ceil(te.x - 8.0);
                int g = static_cast<int>(g0) + pi;
                g = g < 0 ? g + static_cast<int>(ng) : (g >= static_cast<int>(ng) ? g - static_cast<int>(ng) : g);
                const double2 c0 = t[2 * hh], c1 = t[2 * hh + 1];
                // two records of one incidence with small imaginary offsets:
                // lane (pi, hh) evaluates record j + hh's kernel value at point
                // pi (half the Horner work, two independent chains), then both
                // are added in turn
                if (j + 1 < cnt && fabs(te.y) <= Q.eta_poly) {
                    const double2* t1 = t + kSt;
                    const double2 te1 = t1[4];
                    if (fabs(te1.y) <= Q.eta_poly && static_cast<uint32_t>(__double_as_longlong(t1[5].x)) == a) {
                        const double g01 = ceil(te1.x - 8.0);
                        const double x = hh ? __fma_rn(2.0, g01 - te1.x, 15.0) : __fma_rn(2.0, g0 - te.x, 15.0);
                        int g1 = static_cast<int>(g01) + pi;
                        g1 = g1 < 0 ? g1 + static_cast<int>(ng) : (g1 >= static_cast<int>(ng) ? g1 - static_cast<int>(ng) : g1);
                        const double2 d0 = t1[2 * hh], d1 = t1[2 * hh + 1];
                        if (te.y == 0.0 && te1.y == 0.0) {
                            const double w = MCSBR_SPREAD_POLY(cf, x);
                            const double wo = __shfl_xor_sync(0xffffffffu, w, 16);
                            add_real(Gh, ng, g, hh ? wo : w, c0, c1);
                            __syncwarp();
                            add_real(Gh, ng, g1, hh ? w : wo, d0, d1);
                        } else {
                            const Cx w = horner_c(cf, x, -2.0 * (hh ? te1.y : te.y));
                            const Cx wo = {__shfl_xor_sync(0xffffffffu, w.re, 16), __shfl_xor_sync(0xffffffffu, w.im, 16)};
                            add_cx(Gh, ng, g, hh ? wo : w, c0, c1);
                            __syncwarp();
                            add_cx(Gh, ng, g1, hh ? w : wo, d0, d1);
                        }
                        __syncwarp();
                        j += 2;
                        continue;
                    }
                }
                const double d = g0 + static_cast<double>(pi) - te.x;  // [-8, 8)
                const double z = d * 0.125;
                // delta = g0 - t + 8 in [0, 1): psi((delta + pi - 8) / 8) by Horner
                // in x = 2 delta - 1 (+ j 2 Im delta for a complex offset)
                const double x = __fma_rn(2.0, g0 - te.x, 15.0);
                if (te.y == 0.0) {
                    add_real(Gh, ng, g, MCSBR_SPREAD_POLY(cf, x), c0, c1);
                } else if (fabs(te.y) <= Q.eta_poly) {
                    add_cx(Gh, ng, g, horner_c(cf, x, -2.0 * te.y), c0, c1);
                } else if (fabs(te.y) <= Q.eta_max) {
                    // complex offset: psi at (d - j eta) / 8
                    const double zi = -te.y * 0.125;
                    const Cx q = {__fma_rn(-z, z, __fma_rn(zi, zi, 1.0)), -2.0 * z * zi};
                    Cx w = {0.0, 0.0};
                    if (fabs(z) < 1.0) {
                        const Cx sq = csqrt_pos(q);
                        w = polar_la(beta * sq.im, beta * (sq.re - 1.0));
                    }
                    add_cx(Gh, ng, g, w, c0, c1);
                } else {
                    // strongly attenuated path: direct phasors, lanes over
                    // frequencies, straight into the sums (rare)
                    double* out = P.sums + sums_row(P, a) * P.nf * 8;
                    const double hstep = 2.0 * M_PI / dng;
                    for (uint32_t f = lane; f < P.nf; f += 32) {
                        const double m = static_cast<double>(static_cast<int>(f) - static_cast<int>(Q.fc)) * hstep;
                        const Cx z2 = polar_la(m * te.x, -(m * te.y));
#pragma unroll
                        for (int ch = 0; ch < 4; ++ch) {
                            const Cx v = Cx{t[ch].x, t[ch].y} * z2;
                            atomicAdd(out + f * 8 + 2 * ch, v.re);
                            atomicAdd(out + f * 8 + 2 * ch + 1, v.im);
                        }
                    }
                }
                __syncwarp();
                ++j;
            }
        }
        flush();
    }
}

// Records by incidence (a counting sort of their indices): the path kernel
// appends records in completion order, in which incidences interleave (c5:
// runs of ~50 records), and every incidence change flushes a warp's grid.
__global__ void __launch_bounds__(256) bucket_count_kernel(TraceParams P, NufftPlan Q, uint32_t n_inc) {
    extern __shared__ uint32_t hist[];
    for (uint32_t i = threadIdx.x; i < n_inc; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint64_t n = min(static_cast<uint64_t>(*P.rec_count), P.rec_cap);
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t r0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u); r0 < n;
         r0 += static_cast<uint64_t>(gridDim.x) * blockDim.x) {  // warp-uniform trip count
        const uint64_t r = r0 + lane;
        const uint32_t a = r < n ? P.rec_inc[r] : 0xffffffffu;
        // warp-aggregated: consecutive records are mostly one incidence
        const unsigned same = __match_any_sync(0xffffffffu, a);
        if (a != 0xffffffffu && lane == static_cast<uint32_t>(__ffs(same) - 1))
            atomicAdd(&hist[a], static_cast<uint32_t>(__popc(same)));
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n_inc; i += blockDim.x)
        if (hist[i]) atomicAdd(&Q.bucket[i], hist[i]);
}

__global__ void __launch_bounds__(1024) bucket_prefix_kernel(NufftPlan Q, uint32_t n_inc) {
    __shared__ uint32_t part[1024];
    const uint32_t per = (n_inc + 1023) / 1024, b = threadIdx.x * per, e = min(n_inc, b + per);
    uint32_t s = 0;
    for (uint32_t i = b; i < e; ++i) s += Q.bucket[i];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (int i = 0; i < 1024; ++i) {
            const uint32_t v = part[i];
            part[i] = acc;
            acc += v;
        }
    }
    __syncthreads();
    uint32_t acc = part[threadIdx.x];
    for (uint32_t i = b; i < e; ++i) {
        const uint32_t v = Q.bucket[i];
        Q.bucket[n_inc + 1 + i] = acc;  // cursor
        acc += v;
    }
}

// each block: a tile of 4096 records, one cursor reservation per incidence met
__global__ void __launch_bounds__(256) bucket_scatter_kernel(TraceParams P, NufftPlan Q, uint32_t n_inc) {
    extern __shared__ uint32_t hist[];  // [n_inc] counts, then bases
    uint32_t* base = hist + n_inc;
    constexpr uint32_t kTile = 4096;
    const uint64_t n = min(static_cast<uint64_t>(*P.rec_count), P.rec_cap);
    uint32_t* cursor = Q.bucket + n_inc + 1;
    for (uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kTile; t0 < n; t0 += static_cast<uint64_t>(gridDim.x) * kTile) {
        for (uint32_t i = threadIdx.x; i < n_inc; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        uint32_t av[kTile / 256];
#pragma unroll
        for (int k = 0; k < static_cast<int>(kTile / 256); ++k) {
            const uint64_t r = t0 + k * 256 + threadIdx.x;
            av[k] = r < n ? P.rec_inc[r] : 0xffffffffu;
            const unsigned same = __match_any_sync(0xffffffffu, av[k]);
            if (av[k] != 0xffffffffu && (threadIdx.x & 31) == __ffs(same) - 1)
                atomicAdd(&hist[av[k]], static_cast<uint32_t>(__popc(same)));
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n_inc; i += blockDim.x) {
            base[i] = hist[i] ? atomicAdd(&cursor[i], hist[i]) : 0;
            hist[i] = 0;
        }
        __syncthreads();
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int k = 0; k < static_cast<int>(kTile / 256); ++k) {
            const unsigned same = __match_any_sync(0xffffffffu, av[k]);
            const int leader = __ffs(same) - 1;
            uint32_t off = 0;
            if (av[k] != 0xffffffffu && lane == leader) off = atomicAdd(&hist[av[k]], static_cast<uint32_t>(__popc(same)));
            off = __shfl_sync(0xffffffffu, off, leader);
            if (av[k] == 0xffffffffu) continue;
            const uint32_t pos = base[av[k]] + off + __popc(same & ((1u << lane) - 1u));
            Q.idx[pos] = static_cast<uint32_t>(t0 + k * 256 + threadIdx.x);
        }
        __syncthreads();
    }
}

// S_f += (1 / Psi(m)) sum_g G_g e^{j m g h}, one block per incidence of the group
__global__ void __launch_bounds__(256) nufft_finish_kernel(TraceParams P, NufftPlan Q) {
    extern __shared__ double sh[];
    const uint32_t ng = Q.ng, a = blockIdx.x;
    double* G = sh;
    double* cs = sh + 8 * ng;
    double* sn = cs + ng;
    const double* src = Q.grid + static_cast<size_t>(a) * 8 * ng;
    for (uint32_t i = threadIdx.x; i < 8 * ng; i += blockDim.x) G[i] = src[i];
    for (uint32_t i = threadIdx.x; i < ng; i += blockDim.x) sincospi(2.0 * i / ng, &sn[i], &cs[i]);
    __syncthreads();
    double* out = P.sums + sums_row(P, a) * P.nf * 8;
    for (uint32_t o = threadIdx.x; o < P.nf * 4; o += blockDim.x) {
        const uint32_t f = o >> 2, k = o & 3;
        const int m = static_cast<int>(f) - static_cast<int>(Q.fc);
        const uint32_t step = static_cast<uint32_t>(((m % static_cast<int>(ng)) + static_cast<int>(ng)) % static_cast<int>(ng));
        const double* gr = G + 2 * k * ng;
        const double* gi = gr + ng;
        double sr = 0.0, si = 0.0;
        uint32_t idx = 0;
        for (uint32_t g = 0; g < ng; ++g) {
            const double c = cs[idx], s = sn[idx];
            sr = __fma_rn(gr[g], c, __fma_rn(-gi[g], s, sr));
            si = __fma_rn(gr[g], s, __fma_rn(gi[g], c, si));
            idx += step;
            if (idx >= ng) idx -= ng;
        }
        const double inv = Q.inv_hat[f];
        out[f * 8 + 2 * k] += sr * inv;
        out[f * 8 + 2 * k + 1] += si * inv;
    }
}

}  // namespace

// host: the per-point polynomials of psi (Chebyshev interpolation at
// kPolyN points on delta in [0, 1], converted to monomials in x = 2 delta - 1;
// the coefficients stay below 1, so Horner is stable: tools/nufft_error.py)
// and 1 / Psi(m) from the same polynomials at x = -1 (a record on a grid point)
void nufft_tables(uint32_t nf, uint32_t ng, double beta, std::vector<double>& inv_hat, std::vector<double>& coef) {
    constexpr int N = kPolyN;
    coef.assign(16 * N, 0.0);
    const long double pi_l = 3.141592653589793238462643383279502884L;
    for (int i = 0; i < 16; ++i) {
        long double fx[N], c[N];
        for (int j = 0; j < N; ++j) {
            const long double x = std::cos(pi_l * (j + 0.5L) / N);
            const long double z = ((x + 1.0L) / 2.0L + i - 8) / 8.0L;
            const long double q = 1.0L - z * z;
            fx[j] = q > 0 ? std::exp(static_cast<long double>(beta) * (std::sqrt(q) - 1.0L)) : 0.0L;
        }
        for (int k = 0; k < N; ++k) {  // Chebyshev coefficients
            long double acc = 0;
            for (int j = 0; j < N; ++j) acc += fx[j] * std::cos(pi_l * k * (j + 0.5L) / N);
            c[k] = acc * 2.0L / N;
        }
        c[0] *= 0.5L;
        long double tm1[N] = {}, t0[N] = {}, mono[N] = {};  // T_{k-1}, T_k as monomials
        t0[0] = 1;
        for (int k = 0; k < N; ++k) {
            for (int d = 0; d < N; ++d) mono[d] += c[k] * t0[d];
            long double t1[N] = {};
            for (int d = 0; d < N; ++d) {
                if (d + 1 < N) t1[d + 1] += (k == 0 ? 1.0L : 2.0L) * t0[d];
                if (k > 0) t1[d] -= tm1[d];
            }
            for (int d = 0; d < N; ++d) {
                tm1[d] = t0[d];
                t0[d] = t1[d];
            }
        }
        for (int d = 0; d < N; ++d) coef[i * N + d] = static_cast<double>(mono[d]);
    }
    const uint32_t fc = nf / 2;
    const double h = 2.0 * M_PI / ng;
    inv_hat.assign(nf, 0.0);
    for (uint32_t f = 0; f < nf; ++f) {
        const double m = static_cast<double>(static_cast<int>(f) - static_cast<int>(fc));
        double acc = 0.0;
        for (int i = 0; i < 16; ++i) {
            double w = coef[i * N + N - 1];
            for (int k = N - 2; k >= 0; --k) w = w * -1.0 + coef[i * N + k];
            acc += w * std::cos(m * (i - 8) * h);
        }
        inv_hat[f] = 1.0 / acc;
    }
}

bool nufft_supported(uint32_t nf) { return nf >= 32 && nf <= 256; }

size_t nufft_grid_values(uint32_t nf) { return 8ull * 2 * nf; }

cudaError_t launch_spread(const TraceParams& p, const NufftPlan& q, uint32_t n_inc, int device_sms,
                          cudaStream_t stream, uint64_t* launches, uint64_t expected_records) {
    cudaError_t e = cudaMemsetAsync(q.grid, 0, sizeof(double) * 8 * q.ng * n_inc, stream);
    if (e != cudaSuccess) return e;
    NufftPlan qs = q;
    if (q.idx && p.rec_inc && n_inc > 1 && n_inc <= kNufftSortMaxInc) {
        if ((e = cudaMemsetAsync(q.bucket, 0, sizeof(uint32_t) * 2 * (n_inc + 1), stream)) != cudaSuccess) return e;
        bucket_count_kernel<<<device_sms * 4, 256, sizeof(uint32_t) * n_inc, stream>>>(p, q, n_inc);
        bucket_prefix_kernel<<<1, 1024, 0, stream>>>(q, n_inc);
        bucket_scatter_kernel<<<device_sms * 4, 256, sizeof(uint32_t) * 2 * n_inc, stream>>>(p, q, n_inc);
        if (launches) *launches += 3;
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    } else {
        qs.idx = nullptr;  // one incidence (or too many to bucket): record order
    }
    const size_t smem = sizeof(double) * 2 * (8 * q.ng + 32 * 2 * kSt);
    if (smem > 48 * 1024) {
        e = cudaFuncSetAttribute(spread_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    int per_sm = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spread_kernel, 64, smem);
    if (e != cudaSuccess) return e;
    per_sm = std::max(1, per_sm);
    // one wave; more when the launch carries many records per warp (balance)
    const uint64_t per_wave = static_cast<uint64_t>(device_sms) * per_sm * 2 * 8192;
    const unsigned waves = static_cast<unsigned>(std::min<uint64_t>(4, std::max<uint64_t>(1, expected_records / per_wave)));
    spread_kernel<<<static_cast<unsigned>(device_sms) * per_sm * waves, 64, smem, stream>>>(p, qs);
    if (launches) ++*launches;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const size_t smem2 = sizeof(double) * 10 * q.ng;
    if (smem2 > 48 * 1024) {
        e = cudaFuncSetAttribute(nufft_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem2));
        if (e != cudaSuccess) return e;
    }
    nufft_finish_kernel<<<n_inc, 256, smem2, stream>>>(p, q);
    if (launches) ++*launches;
    return cudaGetLastError();
}

}  // namespace mcsbr_int
