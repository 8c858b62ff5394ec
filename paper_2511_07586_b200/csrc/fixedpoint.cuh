// Exact (order-independent) far-field reduction: 192-bit two's-complement
// fixed point, LSB 2^-kFxFrac.
//
// The reference makes its sweep reproducible by merging per-block
// accumulators in block order (solver_mc.cpp:212-216); a GPU that schedules
// paths dynamically cannot fix an fp64 summation order without serialising.
// Instead, MCSBR_REDUCE_EXACT rounds every term (one contribution's product
// with one frequency's phasor, per channel and re / im part) ONCE, to an
// integer multiple of 2^-120 (truncation toward zero, a property of the term
// alone), and adds integers: integer addition is associative, so the sums
// are the same bits whatever the order, launch grouping or number of shards.
// Range: |sum| < 2^71 (fault bit kFaultFixedRange beyond); the truncation
// error per term is < 2^-120 ~ 7.5e-37 (amplitudes are ~1e-9..1e3).
//
// Device accumulators: 3 x uint64 words per value (w0 least significant).
// Cross-rank form: 4 int64 limbs of 48 bits per value (the 192-bit pattern
// split at bits 48 / 96 / 144), which any integer all-reduce can sum for up
// to 2^15 ranks without overflow; host normalisation restores the carries.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define MCSBR_FX_HD __host__ __device__
#else
#define MCSBR_FX_HD
#endif

namespace mcsbr_fx {

constexpr int kFxFrac = 120;
constexpr uint64_t kLimbMask = (uint64_t{1} << 48) - 1;

// x -> 192-bit fixed point (truncated toward zero); returns false when |x|
// is out of range or x is not finite (the words are then zero)
MCSBR_FX_HD inline bool fx_from_double(double x, uint64_t w[3]) {
    w[0] = w[1] = w[2] = 0;
    uint64_t bits;
#ifdef __CUDA_ARCH__
    bits = static_cast<uint64_t>(__double_as_longlong(x));
#else
    __builtin_memcpy(&bits, &x, sizeof(bits));
#endif
    const bool neg = (bits >> 63) != 0;
    int ex = static_cast<int>((bits >> 52) & 0x7ff);
    uint64_t m = bits & ((uint64_t{1} << 52) - 1);
    if (ex == 0x7ff) return false;  // inf / nan
    if (ex == 0) {
        if (m == 0) return true;  // +-0
        ex = 1;                   // subnormal
    } else {
        m |= uint64_t{1} << 52;
    }
    int p = ex - 1075 + kFxFrac;  // bit position of m's least significant bit
    if (p < 0) {
        if (p <= -53) return true;  // below the LSB
        m >>= -p;
        p = 0;
    }
    if (p + 53 > 191) return false;  // |x| >= 2^71 (keep the sign bit free)
    const int wi = p >> 6, off = p & 63;
    w[wi] = m << off;
    if (off && wi + 1 < 3) w[wi + 1] = m >> (64 - off);
    if (neg) {  // two's complement of the 192-bit pattern
        w[0] = ~w[0];
        w[1] = ~w[1];
        w[2] = ~w[2];
        if (++w[0] == 0 && ++w[1] == 0) ++w[2];
    }
    return true;
}

#ifdef __CUDACC__
// a += b (mod 2^192), registers
__device__ __forceinline__ void fx_add(uint64_t a[3], const uint64_t b[3]) {
    asm("add.cc.u64 %0, %0, %3;\n\taddc.cc.u64 %1, %1, %4;\n\taddc.u64 %2, %2, %5;"
        : "+l"(a[0]), "+l"(a[1]), "+l"(a[2])
        : "l"(b[0]), "l"(b[1]), "l"(b[2]));
}

// *g += b (mod 2^192) with device atomics: every word's carry-out is added
// into the next word, so concurrent adds in any interleaving sum exactly
__device__ __forceinline__ void fx_atomic_add(unsigned long long* g, const uint64_t b[3]) {
    unsigned long long carry = 0;
    for (int i = 0; i < 3; ++i) {
        const unsigned long long add = b[i] + carry;
        unsigned long long next = (carry && add == 0) ? 1ull : 0ull;  // b[i] + carry wrapped
        if (add) {
            const unsigned long long old = atomicAdd(g + i, add);
            if (old + add < old) next += 1;
        }
        carry = next;
    }
}
#endif

// 192-bit pattern -> 4 limbs of 48 bits
MCSBR_FX_HD inline void fx_to_limbs(const uint64_t w[3], int64_t l[4]) {
    l[0] = static_cast<int64_t>(w[0] & kLimbMask);
    l[1] = static_cast<int64_t>(((w[0] >> 48) | (w[1] << 16)) & kLimbMask);
    l[2] = static_cast<int64_t>(((w[1] >> 32) | (w[2] << 32)) & kLimbMask);
    l[3] = static_cast<int64_t>((w[2] >> 16) & kLimbMask);
}

// sum of limbs (each the sum over ranks of 48-bit limbs) -> double: carries
// normalised, the 192-bit result read as two's complement, rounded to the
// nearest double from its top 64 significant bits
inline double fx_limbs_to_double(const int64_t l[4]) {
    uint64_t d[4];
    __int128 carry = 0;
    for (int i = 0; i < 4; ++i) {
        const __int128 t = static_cast<__int128>(l[i]) + carry;
        d[i] = static_cast<uint64_t>(t) & kLimbMask;
        carry = (t - static_cast<__int128>(d[i])) >> 48;
    }
    uint64_t w[3] = {d[0] | (d[1] << 48), (d[1] >> 16) | (d[2] << 32), (d[2] >> 32) | (d[3] << 16)};
    const bool neg = (w[2] >> 63) != 0;
    if (neg) {
        w[0] = ~w[0];
        w[1] = ~w[1];
        w[2] = ~w[2];
        if (++w[0] == 0 && ++w[1] == 0) ++w[2];
    }
    int top = -1;
    for (int i = 2; i >= 0 && top < 0; --i)
        if (w[i]) top = 64 * i + 63 - __builtin_clzll(w[i]);
    if (top < 0) return 0.0;
    // the 64 bits below and including `top`
    uint64_t m;
    const int lo = top - 63;
    if (lo <= 0) {  // top < 64: every bit is in w[0]
        m = w[0] << (-lo);
    } else {
        const int wi = lo >> 6, off = lo & 63;
        m = w[wi] >> off;
        if (off && wi + 1 < 3) m |= w[wi + 1] << (64 - off);
    }
    double v = static_cast<double>(m);
    v = __builtin_ldexp(v, lo - kFxFrac);
    return neg ? -v : v;
}

}  // namespace mcsbr_fx
