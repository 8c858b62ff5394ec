// Counter-based random streams for the path kernel.
//
// * Parity mode: the reference's SplitMix64 hash chain keyed by
//   (seed, stratum, sample, bounce, purpose) (proj/include/mcsbr/rng.hpp:19-44),
//   reproduced bit for bit (integer-only).
// * Statistical mode: Philox4x32-10 (Salmon et al., SC'11) keyed by
//   (seed, global ray index), counter = (bounce, purpose): a different but
//   equally valid stream, used when per-ray parity is not required.
#pragma once

#include <cstdint>

namespace mcsbr_dev {

enum : uint64_t { kLaunchU = 0x101, kLaunchV = 0x102, kBranch = 0x201, kRoulette = 0x202 };

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// rng.hpp:29-37.  The (seed, stratum, sample) prefix is shared by every draw
// of a path, so the kernel hashes it once per path and finishes per draw.
__host__ __device__ __forceinline__ uint64_t counter_prefix(uint64_t seed, uint64_t stratum,
                                                            uint64_t sample) {
    uint64_t h = mix64(seed ^ 0x2545f4914f6cdd1dull);
    h = mix64(h ^ stratum);
    return mix64(h ^ (sample + 0x632be59bd9b4e019ull));
}
__host__ __device__ __forceinline__ uint64_t counter_finish(uint64_t prefix, uint64_t bounce,
                                                            uint64_t purpose) {
    const uint64_t h = mix64(prefix ^ (bounce + 0x9e3779b97f4a7c15ull));
    return mix64(h ^ purpose);
}
// rng.hpp:40-44: 53 random bits -> [0, 1)
__host__ __device__ __forceinline__ double u53(uint64_t h) {
    return static_cast<double>(h >> 11) * 0x1.0p-53;
}

// Philox4x32-10
__host__ __device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
        const uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
        const uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
#else
        const uint64_t p0 = static_cast<uint64_t>(M0) * c[0], p1 = static_cast<uint64_t>(M1) * c[2];
        const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
        const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
#endif
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
        k0 += W0;
        k1 += W1;
    }
}

// Stat-mode draw: key = seed, counter = (ray index lo/hi, bounce, purpose).
__host__ __device__ __forceinline__ double philox_uniform(uint64_t seed, uint64_t ray,
                                                          uint32_t bounce, uint32_t purpose) {
    uint32_t c[4] = {static_cast<uint32_t>(ray), static_cast<uint32_t>(ray >> 32), bounce, purpose};
    philox4x32_10(c, static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
    const uint64_t h = (static_cast<uint64_t>(c[0]) << 32) | c[1];
    return u53(h);
}

}  // namespace mcsbr_dev
