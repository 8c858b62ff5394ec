// Bitwise check of the device V3 / double (dmath.cuh: shared-reciprocal
// div.rn.f64 fast path) against three plain IEEE divisions, over random
// operands spread across the whole exponent range plus zeros, denormals,
// infinities and NaNs.  Prints "mismatches N of M".
#include <cstdio>
#include <cstdint>
#include <cstring>
#include "../../paper_2511_07586_b200/csrc/dmath.cuh"
using namespace mcsbr_dev;

__device__ uint64_t mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ double pick(uint64_t h) {
    const uint32_t kind = h & 15;
    const uint64_t sign = (h >> 4 & 1) << 63;
    if (kind == 0) return __longlong_as_double(sign);                        // +-0
    if (kind == 1) return __longlong_as_double(sign | (h >> 12 & 0xfffffffffffffull));  // denormal
    if (kind == 2) return __longlong_as_double(sign | 0x7ff0000000000000ull);  // inf
    if (kind == 3 && (h & 0x300) == 0) return __longlong_as_double(0x7ff8000000000001ull);  // NaN
    if (kind < 8) {  // anywhere in the exponent range
        const uint64_t e = (h >> 5) % 2046 + 1;
        return __longlong_as_double(sign | e << 52 | (h >> 12 & 0xfffffffffffffull));
    }
    // the path kernel's range: |x| in [2^-40, 2^8]
    const uint64_t e = 1023 - 40 + (h >> 5) % 48;
    return __longlong_as_double(sign | e << 52 | (h >> 12 & 0xfffffffffffffull));
}
__global__ void check(uint64_t n, unsigned long long* bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t h = mix(i * 4 + 1);
        V3 a = {pick(mix(h)), pick(mix(h + 1)), pick(mix(h + 2))};
        const double s = pick(mix(h + 3));
        volatile double vs = s;
        const double sd = vs;
        const V3 r = a / sd;
        const double ex[3] = {a.x / sd, a.y / sd, a.z / sd};
        const double got[3] = {r.x, r.y, r.z};
        for (int k = 0; k < 3; ++k) {
            const bool both_nan = ex[k] != ex[k] && got[k] != got[k];
            if (!both_nan && __double_as_longlong(ex[k]) != __double_as_longlong(got[k])) atomicAdd(bad, 1ull);
        }
    }
}
int main() {
    unsigned long long* bad;
    cudaMallocManaged(&bad, 8);
    *bad = 0;
    const uint64_t n = 1ull << 28;
    check<<<148 * 8, 256>>>(n, bad);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("cuda error\n"); return 1; }
    printf("mismatches %llu of %llu\n", *bad, (unsigned long long)(3 * n));
    return *bad != 0;
}
