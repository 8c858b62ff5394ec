// Device sort and scan for the BVH build (bvh.cu): a stable LSD radix sort
// of (u64 Morton key, u32 id) pairs and an exclusive u32 prefix sum.
//
// Radix sort: 8-bit digits, one pass per digit of the key width, ping-pong
// buffers.  Per pass:
//   1. digit_hist_kernel   one block per 4096-element tile counts its digits
//                          (shared-memory atomics) -> hist[digit][tile];
//   2. digit_scan_kernel   (digit-major, so the exclusive prefix of
//                          hist[d][t] is where tile t's digit-d elements go):
//                          one warp per digit, its base from the digit totals
//                          the histogram kernel accumulated;
//   3. digit_scatter_kernel the tile again, each warp owning 512 consecutive
//                          elements in 16 rounds of 32: __match_any_sync
//                          groups a round's lanes by digit, per-warp digit
//                          counts are prefixed across the block's warps in
//                          warp order, so every element's destination keeps
//                          the input order within its digit (stable), and
//                          equal keys stay in id order -- the same
//                          permutation as any stable sort.
// Traffic per pass: the keys and ids read twice, written once (~36 MB per
// pass at 1 M references); a 1 M-reference sort is ~8 x 3 short launches.
//
// Scan: tile sums (4096 per block), an exclusive scan of the tile sums in
// one block, then each tile scanned with its offset.
#include <algorithm>
#include <cstdint>
#include <utility>

#include "internal.h"

namespace mcsbr_int {

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;  // 4096
constexpr int kWarps = kThreads / 32;
constexpr int kWarpSpan = kTile / kWarps;  // 512 consecutive elements per warp
constexpr int kRadix = 256;

__global__ void __launch_bounds__(kThreads) digit_hist_kernel(const uint64_t* __restrict__ keys, uint32_t n,
                                                              int shift, uint32_t n_tiles,
                                                              uint32_t* __restrict__ hist,
                                                              uint32_t* __restrict__ totals) {
    __shared__ uint32_t h[kRadix];
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kTile;
#pragma unroll 4
    for (int k = 0; k < kItems; ++k) {
        const uint64_t i = base + static_cast<uint64_t>(k) * kThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & 0xff], 1u);
    }
    __syncthreads();
    const uint32_t c = h[threadIdx.x];
    hist[static_cast<uint64_t>(threadIdx.x) * n_tiles + blockIdx.x] = c;
    if (c) atomicAdd(totals + threadIdx.x, c);
}

// digit offsets for the scatter: one warp per digit d.  The digit's base is
// the sum of the totals of the digits below it; its row hist[d][0..T) is
// scanned 32 tiles at a time.  (A single block scanning all 256 x T entries
// took ~10x longer: it was ~70% of a 1 M-element sort.)
__global__ void __launch_bounds__(256) digit_scan_kernel(const uint32_t* __restrict__ hist,
                                                         const uint32_t* __restrict__ totals, uint32_t n_tiles,
                                                         uint32_t* __restrict__ offs) {
    const int lane = threadIdx.x & 31;
    const uint32_t d = blockIdx.x * 8 + (threadIdx.x >> 5);
    uint32_t base = 0;
#pragma unroll
    for (int k = 0; k < kRadix / 32; ++k) {
        const uint32_t dd = static_cast<uint32_t>(lane) * (kRadix / 32) + k;
        if (dd < d) base += totals[dd];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) base += __shfl_xor_sync(0xffffffffu, base, o);
    const uint32_t* row = hist + static_cast<uint64_t>(d) * n_tiles;
    uint32_t* orow = offs + static_cast<uint64_t>(d) * n_tiles;
    for (uint32_t t0 = 0; t0 < n_tiles; t0 += 32) {
        const uint32_t t = t0 + lane;
        const uint32_t v = t < n_tiles ? row[t] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (t < n_tiles) orow[t] = base + x - v;
        base += __shfl_sync(0xffffffffu, x, 31);
    }
}

// exclusive scan of n values in ONE block of 1024 threads (each thread a
// contiguous segment); used for the tile sums / digit histograms (<= a few
// hundred thousand values)
__global__ void __launch_bounds__(1024) scan_one_block_kernel(const uint32_t* __restrict__ in,
                                                               uint32_t* __restrict__ out, uint32_t n) {
    __shared__ uint32_t warp_tot[32];
    const uint32_t t = threadIdx.x;
    const uint32_t per = (n + 1023) / 1024;
    const uint32_t a = min(n, t * per), b = min(n, a + per);
    uint32_t sum = 0;
    for (uint32_t i = a; i < b; ++i) sum += in[i];
    // block-wide exclusive scan of the segment sums
    const int lane = t & 31, warp = t >> 5;
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = warp_tot[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        warp_tot[lane] = w;  // inclusive
    }
    __syncthreads();
    uint32_t run = x - sum + (warp ? warp_tot[warp - 1] : 0u);
    for (uint32_t i = a; i < b; ++i) {
        const uint32_t v = in[i];
        out[i] = run;
        run += v;
    }
}

__global__ void __launch_bounds__(kThreads) digit_scatter_kernel(const uint64_t* __restrict__ keys_in,
                                                                 const uint32_t* __restrict__ vals_in, uint32_t n,
                                                                 int shift, uint32_t n_tiles,
                                                                 const uint32_t* __restrict__ offs,
                                                                 uint64_t* __restrict__ keys_out,
                                                                 uint32_t* __restrict__ vals_out) {
    __shared__ uint32_t wcount[kWarps][kRadix];  // per-warp digit counts, then per-warp write cursors
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kWarps * kRadix; i += kThreads) (&wcount[0][0])[i] = 0;
    __syncthreads();
    const uint64_t w0 = static_cast<uint64_t>(blockIdx.x) * kTile + static_cast<uint64_t>(warp) * kWarpSpan;
    const unsigned lt = (1u << lane) - 1u;
    // A: per-warp digit counts (the lowest lane of each digit group adds the group)
    for (int r = 0; r < kWarpSpan / 32; ++r) {
        const uint64_t i = w0 + static_cast<uint64_t>(r) * 32 + lane;
        const bool in = i < n;
        const uint32_t d = in ? static_cast<uint32_t>((keys_in[i] >> shift) & 0xff) : kRadix;
        const unsigned grp = __match_any_sync(0xffffffffu, d);
        if (in && (grp & lt) == 0) wcount[warp][d] += __popc(grp);
        __syncwarp();
    }
    __syncthreads();
    // B: write cursors: the tile's digit offset + the counts of earlier warps
    {
        const uint32_t d = threadIdx.x;  // kThreads == kRadix
        uint32_t run = offs[static_cast<uint64_t>(d) * n_tiles + blockIdx.x];
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t c = wcount[w][d];
            wcount[w][d] = run;
            run += c;
        }
    }
    __syncthreads();
    // C: scatter in input order
    for (int r = 0; r < kWarpSpan / 32; ++r) {
        const uint64_t i = w0 + static_cast<uint64_t>(r) * 32 + lane;
        const bool in = i < n;
        uint64_t k = 0;
        uint32_t v = 0;
        if (in) {
            k = keys_in[i];
            v = vals_in[i];
        }
        const uint32_t d = in ? static_cast<uint32_t>((k >> shift) & 0xff) : kRadix;
        const unsigned grp = __match_any_sync(0xffffffffu, d);
        uint32_t dst = 0;
        if (in) dst = wcount[warp][d] + __popc(grp & lt);
        __syncwarp();
        if (in && (grp & lt) == 0) wcount[warp][d] += __popc(grp);
        __syncwarp();
        if (in) {
            keys_out[dst] = k;
            vals_out[dst] = v;
        }
    }
}

__global__ void __launch_bounds__(kThreads) tile_sum_kernel(const uint32_t* __restrict__ in, uint32_t n,
                                                            uint32_t* __restrict__ sums) {
    __shared__ uint32_t ws[kWarps];
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kTile;
    uint32_t s = 0;
    for (int k = 0; k < kItems; ++k) {
        const uint64_t i = base + static_cast<uint64_t>(k) * kThreads + threadIdx.x;
        if (i < n) s += in[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < kWarps; ++w) t += ws[w];
        sums[blockIdx.x] = t;
    }
}

// each thread scans kItems consecutive values of the tile; thread partials
// are scanned block-wide and offset by the tile's exclusive prefix
__global__ void __launch_bounds__(kThreads) tile_scan_kernel(const uint32_t* __restrict__ in, uint32_t n,
                                                             const uint32_t* __restrict__ tile_off,
                                                             uint32_t* __restrict__ out) {
    __shared__ uint32_t warp_tot[kWarps];
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kTile + static_cast<uint64_t>(threadIdx.x) * kItems;
    uint32_t v[kItems];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const uint64_t i = base + k;
        v[k] = i < n ? in[i] : 0u;
        s += v[k];
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    uint32_t before = 0;
    for (int w = 0; w < warp; ++w) before += warp_tot[w];
    uint32_t run = tile_off[blockIdx.x] + before + x - s;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const uint64_t i = base + k;
        if (i < n) out[i] = run;
        run += v[k];
    }
}

}  // namespace

size_t radix_sort_temp_bytes(uint32_t n) {
    const uint64_t tiles = (static_cast<uint64_t>(n) + kTile - 1) / kTile;
    return sizeof(uint32_t) * (2 * kRadix * std::max<uint64_t>(tiles, 1) + 8 * kRadix);  // + per-pass totals
}

cudaError_t radix_sort_pairs(uint64_t* keys, uint64_t* keys_alt, uint32_t* vals, uint32_t* vals_alt, uint32_t n,
                             int key_bits, void* temp, cudaStream_t stream, bool* result_in_alt) {
    *result_in_alt = false;
    if (n == 0) return cudaSuccess;
    const uint32_t tiles = static_cast<uint32_t>((static_cast<uint64_t>(n) + kTile - 1) / kTile);
    uint32_t* hist = static_cast<uint32_t*>(temp);
    uint32_t* offs = hist + static_cast<uint64_t>(kRadix) * tiles;
    uint32_t* totals = offs + static_cast<uint64_t>(kRadix) * tiles;  // [8 passes][256]
    const int passes = (key_bits + 7) / 8;
    if (passes > 8) return cudaErrorInvalidValue;
    cudaError_t z = cudaMemsetAsync(totals, 0, sizeof(uint32_t) * kRadix * passes, stream);
    if (z != cudaSuccess) return z;
    uint64_t *kin = keys, *kout = keys_alt;
    uint32_t *vin = vals, *vout = vals_alt;
    for (int shift = 0; shift < key_bits; shift += 8) {
        uint32_t* tot = totals + kRadix * (shift / 8);
        digit_hist_kernel<<<tiles, kThreads, 0, stream>>>(kin, n, shift, tiles, hist, tot);
        digit_scan_kernel<<<kRadix / 8, 256, 0, stream>>>(hist, tot, tiles, offs);
        digit_scatter_kernel<<<tiles, kThreads, 0, stream>>>(kin, vin, n, shift, tiles, offs, kout, vout);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        std::swap(kin, kout);
        std::swap(vin, vout);
        *result_in_alt = !*result_in_alt;
    }
    return cudaSuccess;
}

size_t scan_temp_bytes(uint32_t n) {
    const uint64_t tiles = (static_cast<uint64_t>(n) + kTile - 1) / kTile;
    return sizeof(uint32_t) * 2 * std::max<uint64_t>(tiles, 1);
}

cudaError_t exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint32_t n, void* temp, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    const uint32_t tiles = static_cast<uint32_t>((static_cast<uint64_t>(n) + kTile - 1) / kTile);
    uint32_t* sums = static_cast<uint32_t*>(temp);
    uint32_t* offs = sums + tiles;
    tile_sum_kernel<<<tiles, kThreads, 0, stream>>>(in, n, sums);
    scan_one_block_kernel<<<1, 1024, 0, stream>>>(sums, offs, tiles);
    tile_scan_kernel<<<tiles, kThreads, 0, stream>>>(in, n, offs, out);
    return cudaGetLastError();
}

}  // namespace mcsbr_int
