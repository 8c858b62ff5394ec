// Microbenchmark: FP64 MMA (mma.sync m8n8k4 f64) vs FP64 FMA throughput on
// one B200, alone and interleaved (are they separate pipes?).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int kMma, int kFma>
__global__ void k(double* out, int iters, double a, double b) {
    double c[8][2];
    double f[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = threadIdx.x;
#pragma unroll
    for (int i = 0; i < 16; ++i) f[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < kMma; ++i) dmma(c[i & 7][0], c[i & 7][1], a, b);
#pragma unroll
        for (int i = 0; i < kFma; ++i) f[i & 15] = __fma_rn(f[i & 15], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
#pragma unroll
    for (int i = 0; i < 16; ++i) s += f[i];
    if (s == 1.2345) out[0] = s;
}

template <int kMma, int kFma>
void run(const char* name, int blocks_per_sm) {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 4096, threads = 256;
    k<kMma, kFma><<<sms * blocks_per_sm, threads>>>(out, 16, 1.0000001, 1e-9);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<kMma, kFma><<<sms * blocks_per_sm, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = double(sms) * blocks_per_sm * threads / 32;
    const double mma_fma = warps * iters * kMma * 256.0;      // m8n8k4 = 256 FMA
    const double vec_fma = warps * iters * kFma * 32.0;
    printf("%-14s %8.3f ms  mma %7.2f TFLOP/s  vec %7.2f TFLOP/s  total %7.2f TFLOP/s\n", name, ms,
           2 * mma_fma / ms / 1e9, 2 * vec_fma / ms / 1e9, 2 * (mma_fma + vec_fma) / ms / 1e9);
    cudaFree(out);
}

int main() {
    for (int b : {2, 4}) {
        printf("blocks/SM %d (256 threads)\n", b);
        run<16, 0>("mma only", b);
        run<0, 64>("fma only", b);
        run<16, 64>("mma+fma 1:4", b);
        run<16, 32>("mma+fma 1:2", b);
        run<8, 64>("mma+fma 1:8", b);
    }
    return 0;
}
