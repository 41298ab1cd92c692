// Pipe-rate microbenchmark (sm_100a): DFMA-only, IMAD-only and mixed warps.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>  // 0: dfma, 1: imad, 2: half warps dfma half imad
__global__ void k(double* od, uint32_t* oi, int iters) {
    double d[8];
    uint32_t u[8];
    for (int i = 0; i < 8; ++i) { d[i] = threadIdx.x * 1e-3 + i; u[i] = threadIdx.x + i; }
    const bool fp = MODE == 0 || (MODE == 2 && (threadIdx.x >> 5) & 1);
    if (fp) {
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 8; ++i) d[i] = __fma_rn(d[i], 1.0000001, 0.5);
    } else {
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 8; ++i) u[i] = u[i] * 0x9E3779B9u + 7u;
    }
    double s = 0; uint32_t x = 0;
    for (int i = 0; i < 8; ++i) { s += d[i]; x ^= u[i]; }
    od[blockIdx.x * blockDim.x + threadIdx.x] = s;
    oi[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int threads = 512, blocks = sms * 2, iters = 20000;
    double* od; uint32_t* oi;
    cudaMalloc(&od, blocks * threads * 8); cudaMalloc(&oi, blocks * threads * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<blocks, threads>>>(od, oi, iters);
            if (mode == 1) k<1><<<blocks, threads>>>(od, oi, iters);
            if (mode == 2) k<2><<<blocks, threads>>>(od, oi, iters);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double ops = double(blocks) * threads * iters * 8;
            if (rep) printf("mode %d: %.3f ms, %.1f Gop/s, %.1f lane-ops/clk/SM (at max clock %d MHz)\n", mode, ms,
                   ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
        }
    }
    return 0;
}
