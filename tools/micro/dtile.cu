// DFMA register-tile microbenchmark (sm_100a): acc[r][c] = fma(a[r], b[c], acc[r][c]).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int R, int C>
__global__ void tile(double* o, const double* src, int iters) {
    __shared__ double sa[64 * 8], sb[64 * 8];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) { sa[i] = src[i]; sb[i] = src[i + 512]; }
    __syncthreads();
    double acc[R][C];
    for (int r = 0; r < R; ++r) for (int c = 0; c < C; ++c) acc[r][c] = 0;
    const int l = threadIdx.x & 15;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 4
        for (int j = 0; j < 32; ++j) {
            double a[R], b[C];
#pragma unroll
            for (int r = 0; r < R; ++r) a[r] = sa[(j * 16 + l) % 512 + r * 0];
#pragma unroll
            for (int c = 0; c < C; ++c) b[c] = sb[(j * 8 + c) % 512];
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < C; ++c) acc[r][c] = __fma_rn(a[r] + r, b[c], acc[r][c]);
        }
    }
    double s = 0;
    for (int r = 0; r < R; ++r) for (int c = 0; c < C; ++c) s += acc[r][c];
    o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int R, int C>
void run(const char* name, double* o, double* src, int sms, int clk, int threads, int bps) {
    const int iters = 200, blocks = sms * bps;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        tile<R, C><<<blocks, threads>>>(o, src, iters);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = double(blocks) * threads * iters * 32 * R * C;
        if (rep) printf("%s threads %d x %d blocks/SM: %.3f ms, %.1f DFMA lanes/clk/SM\n", name, threads, bps, ms,
                        ops / (ms * 1e-3) / sms / (clk * 1e3));
    }
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double *o, *src; cudaMalloc(&o, 1 << 26); cudaMalloc(&src, 1 << 16);
    cudaMemset(src, 0, 1 << 16);
    run<4, 6>("4x6", o, src, sms, clk, 256, 1);
    run<4, 6>("4x6", o, src, sms, clk, 256, 2);
    run<4, 6>("4x6", o, src, sms, clk, 512, 1);
    run<4, 4>("4x4", o, src, sms, clk, 256, 2);
    run<2, 8>("2x8", o, src, sms, clk, 256, 2);
    run<4, 8>("4x8", o, src, sms, clk, 256, 1);
    run<8, 4>("8x4", o, src, sms, clk, 256, 1);
    return 0;
}
