// Copy-engine write path: can DMA from an L2-resident staging buffer reach the
// memset write rate (7.39 TB/s) that SM stores (<= 6.7 TB/s) cannot?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void fill(float* p, size_t n, float base) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        p[i] = base + float(i);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t bytes = size_t(16) << 30;
    float *out, *stage;
    cudaMalloc(&out, bytes);
    const size_t chunk = size_t(16) << 20;  // 16 MB
    cudaMalloc(&stage, 2 * chunk);
    cudaStream_t s1, s2; cudaStreamCreate(&s1); cudaStreamCreate(&s2);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    fill<<<sms * 4, 256>>>(stage, 2 * chunk / 4, 0.f);
    cudaDeviceSynchronize();
    for (int mode = 0; mode < 3; ++mode) {
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a, s1);
            const size_t nch = bytes / chunk;
            if (mode == 0) {  // CE only: copy the same L2-resident 16 MB chunk 1024 times
                for (size_t c = 0; c < nch; ++c)
                    cudaMemcpyAsync(reinterpret_cast<char*>(out) + c * chunk, stage, chunk, cudaMemcpyDeviceToDevice, s1);
            } else if (mode == 1) {  // one big D2D copy is not possible (no 16 GiB source); two 8 GiB halves
                cudaMemcpyAsync(out, reinterpret_cast<char*>(out) + bytes / 2, bytes / 2, cudaMemcpyDeviceToDevice, s1);
            } else {  // pipelined: SM fills stage[c%2] on s1, CE drains it on s2
                cudaEvent_t ev[2]; cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming); cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
                cudaEvent_t done[2]; cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming); cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming);
                for (size_t c = 0; c < nch; ++c) {
                    float* st = stage + (c & 1) * (chunk / 4);
                    if (c >= 2) cudaStreamWaitEvent(s1, done[c & 1], 0);
                    fill<<<sms * 2, 256, 0, s1>>>(st, chunk / 4, float(c));
                    cudaEventRecord(ev[c & 1], s1);
                    cudaStreamWaitEvent(s2, ev[c & 1], 0);
                    cudaMemcpyAsync(reinterpret_cast<char*>(out) + c * chunk, st, chunk, cudaMemcpyDeviceToDevice, s2);
                    cudaEventRecord(done[c & 1], s2);
                }
                cudaEvent_t fin; cudaEventCreate(&fin); cudaEventRecord(fin, s2); cudaStreamWaitEvent(s1, fin, 0);
            }
            cudaEventRecord(b, s1); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        const double moved = mode == 1 ? bytes / 2 : bytes;
        printf("mode %d (%s): best %.3f ms, written %.1f GB/s [%s]\n", mode,
               mode == 0 ? "CE from L2-resident 16 MB" : mode == 1 ? "CE HBM->HBM 8 GiB" : "SM fill + CE drain",
               best, moved / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
