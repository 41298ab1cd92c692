// Write-bandwidth ceiling on this B200 (sm_100a): 16 GiB written by
//  (a) cudaMemsetAsync, (b) st.global.cs v4 stores from a grid-stride kernel,
//  (c) st.global.cs 4-B stores, 128 B per warp instruction (K1's pattern),
//  (d) TMA bulk stores (cp.async.bulk.global.shared::cta) of 8 KB per warp.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void v4(float4* p, size_t n4) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4; i += size_t(gridDim.x) * blockDim.x) {
        float4 v = make_float4(i, i + 1, i + 2, i + 3);
        asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p + i), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
    }
}
__global__ void v4c(float4* p, size_t n4) {  // constant data
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4; i += size_t(gridDim.x) * blockDim.x)
        asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p + i), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
}
// each warp writes a contiguous 64 KB run with 16-B stores (512 B per instruction)
__global__ void v4run(float4* p, size_t n4) {
    const size_t w = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) >> 5;
    const size_t nw = (size_t(gridDim.x) * blockDim.x) >> 5;
    const int l = threadIdx.x & 31;
    const size_t run = 4096;  // float4 per run = 64 KB
    for (size_t r = w; r * run < n4; r += nw)
        for (size_t i = l; i < run; i += 32) {
            const size_t k = r * run + i;
            asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p + k), "f"(float(k)), "f"(float(k + 1)), "f"(float(k + 2)), "f"(float(k + 3)) : "memory");
        }
}
__global__ void s1(float* p, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p + i), "f"(float(i)) : "memory");
}
// each warp owns contiguous 8 KB chunks; fills a 8 KB smem buffer (double-buffered) and bulk-stores it
__global__ void tma(float* p, size_t n) {
    extern __shared__ __align__(128) float sb[];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    float* mine = sb + w * 2 * 2048;
    const size_t chunks = n / 2048;
    int it = 0;
    for (size_t c = blockIdx.x * size_t(nw) + w; c < chunks; c += size_t(gridDim.x) * nw, ++it) {
        float* buf = mine + (it & 1) * 2048;
        if (l == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
        for (int k = l; k < 2048; k += 32) buf[k] = float(c * 2048 + k);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (l == 0) {
            const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 8192;" ::"l"(p + c * 2048), "r"(sa) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (l == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t bytes = size_t(16) << 30, n = bytes / 4;
    float* p; cudaMalloc(&p, bytes);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaFuncSetAttribute(tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 2 * 8192);
    for (int mode = 0; mode < 6; ++mode) {
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) cudaMemsetAsync(p, rep, bytes);
            if (mode == 1) v4<<<sms * 8, 256>>>(reinterpret_cast<float4*>(p), n / 4);
            if (mode == 2) s1<<<sms * 8, 256>>>(p, n);
            if (mode == 3) tma<<<sms * 2, 256, 8 * 2 * 8192>>>(p, n);
            if (mode == 4) v4c<<<sms * 8, 256>>>(reinterpret_cast<float4*>(p), n / 4);
            if (mode == 5) v4run<<<sms * 8, 256>>>(reinterpret_cast<float4*>(p), n / 4);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("mode %d (%s): best %.3f ms = %.1f GB/s  [%s]\n", mode,
               mode == 0 ? "memset" : mode == 1 ? "st.cs v4" : mode == 2 ? "st.cs 4B" : mode == 3 ? "tma bulk" : mode == 4 ? "st.cs v4 const" : "st.cs v4 64KB runs",
               best, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
