// Micro-test of the tcgen05.mma kind::i8 path (sm_100a) the tensor-core bulk
// kernel uses: D[128 x 112] (s32, TMEM) = sum_k A[m][k] B[n][k], u8 x u8,
// K = 128 in 4 MMAs of K = 32, A and B K-major without swizzle, B built with
// the "16 shifted copies" layout that turns a Hankel matrix B[n][k] = w[n + k]
// into a canonical K-major operand without materialising it. Checked against
// a CPU product; prints "tc_i8 ok" or the first mismatch.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 112, K = 128;

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // version (Blackwell)
    return d;                             // base offset 0, lbo mode 0, SWIZZLE_NONE
}

__global__ void tc_kernel(const uint8_t* __restrict__ A, const uint8_t* __restrict__ w,
                          int32_t* __restrict__ D) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* sa = sm;                 // A: 8 K-chunks x 16 row groups x 128 B = 16 KB
    uint8_t* sb = sm + 16384;         // B: 14 blocks x 16 shifts x 16 B = 3.5 KB
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int t = threadIdx.x;
    // A (row m, k) -> chunk c = k / 16, group g = m / 8: (c * 16 + g) * 128 + (m % 8) * 16 + k % 16
    for (int x = t; x < M * K; x += blockDim.x) {
        const int m = x / K, k = x % K;
        sa[((k / 16) * 16 + m / 8) * 128 + (m % 8) * 16 + (k % 16)] = A[m * K + k];
    }
    // B (row n, k) = w[n + k] -> S[((n / 16 + k / 16) * 16 + n % 16) * 16 + k % 16]
    // i.e. chunk (b, s) holds w[16 b + s .. 16 b + s + 15]
    for (int x = t; x < 14 * 16 * 16; x += blockDim.x) {
        const int b = x / 256, s = (x / 16) % 16, e = x % 16;
        sb[x] = w[16 * b + s + e];
    }
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_base)))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&bar)))
                     : "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tmem_base;
    const uint32_t idesc = (2u << 4) | (0u << 7) | (0u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
                           (static_cast<uint32_t>(M >> 4) << 24);
    if (t == 0) {
        const uint32_t a0 = static_cast<uint32_t>(__cvta_generic_to_shared(sa));
        const uint32_t b0 = static_cast<uint32_t>(__cvta_generic_to_shared(sb));
        for (int ks = 0; ks < K / 32; ++ks) {
            const uint64_t da = smem_desc(a0 + ks * 2 * 2048, 2048, 128);
            const uint64_t db = smem_desc(b0 + ks * 2 * 256, 256, 128);
            const uint32_t acc = ks > 0;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                "l"(da), "l"(db), "r"(idesc), "r"(acc)
                : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                static_cast<uint32_t>(__cvta_generic_to_shared(&bar)))
            : "memory");
    }
    {
        const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(a)
                : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int warp = t >> 5, lane = t & 31;
    if (warp < 4) {
        const int row = 32 * warp + lane;
        for (int c0 = 0; c0 < N; c0 += 16) {
            uint32_t r[16];
            const uint32_t taddr = tm + (static_cast<uint32_t>(32 * warp) << 16) + c0;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                  "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                  "=r"(r[14]), "=r"(r[15])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int q = 0; q < 16; ++q) D[row * N + c0 + q] = static_cast<int32_t>(r[q]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

int main() {
    std::vector<uint8_t> A(M * K), w(256);
    srand(7);
    for (auto& x : A) x = static_cast<uint8_t>(rand());
    for (auto& x : w) x = static_cast<uint8_t>(rand());
    uint8_t *dA, *dw;
    int32_t* dD;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dw, w.size());
    cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dw, w.data(), w.size(), cudaMemcpyHostToDevice);
    cudaMemset(dD, 0xFF, M * N * 4);
    const int smem = 16384 + 4096;
    cudaFuncSetAttribute(tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tc_kernel<<<1, 128, smem>>>(dA, dw, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("cuda error %s\n", cudaGetErrorString(e));
        return 1;
    }
    std::vector<int32_t> D(M * N);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            int64_t ref = 0;
            for (int k = 0; k < K; ++k) ref += int64_t(A[m * K + k]) * w[n + k];
            if (ref != D[m * N + n]) {
                if (bad < 5) printf("mismatch m=%d n=%d got %d want %lld\n", m, n, D[m * N + n], (long long)ref);
                ++bad;
            }
        }
    if (bad) {
        printf("tc_i8 FAILED: %d mismatches\n", bad);
        return 1;
    }
    printf("tc_i8 ok\n");
    return 0;
}
