// Integer-pipe peaks on this B200 (sm_100a): the denominators of the config-3
// (IMAD) and config-4 (integer issue) rooflines.
//
// Every mode runs 8 dependency chains per thread, chain i taking chain i+1
// as its second operand (so ptxas cannot fold repeated ops; ILP stays ~8),
// 2 blocks of 512 threads per SM, and reports lane-operations per clock per SM
// at the clock passed as argv[1] (the caller's nvidia-smi sample) or the max
// clock. The inner loops are inline PTX; `cuobjdump -sass` shows one SASS
// instruction per PTX op, except that ptxas issues half of mode iadd's adds as
// IMAD.IADD (FMA pipe) and mode shfl adds one LOP3 per SHFL (the lane mask).
//
//   imad   : x = x * C + K          (IMAD, FMA pipe)          -> config-3 peak
//   iadd   : x = x + y              (IADD3, ALU pipe)
//   lop3   : x = x ^ y              (LOP3, ALU pipe)
//   mix    : IMAD and IADD3 alternating (both pipes) -> integer issue peak
//   mix3   : IMAD, IADD3, LOP3 in equal parts
//   shfl   : SHFL.IDX               (K1 / K4s mapping)
//   atoms  : red.shared.add.u32 at a private, conflict-free word (K2 histogram)
//
// Output: one JSON line per mode, and a summary object on the last line.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>

constexpr int kChains = 8;

template <int MODE>
__global__ void __launch_bounds__(512) pipe_kernel(uint32_t* out, int iters, uint32_t c) {
    extern __shared__ uint32_t sm[];
    uint32_t x[kChains];
#pragma unroll
    for (int i = 0; i < kChains; ++i) x[i] = threadIdx.x * 2654435761u + i;
    const uint32_t saddr = static_cast<uint32_t>(__cvta_generic_to_shared(sm)) + 4 * threadIdx.x;
    if (MODE == 6) sm[threadIdx.x] = 0;
    __syncthreads();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) {
            if (MODE == 0) {
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(c), "r"(x[(i + 1) % kChains]));
            } else if (MODE == 1) {
                asm volatile("add.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(x[(i + 1) % kChains]));
            } else if (MODE == 2) {
                asm volatile("xor.b32 %0, %0, %1;" : "+r"(x[i]) : "r"(x[(i + 1) % kChains]));
            } else if (MODE == 3) {
                if (i & 1)
                    asm volatile("add.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(x[(i + 1) % kChains]));
                else
                    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(c), "r"(x[(i + 1) % kChains]));
            } else if (MODE == 4) {
                if (i % 3 == 0)
                    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(c), "r"(x[(i + 1) % kChains]));
                else if (i % 3 == 1)
                    asm volatile("add.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(x[(i + 1) % kChains]));
                else
                    asm volatile("xor.b32 %0, %0, %1;" : "+r"(x[i]) : "r"(x[(i + 1) % kChains]));
            } else if (MODE == 5) {
                asm volatile("shfl.sync.idx.b32 %0, %0, %1, 0x1f, 0xffffffff;" : "+r"(x[i]) : "r"(x[(i + 1) % kChains] & 31));
            } else if (MODE == 6) {
                asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(saddr), "r"(x[i]) : "memory");
            }
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kChains; ++i) s ^= x[i];
    if (MODE == 6) {
        __syncthreads();
        s ^= sm[threadIdx.x];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

static const char* kNames[] = {"imad", "iadd", "lop3", "mix_imad_iadd", "mix_imad_iadd_lop3", "shfl", "atoms"};

template <int MODE>
static float run(uint32_t* d, int blocks, int threads, int iters) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int smem = MODE == 6 ? threads * 4 : 0;
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(a);
        pipe_kernel<MODE><<<blocks, threads, smem>>>(d, iters, 0x9E3779B9u);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return best;
}

int main(int argc, char** argv) {
    int sms, clk_khz;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const double clk_mhz = argc > 1 ? atof(argv[1]) : clk_khz / 1000.0;  // measured clock if given
    const int threads = 512, blocks = sms * 2, iters = 1 << 16;
    uint32_t* d;
    cudaMalloc(&d, size_t(blocks) * threads * 4);
    double rate[7];
    for (int mode = 0; mode < 7; ++mode) {
        float ms = 0;
        switch (mode) {
            case 0: ms = run<0>(d, blocks, threads, iters); break;
            case 1: ms = run<1>(d, blocks, threads, iters); break;
            case 2: ms = run<2>(d, blocks, threads, iters); break;
            case 3: ms = run<3>(d, blocks, threads, iters); break;
            case 4: ms = run<4>(d, blocks, threads, iters); break;
            case 5: ms = run<5>(d, blocks, threads, iters); break;
            case 6: ms = run<6>(d, blocks, threads, iters); break;
        }
        const double ops = double(blocks) * threads * iters * kChains;  // lane-ops
        rate[mode] = ops / (ms * 1e-3);
        printf("{\"mode\": \"%s\", \"ms\": %.3f, \"lane_ops_per_s\": %.4e, "
               "\"lane_ops_per_clk_per_sm\": %.2f, \"clock_mhz\": %.0f}\n",
               kNames[mode], ms, rate[mode], rate[mode] / sms / (clk_mhz * 1e6), clk_mhz);
    }
    printf("{\"summary\": true, \"sms\": %d, \"clock_mhz\": %.0f, \"imad_lane_ops_per_s\": %.4e, "
           "\"int_issue_lane_ops_per_s\": %.4e, \"alu_lane_ops_per_s\": %.4e, "
           "\"shfl_lane_ops_per_s\": %.4e, \"atoms_lane_ops_per_s\": %.4e}\n",
           sms, clk_mhz, rate[0], rate[3] > rate[4] ? rate[3] : rate[4], rate[1], rate[5], rate[6]);
    cudaFree(d);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
