// K2: consume-in-kernel (sm_100a) — per-stream u64 sum of the 24-bit outputs
// and a 256-bin histogram of u >> 16, nothing stored (BASELINE config 4).
//
// Thread per stream, with the stream's 97-word Fibonacci ring in REGISTERS:
// slot s holds the latest x_n with n = s (mod 97), so step n is
//   X[s] -= X[(s + 64) % 97]        (x_n = x_{n-97} - x_{n-33}, core.hpp:56)
// and a 97-step unrolled body sees only compile-time slot indices. The first
// body starts at slot 0 because the slots are loaded in canonical order
// (X[s] = u[s] = lane[(i0 - s) mod 97], jump.hpp:32-37); slot s always maps
// back to ring position (i0 - s) mod 97, so the state is written back exactly
// as per_stream calls of step() leave it. No shuffles, no shared-memory
// traffic for generation: per output one IADD for the lag recurrence, two for
// v (VIADD + VIADDMNMX), two for the output, one for the sum, and the
// histogram update.
//
// Histogram: thread-private u16 counters in shared memory, thread t owning
// bank t mod 32 (word (bin >> 1) * kCT + t, half bin & 1): conflict-free and
// atomic-free. A thread flushes them into its stream's u32 histogram in HBM at
// least every 65,535 outputs, so a u16 never overflows.
#include <cstdint>

#include "ranmar_device.cuh"

namespace rb {

namespace {

constexpr int kCT = 384;                               // threads (streams) per block
constexpr int kRows = 128;                             // u16 pairs per thread
constexpr size_t kConsumeSmem = size_t(kRows) * kCT * 4;  // 192 KB
constexpr int kBodiesPerFlush = 65535 / 97;            // 675 bodies = 65,475 outputs

__device__ __forceinline__ int mod97c(int64_t x) {
    int64_t r = x % 97;
    return static_cast<int>(r < 0 ? r + 97 : r);
}

// Byte address of bin u >> 16 in this thread's column, (bin >> 1) 4 kCT + (bin & 1) 2,
// written as bin 2 kCT + (bin & 1) kHalfFix with kHalfFix = 2 - 2 kCT: SHF, LOP3 and
// two IMADs (the second multiplier comes in as a kernel argument so ptxas keeps
// the IMAD instead of turning it into a compare and two selects).
__device__ __forceinline__ uint32_t hist_addr(uint32_t hb, uint32_t u, uint32_t half_fix) {
    const uint32_t bin = u >> 16;
    const uint32_t a = hb + bin * (2 * kCT);
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(bin & 1u), "r"(half_fix), "r"(a));
    return r;
}

__device__ __forceinline__ void hist_add(uint32_t hb, uint32_t u, uint32_t hf) {
    const uint32_t a = hist_addr(hb, u, hf);
    uint32_t c;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(c) : "r"(a));
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "r"(c + 1) : "memory");
}

// Adds (or stores, first time) this thread's u16 counters into gh[256] and
// optionally zeroes them.
__device__ __forceinline__ void flush(uint32_t* col, uint32_t* __restrict__ gh, bool accumulate,
                                      bool zero) {
#pragma unroll 4
    for (int w = 0; w < kRows; ++w) {
        const uint32_t x = col[w * kCT];
        const uint32_t lo = x & 0xFFFFu, hi = x >> 16;
        if (accumulate) {
            gh[2 * w] += lo;
            gh[2 * w + 1] += hi;
        } else {
            gh[2 * w] = lo;
            gh[2 * w + 1] = hi;
        }
        if (zero) col[w * kCT] = 0;
    }
}

// Two outputs' updates with both loads issued before either store, so the
// load -> add -> store latency is paid once per pair. If both land in the
// same counter, both loads saw the same value and the second store (v + 2)
// overwrites the first (v + 1).
__device__ __forceinline__ void hist_add2(uint32_t hb, uint32_t u1, uint32_t u2, uint32_t hf) {
    const uint32_t a1 = hist_addr(hb, u1, hf);
    const uint32_t a2 = hist_addr(hb, u2, hf);
    uint32_t c1, c2;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(c1) : "r"(a1));
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(c2) : "r"(a2));
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a1), "r"(c1 + 1) : "memory");
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a2), "r"(c2 + 1 + (a1 == a2 ? 1u : 0u)) : "memory");
}

template <int S>
struct Body {
    // steps at compile-time slots S and S + 1, then the rest of the body
    static __device__ __forceinline__ void run(uint32_t (&X)[97], uint32_t& V, uint32_t& s32,
                                               uint32_t hb, uint32_t hf) {
        X[S] -= X[(S + 64) % 97];
        V = add_mod_m(V, kStepA);
        const uint32_t u1 = (X[S] - V) & kMask;
        X[S + 1] -= X[(S + 65) % 97];
        V = add_mod_m(V, kStepA);
        const uint32_t u2 = (X[S + 1] - V) & kMask;
        s32 += u1 + u2;
        hist_add2(hb, u1, u2, hf);
        Body<S + 2>::run(X, V, s32, hb, hf);
    }
};
template <>
struct Body<96> {  // the 97th step alone
    static __device__ __forceinline__ void run(uint32_t (&X)[97], uint32_t& V, uint32_t& s32,
                                               uint32_t hb, uint32_t hf) {
        X[96] -= X[63];
        V = add_mod_m(V, kStepA);
        const uint32_t u = (X[96] - V) & kMask;
        s32 += u;
        hist_add(hb, u, hf);
    }
};

__global__ void __launch_bounds__(kCT, 1)
    consume_kernel(ranmar_state* __restrict__ states, uint64_t n_streams, uint64_t per_stream,
                   uint64_t* __restrict__ sums, uint32_t* __restrict__ hist, uint32_t* status,
                   uint32_t half_fix) {
    extern __shared__ uint32_t hsm[];  // [kRows][kCT]
    const int t = threadIdx.x;
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * kCT + t;
    if (k >= n_streams) return;
    uint32_t* col = hsm + t;
#pragma unroll 8
    for (int w = 0; w < kRows; ++w) col[w * kCT] = 0;
    const uint32_t hb = static_cast<uint32_t>(__cvta_generic_to_shared(col));

    ranmar_state* st = states + k;
    const int i0 = st->i, j0 = st->j;
    const uint32_t v0 = st->v;
    if (!state_ok(i0, j0, v0)) {
        atomicOr(status, kStatusBadState);
        return;
    }
    uint32_t X[97];
#pragma unroll
    for (int s = 0; s < 97; ++s) X[s] = st->lane[(i0 - s + 97) % 97];  // canonical order

    uint32_t* gh = hist + k * 256;
    const uint64_t N = per_stream;
    const uint64_t bodies = N / 97;
    const uint32_t tail = static_cast<uint32_t>(N - bodies * 97);
    uint32_t V = v0;
    uint64_t sum64 = 0;
    bool flushed = false;
    int since = 0;
    for (uint64_t b = 0; b < bodies; ++b) {
        uint32_t s32 = 0;  // 97 x (2^24 - 1) < 2^31
        Body<0>::run(X, V, s32, hb, half_fix);
        sum64 += s32;
        if (++since == kBodiesPerFlush) {
            flush(col, gh, flushed, true);
            flushed = true;
            since = 0;
        }
    }
    // tail (< 97 steps): dynamic slots, through local memory
    uint32_t L[97];
#pragma unroll
    for (int s = 0; s < 97; ++s) L[s] = X[s];
    for (uint32_t s = 0; s < tail; ++s) {
        L[s] -= L[(s + 64) % 97];
        V = add_mod_m(V, kStepA);
        const uint32_t u = (L[s] - V) & kMask;
        sum64 += u;
        hist_add(hb, u, half_fix);
    }
    // slot s <-> ring position (i0 - s) mod 97, whatever N is
#pragma unroll
    for (int s = 0; s < 97; ++s) st->lane[(i0 - s + 97) % 97] = L[s] & kMask;
    st->i = mod97c(static_cast<int64_t>(i0) - static_cast<int64_t>(N % 97));
    st->j = mod97c(static_cast<int64_t>(j0) - static_cast<int64_t>(N % 97));
    st->v = V;
    sums[k] = sum64;
    flush(col, gh, flushed, false);
}

}  // namespace

cudaError_t launch_consume(ranmar_state* d_states, uint64_t n_streams, uint64_t per_stream,
                           uint64_t* d_sums, uint32_t* d_hist, uint32_t* status,
                           cudaStream_t stream) {
    if (n_streams == 0) return cudaSuccess;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(consume_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kConsumeSmem));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const uint64_t blocks = (n_streams + kCT - 1) / kCT;
    count_launch();
    consume_kernel<<<static_cast<unsigned>(blocks), kCT, kConsumeSmem, stream>>>(
        d_states, n_streams, per_stream, d_sums, d_hist, status, static_cast<uint32_t>(2 - 2 * kCT));
    return cudaGetLastError();
}

}  // namespace rb
