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
// v (VIADD + VIADDMNMX), two for the output, half an IADD3 for the sum, and
// four for the histogram (shift, IMAD address, LOP3 increment, ATOMS.ADD).
//
// Histogram: thread-private counters in shared memory, thread t owning bank
// t mod 32: the 32-bit word (bin >> 1) * kCT + t holds bin 2w in its low half
// and bin 2w + 1 in its high half. One output is ONE shared-memory reduction
// (red.shared.add, conflict-free since every lane hits its own bank) adding
// inc = (u & 2^16) | 1, one LOP3 (written as inline lop3: the compiler splits the
// C expression into an AND and an OR): the low half counts every output of
// the word's two bins, the high half the odd bin's, and the flush takes
// lo - hi. Config 4: 410 ms with inc = max(u & 2^16, 1) (LOP3 + VIMNMX, both
// ALU-pipe, the pipe ncu shows 87 % busy), 369 ms with the single LOP3; moving
// the u >> 17 shift to an IMAD.HI made it 437 ms. A thread
// flushes its counters into its stream's u32 histogram in HBM at least every
// 65,475 outputs, so the low half never carries into the high one.
#include <cstdint>

#include "ranmar_device.cuh"

namespace rb {

namespace {

constexpr int kCT = 384;                               // threads (streams) per block
constexpr int kRows = 128;                             // counter words per thread
constexpr size_t kConsumeSmem = size_t(kRows) * kCT * 4;  // 192 KB
constexpr int kBodiesPerFlush = 65535 / 97;            // 675 bodies = 65,475 outputs

__device__ __forceinline__ int mod97c(int64_t x) {
    int64_t r = x % 97;
    return static_cast<int>(r < 0 ? r + 97 : r);
}

// Adds (or stores, first time) this thread's counters into gh[256] and
// optionally zeroes them.
__device__ __forceinline__ void flush(uint32_t* col, uint32_t* __restrict__ gh, bool accumulate,
                                      bool zero) {
#pragma unroll 4
    for (int w = 0; w < kRows; ++w) {
        const uint32_t x = col[w * kCT];
        // every output of the word's two bins added 1 to the low half
        const uint32_t hi = x >> 16, lo = (x & 0xFFFFu) - hi;
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

// One output's histogram update: a single shared-memory reduction.
__device__ __forceinline__ void hist_add(uint32_t hb, uint32_t u) {
    const uint32_t a = hb + (u >> 17) * (4 * kCT);
    uint32_t inc;  // (u & 2^16) | 1 as ONE lop3
    asm("lop3.b32 %0, %1, 65536, %2, 0xEA;" : "=r"(inc) : "r"(u), "r"(1u));
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(inc) : "memory");
}

template <int S>
struct Body {
    // steps at compile-time slots S and S + 1, then the rest of the body
    static __device__ __forceinline__ void run(uint32_t (&X)[97], uint32_t& V, uint32_t& s32,
                                               uint32_t hb) {
        X[S] -= X[(S + 64) % 97];
        V = add_mod_m(V, kStepA);
        const uint32_t u1 = (X[S] - V) & kMask;
        X[S + 1] -= X[(S + 65) % 97];
        V = add_mod_m(V, kStepA);
        const uint32_t u2 = (X[S + 1] - V) & kMask;
        s32 += u1 + u2;
        hist_add(hb, u1);
        hist_add(hb, u2);
        Body<S + 2>::run(X, V, s32, hb);
    }
};
template <>
struct Body<96> {  // the 97th step alone
    static __device__ __forceinline__ void run(uint32_t (&X)[97], uint32_t& V, uint32_t& s32,
                                               uint32_t hb) {
        X[96] -= X[63];
        V = add_mod_m(V, kStepA);
        const uint32_t u = (X[96] - V) & kMask;
        s32 += u;
        hist_add(hb, u);
    }
};

__global__ void __launch_bounds__(kCT, 1)
    consume_kernel(ranmar_state* __restrict__ states, uint64_t n_streams, uint64_t per_stream,
                   uint64_t* __restrict__ sums, uint32_t* __restrict__ hist, uint32_t* status) {
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
        Body<0>::run(X, V, s32, hb);
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
        hist_add(hb, u);
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

namespace {
std::atomic<uint64_t> g_cfg_consume{0};
}  // namespace

cudaError_t configure_consume_kernel() {
    return ensure_smem(consume_kernel, static_cast<int>(kConsumeSmem), g_cfg_consume);
}

cudaError_t launch_consume(ranmar_state* d_states, uint64_t n_streams, uint64_t per_stream,
                           uint64_t* d_sums, uint32_t* d_hist, uint32_t* status,
                           cudaStream_t stream) {
    if (n_streams == 0) return cudaSuccess;
    if (cudaError_t e = ensure_smem(consume_kernel, static_cast<int>(kConsumeSmem), g_cfg_consume)) return e;
    const uint64_t blocks = (n_streams + kCT - 1) / kCT;
    count_launch();
    consume_kernel<<<static_cast<unsigned>(blocks), kCT, kConsumeSmem, stream>>>(
        d_states, n_streams, per_stream, d_sums, d_hist, status);
    return cudaGetLastError();
}

}  // namespace rb
