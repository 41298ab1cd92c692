// Generation kernels (sm_100a): K1 store (u32 / f32 / f64), K2 consume
// (per-stream sum + histogram, nothing stored), K4 gaussian (polar).
//
// K1/K2 mapping — one warp per stream, 32 consecutive outputs per round.
// Both lags are 1 mod 32 (97 = 3*32 + 1, 33 = 32 + 1), so with
//   y[r][l] = x_{32 r + l}
// the recurrence x_n = x_{n-97} - x_{n-33} (core.hpp:56; Alg. 2)
// becomes
//   y[r][l] = y[r-3][l-1] - y[r-1][l-1]          (l >= 1)
//   y[r][0] = y[r-4][31]  - y[r-2][31]
// Lane l therefore keeps four registers R1..R4 = y[r-1..r-4][l], computes
// D = R3 - R1 (the difference lane l+1 needs) and passes it on with ONE
// shuffle; lane 0 uses the value lane 31 sent in the previous round. A round
// writes 32 consecutive outputs of one stream: a full 128-B line, coalesced.
// The arithmetic part is per-lane: v for output n is v0 + (n + 1)(m - d) mod m,
// advanced by 32 (m - d) mod m per round with one branch-free min().
//
// After the last round the registers hold x_n for every n in [N - 97, N), so
// each stream's state is written back exactly as N calls of step() leave it
// (ring slot (i0 - n) mod 97 holds x_n, cursors moved by N, v advanced).
#include <cstdint>

#include "ranmar_device.cuh"

namespace rb {

namespace {

__device__ __forceinline__ int mod97(int64_t x) {
    int64_t r = x % 97;
    return static_cast<int>(r < 0 ? r + 97 : r);
}

// Warp-per-stream generator: lane l of round r produces x_{32 r + l}.
struct WarpGen {
    uint32_t R1, R2, R3, R4;  // y[r-1..r-4][l]
    uint32_t prev;            // lane 0's operand for the next round
    uint32_t V;               // v of this lane's next output
    uint32_t A32;             // 32 (m - d) mod m
    int src, l, i0, j0;
    uint32_t v0;

    // Loads the state; false (and the status bit) if it violates the invariants.
    __device__ __forceinline__ bool load(const ranmar_state* st, uint32_t* status) {
        l = threadIdx.x & 31;
        i0 = st->i;
        j0 = st->j;
        v0 = st->v;
        if (!state_ok(i0, j0, v0)) {
            if (l == 0) atomicOr(status, kStatusBadState);
            return false;
        }
        // x_n = lane[(i0 - n) mod 97] for n in [-97, -1].
        const uint32_t* lane = st->lane;
        R1 = lane[(i0 + 32 - l) % 97];
        R2 = lane[(i0 + 64 - l) % 97];
        R3 = lane[(i0 + 96 - l) % 97];
        R4 = (l == 31) ? lane[i0] : 0u;  // x_{-97}; other lanes' round -4 is never read
        src = (l + 31) & 31;
        // Lane 0's operand for round 0 is lane 31's (x_{-97} - x_{-33}).
        prev = __shfl_sync(0xffffffffu, R4 - R2, src);
        V = arith_advance(v0, static_cast<uint64_t>(l) + 1);
        A32 = static_cast<uint32_t>((32ull * kStepA) % kMod);
        return true;
    }

    // One round: returns x_n - v_n (unmasked) for n = 32 r + l.
    __device__ __forceinline__ uint32_t round() {
        const uint32_t S = __shfl_sync(0xffffffffu, R3 - R1, src);
        const uint32_t y = (l == 0) ? prev : S;
        prev = S;
        R4 = R3;
        R3 = R2;
        R2 = R1;
        R1 = y;
        const uint32_t raw = y - V;
        V = add_mod_m(V, A32);
        return raw;
    }

    // Writes the state N = per-stream outputs later, exactly as N step()
    // calls leave it; `rounds` = rounds executed (ceil(N / 32)).
    __device__ __forceinline__ void store(ranmar_state* st, uint64_t N, uint64_t rounds) {
        __syncwarp();
        uint32_t* lane_w = st->lane;
        const int64_t lo = static_cast<int64_t>(N) - 97, hi = static_cast<int64_t>(N);
        const uint32_t regs[4] = {R1, R2, R3, R4};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t n = 32 * (static_cast<int64_t>(rounds) - 1 - k) + l;
            if (n >= lo && n < hi) lane_w[mod97(static_cast<int64_t>(i0) - n)] = regs[k] & kMask;
        }
        if (l == 0) {
            st->i = mod97(static_cast<int64_t>(i0) - static_cast<int64_t>(N % 97));
            st->j = mod97(static_cast<int64_t>(j0) - static_cast<int64_t>(N % 97));
            st->v = arith_advance(v0, N);
        }
    }
};

// Drives a WarpGen over N outputs: emit(r, raw, valid) per round.
template <class Emit>
__device__ __forceinline__ void warp_stream(ranmar_state* st, uint64_t N, uint32_t* status,
                                            Emit&& emit) {
    WarpGen g;
    if (!g.load(st, status)) return;
    const uint64_t full = N >> 5;
    const uint32_t tail = static_cast<uint32_t>(N & 31);
#pragma unroll 4
    for (uint64_t r = 0; r < full; ++r) emit(r, g.round(), true);
    if (tail) emit(full, g.round(), static_cast<uint32_t>(g.l) < tail);
    g.store(st, N, full + (tail ? 1 : 0));
}

template <class T>
__device__ __forceinline__ T convert_out(uint32_t raw);
// u24 as u32 (core.hpp:65)
template <>
__device__ __forceinline__ uint32_t convert_out<uint32_t>(uint32_t raw) {
    return raw & kMask;
}
// next_f64 narrowed to f32 (exact): (raw << 8) keeps the 24 output bits in the
// top of the word, so the u32 -> f32 conversion is exact; * 2^-32 is exact.
template <>
__device__ __forceinline__ float convert_out<float>(uint32_t raw) {
    return __uint2float_rn(raw << 8) * 0x1p-32f;
}
// next_f64 (core.hpp:70-72)
template <>
__device__ __forceinline__ double convert_out<double>(uint32_t raw) {
    return static_cast<double>(raw & kMask) * 0x1p-24;
}

constexpr int kGenWarps = 8;  // streams per 256-thread block

template <class T>
__global__ void __launch_bounds__(32 * kGenWarps)
    gen_store_kernel(ranmar_state* __restrict__ states, uint64_t n_streams, uint64_t per_stream,
                     T* __restrict__ out, uint32_t* status) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * kGenWarps + (threadIdx.x >> 5);
    if (k >= n_streams) return;
    T* o = out + k * per_stream + (threadIdx.x & 31);
    warp_stream(states + k, per_stream, status, [&](uint64_t r, uint32_t raw, bool valid) {
        if (valid) st_cs(o + 32 * r, convert_out<T>(raw));
    });
}

// K2: per-lane private u16 counters, lane l owning bank l:
//   word((b >> 1) * 32 + l), half (b & 1)
// so a warp's 32 updates never conflict and need no atomics. A lane sees at
// most kFlushRounds outputs between flushes, so u16 cannot overflow.
constexpr int kConsumeWarps = 4;
constexpr uint32_t kHistWordsPerWarp = 128 * 32;  // 256 u16 bins x 32 lanes = 16 KB
constexpr uint64_t kFlushRounds = 65535;

__device__ __forceinline__ void flush_hist(uint32_t* hw, uint32_t* __restrict__ ghist, bool zero,
                                           bool accumulate) {
    __syncwarp();
    const int l = threadIdx.x & 31;
    // Lane l reduces bins l, l+32, ..., l+224 over the 32 lane columns.
#pragma unroll 1
    for (int b = l; b < 256; b += 32) {
        const unsigned short* col =
            reinterpret_cast<const unsigned short*>(hw + (b >> 1) * 32) + (b & 1);
        uint32_t s = 0;
#pragma unroll 8
        for (int c = 0; c < 32; ++c) s += col[2 * c];
        ghist[b] = accumulate ? ghist[b] + s : s;
    }
    __syncwarp();
    if (zero)
        for (uint32_t w = l; w < kHistWordsPerWarp; w += 32) hw[w] = 0;
    __syncwarp();
}

// Histogram update for one output u (24-bit): byte offset of bin u >> 16 in
// this lane's column, ((bin >> 1) * 32 words) * 4 + (bin & 1) * 2.
__device__ __forceinline__ void hist_add(uint32_t hb, uint32_t u) {
    // hb: 32-bit shared-window address of this lane's column
    const uint32_t a = hb + (((u >> 10) & 0x3F80u) | ((u >> 15) & 2u));
    uint32_t c;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(c) : "r"(a));
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "r"(c + 1) : "memory");
}

__global__ void __launch_bounds__(32 * kConsumeWarps)
    consume_kernel(ranmar_state* __restrict__ states, uint64_t n_streams, uint64_t per_stream,
                   uint64_t* __restrict__ sums, uint32_t* __restrict__ hist, uint32_t* status) {
    extern __shared__ uint32_t smem_hist[];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * kConsumeWarps + w;
    if (k >= n_streams) return;
    uint32_t* hw = smem_hist + w * kHistWordsPerWarp;
    for (uint32_t i = l; i < kHistWordsPerWarp; i += 32) hw[i] = 0;
    __syncwarp();
    const uint32_t hb = static_cast<uint32_t>(__cvta_generic_to_shared(hw)) + 4 * l;
    uint32_t* gh = hist + k * 256;

    WarpGen g;
    if (!g.load(states + k, status)) return;
    const uint64_t N = per_stream, full = N >> 5;
    const uint32_t tail = static_cast<uint32_t>(N & 31);
    uint64_t sum64 = 0;
    bool flushed = false;
    uint64_t r = 0;
    while (r < full) {
        // <= kFlushRounds rounds between flushes (u16 counters), sums in
        // blocks of <= 128 rounds (128 x 24-bit values fit 32 bits).
        const uint64_t chunk_end = min(full, r + kFlushRounds);
        while (r < chunk_end) {
            const uint64_t left = chunk_end - r;
            const uint32_t blk = left < 128 ? static_cast<uint32_t>(left) : 128u;
            uint32_t s32 = 0;
#pragma unroll 4
            for (uint32_t q = 0; q < blk; ++q) {
                const uint32_t u = g.round() & kMask;
                s32 += u;
                hist_add(hb, u);
            }
            sum64 += s32;
            r += blk;
        }
        if (r < full || tail) {
            flush_hist(hw, gh, true, flushed);
            flushed = true;
        }
    }
    if (tail) {
        const uint32_t u = g.round() & kMask;
        if (static_cast<uint32_t>(l) < tail) {
            sum64 += u;
            hist_add(hb, u);
        }
    }
    g.store(states + k, N, full + (tail ? 1 : 0));
#pragma unroll
    for (int o = 16; o; o >>= 1) sum64 += __shfl_xor_sync(0xffffffffu, sum64, o);
    if (l == 0) sums[k] = sum64;
    flush_hist(hw, gh, false, flushed);
}

}  // namespace

// ---------------------------------------------------------------- launchers

template <class T>
cudaError_t launch_generate(ranmar_state* d_states, uint64_t n_streams, uint64_t per_stream,
                            T* d_out, uint32_t* status, cudaStream_t stream) {
    if (n_streams == 0) return cudaSuccess;
    const uint64_t blocks = (n_streams + kGenWarps - 1) / kGenWarps;
    count_launch();
    gen_store_kernel<T><<<static_cast<unsigned>(blocks), 32 * kGenWarps, 0, stream>>>(
        d_states, n_streams, per_stream, d_out, status);
    return cudaGetLastError();
}
template cudaError_t launch_generate<uint32_t>(ranmar_state*, uint64_t, uint64_t, uint32_t*,
                                               uint32_t*, cudaStream_t);
template cudaError_t launch_generate<float>(ranmar_state*, uint64_t, uint64_t, float*, uint32_t*,
                                            cudaStream_t);
template cudaError_t launch_generate<double>(ranmar_state*, uint64_t, uint64_t, double*,
                                             uint32_t*, cudaStream_t);

cudaError_t launch_consume(ranmar_state* d_states, uint64_t n_streams, uint64_t per_stream,
                           uint64_t* d_sums, uint32_t* d_hist, uint32_t* status,
                           cudaStream_t stream) {
    if (n_streams == 0) return cudaSuccess;
    const int smem = kConsumeWarps * kHistWordsPerWarp * 4;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(consume_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const uint64_t blocks = (n_streams + kConsumeWarps - 1) / kConsumeWarps;
    count_launch();
    consume_kernel<<<static_cast<unsigned>(blocks), 32 * kConsumeWarps, smem, stream>>>(
        d_states, n_streams, per_stream, d_sums, d_hist, status);
    return cudaGetLastError();
}

}  // namespace rb
