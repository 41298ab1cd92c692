// Generation kernel K1 (sm_100a): stored uniforms (u32 / f32 / f64).
// (K2 consume: consume_kernel.cu; K4 gaussian: gauss_kernel.cu.)
//
// Mapping — one warp per stream, 32 consecutive outputs per round.
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

    // One round: returns x_n - v_n (unmasked) for n = 32 r + l; x_n (unmasked)
    // and v_n are left in R1 and last_v.
    uint32_t last_v;
    __device__ __forceinline__ uint32_t round() {
        const uint32_t S = __shfl_sync(0xffffffffu, R3 - R1, src);
        const uint32_t y = (l == 0) ? prev : S;
        prev = S;
        R4 = R3;
        R3 = R2;
        R2 = R1;
        R1 = y;
        const uint32_t raw = y - V;
        last_v = V;
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
    // 32-bit inner counter, unrolled by 8: the only per-round work left is
    // the generator, the conversion and the store
    for (uint64_t r0 = 0; r0 < full; r0 += (1u << 30)) {
        const uint32_t cnt = static_cast<uint32_t>(full - r0 < (1u << 30) ? full - r0 : (1u << 30));
#pragma unroll 8
        for (uint32_t r = 0; r < cnt; ++r) emit(r0 + r, g.round(), true);
    }
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

// The last stream's state re-laid into the ORIGINAL ring layout of *dst, i.e.
// exactly what `count` calls of step() leave on one stream generated as
// substreams (ranmar_generate_single_*): canonical u[k] = lane[(i - k) mod 97]
// is layout-independent, and lane[(i_t - k) mod 97] = u[k] with the target
// cursor i_t = (i0 - count) mod 97 (jump.hpp:32-48). i0 is read from dst (the
// original state) before it is overwritten; an invalid original state was
// already flagged by make_streams and is left untouched. One warp.
__device__ __forceinline__ void warp_relayout(const ranmar_state* __restrict__ src,
                                              ranmar_state* __restrict__ dst, int count_mod97) {
    const int l = threadIdx.x & 31;
    const int i0 = dst->i;
    const bool ok = state_ok(i0, dst->j, dst->v);
    const int i_t = (i0 - count_mod97 + 97) % 97, si = src->i;
    const uint32_t sv = src->v;
    __syncwarp();  // every lane has read dst's cursors before lane 0 rewrites them
    if (!ok) return;
    for (int k = l; k < 97; k += 32) {
        int q = si - k;
        q += q < 0 ? 97 : 0;
        int r = i_t - k;
        r += r < 0 ? 97 : 0;
        dst->lane[r] = src->lane[q];
    }
    if (l == 0) {
        dst->i = i_t;
        dst->j = i_t >= 64 ? i_t - 64 : i_t + 33;
        dst->v = sv;
    }
}

// Warp per stream. per_last = the last stream's output count (per_stream for a
// plain launch); with relay set, the last stream's warp also re-lays its final
// state into *relay (ranmar_generate_single_*: the substreams' tail and the
// re-join ride in the same launch).
template <class T>
__global__ void __launch_bounds__(32 * kGenWarps)
    gen_store_kernel(ranmar_state* __restrict__ states, uint64_t n_streams, uint64_t per_stream,
                     T* __restrict__ out, uint32_t* status, uint64_t per_last,
                     ranmar_state* __restrict__ relay, int count_mod97) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * kGenWarps + (threadIdx.x >> 5);
    if (k >= n_streams) return;
    const bool last = k == n_streams - 1;
    T* o = out + k * per_stream + (threadIdx.x & 31);
    warp_stream(states + k, last ? per_last : per_stream, status, [&](uint64_t r, uint32_t raw, bool valid) {
        if (valid) st_cs(o + 32 * r, convert_out<T>(raw));
    });
    if (relay && last) {
        __syncwarp();  // the stream's state, stored by its lanes, is visible to the warp
        warp_relayout(states + k, relay, count_mod97);
    }
}

// Trace of N steps per stream (the scalar step() of the C++ facade): u[n] =
// output n, x[n] = the value step n writes into lane[i] (x_n), v[n] = the
// residue after step n. States advance like gen_store_kernel.
__global__ void __launch_bounds__(32 * kGenWarps)
    gen_trace_kernel(ranmar_state* __restrict__ states, uint64_t n_streams, uint64_t per_stream,
                     uint32_t* __restrict__ uo, uint32_t* __restrict__ xo, uint32_t* __restrict__ vo,
                     uint32_t* status) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * kGenWarps + (threadIdx.x >> 5);
    if (k >= n_streams) return;
    const uint64_t base = k * per_stream + (threadIdx.x & 31);
    WarpGen g;
    if (!g.load(states + k, status)) return;
    const uint64_t rounds = (per_stream + 31) >> 5;
    for (uint64_t r = 0; r < rounds; ++r) {
        const uint32_t raw = g.round();
        if (32 * r + g.l < per_stream) {
            uo[base + 32 * r] = raw & kMask;
            xo[base + 32 * r] = g.R1 & kMask;
            vo[base + 32 * r] = g.last_v;
        }
    }
    g.store(states + k, per_stream, rounds);
}

}  // namespace

// ---------------------------------------------------------------- launchers

cudaError_t launch_generate_trace(ranmar_state* d_states, uint64_t n_streams, uint64_t per_stream,
                                  uint32_t* d_u, uint32_t* d_x, uint32_t* d_v, uint32_t* status,
                                  cudaStream_t stream) {
    if (n_streams == 0 || per_stream == 0) return cudaSuccess;
    const uint64_t blocks = (n_streams + kGenWarps - 1) / kGenWarps;
    count_launch();
    gen_trace_kernel<<<static_cast<unsigned>(blocks), 32 * kGenWarps, 0, stream>>>(
        d_states, n_streams, per_stream, d_u, d_x, d_v, status);
    return cudaGetLastError();
}

template <class T>
cudaError_t launch_generate_joined(ranmar_state*, uint64_t, uint64_t, uint64_t, T*, ranmar_state*, int,
                                   uint32_t*, cudaStream_t);

template <class T>
cudaError_t launch_generate(ranmar_state* d_states, uint64_t n_streams, uint64_t per_stream,
                            T* d_out, uint32_t* status, cudaStream_t stream) {
    return launch_generate_joined<T>(d_states, n_streams, per_stream, per_stream, d_out, nullptr, 0,
                                     status, stream);
}

// n_streams substreams of per_stream outputs, the last one per_last, in one
// launch; with relay set the last substream's final state is re-laid into it.
template <class T>
cudaError_t launch_generate_joined(ranmar_state* d_states, uint64_t n_streams, uint64_t per_stream,
                                   uint64_t per_last, T* d_out, ranmar_state* relay, int count_mod97,
                                   uint32_t* status, cudaStream_t stream) {
    if (n_streams == 0) return cudaSuccess;
    const uint64_t blocks = (n_streams + kGenWarps - 1) / kGenWarps;
    count_launch();
    gen_store_kernel<T><<<static_cast<unsigned>(blocks), 32 * kGenWarps, 0, stream>>>(
        d_states, n_streams, per_stream, d_out, status, per_last, relay, count_mod97);
    return cudaGetLastError();
}
#define RB_GEN_INST(T)                                                                                \
    template cudaError_t launch_generate<T>(ranmar_state*, uint64_t, uint64_t, T*, uint32_t*,        \
                                            cudaStream_t);                                          \
    template cudaError_t launch_generate_joined<T>(ranmar_state*, uint64_t, uint64_t, uint64_t, T*, \
                                                   ranmar_state*, int, uint32_t*, cudaStream_t);
RB_GEN_INST(uint32_t)
RB_GEN_INST(float)
RB_GEN_INST(double)
#undef RB_GEN_INST

}  // namespace rb
