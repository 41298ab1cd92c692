// K5: the classic floating-point RANMAR (Algorithm 1) on the GPU (sm_100a).
//
// reference/float_ranmar.hpp:33-46 in binary64: y = x_i - x_j (+1 if < 0),
// stored back; c -= d (+ m/M if < 0); output y - c (+1 if < 0). Every value
// is a dyadic a/2^24 and every operation is exact, so the outputs equal the
// integer generator's u/2^24 bit for bit (the reference's own isomorphism,
// core.hpp:4-8). Same warp mapping as K1 (one warp per stream, 32 consecutive
// outputs per round, one 64-bit shuffle per output), here with the
// Fibonacci values and c in fp64 and the +1 fix-ups as in Algorithm 1.
// Config 1 runs its 10^8 outputs through both recurrences.
#include <cstdint>

#include "ranmar_device.cuh"

namespace rb {

namespace {

constexpr double kDeltaF = 7654321.0 / 16777216.0;   // float_ranmar.hpp:19
constexpr double kModF = 16777213.0 / 16777216.0;    // float_ranmar.hpp:20

__device__ __forceinline__ double fix1(double y) { return y < 0.0 ? y + 1.0 : y; }

__device__ __forceinline__ int mod97f(int64_t x) {
    int64_t r = x % 97;
    return static_cast<int>(r < 0 ? r + 97 : r);
}

constexpr int kFWarps = 8;

// kTrace: also store, per step, the value written into x[i] (y) and the new c
// (the scalar step_float of the C++ facade copies them into the caller's
// state, so every word of that state comes from this kernel).
template <bool kTrace>
__global__ void __launch_bounds__(32 * kFWarps)
    float_gen_kernel(ranmar_float_state* __restrict__ states, uint64_t n_streams, uint64_t N,
                     double* __restrict__ out, double* __restrict__ ty, double* __restrict__ tc,
                     uint32_t* status) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * kFWarps + (threadIdx.x >> 5);
    if (k >= n_streams) return;
    const int l = threadIdx.x & 31;
    ranmar_float_state* st = states + k;
    const int i0 = st->i, j0 = st->j;
    const double c0 = st->c;
    if (!(static_cast<unsigned>(i0) < 97u && static_cast<unsigned>(j0) < 97u &&
          (i0 - j0 + 97) % 97 == 64 && c0 >= 0.0 && c0 < kModF)) {
        if (l == 0) atomicOr(status, kStatusBadState);
        return;
    }
    const double* x = st->x;
    double R1 = x[(i0 + 32 - l) % 97], R2 = x[(i0 + 64 - l) % 97], R3 = x[(i0 + 96 - l) % 97];
    double R4 = (l == 31) ? x[i0] : 0.0;
    const int src = (l + 31) & 31;
    double prev = __shfl_sync(0xffffffffu, fix1(R4 - R2), src);
    // c for this lane's first output: c0 - (l + 1) d (mod m/M), stepped exactly
    // as Algorithm 1 does (one subtraction and fix-up per step)
    double c = c0;
    for (int q = 0; q <= l; ++q) {
        c -= kDeltaF;
        if (c < 0.0) c += kModF;
    }
    // per round: c - 32 d (mod m/M) = c + A32 (mod m/M), A32 an exact dyadic
    const double A32 = static_cast<double>((32ull * kStepA) % kMod) * 0x1p-24;
    double* o = out + k * N + l;
    const uint64_t rounds = (N + 31) >> 5;
    for (uint64_t r = 0; r < rounds; ++r) {
        const double S = __shfl_sync(0xffffffffu, fix1(R3 - R1), src);
        const double y = (l == 0) ? prev : S;
        prev = S;
        R4 = R3;
        R3 = R2;
        R2 = R1;
        R1 = y;
        if (32 * r + l < N) {
            o[32 * r] = fix1(y - c);
            if (kTrace) {
                ty[k * N + 32 * r + l] = y;
                tc[k * N + 32 * r + l] = c;
            }
        }
        c += A32;
        if (c >= kModF) c -= kModF;
    }
    __syncwarp();
    double* xw = st->x;
    const int64_t lo = static_cast<int64_t>(N) - 97, hi = static_cast<int64_t>(N);
    const double regs[4] = {R1, R2, R3, R4};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t n = 32 * (static_cast<int64_t>(rounds) - 1 - q) + l;
        if (n >= lo && n < hi) xw[mod97f(static_cast<int64_t>(i0) - n)] = regs[q];
    }
    // c after N steps: lane (N - 1) mod 32 holds it after its last output;
    // recompute from c0 by the closed form on the integer image (exact)
    if (l == 0) {
        st->i = mod97f(static_cast<int64_t>(i0) - static_cast<int64_t>(N % 97));
        st->j = mod97f(static_cast<int64_t>(j0) - static_cast<int64_t>(N % 97));
        const uint32_t v0 = static_cast<uint32_t>(c0 * 16777216.0);
        st->c = static_cast<double>(arith_advance(v0, N)) * 0x1p-24;
    }
}

// The reference's state isomorphism (float_ranmar.hpp:3-8, 84-95) on the
// device: integer state -> float state, x[k] = lane[k] / 2^24, c = v / 2^24,
// same cursors; exact. A warp per state.
__global__ void float_from_states_kernel(const ranmar_state* __restrict__ in, uint64_t n,
                                         ranmar_float_state* __restrict__ out) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (k >= n) return;
    const int l = threadIdx.x & 31;
    for (int q = l; q < 97; q += 32) out[k].x[q] = static_cast<double>(in[k].lane[q] & kMask) * 0x1p-24;
    if (l == 0) {
        out[k].c = static_cast<double>(in[k].v) * 0x1p-24;
        out[k].i = in[k].i;
        out[k].j = in[k].j;
    }
}

}  // namespace

cudaError_t launch_float_from_states(const ranmar_state* d_in, uint64_t n, ranmar_float_state* d_out,
                                     cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    count_launch();
    float_from_states_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, stream>>>(d_in, n, d_out);
    return cudaGetLastError();
}

cudaError_t launch_float_gen(ranmar_float_state* d_states, uint64_t n_streams, uint64_t per_stream,
                             double* d_out, double* d_y, double* d_c, uint32_t* status,
                             cudaStream_t stream) {
    if (n_streams == 0) return cudaSuccess;
    const uint64_t blocks = (n_streams + kFWarps - 1) / kFWarps;
    count_launch();
    if (d_y)
        float_gen_kernel<true><<<static_cast<unsigned>(blocks), 32 * kFWarps, 0, stream>>>(
            d_states, n_streams, per_stream, d_out, d_y, d_c, status);
    else
        float_gen_kernel<false><<<static_cast<unsigned>(blocks), 32 * kFWarps, 0, stream>>>(
            d_states, n_streams, per_stream, d_out, nullptr, nullptr, status);
    return cudaGetLastError();
}

}  // namespace rb
