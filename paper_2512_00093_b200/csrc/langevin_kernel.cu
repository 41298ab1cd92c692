// K6: consumers that advance a state by only a FEW outputs per launch
// (sm_100a): the fix-langevin-style per-atom force update (SURVEY.md §8f rows
// 3-4) and gaussian() with few deviates per atom per launch (the per-step
// launch mode of config 5).
//
// A launch that draws ~3-10 outputs from a stream touches ~3-10 ring words at
// the read cursor i and as many at j = i - 64 (mod 97), plus the cursors and
// v. Staging the whole 97-word ring (K4) would move 832 B per atom for that;
// here each thread steps its state IN PLACE in global memory (core.hpp:54-66
// on the record itself): the touched words come through L1 (a few 32-B
// sectors per atom), and only they are written back. Within a launch a word
// written at step n is read again at step n + 33 at the earliest, by the same
// thread, so in-place stepping is exact.
//
// Langevin force (repo convention; the reference has no consumer, LAMMPS is
// not in the container): for each atom a in the group, type t = type[a],
//   g1 = gfactor1[t], g2 = gfactor2[t] * tsqrt,
//   for d = 0, 1, 2:  r = uniform() - 0.5   (noise 0, LAMMPS' default form)
//                     r = gaussian()        (noise 1)
//                     f[a][d] = f[a][d] + (g1 * v[a][d] + g2 * r)
// every operation rounded separately (oracle/ranmar_oracle.c or_langevin).
// Atoms outside the group (mask[a] & groupbit == 0) draw nothing.
#include <cstdint>

#include "gauss_math.cuh"
#include "ranmar_device.cuh"

namespace rb {

namespace {

// One stream stepped in place in global memory.
struct InPlace {
    uint32_t* lane;
    int i, j;
    uint32_t v;

    __device__ __forceinline__ uint32_t next() {
        const uint32_t x = (lane[i] - lane[j]) & kMask;
        lane[i] = x;
        i = i == 0 ? 96 : i - 1;
        j = j == 0 ? 96 : j - 1;
        v = add_mod_m(v, kStepA);
        return (x - v) & kMask;
    }
};

// gaussian() on an in-place stream (oracle or_gaussian; exact integer test).
__device__ __forceinline__ double gauss_next(InPlace& st, double& saved, bool& has) {
    if (has) {
        has = false;
        return saved;
    }
    uint32_t u0, u1;
    for (;;) {
        u0 = st.next();
        u1 = st.next();
        const int32_t da = static_cast<int32_t>(u0) - (1 << 23);
        const int32_t db = static_cast<int32_t>(u1) - (1 << 23);
        const int64_t s = static_cast<int64_t>(da) * da + static_cast<int64_t>(db) * db;
        if (s > 0 && s < (int64_t(1) << 46)) break;
    }
    const double v1 = polar_v(u0), v2 = polar_v(u1);
    const double fac = polar_fac(u0, u1);
    saved = __dmul_rn(v1, fac);
    has = true;
    return __dmul_rn(v2, fac);
}

template <bool kGauss>
__global__ void __launch_bounds__(256)
    langevin_kernel(ranmar_gauss_state* __restrict__ g, uint64_t n_atoms,
                    const double* __restrict__ vel, double* __restrict__ force,
                    const int32_t* __restrict__ type, const int32_t* __restrict__ mask,
                    int32_t groupbit, const double* __restrict__ gf1,
                    const double* __restrict__ gf2, int32_t n_types, double tsqrt,
                    uint32_t* status) {
    const uint64_t a = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (a >= n_atoms) return;
    if (mask != nullptr && (mask[a] & groupbit) == 0) return;
    const int32_t t = type[a];
    if (t < 0 || t > n_types) {
        atomicOr(status, kStatusBadType);
        return;
    }
    ranmar_gauss_state* gs = g + a;
    InPlace st{gs->s.lane, gs->s.i, gs->s.j, gs->s.v};
    if (!state_ok(st.i, st.j, st.v)) {
        atomicOr(status, kStatusBadState);
        return;
    }
    double saved = 0.0;
    bool has = false;
    if (kGauss) {
        saved = gs->saved;
        has = gs->has_saved != 0;
    }
    const double g1 = gf1[t];
    const double g2 = __dmul_rn(gf2[t], tsqrt);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        double r;
        if (kGauss) {
            r = gauss_next(st, saved, has);
        } else {
            r = __dsub_rn(__dmul_rn(static_cast<double>(st.next()), 0x1p-24), 0.5);
        }
        const double fd = __dadd_rn(__dmul_rn(g1, vel[3 * a + d]), __dmul_rn(g2, r));
        force[3 * a + d] = __dadd_rn(force[3 * a + d], fd);
    }
    gs->s.i = st.i;
    gs->s.j = st.j;
    gs->s.v = st.v;
    if (kGauss) {
        gs->saved = saved;
        gs->has_saved = has ? 1u : 0u;
    }
}

// gaussian() with few deviates per atom per launch: the same calls, output
// layout and state semantics as gaussian_kernel (gauss_kernel.cu), stepping
// the state in place.
__global__ void __launch_bounds__(256)
    gaussian_inplace_kernel(ranmar_gauss_state* __restrict__ g, uint64_t n_atoms,
                            uint64_t per_step, uint64_t steps, double* __restrict__ out,
                            uint32_t* status) {
    const uint64_t a = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (a >= n_atoms) return;
    ranmar_gauss_state* gs = g + a;
    InPlace st{gs->s.lane, gs->s.i, gs->s.j, gs->s.v};
    if (!state_ok(st.i, st.j, st.v)) {
        atomicOr(status, kStatusBadState);
        return;
    }
    double saved = gs->saved;
    bool has = gs->has_saved != 0;
    for (uint64_t s = 0; s < steps; ++s) {
        double* o = out + (s * n_atoms + a) * per_step;
        for (uint64_t c = 0; c < per_step; ++c) st_cs(o + c, gauss_next(st, saved, has));
    }
    gs->s.i = st.i;
    gs->s.j = st.j;
    gs->s.v = st.v;
    gs->saved = saved;
    gs->has_saved = has ? 1u : 0u;
}

// ---- Stream bank: n streams transposed slot-major for consumers that draw the
// same number of outputs from every stream per launch (uniform-noise Langevin).
// Word layout (u32): rows 0..96 hold slot s of every stream (slot s = the
// latest x_m with m = s mod 97, loaded in canonical order X[s] =
// lane[(i0 - s) mod 97] as in K2), row 97 holds v, row 98 the stream's i0.
// After t outputs slot s still maps back to ring position (i0 - s) mod 97 and
// the cursor is (i0 - t) mod 97, so the round trip is byte-identical to t
// calls of step(). A launch that draws 3 outputs touches rows t, t+1, t+2 and
// their lag partners (mod 97) for all streams: every access is coalesced and
// DRAM moves ~44 B of state per stream-step instead of the ~370 B of sectors
// an in-place AoS update touches.
constexpr int kBankRows = 99;

// AoS records <-> slot-major bank, tiled: a block moves 64 records through a
// shared-memory tile [slot][atom] (row stride 65 words, so a record's scattered
// slots and a slot row's consecutive atoms both spread over the banks), with
// coalesced 16-B record accesses on one side and coalesced bank rows on the other.
constexpr int kBankAtoms = 64, kBankThreads = 256, kBankStride = 65;

__global__ void __launch_bounds__(kBankThreads)
    bank_from_states_kernel(const ranmar_state* __restrict__ st, uint64_t n,
                            uint32_t* __restrict__ bank, uint32_t* status) {
    __shared__ uint32_t tile[99 * kBankStride];  // slots 0..96, v, cursor
    __shared__ int ics[kBankAtoms];
    const int t = threadIdx.x;
    const uint64_t a0 = static_cast<uint64_t>(blockIdx.x) * kBankAtoms;
    const int cnt = n - a0 < static_cast<uint64_t>(kBankAtoms) ? static_cast<int>(n - a0) : kBankAtoms;
    if (t < cnt) {
        const ranmar_state* r = st + a0 + t;
        const int i0 = r->i;
        if (!state_ok(i0, r->j, r->v)) atomicOr(status, kStatusBadState);
        const int ic = static_cast<unsigned>(i0) < 97u ? i0 : 0;
        ics[t] = ic;
        tile[97 * kBankStride + t] = r->v;
        tile[98 * kBankStride + t] = static_cast<uint32_t>(ic);
    }
    __syncthreads();
    // record word w of atom a goes to slot (ic - w) mod 97 (canonical order)
    const uint4* src = reinterpret_cast<const uint4*>(st + a0);
    for (int u = t; u < cnt * 25; u += kBankThreads) {
        const int a = u / 25, c = u - 25 * a;
        const uint4 x = src[u];
        int sl = ics[a] - 4 * c;
        sl += sl < 0 ? 97 : 0;
        tile[sl * kBankStride + a] = x.x;
        if (c < 24) {
            sl = sl == 0 ? 96 : sl - 1;
            tile[sl * kBankStride + a] = x.y;
            sl = sl == 0 ? 96 : sl - 1;
            tile[sl * kBankStride + a] = x.z;
            sl = sl == 0 ? 96 : sl - 1;
            tile[sl * kBankStride + a] = x.w;
        }
    }
    __syncthreads();
    for (int x = t; x < 99 * kBankAtoms; x += kBankThreads) {
        const int sl = x / kBankAtoms, a = x - sl * kBankAtoms;
        if (a < cnt) bank[sl * n + a0 + a] = tile[sl * kBankStride + a];
    }
}

__global__ void __launch_bounds__(kBankThreads)
    bank_to_states_kernel(const uint32_t* __restrict__ bank, uint64_t n, uint32_t t97,
                          ranmar_state* __restrict__ st) {
    __shared__ uint32_t tile[99 * kBankStride];
    const int t = threadIdx.x;
    const uint64_t a0 = static_cast<uint64_t>(blockIdx.x) * kBankAtoms;
    const int cnt = n - a0 < static_cast<uint64_t>(kBankAtoms) ? static_cast<int>(n - a0) : kBankAtoms;
    for (int x = t; x < 99 * kBankAtoms; x += kBankThreads) {
        const int sl = x / kBankAtoms, a = x - sl * kBankAtoms;
        if (a < cnt) tile[sl * kBankStride + a] = bank[sl * n + a0 + a];
    }
    __syncthreads();
    uint4* dst = reinterpret_cast<uint4*>(st + a0);
    for (int u = t; u < cnt * 25; u += kBankThreads) {
        const int a = u / 25, c = u - 25 * a;
        const int ic = static_cast<int>(tile[98 * kBankStride + a]);
        int sl = ic - 4 * c;
        sl += sl < 0 ? 97 : 0;
        uint4 x;
        x.x = tile[sl * kBankStride + a] & kMask;
        if (c < 24) {
            sl = sl == 0 ? 96 : sl - 1;
            x.y = tile[sl * kBankStride + a] & kMask;
            sl = sl == 0 ? 96 : sl - 1;
            x.z = tile[sl * kBankStride + a] & kMask;
            sl = sl == 0 ? 96 : sl - 1;
            x.w = tile[sl * kBankStride + a] & kMask;
        } else {  // word 96, then the cursors after t steps and v
            int i = ic - static_cast<int>(t97);
            i += i < 0 ? 97 : 0;
            x.y = static_cast<uint32_t>(i);
            x.z = static_cast<uint32_t>(i >= 64 ? i - 64 : i + 33);
            x.w = tile[97 * kBankStride + a];
        }
        dst[u] = x;
    }
}

// Uniform-noise Langevin on a bank: every stream draws 3 outputs (an atom with
// a type outside [0, n_types] is flagged and its force left alone, but its
// stream still advances, so the bank stays in lockstep).
__global__ void __launch_bounds__(256)
    langevin_bank_kernel(uint32_t* __restrict__ bank, uint64_t n, uint32_t s0,
                         const double* __restrict__ vel, double* __restrict__ force,
                         const int32_t* __restrict__ type, const double* __restrict__ gf1,
                         const double* __restrict__ gf2, int32_t n_types, double tsqrt,
                         uint32_t* status) {
    const uint64_t a = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (a >= n) return;
    const int32_t t = type[a];
    const bool ok = t >= 0 && t <= n_types;
    if (!ok) atomicOr(status, kStatusBadType);
    uint32_t v = bank[97 * n + a];
    double r[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        int sl = static_cast<int>(s0) + d;
        sl -= sl >= 97 ? 97 : 0;
        const int pr = sl >= 33 ? sl - 33 : sl + 64;  // (sl + 64) mod 97: x_{m-33}
        uint32_t* xs = bank + sl * n + a;
        const uint32_t x = (*xs - bank[pr * n + a]) & kMask;
        *xs = x;
        v = add_mod_m(v, kStepA);
        r[d] = __dsub_rn(__dmul_rn(static_cast<double>((x - v) & kMask), 0x1p-24), 0.5);
    }
    bank[97 * n + a] = v;
    if (!ok) return;
    const double g1 = gf1[t];
    const double g2 = __dmul_rn(gf2[t], tsqrt);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double fd = __dadd_rn(__dmul_rn(g1, vel[3 * a + d]), __dmul_rn(g2, r[d]));
        force[3 * a + d] = __dadd_rn(force[3 * a + d], fd);
    }
}

}  // namespace

namespace {

// The same force update with the gaussian noise of this MD step already in HBM
// (noise[a][d], e.g. one K4 launch's deviates for many steps: gaussian() with
// 3 calls per atom per step, out[(step * n + a) * 3 + d]). Element-wise, so
// every access is coalesced (~100 B per atom-step instead of the in-place
// path's ~450). Equal to ranmar_langevin_dev(NOISE_GAUSSIAN) step by step when
// every atom is in the group at every step (the noise was drawn for all atoms).
__global__ void __launch_bounds__(256)
    langevin_noise_kernel(uint64_t n_atoms, const double* __restrict__ noise,
                          const double* __restrict__ vel, double* __restrict__ force,
                          const int32_t* __restrict__ type, const int32_t* __restrict__ mask,
                          int32_t groupbit, const double* __restrict__ gf1,
                          const double* __restrict__ gf2, int32_t n_types, double tsqrt,
                          uint32_t* status) {
    const uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= 3 * n_atoms) return;
    const uint64_t a = e / 3;
    if (mask != nullptr && (mask[a] & groupbit) == 0) return;
    const int32_t t = type[a];
    if (t < 0 || t > n_types) {
        if (e % 3 == 0) atomicOr(status, kStatusBadType);
        return;
    }
    const double g1 = gf1[t];
    const double g2 = __dmul_rn(gf2[t], tsqrt);
    const double fd = __dadd_rn(__dmul_rn(g1, vel[e]), __dmul_rn(g2, noise[e]));
    force[e] = __dadd_rn(force[e], fd);
}

}  // namespace

cudaError_t launch_langevin_noise(uint64_t n_atoms, const double* d_noise, const double* d_v,
                                  double* d_f, const int32_t* d_type, const int32_t* d_mask,
                                  int32_t groupbit, const double* d_gf1, const double* d_gf2,
                                  int32_t n_types, double tsqrt, uint32_t* status,
                                  cudaStream_t stream) {
    if (n_atoms == 0) return cudaSuccess;
    const unsigned blocks = static_cast<unsigned>((3 * n_atoms + 255) / 256);
    count_launch();
    langevin_noise_kernel<<<blocks, 256, 0, stream>>>(n_atoms, d_noise, d_v, d_f, d_type, d_mask,
                                                      groupbit, d_gf1, d_gf2, n_types, tsqrt, status);
    return cudaGetLastError();
}

cudaError_t launch_langevin(ranmar_gauss_state* d_g, uint64_t n_atoms, const double* d_v,
                            double* d_f, const int32_t* d_type, const int32_t* d_mask,
                            int32_t groupbit, const double* d_gf1, const double* d_gf2,
                            int32_t n_types, double tsqrt, int gauss, uint32_t* status,
                            cudaStream_t stream) {
    if (n_atoms == 0) return cudaSuccess;
    const unsigned blocks = static_cast<unsigned>((n_atoms + 255) / 256);
    count_launch();
    if (gauss)
        langevin_kernel<true><<<blocks, 256, 0, stream>>>(d_g, n_atoms, d_v, d_f, d_type, d_mask,
                                                          groupbit, d_gf1, d_gf2, n_types, tsqrt,
                                                          status);
    else
        langevin_kernel<false><<<blocks, 256, 0, stream>>>(d_g, n_atoms, d_v, d_f, d_type, d_mask,
                                                           groupbit, d_gf1, d_gf2, n_types, tsqrt,
                                                           status);
    return cudaGetLastError();
}

cudaError_t launch_gaussian_inplace(ranmar_gauss_state* d_g, uint64_t n_atoms, uint64_t per_step,
                                    uint64_t steps, double* d_out, uint32_t* status,
                                    cudaStream_t stream) {
    if (n_atoms == 0 || per_step == 0 || steps == 0) return cudaSuccess;
    const unsigned blocks = static_cast<unsigned>((n_atoms + 255) / 256);
    count_launch();
    gaussian_inplace_kernel<<<blocks, 256, 0, stream>>>(d_g, n_atoms, per_step, steps, d_out,
                                                        status);
    return cudaGetLastError();
}

cudaError_t launch_bank_from_states(const ranmar_state* d_states, uint64_t n, uint32_t* d_bank,
                                   uint32_t* status, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    count_launch();
    bank_from_states_kernel<<<static_cast<unsigned>((n + kBankAtoms - 1) / kBankAtoms), kBankThreads, 0,
                              stream>>>(d_states, n, d_bank, status);
    return cudaGetLastError();
}

cudaError_t launch_bank_to_states(const uint32_t* d_bank, uint64_t n, uint64_t t,
                                  ranmar_state* d_states, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    count_launch();
    bank_to_states_kernel<<<static_cast<unsigned>((n + kBankAtoms - 1) / kBankAtoms), kBankThreads, 0,
                            stream>>>(d_bank, n, static_cast<uint32_t>(t % 97), d_states);
    return cudaGetLastError();
}

cudaError_t launch_langevin_bank(uint32_t* d_bank, uint64_t n, uint64_t t, const double* d_v,
                                 double* d_f, const int32_t* d_type, const double* d_gf1,
                                 const double* d_gf2, int32_t n_types, double tsqrt,
                                 uint32_t* status, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    count_launch();
    langevin_bank_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(
        d_bank, n, static_cast<uint32_t>(t % 97), d_v, d_f, d_type, d_gf1, d_gf2, n_types, tsqrt,
        status);
    return cudaGetLastError();
}

}  // namespace rb
