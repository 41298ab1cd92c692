// K4: gaussian() on the GPU, thread per atom (sm_100a).
//
// gaussian() has no reference counterpart; the repo
// defines it in oracle/ranmar_oracle.c (or_gaussian): Marsaglia polar method
// on uniform() = next_f64 (core.hpp:70-72), v = 2u - 1, reject rsq >= 1 or
// rsq == 0, return v2 * fac and cache v1 * fac (Numerical Recipes pairing),
// log() being the correctly rounded crlog (gauss_math.cuh) so results are
// bit-identical to the oracle and to RanMars::gaussian with a correctly
// rounded libm log.
//
// Every gaussian() call consumes uniforms in pairs, so an atom's deviates are
// the cached one (if has_saved) followed by (v2 fac, v1 fac) for each
// ACCEPTED attempt pair. Each thread therefore loops over attempts (not one
// rejection loop per call, which would make a warp wait for its unluckiest
// lane at every call): draw two uniforms, test rsq in exact integer
// arithmetic (rsq = s / 2^46 with s = (u1 - 2^23)^2 + (u2 - 2^23)^2), and
// collect kBatch accepted pairs; then the kBatch fp64 chains (log, divide,
// sqrt; branch-free, gauss_math.cuh) run interleaved and emit 2 kBatch
// deviates. The last < 2 kBatch deviates go pair by pair; the last pair's
// second deviate becomes the cached one when the count is odd.
//
// The 97-word ring of each atom lives in shared memory column-major (slot s
// of thread t at s * kGT + t): every access of a warp hits 32 distinct banks
// whatever the (diverged) cursors. States are moved between HBM and the ring
// with 16-B vector accesses (the 416-B records are 16-B aligned).
#include <cstdint>
#include <type_traits>

#include "gauss_math.cuh"
#include "ranmar_device.cuh"

namespace rb {

namespace {

constexpr int kGT = 64;  // threads (atoms) per block: 24.8 KB of ring, 9 blocks/SM
// accepted pairs per fp64 batch. Config 5 (2^24 atoms x 300, per_step 3), with
// the pipelined ring loads and the split log: K = 3 (row-batched stores, 96
// registers, 9 blocks/SM) 20.30 ms; K = 6 (row-batched, 128 registers, 8
// blocks/SM) 21.30; K = 4 / 5 (per_step 3 does not divide 2K: countdown
// stores) 21.36 / 21.31; K = 8 22.05.
constexpr int kBatch = 3;

// The ring is the kernel's only shared memory, so it starts at the fixed
// offset of the CTA's shared window where dynamic shared memory begins (after
// the 1 KB the driver reserves per block on sm_90+). Ring accesses use that
// offset as the instruction's immediate: LDS/STS [R + 0x400], no base register.
// Written through a computed base, ptxas re-derives the window base (S2UR
// SR_CgaCtaId + ULEA) inside the lane-divergent attempt loop, or adds it with an
// IADD per access. The kernel checks the offset on entry and flags
// kStatusInternal (no work done) if a driver ever places it elsewhere.
constexpr uint32_t kRingBase = 0x400;

__device__ __forceinline__ uint32_t ring_ld(uint32_t off) {
    uint32_t x;
    asm volatile("ld.shared.u32 %0, [%1+1024];" : "=r"(x) : "r"(off));
    return x;
}
__device__ __forceinline__ void ring_st(uint32_t off, uint32_t x) {
    asm volatile("st.shared.u32 [%0+1024], %1;" ::"r"(off), "r"(x) : "memory");
}

// P > 0: per_step == P with 2K % P == 0 (compile time). When no lane of a warp
// starts with a cached deviate, every batch of 2K deviates then fills exactly
// 2K / P whole rows of the output, so its 2K stores address row pointers with
// immediate column offsets instead of walking the (row, column) countdown per
// deviate (~6.5 instructions each, ncu source page).
// P == -1: the moments consumer (ranmar_gaussian_moments_dev, §8f row 4): no
// deviate is stored; each atom's steps * per_step deviates (its cached one
// first) are summed in order, s1 = RN(s1 + x), s2 = RN(s2 + RN(x * x)), and
// out[2 atom], out[2 atom + 1] = s1, s2.
template <int K, int P>
__global__ void __launch_bounds__(kGT)
    gaussian_kernel(ranmar_gauss_state* __restrict__ g, uint64_t n_atoms, uint64_t per_step,
                    uint64_t steps, double* __restrict__ out, uint32_t* status) {
    extern __shared__ uint32_t ring[];  // [97][kGT], the only shared memory
    const int t = threadIdx.x;
    if (static_cast<uint32_t>(__cvta_generic_to_shared(ring)) != kRingBase) {
        if (t == 0) atomicOr(status, kStatusInternal);
        return;
    }
    const uint64_t atom = static_cast<uint64_t>(blockIdx.x) * kGT + t;
    if (atom >= n_atoms) return;
    ranmar_gauss_state* gs = g + atom;
    const int i0 = gs->s.i, j0 = gs->s.j;
    const uint32_t v0 = gs->s.v;
    if (!state_ok(i0, j0, v0)) {
        atomicOr(status, kStatusBadState);
        return;
    }
    {   // lanes -> ring column t, 16-B loads (L1 keeps each record's lines)
        const uint4* src = reinterpret_cast<const uint4*>(gs->s.lane);
#pragma unroll 4
        for (int q = 0; q < 24; ++q) {
            const uint4 x = src[q];
            ring[(4 * q + 0) * kGT + t] = x.x;
            ring[(4 * q + 1) * kGT + t] = x.y;
            ring[(4 * q + 2) * kGT + t] = x.z;
            ring[(4 * q + 3) * kGT + t] = x.w;
        }
        ring[96 * kGT + t] = gs->s.lane[96];
    }
    // cursors as byte offsets into the ring: slot s of this thread at 4 t + 4 kGT s.
    // Stepping down with wraparound is one VIADDMNMX: min(a - 4 kGT, top) (unsigned:
    // a < 4 kGT, i.e. slot 0, wraps to a huge value and yields top = slot 96).
    constexpr uint32_t kSlot = 4 * kGT;
    const uint32_t top = 4 * t + 96 * kSlot;
    uint32_t ai = 4 * t + i0 * kSlot;
    uint32_t aj = 4 * t + (i0 >= 64 ? i0 - 64 : i0 + 33) * kSlot;
    uint32_t v = v0;
    double saved = gs->saved;
    bool has = gs->has_saved != 0;

    const uint64_t G = steps * per_step;
    uint64_t q = 0;  // next deviate index of this atom
    // deviate q goes to out[(step * n_atoms + atom) * per_step + c]: a running pointer and a
    // countdown to the end of the atom's row of the current step
    double* po = out + atom * per_step;
    const uint64_t jump = (n_atoms - 1) * per_step;
    const uint32_t row = per_step < 0xFFFFFFFFull ? static_cast<uint32_t>(per_step) : 0xFFFFFFFFu;
    uint32_t left = row;
    double s1 = 0.0, s2 = 0.0;  // P == -1
    auto put = [&](double x) {
        if (P < 0) {
            s1 = __dadd_rn(s1, x);
            s2 = __dadd_rn(s2, __dmul_rn(x, x));
            return;
        }
        st_cs(po, x);
        ++po;
        if (--left == 0) {
            left = row;
            po += jump;
        }
    };
    if (has && G > 0) {
        put(saved);
        has = false;
        q = 1;
    }
    // one attempt: two uniforms (core.hpp:54-66 on the ring); true when
    // 0 < rsq < 1 holds exactly (rsq = s / 2^46). Software-pipelined: the
    // four ring operands of the NEXT attempt are loaded before this attempt's
    // two stores, so their shared-memory latency overlaps this attempt's
    // arithmetic. Safe because x_n = x_{n-97} - x_{n-33} reads nothing written
    // by the previous 32 steps: the next attempt's slots ai - 2, ai - 3 and
    // aj - 2, aj - 3 = ai + 31, ai + 30 (mod 97) are never ai or ai - 1, the
    // slots this attempt writes. a0 / a1 = the slots this attempt writes, aj
    // = the last aj slot loaded; c0..c3 = this attempt's operands.
    uint32_t a1 = min(ai - kSlot, top);
    uint32_t c0 = ring_ld(ai), c1 = ring_ld(aj);
    aj = min(aj - kSlot, top);
    uint32_t c2 = ring_ld(a1), c3 = ring_ld(aj);
    auto attempt = [&](uint32_t& u0, uint32_t& u1) -> bool {
        const uint32_t a2 = min(a1 - kSlot, top), a3 = min(a2 - kSlot, top);
        const uint32_t j2 = min(aj - kSlot, top), j3 = min(j2 - kSlot, top);
        const uint32_t x0 = c0 - c1, x1 = c2 - c3;
        c0 = ring_ld(a2);
        c1 = ring_ld(j2);
        c2 = ring_ld(a3);
        c3 = ring_ld(j3);
        ring_st(ai, x0);
        ring_st(a1, x1);
        ai = a2;
        a1 = a3;
        aj = j3;
        v = add_mod_m(v, kStepA);
        u0 = (x0 - v) & kMask;
        v = add_mod_m(v, kStepA);
        u1 = (x1 - v) & kMask;
        const int32_t da = static_cast<int32_t>(u0) - (1 << 23);
        const int32_t db = static_cast<int32_t>(u1) - (1 << 23);
        const int64_t s = static_cast<int64_t>(da) * da + static_cast<int64_t>(db) * db;
        return s > 0 && s < (int64_t(1) << 46);
    };
    auto accept = [&](uint32_t& u0, uint32_t& u1) {
        while (!attempt(u0, u1)) {
        }
    };
    // Batches of K accepted pairs. One attempt loop collects all K (accepted
    // pairs shift into a[], b[] in order), so a warp waits for its slowest lane
    // once per batch rather than once per pair; then the K independent fp64
    // chains (log, divide, sqrt) are interleaved, so the fp64 pipe sees K-fold
    // instruction-level parallelism instead of one dependent chain per thread.
    static_assert(P == 0 || (2 * K) % P == 0, "whole rows per batch");
    constexpr int kRowsPB = P > 0 ? 2 * K / P : 1;
    const bool rows_fast = P > 0 && __all_sync(__activemask(), q == 0);
    const uint64_t row_stride = n_atoms * per_step;  // elements between an atom's rows
    while (G - q >= 2 * K) {
        uint32_t a[K], b[K];
        for (int got = 0; got < K;) {
            uint32_t u0, u1;
            if (attempt(u0, u1)) {
#pragma unroll
                for (int k = 0; k + 1 < K; ++k) {
                    a[k] = a[k + 1];
                    b[k] = b[k + 1];
                }
                a[K - 1] = u0;
                b[K - 1] = u1;
                ++got;
            }
        }
        double v1[K], v2[K], fac[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            v1[k] = polar_v(a[k]);
            v2[k] = polar_v(b[k]);
        }
        {   // every chain's fast log first, the rare accurate phase after all of them
            double rsq[K];
            bool all_ok = true;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                rsq[k] = polar_rsq(a[k], b[k]);
                bool ok;
                fac[k] = crlog_fast(rsq[k], ok);
                all_ok = all_ok && ok;
            }
            if (__builtin_expect(!all_ok, 0)) {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    bool ok;
                    crlog_fast(rsq[k], ok);
                    if (!ok) fac[k] = crlog_accurate(rsq[k]).y;
                }
            }
#pragma unroll
            for (int k = 0; k < K; ++k) fac[k] = polar_fac_of(rsq[k], fac[k]);
        }
        if (P > 0 && rows_fast) {  // po is at the start of a row
            double* rp[kRowsPB];
            rp[0] = po;
#pragma unroll
            for (int r = 1; r < kRowsPB; ++r) rp[r] = rp[r - 1] + row_stride;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                st_cs(rp[(2 * k) / (P > 0 ? P : 1)] + (2 * k) % (P > 0 ? P : 1), __dmul_rn(v2[k], fac[k]));
                saved = __dmul_rn(v1[k], fac[k]);
                st_cs(rp[(2 * k + 1) / (P > 0 ? P : 1)] + (2 * k + 1) % (P > 0 ? P : 1), saved);
            }
            po = rp[kRowsPB - 1] + row_stride;
        } else {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                put(__dmul_rn(v2[k], fac[k]));
                saved = __dmul_rn(v1[k], fac[k]);  // the oracle keeps the last pair's v1 fac
                put(saved);
            }
        }
        q += 2 * K;
    }
    while (q < G) {
        uint32_t u0, u1;
        accept(u0, u1);
        const double v1 = polar_v(u0), v2 = polar_v(u1);
        const double fac = polar_fac(u0, u1);
        saved = __dmul_rn(v1, fac);
        put(__dmul_rn(v2, fac));
        if (q + 1 < G) {
            put(saved);
        } else {
            has = true;
        }
        q += 2;
    }
    // ring -> lanes (16-B stores), cursors, v, cache
    {
        uint4* dst = reinterpret_cast<uint4*>(gs->s.lane);
#pragma unroll 4
        for (int qq = 0; qq < 24; ++qq)
            dst[qq] = make_uint4(ring[(4 * qq + 0) * kGT + t] & kMask, ring[(4 * qq + 1) * kGT + t] & kMask,
                                 ring[(4 * qq + 2) * kGT + t] & kMask, ring[(4 * qq + 3) * kGT + t] & kMask);
    }
    const int i = static_cast<int>((ai - 4 * t) / kSlot);
    *reinterpret_cast<uint4*>(gs->s.lane + 96) =
        make_uint4(ring[96 * kGT + t] & kMask, static_cast<uint32_t>(i),
                   static_cast<uint32_t>(i >= 64 ? i - 64 : i + 33), v);
    gs->saved = saved;
    gs->has_saved = has ? 1u : 0u;
    if (P < 0) {
        out[2 * atom] = s1;
        out[2 * atom + 1] = s2;
    }
}

}  // namespace

// Self-check of div_rn / sqrt_rn against the library's __ddiv_rn / __dsqrt_rn
// on the operands gaussian() can produce: rsq = s / 2^46 for pseudo-random
// s in [1, 2^46) plus the range ends and powers of two; per value the fac
// division and the sqrt are compared bitwise.
__global__ void fp64_selfcheck_kernel(uint64_t n, uint64_t seed,
                                      unsigned long long* __restrict__ bad) {
    unsigned long long miss = 0;
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n;
         k += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t z = seed + k * 0x9E3779B97F4A7C15ull;  // splitmix64
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        uint64_t s = z & ((uint64_t(1) << 46) - 1);
        if (k < 47) s = uint64_t(1) << k;  // powers of two: z = 0 in crlog
        if (k == 47) s = (uint64_t(1) << 46) - 1;
        if (s == 0 || s >= (uint64_t(1) << 46)) s = 1;
        const double rsq = static_cast<double>(s) * 0x1p-46;
        const double num = __dmul_rn(-2.0, crlog(rsq));
        const double q1 = div_rn(num, rsq), q2 = __ddiv_rn(num, rsq);
        miss += __double_as_longlong(q1) != __double_as_longlong(q2);
        miss += __double_as_longlong(sqrt_rn(q2)) != __double_as_longlong(__dsqrt_rn(q2));
    }
    if (miss) atomicAdd(bad, miss);
}

cudaError_t launch_fp64_selfcheck(uint64_t n, uint64_t seed, unsigned long long* d_bad,
                                  cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    count_launch();
    fp64_selfcheck_kernel<<<148 * 8, 256, 0, stream>>>(n, seed, d_bad);
    return cudaGetLastError();
}

// Exhaustive check of crlog on gaussian()'s domain: rsq = s / 2^46 for
// s in [s0, s0 + n). counts[0] = inputs whose fast phase did not decide,
// counts[1] = inputs whose accurate phase did not decide either (the claim
// "correctly rounded on the whole domain" needs 0 over all 2^46 - 1 inputs),
// counts[2] = (mode 1 only) inputs where the fast phase decided a value other
// than the accurate phase's, counts[3] = number of inputs recorded; their s
// values go to fails[0 .. cap) for the CPU to re-check against the oracle and
// mpmath: the fast-phase failures (modes 0, 1) or only the accurate-phase
// failures (mode 2).
__global__ void crlog_sweep_kernel(uint64_t s0, uint64_t n, int mode,
                                   unsigned long long* __restrict__ counts,
                                   uint64_t* __restrict__ fails, uint64_t cap) {
    unsigned long long nfast = 0, nacc = 0, nmis = 0;
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n;
         k += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t s = s0 + k;
        const double x = static_cast<double>(s) * 0x1p-46;
        bool fast;
        const double y = crlog(x, &fast);
        if (!fast) {
            ++nfast;
            const bool undecided = crlog_accurate(x).ok == 0;
            nacc += undecided;
            if (mode != 2 || undecided) {  // mode 2 records only accurate-phase failures
                const unsigned long long slot = atomicAdd(counts + 3, 1ull);
                if (slot < cap) fails[slot] = s;
            }
        } else if (mode == 1) {
            const CrlogAcc a = crlog_accurate(x);
            nacc += a.ok == 0;
            nmis += __double_as_longlong(a.y) != __double_as_longlong(y);
        }
    }
    if (nfast) atomicAdd(counts + 0, nfast);
    if (nacc) atomicAdd(counts + 1, nacc);
    if (nmis) atomicAdd(counts + 2, nmis);
}

cudaError_t launch_crlog_sweep(uint64_t s0, uint64_t n, int mode, unsigned long long* d_counts,
                               uint64_t* d_fails, uint64_t cap, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    count_launch();
    crlog_sweep_kernel<<<148 * 8, 256, 0, stream>>>(s0, n, mode, d_counts, d_fails, cap);
    return cudaGetLastError();
}

template <int K>
cudaError_t launch_gaussian_k(ranmar_gauss_state* d_g, uint64_t n_atoms, uint64_t per_step,
                              uint64_t steps, double* d_out, uint32_t* status,
                              cudaStream_t stream) {
    const int smem = 97 * kGT * 4;  // 24.8 KB: within the default 48 KB limit
    const uint64_t blocks = (n_atoms + kGT - 1) / kGT;
    count_launch();
    const dim3 grid(static_cast<unsigned>(blocks));
    auto go = [&](auto pc) {
        constexpr int P = decltype(pc)::value;
        if constexpr (P == 0 || (2 * K) % P == 0)
            gaussian_kernel<K, P><<<grid, kGT, smem, stream>>>(d_g, n_atoms, per_step, steps, d_out, status);
        else
            gaussian_kernel<K, 0><<<grid, kGT, smem, stream>>>(d_g, n_atoms, per_step, steps, d_out, status);
    };
    switch (per_step) {  // row-batched stores for the per-step counts that divide 2K
        case 1: go(std::integral_constant<int, 1>{}); break;
        case 2: go(std::integral_constant<int, 2>{}); break;
        case 3: go(std::integral_constant<int, 3>{}); break;
        case 4: go(std::integral_constant<int, 4>{}); break;
        case 6: go(std::integral_constant<int, 6>{}); break;
        default: go(std::integral_constant<int, 0>{});
    }
    return cudaGetLastError();
}

cudaError_t launch_gaussian_moments(ranmar_gauss_state* d_g, uint64_t n_atoms, uint64_t count,
                                    double* d_out, uint32_t* status, cudaStream_t stream) {
    if (n_atoms == 0 || count == 0) return cudaSuccess;
    const int smem = 97 * kGT * 4;
    const uint64_t blocks = (n_atoms + kGT - 1) / kGT;
    count_launch();
    gaussian_kernel<kBatch, -1><<<static_cast<unsigned>(blocks), kGT, smem, stream>>>(d_g, n_atoms, count, 1,
                                                                                      d_out, status);
    return cudaGetLastError();
}

cudaError_t launch_gaussian_inplace(ranmar_gauss_state*, uint64_t, uint64_t, uint64_t, double*,
                                    uint32_t*, cudaStream_t);

cudaError_t launch_gaussian(ranmar_gauss_state* d_g, uint64_t n_atoms, uint64_t per_step,
                            uint64_t steps, double* d_out, uint32_t* status,
                            cudaStream_t stream) {
    if (n_atoms == 0 || per_step == 0 || steps == 0) return cudaSuccess;
    // Few deviates per atom: step the states in place (K6). Measured at 2^24
    // atoms: in place 2.2 / 3.3 / 5.1 / 9.0 ms for 3 / 6 / 12 / 24 deviates,
    // staged ring 6.0 / 6.0 / 6.1 / 6.4 ms.
    constexpr uint64_t kInplaceMax = 12;
    if (steps * per_step <= kInplaceMax)
        return launch_gaussian_inplace(d_g, n_atoms, per_step, steps, d_out, status, stream);
    return launch_gaussian_k<kBatch>(d_g, n_atoms, per_step, steps, d_out, status, stream);
}

}  // namespace rb
