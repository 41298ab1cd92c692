// K4r: gaussian() on the GPU, thread per atom, the 97-word ring in REGISTERS
// (sm_100a).
//
// Convention (oracle/ranmar_oracle.c or_gaussian, LAMMPS RanMars::gaussian's
// form): Marsaglia polar method on uniform() = next_f64 (core.hpp:70-72),
// v = 2u - 1, reject rsq >= 1 or rsq == 0, return v2 * fac and cache v1 * fac,
// log() the correctly rounded crlog (gauss_math.cuh).
//
// An atom's deviates are the cached one (if has_saved) followed by
// (v2 fac, v1 fac) for each ACCEPTED attempt pair, so the kernel splits the
// work in two phases per warp:
//   attempts  every lane runs the same attempt of its own stream in lock-step:
//             the ring lives in 97 registers (slot s holds the latest x_n with
//             n = s mod 97, as in K2 consume_kernel.cu), so attempt A of the
//             97-attempt cycle touches compile-time slots 2A and 2A + 1 mod 97
//             and no lane ever waits for another lane's rejections. Accepted
//             pairs (u1, u2) go to the lane's FIFO column in shared memory.
//   fp64      after every chunk of 16 attempts, batches of K queued pairs per
//             lane run the K interleaved log / divide / sqrt chains
//             (gauss_math.cuh) while every lane holds K pairs (lock-step, so
//             consecutive lanes store consecutive atoms of a step row), or for
//             the lanes whose FIFO could overflow in the next chunk.
// A lane stops attempting once it has queued the pairs this launch needs
// (predicated off; its registers then hold the ring exactly as its n =
// 2 x attempts uniforms left it) and the last queued pairs are drained at the
// end. The ring goes back to the record in its layout: slot s <-> ring position
// (i0 - s) mod 97 whatever n is, cursors moved by n, v advanced (jump.hpp:32-48).
//
// Launch contract: steps * per_step < 2^32 (the launcher splits longer
// launches by steps; consecutive launches compose through the cached deviate).
#include <cstdint>
#include <cstdlib>

#include "gauss_math.cuh"
#include "ranmar_device.cuh"

namespace rb {

namespace {

constexpr int kRT = 128;    // threads (atoms) per block
constexpr int kQCap = 64;   // FIFO column per lane: queued accepted pairs
constexpr int kRK = 3;      // pairs per fp64 batch
constexpr int kChunk = 16;  // attempts between fp64 phases (97 = 6 x 16 + 1)
constexpr int kQStride = kRT * 8;                         // bytes between FIFO rows
constexpr int kRSmem = kQCap * kQStride;                  // 64 KB per block
static_assert(kQCap - kChunk >= kRK, "FIFO headroom");

__device__ __forceinline__ void q_st(uint32_t addr, uint32_t a, uint32_t b) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void q_ld(uint32_t addr, uint32_t& a, uint32_t& b) {
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(addr));
}

struct K4rLane {
    uint32_t v;      // arithmetic part after the uniforms used so far
    uint32_t tail;   // pairs queued (= accepted) so far
    uint32_t head;   // pairs turned into deviates so far
    uint32_t T;      // pairs this launch needs: ceil((G - has) / 2)
    uint32_t att;    // attempts made
    uint32_t qcol;   // shared address of this lane's FIFO column
};

// (k (m - d)) mod m: the arithmetic part's advance over k steps (core.hpp:61)
__host__ __device__ constexpr uint32_t arith_step(int k) {
    return static_cast<uint32_t>((static_cast<uint64_t>(k) * kStepA) % kMod);
}

// Attempt A (0..96) of the 97-attempt cycle: uniforms 2A, 2A + 1 of the cycle
// at ring slots (2A) mod 97 and (2A + 1) mod 97 (core.hpp:54-66).
// SAFE: every lane needs at least as many pairs as the chunk has attempts, so
// no lane can overshoot and the attempt runs unconditionally; v of the k-th
// uniform of the chunk is vb + k (m - d) mod m from the chunk's base vb (two
// independent ops per uniform instead of a serial chain through the chunk).
// Otherwise the attempt is predicated on the lane still needing pairs.
template <int A, int A0, bool SAFE>
__device__ __forceinline__ void attempt(uint32_t (&X)[97], K4rLane& L, uint32_t vb) {
    constexpr int s0 = (2 * A) % 97, s1 = (2 * A + 1) % 97;
    uint32_t u0, u1;
    if (SAFE) {
        X[s0] -= X[(s0 + 64) % 97];
        X[s1] -= X[(s1 + 64) % 97];
        u0 = (X[s0] - add_mod_m(vb, arith_step(2 * (A - A0) + 1))) & kMask;
        u1 = (X[s1] - add_mod_m(vb, arith_step(2 * (A - A0) + 2))) & kMask;
    } else {
        u0 = u1 = 1u << 23;  // inactive: s = 0, rejected
        if (L.tail < L.T) {
            X[s0] -= X[(s0 + 64) % 97];
            L.v = add_mod_m(L.v, kStepA);
            u0 = (X[s0] - L.v) & kMask;
            X[s1] -= X[(s1 + 64) % 97];
            L.v = add_mod_m(L.v, kStepA);
            u1 = (X[s1] - L.v) & kMask;
            ++L.att;
        }
    }
    const int32_t da = static_cast<int32_t>(u0) - (1 << 23);
    const int32_t db = static_cast<int32_t>(u1) - (1 << 23);
    const int64_t s = static_cast<int64_t>(da) * da + static_cast<int64_t>(db) * db;
    if (s > 0 && s < (int64_t(1) << 46)) {  // exact 0 < rsq < 1, rsq = s / 2^46
        q_st(L.qcol + (L.tail & (kQCap - 1)) * kQStride, u0, u1);
        ++L.tail;
    }
}

template <int A, int A0, int E, bool SAFE>
struct Attempts {
    static __device__ __forceinline__ void run(uint32_t (&X)[97], K4rLane& L, uint32_t vb) {
        attempt<A, A0, SAFE>(X, L, vb);
        Attempts<A + 1, A0, E, SAFE>::run(X, L, vb);
    }
};
template <int A0, int E, bool SAFE>
struct Attempts<E, A0, E, SAFE> {
    static __device__ __forceinline__ void run(uint32_t (&)[97], K4rLane&, uint32_t) {}
};

template <int C>
__device__ __forceinline__ void chunk(uint32_t (&X)[97], K4rLane& L) {
    constexpr int a = C * kChunk, e = (a + kChunk < 97) ? a + kChunk : 97;
    if (__all_sync(0xffffffffu, L.T - L.tail >= static_cast<uint32_t>(e - a))) {
        const uint32_t vb = L.v;
        Attempts<a, a, e, true>::run(X, L, vb);
        L.v = add_mod_m(vb, arith_step(2 * (e - a)));
        L.att += e - a;
    } else {
        Attempts<a, a, e, false>::run(X, L, 0);
    }
}

// P > 0: per_step == P divides 2K (compile time). A full batch whose lane sits
// at the start of a step row (q % P == 0) fills 2K / P whole rows, stored
// through row pointers at immediate column offsets instead of the per-deviate
// (row, column) countdown.
template <int P>
__global__ void __launch_bounds__(kRT)
    gaussian_reg_kernel(ranmar_gauss_state* __restrict__ g, uint64_t n_atoms, uint32_t per_step,
                        uint32_t G, double* __restrict__ out, uint32_t* status) {
    static_assert(P == 0 || (2 * kRK) % P == 0, "whole rows per batch");
    extern __shared__ __align__(16) unsigned char k4r_smem[];
    const int t = threadIdx.x;
    const uint64_t atom = static_cast<uint64_t>(blockIdx.x) * kRT + t;
    bool live = atom < n_atoms;
    ranmar_gauss_state* gs = g + (live ? atom : 0);
    int i0 = 0, j0 = 0;
    K4rLane L;
    L.v = 0;
    L.tail = L.head = L.T = L.att = 0;
    L.qcol = static_cast<uint32_t>(__cvta_generic_to_shared(k4r_smem)) + t * 8;
    uint32_t X[97];
    bool has = false;
    double saved = 0.0;
    if (live) {
        i0 = gs->s.i;
        j0 = gs->s.j;
        L.v = gs->s.v;
        if (!state_ok(i0, j0, L.v)) {
            atomicOr(status, kStatusBadState);
            live = false;
        }
    }
    if (live) {
#pragma unroll
        for (int s = 0; s < 97; ++s) X[s] = gs->s.lane[(i0 - s + 97) % 97];  // canonical order
        has = gs->has_saved != 0;
        saved = gs->saved;
        L.T = (G - (has ? 1u : 0u) + 1) / 2;
    } else {
#pragma unroll
        for (int s = 0; s < 97; ++s) X[s] = 0;
    }
    // deviate q of this atom goes to out[(q / per_step * n_atoms + atom) * per_step + q % per_step]:
    // a running pointer and a countdown to the end of the atom's row of the current step
    double* po = out + atom * per_step;
    const uint64_t jump = (n_atoms - 1) * per_step;
    const uint64_t row_stride = n_atoms * per_step;  // elements between an atom's rows
    uint32_t left = per_step;
    uint32_t q = 0;
    auto put = [&](double x) {
        st_cs(po, x);
        ++po;
        if (--left == 0) {
            left = per_step;
            po += jump;
        }
    };
    if (live && has) {
        put(saved);
        has = false;
        q = 1;
    }

    // nv (0..K) queued pairs -> deviates, K chains interleaved
    auto batch = [&](uint32_t nv) {
        uint32_t a[kRK], b[kRK];
#pragma unroll
        for (int k = 0; k < kRK; ++k) {
            a[k] = 0xC00000u;  // an accepted dummy (v1 = 1/2, v2 = 0) for the unused chains
            b[k] = 0x800000u;
            if (static_cast<uint32_t>(k) < nv) q_ld(L.qcol + ((L.head + k) & (kQCap - 1)) * kQStride, a[k], b[k]);
        }
        double rsq[kRK], lg[kRK];
        bool all_ok = true;
#pragma unroll
        for (int k = 0; k < kRK; ++k) {
            rsq[k] = polar_rsq(a[k], b[k]);
            bool ok;
            lg[k] = crlog_fast(rsq[k], ok);
            all_ok = all_ok && ok;
        }
        if (__builtin_expect(!all_ok, 0)) {
#pragma unroll
            for (int k = 0; k < kRK; ++k) {
                bool ok;
                crlog_fast(rsq[k], ok);
                if (!ok) lg[k] = crlog_accurate(rsq[k]).y;
            }
        }
        double d1[kRK], d2[kRK];
#pragma unroll
        for (int k = 0; k < kRK; ++k) {
            const double fac = polar_fac_of(rsq[k], lg[k]);
            d2[k] = __dmul_rn(polar_v(b[k]), fac);
            d1[k] = __dmul_rn(polar_v(a[k]), fac);
        }
        if (P > 0 && nv == kRK && q % (P > 0 ? P : 1) == 0 && q + 2 * kRK <= G) {
            constexpr int kRows = P > 0 ? 2 * kRK / P : 1;
            constexpr int PP = P > 0 ? P : 1;
#pragma unroll
            for (int k = 0; k < kRK; ++k) {
                st_cs(po + ((2 * k) / PP) * row_stride + (2 * k) % PP, d2[k]);
                st_cs(po + ((2 * k + 1) / PP) * row_stride + (2 * k + 1) % PP, d1[k]);
            }
            po += kRows * row_stride;
            saved = d1[kRK - 1];
            q += 2 * kRK;
        } else {
#pragma unroll
            for (int k = 0; k < kRK; ++k) {
                if (static_cast<uint32_t>(k) < nv) {
                    put(d2[k]);
                    if (q + 1 < G) {
                        put(d1[k]);
                    } else {
                        has = true;  // an odd count: v1 fac stays cached
                    }
                    saved = d1[k];
                    q += 2;
                }
            }
        }
        L.head += nv;
    };

    uint32_t c = 0;  // chunk of the 97-attempt cycle
    for (;;) {
        if (!__any_sync(0xffffffffu, L.tail < L.T)) break;
        switch (c) {
            case 0: chunk<0>(X, L); break;
            case 1: chunk<1>(X, L); break;
            case 2: chunk<2>(X, L); break;
            case 3: chunk<3>(X, L); break;
            case 4: chunk<4>(X, L); break;
            case 5: chunk<5>(X, L); break;
            default: chunk<6>(X, L); break;
        }
        c = c == 6 ? 0 : c + 1;
        // lock-step batches while every lane holds K pairs (or has stopped
        // attempting); lanes whose FIFO could overflow in the next chunk are
        // drained regardless
        for (;;) {
            const uint32_t cnt = L.tail - L.head;
            const bool done = L.tail == L.T;
            const bool go = __all_sync(0xffffffffu, cnt >= kRK || done)
                                ? __any_sync(0xffffffffu, cnt > 0)
                                : __any_sync(0xffffffffu, cnt > kQCap - kChunk);
            if (!go) break;
            const uint32_t nv = cnt >= kRK ? kRK : (done ? cnt : 0u);
            if (nv) batch(nv);
        }
    }
    for (;;) {  // drain
        const uint32_t cnt = L.tail - L.head;
        if (!__any_sync(0xffffffffu, cnt > 0)) break;
        if (cnt > 0) batch(cnt < kRK ? cnt : kRK);
    }
    if (!live) return;
    // slot s <-> ring position (i0 - s) mod 97 for any n (see consume_kernel.cu)
#pragma unroll
    for (int s = 0; s < 97; ++s) gs->s.lane[(i0 - s + 97) % 97] = X[s] & kMask;
    const uint32_t n = 2 * L.att;
    const int nm = static_cast<int>(n % 97);
    gs->s.i = (i0 - nm + 97) % 97;
    gs->s.j = (j0 - nm + 97) % 97;
    gs->s.v = L.v;
    gs->saved = saved;
    gs->has_saved = has ? 1u : 0u;
}

// ---------------------------------------------------------------- K4ws
// Warp-specialised K4r: per 128 atoms, four PRODUCER warps own the rings in
// registers and run the attempt chunks (no fp64 state), four CONSUMER warps
// (one per producer warp, same atoms, same lanes) turn the queued pairs into
// deviates with K = kWK interleaved fp64 chains (no ring state), so neither role
// carries the other's registers and both fit 2 blocks = 16 warps per SM.
// Hand-off per warp pair through the FIFO columns and named barriers:
//   producer: [k >= 2: wait EMPTY(k - 2)] chunk k -> tails[k & 1] -> arrive FULL(k)
//   consumer: wait FULL(k) -> tails[k & 1] -> batches -> arrive EMPTY(k) (unless done)
// so the producer runs one chunk ahead. The consumer leaves at most kWLim pairs
// per lane after a phase, hence <= kWLim + 2 x 16 <= kQCap pairs are queued.
constexpr int kWT = 128;           // atoms per block (threads = 2 kWT)
constexpr int kWK = 6;             // pairs per consumer batch
constexpr int kWLim = kQCap - 2 * kChunk;  // leftover bound after a phase
constexpr int kWSmem = kQCap * kQStride + 2 * kWT * 4;  // FIFO + double-buffered tails
static_assert(kWT == kRT, "FIFO layout shared with K4r");

__device__ __forceinline__ void named_sync(int id) {
    asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}
__device__ __forceinline__ void named_arrive(int id) {
    asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory");
}

template <int P>
__global__ void __launch_bounds__(2 * kWT, 2)
    gaussian_ws_kernel(ranmar_gauss_state* __restrict__ g, uint64_t n_atoms, uint32_t per_step,
                       uint32_t G, double* __restrict__ out, uint32_t* status) {
    static_assert(P == 0 || (2 * kWK) % P == 0, "whole rows per batch");
    extern __shared__ __align__(16) unsigned char k4w_smem[];
    const int tid = threadIdx.x;
    const bool producer = tid < kWT;
    const int t = tid & (kWT - 1), w = t >> 5;
    // named barriers of this warp pair: FULL[k & 1] = 4w + (k & 1), EMPTY[k & 1] =
    // 4w + 2 + (k & 1). Alternating two of each keeps a barrier from receiving a
    // second arrival of one side before the other side's sync (a named barrier
    // counts arrivals, it is not a semaphore): chunk k + 2 waits for phase k.
    auto full_id = [&](uint32_t k) { return 4 * w + static_cast<int>(k & 1); };
    auto empty_id = [&](uint32_t k) { return 4 * w + 2 + static_cast<int>(k & 1); };
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(k4w_smem));
    const uint32_t qcol = sbase + t * 8;
    const uint32_t tails = sbase + kQCap * kQStride;  // [2][kWT] u32
    const uint64_t atom = static_cast<uint64_t>(blockIdx.x) * kWT + t;
    bool live = atom < n_atoms;
    ranmar_gauss_state* gs = g + (live ? atom : 0);
    int i0 = 0, j0 = 0;
    uint32_t v = 0;
    if (live) {
        i0 = gs->s.i;
        j0 = gs->s.j;
        v = gs->s.v;
        if (!state_ok(i0, j0, v)) {
            if (producer) atomicOr(status, kStatusBadState);
            live = false;
        }
    }
    const bool has0 = live && gs->has_saved != 0;
    const uint32_t T = live ? (G - (has0 ? 1u : 0u) + 1) / 2 : 0u;

    if (producer) {
        K4rLane L;
        L.v = v;
        L.tail = L.head = L.att = 0;
        L.T = T;
        L.qcol = qcol;
        uint32_t X[97];
        if (live) {
#pragma unroll
            for (int s = 0; s < 97; ++s) X[s] = gs->s.lane[(i0 - s + 97) % 97];  // canonical order
        } else {
#pragma unroll
            for (int s = 0; s < 97; ++s) X[s] = 0;
        }
        uint32_t c = 0, published = 0;
        for (;;) {
            if (!__any_sync(0xffffffffu, L.tail < L.T) && published > 0) break;
            if (published >= 2) named_sync(empty_id(published - 2));
            switch (c) {
                case 0: chunk<0>(X, L); break;
                case 1: chunk<1>(X, L); break;
                case 2: chunk<2>(X, L); break;
                case 3: chunk<3>(X, L); break;
                case 4: chunk<4>(X, L); break;
                case 5: chunk<5>(X, L); break;
                default: chunk<6>(X, L); break;
            }
            c = c == 6 ? 0 : c + 1;
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(tails + ((published & 1) * kWT + t) * 4), "r"(L.tail)
                         : "memory");
            named_arrive(full_id(published));
            ++published;
        }
        if (published >= 2) named_sync(empty_id(published - 2));  // the consumer's last EMPTY arrival
        if (!live) return;
        // slot s <-> ring position (i0 - s) mod 97 for any n (see consume_kernel.cu)
#pragma unroll
        for (int s = 0; s < 97; ++s) gs->s.lane[(i0 - s + 97) % 97] = X[s] & kMask;
        const uint32_t n = 2 * L.att;
        const int nm = static_cast<int>(n % 97);
        gs->s.i = (i0 - nm + 97) % 97;
        gs->s.j = (j0 - nm + 97) % 97;
        gs->s.v = L.v;
        return;
    }

    // ---- consumer
    bool has = has0;
    double saved = live ? gs->saved : 0.0;
    double* po = out + atom * per_step;
    const uint64_t jump = (n_atoms - 1) * per_step;
    const uint64_t row_stride = n_atoms * per_step;
    uint32_t left = per_step;
    uint32_t q = 0, head = 0;
    auto put = [&](double x) {
        st_cs(po, x);
        ++po;
        if (--left == 0) {
            left = per_step;
            po += jump;
        }
    };
    if (has) {
        put(saved);
        has = false;
        q = 1;
    }
    auto batch = [&](uint32_t nv) {
        uint32_t a[kWK], b[kWK];
#pragma unroll
        for (int k = 0; k < kWK; ++k) {
            a[k] = 0xC00000u;  // an accepted dummy (v1 = 1/2, v2 = 0) for the unused chains
            b[k] = 0x800000u;
            if (static_cast<uint32_t>(k) < nv) q_ld(qcol + ((head + k) & (kQCap - 1)) * kQStride, a[k], b[k]);
        }
        double rsq[kWK], lg[kWK];
        bool all_ok = true;
#pragma unroll
        for (int k = 0; k < kWK; ++k) {
            rsq[k] = polar_rsq(a[k], b[k]);
            bool ok;
            lg[k] = crlog_fast(rsq[k], ok);
            all_ok = all_ok && ok;
        }
        if (__builtin_expect(!all_ok, 0)) {
#pragma unroll
            for (int k = 0; k < kWK; ++k) {
                bool ok;
                crlog_fast(rsq[k], ok);
                if (!ok) lg[k] = crlog_accurate(rsq[k]).y;
            }
        }
        double d1[kWK], d2[kWK];
#pragma unroll
        for (int k = 0; k < kWK; ++k) {
            const double fac = polar_fac_of(rsq[k], lg[k]);
            d2[k] = __dmul_rn(polar_v(b[k]), fac);
            d1[k] = __dmul_rn(polar_v(a[k]), fac);
        }
        if (P > 0 && nv == kWK && q % (P > 0 ? P : 1) == 0 && q + 2 * kWK <= G) {
            constexpr int kRows = P > 0 ? 2 * kWK / P : 1;
            constexpr int PP = P > 0 ? P : 1;
#pragma unroll
            for (int k = 0; k < kWK; ++k) {
                st_cs(po + ((2 * k) / PP) * row_stride + (2 * k) % PP, d2[k]);
                st_cs(po + ((2 * k + 1) / PP) * row_stride + (2 * k + 1) % PP, d1[k]);
            }
            po += kRows * row_stride;
            saved = d1[kWK - 1];
            q += 2 * kWK;
        } else {
#pragma unroll
            for (int k = 0; k < kWK; ++k) {
                if (static_cast<uint32_t>(k) < nv) {
                    put(d2[k]);
                    if (q + 1 < G) {
                        put(d1[k]);
                    } else {
                        has = true;  // an odd count: v1 fac stays cached
                    }
                    saved = d1[k];
                    q += 2;
                }
            }
        }
        head += nv;
    };
    for (uint32_t k = 0;; ++k) {
        named_sync(full_id(k));
        uint32_t tail;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tail) : "r"(tails + ((k & 1) * kWT + t) * 4) : "memory");
        const bool done = tail == T;
        const bool all_done = __all_sync(0xffffffffu, done);
        for (;;) {  // lock-step batches; lanes above the leftover bound regardless
            const uint32_t cnt = tail - head;
            const bool go = __all_sync(0xffffffffu, cnt >= kWK || done)
                                ? __any_sync(0xffffffffu, cnt > 0)
                                : __any_sync(0xffffffffu, cnt > kWLim);
            if (!go) break;
            const uint32_t nv = cnt >= kWK ? kWK : (done ? cnt : 0u);
            if (nv) batch(nv);
        }
        if (all_done) break;
        named_arrive(empty_id(k));
    }
    if (!live) return;
    gs->saved = saved;
    gs->has_saved = has ? 1u : 0u;
}

}  // namespace

cudaError_t launch_gaussian_reg(ranmar_gauss_state* d_g, uint64_t n_atoms, uint64_t per_step,
                                uint64_t steps, double* d_out, uint32_t* status, cudaStream_t stream) {
    if (n_atoms == 0 || per_step == 0 || steps == 0) return cudaSuccess;
    if (per_step >= (uint64_t(1) << 32)) return cudaErrorInvalidValue;
    static std::atomic<uint64_t> cfg[5];
    cudaError_t e = ensure_smem(gaussian_reg_kernel<0>, kRSmem, cfg[0]);
    if (!e) e = ensure_smem(gaussian_reg_kernel<1>, kRSmem, cfg[1]);
    if (!e) e = ensure_smem(gaussian_reg_kernel<2>, kRSmem, cfg[2]);
    if (!e) e = ensure_smem(gaussian_reg_kernel<3>, kRSmem, cfg[3]);
    if (!e) e = ensure_smem(gaussian_reg_kernel<6>, kRSmem, cfg[4]);
    static std::atomic<uint64_t> cfgw[6];
    if (!e) e = ensure_smem(gaussian_ws_kernel<0>, kWSmem, cfgw[0]);
    if (!e) e = ensure_smem(gaussian_ws_kernel<1>, kWSmem, cfgw[1]);
    if (!e) e = ensure_smem(gaussian_ws_kernel<2>, kWSmem, cfgw[2]);
    if (!e) e = ensure_smem(gaussian_ws_kernel<3>, kWSmem, cfgw[3]);
    if (!e) e = ensure_smem(gaussian_ws_kernel<4>, kWSmem, cfgw[4]);
    if (!e) e = ensure_smem(gaussian_ws_kernel<6>, kWSmem, cfgw[5]);
    if (e) return e;
    const uint64_t blocks = (n_atoms + kRT - 1) / kRT;
    // at most 2^32 - 1 deviates per atom per launch; longer runs continue from the
    // cached deviate in the next launch, rows further on
    const uint64_t max_steps = 0xFFFFFFFFull / per_step;
    for (uint64_t s0 = 0; s0 < steps; s0 += max_steps) {
        const uint64_t ns = steps - s0 < max_steps ? steps - s0 : max_steps;
        const uint32_t ps = static_cast<uint32_t>(per_step), G = static_cast<uint32_t>(ns * per_step);
        double* o = d_out + s0 * n_atoms * per_step;
        const dim3 grid(static_cast<unsigned>(blocks));
        count_launch();
        static const int mode = [] {  // TEMPORARY A/B switch
            const char* e = getenv("RANMAR_K4R");
            return e ? atoi(e) : 0;
        }();
        if (mode == 0) {
            const dim3 gw(static_cast<unsigned>((n_atoms + kWT - 1) / kWT));
            switch (per_step) {  // row-batched stores for the per-step counts dividing 2K
                case 1: gaussian_ws_kernel<1><<<gw, 2 * kWT, kWSmem, stream>>>(d_g, n_atoms, ps, G, o, status); break;
                case 2: gaussian_ws_kernel<2><<<gw, 2 * kWT, kWSmem, stream>>>(d_g, n_atoms, ps, G, o, status); break;
                case 3: gaussian_ws_kernel<3><<<gw, 2 * kWT, kWSmem, stream>>>(d_g, n_atoms, ps, G, o, status); break;
                case 4: gaussian_ws_kernel<4><<<gw, 2 * kWT, kWSmem, stream>>>(d_g, n_atoms, ps, G, o, status); break;
                case 6: gaussian_ws_kernel<6><<<gw, 2 * kWT, kWSmem, stream>>>(d_g, n_atoms, ps, G, o, status); break;
                default: gaussian_ws_kernel<0><<<gw, 2 * kWT, kWSmem, stream>>>(d_g, n_atoms, ps, G, o, status);
            }
        } else {
        switch (per_step) {  // row-batched stores for the per-step counts dividing 2K
            case 1: gaussian_reg_kernel<1><<<grid, kRT, kRSmem, stream>>>(d_g, n_atoms, ps, G, o, status); break;
            case 2: gaussian_reg_kernel<2><<<grid, kRT, kRSmem, stream>>>(d_g, n_atoms, ps, G, o, status); break;
            case 3: gaussian_reg_kernel<3><<<grid, kRT, kRSmem, stream>>>(d_g, n_atoms, ps, G, o, status); break;
            case 6: gaussian_reg_kernel<6><<<grid, kRT, kRSmem, stream>>>(d_g, n_atoms, ps, G, o, status); break;
            default: gaussian_reg_kernel<0><<<grid, kRT, kRSmem, stream>>>(d_g, n_atoms, ps, G, o, status);
        }
        }
        if (cudaError_t e = cudaGetLastError()) return e;
    }
    return cudaSuccess;
}

}  // namespace rb
