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
#include <cstdlib>
#include <type_traits>

#include "gauss_math.cuh"
#include "ranmar_device.cuh"

namespace rb {

namespace {

constexpr int kGT = 64;  // threads (atoms) per block: 24.8 KB of ring, 9 blocks/SM
// accepted pairs per fp64 batch. Config 5 with the correctly rounded log (2^24
// atoms x 300): K = 2..8 -> 25.24 / 23.76 / 23.54 / 22.99 / 22.96 / 23.37 / 23.32 ms
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
    auto put = [&](double x) {
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
}

// ------------------------------------------------------------------ K4p
// Thread per atom with a warp-wide pool of accepted pairs. Every lane keeps
// drawing attempt pairs on its own ring until its atom has all the pairs this
// launch needs; accepted pairs enter the warp's FIFO pool in shared memory in
// order (ballot + popc), tagged with the owning lane, its cached-deviate bit
// and the low 8 bits of the atom's pair index. Once the pool holds 32 K pairs
// the warp takes them, K per lane, whatever atoms they belong to, and runs the
// K fp64 chains: no lane waits for another lane's rejections (the batch-of-K
// attempt loop above idles ~1/3 of its lane slots), and no accepted pair is
// shifted through registers. A pair's full index is the owning lane's current
// pair count minus its distance (< 256) in the pool; its deviates go to output
// slots 2 j + has, 2 j + 1 + has of the atom, i.e. rows (2 j + has) / P. The
// pair that completes an atom also leaves its v1 fac as the atom's cache.
// Requires steps * per_step < 2^32 and per_step == P (the launcher routes
// other shapes to K4w).
template <int K>
struct K4pShape {
    static constexpr int CAP = 32 * K + 32;  // >= 32 K + 31 queued pairs
    static_assert(CAP <= 256, "pair indices are tagged mod 256");
    static constexpr uint32_t kPoolBase = kRingBase + 97 * kGT * 4;
    static constexpr int smem = 97 * kGT * 4 + (kGT / 32) * CAP * 8;
};

__device__ __forceinline__ void pool_st(uint32_t addr, uint32_t a, uint32_t b) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void pool_ld(uint32_t addr, uint32_t& a, uint32_t& b) {
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(addr));
}

template <int K, int P>
__global__ void __launch_bounds__(kGT)
    gaussian_pool_kernel(ranmar_gauss_state* __restrict__ g, uint64_t n_atoms, uint32_t G,
                         double* __restrict__ out, uint32_t* status) {
    using Sh = K4pShape<K>;
    constexpr int CAP = Sh::CAP;
    extern __shared__ uint32_t ring[];  // [97][kGT], then the warps' pools
    const int t = threadIdx.x, l = t & 31, w = t >> 5;
    if (static_cast<uint32_t>(__cvta_generic_to_shared(ring)) != kRingBase) {
        if (t == 0) atomicOr(status, kStatusInternal);
        return;
    }
    const uint64_t wbase = static_cast<uint64_t>(blockIdx.x) * kGT + w * 32;  // atom of lane 0
    const uint64_t atom = wbase + l;
    bool live = atom < n_atoms;
    ranmar_gauss_state* gs = g + (live ? atom : 0);
    int i0 = 0;
    uint32_t v = 0, has = 0;
    if (live) {
        i0 = gs->s.i;
        v = gs->s.v;
        if (!state_ok(i0, gs->s.j, v)) {
            atomicOr(status, kStatusBadState);
            live = false;
        }
    }
    constexpr uint32_t kSlot = 4 * kGT;
    const uint32_t top = 4 * t + 96 * kSlot;
    uint32_t ai = 4 * t + i0 * kSlot;
    uint32_t aj = 4 * t + (i0 >= 64 ? i0 - 64 : i0 + 33) * kSlot;
    uint32_t T = 0;  // pairs this atom needs: ceil((G - has) / 2)
    if (live) {
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
        has = gs->has_saved != 0 ? 1u : 0u;
        if (has) st_cs(out + atom * P, gs->saved);  // output 0: the cached deviate
        T = (G - has + 1) / 2;
    }
    auto attempt = [&](uint32_t& u0, uint32_t& u1) -> bool {
        uint32_t u[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t x = ring_ld(ai) - ring_ld(aj);
            ring_st(ai, x);
            ai = min(ai - kSlot, top);
            aj = min(aj - kSlot, top);
            v = add_mod_m(v, kStepA);
            u[h] = (x - v) & kMask;
        }
        const int32_t da = static_cast<int32_t>(u[0]) - (1 << 23);
        const int32_t db = static_cast<int32_t>(u[1]) - (1 << 23);
        const int64_t s = static_cast<int64_t>(da) * da + static_cast<int64_t>(db) * db;
        u0 = u[0];
        u1 = u[1];
        return s > 0 && s < (int64_t(1) << 46);
    };
    const uint32_t pbase = Sh::kPoolBase + w * CAP * 8;
    const uint32_t tag = (static_cast<uint32_t>(l) << 24) | (has << 29);
    const uint32_t lt = (1u << l) - 1u;
    const uint64_t rowstride = n_atoms * P;
    uint32_t enq = 0;                  // pairs this lane has queued
    uint32_t head = 0, tail = 0, cnt = 0;  // the warp's pool (warp-uniform)
    for (;;) {
        while (cnt < 32 * K) {
            const bool act = enq < T;
            if (!__any_sync(0xffffffffu, act)) break;
            uint32_t u0 = 0, u1 = 0;
            const bool acc = act && attempt(u0, u1);
            const uint32_t bal = __ballot_sync(0xffffffffu, acc);
            if (acc) {
                uint32_t slot = tail + __popc(bal & lt);
                slot = slot >= CAP ? slot - CAP : slot;
                pool_st(pbase + slot * 8, u0 | tag, u1 | (enq << 24));
                ++enq;
            }
            const uint32_t nb = __popc(bal);
            tail += nb;
            tail = tail >= CAP ? tail - CAP : tail;
            cnt += nb;
        }
        if (cnt == 0) break;
        const uint32_t take = min(cnt, static_cast<uint32_t>(32 * K));
        uint32_t w0[K], w1[K], pid[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t idx = 32 * k + l;
            uint32_t slot = head + idx;
            slot = slot >= CAP ? slot - CAP : slot;
            // a lane without a pair computes an accepted dummy (v1 = 1/2, v2 = 0)
            w0[k] = 0xC00000u | (static_cast<uint32_t>(l) << 24);
            w1[k] = 0x800000u;
            if (idx < take) pool_ld(pbase + slot * 8, w0[k], w1[k]);
            const uint32_t e = __shfl_sync(0xffffffffu, enq, (w0[k] >> 24) & 31);
            pid[k] = e - 1 - ((e - 1 - (w1[k] >> 24)) & 255);
        }
        double rsq[K], lg[K];
        bool all_ok = true;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            rsq[k] = polar_rsq(w0[k] & kMask, w1[k] & kMask);
            bool ok;
            lg[k] = crlog_fast(rsq[k], ok);
            all_ok = all_ok && ok;
        }
        if (__builtin_expect(!all_ok, 0)) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                bool ok;
                crlog_fast(rsq[k], ok);
                if (!ok) lg[k] = crlog_accurate(rsq[k]).y;
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const double fac = polar_fac_of(rsq[k], lg[k]);
            const double d2 = __dmul_rn(polar_v(w1[k] & kMask), fac);
            const double d1 = __dmul_rn(polar_v(w0[k] & kMask), fac);
            if (32 * k + l < take) {
                const uint32_t a = (w0[k] >> 24) & 31, ha = (w0[k] >> 29) & 1;
                const uint32_t q = 2 * pid[k] + ha;
                const uint32_t row = q / P, col = q - row * P;
                double* po = out + row * rowstride + (wbase + a) * P + col;
                st_cs(po, d2);
                if (q + 1 < G) st_cs(col + 1 < P ? po + 1 : po + (rowstride - (P - 1)), d1);
                if (pid[k] == (G - ha - 1) / 2) g[wbase + a].saved = d1;  // the atom's last pair
            }
        }
        head += take;
        head = head >= CAP ? head - CAP : head;
        cnt -= take;
    }
    if (!live) return;
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
    gs->has_saved = (G - has) & 1u;
}

// ------------------------------------------------------------------ K4w
// Warp-cooperative gaussian(): each warp owns A atoms of a CTA tile of
// T = kWW * A atoms, and the output is produced in chunks of CH = 64 PL
// deviates per atom.
//   generation  two rounds of the K1 warp mapping (gen_kernels.cu) give 64
//               consecutive uniforms of one atom = 32 attempt pairs, one per
//               lane; the exact integer test 0 < s < 2^46 runs on every lane
//               and accepted pairs enter the atom's queue in order (ballot +
//               popc). No lane waits for another lane's rejections.
//   fp64        each lane takes pair j = 32 p + l (p < PL) of each of its A
//               atoms: A * PL independent log / divide / sqrt chains per lane,
//               every lane busy.
//   output      deviates land in a shared-memory stage [atom][slot] (slot =
//               output index - chunk start), then the CTA writes the chunk's
//               output rows: per step row the tile's atoms are contiguous
//               (T * per_step doubles), so the stores are coalesced although
//               every atom's deviates are strided by n_atoms * per_step.
// The stage is double-buffered, so one barrier per chunk separates the fp64
// writes of chunk c from its write-out and the write-out of chunk c - 1 from
// the fp64 writes of chunk c + 1.
// Pairs always start at even uniform offsets from the launch's start state (a
// rejected attempt consumes both uniforms; a cached deviate consumes none),
// so pair j of an atom = (u_{2a}, u_{2a+1}) for its j-th accepted attempt a.
// An atom with a cached deviate (has = 1) emits it as output 0, so pair j
// fills output slots 2 j + has, 2 j + 1 + has; the pair that straddles a chunk
// boundary leaves its second deviate as the next chunk's slot 0, which is the
// atom's running `saved` value (the oracle's cache, kept in a register).
// The last pair any atom needs comes from the last generation it ran (a
// generation runs only while the queue holds fewer pairs than the chunk
// needs), so the atom stops at uniform n in (64 g - 64, 64 g] after g
// generations and its ring window [n - 97, n) is among the last five rounds.
constexpr int kWW = 4;  // warps per CTA

template <int A, int PL, int P>
struct K4wShape {
    static constexpr int T = kWW * A;        // atoms per CTA tile
    static constexpr int CH = 64 * PL;       // output slots per atom per chunk
    static constexpr int QCAP = (PL == 1) ? 64 : 128;  // >= 32 PL + 31 queued pairs
    // stage row stride (doubles): >= CH + 1 (the straddling pair's dropped
    // second deviate) and == per_step mod 16, so that the write-out's LDS.64
    // of consecutive (atom, column) elements hit distinct banks
    static constexpr int S = (P > 0) ? CH + 1 + ((P - 1) % 16) : CH + 1;
    static constexpr size_t smem = sizeof(double) * 2 * T * S + sizeof(uint64_t) * T * QCAP;
};

constexpr uint64_t kK4wDummy = (0xC00000ull) | (0x800000ull << 24);

// Per-atom generator registers (the K1 mapping with a fifth round kept).
struct K4wGen {
    uint32_t R1, R2, R3, R4, R5, prev, V;
};

template <int A, int PL, int P>
__global__ void __launch_bounds__(32 * kWW)
    gaussian_warp_kernel(ranmar_gauss_state* __restrict__ g, uint64_t n_atoms, uint64_t per_step,
                         uint64_t steps, double* __restrict__ out, uint32_t* status) {
    using Sh = K4wShape<A, PL, P>;
    constexpr int T = Sh::T, CH = Sh::CH, QCAP = Sh::QCAP, S = Sh::S;
    extern __shared__ __align__(16) unsigned char k4w_smem[];
    double* stage = reinterpret_cast<double*>(k4w_smem);                          // [2][T][S]
    uint64_t* queue = reinterpret_cast<uint64_t*>(k4w_smem + sizeof(double) * 2 * T * S);  // [T][QCAP]

    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t a0 = static_cast<uint64_t>(blockIdx.x) * T;
    const uint64_t ps = P > 0 ? static_cast<uint64_t>(P) : per_step;
    const uint64_t G = steps * ps;
    const int src = (l + 31) & 31;
    const uint32_t A32 = static_cast<uint32_t>((32ull * kStepA) % kMod);

    K4wGen gen[A];
    uint32_t qhead[A], qtail[A], llast[A];
    uint64_t gens[A], total[A];
    double saved[A];
    int has0[A];
    bool act[A];
    uint32_t amask = 0;  // this warp's active atoms (bit k)
#pragma unroll
    for (int k = 0; k < A; ++k) {
        const uint64_t atom = a0 + w * A + k;
        act[k] = false;
        has0[k] = 0;
        saved[k] = 0.0;
        qhead[k] = qtail[k] = llast[k] = 0;
        gens[k] = total[k] = 0;
        gen[k] = K4wGen{0, 0, 0, 0, 0, 0, 0};
        if (atom < n_atoms) {
            const ranmar_gauss_state* gs = g + atom;
            const int i0 = gs->s.i, j0 = gs->s.j;
            const uint32_t v0 = gs->s.v;
            if (!state_ok(i0, j0, v0)) {
                if (l == 0) atomicOr(status, kStatusBadState);
            } else {
                act[k] = true;
                const uint32_t* lane = gs->s.lane;
                K4wGen& s = gen[k];
                s.R1 = lane[(i0 + 32 - l) % 97];
                s.R2 = lane[(i0 + 64 - l) % 97];
                s.R3 = lane[(i0 + 96 - l) % 97];
                s.R4 = (l == 31) ? lane[i0] : 0u;
                s.R5 = 0;
                s.V = arith_advance(v0, static_cast<uint64_t>(l) + 1);
                has0[k] = gs->has_saved != 0 ? 1 : 0;
                saved[k] = gs->saved;
                // pairs this launch needs: ceil((G - has) / 2)
                total[k] = (G - has0[k] + 1) / 2;
            }
        }
        gen[k].prev = __shfl_sync(0xffffffffu, gen[k].R4 - gen[k].R2, src);
        amask |= act[k] ? (1u << k) : 0u;
    }
    // the tile's active atoms (bit w * A + k), for the write-out
    __shared__ uint32_t s_tmask[kWW];
    if (l == 0) s_tmask[w] = amask;
    __syncthreads();
    uint32_t tmask = 0;
#pragma unroll
    for (int ww = 0; ww < kWW; ++ww) tmask |= s_tmask[ww] << (ww * A);

    // write-out position of this thread when a tile row (T * per_step doubles)
    // fits the CTA: rpi rows per pass, element wi = (atom a, column col)
    const uint64_t rowlen64 = static_cast<uint64_t>(T) * ps;
    const bool fixed = rowlen64 <= 32 * kWW;
    const uint32_t rowlen = fixed ? static_cast<uint32_t>(rowlen64) : 1u;
    const uint32_t rpi = (32 * kWW) / rowlen;
    const uint32_t rr0 = threadIdx.x / rowlen, wi = threadIdx.x - rr0 * rowlen;
    const uint32_t a = fixed ? wi / static_cast<uint32_t>(ps) : 0u;
    const uint32_t col = wi - a * static_cast<uint32_t>(ps);
    const bool wact = fixed && rr0 < rpi && ((tmask >> a) & 1u);
    const uint64_t rowstride = n_atoms * ps;

    const uint64_t nch = (G + CH - 1) / CH;
    for (uint64_t c = 0; c < nch; ++c) {
        double* stg = stage + (c & 1) * (T * S);
        const uint64_t q0 = c * CH;
        const uint64_t q1 = min(q0 + CH, G);
        // generation: fill every active atom's queue to this chunk's need
        uint32_t need[A];
#pragma unroll
        for (int k = 0; k < A; ++k) {
            need[k] = 0;
            if (!act[k]) continue;
            const uint64_t pc = min((q1 - has0[k] + 1) / 2, total[k]);  // pairs through this chunk
            const uint64_t p0 = min((q0 - has0[k] + 1) / 2, total[k]);
            need[k] = static_cast<uint32_t>(pc - p0);
            uint64_t* qk = queue + (w * A + k) * QCAP;
            K4wGen& s = gen[k];
            while (qtail[k] - qhead[k] < need[k]) {
                uint32_t uab[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t X = __shfl_sync(0xffffffffu, s.R3 - s.R1, src);
                    const uint32_t y = (l == 0) ? s.prev : X;
                    s.prev = X;
                    s.R5 = s.R4;
                    s.R4 = s.R3;
                    s.R3 = s.R2;
                    s.R2 = s.R1;
                    s.R1 = y;
                    uab[h] = (y - s.V) & kMask;
                    s.V = add_mod_m(s.V, A32);
                }
                const int s1 = (2 * l) & 31;  // attempt l = uniforms 2l, 2l + 1 of the 64
                const uint32_t x1 = __shfl_sync(0xffffffffu, uab[0], s1);
                const uint32_t y1 = __shfl_sync(0xffffffffu, uab[1], s1);
                const uint32_t x2 = __shfl_sync(0xffffffffu, uab[0], s1 + 1);
                const uint32_t y2 = __shfl_sync(0xffffffffu, uab[1], s1 + 1);
                const uint32_t u1 = l < 16 ? x1 : y1, u2 = l < 16 ? x2 : y2;
                const int32_t da = static_cast<int32_t>(u1) - (1 << 23);
                const int32_t db = static_cast<int32_t>(u2) - (1 << 23);
                const int64_t sq = static_cast<int64_t>(da) * da + static_cast<int64_t>(db) * db;
                const bool acc = sq > 0 && sq < (int64_t(1) << 46);
                const uint32_t bal = __ballot_sync(0xffffffffu, acc);
                if (acc) {
                    const uint32_t slot = (qtail[k] + __popc(bal & ((1u << l) - 1u))) & (QCAP - 1);
                    qk[slot] = static_cast<uint64_t>(u1) | (static_cast<uint64_t>(u2) << 24) |
                               (static_cast<uint64_t>(l) << 48);
                }
                qtail[k] += __popc(bal);
                ++gens[k];
            }
        }
        __syncwarp();
        // fp64: pair j = 32 p + l of each atom
        uint64_t e[A][PL];
#pragma unroll
        for (int k = 0; k < A; ++k) {
            const uint64_t* qk = queue + (w * A + k) * QCAP;
#pragma unroll
            for (int p = 0; p < PL; ++p) {
                const uint32_t j = 32 * p + l;
                // a lane without a pair computes an accepted dummy (v1 = 1/2, v2 = 0)
                e[k][p] = j < need[k] ? qk[(qhead[k] + j) & (QCAP - 1)] : kK4wDummy;
            }
        }
        // the fast log of every chain first, the rare accurate phase after all
        // of them (one branch), then the divides and square roots
        double rsq[A][PL], lg[A][PL];
        bool all_ok = true;
#pragma unroll
        for (int k = 0; k < A; ++k) {
#pragma unroll
            for (int p = 0; p < PL; ++p) {
                const uint32_t u1 = static_cast<uint32_t>(e[k][p]) & kMask;
                const uint32_t u2 = static_cast<uint32_t>(e[k][p] >> 24) & kMask;
                rsq[k][p] = polar_rsq(u1, u2);
                bool ok;
                lg[k][p] = crlog_fast(rsq[k][p], ok);
                all_ok = all_ok && ok;
            }
        }
        if (__builtin_expect(!all_ok, 0)) {
#pragma unroll
            for (int k = 0; k < A; ++k) {
#pragma unroll
                for (int p = 0; p < PL; ++p) {
                    bool ok;
                    crlog_fast(rsq[k][p], ok);
                    if (!ok) lg[k][p] = crlog_accurate(rsq[k][p]).y;
                }
            }
        }
        double d1[A][PL], d2[A][PL];
#pragma unroll
        for (int k = 0; k < A; ++k) {
#pragma unroll
            for (int p = 0; p < PL; ++p) {
                const uint32_t u1 = static_cast<uint32_t>(e[k][p]) & kMask;
                const uint32_t u2 = static_cast<uint32_t>(e[k][p] >> 24) & kMask;
                const double fac = polar_fac_of(rsq[k][p], lg[k][p]);
                d2[k][p] = __dmul_rn(polar_v(u2), fac);
                d1[k][p] = __dmul_rn(polar_v(u1), fac);
            }
        }
#pragma unroll
        for (int k = 0; k < A; ++k) {
            double* sk = stg + (w * A + k) * S;
            if (has0[k] && l == 0 && act[k]) sk[0] = saved[k];  // the cached / straddling deviate
            if (need[k] == 0) continue;
#pragma unroll
            for (int p = 0; p < PL; ++p) {
                const uint32_t j = 32 * p + l;
                if (j < need[k]) {
                    sk[2 * j + has0[k]] = d2[k][p];
                    sk[2 * j + 1 + has0[k]] = d1[k][p];
                }
            }
            const uint32_t jl = need[k] - 1;
            double dl = d1[k][0];
#pragma unroll
            for (int p = 1; p < PL; ++p) dl = (jl >> 5) == static_cast<uint32_t>(p) ? d1[k][p] : dl;
            saved[k] = __shfl_sync(0xffffffffu, dl, jl & 31);
            llast[k] = static_cast<uint32_t>(queue[(w * A + k) * QCAP + ((qhead[k] + jl) & (QCAP - 1))] >> 48);
            qhead[k] += need[k];
        }
        __syncthreads();
        // write-out of output slots [q0, q1) of the tile's active atoms
        const uint64_t r_lo = q0 / ps;
        if (fixed) {
            // thread (rr0, wi) writes element wi of rows r_lo + rr0, + rpi, ...
            const uint32_t len = static_cast<uint32_t>(q1 - q0);
            const uint32_t nrows = static_cast<uint32_t>((q1 - 1) / ps - r_lo) + 1;
            int slot = static_cast<int>(rr0 * ps + col) + static_cast<int>(r_lo * ps - q0);
            double* po = out + (r_lo + rr0) * rowstride + a0 * ps + wi;
            const double* sa = stg + a * S;
            if (wact) {
                for (uint32_t rr = rr0; rr < nrows; rr += rpi) {
                    if (static_cast<uint32_t>(slot) < len) st_cs(po, sa[slot]);
                    slot += static_cast<int>(rpi * ps);
                    po += rpi * rowstride;
                }
            }
        } else {
            // long rows: atom-major, consecutive threads on consecutive slots
            const uint32_t len = static_cast<uint32_t>(q1 - q0);
            for (uint32_t x = threadIdx.x; x < T * len; x += 32 * kWW) {
                const uint32_t at = x / len, sl = x - at * len;
                if (!((tmask >> at) & 1u)) continue;
                const uint64_t q = q0 + sl, r = q / ps;
                st_cs(out + (r * n_atoms + a0 + at) * ps + (q - r * ps), stg[at * S + sl]);
            }
        }
    }
    // final states: the ring window, cursors and v after n uniforms; the cache
#pragma unroll
    for (int k = 0; k < A; ++k) {
        if (!act[k]) continue;
        ranmar_gauss_state* gs = g + a0 + w * A + k;
        const int i0 = gs->s.i, j0 = gs->s.j;
        const uint32_t v0 = gs->s.v;
        __syncwarp();
        if (gens[k] > 0) {
            const uint64_t N = 2 * (32 * (gens[k] - 1) + llast[k] + 1);
            const uint64_t rounds = 2 * gens[k];
            uint32_t* lane_w = gs->s.lane;
            const int64_t lo = static_cast<int64_t>(N) - 97, hi = static_cast<int64_t>(N);
            const uint32_t regs[5] = {gen[k].R1, gen[k].R2, gen[k].R3, gen[k].R4, gen[k].R5};
#pragma unroll
            for (int r = 0; r < 5; ++r) {
                const int64_t n = 32 * (static_cast<int64_t>(rounds) - 1 - r) + l;
                if (n >= lo && n < hi) {
                    int64_t m = (static_cast<int64_t>(i0) - n) % 97;
                    lane_w[m < 0 ? m + 97 : m] = regs[r] & kMask;
                }
            }
            __syncwarp();
            if (l == 0) {
                const int nm = static_cast<int>(N % 97);
                gs->s.i = (i0 - nm + 97) % 97;
                gs->s.j = (j0 - nm + 97) % 97;
                gs->s.v = arith_advance(v0, N);
            }
        }
        if (l == 0) {
            gs->saved = saved[k];
            gs->has_saved = G > 0 ? static_cast<uint32_t>((G - has0[k]) & 1) : static_cast<uint32_t>(has0[k]);
        }
    }
}

}  // namespace

template <int A, int PL, int P>
static cudaError_t launch_k4w_p(ranmar_gauss_state* d_g, uint64_t n_atoms, uint64_t per_step,
                                uint64_t steps, double* d_out, uint32_t* status, cudaStream_t stream) {
    using Sh = K4wShape<A, PL, P>;
    static std::atomic<uint64_t> done{0};
    if (cudaError_t e = ensure_smem(gaussian_warp_kernel<A, PL, P>, static_cast<int>(Sh::smem), done))
        return e;
    const uint64_t blocks = (n_atoms + Sh::T - 1) / Sh::T;
    count_launch();
    gaussian_warp_kernel<A, PL, P><<<static_cast<unsigned>(blocks), 32 * kWW, Sh::smem, stream>>>(
        d_g, n_atoms, per_step, steps, d_out, status);
    return cudaGetLastError();
}

template <int K, int P>
static cudaError_t launch_k4p_p(ranmar_gauss_state* d_g, uint64_t n_atoms, uint32_t G, double* d_out,
                                uint32_t* status, cudaStream_t stream) {
    using Sh = K4pShape<K>;
    static std::atomic<uint64_t> done{0};
    if (cudaError_t e = ensure_smem(gaussian_pool_kernel<K, P>, Sh::smem, done)) return e;
    const uint64_t blocks = (n_atoms + kGT - 1) / kGT;
    count_launch();
    gaussian_pool_kernel<K, P><<<static_cast<unsigned>(blocks), kGT, Sh::smem, stream>>>(d_g, n_atoms, G, d_out,
                                                                                          status);
    return cudaGetLastError();
}

template <int K>
static cudaError_t launch_k4p(ranmar_gauss_state* d_g, uint64_t n_atoms, uint64_t per_step, uint64_t steps,
                              double* d_out, uint32_t* status, cudaStream_t stream, bool& done) {
    done = true;
    const uint64_t G = steps * per_step;
    if (G < (uint64_t(1) << 32)) {
        const uint32_t g32 = static_cast<uint32_t>(G);
        switch (per_step) {
            case 1: return launch_k4p_p<K, 1>(d_g, n_atoms, g32, d_out, status, stream);
            case 2: return launch_k4p_p<K, 2>(d_g, n_atoms, g32, d_out, status, stream);
            case 3: return launch_k4p_p<K, 3>(d_g, n_atoms, g32, d_out, status, stream);
            case 4: return launch_k4p_p<K, 4>(d_g, n_atoms, g32, d_out, status, stream);
            case 6: return launch_k4p_p<K, 6>(d_g, n_atoms, g32, d_out, status, stream);
            default: break;
        }
    }
    done = false;
    return cudaSuccess;
}

template <int A, int PL>
static cudaError_t launch_k4w(ranmar_gauss_state* d_g, uint64_t n_atoms, uint64_t per_step,
                              uint64_t steps, double* d_out, uint32_t* status, cudaStream_t stream) {
    switch (per_step) {  // compile-time row shapes for the common per-step counts
        case 1: return launch_k4w_p<A, PL, 1>(d_g, n_atoms, per_step, steps, d_out, status, stream);
        case 2: return launch_k4w_p<A, PL, 2>(d_g, n_atoms, per_step, steps, d_out, status, stream);
        case 3: return launch_k4w_p<A, PL, 3>(d_g, n_atoms, per_step, steps, d_out, status, stream);
        case 4: return launch_k4w_p<A, PL, 4>(d_g, n_atoms, per_step, steps, d_out, status, stream);
        case 6: return launch_k4w_p<A, PL, 6>(d_g, n_atoms, per_step, steps, d_out, status, stream);
        default: return launch_k4w_p<A, PL, 0>(d_g, n_atoms, per_step, steps, d_out, status, stream);
    }
}

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
    static const int mode = [] {  // TEMPORARY A/B switch
        const char* e = getenv("RANMAR_K4");
        return e ? atoi(e) : 1;
    }();
    switch (mode) {
        case 0: return launch_gaussian_k<kBatch>(d_g, n_atoms, per_step, steps, d_out, status, stream);
        case 20: return launch_gaussian_k<4>(d_g, n_atoms, per_step, steps, d_out, status, stream);
        case 21: return launch_gaussian_k<5>(d_g, n_atoms, per_step, steps, d_out, status, stream);
        case 22: return launch_gaussian_k<8>(d_g, n_atoms, per_step, steps, d_out, status, stream);
        case 23: return launch_gaussian_k<3>(d_g, n_atoms, per_step, steps, d_out, status, stream);
        case 1: return launch_k4w<4, 1>(d_g, n_atoms, per_step, steps, d_out, status, stream);
        case 2: return launch_k4w<2, 2>(d_g, n_atoms, per_step, steps, d_out, status, stream);
        case 3: return launch_k4w<2, 1>(d_g, n_atoms, per_step, steps, d_out, status, stream);
        case 4: return launch_k4w<8, 1>(d_g, n_atoms, per_step, steps, d_out, status, stream);
        case 5: return launch_k4w<4, 2>(d_g, n_atoms, per_step, steps, d_out, status, stream);
        default: {
            bool done = false;
            cudaError_t e = cudaSuccess;
            if (mode == 10) e = launch_k4p<4>(d_g, n_atoms, per_step, steps, d_out, status, stream, done);
            if (mode == 11) e = launch_k4p<3>(d_g, n_atoms, per_step, steps, d_out, status, stream, done);
            if (mode == 12) e = launch_k4p<6>(d_g, n_atoms, per_step, steps, d_out, status, stream, done);
            if (mode == 13) e = launch_k4p<2>(d_g, n_atoms, per_step, steps, d_out, status, stream, done);
            if (done) return e;
            return launch_k4w<2, 1>(d_g, n_atoms, per_step, steps, d_out, status, stream);
        }
    }
}

}  // namespace rb
