// K4: gaussian() on the GPU, thread per atom (sm_100a).
//
// gaussian() has no reference counterpart; the repo
// defines it in oracle/ranmar_oracle.c (or_gaussian): Marsaglia polar method
// on uniform() = next_f64 (core.hpp:70-72), v = 2u - 1, reject rsq >= 1 or
// rsq == 0, return v2 * fac and cache v1 * fac (Numerical Recipes pairing),
// log() being the fixed IEEE sequence or_glog so results are bit-identical.
//
// Every gaussian() call consumes uniforms in pairs, so an atom's deviates are
// the cached one (if has_saved) followed by (v2 fac, v1 fac) for each
// ACCEPTED attempt pair. Each thread therefore runs one loop over attempts
// (not one rejection loop per call, which would make a warp wait for its
// unluckiest lane at every call): draw two uniforms, test rsq in exact integer
// arithmetic (rsq = s / 2^46 with s = (u1 - 2^23)^2 + (u2 - 2^23)^2), and on
// acceptance evaluate fac in fp64 and emit two deviates. A lane stops once
// its atom has all steps * per_step deviates; the last pair's second deviate
// becomes the cached one when the count is odd.
//
// The 97-word ring of each atom lives in shared memory column-major (slot s
// of thread t at s * kGT + t): every access of a warp hits 32 distinct banks
// whatever the (diverged) cursors. States are moved between HBM and the ring
// with 16-B vector accesses (the 416-B records are 16-B aligned).
#include <cstdint>

#include "ranmar_device.cuh"

namespace rb {

namespace {

// gaussian()'s log: the repo convention's fixed IEEE sequence (derivation in
// oracle/ranmar_oracle.c or_glog), with explicit round-to-nearest intrinsics
// so nvcc cannot contract or reorder anything. The binary64 coefficients sit
// in constant memory so DFMA reads them as operands (64-bit immediates would
// cost a uniform move each per use inside the attempt loop).
__constant__ double kGlogC[13] = {
    0x1.8618618618618p-5, 0x1.af286bca1af28p-5, 0x1.e1e1e1e1e1e1ep-5, 0x1.1111111111111p-4,
    0x1.3b13b13b13b14p-4, 0x1.745d1745d1746p-4, 0x1.c71c71c71c71cp-4, 0x1.2492492492492p-3,
    0x1.999999999999ap-3, 0x1.5555555555555p-2,          // 1/21 .. 1/3
    0x1.62e42fefa3800p-1, 0x1.ef35793c76730p-45,         // ln2 head, tail
    0x1.6a09e667f3bcdp+0};                               // sqrt(2)

__device__ __forceinline__ double glog(double x) {
    const long long b = __double_as_longlong(x);
    int k = static_cast<int>((b >> 52) & 0x7FF) - 1023;
    double m = __longlong_as_double((b & 0x000FFFFFFFFFFFFFll) | 0x3FF0000000000000ll);
    if (m > kGlogC[12]) {
        m = __dmul_rn(m, 0.5);
        k += 1;
    }
    const double f = __dsub_rn(m, 1.0);
    const double s = __ddiv_rn(f, __dadd_rn(2.0, f));
    const double z = __dmul_rn(s, s);
    double p = kGlogC[0];
#pragma unroll
    for (int c = 1; c < 10; ++c) p = __fma_rn(p, z, kGlogC[c]);
    const double t = __dmul_rn(s, z);
    const double l1p = __dmul_rn(2.0, __fma_rn(t, p, s));
    const double kd = static_cast<double>(k);
    return __fma_rn(kd, kGlogC[10], __fma_rn(kd, kGlogC[11], l1p));
}

// v = 2 (u / 2^24) - 1, exact.
__device__ __forceinline__ double polar_v(uint32_t u) {
    return __dsub_rn(__dmul_rn(static_cast<double>(u), 0x1p-23), 1.0);
}

constexpr int kGT = 128;  // threads (atoms) per block

__global__ void __launch_bounds__(kGT)
    gaussian_kernel(ranmar_gauss_state* __restrict__ g, uint64_t n_atoms, uint64_t per_step,
                    uint64_t steps, double* __restrict__ out, uint32_t* status) {
    extern __shared__ uint32_t ring[];  // [97][kGT]
    const int t = threadIdx.x;
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
    uint32_t* col = ring + t;
    int i = i0;  // cursor; j = i - 64 mod 97
    uint32_t v = v0;
    double saved = gs->saved;
    bool has = gs->has_saved != 0;

    const uint64_t G = steps * per_step;
    uint64_t q = 0;  // next deviate index of this atom
    // out offset of deviate q: (step * n_atoms + atom) * per_step + c, advanced incrementally
    uint64_t off = atom * per_step, c = 0;
    const uint64_t jump = (n_atoms - 1) * per_step;
    auto put = [&](double x) {
        st_cs(out + off, x);
        ++off;
        if (++c == per_step) {
            c = 0;
            off += jump;
        }
    };
    if (has && G > 0) {
        put(saved);
        has = false;
        q = 1;
    }
    while (q < G) {
        // attempts until one is accepted; the fp64 part then runs with the
        // whole warp converged (every lane needs a new pair at the same call)
        uint32_t u0, u1;
        for (;;) {
            uint32_t u[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {  // two uniforms (core.hpp:54-66 on the ring)
                const int j = i >= 64 ? i - 64 : i + 33;
                const uint32_t x = col[i * kGT] - col[j * kGT];
                col[i * kGT] = x;
                i = i == 0 ? 96 : i - 1;
                v = add_mod_m(v, kStepA);
                u[h] = (x - v) & kMask;
            }
            const int32_t da = static_cast<int32_t>(u[0]) - (1 << 23);
            const int32_t db = static_cast<int32_t>(u[1]) - (1 << 23);
            const int64_t s = static_cast<int64_t>(da) * da + static_cast<int64_t>(db) * db;
            u0 = u[0];
            u1 = u[1];
            if (s > 0 && s < (int64_t(1) << 46)) break;  // 0 < rsq < 1, exactly
        }
        const double v1 = polar_v(u0), v2 = polar_v(u1);
        const double rsq = __dadd_rn(__dmul_rn(v1, v1), __dmul_rn(v2, v2));
        const double fac = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, glog(rsq)), rsq));
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
    *reinterpret_cast<uint4*>(gs->s.lane + 96) =
        make_uint4(ring[96 * kGT + t] & kMask, static_cast<uint32_t>(i),
                   static_cast<uint32_t>(i >= 64 ? i - 64 : i + 33), v);
    gs->saved = saved;
    gs->has_saved = has ? 1u : 0u;
}

}  // namespace

cudaError_t launch_gaussian(ranmar_gauss_state* d_g, uint64_t n_atoms, uint64_t per_step,
                            uint64_t steps, double* d_out, uint32_t* status,
                            cudaStream_t stream) {
    if (n_atoms == 0 || per_step == 0 || steps == 0) return cudaSuccess;
    const int smem = 97 * kGT * 4;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(gaussian_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const uint64_t blocks = (n_atoms + kGT - 1) / kGT;
    count_launch();
    gaussian_kernel<<<static_cast<unsigned>(blocks), kGT, smem, stream>>>(d_g, n_atoms, per_step,
                                                                          steps, d_out, status);
    return cudaGetLastError();
}

}  // namespace rb
