// Jump-ahead kernels (sm_100a), K3.
//
// The Fibonacci part of a jump by J is u * P_J(A) with P_J = t^J mod phi(t),
// phi = t^97 + t^64 - 1 over Z/2^24 (jump.hpp:60-76, polyring.hpp:113-124;
// PAPER.md:298-324). All coefficient arithmetic is 32-bit mad.lo with
// wraparound and one final mask: only the low 24 bits of each product matter,
// which replaces the reference's 64-bit accumulation (polyring.hpp:88-96)
// without changing a single residue. Tensor cores are not used: this is
// modular integer arithmetic, not a float contraction.
//
//  pow_kernel        K3a  t^E mod phi by left-to-right square-and-multiply in
//                         shared memory (one CTA per exponent), symmetric
//                         squaring (4,753 MACs instead of 9,409) and the
//                         trinomial fold split into three conflict-free phases
//                         (sources [160,192], [127,159], [97,126]); optional
//                         chain of further squarings P_{2^b E}.
//  mulmod_kernel          batched products a_r * Q mod phi (warp per product);
//                         builds the offset table T_r = P_{rJ} by doubling.
//  apply_kernel      K3b  u * P(A) for a batch of states as a Hankel product
//                         out[m] = sum_j p_j w[j + m] over the 208-term
//                         recurrence extension w of u (no sequential Horner
//                         chain), + K3c the closed-form arithmetic jump.
//  bulk_kernel       K3b  make_streams' stream starts s_{(first + 128h + r)J}
//                         = apply(anchor_h, T_r): per anchor a 128 x 104 x 104
//                         integer "GEMM" tile with a 4 x 8 register tile per
//                         thread; T^T stays in shared memory for all anchors
//                         a CTA visits, results are staged and written as
//                         contiguous 400-B state records.
#include <cstdint>

#include "ranmar_device.cuh"

namespace rb {

constexpr int kPolyN = 97;
constexpr int kWExt = 208;   // recurrence-extension length used by the Hankel products
constexpr int kJPad = 104;   // coefficients padded to 13 x 8
constexpr int kRows = 128;   // offsets per anchor (T table rows)

struct PowJob {
    uint64_t e[4];
    int extra;      // further squarings after t^E (outputs P_{2E}, P_{4E}, ...)
    uint32_t* out;  // (1 + extra) x 97
};
struct PowJobs {
    PowJob job[2];
};

namespace {

constexpr int kPowThreads = 256;

// c[0..192] -> a[0..96] = c mod phi, three phases (see header). c is
// overwritten. Works for any group of threads [t0, t0 + nt) that shares c.
template <class Sync>
__device__ __forceinline__ void fold_to(uint32_t* c, uint32_t* a, int t, int nt, Sync sync) {
    for (int k = 160 + t; k <= 192; k += nt) {
        const uint32_t hi = c[k];
        c[k - 97] += hi;
        c[k - 33] -= hi;
    }
    sync();
    for (int k = 127 + t; k <= 159; k += nt) {
        const uint32_t hi = c[k];
        c[k - 97] += hi;
        c[k - 33] -= hi;
    }
    sync();
    for (int k = 97 + t; k <= 126; k += nt) {
        const uint32_t hi = c[k];
        c[k - 97] += hi;
        c[k - 33] -= hi;
    }
    sync();
    for (int k = t; k < kPolyN; k += nt) a[k] = c[k] & kMask;
    sync();
}

__device__ __forceinline__ void block_square(uint32_t* a, uint32_t* c) {
    const int t = threadIdx.x;
    for (int k = t; k < 193; k += blockDim.x) {
        const int lo = k > 96 ? k - 96 : 0;
        uint32_t acc = 0;
        for (int i = lo; 2 * i < k; ++i) acc += a[i] * a[k - i];
        acc <<= 1;
        if ((k & 1) == 0) acc += a[k >> 1] * a[k >> 1];
        c[k] = acc;
    }
    __syncthreads();
    fold_to(c, a, t, blockDim.x, [] { __syncthreads(); });
}

// a <- a * t (polyring.hpp:101-109)
__device__ __forceinline__ void block_mul_t(uint32_t* a) {
    const int t = threadIdx.x;
    const uint32_t top = a[96];
    uint32_t q = 0;
    if (t < kPolyN) q = t == 0 ? top : a[t - 1];
    __syncthreads();
    if (t < kPolyN) a[t] = t == 64 ? ((q - top) & kMask) : q;
    __syncthreads();
}

__device__ __forceinline__ bool ebit(const uint64_t* e, int b) { return (e[b >> 6] >> (b & 63)) & 1u; }

__global__ void __launch_bounds__(kPowThreads) pow_kernel(PowJobs jobs) {
    __shared__ uint32_t a[kPolyN];
    __shared__ uint32_t c[193];
    const PowJob& job = jobs.job[blockIdx.x];
    int msb = -1;
    for (int w = 3; w >= 0 && msb < 0; --w)
        if (job.e[w]) msb = 64 * w + 63 - __clzll(static_cast<long long>(job.e[w]));
    // Leading bits whose value stays below 97 give a monomial directly.
    int b = msb;
    uint32_t pref = 0;
    while (b >= 0 && 2 * pref + ebit(job.e, b) < 97u) {
        pref = 2 * pref + ebit(job.e, b);
        --b;
    }
    for (int k = threadIdx.x; k < kPolyN; k += blockDim.x) a[k] = (k == static_cast<int>(pref));
    __syncthreads();
    for (; b >= 0; --b) {
        block_square(a, c);
        if (ebit(job.e, b)) block_mul_t(a);
    }
    for (int k = threadIdx.x; k < kPolyN; k += blockDim.x) job.out[k] = a[k];
    for (int x = 1; x <= job.extra; ++x) {
        block_square(a, c);
        for (int k = threadIdx.x; k < kPolyN; k += blockDim.x) job.out[x * kPolyN + k] = a[k];
    }
}

// ---- T table: T_0 = 1, T_{r + half} = T_r * Q for r < half (warp per product)
constexpr int kMulWarps = 4;

__global__ void __launch_bounds__(32 * kMulWarps)
    mulmod_kernel(uint32_t* __restrict__ T, int half, int count, const uint32_t* __restrict__ Q) {
    __shared__ uint32_t q[kPolyN];
    __shared__ uint32_t as[kMulWarps][kPolyN];
    __shared__ uint32_t cs[kMulWarps][193];
    for (int k = threadIdx.x; k < kPolyN; k += blockDim.x) q[k] = Q[k];
    __syncthreads();
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int r = blockIdx.x * kMulWarps + w;
    if (r >= count) return;
    uint32_t* a = as[w];
    uint32_t* c = cs[w];
    for (int k = l; k < kPolyN; k += 32) a[k] = T[r * kPolyN + k];
    __syncwarp();
    for (int k = l; k < 193; k += 32) {
        const int lo = k > 96 ? k - 96 : 0, hi = k < 96 ? k : 96;
        uint32_t acc = 0;
        for (int i = lo; i <= hi; ++i) acc += a[i] * q[k - i];
        c[k] = acc;
    }
    __syncwarp();
    fold_to(c, a, l, 32, [] { __syncwarp(); });
    for (int k = l; k < kPolyN; k += 32) T[(r + half) * kPolyN + k] = a[k];
}

__global__ void t_init_kernel(uint32_t* __restrict__ T) {
    for (int k = threadIdx.x; k < kPolyN; k += blockDim.x) T[k] = (k == 0);
}

// Tt[j][r] = T_r[j] (j < 97), 0 for j in [97, 104).
__global__ void t_transpose_kernel(const uint32_t* __restrict__ T, uint32_t* __restrict__ Tt) {
    const int r = threadIdx.x;  // 128 threads
    for (int j = blockIdx.x; j < kJPad; j += gridDim.x)
        Tt[j * kRows + r] = j < kPolyN ? T[r * kPolyN + j] : 0u;
}

// ---- recurrence extension w[0..207] of a state's canonical vector
// (canonicalize, jump.hpp:32-37; recurrence_extend, test_util.hpp:38-46).
// Phases of <= 33 new terms: w[n] depends on w[n-97], w[n-33] only.
template <class Sync>
__device__ __forceinline__ void extend(uint32_t* W, int t, int nt, Sync sync) {
    for (int p = 0; p < 4; ++p) {
        const int lo = 97 + 33 * p, hi = min(lo + 33, kWExt);
        for (int n = lo + t; n < hi; n += nt) W[n] = W[n - 97] - W[n - 33];
        sync();
    }
}

// ---- K3b/K3c for a batch: out[k] = jump(in[k]) with one shared P and dec.
constexpr int kApplyItems = 8;
constexpr int kApplyThreads = kApplyItems * 13;  // 104: (item, column group of 8)
constexpr int kWStride = kWExt + 1;               // odd stride spreads banks

__global__ void __launch_bounds__(kApplyThreads)
    apply_kernel(const ranmar_state* in, ranmar_state* out, uint64_t n,
                 const uint32_t* __restrict__ P, uint32_t dec) {
    __shared__ uint32_t W[kApplyItems * kWStride];
    __shared__ uint32_t p[kJPad];
    __shared__ uint32_t vin[kApplyItems];
    __shared__ int iin[kApplyItems];
    const int t = threadIdx.x;
    const uint64_t k0 = static_cast<uint64_t>(blockIdx.x) * kApplyItems;
    const int items = static_cast<int>(n - k0 < (uint64_t)kApplyItems ? n - k0 : (uint64_t)kApplyItems);
    for (int k = t; k < kJPad; k += kApplyThreads) p[k] = k < kPolyN ? P[k] : 0u;
    if (t < items) {
        iin[t] = in[k0 + t].i;
        vin[t] = in[k0 + t].v;
    }
    __syncthreads();
    for (int x = t; x < items * kPolyN; x += kApplyThreads) {
        const int it = x / kPolyN, kk = x - it * kPolyN;
        W[it * kWStride + kk] = in[k0 + it].lane[(iin[it] - kk + 97) % 97];
    }
    __syncthreads();
    for (int ph = 0; ph < 4; ++ph) {  // extend() for all items at once, phase by phase
        const int lo = 97 + 33 * ph, len = min(33, kWExt - lo);
        for (int x = t; x < items * len; x += kApplyThreads) {
            const int it = x / len, n = lo + (x - it * len);
            uint32_t* Wi = W + it * kWStride;
            Wi[n] = Wi[n - 97] - Wi[n - 33];
        }
        __syncthreads();
    }

    const int it = t / 13, cg = t - it * 13;
    if (it < items) {
        const uint32_t* w_it = W + it * kWStride + 8 * cg;
        uint32_t acc[8], win[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            acc[c] = 0;
            win[c] = w_it[c];
        }
#pragma unroll 1
        for (int j0 = 0; j0 < kJPad; j0 += 8) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                const uint32_t pj = p[j0 + jj];
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[c] += pj * win[(jj + c) & 7];
                win[jj] = w_it[j0 + jj + 8];
            }
        }
        ranmar_state* o = out + k0 + it;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int m = 8 * cg + c;
            if (m < kPolyN) o->lane[96 - m] = acc[c] & kMask;
        }
        if (cg == 0) {
            o->i = 96;  // decanonicalize, jump.hpp:42-48
            o->j = 32;
            const uint32_t v = vin[it];
            o->v = static_cast<uint32_t>((static_cast<uint64_t>(v) + (kMod - dec)) % kMod);
        }
    }
}

__global__ void put_state_kernel(ranmar_state s, ranmar_state* dst) {
    uint32_t* d = reinterpret_cast<uint32_t*>(dst);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(&s);
    for (int k = threadIdx.x; k < 100; k += blockDim.x) d[k] = src[k];
}

// ---- make_streams bulk: s_{(first + 128 h + r) J} = apply(anchor_h, T_r)
constexpr int kBulkThreads = 13 * 32;  // warp = column group (8 columns), lane = 4 rows
constexpr int kStageWords = kRows * 100;
constexpr size_t kBulkSmem = (kJPad * kRows + kWExt + kStageWords + 8) * 4;

struct BulkArgs {
    const ranmar_state* anchors;
    uint64_t H;           // anchors
    const uint32_t* Tt;   // [104][128]
    ranmar_state* out;    // streams [first, first + n)
    uint64_t first, n;
    uint32_t v_base;      // v of the base state
    uint32_t jm;          // J mod m
    ranmar_state base;    // stream 0 verbatim (when first == 0)
};

__global__ void __launch_bounds__(kBulkThreads, 2) bulk_kernel(const __grid_constant__ BulkArgs args) {
    extern __shared__ uint32_t sm[];
    uint32_t* Tt = sm;                       // [104][128]
    uint32_t* W = Tt + kJPad * kRows;        // [208]
    uint32_t* stage = W + kWExt;             // [128][100] state records
    int* anchor_i = reinterpret_cast<int*>(stage + kStageWords);
    const int t = threadIdx.x;
    const int cg = t >> 5, rg = t & 31;

    {   // T^T tile, loaded once per CTA (vectorised)
        const uint4* src = reinterpret_cast<const uint4*>(args.Tt);
        uint4* dst = reinterpret_cast<uint4*>(Tt);
        for (int x = t; x < kJPad * kRows / 4; x += kBulkThreads) dst[x] = src[x];
    }

    for (uint64_t h = blockIdx.x; h < args.H; h += gridDim.x) {
        const ranmar_state* A = args.anchors + h;
        if (t == 0) *anchor_i = A->i;
        __syncthreads();
        const int ai = *anchor_i;
        for (int kk = t; kk < kPolyN; kk += kBulkThreads) W[kk] = A->lane[(ai - kk + 97) % 97];
        __syncthreads();
        extend(W, t, kBulkThreads, [] { __syncthreads(); });

        uint32_t acc[4][8];
        uint32_t win[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            win[c] = W[8 * cg + c];
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) acc[rr][c] = 0;
        }
        const uint32_t* wcg = W + 8 * cg;
#pragma unroll 1
        for (int j0 = 0; j0 < kJPad; j0 += 8) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                const uint4 tv = *reinterpret_cast<const uint4*>(Tt + (j0 + jj) * kRows + 4 * rg);
                const uint32_t tr[4] = {tv.x, tv.y, tv.z, tv.w};
#pragma unroll
                for (int rr = 0; rr < 4; ++rr)
#pragma unroll
                    for (int c = 0; c < 8; ++c) acc[rr][c] += tr[rr] * win[(jj + c) & 7];
                win[jj] = wcg[j0 + jj + 8];
            }
        }
        // Stage decanonicalized records: lane[96 - m] = out[m] (jump.hpp:42-48).
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
            uint32_t* rec = stage + (4 * rg + rr) * 100;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int m = 8 * cg + c;
                if (m < kPolyN) rec[96 - m] = acc[rr][c] & kMask;
            }
        }
        if (t < kRows) {
            const uint64_t k = args.first + h * kRows + t;  // global stream index
            uint32_t* rec = stage + t * 100;
            rec[97] = 96;
            rec[98] = 32;
            // jump_arith(v_base, k J) (jump.hpp:79-86): (k J) mod m = (k mod m)(J mod m) mod m
            const uint64_t km = (k % kMod) * args.jm % kMod;
            const uint64_t dec = km * kDelta % kMod;
            rec[99] = static_cast<uint32_t>((args.v_base + (kMod - dec)) % kMod);
        }
        __syncthreads();
        const uint64_t row0 = h * kRows;
        if (args.first == 0 && row0 == 0) {  // stream 0 is the base itself (jump.hpp:116)
            if (t < 100) stage[t] = reinterpret_cast<const uint32_t*>(&args.base)[t];
            __syncthreads();
        }
        const int rows = static_cast<int>(args.n - row0 < (uint64_t)kRows ? args.n - row0 : (uint64_t)kRows);
        uint4* dst = reinterpret_cast<uint4*>(args.out + row0);
        const uint4* srcv = reinterpret_cast<const uint4*>(stage);
        for (int x = t; x < rows * 25; x += kBulkThreads) dst[x] = srcv[x];
        __syncthreads();
    }
}

}  // namespace

// ---------------------------------------------------------------- launchers

cudaError_t launch_pow(const PowJobs& jobs, int njobs, cudaStream_t stream) {
    count_launch();
    pow_kernel<<<njobs, kPowThreads, 0, stream>>>(jobs);
    return cudaGetLastError();
}

cudaError_t launch_t_table(uint32_t* T, uint32_t* Tt, const uint32_t* Q, cudaStream_t stream) {
    count_launch();
    t_init_kernel<<<1, 128, 0, stream>>>(T);
    for (int b = 0; (1 << b) < kRows; ++b) {
        const int half = 1 << b;
        count_launch();
        mulmod_kernel<<<(half + kMulWarps - 1) / kMulWarps, 32 * kMulWarps, 0, stream>>>(
            T, half, half, Q + b * kPolyN);
    }
    count_launch();
    t_transpose_kernel<<<kJPad, kRows, 0, stream>>>(T, Tt);
    return cudaGetLastError();
}

cudaError_t launch_apply(const ranmar_state* in, ranmar_state* out, uint64_t n, const uint32_t* P,
                         uint32_t dec, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    const uint64_t blocks = (n + kApplyItems - 1) / kApplyItems;
    count_launch();
    apply_kernel<<<static_cast<unsigned>(blocks), kApplyThreads, 0, stream>>>(in, out, n, P, dec);
    return cudaGetLastError();
}

cudaError_t launch_put_state(const ranmar_state& s, ranmar_state* dst, cudaStream_t stream) {
    count_launch();
    put_state_kernel<<<1, 128, 0, stream>>>(s, dst);
    return cudaGetLastError();
}

cudaError_t launch_bulk(const ranmar_state* anchors, uint64_t H, const uint32_t* Tt,
                        ranmar_state* out, uint64_t first, uint64_t n, uint32_t v_base,
                        uint32_t jm, const ranmar_state& base, int sm_count, cudaStream_t stream) {
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kBulkSmem));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    BulkArgs a{anchors, H, Tt, out, first, n, v_base, jm, base};
    const uint64_t grid = H < uint64_t(2 * sm_count) ? H : uint64_t(2 * sm_count);
    count_launch();
    bulk_kernel<<<static_cast<unsigned>(grid), kBulkThreads, kBulkSmem, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace rb
