// Jump-ahead kernels (sm_100a), K3.
//
// The Fibonacci part of a jump by J is u * P_J(A) with P_J = t^J mod phi(t),
// phi = t^97 + t^64 - 1 over Z/2^24 (jump.hpp:60-76, polyring.hpp:113-124;
// PAPER.md:298-324). All coefficient arithmetic is 32-bit mad.lo with
// wraparound and one final mask: only the low 24 bits of each product matter,
// which replaces the reference's 64-bit accumulation (polyring.hpp:88-96)
// without changing a single residue. Level 0 of make_streams, the one large
// integer contraction, runs EXACTLY on the tensor cores (bulk_tc_kernel: u8
// limbs on tcgen05.mma kind::i8, s32 accumulators that cannot overflow).
//
//  pow_kernel        K3a  the squaring chain t^(2^k) mod phi in shared memory
//                         (one CTA, 256 threads split the 9,409 MACs of each
//                         product four ways) and the trinomial fold split into
//                         three conflict-free phases (sources [160,192],
//                         [127,159], [97,126]). Run once per device to fill
//                         the square table Z_k = t^(2^k), k < 320.
//  pow_table_kernel  K3a  the multiply half: t^(E 2^s) = prod_{k in bits(E)}
//                         Z_{k+s} (right-to-left square-and-multiply with the
//                         cached squares), one CTA per exponent, warps reduce
//                         strided factor subsets then a tree.
//  tables_kernel          offset tables Tab_L[r] = P_{r 128^L J}, r < 128.
//  apply2_kernel     K3b  u * P(A) for a batch of states as a Hankel product
//                         out[m] = sum_j p_j w[j + m] over the recurrence
//                         extension w of u (no sequential Horner chain), + K3c
//                         the closed-form arithmetic jump; 64 states per CTA,
//                         2 x 8 register tiles per lane.
//  level_kernel      K3b  one level of the base-128 stream-start tree
//                         S_L[k] = apply(S_{L+1}[k / 128], Tab_L[k % 128]).
//  bulk_tc_kernel    K3b  level 0 (all stream starts) on the tensor cores
//                         (see its header below); the default.
//  bulk_kernel       K3b  the same on the IMAD pipe (RANMAR_BULK=imad, for
//                         A/B timing): per anchor a 128 x 97
//                         x 97 integer "GEMM" tile, T^T
//                         resident in shared memory, double-buffered anchor
//                         extensions, 4 x 8 register tiles, results stored
//                         from registers as 16-B vectors.
#include <cstdint>
#include <cstdlib>

#include "ranmar_device.cuh"

namespace rb {

constexpr int kPolyN = 97;
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

// CTA-level product out = a * b mod phi for exactly 256 threads: four groups
// of 64 threads each take a quarter of a's coefficients, thread tt of a group
// accumulates c[tt], c[tt + 64], c[tt + 128] over its quarter reading b from a
// zero-padded copy (no range tests), the quarters are summed, then folded.
// Shared scratch: bz[320] + part[4][193] + c[193]. out may alias a or b.
struct BlockMulScratch {
    uint32_t bz[320];
    uint32_t part[4][193];
    uint32_t c[193];
};

__device__ __forceinline__ void block_mulmod(const uint32_t* a, const uint32_t* b, uint32_t* out,
                                             BlockMulScratch& s) {
    const int t = threadIdx.x;
    for (int k = t; k < 320; k += 256) s.bz[k] = (k >= 96 && k < 193) ? b[k - 96] : 0u;
    __syncthreads();
    const int g = t >> 6, tt = t & 63;
    const int i0 = 25 * g, i1 = i0 + 25 < kPolyN ? i0 + 25 : kPolyN;
    uint32_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
#pragma unroll 5
    for (int i = i0; i < i1; ++i) {
        const uint32_t ai = a[i];
        const uint32_t* bi = s.bz + 96 + tt - i;
        acc0 += ai * bi[0];
        acc1 += ai * bi[64];
        acc2 += ai * bi[128];
        acc3 += ai * bi[192];  // only used by tt == 0 (c[192])
    }
    s.part[g][tt] = acc0;
    s.part[g][tt + 64] = acc1;
    s.part[g][tt + 128] = acc2;
    if (tt == 0) s.part[g][192] = acc3;
    __syncthreads();
    if (t < 193) s.c[t] = s.part[0][t] + s.part[1][t] + s.part[2][t] + s.part[3][t];
    __syncthreads();
    fold_to(s.c, out, t, 256, [] { __syncthreads(); });
}

__device__ __forceinline__ void block_square(uint32_t* a, BlockMulScratch& s) {
    block_mulmod(a, a, a, s);
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

// Polynomial primitives for the C++ facade's ranmar::poly (polyring.hpp:60-98),
// one 256-thread CTA per item: mode 0 out = a * b mod phi (mul_mod, items of 97
// words), mode 1 out = raw mod phi (reduce_trinomial, a = items of 193 raw
// words, wrapping u32 fold like the reference's).
__global__ void __launch_bounds__(kPowThreads)
    poly_kernel(int mode, const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                uint32_t* __restrict__ out) {
    __shared__ uint32_t sa[kPolyN], sb[kPolyN], so[kPolyN];
    __shared__ BlockMulScratch scr;
    const uint64_t q = blockIdx.x;
    const int t = threadIdx.x;
    if (mode == 0) {
        if (t < kPolyN) {
            sa[t] = a[q * kPolyN + t];
            sb[t] = b[q * kPolyN + t];
        }
        __syncthreads();
        block_mulmod(sa, sb, so, scr);
    } else {
        if (t < 193) scr.c[t] = a[q * 193 + t];
        __syncthreads();
        fold_to(scr.c, so, t, kPowThreads, [] { __syncthreads(); });
    }
    if (t < kPolyN) out[q * kPolyN + t] = so[t];
}

__global__ void __launch_bounds__(kPowThreads) pow_kernel(PowJobs jobs) {
    __shared__ uint32_t a[kPolyN];
    __shared__ BlockMulScratch c;
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

// ---- warp-level product mod phi: out = a * b (a, b, out in shared memory,
// out may alias a; c is a 320-word scratch). 9,409 MACs, then the fold.
// i-outer: lane l accumulates c[l + 32q] (q < 7) for every a_i at once, reading
// b from a zero-padded copy (bz[96 + j] = b_j) so no lane needs a range test;
// 7 independent accumulators per lane instead of one long dependent chain.
constexpr int kMulScratch = 320;

__device__ __forceinline__ void warp_mulmod(const uint32_t* a, const uint32_t* b, uint32_t* c,
                                            uint32_t* out, int l) {
    uint32_t* bz = c;  // [0, 320): zeros, b at 96..192, zeros
    for (int k = l; k < kMulScratch; k += 32) bz[k] = (k >= 96 && k < 193) ? b[k - 96] : 0u;
    __syncwarp();
    uint32_t acc[7] = {0, 0, 0, 0, 0, 0, 0};
#pragma unroll 4
    for (int i = 0; i < kPolyN; ++i) {
        const uint32_t ai = a[i];
        const uint32_t* bi = bz + 96 + l - i;  // bz[96 + (l + 32q) - i] = b_{k - i}
#pragma unroll
        for (int q = 0; q < 7; ++q) acc[q] += ai * bi[32 * q];
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 7; ++q)
        if (l + 32 * q < 193) c[l + 32 * q] = acc[q];
    __syncwarp();
    fold_to(c, out, l, 32, [] { __syncwarp(); });
}

__device__ __forceinline__ void warp_load_poly(uint32_t* dst, const uint32_t* src, int l) {
    for (int k = l; k < kPolyN; k += 32) dst[k] = src[k];
    __syncwarp();
}

// ---- K3a from the cached squares: t^(E * 2^shift) = prod_{k in bits(E)} Z_{k+shift},
// Z_k = t^(2^k) mod phi (right-to-left square-and-multiply; the squarings are
// the per-device table, built once by pow_kernel). One CTA per job; each warp
// multiplies a strided subset of the factors, then a 3-level tree.
constexpr int kPowTabWarps = 8;
constexpr int kMaxPowJobs = 64;

struct PowTabJob {
    uint64_t e[4];
    int shift;
    uint32_t* out;
};
struct PowTabJobs {
    PowTabJob job[kMaxPowJobs];
};

__global__ void __launch_bounds__(32 * kPowTabWarps)
    pow_table_kernel(const __grid_constant__ PowTabJobs jobs, const uint32_t* __restrict__ Z) {
    __shared__ uint32_t acc[kPowTabWarps][kPolyN];
    __shared__ uint32_t fac[kPowTabWarps][kPolyN];
    __shared__ uint32_t scr[kPowTabWarps][kMulScratch];
    __shared__ int used[kPowTabWarps];
    const PowTabJob& job = jobs.job[blockIdx.x];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    int rank = 0;
    bool have = false;
    for (int k = 0; k < 256; ++k) {
        if (!((job.e[k >> 6] >> (k & 63)) & 1u)) continue;
        if (rank++ % kPowTabWarps != w) continue;
        const uint32_t* zk = Z + static_cast<size_t>(k + job.shift) * kPolyN;
        if (!have) {
            warp_load_poly(acc[w], zk, l);
            have = true;
        } else {
            warp_load_poly(fac[w], zk, l);
            warp_mulmod(acc[w], fac[w], scr[w], acc[w], l);
        }
    }
    if (l == 0) used[w] = have;
    __syncthreads();
    for (int stride = 1; stride < kPowTabWarps; stride *= 2) {
        if (w % (2 * stride) == 0 && used[w + stride]) {
            if (used[w]) {
                warp_mulmod(acc[w], acc[w + stride], scr[w], acc[w], l);
            } else {
                warp_load_poly(acc[w], acc[w + stride], l);
            }
        }
        __syncthreads();
        if (w % (2 * stride) == 0 && l == 0) used[w] = used[w] | used[w + stride];
        __syncthreads();
    }
    if (w == 0)
        for (int k = l; k < kPolyN; k += 32) job.out[k] = used[0] ? acc[0][k] : (k == 0);
}

// ---- offset tables: Tab_L[r] = P_{r 128^L J} = prod_{b in bits(r)} Q_{7L + b}
// (warp per entry); Tab_0 and Tab_1 also written transposed for the bulk kernels.
// One CTA per entry: its <= 6 products run at CTA speed (the chain is the
// latency of the whole setup, not the few MACs).
// With put_dst set, block 0 also writes the base state to put_dst (the launch
// that would otherwise be put_state_kernel's / copy_state_kernel's): the
// host-given `put`, or, when dsrc is set, the device-resident *dsrc after the
// invariant check (core.hpp:29-49; a bad state raises the status bit and is
// replaced by a zero state, so nothing downstream reads out of range).
__global__ void __launch_bounds__(256)
    tables_kernel(const uint32_t* __restrict__ Q, uint32_t* __restrict__ Tab,
                  uint32_t* __restrict__ Tt, const __grid_constant__ ranmar_state put,
                  const ranmar_state* __restrict__ dsrc, ranmar_state* __restrict__ put_dst,
                  uint32_t* status) {
    if (put_dst && blockIdx.x == 0) {
        const int k = threadIdx.x;
        if (!dsrc) {
            if (k < 100) reinterpret_cast<uint32_t*>(put_dst)[k] = reinterpret_cast<const uint32_t*>(&put)[k];
        } else {
            __shared__ int bad;
            if (k == 0) bad = !state_ok(dsrc->i, dsrc->j, dsrc->v);
            __syncthreads();
            if (k < 97 && dsrc->lane[k] > kMask) bad = 1;
            __syncthreads();
            if (bad) {
                if (k == 0) atomicOr(status, kStatusBadState);
                if (k < 97) put_dst->lane[k] = 0;
                if (k == 0) {
                    put_dst->i = 96;
                    put_dst->j = 32;
                    put_dst->v = 0;
                }
            } else if (k < 100) {
                reinterpret_cast<uint32_t*>(put_dst)[k] = reinterpret_cast<const uint32_t*>(dsrc)[k];
            }
        }
    }
    __shared__ uint32_t f[7][kPolyN];  // the entry's factors, fetched together up front
    __shared__ uint32_t acc[kPolyN];
    __shared__ BlockMulScratch scr;
    const int e = blockIdx.x, t = threadIdx.x;
    const int lvl = e / kRows, r = e % kRows;
    // all factor rows in one round of loads (one global latency instead of one per product)
    for (int x = t; x < 7 * kPolyN; x += 256) {
        const int b = x / kPolyN, k = x - b * kPolyN;
        if ((r >> b) & 1) f[b][k] = Q[static_cast<size_t>(7 * lvl + b) * kPolyN + k];
    }
    int first = -1;  // lowest set bit of r: start from that factor directly
    for (int b = 0; b < 7 && first < 0; ++b)
        if ((r >> b) & 1) first = b;
    __syncthreads();
    for (int k = t; k < kPolyN; k += 256) acc[k] = first < 0 ? (k == 0) : f[first][k];
    __syncthreads();
    for (int b = first + 1; first >= 0 && b < 7; ++b) {
        if (!((r >> b) & 1)) continue;
        block_mulmod(acc, f[b], acc, scr);
    }
    for (int k = t; k < kPolyN; k += 256) {
        Tab[static_cast<size_t>(e) * kPolyN + k] = acc[k];
        if (lvl < 2) Tt[static_cast<size_t>(lvl) * kPolyN * kRows + k * kRows + r] = acc[k];
    }
}

// ---- recurrence extension of canonical vectors held in shared memory:
// w[n] = w[n-97] - w[n-33] (test_util.hpp:38-46), phases of <= 33 terms.
__device__ __forceinline__ void extend_items(uint32_t* W, int stride, int items, int len, int t,
                                             int nt) {
    for (int lo = 97; lo < len; lo += 33) {
        const int cnt = min(33, len - lo);
        for (int x = t; x < items * cnt; x += nt) {
            const int it = x / cnt, n = lo + (x - it * cnt);
            uint32_t* Wi = W + it * stride;
            Wi[n] = Wi[n - 97] - Wi[n - 33];
        }
        __syncthreads();
    }
}

// Level kernels process kApplyItems states per CTA (shared-memory Hankel tiles):
// 8, or 1 for small levels (a tree's top levels: 64 states would be 8 CTAs).
constexpr int kApplyItemsMax = 8;
#ifndef RB_LEVEL_JS
#define RB_LEVEL_JS 4
#endif
constexpr int kJPad = 104;                        // coefficients padded to 13 x 8

// ---- K3b/K3c for a batch, tiled: out[k] = jump(in[k]) with one shared P.
// 64 states per CTA (3 CTAs per SM; 128 per CTA measured 16 % slower: its
// gather phase overlaps less): canonical vectors in shared memory (odd stride 193),
// extended by the recurrence to 193 terms, then the Hankel products
// out[m] = sum_j p_j w[j + m] as register tiles: warp g owns columns
// m0 = 89 - 8g .. 96 - 8g (state words 8g .. 8g + 7, 16-B stores), lane l owns
// states l and l + 32 with an 8-wide sliding window each: per j one broadcast
// LDS of p_j, two LDS of the windows and 16 IMADs. Column 0 (word 96) is
// summed by all threads in sixths with shared-memory atomics.
constexpr int kA2Items = 64;
constexpr int kA2Rows = kA2Items / 32;  // states per lane
constexpr int kA2Threads = 384;
constexpr int kA2Stride = 193;  // odd: lanes l (+32 rr) hit distinct banks
constexpr size_t kA2Smem = (size_t(kA2Items) * kA2Stride + 128 + 2 * kA2Items) * 4;

__global__ void __launch_bounds__(kA2Threads, 3)
    apply2_kernel(const ranmar_state* in, ranmar_state* out, uint64_t n,
                  const uint32_t* __restrict__ P, uint32_t dec, uint32_t* status) {
    extern __shared__ uint32_t sm[];
    uint32_t* W = sm;                                   // [128][193]
    uint32_t* p = W + kA2Items * kA2Stride;             // [128] (97 used)
    uint32_t* C0 = p + 128;                             // [kA2Items] column-0 sums
    uint32_t* vin = C0 + kA2Items;                      // [128]
    const int t = threadIdx.x;
    const uint64_t k0 = static_cast<uint64_t>(blockIdx.x) * kA2Items;
    const int items = static_cast<int>(n - k0 < (uint64_t)kA2Items ? n - k0 : (uint64_t)kA2Items);
    if (t < 128) p[t] = t < kPolyN ? P[t] : 0u;
    if (t < kA2Items) {
        C0[t] = 0;
        if (t < items) vin[t] = in[k0 + t].v;
    }
    {   // canonical vectors (jump.hpp:32-37): W[it][kk] = lane[(i - kk) mod 97], a warp per state
        const int g = t >> 5, l = t & 31;
#pragma unroll 2
        for (int it = g; it < items; it += kA2Threads / 32) {
            const ranmar_state* src = in + k0 + it;
            // a state violating the invariants raises the status bit; its
            // cursor is clamped so the reads stay inside the record
            const bool ok = state_ok(src->i, src->j, src->v);
            const int i0 = ok ? src->i : 96;
            uint32_t* Wi = W + it * kA2Stride;
            bool bad = !ok;
#pragma unroll
            for (int kk = l; kk < kPolyN; kk += 32) {
                int q = i0 - kk;
                q += q < 0 ? 97 : 0;
                const uint32_t x = src->lane[q];
                bad |= x > kMask;
                Wi[kk] = x;
            }
            if (__any_sync(0xffffffffu, bad) && l == 0) atomicOr(status, kStatusBadState);
        }
    }
    __syncthreads();
    for (int lo = 97; lo < 193; lo += 33) {  // x_n = x_{n-97} - x_{n-33}, 33 terms at a time
        const int cnt = 193 - lo < 33 ? 193 - lo : 33;
        for (int x = t; x < items * cnt; x += kA2Threads) {
            const int it = x / cnt, nn = lo + (x - it * cnt);
            uint32_t* Wi = W + it * kA2Stride;
            Wi[nn] = Wi[nn - 97] - Wi[nn - 33];
        }
        __syncthreads();
    }
    {   // column 0: state t % 64, a sixth of its terms
        const int it = t % kA2Items, part = t / kA2Items;
        const int j0 = 17 * part, j1 = part == 5 ? kPolyN : j0 + 17;
        const uint32_t* Wi = W + it * kA2Stride;
        uint32_t a0 = 0;
#pragma unroll 6
        for (int j = j0; j < j1; ++j) a0 += p[j] * Wi[j];
        atomicAdd(C0 + it, a0);
    }
    const int g = t >> 5, l = t & 31;
    const int m0 = 89 - 8 * g;
    uint32_t acc[kA2Rows][8], win[kA2Rows][8];
#pragma unroll
    for (int rr = 0; rr < kA2Rows; ++rr)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            acc[rr][c] = 0;
            win[rr][c] = W[(l + 32 * rr) * kA2Stride + m0 + c];
        }
#pragma unroll 1
    for (int j0 = 0; j0 < 96; j0 += 8) {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const uint32_t pj = p[j0 + jj];
#pragma unroll
            for (int rr = 0; rr < kA2Rows; ++rr)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[rr][c] += pj * win[rr][(jj + c) & 7];
#pragma unroll
            for (int rr = 0; rr < kA2Rows; ++rr) win[rr][jj] = W[(l + 32 * rr) * kA2Stride + m0 + j0 + jj + 8];
        }
    }
    {   // j = 96: slot c holds W[96 + m0 + c]
        const uint32_t pj = p[96];
#pragma unroll
        for (int rr = 0; rr < kA2Rows; ++rr)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[rr][c] += pj * win[rr][c];
    }
#pragma unroll
    for (int rr = 0; rr < kA2Rows; ++rr) {
        const int it = l + 32 * rr;
        if (it >= items) continue;
        uint4* dst = reinterpret_cast<uint4*>(out[k0 + it].lane + 8 * g);
        // word 8g + q holds canonical column 96 - 8g - q = m0 + 7 - q (decanonicalize, jump.hpp:42-48)
        dst[0] = make_uint4(acc[rr][7] & kMask, acc[rr][6] & kMask, acc[rr][5] & kMask, acc[rr][4] & kMask);
        dst[1] = make_uint4(acc[rr][3] & kMask, acc[rr][2] & kMask, acc[rr][1] & kMask, acc[rr][0] & kMask);
    }
    __syncthreads();
    if (t < items) {  // word 96, cursors i = 96, j = 32, and v by jump_arith
        const uint32_t v = static_cast<uint32_t>((static_cast<uint64_t>(vin[t]) + (kMod - dec)) % kMod);
        *reinterpret_cast<uint4*>(out[k0 + t].lane + 96) = make_uint4(C0[t] & kMask, 96u, 32u, v);
    }
}

// ---- one level of the base-128 stream-start tree:
//   S_L[k] = apply(S_{L+1}[k / 128], Tab_L[k % 128]),  k < count
// (the arithmetic part by jump_arith with (k % 128) * 128^L * J). WMODE
// writes the 193-term canonical extension + v (what the bulk kernel reads)
// instead of a decanonicalized state.
constexpr int kWAnchor = 196;  // words per anchor extension row (193 used)

// JS > 1 (one state per CTA, the tree's small top levels, where latency is all
// that matters): the 13 j-chunks of 8 are split over JS thread groups and the
// partial columns summed through shared memory.
template <bool WMODE, int kApplyItems, int JS = 1>
__global__ void __launch_bounds__(kApplyItems * (WMODE ? 25 : 13) * JS)
    level_kernel(const ranmar_state* __restrict__ in, uint64_t count,
                 const uint32_t* __restrict__ Tab, uint32_t c_lvl, ranmar_state* __restrict__ out,
                 uint32_t* __restrict__ outW, uint32_t* __restrict__ outV) {
    constexpr int CG = WMODE ? 25 : 13;          // column groups of 8
    constexpr int NT = kApplyItems * CG * JS;
    constexpr int EXT = 97 + 8 * CG;             // 297 / 201
    constexpr int STR = (EXT + 8) | 1;           // odd stride
    __shared__ uint32_t W[kApplyItems * STR];
    __shared__ uint32_t p[kApplyItems][kJPad];
    __shared__ uint32_t vin[kApplyItems];
    __shared__ int iin[kApplyItems];
    __shared__ uint32_t part[JS > 1 ? kApplyItems * (JS - 1) * 8 * CG : 1];
    const int t = threadIdx.x;
    const uint64_t k0 = static_cast<uint64_t>(blockIdx.x) * kApplyItems;
    const int items = static_cast<int>(count - k0 < (uint64_t)kApplyItems ? count - k0 : (uint64_t)kApplyItems);
    for (int x = t; x < items * kJPad; x += NT) {
        const int it = x / kJPad, j = x - it * kJPad;
        p[it][j] = j < kPolyN ? Tab[((k0 + it) % kRows) * kPolyN + j] : 0u;
    }
    if (t < items) {
        const ranmar_state* s = in + (k0 + t) / kRows;
        iin[t] = s->i;
        vin[t] = s->v;
    }
    __syncthreads();
    for (int x = t; x < items * kPolyN; x += NT) {
        const int it = x / kPolyN, kk = x - it * kPolyN;
        W[it * STR + kk] = in[(k0 + it) / kRows].lane[(iin[it] - kk + 97) % 97];
    }
    __syncthreads();
    extend_items(W, STR, items, EXT + 8, t, NT);

    const int it = t / (CG * JS), rem = t - it * (CG * JS);
    const int cg = rem % CG, js = rem / CG;
    const bool live = it < items;
    uint32_t acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = 0;
    if (live) {
        const uint32_t* w_it = W + it * STR + 8 * cg;
        const uint32_t* p_it = p[it];
        uint32_t win[8];
#pragma unroll 1
        for (int q = js; q < kJPad / 8; q += JS) {
            const int j0 = 8 * q;
#pragma unroll
            for (int c = 0; c < 8; ++c) win[c] = w_it[j0 + c];
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                const uint32_t pj = p_it[j0 + jj];
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[c] += pj * win[(jj + c) & 7];
                win[jj] = w_it[j0 + jj + 8];
            }
        }
    }
    if (JS > 1) {
        if (live && js > 0) {
#pragma unroll
            for (int c = 0; c < 8; ++c) part[((it * (JS - 1) + js - 1) * CG + cg) * 8 + c] = acc[c];
        }
        __syncthreads();
        if (!live || js > 0) return;
#pragma unroll
        for (int s2 = 0; s2 < JS - 1; ++s2)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[c] += part[((it * (JS - 1) + s2) * CG + cg) * 8 + c];
    }
    if (!live) return;
    const uint64_t k = k0 + it;
    const uint64_t r = k % kRows;
    const uint32_t dec = static_cast<uint32_t>((r * c_lvl % kMod) * kDelta % kMod);
    const uint32_t v = static_cast<uint32_t>((static_cast<uint64_t>(vin[it]) + (kMod - dec)) % kMod);
    if (WMODE) {
        uint32_t* o = outW + k * kWAnchor;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int m = 8 * cg + c;
            if (m < 193) o[m] = acc[c] & kMask;
        }
        if (cg == 0) outV[k] = v;
    } else {
        ranmar_state* o = out + k;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int m = 8 * cg + c;
            if (m < kPolyN) o->lane[96 - m] = acc[c] & kMask;
        }
        if (cg == 0) {
            o->i = 96;
            o->j = 32;
            o->v = v;
        }
    }
}


// A device-resident base state copied into the workspace and checked there
// (the host path checks it before launching): cursors, v and every lane must
// satisfy the reference's invariants. A bad state raises kStatusBadState and is
// replaced by the all-zero state with fresh cursors, so no later kernel indexes
// out of range.
// ---- make_streams bulk (level 0): s_{(first + 128 h + r) J} = apply(anchor_h, T_r).
// Per anchor a 128 x 97 x 97 integer "GEMM" tile on the IMAD pipe:
//  * T^T (97 x 128) stays in shared memory for every anchor the CTA visits;
//  * the anchor's 193-term extension is prefetched into the other half of a
//    double buffer while the current one is consumed (one barrier per anchor);
//  * warp g owns state words [8g, 8g + 8) (columns m = 89 - 8g .. 96 - 8g of
//    the canonical vector, reversed by decanonicalize), lane rg owns rows
//    4rg .. 4rg + 3: a 4 x 8 register tile, one LDS.128 of T and one sliding
//    LDS of the extension per j for 32 IMADs;
//  * column m = 0 (state word 96) is spread over all warps: thread t sums a
//    third of row (t & 127)'s terms into a shared-memory accumulator
//    (red.shared.add, double-buffered per anchor), and after the next barrier
//    128 threads write the record tails (lane[96], i, j, v) as 16-B stores;
//  * results go straight from registers to HBM as 16-B stores (no staging).
constexpr int kBulkWarps = 12;
constexpr int kBulkThreads = 32 * kBulkWarps;
constexpr size_t kBulkSmem = (size_t(kPolyN) * kRows + 3 * kWAnchor + 3 * kRows) * 4 + 3 * 8;

struct BulkArgs {
    const uint32_t* W1;   // anchors' extensions, H x kWAnchor
    uint64_t H;
    const uint32_t* Tt;   // [97][128]
    ranmar_state* out;    // streams [first, first + n)
    uint64_t first, n;
    uint32_t jm;                // J mod m
    const ranmar_state* base;   // the base state in device memory (stream 0 when first == 0)
};

// Record tail of row `row` of anchor h: word 96 (column 0, summed in C0), the
// normalised cursors and v (closed form, jump_arith with k J mod m); zeroes the
// row's accumulator for the anchor after next.
__device__ __forceinline__ void bulk_tail(const BulkArgs& args, uint32_t v_base, uint32_t* C0,
                                          uint64_t h, int row) {
    const uint32_t a0 = C0[row];
    C0[row] = 0;
    const uint64_t row0 = h * kRows;
    const uint64_t rows = args.n - row0 < (uint64_t)kRows ? args.n - row0 : (uint64_t)kRows;
    if (static_cast<uint64_t>(row) >= rows || (args.first == 0 && h == 0 && row == 0)) return;
    const uint64_t k = args.first + row0 + row;
    const uint64_t dec = ((k % kMod) * args.jm % kMod) * kDelta % kMod;
    const uint32_t v = static_cast<uint32_t>((v_base + (kMod - dec)) % kMod);
    *reinterpret_cast<uint4*>(args.out[row0 + row].lane + 96) = make_uint4(a0 & kMask, 96u, 32u, v);
}

// Split-phase CTA barrier on an mbarrier: every thread arrives once per anchor
// (release) and waits (acquire) only where a later anchor needs that anchor's
// shared-memory writes, so warps are never held at a full barrier per anchor.
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
                 "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    uint32_t done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
}

// Anchors are processed in a 3-deep ring: iteration `it` computes anchor it
// from W[it % 3], prefetches anchor it + 2 into W[(it + 2) % 3] (after waiting
// for the end of it - 1, the last reader of that buffer), adds its column-0
// partials into C0[it % 3], and arrives on bar[it % 3]. The record tails of
// anchor it are written at iteration it + 2, after waiting for its end.
__global__ void __launch_bounds__(kBulkThreads, 2) bulk_kernel(const __grid_constant__ BulkArgs args) {
    extern __shared__ uint4 sm4[];
    uint32_t* Tt = reinterpret_cast<uint32_t*>(sm4);  // [97][128]
    uint32_t* Wb = Tt + kPolyN * kRows;               // [3][196]
    uint32_t* C0 = Wb + 3 * kWAnchor;                 // [3][128] column-0 sums
    uint64_t* bar = reinterpret_cast<uint64_t*>(C0 + 3 * kRows);  // [3]
    const int t = threadIdx.x;
    const int g = t >> 5, rg = t & 31;
    const int m0 = 89 - 8 * g;
    const uint64_t G = gridDim.x;
    const uint32_t v_base = args.base->v;

    {   // T^T tile, loaded once per CTA
        const uint4* src = reinterpret_cast<const uint4*>(args.Tt);
        for (int x = t; x < kPolyN * kRows / 4; x += kBulkThreads) sm4[x] = src[x];
    }
    const uint64_t h0 = blockIdx.x;
    for (int q = 0; q < 2; ++q)
        if (h0 + q * G < args.H && t < 193) Wb[q * kWAnchor + t] = args.W1[(h0 + q * G) * kWAnchor + t];
    if (t < 3 * kRows) C0[t] = 0;
    if (t == 0)
        for (int q = 0; q < 3; ++q) mbar_init(bar + q, kBulkThreads);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    // end of iteration k: bar[k % 3], phase parity (k / 3) & 1
    auto wait_end = [&](int k) { mbar_wait(bar + k % 3, static_cast<uint32_t>((k / 3) & 1)); };
    const int crow = t & (kRows - 1), cpart = t >> 7;  // column 0: row, third of the terms
    const int cj0 = 33 * cpart, cj1 = cpart == 2 ? kPolyN : cj0 + 33;
    int it = 0;
    for (uint64_t h = h0; h < args.H; ++it, h += G) {
        const int slot = it % 3;
        const uint32_t* W = Wb + slot * kWAnchor;
        if (it >= 2) {
            wait_end(it - 2);  // W[slot] (prefetched in it - 2) and C0 of anchor it - 2 are complete
            if (t < kRows) bulk_tail(args, v_base, C0 + ((it - 2) % 3) * kRows, h - 2 * G, t);
        }
        uint32_t acc[4][8];
        uint32_t win[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            win[c] = W[m0 + c];
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) acc[rr][c] = 0;
        }
        const uint32_t* wcg = W + m0;
#pragma unroll 1
        for (int j0 = 0; j0 < 96; j0 += 8) {
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
        {   // j = 96: slot c holds W[96 + m0 + c]
            const uint4 tv = *reinterpret_cast<const uint4*>(Tt + 96 * kRows + 4 * rg);
            const uint32_t tr[4] = {tv.x, tv.y, tv.z, tv.w};
#pragma unroll
            for (int rr = 0; rr < 4; ++rr)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[rr][c] += tr[rr] * win[c];
        }
        const uint64_t row0 = h * kRows;
        const uint64_t rows = args.n - row0 < (uint64_t)kRows ? args.n - row0 : (uint64_t)kRows;
        const bool skip0 = args.first == 0 && h == 0;  // stream 0 is the base itself
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
            const uint64_t row = 4 * rg + rr;
            if (row >= rows || (skip0 && row == 0)) continue;
            uint4* dst = reinterpret_cast<uint4*>(args.out[row0 + row].lane + 8 * g);
            // word 8g + q holds canonical column 96 - 8g - q = m0 + 7 - q
            dst[0] = make_uint4(acc[rr][7] & kMask, acc[rr][6] & kMask, acc[rr][5] & kMask,
                                acc[rr][4] & kMask);
            dst[1] = make_uint4(acc[rr][3] & kMask, acc[rr][2] & kMask, acc[rr][1] & kMask,
                                acc[rr][0] & kMask);
        }
        if (skip0 && t < 100)
            reinterpret_cast<uint32_t*>(args.out)[t] = reinterpret_cast<const uint32_t*>(args.base)[t];
        // W[(it + 2) % 3] and C0[slot]: their last readers / the tail that zeroed
        // C0[slot] ran in iteration it - 1
        if (it >= 1) wait_end(it - 1);
        const uint64_t hn = h + 2 * G;
        if (hn < args.H && t < 193) Wb[((it + 2) % 3) * kWAnchor + t] = args.W1[hn * kWAnchor + t];
        {   // column 0 partial sums of this anchor
            uint32_t a0 = 0;
#pragma unroll 11
            for (int j = cj0; j < cj1; ++j) a0 += Tt[j * kRows + crow] * W[j];
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(static_cast<uint32_t>(
                             __cvta_generic_to_shared(C0 + slot * kRows + crow))),
                         "r"(a0)
                         : "memory");
        }
        mbar_arrive(bar + slot);
    }
    // tails of the last two anchors
    for (int k = it >= 2 ? it - 2 : 0; k < it; ++k) {
        wait_end(k);
        if (t < kRows) bulk_tail(args, v_base, C0 + (k % 3) * kRows, h0 + static_cast<uint64_t>(k) * G, t);
    }
}

// ---- make_streams bulk on the TENSOR CORES (tcgen05.mma kind::i8).
// The same product as bulk_kernel, C[r][m] = sum_j T[r][j] w_h[j + m] mod 2^24
// (r < 128 offsets, m < 97 state words, j < 97), computed EXACTLY from 8-bit
// limbs: with T = T0 + 2^8 T1 + 2^16 T2 and W = W0 + 2^8 W1 + 2^16 W2 (u8),
//   C = D0 + 2^8 D1 + 2^16 D2 mod 2^24,  D0 = T0 W0,  D1 = T0 W1 + T1 W0,
//   D2 = T0 W2 + T1 W1 + T2 W0,
// six u8 x u8 -> s32 GEMMs of 128 x 112 x 128 (K padded with zero T limbs,
// N = 112 >= 97) accumulated in TMEM (D0, D1, D2 = 336 columns); the partial
// sums stay below 3 * 97 * 255^2 < 2^25, so the s32 accumulators are exact and
// the only reduction is the final mask, as in the reference's 64-bit
// accumulation (polyring.hpp:88-96). The Hankel operand W[m][k] = w[m + k] is
// never materialised: in the canonical K-major no-swizzle layout a core
// matrix is 8 rows x 16 bytes at a 16-byte row stride, so storing 16 shifted
// copies of each limb plane interleaved, S[(b * 16 + s) * 16 + e] =
// limb(w[16 b + s + e]), makes row m / K-chunk c start at
// ((m / 16 + c) * 16 + m % 16) * 16: leading-byte offset 256 (K) and
// stride-byte offset 128 (N) describe the whole matrix (tools/micro/tc_i8.cu).
// A CTA per SM (128 threads) runs a software pipeline over its anchors h:
// the 112 output columns are split into halves (N = 64 and N = 48, each
// with its own D0/D1/D2 in TMEM: 192 + 144 of the 512 columns), so while the
// threads read half A of anchor h from TMEM (tcgen05.ld), combine it and
// write state records to shared memory, the tensor core already computes
// half A of the next anchor, and likewise for half B; the W planes of the
// next anchor are built (and its w prefetched from HBM two anchors ahead)
// before that. The CTA's 128 consecutive records (51 KB) leave as ONE TMA
// bulk store (cp.async.bulk) from a double-buffered staging area.
constexpr int kTcConsumerWarps = 8;
constexpr int kTcThreads = 32 * (kTcConsumerWarps + 2);  // + one MMA-issuer warp per column half
constexpr int kTcNA = 64, kTcNB = 48;             // column halves (m < 64, 64 <= m < 112)
constexpr uint32_t kTcAPlane = 16384;             // 8 K-chunks x 16 row groups x 128 B
constexpr uint32_t kTcBPlane = 3584;              // 14 blocks x 16 shifts x 16 B
constexpr uint32_t kTcOffB = 0;                             // 2 buffers x 3 planes
constexpr uint32_t kTcOffW = kTcOffB + 2 * 3 * kTcBPlane;   // 240 words of w
constexpr uint32_t kTcOffOut = kTcOffW + 1024;              // kTcStages x 128 records x 400 B
// staging buffers: TcLayout (3 x 51 KB of records, or 1 x 98 KB of WMODE rows)
constexpr uint32_t kTcColT = 3 * 64 + 3 * 48;               // TMEM columns of the T limbs (96)


struct BulkTcArgs {
    const uint32_t* W1;   // anchors' extensions, H x kWAnchor
    uint64_t H;
    const uint32_t* Tt;   // the offset table: T[r][k] at Tt[k * tt_cs + r * tt_rs]
    int tt_rs, tt_cs;
    ranmar_state* out;    // streams [first, first + n)
    uint64_t first, n;
    uint32_t jm;
    const ranmar_state* base;
    uint32_t* outW;       // WMODE: rows' 193-term extensions (n x kWAnchor) and v
    uint32_t* outV;
    uint32_t* status;     // kStatusInternal if the smem / TMEM placement assumptions fail
};

// Staging per anchor: 128 decanonicalised records (400 B) or, in WMODE (the
// tree's level 1, whose outputs are the next level's anchors), 128 rows of
// canonical vector + recurrence extension (kWAnchor words).
template <bool WMODE>
struct TcLayout {
    static constexpr uint32_t kRowBytes = WMODE ? 4 * 196 : 400;
    static constexpr uint32_t kOut = 128 * kRowBytes;
    static constexpr int kStages = WMODE ? 1 : 3;
    static constexpr uint32_t kSmem = (2 * 3 * 3584 + 1024) + kStages * kOut;
    static constexpr uint32_t kLaunchSmem = kSmem + 128;  // + mbarriers and the TMEM base
};
constexpr uint32_t kTcSmemBase = 0x400;  // dynamic smem offset in the CTA window (1 KB reserved)
static_assert(TcLayout<false>::kLaunchSmem <= 227 * 1024 && TcLayout<true>::kLaunchSmem <= 227 * 1024,
              "tensor-core bulk smem");

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (static_cast<uint64_t>(1) << 46);
}

// The three u8 limbs of four coefficients at once (7 PRMTs instead of 9):
// l_a = byte a of w0..w3 packed little-endian.
__device__ __forceinline__ void limbs3(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t& l0,
                                       uint32_t& l1, uint32_t& l2) {
    const uint32_t x = __byte_perm(w0, w1, 0x5140);  // w0.b0 w1.b0 w0.b1 w1.b1
    const uint32_t y = __byte_perm(w2, w3, 0x5140);  // w2.b0 w3.b0 w2.b1 w3.b1
    l0 = __byte_perm(x, y, 0x5410);
    l1 = __byte_perm(x, y, 0x7632);
    l2 = __byte_perm(__byte_perm(w0, w1, 0x0062), __byte_perm(w2, w3, 0x6200), 0x7610);
}

// byte a of each of w0..w3 packed little-endian (the limb a of four coefficients)
__device__ __forceinline__ uint32_t limb4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t a) {
    const uint32_t sel = a | ((a + 4) << 4);
    return __byte_perm(__byte_perm(w0, w1, sel), __byte_perm(w2, w3, sel), 0x5410);
}

// The 24 MMAs of one column half: D0 += T0 W0; D1 += T0 W1 + T1 W0;
// D2 += T0 W2 + T1 W1 + T2 W0 (K = 128 in 4 steps), then a commit to `bar`.
// The T limbs (operand A) live in TMEM: limb a, K-step ks at columns tmT +
// (4 a + ks) 8 (32 i8 per row = 8 columns); only the per-anchor W planes
// (operand B, descriptor dB = limb plane 0 at K-step 0) are read from shared
// memory. With A in shared memory too, the tensor core's operand reads (276 KB
// per anchor) saturated the SM's shared-memory bandwidth.
// Issued by a whole (converged) warp with warp-uniform operands: elect.sync picks
// the one lane that issues each MMA, and the operands stay in uniform registers
// (issued from a lane-divergent region instead, every MMA paid an ELECT /
// R2UR.BROADCAST loop moving its operands to uniform registers, ~15 instructions).
template <int N>
__device__ __forceinline__ void tc_issue_half(uint32_t tmT, uint64_t dB, uint32_t tmem, uint32_t bar) {
    constexpr uint32_t idesc = (2u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (8u << 24);
    constexpr uint32_t ta[6] = {0, 0, 1, 0, 1, 2}, tb[6] = {0, 1, 0, 2, 1, 0}, td[6] = {0, 1, 1, 2, 2, 2};
#pragma unroll
    for (int p = 0; p < 6; ++p) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
            const uint32_t ta_addr = tmT + (ta[p] * 4 + ks) * 8;
            const uint64_t db = dB + ((tb[p] * kTcBPlane + ks * 512) >> 4);
            const uint32_t acc = (p == 0 || p == 1 || p == 3) && ks == 0 ? 0u : 1u;  // first product of a D
            asm volatile(
                "{ .reg .pred e, a; elect.sync _|e, 0xffffffff; setp.ne.u32 a, %4, 0;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, a; }" ::"r"(tmem + td[p] * N),
                "r"(ta_addr), "l"(db), "r"(idesc), "r"(acc)
                : "memory");
        }
    }
    asm volatile(
        "{ .reg .pred e; elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }" ::"r"(bar)
        : "memory");
}

// 16 columns of this thread's TMEM row starting at column `col` of an
// accumulator set with N columns per accumulator: (D0 + 2^8 D1 + 2^16 D2) & mask.
template <int N>
__device__ __forceinline__ void tc_read_chunk(uint32_t taddr, uint32_t (&val)[16]) {
    uint32_t d[3][16];
#pragma unroll
    for (int a = 0; a < 3; ++a)
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(d[a][0]), "=r"(d[a][1]), "=r"(d[a][2]), "=r"(d[a][3]), "=r"(d[a][4]), "=r"(d[a][5]),
              "=r"(d[a][6]), "=r"(d[a][7]), "=r"(d[a][8]), "=r"(d[a][9]), "=r"(d[a][10]), "=r"(d[a][11]),
              "=r"(d[a][12]), "=r"(d[a][13]), "=r"(d[a][14]), "=r"(d[a][15])
            : "r"(taddr + a * N));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int q = 0; q < 16; ++q) val[q] = (d[0][q] + (d[1][q] << 8) + (d[2][q] << 16)) & kMask;
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
}

template <bool WMODE>
__global__ void __launch_bounds__(kTcThreads, 1) bulk_tc_kernel(const __grid_constant__ BulkTcArgs args) {
    using Lay = TcLayout<WMODE>;
    // All shared memory is dynamic (no static __shared__), so it starts at the fixed
    // window offset kTcSmemBase and every UMMA descriptor is a compile-time constant
    // plus a warp-uniform buffer offset (checked on entry). The mbarriers and the
    // TMEM base live after the staging buffers.
    extern __shared__ __align__(1024) uint32_t tc_smem[];
    uint8_t* sm = reinterpret_cast<uint8_t*>(tc_smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Lay::kSmem);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + Lay::kSmem + 64);
    // mbarriers: MMA half A / B complete (tcgen05.commit), TMEM half A / B drained
    // (8 consumer warps), W planes of buffer b built (8)
    enum { kMmaA = 0, kMmaB = 1, kFreeA = 2, kFreeB = 3, kWReady = 4 };
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const uint32_t s0 = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    if (s0 != kTcSmemBase) {
        if (t == 0) atomicOr(args.status, kStatusInternal);
        return;
    }
    const uint32_t b0 = kTcSmemBase + Lay::kSmem;
    auto bar = [&](int k) { return b0 + 8u * static_cast<uint32_t>(k); };
    uint32_t* sw = reinterpret_cast<uint32_t*>(sm + kTcOffW);
    const uint64_t G = gridDim.x;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot)))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (t == 0) {
        const uint32_t cnt[6] = {1, 1, 8, 8, 8, 8};
        for (int k = 0; k < 6; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar(k)), "r"(cnt[k]) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // All 512 columns of one CTA per SM: the allocation starts at column 0, so the
    // accumulators and the T limbs sit at constant TMEM addresses (checked).
    const uint32_t tm = *tmem_slot;
    constexpr uint32_t tmA = 0, tmB = 3 * kTcNA, tmT = kTcColT;
    const bool tm_ok = tm == 0;
    if (!tm_ok && t == 0) atomicOr(args.status, kStatusInternal);
    // T limbs into TMEM once per CTA (warps 0-3, one row each): row r, limb a, K-step
    // ks, column c holds limb a of T[r][32 ks + 4 c .. + 3] (coalesced Tt reads)
    if (warp < 4) {
        const int r = t;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
            uint32_t v[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) {
                const int k = 32 * ks + e;
                v[e] = k < kPolyN ? args.Tt[k * args.tt_cs + r * args.tt_rs] : 0u;
            }
#pragma unroll
            for (uint32_t a = 0; a < 3; ++a) {
                uint32_t q[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) q[c] = limb4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3], a);
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                        tmT + (static_cast<uint32_t>(32 * warp) << 16) + (a * 4 + ks) * 8),
                    "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]), "r"(q[4]), "r"(q[5]), "r"(q[6]), "r"(q[7])
                    : "memory");
            }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint64_t h0 = blockIdx.x;
    const uint32_t n_anchor = h0 < args.H && tm_ok ? static_cast<uint32_t>((args.H - 1 - h0) / G + 1) : 0u;
    const uint64_t dBase = umma_desc(kTcSmemBase + kTcOffB, 256, 128);  // W planes, buffer 0: a constant

    if (warp >= kTcConsumerWarps) {
        // ---------------- producers: one thread per column half issues its MMAs
        // (two warps, so the halves' issue sequences run in parallel)
        const int half = warp - kTcConsumerWarps;
        if (n_anchor) {
            const uint64_t dB0 = dBase + (half ? (1024 >> 4) : 0);  // rows m' >= 64: 4 blocks in
            const uint64_t dBbuf = (3 * kTcBPlane) >> 4;  // descriptor step to the other W buffer
            mbar_wait_a(bar(kWReady), 0);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (half == 0)
                tc_issue_half<kTcNA>(tmT, dB0, tmA, bar(kMmaA));
            else
                tc_issue_half<kTcNB>(tmT, dB0, tmB, bar(kMmaB));
            for (uint32_t i = 0; i + 1 < n_anchor; ++i) {
                const uint32_t nb = (i + 1) & 1;
                mbar_wait_a(bar(kWReady + nb), ((i + 1) >> 1) & 1);
                mbar_wait_a(bar(half ? kFreeB : kFreeA), i & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (half == 0)
                    tc_issue_half<kTcNA>(tmT, dB0 + nb * dBbuf, tmA, bar(kMmaA));
                else
                    tc_issue_half<kTcNB>(tmT, dB0 + nb * dBbuf, tmB, bar(kMmaB));
            }
        }
    } else if (n_anchor) {
        // ---------------- 8 consumer warps: W planes, TMEM read-back, records
        const int wq = warp & 3;       // TMEM lane quarter: rows 32 wq .. 32 wq + 31
        const int sub = warp >> 2;     // which of the two warps of this quarter
        const int row = 32 * wq + lane;
        const uint32_t trow = static_cast<uint32_t>(32 * wq) << 16;
        const uint32_t v_base = args.base->v;
        // Records: w shifted by 3 (sw[n] = w[n - 3]): output column m' = m + 3 is state
        // word 99 - m', so every 16-column chunk maps onto four whole 16-B record groups.
        // WMODE: no shift, column m is canonical word m of the output row.
        constexpr int kShift = WMODE ? 0 : 3;
        auto load_w = [&](uint64_t hh) -> uint32_t {
            return hh < args.H && t >= kShift && t < 193 + kShift ? args.W1[hh * kWAnchor + t - kShift] : 0u;
        };
        auto store_w = [&](uint32_t w0) {
            if (t < 240) sw[t] = w0;
        };
        auto cbar = [] { asm volatile("bar.sync 1, 256;" ::: "memory"); };
        // the two warps of a lane quarter
        auto qbar = [&] { asm volatile("bar.sync %0, 64;" ::"r"(2 + wq) : "memory"); };
        // W planes into buffer `buf` from sw: chunk (b, s) of plane a = limb_a(sw[16 b + s ..
        // 16 b + s + 15]); 224 chunks over the 256 consumer threads
        auto build_w = [&](int buf) {
            if (t < 14 * 16) {
                const int o = 16 * (t >> 4) + (t & 15);
                uint32_t v[16], q[3][4];
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] = sw[o + e];
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    limbs3(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3], q[0][c], q[1][c], q[2][c]);
#pragma unroll
                for (uint32_t a = 0; a < 3; ++a)
                    *reinterpret_cast<uint4*>(sm + kTcOffB + (3 * buf + a) * kTcBPlane + 16 * t) =
                        make_uint4(q[a][0], q[a][1], q[a][2], q[a][3]);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(kWReady + buf));
        };
        // chunk c (columns m' = 16 c .. 16 c + 15) of this row -> record groups 24 - 4 c - q
        auto put_chunk = [&](uint8_t* rec, int c, const uint32_t (&val)[16], uint32_t v) {
            if (WMODE) {  // canonical words 16 c .. 16 c + 15 of the row
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    reinterpret_cast<uint4*>(rec)[4 * c + q] =
                        make_uint4(val[4 * q], val[4 * q + 1], val[4 * q + 2], val[4 * q + 3]);
                return;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int g = 24 - 4 * c - q;
                if (g < 0) break;
                uint4 x = make_uint4(val[4 * q + 3], val[4 * q + 2], val[4 * q + 1], val[4 * q]);
                if (g == 24) x = make_uint4(val[3], 96u, 32u, v);  // word 96, then i, j, v
                reinterpret_cast<uint4*>(rec)[g] = x;
            }
        };
        // v of this row's stream k (jump_arith: v_base - k (J mod m) d mod m), then
        // stepped by the 128 G streams between this thread's consecutive anchors
        const uint64_t dstep = static_cast<uint64_t>(args.jm) * kDelta % kMod;  // per stream
        uint32_t vrow, vstep;
        {
            const uint64_t k = args.first + h0 * kRows + row;
            vrow = static_cast<uint32_t>((v_base + kMod - (k % kMod) * dstep % kMod) % kMod);
            vstep = static_cast<uint32_t>((kRows * G) % kMod * dstep % kMod);
        }
        store_w(load_w(h0));
        uint32_t nw = load_w(h0 + G);
        cbar();
        build_w(0);
        for (uint32_t i = 0; i < n_anchor; ++i) {
            const uint64_t h = h0 + i * G;
            const uint32_t sb = i % Lay::kStages;
            cbar();  // everyone's build_w has read sw
            if (i + 1 < n_anchor) {
                store_w(nw);
                cbar();
                build_w((i + 1) & 1);  // its previous MMAs (anchor i - 1) completed in iteration i - 1
            }
            nw = load_w(h + 2 * G);
            // this quarter's staging of anchor i - kTcStages has been read by its bulk store
            if (sub == 0 && lane == 0 && i >= Lay::kStages)
                asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(Lay::kStages - 1) : "memory");
            qbar();
            uint8_t* rec = sm + kTcOffOut + sb * Lay::kOut + Lay::kRowBytes * row;
            const uint64_t row0 = h * kRows;
            // stream 0 is the base itself (its own cursor layout); WMODE rows are canonical
            const bool is_base = !WMODE && args.first == 0 && h == 0 && row == 0;
            const uint32_t v = vrow;
            vrow = vrow >= vstep ? vrow - vstep : vrow + (kMod - vstep);  // stream k + 128 G
            // half A: chunks 0..3, two per warp of the quarter
            mbar_wait_a(bar(kMmaA), i & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const int c = 2 * sub + cc;
                uint32_t val[16];
                tc_read_chunk<kTcNA>(tmA + trow + 16 * c, val);
                if (!is_base) put_chunk(rec, c, val, v);
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(kFreeA));
            // half B: chunks 4..6 (sub 0: 4 and 5, sub 1: 6)
            mbar_wait_a(bar(kMmaB), i & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (sub == 0) {
#pragma unroll
                for (int c = 4; c < 6; ++c) {
                    uint32_t val[16];
                    tc_read_chunk<kTcNB>(tmB + trow + 16 * (c - 4), val);
                    if (!is_base) put_chunk(rec, c, val, v);
                }
            } else {  // chunk 6: only m' = 96..99 (state words 3..0) are state words
                uint32_t d[3][4];
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(d[a][0]), "=r"(d[a][1]), "=r"(d[a][2]), "=r"(d[a][3])
                                 : "r"(tmB + trow + 32 + a * kTcNB));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                uint32_t val[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) val[q] = (d[0][q] + (d[1][q] << 8) + (d[2][q] << 16)) & kMask;
                if (WMODE)
                    reinterpret_cast<uint4*>(rec)[24] = make_uint4(val[0], val[1], val[2], val[3]);  // word 96
                else if (!is_base)
                    reinterpret_cast<uint4*>(rec)[0] = make_uint4(val[3], val[2], val[1], val[0]);
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            if (is_base && warp == 0) {
                const uint4* src = reinterpret_cast<const uint4*>(args.base);
#pragma unroll
                for (int p = 0; p < 25; ++p) reinterpret_cast<uint4*>(rec)[p] = src[p];
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // records -> bulk copy engine
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(kFreeB));
            // the quarter's 32 consecutive rows leave as one bulk store, issued by its
            // first warp: four stores per anchor, up to kStages in flight
            qbar();
            if (WMODE) {
                // rows' recurrence extension u_n = u_{n-97} - u_{n-33}, n = 97 .. 192, in
                // three rounds of 32 lanes per row (the quarter's 16 + 16 rows), and v
                if (row0 + row < args.n) args.outV[row0 + row] = v;
                for (int rr = 16 * sub; rr < 16 * sub + 16; ++rr) {
                    uint32_t* R = reinterpret_cast<uint32_t*>(sm + kTcOffOut + sb * Lay::kOut +
                                                              Lay::kRowBytes * (32 * wq + rr));
#pragma unroll
                    for (int lo = 97; lo < 193; lo += 32) {
                        const int nn = lo + lane;
                        R[nn] = (R[nn - 97] - R[nn - 33]) & kMask;
                        __syncwarp();
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                qbar();
            }
            if (sub == 0 && lane == 0) {
                const uint64_t r0 = row0 + 32 * wq;
                const uint64_t nr = args.n > r0 ? (args.n - r0 < 32 ? args.n - r0 : 32) : 0;
                void* dst = WMODE ? static_cast<void*>(args.outW + r0 * kWAnchor) : static_cast<void*>(args.out + r0);
                if (nr)
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                                 "r"(s0 + kTcOffOut + sb * Lay::kOut + Lay::kRowBytes * 32u * wq),
                                 "r"(static_cast<uint32_t>(nr * Lay::kRowBytes))
                                 : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
        if (sub == 0 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

// ---- batched jump_state on the TENSOR CORES: out_s = u_s * P(A) for 128
// states per tile, with one shared P (jump.hpp:60-76). As a GEMM with the
// states on M: OUT[s][m] = sum_i W_s[i] p[i - m] (W_s = the 193-term recurrence
// extension of state s's canonical vector, i < 193 -> K padded to 224). The
// shared operand p[i - m] is Toeplitz in (m, i); with the output columns
// reversed, m~ = 108 - m, it is Hankel: B[m~][i] = pp[m~ + i], pp[n] =
// p[n - 108], so the shifted-copy layout of bulk_tc_kernel describes it
// (leading/stride byte offsets 256/128), built once per CTA. Column m~ is
// state word m~ - 12, so each 16-column chunk is four whole 16-B record
// groups. The per-tile operand (the states' extensions, u8 limbs) goes to
// TMEM (168 columns next to the 336 accumulator columns): A from TMEM, B from
// shared memory, six u8 x u8 -> s32 GEMMs of 128 x 112 x 224 per tile, exact
// as in bulk_tc_kernel. One 16-warp CTA per SM; warps w, w + 4, w + 8, w + 12
// share the tile's states 32 w .. 32 w + 31 (their TMEM lane quarter) and split
// each phase; once a tile's MMAs completed, warps 0-7 read it back while warps
// 8-15 already pack the next tile into TMEM (2^20 jumps: 0.394 -> 0.359 ms).
constexpr int kAtThreads = 512;                       // four warps per TMEM lane quarter
constexpr int kAtWq = kAtThreads / 128;               // warps per quarter
constexpr int kAtN = 112;
constexpr int kAtKSteps = 7;                          // K = 224
constexpr uint32_t kAtBPlane = 21 * 16 * 16;          // (7 + 14) blocks x 16 shifts x 16 B
constexpr int kAtWStride = 196;                       // 16-B rows: LDS.128 per lane, 4 wavefronts
constexpr uint32_t kAtOffW = 3 * kAtBPlane;
constexpr uint32_t kAtOffRaw = kAtOffW + 128 * kAtWStride * 4;  // the next tile's raw records
constexpr uint32_t kAtOffBar = kAtOffRaw + 128 * 400 + 128 * 4;  // after the canonical cursors
constexpr uint32_t kAtSmem = kAtOffBar + 64;                      // + 2 mbarriers, TMEM base: 168 KB
constexpr uint32_t kAtColA = 3 * kAtN;                // TMEM: accumulators, then the A limbs

__global__ void __launch_bounds__(kAtThreads, 1)
    apply_tc_kernel(const ranmar_state* __restrict__ in, ranmar_state* __restrict__ out, uint64_t n,
                    const uint32_t* __restrict__ P, uint32_t dec, uint32_t* status) {
    extern __shared__ __align__(1024) uint32_t at_smem[];
    uint8_t* sm = reinterpret_cast<uint8_t*>(at_smem);
    uint32_t* W = reinterpret_cast<uint32_t*>(sm + kAtOffW);
    // all shared memory is dynamic, at the fixed window offset kTcSmemBase (checked),
    // so the UMMA operands below are constants (see bulk_tc_kernel)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + kAtOffBar + 16);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int wq = warp & 3, sub = warp >> 2;  // TMEM lane quarter, which warp of the quarter
    const uint32_t s0 = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    if (s0 != kTcSmemBase) {
        if (t == 0) atomicOr(status, kStatusInternal);
        return;
    }
    const uint32_t bar = kTcSmemBase + kAtOffBar, raw_bar = bar + 8;

    // B planes from p: item x = 16 b + s holds limbs of pp[16 b + s .. + 15]
    for (int x = t; x < 21 * 16; x += kAtThreads) {
        const int o = 16 * (x >> 4) + (x & 15);
        uint32_t v[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int j = o + e - 108;
            v[e] = j >= 0 && j < kPolyN ? P[j] : 0u;
        }
#pragma unroll
        for (uint32_t a = 0; a < 3; ++a)
            *reinterpret_cast<uint4*>(sm + a * kAtBPlane + 16 * x) =
                make_uint4(limb4(v[0], v[1], v[2], v[3], a), limb4(v[4], v[5], v[6], v[7], a),
                           limb4(v[8], v[9], v[10], v[11], a), limb4(v[12], v[13], v[14], v[15], a));
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot)))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(raw_bar) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B planes -> tensor core
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // all 512 columns of one CTA per SM: the allocation starts at column 0 (checked)
    if (*tmem_slot != 0u) {
        if (t == 0) atomicOr(status, kStatusInternal);
        __syncthreads();
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(*tmem_slot) : "memory");
        return;
    }
    constexpr uint32_t tm = 0, tmA = kAtColA;
    const uint32_t tq = static_cast<uint32_t>(32 * wq) << 16;  // this warp's TMEM lane quarter
    const uint64_t dB = umma_desc(kTcSmemBase, 256, 128);
    constexpr uint32_t idesc = (2u << 4) | (static_cast<uint32_t>(kAtN >> 3) << 17) | (8u << 24);
    const uint64_t n_tiles = (n + 127) / 128;
    uint32_t phase = 0;
    const uint4* raw4 = reinterpret_cast<const uint4*>(sm + kAtOffRaw);
    int* ci = reinterpret_cast<int*>(sm + kAtOffRaw + 128 * 400);  // canonical cursor per state
    if (t == 0 && blockIdx.x < n_tiles) {  // the first tile's raw records
        const uint64_t sb0 = static_cast<uint64_t>(blockIdx.x) * 128;
        const uint32_t bytes = static_cast<uint32_t>((n - sb0 < 128 ? n - sb0 : 128) * 400);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(raw_bar), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         s0 + kAtOffRaw),
                     "l"(in + sb0), "r"(bytes), "r"(raw_bar)
                     : "memory");
    }

    // Tile preparation: the tile's raw records arrived in shared memory (bulk copy
    // issued during the previous preparation); each word goes to its canonical
    // position u[k] = lane[(i - k) mod 97] (jump.hpp:32-37) of its state's W row,
    // the next tile's raw records are fetched, and the rows are extended by the
    // recurrence. Each thread returns its own row's header (lane 96, i, j, v).
    const int row = 32 * wq + lane;
    auto prep = [&](uint64_t tile, uint32_t ph) -> uint4 {
        const uint64_t sb = tile * 128;
        const bool live = sb + row < n;
        const uint64_t rows_here = n - sb < 128 ? n - sb : 128;
        mbar_wait_a(raw_bar, ph);
        uint4 hdr = make_uint4(0u, 96u, 32u, 0u);
        if (live) hdr = raw4[25 * row + 24];
        const bool ok = !live || state_ok(static_cast<int>(hdr.y), static_cast<int>(hdr.z), hdr.w);
        const int i0 = ok ? static_cast<int>(hdr.y) : 96;  // clamped so writes stay inside the row
        bool bad = !ok;
        if (sub == 0) ci[row] = i0;
        __syncthreads();
#pragma unroll 4
        {   // thread (state st = t / 4, part t % 4) re-lays chunks part, part + 4, ... of st
            const int st = t >> 2, part = t & 3;
            const bool in_tile = static_cast<uint64_t>(st) < rows_here;
            uint32_t* Wr = W + st * kAtWStride;
            const uint4* rs = raw4 + 25 * st;
            int k = ci[st] - 4 * part;  // canonical index of the chunk's first word
            k += k < 0 ? 97 : 0;
#pragma unroll
            for (int c = part; c < 25; c += 4) {
                uint4 x = make_uint4(0u, 0u, 0u, 0u);
                if (in_tile) x = rs[c];
                Wr[k] = x.x;
                bad |= x.x > kMask;
                if (c < 24) {
                    int k1 = k == 0 ? 96 : k - 1;
                    Wr[k1] = x.y;
                    k1 = k1 == 0 ? 96 : k1 - 1;
                    Wr[k1] = x.z;
                    k1 = k1 == 0 ? 96 : k1 - 1;
                    Wr[k1] = x.w;
                    bad |= (x.y | x.z | x.w) > kMask;
                }
                k -= 16;  // the next chunk of this thread: 4 chunks = 16 words on
                k += k < 0 ? 97 : 0;
            }
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, kStatusBadState);
        __syncthreads();  // raw staging consumed: fetch the next tile behind this one's work
        if (t == 0) {
            const uint64_t nt = tile + gridDim.x;
            if (nt < n_tiles) {
                const uint64_t nsb = nt * 128;
                const uint32_t bytes = static_cast<uint32_t>((n - nsb < 128 ? n - nsb : 128) * 400);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(raw_bar), "r"(bytes)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        s0 + kAtOffRaw),
                    "l"(in + nsb), "r"(bytes), "r"(raw_bar)
                    : "memory");
            }
        }
        // recurrence extension x_n = x_{n-97} - x_{n-33} into W rows [97, 193): three
        // rounds of 32 per state (each reads only earlier rounds: n - 33 < lo)
        for (int it = 0; it < 128 / (4 * kAtWq); ++it) {
            uint32_t* Wr = W + ((128 / (4 * kAtWq)) * warp + it) * kAtWStride;
#pragma unroll
            for (int lo = 97; lo < 193; lo += 32) {
                const int nn = lo + lane;
                Wr[nn] = Wr[nn - 97] - Wr[nn - 33];
                __syncwarp();
            }
            if (lane < 3) Wr[193 + lane] = 0u;  // K padding read by the 16-B loads
        }
        __syncthreads();
        return hdr;
    };

    // this thread's row of the tile in W as u8 limbs into TMEM: limb a, K-step ks at
    // tmA + (7 a + ks) 8, K-steps ks0, ks0 + kstep, ...
    auto pack = [&](int ks0, int kstep) {
        const uint4* Wr4 = reinterpret_cast<const uint4*>(W + row * kAtWStride);
#pragma unroll 1
        for (int ks = ks0; ks < kAtKSteps; ks += kstep) {
            uint32_t v[32];
#pragma unroll
            for (int e4 = 0; e4 < 8; ++e4) {
                uint4 x = make_uint4(0u, 0u, 0u, 0u);
                if (8 * ks + e4 < kAtWStride / 4) x = Wr4[8 * ks + e4];
                v[4 * e4] = x.x;
                v[4 * e4 + 1] = x.y;
                v[4 * e4 + 2] = x.z;
                v[4 * e4 + 3] = x.w;
            }
            uint32_t q[3][8];
#pragma unroll
            for (int c = 0; c < 8; ++c)
                limbs3(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3], q[0][c], q[1][c], q[2][c]);
#pragma unroll
            for (uint32_t a = 0; a < 3; ++a)
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                        tmA + tq + (a * kAtKSteps + ks) * 8),
                    "r"(q[a][0]), "r"(q[a][1]), "r"(q[a][2]), "r"(q[a][3]), "r"(q[a][4]), "r"(q[a][5]),
                    "r"(q[a][6]), "r"(q[a][7])
                    : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    };
    // read back chunks c0, c0 + cstep, ... of this thread's row, combine the limbs,
    // decanonicalize (jump.hpp:42-48): column m~ of chunk c is word m~ - 12 -> groups
    // 4 c - 3 + q hold val[4 q .. 4 q + 3]
    auto readback = [&](uint64_t tile, const uint4 hdr, int c0, int cstep) {
        const uint64_t srow = tile * 128 + row;
        const uint32_t v = static_cast<uint32_t>((static_cast<uint64_t>(hdr.w) + (kMod - dec)) % kMod);
        uint4* dst = srow < n ? reinterpret_cast<uint4*>(out[srow].lane) : nullptr;
#pragma unroll 1
        for (int c = c0; c < 7; c += cstep) {
            uint32_t val[16];
            tc_read_chunk<kAtN>(tm + tq + 16 * c, val);
            if (dst) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int g = 4 * c - 3 + q;
                    if (g < 0) continue;
                    const uint4 x = g == 24 ? make_uint4(val[12], 96u, 32u, v)
                                            : make_uint4(val[4 * q], val[4 * q + 1], val[4 * q + 2], val[4 * q + 3]);
                    __stcs(dst + g, x);
                }
            }
        }
    };

    uint4 hdr_next = make_uint4(0u, 96u, 32u, 0u);
    if (blockIdx.x < n_tiles) {
        hdr_next = prep(blockIdx.x, 0);
        pack(sub, 4);  // the first tile: K-steps sub, sub + 4 on all 16 warps
    }
    // Per tile: issue its MMAs, prepare the next tile in shared memory while the
    // tensor core runs, then, once the MMAs are done, read this tile back (warps
    // 0-7) while the next tile's rows are packed into TMEM (warps 8-15): the
    // accumulators and the A operand are disjoint TMEM columns, and the A operand
    // is free as soon as this tile's MMAs completed.
    for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, phase ^= 1u) {
        const uint4 hdr = hdr_next;
        const bool has_next = tile + gridDim.x < n_tiles;
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // D0 = A0 B0, D1 = A0 B1 + A1 B0, D2 = A0 B2 + A1 B1 + A2 B0 (K = 224 in 7 steps)
        if (warp == 0) {  // converged warp, elect.sync issues (constant operands)
            constexpr uint32_t ta[6] = {0, 0, 1, 0, 1, 2}, tb[6] = {0, 1, 0, 2, 1, 0}, td[6] = {0, 1, 1, 2, 2, 2};
#pragma unroll
            for (int pq = 0; pq < 6; ++pq) {
#pragma unroll
                for (int ks = 0; ks < kAtKSteps; ++ks) {
                    const uint32_t aa = tmA + (ta[pq] * kAtKSteps + ks) * 8;
                    const uint64_t db = dB + ((tb[pq] * kAtBPlane + ks * 512) >> 4);
                    const uint32_t acc = (pq == 0 || pq == 1 || pq == 3) && ks == 0 ? 0u : 1u;
                    asm volatile(
                        "{ .reg .pred e, a; elect.sync _|e, 0xffffffff; setp.ne.u32 a, %4, 0;\n\t"
                        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, a; }" ::"r"(tm + td[pq] * kAtN),
                        "r"(aa), "l"(db), "r"(idesc), "r"(acc)
                        : "memory");
                }
            }
            asm volatile(
                "{ .reg .pred e; elect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }" ::"r"(bar)
                : "memory");
        }
        if (has_next) hdr_next = prep(tile + gridDim.x, phase ^ 1u);
        mbar_wait_a(bar, phase);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (sub < 2)
            readback(tile, hdr, sub, 2);
        else if (has_next)
            pack(sub - 2, 2);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

}  // namespace

// ---------------------------------------------------------------- launchers

cudaError_t launch_poly(int mode, const uint32_t* a, const uint32_t* b, uint32_t* out, uint64_t n,
                        cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    count_launch();
    poly_kernel<<<static_cast<unsigned>(n), kPowThreads, 0, stream>>>(mode, a, b, out);
    return cudaGetLastError();
}

cudaError_t launch_pow(const PowJobs& jobs, int njobs, cudaStream_t stream) {
    count_launch();
    pow_kernel<<<njobs, kPowThreads, 0, stream>>>(jobs);
    return cudaGetLastError();
}

// jobs: (exponent, shift, out) triples; Z: the per-device square table.
cudaError_t launch_pow_table(const uint64_t (*e)[4], const int* shift, uint32_t* const* out,
                             int njobs, const uint32_t* Z, cudaStream_t stream) {
    for (int b = 0; b < njobs; b += kMaxPowJobs) {
        PowTabJobs jobs{};
        const int cnt = njobs - b < kMaxPowJobs ? njobs - b : kMaxPowJobs;
        for (int q = 0; q < cnt; ++q) {
            for (int w = 0; w < 4; ++w) jobs.job[q].e[w] = e[b + q][w];
            jobs.job[q].shift = shift[b + q];
            jobs.job[q].out = out[b + q];
        }
        count_launch();
        pow_table_kernel<<<cnt, 32 * kPowTabWarps, 0, stream>>>(jobs, Z);
    }
    return cudaGetLastError();
}

cudaError_t launch_tables(const uint32_t* Q, int levels, uint32_t* Tab, uint32_t* Tt,
                          const ranmar_state* put, const ranmar_state* d_src, ranmar_state* put_dst,
                          uint32_t* status, cudaStream_t stream) {
    count_launch();
    ranmar_state pv{};
    if (put) pv = *put;
    tables_kernel<<<levels * kRows, 256, 0, stream>>>(Q, Tab, Tt, pv, put ? nullptr : d_src,
                                                      put || d_src ? put_dst : nullptr, status);
    return cudaGetLastError();
}

namespace {
std::atomic<uint64_t> g_cfg_apply2{0}, g_cfg_bulk{0}, g_cfg_bulk_tc{0}, g_cfg_bulk_tcw{0}, g_cfg_apply_tc{0};
}  // namespace

// Shared-memory limits of the jump kernels, raised by ranmar_device_setup so no
// _dev call (or graph capture) has to do it.
cudaError_t configure_jump_kernels() {
    if (cudaError_t e = ensure_smem(apply2_kernel, static_cast<int>(kA2Smem), g_cfg_apply2)) return e;
    if (cudaError_t e = ensure_smem(bulk_tc_kernel<false>, static_cast<int>(TcLayout<false>::kLaunchSmem), g_cfg_bulk_tc))
        return e;
    if (cudaError_t e = ensure_smem(bulk_tc_kernel<true>, static_cast<int>(TcLayout<true>::kLaunchSmem), g_cfg_bulk_tcw))
        return e;
    if (cudaError_t e = ensure_smem(apply_tc_kernel, static_cast<int>(kAtSmem), g_cfg_apply_tc)) return e;
    return ensure_smem(bulk_kernel, static_cast<int>(kBulkSmem), g_cfg_bulk);
}

cudaError_t launch_apply(const ranmar_state* in, ranmar_state* out, uint64_t n, const uint32_t* P,
                         uint32_t dec, uint32_t* status, int sm_count, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    // batches of >= 128 states on the tensor cores; RANMAR_APPLY=imad keeps the IMAD
    // kernel (A/B timing); single jumps (make_streams' first * J) stay on IMAD
    static const bool use_imad = [] {
        const char* e = std::getenv("RANMAR_APPLY");
        return e && e[0] == 'i';
    }();
    if (!use_imad && n >= 128) {
        if (cudaError_t e = ensure_smem(apply_tc_kernel, static_cast<int>(kAtSmem), g_cfg_apply_tc)) return e;
        const uint64_t tiles = (n + 127) / 128;
        const uint64_t grid = tiles < uint64_t(sm_count) ? tiles : uint64_t(sm_count);
        count_launch();
        apply_tc_kernel<<<static_cast<unsigned>(grid), kAtThreads, kAtSmem, stream>>>(in, out, n, P, dec, status);
        return cudaGetLastError();
    }
    if (cudaError_t e = ensure_smem(apply2_kernel, static_cast<int>(kA2Smem), g_cfg_apply2)) return e;
    count_launch();
    apply2_kernel<<<static_cast<unsigned>((n + kA2Items - 1) / kA2Items), kA2Threads, kA2Smem,
                    stream>>>(in, out, n, P, dec, status);
    return cudaGetLastError();
}

cudaError_t launch_level(const ranmar_state* in, uint64_t count, const uint32_t* Tab,
                         uint32_t c_lvl, ranmar_state* out, uint32_t* outW, uint32_t* outV,
                         cudaStream_t stream) {
    count_launch();
    if (count <= 1024) {  // one state per CTA: the level's latency, not its MACs, matters
        constexpr int JS = RB_LEVEL_JS;  // j-chunks split over JS thread groups
        const unsigned blocks = static_cast<unsigned>(count);
        if (outW)
            level_kernel<true, 1, JS><<<blocks, 25 * JS, 0, stream>>>(in, count, Tab, c_lvl, out, outW, outV);
        else
            level_kernel<false, 1, JS><<<blocks, 13 * JS, 0, stream>>>(in, count, Tab, c_lvl, out, outW, outV);
        return cudaGetLastError();
    }
    constexpr int I = kApplyItemsMax;
    const uint64_t blocks = (count + I - 1) / I;
    if (outW)
        level_kernel<true, I><<<static_cast<unsigned>(blocks), I * 25, 0, stream>>>(
            in, count, Tab, c_lvl, out, outW, outV);
    else
        level_kernel<false, I><<<static_cast<unsigned>(blocks), I * 13, 0, stream>>>(
            in, count, Tab, c_lvl, out, outW, outV);
    return cudaGetLastError();
}



cudaError_t launch_bulk(const uint32_t* W1, uint64_t H, const uint32_t* Tt, ranmar_state* out,
                        uint64_t first, uint64_t n, uint32_t jm, const ranmar_state* d_base,
                        uint32_t* status, int sm_count, cudaStream_t stream) {
    // tensor-core bulk by default; RANMAR_BULK=imad selects the IMAD kernel (A/B timing)
    static const bool use_imad = [] {
        const char* e = std::getenv("RANMAR_BULK");
        return e && e[0] == 'i';
    }();
    const uint64_t grid = H < uint64_t(use_imad ? 2 * sm_count : sm_count) ? H
                                                                           : uint64_t(use_imad ? 2 * sm_count : sm_count);
    if (!use_imad) {
        if (cudaError_t e = ensure_smem(bulk_tc_kernel<false>, static_cast<int>(TcLayout<false>::kLaunchSmem), g_cfg_bulk_tc))
            return e;
        BulkTcArgs a{W1, H, Tt, 1, kRows, out, first, n, jm, d_base, nullptr, nullptr, status};
        count_launch();
        bulk_tc_kernel<false><<<static_cast<unsigned>(grid), kTcThreads, TcLayout<false>::kLaunchSmem, stream>>>(a);
        return cudaGetLastError();
    }
    if (cudaError_t e = ensure_smem(bulk_kernel, static_cast<int>(kBulkSmem), g_cfg_bulk)) return e;
    BulkArgs a{W1, H, Tt, out, first, n, jm, d_base};
    count_launch();
    bulk_kernel<<<static_cast<unsigned>(grid), kBulkThreads, kBulkSmem, stream>>>(a);
    return cudaGetLastError();
}

// Level 1 of the stream-start tree on the tensor cores (large trees): rows
// k = 128 h + r = apply(anchor h, Tab[r]) written as 193-term extensions + v,
// the bulk kernels' anchors. W: the anchors' extensions; Tab transposed [97][128];
// v by jump_arith from `src` (the level's source state) with c_lvl = 128^L J mod m.
cudaError_t launch_level_tc(const uint32_t* W, uint64_t H, const uint32_t* Tab, uint64_t count,
                            uint32_t c_lvl, const ranmar_state* src, uint32_t* outW, uint32_t* outV,
                            uint32_t* status, int sm_count, cudaStream_t stream) {
    if (cudaError_t e = ensure_smem(bulk_tc_kernel<true>, static_cast<int>(TcLayout<true>::kLaunchSmem), g_cfg_bulk_tcw))
        return e;
    const uint64_t grid = H < uint64_t(sm_count) ? H : uint64_t(sm_count);
    BulkTcArgs a{W, H, Tab, 1, kRows, nullptr, 0, count, c_lvl, src, outW, outV, status};
    count_launch();
    bulk_tc_kernel<true><<<static_cast<unsigned>(grid), kTcThreads, TcLayout<true>::kLaunchSmem, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace rb
