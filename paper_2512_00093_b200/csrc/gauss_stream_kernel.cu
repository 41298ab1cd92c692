// K4s: many gaussian() calls on FEW streams — one warp per stream (sm_100a).
//
// The scalar RanMars-style facade (include/ranmar_b200.hpp, §8f row 3) serves
// gaussian() from device-filled blocks of ONE stream. Thread-per-atom K4 would
// run such a block on a single thread; here a warp cooperates on the stream:
//   1. two generator rounds of the K1 warp mapping give 64 consecutive
//      uniforms = 32 attempt pairs, one per lane, tested with the exact
//      integer form of rsq < 1 && rsq != 0; accepted pairs enter a per-warp
//      queue in order (ballot + popc);
//   2. the queue is drained 32 pairs at a time, one pair per lane, so the fp64
//      log / div / sqrt run with every lane busy;
//   3. the stream advances by exactly the attempts up to the last pair used,
//      and the cached deviate / has_saved follow the sequential calls.
// Deviate sequence and convention: as K4 (gauss_kernel.cu, oracle or_gaussian).
// Output: out[s * count + q] = call q of stream s.
#include <cstdint>

#include "gauss_math.cuh"
#include "ranmar_device.cuh"

namespace rb {

namespace {

__device__ __forceinline__ int mod97s(int64_t x) {
    int64_t r = x % 97;
    return static_cast<int>(r < 0 ? r + 97 : r);
}

constexpr int kSW = 4;     // streams (warps) per block
constexpr int kQCap = 64;  // queued accepted pairs per warp (<= 63 in use)

__global__ void __launch_bounds__(32 * kSW)
    gaussian_stream_kernel(ranmar_gauss_state* __restrict__ g, uint64_t n_streams, uint64_t count,
                           double* __restrict__ out, uint32_t* status) {
    __shared__ uint32_t qu1[kSW][kQCap], qu2[kSW][kQCap], qat[kSW][kQCap];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const uint64_t sid = static_cast<uint64_t>(blockIdx.x) * kSW + w;
    if (sid >= n_streams) return;
    ranmar_gauss_state* gs = g + sid;
    ranmar_state* st = &gs->s;
    const int i0 = st->i, j0 = st->j;
    const uint32_t v0 = st->v;
    if (!state_ok(i0, j0, v0)) {
        if (l == 0) atomicOr(status, kStatusBadState);
        return;
    }
    double* o = out + sid * count;
    // K1 warp mapping: R1..R5 = rounds r-1..r-5 of this lane
    const uint32_t* lane = st->lane;
    uint32_t R1 = lane[(i0 + 32 - l) % 97];
    uint32_t R2 = lane[(i0 + 64 - l) % 97];
    uint32_t R3 = lane[(i0 + 96 - l) % 97];
    uint32_t R4 = (l == 31) ? lane[i0] : 0u, R5 = 0;
    const int src = (l + 31) & 31;
    uint32_t prev = __shfl_sync(0xffffffffu, R4 - R2, src);
    uint32_t V = arith_advance(v0, static_cast<uint64_t>(l) + 1);
    const uint32_t A32 = static_cast<uint32_t>((32ull * kStepA) % kMod);

    bool has = gs->has_saved != 0;
    double saved = gs->saved;
    uint64_t q = 0;
    if (has && count > 0) {
        if (l == 0) o[0] = saved;
        has = false;
        q = 1;
    }
    const uint64_t pairs_total = count > q ? (count - q + 1) / 2 : 0;
    uint64_t produced = 0, rounds = 0;
    uint32_t gsteps = 0, qhead = 0, qtail = 0;
    uint64_t last_attempt = 0;
    bool used_any = false;
    while (q < count) {
        const uint32_t qcount = qtail - qhead;
        const uint64_t need = (count - q + 1) / 2;
        if (qcount < 32 && qcount < need && produced < pairs_total) {
            uint32_t uab[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t S = __shfl_sync(0xffffffffu, R3 - R1, src);
                const uint32_t y = (l == 0) ? prev : S;
                prev = S;
                R5 = R4;
                R4 = R3;
                R3 = R2;
                R2 = R1;
                R1 = y;
                uab[h] = (y - V) & kMask;
                V = add_mod_m(V, A32);
            }
            const int s1 = (2 * l) & 31;  // attempt l = uniforms 2l, 2l + 1 of the 64
            const uint32_t a1 = __shfl_sync(0xffffffffu, uab[0], s1);
            const uint32_t b1 = __shfl_sync(0xffffffffu, uab[1], s1);
            const uint32_t a2 = __shfl_sync(0xffffffffu, uab[0], s1 + 1);
            const uint32_t b2 = __shfl_sync(0xffffffffu, uab[1], s1 + 1);
            const uint32_t u1 = l < 16 ? a1 : b1, u2 = l < 16 ? a2 : b2;
            const int32_t da = static_cast<int32_t>(u1) - (1 << 23);
            const int32_t db = static_cast<int32_t>(u2) - (1 << 23);
            const int64_t s = static_cast<int64_t>(da) * da + static_cast<int64_t>(db) * db;
            const bool acc = s > 0 && s < (int64_t(1) << 46);
            const uint32_t bal = __ballot_sync(0xffffffffu, acc);
            const uint64_t left = pairs_total - produced;
            const uint32_t want = left < 32 ? static_cast<uint32_t>(left) : 32u;
            const uint32_t rank = __popc(bal & ((1u << l) - 1u));
            if (acc && rank < want) {
                const uint32_t slot = (qtail + rank) & (kQCap - 1);
                qu1[w][slot] = u1;
                qu2[w][slot] = u2;
                qat[w][slot] = gsteps * 32 + l;
            }
            const uint32_t nacc = __popc(bal);
            const uint32_t take = nacc < want ? nacc : want;
            qtail += take;
            produced += take;
            rounds += 2;
            ++gsteps;
            __syncwarp();
            continue;
        }
        const uint64_t avail = qcount < need ? qcount : need;
        const uint32_t cnt = avail < 32 ? static_cast<uint32_t>(avail) : 32u;
        if (cnt == 0) {  // unreachable by construction; never spin
            if (l == 0) atomicOr(status, kStatusInternal);
            break;
        }
        double g1 = 0.0, g2 = 0.0;
        uint32_t at = 0;
        if (static_cast<uint32_t>(l) < cnt) {
            const uint32_t slot = (qhead + l) & (kQCap - 1);
            const uint32_t u1 = qu1[w][slot], u2 = qu2[w][slot];
            const double v1 = polar_v(u1), v2 = polar_v(u2);
            at = qat[w][slot];
            const double fac = polar_fac(u1, u2);
            g1 = __dmul_rn(v2, fac);
            g2 = __dmul_rn(v1, fac);
            const uint64_t qa = q + 2 * static_cast<uint64_t>(l);
            st_cs(o + qa, g1);
            if (qa + 1 < count) st_cs(o + qa + 1, g2);
        }
        const double g2_last = __shfl_sync(0xffffffffu, g2, cnt - 1);
        const uint32_t at_last = __shfl_sync(0xffffffffu, at, cnt - 1);
        last_attempt = static_cast<uint64_t>(at_last) + 1;
        used_any = true;
        saved = g2_last;
        const uint64_t qn = q + 2 * static_cast<uint64_t>(cnt);
        if (qn > count) {
            has = true;
            q = count;
        } else {
            q = qn;
        }
        qhead += cnt;
        __syncwarp();
    }
    // advance by exactly the attempts used; N lies in the last two rounds, so
    // x_n for n in [N - 97, N) is among R1..R5
    const uint64_t N = used_any ? 2 * last_attempt : 0;
    __syncwarp();
    if (N > 0) {
        uint32_t* lane_w = st->lane;
        const int64_t lo = static_cast<int64_t>(N) - 97, hi = static_cast<int64_t>(N);
        const uint32_t regs[5] = {R1, R2, R3, R4, R5};
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const int64_t n = 32 * (static_cast<int64_t>(rounds) - 1 - k) + l;
            if (n >= lo && n < hi) lane_w[mod97s(static_cast<int64_t>(i0) - n)] = regs[k] & kMask;
        }
        if (l == 0) {
            st->i = mod97s(static_cast<int64_t>(i0) - static_cast<int64_t>(N % 97));
            st->j = mod97s(static_cast<int64_t>(j0) - static_cast<int64_t>(N % 97));
            st->v = arith_advance(v0, N);
        }
    }
    if (l == 0) {
        gs->has_saved = has ? 1u : 0u;
        if (used_any) gs->saved = saved;
    }
}

}  // namespace

cudaError_t launch_gaussian_stream(ranmar_gauss_state* d_g, uint64_t n_streams, uint64_t count,
                                   double* d_out, uint32_t* status, cudaStream_t stream) {
    if (n_streams == 0 || count == 0) return cudaSuccess;
    const uint64_t blocks = (n_streams + kSW - 1) / kSW;
    count_launch();
    gaussian_stream_kernel<<<static_cast<unsigned>(blocks), 32 * kSW, 0, stream>>>(
        d_g, n_streams, count, d_out, status);
    return cudaGetLastError();
}

}  // namespace rb
