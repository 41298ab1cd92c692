// Device-side state persistence: bulk ranmar::to_text /
// from_text (serialize.hpp:21-40 / :81-136) for arrays of device states, so
// stream starts made on the GPU (e.g. config 3's 2^20) can be exported and
// re-imported in the reference's "ranmar24 v1" text without a CPU loop.
//
//   text_len_kernel    thread per state: exact byte length of its text
//   scan kernels       exclusive prefix sum of the lengths -> offsets
//   to_text_kernel     warp per state: lane-parallel line formatting, the
//                      line offsets by a warp prefix sum
//   from_text_kernel   thread per state: the reference's strict parser
//                      (same checks, same 1-based line numbers in the error)
#include <cstdint>

#include "ranmar_device.cuh"

namespace rb {

namespace {

// Decimal digits of x: independent compares instead of a division chain.
__device__ __forceinline__ int ndigits(uint32_t x) {
    return 1 + (x >= 10u) + (x >= 100u) + (x >= 1000u) + (x >= 10000u) + (x >= 100000u) +
           (x >= 1000000u) + (x >= 10000000u) + (x >= 100000000u) + (x >= 1000000000u);
}

// x in decimal at p (no terminator); returns the end. The low and high 4-digit
// groups are converted by two independent chains.
__device__ __forceinline__ char* put_uint(char* p, uint32_t x) {
    const int d = ndigits(x);
    uint32_t hi = x / 10000u, lo = x - hi * 10000u;
    char* e = p + d;
    int k = d - 1;
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // the low group (digits d-1 .. d-4)
        if (k < 0) break;
        const uint32_t t = lo / 10u;
        p[k--] = static_cast<char>('0' + (lo - 10u * t));
        lo = t;
    }
    while (k >= 0) {  // the high group (at most 6 more digits)
        const uint32_t t = hi / 10u;
        p[k--] = static_cast<char>('0' + (hi - 10u * t));
        hi = t;
    }
    return e;
}

// serialize.hpp:21-40 line by line: 0 "ranmar24 v1", 1 "i <i+1> j <j+1>",
// 2 "v <v>", 3 + k "u <k+1> <lane[k]>".
__device__ __forceinline__ int line_len(const ranmar_state& s, int line) {
    if (line == 0) return 12;
    if (line == 1) return 2 + ndigits(s.i + 1) + 3 + ndigits(s.j + 1) + 1;
    if (line == 2) return 2 + ndigits(s.v) + 1;
    const int k = line - 3;  // k + 1 <= 97: at most two digits
    return 2 + (k + 1 >= 10 ? 2 : 1) + 1 + ndigits(s.lane[k]) + 1;
}

// "u <k+1> <x>\n" for x < 10^8 without loops or data-dependent branches: the
// eight decimal digits come from two 4-digit groups by multiply-high, the
// leading zeros are skipped by predicated byte stores (the generic put_uint
// loops cost ~4x the instructions, and this line is 97 of every state's 100).
__device__ __forceinline__ void put_u_line(char* p, uint32_t k1, uint32_t x) {
    p[0] = 'u';
    p[1] = ' ';
    const bool two = k1 >= 10u;
    const uint32_t kt = k1 / 10u;
    p[2] = static_cast<char>('0' + (two ? kt : k1));
    if (two) p[3] = static_cast<char>('0' + (k1 - 10u * kt));
    char* q = p + (two ? 4 : 3);
    *q++ = ' ';
    const int d = ndigits(x);  // 1..8
    const uint32_t hi = x / 10000u, lo = x - 10000u * hi;
    uint32_t dig[8];
    {
        const uint32_t h1 = hi / 100u, h0 = hi - 100u * h1, l1 = lo / 100u, l0 = lo - 100u * l1;
        const uint32_t g[4] = {h1, h0, l1, l0};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t t = g[c] / 10u;
            dig[2 * c] = t;
            dig[2 * c + 1] = g[c] - 10u * t;
        }
    }
    char* z = q - (8 - d);  // digit i of the 8 lands at z + i
#pragma unroll
    for (int i = 0; i < 8; ++i)
        if (i >= 8 - d) z[i] = static_cast<char>('0' + dig[i]);
    q[d] = '\n';
}

__device__ __forceinline__ void put_line(const ranmar_state& s, int line, char* p) {
    if (line >= 3) {
        put_u_line(p, static_cast<uint32_t>(line - 2), s.lane[line - 3]);
        return;
    }
    if (line == 0) {
        const char m[] = "ranmar24 v1\n";
        for (int c = 0; c < 12; ++c) p[c] = m[c];
        return;
    }
    if (line == 1) {
        *p++ = 'i';
        *p++ = ' ';
        p = put_uint(p, static_cast<uint32_t>(s.i + 1));
        *p++ = ' ';
        *p++ = 'j';
        *p++ = ' ';
        p = put_uint(p, static_cast<uint32_t>(s.j + 1));
        *p = '\n';
        return;
    }
    if (line == 2) {
        *p++ = 'v';
        *p++ = ' ';
        p = put_uint(p, s.v);
        *p = '\n';
        return;
    }
    const int k = line - 3;
    *p++ = 'u';
    *p++ = ' ';
    p = put_uint(p, static_cast<uint32_t>(k + 1));
    *p++ = ' ';
    p = put_uint(p, s.lane[k]);
    *p = '\n';
}

// warp per state (coalesced lane reads): the exact byte length of its text.
// A state violating the reference's invariants (cursors, v, 24-bit lanes;
// core.hpp:29-49) raises the status bit and gets an EMPTY text (length 0), so
// text_bound() holds and no kernel writes past the caller's buffer.
__global__ void text_len_kernel(const ranmar_state* __restrict__ st, uint64_t n,
                                uint64_t* __restrict__ len, uint32_t* status) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int l = threadIdx.x & 31;
    if (k >= n) return;
    const ranmar_state& s = st[k];
    bool bad = l == 0 && !state_ok(s.i, s.j, s.v);
    for (int q = l; q < 97; q += 32) bad |= s.lane[q] > kMask;
    if (__any_sync(0xffffffffu, bad)) {
        if (l == 0) {
            len[k] = 0;
            atomicOr(status, kStatusBadState);
        }
        return;
    }
    uint32_t L = 0;
#pragma unroll
    for (int pass = 0; pass < 4; ++pass) {
        const int line = pass * 32 + l;
        if (line < 100) L += static_cast<uint32_t>(line_len(s, line));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    if (l == 0) len[k] = L;
}

// exclusive scan, 1024 items per block; block totals to bsum
constexpr int kScanT = 1024;
__global__ void __launch_bounds__(kScanT)
    scan_block_kernel(const uint64_t* __restrict__ in, uint64_t n, uint64_t* __restrict__ out,
                      uint64_t* __restrict__ bsum) {
    __shared__ uint64_t warp_tot[32];
    const int t = threadIdx.x, l = t & 31, w = t >> 5;
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * kScanT + t;
    const uint64_t x = k < n ? in[k] : 0;
    uint64_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (l >= o) incl += y;
    }
    if (l == 31) warp_tot[w] = incl;
    __syncthreads();
    if (w == 0) {
        uint64_t v = warp_tot[l], wi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (l >= o) wi += y;
        }
        warp_tot[l] = wi - v;  // exclusive warp offsets
        if (l == 31 && bsum) bsum[blockIdx.x] = wi;
    }
    __syncthreads();
    if (k < n) out[k] = warp_tot[w] + incl - x;
}

// out[k] += boff[block] (if any) + *base (if any); then out[n] = out[n-1] + len[n-1]
__global__ void scan_add_kernel(uint64_t* __restrict__ out, uint64_t n,
                                const uint64_t* __restrict__ boff, const uint64_t* base) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * kScanT + threadIdx.x;
    if (k < n) out[k] += (boff ? boff[blockIdx.x] : 0) + (base ? *base : 0);
}

__global__ void total_kernel(uint64_t* __restrict__ off, uint64_t n, const uint64_t* __restrict__ len) {
    off[n] = off[n - 1] + len[n - 1];
}

__global__ void copy_u64_kernel(uint64_t* __restrict__ dst, const uint64_t* __restrict__ src) {
    *dst = *src;
}

// Upper bound of one state's text: 12 + 10 + 11 + 97 * 14.
constexpr uint64_t kMaxStateText = 12 + 10 + 11 + 97 * 14;
constexpr int kTTStates = 8;  // states (warps) per CTA
constexpr int kTTStage = kTTStates * static_cast<int>(kMaxStateText) + 16;

// Warp per state: lane handles lines lane, lane+32, lane+64, lane+96, the
// line offsets by a warp prefix sum. The CTA's 8 consecutive texts are
// formatted into shared memory, placed at the same offset mod 16 as in the
// output, and then written out as aligned 16-B stores (byte stores only for
// the unaligned head and tail of the CTA's range).
__global__ void __launch_bounds__(32 * kTTStates)
    to_text_kernel(const ranmar_state* __restrict__ st, uint64_t n,
                   const uint64_t* __restrict__ off, char* __restrict__ text) {
    __shared__ __align__(16) char stage[kTTStage];
    const uint64_t k0 = static_cast<uint64_t>(blockIdx.x) * kTTStates;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const uint64_t k = k0 + w;
    const uint64_t kend = k0 + kTTStates < n ? k0 + kTTStates : n;
    const uint64_t g0 = off[k0], g1 = off[kend];
    const uint32_t shift = static_cast<uint32_t>(g0 & 15);
    // (invalid states have empty texts). The warp-uniform condition predicates the
    // work instead of branching around it: the shuffles then run in converged code
    // (behind a branch ptxas cannot prove uniform they become WARPSYNC/collective
    // loops).
    const bool act = k < n && off[k + 1] != off[k];
    const ranmar_state& s = st[act ? k : k0];
    char* base = stage + shift + (act ? off[k] - g0 : 0);
    uint32_t before = 0;  // bytes of the lines of previous passes
#pragma unroll
    for (int pass = 0; pass < 4; ++pass) {
        const int line = pass * 32 + l;
        const bool mine = act && line < 100;
        const uint32_t len = mine ? static_cast<uint32_t>(line_len(s, line)) : 0u;
        uint32_t incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (l >= o) incl += y;
        }
        if (mine) put_line(s, line, base + before + incl - len);
        before += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncthreads();
    const uint64_t a = (g0 + 15) & ~uint64_t(15), b = g1 & ~uint64_t(15);
    const int t = threadIdx.x;
    if (a >= b) {  // no aligned chunk: bytes only
        for (uint64_t x = g0 + t; x < g1; x += blockDim.x) text[x] = stage[shift + (x - g0)];
        return;
    }
    if (g0 + t < a) text[g0 + t] = stage[shift + t];
    if (b + t < g1) text[b + t] = stage[shift + (b - g0) + t];
    const uint4* src = reinterpret_cast<const uint4*>(stage + shift + (a - g0));
    uint4* dst = reinterpret_cast<uint4*>(text + a);
    for (uint64_t q = t; q < (b - a) / 16; q += blockDim.x) dst[q] = src[q];
}

// ---- parser (serialize.hpp:81-136), thread per state
struct Cursor {
    const char* p;
    const char* end;
};

// next line without terminator; false at end of input
__device__ __forceinline__ bool next_line(Cursor& c, const char*& b, const char*& e) {
    if (c.p >= c.end) return false;
    b = c.p;
    const char* q = c.p;
    while (q < c.end && *q != '\n') ++q;
    e = q;
    c.p = q < c.end ? q + 1 : q;
    if (e > b && e[-1] == '\r') --e;
    return true;
}

__device__ __forceinline__ bool take_uint(const char*& p, const char* e, uint64_t& v) {
    v = 0;
    int nd = 0;
    while (p < e && *p >= '0' && *p <= '9') {
        v = v * 10 + static_cast<uint64_t>(*p - '0');
        if (v > 0xFFFFFFFFull) return false;
        ++p;
        ++nd;
    }
    return nd > 0;
}

__device__ __forceinline__ bool take_lit(const char*& p, const char* e, const char* lit, int n) {
    if (e - p < n) return false;
    for (int c = 0; c < n; ++c)
        if (p[c] != lit[c]) return false;
    p += n;
    return true;
}

// The reference's strict parser, one thread, on [t0, t1): *out written and
// *err = 0 on success, else *err = the 1-based line of the first error.
__device__ void parse_seq(const char* t0, const char* t1, ranmar_state* out, int32_t* err) {
    Cursor c{t0, t1};
    ranmar_state s;
    int line = 1;
    const char *b, *e;
    auto fail = [&](int ln) { *err = ln; };
    if (!next_line(c, b, e) || !(e - b == 11 && take_lit(b, e, "ranmar24 v1", 11))) return fail(line);
    ++line;
    uint64_t i = 0, j = 0, v = 0;
    if (!next_line(c, b, e) || !take_lit(b, e, "i ", 2) || !take_uint(b, e, i) ||
        !take_lit(b, e, " j ", 3) || !take_uint(b, e, j) || b != e)
        return fail(line);
    if (i < 1 || i > 97 || j < 1 || j > 97 || (i + 97 - j) % 97 != 64) return fail(line);
    ++line;
    if (!next_line(c, b, e) || !take_lit(b, e, "v ", 2) || !take_uint(b, e, v) || b != e ||
        v >= kMod)
        return fail(line);
    s.i = static_cast<int32_t>(i) - 1;
    s.j = static_cast<int32_t>(j) - 1;
    s.v = static_cast<uint32_t>(v);
    for (int q = 0; q < 97; ++q) {
        ++line;
        uint64_t idx = 0, lane = 0;
        if (!next_line(c, b, e) || !take_lit(b, e, "u ", 2) || !take_uint(b, e, idx) ||
            !take_lit(b, e, " ", 1) || !take_uint(b, e, lane) || b != e ||
            idx != static_cast<uint64_t>(q) + 1 || lane > kMask)
            return fail(line);
        s.lane[q] = static_cast<uint32_t>(lane);
    }
    for (const char* p = c.p; p < c.end; ++p)
        if (*p != '\n' && *p != '\r' && *p != ' ' && *p != '\t') return fail(line + 1);
    *out = s;
    *err = 0;
}


// Warp per state: the text is staged in shared memory with coalesced 16-B
// loads, the warp finds the line boundaries (32 bytes per step, ordered by a
// ballot), then lane l checks lines l + 1, l + 33,
// l + 65 and l + 97 with the same rules as parse_seq, and the first failing
// line is the warp minimum. Texts longer than the staging buffer (never a
// valid state with ordinary trailing whitespace) go to parse_seq.
constexpr int kFTWarps = 4;
constexpr int kFTCap = 2048;   // staged bytes per warp
constexpr int kFTLines = 128;  // newline positions kept per warp

__device__ __forceinline__ bool is_digit(char ch) { return ch >= '0' && ch <= '9'; }

// decimal at [p, e): value (fails above 2^32 - 1 or with no digit), advances p
__device__ __forceinline__ bool num_at(const char* sm, int& p, int e, uint64_t& v) {
    v = 0;
    int nd = 0;
    while (p < e && is_digit(sm[p])) {
        v = v * 10 + static_cast<uint64_t>(sm[p] - '0');
        if (v > 0xFFFFFFFFull) return false;
        ++p;
        ++nd;
    }
    return nd > 0;
}

__global__ void __launch_bounds__(32 * kFTWarps)
    from_text_warp_kernel(const char* __restrict__ text, const uint64_t* __restrict__ off,
                          uint64_t n, ranmar_state* __restrict__ out, int32_t* __restrict__ err) {
    __shared__ __align__(16) char stage[kFTWarps][kFTCap + 16];
    __shared__ int nl[kFTWarps][kFTLines];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * kFTWarps + w;
    if (k >= n) return;
    const uint64_t b = off[k], e = off[k + 1];
    const int L = static_cast<int>(e - b < uint64_t(1) << 30 ? e - b : uint64_t(1) << 30);
    if (L > kFTCap) {
        if (l == 0) parse_seq(text + b, text + e, out + k, err + k);
        return;
    }
    char* sm = stage[w];
    {   // aligned 16-B chunks covering [b, e); byte shift = b & 15
        const uint64_t a0 = b & ~uint64_t(15);
        const int sh = static_cast<int>(b - a0);
        const int chunks = (sh + L + 15) >> 4;
        const uint4* src = reinterpret_cast<const uint4*>(text + a0);
        for (int q = l; q < chunks; q += 32) reinterpret_cast<uint4*>(sm)[q] = src[q];
        __syncwarp();
        sm += sh;  // sm[0 .. L) is the text
    }
    // newlines, in order: the warp reads 32 consecutive bytes per step (lane l
    // byte x0 + l, conflict-free) and a ballot places the ones it finds
    int total_nl = 0;
    const uint32_t lt = (1u << l) - 1u;
    for (int x0 = 0; x0 < L && total_nl < kFTLines; x0 += 32) {
        const bool isnl = x0 + l < L && sm[x0 + l] == '\n';
        const uint32_t bal = __ballot_sync(0xffffffffu, isnl);
        const int pos = total_nl + __popc(bal & lt);
        if (isnl && pos < kFTLines) nl[w][pos] = x0 + l;
        total_nl += __popc(bal);
    }
    __syncwarp();
    // line ln (1-based) = [start, end) before '\r' stripping; exists iff start < L
    auto line_span = [&](int ln, int& st, int& en) -> bool {
        st = ln == 1 ? 0 : nl[w][ln - 2] + 1;
        if (ln >= 2 && ln - 2 >= total_nl) return false;  // no newline ends line ln - 1
        if (st >= L) return false;
        en = ln - 1 < total_nl ? nl[w][ln - 1] : L;
        if (en > st && sm[en - 1] == '\r') --en;
        return true;
    };
    int bad = 0x7FFFFFFF;  // first failing line seen by this lane
    uint32_t vals[4] = {0, 0, 0, 0};
    int32_t si = 0, sj = 0;
    uint32_t sv = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int ln = l + 1 + 32 * r;
        if (ln > 100) break;
        int p, en;
        bool ok = line_span(ln, p, en);
        if (ok) {
            if (ln == 1) {
                const char h[] = "ranmar24 v1";
                ok = en - p == 11;
                for (int c = 0; ok && c < 11; ++c) ok = sm[p + c] == h[c];
            } else if (ln == 2) {
                uint64_t i = 0, j = 0;
                ok = en - p >= 2 && sm[p] == 'i' && sm[p + 1] == ' ';
                p += 2;
                ok = ok && num_at(sm, p, en, i);
                ok = ok && en - p >= 3 && sm[p] == ' ' && sm[p + 1] == 'j' && sm[p + 2] == ' ';
                p += 3;
                ok = ok && num_at(sm, p, en, j) && p == en;
                ok = ok && i >= 1 && i <= 97 && j >= 1 && j <= 97 && (i + 97 - j) % 97 == 64;
                si = static_cast<int32_t>(i) - 1;
                sj = static_cast<int32_t>(j) - 1;
            } else if (ln == 3) {
                uint64_t v = 0;
                ok = en - p >= 2 && sm[p] == 'v' && sm[p + 1] == ' ';
                p += 2;
                ok = ok && num_at(sm, p, en, v) && p == en && v < kMod;
                sv = static_cast<uint32_t>(v);
            } else {
                uint64_t idx = 0, lane = 0;
                ok = en - p >= 2 && sm[p] == 'u' && sm[p + 1] == ' ';
                p += 2;
                ok = ok && num_at(sm, p, en, idx);
                ok = ok && p < en && sm[p] == ' ';
                ++p;
                ok = ok && num_at(sm, p, en, lane) && p == en &&
                     idx == static_cast<uint64_t>(ln - 3) && lane <= kMask;
                vals[r] = static_cast<uint32_t>(lane);
            }
        }
        if (!ok && ln < bad) bad = ln;
    }
    // after line 100 only whitespace may follow (serialize.hpp: fail(line + 1))
    {
        int tail = L;  // start of what follows line 100
        if (total_nl >= 100) tail = nl[w][99] + 1;
        bool ws = true;
        for (int x = tail + l; x < L; x += 32) {
            const char ch = sm[x];
            ws = ws && (ch == '\n' || ch == '\r' || ch == ' ' || ch == '\t');
        }
        if (!__all_sync(0xffffffffu, ws) && 101 < bad) bad = 101;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    if (bad != 0x7FFFFFFF) {
        if (l == 0) err[k] = bad;
        return;
    }
    ranmar_state* o = out + k;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int ln = l + 1 + 32 * r;
        if (ln >= 4 && ln <= 100) o->lane[ln - 4] = vals[r];
    }
    if (l == 1) {
        o->i = si;
        o->j = sj;
    }
    if (l == 2) o->v = sv;
    if (l == 0) err[k] = 0;
}

}  // namespace

uint64_t text_bound(uint64_t n) { return n * kMaxStateText; }

constexpr uint64_t kTextChunk = uint64_t(kScanT) * kScanT;  // states per scan (2^20)

size_t text_workspace(uint64_t n) {
    const uint64_t c = n < kTextChunk ? n : kTextChunk;
    const uint64_t blocks = (c + kScanT - 1) / kScanT;
    return static_cast<size_t>((c + 2 * blocks + 2) * sizeof(uint64_t));
}

// Offsets d_off[0..n] (d_off[n] = total bytes) and the concatenated texts;
// chunks of 2^20 states, each continuing where the previous one ended.
cudaError_t launch_to_text(const ranmar_state* d_states, uint64_t n, char* d_text,
                           uint64_t* d_off, void* d_ws, uint32_t* status, cudaStream_t stream) {
    for (uint64_t c0 = 0; c0 < n; c0 += kTextChunk) {
        const uint64_t m = n - c0 < kTextChunk ? n - c0 : kTextChunk;
        const uint64_t blocks = (m + kScanT - 1) / kScanT;
        uint64_t* len = static_cast<uint64_t*>(d_ws);
        uint64_t* bsum = len + m;
        uint64_t* boff = bsum + blocks;
        uint64_t* off = d_off + c0;
        const uint64_t* base = c0 ? d_off + c0 : nullptr;  // the previous chunk's total
        // the previous chunk wrote off[c0] = its end; keep it as this chunk's base
        uint64_t* base_copy = boff + blocks;
        count_launch(3);
        text_len_kernel<<<static_cast<unsigned>((m + 7) / 8), 256, 0, stream>>>(d_states + c0, m,
                                                                                len, status);
        if (base) {
            count_launch();
            copy_u64_kernel<<<1, 1, 0, stream>>>(base_copy, base);
        }
        scan_block_kernel<<<static_cast<unsigned>(blocks), kScanT, 0, stream>>>(len, m, off, bsum);
        if (blocks > 1) {
            count_launch(2);
            scan_block_kernel<<<1, kScanT, 0, stream>>>(bsum, blocks, boff, nullptr);
            scan_add_kernel<<<static_cast<unsigned>(blocks), kScanT, 0, stream>>>(
                off, m, boff, base ? base_copy : nullptr);
        } else if (base) {
            count_launch();
            scan_add_kernel<<<1, kScanT, 0, stream>>>(off, m, nullptr, base_copy);
        }
        count_launch();
        total_kernel<<<1, 1, 0, stream>>>(off, m, len);
        to_text_kernel<<<static_cast<unsigned>((m + kTTStates - 1) / kTTStates), 32 * kTTStates, 0,
                         stream>>>(d_states + c0, m, off, d_text);
    }
    return cudaGetLastError();
}

cudaError_t launch_from_text(const char* d_text, const uint64_t* d_off, uint64_t n,
                             ranmar_state* d_states, int32_t* d_err, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    count_launch();
    from_text_warp_kernel<<<static_cast<unsigned>((n + kFTWarps - 1) / kFTWarps), 32 * kFTWarps, 0,
                            stream>>>(d_text, d_off, n, d_states, d_err);
    return cudaGetLastError();
}

}  // namespace rb
