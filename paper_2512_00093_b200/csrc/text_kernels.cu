// Device-side state persistence: bulk ranmar::to_text /
// from_text (serialize.hpp:21-40 / :81-136) for arrays of device states, so
// stream starts made on the GPU (e.g. config 3's 2^20) can be exported and
// re-imported in the reference's "ranmar24 v1" text without a CPU loop.
//
//   to_text_kernel     one pass, warp per state, 8 states per CTA: lines
//                      formatted in registers, the CTA's byte offset found
//                      by a decoupled look-back over the preceding CTAs'
//                      totals (no separate length / scan kernels), the
//                      texts assembled in shared memory and stored 16 B at
//                      a time; writes the offsets too
//   from_text_warp_kernel  warp per state: the reference's strict parser
//                      (same checks, same 1-based line numbers in the error)
#include <cstdint>

#include "ranmar_device.cuh"

namespace rb {

namespace {

// x < 10^8 in decimal as up to 8 ASCII bytes of a u64 (byte 0 = the first
// character), d = its digit count. The two 4-digit groups are split into
// digits by SWAR multiply-shifts (two 16-bit lanes per u32, then bytes), the
// leading zeros are dropped by one shift: no loop, no division chain, no
// per-byte store.
__device__ __forceinline__ uint64_t dec8(uint32_t x, int& d) {
    const uint32_t hi = x / 10000u, lo = x - 10000u * hi;
    auto split = [](uint32_t g) -> uint32_t {  // g < 10^4 -> 4 digit bytes
        const uint32_t q = (g * 5243u) >> 19;    // g / 100 (exact for g < 43699)
        const uint32_t w = q | ((g - 100u * q) << 16);
        const uint32_t t = ((w * 103u) >> 10) & 0x000F000Fu;  // each lane / 10 (lanes < 100)
        return t | ((w - 10u * t) << 8);
    };
    const uint64_t D = split(hi) | (static_cast<uint64_t>(split(lo)) << 32);
    const int lz = min(__clzll(static_cast<long long>(__brevll(D))) >> 3, 7);  // leading zero digits
    d = 8 - lz;
    return (D + 0x3030303030303030ull) >> (8 * lz);
}

typedef unsigned __int128 u128;

// Header line `line` (0..2) of serialize.hpp:21-27 as bytes of a u128 (byte 0
// first): 0 "ranmar24 v1", 1 "i <i+1> j <j+1>", 2 "v <v>", each with its
// '\n'. (Dx, dx) is dec8 of the line's first number (i + 1 or v), computed
// with the other lanes' lane values; j + 1 <= 97 takes one division.
// Returns the length (<= 14).
__device__ __forceinline__ int format_header(const ranmar_state& s, int line, uint64_t Dx, int dx, u128& V) {
    if (line == 0) {  // "ranmar24 v1\n"
        V = static_cast<u128>(0x343272616D6E6172ull) | (static_cast<u128>(0x0A317620ull) << 64);
        return 12;
    }
    if (line == 1) {  // "i a j b\n"
        const uint32_t j1 = static_cast<uint32_t>(s.j + 1), jt = j1 / 10u;
        const int db = j1 >= 10u ? 2 : 1;
        const uint64_t B = j1 >= 10u ? (('0' + jt) | (uint64_t('0' + j1 - 10u * jt) << 8)) : ('0' + j1);
        V = static_cast<u128>(0x2069u) | (static_cast<u128>(Dx) << 16) |
            (static_cast<u128>(0x206A20u | (B << 24) | (uint64_t('\n') << (24 + 8 * db))) << (16 + 8 * dx));
        return 6 + dx + db;
    }
    V = static_cast<u128>(0x2076u) | (static_cast<u128>(Dx) << 16) | (static_cast<u128>('\n') << (16 + 8 * dx));
    return 3 + dx;  // "v x\n"
}

// The len (<= 14) bytes of V at byte offset p of the zero-initialised stage
// S, as u32 words: the first and last word (shared with the neighbouring
// lines, possibly of another warp's state) by shared-memory OR, the ones in
// between by plain stores.
__device__ __forceinline__ void emit_line(uint32_t* S, uint32_t p, int len, const u128& V) {
    const uint32_t sh = 8u * (p & 3u);
    const u128 W = V << sh;
    const uint32_t w4 = sh ? static_cast<uint32_t>(V >> (128u - sh)) : 0u;
    const uint32_t w0 = static_cast<uint32_t>(W), w1 = static_cast<uint32_t>(W >> 32),
                   w2 = static_cast<uint32_t>(W >> 64), w3 = static_cast<uint32_t>(W >> 96);
    const int nw = static_cast<int>(((p & 3u) + static_cast<uint32_t>(len) + 3u) >> 2);  // 2..5
    uint32_t* q = S + (p >> 2);
    atomicOr(q, w0);
    if (nw > 2) q[1] = w1;
    if (nw > 3) q[2] = w2;
    if (nw > 4) q[3] = w3;
    const uint32_t last = nw == 2 ? w1 : nw == 3 ? w2 : nw == 4 ? w3 : w4;
    atomicOr(q + nw - 1, last);
}

// Upper bound of one state's text: 12 + 10 + 11 + 97 * 14.
constexpr uint64_t kMaxStateText = 12 + 10 + 11 + 97 * 14;
constexpr int kTTStates = 8;  // states (warps) per CTA
constexpr int kTTStage = (kTTStates * static_cast<int>(kMaxStateText) + 16 + 15) & ~15;

// "u <k1> <x>\n" (k1 <= 97, x <= kMask) at byte offset p of the zeroed stage
// S, built as u32 words: the prefix "u k1 " shifted by p & 3, the digits of
// x (dec8) with the '\n' after them shifted by (p & 3) + the prefix length
// with funnel shifts, first and last word by shared-memory OR (shared with
// the neighbouring lines), the words between by plain stores. Returns the
// line's length. format (emit = false) only returns the length.
__device__ __forceinline__ uint32_t u_line_len(uint32_t k1, int d) { return (k1 >= 10u ? 6u : 5u) + d; }

__device__ __forceinline__ void emit_u_line(uint32_t* S, uint32_t p, uint32_t k1, uint64_t D, int d) {
    const uint32_t s = p & 3u;
    const uint32_t kt = k1 / 10u;
    const bool two = k1 >= 10u;
    const uint64_t P = two ? (0x2000002075ull | (uint64_t('0' + kt) << 16) | (uint64_t('0' + k1 - 10u * kt) << 24))
                           : (0x20002075ull | (uint64_t('0' + k1) << 16));
    const uint32_t pl = two ? 5u : 4u;
    const uint64_t Ps = P << (8 * s);  // s + pl <= 8 bytes
    const uint64_t Dn = d == 8 ? D : D | (0x0Aull << (8 * d));
    const uint32_t r0 = static_cast<uint32_t>(Dn), r1 = static_cast<uint32_t>(Dn >> 32), r2 = d == 8 ? 0x0Au : 0u;
    const uint32_t u = s + pl;  // 4..8 bytes: the digits start in word 1 or 2
    const uint32_t bs = 8u * (u & 3u);
    const uint32_t z0 = r0 << bs, z1 = __funnelshift_l(r0, r1, bs), z2 = __funnelshift_l(r1, r2, bs);
    const bool w1 = u < 8u;
    const uint32_t o0 = static_cast<uint32_t>(Ps);
    const uint32_t o1 = static_cast<uint32_t>(Ps >> 32) | (w1 ? z0 : 0u);
    const uint32_t o2 = w1 ? z1 : z0, o3 = w1 ? z2 : z1, o4 = w1 ? 0u : z2;
    const uint32_t nw = (s + pl + static_cast<uint32_t>(d) + 4u) >> 2;  // words touched: 2..5
    uint32_t* q = S + (p >> 2);
    atomicOr(q, o0);
    if (nw > 2) q[1] = o1;
    if (nw > 3) q[2] = o2;
    if (nw > 4) q[3] = o3;
    const uint32_t last = nw == 2 ? o1 : nw == 3 ? o2 : nw == 4 ? o3 : o4;
    atomicOr(q + nw - 1, last);
}

// Decoupled look-back status words, one per CTA tile: the top two bits say
// what the low 62 hold (the tile's own byte total, or the inclusive prefix).
constexpr uint64_t kTileAgg = 1ull << 62, kTileInc = 2ull << 62, kTileVal = kTileAgg - 1;

__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// One pass. Tiles of 8 states are taken in ticket order (so every earlier
// tile is resident or done: the look-back cannot deadlock). Warp w loads its
// state (lane l: the lanes of lines l, l+32, l+64, l+96), checks the
// invariants (core.hpp:29-49; a bad state gets an empty text and raises the
// status bit, so text_bound() holds) and sums its line lengths; after one
// barrier the CTA's total is known: warp 0 publishes it and looks back 32
// tiles at a time for the nearest inclusive prefix while all warps emit their
// lines into the zeroed shared stage at CTA-relative offsets. After a second
// barrier the CTA's range is stored with aligned 16-B stores (the stage read
// at the global offset's misalignment by funnel shifts; bytes only for the
// unaligned head and tail). tile_status[] and *ticket start zeroed.
__global__ void
    __launch_bounds__(32 * kTTStates, 7) to_text_kernel(const ranmar_state* __restrict__ st, uint64_t n, uint64_t* __restrict__ off,
                   char* __restrict__ text, uint64_t* tile_status, uint32_t* ticket, uint32_t* status) {
    __shared__ __align__(16) char stage[kTTStage];
    __shared__ uint32_t warp_len[kTTStates], warp_base[kTTStates];
    __shared__ uint64_t s_g0;
    __shared__ uint32_t s_tile, s_agg;
    const int t = threadIdx.x, w = t >> 5, l = t & 31;
    if (t == 0) s_tile = atomicAdd(ticket, 1u);
    for (int q = t; q < kTTStage / 16; q += 32 * kTTStates) reinterpret_cast<uint4*>(stage)[q] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t k0 = static_cast<uint64_t>(tile) * kTTStates;
    const uint64_t k = k0 + w;
    const bool inr = k < n;
    const ranmar_state& s = st[inr ? k : 0];
    uint32_t x[4];
    bool bad = false;
#pragma unroll
    for (int pass = 0; pass < 4; ++pass) {
        const int line = pass * 32 + l;
        const bool u = line >= 3 && line < 100;
        // header lanes convert their first number with everyone else's
        const uint32_t h = line == 1 ? static_cast<uint32_t>(s.i + 1) : line == 2 ? s.v : 0u;
        x[pass] = !inr ? 0u : u ? s.lane[line - 3] : h;
        bad |= x[pass] > kMask;
    }
    bad = __any_sync(0xffffffffu, bad || (inr && l == 0 && !state_ok(s.i, s.j, s.v)));
    if (bad && l == 0) atomicOr(status, kStatusBadState);
    // The warp-uniform condition predicates the work instead of branching around
    // it: the shuffles then run in converged code.
    const bool act = inr && !bad;
    uint64_t D[4];
    int dx = 0;  // digits of the header lanes' first number (pass 0)
    uint32_t incl[4], tot = 0;
#pragma unroll
    for (int pass = 0; pass < 4; ++pass) {
        const int line = pass * 32 + l;
        int d;
        D[pass] = dec8(x[pass], d);
        if (pass == 0) dx = d;
        uint32_t len = 0;
        if (act && line < 100) {
            if (pass == 0 && l < 3) {
                u128 V;
                len = static_cast<uint32_t>(format_header(s, line, D[0], d, V));
            } else {
                len = u_line_len(static_cast<uint32_t>(line - 2), d);
            }
        }
        uint32_t y = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
            if (l >= o) y += z;
        }
        incl[pass] = (tot + y) | (len << 24);  // the line's end within the state's text, and its length
        tot += __shfl_sync(0xffffffffu, y, 31);
    }
    if (l == 0) warp_len[w] = tot;
    __syncthreads();
    uint32_t vi = 0, agg = 0;
    if (w == 0) {  // the CTA's total and the warps' CTA-relative offsets
        const uint32_t v = l < kTTStates ? warp_len[l] : 0u;
        vi = v;
#pragma unroll
        for (int o = 1; o < kTTStates; o <<= 1) {
            const uint32_t z = __shfl_up_sync(0xffffffffu, vi, o);
            if (l >= o) vi += z;
        }
        agg = __shfl_sync(0xffffffffu, vi, kTTStates - 1);
        if (l < kTTStates) warp_base[l] = vi - v;
        if (l == 0) st_relaxed(tile_status + tile, (tile == 0 ? kTileInc : kTileAgg) | agg);
    }
    __syncthreads();
    {   // emit this warp's lines at their CTA-relative offsets
        uint32_t* S = reinterpret_cast<uint32_t*>(stage);
        const uint32_t base = warp_base[w];
#pragma unroll
        for (int pass = 0; pass < 4; ++pass) {
            const uint32_t len = incl[pass] >> 24, p = base + (incl[pass] & 0xFFFFFFu) - len;
            if (!len) continue;
            if (pass == 0 && l < 3) {  // the header line again (cheap, three lanes)
                u128 V;
                format_header(s, pass * 32 + l, D[0], dx, V);
                emit_line(S, p, static_cast<int>(len), V);
            } else {
                const uint32_t k1 = static_cast<uint32_t>(pass * 32 + l - 2);
                emit_u_line(S, p, k1, D[pass], static_cast<int>(len) - (k1 >= 10u ? 6 : 5));
            }
        }
    }
    if (w == 0) {  // look-back for the tile's global offset
        uint64_t prefix = 0;
        if (tile != 0) {
            int64_t j = static_cast<int64_t>(tile) - 1;  // nearest tile of the window
            for (;;) {
                const int64_t idx = j - l;
                uint64_t xs = kTileInc;  // before tile 0: an inclusive 0
                if (idx >= 0)
                    do xs = ld_relaxed(tile_status + idx); while ((xs >> 62) == 0);
                const uint32_t inc = __ballot_sync(0xffffffffu, (xs >> 62) == 2);
                const int stop = inc ? __ffs(inc) - 1 : 31;  // lanes 0..stop count
                uint64_t c = l <= stop ? (xs & kTileVal) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
                prefix += c;
                if (inc) break;
                j -= 32;
            }
            if (l == 0) st_relaxed(tile_status + tile, kTileInc | (prefix + agg));
        }
        if (l < kTTStates && k0 + l < n) off[k0 + l] = prefix + warp_base[l];
        if (l == 0) {
            s_g0 = prefix;
            s_agg = agg;
            if (k0 + kTTStates >= n) off[n] = prefix + agg;  // the last tile
        }
    }
    __syncthreads();
    const uint64_t g0 = s_g0, g1 = g0 + s_agg;
    const uint64_t a = (g0 + 15) & ~uint64_t(15), b = g1 & ~uint64_t(15);
    if (a >= b) {  // no aligned chunk: bytes only
        for (uint32_t y = t; y < static_cast<uint32_t>(g1 - g0); y += 32 * kTTStates) text[g0 + y] = stage[y];
        return;
    }
    const uint32_t head = static_cast<uint32_t>(a - g0), tail0 = static_cast<uint32_t>(b - g0);
    if (t < head) text[g0 + t] = stage[t];
    if (tail0 + t < static_cast<uint32_t>(g1 - g0)) text[b + t] = stage[tail0 + t];
    // aligned chunk c of the output = stage bytes [head + 16 c, +16): 5 words, funnel-shifted
    const uint32_t* S = reinterpret_cast<const uint32_t*>(stage);
    const uint32_t sb = 8u * (head & 3u), w0 = head >> 2;
    uint4* dst = reinterpret_cast<uint4*>(text + a);
    const uint32_t nchunks = static_cast<uint32_t>((b - a) >> 4);
    for (uint32_t c = t; c < nchunks; c += 32 * kTTStates) {
        const uint32_t* q = S + w0 + 4 * c;
        const uint32_t v0 = q[0], v1 = q[1], v2 = q[2], v3 = q[3], v4 = q[4];
        dst[c] = make_uint4(__funnelshift_r(v0, v1, sb), __funnelshift_r(v1, v2, sb), __funnelshift_r(v2, v3, sb),
                            __funnelshift_r(v3, v4, sb));
    }
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

// 16-bit mask of the '\n' bytes of a 16-B chunk (bit i = byte i): exact
// zero-byte test of x ^ 0x0A0A0A0A per word, bytes gathered by a multiply.
__device__ __forceinline__ uint32_t nl_nibble(uint32_t x) {
    const uint32_t y = x ^ 0x0A0A0A0Au;
    const uint32_t z = ~(((y & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | y | 0x7F7F7F7Fu);  // 0x80 where zero
    return ((z >> 7) * 0x01020408u) >> 24;
}
__device__ __forceinline__ uint32_t nl_mask16(uint4 c) {
    return nl_nibble(c.x) | (nl_nibble(c.y) << 4) | (nl_nibble(c.z) << 8) | (nl_nibble(c.w) << 12);
}

// 16 bytes of the warp's stage from byte q (word view S, readable to q + 20)
__device__ __forceinline__ void load16(const uint32_t* S, int q, uint64_t& lo, uint64_t& hi) {
    const uint32_t* W = S + (q >> 2);
    const uint32_t sh = 8u * (q & 3);
    const uint32_t w0 = W[0], w1 = W[1], w2 = W[2], w3 = W[3], w4 = W[4];
    lo = __funnelshift_r(w0, w1, sh) | (static_cast<uint64_t>(__funnelshift_r(w1, w2, sh)) << 32);
    hi = __funnelshift_r(w2, w3, sh) | (static_cast<uint64_t>(__funnelshift_r(w3, w4, sh)) << 32);
}

// A line in canonical "<prefix><digits>" form: the pl-byte prefix P exactly,
// then 1..8 digits and nothing else. Returns false for anything else (left to
// the character-level checks, which also decide leading zeros, other
// separators, overflow and junk), else the number (<= 99999999, so the
// reference's 2^32 - 1 overflow check cannot fire). The line is [q, q+L) of
// the warp's stage.
__device__ __forceinline__ bool parse_num_fast(const uint32_t* S, int q, int L, uint64_t P, int pl, uint32_t& val) {
    const int nd = L - pl;
    if (nd < 1 || nd > 8) return false;
    uint64_t lo, hi;
    load16(S, q, lo, hi);
    if ((lo & ((1ull << (8 * pl)) - 1)) != P) return false;
    const uint64_t M = nd == 8 ? ~0ull : (1ull << (8 * nd)) - 1;
    const uint64_t D = ((lo >> (8 * pl)) | (hi << (64 - 8 * pl))) & M;  // the digit bytes, first at byte 0
    constexpr uint64_t H = 0x8080808080808080ull;
    const uint64_t ge0 = ((D | H) - 0x3030303030303030ull) & H;   // (c & 0x7F) >= '0'
    const uint64_t gt9 = ((D & ~H) + 0x4646464646464646ull) & H;  // (c & 0x7F) > '9'
    if ((ge0 & ~gt9 & ~D & M & H) != (M & H)) return false;
    uint64_t x = (D - (0x3030303030303030ull & M)) << (8 * (8 - nd));  // right-aligned digit values
    x = ((x & 0x0F0F0F0F0F0F0F0Full) * 2561) >> 8;                // pairs
    x = ((x & 0x00FF00FF00FF00FFull) * 6553601) >> 16;            // groups of 4
    x = ((x & 0x0000FFFF0000FFFFull) * 42949672960001ull) >> 32;  // 8 digits
    val = static_cast<uint32_t>(x);
    return true;
}

// Line 2 "i <a> j <b>" (serialize.hpp:98-105) with 1- or 2-digit numbers and
// single spaces: true and (i, j) = (a, b), else false (the character-level
// checks decide). Same values as the reference's take_uint on such a line.
__device__ __forceinline__ bool parse_ij_fast(const uint32_t* S, int q, int L, uint64_t& i, uint64_t& j) {
    if (L < 7 || L > 9) return false;
    uint64_t lo, hi;
    load16(S, q, lo, hi);
    auto c = [&](int k) -> uint32_t { return static_cast<uint32_t>((k < 8 ? lo >> (8 * k) : hi >> (8 * (k - 8))) & 0xFF); };
    auto dig = [](uint32_t ch) { return ch - '0' <= 9u; };
    if ((lo & 0xFFFF) != 0x2069) return false;  // "i "
    const int da = c(3) == ' ' ? 1 : 2, db = L - 5 - da;
    if (db < 1 || db > 2 || c(2 + da) != ' ' || c(3 + da) != 'j' || c(4 + da) != ' ') return false;
    const uint32_t a0 = c(2), a1 = c(3), b0 = c(5 + da), b1 = c(6 + da);
    if (!dig(a0) || (da == 2 && !dig(a1)) || !dig(b0) || (db == 2 && !dig(b1))) return false;
    i = da == 2 ? 10u * (a0 - '0') + (a1 - '0') : a0 - '0';
    j = db == 2 ? 10u * (b0 - '0') + (b1 - '0') : b0 - '0';
    return true;
}

// Line "u <k1> <x>" (serialize.hpp:115-126) in canonical form: 1 (x <= kMask,
// lane = x), 0 (x > kMask: the reference fails on this line), -1 (not
// canonical: the character-level checks decide).
__device__ __forceinline__ int parse_u_fast(const uint32_t* S, int q, int L, uint32_t k1, uint32_t& lane) {
    const uint32_t kt = k1 / 10u;
    const bool two = k1 >= 10u;
    const uint64_t P = two ? (0x2000002075ull | (uint64_t('0' + kt) << 16) | (uint64_t('0' + k1 - 10u * kt) << 24))
                           : (0x20002075ull | (uint64_t('0' + k1) << 16));
    if (!parse_num_fast(S, q, L, P, two ? 5 : 4, lane)) return -1;
    return lane <= kMask ? 1 : 0;
}

__global__ void __launch_bounds__(32 * kFTWarps, 12)
    from_text_warp_kernel(const char* __restrict__ text, const uint64_t* __restrict__ off,
                          uint64_t n, ranmar_state* __restrict__ out, int32_t* __restrict__ err) {
    __shared__ __align__(16) char stage[kFTWarps][kFTCap + 32];
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
    const uint64_t a0 = b & ~uint64_t(15);
    const int sh = static_cast<int>(b - a0);
    const int chunks = (sh + L + 15) >> 4;
    {   // aligned 16-B chunks covering [b, e); byte shift = b & 15
        const uint4* src = reinterpret_cast<const uint4*>(text + a0);
        for (int q = l; q < chunks; q += 32) reinterpret_cast<uint4*>(sm)[q] = src[q];
        __syncwarp();
    }
    // newlines, in order: lane l tests 16-B chunk 32 r + l (one LDS.128 and a
    // SWAR byte test), a warp scan of the counts places them
    int total_nl = 0;
    for (int c0 = 0; c0 < chunks; c0 += 32) {
        const int c = c0 + l;
        uint32_t m = 0;
        if (c < chunks) {
            m = nl_mask16(reinterpret_cast<const uint4*>(sm)[c]);
            const int lo = sh - 16 * c, hi = sh + L - 16 * c;  // the text's bytes [lo, hi) of the chunk
            if (lo > 0) m &= ~((1u << lo) - 1u);
            if (hi < 16) m &= (1u << hi) - 1u;
        }
        const int cnt = __popc(m);
        int x = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (l >= o) x += y;
        }
        int pos = total_nl + x - cnt;
        while (m) {
            const int bit = __ffs(m) - 1;
            if (pos < kFTLines) nl[w][pos] = 16 * c + bit - sh;
            ++pos;
            m &= m - 1;
        }
        total_nl += __shfl_sync(0xffffffffu, x, 31);
    }
    const uint32_t* S = reinterpret_cast<const uint32_t*>(sm);  // word view of the stage
    sm += sh;  // sm[0 .. L) is the text
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
            if (ln == 1) {  // "ranmar24 v1", compared as two words
                uint64_t lo, hi;
                load16(S, sh + p, lo, hi);
                ok = en - p == 11 && lo == 0x343272616D6E6172ull && (hi & 0xFFFFFFull) == 0x317620ull;
            } else if (ln == 3) {
                uint32_t fv;
                if (parse_num_fast(S, sh + p, en - p, 0x2076ull, 2, fv)) {  // canonical "v <x>"
                    ok = fv < kMod;
                    sv = fv;
                } else {
                    uint64_t v = 0;
                    ok = en - p >= 2 && sm[p] == 'v' && sm[p + 1] == ' ';
                    p += 2;
                    ok = ok && num_at(sm, p, en, v) && p == en && v < kMod;
                    sv = static_cast<uint32_t>(v);
                }
            } else if (ln == 2) {
                uint64_t i = 0, j = 0;
                if (!parse_ij_fast(S, sh + p, en - p, i, j)) {
                    ok = en - p >= 2 && sm[p] == 'i' && sm[p + 1] == ' ';
                    p += 2;
                    ok = ok && num_at(sm, p, en, i);
                    ok = ok && en - p >= 3 && sm[p] == ' ' && sm[p + 1] == 'j' && sm[p + 2] == ' ';
                    p += 3;
                    ok = ok && num_at(sm, p, en, j) && p == en;
                }
                ok = ok && i >= 1 && i <= 97 && j >= 1 && j <= 97 && (i + 97 - j) % 97 == 64;
                si = static_cast<int32_t>(i) - 1;
                sj = static_cast<int32_t>(j) - 1;
            } else {
                uint32_t fl;
                const int f = parse_u_fast(S, sh + p, en - p, static_cast<uint32_t>(ln - 3), fl);
                if (f >= 0) {
                    vals[r] = fl;
                    if (f == 0 && ln < bad) bad = ln;
                    continue;
                }
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

static uint64_t text_tiles(uint64_t n) { return (n + kTTStates - 1) / kTTStates; }

// tile status words + the ticket counter
size_t text_workspace(uint64_t n) { return static_cast<size_t>((text_tiles(n) + 1) * sizeof(uint64_t)); }

// Offsets d_off[0..n] (d_off[n] = total bytes) and the concatenated texts:
// one memset of the look-back workspace and one kernel.
cudaError_t launch_to_text(const ranmar_state* d_states, uint64_t n, char* d_text,
                           uint64_t* d_off, void* d_ws, uint32_t* status, cudaStream_t stream) {
    const uint64_t tiles = text_tiles(n);
    if (tiles > 0x7FFFFFFFull) return cudaErrorInvalidValue;
    uint64_t* tile_status = static_cast<uint64_t*>(d_ws);
    cudaError_t e = cudaMemsetAsync(d_ws, 0, text_workspace(n), stream);
    if (e != cudaSuccess) return e;
    count_launch();
    to_text_kernel<<<static_cast<unsigned>(tiles), 32 * kTTStates, 0, stream>>>(
        d_states, n, d_off, d_text, tile_status, reinterpret_cast<uint32_t*>(tile_status + tiles), status);
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
