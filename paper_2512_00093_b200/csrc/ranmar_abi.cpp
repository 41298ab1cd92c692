// Host runtime behind the C ABI (include/ranmar_b200.h): argument checking
// with the reference's error semantics, 256-bit jump-count arithmetic, the
// stream-range planner for make_streams, kernel orchestration on the caller's
// stream, and the host-buffer (ctx) pipeline. No compute of the hot path runs
// here: generation and jumps are the sm_100a kernels in gen_kernels.cu and
// jump_kernels.cu. The only host arithmetic is the cold seed expansion
// (init.hpp:18-51, ~15 us), closed-form residues mod m, and text persistence.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>
#include <initializer_list>

#include "ranmar_b200.h"

namespace rb {
struct PowJob {
    uint64_t e[4];
    int extra;
    uint32_t* out;
};
struct PowJobs {
    PowJob job[2];
};
template <class T>
cudaError_t launch_generate(ranmar_state*, uint64_t, uint64_t, T*, uint32_t*, cudaStream_t);
cudaError_t launch_consume(ranmar_state*, uint64_t, uint64_t, uint64_t*, uint32_t*, uint32_t*,
                           cudaStream_t);
cudaError_t launch_gaussian_stream(ranmar_gauss_state*, uint64_t, uint64_t, double*, uint32_t*,
                                   cudaStream_t);
cudaError_t launch_float_gen(ranmar_float_state*, uint64_t, uint64_t, double*, double*, double*,
                             uint32_t*, cudaStream_t);
cudaError_t launch_generate_trace(ranmar_state*, uint64_t, uint64_t, uint32_t*, uint32_t*, uint32_t*,
                                  uint32_t*, cudaStream_t);
cudaError_t launch_float_from_states(const ranmar_state*, uint64_t, ranmar_float_state*, cudaStream_t);
cudaError_t launch_poly(int, const uint32_t*, const uint32_t*, uint32_t*, uint64_t, cudaStream_t);
uint64_t text_bound(uint64_t);
size_t text_workspace(uint64_t);
cudaError_t launch_to_text(const ranmar_state*, uint64_t, char*, uint64_t*, void*, uint32_t*,
                           cudaStream_t);
cudaError_t launch_from_text(const char*, const uint64_t*, uint64_t, ranmar_state*, int32_t*,
                             cudaStream_t);
cudaError_t launch_gaussian_moments(ranmar_gauss_state*, uint64_t, uint64_t, double*, uint32_t*, cudaStream_t);
cudaError_t launch_gaussian(ranmar_gauss_state*, uint64_t, uint64_t, uint64_t, double*, uint32_t*,
                            cudaStream_t);
cudaError_t launch_langevin(ranmar_gauss_state*, uint64_t, const double*, double*, const int32_t*,
                            const int32_t*, int32_t, const double*, const double*, int32_t, double,
                            int, uint32_t*, cudaStream_t);
cudaError_t launch_langevin_noise(uint64_t, const double*, const double*, double*, const int32_t*,
                                  const int32_t*, int32_t, const double*, const double*, int32_t,
                                  double, uint32_t*, cudaStream_t);
cudaError_t launch_bank_from_states(const ranmar_state*, uint64_t, uint32_t*, uint32_t*,
                                   cudaStream_t);
cudaError_t launch_bank_to_states(const uint32_t*, uint64_t, uint64_t, ranmar_state*, cudaStream_t);
cudaError_t launch_langevin_bank(uint32_t*, uint64_t, uint64_t, const double*, double*,
                                 const int32_t*, const double*, const double*, int32_t, double,
                                 uint32_t*, cudaStream_t);
template <class T>
cudaError_t launch_generate_joined(ranmar_state*, uint64_t, uint64_t, uint64_t, T*, ranmar_state*, int,
                                   uint32_t*, cudaStream_t);
cudaError_t launch_fp64_selfcheck(uint64_t, uint64_t, unsigned long long*, cudaStream_t);
cudaError_t launch_crlog_sweep(uint64_t, uint64_t, int, unsigned long long*, uint64_t*, uint64_t,
                               cudaStream_t);
cudaError_t launch_pow(const PowJobs&, int, cudaStream_t);
cudaError_t launch_pow_table(const uint64_t (*)[4], const int*, uint32_t* const*, int,
                             const uint32_t*, cudaStream_t);
cudaError_t launch_tables(const uint32_t*, int, uint32_t*, uint32_t*, const ranmar_state*,
                          const ranmar_state*, ranmar_state*, uint32_t*, cudaStream_t);
cudaError_t launch_apply(const ranmar_state*, ranmar_state*, uint64_t, const uint32_t*, uint32_t,
                         uint32_t*, int, cudaStream_t);
cudaError_t launch_level(const ranmar_state*, uint64_t, const uint32_t*, uint32_t, ranmar_state*,
                         uint32_t*, uint32_t*, cudaStream_t);
cudaError_t launch_level_tc(const uint32_t*, uint64_t, const uint32_t*, uint64_t, uint32_t,
                            const ranmar_state*, uint32_t*, uint32_t*, uint32_t*, int, cudaStream_t);
cudaError_t launch_bulk(const uint32_t*, uint64_t, const uint32_t*, ranmar_state*, uint64_t,
                        uint64_t, uint32_t, const ranmar_state*, uint32_t*, int, cudaStream_t);
cudaError_t configure_jump_kernels();
cudaError_t configure_consume_kernel();
std::atomic<uint64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(static_cast<uint64_t>(n), std::memory_order_relaxed); }
}  // namespace rb

namespace {

constexpr uint32_t kMask = 0x00FFFFFFu;
constexpr uint32_t kMod = 16777213u;
constexpr uint32_t kDelta = 7654321u;
constexpr uint32_t kStart = 362436u;
constexpr uint32_t kMaxSeed = 900000000u;
constexpr int kRows = 128;      // must match jump_kernels.cu
constexpr int kPolyN = 97;
constexpr int kWAnchor = 196;   // words per anchor extension row (jump_kernels.cu)
constexpr int kSquares = 320;   // Z_k = t^(2^k), k < 320 (exponents < 2^256, shifts < 64)
constexpr int kMaxLevels = 10;  // 128^9 = 2^63 streams
constexpr int kMaxPlanPows = 7 * kMaxLevels + 1;

static_assert(sizeof(ranmar_state) == 400, "ranmar_state must be the 400-B RanmarState");
static_assert(sizeof(ranmar_gauss_state) == 416, "ranmar_gauss_state layout");

thread_local std::string g_error;

int fail(int code, const std::string& msg) {
    g_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(RANMAR_ECUDA, std::string("ranmar: ") + what + ": " + cudaGetErrorString(e));
}

#define RB_CUDA(call, what)                          \
    do {                                             \
        cudaError_t e_ = (call);                     \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

// ---- 256-bit jump counts ------------------------------------------------
struct U256 {
    uint64_t w[4];
};

U256 from_abi(const ranmar_jump_count* j) {
    U256 r;
    std::memcpy(r.w, j->limb, sizeof r.w);
    return r;
}
bool is_zero(const U256& a) { return (a.w[0] | a.w[1] | a.w[2] | a.w[3]) == 0; }
uint32_t mod_u32(const U256& a, uint32_t m) {
    unsigned __int128 r = 0;
    for (int k = 3; k >= 0; --k) r = ((r << 64) | a.w[k]) % m;
    return static_cast<uint32_t>(r);
}
// a * k; returns false on overflow past 256 bits.
bool mul_u64(const U256& a, uint64_t k, U256* out) {
    unsigned __int128 carry = 0;
    U256 r;
    for (int i = 0; i < 4; ++i) {
        const unsigned __int128 p = static_cast<unsigned __int128>(a.w[i]) * k + carry;
        r.w[i] = static_cast<uint64_t>(p);
        carry = p >> 64;
    }
    *out = r;
    return carry == 0;
}
uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) {
    return static_cast<uint64_t>(static_cast<unsigned __int128>(a) * b % m);
}
// (J mod m) * d mod m: the per-jump decrement of the arithmetic part (jump.hpp:82-84).
uint32_t arith_dec(uint32_t jm) { return static_cast<uint32_t>(mulmod(jm, kDelta, kMod)); }

// ---- per-device resources -------------------------------------------------
// Built once per device by ranmar_device_setup (the only entry point besides
// the ctx_* pipeline that allocates or synchronises): the sticky status word,
// the SM count, and the table of squares Z_k = t^(2^k) mod phi (k < kSquares),
// the squaring half of square-and-multiply, independent of any J, built by
// pow_kernel's squaring chain. The _dev entry points only read them, so they
// never allocate or synchronise and can be captured in a CUDA graph.
struct DevRes {
    uint32_t* status = nullptr;
    uint32_t* squares = nullptr;
    int sms = 0;
};
std::mutex g_dev_mu;
DevRes g_res[64];
std::atomic<bool> g_ready[64];

int current_res(const DevRes** out) {
    int dev = 0;
    RB_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    if (dev < 0 || dev >= 64) return fail(RANMAR_ECUDA, "ranmar: device index out of range");
    if (!g_ready[dev].load(std::memory_order_acquire))
        return fail(RANMAR_ESTATE, "ranmar: device " + std::to_string(dev) +
                                       " is not set up: call ranmar_device_setup(" +
                                       std::to_string(dev) + ", stream) once first");
    *out = &g_res[dev];
    return RANMAR_OK;
}

// ctx_* calls route the kernels' status bits to their context's own word
thread_local uint32_t* g_status_override = nullptr;

int device_status_ptr(uint32_t** out, int* sms) {
    const DevRes* r = nullptr;
    if (int rc = current_res(&r)) return rc;
    *out = g_status_override ? g_status_override : r->status;
    if (sms) *sms = r->sms;
    return RANMAR_OK;
}

int square_table(const uint32_t** out) {
    const DevRes* r = nullptr;
    if (int rc = current_res(&r)) return rc;
    *out = r->squares;
    return RANMAR_OK;
}

// Makes `device` current for a scope and restores the caller's device after.
class DeviceGuard {
  public:
    cudaError_t enter(int device) {
        cudaError_t e = cudaGetDevice(&prev_);
        if (e != cudaSuccess) {
            prev_ = -1;
            return e;
        }
        return prev_ == device ? cudaSuccess : cudaSetDevice(device);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev_ >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev_) cudaSetDevice(prev_);
    }

  private:
    int prev_ = -1;
};

// ---- make_streams workspace plan -----------------------------------------
// Stream starts form a base-128 tree: level L holds count[L] = ceil(n / 128^L)
// states spaced 128^L J apart; the top level (128^top >= n) is the single
// state s_{first J}. Level 1 is kept as 193-word extensions for the bulk.
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Plan {
    int top;         // 128^top >= n, top >= 2
    int tab_levels;  // tables Tab_0 .. Tab_{top-1}
    uint64_t count[kMaxLevels];
    size_t off_q, off_pfirst, off_tab, off_tt, off_a0, off_base, off_w1, off_v1;
    size_t off_lvl[kMaxLevels];
    size_t total;
};

Plan plan_for(uint64_t n) {
    Plan p{};
    p.top = 1;
    for (unsigned __int128 span = kRows; span < n; span *= kRows) ++p.top;
    if (p.top < 2) p.top = 2;
    p.tab_levels = p.top;
    unsigned __int128 span = 1;
    for (int L = 0; L < p.top; ++L, span *= kRows)
        p.count[L] = static_cast<uint64_t>((n + span - 1) / span);
    size_t o = 0;
    p.off_q = o;
    o = align256(o + size_t(7 * p.tab_levels) * kPolyN * 4);
    p.off_pfirst = o;
    o = align256(o + kPolyN * 4);
    p.off_tab = o;
    o = align256(o + size_t(p.tab_levels) * kRows * kPolyN * 4);
    p.off_tt = o;  // Tab_0 and Tab_1 transposed (the tensor-core kernels' coalesced loads)
    o = align256(o + 2 * size_t(kPolyN) * kRows * 4);
    p.off_a0 = o;
    o = align256(o + sizeof(ranmar_state));
    p.off_base = o;
    o = align256(o + sizeof(ranmar_state));
    p.off_w1 = o;
    o = align256(o + size_t(p.count[1]) * kWAnchor * 4);
    p.off_v1 = o;
    o = align256(o + size_t(p.count[1]) * 4);
    for (int L = 2; L < p.top; ++L) {  // level 2 as extension rows (level 1's anchors), above as states
        p.off_lvl[L] = o;
        o = align256(o + size_t(p.count[L]) * (L == 2 ? kWAnchor * 4 : sizeof(ranmar_state)));
    }
    p.total = o;
    return p;
}

void seed_expand(uint32_t seed, ranmar_state* out) {
    // init.hpp:22-49 (signed split with C++ truncation; Remainder form of the mixer).
    const int ij = (static_cast<int>(seed) - 1) / 30082;
    const int kl = (static_cast<int>(seed) - 1) - 30082 * ij;
    int ii = (ij / 177) % 177 + 2, jj = ij % 177 + 2, kk = (kl / 169) % 178 + 1, ll = kl % 169;
    std::memset(out, 0, sizeof *out);
    for (int lane = 0; lane < 97; ++lane) {
        uint32_t acc = 0, t = 1u << 31;
        for (int bit = 0; bit < 24; ++bit) {
            const int mm = ((ii * jj) % 179) * kk % 179;
            ii = jj;
            jj = kk;
            kk = mm;
            ll = (53 * ll + 1) % 169;
            if ((ll * mm) % 64 >= 32) acc += t;
            t >>= 1;
        }
        out->lane[lane] = acc >> 8;
    }
    out->i = 96;
    out->j = 32;
    out->v = kStart;
}

// The reference's invariants of RanmarState (core.hpp:29-49): 24-bit lanes,
// 0-based cursors with (i - j) mod 97 = 64, v < m.
bool host_state_ok(const ranmar_state& s) {
    if (!(s.i >= 0 && s.i < 97 && s.j >= 0 && s.j < 97 && (s.i - s.j + 97) % 97 == 64 && s.v < kMod))
        return false;
    for (int k = 0; k < 97; ++k)
        if (s.lane[k] > kMask) return false;
    return true;
}

}  // namespace

// =========================================================================
extern "C" {

int ranmar_abi_version(void) { return RANMAR_ABI_VERSION; }

int ranmar_device_setup(int device, void* stream) {
    int count = 0;
    RB_CUDA(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (device < 0 || device >= count || device >= 64)
        return fail(RANMAR_ECUDA, "ranmar: no such CUDA device");
    if (g_ready[device].load(std::memory_order_acquire)) return RANMAR_OK;
    DeviceGuard guard;
    RB_CUDA(guard.enter(device), "cudaSetDevice");
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (g_ready[device].load(std::memory_order_relaxed)) return RANMAR_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DevRes r;
    RB_CUDA(cudaDeviceGetAttribute(&r.sms, cudaDevAttrMultiProcessorCount, device),
            "cudaDeviceGetAttribute");
    RB_CUDA(cudaMalloc(&r.status, 256), "cudaMalloc(status)");
    RB_CUDA(cudaMemsetAsync(r.status, 0, 256, s), "cudaMemset(status)");
    RB_CUDA(cudaMalloc(&r.squares, size_t(kSquares) * kPolyN * 4), "cudaMalloc(squares)");
    rb::PowJobs jobs{};
    jobs.job[0].e[0] = 1;  // t^1, then kSquares - 1 squarings
    jobs.job[0].extra = kSquares - 1;
    jobs.job[0].out = r.squares;
    RB_CUDA(rb::launch_pow(jobs, 1, s), "pow_kernel launch (square table)");
    RB_CUDA(cudaStreamSynchronize(s), "square table build");
    RB_CUDA(rb::configure_jump_kernels(), "cudaFuncSetAttribute (jump kernels)");
    RB_CUDA(rb::configure_consume_kernel(), "cudaFuncSetAttribute (consume kernel)");
    g_res[device] = r;
    g_ready[device].store(true, std::memory_order_release);
    return RANMAR_OK;
}
uint64_t ranmar_kernel_launches(void) { return rb::g_launches.load(); }
const char* ranmar_last_error(void) { return g_error.c_str(); }

int ranmar_init(uint32_t seed, ranmar_state* out) {
    if (!out) return fail(RANMAR_EINVAL, "ranmar: null output");
    if (seed > kMaxSeed) return fail(RANMAR_EINVAL, "ranmar: seed must be in [0, 900000000]");
    seed_expand(seed, out);
    return RANMAR_OK;
}

int ranmar_init_unchecked(uint32_t seed, ranmar_state* out) {
    if (!out) return fail(RANMAR_EINVAL, "ranmar: null output");
    seed_expand(seed, out);
    return RANMAR_OK;
}

int ranmar_value_of(uint32_t u24, double* out) {
    if (u24 > kMask) return fail(RANMAR_EINVAL, "ranmar: value_of argument exceeds 24 bits");
    *out = static_cast<double>(u24) * 0x1p-24;
    return RANMAR_OK;
}

int ranmar_parse_jump_count(const char* text, ranmar_jump_count* out) {
    // jumpcount.hpp:16-47: decimal, "2^k", "2^k-1", "2^k+1" (k <= 10^6 there).
    std::memset(out, 0, sizeof *out);
    const std::string bad = std::string("ranmar: bad jump count \"") + (text ? text : "") +
                            "\" (want decimal, 2^k, 2^k-1, or 2^k+1)";
    if (!text || !*text) return fail(RANMAR_EINVAL, bad);
    if (text[0] == '2' && text[1] == '^') {
        const char* p = text + 2;
        unsigned long k = 0;
        int nd = 0;
        while (*p >= '0' && *p <= '9') {
            k = k * 10 + static_cast<unsigned long>(*p - '0');
            if (k > 1000000) return fail(RANMAR_EINVAL, "ranmar: jump exponent too large");
            ++p;
            ++nd;
        }
        if (nd == 0) return fail(RANMAR_EINVAL, bad);
        int delta = 0;
        if (std::strcmp(p, "-1") == 0) delta = -1;
        else if (std::strcmp(p, "+1") == 0) delta = 1;
        else if (*p) return fail(RANMAR_EINVAL, bad);
        if (k > 256 || (k == 256 && delta >= 0))
            return fail(RANMAR_ERANGE, "ranmar: jump count exceeds 2^256 - 1");
        if (k < 256) out->limb[k / 64] = uint64_t(1) << (k % 64);
        if (delta == 1) {
            for (int w = 0; w < 4; ++w)
                if (++out->limb[w] != 0) break;
        } else if (delta == -1) {
            for (int w = 0; w < 4; ++w)
                if (out->limb[w]-- != 0) break;
        }
        return RANMAR_OK;
    }
    for (const char* p = text; *p; ++p)
        if (*p < '0' || *p > '9') return fail(RANMAR_EINVAL, bad);
    U256 acc{};
    for (const char* p = text; *p; ++p) {
        U256 t;
        if (!mul_u64(acc, 10, &t)) return fail(RANMAR_ERANGE, "ranmar: jump count exceeds 2^256 - 1");
        unsigned __int128 carry = static_cast<unsigned>(*p - '0');
        for (int w = 0; w < 4; ++w) {
            const unsigned __int128 s = static_cast<unsigned __int128>(t.w[w]) + carry;
            t.w[w] = static_cast<uint64_t>(s);
            carry = s >> 64;
        }
        if (carry) return fail(RANMAR_ERANGE, "ranmar: jump count exceeds 2^256 - 1");
        acc = t;
    }
    std::memcpy(out->limb, acc.w, sizeof acc.w);
    return RANMAR_OK;
}

int ranmar_jump_arith(uint32_t v, const ranmar_jump_count* j, uint32_t* out) {
    if (!j || !out) return fail(RANMAR_EINVAL, "ranmar: null argument");
    const uint32_t dec = arith_dec(mod_u32(from_abi(j), kMod));
    *out = static_cast<uint32_t>((uint64_t(v) + (kMod - dec)) % kMod);
    return RANMAR_OK;
}

long ranmar_to_text(const ranmar_state* s, char* buf, long cap) {
    // serialize.hpp:21-40
    std::string out = "ranmar24 v1\ni " + std::to_string(s->i + 1) + " j " +
                      std::to_string(s->j + 1) + "\nv " + std::to_string(s->v) + "\n";
    for (int k = 0; k < 97; ++k)
        out += "u " + std::to_string(k + 1) + " " + std::to_string(s->lane[k]) + "\n";
    if (static_cast<long>(out.size()) + 1 > cap) return -1;
    std::memcpy(buf, out.c_str(), out.size() + 1);
    return static_cast<long>(out.size());
}

int ranmar_from_text(const char* text, ranmar_state* out) {
    // serialize.hpp:81-136: strict, line-based; EINVAL with the line number.
    int line = 1;
    const char* t = text ? text : "";
    auto perr = [&](const std::string& what) {
        return fail(RANMAR_EINVAL,
                    "ranmar: state parse error at line " + std::to_string(line) + ": " + what);
    };
    auto next_line = [&](std::string& l) -> bool {
        if (!*t) return false;
        const char* nl = std::strchr(t, '\n');
        size_t n = nl ? size_t(nl - t) : std::strlen(t);
        l.assign(t, n);
        t = nl ? nl + 1 : t + n;
        if (!l.empty() && l.back() == '\r') l.pop_back();
        return true;
    };
    auto take_uint = [&](const std::string& l, size_t& pos, uint64_t& v) -> bool {
        v = 0;
        size_t n = 0;
        while (pos < l.size() && l[pos] >= '0' && l[pos] <= '9') {
            v = v * 10 + uint64_t(l[pos] - '0');
            if (v > 0xFFFFFFFFull) return false;
            ++pos;
            ++n;
        }
        return n > 0;
    };
    auto take_lit = [&](const std::string& l, size_t& pos, const char* lit) -> bool {
        const size_t n = std::strlen(lit);
        if (l.compare(pos, n, lit) != 0) return false;
        pos += n;
        return true;
    };
    std::string l;
    if (!next_line(l)) return perr("unexpected end of input");
    if (l != "ranmar24 v1") return perr("bad magic (want \"ranmar24 v1\")");
    ranmar_state s{};
    ++line;
    if (!next_line(l)) return perr("unexpected end of input");
    size_t pos = 0;
    uint64_t i = 0, j = 0, v = 0;
    if (!take_lit(l, pos, "i ")) return perr("expected \"i \"");
    if (!take_uint(l, pos, i)) return perr("expected a decimal number");
    if (!take_lit(l, pos, " j ")) return perr("expected \" j \"");
    if (!take_uint(l, pos, j)) return perr("expected a decimal number");
    if (pos != l.size()) return perr("trailing characters");
    if (i < 1 || i > 97 || j < 1 || j > 97) return perr("cursor out of range");
    if ((i + 97 - j) % 97 != 64) return perr("cursor separation must be 64");
    s.i = int32_t(i) - 1;
    s.j = int32_t(j) - 1;
    ++line;
    if (!next_line(l)) return perr("unexpected end of input");
    pos = 0;
    if (!take_lit(l, pos, "v ")) return perr("expected \"v \"");
    if (!take_uint(l, pos, v)) return perr("expected a decimal number");
    if (pos != l.size()) return perr("trailing characters");
    if (v >= kMod) return perr("v must be < 16777213");
    s.v = uint32_t(v);
    for (int k = 0; k < 97; ++k) {
        ++line;
        if (!next_line(l)) return perr("unexpected end of input");
        pos = 0;
        uint64_t idx = 0, lane = 0;
        if (!take_lit(l, pos, "u ")) return perr("expected \"u \"");
        if (!take_uint(l, pos, idx)) return perr("expected a decimal number");
        if (!take_lit(l, pos, " ")) return perr("expected \" \"");
        if (!take_uint(l, pos, lane)) return perr("expected a decimal number");
        if (pos != l.size()) return perr("trailing characters");
        if (idx != uint64_t(k) + 1) return perr("lane index out of order");
        if (lane > kMask) return perr("lane value exceeds 24 bits");
        s.lane[k] = uint32_t(lane);
    }
    for (; *t; ++t)
        if (*t != '\n' && *t != '\r' && *t != ' ' && *t != '\t') {
            ++line;
            return perr("trailing content after state");
        }
    *out = s;
    return RANMAR_OK;
}

// ---------------------------------------------------------------- device

size_t ranmar_make_streams_workspace(uint64_t n) { return plan_for(n ? n : 1).total; }

int ranmar_pow_t_mod_dev(const ranmar_jump_count* j, uint32_t* d_coeff, void* stream) {
    if (!j || !d_coeff) return fail(RANMAR_EINVAL, "ranmar: null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint32_t* Z = nullptr;
    if (int rc = square_table(&Z)) return rc;
    const uint64_t(*e)[4] = &j->limb;
    const int shift = 0;
    uint32_t* out = d_coeff;
    RB_CUDA(rb::launch_pow_table(e, &shift, &out, 1, Z, s), "pow_table_kernel launch");
    return RANMAR_OK;
}

int ranmar_jump_dev(const ranmar_state* d_in, ranmar_state* d_out, uint64_t n,
                    const ranmar_jump_count* j, void* d_ws, size_t ws_bytes, void* stream) {
    if (!j) return fail(RANMAR_EINVAL, "ranmar: null jump count");
    if (n == 0) return RANMAR_OK;
    if (!d_in || !d_out || !d_ws) return fail(RANMAR_EINVAL, "ranmar: null argument");
    if (ws_bytes < kPolyN * 4) return fail(RANMAR_ENOMEM, "ranmar: workspace too small");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint32_t* P = static_cast<uint32_t*>(d_ws);
    int rc = ranmar_pow_t_mod_dev(j, P, stream);
    if (rc) return rc;
    const uint32_t dec = arith_dec(mod_u32(from_abi(j), kMod));
    uint32_t* status = nullptr;
    int sms = 148;
    if (int rc2 = device_status_ptr(&status, &sms)) return rc2;
    RB_CUDA(rb::launch_apply(d_in, d_out, n, P, dec, status, sms, s), "apply_kernel launch");
    return RANMAR_OK;
}

}  // extern "C"

namespace {

// make_streams for a base state given on the host (h_base, checked here) or in
// device memory (d_base, checked by tables_kernel, which flags the status
// word): exactly one of them is non-null.
int make_streams_impl(const ranmar_state* h_base, const ranmar_state* d_base,
                      const ranmar_jump_count* j, uint64_t first, uint64_t n, ranmar_state* d_out,
                      void* d_ws, size_t ws_bytes, void* stream) {
    if (!j) return fail(RANMAR_EINVAL, "ranmar: null argument");
    if (n == 0) return fail(RANMAR_EINVAL, "ranmar: need at least one stream");  // jump.hpp:111
    const U256 J = from_abi(j);
    if (is_zero(J)) return fail(RANMAR_EINVAL, "ranmar: block length must be >= 1");  // :112
    if (h_base && !host_state_ok(*h_base))
        return fail(RANMAR_ESTATE, "ranmar: base state violates cursor/residue invariants");
    if (first >= (uint64_t(1) << 62) || n >= (uint64_t(1) << 62) || first + n >= (uint64_t(1) << 62))
        return fail(RANMAR_ERANGE, "ranmar: stream range too large");
    const Plan p = plan_for(n);
    if (!d_out || !d_ws) return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    if (ws_bytes < p.total) return fail(RANMAR_ENOMEM, "ranmar: workspace too small");
    U256 fj;
    if (!mul_u64(J, first, &fj)) return fail(RANMAR_ERANGE, "ranmar: first * J exceeds 2^256");
    {   // every stream start (first + n - 1) * J must be representable too
        U256 lastj;
        if (!mul_u64(J, first + n - 1, &lastj))
            return fail(RANMAR_ERANGE, "ranmar: (first + n - 1) * J exceeds 2^256");
    }
    int sms = 148;
    uint32_t* status = nullptr;
    if (int rc = device_status_ptr(&status, &sms)) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint32_t* Z = nullptr;
    if (int rc = square_table(&Z)) return rc;
    char* ws = static_cast<char*>(d_ws);
    uint32_t* Q = reinterpret_cast<uint32_t*>(ws + p.off_q);
    uint32_t* Pf = reinterpret_cast<uint32_t*>(ws + p.off_pfirst);
    uint32_t* Tab = reinterpret_cast<uint32_t*>(ws + p.off_tab);
    uint32_t* Tt = reinterpret_cast<uint32_t*>(ws + p.off_tt);
    ranmar_state* A0 = reinterpret_cast<ranmar_state*>(ws + p.off_a0);
    ranmar_state* dbase = reinterpret_cast<ranmar_state*>(ws + p.off_base);
    uint32_t* W1 = reinterpret_cast<uint32_t*>(ws + p.off_w1);
    uint32_t* V1 = reinterpret_cast<uint32_t*>(ws + p.off_v1);

    // K3a: Q_b = P_{2^b J} = prod_{k in bits(J)} Z_{k+b} for b < 7 * levels and,
    // if first > 0, P_{first J}; all independent, one launch. When J = 2^k (the
    // usual block length, configs 2-5) Q_b = Z_{k+b} are consecutive rows of the
    // square table and are read in place: no launch.
    int jbit = -1, jpop = 0;
    for (int k = 0; k < 256; ++k)
        if ((J.w[k >> 6] >> (k & 63)) & 1u) {
            jbit = k;
            ++jpop;
        }
    const bool q_in_table = jpop == 1 && jbit + 7 * p.tab_levels <= kSquares;
    const uint32_t* Qsrc = q_in_table ? Z + size_t(jbit) * kPolyN : Q;
    uint64_t e[kMaxPlanPows][4];
    int shift[kMaxPlanPows];
    uint32_t* outs[kMaxPlanPows];
    int njobs = 0;
    for (int b = 0; !q_in_table && b < 7 * p.tab_levels; ++b, ++njobs) {
        std::memcpy(e[njobs], J.w, sizeof J.w);
        shift[njobs] = b;
        outs[njobs] = Q + size_t(b) * kPolyN;
    }
    if (first > 0) {
        std::memcpy(e[njobs], fj.w, sizeof fj.w);
        shift[njobs] = 0;
        outs[njobs] = Pf;
        ++njobs;
    }
    if (njobs) RB_CUDA(rb::launch_pow_table(e, shift, outs, njobs, Z, s), "pow_table_kernel launch");
    // Offset tables Tab_L[r] = P_{r 128^L J}.
    // (a host-given base state rides along as a kernel parameter and is written
    // into the workspace by the same launch)
    // The base state goes into the workspace with the same launch (a device-resident
    // one checked there); A_0 = s_{first J}.
    RB_CUDA(rb::launch_tables(Qsrc, p.tab_levels, Tab, Tt, h_base, d_base, dbase, status, s),
            "tables_kernel launch");
    const uint32_t jm = mod_u32(J, kMod);
    const ranmar_state* a0 = dbase;
    if (first > 0) {
        const uint32_t dec = arith_dec(static_cast<uint32_t>(mulmod(first % kMod, jm, kMod)));
        RB_CUDA(rb::launch_apply(dbase, A0, 1, Pf, dec, status, sms, s), "apply_kernel launch");
        a0 = A0;
    }
    // Levels L-1 .. 1 of the base-128 tree (level 1 writes the anchors'
    // extensions for the bulk kernel), then level 0.
    // With three or more levels, level 2 is written as extension rows and level 1
    // (up to 2^14 x 128 rows) runs on the tensor cores like level 0.
    const ranmar_state* in = a0;
    const uint32_t* w2 = nullptr;
    for (int L = p.top - 1; L >= 1; --L) {
        uint64_t pw = 1;  // 128^L mod m
        for (int x = 0; x < L; ++x) pw = pw * 128 % kMod;
        const uint32_t c_lvl = static_cast<uint32_t>(mulmod(pw, jm, kMod));
        const uint64_t count = p.count[L];
        const uint32_t* tab = Tab + size_t(L) * kRows * kPolyN;
        if (L == 1 && w2) {
            RB_CUDA(rb::launch_level_tc(w2, p.count[2], Tt + size_t(kPolyN) * kRows, count, c_lvl, a0, W1, V1, status, sms, s),
                    "level_tc launch");
        } else if (L == 1) {
            RB_CUDA(rb::launch_level(in, count, tab, c_lvl, nullptr, W1, V1, s), "level launch");
        } else if (L == 2) {
            uint32_t* o = reinterpret_cast<uint32_t*>(ws + p.off_lvl[L]);
            RB_CUDA(rb::launch_level(in, count, tab, c_lvl, nullptr, o, V1, s), "level launch");
            w2 = o;  // (its v row is rewritten by level 1)
        } else {
            ranmar_state* o = reinterpret_cast<ranmar_state*>(ws + p.off_lvl[L]);
            RB_CUDA(rb::launch_level(in, count, tab, c_lvl, o, nullptr, nullptr, s), "level launch");
            in = o;
        }
    }
    RB_CUDA(rb::launch_bulk(W1, p.count[1], Tt, d_out, first, n, jm, dbase, status, sms, s),
            "bulk_kernel launch");
    return RANMAR_OK;
}

}  // namespace

extern "C" {

int ranmar_make_streams_dev(const ranmar_state* base, const ranmar_jump_count* j, uint64_t first,
                            uint64_t n, ranmar_state* d_out, void* d_ws, size_t ws_bytes,
                            void* stream) {
    if (!base) return fail(RANMAR_EINVAL, "ranmar: null argument");
    return make_streams_impl(base, nullptr, j, first, n, d_out, d_ws, ws_bytes, stream);
}

int ranmar_make_streams_from_dev(const ranmar_state* d_base, const ranmar_jump_count* j,
                                 uint64_t first, uint64_t n, ranmar_state* d_out, void* d_ws,
                                 size_t ws_bytes, void* stream) {
    if (!d_base) return fail(RANMAR_EINVAL, "ranmar: null argument");
    return make_streams_impl(nullptr, d_base, j, first, n, d_out, d_ws, ws_bytes, stream);
}

#define RB_STATUS_PTR(var)                               \
    uint32_t* var = nullptr;                             \
    if (int rc_ = device_status_ptr(&var, nullptr)) return rc_

int ranmar_generate_u32_dev(ranmar_state* d_states, uint64_t n_streams, uint64_t per_stream,
                            uint32_t* d_out, void* stream) {
    if (n_streams && (!d_states || (per_stream && !d_out)))
        return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    RB_STATUS_PTR(status);
    RB_CUDA(rb::launch_generate<uint32_t>(d_states, n_streams, per_stream, d_out, status,
                                          static_cast<cudaStream_t>(stream)),
            "gen_store_kernel<u32> launch");
    return RANMAR_OK;
}

int ranmar_generate_f32_dev(ranmar_state* d_states, uint64_t n_streams, uint64_t per_stream,
                            float* d_out, void* stream) {
    if (n_streams && (!d_states || (per_stream && !d_out)))
        return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    RB_STATUS_PTR(status);
    RB_CUDA(rb::launch_generate<float>(d_states, n_streams, per_stream, d_out, status,
                                       static_cast<cudaStream_t>(stream)),
            "gen_store_kernel<f32> launch");
    return RANMAR_OK;
}

// ---- one long stream at full width: substream k starts at s_{kL} (make_streams),
// outputs land in order, and the state ends as `count` calls of step() leave it.
}  // extern "C"

namespace {

constexpr uint64_t kSingleL = 8192;  // outputs per substream

uint64_t single_parts(uint64_t count) { return (count + kSingleL - 1) / kSingleL; }

size_t single_ws_states(uint64_t parts) {
    return static_cast<size_t>((parts * sizeof(ranmar_state) + 255) / 256 * 256);
}

template <class T>
int generate_single(ranmar_state* d_state, uint64_t count, T* d_out, void* d_ws, size_t ws_bytes,
                    void* stream, int (*gen)(ranmar_state*, uint64_t, uint64_t, T*, void*)) {
    if (count == 0) return RANMAR_OK;
    if (!d_state || !d_out) return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    const uint64_t parts = single_parts(count);
    if (parts == 1) return gen(d_state, 1, count, d_out, stream);
    const size_t need = ranmar_generate_single_workspace(count);
    if (!d_ws) return fail(RANMAR_EINVAL, "ranmar: null workspace");
    if (ws_bytes < need) return fail(RANMAR_ENOMEM, "ranmar: workspace too small");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // substream k = s_{k L} from the device-resident state itself (no host read)
    ranmar_state* sub = static_cast<ranmar_state*>(d_ws);
    char* ws2 = static_cast<char*>(d_ws) + single_ws_states(parts);
    ranmar_jump_count J = {{kSingleL, 0, 0, 0}};
    if (int rc = make_streams_impl(nullptr, d_state, &J, 0, parts, sub, ws2,
                                   ws_bytes - single_ws_states(parts), stream))
        return rc;
    // all substreams (the last one shorter) and the re-join into *d_state: one launch
    const uint64_t last = count - (parts - 1) * kSingleL;
    RB_STATUS_PTR(status);
    RB_CUDA(rb::launch_generate_joined<T>(sub, parts, kSingleL, last, d_out, d_state,
                                          static_cast<int>(count % 97), status, s),
            "gen_store_kernel launch");
    return RANMAR_OK;
}

}  // namespace

extern "C" {

size_t ranmar_generate_single_workspace(uint64_t count) {
    const uint64_t parts = single_parts(count);
    if (parts <= 1) return 0;
    return single_ws_states(parts) + ranmar_make_streams_workspace(parts);
}

int ranmar_generate_single_u32_dev(ranmar_state* d_state, uint64_t count, uint32_t* d_out,
                                   void* d_ws, size_t ws_bytes, void* stream) {
    return generate_single<uint32_t>(d_state, count, d_out, d_ws, ws_bytes, stream,
                                     ranmar_generate_u32_dev);
}

int ranmar_generate_single_f32_dev(ranmar_state* d_state, uint64_t count, float* d_out,
                                   void* d_ws, size_t ws_bytes, void* stream) {
    return generate_single<float>(d_state, count, d_out, d_ws, ws_bytes, stream,
                                  ranmar_generate_f32_dev);
}

int ranmar_generate_f64_dev(ranmar_state* d_states, uint64_t n_streams, uint64_t per_stream,
                            double* d_out, void* stream) {
    if (n_streams && (!d_states || (per_stream && !d_out)))
        return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    RB_STATUS_PTR(status);
    RB_CUDA(rb::launch_generate<double>(d_states, n_streams, per_stream, d_out, status,
                                        static_cast<cudaStream_t>(stream)),
            "gen_store_kernel<f64> launch");
    return RANMAR_OK;
}

int ranmar_consume_dev(ranmar_state* d_states, uint64_t n_streams, uint64_t per_stream,
                       uint64_t* d_sums, uint32_t* d_hist, void* stream) {
    if (n_streams && (!d_states || !d_sums || !d_hist))
        return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    RB_STATUS_PTR(status);
    RB_CUDA(rb::launch_consume(d_states, n_streams, per_stream, d_sums, d_hist, status,
                               static_cast<cudaStream_t>(stream)),
            "consume_kernel launch");
    return RANMAR_OK;
}

int ranmar_gaussian_f64_dev(ranmar_gauss_state* d_g, uint64_t n_atoms, uint64_t per_step,
                            uint64_t steps, double* d_out, void* stream) {
    if (n_atoms && (!d_g || (per_step && steps && !d_out)))
        return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    if (per_step >= (uint64_t(1) << 32))
        return fail(RANMAR_EINVAL, "ranmar_gaussian_f64_dev: per_step must be below 2^32");
    RB_STATUS_PTR(status);
    RB_CUDA(rb::launch_gaussian(d_g, n_atoms, per_step, steps, d_out, status,
                                static_cast<cudaStream_t>(stream)),
            "gaussian_kernel launch");
    return RANMAR_OK;
}

int ranmar_gaussian_moments_dev(ranmar_gauss_state* d_g, uint64_t n_atoms, uint64_t count, double* d_out,
                                void* stream) {
    if (n_atoms && count && (!d_g || !d_out)) return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    RB_STATUS_PTR(status);
    RB_CUDA(rb::launch_gaussian_moments(d_g, n_atoms, count, d_out, status, static_cast<cudaStream_t>(stream)),
            "gaussian_kernel (moments) launch");
    return RANMAR_OK;
}

int ranmar_langevin_dev(ranmar_gauss_state* d_g, uint64_t n_atoms, const double* d_v,
                        double* d_f, const int32_t* d_type, const int32_t* d_mask,
                        int32_t groupbit, const double* d_gfactor1, const double* d_gfactor2,
                        int32_t n_types, double tsqrt, int noise, void* stream) {
    if (noise != RANMAR_NOISE_UNIFORM && noise != RANMAR_NOISE_GAUSSIAN)
        return fail(RANMAR_EINVAL, "ranmar_langevin_dev: noise must be RANMAR_NOISE_*");
    if (n_types < 0) return fail(RANMAR_EINVAL, "ranmar_langevin_dev: n_types < 0");
    if (n_atoms && (!d_g || !d_v || !d_f || !d_type || !d_gfactor1 || !d_gfactor2))
        return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    RB_STATUS_PTR(status);
    RB_CUDA(rb::launch_langevin(d_g, n_atoms, d_v, d_f, d_type, d_mask, groupbit, d_gfactor1,
                                d_gfactor2, n_types, tsqrt, noise == RANMAR_NOISE_GAUSSIAN, status,
                                static_cast<cudaStream_t>(stream)),
            "langevin_kernel launch");
    return RANMAR_OK;
}

int ranmar_langevin_noise_dev(uint64_t n_atoms, const double* d_noise, const double* d_v,
                              double* d_f, const int32_t* d_type, const int32_t* d_mask,
                              int32_t groupbit, const double* d_gfactor1, const double* d_gfactor2,
                              int32_t n_types, double tsqrt, void* stream) {
    if (n_types < 0) return fail(RANMAR_EINVAL, "ranmar_langevin_noise_dev: n_types < 0");
    if (n_atoms && (!d_noise || !d_v || !d_f || !d_type || !d_gfactor1 || !d_gfactor2))
        return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    if (n_atoms >= (uint64_t(1) << 62)) return fail(RANMAR_ERANGE, "ranmar_langevin_noise_dev: too many atoms");
    RB_STATUS_PTR(status);
    RB_CUDA(rb::launch_langevin_noise(n_atoms, d_noise, d_v, d_f, d_type, d_mask, groupbit, d_gfactor1,
                                      d_gfactor2, n_types, tsqrt, status, static_cast<cudaStream_t>(stream)),
            "langevin_noise_kernel launch");
    return RANMAR_OK;
}

uint64_t ranmar_bank_words(uint64_t n) { return 99 * n; }

int ranmar_bank_from_states_dev(const ranmar_state* d_states, uint64_t n, uint32_t* d_bank,
                                void* stream) {
    if (n && (!d_states || !d_bank)) return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    RB_STATUS_PTR(status);
    RB_CUDA(rb::launch_bank_from_states(d_states, n, d_bank, status,
                                        static_cast<cudaStream_t>(stream)),
            "bank_from_states_kernel launch");
    return RANMAR_OK;
}

int ranmar_bank_to_states_dev(const uint32_t* d_bank, uint64_t n, uint64_t t,
                              ranmar_state* d_states, void* stream) {
    if (n && (!d_states || !d_bank)) return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    RB_CUDA(rb::launch_bank_to_states(d_bank, n, t, d_states, static_cast<cudaStream_t>(stream)),
            "bank_to_states_kernel launch");
    return RANMAR_OK;
}

int ranmar_langevin_bank_dev(uint32_t* d_bank, uint64_t n_atoms, uint64_t t, const double* d_v,
                             double* d_f, const int32_t* d_type, const double* d_gfactor1,
                             const double* d_gfactor2, int32_t n_types, double tsqrt,
                             void* stream) {
    if (n_types < 0) return fail(RANMAR_EINVAL, "ranmar_langevin_bank_dev: n_types < 0");
    if (n_atoms && (!d_bank || !d_v || !d_f || !d_type || !d_gfactor1 || !d_gfactor2))
        return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    RB_STATUS_PTR(status);
    RB_CUDA(rb::launch_langevin_bank(d_bank, n_atoms, t, d_v, d_f, d_type, d_gfactor1, d_gfactor2,
                                     n_types, tsqrt, status, static_cast<cudaStream_t>(stream)),
            "langevin_bank_kernel launch");
    return RANMAR_OK;
}

int ranmar_fp64_selfcheck_dev(uint64_t n, uint64_t seed, unsigned long long* d_mismatches,
                              void* stream) {
    if (n && !d_mismatches) return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    RB_CUDA(rb::launch_fp64_selfcheck(n, seed, d_mismatches, static_cast<cudaStream_t>(stream)),
            "fp64_selfcheck_kernel launch");
    return RANMAR_OK;
}

int ranmar_crlog_sweep_dev(uint64_t s0, uint64_t n, int32_t mode, unsigned long long* d_counts,
                           uint64_t* d_fails, uint64_t cap, void* stream) {
    if (n && (!d_counts || (cap && !d_fails))) return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    if (mode < 0 || mode > 2) return fail(RANMAR_EINVAL, "ranmar: crlog sweep mode must be 0, 1 or 2");
    if (s0 == 0 || s0 + n > (uint64_t(1) << 46) || s0 + n < s0)
        return fail(RANMAR_EINVAL, "ranmar: crlog sweep range must lie in [1, 2^46)");
    RB_CUDA(rb::launch_crlog_sweep(s0, n, mode, d_counts, d_fails, cap, static_cast<cudaStream_t>(stream)),
            "crlog_sweep_kernel launch");
    return RANMAR_OK;
}

int ranmar_init_float(uint32_t seed, ranmar_float_state* out) {
    ranmar_state s;
    if (int rc = ranmar_init(seed, &s)) return rc;
    for (int k = 0; k < 97; ++k) out->x[k] = static_cast<double>(s.lane[k]) * 0x1p-24;
    out->c = static_cast<double>(s.v) * 0x1p-24;
    out->i = s.i;
    out->j = s.j;
    return RANMAR_OK;
}

int ranmar_generate_float_dev(ranmar_float_state* d_states, uint64_t n_streams,
                              uint64_t per_stream, double* d_out, void* stream) {
    if (n_streams && (!d_states || (per_stream && !d_out)))
        return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    RB_STATUS_PTR(status);
    RB_CUDA(rb::launch_float_gen(d_states, n_streams, per_stream, d_out, nullptr, nullptr, status,
                                 static_cast<cudaStream_t>(stream)),
            "float_gen_kernel launch");
    return RANMAR_OK;
}

int ranmar_generate_float_trace_dev(ranmar_float_state* d_states, uint64_t n_streams,
                                    uint64_t per_stream, double* d_out, double* d_y, double* d_c,
                                    void* stream) {
    if (n_streams && per_stream && (!d_states || !d_out || !d_y || !d_c))
        return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    if (per_stream == 0) return RANMAR_OK;
    RB_STATUS_PTR(status);
    RB_CUDA(rb::launch_float_gen(d_states, n_streams, per_stream, d_out, d_y, d_c, status,
                                 static_cast<cudaStream_t>(stream)),
            "float_gen_kernel<trace> launch");
    return RANMAR_OK;
}

int ranmar_float_from_states_dev(const ranmar_state* d_states, uint64_t n, ranmar_float_state* d_out,
                                 void* stream) {
    if (n && (!d_states || !d_out)) return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    RB_CUDA(rb::launch_float_from_states(d_states, n, d_out, static_cast<cudaStream_t>(stream)),
            "float_from_states_kernel launch");
    return RANMAR_OK;
}

int ranmar_generate_trace_dev(ranmar_state* d_states, uint64_t n_streams, uint64_t per_stream,
                              uint32_t* d_u, uint32_t* d_x, uint32_t* d_v, void* stream) {
    if (n_streams && per_stream && (!d_states || !d_u || !d_x || !d_v))
        return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    RB_STATUS_PTR(status);
    RB_CUDA(rb::launch_generate_trace(d_states, n_streams, per_stream, d_u, d_x, d_v, status,
                                      static_cast<cudaStream_t>(stream)),
            "gen_trace_kernel launch");
    return RANMAR_OK;
}

int ranmar_poly_mul_mod_dev(const uint32_t* d_a, const uint32_t* d_b, uint32_t* d_out, uint64_t n,
                            void* stream) {
    if (n && (!d_a || !d_b || !d_out)) return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    const DevRes* r = nullptr;
    if (int rc = current_res(&r)) return rc;
    RB_CUDA(rb::launch_poly(0, d_a, d_b, d_out, n, static_cast<cudaStream_t>(stream)),
            "poly_kernel launch");
    return RANMAR_OK;
}

int ranmar_poly_reduce_dev(const uint32_t* d_raw, uint32_t* d_out, uint64_t n, void* stream) {
    if (n && (!d_raw || !d_out)) return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    const DevRes* r = nullptr;
    if (int rc = current_res(&r)) return rc;
    RB_CUDA(rb::launch_poly(1, d_raw, nullptr, d_out, n, static_cast<cudaStream_t>(stream)),
            "poly_kernel launch");
    return RANMAR_OK;
}

uint64_t ranmar_to_text_bound(uint64_t n) { return rb::text_bound(n); }
size_t ranmar_text_workspace(uint64_t n) { return rb::text_workspace(n); }

int ranmar_to_text_dev(const ranmar_state* d_states, uint64_t n, char* d_text, uint64_t text_cap,
                       uint64_t* d_offsets, void* d_ws, size_t ws_bytes, void* stream) {
    if (n == 0) {  // no texts: d_offsets[0] = 0 total bytes
        if (d_offsets)
            RB_CUDA(cudaMemsetAsync(d_offsets, 0, sizeof(uint64_t), static_cast<cudaStream_t>(stream)),
                    "offsets memset");
        return RANMAR_OK;
    }
    if (!d_states || !d_text || !d_offsets || !d_ws) return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    if (text_cap < rb::text_bound(n)) return fail(RANMAR_ENOMEM, "ranmar: text buffer below ranmar_to_text_bound(n)");
    if (ws_bytes < rb::text_workspace(n)) return fail(RANMAR_ENOMEM, "ranmar: workspace too small");
    RB_STATUS_PTR(status);
    RB_CUDA(rb::launch_to_text(d_states, n, d_text, d_offsets, d_ws, status,
                               static_cast<cudaStream_t>(stream)),
            "to_text kernels launch");
    return RANMAR_OK;
}

int ranmar_from_text_dev(const char* d_text, const uint64_t* d_offsets, uint64_t n,
                         ranmar_state* d_states, int32_t* d_err, void* stream) {
    if (n == 0) return RANMAR_OK;
    if (!d_text || !d_offsets || !d_states || !d_err) return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    RB_CUDA(rb::launch_from_text(d_text, d_offsets, n, d_states, d_err, static_cast<cudaStream_t>(stream)),
            "from_text_kernel launch");
    return RANMAR_OK;
}

int ranmar_gaussian_stream_f64_dev(ranmar_gauss_state* d_g, uint64_t n_streams, uint64_t count,
                                   double* d_out, void* stream) {
    if (n_streams && (!d_g || (count && !d_out)))
        return fail(RANMAR_EINVAL, "ranmar: null device buffer");
    RB_STATUS_PTR(status);
    RB_CUDA(rb::launch_gaussian_stream(d_g, n_streams, count, d_out, status,
                                       static_cast<cudaStream_t>(stream)),
            "gaussian_stream_kernel launch");
    return RANMAR_OK;
}

int ranmar_current_device(int* device) {
    if (!device) return fail(RANMAR_EINVAL, "ranmar: null output");
    RB_CUDA(cudaGetDevice(device), "cudaGetDevice");
    return RANMAR_OK;
}

int ranmar_device_status(uint32_t* flags, int clear) {
    const DevRes* r = nullptr;
    if (int rc = current_res(&r)) return rc;
    uint32_t* status = r->status;
    RB_CUDA(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    uint32_t h = 0;
    RB_CUDA(cudaMemcpy(&h, status, 4, cudaMemcpyDeviceToHost), "cudaMemcpy(status)");
    if (clear) RB_CUDA(cudaMemset(status, 0, 4), "cudaMemset(status)");
    if (flags) *flags = h;
    return RANMAR_OK;
}

}  // extern "C"

// ------------------------------------------------------- host-buffer context
struct ranmar_ctx {
    int device = 0;
    uint32_t* status = nullptr;  // this context's own sticky status word
    cudaStream_t st[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    void* dbuf[2] = {nullptr, nullptr};  // per-slot output chunk
    size_t dbuf_bytes[2] = {0, 0};
    ranmar_state* dstates = nullptr;
    size_t dstates_n = 0;
    void* dws = nullptr;
    size_t dws_bytes = 0;
    uint64_t h2d = 0, d2h = 0;
};

namespace {

int ctx_reserve(void** p, size_t* have, size_t need) {
    if (*have >= need) return RANMAR_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *have = 0;
    RB_CUDA(cudaMalloc(p, need), "cudaMalloc(ctx)");
    *have = need;
    return RANMAR_OK;
}

int ctx_states(ranmar_ctx* c, uint64_t n) {
    size_t have = c->dstates_n * sizeof(ranmar_state);
    void* p = c->dstates;
    int rc = ctx_reserve(&p, &have, n * sizeof(ranmar_state));
    c->dstates = static_cast<ranmar_state*>(p);
    c->dstates_n = have / sizeof(ranmar_state);
    return rc;
}

constexpr size_t kChunkBytes = size_t(512) << 20;  // output bytes per pipelined chunk

// Routes the status bits of the kernels a ctx_* call launches to the context's
// own word, so concurrent users of the device's word are neither cleared nor
// blamed, and the check needs only the context's stream, not the device.
class StatusScope {
  public:
    explicit StatusScope(uint32_t* word) : prev_(g_status_override) { g_status_override = word; }
    ~StatusScope() { g_status_override = prev_; }

  private:
    uint32_t* prev_;
};

int ctx_check_status(ranmar_ctx* c, cudaStream_t s) {
    uint32_t h = 0;
    RB_CUDA(cudaMemcpyAsync(&h, c->status, 4, cudaMemcpyDeviceToHost, s), "D2H status");
    RB_CUDA(cudaStreamSynchronize(s), "sync");
    if (h == 0) return RANMAR_OK;
    RB_CUDA(cudaMemsetAsync(c->status, 0, 4, s), "clear status");
    RB_CUDA(cudaStreamSynchronize(s), "sync");
    return fail(RANMAR_ESTATE, "ranmar: a device state violated the invariants");
}

template <class T>
int ctx_generate(ranmar_ctx* c, ranmar_state* h_states, uint64_t n, uint64_t per_stream, T* h_out,
                 int (*gen)(ranmar_state*, uint64_t, uint64_t, T*, void*),
                 int (*single)(ranmar_state*, uint64_t, T*, void*, size_t, void*)) {
    if (!c) return fail(RANMAR_EINVAL, "ranmar: null context");
    c->h2d = c->d2h = 0;
    if (n == 0) return RANMAR_OK;
    if (!h_states || (per_stream && !h_out)) return fail(RANMAR_EINVAL, "ranmar: null host buffer");
    for (uint64_t k = 0; k < n; ++k)
        if (!host_state_ok(h_states[k]))
            return fail(RANMAR_ESTATE, "ranmar: state " + std::to_string(k) +
                                           " violates cursor/residue invariants");
    DeviceGuard guard;
    RB_CUDA(guard.enter(c->device), "cudaSetDevice");
    StatusScope scope(c->status);
    if (n == 1 && ranmar_generate_single_workspace(per_stream) > 0) {
        // one long stream: full width through substreams (ranmar_generate_single_*)
        const size_t bytes = per_stream * sizeof(T);
        if (int rc = ctx_states(c, 1)) return rc;
        if (int rc = ctx_reserve(&c->dbuf[0], &c->dbuf_bytes[0], bytes)) return rc;
        if (int rc = ctx_reserve(&c->dws, &c->dws_bytes, ranmar_generate_single_workspace(per_stream)))
            return rc;
        RB_CUDA(cudaMemcpyAsync(c->dstates, h_states, sizeof(ranmar_state), cudaMemcpyHostToDevice,
                                c->st[0]),
                "H2D state");
        if (int rc = single(c->dstates, per_stream, static_cast<T*>(c->dbuf[0]), c->dws, c->dws_bytes,
                            c->st[0]))
            return rc;
        RB_CUDA(cudaMemcpyAsync(h_out, c->dbuf[0], bytes, cudaMemcpyDeviceToHost, c->st[0]), "D2H output");
        RB_CUDA(cudaMemcpyAsync(h_states, c->dstates, sizeof(ranmar_state), cudaMemcpyDeviceToHost,
                                c->st[0]),
                "D2H state");
        c->h2d = sizeof(ranmar_state);
        c->d2h = bytes + sizeof(ranmar_state);
        return ctx_check_status(c, c->st[0]);
    }
    const size_t stream_bytes = per_stream * sizeof(T);
    uint64_t chunk = stream_bytes ? std::max<uint64_t>(1, kChunkBytes / stream_bytes) : n;
    chunk = std::min<uint64_t>(chunk, n);
    if (int rc = ctx_states(c, n)) return rc;
    for (int b = 0; b < 2; ++b)  // one output buffer per pipeline slot
        if (int rc = ctx_reserve(&c->dbuf[b], &c->dbuf_bytes[b], chunk * stream_bytes)) return rc;
    RB_CUDA(cudaMemcpyAsync(c->dstates, h_states, n * sizeof(ranmar_state),
                            cudaMemcpyHostToDevice, c->st[0]),
            "H2D states");
    RB_CUDA(cudaEventRecord(c->ev[0], c->st[0]), "cudaEventRecord");
    RB_CUDA(cudaStreamWaitEvent(c->st[1], c->ev[0], 0), "cudaStreamWaitEvent");
    c->h2d += n * sizeof(ranmar_state);
    // Slot s alternates streams: generation of chunk q+1 overlaps the copy-out of chunk q.
    int q = 0;
    for (uint64_t k0 = 0; k0 < n; k0 += chunk, ++q) {
        const uint64_t cnt = std::min<uint64_t>(chunk, n - k0);
        const int slot = q & 1;
        cudaStream_t s = c->st[slot];
        T* dout = static_cast<T*>(c->dbuf[slot]);
        if (int rc = gen(c->dstates + k0, cnt, per_stream, dout, s)) return rc;
        RB_CUDA(cudaMemcpyAsync(h_out + k0 * per_stream, dout, cnt * stream_bytes,
                                cudaMemcpyDeviceToHost, s),
                "D2H output");
        c->d2h += cnt * stream_bytes;
    }
    RB_CUDA(cudaStreamSynchronize(c->st[1]), "sync");
    RB_CUDA(cudaMemcpyAsync(h_states, c->dstates, n * sizeof(ranmar_state),
                            cudaMemcpyDeviceToHost, c->st[0]),
            "D2H states");
    c->d2h += n * sizeof(ranmar_state);
    return ctx_check_status(c, c->st[0]);
}

}  // namespace

extern "C" {

int ranmar_ctx_create(int device, ranmar_ctx** out) {
    if (!out) return fail(RANMAR_EINVAL, "ranmar: null output");
    int count = 0;
    RB_CUDA(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (device < 0 || device >= count) return fail(RANMAR_ECUDA, "ranmar: no such CUDA device");
    DeviceGuard guard;
    RB_CUDA(guard.enter(device), "cudaSetDevice");
    ranmar_ctx* c = new (std::nothrow) ranmar_ctx();
    if (!c) return fail(RANMAR_ENOMEM, "ranmar: out of host memory");
    c->device = device;
    int rc = RANMAR_OK;
    for (int i = 0; i < 2 && rc == RANMAR_OK; ++i) {
        if (cudaStreamCreateWithFlags(&c->st[i], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming) != cudaSuccess)
            rc = fail(RANMAR_ECUDA, "ranmar: cudaStreamCreate / cudaEventCreate failed");
    }
    if (rc == RANMAR_OK) rc = ranmar_device_setup(device, c->st[0]);
    if (rc == RANMAR_OK && (cudaMalloc(&c->status, 4) != cudaSuccess ||
                            cudaMemsetAsync(c->status, 0, 4, c->st[0]) != cudaSuccess ||
                            cudaStreamSynchronize(c->st[0]) != cudaSuccess))
        rc = fail(RANMAR_ECUDA, "ranmar: context status word");
    if (rc != RANMAR_OK) {
        ranmar_ctx_destroy(c);
        return rc;
    }
    *out = c;
    return RANMAR_OK;
}

void ranmar_ctx_destroy(ranmar_ctx* c) {
    if (!c) return;
    DeviceGuard guard;
    guard.enter(c->device);
    if (c->status) cudaFree(c->status);
    for (int i = 0; i < 2; ++i) {
        if (c->st[i]) cudaStreamDestroy(c->st[i]);
        if (c->ev[i]) cudaEventDestroy(c->ev[i]);
        if (c->dbuf[i]) cudaFree(c->dbuf[i]);
    }
    if (c->dstates) cudaFree(c->dstates);
    if (c->dws) cudaFree(c->dws);
    delete c;
}

int ranmar_ctx_last_traffic(ranmar_ctx* c, uint64_t* h2d, uint64_t* d2h) {
    if (!c) return fail(RANMAR_EINVAL, "ranmar: null context");
    if (h2d) *h2d = c->h2d;
    if (d2h) *d2h = c->d2h;
    return RANMAR_OK;
}

int ranmar_ctx_make_streams(ranmar_ctx* c, uint32_t seed, const ranmar_jump_count* j,
                            uint64_t first, uint64_t n, ranmar_state* h_out) {
    if (!c || !h_out) return fail(RANMAR_EINVAL, "ranmar: null argument");
    c->h2d = c->d2h = 0;
    ranmar_state base;
    if (int rc = ranmar_init(seed, &base)) return rc;  // init.hpp:19-20 range check
    if (n == 0) return fail(RANMAR_EINVAL, "ranmar: need at least one stream");
    DeviceGuard guard;
    RB_CUDA(guard.enter(c->device), "cudaSetDevice");
    StatusScope scope(c->status);
    if (int rc = ctx_states(c, n)) return rc;
    if (int rc = ctx_reserve(&c->dws, &c->dws_bytes, ranmar_make_streams_workspace(n))) return rc;
    if (int rc = ranmar_make_streams_dev(&base, j, first, n, c->dstates, c->dws, c->dws_bytes,
                                         c->st[0]))
        return rc;
    RB_CUDA(cudaMemcpyAsync(h_out, c->dstates, n * sizeof(ranmar_state), cudaMemcpyDeviceToHost,
                            c->st[0]),
            "D2H states");
    c->d2h += n * sizeof(ranmar_state);
    return ctx_check_status(c, c->st[0]);
}

int ranmar_ctx_jump(ranmar_ctx* c, const ranmar_state* h_in, ranmar_state* h_out, uint64_t n,
                    const ranmar_jump_count* j) {
    if (!c || !j) return fail(RANMAR_EINVAL, "ranmar: null argument");
    c->h2d = c->d2h = 0;
    if (n == 0) return RANMAR_OK;
    if (!h_in || !h_out) return fail(RANMAR_EINVAL, "ranmar: null host buffer");
    for (uint64_t k = 0; k < n; ++k)
        if (!host_state_ok(h_in[k]))
            return fail(RANMAR_ESTATE, "ranmar: state " + std::to_string(k) +
                                           " violates cursor/residue invariants");
    DeviceGuard guard;
    RB_CUDA(guard.enter(c->device), "cudaSetDevice");
    StatusScope scope(c->status);
    if (int rc = ctx_states(c, n)) return rc;
    if (int rc = ctx_reserve(&c->dws, &c->dws_bytes, 4096)) return rc;
    RB_CUDA(cudaMemcpyAsync(c->dstates, h_in, n * sizeof(ranmar_state), cudaMemcpyHostToDevice,
                            c->st[0]),
            "H2D states");
    c->h2d += n * sizeof(ranmar_state);
    if (int rc = ranmar_jump_dev(c->dstates, c->dstates, n, j, c->dws, c->dws_bytes, c->st[0]))
        return rc;
    RB_CUDA(cudaMemcpyAsync(h_out, c->dstates, n * sizeof(ranmar_state), cudaMemcpyDeviceToHost,
                            c->st[0]),
            "D2H states");
    c->d2h += n * sizeof(ranmar_state);
    return ctx_check_status(c, c->st[0]);
}

int ranmar_ctx_generate_u32(ranmar_ctx* c, ranmar_state* h_states, uint64_t n, uint64_t per_stream,
                            uint32_t* h_out) {
    return ctx_generate<uint32_t>(c, h_states, n, per_stream, h_out, ranmar_generate_u32_dev,
                                  ranmar_generate_single_u32_dev);
}

int ranmar_ctx_generate_f32(ranmar_ctx* c, ranmar_state* h_states, uint64_t n, uint64_t per_stream,
                            float* h_out) {
    return ctx_generate<float>(c, h_states, n, per_stream, h_out, ranmar_generate_f32_dev,
                               ranmar_generate_single_f32_dev);
}

int ranmar_ctx_consume(ranmar_ctx* c, ranmar_state* h_states, uint64_t n, uint64_t per_stream,
                       uint64_t* h_sums, uint32_t* h_hist) {
    if (!c) return fail(RANMAR_EINVAL, "ranmar: null context");
    c->h2d = c->d2h = 0;
    if (n == 0) return RANMAR_OK;
    if (!h_states || !h_sums || !h_hist) return fail(RANMAR_EINVAL, "ranmar: null host buffer");
    for (uint64_t k = 0; k < n; ++k)
        if (!host_state_ok(h_states[k]))
            return fail(RANMAR_ESTATE, "ranmar: state " + std::to_string(k) +
                                           " violates cursor/residue invariants");
    DeviceGuard guard;
    RB_CUDA(guard.enter(c->device), "cudaSetDevice");
    StatusScope scope(c->status);
    if (int rc = ctx_states(c, n)) return rc;
    const size_t need = n * (8 + 256 * 4);
    if (int rc = ctx_reserve(&c->dbuf[0], &c->dbuf_bytes[0], need)) return rc;
    uint64_t* dsums = static_cast<uint64_t*>(c->dbuf[0]);
    uint32_t* dhist = reinterpret_cast<uint32_t*>(dsums + n);
    cudaStream_t s = c->st[0];
    RB_CUDA(cudaMemcpyAsync(c->dstates, h_states, n * sizeof(ranmar_state), cudaMemcpyHostToDevice,
                            s),
            "H2D states");
    c->h2d += n * sizeof(ranmar_state);
    if (int rc = ranmar_consume_dev(c->dstates, n, per_stream, dsums, dhist, s)) return rc;
    RB_CUDA(cudaMemcpyAsync(h_sums, dsums, n * 8, cudaMemcpyDeviceToHost, s), "D2H sums");
    RB_CUDA(cudaMemcpyAsync(h_hist, dhist, n * 256 * 4, cudaMemcpyDeviceToHost, s), "D2H hist");
    RB_CUDA(cudaMemcpyAsync(h_states, c->dstates, n * sizeof(ranmar_state), cudaMemcpyDeviceToHost,
                            s),
            "D2H states");
    c->d2h += n * (8 + 256 * 4 + sizeof(ranmar_state));
    return ctx_check_status(c, s);
}

int ranmar_ctx_gaussian_stream(ranmar_ctx* c, ranmar_gauss_state* h_g, uint64_t n, uint64_t count,
                               double* h_out) {
    if (!c) return fail(RANMAR_EINVAL, "ranmar: null context");
    c->h2d = c->d2h = 0;
    if (n == 0) return RANMAR_OK;
    if (!h_g || (count && !h_out)) return fail(RANMAR_EINVAL, "ranmar: null host buffer");
    for (uint64_t k = 0; k < n; ++k)
        if (!host_state_ok(h_g[k].s))
            return fail(RANMAR_ESTATE, "ranmar: state " + std::to_string(k) +
                                           " violates cursor/residue invariants");
    DeviceGuard guard;
    RB_CUDA(guard.enter(c->device), "cudaSetDevice");
    StatusScope scope(c->status);
    const size_t gbytes = n * sizeof(ranmar_gauss_state), obytes = n * count * sizeof(double);
    if (int rc = ctx_reserve(&c->dbuf[0], &c->dbuf_bytes[0], gbytes + obytes)) return rc;
    ranmar_gauss_state* dg = static_cast<ranmar_gauss_state*>(c->dbuf[0]);
    double* dout = reinterpret_cast<double*>(static_cast<char*>(c->dbuf[0]) + gbytes);
    cudaStream_t s = c->st[0];
    RB_CUDA(cudaMemcpyAsync(dg, h_g, gbytes, cudaMemcpyHostToDevice, s), "H2D gauss states");
    c->h2d += gbytes;
    if (int rc = ranmar_gaussian_stream_f64_dev(dg, n, count, dout, s)) return rc;
    if (obytes) RB_CUDA(cudaMemcpyAsync(h_out, dout, obytes, cudaMemcpyDeviceToHost, s), "D2H out");
    RB_CUDA(cudaMemcpyAsync(h_g, dg, gbytes, cudaMemcpyDeviceToHost, s), "D2H gauss states");
    c->d2h += gbytes + obytes;
    return ctx_check_status(c, s);
}

}  // extern "C"

namespace {

// Stages `k` host inputs into the context's scratch, runs `launch` on the
// context stream with device pointers, copies `m` outputs back; synchronous.
struct HostSpan {
    const void* h;
    size_t bytes;
};
struct HostOut {
    void* h;
    size_t bytes;
};
template <class Launch>
int ctx_roundtrip(ranmar_ctx* c, std::initializer_list<HostSpan> in, std::initializer_list<HostOut> out,
                  Launch launch) {
    if (!c) return fail(RANMAR_EINVAL, "ranmar: null context");
    c->h2d = c->d2h = 0;
    DeviceGuard guard;
    RB_CUDA(guard.enter(c->device), "cudaSetDevice");
    StatusScope scope(c->status);
    size_t total = 0;
    for (const auto& x : in) total += align256(x.bytes);
    for (const auto& x : out) total += align256(x.bytes);
    if (int rc = ctx_reserve(&c->dbuf[0], &c->dbuf_bytes[0], total ? total : 256)) return rc;
    cudaStream_t s = c->st[0];
    char* p = static_cast<char*>(c->dbuf[0]);
    std::vector<void*> din, dout;
    for (const auto& x : in) {
        if (x.bytes) RB_CUDA(cudaMemcpyAsync(p, x.h, x.bytes, cudaMemcpyHostToDevice, s), "H2D");
        c->h2d += x.bytes;
        din.push_back(p);
        p += align256(x.bytes);
    }
    for (const auto& x : out) {
        dout.push_back(p);
        p += align256(x.bytes);
    }
    if (int rc = launch(din, dout, static_cast<void*>(s))) return rc;
    size_t q = 0;
    for (const auto& x : out) {
        if (x.bytes) RB_CUDA(cudaMemcpyAsync(x.h, dout[q], x.bytes, cudaMemcpyDeviceToHost, s), "D2H");
        c->d2h += x.bytes;
        ++q;
    }
    return ctx_check_status(c, s);
}

}  // namespace

extern "C" {

int ranmar_ctx_generate_trace(ranmar_ctx* c, ranmar_state* h_states, uint64_t n, uint64_t per_stream,
                              uint32_t* h_u, uint32_t* h_x, uint32_t* h_v) {
    if (n && (!h_states || (per_stream && (!h_u || !h_x || !h_v))))
        return fail(RANMAR_EINVAL, "ranmar: null host buffer");
    for (uint64_t k = 0; k < n; ++k)
        if (!host_state_ok(h_states[k]))
            return fail(RANMAR_ESTATE, "ranmar: state " + std::to_string(k) +
                                           " violates cursor/residue invariants");
    const size_t sb = n * sizeof(ranmar_state), ob = n * per_stream * 4;
    return ctx_roundtrip(c, {{h_states, sb}}, {{h_u, ob}, {h_x, ob}, {h_v, ob}, {h_states, sb}},
                         [&](std::vector<void*>& din, std::vector<void*>& dout, void* s) {
                             ranmar_state* d = static_cast<ranmar_state*>(din[0]);
                             if (int rc = ranmar_generate_trace_dev(d, n, per_stream,
                                                                    static_cast<uint32_t*>(dout[0]),
                                                                    static_cast<uint32_t*>(dout[1]),
                                                                    static_cast<uint32_t*>(dout[2]), s))
                                 return rc;
                             RB_CUDA(cudaMemcpyAsync(dout[3], d, sb, cudaMemcpyDeviceToDevice,
                                                     static_cast<cudaStream_t>(s)),
                                     "D2D states");
                             return static_cast<int>(RANMAR_OK);
                         });
}

int ranmar_ctx_float_trace(ranmar_ctx* c, ranmar_float_state* h_states, uint64_t n, uint64_t per_stream,
                           double* h_out, double* h_y, double* h_c) {
    if (n && (!h_states || (per_stream && (!h_out || !h_y || !h_c))))
        return fail(RANMAR_EINVAL, "ranmar: null host buffer");
    const size_t sb = n * sizeof(ranmar_float_state), ob = n * per_stream * 8;
    return ctx_roundtrip(c, {{h_states, sb}}, {{h_out, ob}, {h_y, ob}, {h_c, ob}, {h_states, sb}},
                         [&](std::vector<void*>& din, std::vector<void*>& dout, void* s) {
                             ranmar_float_state* d = static_cast<ranmar_float_state*>(din[0]);
                             if (int rc = ranmar_generate_float_trace_dev(
                                     d, n, per_stream, static_cast<double*>(dout[0]),
                                     static_cast<double*>(dout[1]), static_cast<double*>(dout[2]), s))
                                 return rc;
                             RB_CUDA(cudaMemcpyAsync(dout[3], d, sb, cudaMemcpyDeviceToDevice,
                                                     static_cast<cudaStream_t>(s)),
                                     "D2D states");
                             return static_cast<int>(RANMAR_OK);
                         });
}

int ranmar_ctx_pow_t_mod(ranmar_ctx* c, const ranmar_jump_count* j, uint32_t* h_coeff) {
    if (!j || !h_coeff) return fail(RANMAR_EINVAL, "ranmar: null argument");
    return ctx_roundtrip(c, {}, {{h_coeff, 97 * 4}},
                         [&](std::vector<void*>&, std::vector<void*>& dout, void* s) {
                             return ranmar_pow_t_mod_dev(j, static_cast<uint32_t*>(dout[0]), s);
                         });
}

int ranmar_ctx_poly_mul_mod(ranmar_ctx* c, const uint32_t* h_a, const uint32_t* h_b, uint32_t* h_out,
                            uint64_t n) {
    if (n && (!h_a || !h_b || !h_out)) return fail(RANMAR_EINVAL, "ranmar: null host buffer");
    return ctx_roundtrip(c, {{h_a, n * 97 * 4}, {h_b, n * 97 * 4}}, {{h_out, n * 97 * 4}},
                         [&](std::vector<void*>& din, std::vector<void*>& dout, void* s) {
                             return ranmar_poly_mul_mod_dev(static_cast<uint32_t*>(din[0]),
                                                            static_cast<uint32_t*>(din[1]),
                                                            static_cast<uint32_t*>(dout[0]), n, s);
                         });
}

int ranmar_ctx_poly_reduce(ranmar_ctx* c, const uint32_t* h_raw, uint32_t* h_out, uint64_t n) {
    if (n && (!h_raw || !h_out)) return fail(RANMAR_EINVAL, "ranmar: null host buffer");
    return ctx_roundtrip(c, {{h_raw, n * 193 * 4}}, {{h_out, n * 97 * 4}},
                         [&](std::vector<void*>& din, std::vector<void*>& dout, void* s) {
                             return ranmar_poly_reduce_dev(static_cast<uint32_t*>(din[0]),
                                                           static_cast<uint32_t*>(dout[0]), n, s);
                         });
}

}  // extern "C"
