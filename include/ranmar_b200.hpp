// ranmar_b200.hpp — C++ drop-in facade over the C ABI (ranmar_b200.h).
//
// Restores the reference library's names, types and signatures (namespace
// ranmar, /root/reference/proj/include/ranmar/*.hpp) so a C++ caller switches
// by pointing its include path at this repo's include/ (the shims under
// include/ranmar/ map every reference header here) and linking
// libranmar_b200.so. The reference's own demos and tests/acceptance.cpp
// compile unmodified against it (tests/test_facade.py).
//
//   reference                                      here                    reference file:line
//   RanmarState / FibState / ArithState            same layout (400 B)     core.hpp:29-49
//   step(s) / next_f64(s), one at a time           device trace blocks     core.hpp:54-72
//   value_of(u24)                                  same, throws            core.hpp:75-79
//   init(seed)                                     same, throws            init.hpp:18-51
//   JumpCount (boost cpp_int), parse_jump_count    arbitrary precision     jumpcount.hpp:13-47
//   poly::PolyMod / reduce_trinomial / mul_mod /   same, products on the   polyring.hpp:27-124
//     mul_by_t / pow_t_mod                         GPU
//   canonicalize / decanonicalize / apply_companion                        jump.hpp:32-57
//     / jump_fib / jump_arith / jump_state /       same, jumps on the GPU  jump.hpp:60-124
//     make_streams / StreamMode
//   to_text / from_text                            same                    serialize.hpp:21-136
//   reference::FloatState / init_float /           same; step_float from   float_ranmar.hpp:22-95
//     step_float / is_dyadic24 / to_u24            device trace blocks
//   (north star: LAMMPS RanMars)                   RanMars, UniformStream
//
// std::invalid_argument is thrown exactly where the reference throws it;
// CUDA failures throw std::runtime_error.
//
// Scalar calls. step(s) must advance the caller's state object exactly as
// the reference's step() does, one call at a time. The numbers come from the
// GPU: the first call on a state generates a block of B steps for it
// (ranmar_ctx_generate_trace: per step the output, the word written into
// lane[i] and the new residue), and each call copies the next step's words
// into the caller's state (lane[i], v) and moves the cursors. A thread-local
// cache keyed by the full 400-byte state serves consecutive calls on a state,
// or on a copy of it; anything else (another state, a modified one) starts a
// new block. B grows from 256 to 65,536 while a chain continues. step_float(f)
// works the same way on reference::FloatState. For throughput use the bulk
// forms (generate_f32 / generate_u32, or the _dev C ABI): a scalar call costs
// ~20 ns of host bookkeeping, the bulk path ~0.01 ns per output.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <initializer_list>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <type_traits>
#include <vector>

#include "ranmar_b200.h"

namespace ranmar {

inline constexpr int long_lag = 97;                    // core.hpp:17
inline constexpr int short_lag = 33;                   // core.hpp:18
inline constexpr unsigned word_bits = 24;              // core.hpp:19
inline constexpr std::uint32_t word_mask = 0x00FFFFFFu;
inline constexpr std::uint32_t arith_mod = 16777213u;
inline constexpr std::uint32_t arith_delta = 7654321u;
inline constexpr std::uint32_t arith_start = 362436u;
inline constexpr std::uint32_t max_seed = 900000000u;  // init.hpp:16

struct FibState {
    std::array<std::uint32_t, long_lag> lane{};
    int i = long_lag - 1;
    int j = short_lag - 1;
    bool operator==(const FibState&) const = default;
};
struct ArithState {
    std::uint32_t v = arith_start;
    bool operator==(const ArithState&) const = default;
};
struct RanmarState {
    FibState fib;
    ArithState arith;
    bool operator==(const RanmarState&) const = default;
};
static_assert(sizeof(RanmarState) == sizeof(ranmar_state), "RanmarState must be the ABI record");

// jump.hpp:28
using CanonicalFibVector = std::array<std::uint32_t, long_lag>;

namespace detail {

inline const ranmar_state* abi(const RanmarState* s) { return reinterpret_cast<const ranmar_state*>(s); }
inline ranmar_state* abi(RanmarState* s) { return reinterpret_cast<ranmar_state*>(s); }

[[noreturn]] inline void raise(int rc) {
    const std::string msg = ranmar_last_error();
    if (rc == RANMAR_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}
inline void check(int rc) {
    if (rc != RANMAR_OK) raise(rc);
}

inline int current_device() {
    int d = 0;
    check(ranmar_current_device(&d));
    return d;
}

// One host-buffer context per thread and CUDA device; by default the
// caller's current device (cudaGetDevice), so a thread driving GPU k uses GPU k.
inline ranmar_ctx* context(int device = -1) {
    if (device < 0) device = current_device();
    struct Holder {
        ranmar_ctx* c[64] = {};
        ~Holder() {
            for (ranmar_ctx* x : c) ranmar_ctx_destroy(x);
        }
    };
    thread_local Holder h;
    if (device >= 64) throw std::runtime_error("ranmar: device index out of range");
    if (!h.c[device]) check(ranmar_ctx_create(device, &h.c[device]));
    return h.c[device];
}

}  // namespace detail

// ------------------------------------------------------------- JumpCount
// jumpcount.hpp:13 uses boost::multiprecision::cpp_int. This is the subset of
// cpp_int the reference and its tests use: an arbitrary-precision signed
// integer (sign + 64-bit limbs) with + - * / % << >>, comparisons, msb(),
// bit_test(), decimal strings and integral conversions. Jumps reduce J
// modulo the generator's period before they reach the 256-bit C ABI:
// t has order exactly 2^23 (2^97 - 1) modulo phi over Z/2^24
// (tests/test_facade.py checks t^that = 1 and t^half != 1 on the GPU and the
// oracle) and v has period m = 2^24 - 3, so J and J mod 2^23 (2^97 - 1) m
// (< 2^145) give the same state.
class JumpCount {
 public:
    JumpCount() = default;
    template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
    JumpCount(T v) {  // NOLINT: implicit, like cpp_int
        if constexpr (std::is_signed_v<T>) {
            if (v < 0) {
                neg_ = true;
                mag_.push_back(static_cast<std::uint64_t>(0) - static_cast<std::uint64_t>(v));
                trim();
                return;
            }
        }
        mag_.push_back(static_cast<std::uint64_t>(v));
        trim();
    }
    explicit JumpCount(const std::string& dec) { parse_decimal(dec); }
    explicit JumpCount(const char* dec) { parse_decimal(dec); }

    template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
    explicit operator T() const {  // low bits, like cpp_int's narrowing conversion
        const std::uint64_t lo = mag_.empty() ? 0 : mag_[0];
        const std::uint64_t v = neg_ ? static_cast<std::uint64_t>(0) - lo : lo;
        return static_cast<T>(v);
    }
    explicit operator bool() const { return !mag_.empty(); }

    bool is_negative() const { return neg_; }
    bool is_zero() const { return mag_.empty(); }
    std::size_t limbs() const { return mag_.size(); }
    std::uint64_t limb(std::size_t k) const { return k < mag_.size() ? mag_[k] : 0; }

    std::string str() const {
        if (mag_.empty()) return "0";
        std::vector<std::uint64_t> m = mag_;
        std::string out;
        while (!m.empty()) {  // repeated division by 10^18
            unsigned __int128 r = 0;
            for (std::size_t k = m.size(); k-- > 0;) {
                const unsigned __int128 cur = (r << 64) | m[k];
                m[k] = static_cast<std::uint64_t>(cur / 1000000000000000000ull);
                r = cur % 1000000000000000000ull;
            }
            while (!m.empty() && m.back() == 0) m.pop_back();
            std::string chunk = std::to_string(static_cast<std::uint64_t>(r));
            if (!m.empty()) chunk.insert(0, 18 - chunk.size(), '0');
            out.insert(0, chunk);
        }
        return neg_ ? "-" + out : out;
    }

    friend JumpCount operator-(const JumpCount& a) {
        JumpCount r = a;
        if (!r.mag_.empty()) r.neg_ = !r.neg_;
        return r;
    }
    friend JumpCount operator+(const JumpCount& a, const JumpCount& b) {
        if (a.neg_ == b.neg_) return make(a.neg_, add_mag(a.mag_, b.mag_));
        const int c = cmp_mag(a.mag_, b.mag_);
        if (c == 0) return JumpCount();
        return c > 0 ? make(a.neg_, sub_mag(a.mag_, b.mag_)) : make(b.neg_, sub_mag(b.mag_, a.mag_));
    }
    friend JumpCount operator-(const JumpCount& a, const JumpCount& b) { return a + (-b); }
    friend JumpCount operator*(const JumpCount& a, const JumpCount& b) {
        std::vector<std::uint64_t> r(a.mag_.size() + b.mag_.size(), 0);
        for (std::size_t x = 0; x < a.mag_.size(); ++x) {
            unsigned __int128 carry = 0;
            for (std::size_t y = 0; y < b.mag_.size(); ++y) {
                const unsigned __int128 p =
                    static_cast<unsigned __int128>(a.mag_[x]) * b.mag_[y] + r[x + y] + carry;
                r[x + y] = static_cast<std::uint64_t>(p);
                carry = p >> 64;
            }
            r[x + b.mag_.size()] = static_cast<std::uint64_t>(carry);
        }
        return make(a.neg_ != b.neg_, std::move(r));
    }
    // truncating division and remainder (sign of the dividend), like cpp_int
    friend JumpCount operator/(const JumpCount& a, const JumpCount& b) {
        std::vector<std::uint64_t> q, r;
        divmod_mag(a.mag_, b.mag_, q, r);
        return make(a.neg_ != b.neg_, std::move(q));
    }
    friend JumpCount operator%(const JumpCount& a, const JumpCount& b) {
        std::vector<std::uint64_t> q, r;
        divmod_mag(a.mag_, b.mag_, q, r);
        return make(a.neg_, std::move(r));
    }
    friend JumpCount operator<<(const JumpCount& a, unsigned long s) {
        if (a.mag_.empty()) return a;
        const std::size_t q = s / 64, b = s % 64;
        std::vector<std::uint64_t> r(a.mag_.size() + q + 1, 0);
        for (std::size_t k = 0; k < a.mag_.size(); ++k) {
            r[k + q] |= a.mag_[k] << b;
            if (b) r[k + q + 1] |= a.mag_[k] >> (64 - b);
        }
        return make(a.neg_, std::move(r));
    }
    friend JumpCount operator>>(const JumpCount& a, unsigned long s) {
        const std::size_t q = s / 64, b = s % 64;
        if (q >= a.mag_.size()) return JumpCount();
        std::vector<std::uint64_t> r(a.mag_.size() - q, 0);
        for (std::size_t k = 0; k < r.size(); ++k) {
            r[k] = a.mag_[k + q] >> b;
            if (b && k + q + 1 < a.mag_.size()) r[k] |= a.mag_[k + q + 1] << (64 - b);
        }
        return make(a.neg_, std::move(r));
    }
    JumpCount& operator+=(const JumpCount& b) { return *this = *this + b; }
    JumpCount& operator-=(const JumpCount& b) { return *this = *this - b; }
    JumpCount& operator*=(const JumpCount& b) { return *this = *this * b; }
    JumpCount& operator/=(const JumpCount& b) { return *this = *this / b; }
    JumpCount& operator%=(const JumpCount& b) { return *this = *this % b; }
    JumpCount& operator<<=(unsigned long s) { return *this = *this << s; }
    JumpCount& operator>>=(unsigned long s) { return *this = *this >> s; }

    friend bool operator==(const JumpCount& a, const JumpCount& b) {
        return a.neg_ == b.neg_ && a.mag_ == b.mag_;
    }
    friend bool operator!=(const JumpCount& a, const JumpCount& b) { return !(a == b); }
    friend bool operator<(const JumpCount& a, const JumpCount& b) {
        if (a.neg_ != b.neg_) return a.neg_;
        const int c = cmp_mag(a.mag_, b.mag_);
        return a.neg_ ? c > 0 : c < 0;
    }
    friend bool operator>(const JumpCount& a, const JumpCount& b) { return b < a; }
    friend bool operator<=(const JumpCount& a, const JumpCount& b) { return !(b < a); }
    friend bool operator>=(const JumpCount& a, const JumpCount& b) { return !(a < b); }

    // boost::multiprecision::msb / bit_test (found by ADL, polyring.hpp:119-121)
    friend unsigned msb(const JumpCount& a) {
        if (a.mag_.empty()) throw std::domain_error("ranmar: msb of zero");
        return static_cast<unsigned>(64 * (a.mag_.size() - 1) + 63 - __builtin_clzll(a.mag_.back()));
    }
    friend bool bit_test(const JumpCount& a, unsigned k) { return (a.limb(k / 64) >> (k % 64)) & 1u; }

 private:
    static JumpCount make(bool neg, std::vector<std::uint64_t> m) {
        JumpCount r;
        r.mag_ = std::move(m);
        r.trim();
        r.neg_ = neg && !r.mag_.empty();
        return r;
    }
    void trim() {
        while (!mag_.empty() && mag_.back() == 0) mag_.pop_back();
        if (mag_.empty()) neg_ = false;
    }
    void parse_decimal(std::string_view t) {
        bool neg = false;
        if (!t.empty() && (t[0] == '-' || t[0] == '+')) {
            neg = t[0] == '-';
            t.remove_prefix(1);
        }
        if (t.empty()) throw std::invalid_argument("ranmar: empty integer literal");
        JumpCount r;
        for (char ch : t) {
            if (ch < '0' || ch > '9') throw std::invalid_argument("ranmar: bad integer literal");
            r = r * JumpCount(10) + JumpCount(ch - '0');
        }
        *this = neg ? -r : r;
    }
    static int cmp_mag(const std::vector<std::uint64_t>& a, const std::vector<std::uint64_t>& b) {
        if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
        for (std::size_t k = a.size(); k-- > 0;)
            if (a[k] != b[k]) return a[k] < b[k] ? -1 : 1;
        return 0;
    }
    static std::vector<std::uint64_t> add_mag(const std::vector<std::uint64_t>& a,
                                              const std::vector<std::uint64_t>& b) {
        std::vector<std::uint64_t> r(std::max(a.size(), b.size()) + 1, 0);
        unsigned __int128 c = 0;
        for (std::size_t k = 0; k + 1 < r.size(); ++k) {
            c += static_cast<unsigned __int128>(k < a.size() ? a[k] : 0) + (k < b.size() ? b[k] : 0);
            r[k] = static_cast<std::uint64_t>(c);
            c >>= 64;
        }
        r.back() = static_cast<std::uint64_t>(c);
        return r;
    }
    static std::vector<std::uint64_t> sub_mag(const std::vector<std::uint64_t>& a,
                                              const std::vector<std::uint64_t>& b) {  // a >= b
        std::vector<std::uint64_t> r(a.size(), 0);
        std::uint64_t borrow = 0;
        for (std::size_t k = 0; k < a.size(); ++k) {
            const std::uint64_t y = k < b.size() ? b[k] : 0;
            const std::uint64_t d1 = a[k] - y;
            const std::uint64_t b1 = a[k] < y;
            r[k] = d1 - borrow;
            borrow = b1 | (d1 < borrow);
        }
        return r;
    }
    // binary long division on magnitudes (operands here are at most a few
    // thousand bits; 2^k jump counts go through the shift path instead)
    static void divmod_mag(const std::vector<std::uint64_t>& a, const std::vector<std::uint64_t>& b,
                           std::vector<std::uint64_t>& q, std::vector<std::uint64_t>& r) {
        if (b.empty()) throw std::domain_error("ranmar: division by zero");
        q.assign(a.size(), 0);
        r.clear();
        if (b.size() == 1) {  // fast path: one-limb divisor
            unsigned __int128 rem = 0;
            for (std::size_t k = a.size(); k-- > 0;) {
                const unsigned __int128 cur = (rem << 64) | a[k];
                q[k] = static_cast<std::uint64_t>(cur / b[0]);
                rem = cur % b[0];
            }
            if (rem) r.push_back(static_cast<std::uint64_t>(rem));
            return;
        }
        const std::size_t bits = 64 * a.size();
        for (std::size_t k = bits; k-- > 0;) {
            // r = 2 r + bit k of a
            std::uint64_t carry = (a[k / 64] >> (k % 64)) & 1u;
            for (auto& w : r) {
                const std::uint64_t nc = w >> 63;
                w = (w << 1) | carry;
                carry = nc;
            }
            if (carry) r.push_back(carry);
            if (cmp_mag(r, b) >= 0) {
                r = sub_mag(r, b);
                while (!r.empty() && r.back() == 0) r.pop_back();
                q[k / 64] |= std::uint64_t(1) << (k % 64);
            }
        }
    }

    bool neg_ = false;
    std::vector<std::uint64_t> mag_;  // little-endian, no leading zero limbs
};

namespace detail {

// A multiple of the period of the whole state: ord(t) = 2^23 (2^97 - 1)
// times m = 2^24 - 3 (see JumpCount).
inline const JumpCount& state_period() {
    static const JumpCount p = ((JumpCount(1) << 23) * ((JumpCount(1) << 97) - 1)) * JumpCount(arith_mod);
    return p;
}

// Nonnegative J -> the ABI's 256-bit limbs, reduced modulo the period.
inline ranmar_jump_count to_abi(const JumpCount& j) {
    if (j < 0) throw std::invalid_argument("ranmar: jump count must be nonnegative");  // jump.hpp:80-81
    const JumpCount r = j.limbs() > 2 ? j % state_period() : j;
    ranmar_jump_count out{};
    for (int k = 0; k < 4; ++k) out.limb[k] = r.limb(k);
    return out;
}

}  // namespace detail

// jumpcount.hpp:16-47: decimal, "2^k", "2^k-1", "2^k+1" (k <= 10^6).
inline JumpCount parse_jump_count(std::string_view text) {
    const auto bad = [&] {
        throw std::invalid_argument("ranmar: bad jump count \"" + std::string(text) +
                                    "\" (want decimal, 2^k, 2^k-1, or 2^k+1)");
    };
    if (text.empty()) bad();
    if (text.substr(0, 2) == "2^") {
        std::string_view rest = text.substr(2);
        unsigned long k = 0;
        std::size_t n = 0;
        while (n < rest.size() && rest[n] >= '0' && rest[n] <= '9') {
            k = k * 10 + static_cast<unsigned long>(rest[n] - '0');
            if (k > 1000000) throw std::invalid_argument("ranmar: jump exponent too large");
            ++n;
        }
        if (n == 0) bad();
        rest.remove_prefix(n);
        JumpCount j = JumpCount(1) << k;
        if (rest == "-1")
            j -= 1;
        else if (rest == "+1")
            j += 1;
        else if (!rest.empty())
            bad();
        return j;
    }
    for (char c : text)
        if (c < '0' || c > '9') bad();
    return JumpCount(std::string(text));
}

// ------------------------------------------------------------------ core
// init.hpp:18-51
inline RanmarState init(std::uint32_t seed) {
    RanmarState s;
    detail::check(ranmar_init(seed, detail::abi(&s)));
    return s;
}

// core.hpp:75-79
inline double value_of(std::uint32_t u24) {
    double d = 0;
    detail::check(ranmar_value_of(u24, &d));
    return d;
}

namespace detail {

// Thread-local blocks of device-generated steps for the scalar calls (see the
// header comment). S: the state type; Words: the per-step arrays a block holds.
template <class S, class Words>
struct StepCache {
    struct Entry {
        S cur{};                 // the state after the steps served so far
        Words w;                 // per-step words from the device
        std::size_t pos = 0, size = 0, next_size = 256;
        std::uint64_t used = 0;
    };
    std::array<Entry, 8> e;
    std::uint64_t tick = 0;

    template <class Fill>
    Entry& find(const S& s, Fill fill) {
        ++tick;
        for (auto& x : e)
            if (x.size && std::memcmp(&x.cur, &s, sizeof(S)) == 0) {
                x.used = tick;
                if (x.pos == x.size) {  // the chain continues: a longer block
                    x.next_size = std::min<std::size_t>(2 * x.next_size, 65536);
                    refill(x, s, fill);
                }
                return x;
            }
        Entry* lru = &e[0];
        for (auto& x : e)
            if (x.used < lru->used) lru = &x;
        lru->next_size = 256;
        lru->used = tick;
        refill(*lru, s, fill);
        return *lru;
    }
    template <class Fill>
    void refill(Entry& x, const S& s, Fill fill) {
        x.cur = s;
        S work = s;
        fill(work, x.next_size, x.w);
        x.pos = 0;
        x.size = x.next_size;
    }
};

struct IntWords {
    std::vector<std::uint32_t> u, x, v;
};

inline StepCache<RanmarState, IntWords>& int_cache() {
    thread_local StepCache<RanmarState, IntWords> c;
    return c;
}

}  // namespace detail

// core.hpp:54-66. The output and the words written into the state are the
// device's (gen_trace_kernel); the host moves the cursors.
inline std::uint32_t step(RanmarState& s) {
    auto& ent = detail::int_cache().find(s, [](RanmarState& w, std::size_t n, detail::IntWords& out) {
        out.u.resize(n);
        out.x.resize(n);
        out.v.resize(n);
        detail::check(ranmar_ctx_generate_trace(detail::context(), detail::abi(&w), 1, n, out.u.data(),
                                                out.x.data(), out.v.data()));
    });
    const std::size_t p = ent.pos++;
    // the same word updates on the caller's state and on the cache's copy of it
    // (equal before the call), so they stay equal without a 400-byte copy
    for (RanmarState* x : {&s, &ent.cur}) {
        FibState& f = x->fib;
        f.lane[f.i] = ent.w.x[p];
        f.i = (f.i == 0) ? long_lag - 1 : f.i - 1;
        f.j = (f.j == 0) ? long_lag - 1 : f.j - 1;
        x->arith.v = ent.w.v[p];
    }
    return ent.w.u[p];
}

// core.hpp:70-72
inline double next_f64(RanmarState& s) { return static_cast<double>(step(s)) * 0x1p-24; }

// ------------------------------------------------------------------ poly
namespace poly {

// polyring.hpp:27-54
template <unsigned Bits = 24>
struct PolyMod {
    static_assert(Bits >= 1 && Bits <= 32, "coefficients are stored in 32-bit words");
    static constexpr std::size_t degree_bound = 97;
    static constexpr std::size_t fold_offset = 64;
    static constexpr std::uint32_t coeff_mask =
        (Bits == 32) ? 0xFFFFFFFFu : ((std::uint32_t{1} << Bits) - 1u);

    std::array<std::uint32_t, degree_bound> coeff{};

    static PolyMod one() {
        PolyMod p;
        p.coeff[0] = 1;
        return p;
    }
    static PolyMod monomial(std::size_t k) {
        if (k >= degree_bound) throw std::invalid_argument("ranmar: monomial degree must be < 97");
        PolyMod p;
        p.coeff[k] = 1;
        return p;
    }
    bool operator==(const PolyMod&) const = default;
};

// polyring.hpp:60-80, on the GPU (the device kernels work in Z/2^24)
template <unsigned Bits = 24>
PolyMod<Bits> reduce_trinomial(std::span<const std::uint32_t> raw) {
    static_assert(Bits == 24, "the device kernels implement coefficients mod 2^24");
    if (raw.size() > 2 * PolyMod<Bits>::degree_bound - 1)
        throw std::invalid_argument("ranmar: reduce_trinomial input degree exceeds 192");
    std::array<std::uint32_t, 193> c{};
    std::copy(raw.begin(), raw.end(), c.begin());
    PolyMod<Bits> p;
    detail::check(ranmar_ctx_poly_reduce(detail::context(), c.data(), p.coeff.data(), 1));
    return p;
}
template <unsigned Bits = 24>
PolyMod<Bits> reduce_trinomial(const std::vector<std::uint32_t>& raw) {
    return reduce_trinomial<Bits>(std::span<const std::uint32_t>(raw.data(), raw.size()));
}

// polyring.hpp:85-98, on the GPU
template <unsigned Bits>
PolyMod<Bits> mul_mod(const PolyMod<Bits>& a, const PolyMod<Bits>& b) {
    static_assert(Bits == 24, "the device kernels implement coefficients mod 2^24");
    PolyMod<Bits> p;
    detail::check(ranmar_ctx_poly_mul_mod(detail::context(), a.coeff.data(), b.coeff.data(),
                                          p.coeff.data(), 1));
    return p;
}

// polyring.hpp:101-109 (p * t = p * monomial(1) mod phi), on the GPU
template <unsigned Bits>
PolyMod<Bits> mul_by_t(const PolyMod<Bits>& p) {
    return mul_mod(p, PolyMod<Bits>::monomial(1));
}

// polyring.hpp:113-124, on the GPU (K3 pow_table_kernel over the square table)
template <unsigned Bits = 24>
PolyMod<Bits> pow_t_mod(const JumpCount& j_count) {
    static_assert(Bits == 24, "the device kernels implement coefficients mod 2^24");
    if (j_count < 0) throw std::invalid_argument("ranmar: jump count must be nonnegative");
    const ranmar_jump_count j = detail::to_abi(j_count);
    PolyMod<Bits> p;
    detail::check(ranmar_ctx_pow_t_mod(detail::context(), &j, p.coeff.data()));
    return p;
}

}  // namespace poly

// ------------------------------------------------------------------ jump
// jump.hpp:32-38
inline CanonicalFibVector canonicalize(const FibState& f) {
    CanonicalFibVector u;
    for (int k = 0; k < long_lag; ++k) u[k] = f.lane[(f.i + long_lag - k) % long_lag];
    return u;
}

// jump.hpp:42-48
inline FibState decanonicalize(const CanonicalFibVector& u) {
    FibState f;
    f.i = long_lag - 1;
    f.j = short_lag - 1;
    for (int k = 0; k < long_lag; ++k) f.lane[long_lag - 1 - k] = u[k];
    return f;
}

// jump.hpp:90-95, on the GPU (K3 pow_table + apply2 kernels)
inline RanmarState jump_state(const RanmarState& s, const JumpCount& j) {
    const ranmar_jump_count jc = detail::to_abi(j);
    RanmarState out;
    detail::check(ranmar_ctx_jump(detail::context(), detail::abi(&s), detail::abi(&out), 1, &jc));
    return out;
}

// jump.hpp:60-76: the Fibonacci half of a jump, on the GPU
inline CanonicalFibVector jump_fib(const CanonicalFibVector& u, const JumpCount& j) {
    RanmarState s;
    s.fib = decanonicalize(u);
    s.arith.v = 0;
    return canonicalize(jump_state(s, j).fib);
}

// jump.hpp:52-57: one companion step = a jump by 1
inline CanonicalFibVector apply_companion(const CanonicalFibVector& u) { return jump_fib(u, 1); }

// jump.hpp:79-86
inline ArithState jump_arith(ArithState a, const JumpCount& j) {
    const ranmar_jump_count jc = detail::to_abi(j);
    ArithState r;
    detail::check(ranmar_jump_arith(a.v, &jc, &r.v));
    return r;
}

// jump.hpp:101-104: both modes give identical states (test_jump.cpp:191-196).
enum class StreamMode { incremental, independent };

// jump.hpp:108-124, on the GPU
inline std::vector<RanmarState> make_streams(std::uint32_t seed, const JumpCount& block_length,
                                             std::size_t n_streams,
                                             StreamMode = StreamMode::incremental) {
    if (n_streams == 0) throw std::invalid_argument("ranmar: need at least one stream");
    if (block_length < 1) throw std::invalid_argument("ranmar: block length must be >= 1");
    const ranmar_jump_count jc = detail::to_abi(block_length);
    if (jc.limb[0] == 0 && jc.limb[1] == 0 && jc.limb[2] == 0 && jc.limb[3] == 0) {
        // J a multiple of the period: every stream is the seed state
        return std::vector<RanmarState>(n_streams, init(seed));
    }
    std::vector<RanmarState> out(n_streams);
    detail::check(ranmar_ctx_make_streams(detail::context(), seed, &jc, 0, n_streams,
                                          detail::abi(out.data())));
    return out;
}

// ------------------------------------------------------------ serialize
// serialize.hpp:21-40 / :81-136
inline std::string to_text(const RanmarState& s) {
    char buf[4096];
    const long n = ranmar_to_text(detail::abi(&s), buf, sizeof buf);
    if (n < 0) throw std::runtime_error("ranmar: to_text buffer");
    return std::string(buf, static_cast<std::size_t>(n));
}
inline RanmarState from_text(std::string_view text) {
    RanmarState s;
    const std::string t(text);
    detail::check(ranmar_from_text(t.c_str(), detail::abi(&s)));
    return s;
}

// ------------------------------------------------------------------ bulk
// The GPU form of per_stream calls of step / next_f64 on each state
// (core.hpp:54-72): states advance exactly as step() would advance them.
inline std::vector<float> generate_f32(std::vector<RanmarState>& states, std::size_t per_stream) {
    std::vector<float> out(states.size() * per_stream);
    detail::check(ranmar_ctx_generate_f32(detail::context(), detail::abi(states.data()), states.size(),
                                          per_stream, out.data()));
    return out;
}
inline std::vector<std::uint32_t> generate_u32(std::vector<RanmarState>& states,
                                               std::size_t per_stream) {
    std::vector<std::uint32_t> out(states.size() * per_stream);
    detail::check(ranmar_ctx_generate_u32(detail::context(), detail::abi(states.data()), states.size(),
                                          per_stream, out.data()));
    return out;
}

// ------------------------------------------------------------- reference
// reference/float_ranmar.hpp: the classic floating-point generator. Its
// state is the ABI's ranmar_float_state; step_float comes from device blocks
// (K5 float_gen_kernel's trace) like step().
namespace reference {

inline constexpr double float_delta = 7654321.0 / 16777216.0;    // float_ranmar.hpp:19
inline constexpr double float_modulus = 16777213.0 / 16777216.0;  // float_ranmar.hpp:20

struct FloatState {
    std::array<double, long_lag> x{};
    double c = 362436.0 / 16777216.0;
    int i = long_lag - 1;
    int j = short_lag - 1;
    bool operator==(const FloatState&) const = default;
};
static_assert(sizeof(FloatState) == sizeof(ranmar_float_state), "FloatState must be the ABI record");

namespace detail_f {
struct FloatWords {
    std::vector<double> out, y, c;
};
inline ranmar::detail::StepCache<FloatState, FloatWords>& cache() {
    thread_local ranmar::detail::StepCache<FloatState, FloatWords> c;
    return c;
}
}  // namespace detail_f

// float_ranmar.hpp:33-46
inline double step_float(FloatState& s) {
    auto& ent = detail_f::cache().find(s, [](FloatState& w, std::size_t n, detail_f::FloatWords& o) {
        o.out.resize(n);
        o.y.resize(n);
        o.c.resize(n);
        ranmar::detail::check(ranmar_ctx_float_trace(ranmar::detail::context(),
                                                     reinterpret_cast<ranmar_float_state*>(&w), 1, n,
                                                     o.out.data(), o.y.data(), o.c.data()));
    });
    const std::size_t p = ent.pos++;
    for (FloatState* x : {&s, &ent.cur}) {
        x->x[x->i] = ent.w.y[p];
        x->i = (x->i == 0) ? long_lag - 1 : x->i - 1;
        x->j = (x->j == 0) ? long_lag - 1 : x->j - 1;
        x->c = ent.w.c[p];
    }
    return ent.w.out[p];
}

// float_ranmar.hpp:50-80 (the integer seeding mapped by the isomorphism)
inline FloatState init_float(std::uint32_t seed) {
    FloatState f;
    ranmar::detail::check(ranmar_init_float(seed, reinterpret_cast<ranmar_float_state*>(&f)));
    return f;
}

// float_ranmar.hpp:84-95
inline bool is_dyadic24(double g) {
    if (!(g >= 0.0 && g < 1.0)) return false;
    const double scaled = g * 16777216.0;
    return scaled == static_cast<double>(static_cast<std::uint64_t>(scaled));
}
inline std::uint32_t to_u24(double g) {
    if (!is_dyadic24(g))
        throw std::invalid_argument("ranmar: value is not a 24-bit dyadic in [0,1)");
    return static_cast<std::uint32_t>(g * 16777216.0);
}

}  // namespace reference

// One stream served from device-generated blocks: step() / next_f64() /
// uniform() return exactly the reference's sequence for this state.
class UniformStream {
 public:
    explicit UniformStream(const RanmarState& s, std::size_t block = 1 << 16)
        : state_(1, s), base_(s), block_(block) {}
    explicit UniformStream(std::uint32_t seed, std::size_t block = 1 << 16)
        : UniformStream(init(seed), block) {}

    std::uint32_t step() {
        if (pos_ == buf_.size()) refill();
        return buf_[pos_++];
    }
    double next_f64() { return static_cast<double>(step()) * 0x1p-24; }
    double uniform() { return next_f64(); }
    // The state after everything returned so far (buffered lookahead excluded).
    RanmarState state() const {
        RanmarState s = base_;
        if (pos_ > 0) {
            std::vector<RanmarState> v(1, base_);
            detail::check(ranmar_ctx_generate_u32(detail::context(), detail::abi(v.data()), 1, pos_,
                                                  scratch(pos_)));
            s = v[0];
        }
        return s;
    }

 private:
    void refill() {
        base_ = state_[0];
        buf_.resize(block_);
        detail::check(ranmar_ctx_generate_u32(detail::context(), detail::abi(state_.data()), 1, block_,
                                              buf_.data()));
        pos_ = 0;
    }
    std::uint32_t* scratch(std::size_t n) const {
        scratch_.resize(n);
        return scratch_.data();
    }
    std::vector<RanmarState> state_;
    RanmarState base_{};
    std::size_t block_;
    std::vector<std::uint32_t> buf_;
    std::size_t pos_ = 0;
    mutable std::vector<std::uint32_t> scratch_;
};

// LAMMPS-style generator object: seed constructor,
// uniform() (= next_f64), gaussian() (RanMars::gaussian's polar form with a
// correctly rounded log) and jump-ahead, all on one stream.
// Values come from blocks the GPU generates (K1 for uniforms, the
// warp-per-stream gaussian kernel for deviates); blocks grow from 256 to
// `block` while one kind of call repeats, and switching kind re-derives the
// exact state, so calls interleave freely.
class RanMars {
 public:
    explicit RanMars(std::uint32_t seed, std::size_t block = 1 << 16)
        : RanMars(init(seed), block) {}
    explicit RanMars(const RanmarState& s, std::size_t block = 1 << 16)
        : max_block_(block < kMinBlock ? kMinBlock : block) {
        std::memset(&g_, 0, sizeof g_);
        g_.s = *detail::abi(&s);
    }

    double uniform() { return take(Kind::uniform); }
    double gaussian() { return take(Kind::gaussian); }

    // jump_state (jump.hpp:90-95) on the stream; a cached deviate is kept.
    void jump(const JumpCount& j) {
        sync();
        const ranmar_jump_count jc = detail::to_abi(j);
        detail::check(ranmar_ctx_jump(detail::context(), &g_.s, &g_.s, 1, &jc));
    }

    // Stream state after the values returned so far.
    RanmarState state() {
        sync();
        RanmarState s;
        *detail::abi(&s) = g_.s;
        return s;
    }
    bool has_saved() {
        sync();
        return g_.has_saved != 0;
    }

 private:
    enum class Kind { none, uniform, gaussian };
    static constexpr std::size_t kMinBlock = 256;

    void run(Kind k, ranmar_gauss_state& g, std::size_t n, std::vector<double>& out) {
        out.resize(n);
        if (k == Kind::uniform) {
            std::vector<std::uint32_t> u(n);
            detail::check(ranmar_ctx_generate_u32(detail::context(), &g.s, 1, n, u.data()));
            for (std::size_t q = 0; q < n; ++q) out[q] = static_cast<double>(u[q]) * 0x1p-24;
        } else {
            detail::check(ranmar_ctx_gaussian_stream(detail::context(), &g, 1, n, out.data()));
        }
    }
    void sync() {
        if (kind_ != Kind::none) {
            if (pos_ == buf_.size()) {
                g_ = next_;
            } else if (pos_ > 0) {
                std::vector<double> scratch;
                run(kind_, g_, pos_, scratch);
            }
        }
        kind_ = Kind::none;
        buf_.clear();
        pos_ = 0;
    }
    double take(Kind k) {
        if (kind_ != k || pos_ == buf_.size()) {
            size_ = (kind_ == k) ? (2 * size_ < max_block_ ? 2 * size_ : max_block_) : kMinBlock;
            sync();
            next_ = g_;
            run(k, next_, size_, buf_);
            kind_ = k;
        }
        return buf_[pos_++];
    }

    ranmar_gauss_state g_{};     // state at the start of buf_
    ranmar_gauss_state next_{};  // state after all of buf_
    Kind kind_ = Kind::none;
    std::vector<double> buf_;
    std::size_t pos_ = 0;
    std::size_t size_ = kMinBlock;
    std::size_t max_block_;
};

}  // namespace ranmar
