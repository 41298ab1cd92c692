// TEST INFRASTRUCTURE ONLY (oracle/). Not part of the product.
//
// Minimal stand-in for boost::multiprecision::cpp_int, written for this repo
// because Boost is absent from the image. It lets the UNMODIFIED reference
// headers under /root/reference/proj/include (jumpcount.hpp:13 and
// polyring.hpp:19 include <boost/multiprecision/cpp_int.hpp>) and the
// reference's tests/acceptance.cpp compile, so oracle/_ref can be built from
// the reference's own sources.
//
// Semantics: fixed-width 384-bit two's-complement signed integer. The
// reference only ever uses non-negative jump counts below ~2^141 (period of
// the generator ~2^144) plus the negative literal used to test
// the invalid_argument path (test_jump.cpp:114); 384 bits cover both with a
// wide margin. Overflow wraps silently (unlike Boost, which is unbounded):
// callers that might exceed 2^383 (parse_jump_count("2^1000000")) are not
// exercised by the oracle build.
//
// Operations provided are exactly those the reference path uses
// (SURVEY.md §8c): construction from integral types and decimal strings,
// + - * (also by built-in integers through the implicit constructor), % by a
// value < 2^64, <<, >>, += -=, comparisons, explicit conversion to
// built-in integers, and ADL-found msb() / bit_test().
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <type_traits>

namespace boost {
namespace multiprecision {

class cpp_int {
 public:
    static constexpr int limbs = 6;  // 384 bits

    cpp_int() : w_{} {}

    template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
    cpp_int(T v) : w_{} {  // NOLINT: implicit, like Boost
        if constexpr (std::is_signed_v<T>) {
            const long long s = static_cast<long long>(v);
            w_[0] = static_cast<std::uint64_t>(s);
            const std::uint64_t fill = s < 0 ? ~std::uint64_t{0} : 0;
            for (int k = 1; k < limbs; ++k) w_[k] = fill;
        } else {
            w_[0] = static_cast<std::uint64_t>(v);
        }
    }

    explicit cpp_int(const std::string& text) : w_{} {
        if (text.empty()) throw std::runtime_error("cpp_int: empty string");
        std::size_t pos = 0;
        bool neg = false;
        if (text[0] == '-') { neg = true; pos = 1; }
        if (pos == text.size()) throw std::runtime_error("cpp_int: no digits");
        for (; pos < text.size(); ++pos) {
            const char c = text[pos];
            if (c < '0' || c > '9') throw std::runtime_error("cpp_int: bad digit");
            *this = mul_small(*this, 10);
            *this += cpp_int(static_cast<unsigned>(c - '0'));
        }
        if (neg) *this = -*this;
    }

    bool negative() const { return (w_[limbs - 1] >> 63) != 0; }

    template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
    explicit operator T() const {
        return static_cast<T>(w_[0]);
    }

    friend cpp_int operator+(const cpp_int& a, const cpp_int& b) {
        cpp_int r;
        unsigned __int128 carry = 0;
        for (int k = 0; k < limbs; ++k) {
            const unsigned __int128 s = (unsigned __int128)a.w_[k] + b.w_[k] + carry;
            r.w_[k] = static_cast<std::uint64_t>(s);
            carry = s >> 64;
        }
        return r;
    }
    cpp_int operator-() const {
        cpp_int r;
        for (int k = 0; k < limbs; ++k) r.w_[k] = ~w_[k];
        return r + cpp_int(1);
    }
    friend cpp_int operator-(const cpp_int& a, const cpp_int& b) { return a + (-b); }

    friend cpp_int operator*(const cpp_int& a, const cpp_int& b) {
        // Schoolbook, truncated to `limbs` words (two's complement wraps).
        cpp_int r;
        for (int i = 0; i < limbs; ++i) {
            unsigned __int128 carry = 0;
            for (int j = 0; i + j < limbs; ++j) {
                const unsigned __int128 p =
                    (unsigned __int128)a.w_[i] * b.w_[j] + r.w_[i + j] + carry;
                r.w_[i + j] = static_cast<std::uint64_t>(p);
                carry = p >> 64;
            }
        }
        return r;
    }

    // Remainder by a non-negative divisor below 2^64, for a non-negative
    // dividend (the only use: J % arith_mod, jump.hpp:82).
    friend cpp_int operator%(const cpp_int& a, const cpp_int& b) {
        if (a.negative() || b.negative()) throw std::runtime_error("cpp_int: % of negative");
        for (int k = 1; k < limbs; ++k)
            if (b.w_[k] != 0) throw std::runtime_error("cpp_int: % divisor too wide");
        const std::uint64_t d = b.w_[0];
        if (d == 0) throw std::runtime_error("cpp_int: % by zero");
        unsigned __int128 rem = 0;
        for (int k = limbs - 1; k >= 0; --k) rem = ((rem << 64) | a.w_[k]) % d;
        return cpp_int(static_cast<std::uint64_t>(rem));
    }

    friend cpp_int operator<<(const cpp_int& a, unsigned long s) {
        cpp_int r;
        if (s >= 64u * limbs) return r;
        const unsigned q = static_cast<unsigned>(s / 64), b = static_cast<unsigned>(s % 64);
        for (int k = limbs - 1; k >= static_cast<int>(q); --k) {
            std::uint64_t v = a.w_[k - q] << b;
            if (b != 0 && k - static_cast<int>(q) - 1 >= 0) v |= a.w_[k - q - 1] >> (64 - b);
            r.w_[k] = v;
        }
        return r;
    }
    friend cpp_int operator>>(const cpp_int& a, unsigned long s) {  // logical, non-negative use
        cpp_int r;
        if (s >= 64u * limbs) return r;
        const unsigned q = static_cast<unsigned>(s / 64), b = static_cast<unsigned>(s % 64);
        for (int k = 0; k + static_cast<int>(q) < limbs; ++k) {
            std::uint64_t v = a.w_[k + q] >> b;
            if (b != 0 && k + static_cast<int>(q) + 1 < limbs) v |= a.w_[k + q + 1] << (64 - b);
            r.w_[k] = v;
        }
        return r;
    }
    template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
    friend cpp_int operator<<(const cpp_int& a, T s) { return a << static_cast<unsigned long>(s); }
    template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
    friend cpp_int operator>>(const cpp_int& a, T s) { return a >> static_cast<unsigned long>(s); }

    cpp_int& operator+=(const cpp_int& b) { return *this = *this + b; }
    cpp_int& operator-=(const cpp_int& b) { return *this = *this - b; }
    cpp_int& operator*=(const cpp_int& b) { return *this = *this * b; }

    friend bool operator==(const cpp_int& a, const cpp_int& b) {
        for (int k = 0; k < limbs; ++k)
            if (a.w_[k] != b.w_[k]) return false;
        return true;
    }
    friend bool operator!=(const cpp_int& a, const cpp_int& b) { return !(a == b); }
    friend bool operator<(const cpp_int& a, const cpp_int& b) {
        const bool na = a.negative(), nb = b.negative();
        if (na != nb) return na;
        for (int k = limbs - 1; k >= 0; --k)
            if (a.w_[k] != b.w_[k]) return a.w_[k] < b.w_[k];
        return false;
    }
    friend bool operator>(const cpp_int& a, const cpp_int& b) { return b < a; }
    friend bool operator<=(const cpp_int& a, const cpp_int& b) { return !(b < a); }
    friend bool operator>=(const cpp_int& a, const cpp_int& b) { return !(a < b); }

    std::uint64_t limb(int k) const { return w_[k]; }

 private:
    static cpp_int mul_small(const cpp_int& a, std::uint64_t m) { return a * cpp_int(m); }
    std::uint64_t w_[limbs];
};

// Index of the most significant set bit; the value must be positive.
inline unsigned msb(const cpp_int& a) {
    if (a.negative()) throw std::runtime_error("cpp_int: msb of negative");
    for (int k = cpp_int::limbs - 1; k >= 0; --k)
        if (a.limb(k) != 0)
            return 64u * k + 63u - static_cast<unsigned>(__builtin_clzll(a.limb(k)));
    throw std::runtime_error("cpp_int: msb of zero");
}

inline bool bit_test(const cpp_int& a, unsigned bit) {
    if (bit >= 64u * cpp_int::limbs) return a.negative();
    return ((a.limb(static_cast<int>(bit / 64)) >> (bit % 64)) & 1u) != 0;
}

}  // namespace multiprecision
}  // namespace boost
