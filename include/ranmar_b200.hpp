// ranmar_b200.hpp — C++ drop-in facade over the C ABI (ranmar_b200.h).
//
// Restores the reference library's names and types (namespace ranmar,
// /root/reference/proj/include/ranmar/*.hpp) so C++ callers switch by
// changing an include and a link line:
//
//   reference (ranmar/ranmar.hpp)                 here
//   RanmarState / FibState / ArithState            same layout (400 B)      core.hpp:29-49
//   init(seed)                                     same, throws             init.hpp:18-51
//   value_of(u24)                                  same, throws             core.hpp:75-79
//   JumpCount (boost cpp_int), parse_jump_count    256-bit JumpCount        jumpcount.hpp:13-47
//   jump_arith(ArithState, J)                      same                     jump.hpp:79-86
//   jump_state(state, J)                           same, on the GPU         jump.hpp:90-95
//   make_streams(seed, J, n, mode)                 same, on the GPU         jump.hpp:108-124
//   to_text / from_text                            same                     serialize.hpp:21-136
//   step(state) / next_f64(state), one at a time   UniformStream (device-
//                                                  filled buffer) and bulk
//                                                  generate_f32 / generate_u32
//   (north star: LAMMPS RanMars seed constructor,  RanMars: uniform(), gaussian(),
//    uniform()/gaussian(), jump-ahead)             jump(J), state()
//
// std::invalid_argument is thrown exactly where the reference throws it;
// CUDA failures throw std::runtime_error. Scalar step() has no GPU analogue
// worth calling per number: it is served from device-generated blocks
// (UniformStream), and whole streams are generated in bulk.
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <string_view>
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

// One context per thread, on the current CUDA device 0 by default.
inline ranmar_ctx* context(int device = 0) {
    struct Holder {
        ranmar_ctx* c = nullptr;
        ~Holder() { ranmar_ctx_destroy(c); }
    };
    thread_local Holder h;
    if (!h.c) check(ranmar_ctx_create(device, &h.c));
    return h.c;
}

}  // namespace detail

// Non-negative jump count, 256 bits (the generator's period is ~2^144).
class JumpCount {
 public:
    JumpCount() : j_{} {}
    template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
    JumpCount(T v) : j_{} {  // NOLINT: implicit like cpp_int
        if constexpr (std::is_signed_v<T>)
            if (v < 0) throw std::invalid_argument("ranmar: jump count must be nonnegative");
        j_.limb[0] = static_cast<std::uint64_t>(v);
    }
    static JumpCount from_abi(const ranmar_jump_count& j) {
        JumpCount r;
        r.j_ = j;
        return r;
    }
    const ranmar_jump_count& abi() const { return j_; }

    friend JumpCount operator<<(const JumpCount& a, unsigned s) {
        JumpCount r;
        if (s >= 256) return r;
        const unsigned q = s / 64, b = s % 64;
        for (int k = 3; k >= static_cast<int>(q); --k) {
            std::uint64_t x = a.j_.limb[k - q] << b;
            if (b && k - static_cast<int>(q) - 1 >= 0) x |= a.j_.limb[k - q - 1] >> (64 - b);
            r.j_.limb[k] = x;
        }
        return r;
    }
    friend JumpCount operator+(const JumpCount& a, const JumpCount& b) {
        JumpCount r;
        unsigned __int128 c = 0;
        for (int k = 0; k < 4; ++k) {
            c += static_cast<unsigned __int128>(a.j_.limb[k]) + b.j_.limb[k];
            r.j_.limb[k] = static_cast<std::uint64_t>(c);
            c >>= 64;
        }
        if (c) throw std::overflow_error("ranmar: jump count exceeds 2^256 - 1");
        return r;
    }
    friend JumpCount operator-(const JumpCount& a, const JumpCount& b) {
        if (a < b) throw std::invalid_argument("ranmar: jump count must be nonnegative");
        JumpCount r;
        unsigned __int128 borrow = 0;
        for (int k = 0; k < 4; ++k) {
            const unsigned __int128 x = static_cast<unsigned __int128>(a.j_.limb[k]);
            const unsigned __int128 y = static_cast<unsigned __int128>(b.j_.limb[k]) + borrow;
            r.j_.limb[k] = static_cast<std::uint64_t>(x - y);
            borrow = x < y ? 1 : 0;
        }
        return r;
    }
    friend JumpCount operator*(const JumpCount& a, std::uint64_t m) {
        JumpCount r;
        unsigned __int128 c = 0;
        for (int k = 0; k < 4; ++k) {
            c += static_cast<unsigned __int128>(a.j_.limb[k]) * m;
            r.j_.limb[k] = static_cast<std::uint64_t>(c);
            c >>= 64;
        }
        if (c) throw std::overflow_error("ranmar: jump count exceeds 2^256 - 1");
        return r;
    }
    friend bool operator==(const JumpCount& a, const JumpCount& b) {
        return std::memcmp(a.j_.limb, b.j_.limb, sizeof a.j_.limb) == 0;
    }
    friend bool operator<(const JumpCount& a, const JumpCount& b) {
        for (int k = 3; k >= 0; --k)
            if (a.j_.limb[k] != b.j_.limb[k]) return a.j_.limb[k] < b.j_.limb[k];
        return false;
    }

 private:
    ranmar_jump_count j_;
};

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

// jumpcount.hpp:16-47
inline JumpCount parse_jump_count(std::string_view text) {
    ranmar_jump_count j;
    const std::string t(text);
    detail::check(ranmar_parse_jump_count(t.c_str(), &j));
    return JumpCount::from_abi(j);
}

// jump.hpp:79-86
inline ArithState jump_arith(ArithState a, const JumpCount& j) {
    ArithState r;
    detail::check(ranmar_jump_arith(a.v, &j.abi(), &r.v));
    return r;
}

// jump.hpp:90-95, on the GPU
inline RanmarState jump_state(const RanmarState& s, const JumpCount& j) {
    RanmarState out;
    detail::check(ranmar_ctx_jump(detail::context(), detail::abi(&s), detail::abi(&out), 1, &j.abi()));
    return out;
}

// jump.hpp:101-104: both modes give identical states (test_jump.cpp:191-196).
enum class StreamMode { incremental, independent };

// jump.hpp:108-124, on the GPU
inline std::vector<RanmarState> make_streams(std::uint32_t seed, const JumpCount& block_length,
                                             std::size_t n_streams,
                                             StreamMode = StreamMode::incremental) {
    if (n_streams == 0) throw std::invalid_argument("ranmar: need at least one stream");
    if (block_length == JumpCount(0)) throw std::invalid_argument("ranmar: block length must be >= 1");
    std::vector<RanmarState> out(n_streams);
    detail::check(ranmar_ctx_make_streams(detail::context(), seed, &block_length.abi(), 0, n_streams,
                                          detail::abi(out.data())));
    return out;
}

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

// Bulk generation (the GPU form of per_stream calls of step / next_f64 on each
// state, core.hpp:54-72): states advance exactly as step() would advance them.
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
// uniform() (= next_f64), gaussian() (the repo's polar convention, DESIGN.md
// §5) and jump-ahead, all on one stream. Values come from blocks the GPU
// generates (K1 for uniforms, the warp-per-stream gaussian kernel for
// deviates); blocks grow from 256 to `block` while one kind of call repeats,
// and switching kind re-derives the exact state, so calls interleave freely.
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
        detail::check(ranmar_ctx_jump(detail::context(), &g_.s, &g_.s, 1, &j.abi()));
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
