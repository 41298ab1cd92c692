// TEST INFRASTRUCTURE ONLY (oracle/). Never linked into the product.
//
// extern "C" driver over the UNMODIFIED reference headers
// (/root/reference/proj/include/ranmar/*.hpp, compiled in place with
// -I, never copied). Built by oracle/Makefile into oracle/_ref/libranmar_ref.so,
// which the tests use to pin the C restatement (oracle/ranmar_oracle.c) and
// which bench.py times as the reference CPU arm ("kind": "reference").
//
// Everything below only marshals arguments and threads independent stream
// ranges; every number is computed by the reference's own functions:
//   init            init.hpp:18-51
//   step / next_f64 core.hpp:54-72
//   jump_state      jump.hpp:90-95   (pow_t_mod polyring.hpp:113-124 + Horner jump.hpp:60-76)
//   make_streams    jump.hpp:108-124
//   step_float      reference/float_ranmar.hpp:33-46
//   to_text / from_text serialize.hpp:21-136
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "ranmar/ranmar.hpp"
#include "ranmar/reference/float_ranmar.hpp"

namespace {

using ranmar::JumpCount;
using ranmar::RanmarState;

static_assert(sizeof(RanmarState) == 400, "RanmarState layout");

JumpCount from_limbs(const std::uint64_t* limbs) {
    JumpCount j = 0;
    for (int k = 3; k >= 0; --k) j = (j << 64) + JumpCount(limbs[k]);
    return j;
}

void to_limbs(const JumpCount& j, std::uint64_t* limbs) {
    JumpCount x = j;
    for (int k = 0; k < 4; ++k) {
        limbs[k] = static_cast<std::uint64_t>(x);
        x = x >> 64;
    }
}

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

// Splits [0, n) into `threads` contiguous chunks and runs body(t, lo, hi) on each.
template <class F>
void parallel_ranges(std::uint64_t n, int threads, F&& body) {
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        const std::uint64_t lo = n * t / threads, hi = n * (t + 1) / threads;
        pool.emplace_back([=, &body] { body(t, lo, hi); });
    }
    for (auto& th : pool) th.join();
}

// Stream k of make_streams(base, J) for k in [lo, hi): the first one by an
// independent jump (k*J, jump.hpp:121), the rest incrementally (jump.hpp:119);
// test_jump.cpp:191-196 pins that both modes agree.
template <class F>
void walk_streams(const RanmarState& base, const JumpCount& j, std::uint64_t lo,
                  std::uint64_t hi, F&& per_stream) {
    if (lo >= hi) return;
    RanmarState s = lo == 0 ? base : ranmar::jump_state(base, j * JumpCount(lo));
    for (std::uint64_t k = lo; k < hi; ++k) {
        if (k != lo) s = ranmar::jump_state(s, j);
        per_stream(k, s);
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_init(std::uint32_t seed, RanmarState* out) {
    return guarded([&] { *out = ranmar::init(seed); });
}

int ref_step_n(RanmarState* s, std::uint64_t n, std::uint32_t* out) {
    for (std::uint64_t k = 0; k < n; ++k) {
        const std::uint32_t u = ranmar::step(*s);
        if (out) out[k] = u;
    }
    return 0;
}

int ref_next_f64_n(RanmarState* s, std::uint64_t n, double* out) {
    for (std::uint64_t k = 0; k < n; ++k) out[k] = ranmar::next_f64(*s);
    return 0;
}

int ref_value_of(std::uint32_t u, double* out) {
    return guarded([&] { *out = ranmar::value_of(u); });
}

// Float oracle: init_float(seed) then n calls of step_float.
int ref_step_float_n(std::uint32_t seed, std::uint64_t n, double* out) {
    return guarded([&] {
        auto f = ranmar::reference::init_float(seed);
        for (std::uint64_t k = 0; k < n; ++k) out[k] = ranmar::reference::step_float(f);
    });
}

int ref_init_float(std::uint32_t seed, double* lanes97, double* c) {
    return guarded([&] {
        const auto f = ranmar::reference::init_float(seed);
        for (int k = 0; k < 97; ++k) lanes97[k] = f.x[k];
        *c = f.c;
    });
}

int ref_pow_t_mod(const std::uint64_t* jlimbs, std::uint32_t* coeff97) {
    return guarded([&] {
        const auto p = ranmar::poly::pow_t_mod<24>(from_limbs(jlimbs));
        for (int k = 0; k < 97; ++k) coeff97[k] = p.coeff[k];
    });
}

int ref_mul_mod(const std::uint32_t* a, const std::uint32_t* b, std::uint32_t* out) {
    ranmar::poly::PolyMod<24> pa, pb;
    for (int k = 0; k < 97; ++k) {
        pa.coeff[k] = a[k];
        pb.coeff[k] = b[k];
    }
    const auto r = ranmar::poly::mul_mod(pa, pb);
    for (int k = 0; k < 97; ++k) out[k] = r.coeff[k];
    return 0;
}

int ref_reduce_trinomial(const std::uint32_t* raw, std::uint64_t n, std::uint32_t* out) {
    return guarded([&] {
        const auto r = ranmar::poly::reduce_trinomial<24>(
            std::span<const std::uint32_t>(raw, static_cast<std::size_t>(n)));
        for (int k = 0; k < 97; ++k) out[k] = r.coeff[k];
    });
}

int ref_jump_state(const RanmarState* in, const std::uint64_t* jlimbs, RanmarState* out) {
    return guarded([&] { *out = ranmar::jump_state(*in, from_limbs(jlimbs)); });
}

int ref_jump_arith(std::uint32_t v, const std::uint64_t* jlimbs, std::uint32_t* out) {
    return guarded([&] {
        ranmar::ArithState a{v};
        *out = ranmar::jump_arith(a, from_limbs(jlimbs)).v;
    });
}

int ref_make_streams(std::uint32_t seed, const std::uint64_t* jlimbs, std::uint64_t n,
                     int independent, RanmarState* out) {
    return guarded([&] {
        const auto v = ranmar::make_streams(
            seed, from_limbs(jlimbs), static_cast<std::size_t>(n),
            independent ? ranmar::StreamMode::independent : ranmar::StreamMode::incremental);
        std::memcpy(out, v.data(), v.size() * sizeof(RanmarState));
    });
}

int ref_parse_jump_count(const char* text, std::uint64_t* jlimbs) {
    return guarded([&] { to_limbs(ranmar::parse_jump_count(text), jlimbs); });
}

// to_text into a caller buffer (cap bytes, NUL-terminated); returns length or -1.
long ref_to_text(const RanmarState* s, char* buf, long cap) {
    const std::string t = ranmar::to_text(*s);
    if (static_cast<long>(t.size()) + 1 > cap) return -1;
    std::memcpy(buf, t.c_str(), t.size() + 1);
    return static_cast<long>(t.size());
}

int ref_from_text(const char* text, RanmarState* out) {
    return guarded([&] { *out = ranmar::from_text(text); });
}

// ---- threaded workloads timed by bench.py --impl reference -------------------

// C2 shape: streams [first, first+n) of make_streams(base, J), per_stream
// fp32 uniforms each (next_f64 narrowed to float, exact), stream-major.
// out may be null: the values are then folded into a checksum only.
int ref_generate_f32(const RanmarState* base, const std::uint64_t* jlimbs, std::uint64_t first,
                     std::uint64_t n, std::uint64_t per_stream, int threads, float* out,
                     std::uint64_t* checksum) {
    return guarded([&] {
        const JumpCount j = from_limbs(jlimbs);
        std::vector<std::uint64_t> sums(threads > 0 ? threads : 1, 0);
        parallel_ranges(n, threads, [&](int tid, std::uint64_t lo, std::uint64_t hi) {
            std::uint64_t acc = 0;
            walk_streams(*base, j, first + lo, first + hi, [&](std::uint64_t k, RanmarState s) {
                float* dst = out ? out + (k - first) * per_stream : nullptr;
                for (std::uint64_t t = 0; t < per_stream; ++t) {
                    const float f = static_cast<float>(ranmar::next_f64(s));
                    if (dst) dst[t] = f;
                    acc += static_cast<std::uint64_t>(f * 16777216.0f);
                }
            });
            sums[static_cast<std::size_t>(tid)] = acc;
        });
        if (checksum) {
            std::uint64_t c = 0;
            for (auto x : sums) c += x;
            *checksum = c;
        }
    });
}

// C3 shape: stream starts [first, first+n) of make_streams(base, J).
int ref_stream_starts(const RanmarState* base, const std::uint64_t* jlimbs, std::uint64_t first,
                      std::uint64_t n, int threads, RanmarState* out) {
    return guarded([&] {
        const JumpCount j = from_limbs(jlimbs);
        parallel_ranges(n, threads, [&](int, std::uint64_t lo, std::uint64_t hi) {
            walk_streams(*base, j, first + lo, first + hi,
                         [&](std::uint64_t k, const RanmarState& s) { out[k - first] = s; });
        });
    });
}

// Generic batched jump: out[k] = jump_state(in[k], J), each a full pow_t_mod.
int ref_jump_batch(const RanmarState* in, std::uint64_t n, const std::uint64_t* jlimbs,
                   int threads, RanmarState* out) {
    return guarded([&] {
        const JumpCount j = from_limbs(jlimbs);
        parallel_ranges(n, threads, [&](int, std::uint64_t lo, std::uint64_t hi) {
            for (std::uint64_t k = lo; k < hi; ++k) out[k] = ranmar::jump_state(in[k], j);
        });
    });
}

// Bulk persistence on the host, threaded: to_text of n states into per-state
// slots of `slot` bytes (returns total bytes, or -1 if a slot is too small),
// and from_text of n texts (count of parse failures).
long ref_to_text_bulk(const RanmarState* s, std::uint64_t n, char* buf, long slot, int threads) {
    std::vector<long> tot(threads > 0 ? threads : 1, 0);
    parallel_ranges(n, threads, [&](int tid, std::uint64_t lo, std::uint64_t hi) {
        long t = 0;
        for (std::uint64_t k = lo; k < hi; ++k) {
            const std::string x = ranmar::to_text(s[k]);
            if (static_cast<long>(x.size()) > slot) {
                t = -1;
                break;
            }
            std::memcpy(buf + k * slot, x.data(), x.size());
            t += static_cast<long>(x.size());
        }
        tot[static_cast<std::size_t>(tid)] = t;
    });
    long total = 0;
    for (long t : tot) {
        if (t < 0) return -1;
        total += t;
    }
    return total;
}

long ref_from_text_bulk(const char* buf, const std::uint64_t* off, std::uint64_t n,
                        RanmarState* out, int threads) {
    std::vector<long> bad(threads > 0 ? threads : 1, 0);
    parallel_ranges(n, threads, [&](int tid, std::uint64_t lo, std::uint64_t hi) {
        for (std::uint64_t k = lo; k < hi; ++k) {
            try {
                out[k] = ranmar::from_text(std::string_view(buf + off[k], off[k + 1] - off[k]));
            } catch (const std::invalid_argument&) {
                ++bad[static_cast<std::size_t>(tid)];
            }
        }
    });
    long b = 0;
    for (long x : bad) b += x;
    return b;
}

// C4 shape: per-stream u64 sum of the 24-bit outputs and a 256-bin histogram
// of u >> 16, streams [first, first+n) of make_streams(base, J).
int ref_consume(const RanmarState* base, const std::uint64_t* jlimbs, std::uint64_t first,
                std::uint64_t n, std::uint64_t per_stream, int threads, std::uint64_t* sums,
                std::uint32_t* hist) {
    return guarded([&] {
        const JumpCount j = from_limbs(jlimbs);
        parallel_ranges(n, threads, [&](int, std::uint64_t lo, std::uint64_t hi) {
            walk_streams(*base, j, first + lo, first + hi, [&](std::uint64_t k, RanmarState s) {
                std::uint64_t sum = 0;
                std::uint32_t* h = hist + (k - first) * 256;
                for (int b = 0; b < 256; ++b) h[b] = 0;
                for (std::uint64_t t = 0; t < per_stream; ++t) {
                    const std::uint32_t u = ranmar::step(s);
                    sum += u;
                    ++h[u >> 16];
                }
                sums[k - first] = sum;
            });
        });
    });
}

}  // extern "C"
