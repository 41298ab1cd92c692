// C++ drop-in facade check (include/ranmar_b200.hpp), run by
// tests/test_gpu_facade.py on a GPU. Written like the reference's
// tests/acceptance.cpp: plain main, one PASS/FAIL line per check, using only
// the facade's reference names and the reference's frozen known answers.
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "ranmar_b200.hpp"

using namespace ranmar;

static int failures = 0;
#define CHECK(cond)                                                           \
    do {                                                                      \
        if (!(cond)) {                                                        \
            std::printf("[FAIL] %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
            ++failures;                                                       \
        }                                                                     \
    } while (0)

template <class F>
static bool throws_invalid(F f) {
    try {
        f();
    } catch (const std::invalid_argument&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    // test_core.cpp:118-126 frozen outputs, served from device blocks
    {
        UniformStream s(12345u, 4096);
        const std::uint32_t first[10] = {1905444, 14595391, 174918,   4925251,  346329,
                                         1286474, 5077740,  10808695, 10092480, 6540075};
        for (auto e : first) CHECK(s.step() == e);
        for (int n = 10; n < 999999; ++n) s.step();
        CHECK(s.step() == 7864902u);  // output #1,000,000
        CHECK(s.state().arith.v < arith_mod);
    }
    // test_init.cpp:28-41 and the range check (init.hpp:19-20)
    {
        const auto s = init(12345);
        CHECK(s.fib.lane[0] == 2167695u && s.fib.lane[96] == 1979263u);
        CHECK(s.fib.i == 96 && s.fib.j == 32 && s.arith.v == 362436u);
        CHECK(throws_invalid([] { init(900000001u); }));
        CHECK(throws_invalid([] { value_of(1u << 24); }));
        CHECK(value_of(1u << 23) == 0.5);
    }
    // test_jump.cpp:117-132 jump of 10^5 from seed 12345
    {
        const auto j = jump_state(init(12345), JumpCount(100000));
        UniformStream s(j, 64);
        const std::uint32_t next[5] = {10494747, 9709410, 12229790, 92873, 824205};
        for (auto e : next) CHECK(s.step() == e);
        CHECK(jump_arith(ArithState{362436}, JumpCount(1)).v == 9485328u);
    }
    // additivity at 2^64 scale (acceptance.cpp:110-118)
    {
        const JumpCount big = (JumpCount(1) << 64) - JumpCount(1);
        const auto s = init(555);
        CHECK(jump_state(jump_state(s, big), big) == jump_state(s, (JumpCount(1) << 65) - JumpCount(2)));
        CHECK(parse_jump_count("2^64-1") == big);
        CHECK(throws_invalid([] { parse_jump_count("2^64-2"); }));
    }
    // make_streams tiles the base sequence (acceptance.cpp:195-206), and bulk
    // generation advances states exactly like step()
    {
        auto streams = make_streams(97531, JumpCount(1000), 10);
        auto blocks = generate_u32(streams, 1000);
        UniformStream base(97531u, 10000);
        for (std::size_t n = 0; n < blocks.size(); ++n) CHECK(blocks[n] == base.step());
        UniformStream after(streams[9], 64);  // stream 9 now sits where the base does
        for (int n = 0; n < 100; ++n) CHECK(after.step() == base.step());
        CHECK(throws_invalid([] { make_streams(1, JumpCount(5), 0); }));
        CHECK(throws_invalid([] { make_streams(1, JumpCount(0), 3); }));
        auto st2 = make_streams(12345, JumpCount(1) << 40, 3, StreamMode::independent);
        auto f = generate_f32(st2, 8);
        CHECK(f.size() == 24 && f[0] >= 0.0f && f[0] < 1.0f);
    }
    // RanMars-style object: uniform() is next_f64 of the stream; gaussian()
    // interleaves on the same stream (values pinned by the Python tests)
    {
        RanMars r(12345u, 1024);
        CHECK(r.uniform() == 1905444 * 0x1p-24);
        CHECK(r.uniform() == 14595391 * 0x1p-24);
        const double g1 = r.gaussian();
        CHECK(g1 > -10.0 && g1 < 10.0);
        CHECK(r.has_saved());          // the second deviate of the pair is cached
        const double g2 = r.gaussian();
        CHECK(!r.has_saved() && g2 > -10.0 && g2 < 10.0);
        RanMars same(12345u, 4096);    // another block size, same sequence
        same.uniform();
        same.uniform();
        CHECK(same.gaussian() == g1 && same.gaussian() == g2);
        CHECK(same.state() == r.state());
        CHECK(throws_invalid([] { RanMars bad(900000001u); }));
    }
    // scalar step() / next_f64() on the caller's state (core.hpp:54-72): the
    // reference's frozen outputs, copies of a state continue identically, the
    // state after n calls equals the bulk path's, and a modified state is
    // noticed (test_core.cpp:118-126)
    {
        auto s = init(12345);
        const std::uint32_t first[10] = {1905444, 14595391, 174918,   4925251,  346329,
                                         1286474, 5077740,  10808695, 10092480, 6540075};
        for (auto e : first) {
            auto probe = s;  // demo/basic_usage.cpp's peek
            CHECK(step(probe) == e);
            CHECK(next_f64(s) == e * 0x1p-24);
            CHECK(probe == s);
        }
        for (int n = 10; n < 999999; ++n) step(s);
        CHECK(step(s) == 7864902u);  // output #1,000,000
        std::vector<RanmarState> bulk(1, init(12345));
        generate_u32(bulk, 1000000);
        CHECK(bulk[0] == s);
        auto t = init(12345);
        step(t);
        t.fib.lane[5] ^= 1;  // a modified state must not be served from the cache
        auto t2 = t;
        std::vector<RanmarState> tb(1, t2);
        const auto exp = generate_u32(tb, 3);
        for (int n = 0; n < 3; ++n) CHECK(step(t) == exp[n]);
        CHECK(t == tb[0]);
    }
    // reference::step_float on the caller's FloatState (float_ranmar.hpp:33-46)
    // equals value_of(step()) and keeps the state isomorphic
    {
        auto s = init(900000000u);
        auto f = reference::init_float(900000000u);
        for (int n = 0; n < 300000; ++n) CHECK(value_of(step(s)) == reference::step_float(f));
        for (int k = 0; k < long_lag; ++k) CHECK(reference::to_u24(f.x[k]) == s.fib.lane[k]);
        CHECK(f.i == s.fib.i && f.j == s.fib.j && reference::to_u24(f.c) == s.arith.v);
    }
    // poly on the GPU (polyring.hpp): t has order exactly 2^23 (2^97 - 1) mod
    // phi over Z/2^24 -- the period the facade reduces jump counts by
    {
        using poly::PolyMod;
        const JumpCount ord = (JumpCount(1) << 23) * ((JumpCount(1) << 97) - 1);
        CHECK(poly::pow_t_mod<24>(ord) == PolyMod<24>::one());
        CHECK(!(poly::pow_t_mod<24>(ord / 2) == PolyMod<24>::one()));
        CHECK(!(poly::pow_t_mod<24>((JumpCount(1) << 97) - 1) == PolyMod<24>::one()));
        CHECK(poly::pow_t_mod<24>(JumpCount(97)).coeff[64] == word_mask);  // t^97 = 1 - t^64
        const auto a = poly::pow_t_mod<24>(JumpCount(123456789)), b = poly::pow_t_mod<24>(JumpCount(987654));
        CHECK(poly::mul_mod(a, b) == poly::pow_t_mod<24>(JumpCount(123456789 + 987654)));
        CHECK(poly::mul_by_t(a) == poly::pow_t_mod<24>(JumpCount(123456790)));
        std::vector<std::uint32_t> raw(193, 0);
        raw[192] = 1;  // t^192 mod phi = t^95 * t^97 = t^95 - t^159 = ...
        CHECK(poly::reduce_trinomial<24>(raw) == poly::pow_t_mod<24>(JumpCount(192)));
        // huge jumps reduce by the period: J and J + period give the same state
        const auto s = init(31337);
        const JumpCount huge = parse_jump_count("2^100000+1");
        CHECK(jump_state(s, huge) == jump_state(s, huge + detail::state_period() * JumpCount(3)));
        CHECK(jump_state(s, ord * JumpCount(arith_mod)) == jump_state(s, JumpCount(0)));
        CHECK(canonicalize(jump_state(s, JumpCount(1)).fib) == apply_companion(canonicalize(s.fib)));
    }
    // serialize.hpp round trip
    {
        const auto s = jump_state(init(4711), JumpCount(1) << 100);
        CHECK(from_text(to_text(s)) == s);
        CHECK(throws_invalid([] { from_text("ranmar24 v2\n"); }));
    }
    if (failures) {
        std::printf("%d check(s) FAILED\n", failures);
        return 1;
    }
    std::printf("facade: all checks passed\n");
    return 0;
}
