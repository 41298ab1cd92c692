"""Pins the C restatement (oracle/ranmar_oracle.c) before anything trusts it:
(1) against the frozen known answers of the reference's own unit tests,
(2) against vectors generated from the reference itself (tests/golden/ref_vectors.json),
(3) live against oracle/_ref when it was built here (skipped otherwise)."""
import os
import random

import numpy as np
import pytest

from ranmar_testutil import state_from_json

MASK = 0xFFFFFF


# ---- (1) frozen known answers (reference unit tests) --------------------------------

def test_crafted_step(oracle, known):
    k = known["crafted_step"]  # test_core.cpp:26-45
    s = oracle.init(12345)
    i, j = int(s["i"][0]), int(s["j"][0])
    s["lane"][0][i], s["lane"][0][j], s["v"] = k["lane_i"], k["lane_j"], k["v"]
    out = oracle.step_n(s, 1)[0]
    assert out == k["out"]
    assert s["lane"][0][i] == k["new_lane"] and s["v"][0] == k["new_v"]


def test_seed_outputs(oracle, known):
    for case in known["seed_outputs"]:  # test_core.cpp:118-139
        s = oracle.init(case["seed"])
        assert oracle.step_n(s, len(case["first"])).tolist() == case["first"]
    s = oracle.init(12345)
    assert oracle.step_n(s, 1_000_000)[-1] == known["seed_12345_output_1000000"]["value"]


def test_init_lanes_and_range(oracle, known):
    for case in known["init_lanes"]:  # test_init.cpp:28-59
        s = oracle.init(case["seed"])
        for idx, val in case["lanes"].items():
            assert s["lane"][0][int(idx)] == val
        if "lane_sum" in case:
            assert int(s["lane"][0].astype(np.uint64).sum()) == case["lane_sum"]
        assert (s["i"][0], s["j"][0], s["v"][0]) == (96, 32, 362436)
    oracle.init(known["max_seed"]["value"])
    with pytest.raises(ValueError):  # init.hpp:19-20
        oracle.init(known["max_seed"]["value"] + 1)


def test_jump_known(oracle, known):
    k = known["jump_1e5_seed_12345"]  # test_jump.cpp:123-132
    s = oracle.jump_state(oracle.init(k["seed"]), k["j"])
    assert oracle.step_n(s, 5).tolist() == k["next"]
    for j, v in known["jump_arith"]["cases"]:  # test_jump.cpp:101-105
        assert oracle.jump_arith(known["jump_arith"]["v"], j) == v


def test_t97_relation(oracle, known):
    p = oracle.pow_t_mod(97)  # test_polyring.cpp:75-83
    exp = np.zeros(97, np.uint32)
    for idx, val in known["t97_mod_phi"]["coeff"].items():
        exp[int(idx)] = val
    assert (p == exp).all()


def test_parse_jump_count(oracle, known):
    pj = known["parse_jump_count"]  # test_polyring.cpp:176-189
    for text, val in pj["ok"]:
        assert oracle.parse_jump_count(text) == val
    for text in pj["bad"]:
        with pytest.raises(ValueError):
            oracle.parse_jump_count(text)


def test_float_equivalence_small(oracle):
    # float_ranmar.hpp is the isomorphic oracle: u/2^24 == step_float, bit for bit.
    for seed in (0, 1, 12345, 900000000):
        f = oracle.float_outputs(seed, 20000)
        u = oracle.step_n(oracle.init(seed), 20000)
        assert (u.astype(np.float64) * 2.0 ** -24 == f).all()


# ---- (2) vectors generated from the reference ---------------------------------------

def test_ref_vectors_seeds(oracle, refvec):
    for case in refvec["seeds"]:
        s = oracle.init(case["seed"])
        ref = state_from_json(case["state"])
        assert s.tobytes() == ref.tobytes()
        assert oracle.step_n(s, 1000).tolist() == case["first1000"]


def test_ref_vectors_c1_summary(oracle, refvec):
    c = refvec["c1_seed12345_1e8"]
    s = oracle.init(12345)
    acc_sum = acc_xor = 0
    for _ in range(10):
        out = oracle.step_n(s, 10_000_000)
        acc_sum += int(out.astype(np.uint64).sum())
        acc_xor ^= int(np.bitwise_xor.reduce(out))
    assert (acc_sum, acc_xor, int(out[-1])) == (c["sum"], c["xor"], c["last"])
    assert s.tobytes() == state_from_json(c["final_state"]).tobytes()


def test_ref_vectors_float(oracle, refvec):
    assert oracle.float_outputs(12345, 1000).tolist() == refvec["float_seed12345_first1000"]


def test_ref_vectors_poly(oracle, refvec):
    for case in refvec["pow_t_mod"]:
        assert oracle.pow_t_mod(int(case["j"])).tolist() == case["coeff"], case["j"]
    for case in refvec["mul_mod"]:
        assert oracle.mul_mod(np.array(case["a"]), np.array(case["b"])).tolist() == case["out"]


def test_ref_vectors_jump(oracle, refvec):
    for case in refvec["jump_state"]:
        out = oracle.jump_state(state_from_json(case["in"]), int(case["j"]))
        assert out.tobytes() == state_from_json(case["out"]).tobytes(), case["j"]


def test_ref_vectors_make_streams(oracle, refvec):
    for case in refvec["make_streams"]:
        base = oracle.init(case["seed"])
        ss = oracle.make_streams(base, int(case["j"]), len(case["states"]))
        for got, exp in zip(ss, case["states"]):
            assert got.tobytes() == state_from_json(exp).tobytes()
        # independent chunking (first > 0) agrees with incremental
        tail = oracle.make_streams(base, int(case["j"]), 2, first=len(case["states"]) - 2)
        assert tail.tobytes() == ss[-2:].tobytes()


def test_ref_vectors_c3(oracle, refvec):
    c3 = refvec["c3_starts"]
    base = oracle.init(c3["seed"], checked=False)
    assert base.tobytes() == state_from_json(c3["base"]).tobytes()
    for k, exp in zip(c3["k"], c3["states"]):
        got = oracle.make_streams(base, int(c3["j"]), 1, first=k)
        assert got.tobytes() == state_from_json(exp).tobytes(), k


def test_ref_vectors_consume(oracle, refvec):
    c = refvec["consume"]
    ss = oracle.make_streams(oracle.init(c["seed"]), int(c["j"]), len(c["sums"]))
    sums, hist = oracle.consume(ss, c["per_stream"])
    assert sums.tolist() == c["sums"] and hist.tolist() == c["hist"]


def test_ref_vectors_text(oracle, refvec):
    for case in refvec["to_text"]:
        s = state_from_json(case["state"])
        assert oracle.to_text(s) == case["text"]
        assert oracle.from_text(case["text"]).tobytes() == s.tobytes()
    bad = refvec["to_text"][0]["text"].replace("i 97 j 33", "i 97 j 34")
    with pytest.raises(ValueError):  # serialize.hpp:100-102 cursor separation
        oracle.from_text(bad)


# ---- independent properties (test_util.hpp oracles) ---------------------------------

def test_jump_matches_stepping(oracle):
    rng = random.Random(5)
    for _ in range(5):
        s = oracle.init(rng.randrange(900000001))
        oracle.step_n(s, rng.randrange(200))  # random cursor phase
        for j in (0, 1, 2, 33, 64, 97, 1000, 10_000):
            a = s.copy()
            oracle.step_n(a, j)
            b = oracle.jump_state(s, j)
            assert (oracle.step_n(a, 100) == oracle.step_n(b, 100)).all()


def test_reduce_matches_long_division(oracle):
    # test_util.hpp:52-67 general monic long division by phi = t^97 + t^64 - 1
    rng = np.random.default_rng(7)
    phi = np.zeros(98, np.int64)
    phi[0], phi[64], phi[97] = MASK, 1, 1
    for _ in range(20):
        raw = rng.integers(0, 1 << 24, 193, dtype=np.int64)
        div = [int(x) for x in raw]
        while len(div) > 97:
            q = div[-1] & MASK
            sh = len(div) - 98
            for k in range(98):
                div[sh + k] -= q * int(phi[k])
            div.pop()
        exp = [x & MASK for x in div]
        assert oracle.reduce_trinomial(raw.astype(np.uint32)).tolist() == exp


def test_pow_additivity(oracle):
    rng = random.Random(11)
    for _ in range(5):
        a, b = rng.getrandbits(130), rng.getrandbits(130)
        assert (oracle.pow_t_mod(a + b) == oracle.mul_mod(oracle.pow_t_mod(a), oracle.pow_t_mod(b))).all()


# ---- (3) live reference (when oracle/_ref was built here) ---------------------------

def test_live_reference_agrees(oracle, reference):
    rng = random.Random(3)
    for _ in range(20):
        seed = rng.randrange(900000001)
        a, b = oracle.init(seed), reference.init(seed)
        assert a.tobytes() == b.tobytes()
        assert (oracle.step_n(a, 5000) == reference.step_n(b, 5000)).all()
        j = rng.getrandbits(rng.choice([10, 40, 64, 120, 140]))
        assert oracle.jump_state(a, j).tobytes() == reference.jump_state(a, j).tobytes()
    with pytest.raises(ValueError):
        reference.init(900000001)


def _cr_log(x: float) -> float:
    """log(x) correctly rounded to binary64 (mpmath at 200 bits, then one rounding)."""
    import mpmath
    with mpmath.workprec(200):
        return float(mpmath.log(mpmath.mpf(x)))


def _ulps(a: float, b: float) -> int:
    ia, ib = np.array([a, b]).view(np.int64)
    return abs(int(ia) - int(ib))


def test_crlog_tables_are_fresh():
    # the device and the oracle include the same generated constants
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "gen_crlog.py"), "--check"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_crlog_is_correctly_rounded(oracle):
    # gaussian()'s log (oracle or_crlog) against an exact reference (mpmath)
    import math
    rng = random.Random(9)
    xs = [rng.randrange(1, 2**46) * 2.0**-46 for _ in range(20000)]   # gaussian() domain
    xs += [(rng.randrange(-2**23, 2**23) ** 2 + rng.randrange(-2**23, 2**23) ** 2) / 2.0**46
           for _ in range(5000)]
    xs += [2.0**k for k in range(-46, 1)] + [1 - 2.0**-46, 1 - 2.0**-45, 2.0**-46 * 3,
                                            0.7071067811865476, 0.7071067811865475]
    # and off the domain: it is a general log for positive normal doubles
    xs += [math.ldexp(rng.random() + 0.5, rng.randrange(-1000, 1000)) for _ in range(3000)]
    xs += [1.0, 1 + 2.0**-52, 1.5, 2.0, 1e300, 3e-300]
    xs = [x for x in xs if x > 0]
    glibc_off = 0
    for x in xs:
        y = oracle.crlog(x)
        assert y == _cr_log(x), x
        d = _ulps(y, math.log(x))
        assert d <= 1  # glibc's log is correctly rounded but for rare 1-ulp misses
        glibc_off += d
    print(f"glibc log differs from the correctly rounded log on {glibc_off} of {len(xs)} inputs")


def test_crlog_accurate_phase_on_hard_inputs(oracle):
    # inputs the fast phase cannot decide (about 1 in 2^19) exercise the
    # accurate phase; the scan finds them in a few ranges of the domain
    rng = random.Random(3)
    hard = []
    for _ in range(12):
        s0 = rng.randrange(1, 2**46 - 2_000_000)
        n, fails = oracle.crlog_scan(s0, 2_000_000)
        hard += fails
    assert len(hard) > 10
    # the four domain inputs only the exception table decides (exhaustive
    # sweep, profiles/r2_crlog_sweep.json): within 2^-47 ulp of a midpoint
    for s in (22440254926254, 28850599726852, 31156142270051, 69163099561495):
        y, ok = oracle.crlog_accurate(s * 2.0**-46)
        assert ok and y == _cr_log(s * 2.0**-46)
    for s in hard:
        x = s * 2.0**-46
        y, ok = oracle.crlog_accurate(x)
        assert ok and y == _cr_log(x), s
        assert oracle.crlog_ex(x) == (y, False)
    # and where the fast phase decides, both phases agree
    for _ in range(3000):
        x = rng.randrange(1, 2**46) * 2.0**-46
        y, fast = oracle.crlog_ex(x)
        ya, ok = oracle.crlog_accurate(x)
        assert ok and ya == y


def test_gaussian_vs_glibc_form(oracle):
    # The repo's gaussian() = RanMars::gaussian's form with a correctly rounded
    # log. With glibc's log() instead, a deviate can move only where glibc's
    # log(rsq) is itself not correctly rounded (its 1-ulp error grows to at
    # most 3 ulp through -2 log / rsq, sqrt and v * fac); nowhere else.
    from oracle.bind import GAUSS_DTYPE
    n, per, steps = 4096, 3, 100
    st = oracle.make_streams(oracle.init(7), 2**50, n)
    g1 = np.zeros(n, GAUSS_DTYPE)
    g1["s"] = st
    g2 = g1.copy()
    a = oracle.gaussian_fill(g1, per, steps).reshape(-1)
    b, fl = oracle.gaussian_fill(g2, per, steps, libm_log=True, with_flags=True)
    b, fl = b.reshape(-1), fl.reshape(-1)
    d = np.abs(a.view(np.int64) - b.view(np.int64))
    assert (np.sign(a) == np.sign(b)).all()
    assert (d[fl == 0] == 0).all()
    assert d.max() <= 3
    print(f"glibc log misrounded for {int(fl.sum())} of {fl.size} deviates; "
          f"{np.count_nonzero(d == 1)} differ by 1 ulp, {np.count_nonzero(d == 2)} by 2")


def test_langevin_convention_statistics(oracle):
    # The repo's fix-langevin-style consumer (or_langevin): with v = 0 the force
    # is pure noise, f = g2 r. With rb.langevin_factors the uniform form
    # (variance 24/12) and the gaussian form (variance 2) both give the
    # fluctuation-dissipation variance 2 m kB T / (damp dt).
    import paper_2512_00093_b200 as rb
    from oracle.bind import GAUSS_DTYPE
    n = 20000
    mass, damp, dt, temp = 2.5, 0.2, 0.004, 1.7
    target = 2 * mass * temp / (damp * dt)
    for noise in (rb.NOISE_UNIFORM, rb.NOISE_GAUSSIAN):
        g = np.zeros(n, GAUSS_DTYPE)
        g["s"] = oracle.make_streams(oracle.init(7), 2**50, n)
        gf1, gf2 = rb.langevin_factors([0.0, mass], damp, dt, noise=noise)
        v = np.zeros((n, 3))
        f = np.zeros((n, 3))
        assert oracle.langevin(g, v, f, np.ones(n, np.int32), gf1, gf2, np.sqrt(temp), noise) == 0
        assert abs(f.mean()) < 0.05 * np.sqrt(target)
        assert abs(f.var() / target - 1) < 0.03
    # drag: with zero temperature the force is exactly gfactor1 * v
    g = np.zeros(8, GAUSS_DTYPE)
    g["s"] = oracle.make_streams(oracle.init(7), 2**50, 8)
    v = np.arange(24, dtype=np.float64).reshape(8, 3)
    f = np.zeros((8, 3))
    gf1, gf2 = rb.langevin_factors([0.0, mass], damp, dt)
    oracle.langevin(g, v, f, np.ones(8, np.int32), gf1, gf2, 0.0, rb.NOISE_UNIFORM)
    assert (f == gf1[1] * v).all()
    # atoms outside the group draw nothing
    g2 = g.copy()
    assert oracle.langevin(g2, v, f, np.ones(8, np.int32), gf1, gf2, 1.0, 0,
                           mask=np.zeros(8, np.int32), groupbit=1) == 0
    assert g2.tobytes() == g.tobytes()
