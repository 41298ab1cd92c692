"""GPU parity: the sm_100a kernels, called through the C ABI, against the oracle
(oracle/ranmar_oracle.c, itself pinned to the reference) and the reference's
golden vectors. Integer/byte results must be bit-exact; gaussian() must be
within the north star's 1 ulp of RanMars::gaussian's form (it is 0 ulp: both
sides use the correctly rounded log; vs glibc's log() the deviates differ only
where glibc misrounds)."""
import os
import random

import numpy as np
import pytest

import paper_2512_00093_b200 as rb
from oracle.bind import STATE_DTYPE
from ranmar_testutil import state_from_json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU-only module
    pytest.skip("needs a CUDA device", allow_module_level=True)


@pytest.fixture(autouse=True)
def _clean_status():
    rb.device_status(clear=True)
    yield
    torch.cuda.synchronize()
    assert rb.device_status(clear=True) == 0, "a kernel flagged an invalid state"


def random_states(n, seed, oracle):
    """Valid states with random lanes and random cursor phase (test_util.hpp:20-27)."""
    rng = np.random.default_rng(seed)
    s = np.zeros(n, STATE_DTYPE)
    s["lane"] = rng.integers(0, 1 << 24, (n, 97), dtype=np.uint32)
    s["i"] = rng.integers(0, 97, n)
    s["j"] = (s["i"] + 97 - 64) % 97
    s["v"] = rng.integers(0, 16777213, n, dtype=np.uint32)
    return s


# ---------------------------------------------------------------- K3 jump

def test_pow_t_mod_golden(refvec):
    for case in refvec["pow_t_mod"]:
        got = rb.pow_t_mod_dev(int(case["j"])).cpu().numpy().view(np.uint32)
        assert got.tolist() == case["coeff"], case["j"]


def test_jump_golden(refvec):
    for case in refvec["jump_state"]:
        got = rb.jump_state(state_from_json(case["in"]), int(case["j"]))
        assert got.tobytes() == state_from_json(case["out"]).tobytes(), case["j"]


def test_jump_matches_stepping(oracle):
    # acceptance.cpp:94-108: J <= 10^4 against literal stepping, random states.
    base = random_states(40, 1, oracle)
    d = rb.states_to_device(base)
    for j in (0, 1, 2, 33, 64, 97, 98, 1000, 10_000):
        got = rb.states_to_host(rb.jump_dev(d, j))
        for k in range(len(base)):
            a = base[k:k + 1].copy()
            oracle.step_n(a, j)
            b = got[k:k + 1].copy()
            assert (oracle.step_n(a, 100) == oracle.step_n(b, 100)).all(), (j, k)
            assert got[k:k + 1].tobytes() == oracle.jump_state(base[k:k + 1], j).tobytes()


def test_jump_large_and_additive(oracle):
    base = random_states(300, 2, oracle)
    d = rb.states_to_device(base)
    rng = random.Random(3)
    for j in [2**40, 2**64 - 1, 2**120, 2**120 - 1, rng.getrandbits(141)]:
        got = rb.states_to_host(rb.jump_dev(d, j))
        for k in range(0, len(base), 37):
            assert got[k:k + 1].tobytes() == oracle.jump_state(base[k:k + 1], j).tobytes()
    # additivity (acceptance.cpp:110-118): (2^64-1) twice == 2^65-2 once
    big = 2**64 - 1
    twice = rb.jump_dev(rb.jump_dev(d, big), big)
    once = rb.jump_dev(d, 2**65 - 2)
    assert torch.equal(twice, once)
    # in place
    d2 = d.clone()
    rb.jump_dev(d2, 12345, out=d2)
    assert torch.equal(d2, rb.jump_dev(d, 12345))


def test_jump_commutes_with_stepping(oracle):
    # test_jump.cpp "jumping commutes with stepping", on the device: step n then
    # jump J == jump J then step n (compared through the next outputs, since a
    # stepped ring is rotated and a jumped one renormalised)
    base = random_states(64, 11, oracle)
    for n, j in ((1, 2**40), (97, 12345), (1000, 2**120 - 1)):
        a = rb.states_to_device(base)
        rb.generate(a, n, "u32")
        a = rb.jump_dev(a, j)
        b = rb.jump_dev(rb.states_to_device(base), j)
        rb.generate(b, n, "u32")
        assert torch.equal(rb.generate(a, 500, "u32"), rb.generate(b, 500, "u32")), (n, j)


def test_make_streams_golden(refvec):
    for case in refvec["make_streams"]:
        got = rb.states_to_host(rb.make_streams(case["seed"], int(case["j"]), len(case["states"])))
        for g, e in zip(got, case["states"]):
            assert g.tobytes() == state_from_json(e).tobytes()


@pytest.mark.parametrize("n,first", [(1, 0), (2, 0), (127, 0), (128, 0), (129, 0), (300, 0),
                                     (1000, 0), (200, 5), (257, 1000), (1, 77),
                                     (300, (1 << 40) + 3), (129, (1 << 61) - 200)])
def test_make_streams_shapes(oracle, n, first):
    base = oracle.init(12345)
    got = rb.states_to_host(rb.make_streams_dev(base, 2**40, n, first=first))
    exp = oracle.make_streams(base, 2**40, n, first=first)
    assert got.tobytes() == exp.tobytes()


def test_make_streams_from_phased_base(oracle):
    # a base with a non-fresh cursor phase: stream 0 is the base verbatim
    base = oracle.init(4711)
    oracle.step_n(base, 40)
    got = rb.states_to_host(rb.make_streams_dev(base, 1000, 300))
    assert got.tobytes() == oracle.make_streams(base, 1000, 300).tobytes()


def test_make_streams_tiling(oracle):
    # acceptance.cpp:195-206: stream blocks tile the base sequence
    streams = rb.states_to_host(rb.make_streams(97531, 1000, 10))
    base = oracle.step_n(oracle.init(97531), 10_000)
    tiled = np.concatenate([oracle.step_n(streams[k:k + 1].copy(), 1000) for k in range(10)])
    assert (tiled == base).all()


def test_make_streams_errors():
    with pytest.raises(ValueError):
        rb.make_streams(1, 5, 0)  # jump.hpp:111
    with pytest.raises(ValueError):
        rb.make_streams(1, 0, 3)  # jump.hpp:112
    with pytest.raises(ValueError):
        rb.make_streams(900000001, 5, 3)  # init.hpp:19-20


def test_config3_full(refvec):
    # BASELINE config 3 at full size: 2^20 stream starts at J = 2^120.
    c3 = refvec["c3_starts"]
    base = rb.init_unchecked(c3["seed"])
    n = 1 << 20
    d = rb.make_streams_dev(base, int(c3["j"]), n)
    host = rb.states_to_host(d)
    for k, e in zip(c3["k"], c3["states"]):
        assert host[k:k + 1].tobytes() == state_from_json(e).tobytes(), k
    # size-independent property: s_{k+1} = jump(s_k, J) for every k
    nxt = rb.jump_dev(d[:-1], int(c3["j"]))
    assert torch.equal(nxt, d[1:])


# ---------------------------------------------------------- K1 generation

@pytest.mark.parametrize("fmt", ["u32", "f32", "f64"])
@pytest.mark.parametrize("per_stream", [0, 1, 5, 31, 32, 33, 96, 97, 98, 128, 129, 1000, 4103])
def test_generate_shapes(oracle, fmt, per_stream):
    base = np.concatenate([oracle.init(12345), random_states(13, per_stream + 7, oracle)])
    d = rb.states_to_device(base)
    out = rb.generate(d, per_stream, fmt).cpu().numpy()
    exp_states = base.copy()
    exp_u = oracle.generate_u32(exp_states, per_stream)
    if fmt == "u32":
        assert (out.view(np.uint32) == exp_u).all()
    elif fmt == "f32":
        assert (out == (exp_u.astype(np.float64) * 2.0**-24).astype(np.float32)).all()
    else:
        assert (out == exp_u.astype(np.float64) * 2.0**-24).all()
    # states advance exactly as step() leaves them (ring, cursors, v)
    assert rb.states_to_host(d).tobytes() == exp_states.tobytes()


def test_config1_integer_and_float(refvec, oracle):
    # BASELINE config 1: one stream, seed 12345, 10^8 uniforms; integer path vs
    # the reference summary, f32 path vs the float recurrence (float_ranmar.hpp).
    c = refvec["c1_seed12345_1e8"]
    d = rb.states_to_device(oracle.init(12345))
    u = rb.generate(d, 10**8, "u32")
    u64 = u.to(torch.int64) & 0xFFFFFFFF
    assert int(u64.sum()) == c["sum"]
    x = 0
    for chunk in u64.split(1 << 24):
        x ^= int(np.bitwise_xor.reduce(chunk.cpu().numpy()))
    assert x == c["xor"] and int(u64[-1]) == c["last"]
    assert rb.states_to_host(d).tobytes() == state_from_json(c["final_state"]).tobytes()
    d2 = rb.states_to_device(oracle.init(12345))
    f = rb.generate(d2, 10**8, "f32")
    assert torch.equal((f.double() * 2.0**24).to(torch.int64), u64)
    fl = oracle.float_outputs(12345, 10**6)
    assert (f[:10**6].cpu().numpy().astype(np.float64) == fl).all()


@pytest.mark.parametrize("count", [1, 97, 8192, 8193, 20000, 1_000_007])
def test_generate_single_equals_one_warp(oracle, count):
    # one stream split into 8,192-output substreams: same outputs as the
    # single-warp path, and the state ends byte-identical to count x step()
    base = random_states(1, count, oracle)
    a = rb.states_to_device(base)
    b = rb.states_to_device(base)
    for fmt in ("u32", "f32"):
        ua = rb.generate(a, count, fmt)
        ub = rb.generate_single(b, count, fmt)
        assert torch.equal(ua, ub), fmt
        assert torch.equal(a, b), fmt  # states after 2 x count outputs, same layout


def test_config1_single_stream_full_width(refvec, oracle):
    # config 1 (one stream, 10^8) through the split path: the reference's summary
    c = refvec["c1_seed12345_1e8"]
    d = rb.states_to_device(oracle.init(12345))
    u64 = rb.generate_single(d, 10**8, "u32").to(torch.int64) & 0xFFFFFFFF
    assert int(u64.sum()) == c["sum"] and int(u64[-1]) == c["last"]
    assert rb.states_to_host(d).tobytes() == state_from_json(c["final_state"]).tobytes()


def test_config2_scaled(oracle):
    # config 2 at 1/256 of the streams: make_streams(12345, 2^40, 256), 65536 fp32 each
    states = rb.make_streams(12345, 2**40, 256)
    out = rb.generate(states, 65536, "f32").cpu().numpy()
    exp_states = oracle.make_streams(oracle.init(12345), 2**40, 256)
    exp = oracle.generate_f32(exp_states, 65536)
    assert (out == exp).all()
    assert rb.states_to_host(states).tobytes() == exp_states.tobytes()


def test_config2_full(refvec):
    # config 2 at full size (2^32 fp32 = 16 GiB): per-stream sums of the stored
    # values against the reference's (a checksum of checksums).
    c = refvec["c2_full"]
    n, per = c["n"], c["per_stream"]
    states = rb.make_streams(c["seed"], int(c["j"]), n)
    out = rb.generate(states, per, "f32")
    sums = torch.empty(n, dtype=torch.int64, device="cuda")
    for k0 in range(0, n, 4096):
        blk = out[k0 * per:(k0 + 4096) * per].view(4096, per)
        sums[k0:k0 + 4096] = (blk.double() * 2.0**24).to(torch.int64).sum(dim=1)
    s = sums.cpu().numpy().astype(object)
    assert int(sum(s)) == c["total_sum"]
    assert [int(x) for x in s[:8]] == c["first_sums"]
    assert sum((k + 1) * int(x) for k, x in enumerate(s)) & ((1 << 64) - 1) == c["weighted_digest"]
    del out


# --------------------------------------------------------------- K2 consume

@pytest.mark.parametrize("per_stream", [0, 1, 31, 4096, 100_003])
def test_consume_shapes(oracle, per_stream):
    base = random_states(9, per_stream, oracle)
    d = rb.states_to_device(base)
    sums, hist = rb.consume(d, per_stream)
    es = base.copy()
    exp_sums, exp_hist = oracle.consume(es, per_stream)
    assert (sums.cpu().numpy().view(np.uint64) == exp_sums).all()
    assert (hist.cpu().numpy().view(np.uint32) == exp_hist).all()
    assert rb.states_to_host(d).tobytes() == es.tobytes()


def test_consume_flush_path(oracle):
    # > 65535 rounds per lane forces the u16 private counters to flush
    per = 32 * 65535 + 77
    base = random_states(2, 5, oracle)
    d = rb.states_to_device(base)
    sums, hist = rb.consume(d, per)
    es = base.copy()
    exp_sums, exp_hist = oracle.consume(es, per)
    assert (sums.cpu().numpy().view(np.uint64) == exp_sums).all()
    assert (hist.cpu().numpy().view(np.uint32) == exp_hist).all()


def test_config4_head(refvec):
    c = refvec["c4_head"]
    d = rb.make_streams(c["seed"], int(c["j"]), len(c["sums"]))
    sums, hist = rb.consume(d, c["per_stream"])
    assert sums.cpu().numpy().view(np.uint64).tolist() == c["sums"]
    assert hist.cpu().numpy().view(np.uint32).tolist() == c["hist"]


# -------------------------------------------------------------- K4 gaussian

def ulp_diff(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    ia = a.view(np.int64)
    ib = b.view(np.int64)
    ia = np.where(ia < 0, np.int64(-0x8000000000000000) - ia, ia)
    ib = np.where(ib < 0, np.int64(-0x8000000000000000) - ib, ib)
    return np.abs(ia - ib)


def test_gaussian_within_one_ulp(oracle):
    from oracle.bind import GAUSS_DTYPE
    n, per, steps = 2000, 3, 100
    states = rb.make_streams(7, 2**50, n)
    g = rb.gauss_states_from(states)
    out = rb.gaussian(g, per, steps).cpu().numpy()
    og = np.zeros(n, GAUSS_DTYPE)
    og["s"] = rb.states_to_host(states)
    exp = oracle.gaussian_fill(og, per, steps)
    d = ulp_diff(out.reshape(-1), exp.reshape(-1))
    print(f"gaussian max ulp {d.max()}, differing {np.count_nonzero(d)} of {d.size}")
    assert d.max() <= 1  # north-star tolerance
    assert d.max() == 0  # correctly rounded log on both sides: bit-exact
    og2 = np.zeros(n, GAUSS_DTYPE)
    og2["s"] = rb.states_to_host(states)
    libm, flags = oracle.gaussian_fill(og2, per, steps, libm_log=True, with_flags=True)
    d2 = ulp_diff(out.reshape(-1), libm.reshape(-1))
    print(f"vs the glibc-log() form: max ulp {d2.max()}, differing {np.count_nonzero(d2)}")
    # deviates move only where glibc's own log(rsq) is misrounded
    # (glibc's 1-ulp log error grows to at most 3 ulp through /rsq, sqrt and v*fac)
    assert (d2[flags.reshape(-1) == 0] == 0).all() and d2.max() <= 3
    gh = g.cpu().numpy().view(GAUSS_DTYPE).reshape(-1)
    assert gh["s"].tobytes() == og["s"].tobytes()
    assert (gh["has_saved"] == og["has_saved"]).all()


def test_crlog_sweep_matches_oracle(oracle):
    # the device's correctly rounded log on a slice of gaussian()'s domain:
    # every input the fast phase leaves undecided is decided by the accurate
    # phase, both phases agree where the fast one decides (mode 1), and the
    # undecided inputs equal the oracle's list (the same IEEE sequence)
    import random
    rng = random.Random(11)
    for _ in range(4):
        s0 = rng.randrange(1, 2**46 - 2**27)
        nf, nacc, nmis, fails = rb.crlog_sweep(s0, 2**27, mode=1)
        assert nacc == 0 and nmis == 0
        n2, exp = oracle.crlog_scan(s0, 2**27)
        assert nf == n2 and fails == sorted(exp)
    # a long slice in mode 0 (the mode of the full sweep, tools/crlog_sweep.py)
    nf, nacc, nmis, fails = rb.crlog_sweep(2**45, 2**36, mode=0)
    assert nacc == 0 and nf == len(fails)
    for s in fails[:200]:
        y, ok = oracle.crlog_accurate(s * 2.0**-46)
        assert ok


def test_fp64_fast_paths_match_library():
    # gaussian()'s branch-free divide / sqrt (csrc/gauss_math.cuh) against
    # __ddiv_rn / __dsqrt_rn on 2^28 operand sets rsq = s / 2^46 (bitwise)
    assert rb.fp64_selfcheck(1 << 28, seed=12345) == 0
    assert rb.fp64_selfcheck(1 << 20, seed=7) == 0


def test_gaussian_odd_count_keeps_cache(oracle):
    from oracle.bind import GAUSS_DTYPE
    states = rb.make_streams(7, 2**50, 64)
    g = rb.gauss_states_from(states)
    og = np.zeros(64, GAUSS_DTYPE)
    og["s"] = rb.states_to_host(states)
    for _ in range(3):  # 1 call per step: the cached deviate carries across launches
        out = rb.gaussian(g, 1, 5).cpu().numpy()
        exp = oracle.gaussian_fill(og, 1, 5)
        assert ulp_diff(out.reshape(-1), exp.reshape(-1)).max() <= 1
    gh = g.cpu().numpy().view(GAUSS_DTYPE).reshape(-1)
    assert (gh["has_saved"] == og["has_saved"]).all()
    assert gh.tobytes() == og.tobytes()  # states, cursors, cached deviate


@pytest.mark.parametrize("count", [1, 2, 13, 300, 1001])
def test_gaussian_moments_consumer(oracle, count):
    # §8f row 4: gaussian() consumed in-kernel (K4 without stores): per atom the
    # sum and sum of squares of its `count` deviates in call order (cached one
    # first), bit-exact against sequential sums of the oracle's deviates; states
    # and caches advance exactly as a gaussian() call of the same length
    from oracle.bind import GAUSS_DTYPE
    n = 70
    og = np.zeros(n, GAUSS_DTYPE)
    og["s"] = random_states(n, 9100 + count, oracle)
    og["has_saved"][::4] = 1
    og["saved"][::4] = np.linspace(-1.5, 1.5, len(og[::4]))
    g = torch.from_numpy(og.copy().view(np.int32).reshape(n, rb.GAUSS_WORDS)).cuda()
    mom = rb.gaussian_moments(g, count).cpu().numpy()
    exp = oracle.gaussian_fill(og, count, 1).reshape(n, count)
    s1 = np.cumsum(exp, axis=1)[:, -1]
    s2 = np.cumsum(exp * exp, axis=1)[:, -1]
    assert mom[:, 0].tobytes() == s1.tobytes() and mom[:, 1].tobytes() == s2.tobytes()
    gh = g.cpu().numpy().view(GAUSS_DTYPE).reshape(-1)
    assert gh.tobytes() == og.tobytes()
    assert rb.device_status(clear=True) == 0


@pytest.mark.parametrize("per_step,steps", [(1, 1), (2, 3), (3, 100), (7, 40), (300, 2), (257, 1),
                                            (5, 77)])
def test_gaussian_shapes(oracle, per_step, steps):
    # chunking of the staged output, odd/even deviate counts, the unstaged path
    # (per_step > 256), atoms not a multiple of the block, random cursor phase
    # and a pre-filled cache on some atoms.
    from oracle.bind import GAUSS_DTYPE
    n = 37
    base = random_states(n, per_step * 1000 + steps, oracle)
    og = np.zeros(n, GAUSS_DTYPE)
    og["s"] = base
    og["has_saved"][::3] = 1
    og["saved"][::3] = np.linspace(-2, 2, len(og[::3]))
    g = torch.from_numpy(og.copy().view(np.int32).reshape(n, rb.GAUSS_WORDS)).cuda()
    out = rb.gaussian(g, per_step, steps).cpu().numpy()
    exp = oracle.gaussian_fill(og, per_step, steps)
    assert ulp_diff(out.reshape(-1), exp.reshape(-1)).max() == 0
    gh = g.cpu().numpy().view(GAUSS_DTYPE).reshape(-1)
    assert gh.tobytes() == og.tobytes()


# ------------------------------------------------------ invariants, host API

def test_zero_sized_calls_are_no_ops(oracle):
    # n = 0 or zero outputs per stream: OK, nothing launched on garbage, states unchanged
    d = rb.states_to_device(random_states(3, 4, oracle))
    d0 = d.clone()
    empty = d[:0]
    assert rb.generate(empty, 100, "u32").numel() == 0
    assert rb.generate(d, 0, "f32").numel() == 0
    sums, hist = rb.consume(d, 0)
    assert int(sums.abs().sum()) == 0 and int(hist.abs().sum()) == 0
    assert rb.jump_dev(empty, 2**40).numel() == 0
    g = rb.gauss_states_from(d)
    assert rb.gaussian(g, 3, 0).numel() == 0 and rb.gaussian(g[:0], 3, 5).numel() == 0
    assert torch.equal(d, d0) and torch.equal(g[:, :rb.STATE_WORDS], d0)
    f = torch.zeros((0, 3), dtype=torch.float64, device="cuda")
    gf = torch.zeros(2, dtype=torch.float64, device="cuda")
    rb.langevin(g[:0], f, f, torch.zeros(0, dtype=torch.int32, device="cuda"), gf, gf, 1.0)
    text, off = rb.to_text_dev(empty)
    assert off.numel() == 1 and int(off[0]) == 0 and rb.texts_to_host(text, off) == []
    torch.cuda.synchronize()
    assert rb.device_status() == 0


def test_bad_state_is_flagged(oracle):
    s = oracle.init(1)
    s["j"] = 0  # separation != 64
    d = rb.states_to_device(s)
    rb.generate(d, 64, "u32")
    torch.cuda.synchronize()
    assert rb.device_status(clear=True) & 1


def test_invalid_device_states_are_flagged_not_overrun(oracle):
    # states with unmasked lanes, a huge v or bad cursors must not
    # make the text kernels write past text_bound(n) or the jump kernels read
    # outside the record; each raises the status bit instead
    good = oracle.make_streams(oracle.init(5), 2**40, 6)
    bad = good.copy()
    bad[1]["lane"][7] = 0xFFFFFFFF
    bad[2]["v"] = 0xFFFFFFFF
    bad[3]["i"], bad[3]["j"] = 1 << 30, 5
    bad[4]["i"] = -7
    d = rb.states_to_device(bad)
    text, off = rb.to_text_dev(d)
    torch.cuda.synchronize()
    assert rb.device_status(clear=True) & 1
    o = off.cpu().numpy()
    assert int(o[-1]) <= text.numel()
    lens = np.diff(o)
    assert (lens[1:5] == 0).all() and lens[0] > 0 and lens[5] > 0
    texts = rb.texts_to_host(text, off)
    assert texts[0] == oracle.to_text(good[0:1]) and texts[5] == oracle.to_text(good[5:6])
    for k in (1, 2, 3, 4):
        rb.jump_dev(d[k:k + 1], 2**70)
        torch.cuda.synchronize()
        assert rb.device_status(clear=True) & 1, k
    one = d[3:4].clone()
    rb.generate_single(one, 50000, "u32")  # device-resident base: flagged, not trusted
    torch.cuda.synchronize()
    assert rb.device_status(clear=True) & 1
    assert torch.equal(one, d[3:4])  # an invalid state is left untouched
    ctx = rb.Context()
    with pytest.raises(rb.RanmarError):
        ctx.generate(bad[1:2].copy(), 10, "u32")  # host path: RANMAR_ESTATE (lanes > 2^24 - 1)
    ctx.close()


@pytest.mark.parametrize("n,first", [(1, 0), (129, 0), (70000, 0), (5000, 123457)])
def test_tensor_core_bulk_equals_imad_bulk(n, first):
    # make_streams' level 0 runs on the tensor cores (bulk_tc_kernel, u8 limbs,
    # kind::i8); RANMAR_BULK=imad selects the IMAD kernel. Both must give the
    # same states bit for bit (the config-3 golden vectors pin them further).
    import subprocess
    import sys
    code = (f"import sys; sys.path.insert(0, {ROOT!r}); import numpy as np, paper_2512_00093_b200 as rb; "
            f"s = rb.make_streams_dev(rb.init_unchecked(987654321), 2**120, {n}, first={first}); "
            f"np.save(sys.argv[1], rb.states_to_host(s).view(np.uint32))")
    outs = []
    for mode in ("tc", "imad"):
        path = f"/tmp/bulk_{mode}_{n}.npy"
        env = dict(os.environ, RANMAR_BULK=mode)
        r = subprocess.run([sys.executable, "-c", code, path], env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
    assert outs[0].tobytes() == outs[1].tobytes()


def test_host_buffer_context(oracle):
    ctx = rb.Context(0)
    ss = ctx.make_streams(12345, 2**40, 300)
    exp = oracle.make_streams(oracle.init(12345), 2**40, 300)
    assert ss.tobytes() == exp.tobytes()
    out = ctx.generate(ss, 1000, "f32")
    eo = oracle.generate_f32(exp, 1000)
    assert (out == eo).all() and ss.tobytes() == exp.tobytes()
    h2d, d2h = ctx.traffic()
    assert h2d == 300 * 400 and d2h == 300 * 1000 * 4 + 300 * 400
    sums, hist = ctx.consume(ss, 4096)
    es, eh = oracle.consume(exp, 4096)
    assert (sums == es).all() and (hist == eh).all()
    jumped = ctx.jump(ss, 2**120)
    assert jumped[5:6].tobytes() == oracle.jump_state(exp[5:6], 2**120).tobytes()
    with pytest.raises(ValueError):
        ctx.make_streams(900000001, 5, 2)
    ctx.close()


def test_make_streams_dense_jump_counts_and_determinism(oracle):
    # Jump counts with ~half their bits set exercise every product path of the
    # square-table exponentiation and the offset tables; repeated runs must be
    # byte-identical (a cheap race detector: compute-sanitizer is unavailable).
    rng = random.Random(17)
    base = oracle.init(2024)
    for bits in (37, 64, 131):
        j = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
        ref = None
        for _ in range(4):
            got = rb.states_to_host(rb.make_streams_dev(base, j, 300, first=11))
            if ref is None:
                ref = got
                exp = oracle.make_streams(base, j, 300, first=11)
                assert got.tobytes() == exp.tobytes(), bits
            assert got.tobytes() == ref.tobytes()
        assert rb.pow_t_mod_dev(j).cpu().numpy().view(np.uint32).tolist() == \
            oracle.pow_t_mod(j).tolist()


@pytest.mark.parametrize("n", [127, 128, 129, 300, 4099])
def test_batched_jump_tensor_core_path(oracle, n):
    # batches of >= 128 states run apply_tc_kernel (u8-limb kind::i8 MMAs with the
    # states' extensions in TMEM); 127 stays on the IMAD kernel: both vs the oracle,
    # with random cursor phases, a dense jump count and one invalid state flagged
    base = random_states(n, 1000 + n, oracle)
    d = rb.states_to_device(base)
    for j in (2**120, 3**80 + 12345):
        got = rb.states_to_host(rb.jump_dev(d, j))
        for k in list(range(0, n, max(1, n // 97))) + [n - 1]:
            assert got[k:k + 1].tobytes() == oracle.jump_state(base[k:k + 1], j).tobytes(), (n, j, k)
    assert rb.device_status(clear=True) == 0
    bad = base.copy()
    bad["lane"][n // 2, 5] = 1 << 24  # a lane above 24 bits
    rb.jump_dev(rb.states_to_device(bad), 2**40)
    assert rb.device_status(clear=True) != 0
    bad = base.copy()
    bad["i"][n - 1] = 1000  # a cursor outside the ring: flagged, reads stay inside the record
    rb.jump_dev(rb.states_to_device(bad), 2**40)
    assert rb.device_status(clear=True) != 0


@pytest.mark.parametrize("per_step,steps", [(1, 25), (2, 13), (3, 100), (3, 7), (4, 7), (6, 5), (6, 3)])
def test_gaussian_row_batched_stores(oracle, per_step, steps):
    # per_step dividing 2K: warps whose lanes start without a cached deviate store
    # whole output rows per batch; a second launch starts from the cache an odd
    # deviate count leaves (the countdown path), atoms not a multiple of the block
    from oracle.bind import GAUSS_DTYPE
    n = 100
    og = np.zeros(n, GAUSS_DTYPE)
    og["s"] = random_states(n, 7000 + 10 * per_step + steps, oracle)
    g = torch.from_numpy(og.copy().view(np.int32).reshape(n, rb.GAUSS_WORDS)).cuda()
    for _ in range(2):
        out = rb.gaussian(g, per_step, steps).cpu().numpy()
        exp = oracle.gaussian_fill(og, per_step, steps)
        assert ulp_diff(out.reshape(-1), exp.reshape(-1)).max() == 0
    gh = g.cpu().numpy().view(GAUSS_DTYPE).reshape(-1)
    assert gh.tobytes() == og.tobytes()


@pytest.mark.parametrize("first", [0, 12345, (1 << 40) + 3])
def test_make_streams_three_level_tree(oracle, first):
    # n > 128^2: level 2 on the IMAD level kernel, level 1 and level 0 on the tensor
    # cores, with a stream offset (multi-rank ranges) and a phased base state
    base = oracle.init(4711)
    oracle.step_n(base, 40)
    n = 20000
    got = rb.states_to_host(rb.make_streams_dev(base, 2**40, n, first=first))
    for k in (0, 1, 127, 128, 129, 16383, 16384, 16385, n - 1):
        exp = oracle.make_streams(base, 2**40, 1, first=first + k)
        assert got[k:k + 1].tobytes() == exp.tobytes(), (first, k)
    assert rb.device_status(clear=True) == 0
