"""CPU-only checks of the C-ABI library: it loads without a GPU, exports every
symbol include/ranmar_b200.h declares, and its host-side entry points (seed
expansion, jump-count parsing, closed-form arithmetic jump, text state) match
the oracle and the reference's frozen answers, with the reference's error
behaviour (ValueError where ranmar throws std::invalid_argument)."""
import ctypes
import os
import random
import re

import numpy as np
import pytest

import paper_2512_00093_b200 as rb
from ranmar_testutil import state_from_json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "ranmar_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ranmar_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(rb.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert rb.lib().ranmar_abi_version() == 2


def test_sm100a_cubin_present():
    # The product library carries sm_100a SASS (no PTX JIT, no other arch).
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", rb.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_init_matches_oracle_and_range(oracle, known):
    rng = random.Random(1)
    for seed in [0, 1, 12345, 900000000] + [rng.randrange(900000001) for _ in range(50)]:
        assert rb.init(seed).tobytes() == oracle.init(seed).tobytes()
    with pytest.raises(ValueError):
        rb.init(900000001)  # init.hpp:19-20
    s = rb.init(12345)
    for idx, val in known["init_lanes"][0]["lanes"].items():
        assert s["lane"][0][int(idx)] == val
    # config 3's seed: rejected by init, available through the unchecked expansion
    assert rb.init_unchecked(987654321).tobytes() == oracle.init(987654321, checked=False).tobytes()


def test_value_of():
    assert rb.value_of(0) == 0.0
    assert rb.value_of(0xFFFFFF) == 16777215.0 / 16777216.0
    assert rb.value_of(1 << 23) == 0.5
    with pytest.raises(ValueError):
        rb.value_of(1 << 24)  # core.hpp:76-77


def test_parse_jump_count(known):
    pj = known["parse_jump_count"]
    for text, val in pj["ok"]:
        assert rb.parse_jump_count(text) == val
    for text in pj["bad"]:
        with pytest.raises(ValueError):
            rb.parse_jump_count(text)
    assert rb.parse_jump_count("2^255") == 1 << 255
    assert rb.parse_jump_count("2^256-1") == (1 << 256) - 1
    with pytest.raises(rb.RanmarError):
        rb.parse_jump_count("2^256")  # beyond the ABI's 256-bit jump counts


def test_jump_arith(known, oracle):
    for j, v in known["jump_arith"]["cases"]:
        assert rb.jump_arith(known["jump_arith"]["v"], j) == v
    rng = random.Random(2)
    for _ in range(200):
        v, j = rng.randrange(16777213), rng.getrandbits(rng.choice([8, 64, 130, 200]))
        assert rb.jump_arith(v, j) == oracle.jump_arith(v, j)
    with pytest.raises(ValueError):
        rb.jump_arith(1, -3)  # jump.hpp:80-81


def test_text_round_trip(refvec):
    for case in refvec["to_text"]:
        s = state_from_json(case["state"])
        assert rb.to_text(s) == case["text"]
        assert rb.from_text(case["text"]).tobytes() == s.tobytes()
    good = refvec["to_text"][0]["text"]
    for bad in [good.replace("ranmar24 v1", "ranmar24 v2"), good.replace("i 97 j 33", "i 97 j 34"),
                good.replace("v 362436", "v 16777213"), good + "junk", good[: len(good) // 2],
                good.replace("u 2 ", "u 3 ")]:
        with pytest.raises(ValueError):
            rb.from_text(bad)


def test_device_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(rb.RanmarError):
        rb.make_streams(1, 1000, 4)
    # ctx creation reports a CUDA error instead of computing anything on the CPU
    with pytest.raises(rb.RanmarError):
        rb.Context(0)


def test_device_entry_points_validate_arguments_first():
    # argument errors are reported as RANMAR_EINVAL before any device work, so
    # they behave the same with or without a GPU (the reference throws
    # std::invalid_argument at the same places, jump.hpp:111-112)
    import ctypes as C
    lib = rb.lib()
    EINVAL = rb.EINVAL
    vp = C.c_void_p(0x1000)  # never dereferenced: the checks come first
    assert lib.ranmar_generate_u32_dev(None, 4, 4, vp, None) == EINVAL
    assert lib.ranmar_generate_f32_dev(vp, 4, 4, None, None) == EINVAL
    assert lib.ranmar_consume_dev(vp, 4, 4, None, vp, None) == EINVAL
    assert lib.ranmar_gaussian_f64_dev(None, 4, 3, 2, vp, None) == EINVAL
    assert lib.ranmar_gaussian_moments_dev(vp, 4, 3, None, None) == EINVAL
    assert lib.ranmar_langevin_dev(vp, 4, vp, vp, vp, None, 1, vp, vp, 1, 1.0, 7, None) == EINVAL
    assert lib.ranmar_langevin_dev(vp, 4, vp, vp, vp, None, 1, vp, vp, -1, 1.0, 0, None) == EINVAL
    assert lib.ranmar_langevin_dev(vp, 4, None, vp, vp, None, 1, vp, vp, 1, 1.0, 0, None) == EINVAL
    assert lib.ranmar_langevin_noise_dev(4, None, vp, vp, vp, None, 1, vp, vp, 1, 1.0, None) == EINVAL
    assert lib.ranmar_langevin_noise_dev(4, vp, vp, vp, vp, None, 1, vp, vp, -1, 1.0, None) == EINVAL
    s = rb.init(1)
    j = rb._JumpCount()
    assert lib.ranmar_make_streams_dev(s.ctypes.data, C.byref(j), 0, 4, vp, vp, 1 << 20,
                                       None) == EINVAL  # J = 0 (jump.hpp:112)
    j.limb[0] = 5
    assert lib.ranmar_make_streams_dev(s.ctypes.data, C.byref(j), 0, 0, vp, vp, 1 << 20,
                                       None) == EINVAL  # n = 0 (jump.hpp:111)
    assert lib.ranmar_last_error().decode()  # every failure leaves a message
    j.limb[0], j.limb[3] = 0, 1 << 62  # J = 2^254: stream 4 would need 2^256
    assert lib.ranmar_make_streams_dev(s.ctypes.data, C.byref(j), 0, 5, vp, vp, 1 << 30,
                                       None) == rb.ERANGE
    assert lib.ranmar_make_streams_dev(s.ctypes.data, C.byref(j), 0, 4, vp, vp, 16,
                                       None) == rb.ENOMEM  # workspace too small
