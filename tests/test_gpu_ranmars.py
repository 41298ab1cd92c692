"""§8f row 3 — the LAMMPS-style object (seed constructor, uniform(), gaussian(),
jump-ahead) and the warp-per-stream gaussian kernel behind it, against the
oracle's sequential calls on the same stream."""
import random

import numpy as np
import pytest

import paper_2512_00093_b200 as rb
from oracle.bind import GAUSS_DTYPE, STATE_DTYPE

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU-only module
    pytest.skip("needs a CUDA device", allow_module_level=True)


@pytest.fixture(autouse=True)
def _clean_status():
    rb.device_status(clear=True)
    yield
    torch.cuda.synchronize()
    assert rb.device_status(clear=True) == 0


def _gstates(n, seed, oracle, cache_every=3):
    rng = np.random.default_rng(seed)
    g = np.zeros(n, GAUSS_DTYPE)
    g["s"]["lane"] = rng.integers(0, 1 << 24, (n, 97), dtype=np.uint32)
    g["s"]["i"] = rng.integers(0, 97, n)
    g["s"]["j"] = (g["s"]["i"] + 97 - 64) % 97
    g["s"]["v"] = rng.integers(0, 16777213, n, dtype=np.uint32)
    g["has_saved"][::cache_every] = 1
    g["saved"][::cache_every] = rng.normal(size=len(g[::cache_every]))
    return g


@pytest.mark.parametrize("count", [1, 2, 3, 33, 64, 65, 1000, 4097])
def test_gaussian_stream_kernel(oracle, count):
    g = _gstates(9, count, oracle)
    d = torch.from_numpy(g.copy().view(np.int32).reshape(len(g), rb.GAUSS_WORDS)).cuda()
    out = rb.gaussian_stream(d, count).cpu().numpy()
    exp = oracle.gaussian_fill(g, count, 1)[0]  # [atom][c]
    assert (out.view(np.int64) == exp.view(np.int64)).all()
    assert d.cpu().numpy().view(GAUSS_DTYPE).reshape(-1).tobytes() == g.tobytes()


def test_ranmars_uniform_matches_reference_outputs(known):
    r = rb.RanMars(seed=12345)
    first = known["seed_outputs"][0]["first"]  # test_core.cpp:118-123
    assert [r.uniform() for _ in range(len(first))] == [u * 2.0**-24 for u in first]
    for _ in range(1_000_000 - len(first) - 1):
        r.uniform()
    assert r.uniform() == known["seed_12345_output_1000000"]["value"] * 2.0**-24


def test_ranmars_interleaved_calls(oracle):
    rng = random.Random(5)
    r = rb.RanMars(seed=4711, block=4096)
    og = np.zeros(1, GAUSS_DTYPE)
    og["s"] = oracle.init(4711)
    pattern = [("u", 5), ("g", 7), ("u", 3), ("g", 1), ("g", 2), ("u", 10), ("g", 300),
               ("u", 1), ("g", 3)] + [(rng.choice("ug"), rng.randrange(1, 700)) for _ in range(30)]
    for kind, n in pattern:
        for _ in range(n):
            if kind == "u":
                assert r.uniform() == oracle.uniform_call(og)
            else:
                assert r.gaussian() == oracle.gaussian_call(og)
        if rng.random() < 0.3:
            assert r.state().tobytes() == og.tobytes()
    assert r.state().tobytes() == og.tobytes()


def test_ranmars_jump_and_errors(oracle):
    r = rb.RanMars(seed=31415)
    r.gaussian()  # leaves a cached deviate
    r.jump(2**100)
    og = np.zeros(1, GAUSS_DTYPE)
    og["s"] = oracle.init(31415)
    oracle.gaussian_call(og)
    og["s"] = oracle.jump_state(np.ascontiguousarray(og["s"]), 2**100)
    assert r.gaussian() == oracle.gaussian_call(og)  # the cached one survives the jump
    assert r.uniform() == oracle.uniform_call(og)
    assert r.state().tobytes() == og.tobytes()
    with pytest.raises(ValueError):
        rb.RanMars(seed=900000001)  # init.hpp:19-20
    s = np.zeros(1, STATE_DTYPE)
    s[0] = oracle.init(1)[0]
    assert rb.RanMars(state=s).uniform() == oracle.step_n(oracle.init(1), 1)[0] * 2.0**-24
