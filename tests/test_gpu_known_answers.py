"""The reference's frozen unit-test answers (tests/golden/known_answers.json,
cited per case) reproduced through the DEVICE path: the same crafted states,
seeds and jumps as test_core.cpp, test_jump.cpp and test_float_reference.cpp,
run by the sm_100a kernels instead of the oracle."""
import numpy as np
import pytest

import paper_2512_00093_b200 as rb

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU-only module
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def test_crafted_step_on_device(oracle, known):
    k = known["crafted_step"]  # test_core.cpp:26-45
    s = oracle.init(12345)
    i, j = int(s["i"][0]), int(s["j"][0])
    s["lane"][0][i], s["lane"][0][j], s["v"] = k["lane_i"], k["lane_j"], k["v"]
    d = rb.states_to_device(s)
    assert _u32(rb.generate(d, 1, "u32"))[0] == k["out"]
    h = rb.states_to_host(d)
    assert h["lane"][0][i] == k["new_lane"] and h["v"][0] == k["new_v"]
    # equal operands give a zero difference (test_core.cpp "equal operands")
    s2 = oracle.init(7)
    s2["lane"][0][int(s2["j"][0])] = s2["lane"][0][int(s2["i"][0])]
    d2 = rb.states_to_device(s2)
    rb.generate(d2, 1, "u32")
    assert rb.states_to_host(d2)["lane"][0][int(s2["i"][0])] == 0


def test_seed_outputs_on_device(known):
    for case in known["seed_outputs"]:  # test_core.cpp:118-139
        d = rb.states_to_device(rb.init(case["seed"]))
        assert _u32(rb.generate(d, len(case["first"]), "u32")).tolist() == case["first"]
    d = rb.states_to_device(rb.init(12345))
    assert _u32(rb.generate_single(d, 1_000_000, "u32"))[-1] == \
        known["seed_12345_output_1000000"]["value"]


def test_jump_1e5_on_device(known):
    k = known["jump_1e5_seed_12345"]  # test_jump.cpp:123-132
    d = rb.jump_dev(rb.states_to_device(rb.init(k["seed"])), k["j"])
    assert _u32(rb.generate(d, len(k["next"]), "u32")).tolist() == k["next"]


def test_float_fixup_on_device(known):
    k = known["float_fixup"]  # test_float_reference.cpp:31-41
    f = np.zeros(1, rb.FLOAT_DTYPE)
    f["c"] = 362436 / 16777216
    f["i"], f["j"] = 96, 32
    f["x"][0][96], f["x"][0][32] = k["x_i"], k["x_j"]
    d = torch.from_numpy(f.view(np.uint8).reshape(1, -1).copy()).cuda()
    out = rb.generate_float(d, 1).cpu().numpy()
    assert out[0] == k["out_u24"] / 16777216
    back = d.cpu().numpy().view(rb.FLOAT_DTYPE).reshape(-1)
    assert back["x"][0][96] == k["stored"]
