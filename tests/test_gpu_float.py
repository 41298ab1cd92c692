"""K5 — the classic floating-point RANMAR (reference/float_ranmar.hpp Algorithm 1)
on the GPU: bit-exact against the oracle's restatement of step_float and equal to
the integer path / 2^24 (config 1: "10^8 uniforms via integer and float
recurrence")."""
import numpy as np
import pytest

import paper_2512_00093_b200 as rb

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU-only module
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _dev(f):
    return torch.from_numpy(np.ascontiguousarray(f).view(np.uint8).reshape(len(f), -1).copy()).cuda()


def _host(t):
    return t.cpu().numpy().view(rb.FLOAT_DTYPE).reshape(-1)


def test_init_float_matches_reference(refvec):
    # init_float = the float image of init (test_init.cpp:67-79 equivalence)
    for case in refvec["seeds"]:
        f = rb.init_float(case["seed"])
        assert (f["x"][0] == np.array(case["state"]["lane"], np.float64) * 2.0**-24).all()
        assert f["c"][0] == 362436 / 16777216 and f["i"][0] == 96 and f["j"][0] == 32
    with pytest.raises(ValueError):
        rb.init_float(900000001)


@pytest.mark.parametrize("per_stream", [0, 1, 31, 32, 33, 97, 1000, 4103])
def test_float_recurrence_shapes(oracle, per_stream):
    seeds = [0, 1, 97, 12345, 900000000, 31415]
    f = np.concatenate([rb.init_float(s) for s in seeds])
    d = _dev(f)
    out = rb.generate_float(d, per_stream).cpu().numpy().reshape(len(seeds), per_stream)
    for k, s in enumerate(seeds):
        assert (out[k] == oracle.float_outputs(s, per_stream)).all(), s
    # advanced state: continuing on the device == continuing the oracle
    more = rb.generate_float(d, 50).cpu().numpy().reshape(len(seeds), 50)
    for k, s in enumerate(seeds):
        assert (more[k] == oracle.float_outputs(s, per_stream + 50)[per_stream:]).all()
    h = _host(d)
    assert ((h["c"] >= 0) & (h["c"] < 16777213 / 16777216)).all()


def test_config1_float_recurrence_full(oracle):
    # 10^8 outputs of seed 12345 through the device float recurrence equal the
    # device integer recurrence / 2^24 (itself pinned to the reference's summary
    # in test_config1_integer_and_float) and the oracle's step_float prefix.
    f = _dev(rb.init_float(12345))
    out = rb.generate_float(f, 10**8)
    u = rb.generate(rb.states_to_device(oracle.init(12345)), 10**8, "u32")
    assert torch.equal(out, (u.to(torch.int64) & 0xFFFFFFFF).double() * 2.0**-24)
    assert (out[:10**6].cpu().numpy() == oracle.float_outputs(12345, 10**6)).all()
