"""§8f rows 3-4 — the fix-langevin-style per-atom consumer (K6 langevin_kernel)
and gaussian()'s in-place path for few deviates per launch, bit-exact against
the oracle's restatement (or_langevin / or_gaussian_fill)."""
import numpy as np
import pytest

import paper_2512_00093_b200 as rb
from oracle.bind import GAUSS_DTYPE, STATE_DTYPE

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU-only module
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _atoms(n, seed, oracle, cache_every=0):
    rng = np.random.default_rng(seed)
    s = np.zeros(n, STATE_DTYPE)
    s["lane"] = rng.integers(0, 1 << 24, (n, 97), dtype=np.uint32)
    s["i"] = rng.integers(0, 97, n)
    s["j"] = (s["i"] + 97 - 64) % 97
    s["v"] = rng.integers(0, 16777213, n, dtype=np.uint32)
    g = np.zeros(n, GAUSS_DTYPE)
    g["s"] = s
    if cache_every:
        g["has_saved"][::cache_every] = 1
        g["saved"][::cache_every] = rng.normal(size=len(g[::cache_every]))
    v = rng.normal(size=(n, 3))
    f = rng.normal(size=(n, 3))
    return g, v, f, rng


def _dev(g):
    return torch.from_numpy(g.copy().view(np.int32).reshape(len(g), rb.GAUSS_WORDS)).cuda()


@pytest.mark.parametrize("noise", [rb.NOISE_UNIFORM, rb.NOISE_GAUSSIAN])
@pytest.mark.parametrize("n", [1, 37, 1000, 4099])
def test_langevin_matches_oracle(oracle, noise, n):
    g, v, f, rng = _atoms(n, 100 + n + noise, oracle, cache_every=3)
    mass = np.array([0.0, 1.0, 12.011, 39.948])
    gf1, gf2 = rb.langevin_factors(mass, t_period=0.1, dt=0.005, noise=noise)
    types = rng.integers(1, 4, n).astype(np.int32)
    mask = rng.integers(0, 4, n).astype(np.int32)  # groupbit 2: about half the atoms
    tsqrt = np.sqrt(1.5)
    dg, dv, df = _dev(g), torch.from_numpy(v).cuda(), torch.from_numpy(f.copy()).cuda()
    dt_, dm = torch.from_numpy(types).cuda(), torch.from_numpy(mask).cuda()
    d1, d2 = torch.from_numpy(gf1).cuda(), torch.from_numpy(gf2).cuda()
    fo = f.copy()
    for step in range(5):  # chained MD steps: states and caches carry over
        rb.langevin(dg, dv, df, dt_, d1, d2, tsqrt, noise, mask=dm, groupbit=2)
        assert oracle.langevin(g, v, fo, types, gf1, gf2, tsqrt, noise, mask=mask, groupbit=2) == 0
        assert df.cpu().numpy().tobytes() == fo.tobytes(), step
    gh = dg.cpu().numpy().view(GAUSS_DTYPE).reshape(-1)
    assert gh.tobytes() == g.tobytes()  # states, cursors, cached deviates
    assert rb.device_status() == 0


def test_langevin_without_mask_and_config5_shape(oracle):
    # config 5's stream layout (make_streams(7, 2^50), one stream per atom),
    # every atom in the group, one type
    n = 2048
    states = rb.make_streams(7, 2**50, n)
    dg = rb.gauss_states_from(states)
    g = np.zeros(n, GAUSS_DTYPE)
    g["s"] = rb.states_to_host(states)
    rng = np.random.default_rng(5)
    v = rng.normal(size=(n, 3))
    f = np.zeros((n, 3))
    types = np.ones(n, np.int32)
    gf1, gf2 = rb.langevin_factors([0.0, 1.0], t_period=1.0, dt=0.01, noise=rb.NOISE_GAUSSIAN)
    df = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
    rb.langevin(dg, torch.from_numpy(v).cuda(), df, torch.from_numpy(types).cuda(),
                torch.from_numpy(gf1).cuda(), torch.from_numpy(gf2).cuda(), 1.0,
                rb.NOISE_GAUSSIAN)
    oracle.langevin(g, v, f, types, gf1, gf2, 1.0, rb.NOISE_GAUSSIAN)
    assert df.cpu().numpy().tobytes() == f.tobytes()
    # the noise part equals gfactor2 * gaussian() of the same streams
    g2 = np.zeros(n, GAUSS_DTYPE)
    g2["s"] = rb.states_to_host(states)
    gauss = oracle.gaussian_fill(g2, 3, 1)[0]
    drag = gf1[1] * v
    assert np.allclose(f - drag, gf2[1] * gauss, rtol=1e-12, atol=1e-15)


def test_langevin_bad_type_flagged(oracle):
    g, v, f, _ = _atoms(64, 9, oracle)
    types = np.ones(64, np.int32)
    types[17] = 5  # n_types = 3
    gf1, gf2 = rb.langevin_factors([0.0, 1.0, 2.0, 3.0], 1.0, 0.01)
    dg, df = _dev(g), torch.from_numpy(f.copy()).cuda()
    rb.device_status(clear=True)
    rb.langevin(dg, torch.from_numpy(v).cuda(), df, torch.from_numpy(types).cuda(),
                torch.from_numpy(gf1).cuda(), torch.from_numpy(gf2).cuda(), 1.0)
    assert rb.device_status(clear=True) & 4
    fo = f.copy()
    assert oracle.langevin(g, v, fo, types, gf1, gf2, 1.0, 0) == 1
    assert df.cpu().numpy().tobytes() == fo.tobytes()  # the other atoms were updated
    with pytest.raises(ValueError):
        rb.langevin(dg, torch.from_numpy(v).cuda(), df, torch.from_numpy(types).cuda(),
                    torch.from_numpy(gf1).cuda(), torch.from_numpy(gf2).cuda(), 1.0, noise=7)


@pytest.mark.parametrize("per_step,steps", [(1, 1), (3, 1), (1, 8), (4, 3), (13, 1), (2, 7)])
def test_gaussian_inplace_boundary(oracle, per_step, steps):
    # gaussian() launches of <= 12 deviates per atom step the states in place
    # (K6); 13+ stage the ring (K4). Both must equal the oracle, cache included.
    g, _, _, _ = _atoms(301, per_step * 10 + steps, oracle, cache_every=2)
    dg = _dev(g)
    for _ in range(3):
        out = rb.gaussian(dg, per_step, steps).cpu().numpy()
        exp = oracle.gaussian_fill(g, per_step, steps)
        assert out.tobytes() == exp.tobytes()
    assert dg.cpu().numpy().view(GAUSS_DTYPE).reshape(-1).tobytes() == g.tobytes()


@pytest.mark.parametrize("n", [1, 300, 4099])
def test_stream_bank_round_trip_and_langevin(oracle, n):
    # bank layout (ranmar_bank_*): to_states(from_states(S), t) is byte-identical
    # to t calls of step(); langevin_bank equals the AoS consumer (uniform
    # noise, no mask) bit for bit, across the slot wrap at t = 97
    g, v, f, rng = _atoms(n, 500 + n, oracle)
    states = torch.from_numpy(g["s"].copy().view(np.int32).reshape(n, rb.STATE_WORDS)).cuda()
    bank = rb.bank_from_states(states)
    assert torch.equal(rb.bank_to_states(bank, 0), states)
    mass = np.array([0.0, 1.0, 4.0])
    gf1, gf2 = rb.langevin_factors(mass, 0.2, 0.01)
    types = rng.integers(1, 3, n).astype(np.int32)
    dv, df = torch.from_numpy(v).cuda(), torch.from_numpy(f.copy()).cuda()
    dt_, d1, d2 = torch.from_numpy(types).cuda(), torch.from_numpy(gf1).cuda(), torch.from_numpy(gf2).cuda()
    fo = f.copy()
    t = 0
    for step in range(40):  # 120 outputs per stream: the slots wrap past 97
        t = rb.langevin_bank(bank, t, dv, df, dt_, d1, d2, 1.3)
        oracle.langevin(g, v, fo, types, gf1, gf2, 1.3, rb.NOISE_UNIFORM)
    assert t == 120
    assert df.cpu().numpy().tobytes() == fo.tobytes()
    back = rb.bank_to_states(bank, t).cpu().numpy().view(STATE_DTYPE).reshape(-1)
    assert back.tobytes() == g["s"].tobytes()
    assert rb.device_status() == 0


def test_stream_bank_bad_type_keeps_lockstep(oracle):
    g, v, f, _ = _atoms(64, 77, oracle)
    states = torch.from_numpy(g["s"].copy().view(np.int32).reshape(64, rb.STATE_WORDS)).cuda()
    bank = rb.bank_from_states(states)
    types = np.ones(64, np.int32)
    types[5] = 9
    gf1, gf2 = rb.langevin_factors([0.0, 1.0], 0.2, 0.01)
    df = torch.from_numpy(f.copy()).cuda()
    rb.device_status(clear=True)
    rb.langevin_bank(bank, 0, torch.from_numpy(v).cuda(), df, torch.from_numpy(types).cuda(),
                     torch.from_numpy(gf1).cuda(), torch.from_numpy(gf2).cuda(), 1.0)
    assert rb.device_status(clear=True) & 4
    assert df[5].cpu().numpy().tobytes() == f[5].tobytes()  # force untouched
    back = rb.bank_to_states(bank, 3).cpu().numpy().view(STATE_DTYPE).reshape(-1)
    s5 = g["s"][5:6].copy()
    oracle.step_n(s5, 3)  # the stream still advanced by 3
    assert back[5:6].tobytes() == s5.tobytes()


@pytest.mark.parametrize("n", [37, 4099])
def test_langevin_with_pregenerated_noise(oracle, n):
    # one gaussian() launch for all T steps (K4, per_step 3), then one element-wise
    # consumer per MD step: forces and final states equal the in-place gaussian path
    # and the oracle step by step (every atom in the group)
    g, v, f, rng = _atoms(n, 900 + n, oracle, cache_every=5)
    mass = np.array([0.0, 1.0, 12.011])
    gf1, gf2 = rb.langevin_factors(mass, t_period=0.1, dt=0.005, noise=rb.NOISE_GAUSSIAN)
    types = rng.integers(1, 3, n).astype(np.int32)
    tsqrt = np.sqrt(1.5)
    steps = 7
    dv, dt_ = torch.from_numpy(v).cuda(), torch.from_numpy(types).cuda()
    d1, d2 = torch.from_numpy(gf1).cuda(), torch.from_numpy(gf2).cuda()
    dg_a, df_a = _dev(g), torch.from_numpy(f.copy()).cuda()  # pre-generated noise
    dg_b, df_b = _dev(g), torch.from_numpy(f.copy()).cuda()  # in place
    noise = rb.gaussian(dg_a, 3, steps)                     # [steps, n, 3]
    fo = f.copy()
    for step in range(steps):
        rb.langevin_noise(noise[step], dv, df_a, dt_, d1, d2, tsqrt)
        rb.langevin(dg_b, dv, df_b, dt_, d1, d2, tsqrt, rb.NOISE_GAUSSIAN)
        assert oracle.langevin(g, v, fo, types, gf1, gf2, tsqrt, rb.NOISE_GAUSSIAN) == 0
        assert df_a.cpu().numpy().tobytes() == fo.tobytes(), step
        assert torch.equal(df_a, df_b), step
    assert torch.equal(dg_a, dg_b)
    assert dg_a.cpu().numpy().view(GAUSS_DTYPE).reshape(-1).tobytes() == g.tobytes()
    assert rb.device_status() == 0
    # a type outside [0, n_types] is flagged and that atom keeps its force
    bad = dt_.clone()
    bad[n // 2] = 9
    f0 = df_a.clone()
    rb.langevin_noise(noise[0], dv, df_a, bad, d1, d2, tsqrt)
    assert rb.device_status(clear=True) != 0 and torch.equal(df_a[n // 2], f0[n // 2])
