"""B200-native RANMAR (arXiv 2512.00093) behind the reference's interface.

Python mirror of the reference library's API (/root/reference/proj/include/
ranmar, namespace ``ranmar``) over the C ABI in ``include/ranmar_b200.h``
(``lib/libranmar_b200.so``, sm_100a kernels). Same names, same argument
meaning, and ``ValueError`` wherever the reference throws
``std::invalid_argument``. Device buffers are torch CUDA tensors; torch is
only plumbing (allocation, streams), never the compute path.

There is no CPU fallback: the generation / jump entry points need the built
library and a CUDA device and raise ``RuntimeError`` otherwise.
"""
from __future__ import annotations

import ctypes as C
import enum
import functools
import os
from typing import Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libranmar_b200.so")

# ranmar::RanmarState (core.hpp:29-49) == ranmar_state: 400 bytes.
STATE_DTYPE = np.dtype([("lane", "<u4", (97,)), ("i", "<i4"), ("j", "<i4"), ("v", "<u4")])
GAUSS_DTYPE = np.dtype([("s", STATE_DTYPE), ("saved", "<f8"), ("has_saved", "<u4"), ("pad", "<u4")])
STATE_WORDS = 100
GAUSS_WORDS = 104
# ranmar::reference::FloatState (float_ranmar.hpp:22-29): 792 bytes.
FLOAT_DTYPE = np.dtype([("x", "<f8", (97,)), ("c", "<f8"), ("i", "<i4"), ("j", "<i4")])

long_lag, short_lag, word_bits = 97, 33, 24             # core.hpp:17-19
word_mask = 0x00FFFFFF                                  # core.hpp:20
arith_mod, arith_delta, arith_start = 16777213, 7654321, 362436  # core.hpp:22-24
max_seed = 900000000                                    # init.hpp:16

OK, EINVAL, ERANGE, ECUDA, ESTATE, ENOMEM = range(6)


class StreamMode(enum.Enum):
    """jump.hpp:101-104. Both modes produce identical states."""
    incremental = 0
    independent = 1


class RanmarError(RuntimeError):
    pass


class _JumpCount(C.Structure):
    _fields_ = [("limb", C.c_uint64 * 4)]


_lib = None


def lib() -> C.CDLL:
    """Loads the CUDA library (fails loudly if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `make lib` "
                           f"(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    vp, u32, u64, i32, sz = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_size_t
    jp = C.POINTER(_JumpCount)
    sig = {
        "ranmar_abi_version": (i32, []),
        "ranmar_last_error": (C.c_char_p, []),
        "ranmar_init": (i32, [u32, vp]),
        "ranmar_init_unchecked": (i32, [u32, vp]),
        "ranmar_value_of": (i32, [u32, C.POINTER(C.c_double)]),
        "ranmar_parse_jump_count": (i32, [C.c_char_p, jp]),
        "ranmar_jump_arith": (i32, [u32, jp, C.POINTER(C.c_uint32)]),
        "ranmar_to_text": (C.c_long, [vp, C.c_char_p, C.c_long]),
        "ranmar_from_text": (i32, [C.c_char_p, vp]),
        "ranmar_make_streams_workspace": (sz, [u64]),
        "ranmar_device_setup": (i32, [i32, vp]),
        "ranmar_make_streams_dev": (i32, [vp, jp, u64, u64, vp, vp, sz, vp]),
        "ranmar_make_streams_from_dev": (i32, [vp, jp, u64, u64, vp, vp, sz, vp]),
        "ranmar_jump_dev": (i32, [vp, vp, u64, jp, vp, sz, vp]),
        "ranmar_pow_t_mod_dev": (i32, [jp, vp, vp]),
        "ranmar_generate_u32_dev": (i32, [vp, u64, u64, vp, vp]),
        "ranmar_generate_f32_dev": (i32, [vp, u64, u64, vp, vp]),
        "ranmar_generate_f64_dev": (i32, [vp, u64, u64, vp, vp]),
        "ranmar_consume_dev": (i32, [vp, u64, u64, vp, vp, vp]),
        "ranmar_gaussian_f64_dev": (i32, [vp, u64, u64, u64, vp, vp]),
        "ranmar_gaussian_moments_dev": (i32, [vp, u64, u64, vp, vp]),
        "ranmar_fp64_selfcheck_dev": (i32, [u64, u64, vp, vp]),
        "ranmar_crlog_sweep_dev": (i32, [u64, u64, i32, vp, vp, u64, vp]),
        "ranmar_bank_words": (u64, [u64]),
        "ranmar_generate_single_workspace": (sz, [u64]),
        "ranmar_generate_single_u32_dev": (i32, [vp, u64, vp, vp, sz, vp]),
        "ranmar_generate_single_f32_dev": (i32, [vp, u64, vp, vp, sz, vp]),
        "ranmar_bank_from_states_dev": (i32, [vp, u64, vp, vp]),
        "ranmar_bank_to_states_dev": (i32, [vp, u64, u64, vp, vp]),
        "ranmar_langevin_bank_dev": (i32, [vp, u64, u64, vp, vp, vp, vp, vp, i32, C.c_double, vp]),
        "ranmar_langevin_noise_dev": (i32, [u64, vp, vp, vp, vp, vp, i32, vp, vp, i32, C.c_double, vp]),
        "ranmar_langevin_dev": (i32, [vp, u64, vp, vp, vp, vp, i32, vp, vp, i32, C.c_double,
                                      i32, vp]),
        "ranmar_device_status": (i32, [C.POINTER(C.c_uint32), i32]),
        "ranmar_kernel_launches": (u64, []),
        "ranmar_ctx_create": (i32, [i32, C.POINTER(vp)]),
        "ranmar_ctx_destroy": (None, [vp]),
        "ranmar_ctx_make_streams": (i32, [vp, u32, jp, u64, u64, vp]),
        "ranmar_ctx_jump": (i32, [vp, vp, vp, u64, jp]),
        "ranmar_ctx_generate_u32": (i32, [vp, vp, u64, u64, vp]),
        "ranmar_ctx_generate_f32": (i32, [vp, vp, u64, u64, vp]),
        "ranmar_ctx_consume": (i32, [vp, vp, u64, u64, vp, vp]),
        "ranmar_gaussian_stream_f64_dev": (i32, [vp, u64, u64, vp, vp]),
        "ranmar_init_float": (i32, [u32, vp]),
        "ranmar_generate_float_dev": (i32, [vp, u64, u64, vp, vp]),
        "ranmar_to_text_bound": (u64, [u64]),
        "ranmar_text_workspace": (sz, [u64]),
        "ranmar_to_text_dev": (i32, [vp, u64, vp, u64, vp, vp, sz, vp]),
        "ranmar_from_text_dev": (i32, [vp, vp, u64, vp, vp, vp]),
        "ranmar_ctx_gaussian_stream": (i32, [vp, vp, u64, u64, vp]),
        "ranmar_ctx_last_traffic": (i32, [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    _lib = L
    return L


def _check(rc: int):
    if rc == OK:
        return
    msg = lib().ranmar_last_error().decode()
    if rc == EINVAL:
        raise ValueError(msg)
    raise RanmarError(f"[{rc}] {msg}")


def _jc(j) -> _JumpCount:
    """int (or text accepted by parse_jump_count) -> C jump count."""
    if isinstance(j, str):
        j = parse_jump_count(j)
    j = int(j)
    if j < 0:
        raise ValueError("ranmar: jump count must be nonnegative")  # polyring.hpp:115-116
    if j >= 1 << 256:
        raise RanmarError("ranmar: jump count exceeds 2^256 - 1")
    out = _JumpCount()
    for k in range(4):
        out.limb[k] = (j >> (64 * k)) & ((1 << 64) - 1)
    return out


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RanmarError("no CUDA device: the B200 kernels are the only implementation")
    return torch


def _dptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


_ready = set()


def device_setup(device: Optional[int] = None) -> None:
    """ranmar_device_setup: the one-time per-device resources of the _dev entry
    points (status word, table of squares). Called automatically by every
    device function below; call it yourself before capturing a CUDA graph."""
    torch = _torch()
    dev = torch.cuda.current_device() if device is None else int(device)
    if dev not in _ready:
        with torch.cuda.device(dev):
            s = torch.cuda.current_stream(dev)
            _check(lib().ranmar_device_setup(dev, C.c_void_p(s.cuda_stream)))
        _ready.add(dev)


def _on_device(fn):
    """Run a device function on the device of its first CUDA tensor argument (or
    the current device), set up, and with that device current; the caller's
    current device is restored afterwards (the C ABI works on the current device)."""
    @functools.wraps(fn)
    def wrap(*args, **kw):
        torch = _torch()
        dev = None
        for a in (*args, *kw.values()):
            if isinstance(a, torch.Tensor) and a.is_cuda:
                dev = a.device.index
                break
        if dev is None:
            dev = torch.cuda.current_device()
        device_setup(dev)
        with torch.cuda.device(dev):
            return fn(*args, **kw)
    return wrap


# ----------------------------------------------------------------- host side

def init(seed: int) -> np.ndarray:
    """ranmar::init (init.hpp:18-51). Returns a 1-element STATE_DTYPE array."""
    if not 0 <= seed < 1 << 32:
        raise ValueError("ranmar: seed must be in [0, 900000000]")
    s = np.zeros(1, STATE_DTYPE)
    _check(lib().ranmar_init(seed, _ptr(s)))
    return s


def init_unchecked(seed: int) -> np.ndarray:
    """Seed expansion without init()'s range check (BASELINE config 3's seed)."""
    s = np.zeros(1, STATE_DTYPE)
    _check(lib().ranmar_init_unchecked(seed, _ptr(s)))
    return s


def init_float(seed: int) -> np.ndarray:
    """reference::init_float (float_ranmar.hpp:50-80) -> 1-element FLOAT_DTYPE array."""
    if not 0 <= seed < 1 << 32:
        raise ValueError("ranmar: seed must be in [0, 900000000]")
    f = np.zeros(1, FLOAT_DTYPE)
    _check(lib().ranmar_init_float(seed, _ptr(f)))
    return f


@_on_device
def generate_float(fstates, per_stream: int, out=None, stream=None):
    """per_stream calls of reference::step_float (Algorithm 1, binary64) per float
    state (uint8 CUDA tensor [n, 792]), advanced in place -> float64 [n * per_stream]."""
    torch = _torch()
    n = fstates.shape[0]
    if out is None:
        out = torch.empty(n * per_stream, dtype=torch.float64, device="cuda")
    _check(lib().ranmar_generate_float_dev(_dptr(fstates), n, per_stream, _dptr(out),
                                           _stream_ptr(stream)))
    return out


def value_of(u24: int) -> float:
    """ranmar::value_of (core.hpp:75-79)."""
    out = C.c_double()
    _check(lib().ranmar_value_of(u24, C.byref(out)))
    return out.value


def parse_jump_count(text: str) -> int:
    """ranmar::parse_jump_count (jumpcount.hpp:16-47)."""
    j = _JumpCount()
    _check(lib().ranmar_parse_jump_count(text.encode(), C.byref(j)))
    return sum(int(j.limb[k]) << (64 * k) for k in range(4))


def jump_arith(v: int, j) -> int:
    """ranmar::jump_arith(ArithState{v}, J).v (jump.hpp:79-86)."""
    out = C.c_uint32()
    jc = _jc(j)
    _check(lib().ranmar_jump_arith(v, C.byref(jc), C.byref(out)))
    return out.value


def to_text(state: np.ndarray) -> str:
    """ranmar::to_text (serialize.hpp:21-40)."""
    buf = C.create_string_buffer(4096)
    n = lib().ranmar_to_text(_ptr(np.ascontiguousarray(state, STATE_DTYPE)), buf, 4096)
    if n < 0:
        raise RanmarError("to_text buffer too small")
    return buf.value.decode()


def from_text(text: str) -> np.ndarray:
    """ranmar::from_text (serialize.hpp:81-136)."""
    s = np.zeros(1, STATE_DTYPE)
    _check(lib().ranmar_from_text(text.encode(), _ptr(s)))
    return s


# ---------------------------------------------------------------- device side

def _stream_ptr(stream) -> C.c_void_p:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def states_to_device(states: np.ndarray, device="cuda"):
    """STATE_DTYPE array -> int32 CUDA tensor [n, 100] (same bytes)."""
    torch = _torch()
    a = np.ascontiguousarray(states, STATE_DTYPE).view(np.int32).reshape(-1, STATE_WORDS)
    return torch.from_numpy(a.copy()).to(device)


def states_to_host(t) -> np.ndarray:
    """int32 CUDA tensor [n, 100] -> STATE_DTYPE array."""
    return t.detach().cpu().contiguous().numpy().view(STATE_DTYPE).reshape(-1)


@_on_device
def make_streams_dev(base: np.ndarray, j, n: int, first: int = 0, out=None, workspace=None,
                     stream=None):
    """Streams [first, first+n) of make_streams(base, J) (jump.hpp:108-124) on the GPU.
    Returns an int32 CUDA tensor [n, 100] of ranmar_state records."""
    torch = _torch()
    if n == 0:
        raise ValueError("ranmar: need at least one stream")
    jc = _jc(j)
    if out is None:
        out = torch.empty((n, STATE_WORDS), dtype=torch.int32, device="cuda")
    wsb = lib().ranmar_make_streams_workspace(n)
    if workspace is None or workspace.numel() < wsb:
        workspace = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    b = np.ascontiguousarray(base, STATE_DTYPE).reshape(-1)[:1]
    _check(lib().ranmar_make_streams_dev(_ptr(b), C.byref(jc), first, n, _dptr(out),
                                         _dptr(workspace), workspace.numel(), _stream_ptr(stream)))
    return out


@_on_device
def make_streams(seed: int, block_length, n_streams: int,
                 mode: StreamMode = StreamMode.incremental, first: int = 0):
    """ranmar::make_streams(seed, J, n, mode) (jump.hpp:108-124), computed on the GPU.
    Returns a CUDA tensor of states; `mode` does not change the result."""
    if n_streams == 0:
        raise ValueError("ranmar: need at least one stream")
    if int(block_length) < 1:
        raise ValueError("ranmar: block length must be >= 1")
    return make_streams_dev(init(seed), block_length, n_streams, first=first)


@_on_device
def jump_dev(states, j, out=None, stream=None):
    """out[k] = jump_state(states[k], J) (jump.hpp:90-95)."""
    torch = _torch()
    jc = _jc(j)
    n = states.shape[0]
    if out is None:
        out = torch.empty_like(states)
    ws = torch.empty(4096, dtype=torch.uint8, device="cuda")
    _check(lib().ranmar_jump_dev(_dptr(states), _dptr(out), n, C.byref(jc), _dptr(ws), 4096,
                                 _stream_ptr(stream)))
    return out


def jump_state(state: np.ndarray, j) -> np.ndarray:
    """ranmar::jump_state on one host state, computed on the GPU."""
    return states_to_host(jump_dev(states_to_device(state), j))


@_on_device
def pow_t_mod_dev(j, stream=None):
    """ranmar::poly::pow_t_mod<24>(J) (polyring.hpp:113-124) -> int32 CUDA tensor [97]."""
    torch = _torch()
    jc = _jc(j)
    out = torch.empty(97, dtype=torch.int32, device="cuda")
    _check(lib().ranmar_pow_t_mod_dev(C.byref(jc), _dptr(out), _stream_ptr(stream)))
    return out


_GEN = {"u32": ("ranmar_generate_u32_dev", "int32"), "f32": ("ranmar_generate_f32_dev", "float32"),
        "f64": ("ranmar_generate_f64_dev", "float64")}


@_on_device
def generate(states, per_stream: int, fmt: str = "f32", out=None, stream=None):
    """per_stream x step() per stream (core.hpp:54-72), states advanced in place.
    Returns the stream-major output [n * per_stream] (u32 outputs as int32)."""
    torch = _torch()
    fn, dt = _GEN[fmt]
    n = states.shape[0]
    if out is None:
        out = torch.empty(n * per_stream, dtype=getattr(torch, dt), device="cuda")
    _check(getattr(lib(), fn)(_dptr(states), n, per_stream, _dptr(out), _stream_ptr(stream)))
    return out


@_on_device
def consume(states, per_stream: int, sums=None, hist=None, stream=None):
    """Per-stream u64 sum of the 24-bit outputs and 256-bin histogram of u >> 16."""
    torch = _torch()
    n = states.shape[0]
    if sums is None:
        sums = torch.empty(n, dtype=torch.int64, device="cuda")
    if hist is None:
        hist = torch.empty((n, 256), dtype=torch.int32, device="cuda")
    _check(lib().ranmar_consume_dev(_dptr(states), n, per_stream, _dptr(sums), _dptr(hist),
                                    _stream_ptr(stream)))
    return sums, hist


@_on_device
def gaussian(gstates, per_step: int, steps: int, out=None, stream=None):
    """steps x per_step gaussian() calls per atom -> out[step, atom, c] (float64)."""
    torch = _torch()
    n = gstates.shape[0]
    if out is None:
        out = torch.empty((steps, n, per_step), dtype=torch.float64, device="cuda")
    _check(lib().ranmar_gaussian_f64_dev(_dptr(gstates), n, per_step, steps, _dptr(out),
                                         _stream_ptr(stream)))
    return out


@_on_device
def gaussian_moments(gstates, count: int, out=None, stream=None):
    """count gaussian() calls per atom consumed in-kernel -> out[atom] = (sum, sum of
    squares) in call order (float64 [n, 2]); states advance as gaussian(g, count, 1)."""
    torch = _torch()
    n = gstates.shape[0]
    if out is None:
        out = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    if count == 0:
        out.zero_()
        return out
    _check(lib().ranmar_gaussian_moments_dev(_dptr(gstates), n, count, _dptr(out), _stream_ptr(stream)))
    return out


NOISE_UNIFORM, NOISE_GAUSSIAN = 0, 1


def langevin_factors(mass, t_period: float, dt: float, noise: int = NOISE_UNIFORM,
                     boltz: float = 1.0, mvv2e: float = 1.0, ftm2v: float = 1.0):
    """Per-type (gfactor1, gfactor2) of a Langevin thermostat (Schneider-Stoll
    form as used by fix langevin): drag -m / damp and a random force whose
    variance matches 2 m kB T / (damp dt) — 24 kB T m / (damp dt) for the
    uniform(-1/2, 1/2) noise (variance 1/12), 2 kB T m / (damp dt) for
    gaussian noise. mass is indexed by type (entry 0 unused in LAMMPS)."""
    m = np.asarray(mass, dtype=np.float64)
    c = 24.0 if noise == NOISE_UNIFORM else 2.0
    g1 = -m / t_period / ftm2v
    g2 = np.sqrt(m) * np.sqrt(c * boltz / t_period / dt / mvv2e) / ftm2v
    return np.ascontiguousarray(g1), np.ascontiguousarray(g2)


@_on_device
def langevin(gstates, v, f, types, gfactor1, gfactor2, tsqrt: float, noise: int = NOISE_UNIFORM,
             mask=None, groupbit: int = 1, stream=None):
    """Fix-langevin-style consumer on CUDA tensors: for atoms in the group,
    f[a, d] += gfactor1[t] * v[a, d] + gfactor2[t] * tsqrt * r with
    r = uniform() - 0.5 or gaussian() from atom a's stream (ranmar_langevin_dev).
    v, f: float64 [n, 3]; types: int32 [n]; gfactor*: float64 [n_types + 1]."""
    n = gstates.shape[0]
    for t, dt in ((v, "float64"), (f, "float64"), (gfactor1, "float64"), (gfactor2, "float64")):
        if str(t.dtype) != "torch." + dt or not t.is_contiguous():
            raise ValueError("langevin: v, f, gfactor1, gfactor2 must be contiguous float64")
    if tuple(v.shape) != (n, 3) or tuple(f.shape) != (n, 3) or types.shape[0] != n:
        raise ValueError("langevin: v, f must be [n_atoms, 3] and types [n_atoms]")
    if gfactor1.shape != gfactor2.shape:
        raise ValueError("langevin: gfactor1 and gfactor2 differ in length")
    _check(lib().ranmar_langevin_dev(_dptr(gstates), n, _dptr(v), _dptr(f), _dptr(types),
                                     None if mask is None else _dptr(mask), groupbit,
                                     _dptr(gfactor1), _dptr(gfactor2), gfactor1.shape[0] - 1,
                                     float(tsqrt), noise, _stream_ptr(stream)))
    return f


@_on_device
def langevin_noise(noise, v, f, types, gfactor1, gfactor2, tsqrt: float, mask=None, groupbit: int = 1,
                   stream=None):
    """The fix-langevin-style force update with this step's gaussian noise
    already drawn: noise float64 [n, 3] (e.g. gaussian(g, 3, steps)[step]),
    f[a, d] += gfactor1[t] * v[a, d] + gfactor2[t] * tsqrt * noise[a, d]
    (ranmar_langevin_noise_dev). Step by step equal to langevin(...,
    NOISE_GAUSSIAN) when every atom is in the group at every step."""
    n = v.shape[0]
    for t, dt in ((noise, "float64"), (v, "float64"), (f, "float64"), (gfactor1, "float64"),
                  (gfactor2, "float64")):
        if str(t.dtype) != "torch." + dt or not t.is_contiguous():
            raise ValueError("langevin_noise: noise, v, f, gfactor1, gfactor2 must be contiguous float64")
    if tuple(noise.shape) != (n, 3) or tuple(f.shape) != (n, 3) or types.shape[0] != n:
        raise ValueError("langevin_noise: noise, v, f must be [n_atoms, 3] and types [n_atoms]")
    if gfactor1.shape != gfactor2.shape:
        raise ValueError("langevin_noise: gfactor1 and gfactor2 differ in length")
    _check(lib().ranmar_langevin_noise_dev(n, _dptr(noise), _dptr(v), _dptr(f), _dptr(types),
                                           None if mask is None else _dptr(mask), groupbit,
                                           _dptr(gfactor1), _dptr(gfactor2), gfactor1.shape[0] - 1,
                                           float(tsqrt), _stream_ptr(stream)))
    return f


@_on_device
def generate_single(state, count: int, fmt: str = "f32", out=None, stream=None):
    """count outputs of ONE stream (a [1, 100] CUDA state tensor, advanced in place
    exactly as count calls of step()) computed as 8,192-output substreams."""
    torch = _torch()
    dt = {"u32": torch.int32, "f32": torch.float32}[fmt]
    fn = {"u32": lib().ranmar_generate_single_u32_dev,
          "f32": lib().ranmar_generate_single_f32_dev}[fmt]
    if out is None:
        out = torch.empty(count, dtype=dt, device=state.device)
    wsb = int(lib().ranmar_generate_single_workspace(count))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=state.device)
    _check(fn(_dptr(state), count, _dptr(out), _dptr(ws), wsb, _stream_ptr(stream)))
    return out


@_on_device
def bank_from_states(states, stream=None):
    """[n, 100] (or gauss [n, 104]) state tensor -> stream bank [99, n] (int32 words)."""
    torch = _torch()
    n = states.shape[0]
    src = states if states.shape[1] == STATE_WORDS else states[:, :STATE_WORDS].contiguous()
    bank = torch.empty((99, n), dtype=torch.int32, device=states.device)
    _check(lib().ranmar_bank_from_states_dev(_dptr(src), n, _dptr(bank), _stream_ptr(stream)))
    return bank


@_on_device
def bank_to_states(bank, t: int, out=None, stream=None):
    """Stream bank at t outputs per stream -> [n, 100] states (as t calls of step())."""
    torch = _torch()
    n = bank.shape[1]
    if out is None:
        out = torch.empty((n, STATE_WORDS), dtype=torch.int32, device=bank.device)
    _check(lib().ranmar_bank_to_states_dev(_dptr(bank), n, t, _dptr(out), _stream_ptr(stream)))
    return out


@_on_device
def langevin_bank(bank, t: int, v, f, types, gfactor1, gfactor2, tsqrt: float, stream=None) -> int:
    """Uniform-noise Langevin on a stream bank (every atom draws 3); returns t + 3."""
    n = bank.shape[1]
    if tuple(v.shape) != (n, 3) or tuple(f.shape) != (n, 3) or types.shape[0] != n:
        raise ValueError("langevin_bank: v, f must be [n_atoms, 3] and types [n_atoms]")
    _check(lib().ranmar_langevin_bank_dev(_dptr(bank), n, t, _dptr(v), _dptr(f), _dptr(types),
                                          _dptr(gfactor1), _dptr(gfactor2), gfactor1.shape[0] - 1,
                                          float(tsqrt), _stream_ptr(stream)))
    return t + 3


@_on_device
def fp64_selfcheck(n: int, seed: int = 1) -> int:
    """Bitwise mismatches between gaussian()'s branch-free fp64 divide/sqrt and
    the CUDA library's correctly rounded ones over n operand sets (expected 0)."""
    torch = _torch()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    _check(lib().ranmar_fp64_selfcheck_dev(n, seed, _dptr(bad), None))
    return int(bad.item())


@_on_device
def crlog_sweep(s0: int, n: int, mode: int = 0, cap: int = 1 << 16):
    """Check gaussian()'s correctly rounded log on rsq = s / 2^46, s in
    [s0, s0 + n): returns (fast-phase failures, accurate-phase failures,
    fast/accurate disagreements (mode 1), the failing s values (<= cap))."""
    torch = _torch()
    counts = torch.zeros(4, dtype=torch.int64, device="cuda")
    fails = torch.zeros(max(cap, 1), dtype=torch.int64, device="cuda")
    _check(lib().ranmar_crlog_sweep_dev(s0, n, mode, _dptr(counts), _dptr(fails), cap, None))
    c = counts.cpu().tolist()
    return c[0], c[1], c[2], sorted(fails[: min(c[3], cap)].cpu().tolist())


@_on_device
def gaussian_stream(gstates, count: int, out=None, stream=None):
    """count gaussian() calls on each of a FEW streams (one warp per stream) ->
    out[stream, q] (float64); states and cached deviates advance in place."""
    torch = _torch()
    n = gstates.shape[0]
    if out is None:
        out = torch.empty((n, count), dtype=torch.float64, device="cuda")
    _check(lib().ranmar_gaussian_stream_f64_dev(_dptr(gstates), n, count, _dptr(out),
                                                _stream_ptr(stream)))
    return out


@_on_device
def to_text_dev(states, stream=None, text=None, offsets=None, workspace=None):
    """Bulk ranmar::to_text (serialize.hpp:21-40) on the GPU.
    Returns (text: uint8 CUDA tensor, offsets: int64 CUDA tensor [n + 1]); text /
    offsets / workspace may be passed in (sizes: ranmar_to_text_bound(n), n + 1,
    ranmar_text_workspace(n) bytes) to reuse buffers across calls."""
    torch = _torch()
    n = states.shape[0]
    text = torch.empty(int(lib().ranmar_to_text_bound(n)), dtype=torch.uint8, device="cuda") if text is None else text
    off = torch.empty(n + 1, dtype=torch.int64, device="cuda") if offsets is None else offsets
    ws = (torch.empty(int(lib().ranmar_text_workspace(n)), dtype=torch.uint8, device="cuda")
          if workspace is None else workspace)
    if off.numel() != n + 1 or off.dtype != torch.int64:
        raise ValueError("offsets must be an int64 tensor of n + 1 entries")
    _check(lib().ranmar_to_text_dev(_dptr(states), n, _dptr(text), text.numel(), _dptr(off),
                                    _dptr(ws), ws.numel(), _stream_ptr(stream)))
    return text, off


@_on_device
def from_text_dev(text, offsets, stream=None, out=None, err=None):
    """Bulk ranmar::from_text (serialize.hpp:81-136) on the GPU: texts
    [offsets[k], offsets[k+1]) of `text` -> (states [n, 100], err [n]); err[k]
    is 0 or the 1-based line where the reference's parser throws (states[k] is
    left as it was then: zeros unless `out` is passed in for reuse)."""
    torch = _torch()
    n = offsets.shape[0] - 1
    states = torch.zeros((n, STATE_WORDS), dtype=torch.int32, device="cuda") if out is None else out
    err = torch.empty(n, dtype=torch.int32, device="cuda") if err is None else err
    if states.shape != (n, STATE_WORDS) or states.dtype != torch.int32 or err.numel() != n:
        raise ValueError("out must be an int32 [n, 100] tensor and err an int32 [n] tensor")
    _check(lib().ranmar_from_text_dev(_dptr(text), _dptr(offsets), n, _dptr(states), _dptr(err),
                                      _stream_ptr(stream)))
    return states, err


def texts_to_host(text, offsets) -> list:
    """(text, offsets) from to_text_dev -> list of Python strings."""
    off = offsets.cpu().numpy()
    blob = text[: int(off[-1])].cpu().numpy().tobytes()
    return [blob[off[k]:off[k + 1]].decode() for k in range(len(off) - 1)]


def gauss_states_from(states_t):
    """[n,100] state tensor -> [n,104] ranmar_gauss_state tensor with an empty cache."""
    torch = _torch()
    g = torch.zeros((states_t.shape[0], GAUSS_WORDS), dtype=torch.int32, device=states_t.device)
    g[:, :STATE_WORDS] = states_t
    return g


@_on_device
def device_status(clear: bool = True) -> int:
    """Sticky status bits of the current device (bit 0: a state with bad cursors or v)."""
    flags = C.c_uint32()
    _check(lib().ranmar_device_status(C.byref(flags), int(clear)))
    return flags.value


def kernel_launches() -> int:
    """Kernels launched by the library so far in this process."""
    return int(lib().ranmar_kernel_launches())


class Context:
    """Host-buffer API (ranmar_ctx_*): the call a CPU-side user of the reference
    makes, with the host<->device copies inside."""

    def __init__(self, device: Optional[int] = None):
        self._h = C.c_void_p()
        if device is None:  # the caller's current CUDA device
            device = _torch().cuda.current_device()
        _check(lib().ranmar_ctx_create(device, C.byref(self._h)))

    def close(self):
        if self._h:
            lib().ranmar_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def traffic(self) -> Tuple[int, int]:
        a, b = C.c_uint64(), C.c_uint64()
        _check(lib().ranmar_ctx_last_traffic(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def make_streams(self, seed: int, j, n: int, first: int = 0,
                     out: Optional[np.ndarray] = None) -> np.ndarray:
        jc = _jc(j)
        if out is None:
            out = np.zeros(n, STATE_DTYPE)
        _check(lib().ranmar_ctx_make_streams(self._h, seed, C.byref(jc), first, n, _ptr(out)))
        return out

    def jump(self, states: np.ndarray, j) -> np.ndarray:
        jc = _jc(j)
        states = np.ascontiguousarray(states, STATE_DTYPE)
        out = np.zeros(len(states), STATE_DTYPE)
        _check(lib().ranmar_ctx_jump(self._h, _ptr(states), _ptr(out), len(states), C.byref(jc)))
        return out

    def generate(self, states: np.ndarray, per_stream: int, fmt: str = "f32",
                 out: Optional[np.ndarray] = None) -> np.ndarray:
        """states (STATE_DTYPE, advanced in place) -> host output."""
        assert states.dtype == STATE_DTYPE and states.flags.c_contiguous
        dt = {"f32": np.float32, "u32": np.uint32}[fmt]
        if out is None:
            out = np.empty(len(states) * per_stream, dt)
        fn = lib().ranmar_ctx_generate_f32 if fmt == "f32" else lib().ranmar_ctx_generate_u32
        _check(fn(self._h, _ptr(states), len(states), per_stream, _ptr(out)))
        return out

    def consume(self, states: np.ndarray, per_stream: int):
        assert states.dtype == STATE_DTYPE and states.flags.c_contiguous
        sums = np.empty(len(states), np.uint64)
        hist = np.empty((len(states), 256), np.uint32)
        _check(lib().ranmar_ctx_consume(self._h, _ptr(states), len(states), per_stream,
                                        _ptr(sums), _ptr(hist)))
        return sums, hist

    def gaussian_stream(self, gstates: np.ndarray, count: int) -> np.ndarray:
        """count gaussian() calls on each host GAUSS_DTYPE state (advanced in place)."""
        assert gstates.dtype == GAUSS_DTYPE and gstates.flags.c_contiguous
        out = np.empty((len(gstates), count), np.float64)
        _check(lib().ranmar_ctx_gaussian_stream(self._h, _ptr(gstates), len(gstates), count,
                                                _ptr(out)))
        return out


class RanMars:
    """LAMMPS-style generator object (the north star's "seed
    constructor, uniform()/gaussian(), jump-ahead by J"): one stream whose
    uniform() (= next_f64, core.hpp:70-72) and gaussian() (the repo convention)
    calls return exactly the sequential values, served from blocks the GPU
    generates (K1 for uniforms, the warp-per-stream K4s for deviates).

    Blocks grow from 256 to `block` while one kind of call repeats; switching
    kind (or asking for state()) re-derives the exact state after the values
    already returned, so uniform()/gaussian() may be interleaved freely.
    """

    _MIN_BLOCK = 256

    def __init__(self, seed: Optional[int] = None, state: Optional[np.ndarray] = None,
                 block: int = 1 << 16, device: Optional[int] = None,
                 ctx: Optional["Context"] = None):
        if (seed is None) == (state is None):
            raise ValueError("give exactly one of seed or state")
        self._ctx = ctx or Context(device)
        self._g = np.zeros(1, GAUSS_DTYPE)
        self._g["s"] = init(seed) if seed is not None else np.asarray(state, STATE_DTYPE).reshape(1)
        self._max_block = max(self._MIN_BLOCK, int(block))
        self._kind = None   # 'u' or 'g': what _buf holds
        self._buf = None
        self._pos = 0
        self._next = None   # state after the whole buffer
        self._size = self._MIN_BLOCK

    # -- buffers ----------------------------------------------------------
    def _run(self, kind: str, g: np.ndarray, n: int) -> np.ndarray:
        """n values of `kind` from gauss state g (advanced in place)."""
        if kind == "u":
            s = np.ascontiguousarray(g["s"])
            u = self._ctx.generate(s, n, "u32")
            g["s"] = s
            return u.astype(np.float64) * 2.0**-24
        return self._ctx.gaussian_stream(g, n)[0]

    def _sync(self):
        """Make _g the exact state after the values returned so far."""
        if self._kind is not None:
            if self._pos == len(self._buf):
                self._g = self._next
            elif self._pos > 0:
                g = self._g.copy()
                self._run(self._kind, g, self._pos)
                self._g = g
        self._kind, self._buf, self._pos, self._next = None, None, 0, None

    def _take(self, kind: str) -> float:
        if self._kind != kind or self._pos == len(self._buf):
            if self._kind == kind:  # same kind, buffer used up: grow
                self._size = min(2 * self._size, self._max_block)
            else:
                self._size = self._MIN_BLOCK
            self._sync()
            nxt = self._g.copy()
            self._buf = self._run(kind, nxt, self._size)
            self._next, self._kind, self._pos = nxt, kind, 0
        x = float(self._buf[self._pos])
        self._pos += 1
        return x

    # -- the interface ----------------------------------------------------
    def uniform(self) -> float:
        """Next uniform in [0, 1): next_f64 (core.hpp:70-72)."""
        return self._take("u")

    def gaussian(self) -> float:
        """Next standard normal deviate (repo convention)."""
        return self._take("g")

    def jump(self, j) -> None:
        """Advance the stream by J uniforms (jump_state, jump.hpp:90-95); a cached
        gaussian deviate, if any, is kept."""
        self._sync()
        self._g["s"] = self._ctx.jump(np.ascontiguousarray(self._g["s"]), j)

    def state(self) -> np.ndarray:
        """1-element GAUSS_DTYPE record: the stream state and cached deviate."""
        self._sync()
        return self._g.copy()
