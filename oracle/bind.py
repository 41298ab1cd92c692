"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the CPU checkers.

* ``Oracle``    -> oracle/liboracle.so, the plain-C restatement
                   (oracle/ranmar_oracle.c, each function citing the
                   reference file:line it restates).
* ``Reference`` -> oracle/_ref/libranmar_ref.so, the reference's own headers
                   compiled in place by oracle/Makefile (optional: absent when
                   /root/reference was never available to build it).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module. The product package
(paper_2512_00093_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libranmar_ref.so")
ACCEPTANCE_BIN = os.path.join(HERE, "_ref", "acceptance")

# ranmar::RanmarState (core.hpp:29-49): 97 x u32 lanes, int i, int j, u32 v = 400 B.
STATE_DTYPE = np.dtype([("lane", "<u4", (97,)), ("i", "<i4"), ("j", "<i4"), ("v", "<u4")])
assert STATE_DTYPE.itemsize == 400
# or_gauss_state: state + saved double + flag + pad = 416 B.
GAUSS_DTYPE = np.dtype([("s", STATE_DTYPE), ("saved", "<f8"), ("has_saved", "<u4"), ("pad", "<u4")])
assert GAUSS_DTYPE.itemsize == 416

MASK = 0xFFFFFF
ARITH_MOD = 16777213


def j_limbs(j: int) -> np.ndarray:
    """Python int -> 4 x u64 little-endian limbs (the C-ABI jump-count layout)."""
    if j < 0 or j >= 1 << 256:
        raise ValueError("jump count must be in [0, 2^256)")
    return np.array([(j >> (64 * k)) & ((1 << 64) - 1) for k in range(4)], dtype=np.uint64)


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _build_hint() -> str:
    return "run `make -C oracle` (or __graft_entry__.build())"


class Oracle:
    """The C restatement. All arrays are numpy, states use STATE_DTYPE."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing; {_build_hint()}")
        self.lib = C.CDLL(path)
        L = self.lib
        vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
        sig = {
            "or_init": (i32, [u32, vp]),
            "or_init_unchecked": (None, [u32, vp]),
            "or_step": (u32, [vp]),
            "or_step_n": (None, [vp, u64, vp]),
            "or_value_of": (i32, [u32, vp]),
            "or_init_float": (i32, [u32, vp]),
            "or_step_float_n": (None, [vp, u64, vp]),
            "or_reduce_trinomial": (None, [vp, i32, vp]),
            "or_mul_mod": (None, [vp, vp, vp]),
            "or_mul_by_t": (None, [vp, vp]),
            "or_pow_t_mod": (None, [vp, vp]),
            "or_canonicalize": (None, [vp, vp]),
            "or_apply_companion": (None, [vp, vp]),
            "or_jump_fib": (None, [vp, vp, vp]),
            "or_jump_arith": (u32, [u32, vp]),
            "or_jump_state": (None, [vp, vp, vp]),
            "or_make_streams": (i32, [vp, vp, u64, u64, vp]),
            "or_j256_parse": (i32, [C.c_char_p, vp]),
            "or_generate_u32": (None, [vp, u64, u64, vp]),
            "or_generate_f32": (None, [vp, u64, u64, vp]),
            "or_consume": (None, [vp, u64, u64, vp, vp]),
            "or_gaussian_fill": (None, [vp, u64, u64, u64, vp]),
            "or_gaussian_fill_flags": (None, [vp, u64, u64, u64, vp, vp]),
            "or_crlog": (C.c_double, [C.c_double]),
            "or_crlog_ex": (C.c_double, [C.c_double, C.POINTER(C.c_int)]),
            "or_crlog_accurate": (C.c_double, [C.c_double, C.POINTER(C.c_int)]),
            "or_crlog_scan": (u64, [u64, u64, vp, u64]),
            "or_langevin": (i32, [vp, u64, vp, vp, vp, vp, C.c_int32, vp, vp, C.c_int32,
                                  C.c_double, C.c_int]),
            "or_gaussian": (C.c_double, [vp]),
            "or_to_text": (C.c_long, [vp, C.c_char_p, C.c_long]),
            "or_from_text": (i32, [C.c_char_p, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args

    # -- core ---------------------------------------------------------------
    def init(self, seed: int, checked: bool = True) -> np.ndarray:
        s = np.zeros(1, STATE_DTYPE)
        if checked:
            if self.lib.or_init(seed, _p(s)) != 0:
                raise ValueError("ranmar: seed must be in [0, 900000000]")
        else:
            self.lib.or_init_unchecked(seed, _p(s))
        return s

    def step_n(self, state: np.ndarray, n: int) -> np.ndarray:
        """Advances `state` (1-element STATE_DTYPE array) in place; returns n u24 outputs."""
        out = np.empty(n, np.uint32)
        self.lib.or_step_n(_p(state), n, _p(out))
        return out

    def float_outputs(self, seed: int, n: int) -> np.ndarray:
        st = (C.c_char * (97 * 8 + 8 + 8))()
        if self.lib.or_init_float(seed, C.cast(st, C.c_void_p)) != 0:
            raise ValueError("ranmar: seed must be in [0, 900000000]")
        out = np.empty(n, np.float64)
        self.lib.or_step_float_n(C.cast(st, C.c_void_p), n, _p(out))
        return out

    # -- polynomial ring ----------------------------------------------------
    def pow_t_mod(self, j: int) -> np.ndarray:
        out = np.empty(97, np.uint32)
        self.lib.or_pow_t_mod(_p(j_limbs(j)), _p(out))
        return out

    def mul_mod(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        out = np.empty(97, np.uint32)
        self.lib.or_mul_mod(_p(np.ascontiguousarray(a, np.uint32)),
                            _p(np.ascontiguousarray(b, np.uint32)), _p(out))
        return out

    def reduce_trinomial(self, raw: np.ndarray) -> np.ndarray:
        raw = np.ascontiguousarray(raw, np.uint32)
        out = np.empty(97, np.uint32)
        self.lib.or_reduce_trinomial(_p(raw), len(raw), _p(out))
        return out

    # -- jump ---------------------------------------------------------------
    def canonicalize(self, state: np.ndarray) -> np.ndarray:
        out = np.empty(97, np.uint32)
        self.lib.or_canonicalize(_p(state), _p(out))
        return out

    def jump_state(self, state: np.ndarray, j: int) -> np.ndarray:
        out = np.zeros(1, STATE_DTYPE)
        self.lib.or_jump_state(_p(np.ascontiguousarray(state)), _p(j_limbs(j)), _p(out))
        return out

    def jump_arith(self, v: int, j: int) -> int:
        return int(self.lib.or_jump_arith(v, _p(j_limbs(j))))

    def make_streams(self, base: np.ndarray, j: int, n: int, first: int = 0) -> np.ndarray:
        out = np.zeros(n, STATE_DTYPE)
        if self.lib.or_make_streams(_p(np.ascontiguousarray(base)), _p(j_limbs(j)), first, n,
                                    _p(out)) != 0:
            raise ValueError("ranmar: need n >= 1 and block length >= 1")
        return out

    def parse_jump_count(self, text: str) -> int:
        limbs = np.zeros(4, np.uint64)
        rc = self.lib.or_j256_parse(text.encode(), _p(limbs))
        if rc != 0:
            raise ValueError(f"ranmar: bad jump count {text!r}")
        return sum(int(limbs[k]) << (64 * k) for k in range(4))

    # -- workloads ----------------------------------------------------------
    def generate_u32(self, states: np.ndarray, per_stream: int) -> np.ndarray:
        states = np.ascontiguousarray(states)
        out = np.empty(len(states) * per_stream, np.uint32)
        self.lib.or_generate_u32(_p(states), len(states), per_stream, _p(out))
        return out

    def generate_f32(self, states: np.ndarray, per_stream: int) -> np.ndarray:
        states = np.ascontiguousarray(states)
        out = np.empty(len(states) * per_stream, np.float32)
        self.lib.or_generate_f32(_p(states), len(states), per_stream, _p(out))
        return out

    def consume(self, states: np.ndarray, per_stream: int):
        states = np.ascontiguousarray(states)
        sums = np.empty(len(states), np.uint64)
        hist = np.empty((len(states), 256), np.uint32)
        self.lib.or_consume(_p(states), len(states), per_stream, _p(sums), _p(hist))
        return sums, hist

    def gaussian_fill(self, gstates: np.ndarray, per_step: int, steps: int,
                      libm_log: bool = False, with_flags: bool = False):
        """The repo's gaussian() (RanMars::gaussian's form, correctly rounded
        log); libm_log=True swaps in glibc log() (the same form with the
        platform's libm, which is not correctly rounded on ~0.08 % of inputs).
        with_flags: also return, per deviate, whether its pair's glibc log
        differed from the correctly rounded one (libm mode)."""
        gstates = np.ascontiguousarray(gstates)
        out = np.empty((steps, len(gstates), per_step), np.float64)
        flags = np.zeros(out.shape, np.uint8) if with_flags else None
        flag = C.c_int.in_dll(self.lib, "or_gauss_use_libm_log")
        flag.value = int(libm_log)
        try:
            self.lib.or_gaussian_fill_flags(_p(gstates), len(gstates), per_step, steps, _p(out),
                                            None if flags is None else _p(flags))
        finally:
            flag.value = 0
        return (out, flags) if with_flags else out

    def langevin(self, gstates: np.ndarray, v: np.ndarray, f: np.ndarray, types: np.ndarray,
                 gfactor1: np.ndarray, gfactor2: np.ndarray, tsqrt: float, noise: int,
                 mask: np.ndarray = None, groupbit: int = 1) -> int:
        """The repo's fix-langevin-style consumer: f (n x 3) updated in place,
        gstates advanced; returns 1 if an atom type was out of range."""
        for a in (v, f, types, gfactor1, gfactor2) + ((mask,) if mask is not None else ()):
            assert a.flags["C_CONTIGUOUS"]
        assert v.dtype == np.float64 and f.dtype == np.float64 and types.dtype == np.int32
        return self.lib.or_langevin(_p(gstates), len(gstates), _p(v), _p(f), _p(types),
                                    None if mask is None else _p(mask), groupbit, _p(gfactor1),
                                    _p(gfactor2), len(gfactor1) - 1, tsqrt, noise)

    def crlog(self, x: float) -> float:
        """gaussian()'s correctly rounded log."""
        return self.lib.or_crlog(x)

    def crlog_ex(self, x: float):
        """(log, decided by the fast phase?)"""
        f = C.c_int()
        y = self.lib.or_crlog_ex(x, C.byref(f))
        return y, bool(f.value)

    def crlog_accurate(self, x: float):
        """(accurate phase's log, its rounding test decided?)"""
        ok = C.c_int()
        y = self.lib.or_crlog_accurate(x, C.byref(ok))
        return y, bool(ok.value)

    def crlog_scan(self, s0: int, n: int, cap: int = 1 << 16):
        """Fast-phase failures over rsq = s / 2^46, s in [s0, s0 + n):
        (count, the first <= cap failing s values)."""
        fails = np.zeros(max(cap, 1), np.uint64)
        c = self.lib.or_crlog_scan(s0, n, _p(fails), cap)
        return int(c), fails[: min(c, cap)].tolist()

    def gaussian_call(self, g: np.ndarray) -> float:
        """One gaussian() call on a 1-element GAUSS_DTYPE array (advanced in place)."""
        return self.lib.or_gaussian(_p(g))

    def uniform_call(self, g: np.ndarray) -> float:
        """One uniform() = next_f64 call on the stream of a GAUSS_DTYPE record."""
        out = np.empty(1, np.uint32)
        self.lib.or_step_n(_p(g), 1, _p(out))  # s is at offset 0 of the record
        return float(out[0]) * 2.0**-24

    def to_text(self, state: np.ndarray) -> str:
        buf = C.create_string_buffer(4096)
        n = self.lib.or_to_text(_p(np.ascontiguousarray(state)), buf, 4096)
        assert n > 0
        return buf.value.decode()

    def from_text(self, text: str) -> np.ndarray:
        out = np.zeros(1, STATE_DTYPE)
        if self.lib.or_from_text(text.encode(), _p(out)) != 0:
            raise ValueError("ranmar: state parse error")
        return out


class Reference:
    """The reference's own headers compiled in place (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing; {_build_hint()} with /root/reference present")
        self.lib = C.CDLL(path)
        L = self.lib
        vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
        sig = {
            "ref_init": (i32, [u32, vp]),
            "ref_step_n": (i32, [vp, u64, vp]),
            "ref_step_float_n": (i32, [u32, u64, vp]),
            "ref_pow_t_mod": (i32, [vp, vp]),
            "ref_mul_mod": (i32, [vp, vp, vp]),
            "ref_jump_state": (i32, [vp, vp, vp]),
            "ref_jump_arith": (i32, [u32, vp, vp]),
            "ref_make_streams": (i32, [u32, vp, u64, i32, vp]),
            "ref_parse_jump_count": (i32, [C.c_char_p, vp]),
            "ref_to_text": (C.c_long, [vp, C.c_char_p, C.c_long]),
            "ref_from_text": (i32, [C.c_char_p, vp]),
            "ref_generate_f32": (i32, [vp, vp, u64, u64, u64, i32, vp, vp]),
            "ref_stream_starts": (i32, [vp, vp, u64, u64, i32, vp]),
            "ref_jump_batch": (i32, [vp, u64, vp, i32, vp]),
            "ref_consume": (i32, [vp, vp, u64, u64, u64, i32, vp, vp]),
            "ref_last_error": (C.c_char_p, []),
            "ref_to_text_bulk": (C.c_long, [vp, u64, vp, C.c_long, i32]),
            "ref_from_text_bulk": (C.c_long, [vp, vp, u64, vp, i32]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args

    def _check(self, rc: int):
        if rc == 1:
            raise ValueError(self.lib.ref_last_error().decode())
        if rc != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def init(self, seed: int) -> np.ndarray:
        s = np.zeros(1, STATE_DTYPE)
        self._check(self.lib.ref_init(seed, _p(s)))
        return s

    def step_n(self, state: np.ndarray, n: int) -> np.ndarray:
        out = np.empty(n, np.uint32)
        self.lib.ref_step_n(_p(state), n, _p(out))
        return out

    def float_outputs(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self._check(self.lib.ref_step_float_n(seed, n, _p(out)))
        return out

    def pow_t_mod(self, j: int) -> np.ndarray:
        out = np.empty(97, np.uint32)
        self._check(self.lib.ref_pow_t_mod(_p(j_limbs(j)), _p(out)))
        return out

    def mul_mod(self, a, b) -> np.ndarray:
        out = np.empty(97, np.uint32)
        self.lib.ref_mul_mod(_p(np.ascontiguousarray(a, np.uint32)),
                             _p(np.ascontiguousarray(b, np.uint32)), _p(out))
        return out

    def jump_state(self, state: np.ndarray, j: int) -> np.ndarray:
        out = np.zeros(1, STATE_DTYPE)
        self._check(self.lib.ref_jump_state(_p(np.ascontiguousarray(state)), _p(j_limbs(j)),
                                             _p(out)))
        return out

    def make_streams(self, seed: int, j: int, n: int, independent: bool = False) -> np.ndarray:
        out = np.zeros(n, STATE_DTYPE)
        self._check(self.lib.ref_make_streams(seed, _p(j_limbs(j)), n, int(independent), _p(out)))
        return out

    def stream_starts(self, base: np.ndarray, j: int, first: int, n: int,
                      threads: int = 1) -> np.ndarray:
        out = np.zeros(n, STATE_DTYPE)
        self._check(self.lib.ref_stream_starts(_p(np.ascontiguousarray(base)), _p(j_limbs(j)),
                                               first, n, threads, _p(out)))
        return out

    def jump_batch(self, states: np.ndarray, j: int, threads: int = 1) -> np.ndarray:
        states = np.ascontiguousarray(states)
        out = np.zeros(len(states), STATE_DTYPE)
        self._check(self.lib.ref_jump_batch(_p(states), len(states), _p(j_limbs(j)), threads,
                                            _p(out)))
        return out

    def generate_f32(self, base: np.ndarray, j: int, first: int, n: int, per_stream: int,
                     threads: int = 1, out: np.ndarray | None = None) -> int:
        chk = np.zeros(1, np.uint64)
        self._check(self.lib.ref_generate_f32(
            _p(np.ascontiguousarray(base)), _p(j_limbs(j)), first, n, per_stream, threads,
            _p(out) if out is not None else None, _p(chk)))
        return int(chk[0])

    def consume(self, base: np.ndarray, j: int, first: int, n: int, per_stream: int,
                threads: int = 1):
        sums = np.empty(n, np.uint64)
        hist = np.empty((n, 256), np.uint32)
        self._check(self.lib.ref_consume(_p(np.ascontiguousarray(base)), _p(j_limbs(j)), first, n,
                                         per_stream, threads, _p(sums), _p(hist)))
        return sums, hist

    def parse_jump_count(self, text: str) -> int:
        limbs = np.zeros(4, np.uint64)
        self._check(self.lib.ref_parse_jump_count(text.encode(), _p(limbs)))
        return sum(int(limbs[k]) << (64 * k) for k in range(4))

    def to_text_bulk(self, states: np.ndarray, threads: int = 1, slot: int = 1408):
        """Threaded ranmar::to_text into fixed slots -> (buffer, total bytes)."""
        states = np.ascontiguousarray(states)
        buf = np.zeros(len(states) * slot, np.uint8)
        total = self.lib.ref_to_text_bulk(_p(states), len(states), _p(buf), slot, threads)
        assert total >= 0
        return buf, total

    def from_text_bulk(self, blob: np.ndarray, offsets: np.ndarray, threads: int = 1):
        """Threaded ranmar::from_text of texts [offsets[k], offsets[k+1]) -> (states, failures)."""
        n = len(offsets) - 1
        out = np.zeros(n, STATE_DTYPE)
        bad = self.lib.ref_from_text_bulk(_p(np.ascontiguousarray(blob)),
                                          _p(np.ascontiguousarray(offsets, np.uint64)), n,
                                          _p(out), threads)
        return out, bad

    def to_text(self, state: np.ndarray) -> str:
        buf = C.create_string_buffer(4096)
        n = self.lib.ref_to_text(_p(np.ascontiguousarray(state)), buf, 4096)
        assert n > 0
        return buf.value.decode()

    def from_text(self, text: str) -> np.ndarray:
        out = np.zeros(1, STATE_DTYPE)
        self._check(self.lib.ref_from_text(text.encode(), _p(out)))
        return out


def reference_available() -> bool:
    return os.path.exists(REF_SO)
