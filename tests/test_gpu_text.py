"""§8f row 1 — device-side state persistence: bulk to_text / from_text in the
reference's "ranmar24 v1" format (serialize.hpp), byte-exact against the
oracle's restatement and with the reference's error lines."""
import re

import numpy as np
import pytest

import paper_2512_00093_b200 as rb
from oracle.bind import STATE_DTYPE
from ranmar_testutil import state_from_json

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU-only module
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _random_states(n, seed):
    rng = np.random.default_rng(seed)
    s = np.zeros(n, STATE_DTYPE)
    s["lane"] = rng.integers(0, 1 << 24, (n, 97), dtype=np.uint32)
    s["lane"][::7, :5] = rng.integers(0, 10, (len(s[::7]), 5))  # short numbers too
    s["i"] = rng.integers(0, 97, n)
    s["j"] = (s["i"] + 97 - 64) % 97
    s["v"] = rng.integers(0, 16777213, n, dtype=np.uint32)
    return s


@pytest.mark.parametrize("n", [1, 5, 1023, 1024, 1025, 3000])
def test_to_text_matches_reference_format(oracle, refvec, n):
    s = _random_states(n, n)
    s[0] = state_from_json(refvec["to_text"][0]["state"])[0]
    texts = rb.texts_to_host(*rb.to_text_dev(rb.states_to_device(s)))
    assert texts[0] == refvec["to_text"][0]["text"]
    for k in range(n):
        assert texts[k] == oracle.to_text(s[k:k + 1]), k


def test_invalid_states_across_many_tiles(oracle):
    # empty texts for bad states (whole tiles of them too) inside a long run of
    # tiles: the one-pass look-back must still place every valid text exactly
    n = 5003
    s = _random_states(n, 77)
    bad = np.zeros(n, bool)
    bad[::3] = True
    bad[800:832] = True  # four whole tiles of 8
    bad[n - 1] = True    # the last state (the total comes from the last tile)
    s["v"][bad] = 0xFFFFFFFF
    d = rb.states_to_device(s)
    rb.device_status(clear=True)
    text, off = rb.to_text_dev(d)
    torch.cuda.synchronize()
    assert rb.device_status(clear=True) & 1
    o = off.cpu().numpy()
    lens = np.diff(o)
    assert o[0] == 0 and (lens[bad] == 0).all() and (lens[~bad] > 0).all()
    texts = rb.texts_to_host(text, off)
    for k in np.flatnonzero(~bad)[::37]:
        assert texts[k] == oracle.to_text(s[k:k + 1]), k


def test_round_trip_beyond_one_scan_chunk(oracle):
    # > 2^20 states: 131,077 look-back tiles, offsets past 2^30 bytes
    n = (1 << 20) + 37
    d = rb.make_streams(31415, 2**50, n)
    text, off = rb.to_text_dev(d)
    back, err = rb.from_text_dev(text, off)
    assert int(err.abs().sum()) == 0
    assert torch.equal(back, d)
    host = rb.states_to_host(d)
    o = off.cpu().numpy()
    for k in (0, 1, (1 << 20) - 1, 1 << 20, n - 1):
        blob = text[int(o[k]):int(o[k + 1])].cpu().numpy().tobytes().decode()
        assert blob == oracle.to_text(host[k:k + 1]), k


def _host_error_line(text):
    try:
        rb.from_text(text)
    except ValueError as e:
        return int(re.search(r"line (\d+)", str(e)).group(1))
    return 0


def test_from_text_errors_match_reference(refvec):
    good = refvec["to_text"][0]["text"]
    lines = good.split("\n")
    bad = [
        good.replace("ranmar24 v1", "ranmar24 v2"),
        good.replace("i 97 j 33", "i 97 j 34"),        # separation
        good.replace("i 97 j 33", "i 98 j 34"),        # range
        good.replace("v 362436", "v 16777213"),        # v >= m
        good.replace("v 362436", "v 362436 "),         # trailing
        good.replace("u 2 ", "u 3 "),                  # index order
        good.replace("u 5 ", "u 5  "),                 # double space
        good + "junk",                                 # trailing content
        "\n".join(lines[:50]),                         # truncated
        good.replace(lines[10], "u 8 16777216"),       # lane > mask
        good.replace(lines[10], "u 8 99999999999"),    # overflow
        good.replace("\n", "\r\n"),                    # CRLF is accepted
        good + "\n\n  \t\n",                           # trailing whitespace is accepted
        "",
        good.rstrip("\n"),                             # no final newline is accepted
        good + " " * 3000,                             # oversized (sequential path), accepted
        good + " " * 3000 + "x",                       # oversized with trailing content
        good + "\n" * 200,                             # more newlines than the warp keeps
        good.replace(lines[5] + "\n", lines[5] + "\n\n"),  # an empty line inside
        "ranmar24 v1",                                 # header only
        good[:-30],                                    # cut inside the last line
        # lines the SWAR fast path takes or hands back to the character checks
        good.replace(lines[10], "u 8 0"),               # one digit
        good.replace(lines[10], "u 8 00000012"),        # eight digits, leading zeros
        good.replace(lines[10], "u 8 16777215"),        # the largest lane
        good.replace(lines[10], "u 8 16777216"),        # eight digits, above the mask
        good.replace(lines[10], "u 8 000000000012"),    # twelve digits, leading zeros
        good.replace(lines[10], "u 8 123456789"),       # nine digits
        good.replace(lines[10], "u 8 1677721a"),        # a letter among the digits
        good.replace(lines[10], "u 8 12/"),             # '/' (just below '0')
        good.replace(lines[10], "u 8 12:"),             # ':' (just above '9')
        good.replace(lines[10], "u 8 1\u00b2"),        # a non-ASCII byte pair
        good.replace(lines[10], "u 08 5"),              # index with a leading zero
        good.replace(lines[10], "u  8 5"),              # double space before the index
        good.replace(lines[10], "u 8\t5"),             # tab separator
        good.replace(lines[10], "u 8 "),                # no digits
        good.replace(lines[40], "u 38 7\r"),           # CR on a two-digit index line
        good.replace(lines[40], "v 38 7"),              # wrong tag
        good.replace("v 362436", "v 0362436"),         # v with a leading zero
        good.replace("v 362436", "v 16777212"),        # the largest v
        good.replace("v 362436", "v 3624x6"),          # v with a letter
        good.replace("ranmar24 v1", "Ranmar24 v1"),    # header case
        good.replace("ranmar24 v1", "ranmar24 v10"),   # header one byte long
        good.replace("ranmar24 v1", "ranmar24 v"),     # header one byte short
        good.replace("i 97 j 33", "i 5 j 38"),         # one-digit i
        good.replace("i 97 j 33", "i 72 j 8"),         # one-digit j
        good.replace("i 97 j 33", "i 097 j 33"),       # i with a leading zero
        good.replace("i 97 j 33", "i 97 j 3x"),        # letter in j
        good.replace("i 97 j 33", "i 97  j 33"),       # double space
        good.replace("i 97 j 33", "i 9x j 33"),        # letter in i
        good.replace("i 97 j 33", "i 1 j 35"),         # separation off by one
    ]
    texts = [b.encode() for b in bad]
    offs = np.cumsum([0] + [len(t) for t in texts]).astype(np.int64)
    blob = torch.from_numpy(np.frombuffer(b"".join(texts) or b"\0", np.uint8).copy()).cuda()
    states, err = rb.from_text_dev(blob, torch.from_numpy(offs).cuda())
    err = err.cpu().numpy().tolist()
    for k, b in enumerate(bad):
        assert err[k] == _host_error_line(b), (k, b[:40])
    ok = [k for k, e in enumerate(err) if e == 0]
    assert ok == [11, 12, 14, 15, 17, 21, 22, 23, 25, 31, 35, 37, 38, 43, 44, 45]
    host = rb.states_to_host(states)
    for k in ok:
        assert host[k:k + 1].tobytes() == rb.from_text(bad[k]).tobytes()
