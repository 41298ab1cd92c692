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
