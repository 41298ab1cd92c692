"""§8f row 2 — the GPU-backed CLI (tools/ranmar_cli.cpp), checked with the
reference's own CLI contract (tests/test_cli.cpp:69-209 of the reference):
determinism and agreement with the library, --skip, output formats, jump and
streams files, the bench JSON schema, exit codes 0/1/2."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2512_00093_b200", "bin", "ranmar_b200")


def run(args, **kw):
    if not os.path.exists(CLI):
        subprocess.run(["make", "-C", ROOT, "cli"], check=True, capture_output=True)
    r = subprocess.run([CLI] + args.split(), capture_output=True, text=True, timeout=600, **kw)
    return r.returncode, r.stdout, r.stderr


# ---- usage errors are decided before any device work (CPU) -----------------------

@pytest.mark.parametrize("args", ["nonsense", "generate --count 5", "generate --seed 900000001 --count 5",
                                  "generate --seed 1 --count 5 --format bin",
                                  "generate --seed 1 --count 5 --skip 2^x", "", "jump --by 1",
                                  "generate --seed 1 --count 5 --bogus 3", "generate --seed x --count 5"])
def test_usage_errors_exit_2(args):
    assert run(args)[0] == 2  # test_cli.cpp:185-193


def test_help_exits_cleanly():
    assert run("--help")[0] == 0 and run("generate --help")[0] == 0  # test_cli.cpp:207-209


# ---- GPU -------------------------------------------------------------------------

gpu = pytest.mark.gpu


@gpu
def test_generate_deterministic_and_matches_library(oracle):
    a, b = run("generate --seed 12345 --count 100"), run("generate --seed 12345 --count 100")
    assert a[0] == 0 and a[1] == b[1]
    assert a[1].split("\n")[:-1] == [str(x) for x in oracle.step_n(oracle.init(12345), 100)]
    assert run("generate --seed 1 --count 0")[1] == ""


@gpu
def test_generate_skip_and_large_count(oracle):
    skipped = run("generate --seed 777 --count 50 --skip 1000")[1].split()
    full = run("generate --seed 777 --count 1050")[1].split()
    assert skipped == full[1000:]
    big = run("generate --seed 3 --count 20000000")[1].split()  # crosses the 2^24 block
    exp = oracle.step_n(oracle.init(3), 20_000_000)
    assert len(big) == len(exp) and big[-1] == str(exp[-1]) and big[1 << 24] == str(exp[1 << 24])


@gpu
def test_formats(oracle):
    u = oracle.step_n(oracle.init(5), 20)
    hexs = run("generate --seed 5 --count 20 --format hex")[1].split()
    f64 = run("generate --seed 5 --count 20 --format f64")[1].split()
    assert hexs == ["%06x" % x for x in u]
    assert f64 == ["%.17g" % (x * 2.0**-24) for x in u]


@gpu
def test_jump_file(oracle, tmp_path):
    src, dst = tmp_path / "in.state", tmp_path / "out.state"
    src.write_text(oracle.to_text(oracle.init(31415)))
    assert run(f"jump --state {src} --by 2^20-1 --out {dst}")[0] == 0
    exp = oracle.jump_state(oracle.init(31415), 2**20 - 1)
    assert oracle.from_text(dst.read_text()).tobytes() == exp.tobytes()


@gpu
def test_streams_files_tile(oracle, tmp_path):
    d = tmp_path / "streams"
    rc, out, _ = run(f"streams --seed 42 --block 7 --n 3 --out-dir {d}")
    assert rc == 0 and len(out.split()) == 3
    base = oracle.step_n(oracle.init(42), 21)
    got = np.concatenate([oracle.step_n(oracle.from_text((d / f"stream_{k}.state").read_text()), 7)
                          for k in range(3)])
    assert (got == base).all()


@gpu
def test_bench_report():
    rc, out, _ = run("bench --count 1000000 --jumps 2^32-1,2^20+1 --label test-box")
    assert rc == 0
    r = json.loads(out)
    assert r["count"] == 1000000 and r["machine"] == "test-box"
    assert r["integer_seconds"] > 0 and r["float_seconds"] > 0 and r["speedup"] > 0
    assert [j["j"] for j in r["jumps"]] == ["2^32-1", "2^20+1"]
    assert r["jumps"][0]["bits"] == 32 and r["jumps"][1]["bits"] == 21
    assert r["jumps"][0]["microseconds"] > 0
    rc, out, _ = run("bench --count 1000 --jumps 2^64-1,2^120-1")
    t = json.loads(out)["jumps"]
    ratio = t[1]["microseconds"] / t[0]["microseconds"]  # test_cli.cpp:170-183 band
    assert 0.5 * 120 / 64 < ratio < 2.0 * 120 / 64


@gpu
def test_corrupt_state_exit_1(tmp_path):
    bad, out = tmp_path / "bad.state", tmp_path / "o.state"
    bad.write_text("ranmar24 v1\ni 97 j 34\n")
    assert run(f"jump --state {bad} --by 1 --out {out}")[0] == 1
    assert run(f"jump --state /nonexistent/x --by 1 --out {out}")[0] == 1


@gpu
def test_selftest_passes():
    rc, out, _ = run("selftest")
    assert rc == 0 and "all checks passed" in out
