"""Time batched jump_state (2^20 states by 2^120) with CUDA events, and with
--compare check the tensor-core kernel's states against the IMAD kernel's
(RANMAR_APPLY=imad in a subprocess).

    python tools/time_jump.py [--n 1048576] [--reps 10] [--compare]
"""
import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2512_00093_b200 as rb  # noqa: E402


def run(n, reps):
    st = rb.make_streams(12345, 2**40, n)
    out = torch.empty_like(st)
    for _ in range(3):
        rb.jump_dev(st, 2**120, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        rb.jump_dev(st, 2**120, out=out)
    b.record()
    torch.cuda.synchronize()
    assert rb.device_status() == 0
    return a.elapsed_time(b) / reps, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--compare", action="store_true")
    ap.add_argument("--dump", default="")
    a = ap.parse_args()
    ms, out = run(a.n, a.reps)
    kind = "imad" if os.environ.get("RANMAR_APPLY", "").startswith("i") else "tc"
    print(f"jump n={a.n} apply={kind}: {ms:.4f} ms, {a.n / ms / 1e6:.3e} jumps/s")
    if a.dump:
        torch.save(out.cpu(), a.dump)
    if a.compare:
        path = "/tmp/jump_imad.pt"
        env = dict(os.environ, RANMAR_APPLY="imad")
        subprocess.run([sys.executable, __file__, "--n", str(a.n), "--reps", "2", "--dump", path], env=env,
                       check=True)
        print("tensor-core states == IMAD states:", torch.equal(out.cpu(), torch.load(path)))


if __name__ == "__main__":
    main()
