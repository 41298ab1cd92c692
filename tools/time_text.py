"""Time device persistence of config 3's 2^20 stream starts (to_text / from_text)
with CUDA events.

    python tools/time_text.py [--n 1048576] [--reps 10]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2512_00093_b200 as rb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    st = rb.make_streams_dev(rb.init_unchecked(987654321), 2**120, a.n)
    text, off = rb.to_text_dev(st)
    back, err = rb.from_text_dev(text, off)
    torch.cuda.synchronize()
    assert int(err.abs().sum()) == 0 and torch.equal(back, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {}
    for name, fn in (("to_text", lambda: rb.to_text_dev(st)), ("from_text", lambda: rb.from_text_dev(text, off))):
        fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / a.reps
    print(f"text n={a.n}: to_text {res['to_text']:.3f} ms, from_text {res['from_text']:.3f} ms, "
          f"{int(off[-1])} bytes")


if __name__ == "__main__":
    main()
