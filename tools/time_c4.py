"""Time K2 consume at config 4 (or a given size) with CUDA events.

    python tools/time_c4.py [--streams 1048576] [--per 1048576] [--reps 3]
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
    ap.add_argument("--streams", type=int, default=1 << 20)
    ap.add_argument("--per", type=int, default=1 << 20)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    d = rb.make_streams(42, 2**64, a.streams)
    rb.consume(d.clone(), a.per)
    ts = []
    for _ in range(a.reps):
        x = d.clone()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        sums, hist = rb.consume(x, a.per)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    assert rb.device_status() == 0
    ms = sorted(ts)[len(ts) // 2]
    u = a.streams * a.per
    print(f"c4 streams={a.streams} per={a.per}: median {ms:.3f} ms (all {[round(t, 3) for t in ts]}), "
          f"{u / ms / 1e9:.4e} uniforms/s, sum-of-sums {int(sums.sum())}")


if __name__ == "__main__":
    main()
