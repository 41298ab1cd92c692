"""Experiment: the warp-per-stream gaussian kernel (K4s) at config-5 sizes
(contiguous per-stream output), timed with CUDA events, vs K4 (time_k4.py).

    python tools/time_k4s.py [--atoms N] [--count 300]
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
    ap.add_argument("--atoms", type=int, default=1 << 24)
    ap.add_argument("--count", type=int, default=300)
    a = ap.parse_args()
    g = rb.gauss_states_from(rb.make_streams(7, 2**50, a.atoms))
    out = torch.empty((a.atoms, a.count), dtype=torch.float64, device="cuda")
    for _ in range(2):
        rb.gaussian_stream(g, a.count, out=out)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        rb.gaussian_stream(g, a.count, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    assert rb.device_status() == 0
    ms = sorted(ts)[2]
    print(f"k4s atoms={a.atoms} count={a.count}: median {ms:.3f} ms {[round(t, 3) for t in ts]}, "
          f"{a.atoms * a.count / ms / 1e6:.3e} gaussians/s")


if __name__ == "__main__":
    main()
