"""Time K4 gaussian() at config 5 (or a given size) with CUDA events.

    python tools/time_k4.py [--atoms 16777216] [--per 3] [--steps 100] [--reps 5]
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
    ap.add_argument("--per", type=int, default=3)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--moments", action="store_true", help="time the in-kernel moments consumer instead")
    a = ap.parse_args()
    g = rb.gauss_states_from(rb.make_streams(7, 2**50, a.atoms))
    if a.moments:
        out = torch.empty((a.atoms, 2), dtype=torch.float64, device="cuda")
        run = lambda: rb.gaussian_moments(g, a.per * a.steps, out=out)  # noqa: E731
    else:
        out = torch.empty((a.steps, a.atoms, a.per), dtype=torch.float64, device="cuda")
        run = lambda: rb.gaussian(g, a.per, a.steps, out=out)  # noqa: E731
    for _ in range(2):
        run()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    assert rb.device_status() == 0
    ms = sorted(ts)[len(ts) // 2]
    dev = a.atoms * a.per * a.steps
    by = dev * 8 + a.atoms * 2 * 416
    print(f"k4{' moments' if a.moments else ''} atoms={a.atoms} per={a.per} steps={a.steps}: median {ms:.3f} ms (all {[round(t, 3) for t in ts]}), "
          f"{dev / ms / 1e6:.3e} gaussians/s, {by / ms / 1e6:.1f} GB/s")


if __name__ == "__main__":
    main()
