"""Time config 1 (one stream, seed 12345, 10^8 fp32 uniforms at full width through
substreams) with CUDA events, median of 5 calls after a warm-up call.

    python tools/time_c1.py [--n 100000000]
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2512_00093_b200 as rb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10**8)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    s = rb.states_to_device(rb.init(12345)).cuda()
    out = torch.empty(a.n, dtype=torch.float32, device="cuda")
    rb.generate_single(s.clone(), a.n, "f32", out=out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rb.generate_single(s, a.n, "f32", out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"config1 n={a.n}: {statistics.median(ts):.4f} ms (median of {a.reps}), "
          f"{a.n / statistics.median(ts) * 1e3:.3e} uniforms/s")


if __name__ == "__main__":
    main()
