"""Small invocations of every kernel (a plain smoke run: device status must stay clear).
On pools where compute-sanitizer is available, one tool per run:

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
    compute-sanitizer --tool memcheck  python tools/sanitize_case.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2512_00093_b200 as rb  # noqa: E402


def main():
    st = rb.make_streams(12345, 2**40, 300)             # pow table, tables, levels, bulk
    rb.make_streams_dev(rb.init(7), 2**120 + 12345, 200, first=77)  # apply (first > 0)
    rb.generate(st[:40], 1000, "f32")                   # K1
    rb.generate(st[:5], 37, "u32")
    rb.jump_dev(st[:50], 2**64 - 1)                     # K3 apply
    rb.consume(st[:100], 5000)                          # K2
    rb.gaussian(rb.gauss_states_from(st[:150]), 3, 7)   # K4
    rb.pow_t_mod_dev(2**130 + 5)
    # round-2 paths: three-level tree (level kernel with split j-chunks, tensor-core
    # levels 1 and 0), tensor-core batched jump, K4 row-batched stores and the
    # moments consumer, persistence, Langevin (in place and noise drawn ahead)
    big = rb.make_streams(42, 2**64, 20000)
    rb.jump_dev(big[:300], 2**120)                      # apply_tc (>= 128 states)
    g = rb.gauss_states_from(big[:200])
    rb.gaussian(g, 3, 20)                               # K4<3, 3>
    rb.gaussian_moments(g, 31)                          # K4 moments
    text, off = rb.to_text_dev(big[:64])
    rb.from_text_dev(text, off)
    n = 256
    v = torch.randn((n, 3), dtype=torch.float64, device="cuda")
    f = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
    ty = torch.ones(n, dtype=torch.int32, device="cuda")
    g1, g2 = rb.langevin_factors([0.0, 1.0], 0.1, 0.005, noise=rb.NOISE_GAUSSIAN)
    d1, d2 = torch.from_numpy(g1).cuda(), torch.from_numpy(g2).cuda()
    rb.langevin(rb.gauss_states_from(big[:n]), v, f, ty, d1, d2, 1.0, rb.NOISE_GAUSSIAN)
    torch.cuda.synchronize()
    assert rb.device_status() == 0
    print("sanitize case ok")


if __name__ == "__main__":
    main()
