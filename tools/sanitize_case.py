"""Small invocations of every kernel for compute-sanitizer (one tool per run):

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
    torch.cuda.synchronize()
    assert rb.device_status() == 0
    print("sanitize case ok")


if __name__ == "__main__":
    main()
