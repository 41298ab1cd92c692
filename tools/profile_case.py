"""Small, ncu-friendly drivers for one BASELINE config each (1 GPU).

    python tools/profile_case.py c1|c2|c3|c4|c5|lang|bank|text|jump [--warmup W]

Runs W warm-up repetitions and one more of the config's GPU job, so an ncu
capture with `-k regex:<kernel> -s W -c 1` lands on a warm launch.
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
    ap.add_argument("case", choices=["c1", "c2", "c3", "c4", "c5", "lang", "bank", "text", "jump"])
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--c4-streams", type=int, default=1 << 16)
    args = ap.parse_args()
    reps = args.warmup + 1
    if args.case == "c1":
        # one stream x 10^8 fp32 at full width (substreams by make_streams, re-joined)
        s1 = rb.states_to_device(rb.init(12345)).cuda()
        out = torch.empty(10**8, dtype=torch.float32, device="cuda")
        for _ in range(reps):
            rb.generate_single(s1, 10**8, "f32", out=out)
    elif args.case == "c2":
        n, per = 65536, 65536
        st = torch.empty((n, 100), dtype=torch.int32, device="cuda")
        ws = torch.empty(rb.lib().ranmar_make_streams_workspace(n), dtype=torch.uint8, device="cuda")
        out = torch.empty(n * per, dtype=torch.float32, device="cuda")
        for _ in range(reps):
            rb.make_streams_dev(rb.init(12345), 2**40, n, out=st, workspace=ws)
            rb.generate(st, per, "f32", out=out)
    elif args.case == "c3":
        n = 1 << 20
        st = torch.empty((n, 100), dtype=torch.int32, device="cuda")
        ws = torch.empty(rb.lib().ranmar_make_streams_workspace(n), dtype=torch.uint8, device="cuda")
        for _ in range(reps):
            rb.make_streams_dev(rb.init_unchecked(987654321), 2**120, n, out=st, workspace=ws)
    elif args.case == "jump":
        n = 1 << 20
        st = rb.make_streams(12345, 2**40, n)
        out = torch.empty_like(st)
        for _ in range(reps):
            rb.jump_dev(st, 2**120, out=out)
    elif args.case == "c4":
        n = args.c4_streams
        st = rb.make_streams(42, 2**64, n)
        for _ in range(reps):
            rb.consume(st, 1 << 20)
    elif args.case == "bank":
        # the uniform-noise Langevin consumer on a stream bank, 2^24 atoms
        n = 1 << 24
        bank = rb.bank_from_states(rb.make_streams(7, 2**50, n))
        v = torch.randn((n, 3), dtype=torch.float64, device="cuda")
        f = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
        ty = torch.ones(n, dtype=torch.int32, device="cuda")
        g1, g2 = rb.langevin_factors([0.0, 1.0], 0.1, 0.005)
        d1, d2 = torch.from_numpy(g1).cuda(), torch.from_numpy(g2).cuda()
        t = 0
        for _ in range(reps):
            t = rb.langevin_bank(bank, t, v, f, ty, d1, d2, 1.0)
    elif args.case == "text":
        # device persistence of config 3's 2^20 stream starts
        st = rb.make_streams_dev(rb.init_unchecked(987654321), 2**120, 1 << 20)
        for _ in range(reps):
            text, off = rb.to_text_dev(st)
            rb.from_text_dev(text, off)
    elif args.case == "lang":
        # fix-langevin-style consumer, one launch per MD step, 2^24 atoms (config 5 streams)
        n = 1 << 24
        g = rb.gauss_states_from(rb.make_streams(7, 2**50, n))
        v = torch.randn((n, 3), dtype=torch.float64, device="cuda")
        f = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
        ty = torch.ones(n, dtype=torch.int32, device="cuda")
        g1, g2 = rb.langevin_factors([0.0, 1.0], 0.1, 0.005)
        d1, d2 = torch.from_numpy(g1).cuda(), torch.from_numpy(g2).cuda()
        for _ in range(reps):
            rb.langevin(g, v, f, ty, d1, d2, 1.0, rb.NOISE_UNIFORM)
    else:
        n = 1 << 20
        st = rb.make_streams(7, 2**50, n)
        g = rb.gauss_states_from(st)
        for _ in range(reps):
            rb.gaussian(g, 3, 100)
    torch.cuda.synchronize()
    assert rb.device_status() == 0
    print(f"{args.case} ok, launches={rb.kernel_launches()}")


if __name__ == "__main__":
    main()
