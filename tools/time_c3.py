"""Time config 3 (make_streams of 2^20 starts at J = 2^120) with CUDA events,
and check it against the IMAD bulk kernel's states (RANMAR_BULK=imad in a
subprocess) when --compare is given.

    python tools/time_c3.py [--n 1048576] [--reps 20] [--compare]
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
    base = rb.init_unchecked(987654321)
    st = torch.empty((n, rb.STATE_WORDS), dtype=torch.int32, device="cuda")
    ws = torch.empty(rb.lib().ranmar_make_streams_workspace(n), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        rb.make_streams_dev(base, 2**120, n, out=st, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        rb.make_streams_dev(base, 2**120, n, out=st, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    assert rb.device_status() == 0
    ms_direct = e0.elapsed_time(e1) / reps
    # the same launches captured in a CUDA graph and replayed (device time without host gaps)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        rb.make_streams_dev(base, 2**120, n, out=st, workspace=ws, stream=s)
    torch.cuda.synchronize()
    trials = []
    for _ in range(5):
        e0.record(s)
        with torch.cuda.stream(s):
            for _ in range(reps):
                g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        trials.append(e0.elapsed_time(e1) / reps)
    assert rb.device_status() == 0
    return ms_direct, sorted(trials)[2], st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--compare", action="store_true")
    ap.add_argument("--dump", default="")
    a = ap.parse_args()
    ms, msg, st = run(a.n, a.reps)
    print(f"c3 n={a.n} bulk={os.environ.get('RANMAR_BULK', 'tc')}: {ms:.4f} ms direct, {msg:.4f} ms graph "
          f"replay, {a.n / msg / 1e6:.3e} starts/s")
    if a.dump:
        torch.save(st.cpu(), a.dump)
    if a.compare:
        path = "/tmp/c3_imad.pt"
        env = dict(os.environ, RANMAR_BULK="imad")
        subprocess.run([sys.executable, __file__, "--n", str(a.n), "--reps", "3", "--dump", path],
                       env=env, check=True)
        ref = torch.load(path)
        same = torch.equal(ref, st.cpu())
        print("tensor-core states == IMAD states:", same)
        if not same:
            diff = (ref != st.cpu()).any(dim=1).nonzero().flatten()
            print("differing streams:", diff[:10].tolist(), "count", diff.numel())
            sys.exit(1)


if __name__ == "__main__":
    main()
