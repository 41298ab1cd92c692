"""Opcode mix of one kernel from an ncu report's source page (SASS):
warp-level instructions executed, thread instructions, avg active threads.

    python tools/sass_mix.py report.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    lines = out.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    return list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    r = rows(rep)
    warp = collections.Counter()
    thr = collections.Counter()
    stall = collections.Counter()
    tw = tt = 0
    for x in r:
        op = x["Source"].strip().split()[0] if x["Source"].strip() else "?"
        if op.startswith("@"):
            op = x["Source"].strip().split()[1]
        base = op.split(".")[0]
        w = int(x["Instructions Executed"] or 0)
        t = int(x["Thread Instructions Executed"] or 0)
        warp[base] += w
        thr[base] += t
        stall[base] += int(x["Warp Stall Sampling (All Samples)"] or 0)
        tw += w
        tt += t
    print(f"warp instructions {tw:,}  thread instructions {tt:,}  avg active {tt / max(tw, 1):.1f}")
    st = sum(stall.values())
    for op, w in warp.most_common(top):
        print(f"{op:12s} {w:14,d} {100 * w / tw:5.1f}%  avg threads {thr[op] / max(w, 1):5.1f}  "
              f"stall samples {100 * stall[op] / max(st, 1):5.1f}%")


if __name__ == "__main__":
    main()
