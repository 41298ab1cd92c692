"""Per-source-line totals (warp instructions, stall samples) of one kernel
from an ncu report captured with --import-source on.

    python tools/ncu_lines.py report.ncu-rep [top] [kernel-regex]
"""
import collections
import subprocess
import sys
import csv
import io


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
    out = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout.splitlines()
    path = None
    agg = collections.defaultdict(lambda: [0, 0, 0, ""])
    cur_line = None
    for raw in csv.reader(io.StringIO("\n".join(out))):
        if not raw:
            continue
        if raw[0] == "File Path":
            path = raw[1].split("/")[-1]
            continue
        if raw[0] in ("Function Name", "Line No"):
            continue
        ln, src = raw[0], raw[1]
        if ln:  # a CUDA source line row
            cur_line = (path, ln)
            agg[cur_line][3] = src.strip()[:80]
            continue
        if cur_line is None or len(raw) < 9:
            continue
        try:
            w = int(raw[7] or 0)
            t = int(raw[8] or 0)
            st = int(raw[4] or 0)
        except ValueError:
            continue
        a = agg[cur_line]
        a[0] += w
        a[1] += t
        a[2] += st
    tw = sum(a[0] for a in agg.values())
    ts = sum(a[2] for a in agg.values())
    print(f"total warp instructions {tw:,}")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        if a[0] == 0:
            continue
        print(f"{100 * a[0] / tw:5.1f}% inst {100 * a[2] / max(ts, 1):5.1f}% stall  thr {a[1] / a[0]:4.1f}  "
              f"{k[0]}:{k[1]:>4s}  {a[3]}")


if __name__ == "__main__":
    main()
