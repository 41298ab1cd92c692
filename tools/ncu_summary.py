"""Summarise ncu captures for profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py full <report.ncu-rep> [...]   -> key metrics per kernel (JSON)
    python tools/ncu_summary.py launches <launches.csv>       -> per-kernel share of the launch list
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
    "smsp__inst_executed.sum", "lts__t_bytes.sum",
    "smsp__average_warp_latency_issue_stalled_barrier", "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
]


def full(paths):
    out = {}
    for p in paths:
        raw = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        h, units = rows[0], rows[1]
        for r in rows[2:]:
            name = r[h.index("Kernel Name")].split("(")[0]
            d = {}
            for k in KEYS:
                if k in h:
                    i = h.index(k)
                    d[k] = f"{r[i]} {units[i]}".strip()
            out[f"{p}:{name}"] = d
    print(json.dumps(out, indent=1))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, rows = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    if "Metric Name" in h:  # launch lists may carry DRAM byte counts too: time only
        mi = h.index("Metric Name")
        rows = [r for r in rows if len(r) > mi and r[mi] == "gpu__time_duration.sum"]
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(list)
    for r in rows:
        agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3))
    tot = sum(sum(v) for v in agg.values())
    print(f"{path}: {sum(len(v) for v in agg.values())} launches, {tot:.1f} us total "
          "(ncu: cold cache, serialised)")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"  {k[:70]:70s} n={len(v):4d} mean={sum(v)/len(v):10.2f} us  share={100*sum(v)/tot:5.1f}%")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2:])
    else:
        for p in sys.argv[2:]:
            launches(p)
