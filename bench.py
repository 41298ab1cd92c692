"""Benchmark: B200 RANMAR generation + exact jump-ahead (arXiv 2512.00093).

Headline (BASELINE.json metric "RANMAR uniforms/s & HBM GB/s"): config 2 —
65,536 streams of make_streams(12345, 2^40) x 65,536 fp32 uniforms each
(2^32 values, 16 GiB stored to HBM). One step = the GPU's whole job for that
config: the stream starts (K3, make_streams) and the stored uniforms (K1).
At N GPUs each rank does the same job for its own stream range
[rank * 65536, (rank + 1) * 65536) of the same sequence (weak scaling, no
collective on the data path); NCCL only gathers per-rank checksums afterwards.

Extra keys on the same JSON line: config 3 (2^20 stream starts at J=2^120,
jumps/s), config 4 (consume-in-kernel, uniforms/s), config 5 (gaussians).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C2 = dict(seed=12345, j=2**40, n=65536, per=65536)
C3 = dict(seed=987654321, j=2**120, n=1 << 20)
C4 = dict(seed=42, j=2**64, n=1 << 20, per=1 << 20)
C5 = dict(seed=7, j=2**50, n=1 << 24, per=3, steps=100)
METRIC = "RANMAR uniforms/s & HBM GB/s at 1/2/4/8 B200; jump-aheads/s at J=2^120"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


def measured_int_peaks():
    """Integer-pipe peaks measured on a B200 of this pool by tools/micro/intpipes.cu
    (raw JSON lines committed in profiles/r2_intpipes.txt): IMAD lane-ops/s (the
    config-3 denominator) and the integer issue peak, the best of the IADD3/IMAD
    mixes (the config-4 denominator). None if the file is missing."""
    p = os.path.join(ROOT, "profiles", "r2_intpipes.txt")
    if not os.path.exists(p):
        return None
    modes = {}
    with open(p) as f:
        for line in f:
            if line.startswith("{"):
                d = json.loads(line)
                if "mode" in d:
                    modes[d["mode"]] = d["lane_ops_per_s"]
    issue = max(modes[k] for k in ("iadd", "mix_imad_iadd", "mix_imad_iadd_lop3"))
    return {"imad": modes["imad"], "int_issue": issue, "source": "profiles/r2_intpipes.txt"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.t = None

    def __enter__(self):
        self.started = time.perf_counter()
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def self_launch(args) -> int | None:
    """`python bench.py --gpus N` with N > 1 and no torchrun environment: re-run
    this script under torch.distributed.run with one rank per GPU (the form the
    driver uses), so the N-GPU number is never a 1-GPU run. Returns the exit
    code, or None when this process is already a rank (or N = 1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_setup(gpus: int, need_gpu: bool):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != gpus:
        raise SystemExit(f"bench.py: --gpus {gpus} but WORLD_SIZE={world} ranks were launched")
    # Test hook (never set by the driver): RANMAR_BENCH_SHARED_GPU=1 runs every rank on
    # cuda:0 over gloo, so the N > 1 code path (shards, max over ranks, gathers) can be
    # exercised on a one-GPU box; NCCL refuses two ranks on one device.
    shared = os.environ.get("RANMAR_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    if need_gpu and torch.cuda.device_count() < local + 1:
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{local}, "
                         f"{torch.cuda.device_count()} CUDA device(s) visible")
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl" if torch.cuda.is_available() and not shared else "gloo")
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_checksums(sums, world: int):
    """NCCL all-gather of per-rank checksums (after the timed region only)."""
    from paper_2512_00093_b200.shard import gather_u64
    return gather_u64(sums, device="cuda")


def settle(seconds: float = 1.0) -> None:
    """Idle before each extra config so it is not timed in the power-capped state the
    previous config (e.g. config 2's 100 x 16 GiB of stores) left the board in."""
    import torch
    torch.cuda.synchronize()
    time.sleep(seconds)


def load_traffic(kernel_key: str):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(kernel_key)
    return None


# ------------------------------------------------------------------ CPU arms

def cpu_reference_c2(steps: int = 1, warmup: int = 1, threads: int | None = None,
                     n: int | None = None):
    """The reference's own code (oracle/_ref, headers compiled in place) on the
    host cores: config 2's make_streams + step -> fp32 for n streams (default
    all 65,536: the whole config, ~1 s per step on 16 cores), stored to host RAM.
    Returns a dict, or None."""
    from oracle.bind import Reference, reference_available
    threads = threads or os.cpu_count() or 1
    n = C2["n"] if n is None else n
    per = C2["per"]
    if reference_available():
        import psutil
        ref, kind = Reference(), "reference"
        base = ref.init(C2["seed"])
        # the whole 16 GiB output when the host has room, else the same streams in
        # passes over a 4 GiB buffer (identical work: every uniform is stored once)
        chunk = n if psutil.virtual_memory().available > n * per * 4 + (8 << 30) else min(n, 16384)
        out = np.empty(chunk * per, np.float32)

        def run():
            for lo in range(0, n, chunk):
                ref.generate_f32(base, C2["j"], lo, min(chunk, n - lo), per, threads, out)
    else:  # fall back to the C restatement (single-threaded port)
        from oracle.bind import Oracle
        orc, kind, threads, chunk = Oracle(), "port", 1, 256
        n = min(n, 256)
        out = np.empty(n * per, np.float32)

        def run():
            ss = orc.make_streams(orc.init(C2["seed"]), C2["j"], n)
            out[:] = orc.generate_f32(ss, per)
    for _ in range(max(1, warmup)):
        run()  # warm-up (page-faults the output buffer)
    times = []
    for _ in range(max(1, steps)):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    t = statistics.mean(times)
    return {"value": n * per / t, "unit": "uniforms/s", "cores": threads, "kind": kind,
            "sample": f"config 2 streams [0, {n}) x {per} fp32 (make_streams + next_f64, "
                      f"stored to host RAM{'' if chunk == n else f' in passes of {chunk} streams'}), "
                      f"{threads} threads, mean of {len(times)} steps",
            "streams": n, "seconds": t, "steps": len(times)}


def cpu_reference_c1():
    """Config 1 on the reference's own single-thread loops (the CLI bench,
    ranmar_cli.cpp:195-212): 10^8 x step() and 10^8 x step_float() from seed 12345."""
    from oracle.bind import Reference, reference_available
    if not reference_available():
        return None
    ref = Reference()
    n = 10**8
    s = ref.init(12345)
    t0 = time.perf_counter()
    ref.lib.ref_step_n(s.ctypes.data, n, None)
    t1 = time.perf_counter()
    fbuf = np.empty(n, np.float64)
    t2 = time.perf_counter()
    ref.lib.ref_step_float_n(12345, n, fbuf.ctypes.data)
    t3 = time.perf_counter()
    return {"workload": "one stream, seed 12345, 10^8 outputs, 1 thread",
            "step_per_s": n / (t1 - t0), "step_float_per_s": n / (t3 - t2),
            "step_ms": (t1 - t0) * 1e3, "step_float_ms": (t3 - t2) * 1e3, "cores": 1}


def cpu_reference_text(states: np.ndarray):
    """The reference's to_text / from_text on all host cores, on a sample."""
    from oracle.bind import Reference, reference_available
    if not reference_available():
        return None
    ref, threads = Reference(), os.cpu_count() or 1
    t0 = time.perf_counter()
    buf, total = ref.to_text_bulk(states, threads)
    t1 = time.perf_counter()
    texts = [bytes(buf[k * 1408:(k + 1) * 1408]).rstrip(b"\0") for k in range(len(states))]
    blob = np.frombuffer(b"".join(texts), np.uint8)
    offs = np.cumsum([0] + [len(t) for t in texts]).astype(np.uint64)
    t2 = time.perf_counter()
    _, bad = ref.from_text_bulk(blob, offs, threads)
    t3 = time.perf_counter()
    assert bad == 0
    return {"to_text_states_per_s": len(states) / (t1 - t0),
            "from_text_states_per_s": len(states) / (t3 - t2), "cores": threads,
            "sample": f"{len(states)} states"}


def cpu_reference_extras():
    """Bounded samples of configs 3-5 and persistence on the host cores with
    the reference's own code (oracle/_ref); config 5 has no reference
    counterpart (gaussian() is repo-defined), so its line times the oracle
    port on one core. A few seconds in total."""
    from oracle.bind import GAUSS_DTYPE, Oracle, Reference, reference_available
    if not reference_available():
        return None
    ref, orc, threads = Reference(), Oracle(), os.cpu_count() or 1

    def best(fn, reps=3):
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return min(ts)

    ex = {}
    base3 = orc.init(C3["seed"], checked=False)  # init.hpp:19-20 rejects this seed; see DESIGN §5
    lat = best(lambda: ref.jump_state(base3, C3["j"]), 5)
    n3 = 64 * threads
    starts = best(lambda: ref.stream_starts(base3, C3["j"], 0, n3, threads), 2)
    batch_in = ref.stream_starts(base3, C3["j"], 0, n3, threads)
    jb = best(lambda: ref.jump_batch(batch_in, C3["j"], threads), 2)
    ex["config3"] = {"jump_state_latency_ms_1core": lat * 1e3,
                     "stream_starts_per_s": n3 / starts, "batched_jump_state_per_s": n3 / jb,
                     "cores": threads, "sample": f"k in [0, {n3}) at J = 2^120"}
    n4, per4 = 16 * threads, C4["per"]
    base4 = ref.init(C4["seed"])
    t4 = best(lambda: ref.consume(base4, C4["j"], 0, n4, per4, threads), 2)
    ex["config4"] = {"uniforms_per_s": n4 * per4 / t4, "cores": threads,
                     "sample": f"streams [0, {n4}) x 2^20 consumed (make_streams + step + sum + hist)"}
    n5 = 4096
    g5 = np.zeros(n5, GAUSS_DTYPE)
    g5["s"] = orc.make_streams(orc.init(C5["seed"]), C5["j"], n5)

    def run5():
        g = g5.copy()
        orc.gaussian_fill(g, C5["per"], C5["steps"])
    t5 = best(run5, 2)
    ex["config5"] = {"gaussians_per_s": n5 * C5["per"] * C5["steps"] / t5, "cores": 1,
                     "kind": "port", "sample": f"{n5} atoms x 3 x 100 gaussian() (oracle C port)"}
    ex["persistence"] = cpu_reference_text(ref.stream_starts(base3, C3["j"], 0, 16384, threads))
    return ex


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    # config 2 in full (65,536 streams = one rank's job), exactly --steps timed steps
    cb = cpu_reference_c2(steps=args.steps, warmup=args.warmup)
    line = {"metric": METRIC, "impl": "reference", "value": cb["value"], "unit": "uniforms/s",
            "n_gpus": world, "steps": cb["steps"], "warmup": args.warmup,
            "ms_per_step": cb["seconds"] * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded, BASELINE config 2)",
            "config": {"workload": "config 2: make_streams(12345, 2^40) streams [0, 65536) x 65536 fp32 "
                                   "uniforms stored" + ("" if world == 1 else
                                                        f" (rank 0's share of the {world}-GPU job)"),
                       "streams": cb["streams"], "per_stream": C2["per"],
                       "same_config": cb["streams"] == C2["n"] and cb["kind"] == "reference"},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": "uniforms/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    c1 = cpu_reference_c1()
    if c1:
        line["config1"] = c1
    extras = cpu_reference_extras()
    if extras:
        line.update(extras)
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm

def run_ours(args, rank, world, local):
    import torch

    import paper_2512_00093_b200 as rb

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    peak, peak_kind = measured_peaks()
    extras = {}

    # ---- config 2: make_streams + 2^32 fp32 stored, per rank ----
    n, per = C2["n"], C2["per"]
    from paper_2512_00093_b200.shard import weak_range
    first, _ = weak_range(n, rank)
    base = rb.init(C2["seed"])
    states = torch.empty((n, rb.STATE_WORDS), dtype=torch.int32, device=dev)
    ws = torch.empty(rb.lib().ranmar_make_streams_workspace(n), dtype=torch.uint8, device=dev)
    out = torch.empty(n * per, dtype=torch.float32, device=dev)

    def step(ev=None):
        with torch.cuda.stream(stream):
            rb.make_streams_dev(base, C2["j"], n, first=first, out=states, workspace=ws,
                                stream=stream)
            if ev:
                ev[0].record(stream)
            rb.generate(states, per, "f32", out=out, stream=stream)
            if ev:
                ev[1].record(stream)

    gen_events = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # The clock sampler starts during warm-up (nvidia-smi needs ~0.3 s to emit)
    # and stops right after the timed region, so every sample is under load.
    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        while time.perf_counter() - clk.started < 0.5:
            step()
            torch.cuda.synchronize()
        launches0 = rb.kernel_launches()
        barrier(world)
        torch.cuda.synchronize()
        t0.record(stream)
        for k in range(args.steps):
            step(gen_events[k])
        t1.record(stream)
        torch.cuda.synchronize()
        launches = rb.kernel_launches() - launches0
    barrier(world)
    ms_local = t0.elapsed_time(t1) / args.steps
    ms = max_over_ranks(ms_local, world)
    gen_ms = statistics.mean(a.elapsed_time(b) for a, b in gen_events)
    uniforms_step = n * per * world
    value = uniforms_step / (ms * 1e-3)
    gen_bytes = n * per * 4
    achieved = gen_bytes / (gen_ms * 1e-3) / 1e9
    # checksum of this rank's last step, gathered over NCCL after timing
    with torch.cuda.stream(stream):
        chk = int((out.view(n, per)[:, :1024].double() * 2**24).sum().item())
    torch.cuda.synchronize()
    sums = gather_checksums([first, chk], world)

    # ---- e2e: the same job through the host-buffer C-ABI path ----
    e2e = None
    if not args.no_e2e:
        # Pinned host output per rank: the full 16 GiB unless the ranks together would
        # pin more than a quarter of the host's RAM (then the leading streams of the range).
        import psutil
        budget = psutil.virtual_memory().total // 4 // world
        n_e2e = int(min(n, max(1, budget // (per * 4))))
        ctx = rb.Context(local)
        host_states = np.zeros(n_e2e, rb.STATE_DTYPE)
        host_out = torch.empty(n_e2e * per, dtype=torch.float32, pin_memory=True).numpy()
        e2e_steps = max(1, min(args.steps, 3))
        ctx.make_streams(C2["seed"], C2["j"], n_e2e, first=first, out=host_states)
        ctx.generate(host_states, per, "f32", out=host_out)  # warm-up
        h2d = d2h = 0
        barrier(world)
        tt = time.perf_counter()
        for _ in range(e2e_steps):
            ctx.make_streams(C2["seed"], C2["j"], n_e2e, first=first, out=host_states)
            a, b = ctx.traffic()
            ctx.generate(host_states, per, "f32", out=host_out)
            c, d = ctx.traffic()
            h2d, d2h = a + c, b + d
        e2e_s = max_over_ranks((time.perf_counter() - tt) / e2e_steps, world)
        # host result equals the device result of the timed step
        assert np.array_equal(host_out[:per * 4], out[:per * 4].cpu().numpy())
        e2e = {"value": n_e2e * per * world / e2e_s, "unit": "uniforms/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3,
               "streams_per_rank": n_e2e,
               "path": "ranmar_ctx_make_streams + ranmar_ctx_generate_f32 into pinned host memory"}
        del host_out
        ctx.close()

    # ---- config 1: one stream, seed 12345, 10^8 fp32 uniforms at full width ----
    settle()
    if not args.quick:
        n1 = 10**8
        s1 = rb.states_to_device(rb.init(12345)).to(dev)
        out1 = torch.empty(n1, dtype=torch.float32, device=dev)
        rb.generate_single(s1, n1, "f32", out=out1, stream=stream)  # warm-up
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        rb.generate_single(s1, n1, "f32", out=out1, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        ms1 = max_over_ranks(a.elapsed_time(b), world)
        extras["config1"] = {"workload": "one stream (seed 12345) x 10^8 fp32, split into 8,192-output "
                                         "substreams (make_streams) and re-joined; state ends as 10^8 x step()",
                             "ms": ms1, "uniforms_per_s": n1 / (ms1 * 1e-3),
                             "roofline": {"bound": "hbm", "unit": "GB/s", "achieved": n1 * 4 / (ms1 * 1e-3) / 1e9,
                                          "peak": peak, "frac": n1 * 4 / (ms1 * 1e-3) / 1e9 / peak,
                                          "peak_kind": f"{peak_kind} copy GB/s (MEASURED_PEAKS.json hbm_gbs)",
                                          "algorithmic_per_unit": "4 B stored per uniform (the whole call: "
                                                                  "substream starts, generation, re-join)"}}
        del out1

    # ---- config 3: 2^20 stream starts at J = 2^120 (jump-aheads/s) ----
    settle()
    if not args.quick:
        n3 = C3["n"]
        base3 = rb.init_unchecked(C3["seed"])
        st3 = torch.empty((n3, rb.STATE_WORDS), dtype=torch.int32, device=dev)
        ws3 = torch.empty(rb.lib().ranmar_make_streams_workspace(n3), dtype=torch.uint8, device=dev)
        first3 = rank * n3

        def step3():
            rb.make_streams_dev(base3, C3["j"], n3, first=first3, out=st3, workspace=ws3,
                                stream=stream)

        for _ in range(3):
            step3()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        reps = 10
        for _ in range(reps):
            step3()
        b.record(stream)
        torch.cuda.synchronize()
        ms3_direct = max_over_ranks(a.elapsed_time(b) / reps, world)
        # the same 5 launches captured once in a CUDA graph (the _dev entry points are
        # capturable) and replayed: the device time without host launch gaps
        g3 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g3, stream=stream):
            step3()
        torch.cuda.synchronize()
        trials = []
        for _ in range(5):  # median of 5 trials of 10 replays (0.1 ms launches: clock-sensitive)
            a.record(stream)
            with torch.cuda.stream(stream):
                for _ in range(reps):
                    g3.replay()
            b.record(stream)
            torch.cuda.synchronize()
            trials.append(a.elapsed_time(b) / reps)
        ms3 = max_over_ranks(statistics.median(trials), world)
        # generic batched jump: every state jumped by 2^120 (one P_J, 2^20 applies)
        jo = torch.empty_like(st3)
        rb.jump_dev(st3, C3["j"], out=jo, stream=stream)
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(reps):
            rb.jump_dev(st3, C3["j"], out=jo, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        msj = max_over_ranks(a.elapsed_time(b) / reps, world)
        extras["config3"] = {
            "workload": "make_streams(init_unchecked(987654321), 2^120): 2^20 stream starts s_{kJ} per rank",
            "jump_aheads_per_s": n3 * world / (ms3 * 1e-3), "ms": ms3,
            "timing": "CUDA-graph replay of the make_streams_dev launches, median of 5 x 10 replays",
            "ms_trials": trials,
            "ms_direct_calls": ms3_direct,
            "batched_jump_state_per_s": n3 * world / (msj * 1e-3), "batched_jump_ms": msj,
            "macs_per_start_bulk": 97 * 97}
        ip = measured_int_peaks()
        # Level 0 of the stream-start tree runs on the tensor cores (bulk_tc_kernel,
        # exact u8-limb kind::i8 MMAs); its floor is the HBM write of the states
        # (400 B per start). The whole config (all launches) against that floor,
        # and the 24-bit MAC rate against the measured IMAD peak it replaces.
        state_bytes = n3 * 400
        extras["config3"]["roofline"] = {
            "bound": "hbm", "unit": "GB/s", "achieved": state_bytes / (ms3 * 1e-3) / 1e9, "peak": peak,
            "frac": state_bytes / (ms3 * 1e-3) / 1e9 / peak,
            "peak_kind": f"{peak_kind} copy GB/s (MEASURED_PEAKS.json hbm_gbs)",
            "algorithmic_per_unit": "one 400-B state written per stream start (97 x 97 = 9,409 24-bit MACs)",
            "kernel": "bulk_tc_kernel (tcgen05.mma kind::i8) + pow_table / tables / level"}
        if ip:
            ach = n3 * 97 * 97 / (ms3 * 1e-3)
            extras["config3"]["mac_rate_vs_imad_peak"] = {
                "achieved_TMAC_per_s": ach / 1e12, "imad_peak_TMAC_per_s": ip["imad"] / 1e12,
                "ratio": ach / ip["imad"], "peak_kind": f"measured ({ip['source']}, mode imad)"}
        # §8f row 1: export / re-import the 2^20 starts as reference text on the device
        text, off = rb.to_text_dev(st3, stream=stream)
        back, err = rb.from_text_dev(text, off, stream=stream)
        torch.cuda.synchronize()
        assert int(err.abs().sum()) == 0 and torch.equal(back, st3)
        tb = int(off[-1].item())
        ttw = torch.empty(int(rb.lib().ranmar_text_workspace(n3)), dtype=torch.uint8, device=dev)
        tt_text, tt_off = torch.empty_like(text), torch.empty_like(off)  # buffers reused per call
        rb.to_text_dev(st3, stream=stream, text=tt_text, offsets=tt_off, workspace=ttw)
        a.record(stream)
        for _ in range(reps):
            rb.to_text_dev(st3, stream=stream, text=tt_text, offsets=tt_off, workspace=ttw)
        b.record(stream)
        torch.cuda.synchronize()
        ms_tt = max_over_ranks(a.elapsed_time(b) / reps, world)
        ft_out, ft_err = torch.empty_like(back), torch.empty_like(err)
        a.record(stream)
        for _ in range(reps):
            rb.from_text_dev(text, off, stream=stream, out=ft_out, err=ft_err)
        b.record(stream)
        torch.cuda.synchronize()
        ms_ft = max_over_ranks(a.elapsed_time(b) / reps, world)
        extras["persistence"] = {
            "workload": "to_text / from_text of config 3's 2^20 stream starts (reference text format)",
            "text_bytes": tb, "to_text_states_per_s": n3 * world / (ms_tt * 1e-3),
            "from_text_states_per_s": n3 * world / (ms_ft * 1e-3),
            "to_text_ms": ms_tt, "from_text_ms": ms_ft,
            # algorithmic bytes: the states read + the text written (to_text), and back (from_text)
            "roofline": {"bound": "hbm", "unit": "GB/s", "peak": peak,
                         "to_text_achieved": (tb + n3 * 400) / (ms_tt * 1e-3) / 1e9,
                         "from_text_achieved": (tb + n3 * 400) / (ms_ft * 1e-3) / 1e9,
                         "to_text_frac": (tb + n3 * 400) / (ms_tt * 1e-3) / 1e9 / peak,
                         "from_text_frac": (tb + n3 * 400) / (ms_ft * 1e-3) / 1e9 / peak,
                         "note": "both kernels are instruction-bound (character-level work), see DESIGN §3 K7"}}
        if world == 1 and not args.no_cpu:
            extras["persistence"]["cpu_reference"] = cpu_reference_text(rb.states_to_host(st3[:1 << 16]))
        del st3, ws3, jo, text, off, back, err, tt_text, tt_off, ttw, ft_out, ft_err

    # ---- config 4: consume in kernel (no store) ----
    settle()
    if not args.quick:
        n4 = C4["n"] if not args.c4_streams else args.c4_streams
        st4 = torch.empty((n4, rb.STATE_WORDS), dtype=torch.int32, device=dev)
        ws4 = torch.empty(rb.lib().ranmar_make_streams_workspace(n4), dtype=torch.uint8, device=dev)
        sums4 = torch.empty(n4, dtype=torch.int64, device=dev)
        hist4 = torch.empty((n4, 256), dtype=torch.int32, device=dev)
        first4 = rank * n4

        def step4():
            rb.make_streams_dev(rb.init(C4["seed"]), C4["j"], n4, first=first4, out=st4,
                                workspace=ws4, stream=stream)
            rb.consume(st4, C4["per"], sums=sums4, hist=hist4, stream=stream)

        step4()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step4()
        b.record(stream)
        torch.cuda.synchronize()
        ms4 = max_over_ranks(a.elapsed_time(b), world)
        extras["config4"] = {"workload": f"{n4} streams x 2^20 uniforms consumed per rank "
                                         "(make_streams(42, 2^64) + per-stream u64 sum + 256-bin hist)",
                             "uniforms_per_s": n4 * C4["per"] * world / (ms4 * 1e-3), "ms": ms4}
        ip = measured_int_peaks()
        if ip:
            # 9 int32 ops per uniform (core.hpp:56-65's 7 + sum + histogram)
            ach = 9 * n4 * C4["per"] / (ms4 * 1e-3)
            extras["config4"]["roofline"] = {
                "bound": "int_issue", "unit": "Tops/s", "achieved": ach / 1e12,
                "peak": ip["int_issue"] / 1e12, "frac": ach / ip["int_issue"],
                "peak_kind": f"measured ({ip['source']}, best of the IADD3, IADD3+IMAD and IADD3+IMAD+LOP3 issue rates)",
                "algorithmic_per_unit": "9 int32 ops per uniform (SURVEY §8d C4)"}
        # after timing: all-gather the per-stream sums, all-reduce the histogram
        from paper_2512_00093_b200.shard import allgather_tensor, allreduce_sum
        all_sums = allgather_tensor(sums4)
        hist_tot = allreduce_sum(hist4.to(torch.int64).sum(dim=0))
        assert int(hist_tot.sum()) == n4 * C4["per"] * world  # every uniform counted once
        extras["config4"]["gathered"] = {
            "streams": int(all_sums.numel()), "sum_of_sums": int(all_sums.sum()) & ((1 << 64) - 1),
            "hist_total": int(hist_tot.sum())}
        del st4, ws4, sums4, hist4, all_sums

    # ---- config 5: gaussians ----
    settle()
    if not args.quick:
        n5 = C5["n"]
        st5 = torch.empty((n5, rb.STATE_WORDS), dtype=torch.int32, device=dev)
        ws5 = torch.empty(rb.lib().ranmar_make_streams_workspace(n5), dtype=torch.uint8, device=dev)
        rb.make_streams_dev(rb.init(C5["seed"]), C5["j"], n5, first=rank * n5, out=st5,
                            workspace=ws5, stream=stream)
        g5 = rb.gauss_states_from(st5)
        del st5, ws5
        out5 = torch.empty((C5["steps"], n5, C5["per"]), dtype=torch.float64, device=dev)
        g5w = g5.clone()
        # warm-up: the full launch (the kernel K4 runs; a short launch would take the
        # in-place K6 path and leave K4's first-launch module load in the timed region)
        rb.gaussian(g5w, C5["per"], C5["steps"], out=out5, stream=stream)
        torch.cuda.synchronize()
        trials5 = []
        for _ in range(3):  # each trial from the same start states, copied outside the timing
            g5w.copy_(g5)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            rb.gaussian(g5w, C5["per"], C5["steps"], out=out5, stream=stream)
            b.record(stream)
            torch.cuda.synchronize()
            trials5.append(max_over_ranks(a.elapsed_time(b), world))
        ms5 = sorted(trials5)[1]
        nbytes = out5.numel() * 8 + 2 * n5 * 416
        extras["config5"] = {"workload": "2^24 atoms x 3 gaussian() x 100 steps per rank, fp64 out",
                             "gaussians_per_s": out5.numel() * world / (ms5 * 1e-3), "ms": ms5,
                             "timing": "median of 3 launches after a full warm-up launch",
                             "ms_trials": trials5,
                             "GB_per_s": nbytes / (ms5 * 1e-3) / 1e9,
                             "roofline": {"bound": "hbm", "unit": "GB/s",
                                          "achieved": nbytes / (ms5 * 1e-3) / 1e9, "peak": peak,
                                          "frac": nbytes / (ms5 * 1e-3) / 1e9 / peak}}
        # the same deviates consumed in-kernel (§8f row 4): per-atom sum and sum of
        # squares, nothing stored -- the gaussian() rate without the store
        mom5 = torch.empty((n5, 2), dtype=torch.float64, device=dev)
        g5w.copy_(g5)
        rb.gaussian_moments(g5w, C5["per"] * C5["steps"], out=mom5, stream=stream)  # warm-up
        torch.cuda.synchronize()
        trials_m = []
        for _ in range(3):
            g5w.copy_(g5)
            torch.cuda.synchronize()
            a.record(stream)
            rb.gaussian_moments(g5w, C5["per"] * C5["steps"], out=mom5, stream=stream)
            b.record(stream)
            torch.cuda.synchronize()
            trials_m.append(max_over_ranks(a.elapsed_time(b), world))
        ms_m = sorted(trials_m)[1]
        extras["config5_moments"] = {
            "workload": "config 5's deviates consumed in-kernel: per-atom sum and sum of squares, no store",
            "ms": ms_m, "ms_trials": trials_m,
            "gaussians_per_s": n5 * C5["per"] * C5["steps"] * world / (ms_m * 1e-3)}
        del mom5
        # after timing: every rank's deviate sum and sum of squares, all-gathered
        from paper_2512_00093_b200.shard import allgather_tensor
        # squares by chunked dots (no 40 GB temporary; BLAS dot takes < 2^31 elements)
        flat5 = out5.view(-1)
        sq5 = sum(torch.dot(c, c) for c in flat5.split(1 << 30))
        mom = torch.stack([flat5.sum(dtype=torch.float64), sq5])
        mom = allgather_tensor(mom).view(-1, 2)
        cnt5 = out5.numel() * world
        extras["config5"]["gathered"] = {"mean": float(mom[:, 0].sum()) / cnt5,
                                         "mean_square": float(mom[:, 1].sum()) / cnt5}

        # the same 100 steps launched one MD step at a time (3 deviates per atom
        # per launch: states stepped in place, K6), then the fused consumer
        def timed(fn, reps):
            g5w.copy_(g5)
            fn()  # warm-up launch
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            return max_over_ranks(e0.elapsed_time(e1), world) / reps

        steps5 = C5["steps"]
        ms_ps = timed(lambda: rb.gaussian(g5w, C5["per"], 1, out=out5[0:1], stream=stream), steps5)
        extras["config5"]["per_step_launches"] = {
            "ms_per_step": ms_ps, "ms_100_steps": ms_ps * steps5,
            "gaussians_per_s": n5 * C5["per"] * world / (ms_ps * 1e-3)}
        del out5
        gen = torch.Generator(device=dev).manual_seed(5)
        vel = torch.randn((n5, 3), dtype=torch.float64, device=dev, generator=gen)
        frc = torch.zeros((n5, 3), dtype=torch.float64, device=dev)
        typ = torch.ones(n5, dtype=torch.int32, device=dev)
        lang = {"workload": "2^24 atoms, one stream per atom (config 5 streams), f += g1 v + "
                            "g2 r per component, one launch per MD step"}
        for name, noise in (("uniform", rb.NOISE_UNIFORM), ("gaussian", rb.NOISE_GAUSSIAN)):
            gf1, gf2 = rb.langevin_factors([0.0, 1.0], 0.1, 0.005, noise=noise)
            d1, d2 = torch.from_numpy(gf1).to(dev), torch.from_numpy(gf2).to(dev)
            ms_l = timed(lambda: rb.langevin(g5w, vel, frc, typ, d1, d2, 1.0, noise,
                                             stream=stream), 20)
            # algorithmic bytes per atom-step: v 24 + f 24 read + 24 written + type 4 +
            # state cursors/v 12 read + 12 written + 2 x 3 ring words read + 3 written
            # (uniform: 3 uniforms; gaussian: ~3.8 uniforms, counted as 3)
            lang[name] = {"ms_per_step": ms_l, "atoms_per_s": n5 * world / (ms_l * 1e-3),
                          "algorithmic_GB_per_s": n5 * 136 / (ms_l * 1e-3) / 1e9}
        # the same uniform-noise consumer on a stream bank (slot-major, coalesced)
        gf1, gf2 = rb.langevin_factors([0.0, 1.0], 0.1, 0.005, noise=rb.NOISE_UNIFORM)
        d1, d2 = torch.from_numpy(gf1).to(dev), torch.from_numpy(gf2).to(dev)
        bank = rb.bank_from_states(g5w)
        tb = [0]

        def bank_step():
            tb[0] = rb.langevin_bank(bank, tb[0], vel, frc, typ, d1, d2, 1.0, stream=stream)
        ms_b = timed(bank_step, 20)
        lang["uniform_bank"] = {"ms_per_step": ms_b, "atoms_per_s": n5 * world / (ms_b * 1e-3),
                                "algorithmic_GB_per_s": n5 * 120 / (ms_b * 1e-3) / 1e9,
                                "roofline_frac": n5 * 120 / (ms_b * 1e-3) / 1e9 / peak}
        del bank
        # gaussian noise drawn for all 100 steps by one K4 launch (per_step 3), then one
        # element-wise consumer per MD step (ranmar_langevin_noise_dev): amortised per step
        gf1, gf2 = rb.langevin_factors([0.0, 1.0], 0.1, 0.005, noise=rb.NOISE_GAUSSIAN)
        d1, d2 = torch.from_numpy(gf1).to(dev), torch.from_numpy(gf2).to(dev)
        noise = torch.empty((steps5, n5, 3), dtype=torch.float64, device=dev)
        ms_gen = timed(lambda: rb.gaussian(g5w, 3, steps5, out=noise, stream=stream), 2)
        ts = [0]

        def noise_step():
            rb.langevin_noise(noise[ts[0] % steps5], vel, frc, typ, d1, d2, 1.0, stream=stream)
            ts[0] += 1
        ms_c = timed(noise_step, 20)
        ms_pg = ms_gen / steps5 + ms_c
        lang["gaussian_pregenerated"] = {
            "ms_per_step": ms_pg, "atoms_per_s": n5 * world / (ms_pg * 1e-3),
            "generate_ms_100_steps": ms_gen, "consumer_ms_per_step": ms_c,
            "consumer_GB_per_s": n5 * 100 / (ms_c * 1e-3) / 1e9,
            "consumer_roofline_frac": n5 * 100 / (ms_c * 1e-3) / 1e9 / peak,
            "note": "one gaussian() launch draws 100 steps x 3 deviates per atom (K4), then one "
                    "launch per MD step reads its 24 B of noise per atom (100 B per atom-step)"}
        del noise
        extras["langevin"] = lang
        del g5, g5w, vel, frc, typ

    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        # a bounded sample (a quarter of config 2's streams, ~0.3 s on 16 cores):
        # the full config is the reference arm's job (bench.py --impl reference)
        cb = cpu_reference_c2(steps=1, warmup=1, n=16384)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    line = {
        "metric": METRIC, "value": value, "unit": "uniforms/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded streams, BASELINE config 2)",
        "config": {"workload": "config 2: make_streams(12345, 2^40) streams [rank*65536, +65536) "
                               "x 65536 fp32 uniforms stored per rank (16 GiB/rank)",
                   "streams_per_rank": n, "per_stream": per, "output": "fp32, stream-major",
                   "l2": "output (16 GiB) >> L2 (126 MB): no flush needed",
                   "parallelism": f"stream-range partition x{world}, no data-path collective"},
        "hbm_GB_per_s": n * per * 4 * world / (ms * 1e-3) / 1e9,
        "roofline": {"bound": "hbm", "kernel": "gen_store_kernel<float>", "achieved": achieved,
                     "peak": peak, "peak_kind": f"{peak_kind} copy GB/s (MEASURED_PEAKS.json hbm_gbs)",
                     "unit": "GB/s", "frac": achieved / peak,
                     "traffic": load_traffic("gen_store_kernel<float>"),
                     "algorithmic_bytes_per_launch": gen_bytes, "kernel_ms": gen_ms},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
        "checksums": sums, **extras,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--quick", action="store_true", help="config 2 only")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--c4-streams", type=int, default=0)
    args = ap.parse_args()
    rc = self_launch(args)
    if rc is not None:
        sys.exit(rc)
    rank, world, local = dist_setup(args.gpus, need_gpu=args.impl == "ours")
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
    else:
        run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
