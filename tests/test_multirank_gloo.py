"""World-size-2 check of the multi-GPU path's host side on CPU (gloo): each
rank owns a contiguous stream range (paper_2512_00093_b200.shard), computes
its streams' per-stream sums independently (here with the CPU oracle standing
in for the kernels), and the checksums are all-gathered. Rank 0 verifies the
gathered ranges tile make_streams over the whole range exactly as one process
computes them — the property the GPU ranks rely on (no data-path collective)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_total, per, result_q, mode):
    import torch.distributed as dist

    from oracle.bind import Oracle
    from paper_2512_00093_b200.shard import gather_u64, stream_range, weak_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        base = orc.init(12345)
        first, cnt = stream_range(n_total, world, rank) if mode == "strong" else weak_range(n_total, rank)
        states = orc.make_streams(base, 2**40, cnt, first=first)
        sums, _ = orc.consume(states, per)
        gathered = gather_u64([first, cnt] + [int(x) for x in sums] + [0] * (n_total - cnt))
        if rank == 0:
            result_q.put(gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["strong", "weak"])
def test_two_rank_partition_and_gather(oracle, mode):
    world, n, per = 2, 7, 500
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, per, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # reassemble in rank order and compare with a single-process computation
    total = n if mode == "strong" else world * n
    got = []
    expect_first = 0
    for row in gathered:
        first, cnt = row[0], row[1]
        assert first == expect_first  # contiguous, non-overlapping, in rank order
        got += row[2:2 + cnt]
        expect_first += cnt
    assert expect_first == total
    states = oracle.make_streams(oracle.init(12345), 2**40, total)
    sums, _ = oracle.consume(states, per)
    assert got == [int(x) for x in sums]


def test_stream_range_properties():
    from paper_2512_00093_b200.shard import stream_range
    for n in (0, 1, 7, 65536, 2**20 + 3):
        for w in (1, 2, 3, 8):
            parts = [stream_range(n, w, r) for r in range(w)]
            assert sum(c for _, c in parts) == n
            assert all(parts[r][0] + parts[r][1] == parts[r + 1][0] for r in range(w - 1))
            assert max(c for _, c in parts) - min(c for _, c in parts) <= 1
    with pytest.raises(ValueError):
        stream_range(10, 2, 2)


def _worker_tensors(rank, world, port, n, per, result_q):
    import torch
    import torch.distributed as dist

    from oracle.bind import Oracle
    from paper_2512_00093_b200.shard import allgather_tensor, allreduce_sum, weak_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        first, cnt = weak_range(n, rank)
        sums, hist = orc.consume(orc.make_streams(orc.init(42), 2**64, cnt, first=first), per)
        all_sums = allgather_tensor(torch.from_numpy(sums.view(np.int64).copy()))
        tot = allreduce_sum(torch.from_numpy(hist.astype(np.int64)).sum(dim=0))
        if rank == 0:
            result_q.put((all_sums.numpy().view(np.uint64).tolist(), tot.numpy().tolist()))
    finally:
        dist.destroy_process_group()


def test_two_rank_sums_gather_and_histogram_reduce(oracle):
    # bench.py's config-4 collectives after timing: all-gather of
    # the per-stream u64 sums, all-reduce of the 256-bin histogram
    world, n, per = 2, 5, 700
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_tensors, args=(r, world, port, n, per, q))
             for r in range(world)]
    for p in procs:
        p.start()
    sums, tot = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    exp_sums, exp_hist = oracle.consume(
        oracle.make_streams(oracle.init(42), 2**64, world * n), per)
    assert sums == [int(x) for x in exp_sums]
    assert tot == exp_hist.astype(np.int64).sum(axis=0).tolist()
    assert sum(tot) == world * n * per
