"""Stream-range partitioner for one process per GPU.

The streams of make_streams(base, J, N) are independent units (jump.hpp:97-104:
StreamMode::independent is "safe to compute concurrently"), so rank r of W
simply owns a contiguous range and derives its own starts s_{kJ} from the seed
with ranmar_make_streams_dev(first=range.start). There is no exchange on the
data path; collectives only gather per-rank checksums after the timed region.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def stream_range(n_total: int, world: int, rank: int) -> Tuple[int, int]:
    """Balanced contiguous split: (first, count) of rank `rank` (strong scaling)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    lo = n_total * rank // world
    hi = n_total * (rank + 1) // world
    return lo, hi - lo


def weak_range(n_per_rank: int, rank: int) -> Tuple[int, int]:
    """Weak scaling: every rank owns n_per_rank streams of one global sequence."""
    return rank * n_per_rank, n_per_rank


def _host_if_gloo(t):
    """gloo's all_gather has no CUDA path: carry CUDA tensors through the host there
    (NCCL, the multi-GPU backend, takes them as they are)."""
    import torch.distributed as dist
    return t.cpu() if t.is_cuda and dist.get_backend() == "gloo" else t


def gather_u64(values: Sequence[int], device=None) -> List[List[int]]:
    """All-gather a short list of u64 checksums from every rank (torch.distributed;
    NCCL on GPUs, gloo on CPU). Values are carried as int64 bit patterns."""
    import torch
    import torch.distributed as dist

    def to_i64(x: int) -> int:
        x &= (1 << 64) - 1
        return x - (1 << 64) if x >= 1 << 63 else x

    t = torch.tensor([to_i64(v) for v in values], dtype=torch.int64, device=device)
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return [[v & ((1 << 64) - 1) for v in t.tolist()]]
    t = _host_if_gloo(t)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [[v & ((1 << 64) - 1) for v in o.tolist()] for o in out]


def allgather_tensor(t):
    """All-gather a tensor from every rank (after the timed region only): the
    per-stream u64 sums of config 4, 8 B x streams per rank.
    Returns the concatenation in rank order; the tensor itself at world size 1."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return t
    src = _host_if_gloo(t.contiguous())
    out = [torch.empty_like(src) for _ in range(dist.get_world_size())]
    dist.all_gather(out, src)
    return torch.cat(out).to(t.device)


def allreduce_sum(t):
    """Sum-reduce a tensor over ranks in place (the 256-bin histogram total)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        src = _host_if_gloo(t)
        dist.all_reduce(src, op=dist.ReduceOp.SUM)
        if src is not t:
            t.copy_(src)
    return t
