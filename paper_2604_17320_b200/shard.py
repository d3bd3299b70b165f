"""Data-parallel plumbing for the QUOTA path.

Sequences are independent (no cross-sequence state anywhere in
model.cpp), so a request/image batch is sharded across ranks -- one process per
GPU -- and every rank runs the whole per-layer path on its own shard with no
collective.  torch.distributed (NCCL on the B200 box, gloo in the CPU tests)
is used only after the path: to gather the final logits / retained-index
traces to rank 0 and to take the max-over-ranks step time.
"""
from __future__ import annotations

import torch


def shard_range(n_total: int, world: int, rank: int):
    """Contiguous balanced split of n_total sequences: (first, count) for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def gather_rows(local: torch.Tensor, group=None):
    """Concatenate every rank's [n_r x ...] rows (n_r may differ) in rank order on
    every rank.  Pads to the max row count so one fixed-size all_gather suffices."""
    import torch.distributed as dist
    ws = dist.get_world_size(group)
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    counts = [torch.zeros_like(n) for _ in range(ws)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    mx = max(counts)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(ws)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)


def gather_equal_rows(local: torch.Tensor, out: torch.Tensor, group=None):
    """Every rank's [n x ...] rows (the same n on every rank -- the weak-scaling bench shards
    an equal per-GPU batch) into out [world * n x ...] in rank order, with one
    all_gather_into_tensor and no host synchronisation (it can sit inside a timed region
    and a CUDA stream's order)."""
    import torch.distributed as dist
    dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    return out


def max_over_ranks(value: float, device="cpu", group=None) -> float:
    """The job's time is the slowest rank's (bench.py contract)."""
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
