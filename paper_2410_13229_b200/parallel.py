"""Batch-sharded data parallelism over independent sequences.

Requests are independent (model.py:310 loops over sequences; SPEC: safe to run
concurrently), so B sequences are split contiguously across the ranks of a
`torch.distributed` group (one process per GPU, NCCL over NVLink on the box,
gloo in the CPU tests).  Every rank holds a full model replica; there is no
collective in the forward pass.  The only communication is an all_gather of
the per-rank outputs (generated token ids or last-position logits) at the end.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(B: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced split of B sequences: ranks < B % world get one extra."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("invalid rank / world size")
    base, extra = divmod(B, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard(x: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    s, e = shard_range(x.shape[0], rank, world)
    return x[s:e]


def gather_rows(local: torch.Tensor, B: int, group=None) -> torch.Tensor:
    """All-gather per-rank row blocks (leading dim = that rank's shard size) into
    the full [B, ...] tensor in rank order.  Shards may be ragged: each rank
    pads to the largest shard, gathers, then trims."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [shard_range(B, r, world) for r in range(world)]
    cap = max(e - s for s, e in sizes)
    if local.shape[0] != sizes[rank][1] - sizes[rank][0]:
        raise ValueError("local rows do not match this rank's shard")
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world * cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    parts = [out[r * cap: r * cap + (e - s)] for r, (s, e) in enumerate(sizes)]
    return torch.cat(parts, dim=0)


def dp_greedy_generate(dm, prompts: torch.Tensor, steps: int, group=None) -> torch.Tensor:
    """Greedy generation for all B prompts across the group: each rank decodes its
    shard on its own GPU (DeviceModel.greedy_generate), then the token ids are
    all-gathered so every rank returns the full [B, T + steps] result."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    B = prompts.shape[0]
    mine = shard(prompts, rank, world)
    out = dm.greedy_generate(mine, steps) if mine.shape[0] else torch.empty(
        (0, prompts.shape[1] + steps), dtype=torch.int64, device=prompts.device)
    return gather_rows(out.to(torch.int64), B, group)
