"""Multi-GPU plumbing: one process per GPU over torch.distributed (NCCL).

Ensembles (BASELINE configs 1 and 4) shard by member with no data-path
collective: draws are keyed by (seed, step, cell, member), so the
member->rank mapping cannot change any trajectory.  Ensemble calibration
(config 4) sums the per-member parameter gradients with one all-reduce of
4 fp64 values per iteration, then every rank applies the same AdamW step.
"""
from __future__ import annotations

import os
from typing import List, Tuple

import torch


def env_rank() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def init_distributed(backend: str = None):
    rank, world, local = env_rank()
    if world > 1 and not torch.distributed.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        torch.distributed.init_process_group(backend, rank=rank, world_size=world)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local


def shard_members(n_members: int, rank: int, world: int) -> List[int]:
    """Contiguous member block of this rank (sizes differ by at most one)."""
    base, extra = divmod(n_members, world)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))


def allreduce_sum_(t: torch.Tensor) -> torch.Tensor:
    """In-place sum over ranks (no-op for a single process)."""
    if torch.distributed.is_initialized() and torch.distributed.get_world_size() > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.SUM)
    return t


def allreduce_max(value: float, device=None) -> float:
    if torch.distributed.is_initialized() and torch.distributed.get_world_size() > 1:
        t = torch.tensor([value], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())
    return value


def barrier():
    if torch.distributed.is_initialized() and torch.distributed.get_world_size() > 1:
        torch.distributed.barrier()
