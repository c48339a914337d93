"""Multi-GPU plumbing: pairs are independent, so ranks shard the pair list
with no data-path collective; the only collectives are a barrier around the
timed region and one max-reduction of the per-rank device time."""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env():
    """(rank, world, local_rank) from torchrun's environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def shard(n_pairs: int, world: int, rank: int) -> range:
    """Contiguous block of global pair indices owned by `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n_pairs, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def init(backend: str, local_rank: int | None = None):
    if dist.is_initialized():
        return
    kw = {}
    if backend == "nccl" and local_rank is not None:
        kw["device_id"] = torch.device(f"cuda:{local_rank}")
    dist.init_process_group(backend, **kw)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (the timed region's device milliseconds)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier():
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
