"""Multi-process plumbing for `bench.py --gpus N` (one process per GPU).

The MLK solve of one space-time problem runs on one GPU (north star; SURVEY
section 8(e)).  N > 1 runs replicas: every rank solves its own seeded
instance, with no data-path collective; the only collective is the
max-over-ranks of the measured times (and a barrier around the timed region).
"""

from __future__ import annotations

import os


def rank_info() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str = "nccl") -> None:
    import torch.distributed as dist

    if not dist.is_initialized():
        dist.init_process_group(backend)


def instance_seed(base_seed: int, rank: int) -> int:
    """Seed of a rank's independent instance (rank 0 solves the base case)."""
    return base_seed + rank


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (identity without a process group)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier() -> None:
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.barrier()
