"""Multi-GPU plumbing: one process per GPU, rows sharded across ranks.

CutMax rows are independent, so the data path has no
collective: each rank runs the fused kernels on its contiguous row shard.
torch.distributed is used only to start the ranks, for barriers around the
timed region and to take the max of per-rank device times.
"""
from __future__ import annotations

import os

from .workloads import shard_rows

__all__ = ["DistEnv", "init_from_env", "shard_rows"]


class DistEnv:
    def __init__(self, rank: int, world: int, local_rank: int, backend: str | None):
        self.rank, self.world, self.local_rank, self.backend = rank, world, local_rank, backend

    @property
    def enabled(self) -> bool:
        return self.backend is not None

    def barrier(self) -> None:
        if self.enabled:
            import torch.distributed as dist

            dist.barrier()

    def max_over_ranks(self, value: float) -> float:
        """Max of a per-rank scalar (the job time is the slowest rank's)."""
        if not self.enabled:
            return float(value)
        import torch
        import torch.distributed as dist

        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(self, value: float) -> float:
        if not self.enabled:
            return float(value)
        import torch
        import torch.distributed as dist

        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    def shard(self, B: int):
        return shard_rows(B, self.rank, self.world)

    def close(self) -> None:
        if self.enabled:
            import torch.distributed as dist

            dist.destroy_process_group()


def init_from_env(backend: str = "nccl") -> DistEnv:
    """Read RANK/WORLD_SIZE/LOCAL_RANK (torchrun); single process if absent."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world <= 1:
        return DistEnv(0, 1, 0, None)
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if backend == "nccl":
        import torch

        torch.cuda.set_device(local)
    dist.init_process_group(backend=backend, rank=rank, world_size=world)
    return DistEnv(rank, world, local, backend)
