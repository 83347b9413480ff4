"""Multi-GPU plumbing (one process per GPU): rank discovery, row sharding, NCCL bootstrap.

Data-parallel layout of the hot path:
  * rows of X (and y) are split into `world` contiguous blocks (shard_range);
  * C, v, alpha, the CG state and the preconditioner are replicated;
  * every m-vector product is summed over ranks by ONE NCCL allreduce issued by libfalkon
    on its own communicator (the unique id is broadcast here with torch.distributed);
  * lambda * n uses the global n (libfalkon allreduces n_local once per fit).
No arithmetic of the method lives here.
"""
from __future__ import annotations

import os
from typing import Optional, Tuple


def shard_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Rows [start, stop) of `rank`: contiguous blocks, the first n % world ranks one longer."""
    if world < 1 or not (0 <= rank < world) or n < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def env_ranks() -> Tuple[int, int, int]:
    """(world, rank, local_rank) from the torchrun environment (1, 0, 0 if absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def broadcast_bytes(payload: Optional[bytes], src: int = 0) -> bytes:
    """Broadcast a small byte string from `src` over the default torch.distributed group."""
    import torch.distributed as dist
    obj = [payload if dist.get_rank() == src else None]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def make_context(device: int, world: int, rank: int, stream="torch"):
    """libfalkon context for this rank; for world > 1 the NCCL unique id is created on rank 0
    and broadcast through torch.distributed (which must already be initialised)."""
    from . import binding
    if world == 1:
        return binding.Context(device=device, stream=stream)
    uid = broadcast_bytes(binding.get_unique_id() if rank == 0 else None)
    return binding.Context(device=device, rank=rank, world=world, unique_id=uid, stream=stream)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a host scalar over all ranks (timing: the job is as slow as its slowest rank)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
