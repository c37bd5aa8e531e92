"""One process per GPU: sharding of the batched workload and the result
exchange.

The batched configuration is a set of independent images, so ranks share no
data on the hot path.  Each rank owns a fixed block of images (weak scaling:
``images_per_rank`` per GPU); the only collective is one all-reduce (SUM) of
the [world * images_per_rank, 4] fp64 per-image result table, where every rank
contributes its own rows and zeros elsewhere -- after it every rank holds every
image's (rate, sse, mse, cost).
"""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass(frozen=True)
class Rank:
    rank: int
    local_rank: int
    world: int


def rank_from_env() -> Rank:
    return Rank(int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
                int(os.environ.get("WORLD_SIZE", "1")))


def owned_images(rank: int, images_per_rank: int):
    """Global image indices rank ``rank`` computes (contiguous block)."""
    return list(range(rank * images_per_rank, (rank + 1) * images_per_rank))


def init(backend: str = "nccl"):
    """Initialise torch.distributed from the torchrun environment (no-op at N=1)."""
    import torch
    import torch.distributed as dist
    r = rank_from_env()
    if r.world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(r.local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", r.local_rank))
        else:
            dist.init_process_group(backend)
    elif backend == "nccl" and torch.cuda.is_available():
        torch.cuda.set_device(r.local_rank)
    return r


def scatter_results(local, rank: int, world: int, images_per_rank: int):
    """Place this rank's [images_per_rank, 4] results into a zeroed global
    [world * images_per_rank, 4] table (same device / dtype)."""
    import torch
    table = torch.zeros((world * images_per_rank, local.shape[1]), dtype=local.dtype, device=local.device)
    table[rank * images_per_rank:(rank + 1) * images_per_rank] = local
    return table


def allreduce_results(table):
    """SUM all-reduce of the per-image result table (NCCL on GPU, gloo on CPU)."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(table, op=dist.ReduceOp.SUM)
    return table


def barrier():
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def max_over_ranks(value: float, device=None) -> float:
    """Max of a float over ranks (device timing rule: max over ranks)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
