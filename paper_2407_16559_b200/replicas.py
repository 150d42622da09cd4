"""Multi-GPU mode: independent replicas.

The path does not shard (time stepping is sequential and one RHS fits one GPU), so N GPUs run N
independent workloads: one process per GPU, no data-path collective. torch.distributed carries
only the barrier that brackets the timed region and the max-over-ranks of the device times.
Works with "nccl" (GPU box) and "gloo" (CPU tests, world_size 2).
"""
from __future__ import annotations

import os


def setup(backend: str | None = None):
    """Init from torchrun's env (RANK/LOCAL_RANK/WORLD_SIZE/MASTER_*). Returns (world, rank, local)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if not dist.is_initialized():
            if backend is None:
                backend = "nccl" if torch.cuda.is_available() else "gloo"
            kw = {}
            if backend == "nccl":
                torch.cuda.set_device(local)
                kw["device_id"] = torch.device("cuda", local)
            dist.init_process_group(backend, **kw)
    return world, rank, local


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int, local: int = 0) -> float:
    """Max of a per-rank scalar (device seconds) over all ranks."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = f"cuda:{local}" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_rate(units_per_rank: int, max_seconds: float, world: int) -> float:
    """Whole-job throughput of `world` replicas each processing `units_per_rank` units, timed as
    the max over ranks (weak scaling: per-GPU work fixed)."""
    return world * units_per_rank / max_seconds


def teardown(world: int):
    if world > 1:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()
