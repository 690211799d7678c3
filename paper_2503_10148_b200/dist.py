"""View-parallel data parallelism.

One process per GPU (torchrun); rank r renders views {v : v mod R = r}, all
ranks hold a full parameter replica, the flat fp32 gradient buffer is summed
with one NCCL all-reduce over NVLink/NVSwitch, and every rank then applies
the identical SGHMC/Adam step (same Philox counters), so replicas stay
bit-identical without a parameter broadcast.  torch.distributed is plumbing
only (process group + NCCL); nothing here computes the method.
"""
from __future__ import annotations

import os
from typing import List, Optional

import torch
import torch.distributed as dist


def env_rank_world():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def init(backend: Optional[str] = None):
    """Initialise the default process group from torchrun's environment."""
    rank, world, local = env_rank_world()
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        kw = {}
        if backend == "nccl":
            torch.cuda.set_device(local)
            kw["device_id"] = torch.device("cuda", local)
        dist.init_process_group(backend=backend, rank=rank, world_size=world, **kw)
    return rank, world, local


def shard_views(n_views: int, rank: int, world: int) -> List[int]:
    """Views rendered by `rank` (round robin; 64 and 8 views divide by 1/2/4/8)."""
    return [v for v in range(n_views) if v % world == rank]


def allreduce_sum_(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place sum over ranks (NCCL ring/NVLS on GPUs, gloo on CPU)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def allreduce_max(x: float, device=None) -> float:
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_checksum(t: torch.Tensor) -> torch.Tensor:
    """Bitwise checksum of a float tensor (int64 sum of its 32-bit words)."""
    return t.contiguous().view(torch.int32).to(torch.int64).sum()


def replicas_identical(t: torch.Tensor) -> bool:
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return True
    c = replica_checksum(t).reshape(1)
    lo, hi = c.clone(), c.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX)
    return bool((lo == hi).item())


def barrier():
    if dist.is_initialized():
        dist.barrier()
