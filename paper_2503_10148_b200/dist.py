"""View-parallel data parallelism.

One process per GPU (torchrun); rank r renders views {v : v mod R = r} and
all ranks hold a full parameter replica.  Two exchange schemes for the flat
fp32 [P][n] gradient buffer:
  * replicated: one NCCL all-reduce, then every rank applies the identical
    SGHMC/Adam step (same Philox counters);
  * sharded (ZeRO-1, §8(e) option 2, the default for R > 1): the buffer is
    padded to R * ceil(P / R) planes, reduce-scattered by planes, each rank
    updates only its planes (sss_sghmc_step's plane range; every plane's
    update reads only the replicated pre-update parameters), and the ranks
    all-gather the parameter planes.  Same bytes on the wire as the
    all-reduce; the sampler's HBM work is divided by R.
Either way replicas stay bit-identical.  With the overlapped variant the
gradient is component-blocked (api.BlockedParams): the projection backward
runs block by block and each block's reduce-scatter is issued on a
communication stream as soon as its components are done, so the exchange
overlaps the remaining blocks' computation; the all-gather of the updated
parameter planes follows the sampler step.  torch.distributed is plumbing
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


def allreduce_max_(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place max over ranks (device tensor; no host sync)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t


def plane_shard(P: int, rank: int, world: int):
    """(planes per rank Pr, [begin, end) owned by `rank`) of a [R * Pr][n]
    padded plane buffer."""
    pr = -(-P // world)
    return pr, (min(rank * pr, P), min((rank + 1) * pr, P))


def _nccl(group=None) -> bool:
    return dist.is_initialized() and dist.get_backend(group) == "nccl"


def reduce_scatter_planes_(full: torch.Tensor, scratch: torch.Tensor, group=None) -> torch.Tensor:
    """Sum `full` [R * Pr][n] over ranks into this rank's plane slice (the
    other slices are left stale).  NCCL reduce-scatter; gloo (CPU tests)
    all-reduces, which leaves the same values in the slice."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    pr = full.shape[0] // world
    mine = full[rank * pr:(rank + 1) * pr]
    if _nccl(group):
        dist.reduce_scatter_tensor(scratch, full, op=dist.ReduceOp.SUM, group=group)
        mine.copy_(scratch)
    else:
        dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
    return mine


def reduce_scatter_block_(block: torch.Tensor, group=None) -> torch.Tensor:
    """One block [R * Pr][B] of a component-blocked gradient: the sum over
    ranks of this rank's planes [r Pr, (r + 1) Pr) lands in place (NCCL
    in-place reduce-scatter: output = input + rank * Pr * B); gloo (CPU
    tests) all-reduces the block, which leaves the same values there."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    pr = block.shape[0] // world
    mine = block[rank * pr:(rank + 1) * pr]
    if _nccl(group):
        dist.reduce_scatter_tensor(mine, block, op=dist.ReduceOp.SUM, group=group)
    else:
        dist.all_reduce(block, op=dist.ReduceOp.SUM, group=group)
    return mine


def all_gather_planes_(full: torch.Tensor, scratch: torch.Tensor, group=None) -> torch.Tensor:
    """Every rank's plane slice of `full` [R * Pr][n] to every rank."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    pr = full.shape[0] // world
    scratch.copy_(full[rank * pr:(rank + 1) * pr])
    if _nccl(group):
        dist.all_gather_into_tensor(full, scratch, group=group)
    else:
        dist.all_gather(list(full.view(world, pr, -1).unbind(0)), scratch, group=group)
    return full


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
