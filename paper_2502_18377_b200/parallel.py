"""Batch sharding and the one collective of the multi-GPU step.

Independent PDEs shard over ranks with no data-path exchange; after the backward pass
each rank sums its grad_c over its local batch on the GPU (mpde_batch_sum) and the ranks
all-reduce that sum -- the shared-coefficient gradient -- over NCCL (north_star: "NCCL
over NVLink used only to all-reduce coefficient gradients").  torch.distributed is
plumbing here; the gloo backend runs the same code on CPU for tests.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(total: int, rank: int, world: int):
    """Contiguous [start, start+count) of `total` PDEs owned by `rank` (balanced)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def allreduce_coeff_grad(gsum_local: torch.Tensor, group=None) -> torch.Tensor:
    """In-place SUM all-reduce of the batch-summed coefficient gradient [|M|][P]."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(gsum_local, op=dist.ReduceOp.SUM, group=group)
    return gsum_local


def allreduce_theta_grad(grad_theta: torch.Tensor, group=None) -> torch.Tensor:
    """In-place SUM all-reduce of the template-parameter gradient [|M|+1][K] (a few hundred
    bytes): the collective of the paper's data-parallel discovery step, where theta is
    shared by every PDE of the global batch."""
    return allreduce_coeff_grad(grad_theta, group)


def max_over_ranks(x: float, device=None, group=None) -> float:
    """Max of a host scalar over ranks (device time of the slowest rank)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
