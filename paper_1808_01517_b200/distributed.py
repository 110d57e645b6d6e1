"""Subject/voxel sharding across ranks and the one real exchange: the LSC gradient all-reduce.

The path is a per-voxel map (no spatial coupling, fitting.py:223, lsc.py:194) and
subjects are independent (pkg/tests/test_lsc.py:212-224), so the forward needs no
communication.  Training sums the LSC parameter gradients over all ranks' voxels:
every rank packs its gradients into ONE flat bucket and issues a single
all_reduce(SUM) (NCCL over NVLink on B200; gloo on CPU for tests).
"""

from __future__ import annotations

from typing import Iterable

import torch
import torch.distributed as dist


def shard_range(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) share of n_items for `rank` (first n % world ranks get one more)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, extra = divmod(int(n_items), world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def slab_range(x: torch.Tensor, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of the first spatial axis (X) that `rank` owns when one 5-D volume is split into X-slabs."""
    if x.dim() != 5:
        raise ValueError(f"expected a 5-D (subjects, channels, X, Y, Z) volume, got {tuple(x.shape)}")
    return shard_range(int(x.shape[2]), rank, world)


def voxel_slab(x: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """This rank's contiguous X-slab of a 5-D volume (single-volume sharding).

    The layers are per-voxel maps with no spatial coupling (fitting.py:223, lsc.py:194), so a slab is a
    complete, independent input: its outputs are the volume's outputs on those voxels, and the LSC
    parameter gradient of the volume is the sum of the slabs' gradients (allreduce_gradients).  This
    replaces the reference's in-process voxel spans (lsc.py:202-220, fitting.py:169-187) with ranks.
    """
    lo, hi = slab_range(x, rank, world)
    return x[:, :, lo:hi].contiguous()


def grads_of(params: Iterable[torch.nn.Parameter]) -> list[torch.Tensor]:
    out = []
    for p in params:
        if p.grad is None:
            p.grad = torch.zeros_like(p)
        out.append(p.grad)
    return out


def allreduce_gradients(params: Iterable[torch.nn.Parameter], group=None, scale: float | None = None) -> int:
    """Sum every parameter's .grad over the group with one bucketed all_reduce.

    Returns the bucket size in bytes.  `scale` multiplies the summed gradient
    (e.g. 1/global_voxels when the per-rank loss was an unnormalised sum).
    """
    grads = grads_of(params)
    if not grads:
        return 0
    bucket = torch.cat([g.reshape(-1) for g in grads])
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(bucket, op=dist.ReduceOp.SUM, group=group)
    if scale is not None:
        bucket.mul_(scale)
    off = 0
    for g in grads:
        n = g.numel()
        g.copy_(bucket[off:off + n].view_as(g))
        off += n
    return bucket.numel() * bucket.element_size()


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a host scalar across ranks (timing is reported as the slowest rank)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
