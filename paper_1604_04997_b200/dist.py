"""Multi-GPU plumbing for the hot path (one process per GPU).

The parameter grid shards by problem size: every rank evaluates a
contiguous block of sizes for all kernel variants, so evaluate / predict /
argmin need no collective. The only exchange is the fit's Gram statistics
(SURVEY.md §8e): G and Xᵀ1 are summed, colmax is max-reduced, then every
rank solves the same small system redundantly (no broadcast needed).
"""
from __future__ import annotations


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [begin, end) block of n items for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return n * rank // world, n * (rank + 1) // world


def allreduce_gram(stats, group=None):
    """Combine per-rank GramStats in place: SUM for G, Xᵀ1, row counts; MAX
    for column max|x|. Works with NCCL (CUDA tensors) and gloo (CPU)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return stats
    F = stats.xt1.numel()
    flat = torch.cat([stats.G.reshape(-1), stats.xt1.reshape(-1),
                      torch.tensor([float(stats.n_rows), float(stats.bad_rows)],
                                   dtype=torch.float64, device=stats.G.device)])
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(stats.colmax, op=dist.ReduceOp.MAX, group=group)
    stats.G.copy_(flat[:F * F].view(F, F))
    stats.xt1.copy_(flat[F * F:F * F + F])
    stats.n_rows = int(flat[F * F + F].item())
    stats.bad_rows = int(flat[F * F + F + 1].item())
    return stats


def gather_shards(local, total: int, dst: int = 0, group=None):
    """Concatenate the per-rank output slices (rank order, shard_bounds
    blocks of a length-`total` result along dim 0) on rank `dst`; other
    ranks get None. Works with NCCL (CUDA tensors) and gloo (CPU)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    width = (total + world - 1) // world  # the largest shard
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, parts, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([parts[r][:shard_bounds(total, r, world)[1] - shard_bounds(total, r, world)[0]]
                      for r in range(world)])
