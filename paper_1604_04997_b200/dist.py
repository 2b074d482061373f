"""Multi-GPU plumbing for the hot path (one process per GPU).

The parameter grid shards by problem size: every rank evaluates a
contiguous block of sizes for all kernel variants, so evaluate / predict /
argmin need no collective. The only exchange is the fit's Gram statistics
(SURVEY.md §8e): G and Xᵀ1 are summed, colmax is max-reduced, then every
rank solves the same small system redundantly (no broadcast needed); each
refinement step sums the per-rank gradients Xᵀ(1 - X alpha) the same way.
"""
from __future__ import annotations


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [begin, end) block of n items for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return n * rank // world, n * (rank + 1) // world


def _host_staged(group=None) -> bool:
    """gloo moves CPU tensors: CUDA tensors are staged through the host
    (e.g. several ranks sharing one GPU in a functional dry run)."""
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def _reduce(t, op, group=None):
    import torch.distributed as dist
    if t.is_cuda and _host_staged(group):
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)


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
    _reduce(flat, dist.ReduceOp.SUM, group)
    _reduce(stats.colmax, dist.ReduceOp.MAX, group)
    stats.G.copy_(flat[:F * F].view(F, F))
    stats.xt1.copy_(flat[F * F:F * F + F])
    stats.n_rows = int(flat[F * F + F].item())
    stats.bad_rows = int(flat[F * F + F + 1].item())
    return stats


def allreduce_sum(t, group=None):
    """SUM-reduce a small tensor (e.g. a refinement gradient) in place."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size(group) > 1:
        _reduce(t, dist.ReduceOp.SUM, group)
    return t


def fit_sharded(prog, bindings, T, refine: int = 1, group=None, stream=None):
    """Config 5 on every rank: fused Gram of the local rows, all-reduce,
    redundant solve, `refine` refinement steps (local gradient in twice the
    working precision, all-reduced); the objective at the refined weights
    from the last step's all-reduced sums (api.refined_objective), or the
    fused residual pass when refine = 0.
    Returns (alpha over the program's keys, rank, objective, total rows)."""
    import paper_1604_04997_b200 as kc

    st = kc.gram_fused(prog, bindings, T, stream=stream)
    allreduce_gram(st, group)
    alpha, rank = kc.solve_gram(st)
    K = kc.schema_size()

    def full(a):
        out = [0.0] * K
        for j, k in enumerate(prog.props):
            out[k] = a[j]
        return out
    import torch
    if refine == 0:
        obj = torch.tensor([kc.residual_fused(prog, bindings, T, full(alpha), stream=stream)],
                           dtype=torch.float64, device=T.device)
        allreduce_sum(obj, group)
        return alpha, rank, float(obj.item()), st.n_rows
    for step in range(refine):
        last = step == refine - 1
        r2 = torch.zeros(1, dtype=torch.float64, device=T.device) if last else None
        g = allreduce_sum(kc.residual_grad_fused(prog, bindings, T, full(alpha), stream=stream, r2=r2), group)
        new = kc.refine_gram(st, alpha, g)
        if last:  # objective at the refined weights from this pass's all-reduced sums (no residual pass)
            obj = kc.refined_objective(st, alpha, new, g, allreduce_sum(r2, group))
        alpha = new
    return alpha, rank, obj, st.n_rows


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
    dev = "cpu" if _host_staged(group) else local.device
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=dev)
    pad[:local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, parts, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([parts[r][:shard_bounds(total, r, world)[1] - shard_bounds(total, r, world)[0]]
                      for r in range(world)])
