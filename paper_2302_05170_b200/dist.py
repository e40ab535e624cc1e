"""Multi-GPU plumbing of the 7L path generator: one process per GPU.

Paths are independent (Algorithm I step 4 partitions them over processing units,
PAPER.md:63), and the Philox counter holds the GLOBAL path index, so a rank simulates its shard by
passing ``path_offset`` -- per-path results are bitwise independent of the partition.  The only
exchange step is one SUM all-reduce of the fp64 statistics vectors (moments, strong error,
histogram counts: counts < 2^53 are exact in fp64) after the kernels.
"""
from __future__ import annotations


def strong_shard(n_paths: int, rank: int, world: int) -> tuple[int, int]:
    """Fixed total work: rank r owns [r*ceil(N/W), min(N, (r+1)*ceil(N/W))) -> (offset, count)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("rank/world")
    per = -(-n_paths // world)
    lo = min(n_paths, rank * per)
    hi = min(n_paths, lo + per)
    return lo, hi - lo


def weak_shard(n_per_rank: int, rank: int) -> tuple[int, int]:
    """Fixed work per GPU: rank r owns [r*N, (r+1)*N)."""
    return rank * n_per_rank, n_per_rank


def allreduce_stats(stats, group=None):
    """Sum the per-rank fp64 stats vectors in place (NCCL on GPU tensors, gloo on CPU tensors)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
