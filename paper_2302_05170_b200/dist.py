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


# ------------------------------------------------------------------------------------------------
# Sharded 7L-CDC.  Unlike Algorithm I, the CDC step couples the paths: its m
# marginal collocation points are quantiles of ALL paths.  A rank holding a shard contributes its local
# radix-select digit histograms; the SUM over ranks (four small all-reduces per large step, 64 KB each)
# lets every rank fix the same digits, so each rank's paths evolve exactly as in a single-device run over
# the union of the shards.  The statistics vector is reduced once at the end (allreduce_stats).
# ------------------------------------------------------------------------------------------------

class CdcShard:
    """One device-resident shard of a CDC run, driven through the library's sl7_cdc_* calls."""

    def __init__(self, ctx, y0, dt, n_steps, theta, n_paths, seed, opts, stats=None):
        import torch
        import paper_2302_05170_b200 as sl7
        dev = torch.device("cuda", ctx.device)
        self.ctx = ctx
        self.state = torch.empty(int(n_paths), dtype=torch.float32, device=dev)
        self.hist = torch.empty(sl7.cdc_hist_elems(), dtype=torch.int64, device=dev)   # u64 counts
        self.stats = stats
        ctx.cdc_init(y0, dt, n_steps, theta, n_paths, seed, opts, self.state)

    def local_hist(self, pass_):
        self.ctx.cdc_hist(self.state, pass_, self.hist)
        return self.hist

    def select(self, pass_, hist):
        self.ctx.cdc_select(pass_, hist)

    def step(self, i, last):
        self.ctx.cdc_step(i, self.state, self.state, self.stats if last else None)


def cdc_run(shards, n_steps: int, allreduce=None):
    """Drive the sharded CDC loop over this process's shards (usually one per rank).  `allreduce(t)`
    sums a histogram tensor over the ranks in place (e.g. ``lambda t: dist.all_reduce(t)``); None for a
    single process.  Shards of one process are summed locally first."""
    for i in range(n_steps):
        for p in range(4):
            hs = [s.local_hist(p) for s in shards]
            h = hs[0] if len(hs) == 1 else sum(hs[1:], hs[0].clone())
            if allreduce is not None:
                allreduce(h)
            for s in shards:
                s.select(p, h)
        for s in shards:
            s.step(i, i == n_steps - 1)
    return shards
