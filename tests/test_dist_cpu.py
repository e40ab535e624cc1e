"""The N>1 host path on CPU: world-size-2 gloo group, path partition + SUM all-reduce of the fp64
statistics vector + sl7_stats summary.  The per-rank statistics vectors here come from the oracle
(no GPU on this box); on a GPU box the same helpers reduce the kernels' vectors over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sl7_oracle as O
from paper_2302_05170_b200.dist import allreduce_stats, max_over_ranks, strong_shard, weak_shard

N, SEED, NB, LO, HI = 6001, 424, 64, 0.0, 3.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_stats(rank, world):
    off, n = strong_shard(N, rank, world)
    spec = O.Spec(5, "gbm", (0.05, 0.2), 1.0, 0.25, 4)
    paths = np.arange(off, off + n, dtype=np.uint64)
    Y, Z = O.simulate(spec, SEED, paths)
    R = O.exact_reference("gbm", (0.05, 0.2), 1.0, 0.25, Z)
    return O.stats_vector(Y[-1], 1.0, LO, HI, NB, R)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    v = torch.tensor(_shard_stats(rank, world), dtype=torch.float64)
    allreduce_stats(v)
    t = max_over_ranks(1.0 + rank)
    if rank == 0:
        q.put((v.numpy().copy(), t))
    dist.barrier()
    dist.destroy_process_group()


def test_partition_covers_paths_exactly():
    for n, w in [(10, 3), (6001, 2), (7, 8), (4_000_000_000, 8)]:
        parts = [strong_shard(n, r, w) for r in range(w)]
        assert sum(c for _, c in parts) == n
        assert parts[0][0] == 0
        for (o1, c1), (o2, _) in zip(parts, parts[1:]):
            assert o1 + c1 == o2 or c1 == 0
    assert weak_shard(500_000_000, 3) == (1_500_000_000, 500_000_000)
    with pytest.raises(ValueError):
        strong_shard(10, 3, 3)


def test_gloo_world2_allreduce_equals_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    v, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = _shard_stats(0, 1)
    assert tmax == 2.0
    assert v[0] == ref[0] and np.array_equal(v[8:], ref[8:])           # counts and histogram exact
    np.testing.assert_allclose(v[2:8], ref[2:8], rtol=1e-12)
    import paper_2302_05170_b200 as sl7
    from paper_2302_05170_b200 import build
    build.build(verbose=False)
    opts = sl7.make_opts(stream=False, n_bins=NB, hist_lo=LO, hist_hi=HI, shift=1.0)
    a = sl7.stats_summary(v, opts, q_levels=[0.5])
    b = sl7.stats_summary(ref, opts, q_levels=[0.5])
    for k in ("mean", "var", "skew", "exkurt", "strong_err"):
        assert abs(a[k] - b[k]) <= 1e-12 * max(1.0, abs(b[k]))
    assert a["quantiles"] == b["quantiles"]
