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


# ------------------------------------------------------------------------------------------------
# Sharded 7L-CDC driver (paper_2302_05170_b200.dist.cdc_run) with a world-size-2 gloo group.  The shards
# here implement the library's histogram / select / step protocol in NumPy on fp32 states (keys, digit
# histograms, digit descent, as include/sl7.h describes it) with the oracle's CDC step; the test checks
# the host-side composition: the all-reduced selection yields the exact plotting-position quantiles of
# the UNION of the shards every step, and each rank's paths equal the single-process run's.
# ------------------------------------------------------------------------------------------------

CDC_N, CDC_STEPS, CDC_SEED = 3001, 3, 77


class _RefCdcShard:
    def __init__(self, spec, offset, n, seed):
        import torch as _t
        self.spec = spec
        self.paths = np.arange(offset, offset + n, dtype=np.uint64)
        self.Z = O.normals(seed, self.paths, spec.n_steps)
        self.y = np.full(n, np.float32(spec.y0), dtype=np.float32)
        self.levels = O.normal_cdf(spec.x)
        self.T = 2 * spec.m
        self.hist = _t.zeros(32 * 256, dtype=_t.int64)
        self.z_log = []

    def _keys(self):
        b = self.y.view(np.uint32)
        return np.where(b & 0x80000000, ~b, b | 0x80000000).astype(np.uint32)

    def local_hist(self, p):
        import torch as _t
        k = self._keys()
        shift = 24 - 8 * p
        h = np.zeros((32, 256), dtype=np.int64)
        if p == 0:
            h[0] = np.bincount((k >> shift) & 255, minlength=256)
        else:
            pre = k >> (shift + 8)
            for s, sp in enumerate(self.slots):
                h[s] = np.bincount((k[pre == sp] >> shift) & 255, minlength=256)
        self.hist = _t.from_numpy(h.reshape(-1).copy())
        return self.hist

    def select(self, p, hist):
        h = hist.numpy().reshape(32, 256)
        if p == 0:
            M = int(h[0].sum())
            pos = np.clip(self.levels * M + 0.5, 1.0, M)
            kk = np.floor(pos)
            self.frac = pos - kk
            r0, r1 = kk.astype(np.int64) - 1, np.minimum(kk.astype(np.int64), M - 1)
            self.rank = np.stack([r0, r1], axis=1).reshape(-1)
            self.prefix = np.zeros(self.T, dtype=np.int64)
            slot_of = np.zeros(self.T, dtype=np.int64)
        else:
            slot_of = self.slot_of
        for t in range(self.T):
            c = np.cumsum(h[slot_of[t]])
            b = int(np.searchsorted(c, self.rank[t], side="right"))
            self.rank[t] -= (c[b - 1] if b > 0 else 0)
            self.prefix[t] = (self.prefix[t] << 8) | b
        if p < 3:
            self.slots = sorted(set(int(v) for v in self.prefix))
            self.slot_of = np.array([self.slots.index(int(v)) for v in self.prefix])
        else:
            keys = self.prefix.astype(np.uint32)
            vals = np.where(keys & 0x80000000, keys & 0x7FFFFFFF, ~keys).astype(np.uint32).view(np.float32)
            v = vals.astype(np.float64).reshape(-1, 2)
            self.z = v[:, 0] * (1 - self.frac) + v[:, 1] * self.frac
            self.z_log.append(self.z.copy())

    def step(self, i, last):
        C = self.spec.points(self.z)
        Yn = O.lagrange_eval(self.Z[i], self.spec.x, O.cdc_points(self.z, C, self.y.astype(np.float64)))
        self.y = Yn.astype(np.float32)


def _cdc_spec():
    return O.Spec(5, "ou", (0.0, 1.0, 0.5), 1.0, 0.25, CDC_STEPS)


def _cdc_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2302_05170_b200.dist import cdc_run
    off, n = strong_shard(CDC_N, rank, world)
    sh = _RefCdcShard(_cdc_spec(), off, n, CDC_SEED)
    cdc_run([sh], CDC_STEPS, allreduce=lambda t: dist.all_reduce(t, op=dist.ReduceOp.SUM))
    ys = [None] * world
    dist.all_gather_object(ys, sh.y)
    if rank == 0:
        q.put((np.concatenate(ys), sh.z_log))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sharded_cdc_equals_single_process():
    from paper_2302_05170_b200.dist import cdc_run
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cdc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    y2, z2 = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    one = _RefCdcShard(_cdc_spec(), 0, CDC_N, CDC_SEED)
    ys = [one.y.copy()]
    orig_step = one.step

    def step_and_log(i, last):
        orig_step(i, last)
        ys.append(one.y.copy())
    one.step = step_and_log
    cdc_run([one], CDC_STEPS)
    np.testing.assert_array_equal(y2, one.y)                               # per path, bit for bit
    for i in range(CDC_STEPS):
        np.testing.assert_array_equal(z2[i], one.z_log[i])
        # the exchanged selection gives the exact plotting-position quantiles of the union (R-18)
        np.testing.assert_allclose(z2[i], np.quantile(ys[i].astype(np.float64), one.levels, method="hazen"),
                                   rtol=1e-15, atol=1e-15)
