"""Strong- and weak-scaling emulation of bench.py's configs[4] on ONE B200: each rank's shard of a W-rank run
(`dist.strong_shard` / `weak_shard`, the same path ranges and Philox offsets torchrun would give it) is
launched on its own, one after the other, and timed with CUDA events (L2 flushed before each).  The kernels of
different ranks never wait on one another, so the time a W-GPU run needs is the slowest shard plus the
one stats all-reduce (33 KB; the world-1 NCCL line in profiles/r02_torchrun_world1.json).  Per-shard
statistics are summed on the host (what the all-reduce does) and must equal the one-call run's counts.

  python profiles/shard_emulation.py [W ...]      (default 2 4 8)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2302_05170_b200 as sl7  # noqa: E402
from paper_2302_05170_b200.dist import strong_shard, weak_shard  # noqa: E402
from sl7_inputs import load_golden_blob, workloads  # noqa: E402

torch.cuda.set_device(0)
w = workloads()["cfg4"]
ctx = sl7.Context(w.m, list(w.dims), w.act, device=0)
ctx.load_weights(load_golden_blob(w.blob))
flush = torch.empty((512 << 20) // 4, dtype=torch.float32, device="cuda")
stream = torch.cuda.current_stream()
Ws = [int(a) for a in sys.argv[1:]] or [2, 4, 8]


def shard_ms(offset, n):
    st = torch.zeros(sl7.stats_elems(4096), dtype=torch.float64, device="cuda")
    o = sl7.make_opts(prec=sl7.PREC_BF16, colloc=sl7.COLLOC_ANN, path_offset=offset, n_bins=4096, hist_lo=0.0,
                      hist_hi=0.8, shift=0.1, stream=stream)
    flush.fill_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.simulate(w.y0, w.dt, w.n_steps, w.theta, n, w.seed, sl7.OUT_STATS, o, stats=st)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), st


shard_ms(0, 10_000_000)   # warm-up
ms1, st1 = shard_ms(0, w.n_paths)
print(json.dumps({"scaling": "strong", "W": 1, "paths": w.n_paths, "ms": ms1,
                  "path_steps_per_s": w.n_paths * w.n_steps / (ms1 * 1e-3)}), flush=True)
for W in Ws:
    for mode in ("strong", "weak"):
        times, total = [], None
        for r in range(W):
            off, n = strong_shard(w.n_paths, r, W) if mode == "strong" else weak_shard(500_000_000, r)
            ms, st = shard_ms(off, n)
            times.append(ms)
            total = st if total is None else total + st
        paths = w.n_paths if mode == "strong" else 500_000_000 * W
        t = max(times)
        line = {"scaling": mode, "W": W, "paths": paths, "shard_ms": times, "max_ms": t,
                "emulated_path_steps_per_s": paths * w.n_steps / (t * 1e-3),
                "shard_imbalance": max(times) / min(times) - 1}
        if mode == "strong":
            line["speedup_vs_1"] = ms1 / t
            line["stats_equal_one_call"] = bool(torch.equal(total[0:2], st1[0:2]) and torch.equal(total[8:], st1[8:]))
        print(json.dumps(line), flush=True)
