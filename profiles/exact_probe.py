"""cfg3's exact-collocation FULL run (GBM m=5, 64 steps, step-major [65][N] fp32 to HBM) for timings and ncu:

  python profiles/exact_probe.py [N_PATHS] [REPS] [general]

Default: the fast-normal, closed-form kernel (SL7_FLAG_FAST_NORMALS | SL7_FLAG_SPECIALIZED) on 2e8 paths.
Prints path-steps/s and GB/s from CUDA events (L2 flushed before each timed launch).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2302_05170_b200 as sl7  # noqa: E402
from sl7_inputs import workloads  # noqa: E402

torch.cuda.set_device(0)
w = workloads()["cfg3"]
N = int(sys.argv[1]) if len(sys.argv) > 1 else w.n_paths
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
general = len(sys.argv) > 3 and sys.argv[3] == "general"
n = w.n_steps
out = torch.empty((n + 1) * N, dtype=torch.float32, device="cuda")
flush = torch.empty((512 << 20) // 4, dtype=torch.float32, device="cuda")
ctx = sl7.Context(w.m, device=0)
flags = 0 if general else sl7.FLAG_FAST_NORMALS | sl7.FLAG_SPECIALIZED
opts = sl7.make_opts(prec=sl7.PREC_FP32, colloc=sl7.COLLOC_EXACT_GBM, flags=flags)
stream = torch.cuda.current_stream()
ctx.simulate(w.y0, w.dt, n, w.theta, N, w.seed, sl7.OUT_FULL, opts, out=out)
torch.cuda.synchronize()
ms = []
for _ in range(reps):
    flush.fill_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.simulate(w.y0, w.dt, n, w.theta, N, w.seed, sl7.OUT_FULL, opts, out=out)
    e1.record(stream)
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
best = min(ms)
print(json.dumps({"n_paths": N, "n_steps": n, "ms": ms, "path_steps_per_s": N * n / (best * 1e-3),
                  "GBps": 4 * (n + 1) * N / (best * 1e-3) / 1e9, "checksum": float(out[::1000003].double().sum())}))
