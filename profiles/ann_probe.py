"""One 7L ANN run of a BASELINE workload in a chosen precision, for ncu captures and quick timings:

  python profiles/ann_probe.py WORKLOAD PREC [N_PATHS] [REPS]

WORKLOAD: cfg1 (n = 64 step of the sweep) | cfg2_ou | cfg2_cir | cfg4; PREC: bf16 | tf32 | split | fp32.
Runs REPS (default 1) STATS launches after one warm-up launch and prints path-steps/s from CUDA events
(the first launch is the warm-up; under ncu, `-s 1 -c 1` captures the first timed one).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2302_05170_b200 as sl7  # noqa: E402
from sl7_inputs import load_golden_blob, workloads  # noqa: E402

torch.cuda.set_device(0)
name, prec = sys.argv[1], sys.argv[2]
w = workloads()[name]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 20_000_000
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
n_steps = w.n_steps
dt = w.T / n_steps
th = tuple(w.theta) if w.process != "gbm" else ()
ctx = sl7.Context(w.m, list(w.dims), w.act, device=0)
ctx.load_weights(load_golden_blob(w.blob))
P = {"bf16": sl7.PREC_BF16, "tf32": sl7.PREC_TF32, "split": sl7.PREC_SPLIT, "fp32": sl7.PREC_FP32}[prec]
st = torch.zeros(sl7.stats_elems(4096), dtype=torch.float64, device="cuda")
lo, hi = {"gbm": (0.0, 4.0), "ou": (-3.0, 3.0), "cir": (0.0, 0.6)}[w.process]
opts = sl7.make_opts(prec=P, colloc=sl7.COLLOC_ANN, n_bins=4096, hist_lo=lo, hist_hi=hi, shift=w.y0)
stream = torch.cuda.current_stream()
ctx.simulate(w.y0, dt, n_steps, th, N, w.seed, sl7.OUT_STATS, opts, stats=st)
torch.cuda.synchronize()
ms = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.simulate(w.y0, dt, n_steps, th, N, w.seed, sl7.OUT_STATS, opts, stats=st)
    e1.record(stream)
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
s = sl7.stats_summary(st.cpu().numpy(), opts)
best = min(ms)
print(json.dumps({"workload": name, "prec": prec, "n_paths": N, "n_steps": n_steps, "ms": ms,
                  "path_steps_per_s": N * n_steps / (best * 1e-3), "mean": s["mean"], "var": s["var"]}))
