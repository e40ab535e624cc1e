"""One 7L-CDC run of cfg2 OU (ANN fp32 table, 1e8 paths x 16 steps, STATS) for ncu launch lists:

  ncu --metrics gpu__time_duration.sum -k regex:cdc_ --csv python profiles/cdc_probe.py [N] [pred]

With a second argument "pred": SL7_SCHEME_CDC_PRED (the fused all-steps kernel).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2302_05170_b200 as sl7  # noqa: E402
from sl7_inputs import load_golden_blob, workloads  # noqa: E402

torch.cuda.set_device(0)
w = workloads()[os.environ.get("CDC_PROBE_WORKLOAD", "cfg2_ou")]
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
ctx = sl7.Context(w.m, list(w.dims), w.act, device=0)
ctx.load_weights(load_golden_blob(w.blob))
st = torch.zeros(sl7.stats_elems(4096), dtype=torch.float64, device="cuda")
scheme = sl7.SCHEME_CDC_PRED if (len(sys.argv) > 2 and sys.argv[2] == "pred") else sl7.SCHEME_CDC
opts = sl7.make_opts(prec=sl7.PREC_FP32, colloc=sl7.COLLOC_ANN, scheme=scheme, n_bins=4096, hist_lo=-3.0,
                     hist_hi=3.0, shift=w.y0)
ctx.simulate(w.y0, w.dt, w.n_steps, w.theta, N, w.seed, sl7.OUT_STATS, opts, stats=st)
torch.cuda.synchronize()
reps = int(sys.argv[3]) if len(sys.argv) > 3 else int(os.environ.get("CDC_PROBE_REPS", "0"))   # > 0: time them
ms = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.simulate(w.y0, w.dt, w.n_steps, w.theta, N, w.seed, sl7.OUT_STATS, opts, stats=st)
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
s = sl7.stats_summary(st.cpu().numpy(), opts)
print("ok", s["mean"], s["var"], s.get("clamped_steps"),
      ("%.4g path-steps/s" % (N * w.n_steps / (min(ms) * 1e-3))) if ms else "")
