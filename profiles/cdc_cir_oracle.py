"""The float64 oracle's 7L-CDC on cfg2's CIR network (2e5 paths): per step the mean, min, max of the
states, the count of negative states and of |Y| > 1.  Shows that the divergence of the device's cfg2_cir
CDC moments (r01_bench_configs_cfg2.jsonl) is the scheme's under reading R-18, not the kernel's
(R-25).  Run: PYTHONPATH=. python profiles/cdc_cir_oracle.py"""
import numpy as np

from oracle import sl7_oracle as O
from sl7_inputs import load_golden_blob, workloads

w = workloads()["cfg2_cir"]
blob = load_golden_blob(w.blob)
spec = O.Spec(w.m, "ann", tuple(w.theta), w.y0, w.dt, w.n_steps, net=O.parse_blob(blob))
with np.errstate(all="ignore"):
    Y, Z = O.simulate_cdc(spec, w.seed, np.arange(200_000, dtype=np.uint64))
    print("step mean min max n_negative n_abs_gt_1  marginal z_0 z_6")
    for i in range(w.n_steps + 1):
        y = Y[i]
        z = O.quantiles(y, O.normal_cdf(spec.x)) if i > 0 else np.full(w.m, w.y0)
        print(i, "%.4g %.4g %.4g" % (y.mean(), y.min(), y.max()), int(np.sum(y < 0)), int(np.sum(np.abs(y) > 1)),
              "%.4g %.4g" % (z[0], z[-1]))
