"""Terminal moments of the CIR configs (cfg2_cir: T=2, 16 steps; cfg4: T=4, 32 steps) against the CIR law,
for 7L in BF16 / FP32 and for 7L-CDC with predicted marginal points (CDC_PRED, reading R-26), 1e8 paths.

  python profiles/cir_fit_check.py [N]

CIR law: E Y_T = Y0 e^{-kT} + Ybar (1 - e^{-kT}),
         Var Y_T = Y0 s^2/k (e^{-kT} - e^{-2kT}) + Ybar s^2/(2k) (1 - e^{-kT})^2.
"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2302_05170_b200 as sl7  # noqa: E402
from sl7_inputs import load_golden_blob, workloads  # noqa: E402

torch.cuda.set_device(0)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
for key in ("cfg2_cir", "cfg4"):
    w = workloads()[key]
    k, yb, s = w.theta
    T = w.dt * w.n_steps
    e = math.exp(-k * T)
    law_mean = w.y0 * e + yb * (1 - e)
    law_var = w.y0 * s * s / k * (e - e * e) + yb * s * s / (2 * k) * (1 - e) ** 2
    ctx = sl7.Context(w.m, list(w.dims), w.act, device=0)
    ctx.load_weights(load_golden_blob(w.blob))
    for name, prec, scheme in (("7l_bf16", sl7.PREC_BF16, sl7.SCHEME_7L), ("7l_fp32", sl7.PREC_FP32, sl7.SCHEME_7L),
                               ("cdc_pred", sl7.PREC_FP32, sl7.SCHEME_CDC_PRED)):
        st = torch.zeros(sl7.stats_elems(4096), dtype=torch.float64, device="cuda")
        opts = sl7.make_opts(prec=prec, colloc=sl7.COLLOC_ANN, scheme=scheme, n_bins=4096, hist_lo=0.0,
                             hist_hi=0.8, shift=0.1)
        ctx.simulate(w.y0, w.dt, w.n_steps, w.theta, N, w.seed, sl7.OUT_STATS, opts, stats=st)
        torch.cuda.synchronize()
        v = st.cpu().numpy()
        sm = sl7.stats_summary(v, opts)
        print(json.dumps({"config": key, "run": name, "n": int(v[0]), "n_nonfinite": int(v[1]),
                          "mean": sm["mean"], "var": sm["var"], "law_mean": law_mean, "law_var": law_var,
                          "mean_rel_err": sm["mean"] / law_mean - 1, "var_rel_err": sm["var"] / law_var - 1}),
              flush=True)
