"""One launch each of the Euler-Maruyama kernel and the training-set kernels, for ncu captures:

  ncu --set full -k regex:"em_kernel|em_rows_kernel|row_quantiles" -c 3 python profiles/em_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2302_05170_b200 as sl7  # noqa: E402
from sl7_inputs import OU_THETA, sample_features  # noqa: E402

torch.cuda.set_device(0)
ctx = sl7.Context(7, device=0)
st = torch.zeros(sl7.stats_elems(4096), dtype=torch.float64, device="cuda")
opts = sl7.make_opts(n_bins=4096, hist_lo=-3, hist_hi=3, shift=1.0, ref=sl7.REF_OU, ref_theta=OU_THETA,
                     flags=sl7.FLAG_FAST_NORMALS)
ctx.simulate_em(sl7.MODEL_OU, 1.0, 0.125, 16, 8, OU_THETA, 25_000_000, 1, sl7.OUT_STATS, opts, stats=st)
F = sample_features("ou", 512, seed=3)
ctx.training_set(sl7.MODEL_OU, F, 100_000, 1e-3, 5, sl7.make_opts(flags=sl7.FLAG_FAST_NORMALS))
torch.cuda.synchronize()
print("ok")
