"""One launch of the exact-collocation CIR kernel (cfg2 CIR, 1e5 paths x 16 steps) for ncu:

  ncu --set full -k regex:exact_cir_kernel -c 1 python profiles/cir_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2302_05170_b200 as sl7  # noqa: E402
from sl7_inputs import CIR_THETA  # noqa: E402

torch.cuda.set_device(0)
ctx = sl7.Context(7, device=0)
st = torch.zeros(sl7.stats_elems(4096), dtype=torch.float64, device="cuda")
opts = sl7.make_opts(colloc=sl7.COLLOC_EXACT_CIR, n_bins=4096, hist_lo=0.0, hist_hi=0.6, shift=0.1)
ctx.simulate(0.1, 0.125, 16, CIR_THETA, 100_000, 1, sl7.OUT_STATS, opts, stats=st)
torch.cuda.synchronize()
print("ok")
