"""T-4 (BASELINE north_star): free-running terminal mean and variance over the IDENTICAL
path set within 1e-4 relative of the oracle -- the plain float64 oracle O3 for the fp32-class modes
(SL7_PREC_FP32 on the CUDA cores, SL7_PREC_SPLIT on tcgen05) and the quantisation-aware oracle O6 for the
tensor-core modes (bf16 RNE / tf32 RNA operand rounding, reading R-15).  When |mean| < 1e-3 sd the mean is
compared as |dmean| <= 1e-4 sd.  Both sides start every path at Y0 and run all steps on their own
(nothing is restarted from device states); the normals are the same Philox stream (the BF16 / TF32
kernels draw them with the fast Box-Muller, within 2e-6 (1 + |X|) of the oracle's).

The reference values rest on Eq. 6.6 (the exact OU recursion the exact-collocation mode
reproduces) and on the paper's claim that the scheme's error does not grow on the GPU.

Workloads: cfg0 (GBM m=5, 2 steps), cfg1 at its n = 64 sweep point (GBM m=7, dt = 1/64 --
the bench's longest launch), cfg2 OU and CIR (m=7, 4x50 softplus, 16 steps), and cfg4's shape (CIR,
T = 4, 32 steps), each at 20,000 paths.
"""
import functools

import numpy as np
import pytest

from oracle import sl7_oracle as O
from sl7_inputs import load_golden_blob, workloads

pytestmark = pytest.mark.gpu

N_PATHS = 20_000
WORKLOADS = ["cfg0", "cfg1", "cfg2_ou", "cfg2_cir", "cfg4"]
PRECS = ["fp32", "split", "bf16", "tf32"]
ORACLE_QUANT = {"fp32": None, "split": None, "bf16": "bf16", "tf32": "tf32"}


def _case(name):
    w = workloads()[name]
    theta = tuple(w.theta) if w.process != "gbm" else ()
    return w, load_golden_blob(w.blob), theta


@functools.lru_cache(maxsize=None)
def _oracle_terminal(name, quant):
    w, blob, theta = _case(name)
    spec = O.Spec(w.m, "ann", theta, w.y0, w.T / w.n_steps, w.n_steps, net=O.parse_blob(blob), quant=quant)
    with np.errstate(all="ignore"):
        Y, _ = O.simulate(spec, w.seed, np.arange(N_PATHS, dtype=np.uint64))
    return Y[-1].copy()


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("name", WORKLOADS)
def test_terminal_moments_identical_paths(gpu_lib, name, prec):
    import torch
    sl7 = gpu_lib
    w, blob, theta = _case(name)
    ctx = sl7.Context(w.m, list(w.dims), w.act)
    ctx.load_weights(blob)
    P = {"fp32": sl7.PREC_FP32, "split": sl7.PREC_SPLIT, "bf16": sl7.PREC_BF16, "tf32": sl7.PREC_TF32}[prec]
    opts = sl7.make_opts(prec=P, colloc=sl7.COLLOC_ANN)
    out, _ = ctx.simulate(w.y0, w.T / w.n_steps, w.n_steps, theta, N_PATHS, w.seed, sl7.OUT_TERMINAL, opts)
    torch.cuda.synchronize()
    YT = out.double().cpu().numpy()
    Yo = _oracle_terminal(name, ORACLE_QUANT[prec])
    assert np.all(np.isfinite(YT)) and np.all(np.isfinite(Yo))
    mo, md, vo, vd = Yo.mean(), YT.mean(), Yo.var(), YT.var()
    sd = np.sqrt(vo)
    scale = sd if abs(mo) < 1e-3 * sd else abs(mo)
    rel = np.abs(YT - Yo) / np.maximum(np.abs(Yo), sd)
    print("%s %s: dmean/scale %.2g dvar/var %.2g; per-value median %.2g p99 %.2g max %.2g" % (
        name, prec, abs(md - mo) / scale, abs(vd - vo) / vo, np.median(rel), np.quantile(rel, 0.99), rel.max()))
    assert abs(md - mo) <= 1e-4 * scale
    assert abs(vd - vo) <= 1e-4 * vo
