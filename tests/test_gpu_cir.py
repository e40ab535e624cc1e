"""GPU parity of the exact-collocation CIR mode (SL7_COLLOC_EXACT_CIR) against the
float64 oracle (scipy's noncentral chi-square quantile, itself pinned to the Poisson-mixture definition
at 30 digits in test_oracle_pins.py).

Tolerance T-2: teacher-forced one step, |Y_dev - Y_or| <= 1e-5 * kappa, kappa = sum_j |l_j(X)| |y_j|: the
device computes the quantiles in float64 (to ~1e-14), rounds y_j to fp32 and evaluates g_m in fp32.
"""
import math

import numpy as np
import pytest

from oracle import sl7_oracle as O

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


@pytest.mark.parametrize("m,theta,y0s", [
    (7, (1.0, 0.1, 0.3), (0.1, 0.0, 0.003, 0.6)),        # cfg2 / cfg4 CIR (Feller: d = 4.44)
    (5, (0.5, 0.04, 0.4), (0.04, 0.5)),                   # Feller violated: d = 0.5 < 2
])
def test_exact_cir_teacher_forced(gpu_lib, m, theta, y0s):
    sl7 = gpu_lib
    torch = _torch()
    ctx = sl7.Context(m)
    n, P, dt, seed = 6, 700, 0.125, 31
    # the device's own fp32 normals (checked against the oracle's in test_gpu_parity): near the lowest
    # nodes g_m is steep while kappa is tiny (y_0 ~ 1e-13 when d < 2), so the last-bit difference of X
    # between fp32 and float64 Box-Muller would otherwise dominate the comparison
    z = torch.empty(n * P, dtype=torch.float32, device="cuda")
    sl7.normals(seed, 0, P, n, z)
    torch.cuda.synchronize()
    Z = z.double().cpu().numpy().reshape(n, P)
    spec = O.Spec(m, "cir", theta, 0.1, dt, n)
    for y0 in y0s:
        out, _ = ctx.simulate(y0, dt, n, theta, P, seed, sl7.OUT_FULL, sl7.make_opts(colloc=sl7.COLLOC_EXACT_CIR))
        torch.cuda.synchronize()
        Yd = out.double().cpu().numpy().reshape(n + 1, P)
        assert np.all(np.isfinite(Yd))
        for i in range(n):
            ref = O.step(spec, Yd[i], Z[i])
            kap = O.step_error_scale(spec, Yd[i], Z[i])
            r = np.abs(Yd[i + 1] - ref) / kap
            assert r.max() <= 1e-5, (y0, i, r.max(), int(np.argmax(r)))


def test_exact_cir_moments(gpu_lib):
    """Sanity (not parity): the terminal law after 8 large steps has the CIR closed-form mean/variance
    within Monte-Carlo error plus the Gauss-Hermite collocation error."""
    sl7 = gpu_lib
    torch = _torch()
    k, ybar, s, y0, T, n, P = 1.0, 0.1, 0.3, 0.3, 1.0, 8, 200_000
    ctx = sl7.Context(7)
    st = torch.zeros(sl7.stats_elems(0), dtype=torch.float64, device="cuda")
    opts = sl7.make_opts(colloc=sl7.COLLOC_EXACT_CIR, shift=0.1)
    ctx.simulate(y0, T / n, n, (k, ybar, s), P, 3, sl7.OUT_STATS, opts, stats=st)
    torch.cuda.synchronize()
    md = O.moments_from_stats(st.cpu().numpy(), 0.1)
    y0f = float(np.float32(y0))
    e = math.exp(-k * T)
    mean = ybar + (y0f - ybar) * e
    var = y0f * s * s / k * (e - e * e) + ybar * s * s / (2 * k) * (1 - e) ** 2
    assert abs(md["mean"] - mean) < 4 * math.sqrt(var / P) + 1e-4 * mean
    assert abs(md["var"] - var) < 0.02 * var


def test_exact_cir_validation(gpu_lib):
    sl7 = gpu_lib
    ctx = sl7.Context(5)
    for theta, flags, scheme, msg in [((1.0, 0.1), 0, 0, "EXACT_CIR"), ((0.0, 0.1, 0.3), 0, 0, "kappa"),
                                      ((1.0, 0.1, 0.3), sl7.FLAG_SPECIALIZED, 0, "SPECIALIZED"),
                                      ((1.0, 0.1, 0.3), 0, sl7.SCHEME_CDC, "CDC")]:
        with pytest.raises(sl7.Sl7Error, match=msg):
            ctx.simulate(0.1, 0.5, 2, theta, 10, 1, sl7.OUT_TERMINAL,
                         sl7.make_opts(colloc=sl7.COLLOC_EXACT_CIR, flags=flags, scheme=scheme))
