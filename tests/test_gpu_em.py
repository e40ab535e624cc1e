"""GPU parity of the Euler-Maruyama comparator and the training-set generator
against the float64 oracle (oracle/sl7_em.py), through the C ABI.

Tolerances:
  EM path values: teacher-forced one fine step (K = 1, every fine state recorded),
      |Y_dev - Y_or| <= 1e-5 * kappa, kappa = |Y| + |a(Y) dtau| + |b(Y) sqrt(dtau) Z| (the forward-error
      scale of Eq. 6.2's three-term sum; fp32 rounding is ~2^-23 kappa);
  K > 1: the device's K-sub-step run equals its own K = 1 run at dtau recorded every K-th step, bit for bit;
  labels: the order statistics are integer decisions on the device's fp32 terminal values, so the
      labels lie between the oracle's order statistics OF THOSE VALUES and equal its quantiles up to one
      ulp of the rank position M Phi(x_j) + 1/2 times the gap between them (the levels Phi(x_j) of the
      host erfc and scipy may differ in the last bit);
  terminal values of a row equal sl7_simulate_em of that row (same kernel arithmetic), bit for bit,
      and the oracle's free-running EM within 1e-5 of the accumulated term scale.
"""
import math

import numpy as np
import pytest

from oracle import sl7_em as E
from oracle import sl7_oracle as O
from sl7_inputs import sample_features

pytestmark = pytest.mark.gpu

MODELS = {"gbm": ((0.05, 0.2), 1.0), "ou": ((0.0, 1.0, 0.5), 1.0), "cir": ((1.0, 0.1, 0.3), 0.1)}


def _torch():
    import torch
    return torch


def _model_id(sl7, name):
    return {"gbm": sl7.MODEL_GBM, "ou": sl7.MODEL_OU, "cir": sl7.MODEL_CIR}[name]


def _kappa(model, theta, Y, dtau, Z):
    a, b = E.drift_diffusion(model, theta, Y)
    return np.abs(Y) + np.abs(a * dtau) + np.abs(b * math.sqrt(dtau) * Z) + 1e-30


@pytest.mark.parametrize("fast", [False, True])
@pytest.mark.parametrize("model", ["gbm", "ou", "cir"])
def test_em_teacher_forced(gpu_lib, model, fast):
    sl7 = gpu_lib
    torch = _torch()
    theta, y0 = MODELS[model]
    n, P, dt, seed = 12, 5_003, 0.25, 77
    ctx = sl7.Context(5)
    flags = sl7.FLAG_FAST_NORMALS if fast else 0
    out, _ = ctx.simulate_em(_model_id(sl7, model), y0, dt, n, 1, theta, P, seed, sl7.OUT_FULL,
                             sl7.make_opts(flags=flags))
    if fast:   # the fast Box-Muller is its own (documented) approximation: drive the oracle with its normals
        z = torch.empty(n * P, dtype=torch.float32, device="cuda")
        sl7.normals(seed, 0, P, n, z, flags=sl7.FLAG_FAST_NORMALS)
        Z = z.double().cpu().numpy().reshape(n, P)
    else:
        Z = O.normals(seed, np.arange(P, dtype=np.uint64), n)
    torch.cuda.synchronize()
    Yd = out.double().cpu().numpy().reshape(n + 1, P)
    assert np.all(Yd[0] == np.float32(y0))
    for i in range(n):
        ref = E.euler_step(model, theta, Yd[i], dt, Z[i])
        r = np.abs(Yd[i + 1] - ref) / _kappa(model, theta, Yd[i], dt, Z[i])
        assert r.max() <= 1e-5, (model, i, r.max())


@pytest.mark.parametrize("model", ["gbm", "ou", "cir"])
def test_em_substeps_equal_fine_run(gpu_lib, model):
    sl7 = gpu_lib
    torch = _torch()
    theta, y0 = MODELS[model]
    ctx = sl7.Context(7)
    K, n, P = 5, 6, 1_000
    a, _ = ctx.simulate_em(_model_id(sl7, model), y0, 0.3, n, K, theta, P, 3, sl7.OUT_FULL,
                           sl7.make_opts(path_offset=123))
    b, _ = ctx.simulate_em(_model_id(sl7, model), y0, 0.3 / K, n * K, 1, theta, P, 3, sl7.OUT_FULL,
                           sl7.make_opts(path_offset=123))
    torch.cuda.synchronize()
    A = a.cpu().numpy().reshape(n + 1, P)
    B = b.cpu().numpy().reshape(n * K + 1, P)
    np.testing.assert_array_equal(A, B[::K])


@pytest.mark.parametrize("model", ["gbm", "ou"])
def test_em_stats_and_strong_error(gpu_lib, model):
    """Moments (T-4, 1e-4 relative) and the strong error against the exact solution on the same fine
    normals, free-running on the identical path set."""
    sl7 = gpu_lib
    torch = _torch()
    theta, y0 = MODELS[model]
    n, K, P, seed, dt = 4, 4, 40_000, 5, 0.5
    ref = sl7.REF_GBM if model == "gbm" else sl7.REF_OU
    opts = sl7.make_opts(n_bins=64, hist_lo=-1.0, hist_hi=3.0, shift=y0, ref=ref, ref_theta=theta)
    st = torch.zeros(sl7.stats_elems(64), dtype=torch.float64, device="cuda")
    ctx = sl7.Context(5)
    out, _ = ctx.simulate_em(_model_id(sl7, model), y0, dt, n, K, theta, P, seed, sl7.OUT_TERMINAL, opts, stats=st)
    torch.cuda.synchronize()
    YT = out.double().cpu().numpy()
    v = st.cpu().numpy()
    paths = np.arange(P, dtype=np.uint64)
    Zf = O.normals(seed, paths, n * K)
    Yo = E.simulate_em(model, theta, y0, dt, n, K, seed, paths, Z=Zf)[-1]
    R = O.exact_reference(model, theta, float(np.float32(y0)), dt / K, Zf)
    md = O.moments_from_stats(v, y0)
    assert v[0] == P and v[1] == 0
    assert abs(md["mean"] - Yo.mean()) <= 1e-4 * abs(Yo.mean())
    assert abs(md["var"] - Yo.var()) <= 1e-4 * Yo.var()
    se_or = np.mean(np.abs(Yo - R))
    assert abs(md["strong_err"] - se_or) <= 1e-3 * se_or + 1e-6
    np.testing.assert_allclose(YT, Yo, rtol=2e-5, atol=2e-6)
    ov = O.stats_vector(YT, y0, -1.0, 3.0, 64)          # histogram of the device's own values
    np.testing.assert_array_equal(v[8:], ov[8:])


@pytest.mark.parametrize("fast", [False, True])
@pytest.mark.parametrize("model", ["gbm", "ou", "cir"])
def test_training_set_parity(gpu_lib, model, fast):
    sl7 = gpu_lib
    torch = _torch()
    m, M, dtau, seed, R = 7, 3_001, 0.02, 11, 6
    F = sample_features(model, R, seed=5, dt_range=(0.03, 0.25))
    F[2, 1] = dtau * 3          # exactly K = 3
    ctx = sl7.Context(m)
    flags = sl7.FLAG_FAST_NORMALS if fast else 0
    term = torch.empty((R, M), dtype=torch.float32, device="cuda")
    _, lab = ctx.training_set(_model_id(sl7, model), F, M, dtau, seed, sl7.make_opts(flags=flags, path_offset=17),
                              terminal=term)
    torch.cuda.synchronize()
    T = term.double().cpu().numpy()
    L = lab.cpu().numpy()
    levels = O.normal_cdf(O.gauss_hermite_nodes(m))
    nt = E.N_THETA[model]
    for r in range(R):
        # labels: quantiles of the device's terminal values; the order statistics are exact, the level
        # Phi(x_j) (host erfc vs scipy) may differ in its last bit, so the interpolation weight may too
        Q = O.quantiles(T[r], levels)
        ys = np.sort(T[r])
        k = np.floor(np.clip(levels * M + 0.5, 1, M)).astype(int)
        lo, hi = ys[k - 1], ys[np.minimum(k, M - 1)]
        assert np.all((L[r] >= lo) & (L[r] <= hi))                       # the selected order statistics
        gap_tol = 4 * M * np.finfo(float).eps * (hi - lo)                # one ulp of the rank position
        assert np.all(np.abs(L[r] - Q) <= gap_tol + 1e-15 * np.abs(Q)), (L[r] - Q, gap_tol)
        K = E.em_substeps(F[r, 1], dtau)
        th = tuple(F[r, 2:2 + nt])
        # terminal values: the row is sl7_simulate_em of (y_start, dt/K, K steps) on global ids 17 + r M + q
        y, _ = ctx.simulate_em(_model_id(sl7, model), F[r, 0], F[r, 1] / K, K, 1, th, M, seed, sl7.OUT_TERMINAL,
                               sl7.make_opts(flags=flags, path_offset=17 + r * M))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(T[r], y.double().cpu().numpy())
        if not fast:
            # oracle free-running EM over K sub-steps: error bounded by 1e-5 of the accumulated term scale
            paths = np.uint64(17 + r * M) + np.arange(M, dtype=np.uint64)
            Z = O.normals(seed, paths, K)
            Yo = np.full(M, float(np.float32(F[r, 0])))
            scale = np.zeros(M)
            for k in range(K):
                scale += _kappa(model, th, Yo, F[r, 1] / K, Z[k])
                Yo = E.euler_step(model, th, Yo, F[r, 1] / K, Z[k])
            err = np.abs(T[r] - Yo) / scale
            assert err.max() <= 1e-5, (model, r, K, err.max())


def test_training_set_scratch_and_degenerate_rows(gpu_lib):
    sl7 = gpu_lib
    torch = _torch()
    m, M = 5, 1_000
    F = np.array([[1.5, 0.5, 0.2, 2.0, 0.0],      # sigma = 0: deterministic Euler value
                  [0.3, 0.2, -0.5, 1.0, 0.7],
                  [-1.0, 0.001, 0.0, 1.5, 0.4]])  # dt < dtau: one sub-step
    ctx = sl7.Context(m)
    term = torch.empty((3, M), dtype=torch.float32, device="cuda")
    _, L1 = ctx.training_set(sl7.MODEL_OU, F, M, 0.1, 4, sl7.make_opts(), terminal=term)
    _, L2 = ctx.training_set(sl7.MODEL_OU, F, M, 0.1, 4, sl7.make_opts())          # library scratch
    torch.cuda.synchronize()
    L1, L2 = L1.cpu().numpy(), L2.cpu().numpy()
    np.testing.assert_array_equal(L1, L2)
    det = np.float32(1.5)
    for _ in range(5):
        det = np.float32(np.float32(0.2 * 1.0) * (np.float32(0.2) - det) + det)   # a = lam dtau, fp32 FMA order
    assert np.all(np.abs(L1[0] - float(det)) <= 2e-7 * abs(float(det)))
    assert np.all(L1[0] == L1[0][0])
    assert np.all(np.diff(L1, axis=1) >= 0)


def test_em_and_training_validation(gpu_lib):
    sl7 = gpu_lib
    torch = _torch()
    ctx = sl7.Context(5)
    out = torch.empty(15, dtype=torch.float32, device="cuda")
    for kw, msg in [(dict(model=0), "model"), (dict(model=4), "model"), (dict(theta=(0.1,)), "theta"),
                    (dict(substeps=0), "substeps"), (dict(flags=sl7.FLAG_SPECIALIZED), "flags"),
                    (dict(theta=(0.0, -1.0, 0.5)), "rate"), (dict(dt=-1.0), "dt")]:
        a = dict(model=sl7.MODEL_OU, theta=(0.0, 1.0, 0.5), substeps=1, flags=0, dt=0.5)
        a.update(kw)
        with pytest.raises(sl7.Sl7Error, match=msg):
            ctx.simulate_em(a["model"], 1.0, a["dt"], 2, a["substeps"], a["theta"], 5, 1, sl7.OUT_FULL,
                            sl7.make_opts(flags=a["flags"]), out=out)
    F = np.array([[1.0, 0.5, 0.0, 1.0, 0.5]])
    with pytest.raises(sl7.Sl7Error, match="n_inner"):
        ctx.training_set(sl7.MODEL_OU, F, 4, 0.1, 1, sl7.make_opts())
    with pytest.raises(sl7.Sl7Error, match="dtau"):
        ctx.training_set(sl7.MODEL_OU, F, 100, 0.0, 1, sl7.make_opts())
    bad = F.copy()
    bad[0, 1] = 0.0
    with pytest.raises(sl7.Sl7Error, match=r"features\[0\]"):
        ctx.training_set(sl7.MODEL_OU, bad, 100, 0.1, 1, sl7.make_opts())
    with pytest.raises(sl7.Sl7Error, match="theta"):
        ctx.training_set(sl7.MODEL_GBM, np.array([[1.0, 0.5, 0.1, -0.2]]), 100, 0.1, 1, sl7.make_opts())


def test_training_set_chunked_scratch_equals_caller_buffer(gpu_lib):
    """Without d_terminal the library processes the rows in chunks of its 1 GiB scratch
    (2^28 / M rows): with M = 2^20 that is 256 rows, so 300 rows take two chunks.  The labels must equal
    those of the single-chunk run into a caller buffer, row for row."""
    sl7 = gpu_lib
    torch = _torch()
    M, R = 1 << 20, 300
    F = sample_features("ou", R, seed=12, dt_range=(0.01, 0.02))      # dtau = 0.05 -> K = 1
    ctx = sl7.Context(5)
    term = torch.empty((R, M), dtype=torch.float32, device="cuda")
    _, a = ctx.training_set(sl7.MODEL_OU, F, M, 0.05, 3, sl7.make_opts(flags=sl7.FLAG_FAST_NORMALS), terminal=term)
    _, b = ctx.training_set(sl7.MODEL_OU, F, M, 0.05, 3, sl7.make_opts(flags=sl7.FLAG_FAST_NORMALS))
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    for r in (0, 255, 256, 299):                                          # both sides of the chunk boundary
        T = term[r].double().cpu().numpy()
        lv = O.normal_cdf(O.gauss_hermite_nodes(5))
        Q = O.quantiles(T, lv)
        np.testing.assert_allclose(a[r].cpu().numpy(), Q, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("m,M", [(16, 16), (16, 40), (11, 25), (7, 7)])
def test_training_set_clamped_levels(gpu_lib, m, M):
    """Few inner paths for many levels: several levels clamp to the extreme order statistics, so the
    selection targets repeat rank pairs out of order (0, 1, 0, 1, ...); labels still equal the quantiles of
    the device's terminal values."""
    sl7 = gpu_lib
    torch = _torch()
    F = sample_features("ou", 5, seed=9, dt_range=(0.05, 0.2))
    ctx = sl7.Context(m)
    term = torch.empty((5, M), dtype=torch.float32, device="cuda")
    _, lab = ctx.training_set(sl7.MODEL_OU, F, M, 0.05, 3, sl7.make_opts(), terminal=term)
    torch.cuda.synchronize()
    T, L = term.double().cpu().numpy(), lab.cpu().numpy()
    lv = O.normal_cdf(O.gauss_hermite_nodes(m))
    for r in range(5):
        np.testing.assert_allclose(L[r], O.quantiles(T[r], lv), rtol=1e-12, atol=1e-12)
