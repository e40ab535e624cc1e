"""Pins of the Euler-Maruyama / training-set oracle (oracle/sl7_em.py), CPU only.

Each pin ties the oracle to something other than itself: SPEC.md's worked values, closed forms of the
deterministic (sigma = 0) recursion and of the EM moments, first-order strong convergence against the
exact OU transition (Eq. 6.6), the library quantile (numpy "hazen"), and the exact OU collocation
points."""
import math

import numpy as np
import pytest
import scipy.stats

from oracle import sl7_em as E
from oracle import sl7_oracle as O
from sl7_inputs import sample_features


def test_euler_step_spec_examples():
    # SPEC.md:149-152
    assert E.euler_step("ou", (0.0, 1.0, 0.2), 1.0, 0.01, 0.0) == pytest.approx(0.99, abs=1e-15)
    assert E.euler_step("ou", (0.0, 0.0, 1.0), 0.0, 4.0, 0.5) == pytest.approx(1.0, abs=1e-15)
    assert E.euler_step("gbm", (0.0, 0.0), 1.7, 0.3, 2.0) == 1.7              # a = b = 0: unchanged


def test_drift_diffusion_definitions():
    # Eq. 6.1 coefficients, written out independently at one point per model
    a, b = E.drift_diffusion("gbm", (0.05, 0.2), 2.0)
    assert (a, b) == pytest.approx((0.1, 0.4))
    a, b = E.drift_diffusion("ou", (0.5, 2.0, 0.3), 1.0)
    assert (a, b) == pytest.approx((-1.0, 0.3))
    a, b = E.drift_diffusion("cir", (1.0, 0.1, 0.3), 0.04)
    assert (a, b) == pytest.approx((0.06, 0.06))
    a, b = E.drift_diffusion("cir", (1.0, 0.1, 0.3), -0.01)                  # full truncation (R-22)
    assert (a, b) == pytest.approx((0.1, 0.0))


def test_euler_path_deterministic():
    # sigma = 0, lam = 1, Ybar = 0, Y0 = 1, T = 1, n = 2 -> {1, 0.5, 0.25}
    P = E.simulate_em("ou", (0.0, 1.0, 0.0), 1.0, 0.5, 2, 1, 1, np.arange(3, dtype=np.uint64))
    np.testing.assert_array_equal(P[:, 0], [1.0, 0.5, 0.25])
    # sigma = 0, n = 1e4 vs e^{-1}: |diff| < 1e-3 (the O(dt) Euler error is e^{-1}/(2n))
    Z = np.zeros((10_000, 1))
    P = E.simulate_em("ou", (0.0, 1.0, 0.0), 1.0, 1e-4, 10_000, 1, 0, [0], Z=Z)
    assert abs(P[-1, 0] - math.exp(-1.0)) < 1e-3
    assert P[-1, 0] == pytest.approx((1 - 1e-4) ** 10_000, rel=1e-12)
    # GBM sigma = 0: Y0 (1 + mu dtau)^N
    P = E.simulate_em("gbm", (0.05, 0.0), 1.0, 0.25, 4, 3, 9, np.arange(5, dtype=np.uint64))
    np.testing.assert_allclose(P[:, 2], (1 + 0.05 / 12) ** (3 * np.arange(5)), rtol=1e-14)


def test_substep_identity_and_rng_layout():
    """K sub-steps of dt/K per large step == plain EM at dt/K recorded every K-th step; fine step k of
    path p uses normal Z_{p,k} of the path generator (O2)."""
    paths = np.arange(100, 164, dtype=np.uint64)
    A = E.simulate_em("cir", (1.0, 0.1, 0.3), 0.1, 0.5, 3, 4, 7, paths)
    B = E.simulate_em("cir", (1.0, 0.1, 0.3), 0.1, 0.125, 12, 1, 7, paths)
    np.testing.assert_array_equal(A, B[::4])
    Z = O.normals(7, paths, 12)
    y = np.full(len(paths), float(np.float32(0.1)))           # Y0 is rounded to fp32 (sl7.h)
    for k in range(12):
        y = y + 1.0 * (0.1 - np.maximum(y, 0)) * 0.125 + 0.3 * np.sqrt(np.maximum(y, 0)) * math.sqrt(0.125) * Z[k]
    np.testing.assert_allclose(B[-1], y, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("model,theta,y0", [("gbm", (0.05, 0.2), 1.0), ("ou", (0.3, 1.0, 0.5), 1.0)])
def test_em_moments_closed_form(model, theta, y0):
    """The EM recursion's own first two moments are closed forms (linear models): the sample moments of
    2e5 paths must match within 5 standard errors."""
    P = 200_000
    dtau, N = 0.125, 8
    Y = E.simulate_em(model, theta, y0, dtau * 2, N // 2, 2, 11, np.arange(P, dtype=np.uint64))[-1]
    mean, var = E.em_mean_var_closed_form(model, theta, y0, dtau, N)
    se_mean = math.sqrt(var / P)
    assert abs(Y.mean() - mean) < 5 * se_mean
    kurt = scipy.stats.kurtosis(Y, fisher=False)
    se_var = var * math.sqrt((kurt - 1) / P)
    assert abs(Y.var() - var) < 5 * se_var


def test_strong_convergence_first_order():
    """OU (lam = 1, sigma = 0.5) Euler strong error vs the exact transition (Eq. 6.6) on
    the same normals: the error ratio from dt = 1 to dt = 0.125 is >= 4 (first order: ~8)."""
    theta, P, T = (0.0, 1.0, 0.5), 20_000, 2.0
    paths = np.arange(P, dtype=np.uint64)
    err = {}
    for n in (2, 16):
        dt = T / n
        Y = E.simulate_em("ou", theta, 1.0, dt, n, 1, 5, paths)[-1]
        R = O.exact_reference("ou", theta, 1.0, dt, O.normals(5, paths, n))
        err[n] = np.mean(np.abs(Y - R))
    assert err[2] / err[16] >= 4.0
    assert err[2] / err[16] < 16.0


def test_training_set_labels_are_hazen_quantiles():
    F = sample_features("ou", 3, seed=4, dt_range=(0.05, 0.3))
    term, lab = E.training_set("ou", F, 2001, 0.01, 8, 5)
    levels = scipy.stats.norm.cdf(np.polynomial.hermite_e.hermegauss(5)[0])        # library nodes + cdf
    for r in range(3):
        np.testing.assert_allclose(lab[r], np.quantile(term[r], levels, method="hazen"), rtol=1e-14)
        assert np.all(np.diff(lab[r]) >= 0)
    # terminal values are EM paths from the row's start with ceil(dt/dtau) sub-steps, global ids r*M + q
    for r in range(3):
        K = math.ceil(F[r, 1] / 0.01)
        paths = np.uint64(r * 2001) + np.arange(2001, dtype=np.uint64)
        ref = E.simulate_em("ou", tuple(F[r, 2:5]), F[r, 0], F[r, 1], 1, K, 8, paths)[-1]
        np.testing.assert_array_equal(term[r], ref)


def test_training_set_sigma_zero_row():
    """sigma = 0 -> m identical labels = the deterministic Euler value."""
    F = np.array([[1.5, 0.5, 0.2, 2.0, 0.0]])
    _, lab = E.training_set("ou", F, 64, 0.1, 1, 7)
    det = 0.2 + (1.5 - 0.2) * (1 - 2.0 * 0.1) ** 5
    np.testing.assert_allclose(lab[0], det, rtol=1e-14)


def test_training_set_matches_exact_ou_collocation():
    """OU row (y=1, dt=0.5, lam=1, Ybar=0, sigma=0.5), M = 1e5, dtau = 1e-3 -> labels
    within 3 Monte-Carlo standard errors of the exact collocation points (Eq. 6.6), plus the O(dtau)
    Euler bias."""
    M, m = 100_000, 5
    F = np.array([[1.0, 0.5, 0.0, 1.0, 0.5]])
    _, lab = E.training_set("ou", F, M, 1e-3, 3, m)
    x = O.gauss_hermite_nodes(m)
    exact = O.ou_collocation(np.array([1.0]), 0.5, 0.0, 1.0, 0.5, x)[0]
    _, std = O.ou_conditional_moments(1.0, 0.5, 0.0, 1.0, 0.5)
    p = scipy.stats.norm.cdf(x)
    se = np.sqrt(p * (1 - p) / M) / (scipy.stats.norm.pdf(x) / std)     # quantile standard error
    bias = 1e-3 * (1.0 + std * np.abs(x))                                # O(dtau) Euler bias allowance
    assert np.all(np.abs(lab[0] - exact) <= 3 * se + bias), (lab[0] - exact, se)


def test_em_substeps_rule():
    assert E.em_substeps(0.5, 1e-3) == 500
    assert E.em_substeps(0.0505, 0.01) == 6
    assert E.em_substeps(1e-4, 1e-3) == 1
