"""Pins of the 7L-CDC oracle with predicted marginal points (SL7_SCHEME_CDC_PRED; "only
requires the ANNs to compute a small number of marginal collocation points"; reading R-26 of DESIGN.md),
CPU only."""
import numpy as np
import pytest
import scipy.stats

from oracle import sl7_oracle as O
from sl7_inputs import load_golden_blob, workloads


def test_gbm_marginals_are_lognormal_quantiles():
    # the exact GBM predictor at horizon t_i from Y0: the quantiles of the lognormal law of Y(t_i) at
    # Phi(x_k) (library: scipy.stats.lognorm.ppf)
    mu, s, y0, dt = 0.05, 0.2, 1.3, 0.25
    spec = O.Spec(7, "gbm", (mu, s), y0, dt, 8)
    for i in (1, 3, 7):
        t = i * dt
        ref = scipy.stats.lognorm.ppf(scipy.stats.norm.cdf(spec.x), s=s * np.sqrt(t),
                                      scale=y0 * np.exp((mu - 0.5 * s * s) * t))
        np.testing.assert_allclose(O.cdc_pred_marginals(spec, i), ref, rtol=1e-12)


def test_ou_marginals_are_normal_quantiles():
    # Eq. 6.6 at horizon t_i: N(Ybar + (Y0 - Ybar) e^{-lam t}, s^2 (1 - e^{-2 lam t}) / (2 lam))
    ybar, lam, s, y0, dt = 0.3, 1.5, 0.5, 1.0, 0.125
    spec = O.Spec(5, "ou", (ybar, lam, s), y0, dt, 16)
    for i in (1, 5, 15):
        t = i * dt
        e = np.exp(-lam * t)
        ref = scipy.stats.norm.ppf(scipy.stats.norm.cdf(spec.x), loc=ybar + (y0 - ybar) * e,
                                   scale=s * np.sqrt((1 - e * e) / (2 * lam)))
        np.testing.assert_allclose(O.cdc_pred_marginals(spec, i), ref, rtol=1e-12, atol=1e-14)


def test_step_zero_is_row_zero():
    # t_0: every path at Y0, so all marginal points repeat and R-20's nearest row (row 0 = H(Y0)) applies
    spec = O.Spec(5, "ou", (0.0, 1.0, 0.5), 1.0, 0.25, 3)
    assert np.all(O.cdc_pred_marginals(spec, 0) == 1.0)
    Y = np.full(4, 1.0)
    Z = np.array([-2.0, -0.1, 0.3, 4.0])
    ref = O.lagrange_eval(Z, spec.x, np.tile(spec.points(np.array([1.0]))[0], (4, 1)))
    np.testing.assert_allclose(O.cdc_pred_step(spec, 0, Y, Z), ref, rtol=1e-15)


@pytest.mark.parametrize("colloc, theta, m", [("ou", (0.0, 1.0, 0.5), 7), ("ou", (0.4, 0.3, 1.2), 5),
                                              ("gbm", (0.05, 0.2), 5), ("gbm", (0.1, 0.4), 7)])
def test_cdc_pred_equals_7l_step_for_affine_collocation(colloc, theta, m):
    # exact OU (affine in the state) and exact GBM (linear): the Lagrange interpolant of the table in the
    # state reproduces it exactly, so a CDC_PRED step is the 7L step from the state clamped to the hull
    # (the same 7L step inside it); checked one step at a time on 7L's own states
    spec = O.Spec(m, colloc, theta, 1.0, 0.25, 8)
    paths = np.arange(4000, dtype=np.uint64) * np.uint64(7919)
    Y7, Z = O.simulate(spec, 11, paths)
    outside = 0
    for i in range(spec.n_steps):
        z = O.cdc_pred_marginals(spec, i)
        Yc = np.clip(Y7[i], z[0], z[-1]) if i > 0 else Y7[i]
        outside += int(np.sum(Yc != Y7[i]))
        ref = O.step(spec, Yc, Z[i])
        np.testing.assert_allclose(O.cdc_pred_step(spec, i, Y7[i], Z[i]), ref, rtol=1e-9, atol=1e-11)
        inside = Yc == Y7[i]
        np.testing.assert_allclose(O.cdc_pred_step(spec, i, Y7[i], Z[i])[inside], Y7[i + 1][inside], rtol=1e-9,
                                   atol=1e-11)
    assert outside > 0          # the clamp was exercised


def test_hull_clamp_is_flat_extension():
    # beyond the extreme marginal points a path reads the extreme table row (hand-built table)
    spec = O.Spec(5, "ou", (0.0, 1.0, 0.5), 1.0, 0.25, 3)
    z = O.cdc_pred_marginals(spec, 2)
    C = spec.points(z)
    Y = np.array([z[0] - 5.0, z[-1] + 3.0, np.nan])
    P = O.cdc_points(z, C, O.cdc_pred_state(z, Y))
    np.testing.assert_allclose(P[0], C[0], rtol=1e-13)
    np.testing.assert_allclose(P[1], C[-1], rtol=1e-13)
    assert np.all(np.isnan(P[2]))


def test_paths_are_independent():
    # no cross-path coupling: a subset simulated alone equals the same paths inside a larger set
    w = workloads()["cfg0"]
    spec = O.Spec(w.m, "ann", (), w.y0, w.dt, w.n_steps, net=O.parse_blob(load_golden_blob(w.blob)))
    big = np.arange(500, dtype=np.uint64)
    Yb, _ = O.simulate_cdc_pred(spec, 5, big)
    Ys, _ = O.simulate_cdc_pred(spec, 5, big[123:130])
    np.testing.assert_array_equal(Ys, Yb[:, 123:130])


def test_cir_network_stays_bounded():
    # the motivating property (R-25/R-26): on cfg2's CIR network the empirical-quantile CDC
    # diverges; with predicted marginal points every state stays finite and within the network's range
    w = workloads()["cfg2_cir"]
    spec = O.Spec(w.m, "ann", tuple(w.theta), w.y0, w.dt, w.n_steps, net=O.parse_blob(load_golden_blob(w.blob)))
    with np.errstate(all="ignore"):
        Y, _ = O.simulate_cdc_pred(spec, w.seed, np.arange(20_000, dtype=np.uint64))
    assert np.all(np.isfinite(Y))
    assert np.abs(Y).max() < 2.0
    # the CIR law's mean (0.1 from Y0 = Ybar) within 1% plus 3 standard errors of the 2e4-path mean: the
    # network is fitted for horizons up to T = 4 (oracle/fit_weights.py RANGES), so the predictor is not
    # extrapolated at any t_i of configs 2 and 4
    assert abs(Y[-1].mean() - 0.1) < 0.001 + 3 * Y[-1].std() / np.sqrt(Y.shape[1])


def test_golden_blobs_carry_their_fitted_box():
    # every golden network states the feature box it was fitted on (blob flags bit 2), and the CIR box
    # covers the CDC_PRED horizons of configs 2 and 4 (t_i up to (n_steps - 1) dt)
    import struct
    for key in ("cfg0", "cfg1", "cfg2_ou", "cfg2_cir", "cfg4"):
        w = workloads()[key]
        blob = load_golden_blob(w.blob)
        nd = struct.unpack_from("<I", blob, 8)[0]
        flags = struct.unpack_from("<I", blob, 16 + 4 * nd)[0]
        assert flags & 4, key
        d_in = struct.unpack_from("<I", blob, 12)[0]
        hi = np.frombuffer(blob[-4 * d_in:], dtype="<f4")
        lo = np.frombuffer(blob[-8 * d_in:-4 * d_in], dtype="<f4")
        assert np.all(lo <= hi)
        if w.process == "cir":
            assert lo[1] <= w.dt and (w.n_steps - 1) * w.dt <= hi[1] and lo[0] <= w.y0 <= hi[0]


def test_cdc_pred_clamped_counts_states_outside_the_hull():
    # by hand: 3 steps of exact OU from Y0 = 1; step 0 has every path at Y0 (repeated z: nearest row, no
    # clamp); the states of steps 1 and 2 are placed inside, below and above the predicted hull
    spec = O.Spec(5, "ou", (0.0, 1.0, 0.5), 1.0, 0.25, 3)
    z1, z2 = O.cdc_pred_marginals(spec, 1), O.cdc_pred_marginals(spec, 2)
    Y = np.empty((4, 4))
    Y[0] = 1.0
    Y[1] = [z1[0] - 1e-3, 0.5 * (z1[0] + z1[-1]), z1[-1] + 1.0, np.nan]
    Y[2] = [z2[0], z2[-1], z2[-1] + 1e-9, z2[0] - 5.0]
    Y[3] = 123.0                                   # the terminal row is never read by a table
    assert O.cdc_pred_clamped(spec, Y) == 2 + 2


@pytest.mark.parametrize("m", [5, 7])
def test_bivariate_form_of_the_cdc_step_is_the_same_polynomial(m):
    # the device evaluates the CDC(_PRED) step as ONE bivariate polynomial Y' = sum_a sum_b D[a][b] s^a X^b,
    # D = A^T C B (A, B: monomial coefficients of the Lagrange bases on the hull-normalised marginal points and on
    # the Gauss-Hermite nodes).  Mathematically it is the oracle's two-stage Lagrange step: checked
    # here in float64 on a random table, inside and outside the hull, with numpy's polynomial routines building A, B
    rng = np.random.default_rng(m)
    x = O.gauss_hermite_nodes(m)
    z = np.sort(rng.uniform(-1.0, 2.0, m))
    C = rng.normal(size=(m, m))
    c, h = 0.5 * (z[0] + z[-1]), 0.5 * (z[-1] - z[0])
    sn = (z - c) / h

    def mono(nodes):   # A[k][a] = coefficient of t^a in the k-th Lagrange basis polynomial
        A = np.zeros((len(nodes), len(nodes)))
        for k in range(len(nodes)):
            others = np.delete(nodes, k)
            poly = np.polynomial.polynomial.polyfromroots(others) / np.prod(nodes[k] - others)
            A[k] = poly
        return A

    D = mono(sn).T @ C @ mono(x)
    Y = rng.uniform(z[0] - 0.3, z[-1] + 0.3, 500)
    X = rng.normal(size=500) * 2
    s = (Y - c) / h
    biv = np.einsum("pa,ab,pb->p", np.vander(s, m, increasing=True), D, np.vander(X, m, increasing=True))
    ref = O.lagrange_eval(X, x, O.lagrange_basis(Y, z) @ C)
    np.testing.assert_allclose(biv, ref, rtol=1e-9, atol=1e-9 * np.abs(ref).max())
