"""Pins of the 7L-CDC oracle (readings R-18..R-20 in DESIGN.md), CPU only."""
import numpy as np
import pytest
import scipy.stats

from oracle import sl7_oracle as O
from sl7_inputs import ACT_SOFTPLUS, glorot_mlp, pack_blob


def test_normal_cdf_library():
    x = np.linspace(-6, 6, 101)
    np.testing.assert_allclose(O.normal_cdf(x), scipy.stats.norm.cdf(x), rtol=1e-14, atol=1e-300)


def test_marginal_points_are_hazen_quantiles():
    rng = np.random.default_rng(3)
    Y = rng.normal(size=10_001)
    spec = O.Spec(5, "gbm", (0.05, 0.2), 1.0, 0.5, 2)
    z, C = O.cdc_table(spec, Y)
    ref = np.quantile(Y, scipy.stats.norm.cdf(O.gauss_hermite_nodes(5)), method="hazen")   # library
    np.testing.assert_allclose(z, ref, rtol=1e-14, atol=1e-14)
    assert C.shape == (5, 5)
    np.testing.assert_allclose(C, O.gbm_collocation(z, 0.5, 0.05, 0.2, spec.x), rtol=1e-15)


def test_interpolation_condition_and_constant_rows():
    spec = O.Spec(5, "ou", (0.0, 1.0, 0.5), 1.0, 0.25, 3)
    z = np.array([-1.0, -0.3, 0.1, 0.7, 2.0])
    C = spec.points(z)
    np.testing.assert_allclose(O.cdc_points(z, C, z), C, atol=1e-13)          # y = z_k -> row C[k]
    Cc = np.tile(np.arange(5.0), (5, 1))
    np.testing.assert_allclose(O.cdc_points(z, Cc, np.array([-3.0, 0.5, 4.0])), np.tile(np.arange(5.0), (3, 1)),
                               atol=1e-11)                                       # constant rows


def test_degenerate_states_use_nearest_row():
    spec = O.Spec(5, "gbm", (0.05, 0.2), 1.0, 0.5, 2)
    z, C = O.cdc_table(spec, np.full(100, 1.3))                                  # all paths equal
    assert np.all(z == 1.3)
    np.testing.assert_allclose(C, np.tile(O.gbm_collocation(np.array([1.3]), 0.5, 0.05, 0.2, spec.x)[0], (5, 1)))
    np.testing.assert_array_equal(O.cdc_points(z, C, np.array([1.3, 9.0])), C[[0, 0]])
    z2 = np.array([0.0, 1.0, 1.0, 2.0, 3.0])                                     # partially repeated
    C2 = np.arange(25.0).reshape(5, 5)
    np.testing.assert_array_equal(O.cdc_points(z2, C2, np.array([0.9, 1.2, 2.6])), C2[[1, 1, 4]])


@pytest.mark.parametrize("colloc,theta,m", [("ou", (0.0, 1.0, 0.5), 5), ("ou", (0.3, 0.5, 1.1), 7),
                                            ("gbm", (0.05, 0.2), 5), ("gbm", (0.05, 0.2), 7)])
def test_cdc_equals_7l_for_affine_collocation(colloc, theta, m):
    # with exact collocation the conditional points are affine in the state
    # (OU: mean + std x_j; GBM: Y c_j), which Lagrange interpolation on the z_k reproduces exactly,
    # so CDC and 7L coincide path by path (up to rounding amplified by extrapolation into the tails)
    spec = O.Spec(m, colloc, theta, 1.0, 0.25, 8)
    paths = np.arange(20_000, dtype=np.uint64)
    Y7, _ = O.simulate(spec, 77, paths)
    Yc, _ = O.simulate_cdc(spec, 77, paths)
    scale = np.maximum(1.0, np.abs(Y7))
    assert np.max(np.abs(Yc - Y7) / scale) < 1e-8


def test_cdc_sigma_zero_equals_7l():
    spec = O.Spec(5, "gbm", (0.05, 0.0), 1.0, 0.25, 4)
    paths = np.arange(50, dtype=np.uint64)
    np.testing.assert_allclose(O.simulate_cdc(spec, 1, paths)[0], O.simulate(spec, 1, paths)[0], rtol=1e-14)


def test_cdc_ann_first_step_equals_7l():
    # step 0: every path starts at Y0, so the table has one distinct row H(Y0) = the 7L points
    p = glorot_mlp((5, 16, 16, 7), ACT_SOFTPLUS, seed=4, with_norm=True)
    net = O.parse_blob(pack_blob(p))
    spec = O.Spec(7, "ann", (0.0, 1.0, 0.5), 1.0, 0.125, 1, net=net)
    paths = np.arange(300, dtype=np.uint64)
    np.testing.assert_allclose(O.simulate_cdc(spec, 3, paths)[0], O.simulate(spec, 3, paths)[0], rtol=1e-14)
