"""Pins of the float64 oracle to things other than itself (CPU only, -m "not gpu").

Each pin is chosen so that a plausible slip in oracle/sl7_oracle.py (a dropped term, a wrong sign,
a swapped index or operand) fails at least one test here.  Citations: PAPER.md lines + section.
"""
import math
import os
import struct

import mpmath
import numpy as np
import pytest
import scipy.interpolate
import scipy.integrate
import scipy.stats
import torch

from _helpers import affine_softplus_mlp
from oracle import sl7_oracle as O
from sl7_inputs import ACT_SOFTPLUS, ACT_TANH, MlpParams, glorot_mlp, pack_blob

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- O1 Gauss-Hermite nodes

def _closed_form_nodes(m):
    """Roots of the probabilists' Hermite polynomials He_m written out by hand."""
    s = math.sqrt
    if m == 1:
        return [0.0]
    if m == 2:
        return [-1.0, 1.0]                                   # He2 = x^2 - 1
    if m == 3:
        return [-s(3), 0.0, s(3)]                            # He3 = x^3 - 3x
    if m == 4:
        a, b = s(3 - s(6)), s(3 + s(6))                      # He4 = x^4 - 6x^2 + 3
        return [-b, -a, a, b]
    if m == 5:
        a, b = s(5 - s(10)), s(5 + s(10))                    # He5 = x^5 - 10x^3 + 15x
        return [-b, -a, 0.0, a, b]
    if m == 6:                                               # He6: z^3 - 15 z^2 + 45 z - 15, z = x^2
        z = np.sort(np.roots([1, -15, 45, -15]).real)
        r = np.sqrt(z)
        return sorted(list(-r) + list(r))
    if m == 7:                                               # He7 = x (z^3 - 21 z^2 + 105 z - 105)
        z = np.sort(np.roots([1, -21, 105, -105]).real)
        r = np.sqrt(z)
        return sorted(list(-r) + [0.0] + list(r))
    raise ValueError


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6, 7])
def test_nodes_closed_form(m):
    np.testing.assert_allclose(O.gauss_hermite_nodes(m), _closed_form_nodes(m), rtol=0, atol=5e-15 * max(1, m))


@pytest.mark.parametrize("m", range(1, 17))
def test_nodes_library_and_invariants(m):
    x = O.gauss_hermite_nodes(m)
    ref, _ = np.polynomial.hermite_e.hermegauss(m)          # library (probabilists' Hermite)
    np.testing.assert_allclose(x, ref, atol=1e-13)
    np.testing.assert_allclose(x, -x[::-1], atol=1e-13)     # symmetry
    assert np.all(np.diff(x) > 0)
    c = np.zeros(m + 1)
    c[m] = 1
    val = np.polynomial.hermite_e.hermeval(x, c)            # He_m(x_j) = 0
    scale = np.polynomial.polynomial.polyval(np.abs(x) + 1, np.abs(np.polynomial.hermite_e.herme2poly(c)))
    assert np.all(np.abs(val) <= 1e-12 * scale)


def test_nodes_not_physicists():
    # reading R-1: probabilists'. The physicists' m=2 nodes are +-1/sqrt(2); ours must be +-1.
    assert abs(O.gauss_hermite_nodes(2)[1] - 1.0) < 1e-15


# ---------------------------------------------------------------- barycentric weights

def test_bary_weights_spec_examples():
    np.testing.assert_allclose(O.bary_weights([0, 1, 2]), [0.5, -1, 0.5], rtol=1e-15)
    np.testing.assert_allclose(O.bary_weights([-1, 1]), [-0.5, 0.5], rtol=1e-15)


@pytest.mark.parametrize("m", range(2, 12))
def test_bary_weights_hermite_closed_form(m):
    # He_m' = m He_{m-1}  =>  prod_{k != j}(x_j - x_k) = He_m'(x_j) = m He_{m-1}(x_j)
    x = O.gauss_hermite_nodes(m)
    c = np.zeros(m)
    c[m - 1] = 1
    ref = 1.0 / (m * np.polynomial.hermite_e.hermeval(x, c))
    np.testing.assert_allclose(O.bary_weights(x), ref, rtol=1e-13)
    w = O.bary_weights(x)
    np.testing.assert_allclose(w, (-1) ** (m - 1) * w[::-1], rtol=1e-13)


# ---------------------------------------------------------------- O4 Lagrange interpolation

@pytest.mark.parametrize("m", [1, 2, 3, 5, 7, 9])
def test_lagrange_reproduces_polynomials(m):
    rng = np.random.default_rng(m)
    x = O.gauss_hermite_nodes(m)
    z = np.linspace(-4, 4, 401)
    for deg in range(m):
        coef = rng.normal(size=deg + 1)
        p = np.polynomial.polynomial.polyval(z, coef)
        g = O.lagrange_eval(z, x, np.polynomial.polynomial.polyval(x, coef))
        assert np.all(np.abs(g - p) <= 1e-11 * (1 + np.abs(p)) * max(1, 4 ** deg))
    # degree m is NOT reproduced (catches an interpolant built on the wrong number of nodes)
    if m >= 2:
        coef = np.zeros(m + 1)
        coef[m] = 1
        g = O.lagrange_eval(np.array([3.3]), x, np.polynomial.polynomial.polyval(x, coef))
        assert abs(g[0] - 3.3 ** m) > 1e-3


def test_lagrange_cardinal_and_partition_of_unity():
    x = O.gauss_hermite_nodes(7)
    L = O.lagrange_basis(x, x)
    np.testing.assert_allclose(L, np.eye(7), atol=1e-13)
    z = np.linspace(-5.8, 5.8, 101)
    np.testing.assert_allclose(O.lagrange_basis(z, x).sum(-1), 1.0, atol=1e-10)


def test_lagrange_x_cubed_spec():
    x = O.gauss_hermite_nodes(5)                        # x^3 on m=5, 1e-12 on [-3,3]
    z = np.linspace(-3, 3, 61)
    np.testing.assert_allclose(O.lagrange_eval(z, x, x ** 3), z ** 3, atol=1e-12)


@pytest.mark.parametrize("m", [5, 7])
def test_lagrange_matches_scipy_barycentric(m):
    rng = np.random.default_rng(0)
    x = O.gauss_hermite_nodes(m)
    y = rng.normal(size=m)
    z = rng.uniform(-5.8, 5.8, 500)
    ref = scipy.interpolate.BarycentricInterpolator(x, y)(z)      # library, Berrut-Trefethen
    np.testing.assert_allclose(O.lagrange_eval(z, x, y), ref, rtol=1e-11, atol=1e-11 * np.abs(ref).max())


def test_lagrange_per_path_points():
    # per-path points of shape (P, m) pair with Z of shape (P,) (no transposition)
    x = O.gauss_hermite_nodes(3)
    y = np.array([[1.0, 2.0, 3.0], [5.0, 5.0, 5.0]])
    z = np.array([x[0], 0.3])
    np.testing.assert_allclose(O.lagrange_eval(z, x, y), [1.0, 5.0], atol=1e-14)


# ---------------------------------------------------------------- O2 RNG

def test_philox_known_answers():
    rows = [l.split() for l in open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")) if l.strip() and l[0] != "#"]
    assert len(rows) == 3
    for r in rows:
        v = [int(t, 16) for t in r]
        out = O.philox4x32_10(*v[:6])
        assert [int(o) for o in out] == v[6:]


def test_philox_counter_layout():
    # counter = (block, 0, path_lo, path_hi), key = (seed_lo, seed_hi) (reading R-8); different paths
    # above 2^32 must differ only through ctr3, and the key halves must both matter.
    seed = 0x0123456789ABCDEF
    p = np.array([5, 5 + (1 << 32)], dtype=np.uint64)
    a = O.philox_block(seed, p, 3)
    b0 = O.philox4x32_10(3, 0, 5, 0, 0x89ABCDEF, 0x01234567)
    b1 = O.philox4x32_10(3, 0, 5, 1, 0x89ABCDEF, 0x01234567)
    assert [int(t[0]) for t in a] == [int(t) for t in b0]
    assert [int(t[1]) for t in a] == [int(t) for t in b1]
    c = O.philox_block(seed ^ (1 << 40), p, 3)                      # seed_hi is part of the key
    assert [int(t[0]) for t in a] != [int(t[0]) for t in c]


def test_uniform_grid():
    r = np.array([0, 1 << 9, 0xFFFFFFFF], dtype=np.uint64)
    u = O.u32_to_uniform(r)
    assert u[0] == 2.0 ** -24 and u[1] == 3 * 2.0 ** -24 and u[2] == 1 - 2.0 ** -24
    assert np.all(u.astype(np.float32).astype(np.float64) == u)       # exact in fp32


def test_box_muller_mpmath():
    mpmath.mp.dps = 40
    r = np.array([0, 1, 511, 512, 12345678, 1 << 31, 0xFFFFFE00, 0xFFFFFFFF, 0xDEADBEEF, 0x7FFFFFFF], dtype=np.uint64)
    u = O.u32_to_uniform(r)
    for ua in u:
        for ub in u:
            z0, z1 = O.box_muller(np.array([ua]), np.array([ub]))
            rad = mpmath.sqrt(-2 * mpmath.log(mpmath.mpf(float(ua))))
            ang = 2 * mpmath.pi * mpmath.mpf(float(ub))
            r0, r1 = rad * mpmath.cos(ang), rad * mpmath.sin(ang)
            assert abs(z0[0] - float(r0)) <= 4e-15 * float(rad)
            assert abs(z1[0] - float(r1)) <= 4e-15 * float(rad)


def test_normals_statistics():
    n = 250_000
    Z = O.normals(7, np.arange(n, dtype=np.uint64), 4)       # one Philox block per path
    flat = Z.ravel()
    assert abs(flat.mean()) < 4 / math.sqrt(flat.size)
    assert abs(flat.var() - 1) < 6 * math.sqrt(2 / flat.size)
    assert scipy.stats.kstest(flat, "norm").pvalue > 1e-4
    assert np.abs(flat).max() <= math.sqrt(48 * math.log(2)) + 1e-12
    # cross-path and cross-step independence
    assert abs(np.corrcoef(Z[0, :-1], Z[0, 1:])[0, 1]) < 0.02
    for i, j in [(0, 1), (0, 2), (1, 3), (2, 3)]:
        assert abs(np.corrcoef(Z[i], Z[j])[0, 1]) < 0.02


def test_normals_step_to_block_mapping():
    # step i uses Z_{4b + (i & 3)} of block b = i >> 2; 6 steps span two blocks
    paths = np.array([0, 99, 1 << 33], dtype=np.uint64)
    Z = O.normals(11, paths, 6)
    zs0 = O.normals_block(11, paths, 0)
    zs1 = O.normals_block(11, paths, 1)
    for i in range(4):
        np.testing.assert_array_equal(Z[i], zs0[i])
    np.testing.assert_array_equal(Z[4], zs1[0])
    np.testing.assert_array_equal(Z[5], zs1[1])
    # independent of which subset of paths is requested (sharding transparency)
    np.testing.assert_array_equal(O.normals(11, paths[2:], 6)[:, 0], Z[:, 2])


# ---------------------------------------------------------------- O3 collocation points

def test_gbm_collocation_is_lognormal_quantile():
    # Eq. 6.3: y_j = F^{-1}_{Y(t+dt)|Y}(Phi(x_j)); GBM's law is lognormal (library quantile)
    x = O.gauss_hermite_nodes(7)
    Y, dt, mu, s = 1.7, 0.37, 0.05, 0.2
    ref = scipy.stats.lognorm.ppf(scipy.stats.norm.cdf(x), s=s * math.sqrt(dt),
                                  scale=Y * math.exp((mu - s * s / 2) * dt))
    np.testing.assert_allclose(O.gbm_collocation(np.array([Y]), dt, mu, s, x)[0], ref, rtol=1e-10)


def test_ou_moments_spec_examples():
    m, s = O.ou_conditional_moments(1.0, math.log(2), 0.0, 1.0, 0.0)
    assert abs(m - 0.5) < 1e-15 and s == 0
    m, s = O.ou_conditional_moments(0.0, 1e6, 0.0, 1.0, 1.0)
    assert abs(s - math.sqrt(0.5)) < 1e-9
    m, s = O.ou_conditional_moments(1.3, 0.25, 0.0, 0.0, 0.4)              # SPEC.md:73 (lam -> 0)
    assert abs(m - 1.3) < 1e-15 and abs(s - 0.2) < 1e-15
    m, s = O.ou_conditional_moments(0.0, 1.0, 2.0, 1.0, 0.0)
    assert abs(m - 2 * (1 - math.exp(-1))) < 1e-14


def test_ou_variance_by_quadrature_and_semigroup():
    # Var = sigma^2 int_0^dt e^{-2 lam (dt - s)} ds  (Ito isometry on Eq. 6.5), library quadrature
    for lam, dt, sig in [(1.0, 0.125, 0.5), (0.3, 2.0, 1.1), (5.0, 0.01, 0.2), (1e-8, 0.5, 0.7)]:
        q, _ = scipy.integrate.quad(lambda s_: math.exp(-2 * lam * (dt - s_)), 0, dt, epsabs=1e-14, epsrel=1e-13)
        _, std = O.ou_conditional_moments(0.0, dt, 0.0, lam, sig)
        assert abs(std ** 2 - sig * sig * q) <= 1e-12 * sig * sig * q
    # semigroup: var(d1+d2) = var(d2) + e^{-2 lam d2} var(d1); mean composes
    lam, sig, ybar = 0.7, 0.4, 0.3
    d1, d2 = 0.3, 0.9
    _, s1 = O.ou_conditional_moments(0.0, d1, ybar, lam, sig)
    _, s2 = O.ou_conditional_moments(0.0, d2, ybar, lam, sig)
    _, s12 = O.ou_conditional_moments(0.0, d1 + d2, ybar, lam, sig)
    assert abs(s12 ** 2 - (s2 ** 2 + math.exp(-2 * lam * d2) * s1 ** 2)) < 1e-12
    m1, _ = O.ou_conditional_moments(1.5, d1, ybar, lam, sig)
    m2, _ = O.ou_conditional_moments(m1, d2, ybar, lam, sig)
    m12, _ = O.ou_conditional_moments(1.5, d1 + d2, ybar, lam, sig)
    assert abs(m2 - m12) < 1e-14


def test_ou_series_switch_continuous():
    for dt in (0.5, 2.0):
        lam = 1e-6 / dt
        _, a = O.ou_conditional_moments(0.0, dt, 0.0, lam * (1 - 1e-9), 1.0)
        _, b = O.ou_conditional_moments(0.0, dt, 0.0, lam * (1 + 1e-9), 1.0)
        assert abs(a - b) < 1e-10 * a


def test_ou_collocation_is_normal_quantile():
    x = O.gauss_hermite_nodes(5)
    y = O.ou_collocation(np.array([1.0]), 0.5, 0.0, 1.0, 0.5, x)[0]     # SPEC.md:91 example
    ref = scipy.stats.norm.ppf(scipy.stats.norm.cdf(x), loc=math.exp(-0.5),
                               scale=0.5 * math.sqrt((1 - math.exp(-1)) / 2))
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)


def test_cir_collocation_mean():
    # mean of c * chi'^2(d, lam_nc) = c (d + lam_nc) = Y e^{-k dt} + ybar (1 - e^{-k dt})
    k, ybar, s, Y, dt = 1.0, 0.1, 0.3, 0.1, 0.125
    c = s * s * (1 - math.exp(-k * dt)) / (4 * k)
    d = 4 * k * ybar / (s * s)
    lam_nc = Y * math.exp(-k * dt) / c
    assert abs(c * scipy.stats.ncx2.mean(d, lam_nc) - (Y * math.exp(-k * dt) + ybar * (1 - math.exp(-k * dt)))) < 1e-14
    x = O.gauss_hermite_nodes(7)
    y = O.cir_collocation(np.array([Y]), dt, k, ybar, s, x)[0]
    assert np.all(np.diff(y) > 0) and y[0] > 0
    # the median node x=0 is the conditional median
    assert abs(y[3] - c * scipy.stats.ncx2.median(d, lam_nc)) < 1e-10


# ---------------------------------------------------------------- ANN forward (Eq. 6.4)

def _torch_net(p: MlpParams):
    layers = []
    for l, (W, b) in enumerate(zip(p.W, p.b)):
        lin = torch.nn.Linear(W.shape[1], W.shape[0]).double()
        with torch.no_grad():
            lin.weight.copy_(torch.tensor(W))
            lin.bias.copy_(torch.tensor(b))
        layers.append(lin)
        if l < len(p.W) - 1:
            layers.append(torch.nn.Tanh() if p.act == ACT_TANH else torch.nn.Softplus())
    return torch.nn.Sequential(*layers)


@pytest.mark.parametrize("dims,act", [((2, 50, 50, 50, 5), ACT_TANH), ((5, 50, 50, 50, 50, 7), ACT_SOFTPLUS),
                                      ((3, 17, 9, 4), ACT_TANH)])
def test_mlp_matches_torch(dims, act):
    p = glorot_mlp(dims, act, seed=3, with_norm=True)
    net = O.parse_blob(pack_blob(p))
    rng = np.random.default_rng(1)
    F = rng.normal(size=(257, dims[0]))
    with torch.no_grad():
        ref = _torch_net(p)(torch.tensor((F - p.in_shift) / p.in_scale)).numpy() * p.out_scale + p.out_shift
    np.testing.assert_allclose(O.mlp_forward(net, F), ref, rtol=1e-13, atol=1e-13)


def test_mlp_special_cases():
    dims = (2, 4, 3)
    z = MlpParams(dims, ACT_SOFTPLUS, [np.zeros((4, 2)), np.zeros((3, 4))], [np.zeros(4), np.array([1.0, 2, 3])])
    out = O.mlp_forward(O.parse_blob(pack_blob(z)), np.ones((5, 2)))
    np.testing.assert_array_equal(out, np.tile([1.0, 2, 3], (5, 1)))      # zero weights -> output bias
    # hand-computed 1-input chain: h = softplus(2*x - 1); y = 3*h + 0.5
    hand = MlpParams((1, 1, 1), ACT_SOFTPLUS, [np.array([[2.0]]), np.array([[3.0]])], [np.array([-1.0]), np.array([0.5])])
    xv = 0.8
    y = O.mlp_forward(O.parse_blob(pack_blob(hand)), np.array([[xv]]))[0, 0]
    assert abs(y - (3 * math.log(1 + math.exp(2 * xv - 1)) + 0.5)) < 1e-14
    assert abs(O.softplus(0.0) - math.log(2)) < 1e-16
    assert abs(O.softplus(100.0) - 100.0) < 1e-12
    assert abs(O.softplus(-100.0) / math.exp(-100) - 1) < 1e-6


def test_blob_round_trip_and_errors():
    p = glorot_mlp((5, 50, 50, 7), ACT_SOFTPLUS, seed=9, with_norm=True)
    blob = pack_blob(p)
    net = O.parse_blob(blob)
    for a, b in zip(net.W, p.W):
        np.testing.assert_array_equal(a, b)
    bad = bytearray(blob)
    bad[4] = 2
    with pytest.raises(ValueError, match="version"):
        O.parse_blob(bytes(bad))
    with pytest.raises(ValueError, match="size"):
        O.parse_blob(blob + b"\0\0\0\0")


def test_round_bf16_matches_torch():
    rng = np.random.default_rng(5)
    v = np.concatenate([rng.normal(size=20000) * 3, rng.uniform(-1, 1, 20000)]).astype(np.float32).astype(np.float64)
    # exact ties: fp32 values with the 16 dropped bits = 0x8000
    ties = (np.arange(1, 2001, dtype=np.uint32) << 16 | 0x8000) + np.uint32(0x3F000000)
    v = np.concatenate([v, ties.view(np.float32).astype(np.float64)])
    ref = torch.tensor(v, dtype=torch.float32).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(O.round_bf16(v), ref)


def test_round_tf32_bit_trick():
    rng = np.random.default_rng(6)
    v = rng.normal(size=20000).astype(np.float32)
    ties = ((np.arange(1, 2001, dtype=np.uint32) << 13) | 0x1000) + np.uint32(0x3F000000)
    v = np.concatenate([v, ties.view(np.float32), -ties.view(np.float32)])
    bits = v.view(np.uint32)
    # cvt.rna.tf32: add half an ulp of the 10-bit mantissa to the magnitude bits, truncate
    ref = ((bits + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32).astype(np.float64)
    np.testing.assert_array_equal(O.round_tf32(v.astype(np.float64)), ref)


def test_quantised_forward_reduces_to_plain_when_exact():
    # O6 with weights and activations already on the bf16 grid equals the plain forward
    p = glorot_mlp((2, 8, 8, 3), ACT_TANH, seed=2)
    p.W = [O.round_bf16(w) for w in p.W]
    net = O.parse_blob(pack_blob(p))
    net_id = O.Mlp(net.dims, ACT_TANH, net.W, net.b)
    F = np.random.default_rng(0).normal(size=(50, 2))
    a = O.mlp_forward(net_id, F, "bf16")
    b = O.mlp_forward(net_id, F)
    assert np.max(np.abs(a - b)) < 2e-2 and np.max(np.abs(a - b)) > 0      # activations still rounded
    net_id.act = -1
    # identity "activation" is not allowed; guard that the rounding hits layers >= 2 only:
    W0 = net.W[0]
    assert np.array_equal(O.round_bf16(W0), W0)


# ---------------------------------------------------------------- Algorithm I end to end (exact modes)

def test_exact_ou_path_equals_eq66_recursion_dt_flat():
    # SPEC.md:503-504 + PAPER.md:16 (error does not grow with dt): linear y_j => g_m exact
    for dt in (0.25, 0.5, 1.0, 2.0):
        n = int(round(2.0 / dt))
        spec = O.Spec(5, "ou", (0.0, 1.0, 0.5), 1.0, dt, n)
        Y, Z = O.simulate(spec, 123, np.arange(2000, dtype=np.uint64))
        R = O.exact_reference("ou", (0.0, 1.0, 0.5), 1.0, dt, Z)
        assert np.max(np.abs(Y[-1] - R)) < 1e-9


def test_sigma_zero_deterministic():
    spec = O.Spec(5, "gbm", (0.05, 0.0), 1.0, 0.25, 4)
    Y, _ = O.simulate(spec, 1, np.arange(10, dtype=np.uint64))
    np.testing.assert_allclose(Y[:, 3], np.exp(0.05 * 0.25 * np.arange(5)), rtol=1e-13)
    spec = O.Spec(7, "ou", (0.3, 2.0, 0.0), 1.0, 0.5, 3)
    Y, _ = O.simulate(spec, 1, np.arange(10, dtype=np.uint64))
    t = 0.5 * np.arange(4)
    np.testing.assert_allclose(Y[:, 0], np.exp(-2 * t) + 0.3 * (1 - np.exp(-2 * t)), rtol=1e-13)


def test_m1_is_conditional_median():
    spec = O.Spec(1, "gbm", (0.05, 0.2), 1.0, 0.5, 2)
    Y, _ = O.simulate(spec, 1, np.arange(4, dtype=np.uint64))
    np.testing.assert_allclose(Y[-1], np.exp(2 * (0.05 - 0.02) * 0.5), rtol=1e-14)


@pytest.mark.parametrize("m", [5, 7])
def test_exact_gbm_remainder_bound_and_dt_convergence(m):
    # interpolation remainder: |g_m(Z) - e^{a+bZ}| <= Y b^m/m! e^{b max(|Z|, x_max)} |prod (Z - x_j)|
    mu, s = 0.05, 0.2
    x = O.gauss_hermite_nodes(m)
    errs = []
    for n in (1, 4, 16, 64):
        dt = 1.0 / n
        spec = O.Spec(m, "gbm", (mu, s), 1.0, dt, n)
        Y, Z = O.simulate(spec, 5, np.arange(20000, dtype=np.uint64))
        Yprev = Y[-2]
        b = s * math.sqrt(dt)
        exact_step = Yprev * np.exp((mu - s * s / 2) * dt + b * Z[-1])
        bound = Yprev * b ** m / math.factorial(m) * np.exp(b * np.maximum(np.abs(Z[-1]), x[-1])) * \
            np.abs(np.prod(Z[-1][:, None] - x[None, :], axis=1)) * math.exp((mu - s * s / 2) * dt)
        assert np.all(np.abs(Y[-1] - exact_step) <= bound * (1 + 1e-9) + 1e-15)
        R = O.exact_reference("gbm", (mu, s), 1.0, dt, Z)
        errs.append(np.mean(np.abs(Y[-1] - R)))
    # strong error at T does not grow as dt shrinks; it falls like dt^{(m-1)/2}
    assert all(errs[k + 1] < errs[k] for k in range(len(errs) - 1))
    assert errs[0] / errs[1] > 0.5 * 4 ** ((m - 1) / 2)


def test_exact_ou_terminal_moments_match_eq66():
    # N=4, T=2, 1e5 paths, within 4 standard errors of Eq. 6.6
    spec = O.Spec(5, "ou", (0.0, 1.0, 0.5), 1.0, 0.5, 4)
    Y, _ = O.simulate(spec, 99, np.arange(100_000, dtype=np.uint64))
    mean, std = O.ou_conditional_moments(1.0, 2.0, 0.0, 1.0, 0.5)
    se = std / math.sqrt(1e5)
    assert abs(Y[-1].mean() - mean) < 4 * se
    assert abs(Y[-1].var() - std ** 2) < 4 * std ** 2 * math.sqrt(2 / 1e5)


# ---------------------------------------------------------------- O5 statistics

def test_stats_vector_vs_numpy():
    rng = np.random.default_rng(8)
    y = rng.lognormal(0.0, 0.3, 50_001)
    y[[5, 77]] = [np.nan, np.inf]
    ref = rng.normal(size=y.size) * 1e-3 + y
    v = O.stats_vector(y, 1.0, 0.5, 2.0, 64, ref)
    fin = y[np.isfinite(y)]
    assert v[0] == fin.size and v[1] == 2
    mo = O.moments_from_stats(v, 1.0)
    assert abs(mo["mean"] - fin.mean()) < 1e-13
    assert abs(mo["var"] - fin.var()) < 1e-13
    assert abs(mo["skew"] - scipy.stats.skew(fin)) < 1e-10
    assert abs(mo["exkurt"] - scipy.stats.kurtosis(fin)) < 1e-10
    e = fin - ref[np.isfinite(y)]
    assert abs(mo["strong_err"] - np.mean(np.abs(e))) < 1e-15
    h, _ = np.histogram(fin, bins=64, range=(0.5, 2.0))
    np.testing.assert_array_equal(v[9:9 + 64], h)
    assert v[8] == np.count_nonzero(fin < 0.5) and v[9 + 64] == np.count_nonzero(fin >= 2.0)
    assert v[8:].sum() == fin.size


def test_quantiles_hazen():
    rng = np.random.default_rng(9)
    y = rng.normal(size=1001)
    lv = np.array([0.0005, 0.01, 0.25, 0.5, 0.75, 0.99, 0.9995])
    np.testing.assert_allclose(O.quantiles(y, lv), np.quantile(y, lv, method="hazen"), rtol=1e-14, atol=1e-14)


# ------------------------------------------------------- exact CIR collocation

def _ncx2_cdf_mp(x, d, lam):
    """Definition: Poisson(lam/2) mixture of regularised lower incomplete gammas, 30 digits."""
    import mpmath
    mpmath.mp.dps = 30
    x, d, mu = mpmath.mpf(x), mpmath.mpf(d), mpmath.mpf(lam) / 2
    s, i = mpmath.mpf(0), 0
    while True:
        w = mpmath.exp(-mu + i * mpmath.log(mu) - mpmath.loggamma(i + 1)) if mu > 0 else (1 if i == 0 else 0)
        s += w * mpmath.gammainc(d / 2 + i, 0, x / 2, regularized=True)
        i += 1
        if i > mu + 40 * mpmath.sqrt(mu + 1) + 40:
            return s


@pytest.mark.parametrize("Y", [0.1, 0.02, 0.35, 0.0])
def test_cir_exact_points_vs_definition(Y):
    """y_j = c F^{-1}(Phi(x_j)) with F the noncentral chi-square CDF written out as its Poisson mixture
    and inverted at 30 digits (mpmath), independently of scipy's ncx2."""
    import mpmath
    k, ybar, s, dt = 1.0, 0.1, 0.3, 0.125
    c = s * s * (1 - math.exp(-k * dt)) / (4 * k)
    d = 4 * k * ybar / (s * s)
    lam = Y * math.exp(-k * dt) / c
    x = O.gauss_hermite_nodes(7)
    y = O.cir_exact_points(np.array([Y]), dt, k, ybar, s, x)[0]
    for j in (0, 2, 3, 6):
        p = mpmath.ncdf(x[j])
        q = mpmath.findroot(lambda t: _ncx2_cdf_mp(t, d, lam) - p, y[j] / c)
        assert abs(y[j] - c * float(q)) <= 1e-11 * y[j]


def test_cir_exact_points_negative_state_is_zero_state():
    x = O.gauss_hermite_nodes(5)
    a = O.cir_exact_points(np.array([-0.01, 0.0]), 0.25, 1.0, 0.1, 0.3, x)
    np.testing.assert_array_equal(a[0], a[1])
    c = 0.09 * (1 - math.exp(-0.25)) / 4
    np.testing.assert_allclose(a[1], c * scipy.stats.chi2.ppf(scipy.stats.norm.cdf(x), 4 * 0.1 / 0.09), rtol=1e-12)


def test_cir_exact_collocation_paths_match_cir_moments():
    """7L with exact CIR collocation over 4 large steps reproduces the CIR law's closed-form mean and
    variance (E[Y_T] = Ybar + (Y0 - Ybar) e^{-kT}; Var as below) within 4 standard errors."""
    k, ybar, s, y0, T, n, P = 1.0, 0.1, 0.3, 0.3, 1.0, 4, 3000
    spec = O.Spec(7, "cir", (k, ybar, s), y0, T / n, n)
    Y, _ = O.simulate(spec, 9, np.arange(P, dtype=np.uint64))
    YT = Y[-1]
    y0f = float(np.float32(y0))
    e = math.exp(-k * T)
    mean = ybar + (y0f - ybar) * e
    var = y0f * s * s / k * (e - e * e) + ybar * s * s / (2 * k) * (1 - e) ** 2
    assert abs(YT.mean() - mean) < 4 * math.sqrt(var / P)
    assert abs(YT.var() - var) < 4 * var * math.sqrt(2.0 / P) * 1.5


# --------------------------------------------------- multi-step ANN paths against a closed form

def test_multistep_ann_paths_equal_affine_recursion():
    """Multi-step ANN composition pinned to a closed form: with the OU collocation points of Eq. 6.6
    (y_j = a Y + b + s x_j) built into an exactly-affine softplus network, n 7L steps must equal the
    recursion Y <- a32 Y + L(Z) on the same normals, L the Lagrange interpolant of the (fp32-stored)
    intercepts -- to float64 rounding, over 12 steps -- and, the intercepts being affine in x_j up to their
    fp32 rounding, stay within 1e-6 of the exact Eq. 6.6 path."""
    theta, dt, n, m = (0.3, 1.2, 0.4), 0.25, 12, 7
    ybar, lam, sig = theta
    x = O.gauss_hermite_nodes(m)
    a = math.exp(-lam * dt)
    b = ybar * (1 - a)
    s = sig * math.sqrt((1 - math.exp(-2 * lam * dt)) / (2 * lam))
    net = O.parse_blob(pack_blob(affine_softplus_mlp((5, 50, 50, 50, 50, m), a, b + s * x)))
    a32 = float(np.float32(a))
    c32 = (b + s * x).astype(np.float32).astype(np.float64)
    paths = np.arange(2000, dtype=np.uint64)
    Ya, Z = O.simulate(O.Spec(m, "ann", theta, 0.7, dt, n, net=net), 5, paths)
    Y = np.full(len(paths), 0.7)
    for i in range(n):
        Y = a32 * Y + O.lagrange_eval(Z[i], x, np.broadcast_to(c32, (len(paths), m)))
        np.testing.assert_allclose(Ya[i + 1], Y, rtol=0, atol=1e-12)
    R = O.exact_reference("ou", theta, 0.7, dt, Z)
    np.testing.assert_allclose(Ya[-1], R, rtol=0, atol=1e-6)


def test_residual_blob_reproduces_ou_closed_form():
    """Residual output form (blob flags bit 1, reading R-11): H_j = Y + sqrt(dt) * out_j.  An exactly-affine
    softplus network with slope (a - 1)/sqrt(dt) and intercepts (b + s x_j)/sqrt(dt) must give the Eq. 6.6
    OU points a Y + b + s x_j (up to the fp32 storage of those weights), its 7L paths must track the exact
    OU solution on the same normals, and the forward-error scale must include |Y|."""
    theta, dt, n, m = (0.3, 1.2, 0.4), 0.25, 12, 7
    ybar, lam, sig = theta
    x = O.gauss_hermite_nodes(m)
    a = math.exp(-lam * dt)
    b = ybar * (1 - a)
    s = sig * math.sqrt((1 - math.exp(-2 * lam * dt)) / (2 * lam))
    p = affine_softplus_mlp((5, 50, 50, 50, 50, m), (a - 1) / math.sqrt(dt), (b + s * x) / math.sqrt(dt))
    p.residual = True
    blob = pack_blob(p)
    assert struct.unpack_from("<I", blob, 12 + 4 * 6 + 4)[0] == 2          # flags word: residual, no norm
    net = O.parse_blob(blob)
    assert net.residual
    Ys = np.array([-1.5, 0.0, 0.7, 2.0])
    pts = O.ann_collocation(net, Ys, dt, theta)
    np.testing.assert_allclose(pts, a * Ys[:, None] + b + s * x[None, :], rtol=0, atol=2e-7)
    A = O.mlp_abs_scale(net, O.ann_features(Ys, dt, theta))
    assert np.all(A >= np.abs(Ys)[:, None])
    paths = np.arange(2000, dtype=np.uint64)
    Ya, Z = O.simulate(O.Spec(m, "ann", theta, 0.7, dt, n, net=net), 5, paths)
    R = O.exact_reference("ou", theta, 0.7, dt, Z)
    np.testing.assert_allclose(Ya[-1], R, rtol=0, atol=2e-6)
