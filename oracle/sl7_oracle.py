"""Seven-League (7L) online path generator -- plain float64 CPU ORACLE.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product path (``paper_2302_05170_b200``) never imports it and has
no CPU fallback.  This file shares no code, table or constant generator with
the CUDA library: it re-derives everything from PAPER.md (arXiv 2302.05170)
and the readings listed in DESIGN.md §3.

It computes the method's plain definition step by step, in float64, in the
paper's order (Algorithm I):

  O1  Gauss-Hermite nodes x_j (reading R-1: probabilists')
  O2  normals X_hat ~ N(0,1) from Philox4x32-10 + Box-Muller (reading R-8)
  O3  collocation points y_j | Y_i: ANN H_hat (Eq. 6.4) or exact GBM / OU (Eq. 6.6)
  O4  Y_{i+1} = g_m(X_hat) with g_m the Lagrange interpolant through (x_j, y_j)
      ("g_m ... interpolation"), written as the naive Lagrange sum
  O5  outputs: full path array, terminal values, moments, histogram, quantiles
  O6  quantisation-aware ANN variant (reading R-15) defining the TC-mode result

Pins (tests/test_oracle_*.py, marked "not gpu") tie each part to something
other than itself: closed-form Hermite roots, Random123 known-answer vectors,
mpmath Box-Muller, torch float64 MLP, polynomial reproduction, the GBM and OU
closed forms (Eq. 6.6), numpy statistics; multi-step ANN composition through an exactly-affine
softplus network against the Eq. 6.6 recursion.  Parity unpinned: multi-step paths of a generic
trained network beyond that composition test.
"""
from __future__ import annotations

import struct

import numpy as np

MASK32 = np.uint64(0xFFFFFFFF)

# ----------------------------------------------------------------------------------------------
# O1.  Collocation nodes.  PAPER.md:38 (§Methodology): "x_j are obtained from the standard norm
# distribution X (here Gauss-Hermite quadrature points)".  Reading R-1: probabilists' convention,
# i.e. the roots of He_m, obtained (Golub-Welsch) as the eigenvalues of the symmetric tridiagonal
# Jacobi matrix of the He recurrence  x He_k = He_{k+1} + k He_{k-1}:  zero diagonal,
# off-diagonal sqrt(k), k = 1..m-1.  Library primitive: numpy.linalg.eigvalsh.
# ----------------------------------------------------------------------------------------------


def gauss_hermite_nodes(m: int) -> np.ndarray:
    if m < 1:
        raise ValueError("m must be >= 1")
    J = np.zeros((m, m))
    for k in range(1, m):
        J[k - 1, k] = J[k, k - 1] = np.sqrt(k)
    return np.sort(np.linalg.eigvalsh(J))


def bary_weights(x: np.ndarray) -> np.ndarray:
    """Barycentric weights w_j = 1 / prod_{k != j}(x_j - x_k)  (ref [8] Berrut-Trefethen)."""
    x = np.asarray(x, dtype=np.float64)
    m = len(x)
    w = np.ones(m)
    for j in range(m):
        for k in range(m):
            if k != j:
                w[j] /= (x[j] - x[k])
    return w


# ----------------------------------------------------------------------------------------------
# O4.  Interpolation g_m (Algorithm I steps 5-6).  The plain
# definition of the degree-(m-1) interpolant: g_m(z) = sum_j y_j l_j(z),
# l_j(z) = prod_{k != j} (z - x_k)/(x_j - x_k).  The paper's barycentric form is a
# faster route to the same polynomial; the oracle uses the definition.
# ----------------------------------------------------------------------------------------------


def lagrange_basis(z, x) -> np.ndarray:
    """l_j(z) for every z: shape z.shape + (m,)."""
    z = np.asarray(z, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    m = len(x)
    out = np.ones(z.shape + (m,))
    for j in range(m):
        for k in range(m):
            if k != j:
                out[..., j] *= (z - x[k]) / (x[j] - x[k])
    return out


def lagrange_eval(z, x, y) -> np.ndarray:
    """g_m(z) = sum_j y_j l_j(z); y has shape z.shape + (m,) (per-path points) or (m,)."""
    return np.sum(np.asarray(y, dtype=np.float64) * lagrange_basis(z, x), axis=-1)


# ----------------------------------------------------------------------------------------------
# O2.  Normals.  The paper draws X_hat_{i+1} ~ N(0,1) without naming a
# generator.  Reading R-8 (fixed by BASELINE north_star): counter-based Philox4x32-10 keyed by
# (seed, path, step), Box-Muller, 4 normals per Philox call:
#   key = (seed & 0xffffffff, seed >> 32);  counter = (i >> 2, 0, p & 0xffffffff, p >> 32)
#   u_k = (2*(r_k >> 9) + 1) * 2^-24                       (reading R-9: open (0,1) grid)
#   Z_{4b}   = sqrt(-2 ln u0) cos(2 pi u1),  Z_{4b+1} = sqrt(-2 ln u0) sin(2 pi u1)
#   Z_{4b+2} = sqrt(-2 ln u2) cos(2 pi u3),  Z_{4b+3} = sqrt(-2 ln u2) sin(2 pi u3)
# Philox4x32-10 itself: Salmon et al., SC'11 (Random123): 10 rounds of
#   (hi0,lo0) = mulhilo(M0, c0); (hi1,lo1) = mulhilo(M1, c2)
#   c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0);  key += (W0, W1) between rounds.
# ----------------------------------------------------------------------------------------------

PHILOX_M0 = np.uint64(0xD2511F53)
PHILOX_M1 = np.uint64(0xCD9E8D57)
PHILOX_W0 = np.uint64(0x9E3779B9)
PHILOX_W1 = np.uint64(0xBB67AE85)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 on uint64 arrays holding 32-bit values.  Returns (r0, r1, r2, r3)."""
    c0, c1, c2, c3 = (np.asarray(v, dtype=np.uint64) & MASK32 for v in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint64) & MASK32
    k1 = np.asarray(k1, dtype=np.uint64) & MASK32
    for rnd in range(10):
        if rnd:
            k0 = (k0 + PHILOX_W0) & MASK32
            k1 = (k1 + PHILOX_W1) & MASK32
        p0 = PHILOX_M0 * c0          # < 2^64: exact in uint64
        p1 = PHILOX_M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0), lo1, (hi0 ^ c3 ^ k1), lo0
    return c0, c1, c2, c3


def philox_block(seed: int, paths, block):
    """Raw 4x32-bit outputs for (seed, global path ids, block index b = i >> 2)."""
    paths = np.asarray(paths, dtype=np.uint64)
    block = np.broadcast_to(np.asarray(block, dtype=np.uint64), paths.shape)
    seed = int(seed)
    k0 = np.uint64(seed & 0xFFFFFFFF)
    k1 = np.uint64((seed >> 32) & 0xFFFFFFFF)
    return philox4x32_10(block, np.zeros_like(paths), paths & MASK32, paths >> np.uint64(32), k0, k1)


def u32_to_uniform(r) -> np.ndarray:
    """u = (2*(r >> 9) + 1) * 2^-24 in float64 (exactly representable; never 0 or 1)."""
    r = np.asarray(r, dtype=np.uint64)
    return (2.0 * (r >> np.uint64(9)).astype(np.float64) + 1.0) * 2.0 ** -24


def box_muller(u_a, u_b):
    """(sqrt(-2 ln u_a) cos(2 pi u_b), sqrt(-2 ln u_a) sin(2 pi u_b)) in float64."""
    rad = np.sqrt(-2.0 * np.log(u_a))
    ang = 2.0 * np.pi * u_b
    return rad * np.cos(ang), rad * np.sin(ang)


def normals_block(seed: int, paths, block):
    """The 4 normals Z_{4b..4b+3} of each path for block b."""
    r0, r1, r2, r3 = philox_block(seed, paths, block)
    z0, z1 = box_muller(u32_to_uniform(r0), u32_to_uniform(r1))
    z2, z3 = box_muller(u32_to_uniform(r2), u32_to_uniform(r3))
    return z0, z1, z2, z3


def normals(seed: int, paths, n_steps: int) -> np.ndarray:
    """Z[i, p] = the normal path p consumes at step i (i = 0..n_steps-1)."""
    paths = np.asarray(paths, dtype=np.uint64)
    Z = np.empty((n_steps, len(paths)))
    for b in range((n_steps + 3) // 4):
        zs = normals_block(seed, paths, b)
        for q in range(4):
            i = 4 * b + q
            if i < n_steps:
                Z[i] = zs[q]
    return Z


# ----------------------------------------------------------------------------------------------
# O3.  Conditional collocation points y_j(t_{i+1}) | Y_i = H_j(Y_i, dt, theta)  (Eq. 6.3)
# ----------------------------------------------------------------------------------------------


def gbm_collocation(Y, dt, mu, sigma, x) -> np.ndarray:
    """Exact GBM collocation: y_j = Y exp((mu - sigma^2/2) dt + sigma sqrt(dt) x_j) (BASELINE north_star).

    GBM's conditional law is lognormal, so F^{-1}(Phi(x_j)) (Eq. 6.3) is this closed form."""
    Y = np.asarray(Y, dtype=np.float64)
    c = np.exp((mu - 0.5 * sigma * sigma) * dt + sigma * np.sqrt(dt) * np.asarray(x))
    return Y[..., None] * c


def ou_conditional_moments(y0, dt, ybar, lam, sigma):
    """Eq. 6.6: mean = y0 e^{-lam dt} + ybar (1 - e^{-lam dt}),
    std = sigma sqrt((1 - e^{-2 lam dt}) / (2 lam)).  Reading R-17: when lam*dt < 1e-6
    the variance factor uses its Taylor series dt (1 - lam dt + (2/3)(lam dt)^2)."""
    y0 = np.asarray(y0, dtype=np.float64)
    e = np.exp(-lam * dt)
    mean = y0 * e + ybar * (1.0 - e)
    a = lam * dt
    if a < 1e-6:
        var_f = dt * (1.0 - a + (2.0 / 3.0) * a * a)
    else:
        var_f = (1.0 - np.exp(-2.0 * lam * dt)) / (2.0 * lam)
    return mean, sigma * np.sqrt(var_f)


def ou_collocation(Y, dt, ybar, lam, sigma, x) -> np.ndarray:
    """Exact OU collocation: the conditional law is Gaussian, so y_j = mean + std x_j (Eq. 6.6)."""
    mean, std = ou_conditional_moments(Y, dt, ybar, lam, sigma)
    return mean[..., None] + std * np.asarray(x)


def cir_collocation(Y, dt, kappa, ybar, sigma, x) -> np.ndarray:
    """CIR (square-root) labels for weight fitting only (O7): the conditional law of
    dY = kappa (ybar - Y) dt + sigma sqrt(Y) dW is c * chi'^2(d, lam_nc) with
    c = sigma^2 (1 - e^{-kappa dt}) / (4 kappa), d = 4 kappa ybar / sigma^2,
    lam_nc = Y e^{-kappa dt} / c;  y_j = c * ncx2.ppf(Phi(x_j)).  Library: scipy.stats."""
    from scipy.stats import ncx2, norm
    Y, dt, kappa, ybar, sigma = (a[..., None] for a in np.broadcast_arrays(
        *(np.asarray(v, dtype=np.float64) for v in (Y, dt, kappa, ybar, sigma))))
    c = sigma * sigma * (1.0 - np.exp(-kappa * dt)) / (4.0 * kappa)
    d = 4.0 * kappa * ybar / (sigma * sigma)
    lam_nc = Y * np.exp(-kappa * dt) / c
    q = norm.cdf(np.asarray(x))
    return c * ncx2.ppf(q, d, lam_nc)


def cir_exact_points(Y, dt, kappa, ybar, sigma, x) -> np.ndarray:
    """Exact-collocation CIR: the conditional quantiles of cir_collocation at the
    path's state Y+ = max(Y, 0) (reading R-24: g_m's polynomial extrapolation can leave the state
    slightly negative; the CIR transition from a state <= 0 is the one from 0, a central chi-square)."""
    return cir_collocation(np.maximum(np.asarray(Y, dtype=np.float64), 0.0), dt, kappa, ybar, sigma, x)


# ---- the ANN H_hat (Eq. 6.4; architecture PAPER.md:85) -----------------------

ACT_TANH = 0
ACT_SOFTPLUS = 1


def softplus(z):
    """softplus(z) = ln(1 + e^z), overflow-safe: max(z, 0) + log1p(e^{-|z|})."""
    z = np.asarray(z, dtype=np.float64)
    return np.maximum(z, 0.0) + np.log1p(np.exp(-np.abs(z)))


def activation(z, act):
    return np.tanh(z) if act == ACT_TANH else softplus(z)


class Mlp:
    """One network with m outputs (reading R-4).  W[l] is (out x in), row-major as in the blob."""

    def __init__(self, dims, act, W, b, norm=None, residual=False):
        self.dims = tuple(int(d) for d in dims)
        self.residual = bool(residual)
        self.act = int(act)
        self.W = [np.asarray(w, dtype=np.float64) for w in W]
        self.b = [np.asarray(v, dtype=np.float64) for v in b]
        self.norm = None if norm is None else tuple(np.asarray(a, dtype=np.float64) for a in norm)

    @property
    def m(self):
        return self.dims[-1]


def parse_blob(blob: bytes) -> Mlp:
    """Independent reader of the SL7W container (layout stated in include/sl7.h)."""
    if blob[:4] != b"SL7W":
        raise ValueError("magic")
    ver, nd = struct.unpack_from("<II", blob, 4)
    if ver != 1:
        raise ValueError("version")
    dims = struct.unpack_from("<%dI" % nd, blob, 12)
    off = 12 + 4 * nd
    act, flags = struct.unpack_from("<II", blob, off)
    off += 8
    W, b = [], []
    for l in range(nd - 1):
        fi, fo = dims[l], dims[l + 1]
        W.append(np.frombuffer(blob, dtype="<f4", count=fo * fi, offset=off).astype(np.float64).reshape(fo, fi))
        off += 4 * fo * fi
        b.append(np.frombuffer(blob, dtype="<f4", count=fo, offset=off).astype(np.float64))
        off += 4 * fo
    norm = None
    if flags & 1:
        d_in, m = dims[0], dims[-1]
        arrs = []
        for n in (d_in, d_in, m, m):
            arrs.append(np.frombuffer(blob, dtype="<f4", count=n, offset=off).astype(np.float64))
            off += 4 * n
        norm = tuple(arrs)
    if flags & 4:   # fitted feature box (lo[d_in], hi[d_in]): metadata, not used by the arithmetic
        off += 8 * dims[0]
    if flags & ~7:
        raise ValueError("flags")
    if off != len(blob):
        raise ValueError("size")
    return Mlp(dims, act, W, b, norm, residual=bool(flags & 2))


# O6 rounding of MMA inputs (reading R-15).  bf16: 8 significant bits, round-to-nearest-even;
# TF32: 11 significant bits, round-to-nearest ties-away (cvt.rna).  Exponent range of fp32; our
# operands are far from under/overflow.


def round_bf16(v) -> np.ndarray:
    v = np.asarray(v, dtype=np.float64)
    mant, ex = np.frexp(v)                     # v = mant * 2^ex, 0.5 <= |mant| < 1
    return np.ldexp(np.round(np.ldexp(mant, 8)), ex - 8)   # np.round: half-to-even


def round_tf32(v) -> np.ndarray:
    v = np.asarray(v, dtype=np.float64)
    mant, ex = np.frexp(v)
    q = np.sign(mant) * np.floor(np.abs(np.ldexp(mant, 11)) + 0.5)   # ties away from zero
    return np.ldexp(q, ex - 11)


def mlp_forward(net: Mlp, F, quant: str | None = None) -> np.ndarray:
    """H_hat(F) for feature rows F = (Y, dt, theta...) (Eq. 6.4).  float64.

    quant=None : plain definition (O3).
    quant='bf16'|'tf32' : O6 -- every input of layers 2..L+1 (the contractions the device runs on
    tensor cores: hidden activations and weights) is rounded to the device format before an exact
    product; layer 1 (rank-1 in Y after folding dt, theta) and all biases stay unrounded.
    Residual blobs (flags bit 1, reading R-11): H_hat_j = Y + sqrt(dt) * (out * out_scale + out_shift).
    """
    F = np.asarray(F, dtype=np.float64)
    rnd = {None: (lambda a: a), "bf16": round_bf16, "tf32": round_tf32}[quant]
    h = F
    if net.norm is not None:
        in_shift, in_scale, _, _ = net.norm
        h = (h - in_shift) / in_scale
    L = len(net.W) - 1
    for l in range(L + 1):
        W, b = net.W[l], net.b[l]
        if l == 0:
            z = h @ W.T + b
        else:
            z = rnd(h) @ rnd(W).T + b
        h = z if l == L else activation(z, net.act)
    if net.norm is not None:
        _, _, out_shift, out_scale = net.norm
        h = h * out_scale + out_shift
    if net.residual:
        h = F[..., 0:1] + np.sqrt(F[..., 1:2]) * h
    return h


def mlp_abs_scale(net: Mlp, F, quant: str | None = None) -> np.ndarray:
    """Forward-error scale of each output: A_j = |out_shift_j| + |out_scale_j| (|b_j| + sum_k |W_jk h_k|)
    with h the last hidden layer (the standard bound for a rounded dot product).  Used only to
    scale parity tolerances, not part of the method."""
    F = np.asarray(F, dtype=np.float64)
    rnd = {None: (lambda a: a), "bf16": round_bf16, "tf32": round_tf32}[quant]
    h = F
    if net.norm is not None:
        h = (h - net.norm[0]) / net.norm[1]
    L = len(net.W) - 1
    for l in range(L):
        z = h @ net.W[l].T + net.b[l] if l == 0 else rnd(h) @ rnd(net.W[l]).T + net.b[l]
        h = activation(z, net.act)
    A = np.abs(rnd(h)) @ np.abs(rnd(net.W[L])).T + np.abs(net.b[L])
    if net.norm is not None:
        A = A * np.abs(net.norm[3]) + np.abs(net.norm[2])
    if net.residual:
        A = np.abs(F[..., 0:1]) + np.sqrt(F[..., 1:2]) * A
    return A


def ann_features(Y, dt, theta) -> np.ndarray:
    Y = np.asarray(Y, dtype=np.float64)
    F = np.empty(Y.shape + (2 + len(theta),))
    F[..., 0] = Y
    F[..., 1] = dt
    for c, t in enumerate(theta):
        F[..., 2 + c] = t
    return F


def ann_collocation(net: Mlp, Y, dt, theta, quant=None) -> np.ndarray:
    """y_hat_j(t_{i+1}) | Y_i = H_hat_j(Y_i, dt, theta) (Eq. 6.4); input order (Y, dt, theta...)
    (reading R-10).  No sorting of the predicted points (reading R-6)."""
    return mlp_forward(net, ann_features(Y, dt, theta), quant)


# ----------------------------------------------------------------------------------------------
# Algorithm I (online stage).
# ----------------------------------------------------------------------------------------------


class Spec:
    """What to simulate.  colloc in {'ann', 'gbm', 'ou', 'cir'}; theta in the orders of reading R-10."""

    def __init__(self, m, colloc, theta, y0, dt, n_steps, net=None, quant=None):
        self.m = int(m)
        self.colloc = colloc
        self.theta = tuple(float(t) for t in theta)
        self.y0 = float(y0)
        self.dt = float(dt)
        self.n_steps = int(n_steps)
        self.net = net
        self.quant = quant
        self.x = gauss_hermite_nodes(self.m)

    def points(self, Y) -> np.ndarray:
        """Step 3: the m collocation points of every path at t_{i+1}."""
        if self.colloc == "ann":
            return ann_collocation(self.net, Y, self.dt, self.theta, self.quant)
        if self.colloc == "gbm":
            mu, sigma = self.theta
            return gbm_collocation(Y, self.dt, mu, sigma, self.x)
        if self.colloc == "ou":
            ybar, lam, sigma = self.theta
            return ou_collocation(Y, self.dt, ybar, lam, sigma, self.x)
        if self.colloc == "cir":
            kappa, ybar, sigma = self.theta
            return cir_exact_points(Y, self.dt, kappa, ybar, sigma, self.x)
        raise ValueError(self.colloc)


def step_error_scale(spec: Spec, Y, Z) -> np.ndarray:
    """kappa = sum_j |l_j(Z)| A_j(Y): forward-error scale of one step; A_j = |y_j|
    in the exact modes, mlp_abs_scale in ANN mode.  kappa >= |Y_{i+1}|.  Tolerance helper only."""
    if spec.colloc == "ann":
        A = mlp_abs_scale(spec.net, ann_features(Y, spec.dt, spec.theta), spec.quant)
    elif spec.colloc == "ou":
        # y_j = Y e + Ybar (1 - e) + std x_j: the scale of each term, not of their (cancelling) sum
        ybar, lam, sigma = spec.theta
        e = np.exp(-lam * spec.dt)
        _, std = ou_conditional_moments(Y, spec.dt, ybar, lam, sigma)
        A = (np.abs(np.asarray(Y) * e) + abs(ybar * (1 - e)))[..., None] + np.abs(std * spec.x)
    else:
        A = np.abs(spec.points(Y))
    return np.sum(np.abs(lagrange_basis(Z, spec.x)) * A, axis=-1)


def step(spec: Spec, Y, Z) -> np.ndarray:
    """One 7L step for every path: steps 3, 5, 6 of Algorithm I: Y_{i+1} = g_m(X_hat) through
    (x_j, y_hat_j(Y_i))."""
    return lagrange_eval(Z, spec.x, spec.points(Y))


def simulate(spec: Spec, seed: int, paths) -> tuple[np.ndarray, np.ndarray]:
    """Steps 2-8: full path array Yfull[i, p] (row 0 = Y0) and the normals Z[i, p] consumed."""
    paths = np.asarray(paths, dtype=np.uint64)
    Z = normals(seed, paths, spec.n_steps)
    Y = np.empty((spec.n_steps + 1, len(paths)))
    Y[0] = spec.y0
    for i in range(spec.n_steps):
        Y[i + 1] = step(spec, Y[i], Z[i])
    return Y, Z


# ----------------------------------------------------------------------------------------------
# 7L-CDC ("a variant, the 7L-CDC scheme ... with more interpolations in Step 3";
# PAPER.md:106-108 "a global interpolation technique which is based on the marginal collocation
# points to compute the conditional collocation points for each random path ... only requires the
# ANNs to compute a small number of marginal collocation points").  Readings R-18..R-20:
# per step, the m marginal collocation points z_k are the empirical quantiles of the current states
# of ALL paths at the levels Phi(x_k) (plotting position (k - 0.5)/M, linear interpolation); the table
# row C[k] = H(z_k) is one predictor call per marginal point; each path's conditional points are the
# Lagrange interpolant of k -> C[k][j] on the nodes z_k evaluated at its own state; repeated z_k
# (e.g. step 0, all paths at Y0) fall back to the nearest row (ties: lowest k).  No sorting (R-6).
# ----------------------------------------------------------------------------------------------


def normal_cdf(x) -> np.ndarray:
    """Phi(x) = erfc(-x / sqrt 2) / 2 (library: scipy.special.erfc)."""
    from scipy.special import erfc
    return 0.5 * erfc(-np.asarray(x, dtype=np.float64) / np.sqrt(2.0))


def cdc_table(spec: Spec, Y):
    """Marginal collocation points z (m,) of the current states Y (all paths) and the table C (m, m)."""
    z = quantiles(Y, normal_cdf(spec.x))
    return z, spec.points(z)


def cdc_points(z, C, Y) -> np.ndarray:
    """Conditional collocation points of every path: (P, m)."""
    Y = np.asarray(Y, dtype=np.float64)
    if np.any(np.diff(z) <= 0):
        k = np.argmin(np.abs(Y[:, None] - z[None, :]), axis=1)     # first minimum = lowest k
        return C[k]
    return lagrange_basis(Y, z) @ C


def simulate_cdc(spec: Spec, seed: int, paths) -> tuple[np.ndarray, np.ndarray]:
    """7L-CDC over the FULL path set `paths` (the marginal points couple all paths)."""
    paths = np.asarray(paths, dtype=np.uint64)
    Z = normals(seed, paths, spec.n_steps)
    Y = np.empty((spec.n_steps + 1, len(paths)))
    Y[0] = spec.y0
    for i in range(spec.n_steps):
        Y[i + 1] = cdc_step(spec, Y[i], Z[i])
    return Y, Z


def cdc_step_error_scale(spec: Spec, Y, Z) -> np.ndarray:
    """Forward-error scale of one CDC step (tolerance helper, not part of the method): the outer
    interpolation's sum_j |l_j(Z)| A_j with A_j = sum_k |l_k(Y; z)| S_kj, S the size of the terms of
    the table entries (as in step_error_scale)."""
    Y = np.asarray(Y, dtype=np.float64)
    z, C = cdc_table(spec, Y)
    return _cdc_error_scale(spec, z, C, Y, Z)


def _cdc_error_scale(spec: Spec, z, C, Y, Z) -> np.ndarray:
    Y = np.asarray(Y, dtype=np.float64)
    if spec.colloc == "ann":
        S = mlp_abs_scale(spec.net, ann_features(z, spec.dt, spec.theta), spec.quant)
    elif spec.colloc == "ou":
        ybar, lam, sigma = spec.theta
        e = np.exp(-lam * spec.dt)
        _, std = ou_conditional_moments(z, spec.dt, ybar, lam, sigma)
        S = (np.abs(z * e) + abs(ybar * (1 - e)))[:, None] + np.abs(std * spec.x)
    else:
        S = np.abs(C)
    if np.any(np.diff(z) <= 0):
        A = S[np.argmin(np.abs(Y[:, None] - z[None, :]), axis=1)]
    else:
        A = np.abs(lagrange_basis(Y, z)) @ S
    return np.sum(np.abs(lagrange_basis(Z, spec.x)) * A, axis=-1)


def cdc_step(spec: Spec, Y, Z) -> np.ndarray:
    """One CDC step of every path from the states Y (all paths) with normals Z."""
    z, C = cdc_table(spec, Y)
    return lagrange_eval(Z, spec.x, cdc_points(z, C, Y))


# 7L-CDC with predicted marginal points (SL7_SCHEME_CDC_PRED, reading R-26 of DESIGN.md): PAPER.md:106
# "only requires the ANNs to compute a small number of marginal collocation points" read literally --
# the marginal collocation points of Y(t_i) are the predictor's own at (Y0, horizon t_i = i dt, theta);
# the table and the per-path interpolation are those of cdc_step, at the path's state clamped to the
# marginal hull [z_0, z_{m-1}].  At t_0 every path is at Y0 (the repeated-point rule R-20 gives row 0).
# The paths are independent: any subset can be simulated alone.


def cdc_pred_marginals(spec: Spec, i: int) -> np.ndarray:
    """Marginal collocation points z (m,) of Y(t_i) given Y(0) = y0."""
    if i == 0:
        return np.full(spec.m, spec.y0)
    horizon = Spec(spec.m, spec.colloc, spec.theta, spec.y0, i * spec.dt, spec.n_steps, spec.net, spec.quant)
    return horizon.points(np.array([spec.y0]))[0]


def cdc_pred_state(z, Y) -> np.ndarray:
    """The state at which a path reads the table: clamped to the marginal hull [z_0, z_{m-1}] (R-26: the
    table is extended flat beyond its extreme rows instead of by the degree-(m-1) polynomial); NaN stays
    NaN.  Repeated or unordered z (nearest-row rule R-20): the state as it is."""
    Y = np.asarray(Y, dtype=np.float64)
    return np.clip(Y, z[0], z[-1]) if np.all(np.diff(z) > 0) else Y


def cdc_pred_step(spec: Spec, i: int, Y, Z) -> np.ndarray:
    """Step i of every path: table C[k] = H(z_k, dt, theta) on the predicted marginal points."""
    z = cdc_pred_marginals(spec, i)
    return lagrange_eval(Z, spec.x, cdc_points(z, spec.points(z), cdc_pred_state(z, Y)))


def simulate_cdc_pred(spec: Spec, seed: int, paths) -> tuple[np.ndarray, np.ndarray]:
    """7L-CDC with predicted marginal points over the paths `paths` (global ids)."""
    paths = np.asarray(paths, dtype=np.uint64)
    Z = normals(seed, paths, spec.n_steps)
    Y = np.empty((spec.n_steps + 1, len(paths)))
    Y[0] = spec.y0
    for i in range(spec.n_steps):
        Y[i + 1] = cdc_pred_step(spec, i, Y[i], Z[i])
    return Y, Z


def cdc_pred_clamped(spec: Spec, Y) -> int:
    """Number of path-steps whose state lies outside the marginal hull [z_0, z_{m-1}] of its step and is
    clamped by cdc_pred_state (steps with repeated or unordered z use the nearest row: no clamp).  Y is the
    (n_steps + 1, P) state array of simulate_cdc_pred; NaN states are not counted."""
    n = 0
    for i in range(spec.n_steps):
        z = cdc_pred_marginals(spec, i)
        if np.all(np.diff(z) > 0):
            n += int(np.count_nonzero((Y[i] < z[0]) | (Y[i] > z[-1])))
    return n


def cdc_pred_step_error_scale(spec: Spec, i: int, Y, Z) -> np.ndarray:
    """Forward-error scale of cdc_pred_step (tolerance helper): as cdc_step_error_scale on z_i."""
    z = cdc_pred_marginals(spec, i)
    return _cdc_error_scale(spec, z, spec.points(z), cdc_pred_state(z, Y), Z)


def exact_reference(process: str, theta, y0, dt, Z) -> np.ndarray:
    """Exact solution on the same normals (Eq. 6.6 'used to compute the reference
    value to the path-wise error').  GBM: Y_T = Y0 exp((mu - s^2/2) T + s sqrt(dt) sum_i Z_i);
    OU: the exact Eq. 6.6 transition applied step by step with the same Z_i.  Returns Y_T."""
    n = Z.shape[0]
    if process == "gbm":
        mu, s = theta
        return y0 * np.exp((mu - 0.5 * s * s) * n * dt + s * np.sqrt(dt) * Z.sum(axis=0))
    if process == "ou":
        ybar, lam, s = theta
        R = np.full(Z.shape[1], float(y0))
        for i in range(n):
            mean, std = ou_conditional_moments(R, dt, ybar, lam, s)
            R = mean + std * Z[i]
        return R
    raise ValueError(process)


# ----------------------------------------------------------------------------------------------
# O5.  Statistics of the terminal values (Algorithm I step 7 "collect"), reading R-12.
# Vector layout (an interface, include/sl7.h): [n, n_nonfinite, S1, S2, S3, S4, E1, E2,
# hist_under, hist_0..hist_{B-1}, hist_over] with S_k = sum (Y - shift)^k over finite Y,
# E1 = sum |Y - R|, E2 = sum (Y - R)^2 against a reference R (0 if none).
# ----------------------------------------------------------------------------------------------

STATS_HEAD = 8


def stats_vector(YT, shift, lo, hi, n_bins, ref=None) -> np.ndarray:
    YT = np.asarray(YT, dtype=np.float64)
    fin = np.isfinite(YT)
    y = YT[fin]
    d = y - shift
    v = np.zeros(STATS_HEAD + n_bins + 2)
    v[0] = len(y)
    v[1] = np.count_nonzero(~fin)
    v[2:6] = [np.sum(d), np.sum(d ** 2), np.sum(d ** 3), np.sum(d ** 4)]
    if ref is not None:
        e = y - np.asarray(ref, dtype=np.float64)[fin]
        v[6] = np.sum(np.abs(e))
        v[7] = np.sum(e * e)
    w = (hi - lo) / n_bins
    under = y < lo
    over = y >= hi
    mid = ~(under | over)
    k = np.floor((y[mid] - lo) / w).astype(np.int64)
    k = np.clip(k, 0, n_bins - 1)
    v[STATS_HEAD] = np.count_nonzero(under)
    v[STATS_HEAD + 1:STATS_HEAD + 1 + n_bins] = np.bincount(k, minlength=n_bins)
    v[STATS_HEAD + n_bins + 1] = np.count_nonzero(over)
    return v


def moments_from_stats(v, shift) -> dict:
    """mean, population variance (reading R-12), skewness, excess kurtosis from shifted sums."""
    n = v[0]
    a1, a2, a3, a4 = v[2] / n, v[3] / n, v[4] / n, v[5] / n
    var = a2 - a1 * a1
    m3 = a3 - 3 * a1 * a2 + 2 * a1 ** 3
    m4 = a4 - 4 * a1 * a3 + 6 * a1 * a1 * a2 - 3 * a1 ** 4
    return {"n": n, "mean": shift + a1, "var": var, "skew": m3 / var ** 1.5 if var > 0 else 0.0,
            "exkurt": m4 / var ** 2 - 3.0 if var > 0 else 0.0,
            "strong_err": v[6] / n, "rms_err": np.sqrt(v[7] / n)}


def quantiles(YT, levels) -> np.ndarray:
    """Exact order-statistic quantiles with plotting positions (k - 0.5)/M, linear interpolation
    between order statistics, clamped to the extreme order statistics."""
    y = np.sort(np.asarray(YT, dtype=np.float64)[np.isfinite(YT)])
    M = len(y)
    pos = np.asarray(levels, dtype=np.float64) * M + 0.5     # 1-based fractional rank
    pos = np.clip(pos, 1.0, float(M))
    k = np.floor(pos).astype(np.int64)
    f = pos - k
    k0 = k - 1
    k1 = np.minimum(k, M - 1)
    return y[k0] * (1 - f) + y[k1] * f
