"""Euler-Maruyama comparator and offline training-set generation -- plain float64 CPU ORACLE.

TEST INFRASTRUCTURE ONLY (same rules as ``oracle/sl7_oracle.py``): only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may
import this module; the product path never does and shares no code with it.

SURVEY.md §8(f) rows 2 and 3:

  E1  Euler-Maruyama step (Eq. 6.2):
        Y_{k+1} = Y_k + a(Y_k, theta) dtau + b(Y_k, theta) sqrt(dtau) X_{k+1}
      GBM  a = mu Y,             b = sigma Y                  theta = (mu, sigma)
      OU   a = lam (Ybar - Y),   b = sigma                    theta = (Ybar, lam, sigma)
      CIR  a = kappa (Ybar - Y+), b = sigma sqrt(Y+), Y+ = max(Y, 0)   theta = (kappa, Ybar, sigma)
      (reading R-22: "full truncation" for CIR, the paper's plain Eq. 6.2 is undefined for Y < 0).
  E2  EM paths: a large step dt is taken as K equal sub-steps dtau = dt / K; fine step k of path p
      consumes the normal Z_{p,k} of the path generator's RNG (O2: Philox4x32-10 + Box-Muller keyed
      by (seed, p, k)); the path is recorded at the large steps.
  E3  Training set (Algorithm I step 1; "the Euler-Maruyama scheme will be
      used to generate the training data set ... tiny time steps"): per feature row
      r = (y_start, dt, theta): K_r = ceil(dt / dtau) sub-steps of dt / K_r, M inner
      paths with global ids path_offset + r M + q, labels = empirical quantiles of the M terminal
      values at the levels Phi(x_j) (plotting position (k - 0.5)/M, linear interpolation between
      order statistics; reading R-18 / SPEC.md:179, :240).

Pins (tests/test_oracle_em.py): SPEC.md's worked euler_step / euler_path values, deterministic
closed forms at sigma = 0, the closed-form EM moments of GBM and OU (E[Y] and E[Y^2] of the linear
recursions), first-order strong convergence against Eq. 6.6 on the same normals, the sub-step
identity, and the SPEC.md:170 label check against the exact OU collocation points.
"""
from __future__ import annotations

import math

import numpy as np

from .sl7_oracle import gauss_hermite_nodes, normal_cdf, normals, quantiles

MODELS = ("gbm", "ou", "cir")
N_THETA = {"gbm": 2, "ou": 3, "cir": 3}


def drift_diffusion(model: str, theta, Y):
    """a(Y, theta), b(Y, theta) of Eq. 6.1 for the three models (E1)."""
    Y = np.asarray(Y, dtype=np.float64)
    if model == "gbm":
        mu, s = theta
        return mu * Y, s * Y
    if model == "ou":
        ybar, lam, s = theta
        return lam * (ybar - Y), np.full_like(Y, s)
    if model == "cir":
        kappa, ybar, s = theta
        yp = np.maximum(Y, 0.0)
        return kappa * (ybar - yp), s * np.sqrt(yp)
    raise ValueError(model)


def euler_step(model: str, theta, Y, dtau, X):
    """Eq. 6.2: Y + a(Y) dtau + b(Y) sqrt(dtau) X."""
    a, b = drift_diffusion(model, theta, Y)
    return np.asarray(Y, dtype=np.float64) + a * dtau + b * math.sqrt(dtau) * np.asarray(X, dtype=np.float64)


def simulate_em(model: str, theta, y0, dt, n_steps: int, substeps: int, seed: int, paths,
                Z: np.ndarray | None = None) -> np.ndarray:
    """E2: paths[0..n_steps] (rows = large steps) of K = substeps Euler sub-steps per large step.
    Z (optional): the fine normals [n_steps * K][P]; default: the RNG's (seed, path, fine step)."""
    paths = np.asarray(paths, dtype=np.uint64)
    K = int(substeps)
    dtau = dt / K
    if Z is None:
        Z = normals(seed, paths, n_steps * K)
    Y = np.full(len(paths), float(np.float32(y0)))
    out = np.empty((n_steps + 1, len(paths)))
    out[0] = Y
    for i in range(n_steps):
        for k in range(K):
            Y = euler_step(model, theta, Y, dtau, Z[i * K + k])
        out[i + 1] = Y
    return out


def em_substeps(dt: float, dtau: float) -> int:
    """ceil(dt / dtau) equal sub-steps (at least 1)."""
    return max(1, int(math.ceil(dt / dtau)))


def training_set(model: str, features, M: int, dtau: float, seed: int, m: int,
                 path_offset: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """E3: (terminal values [R][M], labels [R][m]) for feature rows (y_start, dt, theta...)."""
    F = np.asarray(features, dtype=np.float64)
    R = F.shape[0]
    levels = normal_cdf(gauss_hermite_nodes(m))
    term = np.empty((R, M))
    lab = np.empty((R, m))
    for r in range(R):
        y0, dt = F[r, 0], F[r, 1]
        theta = tuple(F[r, 2:2 + N_THETA[model]])
        K = em_substeps(dt, dtau)
        paths = np.uint64(path_offset) + np.uint64(r) * np.uint64(M) + np.arange(M, dtype=np.uint64)
        term[r] = simulate_em(model, theta, y0, dt / K, K, 1, seed, paths)[-1]
        lab[r] = quantiles(term[r], levels)
    return term, lab


def em_mean_var_closed_form(model: str, theta, y0, dtau, N):
    """Exact first two moments of the EM recursion after N steps (linear models only):
    GBM Y_{k+1} = Y_k (1 + mu dtau + s sqrt(dtau) X):  E = y0 (1 + mu dtau)^N,
         E[Y^2] = y0^2 ((1 + mu dtau)^2 + s^2 dtau)^N;
    OU  Y_{k+1} = (1 - lam dtau) Y_k + lam Ybar dtau + s sqrt(dtau) X:
         E = Ybar + (y0 - Ybar)(1 - lam dtau)^N,  Var = s^2 dtau sum_{k<N} (1 - lam dtau)^{2k}."""
    if model == "gbm":
        mu, s = theta
        m1 = y0 * (1 + mu * dtau) ** N
        m2 = y0 * y0 * ((1 + mu * dtau) ** 2 + s * s * dtau) ** N
        return m1, m2 - m1 * m1
    if model == "ou":
        ybar, lam, s = theta
        r = 1 - lam * dtau
        mean = ybar + (y0 - ybar) * r ** N
        var = s * s * dtau * sum(r ** (2 * k) for k in range(N))
        return mean, var
    raise ValueError(model)
