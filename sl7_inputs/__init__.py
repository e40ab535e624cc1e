"""Seeded synthetic inputs shared by the oracle tests, the CUDA-path tests and bench.py.

This module holds NO arithmetic of the Seven-League method (no nodes, no RNG
stream, no collocation, no interpolation).  It only states the workloads of
BASELINE.json ``configs[0..4]`` as plain parameters, draws seeded Glorot
weights ("a Glorot initialization") and packs/unpacks the
``SL7W`` weight-blob container whose layout ``include/sl7.h`` specifies.
Both sides parse the blob with their own code (``oracle/sl7_oracle.py`` in
Python, ``csrc/sl7_host.cpp`` in C++).
"""
from __future__ import annotations

import os
import struct
from dataclasses import dataclass, field

import numpy as np

ACT_TANH = 0
ACT_SOFTPLUS = 1

RUN_SEED_BASE = 2302051700  # run seed = base + config index
WEIGHT_SEED = 17

GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


@dataclass
class Workload:
    """One synthetic workload shaped like BASELINE.json configs[k]."""
    name: str
    process: str            # "gbm" | "ou" | "cir"
    theta: tuple            # GBM (mu, sigma); OU (ybar, lam, sigma); CIR (kappa, ybar, sigma)
    y0: float
    T: float
    n_steps: int
    m: int
    dims: tuple             # [d_in, h1..hL, m]
    act: int
    n_paths: int
    out_mode: str           # "full" | "terminal" | "stats"
    seed: int
    blob: str = ""          # file name under tests/golden (oracle-fitted weights)
    extra: dict = field(default_factory=dict)

    @property
    def dt(self) -> float:
        return self.T / self.n_steps

    @property
    def n_theta(self) -> int:
        return len(self.theta)


GBM_THETA = (0.05, 0.2)
OU_THETA = (0.0, 1.0, 0.5)       # (Ybar, lambda, sigma), Y0 = 1
CIR_THETA = (1.0, 0.1, 0.3)      # (kappa, Ybar, sigma), Y0 = 0.1 (Feller 2*k*Ybar >= sigma^2)


def workloads() -> dict:
    """BASELINE.json configs[0..4] as concrete synthetic workloads."""
    w = {}
    w["cfg0"] = Workload("cfg0_gbm_m5_full", "gbm", GBM_THETA, 1.0, 1.0, 2, 5, (2, 50, 50, 50, 5),
                         ACT_TANH, 10_000, "full", RUN_SEED_BASE + 0, "gbm_m5_tanh3x50.sl7w")
    w["cfg1"] = Workload("cfg1_gbm_m7_sweep", "gbm", GBM_THETA, 1.0, 1.0, 64, 7, (2, 50, 50, 50, 7),
                         ACT_TANH, 10_000_000, "stats", RUN_SEED_BASE + 1, "gbm_m7_tanh3x50.sl7w",
                         extra={"n_sweep": (1, 2, 4, 8, 16, 32, 64)})
    w["cfg2_ou"] = Workload("cfg2_ou_m7_stats", "ou", OU_THETA, 1.0, 2.0, 16, 7, (5, 50, 50, 50, 50, 7),
                            ACT_SOFTPLUS, 100_000_000, "stats", RUN_SEED_BASE + 2, "ou_m7_softplus4x50.sl7w")
    w["cfg2_cir"] = Workload("cfg2_cir_m7_stats", "cir", CIR_THETA, 0.1, 2.0, 16, 7, (5, 50, 50, 50, 50, 7),
                             ACT_SOFTPLUS, 100_000_000, "stats", RUN_SEED_BASE + 2, "cir_m7_softplus4x50.sl7w")
    w["cfg3"] = Workload("cfg3_gbm_m5_full_hbm", "gbm", GBM_THETA, 1.0, 1.0, 64, 5, (2, 50, 50, 50, 5),
                         ACT_TANH, 200_000_000, "full", RUN_SEED_BASE + 3, "gbm_m5_tanh3x50.sl7w")
    w["cfg4"] = Workload("cfg4_cir_m7_scaling", "cir", CIR_THETA, 0.1, 4.0, 32, 7, (5, 50, 50, 50, 50, 7),
                         ACT_SOFTPLUS, 4_000_000_000, "stats", RUN_SEED_BASE + 4, "cir_m7_softplus4x50.sl7w")
    return w


@dataclass
class MlpParams:
    """Plain container: dims, activation, per-layer W[out][in] and b[out], optional affine norm."""
    dims: tuple
    act: int
    W: list
    b: list
    in_shift: np.ndarray | None = None
    in_scale: np.ndarray | None = None
    out_shift: np.ndarray | None = None
    out_scale: np.ndarray | None = None
    residual: bool = False          # blob flags bit 1 (include/sl7.h, 'Weights blob')
    domain: tuple | None = None     # blob flags bit 2: (lo[d_in], hi[d_in]) of the raw features fitted on

    @property
    def has_norm(self) -> bool:
        return self.in_shift is not None


def glorot_mlp(dims, act, seed=WEIGHT_SEED, bias_scale=0.1, with_norm=False, residual=False) -> MlpParams:
    """Seeded Glorot-uniform weights, L = sqrt(6/(fan_in+fan_out)), fp32-representable.

    Biases are small uniform values (not zero) so that every term of the forward pass is exercised.
    """
    rng = np.random.default_rng(seed)
    W, b = [], []
    for l in range(len(dims) - 1):
        fi, fo = dims[l], dims[l + 1]
        L = np.sqrt(6.0 / (fi + fo))
        W.append(rng.uniform(-L, L, size=(fo, fi)).astype(np.float32).astype(np.float64))
        b.append(rng.uniform(-bias_scale, bias_scale, size=fo).astype(np.float32).astype(np.float64))
    p = MlpParams(tuple(dims), act, W, b, residual=residual)
    if with_norm:
        d_in, m = dims[0], dims[-1]
        p.in_shift = rng.uniform(-0.5, 0.5, size=d_in).astype(np.float32).astype(np.float64)
        p.in_scale = rng.uniform(0.5, 2.0, size=d_in).astype(np.float32).astype(np.float64)
        p.out_shift = rng.uniform(-0.5, 0.5, size=m).astype(np.float32).astype(np.float64)
        p.out_scale = rng.uniform(0.5, 2.0, size=m).astype(np.float32).astype(np.float64)
    return p


BLOB_MAGIC = b"SL7W"
BLOB_VERSION = 1


def pack_blob(p: MlpParams) -> bytes:
    """Serialise to the SL7W little-endian container (layout: include/sl7.h, 'Weights blob')."""
    out = bytearray()
    out += BLOB_MAGIC
    out += struct.pack("<II", BLOB_VERSION, len(p.dims))
    out += struct.pack("<%dI" % len(p.dims), *p.dims)
    out += struct.pack("<II", p.act, (1 if p.has_norm else 0) | (2 if p.residual else 0)
                       | (4 if p.domain is not None else 0))
    for W, b in zip(p.W, p.b):
        out += np.asarray(W, dtype="<f4").tobytes()
        out += np.asarray(b, dtype="<f4").tobytes()
    if p.has_norm:
        for a in (p.in_shift, p.in_scale, p.out_shift, p.out_scale):
            out += np.asarray(a, dtype="<f4").tobytes()
    if p.domain is not None:
        for a in p.domain:
            out += np.asarray(a, dtype="<f4").tobytes()
    return bytes(out)


def load_golden_blob(name: str) -> bytes:
    with open(os.path.join(GOLDEN, name), "rb") as f:
        return f.read()


# Training-set feature ranges (SPEC.md:180 for OU; GBM / CIR chosen to cover configs 0-4).  Row layout
# (y_start, dt, theta...) with the SL7 theta order: GBM (mu, sigma), OU (Ybar, lam, sigma),
# CIR (kappa, Ybar, sigma).
FEATURE_RANGES = {
    "gbm": ((0.2, 5.0), (1.0 / 64, 1.0), (0.0, 0.1), (0.1, 0.4)),
    "ou": ((-2.0, 2.0), (0.05, 2.0), (-1.0, 1.0), (0.1, 2.0), (0.1, 1.0)),
    "cir": ((0.01, 0.3), (1.0 / 64, 1.0), (0.5, 2.0), (0.05, 0.2), (0.1, 0.4)),
}


def sample_features(model: str, n_rows: int, seed: int = 0, dt_range=None) -> np.ndarray:
    """Uniform feature rows over FEATURE_RANGES[model], float64 [n_rows][2 + n_theta].
    dt_range overrides the dt column's range (small horizons keep oracle runs short)."""
    rng = np.random.default_rng(seed)
    rg = list(FEATURE_RANGES[model])
    if dt_range is not None:
        rg[1] = dt_range
    return np.stack([rng.uniform(lo, hi, size=n_rows) for lo, hi in rg], axis=1)


def path_ids(n_paths: int, offset: int = 0, stride: int = 1) -> np.ndarray:
    """Global path indices (uint64) of a contiguous or strided subset."""
    return (np.uint64(offset) + np.arange(n_paths, dtype=np.uint64) * np.uint64(stride)).astype(np.uint64)
