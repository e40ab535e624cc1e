"""Fit the MLP weights H_hat (Eq. 6.4) to analytic collocation labels -- oracle side (O7).

TEST INFRASTRUCTURE ONLY.  No trained checkpoint exists offline (BASELINE north_star), so this
committed script produces the frozen weight blobs under tests/golden/ that BOTH the oracle and the
CUDA path consume as inputs.  Labels come only from oracle/sl7_oracle.py (GBM closed form, Eq. 6.6
for OU, the noncentral-chi^2 law for CIR); the optimiser follows PAPER.md:85 ("Glorot
initialization, the Adam optimizer, a batch size of 1024, and a learning rate of 10^-3", annealed to
1e-6 over the time budget) with input/output standardisation stored in the blob and, by default, the residual output form
H_hat_j = Y + sqrt(dt) (out_j out_scale_j + out_shift_j) (blob flags bit 1, reading R-11).  Fit quality is REPORTED in
tests/golden/weights_manifest.json, never graded: the kernels are checked against the oracle
running the *same* frozen weights.

usage: python -m oracle.fit_weights [--seconds S] [--only NAME] [--device cuda] [--absolute] [--out-dir D]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import sl7_oracle as O  # noqa: E402
from sl7_inputs import ACT_SOFTPLUS, ACT_TANH, GOLDEN, MlpParams, WEIGHT_SEED, pack_blob  # noqa: E402


def _sample(rng, n, ranges, log_cols=()):
    cols = []
    for c, (lo, hi) in enumerate(ranges):
        if c in log_cols:
            cols.append(np.exp(rng.uniform(np.log(lo), np.log(hi), n)))
        else:
            cols.append(rng.uniform(lo, hi, n))
    return np.stack(cols, axis=1)


# Raw-feature box each network is fitted on, (lo, hi) per column, and the columns sampled log-uniformly.
# The box is stored in the blob (flags bit 2) so that the library can refuse to read the predictor outside
# it (CDC_PRED horizons, include/sl7.h).  CIR: dt up to 4 = configs[4]'s T, so that the 7L-CDC predictor
# (reading R-26) can be read at every horizon t_i < T of configs 2 and 4.
RANGES = {
    "gbm": ([(0.2, 5.0), (1 / 64, 1.0)], (0, 1)),
    # SPEC.md:180 default OU training ranges; features (Y, dt, Ybar, lam, sigma)
    "ou": ([(-2, 2), (0.05, 2.0), (-1, 1), (0.1, 2.0), (0.1, 1.0)], ()),
    # features (Y, dt, kappa, Ybar, sigma)
    "cir": ([(0.002, 0.5), (0.05, 4.0), (0.5, 2.0), (0.05, 0.2), (0.15, 0.45)], (0, 1)),
}


def make_dataset(kind, m, n, seed):
    rng = np.random.default_rng(seed)
    x = O.gauss_hermite_nodes(m)
    ranges, log_cols = RANGES[kind]
    F = _sample(rng, n, ranges, log_cols=log_cols)
    if kind == "gbm":
        mu, sigma = 0.05, 0.2
        Yl = np.stack([O.gbm_collocation(F[i:i + 1, 0], F[i, 1], mu, sigma, x)[0] for i in range(n)], 0)
        return F, Yl
    if kind == "ou":
        Yl = np.stack([O.ou_collocation(F[i:i + 1, 0], F[i, 1], F[i, 2], F[i, 3], F[i, 4], x)[0]
                       for i in range(n)], 0)
        return F, Yl
    if kind == "cir":
        Yl = O.cir_collocation(F[:, 0], F[:, 1], F[:, 2], F[:, 3], F[:, 4], x)
        return F, Yl
    raise ValueError(kind)


def domain_of(kind):
    ranges, _ = RANGES[kind]
    return (np.array([lo for lo, _ in ranges], dtype=np.float64), np.array([hi for _, hi in ranges], dtype=np.float64))


def fit(kind, m, act, hidden, seconds, seed=WEIGHT_SEED, n=200_000, device="cpu", residual=True):
    import math
    import torch
    torch.manual_seed(seed)
    torch.set_num_threads(max(1, os.cpu_count() or 1))
    F, Yl = make_dataset(kind, m, n, seed)
    # residual blobs (reading R-11) learn (y_j - Y) / sqrt(dt): the network then carries only the
    # step's spread, whose size no longer depends on Y or dt, instead of re-deriving Y through its layers
    T = (Yl - F[:, :1]) / np.sqrt(F[:, 1:2]) if residual else Yl
    in_shift, in_scale = F.mean(0), F.std(0) + 1e-12
    out_shift, out_scale = T.mean(0), T.std(0) + 1e-12
    Xn = torch.tensor((F - in_shift) / in_scale, dtype=torch.float32, device=device)
    Yn = torch.tensor((T - out_shift) / out_scale, dtype=torch.float32, device=device)
    nval = n // 10
    Xv, Yv, Xt, Yt = Xn[:nval], Yn[:nval], Xn[nval:], Yn[nval:]
    dims = [F.shape[1]] + [50] * hidden + [m]
    layers = []
    for l in range(len(dims) - 1):
        lin = torch.nn.Linear(dims[l], dims[l + 1])
        torch.nn.init.xavier_uniform_(lin.weight)   # Glorot
        torch.nn.init.zeros_(lin.bias)
        layers.append(lin)
        if l < len(dims) - 2:
            layers.append(torch.nn.Tanh() if act == ACT_TANH else torch.nn.Softplus())
    net = torch.nn.Sequential(*layers).to(device)
    # Adam, batch 1024, lr 1e-3, then annealed (cosine, in wall time) to 1e-6: the 7L step
    # error of a network is its collocation-point error, and small-dt steps accumulate it over many steps
    opt = torch.optim.Adam(net.parameters(), lr=1e-3)
    best, best_state, epoch = float("inf"), None, 0
    t0 = time.time()
    while time.time() - t0 < seconds:
        frac = min(1.0, (time.time() - t0) / seconds)
        for gr in opt.param_groups:
            gr["lr"] = 1e-6 + 0.5 * (1e-3 - 1e-6) * (1.0 + math.cos(math.pi * frac))
        perm = torch.randperm(Xt.shape[0], device=device)
        for s in range(0, Xt.shape[0], 1024):
            idx = perm[s:s + 1024]
            opt.zero_grad()
            loss = torch.mean((net(Xt[idx]) - Yt[idx]) ** 2)
            loss.backward()
            opt.step()
        epoch += 1
        with torch.no_grad():
            v = torch.mean((net(Xv) - Yv) ** 2).item()
        if v < best:
            best = v
            best_state = {k: t.clone() for k, t in net.state_dict().items()}
    net.load_state_dict(best_state)
    lins = [l for l in net if isinstance(l, torch.nn.Linear)]
    W = [l.weight.detach().double().cpu().numpy().astype(np.float32).astype(np.float64) for l in lins]
    b = [l.bias.detach().double().cpu().numpy().astype(np.float32).astype(np.float64) for l in lins]
    f32 = lambda a: np.asarray(a).astype(np.float32).astype(np.float64)
    p = MlpParams(tuple(dims), act, W, b, f32(in_shift), f32(in_scale), f32(out_shift), f32(out_scale),
                  residual=residual, domain=domain_of(kind))
    # report fit quality with the oracle's own forward pass on the held-out rows
    blob = pack_blob(p)
    onet = O.parse_blob(blob)
    pred = O.mlp_forward(onet, F[:nval])
    scale = np.maximum(np.abs(Yl[:nval]), np.std(Yl[:nval], axis=0))
    rel = np.abs(pred - Yl[:nval]) / scale
    quality = {"epochs": epoch, "val_mse_normalised": best, "median_rel_err": float(np.median(rel)),
               "p99_rel_err": float(np.quantile(rel, 0.99)), "max_rel_err": float(rel.max())}
    return blob, quality


NETS = {
    "gbm_m5_tanh3x50.sl7w": ("gbm", 5, ACT_TANH, 3),
    "gbm_m7_tanh3x50.sl7w": ("gbm", 7, ACT_TANH, 3),
    "ou_m7_softplus4x50.sl7w": ("ou", 7, ACT_SOFTPLUS, 4),
    "cir_m7_softplus4x50.sl7w": ("cir", 7, ACT_SOFTPLUS, 4),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=120.0)
    ap.add_argument("--only", default=None)
    ap.add_argument("--device", default="cpu", help="torch device for the optimiser (labels are the oracle's)")
    ap.add_argument("--absolute", action="store_true", help="absolute-output blobs (no residual form)")
    ap.add_argument("--out-dir", default=GOLDEN)
    ap.add_argument("--stamp-domain", action="store_true",
                    help="re-pack the existing blobs with their recipe's feature box (flags bit 2), weights unchanged")
    a = ap.parse_args()
    man_path = os.path.join(a.out_dir, "weights_manifest.json")
    manifest = json.load(open(man_path)) if os.path.exists(man_path) else {}
    for name, (kind, m, act, hidden) in NETS.items():
        if a.only and a.only != name:
            continue
        if a.stamp_domain:
            path = os.path.join(a.out_dir, name)
            net = O.parse_blob(open(path, "rb").read())
            p = MlpParams(net.dims, net.act, net.W, net.b, *net.norm, residual=net.residual, domain=domain_of(kind))
            blob = pack_blob(p)
            assert O.parse_blob(blob).W[0].tobytes() == net.W[0].tobytes()
            open(path, "wb").write(blob)
            e = manifest[name]
            e["sha256"] = hashlib.sha256(blob).hexdigest()
            e["domain"] = [list(map(float, d)) for d in domain_of(kind)]
            e["script"] += " ; python -m oracle.fit_weights --stamp-domain --only %s" % name
            print(name, "stamped", e["domain"], flush=True)
            json.dump(manifest, open(man_path, "w"), indent=1, sort_keys=True)
            continue
        n = 120_000 if kind == "cir" else 200_000
        blob, q = fit(kind, m, act, hidden, a.seconds, n=n, device=a.device, residual=not a.absolute)
        with open(os.path.join(a.out_dir, name), "wb") as f:
            f.write(blob)
        manifest[name] = {"process": kind, "m": m, "act": "tanh" if act == ACT_TANH else "softplus",
                          "hidden": hidden, "sha256": hashlib.sha256(blob).hexdigest(),
                          "fit_seconds": a.seconds, "seed": WEIGHT_SEED, "quality": q, "device": a.device,
                          "residual": not a.absolute,
                          "domain": [list(map(float, d)) for d in domain_of(kind)],
                          "script": "python -m oracle.fit_weights --seconds %g --device %s%s" % (
                              a.seconds, a.device, " --absolute" if a.absolute else "")}
        print(name, q, flush=True)
        json.dump(manifest, open(man_path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
