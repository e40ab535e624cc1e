"""Test-only constructions shared by the CPU pins and the GPU tests (not part of the product or the oracle)."""
import numpy as np

from sl7_inputs import ACT_SOFTPLUS, MlpParams


def affine_softplus_mlp(dims, slope, intercepts):
    """A softplus MLP whose output is exactly y_j = slope * Y + intercepts[j]: softplus(z) - softplus(-z) = z,
    so hidden units 0 and 1 carry softplus(+Y) and softplus(-Y) through every layer (weights +-1) and all
    other units are dead (zero outgoing weights)."""
    W, bs = [], []
    for l in range(len(dims) - 1):
        fi, fo = dims[l], dims[l + 1]
        w, bb = np.zeros((fo, fi)), np.zeros(fo)
        if l == 0:
            w[0, 0], w[1, 0] = 1.0, -1.0
        elif l < len(dims) - 2:
            w[0, 0], w[0, 1], w[1, 0], w[1, 1] = 1.0, -1.0, -1.0, 1.0
        else:
            w[:, 0], w[:, 1] = slope, -slope
            bb = np.asarray(intercepts, dtype=np.float64)
        W.append(w)
        bs.append(bb)
    return MlpParams(tuple(dims), ACT_SOFTPLUS, W, bs)
