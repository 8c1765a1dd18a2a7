"""Seeded synthetic inputs shared by the tests, bench.py and smoke().

This module holds NONE of the method's arithmetic: it only draws nodes and
coefficients. Both the CUDA path and the CPU oracle receive the arrays it
returns. Recipes re-instantiate the paper's workload
(J = |I_N| i.i.d. uniform nodes in [-1/2,1/2)^D, sigma = 2) and
BASELINE.json configs[0..4].

Draw order with numpy.random.default_rng(seed): nodes, then the N-grid
coefficients, then the M node values. "Complex standard normal" means
re, im i.i.d. N(0, 1/2) (unit complex variance; reading R14).
"""

import math

import numpy as np

# BASELINE.json configs, in order. D, N, M, precision, sigma, m (default),
# batch, node structure.
CONFIGS = {
    "cfg1_1d_256": dict(N=(256,), M=256, precision="c128", sigma=2.0, m=4, batch=1, structure="uniform"),
    "cfg2_1d_2e18": dict(N=(262144,), M=262144, precision="c128", sigma=2.0, m=4, batch=1, structure="uniform"),
    "cfg3_2d_512": dict(N=(512, 512), M=262144, precision="c128", sigma=2.0, m=4, batch=1, structure="uniform"),
    "cfg4_3d_64": dict(N=(64, 64, 64), M=262144, precision="c128", sigma=2.0, m=4, batch=1, structure="uniform"),
    "cfg5_radial_s2": dict(N=(256, 256), M=402 * 512, precision="c64", sigma=2.0, m=4, batch=32, structure="radial"),
    "cfg5_radial_s125": dict(N=(256, 256), M=402 * 512, precision="c64", sigma=1.25, m=4, batch=32, structure="radial"),
}

# Diametric-spoke golden angle pi (sqrt(5) - 1) / 2 (reading R16).
GOLDEN_ANGLE = math.pi * (math.sqrt(5.0) - 1.0) / 2.0


def complex_normal(rng, shape, dtype=np.complex128):
    z = (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / math.sqrt(2.0)
    return z.astype(dtype)


def uniform_nodes(rng, M, D, dtype=np.float64):
    return (rng.random((M, D)) - 0.5).astype(dtype)


def radial_nodes(n_spokes=402, n_samples=512, dtype=np.float32):
    """Golden-angle radial trajectory (reading R16/R17): spoke i at angle
    i * GOLDEN_ANGLE, radii r_s = -1/2 + s / n_samples, spoke-major order;
    computed in fp64 then rounded to `dtype`. r = 0 gives n_spokes coincident
    nodes at the origin."""
    theta = np.arange(n_spokes, dtype=np.float64) * GOLDEN_ANGLE
    r = -0.5 + np.arange(n_samples, dtype=np.float64) / n_samples
    kx = np.cos(theta)[:, None] * r[None, :]
    ky = np.sin(theta)[:, None] * r[None, :]
    return np.stack([kx.reshape(-1), ky.reshape(-1)], axis=1).astype(dtype)


def make(config, seed=0, m=None, batch=None, M=None, N=None):
    """Returns dict(nodes, fhat, f, N, M, m, sigma, precision, batch).

    fhat has shape (batch, *N), f has shape (batch, M); both complex
    (complex64 for c64 configs). Overrides allow scaled-down variants.
    """
    cfg = dict(CONFIGS[config])
    if m is not None:
        cfg["m"] = m
    if batch is not None:
        cfg["batch"] = batch
    if N is not None:
        cfg["N"] = tuple(N)
    if M is not None:
        cfg["M"] = M
    D = len(cfg["N"])
    rdt = np.float64 if cfg["precision"] == "c128" else np.float32
    cdt = np.complex128 if cfg["precision"] == "c128" else np.complex64
    rng = np.random.default_rng(seed)
    if cfg["structure"] == "uniform":
        nodes = uniform_nodes(rng, cfg["M"], D, rdt)
    else:
        nodes = radial_nodes(dtype=rdt)
        if M is not None:
            nodes = nodes[: cfg["M"]]
        cfg["M"] = nodes.shape[0]
    fhat = complex_normal(rng, (cfg["batch"],) + tuple(cfg["N"]), cdt)
    f = complex_normal(rng, (cfg["batch"], cfg["M"]), cdt)
    return dict(nodes=nodes, fhat=fhat, f=f, **cfg)
