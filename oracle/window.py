"""Kaiser–Bessel window pair, written from the paper (TEST INFRASTRUCTURE ONLY).

PAPER.md:124-134 defines the D-dimensional window as a tensor product of a 1-D
pair (phi_hat_Base, phi_Base) with

    phi_hat(k) = prod_d phi_hat_Base(Ntilde_d k_d / m)
    phi(n)     = prod_d (m / Ntilde_d) phi_Base(m n_d / Ntilde_d)

and PAPER.md:691 names the Kaiser–Bessel function for phi and "the corresponding
Fourier transform" for phi_hat, without printing the formulas (DESIGN.md
reading R1). We use the standard pair (shape beta = pi m (2 - 1/sigma)):

    phi_hat_Base(u) = sinh(beta sqrt(1-u^2)) / (pi sqrt(1-u^2)),  |u| <= 1
    phi_Base(v)     = I0( sqrt(beta^2 - (2 pi v)^2) )

phi_Base is the inverse Fourier transform of phi_hat_Base restricted to
[-1, 1] (checked by quadrature in tests/test_oracle_window.py — this is what
fixes the normalisation, reading R2: no extra 1/m).
psi_hat_Base is phi_hat_Base truncated to the half-open [-1, 1).
"""

import math

import numpy as np


def kb_beta(m, sigma):
    """Shape parameter beta = pi m (2 - 1/sigma) (reading R1/R4).

    `sigma` is the effective oversampling Ntilde_d / N_d of the dimension.
    """
    return math.pi * m * (2.0 - 1.0 / sigma)


def i0(x):
    """Modified Bessel function I0 by its defining power series.

    I0(x) = sum_{k>=0} ((x/2)^k / k!)^2. All terms are positive, so summing
    until the term is below 1e-17 of the partial sum gives full fp64 accuracy
    for the arguments used here (0 <= x <= pi m (2 - 1/sigma) <= 38).
    """
    x = np.asarray(x, dtype=np.float64)
    q = (x / 2.0) ** 2
    term = np.ones_like(x)
    total = np.ones_like(x)
    for k in range(1, 400):
        term = term * q / (k * k)
        total = total + term
        if np.all(term <= 1e-17 * total):
            break
    return total


def phi_hat_base(u, beta):
    """Un-truncated 1-D frequency window on [-1, 1]; 0 outside (|u| > 1).

    Continuous at |u| = 1 with the limit beta/pi (sinh(x)/x -> 1).
    """
    u = np.asarray(u, dtype=np.float64)
    out = np.zeros_like(u)
    inside = np.abs(u) < 1.0
    s = np.sqrt(1.0 - u[inside] ** 2)
    out[inside] = np.sinh(beta * s) / (math.pi * s)
    out[np.abs(u) == 1.0] = beta / math.pi
    return out


def phi_hat_continued(u, beta):
    """phi_hat_Base continued analytically beyond |u| = 1 (the NFFT3 window the
    paper contrasts with its own: sampled at 2m+2 points "using
    phi_hat instead of psi_hat"): sinh(beta s)/(pi s), s = sqrt(1-u^2), for
    |u| < 1, beta/pi at |u| = 1, and with s = i sqrt(u^2-1) for |u| > 1,
    sin(beta sqrt(u^2-1)) / (pi sqrt(u^2-1))."""
    u = np.asarray(u, dtype=np.float64)
    out = phi_hat_base(u, beta)
    outside = np.abs(u) > 1.0
    s = np.sqrt(u[outside] ** 2 - 1.0)
    out[outside] = np.sin(beta * s) / (math.pi * s)
    return out


def psi_hat_base(u, beta):
    """Truncated window psi_hat_Base: phi_hat_Base on the half-open [-1, 1)
    and 0 elsewhere ("truncated to [-1,1)")."""
    u = np.asarray(u, dtype=np.float64)
    out = phi_hat_base(u, beta)
    out[(u < -1.0) | (u >= 1.0)] = 0.0
    return out


def phi_base(v, beta):
    """Spatial window phi_Base(v) = I0(sqrt(beta^2 - (2 pi v)^2)).

    Only evaluated for |2 pi v| <= beta, which holds for every n in I_N because
    |v| <= m / (2 sigma) (PAPER.md:134 requires phi(n) != 0 on I_N).
    """
    v = np.asarray(v, dtype=np.float64)
    arg = beta * beta - (2.0 * math.pi * v) ** 2
    if np.any(arg < 0):
        raise ValueError("phi_Base evaluated outside |2 pi v| <= beta")
    return i0(np.sqrt(arg))


def phi(n_axes, Ntilde, m, beta):
    """phi(n) = prod_d (m/Ntilde_d) phi_Base(m n_d / Ntilde_d),
    as a dense array over the Cartesian product of the per-axis index vectors
    `n_axes[d]` (first axis slowest, C order)."""
    out = np.ones(tuple(len(n) for n in n_axes), dtype=np.float64)
    D = len(n_axes)
    for d in range(D):
        fac = (m / Ntilde[d]) * phi_base(m * np.asarray(n_axes[d], np.float64) / Ntilde[d], beta[d])
        shape = [1] * D
        shape[d] = len(n_axes[d])
        out = out * fac.reshape(shape)
    return out
