"""Pins of oracle/window.py against things other than itself (CPU)."""

import json
import math
import os

import numpy as np
import pytest
import scipy.special

from oracle import window

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_i0_matches_library_routine():
    x = np.concatenate([np.linspace(0, 40, 4001), [1e-8, 0.5, 37.699111843077517]])
    ref = scipy.special.i0(x)
    got = window.i0(x)
    assert np.max(np.abs(got - ref) / ref) < 5e-15


def test_i0_golden_values():
    g = GOLDEN["i0"]
    got = window.i0(np.array(g["x"]))
    np.testing.assert_allclose(got, g["value"], rtol=1e-15, atol=0)  # a few ulp: fp64 summation of the series


def _quad_theta(fn, v, beta, n_nodes=400):
    """int_{-1}^{1} g(u) cos(2 pi v u) du with u = sin(theta), for integrands
    g(u) = fn(beta sqrt(1-u^2)) / (pi sqrt(1-u^2)): becomes
    int_{-pi/2}^{pi/2} fn(beta cos theta)/pi cos(2 pi v sin theta) d theta,
    smooth -> Gauss-Legendre converges exponentially. (Imaginary parts vanish
    by evenness.)"""
    x, w = np.polynomial.legendre.leggauss(n_nodes)
    theta = x * (math.pi / 2)
    vals = fn(beta * np.cos(theta)) / math.pi * np.cos(2 * math.pi * v * np.sin(theta))
    return float(np.sum(w * vals) * (math.pi / 2))


@pytest.mark.parametrize("m", [2, 3, 4, 6, 8])
@pytest.mark.parametrize("sigma", [1.25, 2.0])
def test_window_pair_is_a_fourier_pair(m, sigma):
    """phi is the inverse FT of phi_hat.

    (1) Classical Bessel integral: int_{-pi/2}^{pi/2} cosh(z cos t) cos(w sin t) dt
        = pi I0(sqrt(z^2 - w^2)); this pins phi_Base's argument
        sqrt(beta^2 - (2 pi v)^2) and its normalisation (no 1/m, reading R2).
    (2) The sinh-form phi_hat_Base on [-1,1] differs from that cosh integrand
        by exactly e^{-beta cos t}: its truncated transform must equal
        phi_Base minus that (tiny, ~e^{-beta}) remainder. The remainder is what
        the sin-continuation of phi_hat_Base outside [-1,1] carries; it is
        dropped by the truncation psi_hat.
    """
    beta = window.kb_beta(m, sigma)
    vs = np.linspace(0.0, m / (2 * sigma), 9)   # v = m n / Ntilde, |n| <= N/2
    for v in vs:
        ref = window.phi_base(v, beta)
        assert abs(_quad_theta(np.cosh, v, beta) - ref) / ref < 1e-12  # quadrature cancellation ~ e^(beta - sqrt(beta^2 - w^2)) ulp
        trunc = _quad_theta(np.sinh, v, beta)
        rem = _quad_theta(lambda z: np.exp(-z), v, beta)
        assert abs(trunc + rem - ref) / ref < 1e-12
        assert abs(rem) / window.phi_base(0.0, beta) < 2 * math.exp(-beta) * beta


def test_psi_hat_support_is_half_open():
    """psi_hat_Base is phi_hat_Base truncated to [-1, 1)."""
    beta = window.kb_beta(4, 2.0)
    assert window.psi_hat_base(np.array([-1.0]), beta)[0] == pytest.approx(beta / math.pi, rel=1e-15)
    assert window.psi_hat_base(np.array([1.0]), beta)[0] == 0.0
    assert window.psi_hat_base(np.array([1.5, -1.0000001]), beta).tolist() == [0.0, 0.0]
    assert window.psi_hat_base(np.array([0.0]), beta)[0] == pytest.approx(math.sinh(beta) / math.pi, rel=1e-15)
    u = np.linspace(-0.999, 0.999, 101)
    np.testing.assert_array_equal(window.psi_hat_base(u, beta), window.psi_hat_base(-u, beta))
    # strictly decreasing on [0, 1)
    u = np.linspace(0, 0.999, 200)
    assert np.all(np.diff(window.psi_hat_base(u, beta)) < 0)


def test_psi_hat_continuous_at_boundary():
    beta = window.kb_beta(5, 2.0)
    eps = 1e-9
    near = window.psi_hat_base(np.array([-1 + eps, 1 - eps]), beta)
    np.testing.assert_allclose(near, beta / math.pi, rtol=1e-6)


def test_beta_shape_parameter():
    assert window.kb_beta(4, 2.0) == pytest.approx(math.pi * 4 * 1.5)
    assert window.kb_beta(4, 1.25) == pytest.approx(math.pi * 4 * 1.2)
