"""Plain fp64 NFFT: Alg. 1 (direct) and Alg. 2 (adjoint) of PAPER.md, step by
step (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Conventions:
* N-grid arrays are C-contiguous with shape (N_0, ..., N_{D-1}); storage index
  i_d <-> logical n_d = i_d - N_d/2, n_d in [-N_d/2, N_d/2).
* Node coordinate d pairs with grid axis d; nodes are an (M, D) array.
* Oversampled-grid arrays (shape Ntilde) hold the value of logical index
  l in I_Ntilde at storage position (l mod Ntilde_d)_d. This is the periodic
  identification the paper performs with an fftshift; with it
  the grid DFT of PAPER.md:209 is exactly numpy's unnormalised fftn.
* Node footprint (reading R5 "floor form"): with t = Ntilde k and
  a = floor(t), I_{Ntilde,m}(k) = {a-m+1, ..., a+m}, i.e. all l with
  -m <= t - l < m, the half-open support of psi_hat.
"""

import itertools
import math

import numpy as np

from . import window


def geometry(N, sigma, m, window_points="2m"):
    """Plan geometry (readings R3/R4).

    Ntilde_d = 2 ceil(sigma N_d / 2); beta_d = pi m (2 - N_d / Ntilde_d).
    Raises ValueError on the invalid geometries DESIGN.md lists (N_d < 2,
    sigma <= 1, 2m >= Ntilde_d; 2m+2 >= Ntilde_d for the 2m+2 variant). Odd
    N_d are valid: I_N then covers n_d = -(N_d-1)/2 .. (N_d-1)/2,
    storage index i_d = n_d + floor(N_d/2) (reading R18).
    window_points: "2m" (the paper's truncated psi_hat) or
    "2m+2" (NFFT3's variant: 2m+2 samples of the continued
    window, same shape beta and correction).
    """
    if window_points not in ("2m", "2m+2"):
        raise ValueError("window_points must be '2m' or '2m+2'")
    N = tuple(int(n) for n in N)
    if sigma <= 1.0:
        raise ValueError("sigma must be > 1")
    if m < 1:
        raise ValueError("m must be >= 1")
    Ntilde = []
    for n in N:
        if n < 2:
            raise ValueError("N_d must be >= 2")
        Ntilde.append(2 * math.ceil(sigma * n / 2.0))
    npts = 2 * m if window_points == "2m" else 2 * m + 2
    for nt in Ntilde:
        if npts >= nt:
            raise ValueError("the footprint (2m or 2m+2 cells) must be < Ntilde_d")
    beta = [window.kb_beta(m, nt / n) for n, nt in zip(N, Ntilde)]
    return {"D": len(N), "N": N, "Ntilde": tuple(Ntilde), "m": int(m), "beta": beta, "points": npts}


def _logical_axes(N):
    """n_d in I_{N_d} = Z cap [-N_d/2, N_d/2) in storage order:
    -N_d/2 .. N_d/2-1 for even N_d, -(N_d-1)/2 .. (N_d-1)/2 for odd N_d."""
    return [np.arange(-(n // 2), n - n // 2, dtype=np.int64) for n in N]


def correction(geom):
    """1 / (|I_Ntilde| phi(n)) for n in I_N, shape N (Alg. 1 l.3 / Alg. 2 l.8)."""
    n_axes = _logical_axes(geom["N"])
    size = float(np.prod(geom["Ntilde"]))
    return 1.0 / (size * window.phi(n_axes, geom["Ntilde"], geom["m"], geom["beta"]))


def deconvolve_pad(fhat, geom):
    """Alg. 1 lines 1-3: g_n = f_n / (|I_Ntilde| phi(n)) on
    I_N, 0 on I_Ntilde minus I_N; stored at (n mod Ntilde)."""
    g = np.zeros(geom["Ntilde"], dtype=np.complex128)
    n_axes = _logical_axes(geom["N"])
    idx = np.ix_(*[n % nt for n, nt in zip(n_axes, geom["Ntilde"])])
    g[idx] = np.asarray(fhat, np.complex128) * correction(geom)
    return g


def crop_deconvolve(g, geom):
    """Alg. 2 lines 7-9: y_n = g_n / (|I_Ntilde| phi(n)),
    n in I_N, read from storage (n mod Ntilde), written at n + N/2."""
    n_axes = _logical_axes(geom["N"])
    idx = np.ix_(*[n % nt for n, nt in zip(n_axes, geom["Ntilde"])])
    return g[idx] * correction(geom)


def fft_forward(g):
    """Alg. 1 lines 4-6: ghat_l = sum_n g_n e^{-2 pi i n.l/Ntilde}
    (unnormalised; numpy fftn is exactly this sum on mod-Ntilde storage)."""
    return np.fft.fftn(g)


def fft_adjoint(ghat):
    """Alg. 2 lines 4-6: g_n = sum_l ghat_l e^{+2 pi i n.l/Ntilde}
    (unnormalised: numpy's ifftn divides by |I_Ntilde|, so multiply back)."""
    return np.fft.ifftn(ghat) * float(np.prod(ghat.shape))


def local_taps(k_d, Ntilde_d, m, beta_d, points=None):
    """Per-dimension footprint and window values of every node (PAPER.md:489-492,
    reading R7: the unwrapped index l enters the window argument).

    Returns (l0, W): l0 = floor(Ntilde_d k_d) - m + 1 (first footprint index,
    unwrapped) and W[ell] = psi_hat_Base((Ntilde_d k_d - (l0 + ell)) / m),
    ell = 0..2m-1. With points = 2m+2 (NFFT3 variant): l0 =
    floor(Ntilde_d k_d) - m, ell = 0..2m+1, and the continued window
    phi_hat (window.phi_hat_continued) in place of psi_hat.
    """
    points = 2 * m if points is None else points
    t = Ntilde_d * np.asarray(k_d, np.float64)
    a = np.floor(t)
    first = a - m + 1 if points == 2 * m else a - m
    l0 = first.astype(np.int64)
    W = np.empty((points, t.shape[0]), dtype=np.float64)
    for ell in range(points):
        u = (t - (first + ell)) / m
        W[ell] = window.psi_hat_base(u, beta_d) if points == 2 * m else window.phi_hat_continued(u, beta_d)
    return l0, W


def _footprints(nodes, geom):
    D, m = geom["D"], geom["m"]
    P = geom.get("points", 2 * m)
    taps = [local_taps(nodes[:, d], geom["Ntilde"][d], m, geom["beta"][d], P) for d in range(D)]
    for ell in itertools.product(range(P), repeat=D):
        w = np.ones(nodes.shape[0], dtype=np.float64)
        flat = np.zeros(nodes.shape[0], dtype=np.int64)
        for d in range(D):
            l0, W = taps[d]
            w = w * W[ell[d]]
            flat = flat * geom["Ntilde"][d] + (l0 + ell[d]) % geom["Ntilde"][d]
        yield flat, w


def resample_forward(ghat, nodes, geom):
    """Alg. 1 lines 7-9, the sum of eq. (SumOverNode)
    PAPER.md:482: f_j = sum_{l in I_{Ntilde,m}(k_j)} ghat_l psi~(k_j - l/Ntilde),
    with psi~(k - l/Ntilde) = prod_d psi_hat_Base((Ntilde_d k_d - l_d)/m).
    ghat may carry a leading batch axis (B vectors on the same nodes): the
    footprint and taps are evaluated once and applied to every vector (the
    per-vector arithmetic is unchanged); the result is then (B, M)."""
    nodes = np.asarray(nodes, np.float64).reshape(-1, geom["D"])
    ghat = np.asarray(ghat, np.complex128)
    batched = ghat.ndim == geom["D"] + 1
    grid_t = np.ascontiguousarray(ghat.reshape(ghat.shape[0] if batched else 1, -1).T)  # (cells, B)
    f_t = np.zeros((nodes.shape[0], grid_t.shape[1]), dtype=np.complex128)
    for flat, w in _footprints(nodes, geom):
        f_t += w[:, None] * grid_t[flat]
    return f_t.T.copy() if batched else f_t[:, 0].copy()


def resample_adjoint(f, nodes, geom):
    """Alg. 2 lines 1-3 in the node-outer evaluation order
    the paper prescribes: ghat_l += f_j psi~(k_j - l/Ntilde) for
    every l in I_{Ntilde,m}(k_j). f may be (B, M) (B vectors on the same nodes,
    footprints and taps shared); the result is then (B, *Ntilde)."""
    nodes = np.asarray(nodes, np.float64).reshape(-1, geom["D"])
    f = np.asarray(f, np.complex128)
    batched = f.ndim == 2
    fb = f if batched else f.reshape(1, -1)
    size = int(np.prod(geom["Ntilde"]))
    re = np.zeros((fb.shape[0], size))
    im = np.zeros((fb.shape[0], size))
    for flat, w in _footprints(nodes, geom):
        for b in range(fb.shape[0]):
            re[b] += np.bincount(flat, weights=w * fb[b].real, minlength=size)
            im[b] += np.bincount(flat, weights=w * fb[b].imag, minlength=size)
    out = (re + 1j * im).reshape((fb.shape[0],) + tuple(geom["Ntilde"]))
    return out if batched else out[0]


def forward(nodes, fhat, N, m, sigma, rows=None, window_points="2m"):
    """Direct NFFT, Alg. 1: N-grid fhat -> M node values.

    `fhat` has shape N or (B, *N); the result has shape (M,) or (B, M).
    `rows` (optional index array) evaluates only those nodes (the grid steps
    are still done in full). window_points: see geometry()."""
    geom = geometry(N, sigma, m, window_points)
    nodes = np.asarray(nodes, np.float64).reshape(-1, geom["D"])
    if rows is not None:
        nodes = nodes[np.asarray(rows)]
    fhat = np.asarray(fhat, np.complex128)
    batched = fhat.ndim == geom["D"] + 1
    fb = fhat if batched else fhat[None]
    ghat = np.stack([fft_forward(deconvolve_pad(fb[b], geom)) for b in range(fb.shape[0])])
    out = resample_forward(ghat, nodes, geom)
    return out if batched else out[0]


def adjoint(nodes, f, N, m, sigma, window_points="2m"):
    """Adjoint NFFT, Alg. 2: M node values -> N-grid y.

    `f` has shape (M,) or (B, M); the result has shape N or (B, *N).
    window_points: see geometry()."""
    geom = geometry(N, sigma, m, window_points)
    nodes = np.asarray(nodes, np.float64).reshape(-1, geom["D"])
    f = np.asarray(f, np.complex128)
    batched = f.ndim == 2
    fb = f if batched else f[None]
    ghat = resample_adjoint(fb, nodes, geom)
    out = np.stack([crop_deconvolve(fft_adjoint(ghat[b]), geom) for b in range(fb.shape[0])])
    return out if batched else out[0]
