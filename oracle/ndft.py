"""Exact NDFT and adjoint NDFT (TEST INFRASTRUCTURE ONLY).

    fhat_j = sum_{n in I_N} f_n e^{-2 pi i n.k_j}          (eq. NDFT)
    y_n    = sum_{j=1..J} fhat_j e^{+2 pi i n.k_j}         (eq. NDFTH)

The phase n.k is reduced modulo 1 exactly (reading R8): a naive fp64
product n*k loses up to log2(N) bits (a false 1e-11 error floor at N = 2^18).
Each coordinate is split as k = k_hi + k_lo with k_hi = K / 2^30 (K integer) so
that n*K is an exact int64 product reduced mod 2^30, and |n*k_lo| < 2^-11 is
a small, accurately rounded remainder.
"""

import numpy as np

_SHIFT = 30
_SCALE = float(2 ** _SHIFT)


def _split(k):
    k = np.asarray(k, np.float64)
    K = np.round(k * _SCALE)            # exact: power-of-two scaling, |K| < 2^29
    lo = k - K / _SCALE                 # exact (both multiples of ulp(k)), |lo| <= 2^-31
    return K.astype(np.int64), lo


def phase_frac(n, k):
    """(n * k) mod 1 in [-1/2, 1/2), accurate to ~1e-16 absolute, for integer
    n (|n| < 2^31) and fp64 k with |k| < 2^20 (broadcasting)."""
    n = np.asarray(n, np.int64)
    K, lo = _split(k)
    hi = np.mod(n * K, 2 ** _SHIFT).astype(np.float64) / _SCALE   # exact
    p = hi + n.astype(np.float64) * lo
    return p - np.round(p)


def _axes(N):
    return [np.arange(-(n // 2), n - n // 2, dtype=np.int64) for n in N]


def ndft_rows(nodes, fhat, N, rows):
    """fhat_j for the node indices `rows`, each an O(|I_N|) sum (eq. NDFT)."""
    nodes = np.asarray(nodes, np.float64).reshape(-1, len(N))
    f = np.asarray(fhat, np.complex128).reshape(-1)
    axes = _axes(N)
    grids = np.meshgrid(*axes, indexing="ij")
    out = np.empty(len(rows), dtype=np.complex128)
    for i, j in enumerate(rows):
        ph = np.zeros(grids[0].shape, dtype=np.float64)
        for d in range(len(N)):
            ph = ph + phase_frac(grids[d], nodes[j, d])
        out[i] = np.sum(f * np.exp(-2j * np.pi * ph.reshape(-1)))
    return out


def ndft(nodes, fhat, N):
    """Full NDFT (all J rows); O(J |I_N|), for tiny problems."""
    nodes = np.asarray(nodes, np.float64).reshape(-1, len(N))
    return ndft_rows(nodes, fhat, N, range(nodes.shape[0]))


def adjoint_ndft_points(nodes, f, N, points):
    """y_n for the N-grid storage multi-indices `points` (array (P, D) of
    storage indices i_d = n_d + N_d/2), each an O(J) sum (eq. NDFTH)."""
    nodes = np.asarray(nodes, np.float64).reshape(-1, len(N))
    f = np.asarray(f, np.complex128).reshape(-1)
    points = np.asarray(points, np.int64).reshape(-1, len(N))
    out = np.empty(points.shape[0], dtype=np.complex128)
    for i in range(points.shape[0]):
        ph = np.zeros(nodes.shape[0], dtype=np.float64)
        for d in range(len(N)):
            n_d = int(points[i, d]) - N[d] // 2
            ph = ph + phase_frac(n_d, nodes[:, d])
        out[i] = np.sum(f * np.exp(2j * np.pi * ph))
    return out


def adjoint_ndft(nodes, f, N):
    """Full adjoint NDFT over all of I_N; O(J |I_N|), for tiny problems."""
    idx = np.stack(np.meshgrid(*[np.arange(n) for n in N], indexing="ij"), -1).reshape(-1, len(N))
    return adjoint_ndft_points(nodes, f, N, idx).reshape(N)
