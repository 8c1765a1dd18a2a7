"""Max error (relative to the window peak) of the LSQ piecewise-polynomial
window table (one polynomial per tap in zeta in [-1/2, 1/2],
Theta = 2Z equispaced samples) against the exact KB psi_hat, per m, sigma and
degree. Justifies common.cuh: poly_degree (diagnostic, numpy only)."""
import numpy as np


def psi(u, beta):
    s2 = 1 - u * u
    out = np.zeros_like(u)
    pos = s2 > 0
    s = np.sqrt(s2[pos])
    out[pos] = np.sinh(beta * s) / (np.pi * s)
    out[s2 == 0] = beta / np.pi
    return out


for sigma in (2.0, 1.25):
    for m in range(2, 9):
        beta = np.pi * m * (2 - 1 / sigma)
        peak = psi(np.array([0.0]), beta)[0]
        res = []
        for deg in (8, 10, 12, 14, 16):
            Z = deg + 1
            worst = 0
            for l in range(2 * m):
                zs = -0.5 + np.arange(2 * Z) / (2 * Z - 1)
                mu = np.linalg.lstsq(np.vander(zs, Z, increasing=True), psi((zs + 0.5 + (m - 1 - l)) / m, beta),
                                     rcond=None)[0]
                zt = np.linspace(-0.5, 0.5 - 1e-12, 4001)
                err = np.max(np.abs(np.polynomial.polynomial.polyval(zt, mu) - psi((zt + 0.5 + (m - 1 - l)) / m, beta)))
                worst = max(worst, err / peak)
            res.append(f"deg {deg}: {worst:.1e}")
        print(f"sigma {sigma} m {m}: " + ", ".join(res))
