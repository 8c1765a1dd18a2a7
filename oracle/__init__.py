"""CPU oracle for the NFFT hot path of arXiv:2208.00049 (NFFT.jl) — TEST INFRASTRUCTURE.

This package is the slow, plain, obviously-correct fp64 reference that the CUDA
path (`paper_2208_00049_b200`) is checked against. It is NOT part of the
product:

* only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
  `--impl reference` leg may import, call or execute anything in here;
* it shares no code, tables or constants with the CUDA path, and it imports
  nothing from `paper_2208_00049_b200` (inputs are passed in as arrays);
* every function cites the PAPER.md passage (line numbers of
  /root/reference/PAPER.md) or the DESIGN.md reading it follows.

Modules
-------
window   Kaiser–Bessel pair psi_hat_Base / phi_Base, I0, beta
nfft     Alg. 1 (direct) and Alg. 2 (adjoint) step by step, fp64
ndft     exact NDFT / adjoint NDFT with exact phase reduction
binning  block partition R_p / Gamma_p as a stable tile sort

Pins (tests/test_oracle_*.py, `-m "not gpu"`): quadrature of the window pair,
I0 against scipy, NFFT vs brute-force NDFT, error decay in m and sigma,
adjoint inner-product identity, equispaced nodes vs numpy FFT, delta / single
node special cases, hand-checked binning cases. No function is "parity
unpinned".
"""

from . import window, nfft, ndft, binning  # noqa: F401
