"""Diagnostic: run the same forward/adjoint several times (fresh plans and one plan) and compare bitwise."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2208_00049_b200 as pkg
from paper_2208_00049_b200 import workloads

w = workloads.make("cfg3_2d_512", seed=6, N=(32, 48), M=1000, m=4)
nodes = torch.from_numpy(w["nodes"]).cuda(); fhat = torch.from_numpy(w["fhat"]).cuda()
outs = []
for rep in range(3):
    p = pkg.NfftPlan(nodes, w["N"], m=4).precompute()
    outs.append((p.forward(fhat).cpu().numpy(), p.forward(fhat).cpu().numpy()))
    g = torch.empty(1, 64 * 96, dtype=torch.complex128, device="cuda")
    p.close()
for a, b in outs:
    print("same plan twice:", np.array_equal(a, b), " vs first plan:", np.array_equal(a, outs[0][0]),
          np.max(np.abs(a - outs[0][0])))
ph = pkg.NfftPlan(w["nodes"], w["N"], m=4).precompute()
hf = ph.forward(w["fhat"])
print("host path vs device:", np.array_equal(hf, outs[0][0]), np.max(np.abs(hf - outs[0][0])))
# stage-level: compare deconv output and fft output between plans
