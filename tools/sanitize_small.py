"""Small D = 2, 3 transforms through the warp-block and batch adjoints and the
cell-mode interpolation (target for compute-sanitizer memcheck / racecheck /
synccheck; prints the relative l2 errors against the oracle)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2208_00049_b200 as pkg
from oracle import nfft as onfft
from paper_2208_00049_b200 import workloads


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    cases = [("cfg3_2d_512", dict(N=(24, 40), M=600, m=3)), ("cfg4_3d_64", dict(N=(10, 8, 12), M=500, m=2)),
             ("cfg5_radial_s2", dict(N=(24, 32), M=700, m=3, batch=9))]
    for cfg, kw in cases:
        w = workloads.make(cfg, seed=5, **kw)
        nodes = torch.from_numpy(w["nodes"]).cuda()
        p = pkg.NfftPlan(nodes, w["N"], m=w["m"], sigma=w["sigma"], precision=w["precision"],
                         batch=w["batch"]).precompute()
        fo = p.forward(torch.from_numpy(w["fhat"]).cuda()).cpu().numpy()
        yo = p.adjoint(torch.from_numpy(w["f"]).cuda()).cpu().numpy()
        feats = p.features()
        p.close()
        nd = w["nodes"].astype(np.float64)
        rf = onfft.forward(nd, w["fhat"][0].astype(np.complex128), w["N"], w["m"], w["sigma"])
        ry = onfft.adjoint(nd, w["f"][0].astype(np.complex128), w["N"], w["m"], w["sigma"])
        print(cfg, sorted(feats), "fwd %.2e adj %.2e" % (rel(fo[0], rf), rel(yo[0], ry)), flush=True)


if __name__ == "__main__":
    main()
