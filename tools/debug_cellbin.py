"""Diagnostic: cell binning of the plan vs the oracle binning (tile = 1 cell)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2208_00049_b200 as pkg
from paper_2208_00049_b200 import workloads
from oracle import binning as obin

for cfg, over in [("cfg3_2d_512", dict(N=(48, 40), M=3000)), ("cfg2_1d_2e18", {})]:
    w = workloads.make(cfg, seed=1, m=4, **over)
    nodes = torch.from_numpy(w["nodes"]).cuda()
    p = pkg.NfftPlan(nodes, w["N"], m=4, sigma=w["sigma"], precision=w["precision"], batch=1).precompute()
    torch.cuda.synchronize()
    for rep in range(2):
        if rep:
            p.precompute(); torch.cuda.synchronize()
        order, cstart = p.cell_binning()
        info = p.info()
        ref_perm, ref_offs, _ = obin.bin_nodes(w["nodes"], info["Ntilde"], tuple(1 for _ in info["Ntilde"]))
        n = len(cstart) - 1
        T = 4096
        cnt_ok = np.array_equal(np.diff(cstart[:n]), np.diff(ref_offs[:n]))
        tiles = [(t, int(cstart[t * T] - ref_offs[t * T])) for t in range((n + T - 1) // T)]
        print(cfg, "rep", rep, "ncells", n, "counts-equal(excl boundaries)", cnt_ok, "end", cstart[n], ref_offs[n])
        print("  tile excl errors:", [x for x in tiles if x[1] != 0][:20], flush=True)
        # within-tile diffs
        for t in range((n + T - 1) // T):
            a, b = t * T, min(n, (t + 1) * T)
            d = (cstart[a:b] - cstart[a]) - (ref_offs[a:b] - ref_offs[a])
            if np.any(d != 0):
                print("  tile", t, "inner mismatch at", np.nonzero(d)[0][:5]); break
    p.close()
