"""Run one stage of several configs a few times (target for a single ncu capture).

    python tools/prof_stage.py adj_spread[,fwd_interp] cfg4_3d_64:4 cfg3_2d_512:4 cfg5_radial_s2:4

Each config: plan + precompute, then REPS launches of the stage on the plan
stream (no graph, so ncu sees every launch).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2208_00049_b200 as pkg
from paper_2208_00049_b200 import workloads

REPS = int(os.environ.get("PROF_REPS", "2"))


def main():
    stages = sys.argv[1].split(",")
    dev = torch.device("cuda", 0)
    for spec in sys.argv[2:]:
        cfg, m = spec.split(":")
        w = workloads.make(cfg, seed=0, m=int(m))
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            nodes = torch.from_numpy(w["nodes"]).to(dev)
            fhat = torch.from_numpy(w["fhat"]).to(dev)
            f = torch.from_numpy(w["f"]).to(dev)
            p = pkg.NfftPlan(nodes, w["N"], m=int(m), sigma=w["sigma"], precision=w["precision"], batch=w["batch"],
                             stream=st.cuda_stream, check_nodes=False)
            p.run_stage("precompute")
            fo = torch.empty((w["batch"], w["M"]), dtype=p.tdtype_c, device=dev)
            for stage in stages:
                for _ in range(REPS):
                    if stage == "fwd_interp":
                        p.run_stage("fwd_deconv", fhat)
                        p.run_stage("fwd_fft")
                        p.run_stage("fwd_interp", None, fo)
                    else:
                        p.run_stage(stage, f)
        st.synchronize()
        print(spec, p.info().get("tile"), flush=True)
        p.close()


if __name__ == "__main__":
    main()
