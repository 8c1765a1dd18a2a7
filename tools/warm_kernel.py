"""Diagnostic: average duration of single stages replayed back-to-back (warm L2), vs after an L2 flush."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2208_00049_b200 as pkg
from paper_2208_00049_b200 import workloads

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2_1d_2e18"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = workloads.make(cfg, seed=0, m=m)
dev = torch.device("cuda", 0)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    nodes = torch.from_numpy(w["nodes"]).to(dev)
    fhat = torch.from_numpy(w["fhat"]).to(dev)
    f = torch.from_numpy(w["f"]).to(dev)
    p = pkg.NfftPlan(nodes, w["N"], m=m, sigma=w["sigma"], precision=w["precision"], batch=w["batch"],
                     stream=st.cuda_stream, check_nodes=False)
    fo = torch.empty((w["batch"], w["M"]), dtype=p.tdtype_c, device=dev)
    yo = torch.empty((w["batch"],) + tuple(w["N"]), dtype=p.tdtype_c, device=dev)
    p.run_stage("precompute"); p.run_stage("fwd_deconv", fhat); p.run_stage("fwd_fft")
st.synchronize()
res = {}
for name, fn in [("precompute", lambda: p.run_stage("precompute")),
                 ("deconv", lambda: p.run_stage("fwd_deconv", fhat)),
                 ("fft_fwd", lambda: p.run_stage("fwd_fft")),
                 ("interp", lambda: p.run_stage("fwd_interp", None, fo)),
                 ("spread", lambda: p.run_stage("adj_spread", f)),
                 ("fft_adj", lambda: p.run_stage("adj_fft")),
                 ("crop", lambda: p.run_stage("adj_crop", None, yo))]:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(20):
            fn()
    st.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        g.replay()
        e0.record(st)
        for _ in range(5):
            g.replay()
        e1.record(st)
    st.synchronize()
    res[name] = round(e0.elapsed_time(e1) / 100 * 1000, 2)
print(json.dumps({"cfg": cfg, "m": m, "warm_us_per_launch": res}))
