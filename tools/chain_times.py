"""Diagnostic: step time of the direct chain alone, the adjoint chain alone and
both (one nfft_execute each), L2 flushed before every step, CUDA graphs."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2208_00049_b200 as pkg
from paper_2208_00049_b200 import workloads

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2_1d_2e18"
w = workloads.make(cfg, seed=0, m=4)
dev = torch.device("cuda", 0)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    nodes = torch.from_numpy(w["nodes"]).to(dev)
    p = pkg.NfftPlan(nodes, w["N"], m=4, sigma=w["sigma"], precision=w["precision"], batch=w["batch"],
                     stream=st.cuda_stream, check_nodes=False)
    p.precompute()
    fhat = torch.from_numpy(w["fhat"]).to(dev)
    f = torch.from_numpy(w["f"]).to(dev)
    fo = torch.empty((w["batch"], w["M"]), dtype=p.tdtype_c, device=dev)
    yo = torch.empty((w["batch"],) + tuple(w["N"]), dtype=p.tdtype_c, device=dev)
    buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
st.synchronize()
variants = {"fwd": lambda: p.execute(False, fhat, fo), "adj": lambda: p.execute(False, None, None, f, yo),
            "both": lambda: p.execute(False, fhat, fo, f, yo), "pre": lambda: p.execute(True),
            "pre+both": lambda: p.execute(True, fhat, fo, f, yo)}
for name, fn in variants.items():
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        fn()
    st.synchronize()
    with torch.cuda.graph(g, stream=st):
        fn()
    ts = []
    for r in range(60):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            buf.zero_()
            e0.record(st)
            g.replay()
            e1.record(st)
        st.synchronize()
        if r >= 10:
            ts.append(e0.elapsed_time(e1) * 1000)
    print(cfg, name, f"{statistics.median(ts):.1f} us", flush=True)
