"""Per-stage timing sweep (diagnostic; bench.py is the reference harness).

    python tools/stage_bench.py [config m method tile]

Each stage is captured in its own CUDA graph and timed with events on the
plan stream after an L2 flush; prints the median microseconds per stage.
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

# REPS > 1: every stage graph is replayed REPS times back to back between its events
# (L2-warm after the first replay; resolves the ~2 us event granularity)
REPS = int(os.environ.get("STAGE_REPS", "1"))

import paper_2208_00049_b200 as pkg
from paper_2208_00049_b200 import workloads


def run(config, m, method="auto", tile=None, steps=20, flush=True, max_subproblem=0, **over):
    w = workloads.make(config, seed=0, m=m, **over)
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        nodes = torch.from_numpy(w["nodes"]).to(dev)
        fhat = torch.from_numpy(w["fhat"]).to(dev)
        f = torch.from_numpy(w["f"]).to(dev)
        p = pkg.NfftPlan(nodes, w["N"], m=m, sigma=w["sigma"], precision=w["precision"], batch=w["batch"],
                         tile=tile, stream=st.cuda_stream, method=method, check_nodes=False,
                         max_subproblem=max_subproblem, precompute=os.environ.get("STAGE_PRECOMPUTE", "auto"))
        fo = torch.empty((w["batch"], w["M"]), dtype=p.tdtype_c, device=dev)
        yo = torch.empty((w["batch"],) + tuple(w["N"]), dtype=p.tdtype_c, device=dev)
        wmb = int(os.environ.get("FLUSH_WRITE_MB", "256"))
        rmb = int(os.environ.get("FLUSH_READ_MB", "256"))
        buf = torch.empty(max(wmb, 1) << 20, dtype=torch.uint8, device=dev)
        rbuf = torch.ones(max(rmb, 4) << 18, dtype=torch.float32, device=dev)
        sink = torch.empty((), dtype=torch.float32, device=dev)
    stages = [("pre", lambda: p.run_stage("precompute")), ("deconv", lambda: p.run_stage("fwd_deconv", fhat)),
              ("fftF", lambda: p.run_stage("fwd_fft")), ("interp", lambda: p.run_stage("fwd_interp", None, fo)),
              ("spread", lambda: p.run_stage("adj_spread", f)), ("fftA", lambda: p.run_stage("adj_fft")),
              ("crop", lambda: p.run_stage("adj_crop", None, yo))]
    with torch.cuda.stream(st):
        for _, fn in stages:
            fn()
    st.synchronize()
    graphs = []
    for name, fn in stages:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            fn()
        graphs.append((name, g))
    st.synchronize()
    acc = {}
    for s in range(steps + 3):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(graphs) + 1)]
        with torch.cuda.stream(st):
            if flush:
                if wmb > 0:
                    buf.zero_()
                if rmb > 0:
                    sink.copy_(rbuf.sum())
            for k, (_, g) in enumerate(graphs):
                ev[k].record(st)
                for _r in range(REPS):
                    g.replay()
            ev[-1].record(st)
        st.synchronize()
        if s >= 3:
            for k, (name, _) in enumerate(graphs):
                acc.setdefault(name, []).append(ev[k].elapsed_time(ev[k + 1]) * 1000 / REPS)
            acc.setdefault("STEP", []).append(ev[0].elapsed_time(ev[-1]) * 1000)
    info = p.info()
    p.close()
    return {k: round(statistics.median(v), 1) for k, v in acc.items()}, info


if __name__ == "__main__":
    cases = []
    if len(sys.argv) > 1 and sys.argv[1] == "sweep":
        for cfg, tiles in (("cfg2_1d_2e18", [(128,), (256,), (512,), (1024,), (2048,)]),
                           ("cfg3_2d_512", [(16, 16), (16, 32), (32, 32), (32, 64), (64, 64)])):
            for t in tiles:
                for S in (128, 256):
                    r, info = run(cfg, 4, "tiled", t, max_subproblem=S)
                    print(json.dumps({"cfg": cfg, "tile": t, "S": S, "us": r}), flush=True)
        sys.exit(0)
    if len(sys.argv) > 1:
        tile = tuple(int(x) for x in sys.argv[4].split(",")) if len(sys.argv) > 4 else None
        cases = [(sys.argv[1], int(sys.argv[2]), sys.argv[3] if len(sys.argv) > 3 else "auto", tile)]
    else:
        for cfg, ms in (("cfg2_1d_2e18", (4, 8)), ("cfg3_2d_512", (4, 8)), ("cfg4_3d_64", (4,)), ("cfg5_radial_s2", (4,))):
            for m in ms:
                for meth in ("tiled", "direct"):
                    cases.append((cfg, m, meth, None))
    for cfg, m, meth, tile in cases:
        try:
            r, info = run(cfg, m, meth, tile)
            print(json.dumps({"cfg": cfg, "m": m, "method": meth, "tile": info["tile"], "us": r}), flush=True)
        except Exception as e:  # keep sweeping
            print(json.dumps({"cfg": cfg, "m": m, "method": meth, "error": str(e)}), flush=True)
