"""Per-stage timing sweep (diagnostic): python tools/stage_bench.py [config] [m] [method] [tile]"""
import os, sys, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2208_00049_b200 as pkg
from paper_2208_00049_b200 import workloads


def run(config, m, method="auto", tile=None, steps=20, flush=True):
    w = workloads.make(config, seed=0, m=m)
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        nodes = torch.from_numpy(w["nodes"]).to(dev)
        fhat = torch.from_numpy(w["fhat"]).to(dev)
        f = torch.from_numpy(w["f"]).to(dev)
        p = pkg.NfftPlan(nodes, w["N"], m=m, sigma=w["sigma"], precision=w["precision"], batch=w["batch"],
                         tile=tile, stream=st.cuda_stream, method=method, timing=True, check_nodes=False)
        fo = torch.empty((w["batch"], w["M"]), dtype=p.tdtype_c, device=dev)
        yo = torch.empty((w["batch"],) + tuple(w["N"]), dtype=p.tdtype_c, device=dev)
        buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    acc = {}
    for s in range(steps + 3):
        with torch.cuda.stream(st):
            if flush:
                buf.zero_()
            p.precompute(); p.forward(fhat, out=fo); p.adjoint(f, out=yo)
        tf = p.stage_times("forward"); ta = p.stage_times("adjoint")
        if s >= 3:
            for k, v in (("pre", tf["precompute"]), ("deconv", tf["deconv"]), ("fftF", tf["fft"]), ("interp", tf["resample"]),
                         ("zero", ta["zero"]), ("spread", ta["resample"]), ("fftA", ta["fft"]), ("crop", ta["deconv"])):
                acc.setdefault(k, []).append(v * 1000)
    info = p.info()
    p.close()
    return {k: round(statistics.median(v), 1) for k, v in acc.items()}, info


if __name__ == "__main__":
    cases = []
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
        except Exception as e:
            print(json.dumps({"cfg": cfg, "m": m, "method": meth, "error": str(e)}), flush=True)
