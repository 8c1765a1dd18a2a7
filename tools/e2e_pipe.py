import sys, os
sys.path.insert(0, os.getcwd())
import bench, torch
a = bench.parse(["--steps", "20", "--warmup", "3"])
ctx = bench.setup_dist(a)
from paper_2208_00049_b200 import workloads
for cfg in ("cfg2_1d_2e18", "cfg5_radial_s2"):
    w = workloads.make(cfg, seed=0); w["name"] = cfg
    for pipe in (2, 4, 6, 8):
        r = bench.measure_e2e(a, ctx, w, steps=24, pipe=pipe)
        print(cfg, pipe, "%.3g" % r["value"], flush=True)
