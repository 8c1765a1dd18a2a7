"""Sweep every selectable resampling variant and tile size over the BASELINE
configs (diagnostic; prints one JSON line per case with median stage µs).

    python tools/variant_sweep.py [quick]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.stage_bench import run  # noqa: E402

CASES = [
    ("cfg2_1d_2e18", 4, [(256,), (512,), (1024,), (2048,)]),
    ("cfg2_1d_2e18", 8, [(512,), (1024,)]),
    ("cfg3_2d_512", 4, [(16, 16), (32, 32), (16, 64)]),
    ("cfg3_2d_512", 8, [(32, 32)]),
    ("cfg4_3d_64", 4, [(8, 8, 8), (4, 8, 16)]),
    ("cfg5_radial_s2", 4, [(16, 16), (32, 32)]),
    ("cfg5_radial_s125", 4, [(16, 16), (32, 32)]),
]
METHODS = ["tiled", "direct", "tiled_cas", "tiled_loc", "tiled_own", "tiled_sorted"]

if __name__ == "__main__":
    for cfg, m, tiles in CASES:
        for t in tiles:
            for meth in METHODS:
                try:
                    r, info = run(cfg, m, meth, t, steps=10)
                    print(json.dumps({"cfg": cfg, "m": m, "method": meth, "tile": list(t), "us": r}), flush=True)
                except Exception as e:
                    print(json.dumps({"cfg": cfg, "m": m, "method": meth, "tile": list(t), "error": str(e)[:200]}),
                          flush=True)
