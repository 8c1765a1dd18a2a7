"""Host-side pieces of bench.py (no GPU): the algorithmic byte / flop counts
behind roofline.achieved, the derived ALU peak,
and the reference arm (the oracle timed on the host) end to end."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2208_00049_b200 import workloads  # noqa: E402


def test_algorithmic_bytes_and_flops_config2():
    w = workloads.make("cfg2_1d_2e18", seed=0)
    a = bench.algorithmic(w)
    M, nt = 2 ** 18, 2 ** 19
    # grid once (16 B per C128 cell), values once, one fp64 coordinate per node
    assert a["resample_bytes"] == 16 * nt + 16 * M + 8 * M == 14680064
    # 2 flop per FMA: complex value x 2m taps (2 FMAs each) + the degree-2m window evaluation
    assert a["resample_flops"] == 2 * M * (2 * 8 + 8 * 8)
    assert a["deconv_bytes"] == a["crop_bytes"] == 2 * 16 * M
    assert a["grid_cells"] == nt


def test_algorithmic_counts_3d_and_batch():
    w = workloads.make("cfg4_3d_64", seed=0)
    a = bench.algorithmic(w)
    M = 262144
    assert a["resample_bytes"] == 16 * 128 ** 3 + 16 * M + 8 * 3 * M
    assert a["resample_flops"] == 2 * M * (2 * (8 + 64 + 512) + 8 * 3 * 8)
    w = workloads.make("cfg5_radial_s125", seed=0)
    a = bench.algorithmic(w)
    M, B = 205824, 32
    assert a["grid_cells"] == 320 * 320
    assert a["resample_bytes"] == B * 8 * 320 * 320 + B * 8 * M + 4 * 2 * M


def test_alu_peaks_are_the_measured_ones():
    hbm, src, fp = bench.peaks()
    assert hbm > 1000 and src
    # tools/micro/fma_peak.cu on the B200 (profiles/r02/fma_peak.jsonl): close to the unit-count bound
    # 148 SM x 64 FP64 / 128 FP32 FMA lanes x 2 x 1965 MHz = 37.2 / 74.4 TFLOP/s
    assert 30 < fp["fp64"] <= 37.3 and 60 < fp["fp32"] <= 74.5 and "measured" in fp["source"]


def test_reference_arm_prints_one_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config",
                        "cfg1_1d_256", "--steps", "2", "--warmup", "1"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["cpu"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["higher_is_better"] is True and d["unit"] == bench.UNIT
