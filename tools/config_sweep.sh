#!/bin/bash
# One bench line per BASELINE config (GPU box): tools/config_sweep.sh <outdir>
out=${1:-gpurun_out/sweep}
mkdir -p $out
timeout 900 python bench.py --steps 200 --warmup 10 > $out/bench_cfg2.log 2>&1
timeout 900 python bench.py --config cfg3_2d_512 --steps 50 --warmup 5 --no-cpu > $out/bench_cfg3.log 2>&1
timeout 900 python bench.py --config cfg4_3d_64 --steps 20 --warmup 3 --no-cpu --no-sweep > $out/bench_cfg4.log 2>&1
timeout 900 python bench.py --config cfg5_radial_s2 --steps 20 --warmup 3 --no-cpu --no-sweep > $out/bench_cfg5_s2.log 2>&1
timeout 900 python bench.py --config cfg5_radial_s125 --steps 20 --warmup 3 --no-cpu --no-sweep > $out/bench_cfg5_s125.log 2>&1
