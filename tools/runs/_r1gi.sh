#!/bin/bash
# flattened deconv / crop: gpu tests + stage times of all configs
out=gpurun_out/r01gi; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
for cfg in cfg2_1d_2e18 cfg3_2d_512 cfg4_3d_64 cfg5_radial_s2; do
  STAGE_REPS=10 timeout 300 python tools/stage_bench.py $cfg 4 auto >> $out/stages.log 2>&1
done
timeout 600 python bench.py --steps 200 --warmup 10 --no-sweep --no-cpu > $out/bench.log 2>&1
