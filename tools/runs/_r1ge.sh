#!/bin/bash
# interp_cell staging without per-row division: gpu tests + stage times (2D, 3D, radial)
out=gpurun_out/r01ge; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
for cfg in cfg3_2d_512 cfg4_3d_64 cfg5_radial_s2; do
  STAGE_REPS=10 timeout 300 python tools/stage_bench.py $cfg 4 auto >> $out/stages.log 2>&1
done
