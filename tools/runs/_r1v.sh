#!/bin/bash
# wblock spread: gpu tests + stage times (2D, 3D) with and without the warp-block path
out=gpurun_out/r01v; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
for cfg in cfg3_2d_512 cfg4_3d_64; do
  STAGE_REPS=20 timeout 300 python tools/stage_bench.py $cfg 4 auto >> $out/stages.log 2>&1
  NFFTB_NO_WB=1 STAGE_REPS=20 timeout 300 python tools/stage_bench.py $cfg 4 auto >> $out/stages_nowb.log 2>&1
done
ls -la $out
