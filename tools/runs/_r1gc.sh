#!/bin/bash
# interp over stored taps: gpu tests + stage times with / without (NFFTB_INTERP_HORNER)
out=gpurun_out/r01gc; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
for cfg in cfg3_2d_512 cfg4_3d_64 cfg5_radial_s2; do
  STAGE_REPS=10 timeout 300 python tools/stage_bench.py $cfg 4 auto >> $out/stages.log 2>&1
  NFFTB_INTERP_HORNER=1 STAGE_REPS=10 timeout 300 python tools/stage_bench.py $cfg 4 auto >> $out/stages_horner.log 2>&1
done
