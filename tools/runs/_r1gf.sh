#!/bin/bash
# batched interp_cell (regions of 8 / 4 vectors per CTA): gpu tests + radial stage times with / without
out=gpurun_out/r01gf; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
for cfg in cfg5_radial_s2 cfg5_radial_s125; do
  STAGE_REPS=5 timeout 300 python tools/stage_bench.py $cfg 4 auto >> $out/stages.log 2>&1
  NFFTB_NO_INTERP_VB=1 STAGE_REPS=5 timeout 300 python tools/stage_bench.py $cfg 4 auto >> $out/stages_novb.log 2>&1
done
