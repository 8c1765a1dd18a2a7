#!/bin/bash
# 2D default tile 32 x 64 (interp_cell): gpu tests + 2D / radial stage times
out=gpurun_out/r01gn; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
for cfg in cfg3_2d_512 cfg5_radial_s2 cfg5_radial_s125; do STAGE_REPS=10 timeout 300 python tools/stage_bench.py $cfg 4 auto >> $out/stages.log 2>&1; done
