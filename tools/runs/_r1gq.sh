#!/bin/bash
# batched 2D default tile 16 x (32 | 64): gpu tests + radial stage times
out=gpurun_out/r01gq; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
for cfg in cfg5_radial_s2 cfg5_radial_s125 cfg3_2d_512; do STAGE_REPS=5 timeout 300 python tools/stage_bench.py $cfg 4 auto >> $out/stages.log 2>&1; done
