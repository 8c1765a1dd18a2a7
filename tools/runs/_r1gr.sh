#!/bin/bash
# large tiles keep cell mode: full gpu tests + radial stage time at tile 32 x 128
out=gpurun_out/r01gr; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
STAGE_REPS=5 timeout 300 python tools/stage_bench.py cfg5_radial_s2 4 auto 32,128 >> $out/stages.log 2>&1
STAGE_REPS=10 timeout 300 python tools/stage_bench.py cfg3_2d_512 4 auto 64,64 >> $out/stages.log 2>&1
