#!/bin/bash
# transpose with preloaded destinations: batch tests + radial stage times
out=gpurun_out/r01gj; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q -k "batch or radial or seam or window_2m" > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
STAGE_REPS=10 timeout 300 python tools/stage_bench.py cfg5_radial_s2 4 auto >> $out/stages.log 2>&1
timeout 600 python tools/prof_stage.py adj_spread cfg5_radial_s2:4 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:transpose -c 2 --csv python tools/prof_stage.py adj_spread cfg5_radial_s2:4 > $out/ncu_transpose.csv 2>&1
