#!/bin/bash
# permute_f with four positions per thread: tests + 2D/3D stage times + ncu times of permute_f
out=gpurun_out/r01gk; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
for cfg in cfg3_2d_512 cfg4_3d_64; do STAGE_REPS=10 timeout 300 python tools/stage_bench.py $cfg 4 auto >> $out/stages.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:permute -c 4 --csv python tools/prof_stage.py adj_spread cfg4_3d_64:4 cfg3_2d_512:4 > $out/ncu_permute.csv 2>&1
