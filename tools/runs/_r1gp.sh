#!/bin/bash
# interp tile sweep, radial sigma = 1.25 (320^2) and sigma = 2
out=gpurun_out/r01gp; mkdir -p $out
for t in 32,32 32,40 16,64 32,64 16,32 64,32 40,40; do
  STAGE_REPS=5 timeout 300 python tools/stage_bench.py cfg5_radial_s125 4 auto $t >> $out/stages.log 2>&1
done
for t in 32,64 32,128 64,64 16,64; do
  STAGE_REPS=5 timeout 300 python tools/stage_bench.py cfg5_radial_s2 4 auto $t >> $out/stages.log 2>&1
done
for t in 32,64 32,128 64,64 16,128; do
  STAGE_REPS=10 timeout 300 python tools/stage_bench.py cfg3_2d_512 4 auto $t >> $out/stages.log 2>&1
done
