mkdir -p gpurun_out/r01ag
for t in 8,32 16,32 32,32 16,16 8,64 32,64; do
  STAGE_REPS=5 timeout 300 python tools/stage_bench.py cfg3_2d_512 4 auto $t >> gpurun_out/r01ag/tiles2d.log 2>&1
  STAGE_REPS=2 timeout 300 python tools/stage_bench.py cfg5_radial_s2 4 auto $t >> gpurun_out/r01ag/tilesrad.log 2>&1
done
for t in 8,8,16 4,8,16 8,8,8 4,4,32 8,16,16; do
  STAGE_REPS=2 timeout 300 python tools/stage_bench.py cfg4_3d_64 4 auto $t >> gpurun_out/r01ag/tiles3d.log 2>&1
done
