mkdir -p gpurun_out/r01ai
for c in cfg3_2d_512 cfg4_3d_64 cfg5_radial_s2; do
for meth in tiled_cas tiled_loc tiled_own tiled_sorted tiled_v1 direct; do
  STAGE_REPS=2 timeout 200 python tools/stage_bench.py $c 4 $meth >> gpurun_out/r01ai/meth.log 2>&1
done; done
