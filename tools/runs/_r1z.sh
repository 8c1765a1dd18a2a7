mkdir -p gpurun_out/r01z
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01z/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01z/pytest_gpu.log
for c in cfg2_1d_2e18 cfg3_2d_512 cfg5_radial_s2; do
  timeout 300 python tools/stage_bench.py $c 4 auto >> gpurun_out/r01z/stage.log 2>&1
  STAGE_REPS=20 timeout 300 python tools/stage_bench.py $c 4 auto >> gpurun_out/r01z/stage20.log 2>&1
done
