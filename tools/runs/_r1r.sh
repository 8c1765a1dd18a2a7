mkdir -p gpurun_out/r01r
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01r/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01r/pytest_gpu.log
for c in cfg2_1d_2e18 cfg3_2d_512 cfg4_3d_64 cfg5_radial_s2 cfg5_radial_s125; do
  timeout 300 python tools/stage_bench.py $c 4 auto >> gpurun_out/r01r/stage.log 2>&1
done
