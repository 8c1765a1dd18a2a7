mkdir -p gpurun_out/r01ae
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01ae/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01ae/pytest_gpu.log
STAGE_REPS=20 timeout 300 python tools/stage_bench.py cfg2_1d_2e18 4 auto >> gpurun_out/r01ae/stage20.log 2>&1
STAGE_REPS=20 timeout 300 python tools/stage_bench.py cfg2_1d_2e18 8 auto >> gpurun_out/r01ae/stage20.log 2>&1
timeout 300 python tools/stage_bench.py cfg2_1d_2e18 4 auto >> gpurun_out/r01ae/stage.log 2>&1
