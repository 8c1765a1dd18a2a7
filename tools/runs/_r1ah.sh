mkdir -p gpurun_out/r01ah
timeout 1200 python -m pytest tests -m gpu -x -q -k "1d or config1 or cfg2 or batch" > gpurun_out/r01ah/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01ah/pytest_gpu.log
for m in 4 8; do STAGE_REPS=20 timeout 300 python tools/stage_bench.py cfg2_1d_2e18 $m auto >> gpurun_out/r01ah/stage20.log 2>&1; done
timeout 300 python tools/stage_bench.py cfg2_1d_2e18 4 auto >> gpurun_out/r01ah/stage.log 2>&1
