mkdir -p gpurun_out/r01af
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01af/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01af/pytest_gpu.log
for pc in tensor polynomial; do for m in 4 8; do
STAGE_PRECOMPUTE=$pc STAGE_REPS=20 timeout 300 python tools/stage_bench.py cfg2_1d_2e18 $m auto >> gpurun_out/r01af/stage20.log 2>&1
done; done
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu --no-sweep --no-e2e > gpurun_out/r01af/bench.log 2>&1
