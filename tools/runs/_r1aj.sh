mkdir -p gpurun_out/r01aj
python tools/plan_time.py > gpurun_out/r01aj/plan_time.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01aj/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01aj/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu --no-sweep > gpurun_out/r01aj/bench.log 2>&1
