mkdir -p gpurun_out/r01n
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01n/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01n/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu > gpurun_out/r01n/bench.log 2>&1
