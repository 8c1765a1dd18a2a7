mkdir -p gpurun_out/r01b
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01b/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01b/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 10 --no-sweep --no-cpu > gpurun_out/r01b/bench.log 2>&1; echo "exit $?" >> gpurun_out/r01b/bench.log
for q in 256 512 1024 2048; do timeout 300 python tools/stage_bench.py cfg2_1d_2e18 4 auto $q >> gpurun_out/r01b/stage_q.log 2>&1; done
timeout 300 python tools/stage_bench.py cfg2_1d_2e18 8 auto >> gpurun_out/r01b/stage_q.log 2>&1
