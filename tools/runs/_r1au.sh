mkdir -p gpurun_out/r01au
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01au/pytest.log 2>&1; echo exit $? >> gpurun_out/r01au/pytest.log
for rep in 1 2; do timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu --no-sweep --no-e2e > gpurun_out/r01au/b_$rep.log 2>&1; done
