mkdir -p gpurun_out/r01al
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01al/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01al/pytest_gpu.log
for c in cfg5_radial_s2 cfg5_radial_s125; do STAGE_REPS=3 timeout 300 python tools/stage_bench.py $c 4 auto >> gpurun_out/r01al/stage.log 2>&1; done
