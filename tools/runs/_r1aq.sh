mkdir -p gpurun_out/r01aq
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01aq/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01aq/pytest_gpu.log
for c in cfg3_2d_512 cfg4_3d_64 cfg5_radial_s2; do STAGE_REPS=3 timeout 300 python tools/stage_bench.py $c 4 auto >> gpurun_out/r01aq/stage.log 2>&1; done
STAGE_REPS=3 timeout 300 python tools/stage_bench.py cfg3_2d_512 8 auto >> gpurun_out/r01aq/stage.log 2>&1
