mkdir -p gpurun_out/r01av
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01av/pytest.log 2>&1; echo exit $? >> gpurun_out/r01av/pytest.log
python tools/debug_cellbin.py > gpurun_out/r01av/cb.log 2>&1
for c in cfg2_1d_2e18 cfg3_2d_512; do STAGE_REPS=20 timeout 300 python tools/stage_bench.py $c 4 auto >> gpurun_out/r01av/stage.log 2>&1; done
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu --no-sweep --no-e2e > gpurun_out/r01av/b.log 2>&1
