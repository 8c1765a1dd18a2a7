mkdir -p gpurun_out/r01az
timeout 900 python -m pytest tests -m gpu -x -q -k "1d or config1 or cfg2 or batch_and or shard or dense or precompute" > gpurun_out/r01az/pytest.log 2>&1; echo exit $? >> gpurun_out/r01az/pytest.log
STAGE_REPS=20 timeout 300 python tools/stage_bench.py cfg2_1d_2e18 4 auto >> gpurun_out/r01az/stage.log 2>&1
STAGE_REPS=20 timeout 300 python tools/stage_bench.py cfg2_1d_2e18 8 auto >> gpurun_out/r01az/stage.log 2>&1
python tools/chain_times.py > gpurun_out/r01az/chain.log 2>&1
