mkdir -p gpurun_out/r01aw
timeout 900 python -m pytest tests -m gpu -x -q -k "batch or radial" > gpurun_out/r01aw/pytest.log 2>&1; echo exit $? >> gpurun_out/r01aw/pytest.log
for c in cfg5_radial_s2 cfg5_radial_s125; do STAGE_REPS=3 timeout 300 python tools/stage_bench.py $c 4 auto >> gpurun_out/r01aw/stage.log 2>&1; done
