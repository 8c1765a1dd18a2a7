mkdir -p gpurun_out/r01ad
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01ad/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01ad/pytest_gpu.log
for c in cfg2_1d_2e18 cfg3_2d_512 cfg4_3d_64 cfg5_radial_s2; do STAGE_REPS=20 timeout 300 python tools/stage_bench.py $c 4 auto >> gpurun_out/r01ad/stage20.log 2>&1; done
python tools/stage_bench.py cfg3_2d_512 4 auto > gpurun_out/r01ad/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"spread_cell" -s 4 -c 1 \
    -o gpurun_out/r01ad/full python tools/stage_bench.py cfg3_2d_512 4 auto > gpurun_out/r01ad/ncu.log 2>&1
ncu -i gpurun_out/r01ad/full.ncu-rep --page details > gpurun_out/r01ad/details.txt 2>/dev/null
ncu -i gpurun_out/r01ad/full.ncu-rep --page source --csv --print-source sass > gpurun_out/r01ad/src.csv 2>/dev/null
