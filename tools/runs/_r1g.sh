mkdir -p gpurun_out/r01g
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01g/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01g/pytest_gpu.log
for q in 128 256 512; do timeout 300 python tools/stage_bench.py cfg2_1d_2e18 4 auto $q >> gpurun_out/r01g/stage_q.log 2>&1; done
timeout 300 python tools/stage_bench.py cfg2_1d_2e18 8 auto >> gpurun_out/r01g/stage_q.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 10 --no-sweep --no-cpu > gpurun_out/r01g/bench.log 2>&1
python tools/stage_bench.py cfg3_2d_512 4 auto > gpurun_out/r01g/plain2d.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"interp_tiled|spread_gather|spread1d" -s 2 -c 3 \
    -o gpurun_out/r01g/full python tools/stage_bench.py cfg3_2d_512 4 auto > gpurun_out/r01g/ncu.log 2>&1
for k in interp_tiled spread_gather; do
ncu -i gpurun_out/r01g/full.ncu-rep --page source --csv -k regex:$k --print-source sass > gpurun_out/r01g/src_$k.csv 2>/dev/null
done
ncu -i gpurun_out/r01g/full.ncu-rep --page raw --csv > gpurun_out/r01g/full_raw.csv 2>/dev/null
