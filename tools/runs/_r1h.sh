mkdir -p gpurun_out/r01h
timeout 1200 python -m pytest tests -m gpu -x -q -k "1d or binning or config1 or full_size or execute" > gpurun_out/r01h/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01h/pytest_gpu.log
for q in 128 256; do timeout 300 python tools/stage_bench.py cfg2_1d_2e18 4 auto $q >> gpurun_out/r01h/stage_q.log 2>&1; done
python tools/stage_bench.py cfg2_1d_2e18 4 auto 128 > gpurun_out/r01h/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"1d_kernel|binsort" -s 3 -c 6 --csv --log-file gpurun_out/r01h/launches.csv python tools/stage_bench.py cfg2_1d_2e18 4 auto 128 > /dev/null 2>&1
