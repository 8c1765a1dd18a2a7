mkdir -p gpurun_out/r01i
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01i/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01i/pytest_gpu.log
for q in 128 256 512; do timeout 300 python tools/stage_bench.py cfg2_1d_2e18 4 auto $q >> gpurun_out/r01i/stage_q.log 2>&1; done
python tools/stage_bench.py cfg2_1d_2e18 4 auto 128 > gpurun_out/r01i/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none -k regex:"1d_kernel|binsort" -s 3 -c 6 --csv --log-file gpurun_out/r01i/launches.csv python tools/stage_bench.py cfg2_1d_2e18 4 auto 128 > /dev/null 2>&1
