mkdir -p gpurun_out/r01e
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01e/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01e/pytest_gpu.log
for q in 64 128 256 512; do timeout 300 python tools/stage_bench.py cfg2_1d_2e18 4 auto $q >> gpurun_out/r01e/stage_q.log 2>&1; done
timeout 300 python tools/stage_bench.py cfg2_1d_2e18 8 auto >> gpurun_out/r01e/stage_q.log 2>&1
python tools/stage_bench.py cfg2_1d_2e18 4 auto 128 > gpurun_out/r01e/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -s 20 -c 30 --csv --log-file gpurun_out/r01e/launches.csv python tools/stage_bench.py cfg2_1d_2e18 4 auto 128 > /dev/null 2>&1
