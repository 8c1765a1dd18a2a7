mkdir -p gpurun_out/r01l
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01l/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r01l/pytest_gpu.log
for q in 256 512 1024; do timeout 300 python tools/stage_bench.py cfg2_1d_2e18 4 auto $q >> gpurun_out/r01l/stage_q.log 2>&1; done
timeout 300 python tools/stage_bench.py cfg2_1d_2e18 8 auto >> gpurun_out/r01l/stage_q.log 2>&1
python tools/stage_bench.py cfg2_1d_2e18 4 auto > gpurun_out/r01l/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"nfftb" -s 6 -c 14 --csv --log-file gpurun_out/r01l/launches.csv python tools/stage_bench.py cfg2_1d_2e18 4 auto > /dev/null 2>&1
